// slab.cu -- z-slab domain decomposition of ONE design's solve (config C5).
//
// the torus is split into G slabs of whole z-planes; slab
// s owns the active nodes of planes [z0, z1) and keeps one ghost plane on
// each side (z0-1 and z1, periodic).  Field and mask are computed in full by
// every rank (they cost ~0.5 ms at 256^3, less than the setup exchange they
// would need), so the decomposition applies to the solver, where the time
// goes.  Per PCG iteration:
//   update (owned nodes)        -> 12 partial sums  -> cross-slab SUM -> scalars
//   ghost exchange of z (2 planes of 18 components, one per neighbour)
//   apply  (owned nodes, gathers owned + ghost z) -> 6 partial sums -> SUM
// and once at the end an x ghost exchange + the C^H partial sums.
//
// Two transports share every kernel and index map:
//   * emulated: G slabs in one context on one device; the exchange is a
//     pack/unpack device copy and the cross-slab sum is a fixed-order finalize
//     kernel.  Used by the parity tests (no second GPU needed, and no ranks
//     waiting on each other on one device).
//   * NCCL: one slab per rank; ncclSend/ncclRecv of packed ghost planes
//     (periodic ring over NVLink/NVSwitch) and ncclAllReduce of the partial
//     sums.  libnccl is dlopen'ed on first use so the single-GPU library
//     never depends on it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <functional>
#include <memory>
#include <type_traits>
#include <string>
#include <vector>

#include "context.h"
#include "gmg_host.h"

namespace shl {
namespace host {

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void* handle = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // prefer an already-loaded NCCL (torch's), then the system one
    a.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!a.handle) a.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.handle) return a;
    auto sym = [&](const char* n) { return dlsym(a.handle, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.handle || !api.AllReduce || !api.Send)
    throw ShlError(SHL_CUDA, "libnccl.so.2 could not be loaded for the z-slab transport");
  return api;
}

#define NK(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      throw ShlError(SHL_CUDA, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct NcclComm {
  ncclComm_t comm = nullptr;
  unsigned char id[NCCL_UNIQUE_ID_BYTES] = {};
  int rank = -1, nranks = 0;
  ~NcclComm() {
    if (comm) nccl().CommDestroy(comm);
  }
};

// ---------------------------------------------------------------- transports
// What a rank's slab solve needs from the other ranks: an in-place sum of a
// few device values (PCG scalars, C^H, the level-1 multigrid right-hand side)
// and the periodic-ring ghost-plane exchange.  Two backends:
//   NcclTransport -- ncclAllReduce / ncclSend+Recv on the stream (NVLink)
//   HostTransport -- stream sync, D2H into pinned buffers, the caller's
//                    callbacks (shl_slab_transport: e.g. torch.distributed
//                    gloo over TCP), H2D.  No kernel ever waits for another
//                    rank, so ranks may even share one GPU (tests).
struct SlabTransport {
  int rank = 0, nranks = 1;
  virtual ~SlabTransport() = default;
  virtual void allreduce(void* dev, size_t n, bool f64, cudaStream_t s) = 0;
  // send send_hi to rank+1 and send_lo to rank-1; receive recv_lo from rank-1
  // and recv_hi from rank+1 (counts in values).  `during` enqueues work on s
  // that needs none of the received planes (the interior apply): it is issued
  // once the sends are in flight, so it overlaps the transfer; the received
  // planes are ready on s when exchange returns.
  virtual void exchange(const void* send_hi, size_t n_send_hi, const void* send_lo, size_t n_send_lo,
                        void* recv_lo, size_t n_recv_lo, void* recv_hi, size_t n_recv_hi, bool f64,
                        cudaStream_t s, const std::function<void()>& during) = 0;
  // true when exchange() and allreduce() only enqueue device work (capturable
  // into a CUDA graph)
  virtual bool capturable() const { return false; }
};

// A side stream for the transfers and the two events that fork it from / join
// it to the solver's stream.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  SideStream() {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  }
  ~SideStream() {
    if (join) cudaEventDestroy(join);
    if (fork) cudaEventDestroy(fork);
    if (s) cudaStreamDestroy(s);
  }
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
};

struct NcclTransport : SlabTransport {
  NcclComm* comm;
  explicit NcclTransport(NcclComm* c) : comm(c) {
    rank = c->rank;
    nranks = c->nranks;
  }
  void allreduce(void* dev, size_t n, bool f64, cudaStream_t s) override {
    NK(nccl().AllReduce(dev, dev, n, f64 ? ncclFloat64 : ncclFloat32, ncclSum, comm->comm, s));
  }
  // the ring send/recv runs on a side stream forked after the packs, the
  // interior work on s beside it, and s joins the side stream before the unpack
  void exchange(const void* send_hi, size_t n_send_hi, const void* send_lo, size_t n_send_lo, void* recv_lo,
                size_t n_recv_lo, void* recv_hi, size_t n_recv_hi, bool f64, cudaStream_t s,
                const std::function<void()>& during) override {
    const ncclDataType_t dt = f64 ? ncclFloat64 : ncclFloat32;
    const int lo = (rank - 1 + nranks) % nranks, hi = (rank + 1) % nranks;
    CK(cudaEventRecord(side.fork, s));
    CK(cudaStreamWaitEvent(side.s, side.fork, 0));
    NK(nccl().GroupStart());
    NK(nccl().Send(send_hi, n_send_hi, dt, hi, comm->comm, side.s));
    NK(nccl().Send(send_lo, n_send_lo, dt, lo, comm->comm, side.s));
    NK(nccl().Recv(recv_lo, n_recv_lo, dt, lo, comm->comm, side.s));
    NK(nccl().Recv(recv_hi, n_recv_hi, dt, hi, comm->comm, side.s));
    NK(nccl().GroupEnd());
    if (during) during();
    CK(cudaEventRecord(side.join, side.s));
    CK(cudaStreamWaitEvent(s, side.join, 0));
  }
  bool capturable() const override { return true; }
  SideStream side;
};

struct HostTransport : SlabTransport {
  shl_slab_transport cb;
  unsigned char* host = nullptr;  // pinned staging
  size_t cap = 0;
  HostTransport(const shl_slab_transport& t, int r, int n) : cb(t) {
    rank = r;
    nranks = n;
  }
  ~HostTransport() override {
    if (host) cudaFreeHost(host);
  }
  unsigned char* staging(size_t bytes) {
    if (bytes > cap) {
      if (host) cudaFreeHost(host);
      host = nullptr;
      cap = bytes + bytes / 4;
      CK(cudaMallocHost(&host, cap));
    }
    return host;
  }
  void allreduce(void* dev, size_t n, bool f64, cudaStream_t s) override {
    const size_t bytes = n * (f64 ? 8 : 4);
    unsigned char* h = staging(bytes);
    CK(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (cb.allreduce_sum(cb.user, h, n, f64 ? 1 : 0) != 0)
      throw ShlError(SHL_IO, "z-slab transport: allreduce_sum callback failed");
    CK(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, s));
  }
  // D2H of the packed planes on s, then the interior work is enqueued on s and
  // the host waits for the D2H only (not for the interior work); the host
  // round trip and the H2D (side stream) overlap the interior work, and s
  // joins the side stream before the unpack
  void exchange(const void* send_hi, size_t n_send_hi, const void* send_lo, size_t n_send_lo, void* recv_lo,
                size_t n_recv_lo, void* recv_hi, size_t n_recv_hi, bool f64, cudaStream_t s,
                const std::function<void()>& during) override {
    const size_t w = f64 ? 8 : 4;
    unsigned char* h = staging(w * (n_send_hi + n_send_lo + n_recv_lo + n_recv_hi));
    unsigned char *hs_hi = h, *hs_lo = hs_hi + w * n_send_hi, *hr_lo = hs_lo + w * n_send_lo,
                  *hr_hi = hr_lo + w * n_recv_lo;
    if (n_send_hi) CK(cudaMemcpyAsync(hs_hi, send_hi, w * n_send_hi, cudaMemcpyDeviceToHost, s));
    if (n_send_lo) CK(cudaMemcpyAsync(hs_lo, send_lo, w * n_send_lo, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(side.fork, s));
    if (during) during();
    CK(cudaEventSynchronize(side.fork));
    if (cb.ring_exchange(cb.user, hs_hi, n_send_hi, hs_lo, n_send_lo, hr_lo, n_recv_lo, hr_hi, n_recv_hi,
                         f64 ? 1 : 0) != 0)
      throw ShlError(SHL_IO, "z-slab transport: ring_exchange callback failed");
    CK(cudaStreamWaitEvent(side.s, side.fork, 0));
    if (n_recv_lo) CK(cudaMemcpyAsync(recv_lo, hr_lo, w * n_recv_lo, cudaMemcpyHostToDevice, side.s));
    if (n_recv_hi) CK(cudaMemcpyAsync(recv_hi, hr_hi, w * n_recv_hi, cudaMemcpyHostToDevice, side.s));
    CK(cudaEventRecord(side.join, side.s));
    CK(cudaStreamWaitEvent(s, side.join, 0));
    // (the pinned staging is reused by the next exchange / allreduce only after
    // a host wait on s or side.s, so the H2D has finished reading it)
    CK(cudaStreamSynchronize(side.s));
  }
  SideStream side;
};

// ---------------------------------------------------------------- slab plan
struct SlabPlan {
  int z0 = 0, z1 = 0;       // owned planes [z0, z1)
  int zbase = 0, nzl = 0;   // node-map planes: zbase = z0-1 (mod r), nzl = z1-z0+2
  int n_owned = 0, n_glo = 0, n_ghi = 0, n_local = 0;
  int cnt_first = 0, cnt_last = 0;  // owned nodes on planes z0 and z1-1
  int e_lo = 0, e_hi = 0;           // owned elements: range of the global element list
  int noff_z0 = 0;                  // global node id of the first owned node
};

// A slab's share of multigrid level 1 (levels >= 2 stay replicated).  Level-1
// ids are grid-ordered, so the coarse planes [cz0, cz1) a slab owns -- the
// planes cz with z0 <= 2 cz < z1 -- are the id range [c0, c1); the ghost planes
// cz0-1 and cz1 (periodic) are the neighbours' boundary planes, the same ids in
// every slab's full-length level-1 vectors.
struct Level1Plan {
  int c0 = 0, c1 = 0;          // owned ids
  int planes = 0;              // owned planes cz1 - cz0
  int first_n = 0, last0 = 0;  // owned plane cz0: [c0, c0 + first_n); plane cz1-1: [last0, c1)
  int glo0 = 0, glo_n = 0;     // ghost plane cz0-1
  int ghi0 = 0, ghi_n = 0;     // ghost plane cz1
};

struct Slab {
  SlabPlan P;
  DevBuf map, list, vec, partials;
  size_t ld = 0;
  Level1Plan P1;
  DevBuf v1;  // level-1 b, x (two), residual: 4 full-length vectors
};

namespace {

__global__ void plane_count_kernel(const int* __restrict__ flag, int r, int* __restrict__ out) {
  const int z = blockIdx.x;
  const size_t rr = static_cast<size_t>(r) * r;
  int s = 0;
  for (size_t t = threadIdx.x; t < rr; t += blockDim.x) s += flag[z * rr + t];
  s = __reduce_add_sync(0xffffffffu, s);
  __shared__ int w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int q = 0; q < (blockDim.x + 31) / 32; ++q) t += w[q];
    out[z] = t;
  }
}

// local node map over planes zbase .. zbase+nzl-1 and local -> grid id list
__global__ void slab_map_kernel(const int* __restrict__ node_flag, const int* __restrict__ goff,
                                int r, SlabPlan P, const int* __restrict__ plane_off,
                                int* __restrict__ map, int* __restrict__ list) {
  const size_t rr = static_cast<size_t>(r) * r;
  const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (t >= rr * P.nzl) return;
  const int lp = static_cast<int>(t / rr);
  const int gz = (P.zbase + lp) % r;
  const size_t g = gz * rr + t % rr;
  int id = -1;
  if (node_flag[g]) {
    const int pid = goff[g] - plane_off[gz];  // index inside its plane
    if (lp == 0)
      id = P.n_owned + pid;
    else if (lp == P.nzl - 1)
      id = P.n_owned + P.n_glo + pid;
    else
      id = goff[g] - P.noff_z0;
    list[id] = static_cast<int>(g);
  }
  map[t] = id;
}

// totals[6 s + q] = the slab's three apply ranges (low boundary plane,
// interior, high boundary plane) summed in that fixed order
__global__ void sum_ranges_kernel(const double* __restrict__ tr, double* __restrict__ totals, int nloc) {
  const int t = threadIdx.x;
  if (t >= 6 * nloc) return;
  const int s = t / 6, q = t % 6;
  totals[t] = (tr[(3 * s + 0) * 6 + q] + tr[(3 * s + 1) * 6 + q]) + tr[(3 * s + 2) * 6 + q];
}

}  // namespace

// Build the G slab plans + device maps from the resident global mesh.
void build_slabs(shl_ctx* c, int G, int first, int count, std::vector<Slab>& slabs) {
  const int r = c->r;
  if (G < 2 || G > r / 2) throw ShlError(SHL_VALIDATION, "z-slab count must lie in [2, r/2]");
  DevBuf counts;
  counts.ensure(sizeof(int) * (3 * r + 1));
  int* ncnt = counts.as<int>();
  int* ecnt = ncnt + r;
  int* noff_dev = ecnt + r;
  plane_count_kernel<<<r, 256, 0, c->stream>>>(c->node_flag.as<int>(), r, ncnt);
  plane_count_kernel<<<r, 256, 0, c->stream>>>(c->elem_flag.as<int>(), r, ecnt);
  CK(cudaGetLastError());
  std::vector<int> h(2 * r);
  CK(cudaMemcpyAsync(h.data(), ncnt, sizeof(int) * 2 * r, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  std::vector<int> noff(r + 1, 0), eoff(r + 1, 0);
  for (int z = 0; z < r; ++z) {
    noff[z + 1] = noff[z] + h[z];
    eoff[z + 1] = eoff[z] + h[r + z];
  }
  CK(cudaMemcpyAsync(noff_dev, noff.data(), sizeof(int) * r, cudaMemcpyHostToDevice, c->stream));
  slabs.clear();
  slabs.resize(count);
  for (int q = 0; q < count; ++q) {
    const int s = first + q;
    SlabPlan& P = slabs[q].P;
    P.z0 = static_cast<int>(static_cast<long long>(s) * r / G);
    P.z1 = static_cast<int>(static_cast<long long>(s + 1) * r / G);
    P.zbase = (P.z0 - 1 + r) % r;
    P.nzl = P.z1 - P.z0 + 2;
    P.n_owned = noff[P.z1] - noff[P.z0];
    P.n_glo = h[(P.z0 - 1 + r) % r];
    P.n_ghi = h[P.z1 % r];
    P.n_local = P.n_owned + P.n_glo + P.n_ghi;
    P.cnt_first = h[P.z0];
    P.cnt_last = h[P.z1 - 1];
    P.e_lo = eoff[P.z0];
    P.e_hi = eoff[P.z1];
    P.noff_z0 = noff[P.z0];
    Slab& S = slabs[q];
    const size_t cells = static_cast<size_t>(r) * r * P.nzl;
    S.map.ensure(cells * sizeof(int));
    S.list.ensure((static_cast<size_t>(P.n_local) + 1) * sizeof(int));
    slab_map_kernel<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, c->stream>>>(
        c->node_flag.as<int>(), c->off.as<int>(), r, P, noff_dev, S.map.as<int>(), S.list.as<int>());
    CK(cudaGetLastError());
  }
  c->sync();  // `counts` dies here
}

// level-1 plane start ids: out[cz] = off[cz * rc^2] (grid-order exclusive scan)
__global__ void plane_start_kernel(const int* __restrict__ off, int rc, int* __restrict__ out) {
  const int cz = blockIdx.x * blockDim.x + threadIdx.x;
  if (cz < rc) out[cz] = off[static_cast<size_t>(cz) * rc * rc];
}

// ---------------------------------------------------------------- solve
// TX: x, r; TV: p, q and the operator; TZ: z, Dinv and the V-cycle (as in the
// single-device solve).  use_gmg: multigrid-preconditioned, with level 0
// distributed over the slabs (ghost exchange before every level-0 sweep, the
// restriction of the owned fine nodes summed across slabs) and the coarse
// levels 1..L replicated on every process (built from the full mesh each
// process holds; their vectors are small next to level 0).
template <typename TX, typename TV, typename TZ>
void run_solve_slabs(shl_ctx* c, const double* K0, const shl_solve_options& opt, double* C_out,
                     shl_stats* st, int prec, int G, SlabTransport* comm, bool use_gmg) {
  const int r = c->r;
  if (!c->node0_active)
    throw ShlError(SHL_SOLVER, "mesh has no corner node group: cannot prescribe the strain gauge");
  const bool dist = comm != nullptr;
  const int first = dist ? comm->rank : 0;
  const int nloc = dist ? 1 : G;  // slabs driven by this process
  std::vector<Slab> slabs;
  build_slabs(c, G, first, nloc, slabs);

  int max_plane = 0;
  for (auto& S : slabs) {
    const SlabPlan& P = S.P;
    S.ld = round_up(P.n_local + 1, 32);
    const size_t nX = 18 * S.ld;
    // x, r (TX) | p, q (TV) | z, Dinv (TZ) | multigrid level-0 work: xa, xb, res (TZ)
    S.vec.ensure(2 * nX * sizeof(TX) + 2 * nX * sizeof(TV) + (nX + 6 * S.ld + (use_gmg ? 3 * nX : 0)) * sizeof(TZ));
    // per-block partials (<= 2400 blocks x 21) and per-32-node-tile partials of the apply
    S.partials.ensure(sizeof(double) * std::max<size_t>(21 * 2400, static_cast<size_t>((P.n_owned + 31) / 32) * 6));
    max_plane = std::max({max_plane, P.n_glo, P.n_ghi, P.cnt_first, P.cnt_last});
  }
  DevBuf tot, xfer;
  tot.ensure(sizeof(double) * (21 + 18) * nloc);  // totals + the apply's per-range sums
  xfer.ensure(4 * 18 * static_cast<size_t>(std::max(max_plane, 1)) * sizeof(double));
  c->state.ensure(sizeof(PcgState));
  c->cout.ensure(36 * sizeof(double));

  auto X = [&](Slab& S) { return S.vec.as<TX>(); };
  auto R = [&](Slab& S) { return S.vec.as<TX>() + 18 * S.ld; };
  auto Pv = [&](Slab& S) { return reinterpret_cast<TV*>(S.vec.as<TX>() + 36 * S.ld); };
  auto Q = [&](Slab& S) { return Pv(S) + 18 * S.ld; };
  auto Z = [&](Slab& S) { return reinterpret_cast<TZ*>(Pv(S) + 36 * S.ld); };
  auto D = [&](Slab& S) { return Z(S) + 18 * S.ld; };
  auto XA = [&](Slab& S) { return D(S) + 6 * S.ld; };
  auto XB = [&](Slab& S) { return XA(S) + 18 * S.ld; };
  auto RES = [&](Slab& S) { return XB(S) + 18 * S.ld; };

  double T[144], W[144];
  element_loads(K0, r, T, W);
  // ridges as in the single-device solve (shl_api.cu run_solve)
  const double diag_mean = c->n_nodes > 0 ? std::fabs(K0[0]) * 8.0 * c->beta_sum / double(c->n_nodes) : 0.0;
  const double ridge_op = diag_mean * (sizeof(TV) == 8 ? 1e-11 : 1e-8);
  const double ridge = diag_mean * (sizeof(TZ) == 8 ? 1e-11 : 1e-8);
  CK(cudaEventRecord(c->ev[3], c->stream));
  ElementConstLease const_lease(K0, W, T, r, c->stream);
  for (auto& S : slabs) {
    CK(cudaMemsetAsync(S.vec.p, 0, S.vec.cap, c->stream));
    launch_setup<TX, TZ>(S.list.as<int>(), S.P.n_owned, static_cast<int>(S.ld), r, c->beta64.as<double>(),
                         ridge, R(S), D(S), c->stream);
  }
  // replicated coarse hierarchy (levels 1..L) and its V-cycle driver
  Vcycle<TX, TZ, TZ> vc{c, gmg_params()};
  vc.s = c->stream;
  if (vc.gp.nu <= 0) vc.gp.nu = sizeof(TV) == 8 ? 1 : 2;
  const TZ* beta_z = sizeof(TZ) == 8 ? reinterpret_cast<const TZ*>(c->beta64.p)
                                     : reinterpret_cast<const TZ*>(c->beta32.p);
  if (use_gmg) {
    vc.L = gmg_setup<TZ>(c, vc.gp, static_cast<TZ>(ridge));
    if (vc.L == 0) throw ShlError(SHL_VALIDATION, "multigrid needs r divisible by 2 with r/2 >= 8");
    vc.view.push_back({c->node_list.as<int>(), c->node_map.as<int>(), beta_z, nullptr, nullptr, r, c->n_nodes,
                       c->n_nodes, static_cast<TZ>(ridge)});  // level 0 placeholder (slab views below)
    vc.b.push_back(nullptr);
    vc.xa.push_back(nullptr);
    vc.xb.push_back(nullptr);
    vc.res.push_back(nullptr);
    for (int l = 0; l < vc.L; ++l) {
      auto& Lv = c->gmg[l];
      vc.view.push_back({Lv.list.as<int>(), Lv.map.as<int>(), nullptr, Lv.stencil.as<TZ>(), Lv.dinv.as<TZ>(),
                         Lv.r, Lv.n, Lv.n, TZ(0)});
      vc.view.back().bricks = Lv.brick_view();
      TZ* v = Lv.vec.as<TZ>();
      const size_t s18 = static_cast<size_t>(18) * Lv.ld;
      vc.b.push_back(v);
      vc.xa.push_back(v + s18);
      vc.xb.push_back(v + 2 * s18);
      vc.res.push_back(v + 3 * s18);
    }
  }
  // Level 1 distributed over the slabs when there is a level 2 below it (the
  // coarsest level itself stays replicated: it is one cluster kernel)
  const bool dist1 = use_gmg && vc.L >= 2;
  int max_plane1 = 0;
  if (dist1) {
    const auto& L1 = c->gmg[0];
    const int rc = L1.r;
    std::vector<int> ps(rc + 1);
    {
      DevBuf pbuf;
      pbuf.ensure(sizeof(int) * rc);
      plane_start_kernel<<<(rc + 127) / 128, 128, 0, c->stream>>>(L1.off.as<int>(), rc, pbuf.as<int>());
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(ps.data(), pbuf.p, sizeof(int) * rc, cudaMemcpyDeviceToHost, c->stream));
      c->sync();
    }
    ps[rc] = L1.n;
    for (auto& S : slabs) {
      Level1Plan& Q = S.P1;
      const int cz0 = (S.P.z0 + 1) / 2, cz1 = (S.P.z1 + 1) / 2;
      const int glo = (cz0 - 1 + rc) % rc, ghi = cz1 % rc;
      Q.c0 = ps[cz0];
      Q.c1 = ps[cz1];
      Q.planes = cz1 - cz0;
      Q.first_n = ps[cz0 + 1] - ps[cz0];
      Q.last0 = ps[cz1 - 1];
      Q.glo0 = ps[glo];
      Q.glo_n = ps[glo + 1] - ps[glo];
      Q.ghi0 = ps[ghi];
      Q.ghi_n = ps[ghi + 1] - ps[ghi];
      max_plane1 = std::max({max_plane1, Q.first_n, Q.c1 - Q.last0, Q.glo_n, Q.ghi_n});
      const size_t bytes = static_cast<size_t>(4) * 18 * L1.ld * sizeof(TZ);
      S.v1.ensure(bytes);
      CK(cudaMemsetAsync(S.v1.p, 0, bytes, c->stream));
    }
    xfer.ensure(std::max(xfer.cap, 4 * 18 * static_cast<size_t>(std::max(max_plane1, 1)) * sizeof(double)));
  }
  PcgState hs{};
  hs.tol = opt.tol;
  hs.ridge = ridge_op;
  hs.max_iter = opt.max_iter > 0 ? opt.max_iter : 20 * r + 2000;
  std::memcpy(c->hstate, &hs, sizeof(hs));
  CK(cudaMemcpyAsync(c->state.p, c->hstate, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  CK(cudaEventRecord(c->ev[4], c->stream));
  PcgState* dst = c->state.as<PcgState>();
  vc.st = dst;
  vc.partials = slabs[0].partials.as<double>();  // coarse levels never defer
  const TV* beta_apply = sizeof(TV) == 8 ? reinterpret_cast<const TV*>(c->beta64.p)
                                         : reinterpret_cast<const TV*>(c->beta32.p);
  double* totals = tot.as<double>();

  // cross-slab sum: in-process slabs are summed by the finalize kernel; ranks
  // all-reduce their one total first
  auto reduce = [&](int k) {
    if (dist) comm->allreduce(totals, k, true, c->stream);
  };
  // ghost exchange of an 18-component vector (z each iteration, x for C^H)
  auto exchange = [&](auto vec_of, const std::function<void()>& during = {}) {
    using T = std::remove_pointer_t<decltype(vec_of(slabs[0]))>;
    T* buf = xfer.as<T>();
    if (!dist) {
      if (during) during();  // (one stream: nothing to overlap, same order as the ranks)
      for (int s = 0; s < nloc; ++s) {
        Slab& me = slabs[s];
        Slab& lo = slabs[(s - 1 + nloc) % nloc];
        Slab& hi = slabs[(s + 1) % nloc];
        launch_pack<T>(vec_of(lo), lo.P.n_owned - lo.P.cnt_last, lo.P.cnt_last, buf, c->stream);
        launch_unpack<T>(vec_of(me), me.P.n_owned, me.P.n_glo, buf, c->stream);
        launch_pack<T>(vec_of(hi), 0, hi.P.cnt_first, buf, c->stream);
        launch_unpack<T>(vec_of(me), me.P.n_owned + me.P.n_glo, me.P.n_ghi, buf, c->stream);
      }
      return;
    }
    Slab& me = slabs[0];
    const size_t stride = 18 * static_cast<size_t>(std::max(max_plane, 1));
    T *send_hi = buf, *send_lo = buf + stride, *recv_lo = buf + 2 * stride, *recv_hi = buf + 3 * stride;
    launch_pack<T>(vec_of(me), me.P.n_owned - me.P.cnt_last, me.P.cnt_last, send_hi, c->stream);
    launch_pack<T>(vec_of(me), 0, me.P.cnt_first, send_lo, c->stream);
    comm->exchange(send_hi, 18 * static_cast<size_t>(me.P.cnt_last), send_lo, 18 * static_cast<size_t>(me.P.cnt_first),
                   recv_lo, 18 * static_cast<size_t>(me.P.n_glo), recv_hi, 18 * static_cast<size_t>(me.P.n_ghi),
                   sizeof(T) == 8, c->stream, during);
    launch_unpack<T>(vec_of(me), me.P.n_owned, me.P.n_glo, recv_lo, c->stream);
    launch_unpack<T>(vec_of(me), me.P.n_owned + me.P.n_glo, me.P.n_ghi, recv_hi, c->stream);
  };
  auto grid_u = [&](const Slab& S) { return 6 * std::max(1, std::min((S.P.n_owned + 255) / 256, c->num_sms * 2)); };
  auto grid_a_n = [&](int n) { return apply_grid(n, c->num_sms); };
  auto update_all = [&](int init) {
    for (int s = 0; s < nloc; ++s) {
      Slab& S = slabs[s];
      UpdateArgs<TX, TV, TZ> ua{X(S), R(S), Pv(S), Q(S), Z(S), D(S), S.partials.as<double>(), dst,
                                S.P.n_owned, static_cast<int>(S.ld), init, totals + 12 * s, 1,
                                use_gmg ? 1 : 0, use_gmg ? XA(S) : nullptr, static_cast<TZ>(vc.gp.omega)};
      launch_update<TX, TV, TZ>(ua, grid_u(S), c->stream);
    }
    reduce(12);
    if (use_gmg)
      launch_finalize_update_gmg(dst, totals, nloc, init, c->stream);
    else
      launch_finalize_update(dst, totals, nloc, init, c->stream);
  };
  // level-0 view of slab s: owned nodes, slab-local map, ghost planes
  auto fine_view = [&](Slab& S, double* tot_s) {
    GmgLevelView<TZ> v{S.list.as<int>(), S.map.as<int>(), beta_z, nullptr, D(S), r, S.P.n_owned, S.P.n_local,
                       static_cast<TZ>(ridge)};
    v.zbase = S.P.zbase;
    v.totals = tot_s;
    return v;
  };
  // A slab's own ids are plane-ordered: the interior planes read no ghost value
  // and run while the ghost planes are in flight (the exchange's `during`),
  // the first and last planes after the unpack.
  struct NodeRanges {
    int lo0, lo1, in0, in1, hi0, hi1;
  };
  auto node_ranges = [](int a0, int a1, int first_n, int last0, bool one_plane) {
    return one_plane ? NodeRanges{a0, a1, a1, a1, a1, a1} : NodeRanges{a0, a0 + first_n, a0 + first_n, last0, last0, a1};
  };
  auto ranges0 = [&](const Slab& S) {
    return node_ranges(0, S.P.n_owned, S.P.cnt_first, S.P.n_owned - S.P.cnt_last, S.P.z1 - S.P.z0 == 1);
  };
  std::vector<TZ*> cur(nloc), oth(nloc);
  // level-1 vectors of slab s: b, x (two buffers), residual
  const size_t ld1 = dist1 ? static_cast<size_t>(c->gmg[0].ld) : 0;
  auto B1 = [&](Slab& S) { return S.v1.as<TZ>(); };
  auto XA1 = [&](Slab& S) { return S.v1.as<TZ>() + 18 * ld1; };
  auto XB1 = [&](Slab& S) { return S.v1.as<TZ>() + 36 * ld1; };
  auto RES1 = [&](Slab& S) { return S.v1.as<TZ>() + 54 * ld1; };
  auto view1 = [&](Slab& S) {  // level 1 restricted to the slab's own nodes
    GmgLevelView<TZ> v = vc.view[1];
    v.n0 = S.P1.c0;
    v.n = S.P1.c1;
    v.bricks = BrickView{};
    return v;
  };
  // ghost-plane exchange of a level-1 vector: each slab's boundary planes
  // become its neighbours' ghost planes (same ids in every slab's vector)
  std::vector<TZ*> cur1(nloc), oth1(nloc);
  auto exchange1 = [&](std::vector<TZ*>& v, const std::function<void()>& during = {}) {
    TZ* buf = xfer.as<TZ>();
    if (!dist) {
      if (during) during();
      for (int s = 0; s < nloc; ++s) {
        const Level1Plan& Q = slabs[s].P1;
        TZ* lo = v[(s - 1 + nloc) % nloc];
        TZ* hi = v[(s + 1) % nloc];
        launch_pack<TZ>(v[s], Q.c0, Q.first_n, buf, c->stream);
        launch_unpack<TZ>(lo, Q.c0, Q.first_n, buf, c->stream);
        launch_pack<TZ>(v[s], Q.last0, Q.c1 - Q.last0, buf, c->stream);
        launch_unpack<TZ>(hi, Q.last0, Q.c1 - Q.last0, buf, c->stream);
      }
      return;
    }
    const Level1Plan& Q = slabs[0].P1;
    const size_t stride = 18 * static_cast<size_t>(std::max(max_plane1, 1));
    TZ *send_hi = buf, *send_lo = buf + stride, *recv_lo = buf + 2 * stride, *recv_hi = buf + 3 * stride;
    launch_pack<TZ>(v[0], Q.last0, Q.c1 - Q.last0, send_hi, c->stream);
    launch_pack<TZ>(v[0], Q.c0, Q.first_n, send_lo, c->stream);
    comm->exchange(send_hi, 18 * static_cast<size_t>(Q.c1 - Q.last0), send_lo, 18 * static_cast<size_t>(Q.first_n),
                   recv_lo, 18 * static_cast<size_t>(Q.glo_n), recv_hi, 18 * static_cast<size_t>(Q.ghi_n),
                   sizeof(TZ) == 8, c->stream, during);
    launch_unpack<TZ>(v[0], Q.glo0, Q.glo_n, recv_lo, c->stream);
    launch_unpack<TZ>(v[0], Q.ghi0, Q.ghi_n, recv_hi, c->stream);
  };
  // Level 1 on the slabs (dist1): restriction onto each slab's own coarse
  // nodes (after a ghost exchange of the level-0 residual), damped block
  // Jacobi with a ghost exchange before every sweep, the residual's partial
  // restrictions summed into the replicated level 2 (an all-reduce 8x smaller
  // than level 1's), level 2.. as before, prolongation onto the own nodes and
  // a last ghost exchange for the level-0 prolongation.
  auto level1_slabs = [&](int init) {
    const TZ wc = static_cast<TZ>(vc.gp.omega_c);
    const int nu1 = vc.gp.nu_at(1);
    exchange([&](Slab& S) { return RES(S); });
    for (int s = 0; s < nloc; ++s) {
      Slab& S = slabs[s];
      launch_restrict_own<TZ>(view1(S), S.map.as<int>(), S.P.zbase, S.P.nzl, r, RES(S), B1(S), dst, c->stream);
      launch_jacobi_first<TZ, TZ>(view1(S), B1(S), XA1(S), wc, dst, c->stream);
      cur1[s] = XA1(S);
      oth1[s] = XB1(S);
    }
    auto sweep1 = [&](int mode) {  // mode 0: cur1 -> oth1 (swap); 1: cur1 -> RES1
      auto run = [&](int s, int a, int b) {
        Slab& S = slabs[s];
        auto V = view1(S);
        V.n0 = a;
        V.n = b;
        if (b > a)
          launch_level_sweep<TZ, TZ>(V, false, B1(S), cur1[s], mode == 1 ? RES1(S) : oth1[s], wc, mode, dst,
                                     vc.partials, init, apply_grid(b - a, c->num_sms), c->stream);
      };
      auto rg = [&](int s) {
        const Level1Plan& Q = slabs[s].P1;
        return node_ranges(Q.c0, Q.c1, Q.first_n, Q.last0, Q.planes == 1);
      };
      exchange1(cur1, [&] {
        for (int s = 0; s < nloc; ++s) run(s, rg(s).in0, rg(s).in1);
      });
      for (int s = 0; s < nloc; ++s) {
        run(s, rg(s).lo0, rg(s).lo1);
        run(s, rg(s).hi0, rg(s).hi1);
        if (mode == 0) std::swap(cur1[s], oth1[s]);
      }
    };
    for (int k = 1; k < nu1; ++k) sweep1(0);
    sweep1(1);
    TZ* b2 = vc.b[2];
    CK(cudaMemsetAsync(b2, 0, static_cast<size_t>(18) * c->gmg[1].ld * sizeof(TZ), c->stream));
    for (int s = 0; s < nloc; ++s)
      launch_restrict_partial<TZ>(vc.view[2], view1(slabs[s]), RES1(slabs[s]), b2, dst, c->stream);
    if (dist) comm->allreduce(b2, 18 * static_cast<size_t>(c->gmg[1].ld), sizeof(TZ) == 8, c->stream);
    TZ* x2 = vc.level(2, nullptr, init);  // levels 2.., replicated
    for (int s = 0; s < nloc; ++s) launch_prolong<TZ>(view1(slabs[s]), vc.view[2], x2, cur1[s], dst, c->stream);
    for (int k = 1; k <= nu1; ++k) sweep1(0);
    exchange1(cur1);
    for (int s = 0; s < nloc; ++s) {
      Slab& S = slabs[s];
      launch_prolong<TZ>(fine_view(S, nullptr), vc.view[1], cur1[s], cur[s], dst, c->stream);
    }
  };
  // z = M r: the V-cycle with level 0 on the slabs
  auto precondition_all = [&](int init) {
    const TZ w = static_cast<TZ>(vc.gp.omega);
    const int nu = vc.gp.nu_at(0);
    for (int s = 0; s < nloc; ++s) {
      cur[s] = XA(slabs[s]);  // omega Dinv r, written by the update kernel
      oth[s] = XB(slabs[s]);
    }
    auto sweep_all = [&](int mode) {  // mode 0: cur -> oth (swap); 1: cur -> RES
      auto run = [&](int s, int a, int b) {
        Slab& S = slabs[s];
        auto V = fine_view(S, nullptr);
        V.n0 = a;
        V.n = b;
        if (b > a)
          launch_level_sweep<TX, TZ>(V, true, R(S), cur[s], mode == 1 ? RES(S) : oth[s], w, mode, dst,
                                     S.partials.as<double>(), init, apply_grid(b - a, c->num_sms), c->stream);
      };
      exchange([&](Slab& S) { return cur[&S - slabs.data()]; },
               [&] {
                 for (int s = 0; s < nloc; ++s) run(s, ranges0(slabs[s]).in0, ranges0(slabs[s]).in1);
               });
      for (int s = 0; s < nloc; ++s) {
        run(s, ranges0(slabs[s]).lo0, ranges0(slabs[s]).lo1);
        run(s, ranges0(slabs[s]).hi0, ranges0(slabs[s]).hi1);
        if (mode == 0) std::swap(cur[s], oth[s]);
      }
    };
    for (int k = 1; k < nu; ++k) sweep_all(0);
    sweep_all(1);
    if (dist1) {
      level1_slabs(init);
    } else {
      // restriction of the owned fine residuals, summed over slabs / ranks,
      // into the replicated coarse levels
      TZ* b1 = vc.b[1];
      const auto& C1 = vc.view[1];
      CK(cudaMemsetAsync(b1, 0, static_cast<size_t>(18) * c->gmg[0].ld * sizeof(TZ), c->stream));
      for (int s = 0; s < nloc; ++s) {
        Slab& S = slabs[s];
        launch_restrict_slab<TZ>(C1, S.map.as<int>(), S.P.zbase, S.P.nzl, S.P.z0, S.P.z1, r, RES(S), b1, dst,
                                 c->stream);
      }
      if (dist) comm->allreduce(b1, 18 * static_cast<size_t>(c->gmg[0].ld), sizeof(TZ) == 8, c->stream);
      TZ* x1 = vc.level(1, nullptr, init);  // coarse levels, replicated
      for (int s = 0; s < nloc; ++s) {
        Slab& S = slabs[s];
        launch_prolong<TZ>(fine_view(S, nullptr), C1, x1, cur[s], dst, c->stream);
      }
    }
    for (int k = 1; k <= nu; ++k) {
      if (k < nu) {
        sweep_all(0);
        continue;
      }
      exchange([&](Slab& S) { return cur[&S - slabs.data()]; });
      for (int s = 0; s < nloc; ++s) {
        Slab& S = slabs[s];
        launch_level_sweep_out<TX, TZ, TZ>(fine_view(S, totals + 6 * s), R(S), cur[s], Z(S), w, dst,
                                           S.partials.as<double>(), init, apply_grid(S.P.n_owned, c->num_sms),
                                           c->stream);
      }
      reduce(6);
      launch_finalize_gamma(dst, totals, nloc, init, c->stream);
    }
  };
  // The apply in three node ranges per slab: the interior planes read no
  // ghost values, so they run while the ghost planes of z are in flight
  // (SlabTransport::exchange's `during`); the two boundary planes follow the
  // unpack.  Owned ids are plane-ordered: plane z0 = [0, cnt_first), plane
  // z1-1 = [n_owned - cnt_last, n_owned).  Each range defers its 6 sums into
  // rtot[slab][range]; sum_ranges_kernel adds them in fixed order, so the
  // in-process slabs and the ranks produce the same bits.
  double* rtot = totals + 21 * nloc;
  auto apply_range = [&](Slab& S, int s, int k) {
    const SlabPlan& P = S.P;
    const bool one_plane = P.z1 - P.z0 == 1;
    const int lo_end = one_plane ? P.n_owned : P.cnt_first;
    const int hi_beg = one_plane ? P.n_owned : P.n_owned - P.cnt_last;
    const int n0 = k == 0 ? 0 : (k == 1 ? lo_end : hi_beg);
    const int n1 = k == 0 ? lo_end : (k == 1 ? hi_beg : P.n_owned);
    ApplyArgs<TV, TZ> aa{S.list.as<int>(), S.map.as<int>(), beta_apply, Z(S), Pv(S), Q(S),
                         S.partials.as<double>(), dst, r, n1, static_cast<int>(S.ld),
                         P.n_local, P.zbase, P.nzl, rtot + (3 * s + k) * 6, 1};
    aa.n0 = n0;
    launch_apply<TV, TZ>(aa, std::max(1, grid_a_n(n1 - n0)), c->stream);
  };
  auto apply_all = [&]() {
    exchange([&](Slab& S) { return Z(S); },
             [&] {
               for (int s = 0; s < nloc; ++s) apply_range(slabs[s], s, 1);
             });
    for (int s = 0; s < nloc; ++s) {
      apply_range(slabs[s], s, 0);
      apply_range(slabs[s], s, 2);
    }
    sum_ranges_kernel<<<1, 32 * ((6 * nloc + 31) / 32), 0, c->stream>>>(rtot, totals, nloc);
    reduce(6);
    launch_finalize_apply(dst, totals, nloc, c->stream);
  };

  update_all(1);
  if (use_gmg) precondition_all(1);
  apply_all();
  const int check = opt.check_every > 0 ? opt.check_every : 16;
  int64_t launches = 0;
  NvtxRange pcg_range("shellular: z-slab PCG iterations");
  auto iterations = [&]() {
    for (int it = 0; it < check; ++it) {
      update_all(0);
      if (use_gmg) precondition_all(0);
      apply_all();
    }
  };
  // The `check` iterations between host polls as one CUDA graph (in-process
  // slabs, or ranks whose transport only enqueues device work: NCCL on the
  // side stream is captured with its fork/join events).  A capture the
  // transport refuses falls back to eager launches.
  struct ExecGuard {
    cudaGraphExec_t e = nullptr;
    ~ExecGuard() {
      if (e) cudaGraphExecDestroy(e);
    }
  } guard;
  cudaGraphExec_t& exec = guard.e;
  if (!c->profiling && (!dist || comm->capturable())) {
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      iterations();
    } catch (const ShlError&) {
      cudaStreamEndCapture(c->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      graph = nullptr;
      cudaGetLastError();
    }
    if (graph == nullptr && cudaStreamEndCapture(c->stream, &graph) != cudaSuccess) graph = nullptr;
    if (graph && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) exec = nullptr;
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
  }
  for (;;) {
    if (exec)
      CK(cudaGraphLaunch(exec, c->stream));
    else
      iterations();
    launches += check * (2 * nloc + 2 + 11 * nloc);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->hstate, c->state.p, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (c->hstate->stop) break;
  }
  CK(cudaEventRecord(c->ev[5], c->stream));
  const PcgState& fin = *c->hstate;
  if (fin.error) throw ShlError(SHL_SOLVER, "grid CG: operator lost positive definiteness");
  if (!fin.all_done) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "grid CG did not reach tolerance %g in %d iterations", opt.tol,
                  fin.max_iter);
    throw ShlError(SHL_SOLVER, buf);
  }
  // C^H: owned elements need x on the ghost-hi plane
  exchange([&](Slab& S) { return X(S); });
  for (int s = 0; s < nloc; ++s) {
    Slab& S = slabs[s];
    const int ne = S.P.e_hi - S.P.e_lo;
    const int grid_c = std::max(1, std::min((ne + 31) / 32, c->num_sms * 16));
    ChomArgs<TX> ca{c->elem_list.as<int>() + S.P.e_lo, S.map.as<int>(), c->beta64.as<double>(), X(S),
                    S.partials.as<double>(), totals + 21 * s, dst, ne, r, static_cast<int>(S.ld),
                    S.P.zbase, S.P.nzl, 1};
    if (ne > 0)
      launch_chom<TX>(ca, grid_c, c->stream);
    else
      CK(cudaMemsetAsync(totals + 21 * s, 0, 21 * sizeof(double), c->stream));
  }
  reduce(21);
  launch_finalize_chom(totals, nloc, c->cout.as<double>(), c->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->hC, c->cout.p, 36 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->ev[6], c->stream));
  c->sync();
  std::memcpy(C_out, c->hC, 36 * sizeof(double));
  c->launches += launches;
  if (st) {
    st->t_AS = c->ms(3, 4);
    st->t_solve = c->ms(4, 5);
    st->t_C = c->ms(5, 6);
    for (int s = 0; s < 6; ++s) st->iterations[s] = fin.iters[s];
    st->converged = 1;
    st->precision = prec;
    st->gmg_levels = use_gmg ? vc.L + 1 : 0;
  }
}

void homogenize_slabs(shl_ctx* c, int G, SlabTransport* comm, const shl_design* design,
                      const shl_shell_params* sp, const shl_material* mat, int r,
                      const shl_solve_options* o, double* C_out, shl_stats* st) {
  if (!C_out) throw ShlError(SHL_VALIDATION, "null argument");
  const shl_solve_options opt = default_opts(o);
  double K0[576];
  validate_inputs(design, sp, mat, r, K0);
  FieldInputs fin = tagged("field", [&] { return prepare_field(HostDesign::from_abi(*design), r); });
  CK(cudaEventRecord(c->ev[0], c->stream));
  tagged("field", [&] {
    run_field(c, fin);
    return 0;
  });
  CK(cudaEventRecord(c->ev[1], c->stream));
  read_norm(c);
  if (c->norm == 0.0) throw ShlError(SHL_DEGENERATE, "field: design is degenerate (norm = 0)");
  tagged("mesh", [&] {
    run_mesh(c, *sp);
    return 0;
  });
  CK(cudaEventRecord(c->ev[2], c->stream));
  const int prec = resolve_precision(opt);
  // preconditioner choice as in the single-device solve (shl_api.cu)
  const bool gmg = opt.preconditioner == SHL_PRECOND_GMG ||
                   (opt.preconditioner == SHL_PRECOND_AUTO && r % 2 == 0 && r / 2 >= gmg_params().min_r);
  auto once = [&](bool use_gmg) {
    switch (prec) {
      case SHL_PREC_FP64: run_solve_slabs<double, double, double>(c, K0, opt, C_out, st, prec, G, comm, use_gmg); break;
      case SHL_PREC_MIXED:
        if (use_gmg)  // FP64 operator with the FP32 V-cycle (see solve_dispatch_once)
          run_solve_slabs<double, double, float>(c, K0, opt, C_out, st, prec, G, comm, true);
        else
          run_solve_slabs<double, float, float>(c, K0, opt, C_out, st, prec, G, comm, false);
        break;
      default: run_solve_slabs<float, float, float>(c, K0, opt, C_out, st, prec, G, comm, use_gmg); break;
    }
  };
  tagged("solve", [&] {
    if (!gmg || opt.preconditioner != SHL_PRECOND_AUTO) {
      once(gmg);
      return 0;
    }
    try {
      once(true);
    } catch (const ShlError& e) {  // AUTO: a multigrid breakdown is redone with block Jacobi
      if (e.code != SHL_SOLVER || std::string(e.what()).find("positive definiteness") == std::string::npos) throw;
      once(false);
      if (st) st->precond_fallback = 1;
    }
    return 0;
  });
  if (st) {
    st->t_field = c->ms(0, 1);
    st->t_mesh = c->ms(1, 2);
    st->t_fwd = c->ms(0, 6);
    fill_mesh_stats(c, st);
  }
}

}  // namespace host
}  // namespace shl

using namespace shl::host;

extern "C" {

int shl_homogenize_slabs(shl_ctx* c, int n_slabs, const shl_design* design,
                         const shl_shell_params* sp, const shl_material* mat, int r,
                         const shl_solve_options* opt, double* C_out, shl_stats* st) {
  if (!c) return SHL_VALIDATION;
  if (st) std::memset(st, 0, sizeof(*st));
  return guarded(c, [&] { homogenize_slabs(c, n_slabs, nullptr, design, sp, mat, r, opt, C_out, st); });
}

int shl_nccl_unique_id(uint8_t* id_out) {
  if (!id_out) return SHL_VALIDATION;
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    NK(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, NCCL_UNIQUE_ID_BYTES);
  });
}

int shl_homogenize_zslab(shl_ctx* c, const uint8_t* nccl_id, int rank, int nranks,
                         const shl_design* design, const shl_shell_params* sp,
                         const shl_material* mat, int r, const shl_solve_options* opt,
                         double* C_out, shl_stats* st) {
  if (!c || !nccl_id || nranks < 2 || rank < 0 || rank >= nranks) return SHL_VALIDATION;
  if (st) std::memset(st, 0, sizeof(*st));
  return guarded(c, [&] {
    auto* comm = static_cast<NcclComm*>(c->nccl);
    if (!comm || comm->rank != rank || comm->nranks != nranks ||
        std::memcmp(comm->id, nccl_id, NCCL_UNIQUE_ID_BYTES) != 0) {
      delete comm;
      c->nccl = nullptr;
      comm = new NcclComm();
      std::memcpy(comm->id, nccl_id, NCCL_UNIQUE_ID_BYTES);
      comm->rank = rank;
      comm->nranks = nranks;
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, NCCL_UNIQUE_ID_BYTES);
      NK(nccl().CommInitRank(&comm->comm, nranks, id, rank));
      c->nccl = comm;
      c->nccl_deleter = [](void* p) { delete static_cast<NcclComm*>(p); };
    }
    NcclTransport t(comm);
    homogenize_slabs(c, nranks, &t, design, sp, mat, r, opt, C_out, st);
  });
}

int shl_homogenize_zslab_host(shl_ctx* c, const shl_slab_transport* transport, int rank, int nranks,
                              const shl_design* design, const shl_shell_params* sp, const shl_material* mat,
                              int r, const shl_solve_options* opt, double* C_out, shl_stats* st) {
  if (!c || !transport || !transport->allreduce_sum || !transport->ring_exchange || nranks < 2 || rank < 0 ||
      rank >= nranks)
    return SHL_VALIDATION;
  if (st) std::memset(st, 0, sizeof(*st));
  return guarded(c, [&] {
    HostTransport t(*transport, rank, nranks);
    homogenize_slabs(c, nranks, &t, design, sp, mat, r, opt, C_out, st);
  });
}

}  // extern "C"
