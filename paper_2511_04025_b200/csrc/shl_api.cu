// shl_api.cu -- the C ABI of include/shellular_cuda.h: context, device
// workspaces, stage orchestration and error mapping.
//
// Stage map onto the reference's homogenize (pipeline.hpp:61-113):
//   field    host: expand_symmetry, coefficients, cosine tables (host_design.cpp)
//            device: K1 (field.cu)                               -> t_field
//   mesh     K2 classify / dilate / complete / corners / beta   -> t_mesh
//   PBC      node activation + ordered compaction (voxel.cu)      -> t_PBC
//   AS, RHS  block-Jacobi + right-hand sides (solver.cu setup)    -> t_AS (+t_RHS)
//   solve    K4/K5 PCG loop, device-resident scalars               -> t_solve
//   C        K6 energy reduction                                   -> t_C
// Only the norm / counts (one 64-byte readback after meshing), the PCG flag
// (every check_every iterations) and the 6x6 tensor cross PCIe.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <future>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "context.h"
#include "gmg_host.h"

using shl::ShlError;

namespace shl {
namespace host {

thread_local std::string g_thread_error;
thread_local cudaStream_t g_alloc_stream = nullptr;

__global__ void finalize_counts_kernel(Misc* m, const int* node_flag, const int* node_off,
                                       const int* elem_flag, const int* elem_off, int n3,
                                       const double* beta_partials, int nbp) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int b = threadIdx.x; b < nbp; b += blockDim.x) s += beta_partials[2 * b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    m->beta_sum = sh[0];
    m->n_nodes = node_off[n3 - 1] + node_flag[n3 - 1];
    m->n_elem = elem_off[n3 - 1] + elem_flag[n3 - 1];
    m->node0_active = node_flag[0];
  }
}


// element-local affine loads T (grid_solver.hpp:119-126) and W = K0*T
void element_loads(const double* K0, int r, double* T, double* W) {
  for (int n = 0; n < 8; ++n)
    for (int a = 0; a < 3; ++a)
      for (int s = 0; s < 6; ++s) {
        // eps_s (fem.hpp:129-142) times y = corner offset / r
        double e[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (s < 3) e[s][s] = 1.0;
        if (s == 3) e[1][2] = e[2][1] = 0.5;
        if (s == 4) e[0][2] = e[2][0] = 0.5;
        if (s == 5) e[0][1] = e[1][0] = 0.5;
        double y[3] = {shl::kCorner[n][0] / double(r), shl::kCorner[n][1] / double(r),
                       shl::kCorner[n][2] / double(r)};
        T[(3 * n + a) * 6 + s] = e[a][0] * y[0] + e[a][1] * y[1] + e[a][2] * y[2];
      }
  for (int i = 0; i < 24; ++i)
    for (int s = 0; s < 6; ++s) {
      double acc = 0.0;
      for (int j = 0; j < 24; ++j) acc += K0[i * 24 + j] * T[j * 6 + s];
      W[i * 6 + s] = acc;
    }
}


void require_r(int r) {
  if (r < 4) throw ShlError(SHL_VALIDATION, "grid resolution must be >= 4");
  if (r > 1024) throw ShlError(SHL_VALIDATION, "grid resolution must be <= 1024");
}

void alloc_grid(shl_ctx* c, int r) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  c->centres.ensure(n3 * sizeof(double));
  c->corners.ensure(n3 * sizeof(double));
  c->csign.ensure(n3);
  c->misc.ensure(sizeof(Misc));
  c->r = r;
}

// ---- field (sample_grid, field.hpp:488-534) --------------------------------
// Host half: reference arithmetic that must match glibc bit for bit
// (expansion, coefficients, cosine tables).  Device half: K1.


FieldInputs prepare_field(const shl::HostDesign& d, int r) {
  require_r(r);
  FieldInputs f;
  const shl::HostDesign ex = d.expanded();  // validates (field.hpp:149-172)
  f.r = r;
  f.coeff = d.grid_coefficients();
  f.tab = shl::axis_tables(ex, r);
  f.nc = static_cast<int>(ex.sign.size());
  f.n = d.K + 1;
  f.sign.assign(ex.sign.begin(), ex.sign.end());
  return f;
}

void run_field(shl_ctx* c, const FieldInputs& f) {
  const int r = f.r, nc = f.nc, n = f.n;
  alloc_grid(c, r);
  c->grid_ready = c->mesh_ready = false;
  c->tab.ensure(std::max<size_t>(f.tab.size(), 1) * sizeof(double));
  c->coeff.ensure(f.coeff.size() * sizeof(double));
  c->sign8.ensure(std::max<size_t>(f.sign.size(), 1));
  c->sl.ensure(std::max<size_t>(static_cast<size_t>(nc) * 2 * r * n * n, 1) * sizeof(double));
  // pageable sources: the copies are staged before cudaMemcpyAsync returns
  c->h2d += static_cast<int64_t>(f.h2d_bytes());
  if (!f.tab.empty())
    CK(cudaMemcpyAsync(c->tab.p, f.tab.data(), f.tab.size() * sizeof(double),
                       cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->coeff.p, f.coeff.data(), f.coeff.size() * sizeof(double),
                     cudaMemcpyHostToDevice, c->stream));
  if (!f.sign.empty())
    CK(cudaMemcpyAsync(c->sign8.p, f.sign.data(), f.sign.size(), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->misc.p, 0, sizeof(Misc), c->stream));
  shl::launch_field_sl(c->tab.as<double>(), c->coeff.as<double>(), c->sl.as<double>(), nc, r, n,
                       c->stream);
  shl::launch_field_samples(c->tab.as<double>(), c->sl.as<double>(), c->sign8.as<int8_t>(), nc, r,
                            n, c->centres.as<double>(), c->corners.as<double>(),
                            c->csign.as<int8_t>(), &c->misc.as<Misc>()->norm_bits, c->stream);
  c->launches += 2;
  CK(cudaGetLastError());
  c->grid_ready = true;
}

void read_norm(shl_ctx* c) {
  c->d2h += sizeof(Misc);
  CK(cudaMemcpyAsync(c->hmisc, c->misc.p, sizeof(Misc), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  double v;
  std::memcpy(&v, &c->hmisc->norm_bits, sizeof(double));
  c->norm = v;
}

// ---- topology: node ids and element list (ordered compaction) ------------
void build_topology(shl_ctx* c) {
  const int r = c->r;
  const int n3 = r * r * r;
  c->node_flag.ensure(static_cast<size_t>(n3) * sizeof(int));
  c->off.ensure(static_cast<size_t>(n3) * sizeof(int) * 2);
  c->node_map.ensure(static_cast<size_t>(n3) * sizeof(int));
  c->node_list.ensure(static_cast<size_t>(n3) * sizeof(int));
  c->elem_list.ensure(static_cast<size_t>(n3) * sizeof(int));
  const shl::BrickDims bd = shl::brick_dims(r);
  const size_t tb = shl::scan_temp_bytes(static_cast<int>(std::max<long long>(n3, bd.np)));
  c->scan_tmp.ensure(tb);
  c->bflag.ensure(static_cast<size_t>(bd.np) * sizeof(int));
  c->boff.ensure(static_cast<size_t>(bd.np) * sizeof(int));
  c->bact.ensure(static_cast<size_t>(bd.nb) * sizeof(int));
  c->bidx.ensure(static_cast<size_t>(bd.nb) * sizeof(int));
  c->bcoord.ensure(static_cast<size_t>(bd.nb) * sizeof(int));
  c->bstart.ensure(static_cast<size_t>(bd.nb + 1) * sizeof(int));
  int* off_n = c->off.as<int>();
  int* off_e = off_n + n3;
  shl::launch_node_flags(c->elem_flag.as<int>(), r, c->node_flag.as<int>(), c->stream);
  // grid-order offsets (node counts; the z-slab plans number their slabs from them)
  shl::launch_exclusive_scan(c->node_flag.as<int>(), off_n, n3, c->scan_tmp.p, c->scan_tmp.cap,
                             c->stream);
  // level-0 node ids in brick-major order: each active 8x8x4 brick owns a
  // contiguous id range, so the staged brick kernels read their own nodes'
  // rows coalesced (brick.cuh)
  shl::launch_brick_numbering(c->node_flag.as<int>(), r, c->bflag.as<int>(), c->boff.as<int>(),
                              c->bact.as<int>(), c->bidx.as<int>(), c->scan_tmp.p, c->scan_tmp.cap,
                              c->node_map.as<int>(), c->node_list.as<int>(), c->bcoord.as<int>(),
                              c->bstart.as<int>(), &c->misc.as<Misc>()->n_bricks, c->stream);
  shl::launch_exclusive_scan(c->elem_flag.as<int>(), off_e, n3, c->scan_tmp.p, c->scan_tmp.cap,
                             c->stream);
  shl::launch_scatter_compact(c->elem_flag.as<int>(), off_e, n3, nullptr, c->elem_list.as<int>(),
                              c->stream);
  const int nbp = (n3 + 255) / 256;
  finalize_counts_kernel<<<1, 256, 0, c->stream>>>(c->misc.as<Misc>(), c->node_flag.as<int>(),
                                                   off_n, c->elem_flag.as<int>(), off_e, n3,
                                                   c->beta_partials.as<double>(), nbp);
  c->launches += 1 + 2 + 2 + 6 + 1;
  CK(cudaGetLastError());
  c->d2h += sizeof(Misc);
  CK(cudaMemcpyAsync(c->hmisc, c->misc.p, sizeof(Misc), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  c->n_nodes = c->hmisc->n_nodes;
  c->n_elem = c->hmisc->n_elem;
  c->node0_active = c->hmisc->node0_active;
  c->n_bricks = c->hmisc->n_bricks;
  c->beta_sum = c->hmisc->beta_sum;
  c->volume_ratio = c->beta_sum / (double(r) * r * r);
}

// ---- mesh (build_reduced_mesh, voxel.hpp:235-313) --------------------------
void run_mesh(shl_ctx* c, const shl_shell_params& sp) {
  if (!c->grid_ready) throw ShlError(SHL_VALIDATION, "no resident grid: call shl_sample_grid first");
  if (!(sp.sharpness > 0.0)) throw ShlError(SHL_VALIDATION, "sharpness must be positive");
  if (!(sp.floor_ratio > 0.0 && sp.floor_ratio < 1.0))
    throw ShlError(SHL_VALIDATION, "floor must lie in (0, 1)");
  if (sp.expand_layers < 0) throw ShlError(SHL_VALIDATION, "expand_layers must be >= 0");
  if (c->norm == 0.0)
    throw ShlError(SHL_DEGENERATE, "cannot classify surface elements of a degenerate field");
  const int r = c->r;
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const int layers =
      sp.expand_layers > 0 ? sp.expand_layers : std::max(1, static_cast<int>(std::lround(2.0 * r / 64.0)));
  c->occ0.ensure(n3);
  c->occ1.ensure(n3);
  c->beta64.ensure(n3 * sizeof(double));
  c->beta32.ensure(n3 * sizeof(float));
  c->elem_flag.ensure(n3 * sizeof(int));
  c->beta_partials.ensure(((n3 + 255) / 256) * 2 * sizeof(double));
  uint8_t* a = c->occ0.as<uint8_t>();
  uint8_t* b = c->occ1.as<uint8_t>();
  Misc* dm = c->misc.as<Misc>();
  CK(cudaMemsetAsync(&dm->n_surface, 0, sizeof(int) * 2, c->stream));
  shl::launch_classify(c->csign.as<int8_t>(), a, r, &dm->n_surface, c->stream);
  for (int l = 0; l < layers; ++l) {
    shl::launch_dilate(a, b, r, c->stream);
    std::swap(a, b);
  }
  shl::launch_complete(a, b, r, &dm->touches, c->stream);
  std::swap(a, b);
  shl::launch_force_corners(a, r, &dm->touches, c->stream);
  // norm on device: reuse the bits written by the field kernel
  shl::launch_beta(a, c->centres.as<double>(), reinterpret_cast<const double*>(&dm->norm_bits),
                   sp.sharpness, sp.floor_ratio, r, c->beta64.as<double>(), c->beta32.as<float>(),
                   c->elem_flag.as<int>(), c->beta_partials.as<double>(), 0, c->stream);
  c->launches += 4 + layers;
  CK(cudaGetLastError());
  if (a != c->occ0.as<uint8_t>()) {
    // keep the final occupancy in occ0
    CK(cudaMemcpyAsync(c->occ0.p, a, n3, cudaMemcpyDeviceToDevice, c->stream));
  }
  CK(cudaEventRecord(c->ev[7], c->stream));  // t_mesh | t_PBC boundary (voxel.hpp t_select / t_topology)
  c->cc_parent.ensure(n3 * sizeof(int));
  c->cc_corner.ensure(n3 * sizeof(int));
  CK(cudaMemsetAsync(&dm->n_components, 0, sizeof(int) * 2, c->stream));
  shl::launch_components(c->elem_flag.as<int>(), r, c->cc_parent.as<int>(), c->cc_corner.as<int>(),
                         &dm->n_components, &dm->n_floating, c->stream);
  c->launches += 4;
  build_topology(c);
  c->n_surface = c->hmisc->n_surface;
  c->n_components = c->hmisc->n_components;
  c->n_floating = c->hmisc->n_floating;
  if (c->n_surface == 0)
    throw ShlError(SHL_DEGENERATE, "field has no zero crossing: no surface to mesh");
  c->full_fallback = c->n_elem == static_cast<int64_t>(n3);
  c->mesh_ready = true;
}

int resolve_precision(const shl_solve_options& o) {
  if (o.precision >= SHL_PREC_FP64 && o.precision <= SHL_PREC_FP32) return o.precision;
  return o.tol < 1e-7 ? SHL_PREC_FP64 : SHL_PREC_MIXED;
}

// ---- solve on the resident mesh ----------------------------------------------
// TX: r (and x unless TXS says otherwise); TV: p, q and the operator; TZ: z
// and the V-cycle; TXS: storage of x (solver.cuh UpdateArgs).
template <typename TX, typename TV, typename TZ, typename TXS = TX>
void run_solve(shl_ctx* c, const double* K0, const shl_solve_options& opt, double* C_out,
               shl_stats* st, int prec, bool use_gmg) {
  const int r = c->r;
  if (!c->node0_active)
    throw ShlError(SHL_SOLVER,
                   "mesh has no corner node group: cannot prescribe the strain gauge");
  const int n = c->n_nodes;
  // 32-node blocked vectors (solver.cu vbase); node n is an always-zero row
  const int ld = round_up(n + 1, 32);
  const size_t nX = static_cast<size_t>(18) * ld, nV = nX;
  // z: written by the update kernel (block Jacobi) or by the V-cycle's last
  // sweep (multigrid) in TZ, read by the apply.  (An FP64 z for the FP64
  // operator of mixed multigrid removes the FP32->FP64 conversions from the
  // apply but doubles its L1 traffic; measured slower, 364 vs 330 us at 128^3.)
  c->vec.ensure(nX * sizeof(TX) + nX * sizeof(TXS) + 2 * nV * sizeof(TV) +
                (nV + 6 * static_cast<size_t>(ld)) * sizeof(TZ));
  TX* rv = c->vec.as<TX>();
  TXS* x = reinterpret_cast<TXS*>(rv + nX);  // (nX is a multiple of 32: every vector stays 128-byte aligned)
  TV* p = reinterpret_cast<TV*>(x + nX);
  TV* q = p + nV;
  TZ* z = reinterpret_cast<TZ*>(q + nV);
  TZ* dinv = z + nV;
  // update: (node block, load case) blocks; apply: grid-stride over active nodes
  // (node block, load case) CTAs over a grid-stride loop: one 256-node tile
  // per CTA measured 106 vs 77 us (per-CTA reduction and atomics)
  const int grid_u = 6 * std::max(1, std::min((n + 255) / 256, c->num_sms * 2));
  const int grid_a = shl::apply_grid(n, c->num_sms);
  const int grid_c = std::max(1, std::min(static_cast<int>((c->n_elem + 31) / 32), c->num_sms * 16));
  c->partials.ensure(sizeof(double) *
                     std::max<size_t>({static_cast<size_t>(std::max(grid_a, 6 * c->num_sms)) * 6,
                                       static_cast<size_t>((n + 31) / 32) * 6,  // per-tile p.q / r.z
                                       static_cast<size_t>(grid_u) * 2,
                                       static_cast<size_t>(grid_c) * 21,
                                       static_cast<size_t>(c->n_bricks) * 6, 64}));
  c->state.ensure(sizeof(shl::PcgState));
  c->cout.ensure(36 * sizeof(double));

  double T[144], W[144];
  element_loads(K0, r, T, W);
  // ridge 1e-11 * mean|diag A| (fem.hpp:339-341): every K0 diagonal entry is
  // equal, so mean diag = K0[0] * (8 sum beta) / n_nodes
  // Ridge of the reference's singular-system path (fem.hpp:337-343): 1e-11 *
  // mean|diag A| in FP64.  With FP32 vectors the floating components' near-null
  // modes stall the multigrid-preconditioned iteration at that scale (seed 4 at
  // 128^3: breakdown at residual 1e-2), so the FP32-storage modes use 1e-8,
  // still FP32-resolution-small: C^H moves by < 1e-7 relative (tests compare
  // against FP64).  Every K0 diagonal entry is equal, so
  // mean diag = K0[0] * (8 sum beta) / n_nodes.
  // the operator PCG solves uses the Krylov type's ridge; the preconditioner
  // (block Jacobi / V-cycle) the ridge of its own storage type
  const double diag_mean = n > 0 ? std::fabs(K0[0]) * 8.0 * c->beta_sum / double(n) : 0.0;
  const double ridge_op = diag_mean * (sizeof(TV) == 8 ? 1e-11 : 1e-8);
  const double ridge = diag_mean * (sizeof(TZ) == 8 ? 1e-11 : 1e-8);
  CK(cudaEventRecord(c->ev[3], c->stream));
  shl::ElementConstLease const_lease(K0, W, T, r, c->stream);
  CK(cudaMemsetAsync(x, 0, nX * sizeof(TXS), c->stream));
  CK(cudaMemsetAsync(p, 0, 2 * nV * sizeof(TV), c->stream));
  CK(cudaMemsetAsync(z, 0, nV * sizeof(TZ), c->stream));
  CK(cudaEventRecord(c->ev[8], c->stream));
  shl::launch_setup<TX, TZ>(c->node_list.as<int>(), n, ld, r, c->beta64.as<double>(), ridge, rv,
                            dinv, c->stream);
  CK(cudaEventRecord(c->ev[9], c->stream));
  Vcycle<TX, TZ, TZ> vc{c, gmg_params()};
  vc.zout = z;
  vc.s = c->stream;
  if (vc.gp.nu <= 0) vc.gp.nu = sizeof(TV) == 8 ? 1 : 2;
  if (use_gmg) {
    {
      NvtxRange nr("shellular: multigrid setup (Galerkin levels)");
      vc.L = gmg_setup<TZ>(c, vc.gp, static_cast<TZ>(ridge));
    }
    if (vc.L == 0) throw ShlError(SHL_VALIDATION, "multigrid needs r divisible by 2 with r/2 >= 8");
    c->gmg0.ensure(static_cast<size_t>(3) * nV * sizeof(TZ));
    CK(cudaMemsetAsync(c->gmg0.p, 0, static_cast<size_t>(3) * nV * sizeof(TZ), c->stream));
    const TZ* beta_v = sizeof(TZ) == 8 ? reinterpret_cast<const TZ*>(c->beta64.p)
                                       : reinterpret_cast<const TZ*>(c->beta32.p);
    vc.view.push_back({c->node_list.as<int>(), c->node_map.as<int>(), beta_v, nullptr, dinv, r, n, n,
                       static_cast<TZ>(ridge)});
    vc.view.back().bricks = c->brick_view();
    TZ* g0 = c->gmg0.as<TZ>();
    vc.b.push_back(nullptr);
    vc.xa.push_back(g0);
    vc.xb.push_back(g0 + nV);
    vc.res.push_back(g0 + 2 * nV);
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
    vc.partials = c->partials.as<double>();
  }
  shl::PcgState hs{};
  hs.tol = opt.tol;
  hs.ridge = ridge_op;
  hs.max_iter = opt.max_iter > 0 ? opt.max_iter : 20 * r + 2000;
  std::memcpy(c->hstate, &hs, sizeof(hs));
  c->h2d += sizeof(hs) + 576 * 12 + 144 * 16;  // state + element constants
  CK(cudaMemcpyAsync(c->state.p, c->hstate, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  CK(cudaEventRecord(c->ev[4], c->stream));

  shl::PcgState* dst = c->state.as<shl::PcgState>();
  const TV* beta_apply = sizeof(TV) == 8 ? reinterpret_cast<const TV*>(c->beta64.p)
                                         : reinterpret_cast<const TV*>(c->beta32.p);
  shl::UpdateArgs<TX, TV, TZ, TXS> ua{x, rv, p, q, z, dinv, c->partials.as<double>(), dst, n, ld, 1,
                                nullptr, 0, use_gmg ? 1 : 0, use_gmg ? vc.xa[0] : nullptr,
                                static_cast<TZ>(vc.gp.omega)};
  shl::ApplyArgs<TV, TZ> aa{c->node_list.as<int>(), c->node_map.as<int>(), beta_apply, z, p, q,
                        c->partials.as<double>(), dst, r, n, ld, n, 0, r, nullptr, 0};
  aa.bricks = c->brick_view();
  vc.st = dst;
  // z = M r: block Jacobi inside the update kernel, or the V-cycle
  auto precondition = [&](int init) {
    if (use_gmg) vc.level(0, rv, init);
  };
  // z0 = M b, then w0 = A z0, p0 = z0, q0 = w0, alpha0
  shl::launch_update<TX, TV, TZ>(ua, grid_u, c->stream);
  precondition(1);
  shl::launch_apply<TV, TZ>(aa, grid_a, c->stream);
  ua.init = 0;
  // kernels per update + apply (the brick apply is followed by its p.q sum)
  const int it_kernels = 1 + (aa.bricks.nab > 0 ? 2 : 1);
  int64_t launches = 2 + it_kernels;
  int check = opt.check_every > 0 ? opt.check_every : (n < 200000 ? 16 : 32);
#ifdef SHL_DEV_TRACE  // dev build only: per-iteration scalars on stderr
  constexpr bool trace = true;
  check = 1;
#else
  constexpr bool trace = false;
#endif
  double apply_ms = 0.0, update_ms = 0.0;
  int64_t apply_launches = 0;
  int64_t issued = 0;
  // Steady state: the iteration (update, V-cycle, apply: ~30 launches with
  // multigrid) is captured once into a CUDA graph of kGraphIters iterations
  // and replayed, which removes the per-kernel launch gaps of the small
  // coarse-level kernels.  Profiling (shl_set_profiling: per-launch events,
  // per-kernel ncu launch lists) and tracing keep direct launches.
  constexpr int kGraphIters = 4;
  const bool use_graph = !c->profiling && !trace && check % kGraphIters == 0;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;  // kernel launches per graph replay
  // The whole solve loop as ONE graph launch when the driver supports
  // conditional nodes: a WHILE node whose body is kGraphIters iterations plus a
  // one-thread kernel setting the condition to !stop.  No host polls during the
  // solve (host scheduling delays no longer idle the design's stream) and at
  // most kGraphIters-1 no-op iterations after convergence.
  bool use_while = false;
  if (use_graph) {
    // recorded on a side stream: capture + instantiation (host work) overlap the
    // device executing the setup and first iteration already queued on c->stream
    const int64_t before = launches + vc.launches;
    const cudaStream_t cs = c->cap_stream;
    cudaGraph_t graph = nullptr;
    {
      cudaGraph_t g = nullptr;
      CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h;
      cudaGraphNode_t wnode;
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess) {
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        if (cudaGraphAddNode(&wnode, g, nullptr, 0, &cp) == cudaSuccess) {
          cudaGraph_t body = cp.conditional.phGraph_out[0];
          CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
          vc.s = cs;
          for (int it = 0; it < kGraphIters; ++it) {
            shl::launch_update<TX, TV, TZ>(ua, grid_u, cs);
            precondition(0);
            shl::launch_apply<TV, TZ>(aa, grid_a, cs);
            launches += it_kernels;
          }
          shl::launch_set_while(h, dst, cs);
          vc.s = c->stream;
          CK(cudaStreamEndCapture(cs, &body));
          use_while = true;
          graph = g;
        }
      }
      if (!use_while) {
        cudaGetLastError();  // clear a refused conditional node; fall back to host polls
        cudaGraphDestroy(g);
      }
    }
    if (!use_while) {
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      vc.s = cs;
      for (int it = 0; it < kGraphIters; ++it) {
        shl::launch_update<TX, TV, TZ>(ua, grid_u, cs);
        precondition(0);
        shl::launch_apply<TV, TZ>(aa, grid_a, cs);
        launches += it_kernels;
      }
      vc.s = c->stream;
      CK(cudaStreamEndCapture(cs, &graph));
    }
    CK(cudaGraphInstantiate(&gexec, graph, 0));
    CK(cudaGraphDestroy(graph));
    graph_launches = launches + vc.launches - before;
    launches -= it_kernels * kGraphIters;  // counted per replay below
    vc.launches -= graph_launches - it_kernels * kGraphIters;
  }
  struct GraphGuard {
    cudaGraphExec_t g;
    ~GraphGuard() {
      if (g) cudaGraphExecDestroy(g);
    }
  } graph_guard{gexec};
  NvtxRange pcg_range("shellular: PCG iterations");
  if (use_while) {
    CK(cudaGraphLaunch(gexec, c->stream));
    CK(cudaMemcpyAsync(c->hstate, c->state.p, sizeof(shl::PcgState), cudaMemcpyDeviceToHost, c->stream));
    c->d2h += sizeof(shl::PcgState);
    c->sync();
    const int trips = (c->hstate->it + kGraphIters - 1) / kGraphIters;
    launches += static_cast<int64_t>(std::max(trips, 1)) * (graph_launches + 1);
    issued = c->hstate->it;
  }
  for (;;) {
    if (use_while) break;  // the device loop ran the whole solve
    if (use_graph) {
      for (int it = 0; it < check; it += kGraphIters) {
        CK(cudaGraphLaunch(gexec, c->stream));
        launches += graph_launches;
        issued += kGraphIters;
      }
    } else {
      for (int it = 0; it < check; ++it) {
        if (c->profiling) {
          const size_t need = static_cast<size_t>(3 * (issued + 1));
          while (c->prof_ev.size() < need) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            c->prof_ev.push_back(e);
          }
          CK(cudaEventRecord(c->prof_ev[3 * issued], c->stream));
          shl::launch_update<TX, TV, TZ>(ua, grid_u, c->stream);
          precondition(0);
          CK(cudaEventRecord(c->prof_ev[3 * issued + 1], c->stream));
          shl::launch_apply<TV, TZ>(aa, grid_a, c->stream);
          CK(cudaEventRecord(c->prof_ev[3 * issued + 2], c->stream));
        } else {
          shl::launch_update<TX, TV, TZ>(ua, grid_u, c->stream);
          precondition(0);
          shl::launch_apply<TV, TZ>(aa, grid_a, c->stream);
        }
        ++issued;
        launches += it_kernels;
      }
    }
    CK(cudaGetLastError());
    c->d2h += sizeof(shl::PcgState);
    CK(cudaMemcpyAsync(c->hstate, c->state.p, sizeof(shl::PcgState), cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    if (trace) {
      const shl::PcgState& h = *c->hstate;
      std::fprintf(stderr, "it %3d", h.it);
      for (int q = 0; q < 6; ++q)
        std::fprintf(stderr, " | r %.2e g %+.2e pAp %+.2e", h.bnorm[q] > 0 ? std::sqrt(h.rr[q]) / h.bnorm[q] : 0.0,
                     h.gamma[q], h.pap[q]);
      std::fprintf(stderr, "\n");
    }
    if (c->hstate->stop) break;
  }
  if (c->profiling) {
    // per-launch device time of the iterations that did work (later launches exit early)
    const int64_t real = std::min<int64_t>(issued, c->hstate->it);
    for (int64_t i = 0; i < real; ++i) {
      float tu = 0, ta = 0;
      CK(cudaEventElapsedTime(&tu, c->prof_ev[3 * i], c->prof_ev[3 * i + 1]));
      CK(cudaEventElapsedTime(&ta, c->prof_ev[3 * i + 1], c->prof_ev[3 * i + 2]));
      update_ms += tu;
      apply_ms += ta;
    }
    apply_launches = real;
  }
  launches += vc.launches;
  CK(cudaEventRecord(c->ev[5], c->stream));
  const shl::PcgState& fin = *c->hstate;
  if (fin.error) {
    double worst = 0.0;
    for (int q = 0; q < 6; ++q)
      if (fin.bnorm[q] > 0) worst = std::max(worst, std::sqrt(fin.rr[q]) / fin.bnorm[q]);
    char buf[200];
    std::snprintf(buf, sizeof(buf),
                  "grid CG: operator lost positive definiteness (iteration %d, max relative residual %.3g)",
                  fin.it, worst);
    throw ShlError(SHL_SOLVER, buf);
  }
  const bool converged = fin.all_done != 0;
  if (!converged) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "grid CG did not reach tolerance %g in %d iterations", opt.tol,
                  fin.max_iter);
    throw ShlError(SHL_SOLVER, buf);
  }
  shl::ChomArgs<TXS> ca{c->elem_list.as<int>(), c->node_map.as<int>(), c->beta64.as<double>(), x,
                       c->partials.as<double>(), c->cout.as<double>(), dst,
                       static_cast<int>(c->n_elem), r, ld, 0, r, 0};
  {
    NvtxRange nr("shellular: C^H reduction");
    shl::launch_chom<TXS>(ca, grid_c, c->stream);
  }
  launches += 1;
  CK(cudaGetLastError());
  c->d2h += 36 * sizeof(double);
  CK(cudaMemcpyAsync(c->hC, c->cout.p, 36 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->ev[6], c->stream));
  c->sync();
  std::memcpy(C_out, c->hC, 36 * sizeof(double));
  c->launches += launches;
  if (st) {
    // t_RHS: right-hand sides + block-Jacobi inverse (setup kernel); t_AS: the
    // rest of the setup (element constants, workspaces, multigrid Galerkin
    // hierarchy) -- the matrix-free solve assembles no global matrix
    st->t_RHS = c->ms(8, 9);
    st->t_AS = c->ms(3, 4) - st->t_RHS;
    st->t_solve = c->ms(4, 5);
    st->t_C = c->ms(5, 6);
    for (int s = 0; s < 6; ++s) st->iterations[s] = fin.iters[s];
    st->converged = converged;
    st->precision = prec;
    st->apply_ms = apply_ms;
    st->update_ms = update_ms;
    st->apply_launches = apply_launches;
    st->gmg_levels = use_gmg ? vc.L + 1 : 0;
  }
}

bool is_breakdown(const ShlError& e) {
  return e.code == SHL_SOLVER && std::string(e.what()).find("positive definiteness") != std::string::npos;
}

void solve_dispatch_once(shl_ctx* c, const double* K0, const shl_solve_options& opt, double* C_out,
                         shl_stats* st) {
  const int prec = resolve_precision(opt);
  const int r = c->r;
  const bool gmg = opt.preconditioner == SHL_PRECOND_GMG ||
                   (opt.preconditioner == SHL_PRECOND_AUTO && r % 2 == 0 && r / 2 >= gmg_params().min_r);
  switch (prec) {
    case SHL_PREC_FP64: run_solve<double, double, double>(c, K0, opt, C_out, st, prec, gmg); break;
    case SHL_PREC_MIXED: {
      // Multigrid: FP32 V-cycle and z, FP64 Krylov vectors and FP64-accumulated
      // operator (TV = double, TZ = float).  With an FP32 operator, rounding of
      // A p swamps the ridge-sized curvature of a voxel shell's hinge modes
      // (elements sharing only an edge or a corner) and p^T A p loses its sign
      // on ~1 in 16 designs at 128^3; the FP64 operator keeps the reference's
      // 1e-11 ridge and costs ~3% per design (128^3 sweep).
      if (!gmg)
        run_solve<double, float, float>(c, K0, opt, C_out, st, prec, gmg);
      else
        run_solve<double, double, float, float>(c, K0, opt, C_out, st, prec, gmg);
      break;
    }
    default: run_solve<float, float, float>(c, K0, opt, C_out, st, prec, gmg); break;
  }
}

// A multigrid-preconditioned solve that breaks down (p^T A p <= 0: the FP32
// V-cycle lost definiteness on an unusual design) is redone with the
// reference's block-Jacobi PCG rather than failing the design; explicit
// SHL_PRECOND_GMG requests are not retried.
void solve_dispatch(shl_ctx* c, const double* K0, const shl_solve_options& opt, double* C_out,
                    shl_stats* st) {
  if (opt.preconditioner != SHL_PRECOND_AUTO) return solve_dispatch_once(c, K0, opt, C_out, st);
  try {
    solve_dispatch_once(c, K0, opt, C_out, st);
  } catch (const ShlError& e) {
    if (!is_breakdown(e)) throw;
    shl_solve_options jo = opt;
    jo.preconditioner = SHL_PRECOND_JACOBI;
    solve_dispatch_once(c, K0, jo, C_out, st);
    if (st) st->precond_fallback = 1;
  }
}

void fill_mesh_stats(shl_ctx* c, shl_stats* st) {
  if (!st) return;
  st->n_surface = c->n_surface;
  st->n_elements = c->n_elem;
  st->n_nodes = c->n_nodes;
  st->n_tiles = 0;
  st->full_fallback = c->full_fallback;
  st->n_components = c->n_components;
  st->n_floating = c->n_floating;
  st->norm = c->norm;
  st->volume_ratio = c->volume_ratio;
}

shl_solve_options default_opts(const shl_solve_options* o) {
  shl_solve_options d{};
  d.tol = 1e-9;
  d.max_iter = 0;
  d.precision = SHL_PREC_AUTO;
  d.check_every = 0;
  if (o) d = *o;
  if (!(d.tol > 0.0)) throw ShlError(SHL_VALIDATION, "solver tolerance must be positive");
  return d;
}

// homogenize's own checks (pipeline.hpp:64-65: mat.validate, sp.validate) + K0
void validate_inputs(const shl_design* design, const shl_shell_params* sp, const shl_material* mat,
                     int r, double* K0) {
  if (!design || !sp || !mat) throw ShlError(SHL_VALIDATION, "null argument");
  shl::element_stiffness(mat->youngs, mat->poisson, 1.0 / std::max(r, 1), K0);  // mat.validate
  if (!(sp->sharpness > 0.0)) throw ShlError(SHL_VALIDATION, "sharpness must be positive");
  if (!(sp->floor_ratio > 0.0 && sp->floor_ratio < 1.0))
    throw ShlError(SHL_VALIDATION, "floor must lie in (0, 1)");
  if (sp->expand_layers < 0) throw ShlError(SHL_VALIDATION, "expand_layers must be >= 0");
}

void homogenize_one(shl_ctx* c, const shl_design* design, const shl_shell_params* sp,
                    const shl_material* mat, int r, const shl_solve_options* o, double* C_out,
                    shl_stats* st, std::future<FieldInputs>* prepared = nullptr) {
  if (!C_out) throw ShlError(SHL_VALIDATION, "null argument");
  const shl_solve_options opt = default_opts(o);
  double K0[576];
  validate_inputs(design, sp, mat, r, K0);
  const int64_t l0 = c->launches, h0 = c->h2d, d0 = c->d2h;
  // (the batch path prepares the host tables of a lane's next design while the
  // current one runs on the GPU: `prepared` holds them, or their exception)
  NvtxRange design_range("shellular: homogenize");
  FieldInputs fin = tagged("field", [&] {
    return prepared && prepared->valid() ? prepared->get() : prepare_field(shl::HostDesign::from_abi(*design), r);
  });
  CK(cudaEventRecord(c->ev[0], c->stream));
  tagged("field", [&] {
    NvtxRange nr("shellular: field");
    run_field(c, fin);
    return 0;
  });
  CK(cudaEventRecord(c->ev[1], c->stream));
  // The norm comes back with the mesh stage's count readback instead of its
  // own host wait (the mesh kernels read it on the device); a degenerate
  // design (norm 0) still fails with the field-stage error, before any solve.
  c->norm = 1.0;  // placeholder for run_mesh's host-side check
  tagged("mesh", [&] {
    NvtxRange nr("shellular: mesh + topology");
    run_mesh(c, *sp);
    return 0;
  });
  std::memcpy(&c->norm, &c->hmisc->norm_bits, sizeof(double));
  if (c->norm == 0.0) throw ShlError(SHL_DEGENERATE, "field: design is degenerate (norm = 0)");
  CK(cudaEventRecord(c->ev[2], c->stream));
  tagged("solve", [&] {
    NvtxRange nr("shellular: solve + C^H");
    solve_dispatch(c, K0, opt, C_out, st);
    return 0;
  });
  c->sync();
  if (st) {
    st->t_field = c->ms(0, 1);
    st->t_mesh = c->ms(1, 7);  // classify, dilation, completion, corners, beta
    st->t_PBC = c->ms(7, 2);   // components + node numbering (the periodic pairing is implicit on the torus)
    st->t_fwd = c->ms(0, 6);
    fill_mesh_stats(c, st);
    st->kernel_launches = c->launches - l0;
    st->h2d_bytes = c->h2d - h0;
    st->d2h_bytes = c->d2h - d0;
  }
}

}  // namespace host
}  // namespace shl

using namespace shl::host;


// =============================== C ABI =======================================
extern "C" {

int shl_ctx_create(int device, shl_ctx** out) {
  if (!out) return SHL_VALIDATION;
  *out = nullptr;
  auto c = std::make_unique<shl_ctx>();
  c->device = device;
  int rc = guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    // keep freed stream-ordered workspace memory in the device pool (no trim at syncs)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    CK(cudaEventCreateWithFlags(&c->sync_ev, cudaEventBlockingSync | cudaEventDisableTiming));
    CK(cudaMallocHost(&c->hmisc, sizeof(Misc)));
    CK(cudaMallocHost(&c->hlevels, 64 * sizeof(int)));
    CK(cudaMallocHost(&c->hstate, sizeof(shl::PcgState)));
    CK(cudaMallocHost(&c->hC, 36 * sizeof(double)));
  });
  if (rc != SHL_OK) return rc;
  *out = c.release();
  return SHL_OK;
}

void shl_ctx_destroy(shl_ctx* c) {
  if (!c) return;
  for (shl_ctx* l : c->lanes) shl_ctx_destroy(l);
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->nccl && c->nccl_deleter) c->nccl_deleter(c->nccl);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->sync_ev) cudaEventDestroy(c->sync_ev);
  for (auto& e : c->prof_ev)
    if (e) cudaEventDestroy(e);
  if (c->hmisc) cudaFreeHost(c->hmisc);
  if (c->hlevels) cudaFreeHost(c->hlevels);
  if (c->hstate) cudaFreeHost(c->hstate);
  if (c->hC) cudaFreeHost(c->hC);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

const char* shl_last_error(const shl_ctx* c) {
  return c ? c->err.c_str() : g_thread_error.c_str();
}

int shl_set_profiling(shl_ctx* c, int on) {
  if (!c) return SHL_VALIDATION;
  c->profiling = on != 0;
  return SHL_OK;
}

int shl_sample_grid(shl_ctx* c, const shl_design* design, int r, double* centres, double* corners,
                    double* norm) {
  if (!c || !design) return SHL_VALIDATION;
  return guarded(c, [&] {
    run_field(c, prepare_field(shl::HostDesign::from_abi(*design), r));
    read_norm(c);
    const size_t n3 = static_cast<size_t>(r) * r * r;
    if (centres)
      CK(cudaMemcpy(centres, c->centres.p, n3 * sizeof(double), cudaMemcpyDeviceToHost));
    if (corners) {
      std::vector<double> u(n3);
      CK(cudaMemcpy(u.data(), c->corners.p, n3 * sizeof(double), cudaMemcpyDeviceToHost));
      const int r1 = r + 1;
      for (int k = 0; k < r1; ++k)
        for (int j = 0; j < r1; ++j)
          for (int i = 0; i < r1; ++i)
            corners[(static_cast<size_t>(k) * r1 + j) * r1 + i] =
                u[(static_cast<size_t>(k % r) * r + j % r) * r + i % r];
    }
    if (norm) *norm = c->norm;
  });
}

int shl_load_grid(shl_ctx* c, int r, const double* centres, const double* corners, double norm) {
  if (!c || !centres || !corners) return SHL_VALIDATION;
  return guarded(c, [&] {
    require_r(r);
    alloc_grid(c, r);
    c->grid_ready = c->mesh_ready = false;
    const size_t n3 = static_cast<size_t>(r) * r * r;
    std::vector<double> u(n3);
    const int r1 = r + 1;
    for (int k = 0; k < r; ++k)
      for (int j = 0; j < r; ++j)
        for (int i = 0; i < r; ++i)
          u[(static_cast<size_t>(k) * r + j) * r + i] = corners[(static_cast<size_t>(k) * r1 + j) * r1 + i];
    CK(cudaMemcpy(c->centres.p, centres, n3 * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->corners.p, u.data(), n3 * sizeof(double), cudaMemcpyHostToDevice));
    Misc m{};
    std::memcpy(&m.norm_bits, &norm, sizeof(double));
    CK(cudaMemcpy(c->misc.p, &m, sizeof(Misc), cudaMemcpyHostToDevice));
    shl::launch_corner_signs(c->corners.as<double>(), c->csign.as<int8_t>(), r, c->stream);
    CK(cudaGetLastError());
    c->sync();
    c->norm = norm;
    c->grid_ready = true;
  });
}

int shl_classify_surface(shl_ctx* c, uint32_t* elements, int64_t* n_surface) {
  if (!c) return SHL_VALIDATION;
  return guarded(c, [&] {
    if (!c->grid_ready) throw ShlError(SHL_VALIDATION, "no resident grid");
    if (c->norm == 0.0)
      throw ShlError(SHL_DEGENERATE, "cannot classify surface elements of a degenerate field");
    const int r = c->r;
    const size_t n3 = static_cast<size_t>(r) * r * r;
    c->occ1.ensure(n3);
    Misc* dm = c->misc.as<Misc>();
    CK(cudaMemsetAsync(&dm->n_surface, 0, sizeof(int), c->stream));
    shl::launch_classify(c->csign.as<int8_t>(), c->occ1.as<uint8_t>(), r, &dm->n_surface, c->stream);
    std::vector<uint8_t> occ(n3);
    CK(cudaMemcpyAsync(occ.data(), c->occ1.p, n3, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    int64_t cnt = 0;
    for (size_t e = 0; e < n3; ++e)
      if (occ[e]) {
        if (elements) elements[cnt] = static_cast<uint32_t>(e);
        ++cnt;
      }
    if (n_surface) *n_surface = cnt;
    c->mesh_ready = false;
  });
}

int shl_build_reduced_mesh(shl_ctx* c, const shl_shell_params* sp, uint32_t* elements,
                           double* beta, int64_t* n_elements, int32_t* full_fallback) {
  if (!c || !sp) return SHL_VALIDATION;
  return guarded(c, [&] {
    run_mesh(c, *sp);
    const int r = c->r;
    const size_t n3 = static_cast<size_t>(r) * r * r;
    if (elements || beta) {
      std::vector<int> el(c->n_elem);
      if (c->n_elem)
        CK(cudaMemcpy(el.data(), c->elem_list.p, el.size() * sizeof(int), cudaMemcpyDeviceToHost));
      if (elements)
        for (size_t q = 0; q < el.size(); ++q) elements[q] = static_cast<uint32_t>(el[q]);
      if (beta) {
        std::vector<double> b(n3);
        CK(cudaMemcpy(b.data(), c->beta64.p, n3 * sizeof(double), cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < el.size(); ++q) beta[q] = b[el[q]];
      }
    }
    if (n_elements) *n_elements = c->n_elem;
    if (full_fallback) *full_fallback = c->full_fallback;
  });
}

int shl_grid_solve(shl_ctx* c, int r, const double* beta, const double* K0,
                   const shl_solve_options* o, double* C_out, shl_stats* st) {
  if (!c || !beta || !K0 || !C_out) return SHL_VALIDATION;
  return guarded(c, [&] {
    require_r(r);
    const shl_solve_options opt = default_opts(o);
    const size_t n3 = static_cast<size_t>(r) * r * r;
    for (size_t e = 0; e < n3; ++e)
      if (!(beta[e] >= 0.0)) throw ShlError(SHL_VALIDATION, "beta must be >= 0");
    const int64_t l0 = c->launches;
    CK(cudaEventRecord(c->ev[0], c->stream));
    alloc_grid(c, r);
    c->grid_ready = false;
    c->occ0.ensure(n3);
    c->beta64.ensure(n3 * sizeof(double));
    c->beta32.ensure(n3 * sizeof(float));
    c->elem_flag.ensure(n3 * sizeof(int));
    c->beta_partials.ensure(((n3 + 255) / 256) * 2 * sizeof(double));
    CK(cudaMemsetAsync(c->beta_partials.p, 0, ((n3 + 255) / 256) * 2 * sizeof(double), c->stream));
    CK(cudaMemcpyAsync(c->beta64.p, beta, n3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    shl::launch_beta_from_dense(c->beta64.as<double>(), r, c->beta32.as<float>(),
                                c->elem_flag.as<int>(), c->occ0.as<uint8_t>(), c->stream);
    c->launches += 1;
    CK(cudaEventRecord(c->ev[1], c->stream));
    CK(cudaEventRecord(c->ev[2], c->stream));
    build_topology(c);
    double s = 0.0;
    for (size_t e = 0; e < n3; ++e) s += beta[e];
    c->beta_sum = s;
    c->volume_ratio = s / double(n3);
    c->n_surface = 0;
    c->full_fallback = c->n_elem == static_cast<int64_t>(n3);
    c->mesh_ready = true;
    if (c->n_elem == 0) throw ShlError(SHL_DEGENERATE, "no elements with beta > 0");
    solve_dispatch(c, K0, opt, C_out, st);
    if (st) {
      st->t_field = 0.0;
      st->t_mesh = c->ms(0, 2);
      st->t_PBC = 0.0;
      st->t_fwd = c->ms(0, 6);
      fill_mesh_stats(c, st);
      st->kernel_launches = c->launches - l0;
    }
  });
}

int shl_solve_mesh(shl_ctx* c, const double* K0, const shl_solve_options* o, double* C_out,
                   shl_stats* st) {
  if (!c || !K0 || !C_out) return SHL_VALIDATION;
  return guarded(c, [&] {
    if (!c->mesh_ready) throw ShlError(SHL_VALIDATION, "no resident mesh: call shl_build_reduced_mesh");
    const shl_solve_options opt = default_opts(o);
    const int64_t l0 = c->launches;
    solve_dispatch(c, K0, opt, C_out, st);
    if (st) {
      st->t_fwd = c->ms(3, 6);
      fill_mesh_stats(c, st);
      st->kernel_launches = c->launches - l0;
    }
  });
}

int shl_homogenize(shl_ctx* c, const shl_design* design, const shl_shell_params* sp,
                   const shl_material* mat, int r, const shl_solve_options* opt, double* C_out,
                   shl_stats* st) {
  if (!c) return SHL_VALIDATION;
  if (st) std::memset(st, 0, sizeof(*st));
  return guarded(c, [&] { homogenize_one(c, design, sp, mat, r, opt, C_out, st); });
}

int shl_set_batch_lanes(shl_ctx* c, int lanes) {
  if (!c || lanes < 1 || lanes > 16) return SHL_VALIDATION;
  c->n_lanes = lanes;
  return SHL_OK;
}

// Designs are independent, so a batch keeps several in flight: lane 0 is this
// context, lanes 1.. are sub-contexts on the same device (own stream, own
// workspaces, created once), each driven by a host thread pulling the next
// design index from a shared counter.  One design's latency-bound phases
// (coarse multigrid levels, host polls, graph launch gaps) then overlap
// another's bandwidth-bound kernels.
int shl_homogenize_batch(shl_ctx* c, int n, const shl_design* designs, const shl_shell_params* sp,
                         const shl_material* mat, int r, const shl_solve_options* opt,
                         double* C_out, shl_stats* stats, int32_t* status) {
  if (!c || n < 0 || (n > 0 && (!designs || !C_out))) return SHL_VALIDATION;
  const int L = std::max(1, std::min(c->n_lanes, n));
  while (static_cast<int>(c->lanes.size()) < L - 1) {
    shl_ctx* sub = nullptr;
    const int rc = shl_ctx_create(c->device, &sub);
    if (rc != SHL_OK) return rc;
    c->lanes.push_back(sub);
  }
  // Lane 0 runs at the greatest stream priority, the other lanes at the
  // default: whenever CTA slots free up the block scheduler serves lane 0 first
  // and the others fill the gaps.  With equal priorities the lanes' phases
  // drifted into lockstep contention on about one run in three (one lane's
  // setup kernels queued behind the other's resident solve kernels: 26 vs 35
  // designs/s at 2 lanes); with lane 0 prioritised 2 lanes measure 33.5-34.4
  // designs/s on most runs (not on every box).
  if (L > 1 && !c->high_priority) {
    const int rc = shl::host::guarded(c, [&] {
      int least = 0, greatest = 0;
      CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      // new streams first: on failure the context keeps its working streams
      cudaStream_t s0 = nullptr, s1 = nullptr;
      CK(cudaStreamCreateWithPriority(&s0, cudaStreamNonBlocking, greatest));
      if (cudaStreamCreateWithPriority(&s1, cudaStreamNonBlocking, greatest) != cudaSuccess) {
        cudaStreamDestroy(s0);
        throw ShlError(SHL_CUDA, "cudaStreamCreateWithPriority failed");
      }
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaStreamSynchronize(c->cap_stream));
      CK(cudaStreamDestroy(c->stream));
      CK(cudaStreamDestroy(c->cap_stream));
      c->stream = s0;
      c->cap_stream = s1;
      c->high_priority = true;
    });
    if (rc != SHL_OK) return rc;
  }
  std::atomic<int> next{0};
  std::atomic<int> device_failed{0};
  std::string device_msg;
  // Each lane claims its next design one step ahead and builds that design's
  // host inputs (symmetry expansion, glibc cosine tables: ~1 ms at 128^3) on a
  // helper thread while the current design runs, so the GPU does not wait for
  // the host between designs.
  auto prepare_async = [&](int k) {
    return std::async(std::launch::async,
                      [&designs, r, k] { return prepare_field(shl::HostDesign::from_abi(designs[k]), r); });
  };
  auto work = [&](shl_ctx* lc, int lane) {
    cudaSetDevice(c->device);
    lc->profiling = c->profiling;
    int i = next.fetch_add(1);
    std::future<FieldInputs> pre;
    if (i < n) pre = prepare_async(i);
    while (i < n && !device_failed.load()) {
      const int j = next.fetch_add(1);
      std::future<FieldInputs> pre_next;
      if (j < n) pre_next = prepare_async(j);
      shl_stats* st = stats ? stats + i : nullptr;
      if (st) std::memset(st, 0, sizeof(*st));
      const int rc =
          guarded(lc, [&] { homogenize_one(lc, designs + i, sp, mat, r, opt, C_out + 36 * i, st, &pre); });
      if (st) st->lane = lane;
      if (status) status[i] = rc;
      if (rc == SHL_CUDA && !device_failed.exchange(1)) device_msg = lc->err;
      i = j;
      pre = std::move(pre_next);
    }
    // a design claimed but not run (device failure): report it
    if (i < n && status) status[i] = SHL_CUDA;
  };
  std::vector<std::thread> threads;
  for (int l = 1; l < L; ++l) threads.emplace_back(work, c->lanes[l - 1], l);
  work(c, 0);
  for (auto& t : threads) t.join();
  if (device_failed.load()) {
    c->err = device_msg;
    g_thread_error = device_msg;
    return SHL_CUDA;
  }
  return SHL_OK;
}

int shl_element_stiffness(const shl_material* mat, double edge, double* K) {
  if (!mat || !K) return SHL_VALIDATION;
  return guarded(nullptr, [&] { shl::element_stiffness(mat->youngs, mat->poisson, edge, K); });
}

int shl_random_design(int symmetry, int n_pre, int K, double lo, double hi, uint64_t seed,
                      double* positions, int32_t* signs, double* weights) {
  return guarded(nullptr, [&] {
    shl::HostDesign d = shl::random_design(symmetry, n_pre, K, lo, hi, seed);
    std::copy(d.pos.begin(), d.pos.end(), positions);
    std::copy(d.sign.begin(), d.sign.end(), signs);
    std::copy(d.weights.begin(), d.weights.end(), weights);
  });
}

int shl_expand_symmetry(const shl_design* design, double* positions_out, int32_t* signs_out,
                        int32_t* n_out) {
  if (!design) return SHL_VALIDATION;
  return guarded(nullptr, [&] {
    shl::HostDesign e = shl::HostDesign::from_abi(*design).expanded();
    std::copy(e.pos.begin(), e.pos.end(), positions_out);
    std::copy(e.sign.begin(), e.sign.end(), signs_out);
    if (n_out) *n_out = static_cast<int32_t>(e.sign.size());
  });
}

}  // extern "C"
