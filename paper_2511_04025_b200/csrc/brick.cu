// brick.cu -- level-0 operator kernels on shared-memory-staged bricks (sm_100a).
//
// The matrix-free masked operator of the reference's GridSolver::apply
// (grid_solver.hpp:154-176: y_n = sum_e beta_e K0 u_e, node 0 pinned) applied
// brick by brick.  Level-0 node ids are numbered brick-major (voxel.cu
// brick_* kernels): the torus is cut into 8x4x4-node bricks, each active brick
// owns a contiguous id range [bstart[t], bstart[t+1]).  One CTA per active brick
//   1. stages the node map of the brick + 1-node halo (10x6x6 = 360
//      positions) and beta of its 9x5x5 elements in shared memory (cp.async),
//   2. stages the 18 components (3 dof x 6 load cases) of the input vector at
//      every staged position in shared memory (cp.async, bank-swizzled rows),
//   3. gives each active node of the brick one thread, which builds the 27
//      neighbour blocks S_m = sum_e beta_e K0[a(n,e), b(m,e)] and applies them
//      to all six load cases from shared memory,
//   4. runs the caller's epilogue (PCG direction update, smoother or
//      residual) on the node's own coalesced rows, and reduces its dot
//      products per brick (fixed order -> reproducible).
// The dependent map -> vector load chain of a per-node gather becomes two
// bulk phases per brick; the arithmetic reads shared memory only.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "internal.h"
#include "pcg_common.cuh"
#include "stencil_patterns.h"

namespace shl {

// this translation unit's copy of K0 (uploaded with the solver's element
// constants, ElementConstLease in solver.cu)
__constant__ double c_bK0d[576];
__constant__ float c_bK0f[576];
// FP32 stencil coefficients coef_m(c,d) = K0[3 a0(m) + c][3 b0(m) + d] (stencil_patterns.h)
__constant__ float c_bcoeff[243];

namespace {

template <typename T>
__device__ __forceinline__ T k0(int i);
template <>
__device__ __forceinline__ double k0<double>(int i) {
  return c_bK0d[i];
}
template <>
__device__ __forceinline__ float k0<float>(int i) {
  return c_bK0f[i];
}

constexpr int kBX = 8, kBY = 4, kBZ = 4;  // nodes per brick (must match voxel.cu)
constexpr int kRX = kBX + 2, kRY = kBY + 2, kRZ = kBZ + 2;
constexpr int kRegion = kRX * kRY * kRZ;  // 360 staged node positions (brick + 1-node halo)
constexpr int kEX = kBX + 1, kEY = kBY + 1, kEZ = kBZ + 1;
constexpr int kERegion = kEX * kEY * kEZ;  // 225 staged elements
constexpr int kNodes = kBX * kBY * kBZ;    // 128 nodes per brick
constexpr int kThreads = kNodes;           // one thread per brick node
constexpr int kWarps = kThreads / 32;

// Staged vector layout.  FP32 arithmetic reads [c][load-case pair][position]
// as float2 (packed FFMA2 over load-case pairs, one 64-bit word per pair); a
// position (lx, ly, lz) of the 10x6x6 region lives in row slot 4*ly + prow(lz)
// of 10 positions, so consecutive y rows sit 40 positions apart and the 2 rows
// of 8 nodes a half warp reads in a full brick plane fall on disjoint banks
// (with the packed 10-position row stride 2 of every 16 lanes collided).
// Planes 0-3 interleave in row slots 0..23, planes 4-5 in 24..45 (460
// positions instead of 360).  The FP64 operator's [q][position] layout stays
// packed (its smem footprint sets the CTAs per SM, and it is not bank-bound).
constexpr int kPhys = 460;
__device__ __forceinline__ int plane_base(int lz) { return kRX * ((lz & 3) + 24 * (lz >> 2)); }
constexpr int kRowStep = 4 * kRX;  // positions between staged rows ly and ly + 1 (swizzled)
template <bool kPairs>
__device__ __forceinline__ int stage_pos(int lx, int ly, int lz) {
  if constexpr (kPairs)
    return plane_base(lz) + kRowStep * ly + lx;
  else
    return lx + kRX * (ly + kRY * lz);
}
template <bool kPairs>
constexpr int stage_words() {
  return kPairs ? kPhys : kRegion;
}

template <typename TS, bool kPairs = (sizeof(TS) == 4)>
__device__ __forceinline__ int xs_index(int q, int pos) {
  if constexpr (kPairs)
    return (((q / 6) * 3 + (q % 6) / 2) * kPhys + pos) * 2 + (q & 1);
  else
    return q * kRegion + pos;
}

// v in [-r, 3r) -> [0, r)   (staged coordinates never leave that range for r >= 4)
__device__ __forceinline__ int wrap3(int v, int r) {
  v += v < 0 ? r : 0;
  v -= v >= r ? r : 0;
  v -= v >= r ? r : 0;
  return v;
}

// Shared memory of one CTA: the staged input vector, the element betas and the
// brick's node positions, and the reduction scratch.
template <typename TS, typename TB = TS>
struct alignas(16) BrickShared {  // (16: the float2 reads of the second buffer)
  TS xs[18 * stage_words<sizeof(TS) == 4 && sizeof(TB) == 4>()];  // [q][position], 0 where absent
  TB bs[kERegion];            // element betas of the region
  unsigned short pc[kNodes];  // region position of brick node first + i
};
template <typename TS, typename TB = TS>
struct BrickCta {
  BrickShared<TS, TB> buf;
  double red[kWarps * 6];
};
template <typename TS, typename TB = TS>
constexpr size_t brick_smem_bytes() {
  return sizeof(BrickCta<TS, TB>);
}

__device__ __forceinline__ void brick_origin(const BrickView& B, int t, int& x0, int& y0, int& z0) {
  const int b = __ldg(B.bcoord + t);
  x0 = (b % B.nbx) * kBX;
  y0 = ((b / B.nbx) % B.nby) * kBY;
  z0 = (b / (B.nbx * B.nby)) * kBZ;
}

// Neighbour table of the 27-point node stencil, grouped by how many elements a
// node shares with the neighbour (centre 8, faces 4, edges 2, corners 1):
// staged-region offset of the neighbour, and per shared element its offset in
// the staged beta region and the K0 block base (3a)*24 + 3b (a, b the corners
// of node and neighbour in that element).  The gather loops over neighbours at
// run time (uniform indices, K0 from the constant bank) so the kernel body is
// ~2 KB of code instead of a 90 KB unrolled stencil that thrashed the
// instruction cache.
struct NbEntry {
  int roff;
  int eoff[8];
  int kb[8];
};
__constant__ NbEntry c_nb[27];
constexpr int kNbFace = 1, kNbEdge = 7, kNbCorner = 19;  // class starts: centre [0,1), faces, edges, corners

template <int K, typename TS, typename TX = TS>
__device__ __forceinline__ void gather_class(TS (&y)[18], const TX* __restrict__ xs, const TS* __restrict__ bs,
                                             int pc, int ec, int m0, int m1) {
#pragma unroll 2
  for (int m = m0; m < m1; ++m) {
    TS Sm[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) Sm[q] = TS(0);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const TS bej = bs[ec + c_nb[m].eoff[j]];
      const int kb = c_nb[m].kb[j];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) Sm[c * 3 + d] = fma_t(bej, k0<TS>(kb + c * 24 + d), Sm[c * 3 + d]);
    }
    const TX* xn = xs + pc + c_nb[m].roff;
#pragma unroll
    for (int s = 0; s < 6; ++s) {  // (an FP32-staged vector widens exactly)
      const TS z0 = static_cast<TS>(xn[(0 * 6 + s) * kRegion]), z1 = static_cast<TS>(xn[(1 * 6 + s) * kRegion]),
               z2 = static_cast<TS>(xn[(2 * 6 + s) * kRegion]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        TS v = y[c * 6 + s];
        v = fma_t(Sm[c * 3 + 0], z0, v);
        v = fma_t(Sm[c * 3 + 1], z1, v);
        v = fma_t(Sm[c * 3 + 2], z2, v);
        y[c * 6 + s] = v;
      }
    }
  }
}

// The S-build through the stencil's sign structure (stencil_patterns.h): per
// neighbour the distinct signed beta sums (60 per node, 124 adds) times the
// 243 stencil coefficients, instead of 576 beta*K0 FMAs with 576 constants.
// Every index is a compile-time constant after unrolling.
__device__ __forceinline__ void stencil_block_f32(int m, const float (&be)[8], float (&Sm)[9]) {
  float P[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    if (p >= pat::npat(m)) break;
    float acc = be[pat::elem(m, 0)];  // the first sign of every pattern is +1
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      if (j >= pat::shared(m)) break;
      acc = pat::sign(m, p, j) > 0 ? acc + be[pat::elem(m, j)] : acc - be[pat::elem(m, j)];
    }
    P[p] = acc;
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) Sm[q] = c_bcoeff[m * 9 + q] * P[pat::pat_of(m, q)];
}

// FP32 operator: the stencil unrolled with the structured S-build and the
// application on packed FFMA2 over load-case pairs (one FFMA2 = two load cases).
__device__ __forceinline__ void brick_gather_f32(float (&y)[18], const float* __restrict__ xs,
                                                 const float* __restrict__ bs, int pxy, int lz, int ec) {
  float2 acc[9];  // [c][load-case pair]
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = make_float2(0.f, 0.f);
  float be[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;
    be[e] = bs[ec - oz * (kEX * kEY) - oy * kEX - ox];
  }
  const float2* __restrict__ x2 = reinterpret_cast<const float2*>(xs);
#pragma unroll
  for (int m = 0; m < 27; ++m) {
    const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = m / 9 - 1;
    float Sm[9];
    stencil_block_f32(m, be, Sm);
    const float2* xn = x2 + plane_base(lz + dz) + pxy + dy * kRowStep + dx;
#pragma unroll
    for (int sp = 0; sp < 3; ++sp) {
      const float2 z0 = xn[(0 * 3 + sp) * kPhys], z1 = xn[(1 * 3 + sp) * kPhys], z2 = xn[(2 * 3 + sp) * kPhys];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float2 v = acc[c * 3 + sp];
        v = __ffma2_rn(make_float2(Sm[c * 3 + 0], Sm[c * 3 + 0]), z0, v);
        v = __ffma2_rn(make_float2(Sm[c * 3 + 1], Sm[c * 3 + 1]), z1, v);
        v = __ffma2_rn(make_float2(Sm[c * 3 + 2], Sm[c * 3 + 2]), z2, v);
        acc[c * 3 + sp] = v;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int sp = 0; sp < 3; ++sp) {
      y[c * 6 + 2 * sp] = acc[c * 3 + sp].x;
      y[c * 6 + 2 * sp + 1] = acc[c * 3 + sp].y;
    }
}

// y (18, component-major q = c*6 + s) = sum over the 27 neighbours of S_m x_m,
// S_m = sum_e beta_e K0[a(n,e), b(m,e)] built from the staged element betas.
template <typename TS, typename TX = TS>
__device__ __forceinline__ void brick_gather(TS (&y)[18], const TX* __restrict__ xs, const TS* __restrict__ bs, int pc,
                                             int pxy, int lz, int ec) {
  if constexpr (sizeof(TS) == 4) {
    brick_gather_f32(y, xs, bs, pxy, lz, ec);
    return;
  }
#pragma unroll
  for (int q = 0; q < 18; ++q) y[q] = TS(0);
  gather_class<8, TS, TX>(y, xs, bs, pc, ec, 0, kNbFace);
  gather_class<4, TS, TX>(y, xs, bs, pc, ec, kNbFace, kNbEdge);
  gather_class<2, TS, TX>(y, xs, bs, pc, ec, kNbEdge, kNbCorner);
  gather_class<1, TS, TX>(y, xs, bs, pc, ec, kNbCorner, 27);
}

// Staging, split so that it pipelines across a CTA's bricks:
//   stage_ids   -- the node ids of the region positions this thread stages
//                  (plain loads into registers, consumed one brick later),
//   stage_issue -- cp.async of the element betas and of the 18 components at
//                  every region position into a brick buffer (absent
//                  positions zero-filled), and the brick's own node positions;
//                  one commit group per brick.
constexpr int kPer = (kRegion + kThreads - 1) / kThreads;  // 3 region positions per thread

__device__ __forceinline__ void stage_ids(int (&id)[kPer], const BrickView& B, int t, int r,
                                          const int* __restrict__ nmap) {
  int x0, y0, z0;
  brick_origin(B, t, x0, y0, z0);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int p = threadIdx.x + j * kThreads;
    id[j] = -1;
    if (p < kRegion) {
      const int lx = p % kRX, ly = (p / kRX) % kRY, lz = p / (kRX * kRY);
      const int gx = wrap3(x0 + lx - 1, r), gy = wrap3(y0 + ly - 1, r), gz = wrap3(z0 + lz - 1, r);
      id[j] = __ldg(nmap + (static_cast<size_t>(gz) * r + gy) * r + gx);
      SHL_DCHECK(id[j] < 0 || B.n_nodes == 0 || id[j] < B.n_nodes);
    }
  }
}

template <typename TS, typename TB>
__device__ __forceinline__ void stage_issue(BrickShared<TS, TB>& S, const BrickView& B, int t, int r,
                                            const int (&id)[kPer], const TB* __restrict__ beta,
                                            const TS* __restrict__ v) {
  constexpr bool kPairs = sizeof(TS) == 4 && sizeof(TB) == 4;
  int x0, y0, z0;
  brick_origin(B, t, x0, y0, z0);
  const int first = __ldg(B.bstart + t), last = __ldg(B.bstart + t + 1);
  SHL_DCHECK(t >= 0 && t < B.nab && first >= 0 && first <= last && last - first <= kNodes);
  for (int e = threadIdx.x; e < kERegion; e += kThreads) {
    const int lx = e % kEX, ly = (e / kEX) % kEY, lz = e / (kEX * kEY);
    const int gx = wrap3(x0 + lx - 1, r), gy = wrap3(y0 + ly - 1, r), gz = wrap3(z0 + lz - 1, r);
    cp_async<sizeof(TB)>(&S.bs[e], beta + (static_cast<size_t>(gz) * r + gy) * r + gx);
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int p = threadIdx.x + j * kThreads;
    if (p >= kRegion) continue;
    const int lx = p % kRX, ly = (p / kRX) % kRY, lz = p / (kRX * kRY);
    const int ph = stage_pos<kPairs>(lx, ly, lz);
    // interior, unwrapped positions carry the brick's own ids
    const bool inner = lx >= 1 && lx <= kBX && ly >= 1 && ly <= kBY && lz >= 1 && lz <= kBZ && x0 + lx - 1 < r &&
                       y0 + ly - 1 < r && z0 + lz - 1 < r;
    if (inner && id[j] >= first && id[j] < last) S.pc[id[j] - first] = static_cast<unsigned short>(p);
    SHL_DCHECK(!(inner && id[j] >= 0) || (id[j] >= first && id[j] < last));  // a brick's nodes are its id range
    if (id[j] >= 0) {
      const TS* src = v + vbase(id[j], 18);
#pragma unroll
      for (int q = 0; q < 18; ++q) cp_async<sizeof(TS)>(&S.xs[xs_index<TS, kPairs>(q, ph)], src + q * 32);
    } else {
#pragma unroll
      for (int q = 0; q < 18; ++q) S.xs[xs_index<TS, kPairs>(q, ph)] = TS(0);
    }
  }
  cp_async_commit();
}

// Stage brick t = blockIdx.x into the CTA's buffer and run body(S, t) on it.
// (One CTA per active brick: the hardware keeps 4 independent bricks per SM in
// flight, which hides the staging of one behind the arithmetic of the others
// better than a persistent double-buffered CTA did -- 3 CTAs/SM fit then,
// 985 vs 879 us per PCG iteration.)
template <typename TS, typename TB, typename Body>
__device__ __forceinline__ void brick_run(BrickCta<TS, TB>& C, const BrickView& B, int r,
                                          const int* __restrict__ nmap, const TB* __restrict__ beta,
                                          const TS* __restrict__ v, Body&& body) {
  const int t = blockIdx.x;
  int id[kPer];
  stage_ids(id, B, t, r, nmap);
  stage_issue(C.buf, B, t, r, id, beta, v);
  cp_async_wait<0>();
  __syncthreads();  // brick t staged
  body(C.buf, t);
}

// Per-brick fixed-order sum of six doubles into partials[t*6 + s].
__device__ __forceinline__ void brick_reduce6(double (&v)[6], double* red, double* partials, int t) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_xor_sync(0xffffffffu, v[s], o);
    if (lane == 0) red[w * 6 + s] = v[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // (summed after the kernel by brick_sum_kernel)
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      double tot = 0.0;
#pragma unroll
      for (int u = 0; u < kWarps; ++u) tot += red[u * 6 + s];
      partials[t * 6 + s] = tot;
    }
  }
}

// ---- K4 on bricks: w = A z, p = z + beta p, q = w + beta q, p.q ----------------
// One CTA per active brick (brick_run).
template <typename TV, typename TZ, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) brick_apply_kernel(const ApplyArgs<TV, TZ> A) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char brick_raw[];
  __shared__ double scratch[32 * 6];
  PcgState* st = A.state;
  if (st->stop) return;
  // z staged in its storage type (FP32 in mixed multigrid: half the shared
  // memory of an FP64 copy), widened exactly on use
  BrickCta<TZ, TV>& C = *reinterpret_cast<BrickCta<TZ, TV>*>(brick_raw);
  const BrickView& B = A.bricks;
  constexpr bool kPairs = sizeof(TZ) == 4 && sizeof(TV) == 4;  // the staged layout
  brick_run(C, B, A.r, A.node_map, A.beta, A.z, [&](const BrickShared<TZ, TV>& S, int t) {
    const int first = __ldg(B.bstart + t), last = __ldg(B.bstart + t + 1);
    const int idx = first + threadIdx.x;
    double pq[6] = {0, 0, 0, 0, 0, 0};
    if (idx < last) {
      const size_t ob = vbase(idx, 18);
      const TV ridge = static_cast<TV>(st->ridge);
      const int pc = S.pc[threadIdx.x];
      const int lx = pc % kRX, ly = (pc / kRX) % kRY, lz = pc / (kRX * kRY);
      const int ph = stage_pos<kPairs>(lx, ly, lz);
      TV y[18];
      brick_gather<TV, TZ>(y, S.xs, S.bs, pc, kRowStep * ly + lx, lz, lz * (kEX * kEY) + ly * kEX + lx);
      TV* __restrict__ pg = A.p + ob;
      TV* __restrict__ qg = A.q + ob;
      TV pv[18], qv[18];
#pragma unroll
      for (int q = 0; q < 18; ++q) {  // every load in flight before the first store
        pv[q] = pg[q * 32];
        qv[q] = qg[q * 32];
      }
#pragma unroll
      for (int q = 0; q < 18; ++q) {
        const int s = q % 6;
        const TV zq = static_cast<TV>(S.xs[xs_index<TZ, kPairs>(q, ph)]);
        const TV w = idx == 0 ? TV(0) : fma_t(ridge, zq, y[q]);  // node 0 (id 0) pinned
        TV pn = TV(0), qn = TV(0);
        if (!st->done[s]) {
          const TV bc = static_cast<TV>(st->beta[s]);
          pn = fma_t(bc, pv[q], zq);
          qn = fma_t(bc, qv[q], w);
        }
        pg[q * 32] = pn;
        qg[q * 32] = qn;
        pq[s] += static_cast<double>(pn) * static_cast<double>(qn);
      }
    }
    brick_reduce6(pq, C.red, A.partials, t);
  });
  (void)scratch;  // (p.q is summed by brick_sum_kernel, launched after this one)
}

// ---- level-0 V-cycle sweep on bricks ---------------------------------------------
// mode 0: xout = xin + w Dinv (b - A xin)
//      1: xout = b - A xin
//      2: as 0, plus gamma = b.xout (the V-cycle output z = M r; updates beta)
template <typename TB, typename TV, typename TO, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    brick_sweep_kernel(const GmgLevelView<TV> L, const TB* __restrict__ b, const TV* __restrict__ xin,
                       TO* __restrict__ xout, TV omega, int mode, PcgState* st, double* partials, int init) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char brick_raw[];
  __shared__ double scratch[32 * 6];
  if (st->stop) return;
  BrickCta<TV>& C = *reinterpret_cast<BrickCta<TV>*>(brick_raw);
  const BrickView& B = L.bricks;
  brick_run(C, B, L.r, L.node_map, L.beta, xin, [&](const BrickShared<TV>& S, int t) {
    const int first = __ldg(B.bstart + t), last = __ldg(B.bstart + t + 1);
    const int idx = first + threadIdx.x;
    double gam[6] = {0, 0, 0, 0, 0, 0};
    if (idx < last) {
      const size_t ob = vbase(idx, 18);
      TV D[6];
      TB bv[18];
      if (mode != 1) {
#pragma unroll
        for (int q = 0; q < 6; ++q) D[q] = L.dinv[vbase(idx, 6) + q * 32];
      }
#pragma unroll
      for (int q = 0; q < 18; ++q) bv[q] = b[ob + q * 32];  // in flight during the gather
      const int pc = S.pc[threadIdx.x];
      const int lx = pc % kRX, ly = (pc / kRX) % kRY, lz = pc / (kRX * kRY);
      const int ph = stage_pos<sizeof(TV) == 4>(lx, ly, lz);
      TV y[18];
      brick_gather<TV>(y, S.xs, S.bs, pc, kRowStep * ly + lx, lz, lz * (kEX * kEY) + ly * kEX + lx);
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        TV res[3], xo[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int q = c * 6 + s;
          const TV xi = S.xs[xs_index<TV>(q, ph)];
          const TV wv = idx == 0 ? TV(0) : fma_t(L.ridge, xi, y[q]);  // node 0 (id 0) pinned
          res[c] = static_cast<TV>(bv[q]) - wv;
          xo[c] = xi;
        }
        if (mode == 1) {
#pragma unroll
          for (int c = 0; c < 3; ++c) xout[ob + (c * 6 + s) * 32] = static_cast<TO>(idx == 0 ? TV(0) : res[c]);
          continue;
        }
        const TV z0v = D[0] * res[0] + D[1] * res[1] + D[2] * res[2];
        const TV z1v = D[1] * res[0] + D[3] * res[1] + D[4] * res[2];
        const TV z2v = D[2] * res[0] + D[4] * res[1] + D[5] * res[2];
        xo[0] = fma_t(omega, z0v, xo[0]);
        xo[1] = fma_t(omega, z1v, xo[1]);
        xo[2] = fma_t(omega, z2v, xo[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xout[ob + (c * 6 + s) * 32] = static_cast<TO>(xo[c]);
          if (mode == 2) gam[s] += static_cast<double>(bv[c * 6 + s]) * static_cast<double>(xo[c]);
        }
      }
    }
    if (mode == 2) brick_reduce6(gam, C.red, partials, t);
  });
  // (mode 2: r.z is summed by brick_sum_kernel, launched after this one)
  (void)scratch;
  (void)init;
}

// The per-brick partials of the apply (p.q) or of the V-cycle's last level-0
// sweep (r.z) summed in brick order by ONE CTA launched right after the brick
// kernel (programmatic dependent launch), then the PCG scalars (alpha / beta)
// or, for a deferred sum, the 6 totals.  Round 1/2 let the last brick CTA to
// arrive on an atomic counter do this; the arrival's L2 round trip and two
// barriers at the end of EVERY brick CTA cost more than this launch (final
// sweep 148 vs 106 us for the same sweep without a reduction; 773 vs 791 us
// per PCG iteration for the sweep alone).
constexpr int kSumThreads = 512;
constexpr int kSumCtas = 8;  // one portable cluster
__global__ void __cluster_dims__(kSumCtas, 1, 1) __launch_bounds__(kSumThreads)
    brick_sum_kernel(const double* __restrict__ partials, int nab, PcgState* st, int kind, int init,
                     double* totals) {
  namespace cg = cooperative_groups;
  pdl_wait();
  __shared__ double scratch[32 * 6];
  __shared__ double cta_tot[6];
  if (st->stop) return;  // (every CTA of the cluster sees the same flag)
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  // CTA `rank` sums the contiguous chunk of bricks [t0, t1), 16-byte loads
  SHL_DCHECK(nab > 0);
  const int chunk = (nab + kSumCtas - 1) / kSumCtas;
  const int t0 = rank * chunk, t1 = min(nab, t0 + chunk);
  double tot[6] = {0, 0, 0, 0, 0, 0};
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(partials);
  for (int tb = t0 + static_cast<int>(threadIdx.x); tb < t1; tb += 2 * kSumThreads) {
    double2 v[2][3];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = tb + u * kSumThreads;
#pragma unroll
      for (int h = 0; h < 3; ++h) v[u][h] = t < t1 ? __ldcg(p2 + t * 3 + h) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        tot[2 * h] += v[u][h].x;
        tot[2 * h + 1] += v[u][h].y;
      }
  }
  block_sum<6>(tot, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) cta_tot[q] = tot[q];
  cluster.sync();  // every CTA's total in its shared memory
  if (rank == 0 && threadIdx.x == 0) {
    double g[6] = {0, 0, 0, 0, 0, 0};
    for (int c = 0; c < kSumCtas; ++c) {  // CTA order: fixed summation order
      const double* ct = cluster.map_shared_rank(cta_tot, c);
      for (int q = 0; q < 6; ++q) g[q] += ct[q];
    }
    if (totals) {
      for (int q = 0; q < 6; ++q) totals[q] = g[q];
    } else if (kind == 0) {
      finalize_apply_state(st, g);
    } else {
      finalize_gamma_state(st, g, init);
    }
  }
  cluster.sync();  // (no CTA exits while CTA 0 may still read its total)
}

// ---- stored (Galerkin) levels on bricks ------------------------------------------
// The coarse levels' 27-point 3x3-block stencils are stored (243 floats per
// node); the per-node gather of the neighbours' 18 components was a chain of
// dependent L2 loads (level_sweep3 / coarse_warp_sweep).  Here one CTA per
// active 8x4x4-position brick of the level stages the iterate of the brick +
// halo in shared memory (node map -> ids in registers, cp.async, the FP32
// load-case-pair layout with swizzled rows of the level-0 sweeps) and each
// thread owns one brick position: it streams its node's stencil (each warp
// load is 4 row segments of consecutive grid-ordered ids) and gathers the
// neighbours from shared memory.  mode 0: xout = xin + w Dinv (b - A xin);
// mode 1: xout = b - A xin.  Node 0 (grid index 0) is pinned: output 0.
// Three threads per brick position (one per neighbour plane dz = -1, 0, +1,
// 9 stencil blocks each; 384-thread CTAs): the stored levels that take this
// kernel have few active bricks (32^3: ~220, 1.5 per SM), so one thread per
// position left 6 warps per SM to cover the stencil loads' latency.  The
// three partial sums meet in shared memory (fixed order), plane 0's threads
// finish.
constexpr int kSBParts = 3;
constexpr int kSBThreads = kSBParts * kNodes;
struct alignas(16) StencilBrickShared {
  float xs[18 * kPhys];
  float2 part[kSBParts][9][kNodes];  // [plane][c * 3 + load-case pair][position]
};

__global__ void __launch_bounds__(kSBThreads)
    stencil_brick_sweep_kernel(const GmgLevelView<float> L, const float* __restrict__ b,
                               const float* __restrict__ xin, float* __restrict__ xout, float omega, int mode,
                               const PcgState* st) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sb_raw[];
  if (st->stop) return;
  StencilBrickShared& S = *reinterpret_cast<StencilBrickShared*>(sb_raw);
  const BrickView& B = L.bricks;
  const int t = blockIdx.x, tid = threadIdx.x, r = L.r;
  int x0, y0, z0;
  brick_origin(B, t, x0, y0, z0);
  if (tid < kRegion) {  // one staged position per thread
    const int lx = tid % kRX, ly = (tid / kRX) % kRY, lz = tid / (kRX * kRY);
    const int gx = wrap3(x0 + lx - 1, r), gy = wrap3(y0 + ly - 1, r), gz = wrap3(z0 + lz - 1, r);
    const int id = __ldg(L.node_map + (static_cast<size_t>(gz) * r + gy) * r + gx);
    const int ph = stage_pos<true>(lx, ly, lz);
    if (id >= 0) {
      const float* src = xin + vbase(id, 18);
#pragma unroll
      for (int q = 0; q < 18; ++q) cp_async<4>(&S.xs[xs_index<float, true>(q, ph)], src + q * 32);
    } else {
#pragma unroll
      for (int q = 0; q < 18; ++q) S.xs[xs_index<float, true>(q, ph)] = 0.f;
    }
  }
  cp_async_commit();
  // this thread's brick position, node and neighbour plane
  const int part = tid / kNodes, pos = tid % kNodes;
  const int bx = pos & 7, by = (pos >> 3) & 3, bz = pos >> 5;
  const int gx = x0 + bx, gy = y0 + by, gz = z0 + bz;
  const int G = (gz * r + gy) * r + gx;
  const int idx = __ldg(L.node_map + G);
  cp_async_wait<0>();
  __syncthreads();
  const int lx = bx + 1, ly = by + 1, lz = bz + 1;
  const int pxy = kRowStep * ly + lx;
  if (idx >= 0 && G != 0) {
    const float* __restrict__ Sg = L.stencil + vbase(idx, 243);  // 27 x 3x3 blocks per node
    const float2* __restrict__ x2 = reinterpret_cast<const float2*>(S.xs);
    float2 acc[9];  // [c][load-case pair]
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = make_float2(0.f, 0.f);
    const int dz = part - 1;
#pragma unroll 3
    for (int mm = 0; mm < 9; ++mm) {
      const int m = part * 9 + mm;
      const int dx = mm % 3 - 1, dy = mm / 3 - 1;
      float Sm[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) Sm[q] = __ldg(Sg + (m * 9 + q) * 32);
      const float2* xn = x2 + plane_base(lz + dz) + pxy + dy * kRowStep + dx;
#pragma unroll
      for (int sp = 0; sp < 3; ++sp) {
        const float2 z0v = xn[(0 * 3 + sp) * kPhys], z1v = xn[(1 * 3 + sp) * kPhys],
                     z2v = xn[(2 * 3 + sp) * kPhys];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float2 v = acc[c * 3 + sp];
          v = __ffma2_rn(make_float2(Sm[c * 3 + 0], Sm[c * 3 + 0]), z0v, v);
          v = __ffma2_rn(make_float2(Sm[c * 3 + 1], Sm[c * 3 + 1]), z1v, v);
          v = __ffma2_rn(make_float2(Sm[c * 3 + 2], Sm[c * 3 + 2]), z2v, v);
          acc[c * 3 + sp] = v;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) S.part[part][q][pos] = acc[q];
  }
  __syncthreads();
  if (part != 0 || idx < 0) return;
  const size_t ob = vbase(idx, 18);
  if (G == 0) {  // pinned node
#pragma unroll
    for (int q = 0; q < 18; ++q) xout[ob + q * 32] = 0.f;
    return;
  }
  float D[6];
  if (mode != 1) {
#pragma unroll
    for (int q = 0; q < 6; ++q) D[q] = L.dinv[vbase(idx, 6) + q * 32];
  }
  const int ph = plane_base(lz) + pxy;
#pragma unroll
  for (int sp = 0; sp < 3; ++sp)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s_ = 2 * sp + h;
      float res[3], xo[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float2 p0 = S.part[0][c * 3 + sp][pos], p1 = S.part[1][c * 3 + sp][pos],
                     p2 = S.part[2][c * 3 + sp][pos];
        const float y = h ? (p0.y + p1.y) + p2.y : (p0.x + p1.x) + p2.x;
        res[c] = b[ob + (c * 6 + s_) * 32] - y;
        xo[c] = S.xs[xs_index<float, true>(c * 6 + s_, ph)];
      }
      if (mode == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) xout[ob + (c * 6 + s_) * 32] = res[c];
        continue;
      }
      xout[ob + (0 * 6 + s_) * 32] = fma_t(omega, D[0] * res[0] + D[1] * res[1] + D[2] * res[2], xo[0]);
      xout[ob + (1 * 6 + s_) * 32] = fma_t(omega, D[1] * res[0] + D[3] * res[1] + D[4] * res[2], xo[1]);
      xout[ob + (2 * 6 + s_) * 32] = fma_t(omega, D[2] * res[0] + D[4] * res[1] + D[5] * res[2], xo[2]);
    }
}

// Opt a brick kernel into its dynamic shared memory (> 48 KB for FP64).
template <typename K>
bool brick_configure(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return true;
}

}  // namespace

static void build_nb_table(NbEntry (&t)[27]) {
  int n = 0;
  for (int k : {8, 4, 2, 1}) {
    for (int m = 0; m < 27; ++m) {
      const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = m / 9 - 1;
      const int shared = (2 - (dx != 0)) * (2 - (dy != 0)) * (2 - (dz != 0));
      if (shared != k) continue;
      NbEntry& e = t[n++];
      e.roff = dz * (kRX * kRY) + dy * kRX + dx;
      int j = 0;
      for (int el = 0; el < 8; ++el) {
        const int ox = el & 1, oy = (el >> 1) & 1, oz = (el >> 2) & 1;  // node's corner in the element
        const int bx = ox + dx, by = oy + dy, bz = oz + dz;
        if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
        e.eoff[j] = -(oz * (kEX * kEY) + oy * kEX + ox);
        e.kb[j] = 3 * corner_id(ox, oy, oz) * 24 + 3 * corner_id(bx, by, bz);
        ++j;
      }
      for (; j < 8; ++j) e.eoff[j] = e.kb[j] = 0;
    }
  }
}

void brick_upload_constants(const double* K0d, const float* K0f, cudaStream_t s) {
  // coef_m(c,d) = K0[3 a0 + c][3 b0 + d]; every other term of the entry must be
  // +-coef (the isotropic sign structure of stencil_patterns.h)
  static thread_local float cf[243];
  double kmax = 0.0;
  for (int i = 0; i < 576; ++i) kmax = std::max(kmax, std::fabs(K0d[i]));
  for (int m = 0; m < 27; ++m) {
    const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = m / 9 - 1;
    for (int q = 0; q < 9; ++q) {
      const int c = q / 3, d = q % 3;
      const double coef = K0d[(3 * pat::a0(m) + c) * 24 + 3 * pat::b0(m) + d];
      for (int j = 0; j < pat::shared(m); ++j) {
        const int e = pat::elem(m, j), ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;
        const int a = corner_id(ox, oy, oz), b = corner_id(ox + dx, oy + dy, oz + dz);
        if (std::fabs(K0d[(3 * a + c) * 24 + 3 * b + d] - coef * pat::sign(m, pat::pat_of(m, q), j)) > 1e-12 * kmax)
          throw ShlError(SHL_VALIDATION, "element stiffness lacks the isotropic stencil sign structure");
      }
      cf[m * 9 + q] = static_cast<float>(coef);
    }
  }
  cudaMemcpyToSymbolAsync(c_bcoeff, cf, sizeof(cf), 0, cudaMemcpyHostToDevice, s);
  static NbEntry table[27];
  static const bool built = (build_nb_table(table), true);
  (void)built;
  cudaMemcpyToSymbolAsync(c_nb, table, sizeof(table), 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_bK0d, K0d, sizeof(double) * 576, 0, cudaMemcpyHostToDevice, s);
  cudaMemcpyToSymbolAsync(c_bK0f, K0f, sizeof(float) * 576, 0, cudaMemcpyHostToDevice, s);
}

// Level-0 apply: one CTA per active brick.
template <typename TV, typename TZ>
void launch_brick_apply(const ApplyArgs<TV, TZ>& a, cudaStream_t s) {
  constexpr size_t smem = brick_smem_bytes<TZ, TV>();
  constexpr int kMinB = sizeof(TZ) == 8 ? 3 : 4;
  static const bool configured = brick_configure(brick_apply_kernel<TV, TZ, kMinB>, smem);
  (void)configured;
  launch_pdl(brick_apply_kernel<TV, TZ, kMinB>, a.bricks.nab, kThreads, smem, s, a);
  launch_pdl(brick_sum_kernel, kSumCtas, kSumThreads, 0, s, static_cast<const double*>(a.partials), a.bricks.nab, a.state, 0, 0,
             a.defer ? a.totals : static_cast<double*>(nullptr));
}

// Level-0 sweep: one CTA per active brick.
template <typename TB, typename TV, typename TO>
void launch_brick_sweep(const GmgLevelView<TV>& L, const TB* b, const TV* xin, TO* xout, TV omega, int mode,
                        PcgState* st, double* partials, int init, cudaStream_t s) {
  constexpr size_t smem = brick_smem_bytes<TV>();
  constexpr int kMinB = sizeof(TV) == 8 ? 3 : 4;
  static const bool configured = brick_configure(brick_sweep_kernel<TB, TV, TO, kMinB>, smem);
  (void)configured;
  launch_pdl(brick_sweep_kernel<TB, TV, TO, kMinB>, L.bricks.nab, kThreads, smem, s, L, b, xin, xout, omega, mode,
             st, partials, init);
  if (mode == 2)
    launch_pdl(brick_sum_kernel, kSumCtas, kSumThreads, 0, s, static_cast<const double*>(partials), L.bricks.nab, st, 1, init,
               L.totals);
}

// Stored-level sweep on the level's active bricks (FP32 levels).
void launch_stencil_brick_sweep(const GmgLevelView<float>& L, const float* b, const float* xin, float* xout,
                                float omega, int mode, const PcgState* st, cudaStream_t s) {
  static const bool configured = brick_configure(stencil_brick_sweep_kernel, sizeof(StencilBrickShared));
  (void)configured;
  launch_pdl(stencil_brick_sweep_kernel, L.bricks.nab, kSBThreads, sizeof(StencilBrickShared), s, L, b, xin, xout,
             omega, mode, st);
}

template void launch_brick_apply<double, float>(const ApplyArgs<double, float>&, cudaStream_t);
template void launch_brick_apply<double, double>(const ApplyArgs<double, double>&, cudaStream_t);
template void launch_brick_apply<float, float>(const ApplyArgs<float, float>&, cudaStream_t);
template void launch_brick_sweep<double, float, float>(const GmgLevelView<float>&, const double*, const float*,
                                                       float*, float, int, PcgState*, double*, int, cudaStream_t);
template void launch_brick_sweep<double, float, double>(const GmgLevelView<float>&, const double*, const float*,
                                                        double*, float, int, PcgState*, double*, int, cudaStream_t);
template void launch_brick_sweep<float, float, float>(const GmgLevelView<float>&, const float*, const float*,
                                                      float*, float, int, PcgState*, double*, int, cudaStream_t);
template void launch_brick_sweep<double, double, double>(const GmgLevelView<double>&, const double*,
                                                         const double*, double*, double, int, PcgState*, double*,
                                                         int, cudaStream_t);

}  // namespace shl
