// solver.cu -- K3..K6: matrix-free six-load-case PCG on the masked torus (sm_100a).
//
// The reference's GridSolver (grid_solver.hpp:18-207) generalized to the
// reduced shell mesh: absent elements carry beta = 0, torus nodes touched by
// no present element carry no unknowns, node 0 is pinned (the corner gauge of
// build_periodic_system, fem.hpp:190-203; equivalence argued in SURVEY.md
// row A14 and pinned in tests/test_oracle_fem.py).
//
// Storage: active nodes are numbered in grid order (voxel.cu); every PCG
// vector is 18 planes [comp*6 + loadcase][node] so consecutive active nodes
// are consecutive addresses (coalesced, no bytes spent on void voxels).
//
//   K3 rhs_kernel      b_n = -sum_e beta_e (K0 T)_{a(e,n)}      grid_solver.hpp:141-152
//   K4 apply_kernel    w = A z by node-centric gather (no atomics, one thread
//                      per active node), p = z + beta p, q = w + beta q in
//                      place (single-SpMV PCG: A is applied to z, q = A p by
//                      recurrence), partial p.q
//   K5 update_kernel   x += alpha p, r -= alpha q, z = Dinv r, partial r.z, r.r
//   K6 chom_kernel     C_ab = sum_e beta_e (x_e+T)_a^T K0 (x_e+T)_b        :183-197
//
// Scalars never leave the device: the last block of each reduction kernel
// (fixed-order sum of the per-block partials -> deterministic) updates the
// PcgState, so the host only polls a flag every few iterations.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "device.cuh"
#include "solver.cuh"
#include "pcg_common.cuh"

namespace shl {

__constant__ double c_K0d[576];
__constant__ float c_K0f[576];
__constant__ double c_W[144];  // (K0 * T)[24][6]
__constant__ double c_T[144];  // element-local affine displacements T[24][6]

template <typename T>
__device__ __forceinline__ T k0(int i);
template <>
__device__ __forceinline__ double k0<double>(int i) {
  return c_K0d[i];
}
template <>
__device__ __forceinline__ float k0<float>(int i) {
  return c_K0f[i];
}

namespace {

// ---- K3 + preconditioner setup -------------------------------------------
// One thread per active node: block-Jacobi inverse (grid_solver.hpp:129-139)
// and the strain right-hand sides (grid_solver.hpp:141-152), node 0 pinned.
template <typename TX, typename TV>
__global__ void setup_kernel(const int* __restrict__ node_list, int n_nodes, int ld, int r,
                             const double* __restrict__ beta64, double ridge, TX* __restrict__ rvec,
                             TV* __restrict__ dinv) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_nodes) return;
  const int g = node_list[idx];
  const int i = g % r, j = (g / r) % r, k = g / (r * r);
  double D[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double b[18];
#pragma unroll
  for (int q = 0; q < 18; ++q) b[q] = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;  // node offset inside element
    const int ei = i - ox < 0 ? r - 1 : i - ox, ej = j - oy < 0 ? r - 1 : j - oy,
              ek = k - oz < 0 ? r - 1 : k - oz;
    const double be = beta64[(static_cast<size_t>(ek) * r + ej) * r + ei];
    if (be == 0.0) continue;
    const int a = corner_id(ox, oy, oz);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int d = 0; d < 3; ++d) D[c * 3 + d] += be * c_K0d[(3 * a + c) * 24 + 3 * a + d];
#pragma unroll
      for (int s = 0; s < 6; ++s) b[c * 6 + s] -= be * c_W[(3 * a + c) * 6 + s];
    }
  }
  double inv[6] = {0, 0, 0, 0, 0, 0};  // symmetric: 00 01 02 11 12 22
  if (g != 0) {
    D[0] += ridge;
    D[4] += ridge;
    D[8] += ridge;
    const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[5] * D[6] - D[3] * D[8],
                 c02 = D[3] * D[7] - D[4] * D[6];
    const double det = D[0] * c00 + D[1] * c01 + D[2] * c02;
    const double id = 1.0 / det;
    inv[0] = c00 * id;
    inv[1] = c01 * id;
    inv[2] = c02 * id;
    inv[3] = (D[0] * D[8] - D[2] * D[6]) * id;
    inv[4] = (D[2] * D[3] - D[0] * D[5]) * id;
    inv[5] = (D[0] * D[4] - D[1] * D[3]) * id;
  } else {
#pragma unroll
    for (int q = 0; q < 18; ++q) b[q] = 0.0;
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) dinv[vbase(idx, 6) + q * 32] = static_cast<TV>(inv[q]);
#pragma unroll
  for (int q = 0; q < 18; ++q) rvec[vbase(idx, 18) + q * 32] = static_cast<TX>(b[q]);
}

// ---- K4: w = A z by gather, fused with the direction update -------------------
// Chronopoulos-Gear form of PCG: the operator is applied to z (the freshly
// preconditioned residual) instead of p, so the neighbourhood gather reads one
// vector and p, q are updated in place for the thread's own node:
//   w = A z,  p = z + beta p,  q = w + beta q,  delta = z.w
// One thread per ACTIVE node (no lanes spent on void voxels).  For neighbour m
// of node n the 3x3 block S_m = sum_{e ni n,m} beta_e K0[a(n,e), b(m,e)] is
// built once (K0 entries are constant-bank operands, single-issue FFMA) and
// applied to all six load cases.  In FP32 the application runs on packed
// FFMA2 over load-case pairs (S scalar broadcast x (z_s, z_s+1)), halving the
// 3-register FFMAs that bound this kernel.  Inactive neighbours read a zero
// slot (index n_nodes).
template <typename TV>
struct GatherAcc;

template <>
struct GatherAcc<float> {
  float2 y[9];  // [comp][loadcase pair]
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < 9; ++q) y[q] = make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ void add(const float (&S)[9], const float* __restrict__ zn) {
#pragma unroll
    for (int sp = 0; sp < 3; ++sp) {
      const float2 z0 = make_float2(zn[(0 * 6 + 2 * sp) * 32], zn[(0 * 6 + 2 * sp + 1) * 32]);
      const float2 z1 = make_float2(zn[(1 * 6 + 2 * sp) * 32], zn[(1 * 6 + 2 * sp + 1) * 32]);
      const float2 z2 = make_float2(zn[(2 * 6 + 2 * sp) * 32], zn[(2 * 6 + 2 * sp + 1) * 32]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float2 v = y[c * 3 + sp];
        v = __ffma2_rn(make_float2(S[c * 3 + 0], S[c * 3 + 0]), z0, v);
        v = __ffma2_rn(make_float2(S[c * 3 + 1], S[c * 3 + 1]), z1, v);
        v = __ffma2_rn(make_float2(S[c * 3 + 2], S[c * 3 + 2]), z2, v);
        y[c * 3 + sp] = v;
      }
    }
  }
  __device__ __forceinline__ float get(int q) const {  // q = c*6 + s
    const float2 v = y[(q / 6) * 3 + (q % 6) / 2];
    return (q & 1) ? v.y : v.x;
  }
};

template <>
struct GatherAcc<double> {
  double y[18];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < 18; ++q) y[q] = 0.0;
  }
  template <typename TZ>
  __device__ __forceinline__ void add(const double (&S)[9], const TZ* __restrict__ zn) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const double z0 = zn[(0 * 6 + s) * 32], z1 = zn[(1 * 6 + s) * 32], z2 = zn[(2 * 6 + s) * 32];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = y[c * 6 + s];
        v = fma(S[c * 3 + 0], z0, v);
        v = fma(S[c * 3 + 1], z1, v);
        v = fma(S[c * 3 + 2], z2, v);
        y[c * 6 + s] = v;
      }
    }
  }
  __device__ __forceinline__ double get(int q) const { return y[q]; }
};

// FP64 accumulator for three load cases (3h .. 3h+2): the six-warp apply
// splits the load cases in halves to keep the FP64 register footprint small.
struct GatherAccHalf {
  double y[9];  // [comp][load case in half]
  int off;      // 3h * 32: first load case of the half
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < 9; ++q) y[q] = 0.0;
  }
  template <typename TZ>
  __device__ __forceinline__ void add(const double (&S)[9], const TZ* __restrict__ zn) {
    zn += off;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const double z0 = zn[(0 * 6 + s) * 32], z1 = zn[(1 * 6 + s) * 32], z2 = zn[(2 * 6 + s) * 32];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = y[c * 3 + s];
        v = fma(S[c * 3 + 0], z0, v);
        v = fma(S[c * 3 + 1], z1, v);
        v = fma(S[c * 3 + 2], z2, v);
        y[c * 3 + s] = v;
      }
    }
  }
};

// w = A x at active node idx (grid id g): the matrix-free level-0 operator.
// beta is global (every rank holds the full mask); the node map covers local
// planes [zbase, zbase + nzl) (the whole torus when not slabbed).
template <typename TV>
__device__ __forceinline__ void fine_gather(GatherAcc<TV>& acc, int idx, int g,
                                            const TV* __restrict__ xv,
                                            const TV* __restrict__ betav,
                                            const int* __restrict__ nmap, int r, int zbase,
                                            int zero_slot) {
  acc.zero();
  if (g == 0) return;  // pinned node (grid_solver.hpp:175)
  const int rr = r * r;
  const int i = g % r, j = (g / r) % r, k = g / rr;
  const int xs[3] = {i == 0 ? r - 1 : i - 1, i, i == r - 1 ? 0 : i + 1};
  const int ys[3] = {(j == 0 ? r - 1 : j - 1) * r, j * r, (j == r - 1 ? 0 : j + 1) * r};
  const int kz[3] = {k == 0 ? r - 1 : k - 1, k, k == r - 1 ? 0 : k + 1};
  const int zs[3] = {kz[0] * rr, kz[1] * rr, kz[2] * rr};
  int zl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int lz = kz[d] - zbase;
    lz += lz < 0 ? r : 0;
    zl[d] = lz * rr;
  }
  TV be[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;  // node's corner in e
    be[e] = betav[zs[1 - oz] + ys[1 - oy] + xs[1 - ox]];
  }
#pragma unroll
  for (int m = 0; m < 27; ++m) {
    const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = m / 9 - 1;
    int nb = (m == 13) ? idx : nmap[zl[dz + 1] + ys[dy + 1] + xs[dx + 1]];
    nb = nb < 0 ? zero_slot : nb;
    TV S[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) S[q] = TV(0);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;
      const int bx = ox + dx, by = oy + dy, bz = oz + dz;  // neighbour's corner in e
      if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
      const int a = corner_id(ox, oy, oz), b = corner_id(bx, by, bz);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          S[c * 3 + d] = fma_t(be[e], k0<TV>((3 * a + c) * 24 + 3 * b + d), S[c * 3 + d]);
    }
    acc.add(S, xv + vbase(nb, 18));
  }
}

// Partial w = A x over the nine neighbours in plane dz = PLANE-1 (PLANE is a
// compile-time constant so the K0 indices stay immediates).
template <typename TV, int PLANE, typename TZ, typename Acc>
__device__ __forceinline__ void fine_gather_plane(Acc& acc, int idx, int g,
                                                  const TZ* __restrict__ xv,
                                                  const TV* __restrict__ betav,
                                                  const int* __restrict__ nmap, int r, int zbase,
                                                  int zero_slot) {
  acc.zero();
  if (g == 0) return;
  const int rr = r * r;
  const int i = g % r, j = (g / r) % r, k = g / rr;
  const int xs[3] = {i == 0 ? r - 1 : i - 1, i, i == r - 1 ? 0 : i + 1};
  const int ys[3] = {(j == 0 ? r - 1 : j - 1) * r, j * r, (j == r - 1 ? 0 : j + 1) * r};
  constexpr int dz = PLANE - 1;
  const int kn = dz < 0 ? (k == 0 ? r - 1 : k - 1) : (dz > 0 ? (k == r - 1 ? 0 : k + 1) : k);
  int lz = kn - zbase;
  lz += lz < 0 ? r : 0;
  const int zl = lz * rr;
  // the elements shared with this plane: node corner oz with oz + dz in {0,1}
  TV be[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;
    if (oz + dz < 0 || oz + dz > 1) {
      be[e] = TV(0);
      continue;
    }
    const int ek = oz ? (k == 0 ? r - 1 : k - 1) : k;
    be[e] = betav[ek * rr + ys[1 - oy] + xs[1 - ox]];
  }
#pragma unroll
  for (int mm = 0; mm < 9; ++mm) {
    const int dx = mm % 3 - 1, dy = mm / 3 - 1;
    int nb = (dx == 0 && dy == 0 && dz == 0) ? idx : nmap[zl + ys[dy + 1] + xs[dx + 1]];
    nb = nb < 0 ? zero_slot : nb;
    TV S[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) S[q] = TV(0);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ox = e & 1, oy = (e >> 1) & 1, oz = (e >> 2) & 1;
      const int bx = ox + dx, by = oy + dy, bz = oz + dz;
      if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
      const int a = corner_id(ox, oy, oz), b = corner_id(bx, by, bz);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          S[c * 3 + d] = fma_t(be[e], k0<TV>((3 * a + c) * 24 + 3 * b + d), S[c * 3 + d]);
    }
    acc.add(S, xv + vbase(nb, 18));
  }
}

// Three warps cooperate on 32 consecutive nodes: warp p gathers plane dz=p-1,
// the partial sums meet in shared memory, and the caller's epilogue runs on
// warp p for load-case pair p (s = 2p, 2p+1).  part_s: [3][18][32].
template <typename TV, typename TZ>
__device__ __forceinline__ void gather3_tile(TV* part_s, int part, int lane, int idx, bool valid,
                                             int g, const TZ* __restrict__ xv,
                                             const TV* __restrict__ betav,
                                             const int* __restrict__ nmap, int r, int zbase,
                                             int zero_slot) {
  GatherAcc<TV> acc;
  if (!valid) {
    acc.zero();
  } else if (part == 0) {
    fine_gather_plane<TV, 0>(acc, idx, g, xv, betav, nmap, r, zbase, zero_slot);
  } else if (part == 1) {
    fine_gather_plane<TV, 1>(acc, idx, g, xv, betav, nmap, r, zbase, zero_slot);
  } else {
    fine_gather_plane<TV, 2>(acc, idx, g, xv, betav, nmap, r, zbase, zero_slot);
  }
#pragma unroll
  for (int q = 0; q < 18; ++q) part_s[(part * 18 + q) * 32 + lane] = acc.get(q);
}

template <typename TV>
__device__ __forceinline__ TV gather3_sum(const TV* part_s, int q, int lane) {
  return part_s[(0 * 18 + q) * 32 + lane] + part_s[(1 * 18 + q) * 32 + lane] + part_s[(2 * 18 + q) * 32 + lane];
}

// w = A z, p = z + beta p, q = w + beta q, p.q (the FP32 operator), latency-split
// three ways (gather3_tile).
template <typename TV, typename TZ>
__global__ void __launch_bounds__(192) apply3_kernel(const ApplyArgs<TV, TZ> A) {
  __shared__ __align__(16) TV part_s[2][3 * 18 * 32];
  __shared__ double scratch[32 * 6];
  PcgState* st = A.state;
  if (st->stop) return;
  const TZ* __restrict__ zv = A.z;
  TV* __restrict__ pv = A.p;
  TV* __restrict__ qv = A.q;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = w / 3, part = w % 3;
  const TV ridge = static_cast<TV>(st->ridge);
  bool dn[2];
  TV bcoef[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    dn[k] = st->done[2 * part + k] != 0;
    bcoef[k] = static_cast<TV>(st->beta[2 * part + k]);
  }
  double pq2[2] = {0, 0};
  for (int tile = blockIdx.x; A.n0 + tile * 64 < A.n; tile += gridDim.x) {
    const int idx = A.n0 + tile * 64 + grp * 32 + lane;
    const bool valid = idx < A.n;
    const int g = valid ? A.node_list[idx] : -1;
    gather3_tile<TV, TZ>(part_s[grp], part, lane, idx, valid, g, zv, A.beta, A.node_map, A.r, A.zbase,
                         A.zero_slot);
    __syncthreads();
    if (valid) {
      const size_t ob = vbase(idx, 18);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int s_ = 2 * part + k, q = c * 6 + s_;
          const size_t o = ob + q * 32;
          const TV zq = static_cast<TV>(zv[o]);
          const TV wv = g != 0 ? fma_t(ridge, zq, gather3_sum<TV>(part_s[grp], q, lane)) : TV(0);
          TV pn = TV(0), qn = TV(0);
          if (!dn[k]) {
            pn = fma_t(bcoef[k], pv[o], zq);
            qn = fma_t(bcoef[k], qv[o], wv);
          }
          pv[o] = pn;
          qv[o] = qn;
          pq2[k] += static_cast<double>(pn) * static_cast<double>(qn);
        }
    }
    __syncthreads();
  }
  double pq[6];
#pragma unroll
  for (int s_ = 0; s_ < 6; ++s_) pq[s_] = (s_ >> 1) == part ? pq2[s_ & 1] : 0.0;
  block_sum<6>(pq, scratch);
  if (publish_partial<6>(pq, A.partials, &st->counter_apply)) {
    double tot[6];
    __syncthreads();
    reduce_partials<6>(A.partials, tot, scratch);
    if (threadIdx.x == 0) {
      if (A.defer) {
        for (int s_ = 0; s_ < 6; ++s_) A.totals[s_] = tot[s_];
      } else {
        finalize_apply_state(st, tot);
      }
      st->counter_apply = 0;
    }
  }
}

// FP64 operator: six warps per 32 nodes, warp (plane p, half h) gathers plane
// dz=p-1 for load cases 3h..3h+2, then finishes load case s = 3h + p.  G groups
// of six warps per block, MINB blocks per SM (register budget).
template <typename TZ, int G, int MINB>
__global__ void __launch_bounds__(192 * G, MINB) apply6_kernel(const ApplyArgs<double, TZ> A) {
  __shared__ __align__(16) double part_s[G][3 * 18 * 32];
  __shared__ double scratch[32 * 6];
  PcgState* st = A.state;
  if (st->stop) return;
  const TZ* __restrict__ zv = A.z;
  double* __restrict__ pv = A.p;
  double* __restrict__ qv = A.q;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = w / 6, plane = w % 3, half = (w % 6) / 3;
  const int s_ = 3 * half + plane;  // epilogue load case
  const double ridge = st->ridge;
  const bool dn = st->done[s_] != 0;
  const double bcoef = st->beta[s_];
  __shared__ double red[G][6];
  // Tiles come from the shared counter (TileQueue); p.q is reduced PER TILE
  // (warp butterfly, groups in fixed order) into partials[tile][6], and the
  // last CTA sums the tiles in index order: the same bits whichever CTA ran
  // which tile (reproducible C^H under any residency).
  __shared__ int tq_slot[2];
  TileQueue tq{&st->tile_next[0], tq_slot};
  for (int tile = tq.first();; tile = tq.advance()) {
    if (A.n0 + tile * (32 * G) >= A.n) break;
    tq.request();
    const int idx = A.n0 + tile * (32 * G) + grp * 32 + lane;
    const bool valid = idx < A.n;
    const int g = valid ? A.node_list[idx] : -1;
    {
      GatherAccHalf acc;
      acc.off = 3 * half * 32;
      if (!valid)
        acc.zero();
      else if (plane == 0)
        fine_gather_plane<double, 0>(acc, idx, g, zv, A.beta, A.node_map, A.r, A.zbase, A.zero_slot);
      else if (plane == 1)
        fine_gather_plane<double, 1>(acc, idx, g, zv, A.beta, A.node_map, A.r, A.zbase, A.zero_slot);
      else
        fine_gather_plane<double, 2>(acc, idx, g, zv, A.beta, A.node_map, A.r, A.zbase, A.zero_slot);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 3; ++k) part_s[grp][(plane * 18 + c * 6 + 3 * half + k) * 32 + lane] = acc.y[c * 3 + k];
    }
    tq.publish();
    __syncthreads();
    double pq = 0.0;
    if (valid) {
      const size_t ob = vbase(idx, 18);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int q = c * 6 + s_;
        const size_t o = ob + q * 32;
        const double zq = static_cast<double>(zv[o]);
        const double wv = g != 0 ? fma(ridge, zq, gather3_sum<double>(part_s[grp], q, lane)) : 0.0;
        double pn = 0.0, qn = 0.0;
        if (!dn) {
          pn = fma(bcoef, pv[o], zq);
          qn = fma(bcoef, qv[o], wv);
        }
        pv[o] = pn;
        qv[o] = qn;
        pq += pn * qn;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pq += __shfl_xor_sync(0xffffffffu, pq, o);
    if (lane == 0) red[grp][s_] = pq;
    __syncthreads();
    if (threadIdx.x < 6) {
      double t = red[0][threadIdx.x];
#pragma unroll
      for (int gg = 1; gg < G; ++gg) t += red[gg][threadIdx.x];
      A.partials[tile * 6 + threadIdx.x] = t;
    }
  }
  tiles_done(&st->tile_next[0], &st->tile_done[0]);
  __shared__ bool last;
  __syncthreads();  // every thread's partial writes ordered before thread 0's release
  if (threadIdx.x == 0) last = arrive_last(&st->counter_apply);
  __syncthreads();
  if (!last) return;
  const int ntiles = (A.n - A.n0 + 32 * G - 1) / (32 * G);
  double tot[6] = {0, 0, 0, 0, 0, 0};
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x)
#pragma unroll
    for (int q = 0; q < 6; ++q) tot[q] += __ldcg(A.partials + t * 6 + q);
  block_sum<6>(tot, scratch);
  if (threadIdx.x == 0) {
    if (A.defer) {
      for (int t = 0; t < 6; ++t) A.totals[t] = tot[t];
    } else {
      finalize_apply_state(st, tot);
    }
    st->counter_apply = 0;
  }
}

// ---- K5: vector update + preconditioner + dots ------------------------------
//   x += alpha p, r -= alpha q, z = Dinv r, partial r.r and r.z
// One thread per (node, load case): 3 components of x, r, p, q, z and the 6
// Dinv entries -> ~30 registers, full occupancy, every access a coalesced
// 32-node plane segment.  blockIdx.x = node_block * 6 + s so the six blocks
// of a node block run together and Dinv is re-read from L2, not DRAM.
template <typename TX, typename TV, typename TZ, typename TXS>
__global__ void __launch_bounds__(256) update_kernel(const UpdateArgs<TX, TV, TZ, TXS> U) {
  pdl_wait();
  __shared__ double scratch[32 * 2];
  PcgState* st = U.state;
  if (st->stop) return;
  TXS* __restrict__ xv = U.x;
  TX* __restrict__ rv = U.r;
  const TV* __restrict__ pv = U.p;
  const TV* __restrict__ qv = U.q;
  TZ* __restrict__ zv = U.z;
  const TZ* __restrict__ dv = U.dinv;
  const int s = blockIdx.x % 6;
  const int nbx = gridDim.x / 6;
  const TX a = static_cast<TX>(st->alpha[s]);
  double acc[2] = {0.0, 0.0};  // r.r, r.z for load case s
  for (int idx = (blockIdx.x / 6) * blockDim.x + threadIdx.x; idx < U.n; idx += nbx * blockDim.x) {
    const size_t ob = vbase(idx, 18) + s * 32;
    const size_t od = vbase(idx, 6);
    // all loads first (keeps ~15 independent requests in flight per thread)
    TX xc[3], rc[3];
    TV pc[3], qc[3];
    TZ D[6] = {};
#pragma unroll
    for (int c = 0; c < 3; ++c) rc[c] = rv[ob + c * 192];
    if (!U.init) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xc[c] = static_cast<TX>(xv[ob + c * 192]);
        pc[c] = pv[ob + c * 192];
        qc[c] = qv[ob + c * 192];
      }
    }
    if (!U.gmg || U.gmg_x0) {
#pragma unroll
      for (int q = 0; q < 6; ++q) D[q] = dv[od + q * 32];
    }
    if (!U.init) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xc[c] = fma_t(a, static_cast<TX>(pc[c]), xc[c]);
        rc[c] = fma_t(-a, static_cast<TX>(qc[c]), rc[c]);
      }
    }
    const double d0 = rc[0], d1 = rc[1], d2 = rc[2];
    acc[0] += d0 * d0 + d1 * d1 + d2 * d2;
    if (U.gmg) {
      if (!U.init) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xv[ob + c * 192] = static_cast<TXS>(xc[c]);
          rv[ob + c * 192] = rc[c];
        }
      }
      if (U.gmg_x0) {  // fused first smoothing sweep of the V-cycle (x = w Dinv r)
        const TZ r0 = static_cast<TZ>(rc[0]), r1 = static_cast<TZ>(rc[1]), r2 = static_cast<TZ>(rc[2]);
        const TZ w = U.gmg_omega;
        U.gmg_x0[ob + 0 * 192] = w * (D[0] * r0 + D[1] * r1 + D[2] * r2);
        U.gmg_x0[ob + 1 * 192] = w * (D[1] * r0 + D[3] * r1 + D[4] * r2);
        U.gmg_x0[ob + 2 * 192] = w * (D[2] * r0 + D[4] * r1 + D[5] * r2);
      }
      continue;
    }
    const TZ r0 = static_cast<TZ>(rc[0]), r1 = static_cast<TZ>(rc[1]), r2 = static_cast<TZ>(rc[2]);
    const TZ z0 = D[0] * r0 + D[1] * r1 + D[2] * r2;
    const TZ z1 = D[1] * r0 + D[3] * r1 + D[4] * r2;
    const TZ z2 = D[2] * r0 + D[4] * r1 + D[5] * r2;
    if (!U.init) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xv[ob + c * 192] = static_cast<TXS>(xc[c]);
        rv[ob + c * 192] = rc[c];
      }
    }
    zv[ob + 0 * 192] = z0;
    zv[ob + 1 * 192] = z1;
    zv[ob + 2 * 192] = z2;
    acc[1] += d0 * static_cast<double>(z0) + d1 * static_cast<double>(z1) + d2 * static_cast<double>(z2);
  }
  block_sum<2>(acc, scratch);
  if (publish_partial<2>(acc, U.partials, &st->counter_update)) {
    __syncthreads();
    // fixed-order reduction per load case: partials[(b*6 + s)*2 + {0,1}]
    double tot[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) tot[q] = 0.0;
    for (int b = threadIdx.x; b < nbx; b += blockDim.x)
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        tot[t] += __ldcg(U.partials + (b * 6 + t) * 2 + 0);
        tot[6 + t] += __ldcg(U.partials + (b * 6 + t) * 2 + 1);
      }
    __shared__ double scratch12[32 * 12];
    block_sum<12>(tot, scratch12);
    if (threadIdx.x == 0) {
      if (U.defer) {
        for (int q = 0; q < 12; ++q) U.totals[q] = tot[q];
      } else if (U.gmg) {
        finalize_update_gmg(st, tot, U.init);
      } else {
        finalize_update_state(st, tot, U.init);
      }
      st->counter_update = 0;
    }
  }
}

// ---- K6: C^H energy reduction ------------------------------------------------
// One thread per active element; U = x_e + T (24x6) staged in shared memory,
// the 21 upper-triangle accumulators too, W = K0 U_b per column in registers.
template <typename TX>
__global__ void __launch_bounds__(32) chom_kernel(const ChomArgs<TX> Cg) {
  __shared__ double scratch[32 * 21];
  __shared__ double Us[32][145];
  __shared__ double As[32][21];
  PcgState* st = Cg.state;
  const int r = Cg.r;
  double* U = Us[threadIdx.x];
  double* acc_s = As[threadIdx.x];
  for (int q = 0; q < 21; ++q) acc_s[q] = 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Cg.n_elem; t += gridDim.x * blockDim.x) {
    const int e = Cg.elem_list[t];
    const int i = e % r, j = (e / r) % r, k = e / (r * r);
    const double be = Cg.beta64[e];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int gx = (i + (n == 1 || n == 2 || n == 5 || n == 6)) % r;
      const int gy = (j + (n == 2 || n == 3 || n == 6 || n == 7)) % r;
      int lz = (k + (n >= 4)) % r - Cg.zbase;
      lz += lz < 0 ? r : 0;
      const int idx = Cg.node_map[(static_cast<size_t>(lz) * r + gy) * r + gx];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int s = 0; s < 6; ++s)
          U[(3 * n + c) * 6 + s] =
              (idx >= 0 ? static_cast<double>(Cg.x[vbase(idx, 18) + (c * 6 + s) * 32]) : 0.0) +
              c_T[(3 * n + c) * 6 + s];
    }
#pragma unroll 1
    for (int b = 0; b < 6; ++b) {
      double W[24];
#pragma unroll
      for (int ii = 0; ii < 24; ++ii) {
        double w = 0.0;
#pragma unroll
        for (int jj = 0; jj < 24; ++jj) w += c_K0d[ii * 24 + jj] * U[jj * 6 + b];
        W[ii] = w;
      }
#pragma unroll 1
      for (int a = 0; a <= b; ++a) {
        double d = 0.0;
#pragma unroll
        for (int ii = 0; ii < 24; ++ii) d += U[ii * 6 + a] * W[ii];
        acc_s[b * (b + 1) / 2 + a] += be * d;
      }
    }
  }
  double acc[21];
#pragma unroll
  for (int q = 0; q < 21; ++q) acc[q] = acc_s[q];
  block_sum<21>(acc, scratch);
  if (publish_partial<21>(acc, Cg.partials, &st->counter_misc)) {
    double tot[21];
    __syncthreads();
    reduce_partials<21>(Cg.partials, tot, scratch);
    if (threadIdx.x == 0) {
      if (Cg.defer) {
        for (int q = 0; q < 21; ++q) Cg.C_out[q] = tot[q];
      } else {
        for (int b = 0; b < 6; ++b)
          for (int a = 0; a <= b; ++a) {
            Cg.C_out[a * 6 + b] = tot[b * (b + 1) / 2 + a];
            Cg.C_out[b * 6 + a] = tot[b * (b + 1) / 2 + a];
          }
      }
      st->counter_misc = 0;
    }
  }
}

// ---- cross-slab finalize + ghost-plane transport ---------------------------
__global__ void finalize_update_kernel(PcgState* st, const double* totals, int nslab, int init) {
  double tot[12];
  for (int q = 0; q < 12; ++q) {
    double s = 0.0;
    for (int b = 0; b < nslab; ++b) s += totals[b * 12 + q];
    tot[q] = s;
  }
  if (st->stop && !init) return;
  finalize_update_state(st, tot, init);
}

__global__ void finalize_update_gmg_kernel(PcgState* st, const double* totals, int nslab, int init) {
  double rr[6];
  for (int q = 0; q < 6; ++q) {
    double s = 0.0;
    for (int b = 0; b < nslab; ++b) s += totals[b * 12 + q];
    rr[q] = s;
  }
  if (st->stop && !init) return;
  finalize_update_gmg(st, rr, init);
}

__global__ void finalize_gamma_kernel(PcgState* st, const double* totals, int nslab, int init) {
  if (st->stop) return;
  double g[6];
  for (int q = 0; q < 6; ++q) {
    double s = 0.0;
    for (int b = 0; b < nslab; ++b) s += totals[b * 6 + q];
    g[q] = s;
  }
  finalize_gamma_state(st, g, init);
}

__global__ void finalize_apply_kernel(PcgState* st, const double* totals, int nslab) {
  if (st->stop) return;
  double tot[6];
  for (int q = 0; q < 6; ++q) {
    double s = 0.0;
    for (int b = 0; b < nslab; ++b) s += totals[b * 6 + q];
    tot[q] = s;
  }
  finalize_apply_state(st, tot);
}

__global__ void finalize_chom_kernel(const double* totals, int nslab, double* C) {
  for (int b = 0; b < 6; ++b)
    for (int a = 0; a <= b; ++a) {
      double s = 0.0;
      for (int q = 0; q < nslab; ++q) s += totals[q * 21 + b * (b + 1) / 2 + a];
      C[a * 6 + b] = s;
      C[b * 6 + a] = s;
    }
}

template <typename T>
__global__ void pack_kernel(const T* __restrict__ vec, int first, int count, T* __restrict__ buf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 18) return;
  const int q = t / count, i = t % count;
  buf[t] = vec[vbase(first + i, 18) + q * 32];
}

template <typename T>
__global__ void unpack_kernel(T* __restrict__ vec, int first, int count, const T* __restrict__ buf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * 18) return;
  const int q = t / count, i = t % count;
  vec[vbase(first + i, 18) + q * 32] = buf[t];
}

}  // namespace

void launch_finalize_update(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s) {
  finalize_update_kernel<<<1, 1, 0, s>>>(st, totals, nslab, init);
}
// Device-side loop control of the solve graph: keep iterating while the PCG
// state has not stopped (converged, broken down or out of iterations).
__global__ void set_while_kernel(cudaGraphConditionalHandle h, const PcgState* st) {
  pdl_wait();
  cudaGraphSetConditional(h, st->stop ? 0u : 1u);
}
void launch_set_while(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s) {
  launch_pdl(set_while_kernel, 1, 1, 0, s, h, st);
}

void launch_finalize_update_gmg(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s) {
  finalize_update_gmg_kernel<<<1, 1, 0, s>>>(st, totals, nslab, init);
}
void launch_finalize_gamma(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s) {
  finalize_gamma_kernel<<<1, 1, 0, s>>>(st, totals, nslab, init);
}
void launch_finalize_apply(PcgState* st, const double* totals, int nslab, cudaStream_t s) {
  finalize_apply_kernel<<<1, 1, 0, s>>>(st, totals, nslab);
}
void launch_finalize_chom(const double* totals, int nslab, double* C_out, cudaStream_t s) {
  finalize_chom_kernel<<<1, 1, 0, s>>>(totals, nslab, C_out);
}
template <typename T>
void launch_pack(const T* vec, int first, int count, T* buf, cudaStream_t s) {
  if (count > 0) pack_kernel<T><<<(count * 18 + 255) / 256, 256, 0, s>>>(vec, first, count, buf);
}
template <typename T>
void launch_unpack(T* vec, int first, int count, const T* buf, cudaStream_t s) {
  if (count > 0) unpack_kernel<T><<<(count * 18 + 255) / 256, 256, 0, s>>>(vec, first, count, buf);
}
template void launch_pack<float>(const float*, int, int, float*, cudaStream_t);
template void launch_pack<double>(const double*, int, int, double*, cudaStream_t);
template void launch_unpack<float>(float*, int, int, const float*, cudaStream_t);
template void launch_unpack<double>(double*, int, int, const double*, cudaStream_t);

#include "gmg.cuh"

// ---- host-side launchers -----------------------------------------------------
// The element matrices live in __constant__ memory (FMA operands straight from
// the constant bank) and the level-1 Galerkin cell matrices in device globals:
// one copy per device, shared by every context.  A solve holds a lease on the
// copy for its whole duration; the copy is rewritten only when a solve needs
// different constants (another r or material) and no other solve on the device
// still uses the old ones.  Concurrent batch lanes (same r and material) then
// never write constant memory while each other's kernels run, and independent
// contexts with different constants serialize instead of racing.
namespace {
struct ConstSlot {
  std::mutex m;
  std::condition_variable cv;
  bool valid = false;
  double key[577] = {};  // K0 (576) and r: W and T follow from them
  int users = 0;
};
ConstSlot& const_slot(int device) {
  static ConstSlot slots[64];
  return slots[device & 63];
}
}  // namespace

ElementConstLease::ElementConstLease(const double* K0, const double* W, const double* T, int r, cudaStream_t s) {
  cudaGetDevice(&device_);
  ConstSlot& cs = const_slot(device_);
  double key[577];
  std::memcpy(key, K0, 576 * sizeof(double));
  key[576] = static_cast<double>(r);
  std::unique_lock<std::mutex> lk(cs.m);
  auto same = [&] { return cs.valid && std::memcmp(cs.key, key, sizeof(key)) == 0; };
  cs.cv.wait(lk, [&] { return same() || cs.users == 0; });
  if (!same()) {
    float K0f[576];
    for (int q = 0; q < 576; ++q) K0f[q] = static_cast<float>(K0[q]);
    cudaMemcpyToSymbolAsync(c_K0d, K0, sizeof(double) * 576, 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_K0f, K0f, sizeof(float) * 576, 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_W, W, sizeof(double) * 144, 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_T, T, sizeof(double) * 144, 0, cudaMemcpyHostToDevice, s);
    brick_upload_constants(K0, K0f, s);  // brick.cu keeps its own copy of K0
    cell_matrices_kernel<<<8, 576, 0, s>>>();  // P_j^T K0 P_j for the level-1 Galerkin product
    // K0f lives on this stack frame; other streams read the result next
    cudaStreamSynchronize(s);
    std::memcpy(cs.key, key, sizeof(key));
    cs.valid = true;
  }
  ++cs.users;
}

ElementConstLease::~ElementConstLease() {
  ConstSlot& cs = const_slot(device_);
  {
    std::lock_guard<std::mutex> lk(cs.m);
    --cs.users;
  }
  cs.cv.notify_all();
}

template <typename TX, typename TV>
void launch_setup(const int* node_list, int n_nodes, int ld, int r, const double* beta64,
                  double ridge, TX* rvec, TV* dinv, cudaStream_t s) {
  if (n_nodes == 0) return;
  setup_kernel<TX, TV><<<(n_nodes + 127) / 128, 128, 0, s>>>(node_list, n_nodes, ld, r, beta64,
                                                            ridge, rvec, dinv);
}

template <typename TV, typename TZ>
void launch_apply(const ApplyArgs<TV, TZ>& a, int grid, cudaStream_t s) {
  if (a.bricks.nab > 0) {
    launch_brick_apply<TV, TZ>(a, s);
    return;
  }
  // per-node gather kernels: the z-slab levels (slab-local numbering)
  if constexpr (sizeof(TV) == 8) {
    // one six-warp group per CTA, 4 CTAs per SM, one CTA per resident slot
    // (tiles are dynamic, so the grid-stride loop has no tail wave)
    static const int nsm = [] {
      int dev = 0, v = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v;
    }();
    apply6_kernel<TZ, 1, 4><<<std::min(grid, 4 * nsm), 192, 0, s>>>(a);
  } else {
    apply3_kernel<TV, TZ><<<grid, 192, 0, s>>>(a);
  }
}

int apply_grid(int n, int num_sms) { return std::max(1, std::min((n + 63) / 64, num_sms * 4)); }

template <typename TX, typename TV, typename TZ, typename TXS>
void launch_update(const UpdateArgs<TX, TV, TZ, TXS>& u, int grid, cudaStream_t s) {
  launch_pdl(update_kernel<TX, TV, TZ, TXS>, grid, 256, 0, s, u);
}

template <typename TX>
void launch_chom(const ChomArgs<TX>& c, int grid, cudaStream_t s) {
  chom_kernel<TX><<<grid, 32, 0, s>>>(c);
}

template void launch_setup<double, double>(const int*, int, int, int, const double*, double,
                                           double*, double*, cudaStream_t);
template void launch_setup<double, float>(const int*, int, int, int, const double*, double, double*,
                                          float*, cudaStream_t);
template void launch_setup<float, float>(const int*, int, int, int, const double*, double, float*,
                                         float*, cudaStream_t);
template void launch_apply<double, double>(const ApplyArgs<double, double>&, int, cudaStream_t);
template void launch_apply<double, float>(const ApplyArgs<double, float>&, int, cudaStream_t);
template void launch_apply<float, float>(const ApplyArgs<float, float>&, int, cudaStream_t);
template void launch_update<double, double, double>(const UpdateArgs<double, double>&, int, cudaStream_t);
template void launch_update<double, double, float>(const UpdateArgs<double, double, float>&, int, cudaStream_t);
template void launch_update<double, double, float, float>(const UpdateArgs<double, double, float, float>&, int,
                                                         cudaStream_t);
template void launch_update<double, float, float>(const UpdateArgs<double, float>&, int, cudaStream_t);
template void launch_update<float, float, float>(const UpdateArgs<float, float>&, int, cudaStream_t);
template void launch_chom<double>(const ChomArgs<double>&, int, cudaStream_t);
template void launch_chom<float>(const ChomArgs<float>&, int, cudaStream_t);

}  // namespace shl
