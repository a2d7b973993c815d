// gmg.cuh -- geometric multigrid preconditioner kernels (included by solver.cu,
// which owns the __constant__ element matrices).
//
// Hierarchy on the periodic torus: level 0 is the matrix-free masked operator
// (fine_gather); level l+1 has r/2^(l+1) nodes per axis and the Galerkin
// operator A_{l+1} = P^T A_l P for trilinear interpolation P (weights 1, 1/2
// per axis, periodic), restricted to coarse nodes whose support touches an
// active fine node.  Coarse operators are stored as 27-point stencils of 3x3
// blocks (243 values per node, 32-node blocked like every vector).  Galerkin
// coarsening keeps the masked, 1e3-contrast shell operator faithful on every
// level (no re-discretization of void/floor voxels).  The pinned node 0 is a
// zero row/column on every level.  Smoother: damped 3x3 block Jacobi.
//
// All vectors carry the six load cases x three components (18 per node).

namespace {

constexpr int kStencil = 243;

// Thread t -> (node, load case) with each warp on ONE load case of 32
// consecutive nodes, so a warp's access to a component plane of the 32-node
// blocked vectors is one contiguous 128-byte line (t/6, t%6 spread a warp over
// six planes of ~5 nodes each).  Launch ceil(n/32)*192 threads.
__device__ __forceinline__ void node_case(long long t, int& idx, int& s) {
  const long long w = t >> 5;
  idx = static_cast<int>((w / 6) * 32 + (t & 31));
  s = static_cast<int>(w % 6);
}
__host__ __device__ inline unsigned node_case_blocks(int n, int threads_per_block) {
  return static_cast<unsigned>((static_cast<long long>((n + 31) / 32) * 192 + threads_per_block - 1) /
                               threads_per_block);
}


template <typename TV>
struct LevelArgs {
  const int* node_list;
  const int* node_map;
  const TV* beta;     // level 0 only (dense r^3)
  const TV* stencil;  // levels >= 1
  const TV* dinv;     // 6 per node
  int r, n, zero_slot;
  TV ridge;           // level 0 only
  int zbase;          // level 0 of a z-slab (0 otherwise)
  double* totals;     // mode 2: write the r.z sums here instead of finalizing (slabs)
  int n0;             // nodes [n0, n) are swept (a z-slab's owned level-1 planes; 0 otherwise)
};

// stencil_gather restricted to neighbour plane dz = PLANE-1.
template <typename TV, int PLANE>
__device__ __forceinline__ void stencil_gather_plane(GatherAcc<TV>& acc, int idx, int g,
                                                     const TV* __restrict__ xv,
                                                     const TV* __restrict__ stencil,
                                                     const int* __restrict__ nmap, int r, int zero_slot) {
  acc.zero();
  if (g == 0) return;
  const int rr = r * r;
  const int i = g % r, j = (g / r) % r, k = g / rr;
  const int xs[3] = {i == 0 ? r - 1 : i - 1, i, i == r - 1 ? 0 : i + 1};
  const int ys[3] = {(j == 0 ? r - 1 : j - 1) * r, j * r, (j == r - 1 ? 0 : j + 1) * r};
  constexpr int dz = PLANE - 1;
  const int zl = (dz < 0 ? (k == 0 ? r - 1 : k - 1) : (dz > 0 ? (k == r - 1 ? 0 : k + 1) : k)) * rr;
  const TV* sb = stencil + vbase(idx, kStencil);
#pragma unroll
  for (int mm = 0; mm < 9; ++mm) {
    const int m = PLANE * 9 + mm;
    const int dx = mm % 3 - 1, dy = mm / 3 - 1;
    const int nb = (m == 13) ? idx : nmap[zl + ys[dy + 1] + xs[dx + 1]];
    if (nb < 0) continue;  // absent neighbour: no coupling
    TV S[9];
    if (m < 13) {
      // backward neighbour: the Galerkin operator is symmetric, S_m(n) =
      // S_{26-m}(n+m)^T, so read the neighbour's forward block transposed.
      // Each forward block is then read twice in a sweep (by its node and by
      // that neighbour), the second time mostly from L2: the stencils' DRAM
      // traffic halves, and the operator applied is exactly symmetric.
      const TV* sn = stencil + vbase(nb, kStencil) + (26 - m) * 9 * 32;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) S[c * 3 + d] = sn[(d * 3 + c) * 32];
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) S[q] = sb[(m * 9 + q) * 32];
    }
    acc.add(S, xv + vbase(nb, 18));
  }
  (void)zero_slot;
}

// level_sweep_kernel latency-split three ways: three warps per 32 nodes, warp p
// gathers plane dz=p-1, warp p then finishes load-case pair p (gather3_tile).
// kQueue: CTAs take 64-node tiles from the shared counter (level 0 of the
// z-slabs); otherwise one CTA per tile (grid = tiles: the stored levels, no
// tile atomics, and lanes cannot leave a CTA with a late full share).
template <typename TB, typename TV, bool kFine, typename TO = TV, bool kQueue = kFine>
__global__ void __launch_bounds__(192)
    level_sweep3_kernel(const LevelArgs<TV> L, const TB* __restrict__ b, const TV* __restrict__ xin,
                        TO* __restrict__ xout, TV omega, int mode, PcgState* st, double* partials,
                        int init) {
  pdl_wait();
  __shared__ __align__(16) TV part_s[2][3 * 18 * 32];
  __shared__ double scratch[32 * 6];
  if (st->stop) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = w / 3, part = w % 3;
  double gam2[2] = {0, 0};
  // tiles from the shared counter; mode 2 reduces r.z per tile (fixed order,
  // see apply6_kernel) so the sum does not depend on which CTA ran which tile
  __shared__ double red[2][6];
  __shared__ int tq_slot[2];
  TileQueue tq{&st->tile_next[1], tq_slot};
  for (int tile = kQueue ? tq.first() : static_cast<int>(blockIdx.x);; tile = tq.advance()) {
    if (L.n0 + tile * 64 >= L.n) break;
    if (kQueue) tq.request();
    gam2[0] = gam2[1] = 0.0;
    const int idx = L.n0 + tile * 64 + grp * 32 + lane;
    const bool valid = idx < L.n;
    const int g = valid ? L.node_list[idx] : -1;
    {
      GatherAcc<TV> acc;
      if (!valid) {
        acc.zero();
      } else if (kFine) {
        if (part == 0)
          fine_gather_plane<TV, 0>(acc, idx, g, xin, L.beta, L.node_map, L.r, L.zbase, L.zero_slot);
        else if (part == 1)
          fine_gather_plane<TV, 1>(acc, idx, g, xin, L.beta, L.node_map, L.r, L.zbase, L.zero_slot);
        else
          fine_gather_plane<TV, 2>(acc, idx, g, xin, L.beta, L.node_map, L.r, L.zbase, L.zero_slot);
      } else {
        if (part == 0)
          stencil_gather_plane<TV, 0>(acc, idx, g, xin, L.stencil, L.node_map, L.r, L.zero_slot);
        else if (part == 1)
          stencil_gather_plane<TV, 1>(acc, idx, g, xin, L.stencil, L.node_map, L.r, L.zero_slot);
        else
          stencil_gather_plane<TV, 2>(acc, idx, g, xin, L.stencil, L.node_map, L.r, L.zero_slot);
      }
#pragma unroll
      for (int q = 0; q < 18; ++q) part_s[grp][(part * 18 + q) * 32 + lane] = acc.get(q);
    }
    if (kQueue) tq.publish();
    __syncthreads();
    if (valid) {
      const size_t ob = vbase(idx, 18);
      TV D[6];
      if (mode != 1) {
#pragma unroll
        for (int q = 0; q < 6; ++q) D[q] = L.dinv[vbase(idx, 6) + q * 32];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int s_ = 2 * part + k;
        TV res[3], xo[3], bb[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const size_t o = ob + (c * 6 + s_) * 32;
          const TV xi = xin[o];
          TV wv = gather3_sum<TV>(part_s[grp], c * 6 + s_, lane);
          if (kFine && g != 0) wv = fma_t(L.ridge, xi, wv);
          bb[c] = static_cast<TV>(b[o]);
          res[c] = bb[c] - wv;
          xo[c] = xi;
        }
        if (mode == 1) {
#pragma unroll
          for (int c = 0; c < 3; ++c) xout[ob + (c * 6 + s_) * 32] = static_cast<TO>(g == 0 ? TV(0) : res[c]);
          continue;
        }
        const TV z0 = D[0] * res[0] + D[1] * res[1] + D[2] * res[2];
        const TV z1 = D[1] * res[0] + D[3] * res[1] + D[4] * res[2];
        const TV z2 = D[2] * res[0] + D[4] * res[1] + D[5] * res[2];
        xo[0] = fma_t(omega, z0, xo[0]);
        xo[1] = fma_t(omega, z1, xo[1]);
        xo[2] = fma_t(omega, z2, xo[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xout[ob + (c * 6 + s_) * 32] = static_cast<TO>(xo[c]);
          if (mode == 2) gam2[k] += static_cast<double>(b[ob + (c * 6 + s_) * 32]) * static_cast<double>(xo[c]);
        }
      }
    }
    if (mode == 2) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gam2[k] += __shfl_xor_sync(0xffffffffu, gam2[k], o);
        if (lane == 0) red[grp][2 * part + k] = gam2[k];
      }
    }
    __syncthreads();
    if (mode == 2 && threadIdx.x < 6) partials[tile * 6 + threadIdx.x] = red[0][threadIdx.x] + red[1][threadIdx.x];
    if (!kQueue) break;
  }
  if (!kQueue) return;  // (stored levels: mode 0 / 1 only)
  tiles_done(&st->tile_next[1], &st->tile_done[1]);
  if (mode != 2) return;
  __shared__ bool last;
  __syncthreads();  // every thread's partial writes ordered before thread 0's release
  if (threadIdx.x == 0) last = arrive_last(&st->counter_misc);
  __syncthreads();
  if (!last) return;
  const int ntiles = (L.n + 63) / 64;
  double tot[6] = {0, 0, 0, 0, 0, 0};
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x)
#pragma unroll
    for (int q = 0; q < 6; ++q) tot[q] += __ldcg(partials + t * 6 + q);
  block_sum<6>(tot, scratch);
  if (threadIdx.x == 0) {
    if (L.totals) {
      for (int q = 0; q < 6; ++q) L.totals[q] = tot[q];
    } else {
      finalize_gamma_state(st, tot, init);
    }
    st->counter_misc = 0;
  }
}

// Stored (Galerkin) levels are small, so a per-node loop over 27 neighbours is
// a pure dependent-load chain (~30 us per sweep regardless of size).  Here one
// WARP owns a node and lane m < 27 owns stencil neighbour m: each lane does one
// node-map lookup and one block-times-vector (9 x 6 FMA), a butterfly shuffle
// sums the 18 outputs, and lanes 0..5 finish load case s = lane.
template <typename TV>
__device__ __forceinline__ void coarse_warp_node(const LevelArgs<TV>& L, const TV* __restrict__ b,
                                                 const TV* __restrict__ xin, TV* __restrict__ xout, TV omega,
                                                 int mode, int idx, int lane) {
  const int g = L.node_list[idx];
  TV y[18];
#pragma unroll
  for (int q = 0; q < 18; ++q) y[q] = TV(0);
  if (g != 0 && lane < 27) {
    const int r = L.r, rr = r * r;
    const int i = g % r, j = (g / r) % r, k = g / rr;
    const int dx = lane % 3 - 1, dy = (lane / 3) % 3 - 1, dz = lane / 9 - 1;
    const int xi = (i + dx + r) % r, yj = (j + dy + r) % r, zk = (k + dz + r) % r;
    int nb = (lane == 13) ? idx : L.node_map[(zk * r + yj) * r + xi];
    if (nb >= 0) {
      const TV* S = L.stencil + vbase(idx, kStencil) + lane * 9 * 32;
      const TV* xm = xin + vbase(nb, 18);
      TV Sv[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) Sv[q] = S[q * 32];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const TV x0 = xm[s * 32], x1 = xm[(6 + s) * 32], x2 = xm[(12 + s) * 32];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          y[c * 6 + s] = fma_t(Sv[c * 3 + 0], x0, fma_t(Sv[c * 3 + 1], x1, Sv[c * 3 + 2] * x2));
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 18; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y[q] += __shfl_xor_sync(0xffffffffu, y[q], o);
  if (lane >= 6) return;
  const int sl = lane;
  const size_t ob = vbase(idx, 18) + sl * 32;
  if (g == 0) {
    xout[ob] = xout[ob + 192] = xout[ob + 384] = TV(0);
    return;
  }
  // select this lane's load case without dynamic register indexing
  TV y0 = y[sl], y1 = y[6 + sl], y2 = y[12 + sl];
#pragma unroll
  for (int s = 0; s < 6; ++s)
    if (s == sl) {
      y0 = y[s];
      y1 = y[6 + s];
      y2 = y[12 + s];
    }
  const TV r0 = b[ob] - y0, r1 = b[ob + 192] - y1, r2 = b[ob + 384] - y2;
  if (mode == 1) {
    xout[ob] = r0;
    xout[ob + 192] = r1;
    xout[ob + 384] = r2;
    return;
  }
  TV D[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) D[q] = L.dinv[vbase(idx, 6) + q * 32];
  xout[ob] = fma_t(omega, D[0] * r0 + D[1] * r1 + D[2] * r2, xin[ob]);
  xout[ob + 192] = fma_t(omega, D[1] * r0 + D[3] * r1 + D[4] * r2, xin[ob + 192]);
  xout[ob + 384] = fma_t(omega, D[2] * r0 + D[4] * r1 + D[5] * r2, xin[ob + 384]);
}

// Stored (Galerkin) levels are small, so a per-node loop over 27 neighbours is
// a pure dependent-load chain (~30 us per sweep regardless of size).  Here one
// WARP owns a node and lane m < 27 owns stencil neighbour m: each lane does one
// node-map lookup and one block-times-vector (9 x 6 FMA), a butterfly shuffle
// sums the 18 outputs, and lanes 0..5 finish load case s = lane.
template <typename TV>
__global__ void __launch_bounds__(256) coarse_warp_sweep_kernel(const LevelArgs<TV> L, const TV* __restrict__ b,
                                                                const TV* __restrict__ xin, TV* __restrict__ xout,
                                                                TV omega, int mode, const PcgState* st) {
  pdl_wait();
  if (st->stop) return;
  const int warp = L.n0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (warp >= L.n) return;  // whole warps exit together
  coarse_warp_node<TV>(L, b, xin, xout, omega, mode, warp, lane);
}

// ---- coarsest level (8^3 torus) as one thread-block cluster ---------------------
// The coarsest solve is jacobi_first + (sweeps - 1) damped block-Jacobi sweeps
// over <= 512 nodes: as separate launches each sweep costs a launch and a
// grid-wide dependency for ~6 us of latency (about 10% of a PCG iteration at
// 128^3).  Here one cluster of 8 CTAs runs them all: CTA c owns z-plane c,
// keeps its nodes' stencils (up to 64 x 243) in shared memory and its plane of
// the iterate as a dense 8x8 plane (absent positions 0, so no node-map
// lookups), double-buffered; each sweep starts with one cluster barrier and a
// vectorized read of the two neighbour planes from the neighbours' shared
// memory (distributed shared memory).  Same arithmetic as jacobi_first +
// coarse_warp_sweep_kernel (mode 0) up to the summation order of the 27
// neighbour blocks.
constexpr int kCoR = 8;                // coarsest grid (nodes per axis) this kernel takes
constexpr int kCoP = kCoR * kCoR;      // positions per plane
constexpr int kCoThreads = 3 * kCoP;   // (node, neighbour plane) per thread
constexpr int kCoPlane = 9 * kCoP;     // float2 per plane: [component][load-case pair][position]
struct CoarsestShared {
  float S[kStencil][kCoP];             // own nodes' stencils [m*9 + q][local node]
  float2 own[2][kCoPlane];             // own plane c, double-buffered
  float2 nb[2][kCoPlane];              // copies of planes c-1 and c+1 for the current sweep
  float part[3][18][kCoP];             // per-neighbour-plane partial A x
  float b[18][kCoP];
  float D[6][kCoP];
  short pos[kCoP];                     // position of local node u in its plane
  int range[2];                        // own id range [lo, hi)
};

__global__ void __cluster_dims__(kCoR, 1, 1) __launch_bounds__(kCoThreads, 1)
    coarsest_cluster_kernel(const int* __restrict__ node_list, int n, const float* __restrict__ stencil,
                            const float* __restrict__ dinv, const float* __restrict__ b, float* __restrict__ x,
                            float omega, int sweeps, const PcgState* st) {
  namespace cg = cooperative_groups;
  pdl_wait();
  if (st->stop) return;  // (uniform: every CTA of the cluster returns)
  extern __shared__ __align__(16) unsigned char co_raw[];
  CoarsestShared& C = *reinterpret_cast<CoarsestShared*>(co_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int c = static_cast<int>(cl.block_rank()), tid = threadIdx.x;
  // own id range: node ids are ordered by grid index, plane c = ids with g / 64 == c
  if (tid < 2) C.range[tid] = 0;
  for (int e = tid; e < 2 * kCoPlane; e += kCoThreads) (&C.own[0][0])[e] = make_float2(0.f, 0.f);
  __syncthreads();
  int below = 0, upto = 0;
  for (int i = tid; i < n; i += kCoThreads) {
    const int g = node_list[i];
    below += g < c * kCoP;
    upto += g < (c + 1) * kCoP;
  }
  if (below) atomicAdd(&C.range[0], below);
  if (upto) atomicAdd(&C.range[1], upto);
  __syncthreads();
  const int lo = C.range[0], nl = C.range[1] - C.range[0];
  // stage the own nodes' stencils, rhs and Dinv (cp.async: every load in flight at once)
  for (int e = tid; e < kStencil * kCoP; e += kCoThreads) {
    const int q = e / kCoP, u = e % kCoP;
    if (u < nl)
      cp_async<4>(&C.S[q][u], stencil + vbase(lo + u, kStencil) + q * 32);
    else
      C.S[q][u] = 0.f;
  }
  for (int e = tid; e < 18 * kCoP; e += kCoThreads) {
    const int q = e / kCoP, u = e % kCoP;
    if (u < nl)
      cp_async<4>(&C.b[q][u], b + vbase(lo + u, 18) + q * 32);
    else
      C.b[q][u] = 0.f;
  }
  for (int e = tid; e < 6 * kCoP; e += kCoThreads) {
    const int q = e / kCoP, u = e % kCoP;
    if (u < nl)
      cp_async<4>(&C.D[q][u], dinv + vbase(lo + u, 6) + q * 32);
    else
      C.D[q][u] = 0.f;
  }
  cp_async_commit();
  if (tid < nl) C.pos[tid] = static_cast<short>(node_list[lo + tid] - c * kCoP);
  cp_async_wait<0>();
  __syncthreads();
  const float4* own_lo = reinterpret_cast<const float4*>(cl.map_shared_rank(&C.own[0][0], (c + kCoR - 1) % kCoR));
  const float4* own_hi = reinterpret_cast<const float4*>(cl.map_shared_rank(&C.own[0][0], (c + 1) % kCoR));
  const bool pinned0 = c == 0 && nl > 0 && node_list[lo] == 0;  // node 0 stays 0
  float* const ownf = reinterpret_cast<float*>(&C.own[0][0]);
  // x_new of this thread's (node, load case) pairs into own[nb]
  auto finish = [&](int nb, bool first) {
    for (int k = tid; k < 6 * kCoP; k += kCoThreads) {
      const int u = k % kCoP, s_ = k / kCoP;
      if (u >= nl) continue;
      const int ps = C.pos[u];
      float xo[3];
      if (first) {  // from x = 0: x = w Dinv b
        const float r0 = C.b[s_][u], r1 = C.b[6 + s_][u], r2 = C.b[12 + s_][u];
        xo[0] = omega * (C.D[0][u] * r0 + C.D[1][u] * r1 + C.D[2][u] * r2);
        xo[1] = omega * (C.D[1][u] * r0 + C.D[3][u] * r1 + C.D[4][u] * r2);
        xo[2] = omega * (C.D[2][u] * r0 + C.D[4][u] * r1 + C.D[5][u] * r2);
      } else {
        float res[3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const int q = cc * 6 + s_;
          res[cc] = C.b[q][u] - (C.part[0][q][u] + C.part[1][q][u] + C.part[2][q][u]);
          xo[cc] = ownf[(((nb ^ 1) * 3 + cc) * 3 * kCoP + (s_ >> 1) * kCoP + ps) * 2 + (s_ & 1)];
        }
        xo[0] = fma_t(omega, C.D[0][u] * res[0] + C.D[1][u] * res[1] + C.D[2][u] * res[2], xo[0]);
        xo[1] = fma_t(omega, C.D[1][u] * res[0] + C.D[3][u] * res[1] + C.D[4][u] * res[2], xo[1]);
        xo[2] = fma_t(omega, C.D[2][u] * res[0] + C.D[4][u] * res[1] + C.D[5][u] * res[2], xo[2]);
      }
      if (pinned0 && u == 0) xo[0] = xo[1] = xo[2] = 0.f;
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        ownf[((nb * 3 + cc) * 3 * kCoP + (s_ >> 1) * kCoP + ps) * 2 + (s_ & 1)] = xo[cc];
    }
  };
  finish(0, true);
  const int pl = tid / kCoP, u = tid % kCoP;  // gather: neighbour plane pl (dz = pl - 1) of local node u
  for (int k = 1; k < sweeps; ++k) {
    const int cur = (k - 1) & 1;
    cl.sync();  // every plane of sweep k-1 complete
    {
      float4* dst = reinterpret_cast<float4*>(&C.nb[0][0]);
      constexpr int kV = kCoPlane / 2;  // float4 per plane
      for (int e = tid; e < 2 * kV; e += kCoThreads)
        dst[e] = e < kV ? own_lo[cur * kV + e] : own_hi[cur * kV + e - kV];
    }
    __syncthreads();
    if (u < nl) {
      const int ps = C.pos[u], i = ps % kCoR, j = ps / kCoR;
      const float2* xp = pl == 1 ? C.own[cur] : C.nb[pl >> 1];
      float2 y[9];  // [component][load-case pair], packed FFMA2 over the pair
#pragma unroll
      for (int q = 0; q < 9; ++q) y[q] = make_float2(0.f, 0.f);
#pragma unroll
      for (int mm = 0; mm < 9; ++mm) {
        const int dx = mm % 3 - 1, dy = mm / 3 - 1, m = pl * 9 + mm;
        const int np = ((i + dx + kCoR) % kCoR) + kCoR * ((j + dy + kCoR) % kCoR);
        float Sv[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) Sv[q] = C.S[m * 9 + q][u];
#pragma unroll
        for (int sp = 0; sp < 3; ++sp) {
          const float2 x0 = xp[(0 * 3 + sp) * kCoP + np], x1 = xp[(1 * 3 + sp) * kCoP + np],
                       x2 = xp[(2 * 3 + sp) * kCoP + np];
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            float2 v = y[cc * 3 + sp];
            v = __ffma2_rn(make_float2(Sv[cc * 3 + 2], Sv[cc * 3 + 2]), x2, v);
            v = __ffma2_rn(make_float2(Sv[cc * 3 + 1], Sv[cc * 3 + 1]), x1, v);
            v = __ffma2_rn(make_float2(Sv[cc * 3 + 0], Sv[cc * 3 + 0]), x0, v);
            y[cc * 3 + sp] = v;
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
#pragma unroll
        for (int sp = 0; sp < 3; ++sp) {
          C.part[pl][cc * 6 + 2 * sp][u] = y[cc * 3 + sp].x;
          C.part[pl][cc * 6 + 2 * sp + 1][u] = y[cc * 3 + sp].y;
        }
    }
    __syncthreads();
    finish(cur ^ 1, false);
  }
  __syncthreads();
  const int fin = (sweeps - 1) & 1;
  for (int k = tid; k < 18 * kCoP; k += kCoThreads) {
    const int q = k / kCoP, uu = k % kCoP, cc = q / 6, s_ = q % 6;
    if (uu < nl) x[vbase(lo + uu, 18) + q * 32] = ownf[((fin * 3 + cc) * 3 * kCoP + (s_ >> 1) * kCoP + C.pos[uu]) * 2 + (s_ & 1)];
  }
  cl.sync();  // no CTA leaves while a neighbour may still read its plane
}

// first sweep from x = 0: xout = w Dinv b (pointwise)
template <typename TB, typename TV>
__global__ void jacobi_first_kernel(const int* __restrict__ node_list, const TV* __restrict__ dinv,
                                    int n, const TB* __restrict__ b, TV* __restrict__ xout, TV omega,
                                    const PcgState* st, int n0) {
  pdl_wait();
  if (st->stop) return;
  int idx, s;
  node_case(blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x, idx, s);
  idx += n0;
  if (idx >= n) return;
  const size_t ob = vbase(idx, 18) + s * 32;
  TV D[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) D[q] = dinv[vbase(idx, 6) + q * 32];
  const TV r0 = static_cast<TV>(b[ob]), r1 = static_cast<TV>(b[ob + 192]), r2 = static_cast<TV>(b[ob + 384]);
  xout[ob] = omega * (D[0] * r0 + D[1] * r1 + D[2] * r2);
  xout[ob + 192] = omega * (D[1] * r0 + D[3] * r1 + D[4] * r2);
  xout[ob + 384] = omega * (D[2] * r0 + D[4] * r1 + D[5] * r2);
  (void)node_list;
}

// ---------------------------------------------------------------- transfers
// b_c(N) = sum_{n in supp(N)} w(n,N) res_f(n), w = prod over axes (1 | 1/2)
// (f1 > 0: only fine ids in [f0, f1) contribute and b_c accumulates -- the
// partial restriction of a z-slab's owned level-1 nodes, summed over slabs)
// (x_c != nullptr: also the coarse level's first damped Jacobi sweep from
// x = 0, x_c = omega Dinv b_c -- jacobi_first_kernel fused into the
// restriction that produces b_c, same arithmetic)
template <typename TV>
__global__ void restrict_kernel(const int* __restrict__ list_c, int n_c, int r_c,
                                const int* __restrict__ map_f, int r_f, const TV* __restrict__ res_f,
                                TV* __restrict__ b_c, const PcgState* st, int f0 = 0, int f1 = 0,
                                const TV* __restrict__ dinv_c = nullptr, TV* __restrict__ x_c = nullptr,
                                TV omega = TV(0)) {
  pdl_wait();
  if (st->stop) return;
  int idx, s;
  node_case(blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x, idx, s);
  if (idx >= n_c) return;
  const int G = list_c[idx];
  const int I = G % r_c, J = (G / r_c) % r_c, K = G / (r_c * r_c);
  TV acc[3] = {TV(0), TV(0), TV(0)};
  if (G != 0) {
    // the 27 map lookups first (all in flight at once), then the gathers
    int fx[3], fy[3], fz[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      fx[d] = (2 * I + d - 1 + r_f) % r_f;
      fy[d] = (2 * J + d - 1 + r_f) % r_f;
      fz[d] = (2 * K + d - 1 + r_f) % r_f;
    }
    int nf[27];
#pragma unroll
    for (int m = 0; m < 27; ++m)
      nf[m] = map_f[(static_cast<size_t>(fz[m / 9]) * r_f + fy[(m / 3) % 3]) * r_f + fx[m % 3]];
#pragma unroll
    for (int m = 0; m < 27; ++m) {
      if (nf[m] < 0 || (f1 > 0 && (nf[m] < f0 || nf[m] >= f1))) continue;
      const int di = m % 3 - 1, dj = (m / 3) % 3 - 1, dk = m / 9 - 1;
      const TV w = TV((di ? 0.5 : 1.0) * (dj ? 0.5 : 1.0) * (dk ? 0.5 : 1.0));
      const size_t o = vbase(nf[m], 18) + s * 32;
      acc[0] = fma_t(w, res_f[o], acc[0]);
      acc[1] = fma_t(w, res_f[o + 192], acc[1]);
      acc[2] = fma_t(w, res_f[o + 384], acc[2]);
    }
  }
  const size_t oc = vbase(idx, 18) + s * 32;
  if (f1 > 0) {
    b_c[oc] += acc[0];
    b_c[oc + 192] += acc[1];
    b_c[oc + 384] += acc[2];
  } else {
    b_c[oc] = acc[0];
    b_c[oc + 192] = acc[1];
    b_c[oc + 384] = acc[2];
    if (x_c) {
      TV D[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) D[q] = dinv_c[vbase(idx, 6) + q * 32];
      x_c[oc] = omega * (D[0] * acc[0] + D[1] * acc[1] + D[2] * acc[2]);
      x_c[oc + 192] = omega * (D[1] * acc[0] + D[3] * acc[1] + D[4] * acc[2]);
      x_c[oc + 384] = omega * (D[2] * acc[0] + D[4] * acc[1] + D[5] * acc[2]);
    }
  }
}

// z-slab restriction onto the slab's OWNED coarse (level-1) nodes [c0, c1)
// from the slab's level-0 residual, ghost planes included (the coarse planes a
// slab owns gather fine planes z0-1 .. z1, all inside its local node map)
template <typename TV>
__global__ void restrict_own_kernel(const int* __restrict__ list_c, int c0, int c1, int r_c,
                                    const int* __restrict__ map_s, int zbase, int nzl, int r_f,
                                    const TV* __restrict__ res_f, TV* __restrict__ b_c, const PcgState* st) {
  pdl_wait();
  if (st->stop) return;
  int idx, s;
  node_case(blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x, idx, s);
  idx += c0;
  if (idx >= c1) return;
  SHL_DCHECK(c0 >= 0 && c0 <= c1);
  const int G = list_c[idx];
  const int I = G % r_c, J = (G / r_c) % r_c, K = G / (r_c * r_c);
  TV acc[3] = {TV(0), TV(0), TV(0)};
  if (G != 0) {
    for (int dk = -1; dk <= 1; ++dk) {
      int lz = (2 * K + dk + r_f) % r_f - zbase;
      lz += lz < 0 ? r_f : 0;
      if (lz >= nzl) continue;  // (never for an owned coarse plane)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int fi = (2 * I + di + r_f) % r_f, fj = (2 * J + dj + r_f) % r_f;
          const int nf = map_s[(static_cast<size_t>(lz) * r_f + fj) * r_f + fi];
          if (nf < 0) continue;
          const TV w = TV((di ? 0.5 : 1.0) * (dj ? 0.5 : 1.0) * (dk ? 0.5 : 1.0));
          const size_t o = vbase(nf, 18) + s * 32;
          acc[0] = fma_t(w, res_f[o], acc[0]);
          acc[1] = fma_t(w, res_f[o + 192], acc[1]);
          acc[2] = fma_t(w, res_f[o + 384], acc[2]);
        }
    }
  }
  SHL_DCHECK(G != 0 || idx == 0);
  const size_t oc = vbase(idx, 18) + s * 32;
  b_c[oc] = acc[0];
  b_c[oc + 192] = acc[1];
  b_c[oc + 384] = acc[2];
}

// z-slab restriction: the slab's OWNED fine nodes only, accumulated into b_c
template <typename TV>
__global__ void restrict_slab_kernel(const int* __restrict__ list_c, int n_c, int r_c, const int* __restrict__ map_s,
                                     int zbase, int nzl, int z0, int z1, int r_f, const TV* __restrict__ res_f,
                                     TV* __restrict__ b_c, const PcgState* st) {
  if (st->stop) return;
  int idx, s;
  node_case(blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x, idx, s);
  if (idx >= n_c) return;
  const int G = list_c[idx];
  const int I = G % r_c, J = (G / r_c) % r_c, K = G / (r_c * r_c);
  TV acc[3] = {TV(0), TV(0), TV(0)};
  bool any = false;
  if (G != 0) {
    for (int dk = -1; dk <= 1; ++dk) {
      const int fk = (2 * K + dk + r_f) % r_f;
      if (fk < z0 || fk >= z1) continue;  // not owned by this slab
      int lz = fk - zbase;
      lz += lz < 0 ? r_f : 0;
      if (lz >= nzl) continue;
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int fi = (2 * I + di + r_f) % r_f, fj = (2 * J + dj + r_f) % r_f;
          const int nf = map_s[(static_cast<size_t>(lz) * r_f + fj) * r_f + fi];
          if (nf < 0) continue;
          const TV w = TV((di ? 0.5 : 1.0) * (dj ? 0.5 : 1.0) * (dk ? 0.5 : 1.0));
          const size_t o = vbase(nf, 18) + s * 32;
          acc[0] = fma_t(w, res_f[o], acc[0]);
          acc[1] = fma_t(w, res_f[o + 192], acc[1]);
          acc[2] = fma_t(w, res_f[o + 384], acc[2]);
          any = true;
        }
    }
  }
  if (!any) return;
  const size_t oc = vbase(idx, 18) + s * 32;
  b_c[oc] += acc[0];
  b_c[oc + 192] += acc[1];
  b_c[oc + 384] += acc[2];
}

// x_f(n) += sum_N w(n,N) x_c(N) over the 1..8 coarse parents of n.  One
// thread per fine node and all 18 components: the parent lookup (two integer
// divisions and up to 8 dependent map loads) is done once per node, not once
// per load case.
template <typename TV>
__global__ void __launch_bounds__(128) prolong_kernel(const int* __restrict__ list_f, int n_f, int r_f,
                                                      const int* __restrict__ map_c, int r_c,
                                                      const TV* __restrict__ x_c, TV* __restrict__ x_f,
                                                      const PcgState* st, int n0) {
  pdl_wait();
  if (st->stop) return;
  const int idx = n0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_f) return;
  const int g = list_f[idx];
  if (g == 0) return;
  const int i = g % r_f, j = (g / r_f) % r_f, k = g / (r_f * r_f);
  const int pi[2] = {i >> 1, ((i + 1) >> 1) % r_c}, pj[2] = {j >> 1, ((j + 1) >> 1) % r_c},
            pk[2] = {k >> 1, ((k + 1) >> 1) % r_c};
  const int ni = (i & 1) ? 2 : 1, nj = (j & 1) ? 2 : 1, nk = (k & 1) ? 2 : 1;
  int nc[8];  // parents in (c, b, a) order, -1 where absent
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int a = u & 1, b = (u >> 1) & 1, c = u >> 2;
    nc[u] = (a < ni && b < nj && c < nk) ? map_c[(static_cast<size_t>(pk[c]) * r_c + pj[b]) * r_c + pi[a]] : -1;
  }
  const TV w = TV(1.0 / (ni * nj * nk));
  const size_t of = vbase(idx, 18);
  TV acc[18], xf[18];
#pragma unroll
  for (int q = 0; q < 18; ++q) {
    acc[q] = TV(0);
    xf[q] = x_f[of + q * 32];
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if (nc[u] < 0) continue;
    const size_t o = vbase(nc[u], 18);
#pragma unroll
    for (int q = 0; q < 18; ++q) acc[q] += x_c[o + q * 32];
  }
#pragma unroll
  for (int q = 0; q < 18; ++q) x_f[of + q * 32] = fma_t(w, acc[q], xf[q]);
}

// ---------------------------------------------------------------- setup
// brick (8x4x4 positions of a coarse level, r % 8 == 0, r % 4 == 0) active iff
// one of its nodes is
__global__ void coarse_brick_flag_kernel(const int* __restrict__ map, int r, int* __restrict__ flag) {
  const int nbx = r / 8, nby = r / 4, nb = nbx * nby * (r / 4);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb) return;
  const int x0 = (t % nbx) * 8, y0 = ((t / nbx) % nby) * 4, z0 = (t / (nbx * nby)) * 4;
  int any = 0;
  for (int k = 0; k < 128 && !any; ++k)
    any = map[(static_cast<size_t>(z0 + (k >> 5)) * r + y0 + ((k >> 3) & 3)) * r + x0 + (k & 7)] >= 0;
  flag[t] = any;
}

// coarse node active iff a fine node of its support is active
__global__ void coarse_flag_kernel(const int* __restrict__ map_f, int r_f, int r_c,
                                   int* __restrict__ flag_c) {
  const size_t n3 = static_cast<size_t>(r_c) * r_c * r_c;
  const size_t G = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (G >= n3) return;
  const int I = static_cast<int>(G % r_c), J = static_cast<int>((G / r_c) % r_c),
            K = static_cast<int>(G / (static_cast<size_t>(r_c) * r_c));
  int on = 0;
  for (int dk = -1; dk <= 1 && !on; ++dk)
    for (int dj = -1; dj <= 1 && !on; ++dj)
      for (int di = -1; di <= 1 && !on; ++di) {
        const int fi = (2 * I + di + r_f) % r_f, fj = (2 * J + dj + r_f) % r_f, fk = (2 * K + dk + r_f) % r_f;
        on = map_f[(static_cast<size_t>(fk) * r_f + fj) * r_f + fi] >= 0;
      }
  flag_c[G] = on;
}

// ---- level-1 Galerkin from elements -------------------------------------
// Inside one coarse cell the trilinear P maps the cell's 8 coarse corners onto
// the 27 fine nodes of its 8 fine elements, so P^T A_f P restricted to the cell
// is sum_j beta_j M_j with M_j = P_j^T K0 P_j (24x24, coarse corners in bit
// order x + 2y + 4z).  A_1(N, N+D) is then plain element assembly over the (up
// to 8) cells holding both N and N+D: 8 fine elements x 9 FMA per cell.  Rows
// and columns through fine node 0 only reach coarse node 0, whose row is zero
// and whose value is held at zero, so the operator equals the node-wise form.
__device__ double g_cellMd[8 * 576];
__device__ float g_cellMf[8 * 576];

__device__ __forceinline__ double tri_w(int t, int cc) {  // fine offset t in {0,1,2} from corner cc
  return t == 1 ? 0.5 : ((t == 0) == (cc == 0) ? 1.0 : 0.0);
}

__global__ void cell_matrices_kernel() {
  const int j = blockIdx.x, e = threadIdx.x;
  const int row = e / 24, col = e % 24;
  const int C = row / 3, c = row % 3, C2 = col / 3, c2 = col % 3;
  const int jx = j & 1, jy = (j >> 1) & 1, jz = (j >> 2) & 1;
  double acc = 0.0;
  for (int a = 0; a < 8; ++a) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = (a >> 2) & 1;
    const double wa = tri_w(jx + ax, C & 1) * tri_w(jy + ay, (C >> 1) & 1) * tri_w(jz + az, C >> 2);
    if (wa == 0.0) continue;
    for (int b = 0; b < 8; ++b) {
      const int bx = b & 1, by = (b >> 1) & 1, bz = (b >> 2) & 1;
      const double wb = tri_w(jx + bx, C2 & 1) * tri_w(jy + by, (C2 >> 1) & 1) * tri_w(jz + bz, C2 >> 2);
      if (wb == 0.0) continue;
      acc += wa * wb * c_K0d[(3 * corner_id(ax, ay, az) + c) * 24 + 3 * corner_id(bx, by, bz) + c2];
    }
  }
  g_cellMd[j * 576 + e] = acc;
  g_cellMf[j * 576 + e] = static_cast<float>(acc);
}

template <typename TV>
__device__ __forceinline__ const TV* cell_matrices();
template <>
__device__ __forceinline__ const double* cell_matrices<double>() { return g_cellMd; }
template <>
__device__ __forceinline__ const float* cell_matrices<float>() { return g_cellMf; }

// block (32 coarse nodes, 27 stencil slots): thread (x, m) owns block m of node x,
// so each stencil store is one coalesced 32-node line.
// The 4x4x4 fine elements around each of the block's 32 coarse nodes are
// staged in shared memory first (64 loads per node instead of 8 per shared
// coarse element per slot thread).
template <typename TV>
struct GalerkinFineShared {
  TV M[8 * 576];
  TV B[32][64];  // [node][fine element (tz*4 + ty)*4 + tx], origin 2N - 2
};
template <typename TV>
// (grid.y = 3: each CTA computes 9 of the 27 neighbour blocks of its 32 coarse
// nodes, 288 threads -- an 864-thread CTA waited for a nearly empty SM while
// other batch lanes' small CTAs kept backfilling, starving the setup)
__global__ void __launch_bounds__(288) galerkin_fine_kernel(const int* __restrict__ list_c, int n_c, int r_c,
                                                            const int* __restrict__ map_f, int r_f,
                                                            const TV* __restrict__ betav, TV ridge,
                                                            TV* __restrict__ stencil_c) {
  extern __shared__ __align__(16) unsigned char gf_raw[];
  GalerkinFineShared<TV>& Sh = *reinterpret_cast<GalerkinFineShared<TV>*>(gf_raw);
  TV* M = Sh.M;
  const TV* Mg = cell_matrices<TV>();
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int nthr = blockDim.x * blockDim.y;
  for (int t = tid; t < 8 * 576; t += nthr) M[t] = Mg[t];
  for (int t = tid; t < 32 * 64; t += nthr) {
    const int x = t / 64, e = t % 64, id = blockIdx.x * 32 + x;
    TV v = TV(0);
    if (id < n_c) {
      const int Gx = list_c[id];
      const int I = Gx % r_c, J = (Gx / r_c) % r_c, K = Gx / (r_c * r_c);
      const int ex = (2 * I - 2 + (e & 3) + r_f) % r_f, ey = (2 * J - 2 + ((e >> 2) & 3) + r_f) % r_f,
                ez = (2 * K - 2 + (e >> 4) + r_f) % r_f;
      v = betav[(static_cast<size_t>(ez) * r_f + ey) * r_f + ex];
    }
    Sh.B[x][e] = v;
  }
  __syncthreads();
  const int idx = blockIdx.x * 32 + threadIdx.x;
  if (idx >= n_c) return;
  const TV* Bn = Sh.B[threadIdx.x];
  const int m = blockIdx.y * blockDim.y + threadIdx.y;
  const int Dx = m % 3 - 1, Dy = (m / 3) % 3 - 1, Dz = m / 9 - 1;
  const int G = list_c[idx];
  TV S[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) S[q] = TV(0);
  if (G != 0) {
    const int rc2 = r_c * r_c;
    const int I = G % r_c, J = (G / r_c) % r_c, K = G / rc2;
    for (int az = 0; az < 2; ++az) {
      const int bz = az + Dz;
      if (bz < 0 || bz > 1) continue;
      for (int ay = 0; ay < 2; ++ay) {
        const int by = ay + Dy;
        if (by < 0 || by > 1) continue;
        for (int ax = 0; ax < 2; ++ax) {
          const int bx = ax + Dx;
          if (bx < 0 || bx > 1) continue;
          const int A = ax + 2 * ay + 4 * az, B = bx + 2 * by + 4 * bz;
          // coarse element 2(N - a) = fine elements 2N - 2 + 2(1 - a) + child offset
          const TV* Be = Bn + (2 * (1 - az)) * 16 + (2 * (1 - ay)) * 4 + 2 * (1 - ax);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const TV be = Be[(j >> 2) * 16 + ((j >> 1) & 1) * 4 + (j & 1)];
            const TV* Mj = M + j * 576 + (3 * A) * 24 + 3 * B;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int d = 0; d < 3; ++d) S[c * 3 + d] = fma_t(be, Mj[c * 24 + d], S[c * 3 + d]);
          }
        }
      }
    }
    if (ridge != TV(0)) {  // ridge * sum_n w(n,N) w(n,N+D) over active fine n != 0
      TV wsum = TV(0);
      for (int nz = -1; nz <= 1; ++nz) {
        if (Dz != 0 && nz != Dz) continue;
        for (int ny = -1; ny <= 1; ++ny) {
          if (Dy != 0 && ny != Dy) continue;
          for (int nx = -1; nx <= 1; ++nx) {
            if (Dx != 0 && nx != Dx) continue;
            const int fi = (2 * I + nx + r_f) % r_f, fj = (2 * J + ny + r_f) % r_f, fk = (2 * K + nz + r_f) % r_f;
            const size_t gn = (static_cast<size_t>(fk) * r_f + fj) * r_f + fi;
            if (gn == 0 || map_f[gn] < 0) continue;
            wsum += TV((nx ? 0.25 : 1.0) * (ny ? 0.25 : 1.0) * (nz ? 0.25 : 1.0));
          }
        }
      }
      S[0] = fma_t(ridge, wsum, S[0]);
      S[4] = fma_t(ridge, wsum, S[4]);
      S[8] = fma_t(ridge, wsum, S[8]);
    }
  }
  TV* out = stencil_c + vbase(idx, kStencil) + m * 9 * 32;
#pragma unroll
  for (int q = 0; q < 9; ++q) out[q * 32] = S[q];
}

// ---- Galerkin from a stored level ----------------------------------------
// A_c(N, N+D) = sum_{n in supp(N)} sum_{m in supp(N+D)} w(n,N) A_f(n,m) w(m,N+D).
// One warp per coarse node N, lane t < 27 owns fine node n = 2N + off(t) of
// N's support and reads each of its 27 fine blocks A_f(n, m) once, adding it
// to every coarse slot D whose support holds m; the 27 slots are done one
// z-plane (9 slots, 81 register accumulators) at a time and summed over the
// lanes by a butterfly (fixed order -> reproducible).  8 consecutive coarse
// nodes per CTA read overlapping fine stencils, which the L1 serves.
template <typename TV>
__global__ void __launch_bounds__(256) galerkin_stored_kernel(const int* __restrict__ list_c, int n_c, int r_c,
                                                              const int* __restrict__ map_f, int r_f,
                                                              const TV* __restrict__ stencil_f,
                                                              TV* __restrict__ stencil_c) {
  const int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (idx >= n_c) return;  // whole warps exit together
  const int G = list_c[idx];
  const int nx = lane % 3 - 1, ny = (lane / 3) % 3 - 1, nz = lane / 9 - 1;
  int fi = 0, fj = 0, fk = 0;
  bool act = false;
  const TV* sb = stencil_f;
  if (G != 0 && lane < 27) {
    const int I = G % r_c, J = (G / r_c) % r_c, K = G / (r_c * r_c);
    fi = (2 * I + nx + r_f) % r_f;
    fj = (2 * J + ny + r_f) % r_f;
    fk = (2 * K + nz + r_f) % r_f;
    const size_t gn = (static_cast<size_t>(fk) * r_f + fj) * r_f + fi;
    const int nf = map_f[gn];
    act = nf >= 0 && gn != 0;
    if (act) sb = stencil_f + vbase(nf, kStencil);
  }
  const TV wn = TV((nx ? 0.5 : 1.0) * (ny ? 0.5 : 1.0) * (nz ? 0.5 : 1.0));
  auto w1 = [](int e) { return e == 0 ? TV(1) : TV(0.5); };
#pragma unroll 1
  for (int Dz = -1; Dz <= 1; ++Dz) {
    TV S[9][9];  // [slot (Dy, Dx)][q]
#pragma unroll
    for (int d = 0; d < 9; ++d)
#pragma unroll
      for (int q = 0; q < 9; ++q) S[d][q] = TV(0);
    if (act) {
#pragma unroll
      for (int m = 0; m < 27; ++m) {
        const int dx = m % 3 - 1, dy = (m / 3) % 3 - 1, dz = m / 9 - 1;
        const int ez = nz + dz - 2 * Dz;  // m relative to 2(N+D) along z
        if (ez < -1 || ez > 1) continue;
        // an inactive fine neighbour's block is exactly zero (no active element
        // couples to it on any level), so only the pinned node needs skipping
        if ((fi + dx + r_f) % r_f == 0 && (fj + dy + r_f) % r_f == 0 && (fk + dz + r_f) % r_f == 0) continue;
        TV A[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = sb[(m * 9 + q) * 32];
        const TV wz = wn * w1(ez);
#pragma unroll
        for (int Dy = -1; Dy <= 1; ++Dy) {
          const int ey = ny + dy - 2 * Dy;
          if (ey < -1 || ey > 1) continue;
#pragma unroll
          for (int Dx = -1; Dx <= 1; ++Dx) {
            const int ex = nx + dx - 2 * Dx;
            if (ex < -1 || ex > 1) continue;
            const TV w = wz * w1(ey) * w1(ex);
#pragma unroll
            for (int q = 0; q < 9; ++q) S[(Dy + 1) * 3 + Dx + 1][q] = fma_t(w, A[q], S[(Dy + 1) * 3 + Dx + 1][q]);
          }
        }
      }
    }
#pragma unroll
    for (int d = 0; d < 9; ++d)
#pragma unroll
      for (int q = 0; q < 9; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S[d][q] += __shfl_xor_sync(0xffffffffu, S[d][q], o);
      }
    // lane d < 9 writes slot (Dz, d) -- the 9 values without dynamic register indexing
    if (lane < 9) {
      TV v[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) v[q] = S[0][q];
#pragma unroll
      for (int d = 1; d < 9; ++d)
        if (lane == d) {
#pragma unroll
          for (int q = 0; q < 9; ++q) v[q] = S[d][q];
        }
      const int slot = (Dz + 1) * 9 + lane;
#pragma unroll
      for (int q = 0; q < 9; ++q) stencil_c[vbase(idx, kStencil) + (slot * 9 + q) * 32] = v[q];
    }
  }
}

// Dinv of a stored level: inverse of the centre 3x3 block (0 for node 0 /
// singular).  l1 != 0: l1-block-Jacobi -- each diagonal entry also gets the
// row's off-block absolute sum, which makes the smoother convergent for any
// SPD matrix (no damping to tune on Galerkin levels, whose lambda_max(D^-1 A)
// exceeds the fine level's).
template <typename TV>
__global__ void coarse_dinv_kernel(const int* __restrict__ list_c, int n_c,
                                   const TV* __restrict__ stencil, TV* __restrict__ dinv, int l1) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_c) return;
  const TV* sb = stencil + vbase(idx, kStencil) + 13 * 9 * 32;
  double D[9];
  for (int q = 0; q < 9; ++q) D[q] = static_cast<double>(sb[q * 32]);
  if (l1) {
    const TV* s0 = stencil + vbase(idx, kStencil);
    for (int c = 0; c < 3; ++c) {
      double extra = 0.0;
      for (int m = 0; m < 27; ++m) {
        if (m == 13) continue;
        for (int d = 0; d < 3; ++d) extra += fabs(static_cast<double>(s0[(m * 9 + c * 3 + d) * 32]));
      }
      D[c * 3 + c] += extra;
    }
  }
  double inv[6] = {0, 0, 0, 0, 0, 0};
  const double c00 = D[4] * D[8] - D[5] * D[7], c01 = D[5] * D[6] - D[3] * D[8],
               c02 = D[3] * D[7] - D[4] * D[6];
  const double det = D[0] * c00 + D[1] * c01 + D[2] * c02;
  if (list_c[idx] != 0 && det > 0.0) {
    const double id = 1.0 / det;
    inv[0] = c00 * id;
    inv[1] = c01 * id;
    inv[2] = c02 * id;
    inv[3] = (D[0] * D[8] - D[2] * D[6]) * id;
    inv[4] = (D[2] * D[3] - D[0] * D[5]) * id;
    inv[5] = (D[0] * D[4] - D[1] * D[3]) * id;
  }
  for (int q = 0; q < 6; ++q) dinv[vbase(idx, 6) + q * 32] = static_cast<TV>(inv[q]);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_coarse_brick_flags(const int* map, int r, int* flag, cudaStream_t s) {
  const int nb = (r / 8) * (r / 4) * (r / 4);
  coarse_brick_flag_kernel<<<(nb + 127) / 128, 128, 0, s>>>(map, r, flag);
}

void launch_coarse_flags(const int* map_f, int r_f, int r_c, int* flag_c, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r_c) * r_c * r_c;
  coarse_flag_kernel<<<static_cast<unsigned>((n3 + 255) / 256), 256, 0, s>>>(map_f, r_f, r_c, flag_c);
}

template <typename TV>
void launch_galerkin(const int* list_c, int n_c, int r_c, const int* map_f, int r_f,
                     const TV* beta_f, const TV* stencil_f, TV ridge, TV* stencil_c, cudaStream_t s) {
  if (n_c == 0) return;
  if (stencil_f == nullptr) {
    static const bool configured = [] {
      cudaFuncSetAttribute(galerkin_fine_kernel<TV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(GalerkinFineShared<TV>)));
      return true;
    }();
    (void)configured;
    galerkin_fine_kernel<TV><<<dim3((n_c + 31) / 32, 3), dim3(32, 9), sizeof(GalerkinFineShared<TV>), s>>>(
        list_c, n_c, r_c, map_f, r_f, beta_f, ridge, stencil_c);
  } else {
    galerkin_stored_kernel<TV><<<static_cast<unsigned>((n_c + 7) / 8), 256, 0, s>>>(list_c, n_c, r_c, map_f, r_f,
                                                                                     stencil_f, stencil_c);
  }
}

template <typename TV>
void launch_coarse_dinv(const int* list_c, int n_c, const TV* stencil, TV* dinv, int l1, cudaStream_t s) {
  if (n_c) coarse_dinv_kernel<TV><<<(n_c + 127) / 128, 128, 0, s>>>(list_c, n_c, stencil, dinv, l1);
}

template <typename TB, typename TV>
void launch_level_sweep(const GmgLevelView<TV>& L, bool fine, const TB* b, const TV* xin, TV* xout,
                        TV omega, int mode, PcgState* st, double* partials, int init, int grid,
                        cudaStream_t s) {
  if (fine && L.bricks.nab > 0) {
    launch_brick_sweep<TB, TV, TV>(L, b, xin, xout, omega, mode, st, partials, init, s);
    return;
  }
  if constexpr (std::is_same<TV, float>::value && std::is_same<TB, float>::value) {
    // (at 64^3 and up the node-ordered level_sweep3 streams the stencils better:
    //  61 vs 38 us at level 1 of 128^3; at 16^3 the warp-per-node sweep wins:
    //  14 vs 10 us; at 32^3 the staged bricks: 20 vs 29 us)
    if (!fine && L.bricks.nab > 0 && L.n0 == 0 && mode != 2 && L.n <= 32768 && L.r >= 32) {
      launch_stencil_brick_sweep(L, b, xin, xout, omega, mode, st, s);
      return;
    }
  }
  LevelArgs<TV> a{L.node_list, L.node_map, L.beta, L.stencil, L.dinv, L.r, L.n, L.zero_slot, L.ridge, L.zbase, L.totals,
                  L.n0};
  if (fine) {
    launch_pdl(level_sweep3_kernel<TB, TV, true>, grid, 192, 0, s, a, b, xin, xout, omega, mode, st, partials, init);
  } else if (L.n - L.n0 > 32768) {  // large stored level: thread per node is throughput-bound
    launch_pdl(level_sweep3_kernel<TB, TV, false>, (L.n - L.n0 + 63) / 64, 192, 0, s, a, b, xin, xout, omega, mode, st,
               partials, init);
  } else {  // small stored level: latency-bound, one warp per node (mode 2 is level-0 only)
    launch_pdl(coarse_warp_sweep_kernel<TV>, std::max(1, (L.n - L.n0 + 7) / 8), 256, 0, s, a,
               reinterpret_cast<const TV*>(b), xin, xout, omega, mode, st);
  }
}

template <typename TB, typename TV, typename TO>
void launch_level_sweep_out(const GmgLevelView<TV>& L, const TB* b, const TV* xin, TO* xout, TV omega,
                            PcgState* st, double* partials, int init, int grid, cudaStream_t s) {
  if (L.bricks.nab > 0) {
    launch_brick_sweep<TB, TV, TO>(L, b, xin, xout, omega, 2, st, partials, init, s);
    return;
  }
  LevelArgs<TV> a{L.node_list, L.node_map, L.beta, L.stencil, L.dinv, L.r, L.n, L.zero_slot, L.ridge, L.zbase, L.totals,
                  L.n0};
  launch_pdl(level_sweep3_kernel<TB, TV, true, TO>, grid, 192, 0, s, a, b, xin, xout, omega, 2, st, partials, init);
}

template <typename TB, typename TV>
void launch_jacobi_first(const GmgLevelView<TV>& L, const TB* b, TV* xout, TV omega, const PcgState* st,
                         cudaStream_t s) {
  if (L.n > L.n0)
    launch_pdl(jacobi_first_kernel<TB, TV>, node_case_blocks(L.n - L.n0, 192), 192, 0, s, L.node_list, L.dinv, L.n, b,
               xout, omega, st, L.n0);
}

// The coarsest solve (jacobi_first + sweeps - 1 sweeps) as one cluster
// kernel when the level is the 8^3 torus in FP32; false otherwise (the caller
// then launches the sweeps one by one).
template <typename TV>
bool launch_coarsest(const GmgLevelView<TV>& L, const TV* b, TV* x, TV omega, int sweeps, const PcgState* st,
                     cudaStream_t s) {
  if constexpr (!std::is_same<TV, float>::value) {
    return false;
  } else {
    if (L.r != kCoR || L.n > kCoR * kCoP || L.n == 0 || sweeps < 1) return false;
    static const bool configured = [] {
      cudaFuncSetAttribute(coarsest_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(CoarsestShared)));
      return true;
    }();
    (void)configured;
    launch_pdl(coarsest_cluster_kernel, kCoR, kCoThreads, sizeof(CoarsestShared), s, L.node_list, L.n, L.stencil,
               L.dinv, b, x, omega, sweeps, st);
    return true;
  }
}

template <typename TV>
void launch_restrict(const GmgLevelView<TV>& C, const GmgLevelView<TV>& F, const TV* res_f, TV* b_c,
                     const PcgState* st, cudaStream_t s, TV* x_c, TV omega) {
  if (C.n)
    launch_pdl(restrict_kernel<TV>, node_case_blocks(C.n, 192), 192, 0, s, C.node_list, C.n, C.r, F.node_map, F.r,
               res_f, b_c, st, 0, 0, static_cast<const TV*>(C.dinv), x_c, omega);
}

template <typename TV>
void launch_restrict_partial(const GmgLevelView<TV>& C, const GmgLevelView<TV>& F, const TV* res_f, TV* b_c,
                             const PcgState* st, cudaStream_t s) {
  if (C.n)
    launch_pdl(restrict_kernel<TV>, node_case_blocks(C.n, 192), 192, 0, s, C.node_list, C.n, C.r, F.node_map, F.r,
               res_f, b_c, st, F.n0, std::max(F.n, 1), static_cast<const TV*>(nullptr), static_cast<TV*>(nullptr),
               TV(0));
}

template <typename TV>
void launch_restrict_own(const GmgLevelView<TV>& C, const int* map_s, int zbase, int nzl, int r_f, const TV* res_f,
                         TV* b_c, const PcgState* st, cudaStream_t s) {
  if (C.n > C.n0)
    launch_pdl(restrict_own_kernel<TV>, node_case_blocks(C.n - C.n0, 192), 192, 0, s, C.node_list, C.n0, C.n, C.r,
               map_s, zbase, nzl, r_f, res_f, b_c, st);
}

template <typename TV>
void launch_restrict_slab(const GmgLevelView<TV>& C, const int* map_s, int zbase, int nzl, int z0, int z1, int r_f,
                          const TV* res_f, TV* b_c, const PcgState* st, cudaStream_t s) {
  if (C.n)
    restrict_slab_kernel<TV><<<node_case_blocks(C.n, 192), 192, 0, s>>>(C.node_list, C.n, C.r, map_s, zbase, nzl, z0,
                                                                          z1, r_f, res_f, b_c, st);
}

template <typename TV>
void launch_prolong(const GmgLevelView<TV>& F, const GmgLevelView<TV>& C, const TV* x_c, TV* x_f,
                    const PcgState* st, cudaStream_t s) {
  if (F.n > F.n0)
    launch_pdl(prolong_kernel<TV>, (F.n - F.n0 + 127) / 128, 128, 0, s, F.node_list, F.n, F.r, C.node_map, C.r, x_c,
               x_f, st, F.n0);
}

#define SHL_GMG_INST(TV)                                                                               \
  template void launch_galerkin<TV>(const int*, int, int, const int*, int, const TV*, const TV*, TV, TV*, \
                                    cudaStream_t);                                                     \
  template void launch_coarse_dinv<TV>(const int*, int, const TV*, TV*, int, cudaStream_t);            \
  template void launch_restrict<TV>(const GmgLevelView<TV>&, const GmgLevelView<TV>&, const TV*, TV*,  \
                                    const PcgState*, cudaStream_t, TV*, TV);                          \
  template void launch_prolong<TV>(const GmgLevelView<TV>&, const GmgLevelView<TV>&, const TV*, TV*,   \
                                   const PcgState*, cudaStream_t);                                   \
  template bool launch_coarsest<TV>(const GmgLevelView<TV>&, const TV*, TV*, TV, int, const PcgState*, \
                                    cudaStream_t);                                                   \
  template void launch_restrict_slab<TV>(const GmgLevelView<TV>&, const int*, int, int, int, int, int,   \
                                         const TV*, TV*, const PcgState*, cudaStream_t);                \
  template void launch_restrict_partial<TV>(const GmgLevelView<TV>&, const GmgLevelView<TV>&, const TV*, \
                                            TV*, const PcgState*, cudaStream_t);                        \
  template void launch_restrict_own<TV>(const GmgLevelView<TV>&, const int*, int, int, int, const TV*, TV*, \
                                        const PcgState*, cudaStream_t);
SHL_GMG_INST(float)
SHL_GMG_INST(double)
template void launch_level_sweep<double, float>(const GmgLevelView<float>&, bool, const double*, const float*,
                                                float*, float, int, PcgState*, double*, int, int, cudaStream_t);
template void launch_level_sweep<float, float>(const GmgLevelView<float>&, bool, const float*, const float*,
                                               float*, float, int, PcgState*, double*, int, int, cudaStream_t);
template void launch_level_sweep<double, double>(const GmgLevelView<double>&, bool, const double*,
                                                 const double*, double*, double, int, PcgState*, double*,
                                                 int, int, cudaStream_t);
template void launch_level_sweep_out<double, float, double>(const GmgLevelView<float>&, const double*,
                                                           const float*, double*, float, PcgState*, double*,
                                                           int, int, cudaStream_t);
template void launch_level_sweep_out<double, float, float>(const GmgLevelView<float>&, const double*,
                                                          const float*, float*, float, PcgState*, double*,
                                                          int, int, cudaStream_t);
template void launch_level_sweep_out<float, float, float>(const GmgLevelView<float>&, const float*, const float*,
                                                          float*, float, PcgState*, double*, int, int, cudaStream_t);
template void launch_level_sweep_out<double, double, double>(const GmgLevelView<double>&, const double*,
                                                             const double*, double*, double, PcgState*, double*,
                                                             int, int, cudaStream_t);
template void launch_jacobi_first<double, float>(const GmgLevelView<float>&, const double*, float*, float,
                                                 const PcgState*, cudaStream_t);
template void launch_jacobi_first<float, float>(const GmgLevelView<float>&, const float*, float*, float,
                                                const PcgState*, cudaStream_t);
template void launch_jacobi_first<double, double>(const GmgLevelView<double>&, const double*, double*, double,
                                                  const PcgState*, cudaStream_t);
