// voxel.cu -- K2: shell mask on device (sm_100a).
//
// Replaces build_reduced_mesh's element selection (voxel.hpp:235-307) and
// classify_surface_elements (voxel.hpp:118-141), and the node bookkeeping of
// build_topology (voxel.hpp:147-228), which on the torus reduces to index
// arithmetic plus an ordered compaction:
//
//   classify   element surface iff a corner sign is 0 or signs differ
//   dilate xL  BFS with 6-connectivity and periodic wrap == L dilation passes
//   complete   orbit closure under boundary-index flips (one pass in the ref)
//   corners    8 corner voxels forced when any element touches the boundary
//   beta       h(F_centre / norm), step_function voxel.hpp:38-41
//   nodes      torus node active iff an incident element is active; ordered
//              exclusive scan gives node ids in grid order (node_map, node_list)
//
// Occupancy is one byte per voxel: at 128^3 a dilation pass moves ~2 MB, a few
// microseconds of HBM time, so bit packing would not move the stage total.
#include <cub/device/device_scan.cuh>

#include "device.cuh"

namespace shl {

namespace {

__device__ __forceinline__ int wrapi(int v, int r) { return v < 0 ? v + r : (v >= r ? v - r : v); }

__global__ void corner_sign_kernel(const double* __restrict__ corners, int8_t* __restrict__ sg,
                                   size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = corners[i];
  sg[i] = v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);
}

__global__ void classify_kernel(const int8_t* __restrict__ cs, uint8_t* __restrict__ occ, int r,
                                int* n_surface) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  int hit = 0;
  if (e < n3) {
    const int i = static_cast<int>(e % r), j = static_cast<int>((e / r) % r),
              k = static_cast<int>(e / (static_cast<size_t>(r) * r));
    bool pos = false, neg = false, zero = false;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const int ci = wrapi(i + (d & 1), r), cj = wrapi(j + ((d >> 1) & 1), r),
                ck = wrapi(k + ((d >> 2) & 1), r);
      const int8_t s = cs[(static_cast<size_t>(ck) * r + cj) * r + ci];
      pos |= s > 0;
      neg |= s < 0;
      zero |= s == 0;
    }
    hit = (zero || (pos && neg)) ? 1 : 0;
    occ[e] = static_cast<uint8_t>(hit);
  }
  const int cnt = __syncthreads_count(hit);
  if (threadIdx.x == 0 && cnt) atomicAdd(n_surface, cnt);
}

__global__ void dilate_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int r) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (e >= n3) return;
  const int i = static_cast<int>(e % r), j = static_cast<int>((e / r) % r),
            k = static_cast<int>(e / (static_cast<size_t>(r) * r));
  const size_t rr = static_cast<size_t>(r) * r;
  const size_t row = (static_cast<size_t>(k) * r + j) * r;
  uint8_t v = in[e];
  v |= in[row + wrapi(i - 1, r)] | in[row + wrapi(i + 1, r)];
  v |= in[static_cast<size_t>(k) * rr + static_cast<size_t>(wrapi(j - 1, r)) * r + i];
  v |= in[static_cast<size_t>(k) * rr + static_cast<size_t>(wrapi(j + 1, r)) * r + i];
  v |= in[static_cast<size_t>(wrapi(k - 1, r)) * rr + static_cast<size_t>(j) * r + i];
  v |= in[static_cast<size_t>(wrapi(k + 1, r)) * rr + static_cast<size_t>(j) * r + i];
  out[e] = v;
}

// Orbit closure (voxel.hpp:266-282) + the "touches boundary" flag (:286-292).
__global__ void complete_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int r,
                                int* touches) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  int t = 0;
  if (e < n3) {
    const int c[3] = {static_cast<int>(e % r), static_cast<int>((e / r) % r),
                      static_cast<int>(e / (static_cast<size_t>(r) * r))};
    int axes[3], nf = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (c[a] == 0 || c[a] == r - 1) axes[nf++] = a;
    uint8_t v = in[e];
    for (int mask = 1; mask < (1 << nf) && !v; ++mask) {
      int q[3] = {c[0], c[1], c[2]};
      for (int b = 0; b < nf; ++b)
        if (mask & (1 << b)) q[axes[b]] = q[axes[b]] == 0 ? r - 1 : 0;
      v |= in[(static_cast<size_t>(q[2]) * r + q[1]) * r + q[0]];
    }
    out[e] = v;
    t = (v && nf > 0) ? 1 : 0;
  }
  if (__syncthreads_or(t) && threadIdx.x == 0) atomicOr(touches, 1);
}

__global__ void force_corners_kernel(uint8_t* occ, int r, const int* touches) {
  if (!*touches) return;
  const int t = threadIdx.x;  // 8 threads
  const int i = (t & 1) ? r - 1 : 0, j = (t & 2) ? r - 1 : 0, k = (t & 4) ? r - 1 : 0;
  occ[(static_cast<size_t>(k) * r + j) * r + i] = 1;
}

// beta = 1 + v0/2 - v0 / (1 + exp(-k v^2)), v = F/norm (voxel.hpp:38-41,304-307)
__global__ void beta_kernel(const uint8_t* __restrict__ occ, const double* __restrict__ centres,
                            const double* __restrict__ norm, double sharp, double floor_ratio,
                            size_t n3, double* __restrict__ beta64, float* __restrict__ beta32,
                            int* __restrict__ elem_flag, double* __restrict__ partial) {
  const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double b = 0.0;
  int on = 0;
  if (e < n3) {
    on = occ[e] ? 1 : 0;
    if (on) {
      const double v0 = 2.0 * (1.0 - floor_ratio);
      const double v = centres[e] / *norm;
      const double ex = exp(__dmul_rn(__dmul_rn(-sharp, v), v));
      b = __dsub_rn(__dadd_rn(1.0, __dmul_rn(0.5, v0)), v0 / __dadd_rn(1.0, ex));
    }
    beta64[e] = b;
    beta32[e] = static_cast<float>(b);
    elem_flag[e] = on;
  }
  // deterministic per-block partial sums of (count, sum beta)
  __shared__ double sb[32];
  __shared__ int sc[32];
  double s = b;
  int c = on;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sb[w] = s;
    sc[w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0;
    int tc = 0;
    for (int q = 0; q < (blockDim.x + 31) / 32; ++q) {
      ts += sb[q];
      tc += sc[q];
    }
    partial[2 * blockIdx.x] = ts;
    partial[2 * blockIdx.x + 1] = static_cast<double>(tc);
  }
}

__global__ void beta_dense_kernel(const double* __restrict__ beta_in, size_t n3,
                                  float* __restrict__ beta32, int* __restrict__ elem_flag,
                                  uint8_t* __restrict__ occ) {
  const size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (e >= n3) return;
  const double b = beta_in[e];
  beta32[e] = static_cast<float>(b);
  elem_flag[e] = b != 0.0;
  occ[e] = b != 0.0;
}

__global__ void node_flag_kernel(const int* __restrict__ ef, int r, int* __restrict__ node_flag) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  const size_t n = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (n >= n3) return;
  const int i = static_cast<int>(n % r), j = static_cast<int>((n / r) % r),
            k = static_cast<int>(n / (static_cast<size_t>(r) * r));
  int on = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int ei = wrapi(i - (d & 1), r), ej = wrapi(j - ((d >> 1) & 1), r),
              ek = wrapi(k - ((d >> 2) & 1), r);
    on |= ef[(static_cast<size_t>(ek) * r + ej) * r + ei];
  }
  node_flag[n] = on;
}

__global__ void scatter_kernel(const int* __restrict__ flag, const int* __restrict__ off, int n,
                               int* __restrict__ map, int* __restrict__ list) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int f = flag[i];
  if (map) map[i] = f ? off[i] : -1;
  if (f) list[off[i]] = i;
}

// ---- brick-major level-0 node numbering (brick.cuh) -------------------------
// Padded brick-major index p = brick * 128 + (lz*4 + ly)*8 + lx over
// ceil(r/8) x ceil(r/4) x ceil(r/4) bricks of 8x4x4 nodes; positions outside
// the torus (ragged last bricks) are never active.
constexpr int kBrickX = 8, kBrickY = 4, kBrickZ = 4, kBrickN = kBrickX * kBrickY * kBrickZ;

__device__ __forceinline__ long long brick_to_grid(long long p, int r, int nbx, int nby) {
  const long long b = p / kBrickN;
  const int w = static_cast<int>(p % kBrickN);
  const int x = static_cast<int>(b % nbx) * kBrickX + w % kBrickX;
  const int y = static_cast<int>((b / nbx) % nby) * kBrickY + (w / kBrickX) % kBrickY;
  const int z = static_cast<int>(b / (static_cast<long long>(nbx) * nby)) * kBrickZ + w / (kBrickX * kBrickY);
  if (x >= r || y >= r || z >= r) return -1;
  return (static_cast<long long>(z) * r + y) * r + x;
}

__global__ void brick_flag_kernel(const int* __restrict__ node_flag, int r, int nbx, int nby, long long np,
                                  int* __restrict__ bflag) {
  const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p >= np) return;
  const long long g = brick_to_grid(p, r, nbx, nby);
  bflag[p] = g >= 0 ? node_flag[g] : 0;
}

__global__ void brick_scatter_kernel(const int* __restrict__ bflag, const int* __restrict__ boff, int r, int nbx,
                                     int nby, long long np, int* __restrict__ map, int* __restrict__ list) {
  const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p >= np) return;
  const long long g = brick_to_grid(p, r, nbx, nby);
  if (g < 0) return;
  const int f = bflag[p];
  map[g] = f ? boff[p] : -1;
  if (f) list[boff[p]] = static_cast<int>(g);
}

__global__ void brick_active_kernel(const int* __restrict__ bflag, const int* __restrict__ boff, int nb,
                                    int* __restrict__ bact) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const long long first = static_cast<long long>(b) * kBrickN, last = first + kBrickN - 1;
  bact[b] = (boff[last] + bflag[last] - boff[first]) > 0;
}

__global__ void brick_table_kernel(const int* __restrict__ bact, const int* __restrict__ bidx,
                                   const int* __restrict__ boff, const int* __restrict__ bflag, int nb,
                                   int* __restrict__ bcoord, int* __restrict__ bstart, int* __restrict__ nab_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  if (bact[b]) {
    bcoord[bidx[b]] = b;
    bstart[bidx[b]] = boff[static_cast<long long>(b) * kBrickN];
  }
  if (b == nb - 1) {
    const int nab = bidx[b] + bact[b];
    const long long lastp = static_cast<long long>(nb) * kBrickN - 1;
    bstart[nab] = boff[lastp] + bflag[lastp];
    *nab_out = nab;
  }
}

// ---- mechanical connectivity (fem.hpp:288-317) ---------------------------------
// Elements are coupled when they share a torus node (the reference's canonical
// (mod r) node key), i.e. they are 26-neighbours on the periodic element grid.
// Lock-free union-find on the dense r^3 element grid: parents only ever point
// to smaller ids (a root is hooked under the smaller root by CAS), so path
// halving races are benign.
__device__ __forceinline__ int uf_find(int* p, int x) {
  int cur = p[x];
  if (cur == x) return x;
  int prev = x, next;
  while (cur > (next = p[cur])) {
    p[prev] = next;
    prev = cur;
    cur = next;
  }
  return cur;
}

__device__ __forceinline__ void uf_union(int* p, int a, int b) {
  for (;;) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(&p[a], a, b) == a) return;  // a still a root: hooked under b
  }
}

__global__ void cc_init_kernel(const int* __restrict__ ef, int n3, int* __restrict__ parent, int* __restrict__ corner) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n3) return;
  parent[e] = ef[e] ? e : -1;
  corner[e] = 0;
}

__global__ void cc_union_kernel(const int* __restrict__ ef, int r, int* __restrict__ parent) {
  const int n3 = r * r * r;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n3 || !ef[e]) return;
  const int i = e % r, j = (e / r) % r, k = e / (r * r);
  // the 13 "forward" neighbours of the 26 (each pair is united once)
  for (int d = 14; d < 27; ++d) {
    const int di = d % 3 - 1, dj = (d / 3) % 3 - 1, dk = d / 9 - 1;
    const int f = (wrapi(k + dk, r) * r + wrapi(j + dj, r)) * r + wrapi(i + di, r);
    if (f != e && ef[f]) uf_union(parent, e, f);
  }
}

// every element's root; roots of components holding an element at torus node 0
__global__ void cc_mark_kernel(const int* __restrict__ ef, int r, int* __restrict__ parent, int* __restrict__ corner) {
  const int n3 = r * r * r;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n3 || !ef[e]) return;
  const int root = uf_find(parent, e);
  const int i = e % r, j = (e / r) % r, k = e / (r * r);
  const bool at0 = (i == 0 || i == r - 1) && (j == 0 || j == r - 1) && (k == 0 || k == r - 1);
  if (at0) corner[root] = 1;
}

__global__ void cc_count_kernel(const int* __restrict__ parent, const int* __restrict__ corner, int n3,
                                int* __restrict__ n_comp, int* __restrict__ n_float) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  int c = 0, f = 0;
  if (e < n3 && parent[e] == e) {
    c = 1;
    f = corner[e] == 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  f = __reduce_add_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && c) {
    atomicAdd(n_comp, c);
    if (f) atomicAdd(n_float, f);
  }
}

__global__ void fill_int_kernel(int* p, int v, size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = v;
}

inline unsigned blocks(size_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

void launch_corner_signs(const double* corners, int8_t* cs, int r, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  corner_sign_kernel<<<blocks(n3, 256), 256, 0, s>>>(corners, cs, n3);
}

void launch_classify(const int8_t* cs, uint8_t* occ, int r, int* n_surface, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  classify_kernel<<<blocks(n3, 256), 256, 0, s>>>(cs, occ, r, n_surface);
}

void launch_dilate(const uint8_t* in, uint8_t* out, int r, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  dilate_kernel<<<blocks(n3, 256), 256, 0, s>>>(in, out, r);
}

void launch_complete(const uint8_t* in, uint8_t* out, int r, int* touches, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  complete_kernel<<<blocks(n3, 256), 256, 0, s>>>(in, out, r, touches);
}

void launch_force_corners(uint8_t* occ, int r, const int* touches, cudaStream_t s) {
  force_corners_kernel<<<1, 8, 0, s>>>(occ, r, touches);
}

void launch_beta(const uint8_t* occ, const double* centres, const double* norm, double sharp,
                 double floor_ratio, int r, double* beta64, float* beta32, int* elem_flag,
                 double* partial, int nblocks_partial, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  (void)nblocks_partial;
  beta_kernel<<<blocks(n3, 256), 256, 0, s>>>(occ, centres, norm, sharp, floor_ratio, n3, beta64,
                                              beta32, elem_flag, partial);
}

void launch_beta_from_dense(const double* beta_in, int r, float* beta32, int* elem_flag,
                            uint8_t* occ, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  beta_dense_kernel<<<blocks(n3, 256), 256, 0, s>>>(beta_in, n3, beta32, elem_flag, occ);
}

void launch_node_flags(const int* elem_flag, int r, int* node_flag, cudaStream_t s) {
  const size_t n3 = static_cast<size_t>(r) * r * r;
  node_flag_kernel<<<blocks(n3, 256), 256, 0, s>>>(elem_flag, r, node_flag);
}

void launch_scatter_compact(const int* flag, const int* off, int n, int* map, int* list,
                            cudaStream_t s) {
  scatter_kernel<<<blocks(n, 256), 256, 0, s>>>(flag, off, n, map, list);
}

void launch_fill_int(int* p, int v, size_t n, cudaStream_t s) {
  if (n) fill_int_kernel<<<blocks(n, 256), 256, 0, s>>>(p, v, n);
}

BrickDims brick_dims(int r) {
  BrickDims d;
  d.nbx = (r + kBrickX - 1) / kBrickX;
  d.nby = (r + kBrickY - 1) / kBrickY;
  d.nbz = (r + kBrickZ - 1) / kBrickZ;
  d.nb = d.nbx * d.nby * d.nbz;
  d.np = static_cast<long long>(d.nb) * kBrickN;
  return d;
}

void launch_brick_numbering(const int* node_flag, int r, int* bflag, int* boff, int* bact, int* bidx,
                            void* temp, size_t temp_bytes, int* node_map, int* node_list, int* bcoord,
                            int* bstart, int* nab_out, cudaStream_t s) {
  const BrickDims d = brick_dims(r);
  brick_flag_kernel<<<blocks(d.np, 256), 256, 0, s>>>(node_flag, r, d.nbx, d.nby, d.np, bflag);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, bflag, boff, static_cast<int>(d.np), s);
  brick_scatter_kernel<<<blocks(d.np, 256), 256, 0, s>>>(bflag, boff, r, d.nbx, d.nby, d.np, node_map,
                                                         node_list);
  brick_active_kernel<<<blocks(d.nb, 256), 256, 0, s>>>(bflag, boff, d.nb, bact);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, bact, bidx, d.nb, s);
  brick_table_kernel<<<blocks(d.nb, 256), 256, 0, s>>>(bact, bidx, boff, bflag, d.nb, bcoord, bstart, nab_out);
}

void launch_components(const int* elem_flag, int r, int* parent, int* corner, int* n_comp, int* n_float,
                       cudaStream_t s) {
  const int n3 = r * r * r;
  cc_init_kernel<<<blocks(n3, 256), 256, 0, s>>>(elem_flag, n3, parent, corner);
  cc_union_kernel<<<blocks(n3, 256), 256, 0, s>>>(elem_flag, r, parent);
  cc_mark_kernel<<<blocks(n3, 256), 256, 0, s>>>(elem_flag, r, parent, corner);
  cc_count_kernel<<<blocks(n3, 256), 256, 0, s>>>(parent, corner, n3, n_comp, n_float);
}

size_t scan_temp_bytes(int n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const int*>(nullptr),
                                static_cast<int*>(nullptr), n);
  return bytes;
}

void launch_exclusive_scan(const int* in, int* out, int n, void* temp, size_t temp_bytes,
                           cudaStream_t s) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n, s);
}

}  // namespace shl
