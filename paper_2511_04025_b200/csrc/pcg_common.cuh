// pcg_common.cuh -- device helpers shared by the PCG kernels of solver.cu and
// the staged brick kernels of brick.cu: vector layout, reductions, the dynamic
// tile queue and the PcgState scalar updates.  Internal.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "solver.cuh"

namespace shl {

// ---- programmatic dependent launch -------------------------------------------
// The solve loop is a chain of ~35 dependent kernels per PCG iteration, most of
// them small (coarse multigrid levels).  Launched with programmatic stream
// serialization, a kernel's launch is processed while its predecessor still
// runs; pdl_wait() (griddepcontrol.wait) then holds it until the predecessor
// has completed and its writes are visible.  Every kernel launched this way
// calls pdl_wait() before touching global memory; launched normally it is a
// no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// cp.async (4/8/16-byte global -> shared copies, completion by commit group)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_addr(dst)), "l"(src), "n"(BYTES)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ float fma_t(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_t(double a, double b, double c) { return fma(a, b, c); }

// PCG vectors are stored in 32-node blocks, [idx/32][q][idx%32]: a warp's
// access to one component q of 32 consecutive nodes is one 128-byte line (FP32)
// and every component offset is an immediate (q*32 elements) from the node's
// base address.
__host__ __device__ __forceinline__ size_t vbase(int idx, int nq) {
  return static_cast<size_t>(idx >> 5) * (nq * 32) + (idx & 31);
}

__host__ __device__ constexpr int corner_id(int x, int y, int z) {
  return 4 * z + (y ? (x ? 2 : 3) : (x ? 1 : 0));
}

namespace {

// ---- reductions -----------------------------------------------------------
template <int NV>
__device__ __forceinline__ void warp_sum(double (&v)[NV]) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
}

// Block sum of NV doubles; result valid in thread 0.  scratch: 32*NV doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  warp_sum<NV>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  if (l == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) scratch[w * NV + q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int u = 0; u < nw; ++u) s += scratch[u * NV + q];
      v[q] = s;
    }
  }
}

// Writes this block's partial; returns true in exactly one block (the last to
// finish), whose threads then see every partial.
// Thread 0's arrival at a last-block counter: an acq_rel atomic at GPU scope
// (release: this block's partials, ordered before it by the preceding
// barrier; acquire: every other block's, for the last one) instead of a
// sequentially consistent __threadfence() + atomicAdd.
__device__ __forceinline__ bool arrive_last(uint32_t* counter) {
  uint32_t t;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter) : "memory");
  return t == gridDim.x - 1;
}

template <int NV>
__device__ __forceinline__ bool publish_partial(const double (&v)[NV], double* partials,
                                                uint32_t* counter) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[blockIdx.x * NV + q] = v[q];
    last = arrive_last(counter);
  }
  __syncthreads();
  return last;
}

// Fixed-order reduction of gridDim.x partials (called by the last block).
template <int NV>
__device__ __forceinline__ void reduce_partials(const double* partials, double (&out)[NV],
                                                double* scratch) {
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = 0.0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] += __ldcg(partials + b * NV + q);
  block_sum<NV>(out, scratch);
}

// ---- dynamic tile scheduling ------------------------------------------------
// The gather kernels keep one CTA per resident slot and hand out 32/64-node
// tiles from an atomic counter instead of a fixed grid stride.  With several
// designs in flight (batch lanes) a kernel is often only partly resident; a
// fixed stride then runs the late CTAs' full shares as a second wave (measured:
// two lanes at half the throughput of one), while a shared counter lets the
// resident CTAs take the work.  The last CTA to finish resets the counter.
// The next grab is kept in flight: thread 0 requests tile i+1 while
// the CTA gathers tile i (the atomic's L2 round trip overlaps the loads instead
// of holding every warp at a barrier), publishes it before the tile's mid
// barrier, and everyone reads it after the end barrier.  Two slots, so a warp
// still reading tile i+1's id never sees tile i+2's.  Per tile this needs only
// the kernel's own two barriers (a grab-then-broadcast needs two more).
struct TileQueue {
  uint32_t* next;
  int* slot;  // __shared__ int[2]
  unsigned pending = 0;
  int it = 0;
  __device__ __forceinline__ int first() {
    if (threadIdx.x == 0) slot[1] = static_cast<int>(atomicAdd(next, 1u));
    __syncthreads();
    return slot[1];
  }
  __device__ __forceinline__ void request() {
    if (threadIdx.x == 0) pending = atomicAdd(next, 1u);
  }
  __device__ __forceinline__ void publish() {  // before the tile's mid barrier
    if (threadIdx.x == 0) slot[it & 1] = static_cast<int>(pending);
  }
  __device__ __forceinline__ int advance() {  // after the tile's end barrier
    return slot[(it++) & 1];
  }
};

__device__ __forceinline__ void tiles_done(uint32_t* next, uint32_t* done) {
  if (threadIdx.x == 0 && atomicAdd(done, 1u) == gridDim.x - 1) {
    atomicExch(next, 0u);
    atomicExch(done, 0u);
  }
}

// ---- scalar updates (shared by the last block and the cross-slab finalize) --
__device__ void finalize_apply_state(PcgState* st, const double (&tot)[6]) {
  for (int s = 0; s < 6; ++s) {
    st->delta[s] = tot[s];  // p.q
    if (st->done[s]) {
      st->alpha[s] = 0.0;
      continue;
    }
    const double den = tot[s];  // p^T A p (grid_solver.hpp:62-63)
    if (!(den > 0.0)) st->error = 1;
    st->pap[s] = den;
    st->alpha[s] = st->gamma[s] / den;
  }
  if (st->error) st->stop = 1;
}

__device__ void finalize_update_state(PcgState* st, const double (&tot)[12], int init) {
  bool all = true;
  for (int t = 0; t < 6; ++t) {
    st->rr[t] = tot[t];
    const double rn = sqrt(tot[t]);
    if (init) {
      st->bnorm[t] = rn;
      st->gamma[t] = tot[6 + t];
      st->done[t] = rn == 0.0;
      st->beta[t] = 0.0;
      st->alpha[t] = 0.0;
      st->iters[t] = 0;
    } else if (!st->done[t]) {
      st->iters[t] = st->it + 1;           // grid_solver.hpp:67
      if (rn <= st->tol * st->bnorm[t]) {  // grid_solver.hpp:68-72
        st->done[t] = 1;
        st->beta[t] = 0.0;
      } else {
        st->beta[t] = tot[6 + t] / st->gamma[t];
        st->gamma[t] = tot[6 + t];
      }
    }
    all = all && st->done[t];
  }
  if (!init) st->it += 1;
  st->all_done = all;
  st->stop = all || st->error || st->it >= st->max_iter;
}

// GMG mode: the update kernel only reduces r.r (convergence); beta comes
// from gamma = r.z reduced by the V-cycle's last sweep.
__device__ void finalize_update_gmg(PcgState* st, const double* rr, int init) {
  bool all = true;
  for (int t = 0; t < 6; ++t) {
    st->rr[t] = rr[t];
    const double rn = sqrt(rr[t]);
    if (init) {
      st->bnorm[t] = rn;
      st->done[t] = rn == 0.0;
      st->beta[t] = 0.0;
      st->alpha[t] = 0.0;
      st->iters[t] = 0;
    } else if (!st->done[t]) {
      st->iters[t] = st->it + 1;
      if (rn <= st->tol * st->bnorm[t]) {
        st->done[t] = 1;
        st->beta[t] = 0.0;
      }
    }
    all = all && st->done[t];
  }
  if (!init) st->it += 1;
  st->all_done = all;
  st->stop = all || st->error || st->it >= st->max_iter;
}

__device__ void finalize_gamma_state(PcgState* st, const double (&g)[6], int init) {
  for (int t = 0; t < 6; ++t) {
    if (init) {
      st->gamma[t] = g[t];
      st->beta[t] = 0.0;
    } else if (!st->done[t]) {
      st->beta[t] = g[t] / st->gamma[t];
      st->gamma[t] = g[t];
    }
  }
}

}  // namespace
}  // namespace shl
