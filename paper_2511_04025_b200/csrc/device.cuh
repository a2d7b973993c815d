// device.cuh -- device-side types, launch wrappers and small helpers shared by
// the kernels of libshellular_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace shl {

// Bounds-checked build (compute-sanitizer is closed on the gpurun pool):
// `make DEBUG_CHECKS=1` compiles device-side index checks that trap on the
// first out-of-range access; the product build compiles them out.
#ifdef SHL_DEBUG_CHECKS
#define SHL_DCHECK(cond)                                                                         \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("SHL_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                       \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define SHL_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

constexpr int kFieldRows = 8;        // (y,z)-rows per field block (charge tables reused 8x)
constexpr int kFieldThreads = 128;   // x samples per field block pass
constexpr int kFieldChargeChunk = 128;

// ---- PCG control block (one per solve, device resident) -------------------
struct PcgState {
  double alpha[6];   // step of the current iteration
  double beta[6];    // gamma_{k+1} / gamma_k
  double gamma[6];   // r.z of the current residual
  double delta[6];   // z.Az
  double pap[6];     // p.Ap (Chronopoulos-Gear recurrence)
  double bnorm[6];
  double rr[6];
  double tol;
  double ridge;      // diagonal ridge (fem.hpp:337-343), added to A
  int32_t done[6];
  int32_t iters[6];
  int32_t it;
  int32_t max_iter;
  int32_t all_done;
  int32_t error;  // 1: p^T A p <= 0 on an unconverged column
  int32_t stop;   // all_done || error || it >= max_iter
  uint32_t counter_apply;
  uint32_t counter_update;
  uint32_t counter_misc;
  // dynamic tile schedulers (TileQueue / tiles_done): [0] apply, [1] V-cycle sweeps
  uint32_t tile_next[2];
  uint32_t tile_done[2];
};

// ---- launch wrappers (defined in field.cu / voxel.cu / solver.cu) ---------
// field
void launch_field_sl(const double* tab, const double* coeff, double* sl, int nc, int r, int n,
                     cudaStream_t s);
void launch_field_samples(const double* tab, const double* sl, const int8_t* sign, int nc, int r,
                          int n, double* centres, double* corners, int8_t* corner_sign,
                          unsigned long long* norm_bits, cudaStream_t s);
// voxelize
void launch_corner_signs(const double* corners, int8_t* corner_sign, int r, cudaStream_t s);
void launch_classify(const int8_t* corner_sign, uint8_t* occ, int r, int* n_surface,
                     cudaStream_t s);
void launch_dilate(const uint8_t* in, uint8_t* out, int r, cudaStream_t s);
void launch_complete(const uint8_t* in, uint8_t* out, int r, int* touches, cudaStream_t s);
void launch_force_corners(uint8_t* occ, int r, const int* touches, cudaStream_t s);
void launch_beta(const uint8_t* occ, const double* centres, const double* norm, double sharp,
                 double floor_ratio, int r, double* beta64, float* beta32, int* elem_flag,
                 double* partial, int nblocks_partial, cudaStream_t s);
void launch_beta_from_dense(const double* beta_in, int r, float* beta32, int* elem_flag,
                            uint8_t* occ, cudaStream_t s);
void launch_node_flags(const int* elem_flag, int r, int* node_flag, cudaStream_t s);
void launch_scatter_compact(const int* flag, const int* offset, int n, int* map_or_null,
                            int* list, cudaStream_t s);
void launch_fill_int(int* p, int v, size_t n, cudaStream_t s);
size_t scan_temp_bytes(int n);
// Connected components of the active elements under the reference's coupling
// (shared torus node, fem.hpp:288-317): *n_comp += components, *n_float +=
// components without an element at torus node 0 (floating: rigid null modes).
// parent / corner: r^3 int workspaces.
void launch_components(const int* elem_flag, int r, int* parent, int* corner, int* n_comp, int* n_float,
                       cudaStream_t s);
// brick-major level-0 numbering (8x4x4-node bricks, brick.cu): node_map /
// node_list in brick order, active brick table (bcoord, bstart[nab+1]) and
// nab written to *nab_out.  Scan temp must hold scan_temp_bytes(np).
struct BrickDims {
  int nbx = 0, nby = 0, nbz = 0, nb = 0;
  long long np = 0;  // padded positions = nb * 256
};
BrickDims brick_dims(int r);
void launch_brick_numbering(const int* node_flag, int r, int* bflag, int* boff, int* bact, int* bidx,
                            void* temp, size_t temp_bytes, int* node_map, int* node_list, int* bcoord,
                            int* bstart, int* nab_out, cudaStream_t s);
void launch_exclusive_scan(const int* in, int* out, int n, void* temp, size_t temp_bytes,
                           cudaStream_t s);

}  // namespace shl
