// solver.cuh -- argument blocks and launchers of the PCG kernels (solver.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device.cuh"

namespace shl {

// Level-0 brick tables (brick.cu): active bricks of 8x4x4 nodes in
// brick-major order, each owning the contiguous node ids
// [bstart[t], bstart[t+1]).  nab == 0: no brick numbering (z-slab levels), the
// per-node gather kernels run instead.
struct BrickView {
  const int* bcoord = nullptr;  // active brick t -> brick id bx + nbx*(by + nby*bz)
  const int* bstart = nullptr;  // nab + 1 entries
  int nab = 0;
  int nbx = 0, nby = 0;
  int n_nodes = 0;  // node ids in [0, n_nodes) (bounds-checked build)
};

// TV: Krylov vectors p, q and the operator arithmetic; TZ: the preconditioned
// residual z (the multigrid V-cycle's type).  Mixed multigrid runs TV = double
// with TZ = float: w = A z is accumulated in FP64 from the FP32 z, so p^T A p
// keeps its sign on the near-null hinge modes of voxel shells.
template <typename TV, typename TZ = TV>
struct ApplyArgs {
  const int* node_list;  // active node -> grid id
  const int* node_map;   // r^3 -> active node id or -1
  const TV* beta;        // r^3 dense, 0 = absent
  const TZ* z;           // 18 planes, slot n is a zero row
  TV* p;
  TV* q;
  double* partials;
  PcgState* state;
  int r;
  int n;          // nodes this launch owns (iterated)
  int ld;
  int zero_slot;  // local id of the always-zero row (= owned + ghost nodes)
  int zbase;      // global z of local node-map plane 0 (0 when not slabbed)
  int nzl;        // node-map planes (r when not slabbed)
  double* totals; // defer != 0: write the 6 reduced sums here, leave state alone
  int defer;
  BrickView bricks;  // nab > 0: staged brick kernel (brick.cuh)
  int n0 = 0;        // per-node gather kernels: iterate nodes [n0, n) (z-slab interior / boundary planes)
};

// TXS: storage type of the solution x (FP32 in mixed multigrid: x is only
// accumulated, x += alpha p, and read once for C^H, whose error is second
// order in x's rounding since C^H is the energy at its minimiser)
template <typename TX, typename TV, typename TZ = TV, typename TXS = TX>
struct UpdateArgs {
  TXS* x;
  TX* r;
  const TV* p;
  const TV* q;
  TZ* z;
  const TZ* dinv;
  double* partials;
  PcgState* state;
  int n;
  int ld;
  int init;
  double* totals;  // defer != 0: write the 12 reduced sums here, leave state alone
  int defer;
  int gmg;         // 1: z comes from the multigrid V-cycle (this kernel only reduces r.r)
  TZ* gmg_x0;      // gmg: also write the V-cycle's first sweep omega*Dinv*r here
  TZ gmg_omega;
};

template <typename TX>
struct ChomArgs {
  const int* elem_list;
  const int* node_map;
  const double* beta64;
  const TX* x;
  double* partials;
  double* C_out;  // defer == 0: symmetric 6x6; defer != 0: 21 raw sums
  PcgState* state;
  int n_elem;
  int r;
  int ld;
  int zbase;
  int nzl;
  int defer;
};

// Cross-slab reduction: sum `nslab` deferred totals in slab order and update
// the PcgState (emulated slabs on one device, or after an NCCL all-reduce
// with nslab = 1).
void launch_finalize_update(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s);
void launch_finalize_apply(PcgState* st, const double* totals, int nslab, cudaStream_t s);
void launch_finalize_chom(const double* totals, int nslab, double* C_out, cudaStream_t s);
// Ghost-plane transport: nodes [first, first+count) of an 18-component
// blocked vector <-> dense [18][count] buffer.
template <typename T>
void launch_pack(const T* vec, int first, int count, T* buf, cudaStream_t s);
template <typename T>
void launch_unpack(T* vec, int first, int count, const T* buf, cudaStream_t s);

// One multigrid level as the kernels see it (gmg.cuh).
template <typename TV>
struct GmgLevelView {
  const int* node_list;
  const int* node_map;
  const TV* beta;     // level 0: dense r^3 beta (matrix-free operator)
  const TV* stencil;  // levels >= 1: Galerkin 27-point 3x3-block stencils
  const TV* dinv;
  int r, n, zero_slot;
  TV ridge;
  int zbase = 0;             // level 0 of a z-slab: global z of local node-map plane 0
  int n0 = 0;                // sweeps / Jacobi / prolongation cover nodes [n0, n) (a slab's own level-1 planes)
  double* totals = nullptr;  // non-null: the last sweep writes its 6 r.z sums here (slabs)
  BrickView bricks{};        // level 0 with brick numbering: staged brick sweeps
};

void launch_coarse_flags(const int* map_f, int r_f, int r_c, int* flag_c, cudaStream_t s);
// z-slab restriction: b_c += P^T res over the fine nodes the slab owns (planes
// [z0, z1), slab-local node map over planes zbase..).  The slabs' calls (or the
// ranks' all-reduce) sum to the undecomposed restriction.
template <typename TV>
void launch_restrict_slab(const GmgLevelView<TV>& C, const int* map_s, int zbase, int nzl, int z0, int z1, int r_f,
                          const TV* res_f, TV* b_c, const PcgState* st, cudaStream_t s);
// b_c += P^T res_f over the fine nodes [F.n0, F.n) only (a slab's own level-1
// nodes; the slabs' / ranks' partial sums add up to the full restriction)
template <typename TV>
void launch_restrict_partial(const GmgLevelView<TV>& C, const GmgLevelView<TV>& F, const TV* res_f, TV* b_c,
                             const PcgState* st, cudaStream_t s);
// b_c = P^T res on the coarse nodes [C.n0, C.n) a slab owns, from its level-0
// residual (local node map over planes zbase.., ghost planes exchanged first)
template <typename TV>
void launch_restrict_own(const GmgLevelView<TV>& C, const int* map_s, int zbase, int nzl, int r_f, const TV* res_f,
                         TV* b_c, const PcgState* st, cudaStream_t s);
// cross-slab finalize of the multigrid update (r.r only) and of the last sweep's r.z
void launch_finalize_update_gmg(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s);
// set a graph WHILE node's condition to !st->stop (the solve loop runs on the device)
void launch_set_while(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s);
void launch_finalize_gamma(PcgState* st, const double* totals, int nslab, int init, cudaStream_t s);
template <typename TV>
void launch_galerkin(const int* list_c, int n_c, int r_c, const int* map_f, int r_f, const TV* beta_f,
                     const TV* stencil_f, TV ridge, TV* stencil_c, cudaStream_t s);
template <typename TV>
void launch_coarse_dinv(const int* list_c, int n_c, const TV* stencil, TV* dinv, int l1, cudaStream_t s);
// mode 0 smooth, 1 residual, 2 final smooth + gamma = b.x reduction (updates beta)
template <typename TB, typename TV>
void launch_level_sweep(const GmgLevelView<TV>& L, bool fine, const TB* b, const TV* xin, TV* xout,
                        TV omega, int mode, PcgState* st, double* partials, int init, int grid,
                        cudaStream_t s);
// Last level-0 sweep of the V-cycle (mode 2) writing z = M r in the Krylov
// vectors' type TO (FP64 in mixed multigrid, so the apply needs no conversions).
template <typename TB, typename TV, typename TO>
void launch_level_sweep_out(const GmgLevelView<TV>& L, const TB* b, const TV* xin, TO* xout, TV omega,
                            PcgState* st, double* partials, int init, int grid, cudaStream_t s);
template <typename TB, typename TV>
void launch_jacobi_first(const GmgLevelView<TV>& L, const TB* b, TV* xout, TV omega, const PcgState* st,
                         cudaStream_t s);
template <typename TV>
void launch_restrict(const GmgLevelView<TV>& C, const GmgLevelView<TV>& F, const TV* res_f, TV* b_c,
                     const PcgState* st, cudaStream_t s, TV* x_c = nullptr,
                     TV omega = TV(0));
// The whole coarsest-level solve in one cluster kernel (8^3 torus, FP32);
// false when the level does not qualify.
template <typename TV>
bool launch_coarsest(const GmgLevelView<TV>& L, const TV* b, TV* x, TV omega, int sweeps, const PcgState* st,
                     cudaStream_t s);
template <typename TV>
void launch_prolong(const GmgLevelView<TV>& F, const GmgLevelView<TV>& C, const TV* x_c, TV* x_f,
                    const PcgState* st, cudaStream_t s);

// Lease on the device's element constants (K0 in FP64/FP32, K0*T, T and the
// level-1 Galerkin cell matrices), uploaded only when (K0, r) changes and no
// other solve still holds the old ones.  Hold it for the whole solve.
class ElementConstLease {
 public:
  ElementConstLease(const double* K0, const double* W, const double* T, int r, cudaStream_t s);
  ~ElementConstLease();
  ElementConstLease(const ElementConstLease&) = delete;
  ElementConstLease& operator=(const ElementConstLease&) = delete;

 private:
  int device_ = 0;
};
template <typename TX, typename TV>
void launch_setup(const int* node_list, int n_nodes, int ld, int r, const double* beta64,
                  double ridge, TX* rvec, TV* dinv, cudaStream_t s);
template <typename TV, typename TZ>
void launch_apply(const ApplyArgs<TV, TZ>& a, int grid, cudaStream_t s);
// Staged brick kernels of level 0 (brick.cu); used when a.bricks.nab > 0.
template <typename TV, typename TZ>
void launch_brick_apply(const ApplyArgs<TV, TZ>& a, cudaStream_t s);
template <typename TB, typename TV, typename TO>
void launch_brick_sweep(const GmgLevelView<TV>& L, const TB* b, const TV* xin, TO* xout, TV omega, int mode,
                        PcgState* st, double* partials, int init, cudaStream_t s);
void brick_upload_constants(const double* K0d, const float* K0f, cudaStream_t s);
// stored (Galerkin) FP32 level, one CTA per active 8x4x4 brick (L.bricks: bcoord = active brick ids)
void launch_stencil_brick_sweep(const GmgLevelView<float>& L, const float* b, const float* xin, float* xout,
                                float omega, int mode, const PcgState* st, cudaStream_t s);
// active 8x4x4 bricks of a coarse level's node map: flags, then (scan + compaction) their ids
void launch_coarse_brick_flags(const int* map, int r, int* flag, cudaStream_t s);
// Grid (block count) launch_apply / launch_level_sweep use for n nodes; the
// caller sizes its partials buffer as 6 doubles per block.
int apply_grid(int n, int num_sms);
template <typename TX, typename TV, typename TZ, typename TXS = TX>
void launch_update(const UpdateArgs<TX, TV, TZ, TXS>& u, int grid, cudaStream_t s);
template <typename TX>
void launch_chom(const ChomArgs<TX>& c, int grid, cudaStream_t s);

}  // namespace shl
