/* shellular_cuda.h -- C ABI of the B200-native shellular hot path.
 *
 * The reference (arxiv/paper_2511_04025, /root/reference/proj) has no FFI:
 * its boundary is the inline C++ API in proj/include/shellular/ (*.hpp).  Each
 * entry point below replaces the body of one reference function; the C++
 * drop-in headers in include/shellular/ keep the reference names and call
 * these.  Plain pointers and sizes only, no exceptions across the ABI.
 *
 *   shl_sample_grid        <- sample_grid            field.hpp:488-534
 *   shl_load_grid          <- sample_grid_fn         field.hpp:538-559 (host-sampled fields)
 *   shl_build_reduced_mesh <- build_reduced_mesh     voxel.hpp:235-313
 *                             classify_surface_elements voxel.hpp:118-141
 *   shl_grid_solve         <- GridSolver(...).solve  grid_solver.hpp:20-96
 *   shl_solve_mesh         <- build_periodic_system + solve_test_strains +
 *                             effective_tensor       fem.hpp:179-428
 *   shl_homogenize         <- homogenize             pipeline.hpp:61-113
 *   shl_homogenize_batch   <- (new) many designs, one call (SPEC sample_campaign)
 *   shl_homogenize_slabs / shl_homogenize_zslab
 *                          <- (new) z-slab decomposition of one design (C5)
 *   shl_extract_isosurface <- extract_isosurface     geomio.hpp:45-108
 *   shl_voxel_raw          <- VoxelMesh::write_raw   voxel.hpp:105-114 (bytes)
 *   shl_element_stiffness  <- element_stiffness      fem.hpp:50-92
 *   shl_random_design      <- random_design          field.hpp:569-593
 *   shl_expand_symmetry    <- expand_symmetry        field.hpp:236-249
 *
 * Status codes mirror the reference exception classes (common.hpp:25-48).
 * Host buffers are caller-allocated; device workspaces are owned by the
 * context and reused across calls.  A context is bound to one device and is
 * not thread-safe; distinct contexts are independent.
 */
#ifndef SHELLULAR_CUDA_H
#define SHELLULAR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SHL_OK = 0,
  SHL_VALIDATION = 1, /* ValidationError       */
  SHL_DEGENERATE = 2, /* DegenerateDesignError */
  SHL_SOLVER = 3,     /* SolverError           */
  SHL_IO = 4,         /* IoError               */
  SHL_CUDA = 5,       /* device / driver failure (no reference analogue) */
  SHL_ERROR = 6       /* shellular::Error itself (e.g. empty isosurface) */
};

enum { SHL_SYM_NONE = 0, SHL_SYM_CUBIC_OCTANT = 1, SHL_SYM_TETRAHEDRAL = 2 };

/* arithmetic of the PCG vectors (x, r | p, q, z) and of the K.u apply */
enum {
  SHL_PREC_AUTO = -1,  /* FP64 when tol < 1e-7, else MIXED */
  SHL_PREC_FP64 = 0,   /* everything FP64 */
  SHL_PREC_MIXED = 1,  /* FP32 apply/p/q/z, FP64 x/r/dots */
  SHL_PREC_FP32 = 2    /* FP32 vectors, FP64 dots */
};

typedef struct shl_ctx shl_ctx;

/* DesignParams (field.hpp:131-231), pre-expansion. positions: 3*n_charges
 * (wrapped into [0,1) like the Charge ctor), signs: +-1, weights: (K+1)^3. */
typedef struct {
  int symmetry;
  int K;
  int n_charges;
  const double* positions;
  const int32_t* signs;
  const double* weights;
} shl_design;

/* ShellParams (voxel.hpp:18-34) */
typedef struct {
  double sharpness;   /* 500   */
  double floor_ratio; /* 1e-3  */
  int expand_layers;  /* 0 = max(1, round(2r/64)) */
} shl_shell_params;

/* BaseMaterial (fem.hpp:19-30) */
typedef struct {
  double youngs;  /* 1.0 */
  double poisson; /* 0.3 */
} shl_material;

/* PCG preconditioner */
enum {
  SHL_PRECOND_JACOBI = 0, /* 3x3 block Jacobi (grid_solver.hpp:129-139) */
  SHL_PRECOND_GMG = 1,    /* Galerkin geometric multigrid V-cycle (new) */
  SHL_PRECOND_AUTO = 2    /* GMG when r is even and r/2 >= 8, else block Jacobi */
};

/* Solver options.  Ridge: the reference regularizes a singular system with
 * 1e-11 * mean|diag A| when a component floats or the factorization fails
 * (fem.hpp:337-350).  Floating components are the common case for shell
 * meshes and hinge modes are not detected up front, so the device
 * PCG always adds that ridge to its Krylov operator when it is FP64 (C^H moves
 * by O(1e-11), tested against the unridged direct solve at 1e-8); FP32-storage
 * operators and preconditioners use 1e-8 * mean|diag A| (tested against the
 * FP64 solve at 1e-6).  stats.n_floating reports whether the reference would
 * have ridged (expect_singular). */
typedef struct {
  double tol;         /* per-column ||r|| <= tol*||b|| (grid_solver.hpp:68) */
  int max_iter;       /* 0 = 20r+2000 (grid_solver.hpp:38) */
  int precision;      /* SHL_PREC_* */
  int check_every;    /* host convergence poll period in iterations (0 = auto) */
  int preconditioner; /* SHL_PRECOND_* */
} shl_solve_options;

/* StageTimings (common.hpp:145-160) + solver / mesh statistics */
typedef struct {
  double t_field, t_mesh, t_PBC, t_AS, t_RHS, t_solve, t_C, t_fwd; /* ms, CUDA events */
  int32_t iterations[6];
  int32_t converged;
  int32_t full_fallback;
  int32_t precision; /* resolved SHL_PREC_* */
  int32_t lane;      /* batch lane that ran this design (shl_set_batch_lanes) */
  int64_t n_surface;  /* surface elements before dilation */
  int64_t n_elements; /* active (reduced-mesh) elements */
  int64_t n_nodes;    /* active torus nodes */
  int64_t n_tiles;    /* active apply tiles */
  double norm;        /* max |centre sample| */
  double volume_ratio;
  double apply_ms;  /* summed device time of the K.u apply launches (0 unless profiled) */
  double update_ms; /* update kernel + (GMG) V-cycle, same accounting */
  int64_t apply_launches;
  int64_t kernel_launches; /* kernels launched by this call */
  int64_t h2d_bytes;       /* host->device bytes moved by this call */
  int64_t d2h_bytes;       /* device->host bytes moved by this call */
  int32_t gmg_levels;      /* multigrid levels incl. the fine one (0 = block Jacobi) */
  int32_t precond_fallback; /* 1: AUTO multigrid broke down, solved with block Jacobi;
                               2: mixed multigrid redone with the FP64-accumulated operator */
  int32_t n_components;     /* mechanically connected element components: elements sharing a
                               torus node are coupled (fem.hpp:288-317 union-find criterion) */
  int32_t n_floating;       /* components without an element at torus node 0: their rigid
                               motions are null modes (the reference's expect_singular) */
} shl_stats;

int shl_ctx_create(int device, shl_ctx** out);
void shl_ctx_destroy(shl_ctx* ctx);
/* Message of the last failing call on ctx (or of the calling thread when ctx
 * is NULL). */
const char* shl_last_error(const shl_ctx* ctx);
/* Device-time profiling of apply / update kernels (CUDA events per launch). */
int shl_set_profiling(shl_ctx* ctx, int on);

/* Field sampling on device (bit-exact FP64 reference order).  Any output
 * pointer may be NULL.  centres: r^3, corners: (r+1)^3 incl. wrapped copies,
 * both x fastest.  The grid stays resident in ctx for shl_build_reduced_mesh. */
int shl_sample_grid(shl_ctx* ctx, const shl_design* design, int r, double* centres,
                    double* corners, double* norm);

/* Make a host-sampled grid (sample_grid_fn fixtures) resident in ctx. */
int shl_load_grid(shl_ctx* ctx, int r, const double* centres, const double* corners,
                  double norm);

/* Surface classification only (classify_surface_elements), on the resident
 * grid: writes sorted element ids (capacity r^3) and their count. */
int shl_classify_surface(shl_ctx* ctx, uint32_t* elements, int64_t* n_surface);

/* Reduced mesh on the resident grid.  elements: sorted ids (capacity r^3),
 * beta: per listed element; either may be NULL. */
int shl_build_reduced_mesh(shl_ctx* ctx, const shl_shell_params* sp, uint32_t* elements,
                           double* beta, int64_t* n_elements, int32_t* full_fallback);

/* Six-load-case homogenization of a voxel mesh given by a dense r^3 beta
 * array (0 = absent element), with torus node 0 pinned: the GridSolver of
 * grid_solver.hpp generalized to masked meshes.  K0: 24x24 row-major. */
int shl_grid_solve(shl_ctx* ctx, int r, const double* beta, const double* K0,
                   const shl_solve_options* opt, double* C_out, shl_stats* stats);

/* Same solve on the reduced mesh resident in ctx (after
 * shl_build_reduced_mesh). */
int shl_solve_mesh(shl_ctx* ctx, const double* K0, const shl_solve_options* opt, double* C_out,
                   shl_stats* stats);

/* End-to-end: field -> shell mask -> six-load-case PCG -> C^H (36, row-major). */
int shl_homogenize(shl_ctx* ctx, const shl_design* design, const shl_shell_params* sp,
                   const shl_material* mat, int r, const shl_solve_options* opt, double* C_out,
                   shl_stats* stats);

/* n designs at one resolution; C_out: n*36, stats: n (may be NULL), status:
 * n per-design codes (may be NULL).  Returns SHL_OK unless a device error
 * stops the batch; per-design failures are reported through status. */
/* Designs a batch keeps in flight concurrently (default 1): lanes >= 2 run
 * that many designs at once on sub-contexts of ctx (same device, one stream
 * and host thread each); results and per-design stats are unchanged.  ctx's
 * own streams are recreated at the greatest stream priority on the first
 * multi-lane batch (lane 0 first, other lanes fill its gaps). */
int shl_set_batch_lanes(shl_ctx* ctx, int lanes);
int shl_homogenize_batch(shl_ctx* ctx, int n, const shl_design* designs,
                         const shl_shell_params* sp, const shl_material* mat, int r,
                         const shl_solve_options* opt, double* C_out, shl_stats* stats,
                         int32_t* status);

/* z-slab decomposition of one design's solve (config C5, SURVEY.md §8 e):
 * the torus is split into n_slabs slabs of whole z-planes with one ghost
 * plane per side; per PCG iteration one ghost exchange of z and two small
 * cross-slab sums.
 *   shl_homogenize_slabs : all slabs in this context on one device (the
 *                          exchange is a device copy) -- parity/testing
 *   shl_homogenize_zslab : one slab per rank over NCCL (libnccl dlopen'ed);
 *                          nccl_id from shl_nccl_unique_id on rank 0,
 *                          broadcast by the caller (e.g. torch.distributed). */
int shl_homogenize_slabs(shl_ctx* ctx, int n_slabs, const shl_design* design,
                         const shl_shell_params* sp, const shl_material* mat, int r,
                         const shl_solve_options* opt, double* C_out, shl_stats* stats);
int shl_nccl_unique_id(uint8_t* id_out /*128 bytes*/);
int shl_homogenize_zslab(shl_ctx* ctx, const uint8_t* nccl_id, int rank, int nranks,
                         const shl_design* design, const shl_shell_params* sp,
                         const shl_material* mat, int r, const shl_solve_options* opt,
                         double* C_out, shl_stats* stats);

/* Host-staged transport for the per-rank z-slab solve: the caller's
 * communicator (e.g. torch.distributed over gloo) moves host buffers; the
 * library syncs its stream and stages device data through pinned memory
 * around each call.  Counts are in values (double if f64, else float).
 * Callbacks return 0 on success. */
typedef struct {
  void* user;
  /* element-wise sum over all ranks, in place */
  int (*allreduce_sum)(void* user, void* buf, size_t n, int f64);
  /* periodic ring: send send_hi to rank+1 and send_lo to rank-1; receive
   * recv_lo from rank-1 and recv_hi from rank+1 */
  int (*ring_exchange)(void* user, const void* send_hi, size_t n_send_hi, const void* send_lo,
                       size_t n_send_lo, void* recv_lo, size_t n_recv_lo, void* recv_hi,
                       size_t n_recv_hi, int f64);
} shl_slab_transport;
int shl_homogenize_zslab_host(shl_ctx* ctx, const shl_slab_transport* transport, int rank,
                              int nranks, const shl_design* design, const shl_shell_params* sp,
                              const shl_material* mat, int r, const shl_solve_options* opt,
                              double* C_out, shl_stats* stats);

/* Marching cubes on the resident grid's corner samples: the zero level set
 * with linear edge interpolation, vertices/triangles in exactly the
 * reference's order.  vertices: 3*n_vertices doubles, triangles:
 * 3*n_triangles vertex ids.  Counts are always written; the arrays only when
 * both are non-NULL and their capacities (in vertices / triangles) suffice,
 * so a NULL first call sizes the buffers.  SHL_ERROR when nothing crosses
 * zero. */
int shl_extract_isosurface(shl_ctx* ctx, double* vertices, int64_t vertex_capacity,
                           uint32_t* triangles, int64_t triangle_capacity, int64_t* n_vertices,
                           int64_t* n_triangles);

/* write_raw bytes of the resident reduced mesh: r^3 bytes, 0 = absent,
 * 1 + lround(254 beta) for a mesh element. */
int shl_voxel_raw(shl_ctx* ctx, uint8_t* occupancy);

/* Host helpers (reference arithmetic, no device work). */
int shl_element_stiffness(const shl_material* mat, double edge, double* K_out /*576*/);
int shl_random_design(int symmetry, int n_pre, int K, double weight_lo, double weight_hi,
                      uint64_t seed, double* positions /*3*n_pre*/, int32_t* signs /*n_pre*/,
                      double* weights /*(K+1)^3*/);
int shl_expand_symmetry(const shl_design* design, double* positions_out, int32_t* signs_out,
                        int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* SHELLULAR_CUDA_H */
