"""ctypes binding of libshellular_cuda.so (the C ABI of include/shellular_cuda.h).

The product path has no CPU fallback: importing this module when the CUDA
library has not been built raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SHL_LIB") or os.path.join(HERE, "libshellular_cuda.so")

SHL_OK, SHL_VALIDATION, SHL_DEGENERATE, SHL_SOLVER, SHL_IO, SHL_CUDA, SHL_ERROR = range(7)
PREC_AUTO, PREC_FP64, PREC_MIXED, PREC_FP32 = -1, 0, 1, 2
PRECOND_JACOBI, PRECOND_GMG, PRECOND_AUTO = 0, 1, 2


class shl_design(C.Structure):
    _fields_ = [("symmetry", C.c_int), ("K", C.c_int), ("n_charges", C.c_int),
                ("positions", C.POINTER(C.c_double)), ("signs", C.POINTER(C.c_int32)),
                ("weights", C.POINTER(C.c_double))]


class shl_shell_params(C.Structure):
    _fields_ = [("sharpness", C.c_double), ("floor_ratio", C.c_double),
                ("expand_layers", C.c_int)]


class shl_material(C.Structure):
    _fields_ = [("youngs", C.c_double), ("poisson", C.c_double)]


class shl_solve_options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("precision", C.c_int),
                ("check_every", C.c_int), ("preconditioner", C.c_int)]


class shl_stats(C.Structure):
    _fields_ = [("t_field", C.c_double), ("t_mesh", C.c_double), ("t_PBC", C.c_double),
                ("t_AS", C.c_double), ("t_RHS", C.c_double), ("t_solve", C.c_double),
                ("t_C", C.c_double), ("t_fwd", C.c_double),
                ("iterations", C.c_int32 * 6), ("converged", C.c_int32),
                ("full_fallback", C.c_int32), ("precision", C.c_int32), ("lane", C.c_int32),
                ("n_surface", C.c_int64), ("n_elements", C.c_int64), ("n_nodes", C.c_int64),
                ("n_tiles", C.c_int64), ("norm", C.c_double), ("volume_ratio", C.c_double),
                ("apply_ms", C.c_double), ("update_ms", C.c_double),
                ("apply_launches", C.c_int64), ("kernel_launches", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("gmg_levels", C.c_int32), ("precond_fallback", C.c_int32),
                ("n_components", C.c_int32), ("n_floating", C.c_int32)]


# shl_slab_transport (host-staged z-slab transport callbacks)
SLAB_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int)
SLAB_EXCHANGE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                            C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int)


class shl_slab_transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum", SLAB_ALLREDUCE), ("ring_exchange", SLAB_EXCHANGE)]


# every symbol include/shellular_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "shl_ctx_create", "shl_ctx_destroy", "shl_last_error", "shl_set_profiling",
    "shl_sample_grid", "shl_load_grid", "shl_classify_surface", "shl_build_reduced_mesh",
    "shl_grid_solve", "shl_solve_mesh", "shl_homogenize", "shl_homogenize_batch",
    "shl_element_stiffness", "shl_random_design", "shl_expand_symmetry",
    "shl_homogenize_slabs", "shl_nccl_unique_id", "shl_homogenize_zslab", "shl_homogenize_zslab_host",
    "shl_extract_isosurface", "shl_voxel_raw", "shl_set_batch_lanes",
)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
            "paper_2511_04025_b200/csrc). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.shl_ctx_create.argtypes = [C.c_int, P(vp)]
    L.shl_ctx_destroy.argtypes = [vp]
    L.shl_ctx_destroy.restype = None
    L.shl_last_error.argtypes = [vp]
    L.shl_last_error.restype = C.c_char_p
    L.shl_set_profiling.argtypes = [vp, C.c_int]
    L.shl_sample_grid.argtypes = [vp, P(shl_design), C.c_int, vp, vp, P(C.c_double)]
    L.shl_load_grid.argtypes = [vp, C.c_int, vp, vp, C.c_double]
    L.shl_classify_surface.argtypes = [vp, vp, P(C.c_int64)]
    L.shl_build_reduced_mesh.argtypes = [vp, P(shl_shell_params), vp, vp, P(C.c_int64),
                                         P(C.c_int32)]
    L.shl_grid_solve.argtypes = [vp, C.c_int, vp, vp, P(shl_solve_options), vp, P(shl_stats)]
    L.shl_solve_mesh.argtypes = [vp, vp, P(shl_solve_options), vp, P(shl_stats)]
    L.shl_homogenize.argtypes = [vp, P(shl_design), P(shl_shell_params), P(shl_material), C.c_int,
                                 P(shl_solve_options), vp, P(shl_stats)]
    L.shl_homogenize_batch.argtypes = [vp, C.c_int, P(shl_design), P(shl_shell_params),
                                       P(shl_material), C.c_int, P(shl_solve_options), vp,
                                       P(shl_stats), vp]
    L.shl_element_stiffness.argtypes = [P(shl_material), C.c_double, vp]
    L.shl_random_design.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_uint64, vp, vp, vp]
    L.shl_expand_symmetry.argtypes = [P(shl_design), vp, vp, P(C.c_int32)]
    L.shl_homogenize_slabs.argtypes = [vp, C.c_int, P(shl_design), P(shl_shell_params),
                                       P(shl_material), C.c_int, P(shl_solve_options), vp,
                                       P(shl_stats)]
    L.shl_nccl_unique_id.argtypes = [vp]
    L.shl_homogenize_zslab.argtypes = [vp, vp, C.c_int, C.c_int, P(shl_design),
                                       P(shl_shell_params), P(shl_material), C.c_int,
                                       P(shl_solve_options), vp, P(shl_stats)]
    L.shl_homogenize_zslab_host.argtypes = [vp, P(shl_slab_transport), C.c_int, C.c_int, P(shl_design),
                                            P(shl_shell_params), P(shl_material), C.c_int,
                                            P(shl_solve_options), vp, P(shl_stats)]
    L.shl_extract_isosurface.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, P(C.c_int64),
                                         P(C.c_int64)]
    L.shl_voxel_raw.argtypes = [vp, vp]
    L.shl_set_batch_lanes.argtypes = [vp, C.c_int]
    _lib = L
    return L
