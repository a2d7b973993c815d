"""ctypes bindings for the oracle libraries -- TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libshellular_ref.so")

SYM = {"none": 0, "cubic_octant": 1, "tetrahedral": 2}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/include/shellular"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_random_design.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_uint64, _dp, _ip, _dp]
        L.orc_expand_symmetry.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, _dp, _ip,
                                          C.POINTER(C.c_int)]
        L.orc_sample_grid.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, C.c_int, C.c_int,
                                      _dp, _dp, C.POINTER(C.c_double)]
        L.orc_build_reduced_mesh.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                             C.c_int, _u8, _dp, C.POINTER(C.c_int64),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.orc_step_function.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.orc_element_stiffness.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.orc_grid_solve.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_int, C.c_int, C.c_int,
                                     _dp, _ip, _dp, C.c_void_p]
        L.orc_homogenize.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, C.c_double,
                                     C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int, _dp, _ip, _dp, _dp]
        L.orc_extract_isosurface.argtypes = [C.c_int, _dp, C.c_double, _dp, C.c_int64, _u32,
                                             C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def ref():
    """The reference's own field/voxel code (oracle/_ref); None if not built."""
    global _ref
    if _ref is None:
        if not have_ref():
            return None
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_design.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_uint64, _dp, _ip, _dp]
        L.ref_expand_symmetry.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, _dp, _ip,
                                          C.POINTER(C.c_int)]
        L.ref_field_value.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, C.c_int, _dp, _dp]
        L.ref_sample_grid.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, C.c_int, C.c_int,
                                      _dp, _dp, C.POINTER(C.c_double)]
        L.ref_classify.argtypes = [C.c_int, _dp, _dp, C.c_double, _u32, C.POINTER(C.c_int64)]
        L.ref_build_reduced_mesh.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                             C.c_int, _u32, _dp, _i64]
        L.ref_step_function.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.ref_extract_isosurface.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp, C.c_int64, _u32,
                                             C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_write_raw.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_double, C.c_int,
                                    C.c_char_p]
        L.ref_export_mesh.argtypes = [_dp, C.c_int64, _u32, C.c_int64, C.c_char_p, C.c_int]
        _ref = L
    return _ref


def _check(code: int, L, which="orc") -> None:
    if code != 0:
        msg = (L.orc_last_error() if which == "orc" else L.ref_last_error()).decode()
        raise OracleError(code, msg)


# --------------------------------------------------------------------------
@dataclass
class Design:
    """Pre-expansion design (field.hpp:131-231)."""
    symmetry: str = "none"
    K: int = 2
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    signs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(27))

    def arrays(self):
        return (np.ascontiguousarray(self.positions, np.float64).reshape(-1),
                np.ascontiguousarray(self.signs, np.int32),
                np.ascontiguousarray(self.weights, np.float64))


def random_design(symmetry="cubic_octant", n_pre=8, K=2, lo=-1.0, hi=1.0, seed=1,
                  use_ref=False) -> Design:
    """field.hpp:569-593 (splitmix64 draws)."""
    L = ref() if use_ref else lib()
    n = K + 1
    pos = np.zeros(3 * max(n_pre, 0), np.float64)
    sg = np.zeros(max(n_pre, 0), np.int32)
    w = np.zeros(n ** 3, np.float64)
    fn = L.ref_random_design if use_ref else L.orc_random_design
    _check(fn(SYM[symmetry], n_pre, K, lo, hi, seed, pos, sg, w), L, "ref" if use_ref else "orc")
    return Design(symmetry, K, pos.reshape(-1, 3), sg, w)


def expand_symmetry(d: Design, use_ref=False):
    L = ref() if use_ref else lib()
    pos, sg, w = d.arrays()
    mult = {"none": 1, "cubic_octant": 8, "tetrahedral": 48}[d.symmetry]
    po = np.zeros(3 * len(sg) * mult)
    so = np.zeros(len(sg) * mult, np.int32)
    n = C.c_int(0)
    fn = L.ref_expand_symmetry if use_ref else L.orc_expand_symmetry
    _check(fn(SYM[d.symmetry], d.K, len(sg), pos, sg, w, po, so, C.byref(n)), L,
           "ref" if use_ref else "orc")
    return po[: 3 * n.value].reshape(-1, 3), so[: n.value]


@dataclass
class Grid:
    r: int
    samples: np.ndarray  # (r,r,r) indexed [k,j,i]
    corners: np.ndarray  # (r+1,)*3 indexed [k,j,i]
    norm: float


def sample_grid(d: Design, r: int, threads: int = 0, use_ref=False) -> Grid:
    """field.hpp:488-534."""
    L = ref() if use_ref else lib()
    pos, sg, w = d.arrays()
    cen = np.zeros(r ** 3)
    cor = np.zeros((r + 1) ** 3)
    nrm = C.c_double(0)
    fn = L.ref_sample_grid if use_ref else L.orc_sample_grid
    _check(fn(SYM[d.symmetry], d.K, len(sg), pos, sg, w, r, threads, cen, cor, C.byref(nrm)), L,
           "ref" if use_ref else "orc")
    return Grid(r, cen.reshape(r, r, r), cor.reshape(r + 1, r + 1, r + 1), nrm.value)


@dataclass
class Mesh:
    r: int
    occupancy: np.ndarray  # (r,r,r) uint8 [k,j,i]
    beta: np.ndarray  # (r,r,r) float64, 0 = absent
    n_elements: int
    n_surface: int
    full_fallback: bool

    @property
    def elements(self):
        return np.flatnonzero(self.occupancy.reshape(-1)).astype(np.uint32)


def build_reduced_mesh(g: Grid, sharpness=500.0, floor_ratio=1e-3, expand_layers=0) -> Mesh:
    """voxel.hpp:235-313 (element selection + beta)."""
    L = lib()
    r = g.r
    occ = np.zeros(r ** 3, np.uint8)
    beta = np.zeros(r ** 3)
    ne, ns, ff = C.c_int64(0), C.c_int64(0), C.c_int(0)
    _check(L.orc_build_reduced_mesh(r, np.ascontiguousarray(g.samples.reshape(-1)),
                                    np.ascontiguousarray(g.corners.reshape(-1)), g.norm,
                                    sharpness, floor_ratio, expand_layers, occ, beta,
                                    C.byref(ne), C.byref(ns), C.byref(ff)), L)
    return Mesh(r, occ.reshape(r, r, r), beta.reshape(r, r, r), ne.value, ns.value, bool(ff.value))


def ref_build_reduced_mesh(g: Grid, sharpness=500.0, floor_ratio=1e-3, expand_layers=0):
    """The reference's own build_reduced_mesh (incl. topology). Returns (elements, beta, info)."""
    L = ref()
    r = g.r
    el = np.zeros(r ** 3, np.uint32)
    be = np.zeros(r ** 3)
    info = np.zeros(6, np.int64)
    _check(L.ref_build_reduced_mesh(r, np.ascontiguousarray(g.samples.reshape(-1)),
                                    np.ascontiguousarray(g.corners.reshape(-1)), g.norm,
                                    sharpness, floor_ratio, expand_layers, el, be, info), L, "ref")
    n = int(info[0])
    return el[:n].copy(), be[:n].copy(), dict(n_elements=n, n_nodes=int(info[1]),
                                             n_groups=int(info[2]), corner_group=int(info[3]),
                                             full_fallback=bool(info[4]),
                                             corner_group_size=int(info[5]))


def step_function(v, sharpness=500.0, floor_ratio=1e-3, use_ref=False) -> float:
    L = ref() if use_ref else lib()
    out = C.c_double(0)
    fn = L.ref_step_function if use_ref else L.orc_step_function
    _check(fn(float(v), sharpness, floor_ratio, C.byref(out)), L, "ref" if use_ref else "orc")
    return out.value


def element_stiffness(E=1.0, nu=0.3, edge=1.0) -> np.ndarray:
    """fem.hpp:50-92, 24x24."""
    K = np.zeros(576)
    _check(lib().orc_element_stiffness(E, nu, edge, K), lib())
    return K.reshape(24, 24)


@dataclass
class SolveResult:
    C: np.ndarray
    iterations: np.ndarray
    t_rhs_ms: float
    t_solve_ms: float
    t_reduce_ms: float
    n_nodes: int
    n_elements: int
    converged: bool
    x: np.ndarray | None = None


def grid_solve(beta: np.ndarray, K0: np.ndarray, tol=1e-9, max_iter=0, threads=0,
               allow_unconverged=False, want_x=False) -> SolveResult:
    """Masked GridSolver (grid_solver.hpp:18-207 on the masked torus)."""
    beta = np.ascontiguousarray(beta, np.float64)
    r = beta.shape[0]
    C_out = np.zeros(36)
    it = np.zeros(6, np.int32)
    st = np.zeros(6)
    x = np.zeros(r ** 3 * 18) if want_x else None
    _check(lib().orc_grid_solve(r, beta.reshape(-1), np.ascontiguousarray(K0, np.float64).reshape(-1),
                                tol, max_iter, threads, int(allow_unconverged), C_out, it, st,
                                x.ctypes.data if want_x else None), lib())
    return SolveResult(C_out.reshape(6, 6), it, st[0], st[1], st[2], int(st[3]), int(st[4]),
                       bool(st[5]), x.reshape(r, r, r, 3, 6) if want_x else None)


@dataclass
class HomogenizeResult:
    C: np.ndarray
    iterations: np.ndarray
    timings: dict
    n_elements: int
    n_nodes: int
    volume_ratio: float
    full_fallback: bool
    converged: bool


TIMING_KEYS = ("t_field", "t_mesh", "t_PBC", "t_AS", "t_RHS", "t_solve", "t_C", "t_fwd")


def homogenize(d: Design, r: int, sharpness=500.0, floor_ratio=1e-3, expand_layers=0, E=1.0,
               nu=0.3, threads=0, tol=1e-9, max_iter=0, allow_unconverged=False) -> HomogenizeResult:
    """pipeline.hpp:61-113 with the masked matrix-free solve."""
    pos, sg, w = d.arrays()
    C_out = np.zeros(36)
    it = np.zeros(6, np.int32)
    tm = np.zeros(8)
    info = np.zeros(5)
    _check(lib().orc_homogenize(SYM[d.symmetry], d.K, len(sg), pos, sg, w, sharpness, floor_ratio,
                                expand_layers, E, nu, r, threads, tol, max_iter,
                                int(allow_unconverged), C_out, it, tm, info), lib())
    return HomogenizeResult(C_out.reshape(6, 6), it, dict(zip(TIMING_KEYS, tm.tolist())),
                            int(info[0]), int(info[1]), float(info[2]), bool(info[3]),
                            bool(info[4]))


# ---- fixtures used throughout the reference tests -------------------------
def seeded_design(seed: int) -> Design:
    """test_voxel.cpp:26-31 / test_fem.cpp:17-22: CubicOctant, 4 pre, K=2."""
    return random_design("cubic_octant", 4, 2, -1.0, 1.0, seed)


def plane_design_z(shift: float = 0.0) -> Design:
    """test_voxel.cpp:15-24."""
    w = np.zeros(27)
    w[1] = 1.0  # weight(0,0,1)
    return Design("none", 2, np.array([[0.5, 0.5, 0.25 + shift], [0.5, 0.5, 0.75 + shift]]),
                  np.array([1, -1], np.int32), w)


def gyroid_design() -> Design:
    """Config C2: 16 charges at the gyroid extrema, alpha=1 for |hkl|^2 <= 2."""
    plus = [(1, 1, 1), (1, 7, 3), (3, 1, 7), (3, 7, 5), (5, 3, 7), (5, 5, 5), (7, 3, 1), (7, 5, 3)]
    minus = [(1, 3, 5), (1, 5, 7), (3, 3, 3), (3, 5, 1), (5, 1, 3), (5, 7, 1), (7, 1, 5), (7, 7, 7)]
    pos = np.array(plus + minus, np.float64) / 8.0
    sg = np.array([1] * 8 + [-1] * 8, np.int32)
    w = np.zeros(27)
    for h in range(3):
        for k in range(3):
            for l in range(3):
                if (h, k, l) != (0, 0, 0) and h * h + k * k + l * l <= 2:
                    w[(h * 3 + k) * 3 + l] = 1.0
    return Design("none", 2, pos, sg, w)


def extract_isosurface(g: Grid, use_ref=False):
    """geomio.hpp:45-108 marching cubes.  Returns (vertices (n,3) f64, triangles (m,3) u32)."""
    L = ref() if use_ref else lib()
    cor = np.ascontiguousarray(g.corners.reshape(-1))
    nv, nt = C.c_int64(0), C.c_int64(0)
    empty_d, empty_u = np.zeros(1), np.zeros(1, np.uint32)
    if use_ref:
        cen = np.ascontiguousarray(g.samples.reshape(-1))
        call = lambda v, vc, t, tc: L.ref_extract_isosurface(g.r, cen, cor, g.norm, v, vc, t, tc,
                                                             C.byref(nv), C.byref(nt))
    else:
        call = lambda v, vc, t, tc: L.orc_extract_isosurface(g.r, cor, g.norm, v, vc, t, tc,
                                                             C.byref(nv), C.byref(nt))
    _check(call(empty_d, 0, empty_u, 0), L, "ref" if use_ref else "orc")
    v = np.zeros(3 * nv.value)
    t = np.zeros(3 * nt.value, np.uint32)
    _check(call(v, nv.value, t, nt.value), L, "ref" if use_ref else "orc")
    return v.reshape(-1, 3), t.reshape(-1, 3)


def ref_write_raw(g: Grid, path: str, sharpness=500.0, floor_ratio=1e-3, expand_layers=0) -> None:
    """VoxelMesh::write_raw (voxel.hpp:105-114) of the reference's build_reduced_mesh."""
    L = ref()
    _check(L.ref_write_raw(g.r, np.ascontiguousarray(g.samples.reshape(-1)),
                           np.ascontiguousarray(g.corners.reshape(-1)), g.norm, sharpness,
                           floor_ratio, expand_layers, path.encode()), L, "ref")


def ref_export_mesh(vertices: np.ndarray, triangles: np.ndarray, path: str, fmt: str = "stl") -> None:
    """export_mesh (geomio.hpp:277-316): fmt 'stl' (binary) or 'obj'."""
    L = ref()
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
    t = np.ascontiguousarray(triangles, np.uint32).reshape(-1)
    _check(L.ref_export_mesh(v, len(v) // 3, t, len(t) // 3, path.encode(), 0 if fmt == "stl" else 1),
           L, "ref")


__all__ = [n for n in dir() if not n.startswith("_")]
