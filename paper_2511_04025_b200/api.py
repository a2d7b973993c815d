"""Python mirror of the reference ``shellular`` API over the CUDA C ABI.

Same names, argument meaning and error classes as
``/root/reference/proj/include/shellular`` (field.hpp, voxel.hpp, fem.hpp,
grid_solver.hpp, pipeline.hpp); every call crosses into libshellular_cuda.so.
The C++ drop-in (include/shellular/*.hpp) is the primary host API; this
module is what tests, the sweep driver and bench.py use from Python.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib as L

# ---- errors (common.hpp:25-48) ---------------------------------------------


class Error(RuntimeError):
    """Base of the shellular error hierarchy."""


class ValidationError(Error):
    pass


class DegenerateDesignError(Error):
    pass


class SolverError(Error):
    pass


class IoError(Error):
    pass


class CudaError(Error):
    """Device / driver failure (no reference analogue)."""


_ERR = {L.SHL_VALIDATION: ValidationError, L.SHL_DEGENERATE: DegenerateDesignError,
        L.SHL_SOLVER: SolverError, L.SHL_IO: IoError, L.SHL_CUDA: CudaError, L.SHL_ERROR: Error}


def _check(code: int, ctx=None) -> None:
    if code != L.SHL_OK:
        msg = L.lib().shl_last_error(ctx.handle if ctx is not None else None)
        raise _ERR.get(code, Error)(msg.decode() if msg else f"status {code}")


# ---- design space (field.hpp) -----------------------------------------------
SYMMETRY = {"none": 0, "cubic_octant": 1, "tetrahedral": 2}


@dataclass
class DesignParams:
    """field.hpp:131-231 -- pre-expansion charges (n,3) + signs, flat weights (K+1)^3."""
    symmetry: str = "none"
    truncation: int = 2
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    signs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(27))

    def weight_index(self, h: int, k: int, l: int) -> int:
        n = self.truncation + 1
        return (h * n + k) * n + l

    def _abi(self):
        pos = np.ascontiguousarray(np.asarray(self.positions, np.float64).reshape(-1))
        sg = np.ascontiguousarray(np.asarray(self.signs, np.int32).reshape(-1))
        w = np.ascontiguousarray(np.asarray(self.weights, np.float64).reshape(-1))
        d = L.shl_design(SYMMETRY[self.symmetry], int(self.truncation), len(sg),
                         pos.ctypes.data_as(C.POINTER(C.c_double)),
                         sg.ctypes.data_as(C.POINTER(C.c_int32)),
                         w.ctypes.data_as(C.POINTER(C.c_double)))
        return d, (pos, sg, w)  # keep the arrays alive with the struct


@dataclass
class RandomDesignSpec:
    """field.hpp:561-567."""
    symmetry: str = "cubic_octant"
    n_charges_pre_expansion: int = 8
    truncation: int = 2
    weight_lo: float = -1.0
    weight_hi: float = 1.0


def random_design(spec: RandomDesignSpec, seed: int) -> DesignParams:
    """field.hpp:569-593 (splitmix64; bit-identical to the compiled reference)."""
    n = spec.truncation + 1
    npre = max(spec.n_charges_pre_expansion, 0)
    pos = np.zeros(3 * npre)
    sg = np.zeros(npre, np.int32)
    w = np.zeros(max(n, 1) ** 3)
    _check(L.lib().shl_random_design(SYMMETRY[spec.symmetry], spec.n_charges_pre_expansion,
                                     spec.truncation, spec.weight_lo, spec.weight_hi,
                                     int(seed) & (2 ** 64 - 1), pos.ctypes.data, sg.ctypes.data,
                                     w.ctypes.data))
    return DesignParams(spec.symmetry, spec.truncation, pos.reshape(-1, 3), sg, w)


def expand_symmetry(p: DesignParams) -> DesignParams:
    """field.hpp:236-249."""
    mult = {"none": 1, "cubic_octant": 8, "tetrahedral": 48}[p.symmetry]
    d, keep = p._abi()
    cap = max(d.n_charges * mult, 1)
    pos = np.zeros(3 * cap)
    sg = np.zeros(cap, np.int32)
    n = C.c_int32(0)
    _check(L.lib().shl_expand_symmetry(C.byref(d), pos.ctypes.data, sg.ctypes.data, C.byref(n)))
    m = n.value
    return DesignParams("none", p.truncation, pos[: 3 * m].reshape(-1, 3), sg[:m].copy(),
                        np.asarray(p.weights, np.float64).copy())


# ---- device context ----------------------------------------------------------
class Context:
    """One shl_ctx: a device, a stream and reusable device workspaces."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(L.lib().shl_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            L.lib().shl_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on: bool) -> None:
        _check(L.lib().shl_set_profiling(self.handle, int(bool(on))), self)


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ---- field (field.hpp:397-559) -------------------------------------------------
@dataclass
class FieldGrid:
    resolution: int
    samples: np.ndarray          # (r,r,r) [k,j,i]
    corner_samples: np.ndarray   # (r+1,)*3 [k,j,i]
    norm: float

    def degenerate(self) -> bool:
        return self.norm == 0.0

    def center(self, i, j, k):
        return self.samples[k, j, i]

    def corner(self, i, j, k):
        return self.corner_samples[k, j, i]


def sample_grid(params: DesignParams, r: int, ctx: Context | None = None) -> FieldGrid:
    """field.hpp:488-534 on the device (FP64, bit-identical to the reference)."""
    ctx = ctx or default_context()
    d, keep = params._abi()
    r = int(r)
    cen = np.zeros(max(r, 0) ** 3)
    cor = np.zeros((max(r, 0) + 1) ** 3)
    nrm = C.c_double(0.0)
    _check(L.lib().shl_sample_grid(ctx.handle, C.byref(d), r, cen.ctypes.data, cor.ctypes.data,
                                   C.byref(nrm)), ctx)
    return FieldGrid(r, cen.reshape(r, r, r), cor.reshape(r + 1, r + 1, r + 1), nrm.value)


def sample_grid_fn(fn: Callable[[np.ndarray, np.ndarray, np.ndarray], np.ndarray],
                   r: int) -> FieldGrid:
    """field.hpp:538-559 (host-evaluated analytic fixtures; fn is vectorized over x,y,z)."""
    if r < 4:
        raise ValidationError("grid resolution must be >= 4")
    c = (np.arange(r) + 0.5) / r
    k, j, i = np.meshgrid(c, c, c, indexing="ij")
    cen = np.asarray(fn(i, j, k), np.float64) * np.ones_like(i)
    e = np.arange(r + 1) / r
    k, j, i = np.meshgrid(e, e, e, indexing="ij")
    cor = np.asarray(fn(i, j, k), np.float64) * np.ones_like(i)
    return FieldGrid(r, cen, cor, float(np.max(np.abs(cen))))


def _load_grid(grid: FieldGrid, ctx: Context) -> None:
    cen = np.ascontiguousarray(grid.samples, np.float64).reshape(-1)
    cor = np.ascontiguousarray(grid.corner_samples, np.float64).reshape(-1)
    _check(L.lib().shl_load_grid(ctx.handle, int(grid.resolution), cen.ctypes.data,
                                 cor.ctypes.data, float(grid.norm)), ctx)


# ---- voxelization (voxel.hpp) -------------------------------------------------------
@dataclass
class ShellParams:
    """voxel.hpp:18-34."""
    sharpness: float = 500.0
    floor_ratio: float = 1e-3
    expand_layers: int = 0

    def layers_for(self, r: int) -> int:
        if self.expand_layers > 0:
            return self.expand_layers
        return max(1, int(np.floor(2.0 * r / 64.0 + 0.5)))

    def _abi(self):
        return L.shl_shell_params(float(self.sharpness), float(self.floor_ratio),
                                  int(self.expand_layers))


@dataclass
class VoxelMesh:
    resolution: int
    elements: np.ndarray  # sorted linear ids (k*r + j)*r + i
    beta: np.ndarray
    full_fallback: bool

    def num_elements(self) -> int:
        return len(self.elements)

    def element_fraction(self) -> float:
        return len(self.elements) / float(self.resolution) ** 3

    def volume_ratio(self) -> float:
        return float(np.sum(self.beta)) / float(self.resolution) ** 3

    def raw_bytes(self) -> np.ndarray:
        """voxel.hpp:105-114 occupancy bytes: 0 absent, 1 + lround(254 beta)."""
        occ = np.zeros(self.resolution ** 3, np.uint8)
        x = np.asarray(self.beta, np.float64) * 254.0
        f = np.floor(x)
        occ[self.elements] = (1 + f + (x - f >= 0.5)).astype(np.uint8)  # lround, x >= 0
        return occ

    def write_raw(self, path: str) -> None:
        """VoxelMesh::write_raw (voxel.hpp:105-114)."""
        try:
            with open(path, "wb") as f:
                f.write(self.raw_bytes().tobytes())
        except OSError as e:
            raise IoError(f"cannot open '{path}' for writing") from e


def classify_surface_elements(grid: FieldGrid, ctx: Context | None = None) -> np.ndarray:
    """voxel.hpp:118-141."""
    ctx = ctx or default_context()
    if grid.degenerate():
        raise DegenerateDesignError("cannot classify surface elements of a degenerate field")
    _load_grid(grid, ctx)
    out = np.zeros(grid.resolution ** 3, np.uint32)
    n = C.c_int64(0)
    _check(L.lib().shl_classify_surface(ctx.handle, out.ctypes.data, C.byref(n)), ctx)
    return out[: n.value].copy()


def build_reduced_mesh(grid: FieldGrid, sp: ShellParams = ShellParams(),
                       ctx: Context | None = None) -> VoxelMesh:
    """voxel.hpp:235-313 (element set + beta; topology is implicit on the torus)."""
    ctx = ctx or default_context()
    _load_grid(grid, ctx)
    r = grid.resolution
    el = np.zeros(r ** 3, np.uint32)
    be = np.zeros(r ** 3)
    n = C.c_int64(0)
    ff = C.c_int32(0)
    spa = sp._abi()
    _check(L.lib().shl_build_reduced_mesh(ctx.handle, C.byref(spa), el.ctypes.data,
                                          be.ctypes.data, C.byref(n), C.byref(ff)), ctx)
    return VoxelMesh(r, el[: n.value].copy(), be[: n.value].copy(), bool(ff.value))


def voxel_raw(grid: FieldGrid, sp: ShellParams = ShellParams(),
              ctx: Context | None = None) -> np.ndarray:
    """write_raw bytes of build_reduced_mesh(grid, sp), quantized on the device (r^3 uint8)."""
    ctx = ctx or default_context()
    build_reduced_mesh(grid, sp, ctx)
    occ = np.zeros(grid.resolution ** 3, np.uint8)
    _check(L.lib().shl_voxel_raw(ctx.handle, occ.ctypes.data), ctx)
    return occ


def full_solid_mesh(r: int, beta_value: float = 1.0) -> VoxelMesh:
    """voxel.hpp:316-326."""
    return VoxelMesh(r, np.arange(r ** 3, dtype=np.uint32), np.full(r ** 3, float(beta_value)),
                     True)


# ---- geometry export (geomio.hpp) --------------------------------------------------
@dataclass
class TriMesh:
    """geomio.hpp:18-39."""
    vertices: np.ndarray   # (n, 3) float64
    triangles: np.ndarray  # (m, 3) uint32

    def area(self) -> float:
        v = self.vertices
        t = self.triangles.astype(np.int64)
        e1, e2 = v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]]
        return float(0.5 * np.linalg.norm(np.cross(e1, e2), axis=1).sum())

    def signed_volume(self) -> float:
        v = self.vertices
        t = self.triangles.astype(np.int64)
        return float(np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6.0)


def extract_isosurface(grid: FieldGrid, ctx: Context | None = None) -> TriMesh:
    """geomio.hpp:45-108: marching cubes on the device; the reference's vertices,
    triangles and ordering, bit for bit."""
    ctx = ctx or default_context()
    if grid.degenerate():
        raise DegenerateDesignError("cannot extract isosurface of a degenerate field")
    _load_grid(grid, ctx)
    nv, nt = C.c_int64(0), C.c_int64(0)
    _check(L.lib().shl_extract_isosurface(ctx.handle, None, 0, None, 0, C.byref(nv), C.byref(nt)), ctx)
    v = np.zeros((nv.value, 3))
    t = np.zeros((nt.value, 3), np.uint32)
    _check(L.lib().shl_extract_isosurface(ctx.handle, v.ctypes.data, nv.value, t.ctypes.data, nt.value,
                                          C.byref(nv), C.byref(nt)), ctx)
    return TriMesh(v, t)


def export_mesh(mesh: TriMesh, path: str, fmt: str = "stl") -> None:
    """geomio.hpp:272-316: fmt "stl" (binary) or "obj"; same bytes as the reference."""
    if len(mesh.triangles) == 0:
        raise ValidationError("refusing to export an empty mesh")
    if fmt not in ("stl", "obj"):
        raise ValidationError(f"unknown mesh format '{fmt}'")
    v = np.asarray(mesh.vertices, np.float64)
    t = np.asarray(mesh.triangles, np.int64)
    try:
        f = open(path, "wb")
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing") from e
    with f:
        if fmt == "stl":
            header = b"shellular voxel cell export".ljust(80, b"\0")
            a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
            # Vec3 cross / norm / division in the reference's order (no FMA in numpy)
            e1, e2 = b - a, c - a
            n = np.stack([e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1],
                          e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2],
                          e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]], axis=1)
            ln = np.sqrt((n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1]) + n[:, 2] * n[:, 2])
            nz = ln > 0.0
            n[nz] = n[nz] / ln[nz, None]
            rec = np.zeros(len(t), dtype=[("f", "<f4", 12), ("attr", "<u2")])
            rec["f"] = np.concatenate([n, a, b, c], axis=1).astype(np.float32)
            f.write(header)
            f.write(np.uint32(len(t)).tobytes())
            f.write(rec.tobytes())
        else:
            lines = [f"v {_g17(x)} {_g17(y)} {_g17(z)}\n" for x, y, z in v]
            lines += [f"f {i + 1} {j + 1} {k + 1}\n" for i, j, k in t]
            f.write("".join(lines).encode())


def _g17(x: float) -> str:
    """std::ostream << double with precision(17) (%.17g)."""
    return "%.17g" % x


# ---- FEM (fem.hpp) ------------------------------------------------------------------
@dataclass
class BaseMaterial:
    """fem.hpp:19-30."""
    youngs: float = 1.0
    poisson: float = 0.3

    def lam(self) -> float:
        E, nu = self.youngs, self.poisson
        return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))

    def mu(self) -> float:
        return self.youngs / (2.0 * (1.0 + self.poisson))

    def _abi(self):
        return L.shl_material(float(self.youngs), float(self.poisson))


def element_stiffness(mat: BaseMaterial, edge: float) -> np.ndarray:
    """fem.hpp:50-92 -> (24, 24)."""
    K = np.zeros(576)
    m = mat._abi()
    _check(L.lib().shl_element_stiffness(C.byref(m), float(edge), K.ctypes.data))
    return K.reshape(24, 24)


def isotropic_tensor(mat: BaseMaterial) -> np.ndarray:
    """ElasticTensor::isotropic (fem.hpp:99-106)."""
    C6 = np.zeros((6, 6))
    C6[:3, :3] = mat.lam()
    for a in range(3):
        C6[a, a] = mat.lam() + 2 * mat.mu()
        C6[3 + a, 3 + a] = mat.mu()
    return C6


PRECISION = {"auto": L.PREC_AUTO, "fp64": L.PREC_FP64, "mixed": L.PREC_MIXED,
             "fp32": L.PREC_FP32}
PRECISION_NAME = {v: k for k, v in PRECISION.items()}
PRECONDITIONER = {"jacobi": L.PRECOND_JACOBI, "gmg": L.PRECOND_GMG, "auto": L.PRECOND_AUTO}


@dataclass
class HomogenizeOptions:
    """pipeline.hpp:15-20, with the device solver's knobs."""
    residual_tol: float = 1e-9
    max_iter: int = 0
    precision: str = "auto"
    check_every: int = 0
    # "auto" (multigrid when r is even and r/2 >= 8) | "gmg" | "jacobi" (grid_solver.hpp:129-139)
    preconditioner: str = "auto"

    def _abi(self):
        return L.shl_solve_options(float(self.residual_tol), int(self.max_iter),
                                   PRECISION[self.precision], int(self.check_every),
                                   PRECONDITIONER[self.preconditioner])


TIMING_KEYS = ("t_field", "t_mesh", "t_PBC", "t_AS", "t_RHS", "t_solve", "t_C", "t_fwd")


@dataclass
class SolveStats:
    timings: dict
    iterations: np.ndarray
    converged: bool
    precision: str
    n_surface: int
    n_elements: int
    n_nodes: int
    n_tiles: int
    norm: float
    volume_ratio: float
    full_fallback: bool
    apply_ms: float
    update_ms: float
    apply_launches: int
    kernel_launches: int
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    gmg_levels: int = 0
    precond_fallback: int = 0  # 1: block-Jacobi redo, 2: FP64-operator redo (shellular_cuda.h)
    lane: int = 0              # batch lane (homogenize_batch(lanes=...))
    n_components: int = 0      # mechanically connected element components (fem.hpp:288-317)
    n_floating: int = 0        # ... without an element at torus node 0 (expect_singular)

    @classmethod
    def from_abi(cls, s: L.shl_stats) -> "SolveStats":
        return cls({k: getattr(s, k) for k in TIMING_KEYS}, np.array(list(s.iterations)),
                   bool(s.converged), PRECISION_NAME.get(s.precision, "?"), s.n_surface,
                   s.n_elements, s.n_nodes, s.n_tiles, s.norm, s.volume_ratio,
                   bool(s.full_fallback), s.apply_ms, s.update_ms, s.apply_launches,
                   s.kernel_launches, s.h2d_bytes, s.d2h_bytes, s.gmg_levels, s.precond_fallback,
                   s.lane, s.n_components, s.n_floating)


class GridSolver:
    """grid_solver.hpp:18-207, generalized to masked meshes (beta == 0 -> absent)."""

    @dataclass
    class Result:
        tensor: np.ndarray
        iterations: np.ndarray
        t_rhs_ms: float
        t_solve_ms: float
        t_reduce_ms: float
        stats: SolveStats

    def __init__(self, beta: np.ndarray, r: int, K0: np.ndarray, ctx: Context | None = None,
                 precision: str = "auto", preconditioner: str = "jacobi"):
        beta = np.ascontiguousarray(beta, np.float64).reshape(-1)
        if beta.size != r ** 3:
            raise ValidationError("beta array does not match resolution")
        self.beta, self.r = beta, int(r)
        self.K0 = np.ascontiguousarray(K0, np.float64).reshape(-1)
        self.ctx = ctx or default_context()
        self.precision = precision
        self.preconditioner = preconditioner

    def solve(self, tol: float = 1e-9, max_iter: int = 0) -> "GridSolver.Result":
        opt = HomogenizeOptions(tol, max_iter, self.precision, 0, self.preconditioner)._abi()
        Cm = np.zeros(36)
        st = L.shl_stats()
        _check(L.lib().shl_grid_solve(self.ctx.handle, self.r, self.beta.ctypes.data,
                                      self.K0.ctypes.data, C.byref(opt), Cm.ctypes.data,
                                      C.byref(st)), self.ctx)
        s = SolveStats.from_abi(st)
        return GridSolver.Result(Cm.reshape(6, 6), s.iterations, s.timings["t_RHS"],
                                 s.timings["t_solve"], s.timings["t_C"], s)


def solve_mesh(mesh: VoxelMesh, K0: np.ndarray, opt: HomogenizeOptions = HomogenizeOptions(),
               ctx: Context | None = None):
    """build_periodic_system + solve_test_strains + effective_tensor (fem.hpp:179-428)
    for an explicit mesh, through the masked-torus device solver."""
    r = mesh.resolution
    beta = np.zeros(r ** 3)
    beta[np.asarray(mesh.elements, np.int64)] = mesh.beta
    solver = GridSolver(beta, r, K0, ctx, opt.precision)
    return solver.solve(opt.residual_tol, opt.max_iter)


# ---- pipeline (pipeline.hpp) ---------------------------------------------------------
@dataclass
class HomogenizationResult:
    """pipeline.hpp:22-38 (grid/mesh are not copied back; see stats)."""
    tensor: np.ndarray
    resolution: int
    timings: dict
    volume_ratio: float
    element_fraction: float
    solver_used: str
    iterations: np.ndarray
    stats: SolveStats

    def to_json(self) -> dict:
        return {"C": self.tensor.tolist(), "resolution": self.resolution,
                "volume_ratio": self.volume_ratio, "element_fraction": self.element_fraction,
                "solver": self.solver_used, "timings_ms": dict(self.timings),
                "iterations": [int(v) for v in self.iterations]}


def homogenize(params: DesignParams, sp: ShellParams, mat: BaseMaterial, r: int,
               opt: HomogenizeOptions = HomogenizeOptions(),
               ctx: Context | None = None) -> HomogenizationResult:
    """pipeline.hpp:61-113 entirely on the device."""
    ctx = ctx or default_context()
    d, keep = params._abi()
    spa, ma, oa = sp._abi(), mat._abi(), opt._abi()
    Cm = np.zeros(36)
    st = L.shl_stats()
    _check(L.lib().shl_homogenize(ctx.handle, C.byref(d), C.byref(spa), C.byref(ma), int(r),
                                  C.byref(oa), Cm.ctypes.data, C.byref(st)), ctx)
    s = SolveStats.from_abi(st)
    return HomogenizationResult(Cm.reshape(6, 6), int(r), s.timings, s.volume_ratio,
                                s.n_elements / float(r) ** 3, f"device_pcg_{s.precision}",
                                s.iterations, s)


def homogenize_batch(designs: Sequence[DesignParams], sp: ShellParams, mat: BaseMaterial, r: int,
                     opt: HomogenizeOptions = HomogenizeOptions(),
                     ctx: Context | None = None, lanes: int = 1):
    """Many designs in one C-ABI call (shl_homogenize_batch), `lanes` of them in
    flight at once on the device. Returns (C[n,6,6], status[n], stats)."""
    ctx = ctx or default_context()
    _check(L.lib().shl_set_batch_lanes(ctx.handle, int(lanes)), ctx)
    n = len(designs)
    arr = (L.shl_design * max(n, 1))()
    keep = []
    for i, p in enumerate(designs):
        d, k = p._abi()
        arr[i] = d
        keep.append(k)
    spa, ma, oa = sp._abi(), mat._abi(), opt._abi()
    Cm = np.zeros(36 * max(n, 1))
    stats = (L.shl_stats * max(n, 1))()
    status = np.zeros(max(n, 1), np.int32)
    _check(L.lib().shl_homogenize_batch(ctx.handle, n, arr, C.byref(spa), C.byref(ma), int(r),
                                        C.byref(oa), Cm.ctypes.data, stats, status.ctypes.data),
           ctx)
    return (Cm[: 36 * n].reshape(n, 6, 6), status[:n].copy(),
            [SolveStats.from_abi(stats[i]) for i in range(n)])


# ---- z-slab decomposition of one design (config C5) -----------------------------
def homogenize_slabs(params: DesignParams, sp: ShellParams, mat: BaseMaterial, r: int,
                     n_slabs: int, opt: HomogenizeOptions = HomogenizeOptions(),
                     ctx: Context | None = None) -> HomogenizationResult:
    """The z-slab solver with all `n_slabs` slabs in one context (device-copy
    ghost exchange, fixed-order cross-slab sums) -- the multi-rank code path
    exercised on a single GPU."""
    ctx = ctx or default_context()
    d, keep = params._abi()
    spa, ma, oa = sp._abi(), mat._abi(), opt._abi()
    Cm = np.zeros(36)
    st = L.shl_stats()
    _check(L.lib().shl_homogenize_slabs(ctx.handle, int(n_slabs), C.byref(d), C.byref(spa),
                                        C.byref(ma), int(r), C.byref(oa), Cm.ctypes.data,
                                        C.byref(st)), ctx)
    s = SolveStats.from_abi(st)
    return HomogenizationResult(Cm.reshape(6, 6), int(r), s.timings, s.volume_ratio,
                                s.n_elements / float(r) ** 3, f"device_pcg_{s.precision}_zslab{n_slabs}",
                                s.iterations, s)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(L.lib().shl_nccl_unique_id(buf))
    return bytes(buf)


def homogenize_zslab_host(params: DesignParams, sp: ShellParams, mat: BaseMaterial, r: int,
                          rank: int, nranks: int, transport,
                          opt: HomogenizeOptions = HomogenizeOptions(),
                          ctx: Context | None = None) -> HomogenizationResult:
    """One z-slab per rank over a host-staged transport (shl_homogenize_zslab_host):
    `transport.allreduce_sum(buf)` sums a host numpy array over the ranks in
    place; `transport.ring_exchange(send_hi, send_lo, recv_lo, recv_hi)` sends
    to rank+1 / rank-1 and receives from rank-1 / rank+1 (numpy views of the
    library's pinned staging buffers).  See zslab.TorchSlabTransport."""
    ctx = ctx or default_context()
    d, keep = params._abi()
    spa, ma, oa = sp._abi(), mat._abi(), opt._abi()

    def view(ptr, n, f64):
        if n == 0:
            return np.zeros(0, np.float64 if f64 else np.float32)
        ct = (C.c_double if f64 else C.c_float) * n
        return np.ctypeslib.as_array(ct.from_address(ptr))

    def allreduce(user, buf, n, f64):
        try:
            transport.allreduce_sum(view(buf, n, f64))
            return 0
        except Exception:  # noqa: BLE001 - no exception may cross the C ABI
            import traceback
            traceback.print_exc()
            return 1

    def exchange(user, shi, nshi, slo, nslo, rlo, nrlo, rhi, nrhi, f64):
        try:
            transport.ring_exchange(view(shi, nshi, f64), view(slo, nslo, f64), view(rlo, nrlo, f64),
                                    view(rhi, nrhi, f64))
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    cbs = (L.SLAB_ALLREDUCE(allreduce), L.SLAB_EXCHANGE(exchange))  # kept alive for the call
    tr = L.shl_slab_transport(None, cbs[0], cbs[1])
    Cm = np.zeros(36)
    st = L.shl_stats()
    _check(L.lib().shl_homogenize_zslab_host(ctx.handle, C.byref(tr), int(rank), int(nranks), C.byref(d),
                                             C.byref(spa), C.byref(ma), int(r), C.byref(oa),
                                             Cm.ctypes.data, C.byref(st)), ctx)
    s = SolveStats.from_abi(st)
    return HomogenizationResult(Cm.reshape(6, 6), int(r), s.timings, s.volume_ratio,
                                s.n_elements / float(r) ** 3, f"device_pcg_{s.precision}_zslab_host",
                                s.iterations, s)


def homogenize_zslab(params: DesignParams, sp: ShellParams, mat: BaseMaterial, r: int,
                     nccl_id: bytes, rank: int, nranks: int,
                     opt: HomogenizeOptions = HomogenizeOptions(),
                     ctx: Context | None = None) -> HomogenizationResult:
    """One z-slab per rank over NCCL (every rank passes the same nccl_id)."""
    ctx = ctx or default_context()
    d, keep = params._abi()
    spa, ma, oa = sp._abi(), mat._abi(), opt._abi()
    idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
    Cm = np.zeros(36)
    st = L.shl_stats()
    _check(L.lib().shl_homogenize_zslab(ctx.handle, idb, int(rank), int(nranks), C.byref(d),
                                        C.byref(spa), C.byref(ma), int(r), C.byref(oa),
                                        Cm.ctypes.data, C.byref(st)), ctx)
    s = SolveStats.from_abi(st)
    return HomogenizationResult(Cm.reshape(6, 6), int(r), s.timings, s.volume_ratio,
                                s.n_elements / float(r) ** 3, f"device_pcg_{s.precision}_zslab",
                                s.iterations, s)
