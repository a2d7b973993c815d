"""Reference master-slave direct path + test oracles -- TEST INFRASTRUCTURE ONLY.

numpy/scipy restatement of
  * ``detail::build_topology``       voxel.hpp:147-228
  * ``build_periodic_system``        fem.hpp:179-319
  * ``detail::factor_and_solve``     fem.hpp:334-380 (scipy sparse LU stands in
    for Eigen SimplicialLDLT / CHOLMOD; same ridge 1e-11*mean|diag| + 2
    refinement passes, same residual check)
  * ``solve_test_strains``           fem.hpp:385-409
  * ``effective_tensor``             fem.hpp:413-428
and of the reference test oracles (tests/oracles.hpp): ``dense_kkt_solve``
(:77-134), ``laminate_constants`` (:143-161), ``element_energy_quadrature``
(:166-197).  Used to pin the masked-torus solver (oracle and CUDA) to the
reference's direct path, as test_fem.cpp:220-232 does for GridSolver.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

OFF = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]])


def unit_test_strains() -> np.ndarray:
    """fem.hpp:129-142 (engineering shear -> tensor 1/2)."""
    s = np.zeros((6, 3, 3))
    s[0, 0, 0] = s[1, 1, 1] = s[2, 2, 2] = 1.0
    s[3, 1, 2] = s[3, 2, 1] = 0.5
    s[4, 0, 2] = s[4, 2, 0] = 0.5
    s[5, 0, 1] = s[5, 1, 0] = 0.5
    return s


@dataclass
class VoxelMesh:
    r: int
    elements: np.ndarray  # sorted linear ids
    beta: np.ndarray
    element_nodes: np.ndarray  # (E, 8)
    node_coords: np.ndarray  # (N, 3) in [0, r]
    groups: list  # [(master, [(slave, delta(3,)), ...])]
    corner_group: int


def build_topology(r: int, elements: np.ndarray, beta: np.ndarray) -> VoxelMesh:
    """voxel.hpp:147-228 (node ids in first-seen order; groups by sorted key)."""
    elements = np.asarray(elements, np.int64)
    ei = elements % r
    ej = (elements // r) % r
    ek = elements // (r * r)
    c = np.stack([ei, ej, ek], 1)[:, None, :] + OFF[None, :, :]  # (E,8,3)
    flat = c.reshape(-1, 3)
    keys = (flat[:, 2] * (r + 1) + flat[:, 1]) * (r + 1) + flat[:, 0]
    uk, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    node_id = rank[inv]
    coords = flat[first[order]]
    element_nodes = node_id.reshape(-1, 8)
    boundary = ((coords == 0) | (coords == r)).sum(1)
    groups = []
    corner_group = -1
    bmask = boundary > 0
    bn = np.flatnonzero(bmask)
    canon = coords[bn] % r
    ckey = (canon[:, 2] * (r + 1) + canon[:, 1]) * (r + 1) + canon[:, 0]
    srt = np.lexsort((bn, ckey))
    bn, ckey = bn[srt], ckey[srt]
    splits = np.flatnonzero(np.diff(ckey)) + 1
    for members in np.split(bn, splits):
        master = None
        slaves = []
        for n in members:  # bucket order = node order (push_back in node loop)
            delta = (coords[n] == r).astype(np.int64)
            if not delta.any():
                master = int(n)
            else:
                slaves.append((int(n), delta))
        if master is None:
            raise RuntimeError("periodic group without master node")
        axes = int(((coords[master] % r) == 0).sum())
        if len(members) != (1 << axes):
            raise RuntimeError(f"periodic group has {len(members)} members, expected {1 << axes}")
        if axes == 3:
            corner_group = len(groups)
        groups.append((master, slaves))
    return VoxelMesh(r, elements, np.asarray(beta, np.float64), element_nodes, coords, groups,
                     corner_group)


@dataclass
class PeriodicSystem:
    A: sp.csr_matrix
    rhs: np.ndarray  # (n_master_dofs, 6)
    node_dof: np.ndarray
    node_offset: np.ndarray
    n_components: int
    expect_singular: bool


def build_periodic_system(mesh: VoxelMesh, K0: np.ndarray, gauge: int = 0) -> PeriodicSystem:
    """fem.hpp:179-319."""
    if mesh.corner_group < 0:
        raise RuntimeError("mesh has no corner node group")
    nn = len(mesh.node_coords)
    node_dof = np.full(nn, -2, np.int64)
    node_offset = np.zeros((nn, 3))
    master, slaves = mesh.groups[mesh.corner_group]
    members = [(master, np.zeros(3, np.int64))] + slaves
    if gauge < 0 or gauge >= len(members):
        raise ValueError("corner gauge member out of range")
    ref = members[gauge][1]
    for node, delta in members:
        node_dof[node] = -1
        node_offset[node] = delta - ref
    master_of = np.arange(nn)
    for gi, (m, sl) in enumerate(mesh.groups):
        if gi == mesh.corner_group:
            continue
        for node, delta in sl:
            master_of[node] = m
            node_offset[node] = delta
    nxt = 0
    for n in range(nn):
        if node_dof[n] == -1:
            continue
        if master_of[n] == n:
            node_dof[n] = 3 * nxt
            nxt += 1
    free = (node_dof != -1) & (master_of != np.arange(nn))
    node_dof[free] = node_dof[master_of[free]]
    ndof = 3 * nxt
    en = mesh.element_nodes
    E = len(en)
    da = node_dof[en]  # (E,8)
    Kb = K0.reshape(8, 3, 8, 3)
    # triplets for a,b with both dofs free
    ia = (da[:, :, None, None, None] + np.arange(3)[None, None, :, None, None])
    jb = (da[:, None, None, :, None] + np.arange(3)[None, None, None, None, :])
    ia = np.broadcast_to(ia, (E, 8, 3, 8, 3))
    jb = np.broadcast_to(jb, (E, 8, 3, 8, 3))
    val = mesh.beta[:, None, None, None, None] * Kb[None]
    ok = (np.broadcast_to(da[:, :, None, None, None], (E, 8, 3, 8, 3)) >= 0) & \
         (np.broadcast_to(da[:, None, None, :, None], (E, 8, 3, 8, 3)) >= 0)
    A = sp.coo_matrix((val[ok], (ia[ok], jb[ok])), shape=(ndof, ndof)).tocsr()
    # RHS: -K_ab * (eps_s * dy_b) for rows with free dofs
    strains = unit_test_strains()
    t = np.einsum("sab,nb->nsa", strains, node_offset)  # (nn,6,3)
    tb = t[en]  # (E,8,6,3)
    f = -np.einsum("e,aibj,ebsj->eais", mesh.beta, Kb, tb)  # (E,8,3,6)
    rows = da[:, :, None] + np.arange(3)[None, None, :]
    okr = np.broadcast_to(da[:, :, None] >= 0, rows.shape)
    rhs = np.zeros((ndof, 6))
    np.add.at(rhs, rows[okr], f[okr])
    # union-find components (fem.hpp:288-317) via connected components
    r = mesh.r
    canon = mesh.node_coords % r
    ckey = (canon[:, 2] * r + canon[:, 1]) * r + canon[:, 0]
    ek = ckey[en]  # (E,8)
    g = sp.coo_matrix((np.ones(E * 8), (np.repeat(np.arange(E), 8), ek.reshape(-1))),
                      shape=(E, r ** 3)).tocsr()
    adj = (g @ g.T).tocsr()
    ncomp, lab = sp.csgraph.connected_components(adj, directed=False)
    has_corner = np.zeros(ncomp, bool)
    np.logical_or.at(has_corner, lab, (ek == 0).any(1))
    return PeriodicSystem(A, rhs, node_dof, node_offset, int(ncomp), bool((~has_corner).any()))


def solve_test_strains(sys_: PeriodicSystem, residual_tol: float = 1e-9):
    """fem.hpp:334-409. Returns (u (nn,6,3), stats)."""
    A = sys_.A.tocsc()
    B = sys_.rhs
    ridged = sys_.expect_singular

    def factor(M):
        return spla.splu(M.tocsc())

    lu = None
    if not ridged:
        try:
            lu = factor(A)
        except RuntimeError:
            ridged = True
    if ridged:
        mean_diag = np.abs(A.diagonal()).mean()
        lu = factor(A + sp.identity(A.shape[0], format="csc") * (1e-11 * mean_diag))
    U = lu.solve(B)
    if ridged:
        for _ in range(2):
            U = U + lu.solve(B - A @ U)
    worst = 0.0
    for s in range(6):
        bn = max(np.linalg.norm(B[:, s]), 1e-30)
        rn = np.linalg.norm(A @ U[:, s] - B[:, s]) / bn
        worst = max(worst, rn)
        if not rn <= residual_tol:
            raise RuntimeError(f"linear solve residual {rn} exceeds tolerance for strain {s}")
    strains = unit_test_strains()
    t = np.einsum("sab,nb->nsa", strains, sys_.node_offset)
    u = t.copy()
    free = sys_.node_dof >= 0
    idx = sys_.node_dof[free][:, None] + np.arange(3)[None, :]
    u[free] += np.transpose(U[idx], (0, 2, 1))
    return u, dict(regularized=ridged, worst_residual=worst, n_components=sys_.n_components)


def effective_tensor(mesh: VoxelMesh, K0: np.ndarray, u: np.ndarray) -> np.ndarray:
    """fem.hpp:413-428. u: (nn, 6, 3)."""
    Ue = u[mesh.element_nodes]  # (E,8,6,3)
    Ue = np.transpose(Ue, (0, 1, 3, 2)).reshape(len(mesh.element_nodes), 24, 6)
    W = np.einsum("ij,ejs->eis", K0, Ue)
    C = np.einsum("e,eia,eib->ab", mesh.beta, Ue, W)
    return 0.5 * (C + C.T)


def direct_homogenize(r: int, elements, beta, K0, gauge=0, tol=1e-9):
    mesh = build_topology(r, elements, beta)
    sys_ = build_periodic_system(mesh, K0, gauge)
    u, st = solve_test_strains(sys_, tol)
    return effective_tensor(mesh, K0, u), st, mesh, sys_, u


def full_solid(r: int, beta=1.0):
    """voxel.hpp:316-326."""
    el = np.arange(r ** 3)
    return el, np.full(r ** 3, float(beta))


# ---- tests/oracles.hpp ----------------------------------------------------
def dense_kkt_solve(mesh: VoxelMesh, K0: np.ndarray, strain: np.ndarray) -> np.ndarray:
    """oracles.hpp:77-134: full stiffness + Lagrange rows for every periodic pair."""
    nn = len(mesh.node_coords)
    N = 3 * nn
    K = np.zeros((N, N))
    for e in range(len(mesh.element_nodes)):
        d = (3 * mesh.element_nodes[e][:, None] + np.arange(3)[None, :]).reshape(-1)
        K[np.ix_(d, d)] += mesh.beta[e] * K0
    rows, vals = [], []
    for gi, (m, sl) in enumerate(mesh.groups):
        if gi == mesh.corner_group:
            for c in range(3):
                row = np.zeros(N)
                row[3 * m + c] = 1.0
                rows.append(row)
                vals.append(0.0)
            for node, delta in sl:
                t = strain @ delta
                for c in range(3):
                    row = np.zeros(N)
                    row[3 * node + c] = 1.0
                    rows.append(row)
                    vals.append(t[c])
        else:
            for node, delta in sl:
                t = strain @ delta
                for c in range(3):
                    row = np.zeros(N)
                    row[3 * node + c] = 1.0
                    row[3 * m + c] = -1.0
                    rows.append(row)
                    vals.append(t[c])
    G = np.array(rows)
    M = len(rows)
    KKT = np.zeros((N + M, N + M))
    KKT[:N, :N] = K
    KKT[:N, N:] = G.T
    KKT[N:, :N] = G
    rhs = np.zeros(N + M)
    rhs[N:] = vals
    sol = np.linalg.lstsq(KKT, rhs, rcond=None)[0]
    return sol[:N]


def laminate_constants(scale, lam, mu):
    """oracles.hpp:143-161."""
    scale = np.asarray(scale, np.float64)
    la, m = scale * lam, scale * mu
    inv_a = np.mean(1.0 / (la + 2 * m))
    la_over_a = np.mean(la / (la + 2 * m))
    C33 = 1.0 / inv_a
    C13 = la_over_a * C33
    C11 = np.mean(4 * m * (la + m) / (la + 2 * m)) + la_over_a ** 2 * C33
    C12 = np.mean(2 * m * la / (la + 2 * m)) + la_over_a ** 2 * C33
    C44 = 1.0 / np.mean(1.0 / m)
    C66 = np.mean(m)
    return dict(C11=C11, C12=C12, C13=C13, C33=C33, C44=C44, C66=C66)


def element_energy_quadrature(E, nu, edge, u):
    """oracles.hpp:166-197 (3-point Gauss energy of one trilinear voxel)."""
    la = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    gx = [0.5 * (1 - math.sqrt(3 / 5)), 0.5, 0.5 * (1 + math.sqrt(3 / 5))]
    gw = [5 / 18, 8 / 18, 5 / 18]
    energy = 0.0
    for a in range(3):
        for b in range(3):
            for c in range(3):
                x, y, z = gx[a], gx[b], gx[c]
                grad = np.zeros((3, 3))
                for n in range(8):
                    fx = x if OFF[n][0] else 1 - x
                    fy = y if OFF[n][1] else 1 - y
                    fz = z if OFF[n][2] else 1 - z
                    sx = 1.0 if OFF[n][0] else -1.0
                    sy = 1.0 if OFF[n][1] else -1.0
                    sz = 1.0 if OFF[n][2] else -1.0
                    dN = np.array([sx * fy * fz, fx * sy * fz, fx * fy * sz]) / edge
                    grad += np.outer(u[3 * n:3 * n + 3], dN)
                eps = 0.5 * (grad + grad.T)
                tr = np.trace(eps)
                dens = 0.5 * la * tr * tr + mu * np.sum(eps * eps)
                energy += gw[a] * gw[b] * gw[c] * dens * edge ** 3
    return energy


def isotropic(E=1.0, nu=0.3) -> np.ndarray:
    la = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    C = np.zeros((6, 6))
    C[:3, :3] = la
    C[0, 0] = C[1, 1] = C[2, 2] = la + 2 * mu
    C[3, 3] = C[4, 4] = C[5, 5] = mu
    return C
