"""Pin the FEM half of the oracle to the reference's known answers (CPU only).

The reference's direct path needs Eigen/CHOLMOD (absent), so the pins are the
reference's own solver-independent tests (test_fem.cpp), restated:
K0 properties, dense KKT, isotropic tensor, laminate closed form, gauge
invariance, E-scaling, and GridSolver == direct -- plus the masked-torus
solver (what the CUDA path implements) == the master-slave direct solve on
seeded reduced meshes with floating components.
"""
import numpy as np
import pytest

from oracle import direct as D


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_element_stiffness_properties(O):
    """test_fem.cpp:33-91."""
    K = O.element_stiffness(1.0, 0.3, 0.25)
    scale = np.abs(K).max()
    t = np.tile([0.3, -1.2, 0.7], 8)
    assert np.abs(K @ t).max() < 1e-12 * scale
    w = np.array([0.2, -0.5, 1.0])
    rot = np.concatenate([np.cross(w, D.OFF[n] * 0.25) for n in range(8)])
    assert np.abs(K @ rot).max() < 1e-12 * scale
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12 * scale) == 6
    assert ev[0] > -1e-12 * scale
    assert np.abs(K - K.T).max() < 1e-12 * scale
    k1 = O.element_stiffness(1.0, 0.25, 1.0)
    kh = O.element_stiffness(1.0, 0.25, 0.5)
    assert np.abs(kh - 0.5 * k1).max() < 1e-12 * np.abs(k1).max()
    rng = np.random.default_rng(4)
    u = rng.uniform(-1, 1, 24)
    K5 = O.element_stiffness(1.0, 0.3, 0.5)
    assert D.element_energy_quadrature(1.0, 0.3, 0.5, u) == pytest.approx(0.5 * u @ K5 @ u, rel=1e-10)


def test_product_stiffness_matches_oracle(S, O):
    """Host helper of the C ABI (no device work): fem.hpp:50-92."""
    for nu, edge in ((0.3, 1 / 32), (0.25, 1.0), (-0.2, 0.1)):
        Kp = S.element_stiffness(S.BaseMaterial(1.0, nu), edge)
        Ko = O.element_stiffness(1.0, nu, edge)
        assert np.abs(Kp - Ko).max() <= 1e-14 * np.abs(Ko).max()


def test_full_solid_dofs_and_isotropic(O):
    """test_fem.cpp:102-109, 131-144, 183-195."""
    r = 4
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    el, be = D.full_solid(r)
    C, st, mesh, sys_, u = D.direct_homogenize(r, el, be, K0)
    assert sys_.A.shape[0] == 3 * (r ** 3 - 1)
    strains = D.unit_test_strains()
    y = mesh.node_coords / r
    for s in range(6):
        assert np.abs(u[:, s, :] - y @ strains[s].T).max() < 1e-10
    assert rel(C, D.isotropic()) < 1e-6
    res = O.grid_solve(be.reshape(r, r, r), K0, tol=1e-12)
    assert rel(res.C, D.isotropic()) < 1e-6


@pytest.mark.parametrize("fixture", ["solid", "rand7", "rand1"])
def test_master_slave_matches_dense_kkt(O, fixture):
    """test_fem.cpp:165-181."""
    r = 4
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    el = np.arange(r ** 3)
    if fixture == "solid":
        be = np.ones(r ** 3)
    else:
        seed, lo = (7, 0.05) if fixture == "rand7" else (1, 0.001)
        be = np.random.default_rng(seed).uniform(lo, 1.0, r ** 3)
    C, st, mesh, sys_, u = D.direct_homogenize(r, el, be, K0)
    strains = D.unit_test_strains()
    for s in range(6):
        ud = D.dense_kkt_solve(mesh, K0, strains[s])
        assert np.abs(u[:, s, :].reshape(-1) - ud).max() <= 1e-8 * max(np.abs(ud).max(), 1e-12)


def test_laminate(O):
    """test_fem.cpp:197-218 through both the direct path and the masked grid solver."""
    r = 8
    layers = [1.0, 0.4, 1e-3, 0.02, 1.0, 0.7, 1e-3, 0.15]
    be = np.repeat(np.array(layers), r * r)
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    lam = D.laminate_constants(layers, 0.3 / (1.3 * 0.4), 1 / 2.6)
    Cd = D.direct_homogenize(r, np.arange(r ** 3), be, K0, tol=1e-12)[0]
    Cg = O.grid_solve(be.reshape(r, r, r), K0, tol=1e-12).C
    for C in (Cd, Cg):
        assert C[0, 0] == pytest.approx(lam["C11"], rel=1e-8)
        assert C[0, 1] == pytest.approx(lam["C12"], rel=1e-8)
        assert C[0, 2] == pytest.approx(lam["C13"], rel=1e-8)
        assert C[2, 2] == pytest.approx(lam["C33"], rel=1e-8)
        assert C[3, 3] == pytest.approx(lam["C44"], rel=1e-8)
        assert C[5, 5] == pytest.approx(lam["C66"], rel=1e-8)


def test_grid_solver_matches_direct(O):
    """test_fem.cpp:220-232."""
    r = 8
    be = np.random.default_rng(31).uniform(0.05, 1.0, r ** 3)
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    Cd = D.direct_homogenize(r, np.arange(r ** 3), be, K0)[0]
    Cg = O.grid_solve(be.reshape(r, r, r), K0, tol=1e-11).C
    assert rel(Cg, Cd) < 1e-8


@pytest.mark.parametrize("seed", [3, 5, 12, 21])
def test_masked_torus_equals_master_slave(O, seed):
    """the masked torus with node 0 pinned reproduces the
    reference's reduced master-slave system (incl. floating components)."""
    r = 12
    g = O.sample_grid(O.seeded_design(seed), r)
    m = O.build_reduced_mesh(g)
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    Cd, st, *_ = D.direct_homogenize(r, m.elements, m.beta.reshape(-1)[m.elements], K0)
    Cg = O.grid_solve(m.beta, K0, tol=1e-11).C
    assert rel(Cg, Cd) < 1e-8


def test_gauge_invariance_and_modulus_scaling(O):
    """test_fem.cpp:234-259."""
    r = 8
    g = O.sample_grid(O.seeded_design(12), r)
    m = O.build_reduced_mesh(g)
    be = m.beta.reshape(-1)[m.elements]
    K0 = O.element_stiffness(1.0, 0.3, 1 / r)
    ref = D.direct_homogenize(r, m.elements, be, K0, gauge=0)[0]
    for gauge in (3, 7):
        assert rel(D.direct_homogenize(r, m.elements, be, K0, gauge=gauge)[0], ref) < 1e-10
    K3 = O.element_stiffness(3.0, 0.3, 1 / r)
    C1 = O.grid_solve(m.beta, K0, tol=1e-12).C
    C3 = O.grid_solve(m.beta, K3, tol=1e-12).C
    assert rel(C3, 3.0 * C1) < 1e-10


def test_oracle_homogenize_composition(O):
    """test_fem.cpp:261-280 (stage keys, full fallback at r=8, degenerate throws)."""
    res = O.homogenize(O.seeded_design(5), 8, tol=1e-9)
    assert res.full_fallback
    assert set(res.timings) == {"t_field", "t_mesh", "t_PBC", "t_AS", "t_RHS", "t_solve", "t_C", "t_fwd"}
    assert res.volume_ratio > 0 and np.abs(res.C).max() > 0
    res16 = O.homogenize(O.seeded_design(5), 16, tol=1e-6)
    assert not res16.full_fallback
    d = O.seeded_design(5)
    d.weights[:] = 0.0
    with pytest.raises(O.OracleError) as e:
        O.homogenize(d, 8)
    assert e.value.code == 2


def test_plane_design_orthotropic(O):
    """test_fem.cpp:282-297."""
    d = O.plane_design_z(0.0)
    res = O.homogenize(d, 16, sharpness=100.0, tol=1e-10)
    c11 = res.C[0, 0]
    assert np.abs(res.C[:3, 3:]).max() < 1e-6 * c11
