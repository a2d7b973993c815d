"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): field samples and the voxel mask bit-exact in
FP64; beta within 1e-12 relative (device exp vs glibc exp); C^H within 1e-4
relative Frobenius of the oracle, with iteration counts reported; the
reference's known-answer tests (test_fem.cpp) at their own tolerances.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_max(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def rel_fro(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def pair(S, O, kind, seed=1, n_pre=4):
    """(product design, oracle design) built independently from the same seed."""
    if kind == "gyroid":
        od = O.gyroid_design()
        return S.DesignParams("none", 2, od.positions, od.signs, od.weights), od
    if kind == "plane":
        od = O.plane_design_z(0.5 / 32)
        return S.DesignParams("none", 2, od.positions, od.signs, od.weights), od
    sd = S.random_design(S.RandomDesignSpec(kind, n_pre, 2, -1.0, 1.0), seed)
    od = O.random_design(kind, n_pre, 2, -1.0, 1.0, seed)
    assert np.array_equal(sd.positions, od.positions)
    assert np.array_equal(sd.weights, od.weights)
    return sd, od


FIELD_CASES = [("cubic_octant", 3, 4, 16), ("cubic_octant", 12, 4, 16), ("cubic_octant", 1, 2, 32),
               ("none", 7, 64, 32), ("tetrahedral", 5, 2, 16), ("cubic_octant", 2024, 4, 64),
               ("gyroid", 0, 0, 64), ("plane", 0, 0, 32), ("cubic_octant", 11, 8, 8),
               ("none", 3, 4, 5)]


@pytest.mark.parametrize("kind,seed,n_pre,r", FIELD_CASES)
def test_field_bit_exact(S, O, kind, seed, n_pre, r):
    sd, od = pair(S, O, kind, seed, n_pre)
    g = S.sample_grid(sd, r)
    og = O.sample_grid(od, r)
    assert np.array_equal(g.samples, og.samples)
    assert np.array_equal(g.corner_samples, og.corners)
    assert g.norm == og.norm


@pytest.mark.parametrize("kind,seed,n_pre,r", FIELD_CASES)
def test_mask_exact(S, O, kind, seed, n_pre, r):
    sd, od = pair(S, O, kind, seed, n_pre)
    og = O.sample_grid(od, r)
    om = O.build_reduced_mesh(og)
    m = S.build_reduced_mesh(S.sample_grid(sd, r), S.ShellParams())
    assert np.array_equal(m.elements, om.elements)
    ob = om.beta.reshape(-1)[om.elements]
    assert np.abs(m.beta - ob).max() <= 1e-12 * np.abs(ob).max()
    assert m.full_fallback == om.full_fallback


def test_classify_matches_oracle(S, O):
    sd, od = pair(S, O, "gyroid")
    g = S.sample_grid(sd, 64)
    surf = S.classify_surface_elements(g)
    og = O.sample_grid(od, 64)
    m1 = O.build_reduced_mesh(og, expand_layers=1)
    assert len(surf) == O.build_reduced_mesh(og).n_surface
    assert set(surf.tolist()) <= set(m1.elements.tolist())


def test_plane_two_slabs(S):
    """test_voxel.cpp:144-152: off-lattice plane -> exactly 2 r^2 surface voxels."""
    r = 32
    w = np.zeros(27)
    w[1] = 1.0
    p = S.DesignParams("none", 2, np.array([[0.5, 0.5, 0.25 + 0.5 / r], [0.5, 0.5, 0.75 + 0.5 / r]]),
                       np.array([1, -1], np.int32), w)
    surf = S.classify_surface_elements(S.sample_grid(p, r))
    assert len(surf) == 2 * r * r
    assert len(set((surf // (r * r)).tolist())) == 2


def test_schwarz_p_classification(S):
    """test_voxel.cpp:166-187 (host-sampled analytic field through shl_load_grid)."""
    f = lambda x, y, z: np.cos(2 * np.pi * x) + np.cos(2 * np.pi * y) + np.cos(2 * np.pi * z)
    r = 32
    g = S.sample_grid_fn(f, r)
    got = set(S.classify_surface_elements(g).tolist())
    c = g.corner_samples
    want = set()
    for k in range(r):
        for j in range(r):
            for i in range(r):
                blk = c[k:k + 2, j:j + 2, i:i + 2]
                if blk.min() <= 0.0 <= blk.max():
                    want.add((k * r + j) * r + i)
    assert got == want


@pytest.mark.parametrize("seed,r,prec,tol,bar", [(3, 16, "fp64", 1e-11, 1e-8), (12, 16, "fp64", 1e-11, 1e-8),
                                                 (5, 16, "mixed", 1e-6, 1e-5), (21, 16, "fp32", 1e-5, 1e-4)])
def test_grid_solve_vs_oracle(S, O, seed, r, prec, tol, bar):
    od = O.seeded_design(seed)
    om = O.build_reduced_mesh(O.sample_grid(od, r))
    K0 = O.element_stiffness(1.0, 0.3, 1.0 / r)
    ref = O.grid_solve(om.beta, K0, tol=1e-11)
    res = S.GridSolver(om.beta, r, K0, precision=prec, preconditioner="jacobi").solve(tol)
    assert rel_max(res.tensor, ref.C) < bar
    assert np.all(res.iterations > 0)
    if prec == "fp64":
        # same algorithm, same arithmetic class: iteration counts agree closely
        assert np.abs(res.iterations - O.grid_solve(om.beta, K0, tol=tol).iterations).max() <= 2


def test_full_solid_isotropic(S):
    """test_fem.cpp:183-195."""
    r = 4
    K0 = S.element_stiffness(S.BaseMaterial(), 1.0 / r)
    res = S.GridSolver(np.ones(r ** 3), r, K0, precision="fp64").solve(1e-12)
    iso = S.isotropic_tensor(S.BaseMaterial())
    assert rel_max(res.tensor, iso) < 1e-6
    assert iso[0, 0] == pytest.approx(1.34615384615, rel=1e-9)


def test_laminate_constants(S, O):
    """test_fem.cpp:197-218 at the reference tolerance 1e-8."""
    from oracle import direct as D
    r = 8
    layers = [1.0, 0.4, 1e-3, 0.02, 1.0, 0.7, 1e-3, 0.15]
    beta = np.repeat(np.array(layers), r * r)
    mat = S.BaseMaterial()
    K0 = S.element_stiffness(mat, 1.0 / r)
    C = S.GridSolver(beta, r, K0, precision="fp64").solve(1e-12).tensor
    lam = D.laminate_constants(layers, mat.lam(), mat.mu())
    assert C[0, 0] == pytest.approx(lam["C11"], rel=1e-8)
    assert C[1, 1] == pytest.approx(lam["C11"], rel=1e-8)
    assert C[0, 1] == pytest.approx(lam["C12"], rel=1e-8)
    assert C[0, 2] == pytest.approx(lam["C13"], rel=1e-8)
    assert C[2, 2] == pytest.approx(lam["C33"], rel=1e-8)
    assert C[3, 3] == pytest.approx(lam["C44"], rel=1e-8)
    assert C[4, 4] == pytest.approx(lam["C44"], rel=1e-8)
    assert C[5, 5] == pytest.approx(lam["C66"], rel=1e-8)


def test_grid_solver_matches_direct(S, O):
    """test_fem.cpp:220-232: random-beta r=8 against the master-slave direct solve."""
    from oracle import direct as D
    r = 8
    rng = np.random.default_rng(31)
    beta = rng.uniform(0.05, 1.0, r ** 3)
    K0 = O.element_stiffness(1.0, 0.3, 1.0 / r)
    Cd = D.direct_homogenize(r, np.arange(r ** 3), beta, K0)[0]
    Cg = S.GridSolver(beta, r, K0, precision="fp64").solve(1e-11).tensor
    assert rel_max(Cg, Cd) < 1e-8


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_homogenize_c1_vs_oracle(S, O, seed):
    """Config C1: 32^3, CubicOctant 2 pre (16 charges); C^H <= 1e-4 rel Frobenius."""
    r = 32
    sd, od = pair(S, O, "cubic_octant", seed, 2)
    res = S.homogenize(sd, S.ShellParams(), S.BaseMaterial(), r,
                       S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"))
    ref = O.homogenize(od, r, tol=1e-8)
    assert rel_fro(res.tensor, ref.C) < 1e-4
    assert res.stats.n_elements == ref.n_elements
    assert res.stats.n_nodes == ref.n_nodes
    assert res.volume_ratio == pytest.approx(ref.volume_ratio, rel=1e-12)
    assert res.stats.converged


@pytest.mark.parametrize("r,seed,prec,tol,bar", [(20, 3, "mixed", 1e-6, 1e-4), (25, 5, "mixed", 1e-6, 1e-4),
                                                 (36, 7, "mixed", 1e-6, 1e-4), (44, 9, "fp64", 1e-10, 1e-7),
                                                 (18, 11, "fp64", 1e-10, 1e-7)])
def test_homogenize_ragged_sizes_vs_oracle(S, O, r, seed, prec, tol, bar):
    """Grid sizes that are not multiples of the 8x4x4 level-0 brick (ragged last
    bricks on the periodic seam), odd r (AUTO picks block Jacobi: no multigrid)
    and even r whose multigrid hierarchy stops at an odd coarse size (36 -> 18
    -> 9, 44 -> 22 -> 11, 18 -> 9): C^H from the product path against the
    oracle's masked PCG (pipeline.hpp:61-113), same element and node sets."""
    sd, od = pair(S, O, "cubic_octant", seed, 4)
    res = S.homogenize(sd, S.ShellParams(), S.BaseMaterial(), r,
                       S.HomogenizeOptions(residual_tol=tol, precision=prec))
    ref = O.homogenize(od, r, tol=min(tol, 1e-9) * 1e-2)
    assert res.stats.n_elements == ref.n_elements
    assert res.stats.n_nodes == ref.n_nodes
    assert res.stats.converged and np.all(res.iterations > 0)
    if r % 2 == 0 and r // 2 >= 8:
        assert res.stats.gmg_levels >= 1
    else:
        assert res.stats.gmg_levels == 0
    assert rel_fro(res.tensor, ref.C) < bar


def test_homogenize_gyroid_c2(S, O):
    """Config C2: 64^3 gyroid fixture -> cubic C^H, against the oracle."""
    r = 64
    sd, od = pair(S, O, "gyroid")
    res = S.homogenize(sd, S.ShellParams(), S.BaseMaterial(), r,
                       S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"))
    C = res.tensor
    assert abs(C[0, 0] - C[1, 1]) < 1e-4 * C[0, 0] and abs(C[0, 0] - C[2, 2]) < 1e-4 * C[0, 0]
    assert abs(C[3, 3] - C[4, 4]) < 1e-4 * C[0, 0]
    ref = O.homogenize(od, r, tol=1e-7)
    assert rel_fro(C, ref.C) < 1e-4


def test_errors_map_to_reference_classes(S):
    r = 8
    p = S.random_design(S.RandomDesignSpec("cubic_octant", 4), 5)
    zero = S.DesignParams(p.symmetry, p.truncation, p.positions, p.signs, np.zeros(27))
    with pytest.raises(S.DegenerateDesignError, match="field: design is degenerate"):
        S.homogenize(zero, S.ShellParams(), S.BaseMaterial(), r)
    with pytest.raises(S.ValidationError, match="field: grid resolution"):
        S.homogenize(p, S.ShellParams(), S.BaseMaterial(), 3)
    with pytest.raises(S.ValidationError):
        S.homogenize(p, S.ShellParams(floor_ratio=1.5), S.BaseMaterial(), r)
    with pytest.raises(S.ValidationError):
        S.homogenize(p, S.ShellParams(), S.BaseMaterial(poisson=0.5), r)
    bad = S.DesignParams("cubic_octant", 2, np.array([[0.7, 0.2, 0.2], [0.1, 0.1, 0.1]]),
                         np.array([1, -1], np.int32), p.weights)
    with pytest.raises(S.ValidationError, match="fundamental"):
        S.homogenize(bad, S.ShellParams(), S.BaseMaterial(), r)
    f = S.sample_grid_fn(lambda x, y, z: 1.0 + 0 * x, 8)
    with pytest.raises(S.DegenerateDesignError, match="no zero crossing"):
        S.build_reduced_mesh(f)


def test_full_fallback_and_small_r(S, O):
    """test_voxel.cpp:289-297 and pipeline r=8 full-fallback."""
    sd, od = pair(S, O, "cubic_octant", 5, 4)
    m = S.build_reduced_mesh(S.sample_grid(sd, 8), S.ShellParams(expand_layers=8))
    assert m.full_fallback and m.num_elements() == 512
    res = S.homogenize(sd, S.ShellParams(), S.BaseMaterial(), 8,
                       S.HomogenizeOptions(residual_tol=1e-10))
    ref = O.homogenize(od, 8, tol=1e-10)
    assert rel_max(res.tensor, ref.C) < 1e-7
    assert res.stats.full_fallback == ref.full_fallback


def test_batch_matches_single(S):
    designs = [S.random_design(S.RandomDesignSpec("cubic_octant", 2), s) for s in range(4)]
    opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed")
    Cb, status, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), 16, opt)
    assert np.all(status == 0)
    for i, d in enumerate(designs):
        Cs = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 16, opt).tensor
        assert np.array_equal(Cs, Cb[i])  # deterministic reductions


@pytest.mark.parametrize("r,lanes", [(32, 3), (64, 4)])
def test_batch_lanes_match_single(S, r, lanes):
    """Designs in flight on concurrent lanes give bit-identical C^H and iteration
    counts (each design's reductions are fixed-order, whatever runs beside it)."""
    designs = [S.random_design(S.RandomDesignSpec("cubic_octant", 4), s) for s in range(7)]
    opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed")
    ctx = S.Context(0)
    Cb, status, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), r, opt,
                                           ctx=ctx, lanes=lanes)
    assert np.all(status == 0)
    assert len({s.lane for s in stats}) > 1
    for i, d in enumerate(designs):
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt, ctx=ctx)
        assert np.array_equal(res.tensor, Cb[i])
        assert np.array_equal(res.iterations, stats[i].iterations)
    ctx.close()


def test_c4_sweep_subset(S):
    """Config C4 (64^3, CubicOctant 8 pre-expansion charges): seeds 0..15 in one
    batch with 4 designs in flight, every one against the oracle's C^H
    (tests/golden/c4_chom.npz, masked block-Jacobi PCG to rtol 1e-8; the
    fixed 16-seed subset of SURVEY.md §8 d) at the 1e-4 relative Frobenius
    bar, and all 16 finite, symmetric and positive definite."""
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "c4_chom.npz"))
    spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
    designs = [S.random_design(spec, s) for s in range(16)]
    opt = S.HomogenizeOptions(residual_tol=1e-6, precision="mixed")
    C, status, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), 64, opt, lanes=4)
    assert np.all(status == 0)
    for i, s in enumerate(gold["seeds"]):
        err = np.linalg.norm(C[s] - gold["C"][i]) / np.linalg.norm(gold["C"][i])
        assert err < 1e-4, (s, err)
    for c in C:
        assert np.all(np.isfinite(c))
        assert np.allclose(c, c.T, rtol=0, atol=1e-12 * np.abs(c).max())
        assert np.linalg.eigvalsh(c).min() > 0


@pytest.mark.parametrize("r,G,prec,tol", [(16, 2, "fp64", 1e-10), (32, 3, "mixed", 1e-6),
                                          (32, 4, "fp32", 1e-5), (64, 8, "mixed", 1e-5)])
def test_zslab_matches_single_device(S, r, G, prec, tol):
    """Config C5 code path (emulated slabs): same C^H and iteration counts as the
    undecomposed solve; only the cross-slab summation order differs."""
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), 3)
    opt = S.HomogenizeOptions(residual_tol=tol, precision=prec, preconditioner="jacobi")
    ref = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
    got = S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), r, G, opt)
    assert rel_fro(got.tensor, ref.tensor) < (1e-10 if prec == "fp64" else 1e-6)
    assert np.abs(got.iterations - ref.iterations).max() <= 2
    assert got.stats.n_nodes == ref.stats.n_nodes


@pytest.mark.parametrize("r,G,prec,tol", [(32, 2, "fp64", 1e-10), (64, 3, "mixed", 1e-6),
                                          (64, 4, "fp32", 1e-5), (128, 4, "mixed", 1e-5),
                                          (32, 3, "fp64", 1e-10), (32, 16, "fp64", 1e-10),
                                          (16, 2, "fp64", 1e-10)])
def test_zslab_multigrid_matches_single_device(S, r, G, prec, tol):
    """Multigrid z-slab solve (levels 0 and 1 on the slabs with ghost exchanges
    before every sweep, the level-2 restriction summed over slabs, levels >= 2
    replicated; with only one coarse level it stays replicated): same C^H as the
    undecomposed multigrid solve, iteration counts within 1.  G = 3 at r = 32
    puts slab boundaries on odd planes; G = r/2 leaves each slab two fine
    planes and one level-1 plane."""
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), 3)
    opt = S.HomogenizeOptions(residual_tol=tol, precision=prec, preconditioner="gmg")
    ref = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
    got = S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), r, G, opt)
    assert got.stats.gmg_levels == ref.stats.gmg_levels > 1
    assert rel_fro(got.tensor, ref.tensor) < (1e-10 if prec == "fp64" else 1e-6)
    assert np.abs(got.iterations - ref.iterations).max() <= 1


def test_zslab_validation(S):
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), 3)
    with pytest.raises(S.ValidationError):
        S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), 16, 9)


@pytest.mark.parametrize("r,prec,seed", [(32, "mixed", 1), (64, "mixed", 2), (64, "fp64", 3),
                                         (128, "mixed", 1), (32, "fp32", 4)])
def test_gmg_matches_block_jacobi(S, r, prec, seed):
    """Multigrid-preconditioned CG reaches the same C^H as the reference's
    block-Jacobi PCG, in an r-independent handful of iterations."""
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), seed)
    tol = 1e-5
    ja = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                      S.HomogenizeOptions(residual_tol=tol, precision=prec, preconditioner="jacobi"))
    mg = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                      S.HomogenizeOptions(residual_tol=tol, precision=prec, preconditioner="gmg"))
    assert mg.stats.gmg_levels >= 2
    assert rel_fro(mg.tensor, ja.tensor) < 1e-6
    assert max(mg.iterations) < 60 < max(ja.iterations)


def test_gmg_vs_oracle_and_direct(S, O):
    """GMG on a seeded r=16 reduced mesh against the oracle's masked PCG (which is
    pinned to the reference's master-slave direct solve)."""
    r = 16
    od = O.seeded_design(12)
    om = O.build_reduced_mesh(O.sample_grid(od, r))
    K0 = O.element_stiffness(1.0, 0.3, 1.0 / r)
    ref = O.grid_solve(om.beta, K0, tol=1e-11)
    res = S.GridSolver(om.beta, r, K0, precision="fp64", preconditioner="gmg").solve(1e-11)
    assert res.stats.gmg_levels == 2
    assert rel_max(res.tensor, ref.C) < 1e-8


@pytest.mark.parametrize("seed", [4, 44])
def test_fp32_ridge_keeps_ch(S, seed):
    """Designs whose floating components stalled the FP32 multigrid iteration at
    the FP64 ridge: the FP32-mode ridge (1e-8 mean|diag|) converges without
    falling back, and C^H matches the FP64 solve far inside the 1e-4 bar."""
    r = 128 if seed == 4 else 64
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), seed)
    mixed = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                         S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg"))
    fp64 = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                        S.HomogenizeOptions(residual_tol=1e-8, precision="fp64", preconditioner="gmg"))
    assert max(mixed.iterations) < 60
    assert rel_fro(mixed.tensor, fp64.tensor) < 1e-6


@pytest.mark.gpu
def test_mixed_gmg_hinge_breakdown_retried_in_fp64_operator(S):
    """Seed 10 at 128^3: the FP32 operator loses p^T A p on the hinge modes of
    the voxel shell; the mixed solve is redone with FP64 Krylov vectors and an
    FP64-accumulated operator (precond_fallback 2), never with block Jacobi,
    and matches the FP64 C^H."""
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8), 10)
    mixed = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 128,
                         S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"))
    fp64 = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 128,
                        S.HomogenizeOptions(residual_tol=1e-8, precision="fp64", preconditioner="gmg"))
    assert mixed.stats.precond_fallback in (0, 2)
    assert mixed.stats.gmg_levels >= 2
    assert max(mixed.iterations) < 60
    assert rel_fro(mixed.tensor, fp64.tensor) < 1e-6


# ---- the bench configuration (BASELINE.json configs[2], C3: 128^3) and C5 (256^3) ----
def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ref_gold():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.npz"))


@pytest.mark.parametrize("key", ["c3_seed1/r128", "c3_seed2/r128", "c3_seed3/r128", "c3_seed1/r256"])
def test_bench_config_field_and_mask_vs_reference(S, ref_gold, key):
    """C3 at 128^3 (the bench workload, first bench seeds) and C5 at 256^3: the
    device field (centres, corners, norm) and element set are bit-identical to
    the reference's OWN sample_grid / build_reduced_mesh (field.hpp:488-534,
    voxel.hpp:235-313, digests written from oracle/_ref by
    tests/golden/make_golden.py); beta within 1e-12 relative on a fixed sample
    of elements and in its sum (device exp vs glibc exp)."""
    name, rr = key.split("/")
    r, seed = int(rr[1:]), int(name[len("c3_seed"):])
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    assert np.array_equal(d.positions, ref_gold[f"{name}/positions"])
    keys = list(ref_gold["digest/keys"])
    hc, hk, he, _ = ref_gold["digest/values"][keys.index(key)]
    g = S.sample_grid(d, r)
    assert _sha(g.samples) == hc, "centres differ from the reference"
    assert _sha(g.corner_samples) == hk, "corners differ from the reference"
    assert g.norm == ref_gold[f"{key}/norm"][0]
    m = S.build_reduced_mesh(g, S.ShellParams())
    assert _sha(np.asarray(m.elements, np.uint32)) == he, "element set differs from the reference"
    info = ref_gold[f"{key}/info"]
    assert len(m.elements) == info[0] and bool(m.full_fallback) == bool(info[4])
    idx = ref_gold[f"{key}/beta_sample_idx"]
    ref = ref_gold[f"{key}/beta_sample"]
    assert np.abs(m.beta[idx] - ref).max() <= 1e-12 * np.abs(ref).max()
    bs = ref_gold[f"{key}/beta_sum"][0]
    assert abs(m.beta.sum() - bs) <= 1e-12 * bs


@pytest.mark.parametrize("lanes", [1, 2])
def test_bench_config_chom_vs_oracle(S, lanes):
    """C^H at the bench configuration with the bench's exact options (C3 128^3,
    rtol 1e-5, mixed precision, automatic preconditioner = multigrid,
    shl_homogenize_batch with `lanes` designs in flight) against the oracle's
    masked block-Jacobi PCG of the reference pipeline (grid_solver.hpp:37-96,
    rtol 1e-7; tests/golden/c3_chom.npz): the 1e-4 relative Frobenius bar of
    BASELINE.json north_star, with the lockstep iteration counts reported."""
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3_chom.npz"))
    seeds = [int(s) for s in gold["seeds"]]
    spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
    designs = [S.random_design(spec, s) for s in seeds]
    opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="auto")
    C, status, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), 128, opt, lanes=lanes)
    assert np.all(status == 0)
    for i, s in enumerate(seeds):
        err = rel_fro(C[i], gold["C"][i])
        print(f"C3 seed {s}: rel Frobenius {err:.2e}, GPU multigrid iterations {list(stats[i].iterations)}, "
              f"oracle block-Jacobi iterations {list(gold['iterations'][i])}, nodes {stats[i].n_nodes}")
        assert stats[i].n_nodes == gold["n_nodes"][i]
        assert stats[i].gmg_levels > 0
        assert err < 1e-4, (s, err)


@pytest.mark.parametrize("seed,r", [(3, 16), (12, 16), (21, 16), (1, 32), (5, 32)])
def test_floating_components_vs_reference_criterion(S, O, seed, r):
    """shl_stats.n_components / n_floating: the union-find connectivity scan of
    build_periodic_system (fem.hpp:288-317: elements sharing a torus node are
    coupled; a component with no element at torus node 0 floats), on the
    device, against the oracle's restatement (oracle/direct.py)."""
    from oracle import direct as D
    sd, od = pair(S, O, "cubic_octant", seed, 4)
    res = S.homogenize(sd, S.ShellParams(), S.BaseMaterial(), r,
                       S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"))
    om = O.build_reduced_mesh(O.sample_grid(od, r))
    mesh = D.build_topology(r, om.elements, om.beta.reshape(-1)[om.elements])
    sys_ = D.build_periodic_system(mesh, O.element_stiffness(1.0, 0.3, 1.0 / r))
    assert res.stats.n_components == sys_.n_components
    assert (res.stats.n_floating > 0) == sys_.expect_singular


def test_repeat_runs_bitwise_identical(S):
    """Race check without a sanitizer (compute-sanitizer is closed on this GPU
    pool): the same 64^3 design solved repeatedly, alone and interleaved with
    other designs on 1 and 3 batch lanes, gives bitwise identical C^H and
    iteration counts -- every reduction (per-brick partials, last-CTA sums,
    tile queues, union-find component count) is order-deterministic, so any
    data race on them would show up as a changed bit."""
    spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
    sp, mat = S.ShellParams(), S.BaseMaterial()
    opt = S.HomogenizeOptions(residual_tol=1e-6, precision="mixed")
    d = S.random_design(spec, 7)
    ctx = S.Context(0)
    ref = S.homogenize(d, sp, mat, 64, opt, ctx=ctx)
    for _ in range(3):
        res = S.homogenize(d, sp, mat, 64, opt, ctx=ctx)
        assert np.array_equal(res.tensor, ref.tensor)
        assert np.array_equal(res.iterations, ref.iterations)
        assert res.stats.n_components == ref.stats.n_components
    others = [S.random_design(spec, s) for s in (8, 9, 10, 11, 12)]
    for lanes in (1, 3):
        C, status, st = S.homogenize_batch(others[:3] + [d] + others[3:], sp, mat, 64, opt, ctx=ctx, lanes=lanes)
        assert np.all(status == 0)
        assert np.array_equal(C[3], ref.tensor)
        assert np.array_equal(st[3].iterations, ref.iterations)
    ctx.close()
