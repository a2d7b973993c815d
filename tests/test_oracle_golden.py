"""Pin the oracle's C++ restatement to the reference's own code (CPU only).

tests/golden/reference_fixtures.npz was produced by the reference's field.hpp /
voxel.hpp compiled unmodified (tests/golden/make_golden.py via oracle/_ref).
Everything here is bit-exact; when oracle/_ref is present (dev container) the
restatement is additionally compared live against it.
"""
import hashlib
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.npz")
SYMS = {0: "none", 1: "cubic_octant", 2: "tetrahedral"}


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def names(gold):
    return sorted({k.split("/")[0] for k in gold if k.endswith("/positions")})


def design(O, gold, name):
    return O.Design(SYMS[int(gold[f"{name}/symmetry"][0])], 2, gold[f"{name}/positions"],
                    gold[f"{name}/signs"].astype(np.int32), gold[f"{name}/weights"])


RANDOM = {"seeded_3": ("cubic_octant", 4, 3), "seeded_12": ("cubic_octant", 4, 12),
          "seeded_21": ("cubic_octant", 4, 21), "seeded_2024": ("cubic_octant", 4, 2024),
          "c1_seed1": ("cubic_octant", 2, 1), "none64_seed7": ("none", 64, 7),
          "tetra_seed5": ("tetrahedral", 2, 5), "c3_seed1": ("cubic_octant", 8, 1),
          "c3_seed2": ("cubic_octant", 8, 2), "c3_seed3": ("cubic_octant", 8, 3)}


@pytest.mark.parametrize("name", sorted(RANDOM))
def test_random_design_matches_reference(O, gold, name):
    sym, npre, seed = RANDOM[name]
    d = O.random_design(sym, npre, 2, -1.0, 1.0, seed)
    assert np.array_equal(d.positions, gold[f"{name}/positions"])
    assert np.array_equal(d.weights, gold[f"{name}/weights"])
    assert np.array_equal(d.signs, gold[f"{name}/signs"])


def test_expand_symmetry_matches_reference(O, gold):
    for name in names(gold):
        p, s = O.expand_symmetry(design(O, gold, name))
        assert np.array_equal(p, gold[f"{name}/expanded_positions"]), name
        assert np.array_equal(s, gold[f"{name}/expanded_signs"]), name


def test_grids_and_meshes_match_reference(O, gold):
    keys = list(gold["digest/keys"])
    vals = gold["digest/values"]
    checked = 0
    for key, (hc, hk, he, hb) in zip(keys, vals):
        name, rr = key.split("/")
        r = int(rr[1:])
        if r > 32 and name not in ("seeded_2024", "gyroid") and key != "c3_seed1/r128":
            continue  # keep the CPU suite quick: 64^3 by two designs, the bench config 128^3 by one
        g = O.sample_grid(design(O, gold, name), r)
        assert sha(g.samples) == hc, key
        assert sha(g.corners) == hk, key
        assert g.norm == gold[f"{key}/norm"][0], key
        m = O.build_reduced_mesh(g)
        el = m.elements
        be = m.beta.reshape(-1)[el]
        assert sha(el) == he, key
        assert sha(be) == hb, key
        info = gold[f"{key}/info"]
        assert m.n_elements == info[0] and m.full_fallback == bool(info[4]), key
        if f"{key}/centres" in gold:
            assert np.array_equal(g.samples, gold[f"{key}/centres"])
            assert np.array_equal(g.corners, gold[f"{key}/corners"])
        checked += 1
    assert checked >= 15


def test_step_function_matches_reference(O, gold):
    v = gold["step/v"]
    for key in gold:
        if key.startswith("step/") and key != "step/v":
            sharp, fl = map(float, key.split("/")[1].split("_"))
            got = np.array([O.step_function(x, sharp, fl) for x in v])
            assert np.array_equal(got, gold[key]), key


def test_reference_known_answers(O, gold):
    """test_voxel.cpp: seed-2024 fraction band at r=64 L=2; full periodic corner group."""
    info = gold["seeded_2024/r64/info"]
    frac = info[0] / 64 ** 3
    assert 0.03 <= frac <= 0.35
    assert info[5] == 8  # corner group has 1 master + 7 slaves (test_voxel.cpp:246-247)
    assert O.step_function(0.0) == pytest.approx(1.0, abs=1e-15)
    assert O.step_function(10.0) == pytest.approx(1e-3, abs=1e-9)


def test_gyroid_has_exact_zero_corners(O, gold):
    """The bit-exactness stress case: lattice points where F is exactly 0."""
    c = gold["gyroid/r16/corners"]
    assert np.count_nonzero(c == 0.0) > 0


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)),
                                                    "oracle", "_ref", "libshellular_ref.so")),
                    reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("sym,npre", [("none", 6), ("cubic_octant", 4), ("tetrahedral", 2)])
def test_restatement_vs_live_reference(O, sym, npre):
    for seed in range(20):
        a = O.random_design(sym, npre, 2, -1, 1, seed)
        b = O.random_design(sym, npre, 2, -1, 1, seed, use_ref=True)
        assert np.array_equal(a.positions, b.positions)
        ga, gb = O.sample_grid(a, 12), O.sample_grid(a, 12, use_ref=True)
        assert np.array_equal(ga.samples, gb.samples) and np.array_equal(ga.corners, gb.corners)
        try:
            ma = O.build_reduced_mesh(ga)
        except O.OracleError:
            continue
        el, be, _ = O.ref_build_reduced_mesh(gb)
        assert np.array_equal(ma.elements, el)
        assert np.array_equal(ma.beta.reshape(-1)[el], be)
