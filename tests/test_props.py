"""props.make_report and its pieces against the reference's own test cases
(proj/tests/test_props.cpp, the 13 TEST_CASEs restated with their tolerances;
props.hpp:1-182).  Host-only, no GPU."""
import math

import numpy as np
import pytest

from paper_2511_04025_b200 import props as P
from paper_2511_04025_b200.api import ValidationError

MASK = (1 << 64) - 1


class Rng:
    """common.hpp:86-103 (splitmix64, 53-bit uniforms) for the random_spd fixture."""

    def __init__(self, seed):
        self.s = seed or 0x9E3779B97F4A7C15

    def u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self, lo, hi):
        return lo + (hi - lo) * ((self.u64() >> 11) * 2.0 ** -53)


def isotropic(E=1.0, nu=0.3):
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] += 2 * mu
    C[np.arange(3, 6), np.arange(3, 6)] = mu
    return C


def cubic_fixture():
    C = np.zeros((6, 6))
    C[:3, :3] = 1.0
    C[np.arange(3), np.arange(3)] = 2.0
    C[np.arange(3, 6), np.arange(3, 6)] = 1.0
    return C


def random_spd(seed):
    rng = Rng(seed)
    M = np.array([[rng.uniform(-1.0, 1.0) for _ in range(6)] for _ in range(6)])
    return M.T @ M + 0.5 * np.eye(6)


PAIRS = ((0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1))


def rotate_voigt(C, R):
    T = np.zeros((3, 3, 3, 3))
    for a, (i, j) in enumerate(PAIRS):
        for b, (k, l) in enumerate(PAIRS):
            for (p, q) in ((i, j), (j, i)):
                for (u, v) in ((k, l), (l, k)):
                    T[p, q, u, v] = C[a, b]
    Tr = np.einsum("ia,jb,kc,ld,abcd->ijkl", R, R, R, R, T)
    return np.array([[Tr[i, j, k, l] for (k, l) in PAIRS] for (i, j) in PAIRS])


def test_directional_young_isotropic():
    for a in (1, 2, 3):
        assert P.directional_young(isotropic(), a) == pytest.approx(1.0, abs=1e-10)
    with pytest.raises(ValidationError):
        P.directional_young(isotropic(), 0)


def test_directional_young_independent_solve():
    C = random_spd(5)
    for a in (1, 2, 3):
        e = np.zeros(6)
        e[a - 1] = 1.0
        s = np.linalg.lstsq(C, e, rcond=None)[0]
        assert P.directional_young(C, a) == pytest.approx(1.0 / s[a - 1], rel=1e-10)


def test_vrh_isotropic_analytic():
    m = P.voigt_reuss_hill(isotropic())
    K, G = 1.0 / (3.0 * (1.0 - 0.6)), 1.0 / 2.6
    for key, want in (("K_V", K), ("K_R", K), ("G_V", G), ("G_R", G), ("E_eff", 1.0)):
        assert m[key] == pytest.approx(want, rel=1e-12)


def test_vrh_cubic_fixture():
    m = P.voigt_reuss_hill(cubic_fixture())
    assert m["K_V"] == pytest.approx(4.0 / 3.0, rel=1e-14)
    assert m["K_R"] == pytest.approx(4.0 / 3.0, rel=1e-14)
    S11, S12, S44 = 0.75, -0.25, 1.0
    assert m["G_V"] == pytest.approx(0.8, rel=1e-14)
    assert m["G_R"] == pytest.approx(15.0 / (12.0 * S11 - 12.0 * S12 + 9.0 * S44), rel=1e-12)


def test_reuss_never_exceeds_voigt():
    for seed in range(1, 9):
        m = P.voigt_reuss_hill(random_spd(seed))
        assert m["K_R"] <= m["K_V"] + 1e-12 and m["G_R"] <= m["G_V"] + 1e-12
        assert m["K_R"] <= m["K_eff"] <= m["K_V"]


def test_universal_anisotropy():
    assert P.universal_anisotropy(isotropic()) == pytest.approx(0.0, abs=1e-12)
    m = P.voigt_reuss_hill(cubic_fixture())
    want = 5.0 * m["G_V"] / m["G_R"] + m["K_V"] / m["K_R"] - 6.0
    assert P.universal_anisotropy(cubic_fixture()) == pytest.approx(want, rel=1e-12)
    assert P.universal_anisotropy(3.0 * cubic_fixture()) == pytest.approx(want, rel=1e-12)
    assert P.universal_anisotropy(random_spd(3)) >= 0.0


def test_hs_upper_bounds():
    K1, G1 = 1.0 / (3.0 * 0.4), 1.0 / 2.6
    k1, g1 = P.hs_upper_bounds(1.0)
    assert k1 == pytest.approx(K1, rel=1e-14) and g1 == pytest.approx(G1, rel=1e-14)
    k0, g0 = P.hs_upper_bounds(0.0)
    assert k0 == pytest.approx(0.0, abs=1e-14) and g0 == pytest.approx(0.0, abs=1e-14)
    v = 0.1
    K_want = K1 + (1 - v) / (-1 / K1 + 3 * v / (3 * K1 + 4 * G1))
    G_want = G1 + (1 - v) / (-1 / G1 + 6 * v * (K1 + 2 * G1) / (5 * G1 * (3 * K1 + 4 * G1)))
    kv, gv = P.hs_upper_bounds(v)
    assert kv == pytest.approx(K_want, rel=1e-12) and gv == pytest.approx(G_want, rel=1e-12)
    pk = pg = 0.0
    for f in np.arange(0.0, 1.0001, 0.01):
        k, g = P.hs_upper_bounds(min(f, 1.0))
        assert k >= pk - 1e-12 and g >= pg - 1e-12
        pk, pg = k, g
    with pytest.raises(ValidationError):
        P.hs_upper_bounds(1.5)


def test_offdiag_sum():
    assert P.offdiag_sum(isotropic()) == 0.0
    C = isotropic()
    C[0, 3] = C[3, 0] = 0.2
    assert P.offdiag_sum(C) == pytest.approx(0.2, rel=1e-14)


def test_isotropic_distance_zero():
    assert P.isotropic_distance(isotropic()) == pytest.approx(0.0, abs=1e-12)


def test_isotropic_distance_orthogonal_perturbation():
    C = isotropic()
    eps = 1e-3
    C[0, 0] += eps
    C[1, 1] -= eps
    assert P.isotropic_distance(C) == pytest.approx(math.sqrt(2.0) * eps, rel=1e-10)


def test_isotropic_distance_least_squares():
    w = np.outer(*(2 * [np.where(np.arange(6) >= 3, 2.0, 1.0)]))
    for seed in (2, 9):
        C = random_spd(seed)
        m = P.voigt_reuss_hill(C)
        Ks = np.arange(0.2 * m["K_V"], 3.0 * m["K_V"], m["K_V"] * 1e-3)
        Gs = np.arange(0.2 * m["G_V"], 3.0 * m["G_V"], m["G_V"] * 1e-2)
        best = np.inf
        for G in Gs:  # vectorised over K
            la = Ks - 2.0 * G / 3.0
            I = np.zeros((len(Ks), 6, 6))
            I[:, :3, :3] = la[:, None, None]
            I[:, np.arange(3), np.arange(3)] += 2.0 * G
            I[:, np.arange(3, 6), np.arange(3, 6)] = G
            best = min(best, float((w * (C[None] - I) ** 2).sum(axis=(1, 2)).min()))
        d = P.isotropic_distance(C)
        assert math.sqrt(best) * 0.999 <= d <= math.sqrt(best) + 1e-9


def signed_permutations():
    """The 48 operators of symmetry_operators(Tetrahedral) (field.hpp:63-99): all
    signed 3x3 permutation matrices."""
    import itertools
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1.0, -1.0), repeat=3):
            R = np.zeros((3, 3))
            for i in range(3):
                R[i, perm[i]] = signs[i]
            yield R


def test_isotropic_distance_cubic_invariance():
    C = random_spd(12)
    C = 0.5 * (C + C.T)
    ref = P.isotropic_distance(C)
    for R in signed_permutations():
        assert P.isotropic_distance(rotate_voigt(C, R)) == pytest.approx(ref, rel=1e-10)


def test_report_aggregates():
    rep = P.make_report(isotropic(), 1.0)
    assert rep["E_x"] == pytest.approx(1.0, abs=1e-10)
    assert rep["K_eff"] == pytest.approx(1.0 / 1.2, rel=1e-12)
    assert rep["K_HS_upper"] == pytest.approx(1.0 / 1.2, rel=1e-12)
    assert rep["E_voigt"] == pytest.approx(1.0, rel=1e-12)
    assert rep["uai"] == pytest.approx(0.0, abs=1e-10)
    assert P.CSV_HEADER.count(",") == P.csv_row(rep).count(",")
