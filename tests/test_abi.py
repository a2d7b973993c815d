"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/shellular_cuda.h declares, the host helpers (reference
arithmetic, no device work) agree with the oracle, and device calls fail
loudly -- never silently on a CPU -- when no device is present."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "shellular_cuda.h")).read()
    return sorted(set(re.findall(r"\b(shl_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(S):
    from paper_2511_04025_b200 import _lib
    L = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.EXPORTS)


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX JIT fallback to other archs)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2511_04025_b200", "libshellular_cuda.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("sym,npre", [("none", 6), ("cubic_octant", 8), ("tetrahedral", 2)])
def test_host_random_design_matches_oracle(S, O, sym, npre):
    for seed in (0, 1, 7, 2024, 2 ** 63 + 5):
        a = S.random_design(S.RandomDesignSpec(sym, npre, 2, -1.0, 1.0), seed)
        b = O.random_design(sym, npre, 2, -1.0, 1.0, seed)
        assert np.array_equal(a.positions, b.positions)
        assert np.array_equal(a.weights, b.weights)
        assert np.array_equal(a.signs, b.signs)


def test_host_expand_symmetry_matches_oracle(S, O):
    for sym, npre in (("cubic_octant", 4), ("tetrahedral", 2), ("none", 4)):
        d = S.random_design(S.RandomDesignSpec(sym, npre), 3)
        e = S.expand_symmetry(d)
        p, s = O.expand_symmetry(O.Design(sym, 2, d.positions, d.signs, d.weights))
        assert np.array_equal(e.positions, p) and np.array_equal(e.signs, s)


def test_validation_errors_without_device(S):
    with pytest.raises(S.ValidationError):
        S.random_design(S.RandomDesignSpec("none", 3), 1)
    bad = S.DesignParams("cubic_octant", 2, np.array([[0.7, 0.2, 0.2], [0.1, 0.1, 0.1]]),
                         np.array([1, -1], np.int32), np.r_[0.0, np.ones(26)])
    with pytest.raises(S.ValidationError, match="fundamental"):
        S.expand_symmetry(bad)
    with pytest.raises(S.ValidationError):
        S.element_stiffness(S.BaseMaterial(poisson=0.5), 1.0)


def test_device_call_fails_loudly_without_gpu(S):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(S.CudaError):
        S.Context(0)
