"""C^H golden values for config C4 (design-space sweep at 64^3, CubicOctant 8
pre-expansion charges, K=2, seeds 0..3) from the CPU oracle's masked-PCG
restatement of the reference pipeline (oracle/shellular_oracle.cpp,
pipeline.hpp:61-113 + grid_solver.hpp), solved to rtol 1e-8.  The oracle needs
~3-5 CPU-minutes per 64^3 design, too slow for the test suite, so the values
are committed (tests/golden/c4_chom.npz) and the GPU sweep test compares to
them.  Run: python tests/golden/make_golden_c4.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

SEEDS = (0, 1, 2, 3)


def main():
    Cs, its = [], []
    for s in SEEDS:
        d = O.random_design("cubic_octant", 8, 2, -1.0, 1.0, s)
        res = O.homogenize(d, 64, tol=1e-8)
        Cs.append(res.C)
        its.append(res.iterations)
        print(s, res.iterations, flush=True)
    np.savez_compressed(os.path.join(HERE, "c4_chom.npz"), seeds=np.array(SEEDS), C=np.array(Cs),
                        iterations=np.array(its), tol=np.array([1e-8]))


if __name__ == "__main__":
    main()
