"""Dev aid: diagnose GMG breakdown on given seeds (precision / smoother knobs via env)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04025_b200 as S
r = int(sys.argv[1]); seeds = [int(x) for x in sys.argv[2].split(",")]
for seed in seeds:
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    for pc, prec in (("jacobi", "mixed"), ("gmg", "mixed"), ("gmg", "fp64"), ("gmg", "fp32")):
        try:
            res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                               S.HomogenizeOptions(residual_tol=1e-5, precision=prec, preconditioner=pc))
            print(seed, pc, prec, "ok", list(map(int, res.iterations)), f"vol={res.volume_ratio:.4f} nodes={res.stats.n_nodes}")
        except S.Error as e:
            print(seed, pc, prec, "FAIL", e)
