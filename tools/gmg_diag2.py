import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04025_b200 as S
r = int(sys.argv[1]); seeds = [int(x) for x in sys.argv[2].split(",")]; prec = sys.argv[3] if len(sys.argv) > 3 else "mixed"
for seed in seeds:
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    try:
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                           S.HomogenizeOptions(residual_tol=1e-5, precision=prec, preconditioner="gmg"))
        print(seed, prec, "ok", list(map(int, res.iterations)), flush=True)
    except S.Error as e:
        print(seed, prec, "FAIL", e, flush=True)
