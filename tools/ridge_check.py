"""Dev aid: C^H of mixed/GMG under SHL_RIDGE_REL against the FP64 Jacobi solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S
r = int(sys.argv[1]); seeds = [int(x) for x in sys.argv[2].split(",")]
for seed in seeds:
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    ref = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                       S.HomogenizeOptions(residual_tol=1e-9, precision="fp64", preconditioner="gmg"))
    for prec in ("mixed", "fp32"):
        try:
            res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                               S.HomogenizeOptions(residual_tol=1e-5, precision=prec, preconditioner="gmg"))
            err = np.linalg.norm(np.asarray(res.tensor) - np.asarray(ref.tensor)) / np.linalg.norm(np.asarray(ref.tensor))
            print(f"seed {seed} {prec} ridge={os.environ.get('SHL_RIDGE_REL')} ok "
                  f"it={list(map(int, res.iterations))} relF={err:.2e}", flush=True)
        except S.Error as e:
            print(f"seed {seed} {prec} ridge={os.environ.get('SHL_RIDGE_REL')} FAIL {e}", flush=True)
