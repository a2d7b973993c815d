"""Dev aid: robustness/iterations of GMG settings over many designs (env-configured)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S
ctx = S.default_context(0)
cases = [(32, "cubic_octant", 2, s) for s in (1, 2, 3)] + [(64, "cubic_octant", 8, s) for s in range(1, 7)] + \
        [(64, "none", 64, 1), (64, "tetrahedral", 8, 1), (128, "cubic_octant", 8, 1), (128, "cubic_octant", 8, 3)]
its, ts, fails = [], [], 0
for r, sym, npre, seed in cases:
    d = S.random_design(S.RandomDesignSpec(sym, npre, 2, -1.0, 1.0), seed)
    try:
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r,
                           S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg"), ctx=ctx)
        its.append(int(max(res.iterations))); ts.append(res.timings["t_fwd"])
    except S.SolverError:
        fails += 1; its.append(-1); ts.append(0)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SHL_GMG"))
print(f"[{tag}] fails={fails} iters={its} t_fwd_ms={[round(t,1) for t in ts]}", flush=True)
