"""Dev aid: mean per-design time and lockstep iterations at the bench setting
(128^3, cubic_octant n_pre=8, mixed, rtol 1e-5) under the SHL_GMG_* env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S
ctx = S.default_context(0)
r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
seeds = range(1, 1 + (int(sys.argv[2]) if len(sys.argv) > 2 else 6))
opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg")
its, ts, fails = [], [], 0
S.homogenize(S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 99), S.ShellParams(),
             S.BaseMaterial(), r, opt, ctx=ctx)
for seed in seeds:
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    try:
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt, ctx=ctx)
        its.append(int(max(res.iterations))); ts.append(res.timings["t_fwd"])
    except Exception as e:  # noqa: BLE001 - report and continue
        fails += 1
        print(f"seed {seed}: {type(e).__name__}: {e}", flush=True)
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SHL_"))
print(f"[{tag}] fails={fails} mean_ms={np.mean(ts):.2f} iters={its}", flush=True)
