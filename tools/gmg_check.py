"""Dev aid: GMG vs block-Jacobi PCG on the same designs (C^H agreement, iterations, time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S

r = int(sys.argv[1]) if len(sys.argv) > 1 else 64
seeds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2]
prec = sys.argv[3] if len(sys.argv) > 3 else "mixed"
ctx = S.default_context(0)
spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
for seed in seeds:
    d = S.random_design(spec, seed)
    out = {}
    for pc in ("jacobi", "gmg"):
        opt = S.HomogenizeOptions(residual_tol=1e-5, precision=prec, preconditioner=pc)
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt, ctx=ctx)
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt, ctx=ctx)
        out[pc] = res
        t = res.timings
        print(f"r={r} seed={seed} {pc:6s} lv={res.stats.gmg_levels} iters={list(map(int,res.iterations))} "
              f"t_AS={t['t_AS']:.2f} t_solve={t['t_solve']:.2f} t_fwd={t['t_fwd']:.2f} ms "
              f"per_iter={t['t_solve']/max(1,max(res.iterations))*1e3:.0f}us", flush=True)
    a, b = out["jacobi"].tensor, out["gmg"].tensor
    print(f"   rel fro diff gmg vs jacobi: {np.linalg.norm(a-b)/np.linalg.norm(a):.2e}")
