"""Dev aid: one-GPU numbers for the non-headline BASELINE configs.

C5: single design at 256^3 (C3 design spec, L = 8), multigrid mixed PCG, and
the same design through 4 emulated z-slabs (C^H agreement).  C4: design-space
sweep throughput at 64^3 through homogenize_batch with 1/2/4 lanes.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04025_b200 as S  # noqa: E402

spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed")
ctx = S.Context(0)
d = S.random_design(spec, 1)
S.homogenize(S.random_design(spec, 2), S.ShellParams(), S.BaseMaterial(), 256, opt, ctx=ctx)  # warm
for rep in range(2):
    t = time.perf_counter()
    res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 256, opt, ctx=ctx)
    wall = time.perf_counter() - t
    print(f"C5 256^3 seed 1: wall {wall*1e3:.1f} ms, stages {dict((k, round(v, 2)) for k, v in res.timings.items())}, "
          f"iterations {list(res.iterations)}, nodes {res.stats.n_nodes}, gmg levels {res.stats.gmg_levels}", flush=True)
for pre in ("gmg", "jacobi"):
    o = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner=pre)
    ref = res if pre == "gmg" else S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 256, o, ctx=ctx)
    S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), 256, 4, o, ctx=ctx)  # warm (allocations, module loads)
    sl = S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), 256, 4, o, ctx=ctx)
    print(f"C5 4 emulated slabs ({pre}): rel diff vs undecomposed "
          f"{np.linalg.norm(sl.tensor - ref.tensor) / np.linalg.norm(ref.tensor):.2e}, "
          f"iterations {list(sl.iterations)} vs {list(ref.iterations)}, t_fwd {sl.timings['t_fwd']:.0f} ms "
          f"(undecomposed {ref.timings['t_fwd']:.0f} ms)", flush=True)
designs = [S.random_design(spec, s) for s in range(64)]
S.homogenize_batch(designs[:8], S.ShellParams(), S.BaseMaterial(), 64, opt, ctx=ctx, lanes=4)
for lanes in (1, 2, 4):
    t = time.perf_counter()
    C, st, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), 64, opt, ctx=ctx, lanes=lanes)
    wall = time.perf_counter() - t
    print(f"C4 64^3 sweep, 64 designs, lanes {lanes}: {len(designs)/wall:.1f} designs/s "
          f"(mean t_fwd {np.mean([s.timings['t_fwd'] for s in stats]):.2f} ms, failures {int((st != 0).sum())})", flush=True)
