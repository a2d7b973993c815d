"""Dev aid: two homogenizations of C3 seed 1 (mixed, multigrid) at r (default 128).
With --profiling the solve runs without CUDA graphs (per-launch events), so an
ncu launch list shows every kernel of every iteration (tools/iter_breakdown.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04025_b200 as S  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
r = int(args[0]) if args else 128
ctx = S.Context(0)
ctx.set_profiling("--profiling" in sys.argv)
d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 1)
opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg")
for _ in range(2):
    res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt, ctx=ctx)
print(list(res.iterations), res.timings, "nodes", res.stats.n_nodes, "components", res.stats.n_components, "floating", res.stats.n_floating)
