"""Quick device timing probe (development aid): one design at r through the C ABI."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S

r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
prec = sys.argv[2] if len(sys.argv) > 2 else "mixed"
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-5
prof = int(sys.argv[4]) if len(sys.argv) > 4 else 0
pc = os.environ.get("PRECOND", "jacobi")
ctx = S.default_context(0)
ctx.set_profiling(bool(prof))
spec = S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0)
seeds = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [1, 1, 2]
for seed in seeds:
    d = S.random_design(spec, seed)
    t = time.perf_counter()
    res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, S.HomogenizeOptions(residual_tol=tol, precision=prec, preconditioner=pc), ctx=ctx)
    wall = (time.perf_counter() - t) * 1e3
    st = res.stats
    it = int(max(res.iterations))
    print(f"r={r} seed={seed} prec={st.precision} wall={wall:.1f}ms timings=" +
          " ".join(f"{k}={v:.2f}" for k, v in res.timings.items()) +
          f" iters={list(res.iterations)} elems={st.n_elements} nodes={st.n_nodes} tiles={st.n_tiles}"
          f" lv={st.gmg_levels} per_iter={st.timings['t_solve']/max(it,1)*1e3:.1f}us apply_ms={st.apply_ms:.2f} update_ms={st.update_ms:.2f} launches={st.kernel_launches}")
    if prof and st.apply_launches:
        print(f"   apply avg {st.apply_ms/st.apply_launches*1e3:.1f}us update avg {st.update_ms/st.apply_launches*1e3:.1f}us")
print("C=", np.array2string(res.tensor, precision=5))
