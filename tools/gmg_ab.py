"""Dev aid: iterations, C^H and solve time for a few designs (run twice with an
env toggle such as SHL_GALERKIN_NODEWISE=1 / SHL_APPLY1=1 and diff)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_04025_b200 as S
out = []
for r in (int(a) for a in sys.argv[1].split(",")):
    for seed in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
        d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
        opt = S.HomogenizeOptions(preconditioner="gmg")
        S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
        res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
        out.append({"r": r, "seed": seed, "it": [int(v) for v in res.iterations], "t_AS": res.timings["t_AS"],
                    "t_solve": res.timings["t_solve"], "C": np.asarray(res.tensor).ravel().tolist()})
        print(r, seed, out[-1]["it"], f"AS {res.timings["t_AS"]:.2f} solve {res.timings["t_solve"]:.2f} ms", flush=True)
if len(sys.argv) > 3:
    json.dump(out, open(sys.argv[3], "w"))
