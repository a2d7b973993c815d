import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04025_b200 as S
d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 1)
res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), 32, S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg"))
print("ok", list(res.iterations), res.stats.gmg_levels)
