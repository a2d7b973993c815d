import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04025_b200 as S
r = int(sys.argv[1]) if len(sys.argv) > 1 else 128
d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 1)
opt = S.HomogenizeOptions(residual_tol=1e-5, precision="mixed", preconditioner="gmg")
for _ in range(2):
    res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
print(list(res.iterations), res.timings)
