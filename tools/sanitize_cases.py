"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, one tool per run): the 32^3 and 64^3 single-design, batch-lane,
block-Jacobi, FP64, z-slab and geometry paths.  Exits non-zero on any failure.

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04025_b200 as S  # noqa: E402

spec = S.RandomDesignSpec("cubic_octant", 2, 2, -1.0, 1.0)
sp, mat = S.ShellParams(), S.BaseMaterial()
ctx = S.Context(0)
d1 = S.random_design(spec, 1)
out = []
for prec, pc in (("mixed", "auto"), ("mixed", "jacobi"), ("fp64", "auto"), ("fp32", "auto")):
    res = S.homogenize(d1, sp, mat, 32, S.HomogenizeOptions(residual_tol=1e-5, precision=prec, preconditioner=pc),
                       ctx=ctx)
    out.append((prec, pc, list(res.iterations)))
designs = [S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), s) for s in range(4)]
C, status, st = S.homogenize_batch(designs, sp, mat, 64, S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"),
                                   ctx=ctx, lanes=2)
assert np.all(status == 0)
out.append(("batch64 lanes2", [list(s.iterations) for s in st]))
rs = S.homogenize_slabs(d1, sp, mat, 32, 2, S.HomogenizeOptions(residual_tol=1e-5, precision="mixed"), ctx=ctx)
out.append(("slabs G=2", list(rs.iterations)))
g = S.sample_grid(d1, 32, ctx=ctx)
tri = S.extract_isosurface(g, ctx=ctx)
out.append(("isosurface", len(tri.vertices)))
for o in out:
    print(o)
ctx.close()
print("sanitize cases ok")
