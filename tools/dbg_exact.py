"""exact_solve (restarted MG-PCG) on the acceptance L-shape, with and without the MG tail."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B

spec = B.catalog()["lshape"].scale(0.4)
grid = B.resolve(spec)
print("grid", grid.nx, grid.ny)
for lim in ("0", "2048", "100000"):
    os.environ["BSP_MG_TAIL"] = lim
    for vf in (0.5, 1.0):
        a = np.full(grid.nx * grid.ny, vf ** 3)
        try:
            u = B.exact_solve(grid, a, 1e-10)
            r = B.apply_stiffness(grid, a, u) - grid.load
            r[grid.fixed_dofs] = 0
            print(lim, vf, "ok", np.abs(r).max(), flush=True)
        except Exception as e:
            print(lim, vf, "FAIL", e, flush=True)
    mg = B.Multigrid(grid)
    print("levels", mg.num_levels, [mg.level(l)[:2] for l in range(mg.num_levels)], mg.coarse_dofs)
