"""GPU V-cycle / MG-PCG vs the numpy oracle on the acceptance L-shape start design."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B
from oracle import approx_inverse_oracle as M
from oracle import bisimp_oracle as O

spec = B.catalog()["lshape"].scale(0.4)
grid = B.resolve(spec)
og = O.Grid.from_model(grid)
pm = spec.passive_mask()
a = np.where(pm, 0.1, 0.4) ** 3
b = grid.load.copy()
b[og.fixed] = 0
lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed)
acts = M.activations(lv, a)
mg = B.Multigrid(grid).setup(a)
print("levels", mg.num_levels, len(lv), "nc", mg.coarse_dofs)
for l in range(mg.num_levels):
    nx, ny, fx = mg.level(l)
    print(" level", l, nx, ny, "mask equal", np.array_equal(fx, lv[l].fixed), int(fx.sum()))
for nu in (1, 2):
    x = mg.vcycle(b, 0.6, nu)
    ref = M.vcycle(lv, acts, b, 0.6, nu)
    print("nu", nu, "vcycle rel", np.linalg.norm(x - ref) / np.linalg.norm(ref))
    for steps in (1, 4, 16):
        xg = B.pcg_apply(grid, a, b, steps, multigrid=mg, nu=nu)
        xo = M.pcg(og, a, b, steps, levels=lv, nu=nu)
        r = B.apply_stiffness(grid, a, xg) - b
        r[og.fixed] = 0
        print("  pcg", steps, "rel", np.linalg.norm(xg - xo) / np.linalg.norm(xo), "res", np.abs(r).max())
try:
    u = B.exact_solve(grid, a, 1e-10)
    print("exact ok")
except Exception as e:
    print("exact FAIL", e)
