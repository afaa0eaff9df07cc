"""Replicates pgd_exact's first exact_solve on the acceptance L-shape."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S
from oracle import approx_inverse_oracle as M
from oracle import bisimp_oracle as O

spec = B.catalog()["lshape"].scale(0.4)
cfg = B.SolverConfig(algorithm="pgd_exact", max_iters=10)
ws = S._prepare(spec, cfg)
grid = ws.grid
vp, a = S.apply_filter_and_activation(ws.v_init, grid.nx, grid.ny, ws.filter_spec, ws.eta)
a_h = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
print("a range", a_h.min(), a_h.max())
og = O.Grid.from_model(grid)
b = grid.load.copy()
b[og.fixed] = 0
lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed)
x, hist = M.pcg(og, a_h, b, 64, levels=lv, nu=1, history=True)
print("oracle pcg nu=1", [f"{h:.1e}" for h in np.asarray(hist)[::8]])
mg = B.Multigrid(grid).setup(a_h)
for steps in (4, 16, 64):
    xg = B.pcg_apply(grid, a_h, b, steps, multigrid=mg, nu=1)
    xo = M.pcg(og, a_h, b, steps, levels=lv, nu=1)
    print("pcg", steps, "rel", np.linalg.norm(xg - xo) / np.linalg.norm(xo))
for x0 in (None, np.zeros(grid.num_dofs)):
    try:
        u = B.exact_solve(grid, a, 1e-10, x0=x0)
        print("exact ok (tensor a)")
    except Exception as e:
        print("exact FAIL (tensor a)", e)
    try:
        u = B.exact_solve(grid, a_h, 1e-10, x0=x0)
        print("exact ok (numpy a)")
    except Exception as e:
        print("exact FAIL (numpy a)", e)
