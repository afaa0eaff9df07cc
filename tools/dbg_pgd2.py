"""Capture the failing exact_solve inputs of pgd_exact on the L-shape and replay them."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S
from oracle import approx_inverse_oracle as M
from oracle import bisimp_oracle as O

orig = S.exact_solve
cap = {}


def wrapped(grid, a, tol, x0=None, **kw):
    try:
        return orig(grid, a, tol, x0=x0, **kw)
    except Exception:
        cap.update(grid=grid, a=a.cpu().numpy().copy(), x0=None if x0 is None else x0.cpu().numpy().copy())
        raise


S.exact_solve = wrapped
spec = B.catalog()["lshape"].scale(0.4)
try:
    B.run(spec, B.SolverConfig(algorithm="pgd_exact", max_iters=50000))
except Exception as e:
    print("failed:", e)
grid, a, x0 = cap["grid"], cap["a"], cap["x0"]
np.savez("gpurun_out/exact_fail.npz", a=a, x0=x0)
og = O.Grid.from_model(grid)
b = grid.load.copy()
b[og.fixed] = 0
lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed)
acts = M.activations(lv, a)
mg = B.Multigrid(grid).setup(a)
for nu in (1, 2):
    xg = mg.vcycle(b, 0.6, nu)
    xo = M.vcycle(lv, acts, b, 0.6, nu)
    print("vcycle nu", nu, "rel", np.linalg.norm(xg - xo) / np.linalg.norm(xo), "b.Vb gpu", b @ xg, "oracle", b @ xo)
r0 = b - B.apply_stiffness(grid, a, x0)
r0[og.fixed] = 0
for nu in (1,):
    zg = mg.vcycle(r0, 0.6, nu)
    zo = M.vcycle(lv, acts, r0, 0.6, nu)
    print("r0: |r0|inf", np.abs(r0).max(), "rel", np.linalg.norm(zg - zo) / np.linalg.norm(zo), "r.z gpu", r0 @ zg, "oracle", r0 @ zo)
    for steps in (1, 8, 32):
        xg = B.pcg_apply(grid, a, r0, steps, multigrid=mg, nu=nu)
        xo = M.pcg(og, a, r0, steps, levels=lv, nu=nu)
        print("  pcg", steps, "rel", np.linalg.norm(xg - xo) / max(np.linalg.norm(xo), 1e-300))
try:
    B.exact_solve(grid, a, 1e-10, x0=x0)
    print("replay ok")
except Exception as e:
    print("replay FAIL", e)
try:
    B.exact_solve(grid, a, 1e-10)
    print("replay from 0 ok")
except Exception as e:
    print("replay from 0 FAIL", e)
