"""V-cycle with and without the one-CTA coarse tail: max relative difference."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B
import paper_2204_06204_b200.problems as P
from oracle import bisimp_oracle as O

for name, spec in {"mbb": P.mbb_half_beam(60, 34), "tiny": P.mbb_half_beam(6, 4),
                   "lb": P.l_bracket(48)}.items():
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(5)
    a = rng.uniform(1e-3, 1.0, og.n_elem)
    b = rng.standard_normal(og.n_dofs)
    b[og.fixed] = 0.0
    mg = B.Multigrid(grid).setup(a)
    for nu in (1, 2):
        out = {}
        for lim in ("0", "300", str(10 ** 9)):
            os.environ["BSP_MG_TAIL"] = lim
            out[lim] = mg.vcycle(b, omega=0.6, nu=nu)
        for lim in ("300", str(10 ** 9)):
            d = np.abs(out[lim] - out["0"])
            print(name, mg.num_levels, nu, lim, "max|d|", d.max(), "rel", d.max() / np.abs(out["0"]).max(),
                  "n_diff", int((d > 0).sum()), "of", d.size, flush=True)
