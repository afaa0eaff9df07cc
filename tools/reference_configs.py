"""The unmodified reference (baseline/_ref) on every BASELINE.json config, in
bounded samples, on the host cores (SURVEY §8(d) "CPU baseline beside it").

    python tools/reference_configs.py [--json OUT]

Each entry: bisimp.solvers.run(spec, SolverConfig(algorithm, max_iters=W+K),
threads=1, clock=time.perf_counter) with BLAS on one thread; the median of
diff(elapsed_s) over the last K iterations.  The reference has no multigrid
or PCG low-level step, so C3 / C4 time its pfbto_jacobi (and cpfbto_krylov at
C3) -- the nearest reference algorithms on the same grids.  C4 / C5 pass
beta (0.2) so the set-up does not spend ~100 matvecs on its power
iteration; an iteration's cost does not depend on beta.  C5 (134M cells,
~45 GB, ~1 min per iteration) runs on its 16384x1024 band (1/8) and is
scaled by 8: the reference's cost is linear in the cells.
"""
import json
import os
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def cases(ref):
    P = ref.problems
    mbb = dict(volume_fraction=0.5,
               fixtures=({"edge": "left", "dofs": "x"}, {"point": (1.0, 1.0), "dofs": "y"}),
               loads=({"edge": "top", "span": (0.0, 0.02), "fy": -1.0},))
    lsh = P.catalog()["lshape"]
    c3 = P.ProblemSpec(nx=300, ny=300, volume_fraction=0.5, fixtures=lsh.fixtures,
                       loads=lsh.loads, passive=lsh.passive)
    c4 = P.ProblemSpec(nx=4096, ny=4096, volume_fraction=0.4,
                       fixtures=({"edge": "left", "dofs": "xy"},),
                       loads=({"edge": "right", "span": (0.47, 0.53), "fy": -1.0},))
    return [
        ("C1", P.catalog()["teaser"], "cpfbto_krylov", {}, 2, 5, 1.0),
        ("C2", P.ProblemSpec(nx=440, ny=250, **mbb), "pfbto_jacobi", {}, 5, 20, 1.0),
        ("C3", c3, "pfbto_jacobi", {}, 3, 10, 1.0),
        ("C3_cpfbto", c3, "cpfbto_krylov", {}, 1, 4, 1.0),
        ("C4", c4, "pfbto_jacobi", {"beta": 0.2}, 1, 2, 1.0),
        ("C5_band_x8", P.ProblemSpec(nx=16384, ny=1024, **mbb), "pfbto_jacobi", {"beta": 0.2}, 1,
         2, 8.0),
    ]


def main(out=None, log=sys.stderr):
    if not os.path.isdir(os.path.join(REF, "bisimp")):
        print(json.dumps({"unavailable": "baseline/_ref is not installed"}), file=log)
        return None
    sys.path.insert(0, REF)
    warnings.filterwarnings("ignore")
    import bisimp.problems
    import bisimp.solvers
    import bisimp as ref
    from threadpoolctl import threadpool_limits
    res = {}
    for key, spec, algo, kw, W, K, scale in cases(ref):
        cfg = ref.solvers.SolverConfig(algorithm=algo, max_iters=W + K, **kw)
        t0 = time.perf_counter()
        with threadpool_limits(limits=1):
            r = ref.solvers.run(spec, cfg, threads=1, clock=time.perf_counter)
        d = np.diff(np.asarray(r.record.elapsed_s))[W - 1:] * 1e3
        res[key] = {"algorithm": algo, "cells": spec.nx * spec.ny,
                    "ms_per_iter": float(np.median(d)) * scale, "iters_timed": K,
                    "scaled_by": scale, "wall_s": time.perf_counter() - t0, "cores": 1}
        print(key, json.dumps(res[key]), file=log, flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    main(sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None, log=sys.stdout)
