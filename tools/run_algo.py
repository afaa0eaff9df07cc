"""Run one problem / algorithm to convergence on the device loop and report it.

    python tools/run_algo.py <problem> <algorithm> [max_iters] [key=value ...]

<problem>: lshape64 | lbracket300 | mbb440 | teaser | cant4096 | mbb<nx>x<ny>
Prints iterations, reason, wall time, ms/iter, final record row and the exact
compliance 1/2 f.u(v) (u by exact_solve to 1e-10).
"""
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import numpy as np  # noqa: E402

import paper_2204_06204_b200 as B  # noqa: E402


def problem(name):
    P = B.problems
    if name == "lshape64":
        return B.catalog()["lshape"].scale(0.4)
    if name == "lbracket300":
        return P.l_bracket(300)
    if name == "mbb440":
        return P.mbb_half_beam(440, 250)
    if name == "teaser":
        return B.catalog()["teaser"]
    if name == "cant4096":
        return P.cantilever_square(4096)
    if name.startswith("mbb"):
        nx, ny = name[3:].split("x")
        return P.mbb_half_beam(int(nx), int(ny))
    raise SystemExit(f"unknown problem {name}")


def main():
    spec = problem(sys.argv[1])
    algo = sys.argv[2]
    max_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
    kw = {}
    for a in sys.argv[4:]:
        k, v = a.split("=")
        kw[k] = float(v) if "." in v or "e" in v else int(v)
    cfg = B.SolverConfig(algorithm=algo, max_iters=max_iters, **kw)
    t0 = time.perf_counter()
    res = B.run(spec, cfg)
    dt = time.perf_counter() - t0
    grid = B.resolve(spec)
    vp = B.apply_filter(res.state.v.values, spec.nx, spec.ny, spec.filter)
    u = B.exact_solve(grid, vp ** spec.eta, 1e-10)
    exact = 0.5 * float(np.asarray(grid.load) @ u)
    print(f"{sys.argv[1]} {algo} {kw}: {res.reason} at {res.state.iter} iterations, {dt:.2f} s "
          f"({dt / max(res.state.iter, 1) * 1e3:.3f} ms/iter incl. setup), last row "
          f"compliance={res.record.compliance[-1]:.4f} res_inf={res.record.residual_inf[-1]:.2e} "
          f"dv_inf={res.record.dv_inf[-1]:.2e}; exact compliance {exact:.4f}")


if __name__ == "__main__":
    main()
