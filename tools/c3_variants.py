"""C3 (L-bracket 300x300, passive void) endpoints of the low-level solver
variants, each run to the reference termination test, graded by the exact
compliance of the final design (device exact_solve to 1e-10).

    python tools/c3_variants.py [n] > gpurun_out/c3_variants.log
"""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
warnings.filterwarnings("ignore", message="decay exponent")

import paper_2204_06204_b200 as B  # noqa: E402

VARIANTS = [
    ("cpfbto_krylov", {}),
    ("mg_pcg", {}),
    ("mg_pcg", {"beta": 0.5}),
    ("mg_pcg", {"beta": 0.3}),
    ("mg_pcg", {"inner_steps": 1}),
    ("mg_pcg", {"inner_steps": 2, "beta": 0.5}),
    ("mg_vcycle", {}),
    ("mg_vcycle", {"mg_smooth": 1}),
    ("mg_vcycle", {"mg_smooth": 3}),
    ("pcg_jacobi", {"beta": 0.5}),
    ("pgd_exact", {}),
]


# exact compliance of the converged pgd_exact designs measured on B200 (r02)
KNOWN_PGD = {64: 777.803, 300: 2919.129}


def main(n, only=None):
    spec = B.problems.l_bracket(n) if n != 64 else B.catalog()["lshape"].scale(0.4)
    grid = B.resolve(spec)

    def exact_compliance(v):
        vp = B.apply_filter(v, spec.nx, spec.ny, spec.filter)
        u = B.exact_solve(grid, vp ** spec.eta, 1e-10)
        return 0.5 * float(np.asarray(grid.load) @ u)

    for algo, kw in VARIANTS:
        if only is not None and algo not in only:
            continue
        if algo == "pgd_exact" and n in KNOWN_PGD:
            print(f"{n} pgd_exact (earlier run) exact {KNOWN_PGD[n]:10.3f}", flush=True)
            continue
        t0 = time.perf_counter()
        try:
            r = B.run(spec, B.SolverConfig(algorithm=algo, max_iters=60_000, **kw))
        except Exception as exc:  # report and go on
            print(f"{algo} {kw}: {exc!r}", flush=True)
            continue
        dt = time.perf_counter() - t0
        c = exact_compliance(r.state.v.values)
        vol = np.asarray(r.record.volume)
        print(f"{n} {algo:14s} {str(kw):22s} {r.reason:9s} it {r.state.iter:6d} {dt:6.1f}s "
              f"exact {c:10.3f} final vol {vol[-1]:.1f} min vol {vol.min():.1f}", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["300"]
    only = None
    if "--only" in args:
        i = args.index("--only")
        only, args = set(args[i + 1].split(",")), args[:i]
    for n in (int(a) for a in args):
        main(n, only)
