"""Converged C3 endpoints on the GPU (BASELINE configs[2]: L-bracket 300x300
with the passive void): pgd_exact (exact inversion) and the multigrid
approximate inverse mg_pcg, each run to the reference's termination test.

    python tools/c3_endpoints.py gpurun_out/c3_endpoints.npz

The pgd_exact endpoint is then certified by the REAL reference in the builder
container (`tests/golden/make_golden.py c3_certificate`): one reference
pgd step from it (SuperLU solve, sensitivity, projection) must move the
design by less than tol_dv, and the reference's exact compliance of both
endpoints is recorded (tests/golden/c3_endpoint.npz)."""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
warnings.filterwarnings("ignore", message="decay exponent")

import paper_2204_06204_b200 as B  # noqa: E402


def main(out):
    spec = B.problems.l_bracket(300)
    res = {}
    for algo in ("pgd_exact", "mg_pcg"):
        t0 = time.perf_counter()
        r = B.run(spec, B.SolverConfig(algorithm=algo, max_iters=200_000))
        dt = time.perf_counter() - t0
        print(f"{algo}: {r.reason} after {r.state.iter} iterations, {dt:.1f} s, "
              f"compliance {r.record.compliance[-1]:.6f}", flush=True)
        res[f"{algo}_v"] = r.state.v.values
        res[f"{algo}_iter"] = np.int64(r.state.iter)
        res[f"{algo}_reason"] = r.reason
        res[f"{algo}_rec"] = np.array([r.record.iters, r.record.compliance, r.record.residual_inf,
                                       r.record.dv_inf, r.record.volume]).T
        res[f"{algo}_seconds"] = dt
    np.savez_compressed(out, **res)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c3_endpoints.npz")
