"""Wall time of the public run() on C2 for growing iteration counts."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import paper_2204_06204_b200 as B
spec = B.problems.mbb_half_beam(440, 250, 0.5)
prev = None
for n in (20, 20, 520, 1020, 2020, 4020, 8020):
    t0 = time.perf_counter()
    res = B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=n))
    dt = time.perf_counter() - t0
    print(n, f"{dt*1e3:.1f} ms", res.reason, res.state.iter, f"last dv {res.record.dv_inf[-1]:.2e} res {res.record.residual_inf[-1]:.2e}")
