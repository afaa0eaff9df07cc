"""Where does the wall time of run() go?  Phase timings of repeated C2 runs."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import numpy as np
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S
spec = B.problems.mbb_half_beam(440, 250, 0.5)
for rep in range(8):
    t = [time.perf_counter()]
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=2020)
    ws = S._prepare(spec, cfg); t.append(time.perf_counter())
    loop = S.DeviceLoop(ws, cfg); t.append(time.perf_counter())
    k = 1
    while k <= 2020:
        n = min(256, 2021 - k)
        done, status, rows = loop.run(k, [cfg.step_size(j) for j in range(k, k + n)])
        k += done
    t.append(time.perf_counter())
    st = loop.read("u"); t.append(time.perf_counter())
    del loop, ws
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("prepare %.1f  loop-create %.1f  2020 iters %.1f  read %.1f  free %.1f ms" % tuple(d))
