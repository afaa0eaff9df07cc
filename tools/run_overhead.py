"""Host overhead of run(): time inside DeviceLoop.run vs. between calls (C2)."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import numpy as np
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S
spec = B.problems.mbb_half_beam(440, 250, 0.5)
inside, marks = [], []
orig = S.DeviceLoop.run
def timed(self, k, alphas):
    t0 = time.perf_counter(); out = orig(self, k, alphas); inside.append(time.perf_counter() - t0)
    marks.append(time.perf_counter()); return out
S.DeviceLoop.run = timed
for snap in (0, 256):
    inside.clear(); marks.clear()
    t0 = time.perf_counter()
    B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=4096, snapshot_every=snap),
          sink=(lambda s: None) if snap else None)
    tot = time.perf_counter() - t0
    gaps = np.diff(marks) - np.array(inside[1:])
    print(f"snapshot_every={snap}: total {tot*1e3:.1f} ms, batches {len(inside)}, "
          f"inside run() median {np.median(inside)*1e3:.2f} ms, between calls median {np.median(gaps)*1e3:.3f} ms")
