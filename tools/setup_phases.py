"""Set-up cost of a large problem (C5: 16384 x 8192) by phase."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import numpy as np
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S
import torch
torch.cuda.init()
nx, ny = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (16384, 8192)
spec = B.problems.mbb_half_beam(nx, ny)
cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=10)
t = time.perf_counter()
grid = B.resolve(spec); t1 = time.perf_counter(); print(f"resolve {t1-t:.2f} s")
grid.native(); t2 = time.perf_counter(); print(f"bsp_grid_create {t2-t1:.2f} s")
v = np.full(spec.num_elements, 0.5)
rho = S._squared_jacobi_rho(grid, v, 3.0, spec.filter, 0); t3 = time.perf_counter(); print(f"beta power iteration {t3-t2:.2f} s")
ws = S._prepare(spec, cfg); t4 = time.perf_counter(); print(f"_prepare total {t4-t3:.2f} s")
loop = S.DeviceLoop(ws, cfg); t5 = time.perf_counter(); print(f"DeviceLoop create {t5-t4:.2f} s")
