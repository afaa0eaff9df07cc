"""lambda-search rounds per iteration (DeviceLoop.info) on a config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B
from paper_2204_06204_b200 import solvers as S

nx, ny, it = (int(a) for a in sys.argv[1:4])
spec = B.problems.mbb_half_beam(nx, ny)
cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=10 ** 9)
ws = S._prepare(spec, cfg)
loop = S.DeviceLoop(ws, cfg, max_batch=1)
rounds = []
for k in range(1, it + 1):
    loop.run(k, [cfg.step_size(k)])
    rounds.append(loop.info()["lambda_rounds"])
print("rounds per iteration:", rounds)
