"""How often the bounded-simplex projection needs its lambda search (the box
early exit fails) over a run, and what those iterations cost.

    python tools/lam_freq.py [C2|C5] [--iters N]

Runs the device loop one iteration per batch (so DeviceLoop.info() reports
each iteration's lambda rounds) and prints the count of iterations with
rounds > 0, their rounds, and the device ms of the batches with and without.
"""
import json
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")


def main(name="C5", iters=300):
    import torch

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    spec = B.problems.mbb_half_beam(16384, 8192) if name == "C5" else B.problems.mbb_half_beam(440, 250)
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=10 ** 9)
    ws = S._prepare(spec, cfg)
    loop = S.DeviceLoop(ws, cfg, max_batch=4)
    st = torch.cuda.ExternalStream(loop.stream())
    rounds, ms = [], []
    for k in range(1, iters + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        done, status, _ = loop.run(k, [cfg.step_size(k)])
        e1.record(st)
        torch.cuda.synchronize()
        assert done == 1 and status == 0, (k, done, status)
        rounds.append(loop.info()["lambda_rounds"])
        ms.append(e0.elapsed_time(e1))
    r, m = np.array(rounds), np.array(ms)
    lam = r > 0
    out = {"config": name, "iters": iters, "lambda_iters": int(lam.sum()),
           "first_lambda_iters": [int(i + 1) for i in np.nonzero(lam)[0][:20]],
           "rounds_hist": {int(k): int(v) for k, v in zip(*np.unique(r[lam], return_counts=True))},
           "ms_median_no_lambda": float(np.median(m[~lam][3:])) if (~lam).sum() > 3 else None,
           "ms_median_lambda": float(np.median(m[lam])) if lam.any() else None,
           "lambda_iters_after_50": int(lam[50:].sum())}
    print(json.dumps(out))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a and not a[0].startswith("--") else "C5",
         int(a[a.index("--iters") + 1]) if "--iters" in a else 300)
