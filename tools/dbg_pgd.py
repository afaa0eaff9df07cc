"""pgd_exact on the acceptance L-shape: does exact_solve (MG-PCG) converge along the run?
On failure the last design is saved to gpurun_out/v_fail.npy."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06204_b200 as B

spec = B.catalog()["lshape"].scale(0.4)
for lim in sys.argv[1:] or ["0", "2048"]:
    os.environ["BSP_MG_TAIL"] = lim
    t = time.time()
    last = {}
    try:
        r = B.run(spec, B.SolverConfig(algorithm="pgd_exact", max_iters=50000, snapshot_every=1),
                  sink=lambda s: last.update(v=s.v.values.copy(), k=s.iter))
        print(lim, r.reason, r.state.iter, r.state.compliance, f"{time.time() - t:.1f}s", flush=True)
    except Exception as e:
        print(lim, "FAIL after iteration", last.get("k"), e, f"{time.time() - t:.1f}s", flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        np.save("gpurun_out/v_fail.npy", last["v"])
