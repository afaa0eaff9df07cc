"""Row-slab (multi-GPU) timing of one rank, run as an isolated child process.

    python tools/sharded_bench.py --world N --rank r --device d [--nx 16384 --ny 8192]
                                  [--algo pfbto_jacobi] [--steps K] [--warmup W]

`bench.py` starts one of these per rank under torchrun.  The children form
their own NCCL communicator through the library (`bsp_dist_*`), so a failure
or a hang stays in the child and the parent's time-out contains it.  Rank 0
prints `ID <hex>` with the NCCL unique id; the other ranks read the same line
on stdin (the parents relay it over torch.distributed).  Output is one line,
`RESULT <json>`: device ms/iter over K timed iterations (CUDA events on the
slab stream), the halo-exchange and all-gather device ms, and the slab
geometry.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--nx", type=int, default=16384)
    ap.add_argument("--ny", type=int, default=8192)
    ap.add_argument("--algo", default="pfbto_jacobi")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(a.device)
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200.distributed import SlabLoop, nccl_unique_id, slab_rows

    if a.rank == 0:
        nid = nccl_unique_id()
        print("ID " + nid.hex(), flush=True)
    else:
        line = sys.stdin.readline().strip()
        assert line.startswith("ID "), line
        nid = bytes.fromhex(line[3:])
    spec = B.problems.mbb_half_beam(a.nx, a.ny)
    cfg = B.SolverConfig(algorithm=a.algo, max_iters=10 ** 9)
    t0 = time.perf_counter()
    K, W = a.steps, a.warmup
    loop = SlabLoop(spec, cfg, world=a.world, rank=a.rank, nccl_id=nid, local=False,
                    max_batch=max(K, W))
    setup_s = time.perf_counter() - t0
    done, status, _ = loop.run(1, [cfg.step_size(k) for k in range(1, W + 1)])
    assert status == 0 and done == W, (done, status)
    stream = torch.cuda.ExternalStream(loop.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    done, status, rows = loop.run(W + 1, [cfg.step_size(k) for k in range(W + 1, W + K + 1)])
    e1.record(stream)
    torch.cuda.synchronize()
    assert status == 0 and done == K, (done, status)
    ms = e0.elapsed_time(e1) / K
    halo_ms, gather_ms = loop.comm_ms(50)
    e0_, e1_, w0, w1 = slab_rows(a.ny, a.world, a.rank, loop.halo)
    info = loop.info()
    print("RESULT " + json.dumps({
        "rank": a.rank, "ms_per_iter": ms, "halo_ms": halo_ms, "allgather_ms": gather_ms,
        "rows": [e0_, e1_], "window": [w0, w1], "setup_s": setup_s, "graphs": info["graphs"],
        "host_lambda_iters": info["host_lambda_iters"],
        "last_row": [float(x) for x in rows[K - 1]]}), flush=True)


if __name__ == "__main__":
    main()
