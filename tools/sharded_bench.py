"""Row-slab (multi-GPU) timing of one rank, run as an isolated child process.

    python tools/sharded_bench.py --world N --rank r --device d --port P
                                  [--nx 16384 --ny 8192] [--algo pfbto_jacobi]
                                  [--steps K] [--warmup W] [--no-e2e]

`bench.py` starts one of these per rank under torchrun.  The children form
their own process group (gloo over 127.0.0.1:P, for the NCCL id broadcast and
the host gathers) and the library builds its own NCCL communicator, so a
failure or a hang stays in the children and the parent's time-out contains
it.  Output is one line, `RESULT <json>`:
  * ms_per_iter: device ms/iter over K timed iterations of the slab loop
    (CUDA events on the slab stream); the halo-exchange and all-gather
    device ms; the slab geometry and set-up time;
  * e2e_ms_per_iter: the same iterations through the public API,
    run(problem, SolverConfig(...), slabs="nccl") -- set-up, the device loop
    in batches with the step sizes in and the record rows out, and the final
    state gathered to every rank -- as (T(W + KE) - T(W)) / KE of two
    wall-clock runs (KE = max(K, 600), after an untimed run), so the set-up
    cancels.
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
    ap.add_argument("--port", type=int, default=0, help="gloo rendezvous port (0: pick, world 1)")
    ap.add_argument("--nx", type=int, default=16384)
    ap.add_argument("--ny", type=int, default=8192)
    ap.add_argument("--algo", default="pfbto_jacobi")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(a.device)
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200.distributed import SlabLoop, broadcast_nccl_id, slab_rows

    port = a.port
    if port == 0:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=a.rank,
                            world_size=a.world)
    spec = B.problems.mbb_half_beam(a.nx, a.ny)
    cfg = B.SolverConfig(algorithm=a.algo, max_iters=10 ** 9)
    K, W = a.steps, a.warmup
    t0 = time.perf_counter()
    loop = SlabLoop(spec, cfg, world=a.world, rank=a.rank, nccl_id=broadcast_nccl_id(a.rank),
                    local=False, max_batch=max(K, W))
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
    del loop
    torch.cuda.empty_cache()
    e2e = None
    if not a.no_e2e:
        # an untimed first run: one-time costs (module loads, NCCL set-up,
        # graph instantiation paths) must not land in T(W)
        B.run(spec, B.SolverConfig(algorithm=a.algo, max_iters=W), slabs="nccl")
        # the difference must dwarf the set-up's run-to-run noise (~0.3 s)
        KE = max(K, 600)
        wall = {}
        for n in (W, W + KE):
            dist.barrier()
            t = time.perf_counter()
            res = B.run(spec, B.SolverConfig(algorithm=a.algo, max_iters=n), slabs="nccl")
            wall[n] = time.perf_counter() - t
            assert res.state.iter == n, (res.reason, res.state.iter)
        e2e = (wall[W + KE] - wall[W]) * 1e3 / KE
    print("RESULT " + json.dumps({
        "rank": a.rank, "ms_per_iter": ms, "halo_ms": halo_ms, "allgather_ms": gather_ms,
        "rows": [e0_, e1_], "window": [w0, w1], "setup_s": setup_s, "graphs": info["graphs"],
        "host_lambda_iters": info["host_lambda_iters"], "e2e_ms_per_iter": e2e,
        "last_row": [float(x) for x in rows[K - 1]]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
