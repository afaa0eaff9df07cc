"""Per-iteration device time of every BASELINE.json config (C1..C5 on one GPU).

    python tools/config_sweep.py [C1 C2 ...] [--iters K] [--warmup W]

Each config runs its outer loop on the device (`DeviceLoop`, CUDA-graph
replays) for W warm-up iterations, then K iterations bracketed by CUDA events
on the solver stream, without L2 flushes (steady state of a long run).
Prints one line per config, plus a JSON summary on the last line.
"""
from __future__ import annotations

import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")

CONFIGS = {
    # name: (problem factory, algorithm, extra SolverConfig kwargs, description)
    "C1": ("teaser", "cpfbto_krylov", {}, "cantilever 128x256 (teaser), cpfbto_krylov D=20"),
    "C2": ("mbb440", "pfbto_jacobi", {}, "MBB half-beam 440x250, pfbto_jacobi"),
    "C3": ("lbracket300", "mg_pcg", {}, "L-bracket 300x300 passive void, MG-PCG-4"),
    "C4": ("cant4096", "mg_pcg", {}, "cantilever 4096x4096, MG-PCG-4"),
    "C4v": ("cant4096", "mg_vcycle", {}, "cantilever 4096x4096, one MG V-cycle"),
    "C5": ("mbb16384x8192", "pfbto_jacobi", {}, "MBB 16384x8192 (134M cells) on 1 GPU, pfbto_jacobi"),
    "C5k": ("mbb16384x8192", "cpfbto_krylov", {},
            "MBB 16384x8192 (134M cells) on 1 GPU, cpfbto_krylov D=20"),
}


def problem(B, name):
    P = B.problems
    if name == "teaser":
        return B.catalog()["teaser"]
    if name == "mbb440":
        return P.mbb_half_beam(440, 250)
    if name == "lbracket300":
        return P.l_bracket(300)
    if name == "cant4096":
        return P.cantilever_square(4096)
    if name.startswith("mbb"):
        nx, ny = name[3:].split("x")
        return P.mbb_half_beam(int(nx), int(ny))
    raise KeyError(name)


def time_config(key, iters=20, warmup=3):
    import numpy as np
    import torch

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    from paper_2204_06204_b200._native import call

    pname, algo, kw, desc = CONFIGS[key]
    spec = problem(B, pname)
    cfg = B.SolverConfig(algorithm=algo, max_iters=10 ** 9, **kw)
    t0 = time.perf_counter()
    ws = S._prepare(spec, cfg)
    loop = S.DeviceLoop(ws, cfg, max_batch=max(iters, warmup))
    setup_s = time.perf_counter() - t0
    done, status, _ = loop.run(1, [cfg.step_size(j) for j in range(1, warmup + 1)])
    assert status == 0 and done == warmup, (key, done, status)
    k = warmup + 1
    stream = torch.cuda.ExternalStream(loop.stream())
    call("bsp_solver_set_alphas", loop._h, k, iters,
         np.array([cfg.step_size(j) for j in range(k, k + iters)]).ctypes.data)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(iters):
        call("bsp_solver_launch", loop._h, k + i)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    import ctypes as C
    rec = np.zeros((iters, 4))
    dn, st = C.c_int(), C.c_int()
    call("bsp_solver_finish", loop._h, k, iters, rec.ctypes.data, C.byref(dn), C.byref(st))
    info = loop.info()
    g = ws.grid
    out = {"workload": desc, "algorithm": algo, "cells": g.num_elements, "dofs": g.num_dofs,
           "ms_per_iter": ms, "iters": iters, "kernels_per_iter": info["kernels_per_iter"],
           "setup_s": setup_s, "status": int(st.value),
           "last_compliance": float(rec[dn.value - 1, 0]) if dn.value else None}
    del loop, ws
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    iters = 20
    warmup = 3
    if "--iters" in sys.argv:
        iters = int(sys.argv[sys.argv.index("--iters") + 1])
    if "--warmup" in sys.argv:
        warmup = int(sys.argv[sys.argv.index("--warmup") + 1])
    keys = [a for a in args if a in CONFIGS] or list(CONFIGS)
    res = {}
    for k in keys:
        r = time_config(k, iters, warmup)
        res[k] = r
        print(f"{k}: {r['workload']}: {r['ms_per_iter']:.3f} ms/iter ({r['kernels_per_iter']} kernels, "
              f"setup {r['setup_s']:.1f} s, compliance {r['last_compliance']})", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
