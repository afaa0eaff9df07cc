"""Roofline of the CG/MG half of the matvec/CG path (north star: ">= 70% of
HBM roofline at >= 64M cells"; "PCG/MG bytes must be declared").

    python tools/cg_roofline.py [cg|mg|both] [--json OUT]

cg: Jacobi-PCG, `steps` CG iterations through the public C entry point
    bsp_pcg_apply at C5 (MBB 16384x8192: 134M cells, 268M DOFs).  Declared
    algorithmic bytes (each array read once and written once per kernel,
    8 bytes per value; n DOFs, E cells):
      k_diag                      8E + 8n        (a in, D out)
      k_pcg_init_jacobi           32n            (b, D in; R, P out)
      per step: K p + p.Kp         16n + 8E       (p, a in; q out)
      k_pcg_update (first)         48n            (P, Q, R, D in; X, R out)
      k_pcg_update (middle)        56n            (+ X in)
      k_pcg_update (last)          32n            (P, X, base in; out out)
      k_pcg_dir (all but last)     32n            (R, D, P in; P out)
    i.e. 104n + 8E per interior CG step.
mg: one V-cycle / one MG-PCG-4 iteration of C4 (cantilever 4096^2) for an
    ncu capture (kernel list and DRAM bytes per kernel; tools/README).
"""
import argparse
import json
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore", message="decay exponent")


def cg_bytes(n, E, steps):
    b = (8 * E + 8 * n) + 32 * n
    for j in range(steps):
        b += 16 * n + 8 * E
        last, first = j == steps - 1, j == 0
        b += 32 * n if last else (48 * n if first else 56 * n)
        if not last:
            b += 32 * n
    return b


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def run_cg(steps=20, reps=5):
    import torch

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import fea
    from paper_2204_06204_b200._native import call
    spec = B.problems.mbb_half_beam(16384, 8192)
    grid = B.problems.resolve_device(spec)
    n, E = grid.num_dofs, grid.num_elements
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = torch.rand(E, dtype=torch.float64, device="cuda", generator=gen) * 0.999 + 1e-3
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    b[torch.from_numpy(np.asarray(grid.fixed_dofs)).to("cuda")] = 0.0
    out = torch.empty_like(b)
    s = torch.cuda.current_stream()
    h = fea.grid_handle(grid)
    args = (h, None, a.data_ptr(), b.data_ptr(), steps, 0.6, 1, None, 1.0, out.data_ptr(),
            s.cuda_stream)
    call("bsp_pcg_apply", *args)  # warm-up (allocates the workspace)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(s)
    for i in range(reps):
        call("bsp_pcg_apply", *args)
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    ms = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))
    nbytes = cg_bytes(n, E, steps)
    hbm, src = peak()
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"workload": f"Jacobi-PCG-{steps} (bsp_pcg_apply) on C5 MBB 16384x8192, "
                        "134M cells, 268M DOFs",
            "steps": steps, "ms_per_apply": ms, "ms_per_cg_step": ms / steps,
            "alg_bytes_per_apply": nbytes,
            "alg_bytes_per_interior_step": 104 * n + 8 * E,
            "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
            "peak_source": src, "bound": "hbm"}


def run_mg(iters=3):
    import torch

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    spec = B.problems.cantilever_square(4096)
    out = {}
    for algo in ("mg_pcg", "mg_vcycle"):
        cfg = B.SolverConfig(algorithm=algo, max_iters=10 ** 9)
        ws = S._prepare(spec, cfg)
        loop = S.DeviceLoop(ws, cfg, max_batch=iters + 2)
        loop.run(1, [cfg.step_size(k) for k in (1, 2)])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.ExternalStream(loop.stream())
        e0.record(st)
        loop.run(3, [cfg.step_size(k) for k in range(3, 3 + iters)])
        e1.record(st)
        torch.cuda.synchronize()
        out[algo] = {"ms_per_iter": e0.elapsed_time(e1) / iters,
                     "kernels_per_iter": loop.info()["kernels_per_iter"]}
        del loop
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="both", choices=["cg", "mg", "both"])
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    res = {}
    if a.what in ("cg", "both"):
        res["cg"] = run_cg()
    if a.what in ("mg", "both"):
        res["mg"] = run_mg()
    print(json.dumps(res, indent=1))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(res, fh, indent=1)
