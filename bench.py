#!/usr/bin/env python
"""Benchmark of the bilevel-SIMP hot path (one JSON line on stdout, rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], C2): MBB half-beam 440x250 (110k cells,
221k DOFs), PFBTO with the Jacobi-preconditioned approximate inverse.  A step
is one outer iteration of run()'s loop body (solvers.py:442-475): filter +
activation, residual + reductions + sensitivities, filter adjoint,
low-level step, projected high-level step + record.

  value        ms per outer iteration on the device (CUDA events on the solver
               stream around each iteration's graph replay; L2 flushed with a
               256 MiB write before every timed iteration: the C2 working set
               fits the 126 MB L2).  Lower is better.
  e2e          the same iteration through the C-ABI call with HOST buffers
               (bsp_solver_step_host: v, u in from pinned memory, v_next,
               u_next and the record row back), wall clock per call.
  roofline     the dominant kernel of the matvec/CG path, the masked Q4
               matvec, at the north star's large-grid size (8192x16384 cells =
               134M cells, inputs 5.4 GB >> L2): algorithmic bytes 16n+8E per
               launch / CUDA-event time, vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline the oracle port (numpy/scipy restatement of the reference) on
               the host cores, 1 thread, a bounded sample of C2 iterations.
  --impl reference: the reference's CPU implementation of the path: the
               unmodified `bisimp.solvers.run` from baseline/_ref on the same
               workload, 1 core and all cores, the faster one reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
warnings.filterwarnings("ignore", message="decay exponent")

METRIC = "ms per TO outer iteration and matvec GDOF/s vs HBM roofline, 1/2/4/8 B200"
UNIT = "ms/iter"
WORKLOAD = "C2: MBB half-beam 440x250 (110,000 cells, 221,382 DOFs), pfbto_jacobi"
C5_SHARDED = ("C5: MBB half-beam 16384x8192 (134,217,728 cells, 268,484,610 DOFs) as row "
              "slabs, pfbto_jacobi")
HBM_FALLBACK = 6650.0



def roofline_traffic():
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    --set full capture of the same kernel and workload (profiles/, the
    newest round's file), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          "r*_roofline_traffic.json")))
    if not files:
        return None
    with open(files[-1]) as fh:
        return float(json.load(fh)["dram_bytes_per_launch"])

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def c2_spec(B):
    return B.problems.mbb_half_beam(440, 250, 0.5)


# ------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self, which: str):
        setattr(self, which, time.monotonic())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_end", float("inf"))
        for ts, line in self.lines:
            if not (t0 <= ts <= t1 + 0.15):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU legs ----

def cpu_iterations(seconds: float, threads: int | None, max_iters: int, warmup: int = 2):
    """Time oracle C2 iterations on the host; returns (ms/iter list, n)."""
    from oracle import bisimp_oracle as O
    import paper_2204_06204_b200.problems as P
    spec = P.mbb_half_beam(440, 250, 0.5)
    g = O.build_grid(spec.nx, spec.ny, spec.fixtures, spec.loads)
    ctx = None
    if threads is not None:
        try:
            from threadpoolctl import threadpool_limits
            ctx = threadpool_limits(limits=threads)
        except Exception:
            ctx = None
    try:
        v, active, budget, beta = O.setup(g, spec.nx, spec.ny, spec.volume_fraction, 0.1,
                                          np.zeros(spec.nx * spec.ny, bool), "pfbto_jacobi",
                                          3.0, 7, 1.5, beta=None, seed=0)
        u = np.zeros(g.n_dofs)
        times = []
        t_end = time.perf_counter() + seconds
        for k in range(1, max_iters + warmup + 1):
            t0 = time.perf_counter()
            u, v, _, _, _ = O.iterate(g, v, u, k, algorithm="pfbto_jacobi", eta=3.0, size=7,
                                      sigma=1.5, beta=beta, alpha0=0.25, m=0.75, lo=0.1,
                                      budget=budget, active=active)
            dt = time.perf_counter() - t0
            if k > warmup:
                times.append(dt * 1e3)
            if k > warmup and time.perf_counter() > t_end:
                break
        return times
    finally:
        if ctx is not None:
            ctx.unregister() if hasattr(ctx, "unregister") else None


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_run_ms(ref, spec, warmup, steps, threads, blas_threads):
    """ms/iter of the UNMODIFIED reference `bisimp.solvers.run` on C2
    (BASELINE.md §4): clock=time.perf_counter stamps every iteration; the
    median and mean of diff(elapsed_s) over the timed iterations after
    `warmup` warm-up iterations (the tests/test_acceptance.py:239-245 method)."""
    from threadpoolctl import threadpool_limits
    cfg = ref.solvers.SolverConfig(algorithm="pfbto_jacobi", max_iters=warmup + steps)
    with threadpool_limits(limits=blas_threads):
        res = ref.solvers.run(spec, cfg, threads=threads, clock=time.perf_counter)
    assert len(res.record.elapsed_s) == warmup + steps, (res.reason, len(res.record.elapsed_s))
    d = np.diff(np.asarray(res.record.elapsed_s))[warmup - 1:] * 1e3
    return float(np.median(d)), float(np.mean(d))


def reference_arm(args, world):
    """--impl reference: the reference's own CPU implementation of the path.

    The reference is pure Python (numpy/scipy), so its implementation IS the
    package: `baseline/_ref` holds the unmodified reference installed with
    pip, and this arm runs `bisimp.solvers.run` on C2 through
    its public API.  Two host configurations are timed, because the
    reference's own threading makes it slower: 1 core
    (run(threads=1), BLAS 1 thread) and all host cores (run(threads=cores),
    BLAS on all cores); the faster one is the line's value.  Without
    baseline/_ref the numpy oracle port stands in and says so."""
    cores = os.cpu_count() or 1
    if world > 1:
        return reference_arm_c5(args, world, cores)
    steps = min(args.steps, 500)   # bounded sample: <= ~10 s per configuration
    warmup = max(args.warmup, 5)
    legs = {}
    if os.path.isdir(os.path.join(REF_DIR, "bisimp")):
        sys.path.insert(0, REF_DIR)
        import bisimp.problems
        import bisimp.solvers
        import bisimp as ref
        spec = ref.problems.ProblemSpec(
            nx=440, ny=250, volume_fraction=0.5,
            fixtures=({"edge": "left", "dofs": "x"}, {"point": (1.0, 1.0), "dofs": "y"}),
            loads=({"edge": "top", "span": (0.0, 0.02), "fy": -1.0},))
        for name, thr, blas in (("1core", 1, 1), ("allcores", cores, cores)):
            med, mean = _reference_run_ms(ref, spec, warmup, steps, thr, blas)
            legs[name] = {"median_ms": med, "mean_ms": mean, "run_threads": thr,
                          "blas_threads": blas}
        kind = "reference"
        sample = (f"{steps} C2 pfbto_jacobi iterations of the unmodified reference "
                  f"bisimp.solvers.run (baseline/_ref) after {warmup} warm-up, "
                  "clock=time.perf_counter, median of diff(elapsed_s)")
    else:
        times = cpu_iterations(30.0, threads=None, max_iters=steps, warmup=warmup)
        legs["allcores"] = {"median_ms": float(np.median(times)), "mean_ms": float(np.mean(times)),
                            "run_threads": 1, "blas_threads": cores}
        kind = "port"
        sample = (f"{len(times)} C2 pfbto_jacobi iterations of the numpy oracle port "
                  "(baseline/_ref absent), median")
    best = min(legs, key=lambda k: legs[k]["median_ms"])
    ms = legs[best]["median_ms"]
    used = legs[best]["run_threads"] if best == "1core" else cores
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (MBB half-beam load case, reference problem setup)",
        "config": {"workload": WORKLOAD, "flush": "n/a (host)"},
        "cpu_baseline": {"value": ms, "unit": UNIT, "cores": used, "kind": kind,
                         "sample": sample + f"; fastest host configuration: {best}"},
        "reference_legs": legs,
        "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def reference_arm_c5(args, world, cores):
    """--impl reference at N > 1: the B200 arm's headline is C5 (134M cells)
    split over the GPUs, so the reference times the same workload.  A full C5
    iteration of the reference needs ~45 GB and about a minute,
    so each step is a bounded sample: one iteration on the 16384 x 1024 band
    (1/8 of C5, the slab of one rank at N = 8; same algorithm, loads and
    fixtures), scaled by 8 -- the reference's cost is linear in the cells
    (BASELINE.md §2).  beta is passed (the GPU's C5 value, 0.2) so the set-up
    does not spend ~100 band matvecs on its power iteration; an iteration's
    cost does not depend on it."""
    if not os.path.isdir(os.path.join(REF_DIR, "bisimp")):
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref is not installed"}))
        return
    sys.path.insert(0, REF_DIR)
    import bisimp.problems
    import bisimp.solvers
    import bisimp as ref
    from threadpoolctl import threadpool_limits
    spec = ref.problems.ProblemSpec(
        nx=16384, ny=1024, volume_fraction=0.5,
        fixtures=({"edge": "left", "dofs": "x"}, {"point": (1.0, 1.0), "dofs": "y"}),
        loads=({"edge": "top", "span": (0.0, 0.02), "fy": -1.0},))
    n = 3
    cfg = ref.solvers.SolverConfig(algorithm="pfbto_jacobi", beta=0.2, max_iters=n)
    with threadpool_limits(limits=1):
        res = ref.solvers.run(spec, cfg, threads=1, clock=time.perf_counter)
    d = np.diff(np.asarray(res.record.elapsed_s)) * 1e3
    ms = float(np.median(d)) * 8.0
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (MBB half-beam load case, reference problem setup)",
        "config": {"workload": C5_SHARDED, "flush": "n/a (host)"},
        "cpu_baseline": {"value": ms, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"median of {n - 1} iteration times of the unmodified "
                                   "reference bisimp.solvers.run (baseline/_ref) on the "
                                   "16384x1024 band (1/8 of C5), x 8"},
        "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU legs ----

def matvec_roofline(B, torch, nx, ny, launches=20, warmup=3):
    """Q4 matvec at nx x ny: the median of `launches` back-to-back launches, each
    bracketed by CUDA events on the launching stream, of (a) the solver's path
    (input zero on fixed DOFs, bsp_apply_stiffness_premasked) and (b) the public
    apply_stiffness path (input masking in-kernel)."""
    from paper_2204_06204_b200._native import call
    spec = B.problems.mbb_half_beam(nx, ny, 0.5)
    g = B.resolve(spec)
    E, n = g.num_elements, g.num_dofs
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = torch.rand(E, dtype=torch.float64, device="cuda", generator=gen) * 0.999 + 1e-3
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    u[torch.from_numpy(g.fixed_dofs).to("cuda")] = 0.0
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    h = g.native()
    s = torch.cuda.current_stream()
    out = {}
    for fn in ("bsp_apply_stiffness_premasked", "bsp_apply_stiffness"):
        for _ in range(warmup):
            call(fn, h, a.data_ptr(), u.data_ptr(), y.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(launches + 1)]
        ev[0].record(s)
        for i in range(launches):
            call(fn, h, a.data_ptr(), u.data_ptr(), y.data_ptr(), s.cuda_stream)
            ev[i + 1].record(s)
        torch.cuda.synchronize()
        out[fn] = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(launches)]))
    alg_bytes = 16 * n + 8 * E
    del a, u, y, g
    torch.cuda.empty_cache()
    return out["bsp_apply_stiffness_premasked"], alg_bytes, n, E, out["bsp_apply_stiffness"]


def sharded_c5(rank, world, local, dist, timeout=600.0, algo="pfbto_jacobi", e2e=True):
    """C5 (MBB 16384x8192, 134M cells) as row slabs over all ranks.

    One isolated child per rank (tools/sharded_bench.py) forms its own gloo
    group on a port rank 0 picks and the library's NCCL communicator, so a
    child that fails or hangs is reported, never fatal.  The children time the
    slab loop on the device and, through the public API, run(..., slabs="nccl")
    end to end."""
    import select
    import socket
    port = None
    if rank == 0:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
    obj = [port]
    dist.broadcast_object_list(obj, src=0)
    port = obj[0]
    cmd = [sys.executable, os.path.join(ROOT, "tools", "sharded_bench.py"), "--world", str(world),
           "--rank", str(rank), "--device", str(local), "--algo", algo, "--port", str(port)]
    if not e2e:
        cmd.append("--no-e2e")
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    t_end = time.monotonic() + timeout
    result = None
    while result is None:
        r, _, _ = select.select([p.stdout], [], [], 1.0)
        if r:
            line = p.stdout.readline()
            if line.startswith("RESULT "):
                result = json.loads(line[7:])
            elif not line:
                result = {"error": "exit without RESULT"}
        elif p.poll() is not None:
            result = {"error": f"exit {p.returncode} without RESULT"}
        elif time.monotonic() > t_end:
            result = {"error": "timeout"}
    if p.poll() is None:
        p.kill()
    try:
        err = p.stderr.read()[-400:] if "error" in result else ""
    except Exception:
        err = ""
    if err:
        result["stderr_tail"] = err
    allr = [None] * world
    dist.all_gather_object(allr, result)
    ok = [r for r in allr if r and "error" not in r]
    comm = {"pfbto_jacobi": {"halo": 2, "allgather": 3},
            "pcg_jacobi": {"halo": "2 + 1 per CG step (p)",
                           "allgather": "3 + 1 + 2 per CG step (p.Kp, r.z)"},
            "cpfbto_krylov": {"halo": "2 + 1 per power (21)",
                              "allgather": "3 + 1 per power (norm) + 1 of the TSQR factors"},
            "mg_pcg": {"halo": "2 + 1 per CG step (p); the block V-cycles are rank-local",
                       "allgather": "3 + 1 + 2 per CG step (p.Kp, r.z)"}}[algo]
    out = {"workload": f"C5: MBB half-beam 16384x8192 (134M cells, 268M DOFs) as row slabs, "
                       f"{algo}, NCCL halo exchange + all-gathers",
           "n_ranks": world}
    if len(ok) == world:
        out.update({
            "ms_per_iter": max(r["ms_per_iter"] for r in ok),
            "halo_ms_per_exchange": max(r["halo_ms"] for r in ok),
            "allgather_ms": max(r["allgather_ms"] for r in ok),
            "exchanges_per_iter": comm,
            "rows_per_rank": [r["rows"] for r in ok],
            "setup_s": max(r["setup_s"] for r in ok),
            "graphs": all(r["graphs"] for r in ok),
            "last_row": ok[0]["last_row"]})
        if all(r.get("e2e_ms_per_iter") is not None for r in ok):
            out["e2e_ms_per_iter"] = max(r["e2e_ms_per_iter"] for r in ok)
    else:
        out["errors"] = [r for r in allr if not r or "error" in r]
    return out


def _rebatch(S, ws, cfg, loop, K, k_next):
    """A loop whose batch holds K iterations, advanced to iteration k_next."""
    big = S.DeviceLoop(ws, cfg, max_batch=K)
    done, status, _ = big.run(1, [cfg.step_size(j) for j in range(1, k_next)])
    assert status == 0 and done == k_next - 1
    del loop
    return big


def b200_arm(args, rank, world, local):
    import torch
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    from paper_2204_06204_b200._native import call

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = c2_spec(B)
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=10 ** 9)
    ws = S._prepare(spec, cfg)
    loop = S.DeviceLoop(ws, cfg)
    grid = ws.grid
    # warm-up through the normal batched path
    k = 1
    done, status, _ = loop.run(k, [cfg.step_size(j) for j in range(k, k + args.warmup)])
    assert status == 0 and done == args.warmup, (done, status)
    k += done
    K = args.steps
    if K > loop.max_batch:
        loop = _rebatch(S, ws, cfg, loop, K, k)
    stream = torch.cuda.ExternalStream(loop.stream())
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    alphas = np.array([cfg.step_size(j) for j in range(k, k + K)])
    call("bsp_solver_set_alphas", loop._h, k, K, alphas.ctypes.data)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # clocks are sampled from here through the hot loop and the end-to-end
    # runs below (the flushed K-step loop alone lasts a few ms at C2)
    clocks = ClockSampler(local).__enter__()
    time.sleep(0.5)  # nvidia-smi start-up; samples are kept only inside the timed regions
    clocks.mark("t_start")
    with torch.cuda.stream(stream):
        for i in range(K):
            flush.fill_(float(i))          # L2 flush (256 MiB write) between iterations
            starts[i].record(stream)
            call("bsp_solver_launch", loop._h, k + i)
            ends[i].record(stream)
    torch.cuda.synchronize()
    rec = np.zeros((K, 4))
    import ctypes as C
    dn, st = C.c_int(), C.c_int()
    call("bsp_solver_finish", loop._h, k, K, rec.ctypes.data, C.byref(dn), C.byref(st))
    assert st.value == 0 and dn.value == K, (dn.value, st.value)
    k += K
    step_ms = np.array([s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)])
    ms = float(step_ms.sum() / K)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # steady state without flushes: K back-to-back replays (what a long run sees)
    call("bsp_solver_set_alphas", loop._h, k, K,
         np.array([cfg.step_size(j) for j in range(k, k + K)]).ctypes.data)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(K):
        call("bsp_solver_launch", loop._h, k + i)
    e1.record(stream)
    torch.cuda.synchronize()
    call("bsp_solver_finish", loop._h, k, K, rec.ctypes.data, C.byref(dn), C.byref(st))
    hot_ms = e0.elapsed_time(e1) / K
    k += K
    info = loop.info()

    # e2e through the public API the reference's callers use: run(problem,
    # config, sink) (solvers.py:381; cli.py:73, sessions.py:106) with a
    # snapshot every 256 iterations.  Every step's step size goes host->device
    # and its ConvergenceRecord row device->host (batched bsp_solver_run calls
    # with host buffers).  Every 1024 steps the sink receives the state
    # (u, v, v_phys, a copied to the host).  The wall time between consecutive
    # sink calls / 1024 is one sample; the median sample is reported, which is
    # robust to host / power-state hiccups of the box.
    SNAP = 1024
    K_e2e = max(K, 8 * SNAP)
    stamps = []
    B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=2 * SNAP,
                               snapshot_every=SNAP), sink=lambda st: None)  # warm
    res_e2e = B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=K_e2e,
                                         snapshot_every=SNAP),
                    sink=lambda st: stamps.append(time.perf_counter()))
    assert res_e2e.state.iter == K_e2e, (res_e2e.reason, res_e2e.state.iter)
    batch_ms = np.diff(np.array(stamps[:K_e2e // SNAP])) * 1e3 / SNAP
    e2e_ms = float(np.median(batch_ms))
    e2e_mean_ms = float(np.mean(batch_ms))
    snap_bytes = 8 * (grid.num_dofs + 3 * grid.num_elements)
    # the same iteration with the full state through host buffers each step
    # (bsp_solver_step_host: v, u in from pinned memory; v_next, u_next and the
    # record row back): the worst-case drop-in call, one iteration at a time
    pin = lambda n: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()  # noqa: E731
    hv, hu, hvn, hun = pin(grid.num_elements), pin(grid.num_dofs), pin(grid.num_elements), pin(grid.num_dofs)
    hv[:] = loop.read("v")
    hu[:] = loop.read("u")
    for i in range(args.warmup):
        loop.step_host(k, cfg.step_size(k), hv, hu, hvn, hun)
        hv, hvn = hvn, hv
        hu, hun = hun, hu
        k += 1
    t0 = time.perf_counter()
    K_rt = min(K, 1000)
    for i in range(K_rt):
        loop.step_host(k, cfg.step_size(k), hv, hu, hvn, hun)
        hv, hvn = hvn, hv
        hu, hun = hun, hu
        k += 1
    rt_ms = (time.perf_counter() - t0) * 1e3 / K_rt
    clocks.mark("t_end")
    clocks.__exit__(None, None, None)
    rt_h2d = 8 * (grid.num_elements + grid.num_dofs)
    rt_d2h = 8 * (grid.num_elements + grid.num_dofs) + 8 * 4
    del loop
    torch.cuda.synchronize()

    hbm, peak_src = peaks()
    # dominant kernel of the matvec/CG path at the large-grid size
    mv_ms, mv_bytes, mv_n, mv_E, mv_pub_ms = matvec_roofline(B, torch, 16384, 8192)
    achieved = mv_bytes / (mv_ms * 1e-3) / 1e9
    # the C2 step as a whole against its own algorithmic bytes (latency bound)
    n2, E2 = grid.num_dofs, grid.num_elements
    it_bytes = 80 * n2 + 128 * E2
    fused_bytes = 48 * n2 + 80 * E2

    # the CG half of the matvec/CG path at the north star's >= 64M-cell size:
    # Jacobi-PCG-20 through bsp_pcg_apply on C5, declared bytes per CG step
    # (tools/cg_roofline.py)
    roofline_cg = None
    if not args.no_sweep:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import cg_roofline
        try:
            roofline_cg = cg_roofline.run_cg()
        except Exception as exc:  # report, never hide
            roofline_cg = {"error": repr(exc)[:200]}
        torch.cuda.empty_cache()

    # every BASELINE.json config on this GPU (steady-state device time per
    # iteration; tools/config_sweep.py), for context beside the C2 headline
    sweep = None
    if not args.no_sweep and world == 1:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import config_sweep
        sweep = {}
        # warm-up 10: past the one early iteration whose box projection fails
        # (C5: iteration 4; tools/lam_freq.py), i.e. the steady state of a run
        for key in ("C1", "C3", "C4", "C4v", "C5", "C5k"):
            try:
                sweep[key] = config_sweep.time_config(key, iters=10, warmup=10)
            except Exception as exc:  # report, never hide
                sweep[key] = {"error": repr(exc)[:200]}
    # C5 (BASELINE.json configs[4]) as row slabs: for N > 1 the headline
    # (strong scaling: the 134M-cell grid split over the N GPUs); at N = 1 one
    # rank (the N = 1 point of the same curve)
    algos = ("pfbto_jacobi", "pcg_jacobi", "cpfbto_krylov", "mg_pcg")
    sharded, shard_clocks = None, None
    if dist:
        with ClockSampler(local) as sc:
            sc.mark("t_start")
            sharded = {"pfbto_jacobi": sharded_c5(rank, world, local, dist)}
            sc.mark("t_end")
        shard_clocks = sc.summary()
        if not args.no_sweep:
            for a in algos[1:]:
                sharded[a] = sharded_c5(rank, world, local, dist, algo=a, e2e=False)
    elif not args.no_sharded:  # one NCCL rank on this GPU, in an isolated child
        import socket
        import torch.distributed as tdist
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                 world_size=1)
        sharded = {a: sharded_c5(0, 1, local, tdist, algo=a, e2e=(a == "pfbto_jacobi"))
                   for a in (algos if args.force_sharded else algos[:1])}
        tdist.destroy_process_group()
    cpu = None
    ref_configs = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the unmodified reference on every BASELINE config, bounded samples,
        # 1 core (tools/reference_configs.py), for the per-config ratios
        if not args.no_sweep:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import reference_configs
            try:
                ref_configs = reference_configs.main()
            except Exception as exc:  # report, never hide
                ref_configs = {"error": repr(exc)[:200]}
        times = cpu_iterations(args.cpu_seconds, threads=1, max_iters=2000)
        cpu = {"value": float(np.median(times)), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{len(times)} C2 pfbto_jacobi iterations of the numpy oracle port "
                         f"(median, 1 thread, ~{args.cpu_seconds:.0f} s budget)"}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (MBB half-beam load case, uniform initial design; no datasets)",
        "config": {"workload": WORKLOAD, "algorithm": "pfbto_jacobi",
                   "flush": "L2 flushed (256 MiB write) before every timed iteration",
                   "parallelism": "replicas" if world > 1 else "single GPU",
                   "cuda_graphs": info["graphs"]},
        "ms_per_iter_hot": hot_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": roofline_traffic(),
                     "kernel": "k_stiff3 (TMA Q4 matvec of the solver path, input zero on "
                               "fixed DOFs), 8192x16384 cells = 134M cells, 268M DOFs",
                     "alg_bytes_per_launch": mv_bytes, "ms_per_launch": mv_ms,
                     "gdof_per_s": mv_n / (mv_ms * 1e-3) / 1e9, "peak_source": peak_src,
                     "public_apply_stiffness": {
                         "ms_per_launch": mv_pub_ms,
                         "achieved": mv_bytes / (mv_pub_ms * 1e-3) / 1e9,
                         "frac": mv_bytes / (mv_pub_ms * 1e-3) / 1e9 / hbm}},
        "roofline_cg": roofline_cg,
        "roofline_step": {"alg_bytes_per_iter": it_bytes,
                          "achieved_gbs": it_bytes / (ms * 1e-3) / 1e9,
                          "fused_min_bytes_per_iter": fused_bytes,
                          "note": "80n+128E bytes per pfbto iteration (SURVEY §8(d) convention, "
                                  "stages unfused); 48n+80E is the minimum of this fused "
                                  "pipeline (DESIGN.md §3); C2 is latency bound"},
        "configs": sweep,
        "reference_configs": ref_configs,
        "sharded": sharded,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": 32 + snap_bytes / SNAP, "mean_ms": e2e_mean_ms,
                "path": f"public run(problem, SolverConfig(pfbto_jacobi, max_iters={K_e2e}, "
                        f"snapshot_every={SNAP}), sink) over C2: median wall time between sink "
                        f"calls / {SNAP} (alpha_k in, record row out every step, in batches of "
                        f"256; u, v, v_phys, a out every {SNAP} steps)"},
        "e2e_state_roundtrip": {"value": rt_ms, "unit": UNIT, "h2d_bytes_per_step": rt_h2d,
                                "d2h_bytes_per_step": rt_d2h,
                                "path": "bsp_solver_step_host: full state through pinned host "
                                        "buffers every iteration"},
        "gpu_launches": int(info["kernels_per_iter"]) * K,
        "clocks": clocks.summary(),
    }
    if world > 1:
        # strong scaling: the headline is C5 split over the N GPUs; the C2
        # replica numbers stay beside it
        sp = (sharded or {}).get("pfbto_jacobi", {})
        line["c2_replicas"] = {"value": ms, "ms_per_iter_hot": hot_ms, "e2e": line["e2e"],
                               "workload": WORKLOAD + f", one independent replica per GPU"}
        line.update({
            "value": sp.get("ms_per_iter"), "ms_per_step": sp.get("ms_per_iter"),
            "scaling": "strong",
            "config": {"workload": C5_SHARDED, "algorithm": "pfbto_jacobi",
                       "flush": "inputs 23 GB per iteration >> L2",
                       "parallelism": f"row slabs x{world} (NCCL halo exchange + all-gathers)",
                       "cuda_graphs": sp.get("graphs")},
            "e2e": {"value": sp.get("e2e_ms_per_iter"), "unit": UNIT, "h2d_bytes_per_step": 8,
                    "d2h_bytes_per_step": 32,
                    "path": "public run(problem, SolverConfig(pfbto_jacobi), slabs='nccl') on "
                            "every rank: (T(W+K) - T(W)) / K of two wall-clock runs (set-up and "
                            "the final gathered state cancel); alpha_k in, record row out per "
                            "step"},
            "gpu_launches": 6 * K,
            "clocks": shard_clocks,
        })
        if sp.get("ms_per_iter") is None:
            line["error"] = "row-slab C5 failed: " + json.dumps(sp)[:300]
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C1/C3/C4/C5 sweep")
    ap.add_argument("--force-sharded", action="store_true",
                    help="at N = 1 time all four slab algorithms at C5 (default: pfbto only)")
    ap.add_argument("--no-sharded", action="store_true",
                    help="at N = 1 skip the one-rank C5 row-slab point")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = dist_env()
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return
    b200_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
