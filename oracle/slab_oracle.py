"""CPU ORACLE — TEST INFRASTRUCTURE ONLY — row-slab emulation over torch.distributed.

This restates the slab-decomposed outer iteration of
`paper_2204_06204_b200/csrc/distributed.cu` in numpy.  Each
rank is a process running on the gloo backend.  Every rank holds only its
window rows and runs the global oracle kernels (`bisimp_oracle`) on its
window, embedded in a zero grid.  The rows just outside the window read zero,
as in the CUDA kernels, so owned rows come out exact only when the halos are
right.  Halos move with point-to-point send/recv.  Scalars are all-gathered
and summed in rank order.

The decomposition logic under test is product code: `slab_rows`,
`owned_node_rows`, `halo_rows` and `halo_plan` from
`paper_2204_06204_b200.distributed`.  The test compares the record rows
against the global oracle loop (`bisimp_oracle.run_loop`).  That loop is
itself pinned to the reference goldens.

Low-level step: pfbto_jacobi (solvers.py:275-278) or fbto (273-274).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import bisimp_oracle as O


def _exchange(arr, plan, rank, world):
    """Fill arr's halo rows from the neighbours (arr: rows-first window array)."""
    reqs, bufs = [], []
    if rank > 0:
        a, b = plan["send_up"]
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[a:b])), rank - 1))
        a, b = plan["recv_up"]
        buf = torch.empty(arr[a:b].shape, dtype=torch.float64)
        reqs.append(dist.irecv(buf, rank - 1))
        bufs.append((a, b, buf))
    if rank + 1 < world:
        a, b = plan["send_dn"]
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr[a:b])), rank + 1))
        a, b = plan["recv_dn"]
        buf = torch.empty(arr[a:b].shape, dtype=torch.float64)
        reqs.append(dist.irecv(buf, rank + 1))
        bufs.append((a, b, buf))
    for r in reqs:
        r.wait()
    for a, b, buf in bufs:
        arr[a:b] = buf.numpy()


def _gather(vals, world):
    """All-gather a small vector of partials; returns [world, len] (rank order)."""
    t = torch.tensor(np.asarray(vals, dtype=np.float64))
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.stack([o.numpy() for o in out])


def _lambda(gsum, w_own, act_own, lo, hi, budget, guess, wmax, world):
    """Regime-Newton lambda search over the slabs (highlevel.cu / distributed.cu)."""
    L, U = 0.0, wmax - lo
    lam = guess if L < guess < U else 0.5 * (L + U)
    wa = w_own[act_own]
    for _ in range(200):
        d = wa - lam
        mlo, mhi = d <= lo, d >= hi
        mid = ~mlo & ~mhi
        part = _gather([wa[mid].sum(), mid.sum(), mlo.sum(), mhi.sum()], world)
        smid, nmid, nlo, nhi = (float(sum(part[r, i] for r in range(world))) for i in range(4))
        f = smid - nmid * lam + nlo * lo + nhi * hi
        if f > budget:
            L = lam
        else:
            U = lam
        if nmid > 0:
            root = (smid + nlo * lo + nhi * hi - budget) / nmid
            if abs(root - lam) <= 1e-15 * max(1.0, abs(lam)):
                lam = root if L < root < U else lam
                break
            nxt = root if L < root < U else 0.5 * (L + U)
        else:
            nxt = 0.5 * (L + U)
        if not (U - L > 0) or nxt == lam:
            lam = U if f > budget else lam
            break
        lam = nxt
    return max(lam, 0.0)


def run_slab_loop(spec, algorithm, iters, rank, world, eta=3.0, size=7, sigma=1.5, v_lo=0.1):
    """Record rows (compliance, residual_inf, dv_inf, volume) of `iters` iterations."""
    from paper_2204_06204_b200.distributed import halo_plan, halo_rows, owned_node_rows, slab_rows
    nx, ny = spec.nx, spec.ny
    g = O.build_grid(nx, ny, spec.fixtures, spec.loads)
    passive = spec.passive_mask()
    v_glob, active, budget, beta = O.setup(g, nx, ny, spec.volume_fraction, v_lo, passive,
                                           algorithm, eta, size, sigma)
    act_glob = np.ones(nx * ny, bool) if active is None else active
    n_active = float(act_glob.sum())
    H = halo_rows(size)
    r_f = size // 2
    e0, e1, w0, w1 = slab_rows(ny, world, rank, H)
    n0, n1 = owned_node_rows(ny, world, rank)
    own = slice(e0 - w0, e1 - w0)
    nown = slice(n0 - w0, n1 - w0)
    v = v_glob.reshape(ny, nx)[w0:w1].copy()        # window element rows
    act = act_glob.reshape(ny, nx)[w0:w1]
    u = np.zeros((w1 - w0 + 1, nx + 1, 2))           # window node rows
    fixed = g.fixed.reshape(ny + 1, nx + 1, 2)[w0:w1 + 1]
    load_ = g.load.reshape(ny + 1, nx + 1, 2)[w0:w1 + 1]

    def embed_e(x):
        full = np.zeros((ny, nx))
        full[w0:w1] = x
        return full.ravel()

    def embed_n(x):
        full = np.zeros((ny + 1, nx + 1, 2))
        full[w0:w1 + 1] = x
        return full.ravel()

    def win_e(full):
        return full.reshape(ny, nx)[w0:w1]

    def win_n(full):
        return full.reshape(ny + 1, nx + 1, 2)[w0:w1 + 1]

    rows = []
    for k in range(1, iters + 1):
        vp = win_e(O.filter_fwd(embed_e(v), nx, ny, size, sigma))
        a = vp ** eta
        ku = win_n(O.matvec(g, embed_e(a), embed_n(u)))
        r = ku - load_
        part = _gather([float((u[nown] * ku[nown]).sum()), float(np.abs(r[nown]).max())], world)
        compliance = 0.5 * float(sum(part[i, 0] for i in range(world)))
        res_inf = float(max(part[i, 1] for i in range(world)))
        sens = eta * vp ** (eta - 1) * win_e(O.energies(g, embed_n(u)))
        _exchange(sens, halo_plan(e0, e1, w0, r_f, False), rank, world)
        gr = win_e(O.filter_adj(embed_e(sens), nx, ny, size, sigma))
        part = _gather([float(gr[own][act[own]].sum())], world)
        mean = float(sum(part[i, 0] for i in range(world))) / n_active
        if algorithm == "pfbto_jacobi":
            d = win_n(O.stiffness_diag(g, embed_e(a)))
            z = np.where(fixed, 0.0, r / d ** 2)
            _exchange(z, halo_plan(e0, e1, w0, 1, True), rank, world)
            u_next = u - beta * win_n(O.matvec(g, embed_e(a), embed_n(z)))
        else:
            u_next = u - beta * r
        alpha = 0.25 * float(k) ** -0.75 if algorithm != "fbto" else 0.001 * float(k) ** -0.75
        vo, ao = v[own], act[own]
        w = vo + alpha * (gr[own] - mean)
        clip = np.where(ao, np.clip(w, v_lo, 1.0), vo)
        part = _gather([float(clip[ao].sum()), float(w[ao].max()),
                        float(((w > v_lo) & (w < 1.0) & ao).sum())], world)
        box = float(sum(part[i, 0] for i in range(world)))
        if box > budget:
            wmax = float(max(part[i, 1] for i in range(world)))
            nmid0 = float(sum(part[i, 2] for i in range(world)))
            guess = (box - budget) / nmid0 if nmid0 > 0 else -1.0
            lam = _lambda(mean, w, ao, v_lo, 1.0, budget, guess, wmax, world)
            clip = np.where(ao, np.clip(w - lam, v_lo, 1.0), vo)
        part = _gather([float(np.abs(clip - vo).max()), float(vo.sum())], world)
        dv = float(max(part[i, 0] for i in range(world)))
        vol = float(sum(part[i, 1] for i in range(world)))
        rows.append((compliance, res_inf, dv, vol))
        v_next = v.copy()
        v_next[own] = clip
        _exchange(v_next, halo_plan(e0, e1, w0, H, False), rank, world)
        _exchange(u_next, halo_plan(e0, e1, w0, 1, True), rank, world)
        u, v = u_next, v_next
    return rows
