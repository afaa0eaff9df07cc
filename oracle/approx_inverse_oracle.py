"""CPU ORACLE — TEST INFRASTRUCTURE ONLY — for the approximate inverses that
have NO reference implementation (SURVEY §8(a')).

The reference package has no PCG or multigrid low-level step (`SPEC.md:353`
lists multigrid as a non-goal).  The north star still asks for both.  SURVEY
§8(a') grades them by:
(1) this numpy restatement of the builder's algorithm, at 1e-10 per CG step or
    per V-cycle;
(2) energy monotonicity at a fixed design (the `tests/test_solvers.py:203-217`
    pattern);
(3) converged compliance within 5% of `pgd_exact` (`test_acceptance.py:198-226`).

Parity status: **unpinned to the reference** (nothing exists to pin against).
The restatement shares no code with the CUDA path.  The K(a) products go
through `bisimp_oracle.matvec`, which is itself pinned to the reference's
`apply_stiffness` goldens.

Algorithm (must match `include/bisimp_b200.h` bsp_mg_* / bsp_pcg_apply):
* levels: level l+1 has ceil(nx_l/2) x ceil(ny_l/2) elements.  Coarsen while
  (nx+1)(ny+1) > 40 nodes and the grid is larger than 1x1, up to
  `max_levels` levels in total (0 means 24).
* coarse activation: the mean of the 4 children; virtual children outside the
  grid count as 0.
* coarse fixed mask: a DOF is fixed iff a fine DOF of the same component at
  (2X+dx, 2Y+dy), dx, dy in {-1, 0, 1}, is fixed.
* P: masked bilinear interpolation.  R = P^T.
* smoother: damped Jacobi with weight omega, nu sweeps before and nu after.
  The first pre-sweep starts from zero.
* coarsest level: dense direct solve, with fixed DOFs as identity rows.
* PCG: `steps` iterations from x = 0.  alpha = rz/pKp (0 if either is <= 0);
  steps = 0 returns M b.
"""
from __future__ import annotations

import numpy as np

from . import bisimp_oracle as O

COARSE_NODES = 40
MAX_LEVELS = 24


class Level:
    def __init__(self, nx, ny, ke, fixed):
        self.nx, self.ny = int(nx), int(ny)
        self.grid = O.Grid(nx, ny, ke, fixed, np.zeros(fixed.size))
        self.fixed = self.grid.fixed


def hierarchy(nx, ny, ke, fixed, max_levels=0):
    """Levels 0..L (level 0 = the given grid)."""
    if max_levels < 1:
        max_levels = MAX_LEVELS
    max_levels = min(max_levels, MAX_LEVELS)
    levels = [Level(nx, ny, ke, np.asarray(fixed, bool))]
    while (len(levels) < max_levels and (nx + 1) * (ny + 1) > COARSE_NODES
           and (nx > 1 or ny > 1)):
        cx, cy = (nx + 1) // 2, (ny + 1) // 2
        fine = levels[-1].fixed.reshape(ny + 1, nx + 1, 2)
        coarse = np.zeros((cy + 1, cx + 1, 2), bool)
        Y, X = np.arange(cy + 1), np.arange(cx + 1)
        for dy in (-1, 0, 1):
            y = 2 * Y + dy
            vy = (y >= 0) & (y <= ny)
            for dx in (-1, 0, 1):
                x = 2 * X + dx
                vx = (x >= 0) & (x <= nx)
                coarse[np.ix_(Y[vy], X[vx])] |= fine[np.ix_(y[vy], x[vx])]
        levels.append(Level(cx, cy, ke, coarse.ravel()))
        nx, ny = cx, cy
    return levels


def coarsen_activation(a, nx, ny):
    """Mean of the 4 children, virtual children (outside the grid) = 0."""
    cx, cy = (nx + 1) // 2, (ny + 1) // 2
    A = np.zeros((2 * cy, 2 * cx))
    A[:ny, :nx] = np.asarray(a).reshape(ny, nx)
    return 0.25 * ((A[0::2, 0::2] + A[0::2, 1::2]) + (A[1::2, 0::2] + A[1::2, 1::2])).ravel()


def restrict(t, fine: Level, coarse: Level):
    """-M_c P~^T t (t = K x - b on the fine level)."""
    nx, ny, cx, cy = fine.nx, fine.ny, coarse.nx, coarse.ny
    T = np.asarray(t).reshape(ny + 1, nx + 1, 2)
    S = np.zeros((cy + 1, cx + 1, 2))
    Y, X = np.arange(cy + 1), np.arange(cx + 1)
    for dy in (-1, 0, 1):
        y = 2 * Y + dy
        vy = (y >= 0) & (y <= ny)
        wy = 1.0 if dy == 0 else 0.5
        for dx in (-1, 0, 1):
            x = 2 * X + dx
            vx = (x >= 0) & (x <= nx)
            w = wy * (1.0 if dx == 0 else 0.5)
            S[np.ix_(Y[vy], X[vx])] += w * T[np.ix_(y[vy], x[vx])]
    b = -S.ravel()
    b[coarse.fixed] = 0.0
    return b


def prolong(xc, fine: Level, coarse: Level):
    """M_f P~ x_c."""
    nx, ny, cx = fine.nx, fine.ny, coarse.nx
    XC = np.asarray(xc).reshape(coarse.ny + 1, cx + 1, 2)
    y, x = np.arange(ny + 1), np.arange(nx + 1)
    Y0, oy, X0, ox = y >> 1, y & 1, x >> 1, x & 1
    w = np.outer(np.where(oy == 1, 0.5, 1.0), np.where(ox == 1, 0.5, 1.0))[:, :, None]
    out = np.zeros((ny + 1, nx + 1, 2))
    for iy in (0, 1):
        for ix in (0, 1):
            take = np.outer(iy <= oy, ix <= ox)[:, :, None]
            yy = np.minimum(Y0 + iy, coarse.ny)
            xx = np.minimum(X0 + ix, cx)
            out += np.where(take, w * XC[np.ix_(yy, xx)], 0.0)
    out = out.ravel()
    out[fine.fixed] = 0.0
    return out


def dense_operator(level: Level, a):
    """Dense masked K(a) with identity rows/cols on fixed DOFs."""
    n = level.grid.n_dofs
    K = np.zeros((n, n))
    ke = level.grid.ke
    for e, dofs in enumerate(level.grid.edof):
        K[np.ix_(dofs, dofs)] += a[e] * ke
    f = level.fixed
    K[f, :] = 0.0
    K[:, f] = 0.0
    K[f, f] = 1.0
    return K


def jacobi_sweep(level: Level, a, b, x, omega):
    d = O.stiffness_diag(level.grid, a)
    return x - omega * (O.matvec(level.grid, a, x) - b) / d


def vcycle(levels, acts, b, omega=0.6, nu=2, coarse_inverse=None):
    """x = V(b); acts[l] = activation of level l; b zero on fixed DOFs."""
    L = len(levels) - 1
    if coarse_inverse is None:
        coarse_inverse = np.linalg.inv(dense_operator(levels[L], acts[L]))

    def cycle(l, b):
        lev = levels[l]
        if l == L:
            return coarse_inverse @ b
        d = O.stiffness_diag(lev.grid, acts[l])
        x = omega * b / d
        x[lev.fixed] = 0.0
        for _ in range(nu - 1):
            x = jacobi_sweep(lev, acts[l], b, x, omega)
        t = O.matvec(lev.grid, acts[l], x) - b
        xc = cycle(l + 1, restrict(t, lev, levels[l + 1]))
        x = x + prolong(xc, lev, levels[l + 1])
        for _ in range(nu):
            x = jacobi_sweep(lev, acts[l], b, x, omega)
        return x

    return cycle(0, np.asarray(b, float))


def activations(levels, a):
    acts = [np.asarray(a, float)]
    for l in range(1, len(levels)):
        acts.append(coarsen_activation(acts[-1], levels[l - 1].nx, levels[l - 1].ny))
    return acts


def pcg(grid: O.Grid, a, b, steps, levels=None, omega=0.6, nu=2, history=False):
    """`steps` PCG iterations from 0 on K(a)x = b; Jacobi if levels is None.

    Returns x (and the list of ||r_j|| if history)."""
    b = np.where(grid.fixed, 0.0, np.asarray(b, float))
    if levels is not None:
        acts = activations(levels, a)
        cinv = np.linalg.inv(dense_operator(levels[-1], acts[-1]))
        prec = lambda r: vcycle(levels, acts, r, omega, nu, cinv)  # noqa: E731
    else:
        d = O.stiffness_diag(grid, a)
        prec = lambda r: r / d  # noqa: E731
    z = prec(b)
    if steps == 0:
        return (z, []) if history else z
    x = np.zeros_like(b)
    r = b.copy()
    p = z.copy()
    rz = float(r @ z)
    hist = [float(np.linalg.norm(r))]
    for j in range(steps):
        q = O.matvec(grid, a, p)
        pq = float(p @ q)
        alpha = rz / pq if (pq > 0 and rz > 0) else 0.0
        x = x + alpha * p
        r = r - alpha * q
        hist.append(float(np.linalg.norm(r)))
        if j == steps - 1:
            break
        z = prec(r)
        rz_new = float(r @ z)
        beta = rz_new / rz if (rz > 0 and rz_new > 0) else 0.0
        rz = rz_new
        p = z + beta * p
    return (x, hist) if history else x


def low_level(grid: O.Grid, a, u, algorithm, beta=1.0, residual=None, steps=None, omega=0.6,
              nu=2, max_levels=0):
    """u - beta M~^{-1} r for pcg_jacobi / mg_vcycle / mg_pcg."""
    r = residual if residual is not None else O.matvec(grid, a, u) - grid.load
    if algorithm == "pcg_jacobi":
        return u - beta * pcg(grid, a, r, 20 if steps is None else steps)
    levels = hierarchy(grid.nx, grid.ny, grid.ke, grid.fixed, max_levels)
    if algorithm == "mg_vcycle":
        return u - beta * pcg(grid, a, r, 0, levels, omega, nu)
    if algorithm == "mg_pcg":
        return u - beta * pcg(grid, a, r, 4 if steps is None else steps, levels, omega, nu)
    raise ValueError(algorithm)
