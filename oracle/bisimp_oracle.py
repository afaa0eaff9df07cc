"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A from-scratch numpy/scipy restatement of the per-iteration hot path of the
reference package `bisimp` (arXiv 2204.06204, `/root/reference/pkg/src/bisimp`).
Every function cites the reference file:line whose behaviour it restates.

Who may import this module: `tests/`, `__graft_entry__.smoke()` (as the
checker) and `bench.py` (the `cpu_baseline` leg and `--impl reference`).
The product package `paper_2204_06204_b200` never imports it; its compute
path is the CUDA library and fails loudly when that library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
the real reference in this container (`tests/golden/make_golden.py` →
`tests/golden/*.npz`, test `tests/test_oracle_golden.py`).

The numerical primitives deliberately match the reference's third-party
calls (numpy 2.x / scipy 1.1x, versions unpinned upstream:
`pkg/pyproject.toml:10-15`) so that the CPU timing beside the GPU numbers is
representative of the reference: `np.bincount` scatter-add, BLAS `(E,8)@(8,8)`,
`scipy.ndimage.correlate1d`, LAPACK `geqrf/ormqr/trtrs`, stable argsort.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg
from scipy.ndimage import correlate1d

# --------------------------------------------------------------------------
# grid model (fea.py)
# --------------------------------------------------------------------------


def q4_stiffness(young: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """Unit-square bilinear quad, plane stress, 2x2 Gauss (fea.py:61-87).

    Local nodes (0,0),(1,0),(1,1),(0,1); DOFs interleaved (ux, uy)."""
    c = young / (1.0 - nu * nu)
    dmat = c * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, 0.5 * (1.0 - nu)]])
    out = np.zeros((8, 8))
    pts = (0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0))
    for xi in pts:
        for eta in pts:
            gx = np.array([eta - 1.0, 1.0 - eta, eta, -eta])
            gy = np.array([xi - 1.0, -xi, xi, 1.0 - xi])
            bm = np.zeros((3, 8))
            bm[0, 0::2] = gx
            bm[1, 1::2] = gy
            bm[2, 0::2] = gy
            bm[2, 1::2] = gx
            out += 0.25 * (bm.T @ dmat @ bm)
    return out


def element_dofs(nx: int, ny: int) -> np.ndarray:
    """(E,8) global DOF table, element e = ey*nx+ex, node = y*(nx+1)+x (fea.py:90-101)."""
    ey, ex = np.divmod(np.arange(nx * ny), nx)
    n0 = ey * (nx + 1) + ex
    corners = np.stack([n0, n0 + 1, n0 + nx + 2, n0 + nx + 1], axis=1)
    table = np.empty((nx * ny, 8), dtype=np.int64)
    table[:, 0::2] = 2 * corners
    table[:, 1::2] = 2 * corners + 1
    return table


class Grid:
    """Plain container for the oracle (mirrors fea.GridModel fields, fea.py:104-143)."""

    def __init__(self, nx, ny, ke, fixed, load):
        self.nx, self.ny = int(nx), int(ny)
        self.ke = np.asarray(ke, dtype=float)
        self.fixed = np.asarray(fixed, dtype=bool)
        self.load = np.asarray(load, dtype=float)
        self.edof = element_dofs(self.nx, self.ny)
        self.n_dofs = 2 * (self.nx + 1) * (self.ny + 1)
        self.n_elem = self.nx * self.ny

    @classmethod
    def from_model(cls, model):
        return cls(model.nx, model.ny, model.ke, model.fixed_dofs, model.load)


def matvec(grid: Grid, a: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Masked K(a)u: gather, (E,8)@ke, scale by a, bincount scatter (fea.py:150-181)."""
    um = u.copy()
    um[grid.fixed] = 0.0
    local = (um[grid.edof] @ grid.ke) * a[:, None]
    y = np.bincount(grid.edof.ravel(), weights=local.ravel(), minlength=grid.n_dofs)
    y[grid.fixed] = 0.0
    return y


def stiffness_diag(grid: Grid, a: np.ndarray) -> np.ndarray:
    """diag K(a) with 1 on fixed DOFs (fea.py:184-189)."""
    w = a[:, None] * np.diag(grid.ke)[None, :]
    d = np.bincount(grid.edof.ravel(), weights=w.ravel(), minlength=grid.n_dofs)
    d[grid.fixed] = 1.0
    return d


def energies(grid: Grid, u: np.ndarray) -> np.ndarray:
    """Per-element ½ u_eᵀ ke u_e, fixed DOFs of u read as 0 (fea.py:197-201)."""
    um = np.where(grid.fixed, 0.0, u)
    ue = um[grid.edof]
    return 0.5 * np.einsum("ei,ei->e", ue @ grid.ke, ue)


def power_rho(grid: Grid, a: np.ndarray, iters: int, seed: int = 0) -> float:
    """Seeded power iteration, Rayleigh quotient (fea.py:278-301)."""
    x = np.random.default_rng(seed).standard_normal(grid.n_dofs)
    x[grid.fixed] = 0.0
    x = x / np.linalg.norm(x)
    rho = 0.0
    for _ in range(iters):
        y = matvec(grid, a, x)
        rho = float(x @ y)
        nrm = np.linalg.norm(y)
        if nrm == 0.0:
            break
        x = y / nrm
    return rho


# --------------------------------------------------------------------------
# density filter (filtering.py)
# --------------------------------------------------------------------------


def gauss_taps(size: int, sigma: float) -> np.ndarray:
    """Normalised 1-D Gaussian taps (filtering.py:30-35)."""
    r = size // 2
    t = np.exp(-0.5 * (np.arange(-r, r + 1, dtype=float) / sigma) ** 2)
    return t / t.sum()


def _mass(length: int, taps: np.ndarray) -> np.ndarray:
    # in-range kernel mass per index, zero padding (filtering.py:38-43)
    return correlate1d(np.ones(length), taps, mode="constant", cval=0.0)


def filter_fwd(field, nx, ny, size=7, sigma=1.5):
    """C(v): x-correlate / sx, then y-correlate / sy (filtering.py:46-55)."""
    taps = gauss_taps(size, sigma)
    img = field.reshape(ny, nx)
    img = correlate1d(img, taps, axis=1, mode="constant", cval=0.0) / _mass(nx, taps)[None, :]
    img = correlate1d(img, taps, axis=0, mode="constant", cval=0.0) / _mass(ny, taps)[:, None]
    return img.ravel()


def filter_adj(field, nx, ny, size=7, sigma=1.5):
    """Cᵀ s: /sy, y-correlate, /sx, x-correlate (filtering.py:58-72)."""
    taps = gauss_taps(size, sigma)
    img = field.reshape(ny, nx)
    img = correlate1d(img / _mass(ny, taps)[:, None], taps, axis=0, mode="constant", cval=0.0)
    img = correlate1d(img / _mass(nx, taps)[None, :], taps, axis=1, mode="constant", cval=0.0)
    return img.ravel()


# --------------------------------------------------------------------------
# bounded-simplex projection (projection.py)
# --------------------------------------------------------------------------


def _bisect(v, lo, hi, budget):
    # 100 halvings on [0, max(v)-lo] (projection.py:38-47)
    left, right = 0.0, float(v.max() - lo)
    for _ in range(100):
        mid = 0.5 * (left + right)
        if np.clip(v - mid, lo, hi).sum() > budget:
            left = mid
        else:
            right = mid
    return right


def project(v, lo, hi, budget):
    """argmin ½‖x−v‖² s.t. lo≤x≤hi, Σx≤budget (projection.py:50-91).

    Box early exit; otherwise breakpoint sort + slope sweep, with the
    reference's two bisection fallbacks."""
    n = v.size
    if not (0.0 < lo < hi):
        raise ValueError("need 0 < lo < hi")
    if not (n * lo <= budget <= n * hi):
        raise ValueError("infeasible budget")
    box = np.clip(v, lo, hi)
    if box.sum() <= budget:
        return box
    pts = np.concatenate([v - hi, v - lo])
    step = np.concatenate([np.full(n, -1.0), np.full(n, 1.0)])
    order = np.argsort(pts, kind="stable")
    pts = pts[order]
    slope = np.cumsum(step[order])
    total = n * hi + np.concatenate([[0.0], np.cumsum(slope[:-1] * np.diff(pts))])
    lam = None
    hit = np.flatnonzero(total <= budget)
    if hit.size and hit[0] > 0:
        j = int(hit[0])
        if slope[j - 1] < 0:
            lam = pts[j - 1] + (total[j - 1] - budget) / (-slope[j - 1])
    if lam is None or lam < 0:
        lam = _bisect(v, lo, hi, budget)
    out = np.clip(v - lam, lo, hi)
    if abs(out.sum() - budget) > 1e-7:
        out = np.clip(v - _bisect(v, lo, hi, budget), lo, hi)
    return out


# --------------------------------------------------------------------------
# solver pieces (solvers.py)
# --------------------------------------------------------------------------


def sensitivity(grid, v_phys, u, eta, size=7, sigma=1.5):
    """Cᵀ(η v_phys^(η−1) ⊙ energies) (solvers.py:181-190)."""
    s = eta * v_phys ** (eta - 1.0) * energies(grid, u)
    return filter_adj(s, grid.nx, grid.ny, size, sigma)


_GEQRF, _ORMQR, _TRTRS = scipy.linalg.get_lapack_funcs(("geqrf", "ormqr", "trtrs"),
                                                       (np.zeros(1),))


def lstsq_householder(cols: np.ndarray, b: np.ndarray) -> np.ndarray:
    """min‖b − cols·c‖ via LAPACK geqrf/ormqr/trtrs with the 1e-13 rank cut
    (solvers.py:205-219)."""
    k = cols.shape[1]
    fact, tau, _, _ = _GEQRF(np.asfortranarray(cols))
    qtb, _, _ = _ORMQR("L", "T", fact, tau, np.asfortranarray(b.reshape(-1, 1)),
                       lwork=max(64, 8 * k))
    rdiag = np.abs(np.diag(fact[:k, :k]))
    tiny = rdiag <= 1e-13 * rdiag[0]
    rank = int(np.argmax(tiny)) if tiny.any() else k
    c = np.zeros(k)
    if rank:
        sol, _ = _TRTRS(fact[:rank, :rank], qtb[:rank])
        c[:rank] = sol.ravel()
    return c


def krylov(grid, a, b, dim, return_parts=False):
    """Least-squares Krylov polynomial applied to b (solvers.py:222-255)."""
    if dim < 1:
        raise ValueError("Krylov dimension must be at least 1")
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b)
    npow = min(dim + 1, b.size)
    basis = np.empty((b.size, npow + 1), order="F")
    basis[:, 0] = b / nb
    growth = np.empty(npow)
    used = 0
    for i in range(npow):
        t = matvec(grid, a, basis[:, i])
        m = np.linalg.norm(t)
        if m == 0.0:
            break
        basis[:, i + 1] = t / m
        growth[i] = m
        used += 1
    if used == 0:
        return np.zeros_like(b)
    coeff = lstsq_householder(basis[:, 1:used + 1].copy(order="F"), b)
    out = basis[:, :used] @ (coeff / growth[:used])
    if return_parts:
        return out, coeff, growth[:used]
    return out


def low_level(grid, a, u, algorithm, beta, residual=None, dim=20):
    """One damped displacement update (solvers.py:258-281)."""
    r = matvec(grid, a, u) - grid.load if residual is None else residual
    if algorithm == "fbto":
        return u - beta * r
    if algorithm == "pfbto_jacobi":
        d = stiffness_diag(grid, a)
        return u - beta * matvec(grid, a, r / d ** 2)
    if algorithm == "cpfbto_krylov":
        return u - beta * krylov(grid, a, r, dim)
    raise ValueError(f"no low-level step for {algorithm!r}")


def high_level(v, g, alpha, lo, hi, budget, active=None, mean_projection=True):
    """Projected ascent with optional mean removal; passive pinned (solvers.py:284-302)."""
    if active is None:
        step = g - g.mean() if mean_projection else g
        return project(v + alpha * step, lo, hi, budget)
    ga = g[active]
    if mean_projection:
        ga = ga - ga.mean()
    out = v.copy()
    out[active] = project(v[active] + alpha * ga, lo, hi, budget)
    return out


def sq_jacobi_rho(grid, v, eta, size, sigma, seed, iters=50):
    """Power iteration on K M⁻² K at the initial design (solvers.py:348-364)."""
    a = filter_fwd(v, grid.nx, grid.ny, size, sigma) ** eta
    d2 = stiffness_diag(grid, a) ** 2
    x = np.random.default_rng(seed).standard_normal(grid.n_dofs)
    x[grid.fixed] = 0.0
    x = x / np.linalg.norm(x)
    rho = 1.0
    for _ in range(iters):
        y = matvec(grid, a, matvec(grid, a, x) / d2)
        rho = float(x @ y)
        nrm = np.linalg.norm(y)
        if nrm == 0.0:
            break
        x = y / nrm
    return rho


ALPHA0 = {"fbto": 0.001, "pfbto_jacobi": 0.25, "cpfbto_krylov": 0.25, "pgd_exact": 0.25,
          # builder extensions (no reference): approx_inverse_oracle.low_level
          "pcg_jacobi": 0.25, "mg_vcycle": 0.25, "mg_pcg": 0.25}


def setup(grid, nx, ny, volume_fraction, v_lo, passive_mask, algorithm, eta,
          size, sigma, beta=None, seed=0):
    """Initial design, bounds and β (solvers.py:319-345)."""
    active = None if not passive_mask.any() else ~passive_mask
    n_act = nx * ny if active is None else int(active.sum())
    budget = volume_fraction * n_act
    v = np.full(nx * ny, v_lo)
    level = min(max(volume_fraction, v_lo), 1.0)
    if active is None:
        v[:] = level
    else:
        v[active] = level
    if beta is None:
        if algorithm == "fbto":
            beta = 1.0 / power_rho(grid, np.ones(nx * ny), 50, seed)
        elif algorithm == "pfbto_jacobi":
            beta = 1.0 / sq_jacobi_rho(grid, v, eta, size, sigma, seed)
        else:
            beta = 1.0
    return v, active, budget, beta


def iterate(grid, v, u, k, *, algorithm, eta, size, sigma, beta, alpha0, m,
            lo, budget, active, mean_projection=True, dim=20, low_level_fn=None):
    """One outer iteration k of the run() loop body (solvers.py:442-466).

    Returns (u_next, v_next, record_row, v_phys, a) where record_row is
    (compliance, residual_inf, dv_inf, volume) measured at (u, v)."""
    v_phys = filter_fwd(v, grid.nx, grid.ny, size, sigma)
    a = v_phys ** eta
    r = matvec(grid, a, u) - grid.load
    res_inf = float(np.abs(r).max())
    compliance = 0.5 * float(u @ (r + grid.load))
    if not (np.isfinite(res_inf) and np.isfinite(compliance)):
        raise FloatingPointError(f"non-finite iterate at iteration {k}")
    g = sensitivity(grid, v_phys, u, eta, size, sigma)
    if low_level_fn is not None:  # builder extensions (approx_inverse_oracle)
        u_next = low_level_fn(grid, a, u, r)
    else:
        u_next = low_level(grid, a, u, algorithm, beta, residual=r, dim=dim)
    alpha_k = alpha0 * float(k) ** (-m)
    v_next = high_level(v, g, alpha_k, lo, 1.0, budget, active, mean_projection)
    dv = float(np.abs(v_next - v).max())
    return u_next, v_next, (compliance, res_inf, dv, float(v.sum())), v_phys, a


def run_loop(grid, *, nx, ny, volume_fraction, v_lo=0.1, eta=3.0, size=7, sigma=1.5,
             passive_mask=None, algorithm="cpfbto_krylov", alpha0=None, m=0.75,
             beta=None, dim=20, max_iters=100, tol_dv=1e-4, tol_res=1e-2, seed=0,
             mean_projection=True, low_level_fn=None):
    """The run() outer loop without control/sink plumbing (solvers.py:381-484)."""
    if passive_mask is None:
        passive_mask = np.zeros(nx * ny, dtype=bool)
    alpha0 = ALPHA0[algorithm] if alpha0 is None else alpha0
    v, active, budget, beta = setup(grid, nx, ny, volume_fraction, v_lo, passive_mask,
                                    algorithm, eta, size, sigma, beta, seed)
    u = np.zeros(grid.n_dofs)
    rows = []
    reason = "budget"
    last = None
    for k in range(1, max_iters + 1):
        u_next, v_next, row, v_phys, a = iterate(
            grid, v, u, k, algorithm=algorithm, eta=eta, size=size, sigma=sigma, beta=beta,
            alpha0=alpha0, m=m, lo=v_lo, budget=budget, active=active,
            mean_projection=mean_projection, dim=dim, low_level_fn=low_level_fn)
        rows.append((k,) + row)
        last = (k, u, v, v_phys, a)
        u, v = u_next, v_next
        if row[2] < tol_dv and row[1] < tol_res:
            reason = "converged"
            break
    return {"rows": rows, "reason": reason, "last": last, "beta": beta,
            "u_next": u, "v_next": v}


# --------------------------------------------------------------------------
# problem setup (problems.py) — used to build oracle grids from specs
# --------------------------------------------------------------------------


def selector_nodes(sel: dict, nx: int, ny: int) -> np.ndarray:
    """Edge/point selector → node ids (problems.py:48-71; Python round())."""
    if "edge" in sel:
        a, b = sel.get("span", (0.0, 1.0))
        edge = sel["edge"]
        length = ny if edge in ("left", "right") else nx
        k = np.arange(round(a * length), round(b * length) + 1)
        return {"left": k * (nx + 1), "right": k * (nx + 1) + nx,
                "top": k, "bottom": ny * (nx + 1) + k}[edge]
    rx, ry = sel["point"]
    return np.array([round(ry * ny) * (nx + 1) + round(rx * nx)])


def build_grid(nx, ny, fixtures, loads, young=1.0, nu=0.3) -> Grid:
    """Fixed mask + 2-norm-normalised load (problems.py:138-164)."""
    n = 2 * (nx + 1) * (ny + 1)
    fixed = np.zeros(n, dtype=bool)
    for sel in fixtures:
        nodes = selector_nodes(sel, nx, ny)
        dofs = sel.get("dofs", "xy")
        if "x" in dofs:
            fixed[2 * nodes] = True
        if "y" in dofs:
            fixed[2 * nodes + 1] = True
    f = np.zeros(n)
    for sel in loads:
        nodes = selector_nodes(sel, nx, ny)
        f[2 * nodes] += sel.get("fx", 0.0) / nodes.size
        f[2 * nodes + 1] += sel.get("fy", 0.0) / nodes.size
    f[fixed] = 0.0
    f /= np.linalg.norm(f)
    return Grid(nx, ny, q4_stiffness(young, nu), fixed, f)


def passive_mask(nx, ny, rects) -> np.ndarray:
    """Element mask of passive rectangles (problems.py:123-130)."""
    m = np.zeros((ny, nx), dtype=bool)
    for (x0, y0, x1, y1) in rects:
        m[round(y0 * ny):round(y1 * ny), round(x0 * nx):round(x1 * nx)] = True
    return m.ravel()


# --------------------------------------------------------------------------
# density frames

def pgm_bytes(v_phys: np.ndarray, nx: int, ny: int) -> bytes:
    """Binary PGM of a density field (outputs.py:21-30): header
    "P5\\n{nx} {ny}\\n255\\n", pixel = round-half-up of 255·(1 − v), solid black."""
    v = np.asarray(v_phys, dtype=np.float64)
    if v.shape != (nx * ny,):
        raise ValueError(f"field has length {v.shape}, expected {nx * ny}")
    if v.min() < 0.0 or v.max() > 1.0:
        raise ValueError("density values must lie in [0, 1]")
    scaled = np.multiply(255.0, np.subtract(1.0, v))
    pix = np.floor(np.add(scaled, 0.5)).astype(np.uint8)
    return f"P5\n{nx} {ny}\n255\n".encode("ascii") + pix.tobytes()


def frame_payload(v_phys: np.ndarray) -> bytes:
    """Service frame payload: row-major little-endian float32 of v_phys
    (service/sessions.py:97), numpy's round-to-nearest-even cast."""
    with np.errstate(over="ignore"):
        return np.asarray(v_phys, dtype=np.float64).astype("<f4").tobytes()
