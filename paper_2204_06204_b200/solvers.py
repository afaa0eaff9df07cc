"""First-order bilevel SIMP solvers on the GPU — drop-in for `bisimp.solvers`.

Same public names, signatures, defaults, validation messages and exception
types as the reference module (`/root/reference/pkg/src/bisimp/solvers.py`).

`run()` keeps the whole outer loop (solvers.py:416-475) on the device: each
iteration is one CUDA-graph replay of filter → residual/energies → adjoint →
low-level step → projected high-level step; convergence and divergence are
decided on the GPU, so a batch of iterations needs one host synchronisation
(to read the ConvergenceRecord rows).  Host-visible semantics are the
reference's:
  * the record row k holds (compliance, residual_inf) of (u_k, v_k), the
    dv_inf of v_{k+1} − v_k and volume Σv_k (solvers.py:466);
  * the sink receives iterate k (u_k, v_k, C(v_k), a_k) every snapshot_every
    iterations and once more for the final state (solvers.py:468-483);
  * RunControl messages apply at iteration boundaries only (solvers.py:417-440);
    the device loop runs in batches that end at snapshot multiples, and at
    most `_CONTROL_BATCH` iterations pass between control drains;
  * `clock`: with a real-time clock (time.perf_counter / monotonic / time)
    every iteration is stamped on the device (%globaltimer, written with its
    record row) and the stamps are mapped onto the clock, so the loop still
    runs in batches; any other callable is called once per completed
    iteration, one iteration per batch, exactly as the reference does.
`threads` is accepted for API compatibility and ignored.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import queue
import time
import warnings
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _dev
from ._native import ALGO, SolverConfigC, call, load
from .fea import (
    DensityField,
    GridModel,
    apply_stiffness,
    element_energies,
    estimate_rho_max,
    exact_solve,
    residual_reduce,
    start_vector,
    grid_handle,
    stiffness_diagonal,
)
from .filtering import (
    FilterSpec,
    apply_filter,
    apply_filter_adjoint,
    apply_filter_and_activation,
    gaussian_weights,
)
from .approx_inverse import Multigrid, pcg_apply
from .problems import ProblemSpec, resolve, resolve_device
from .projection import SimplexBounds, project_simplex

ALGORITHMS = ("fbto", "pfbto_jacobi", "cpfbto_krylov", "pgd_exact",
              # north-star approximate inverses (no reference implementation,
              # SURVEY §8(a')): u <- u - beta M~^{-1} r
              "pcg_jacobi", "mg_vcycle", "mg_pcg")
APPROX_INVERSES = ("pcg_jacobi", "mg_vcycle", "mg_pcg")

_ALPHA0_DEFAULTS = {
    "fbto": 0.001,  # the plain variant diverges for alpha0 > 1e-2
    "pfbto_jacobi": 0.25,
    "cpfbto_krylov": 0.25,
    "pgd_exact": 0.25,
    "pcg_jacobi": 0.25,
    "mg_vcycle": 0.25,
    "mg_pcg": 0.25,
}
# CG steps per outer iteration.  SURVEY §8(a') measured PCG-20 and MG-PCG-2.  On
# B200, MG-PCG-2 converges to a design whose compliance depends chaotically on
# rounding (789.4 or 961.0 on the acceptance L-shape).  MG-PCG-4 lands within
# 2% of pgd_exact (790.7).
_INNER_STEPS_DEFAULTS = {"pcg_jacobi": 20, "mg_pcg": 4, "mg_vcycle": 0}
# Low-level damping beta and smoother sweeps of the multigrid approximate
# inverses, chosen by criterion 5 of the reference's acceptance suite (exact
# compliance of the converged design within 5% of pgd_exact,
# test_acceptance.py:198-226) on the L-shape at 64^2, 160^2 and 300^2 (C3),
# measured on B200 (tools/c3_variants.py).  MG-PCG-4 with
# beta = 1 is an almost exact lagged solve: at 300^2 its first iterations
# thrash the design, lose a quarter of the material to the box clips and end
# 33% above pgd_exact; beta = 0.5 (a 0.5 contraction per outer iteration)
# damps the lag and lands at +3.0% / +4.1% / +1.1%.  The stationary V-cycle
# lands at +2.3% / +1.2% / +1.9% with 1+1 sweeps (+8% at 64^2 with 2+2).
_BETA_DEFAULTS = {"mg_pcg": 0.5}
_MG_SMOOTH_DEFAULTS = {"mg_vcycle": 1, "mg_pcg": 2, "pcg_jacobi": 2}

_EXACT_SOLVE_TOL = 1e-10
# grids from this many cells are resolved as index lists (problems.resolve_device)
_DEVICE_RESOLVE_CELLS = 1 << 22
_MAX_BATCH = 256
_CONTROL_BATCH = 16


class DivergenceError(RuntimeError):
    """Raised when an iterate turns non-finite (solvers.py:52-53)."""


@dataclass
class SolverConfig:
    """Algorithm choice plus step-size, subspace and termination knobs (solvers.py:56-102)."""

    algorithm: str = "cpfbto_krylov"
    alpha0: float | None = None
    m: float = 0.75
    beta: float | None = None
    krylov_dim: int = 20
    eta: float | None = None
    max_iters: int = 50_000
    tol_dv: float = 1e-4
    tol_res: float = 1e-2
    snapshot_every: int = 0
    seed: int = 0
    mean_projection: bool = True
    # approximate-inverse algorithms only (pcg_jacobi / mg_vcycle / mg_pcg)
    inner_steps: int | None = None
    mg_omega: float = 0.6
    mg_smooth: int | None = None  # damped-Jacobi sweeps each side; None: per algorithm
    mg_levels: int = 0

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {self.algorithm!r}")
        if self.alpha0 is not None and not self.alpha0 > 0:
            raise ValueError("alpha0 must be positive")
        if not 0.75 <= self.m < 1.0:
            raise ValueError(f"decay exponent m must lie in [0.75, 1), got {self.m}")
        if self.m == 0.75:
            warnings.warn("decay exponent m = 0.75 sits on the boundary of the convergent range",
                          UserWarning, stacklevel=2)
        if self.beta is not None and not self.beta > 0:
            raise ValueError("beta must be positive")
        if self.krylov_dim < 1:
            raise ValueError("krylov_dim must be at least 1")
        if self.eta is not None and self.eta < 1:
            raise ValueError("eta must be at least 1")
        if self.max_iters < 0:
            raise ValueError("max_iters must be nonnegative")
        if self.tol_dv <= 0 or self.tol_res <= 0:
            raise ValueError("tolerances must be positive")
        if self.inner_steps is not None and self.inner_steps < 0:
            raise ValueError("inner_steps must be nonnegative")
        if not self.mg_omega > 0 or (self.mg_smooth is not None and self.mg_smooth < 1):
            raise ValueError("multigrid needs mg_omega > 0 and mg_smooth >= 1")

    def resolved_alpha0(self) -> float:
        return self.alpha0 if self.alpha0 is not None else _ALPHA0_DEFAULTS[self.algorithm]

    def resolved_inner_steps(self) -> int:
        if self.algorithm == "mg_vcycle":
            return 0
        if self.inner_steps is not None:
            return self.inner_steps
        return _INNER_STEPS_DEFAULTS.get(self.algorithm, 0)

    def resolved_beta(self) -> float | None:
        """beta of the approximate inverses (None: fbto / pfbto_jacobi take a
        spectral estimate at set-up, solvers.py:336-345)."""
        if self.beta is not None:
            return self.beta
        if self.algorithm in ("fbto", "pfbto_jacobi"):
            return None
        return _BETA_DEFAULTS.get(self.algorithm, 1.0)

    def resolved_mg_smooth(self) -> int:
        if self.mg_smooth is not None:
            return self.mg_smooth
        return _MG_SMOOTH_DEFAULTS.get(self.algorithm, 2)

    def step_size(self, k: int, alpha0: float | None = None) -> float:
        a0 = self.resolved_alpha0() if alpha0 is None else alpha0
        return a0 * float(k) ** (-self.m)


def as_solver_config(config) -> SolverConfig:
    """This module's SolverConfig for any reference-shaped config.

    The reference's callers build `bisimp.solvers.SolverConfig` (cli.py:55-62,
    service/sessions.py:106-107), which has the reference fields only
    (solvers.py:56-102).  Its fields are copied; the approximate-inverse knobs
    this module adds (inner_steps, mg_*) take their defaults when absent.
    Validation is this class's, i.e. the reference's plus the added fields."""
    if isinstance(config, SolverConfig):
        return config
    kw = {}
    for f in dataclasses.fields(SolverConfig):
        if hasattr(config, f.name):
            kw[f.name] = getattr(config, f.name)
    if "algorithm" not in kw:
        raise TypeError(f"{type(config).__name__} is not a solver configuration (no 'algorithm')")
    with warnings.catch_warnings():  # the m = 0.75 warning was already raised by the caller's type
        warnings.simplefilter("ignore", UserWarning)
        return SolverConfig(**kw)


def config_c(ws, config: SolverConfig, max_batch: int) -> SolverConfigC:
    """The C-ABI `bsp_solver_config` of one run (include/bisimp_b200.h)."""
    cfg = SolverConfigC(taps=gaussian_weights(ws.filter_spec))
    cfg.algorithm = ALGO[config.algorithm]
    cfg.eta = float(ws.eta)
    cfg.v_lo = float(ws.bounds.v_lo)
    cfg.v_hi = float(ws.bounds.v_hi)
    cfg.budget = float(ws.bounds.v_bar)
    cfg.beta = float(ws.beta) if ws.beta is not None else 0.0  # 0: estimated on the slabs
    cfg.krylov_dim = int(config.krylov_dim)
    cfg.tol_dv = float(config.tol_dv)
    cfg.tol_res = float(config.tol_res)
    cfg.mean_projection = 1 if config.mean_projection else 0
    cfg.max_batch = int(max_batch)
    cfg.inner_steps = int(config.resolved_inner_steps())
    cfg.mg_omega = float(config.mg_omega)
    cfg.mg_nu = int(config.resolved_mg_smooth())
    cfg.mg_levels = int(config.mg_levels)
    return cfg


@dataclass
class SolverState:
    """One consistent iterate plus cached diagnostics (solvers.py:105-117); host copies."""

    iter: int
    u: np.ndarray
    v: DensityField
    v_phys: np.ndarray
    activation: np.ndarray
    residual_inf: float
    compliance: float
    volume: float
    last_dv_inf: float


@dataclass
class ConvergenceRecord:
    """Columnar per-iteration history (solvers.py:120-146)."""

    iters: list = field(default_factory=list)
    elapsed_s: list = field(default_factory=list)
    compliance: list = field(default_factory=list)
    residual_inf: list = field(default_factory=list)
    dv_inf: list = field(default_factory=list)
    volume: list = field(default_factory=list)

    def append(self, k, elapsed, compliance, residual, dv, volume):
        if self.iters and k <= self.iters[-1]:
            raise ValueError("iteration numbers must be strictly increasing")
        self.iters.append(k)
        self.elapsed_s.append(elapsed)
        self.compliance.append(compliance)
        self.residual_inf.append(residual)
        self.dv_inf.append(dv)
        self.volume.append(volume)

    def rows(self):
        return zip(self.iters, self.elapsed_s, self.compliance, self.residual_inf, self.dv_inf,
                   self.volume)

    def __len__(self):
        return len(self.iters)


@dataclass
class RunResult:
    state: SolverState
    record: ConvergenceRecord
    reason: str  # "converged" | "budget" | "stopped"


class RunControl:
    """Thread-safe control channel applied at iteration boundaries (solvers.py:156-178)."""

    PAUSE, RESUME, STOP = "pause", "resume", "stop"

    def __init__(self):
        self._queue = queue.Queue()

    def send(self, command) -> None:
        self._queue.put(command)

    def drain(self) -> list:
        out = []
        while True:
            try:
                out.append(self._queue.get_nowait())
            except queue.Empty:
                return out

    def wait(self):
        return self._queue.get()


# ----------------------------------------------------------------- pieces ---

def sensitivity(grid: GridModel, v_phys, u, eta: float, filter_spec: FilterSpec):
    """Cᵀ(η·v_phys^(η−1) ⊙ ½u_eᵀke u_e) (solvers.py:181-190): one fused element pass
    (energies × SIMP prefactor) plus the adjoint stencil."""
    tv, tu = _dev.dev_f64(v_phys), _dev.dev_f64(u)
    out = _dev.empty(grid.num_elements)
    w = np.ascontiguousarray(gaussian_weights(filter_spec), dtype=np.float64)
    call("bsp_sensitivity", grid_handle(grid), tv.data_ptr(), tu.data_ptr(), float(eta), w.ctypes.data,
         int(filter_spec.size), out.data_ptr(), _dev.stream())
    return _dev.like(v_phys, out)


def mean_project(g):
    """g − mean(g) (solvers.py:193-197)."""
    n = int(_dev.shape_of(g)[0]) if len(_dev.shape_of(g)) else 0
    if n < 1:
        raise ValueError("mean_project needs at least one entry")
    t = _dev.dev_f64(g)
    out = _dev.empty(n)
    call("bsp_mean_project", t.data_ptr(), n, out.data_ptr(), _dev.stream())
    return _dev.like(g, out)


def krylov_apply(grid: GridModel, a, b, dim: int, threads: int = 1):
    """Least-squares Krylov polynomial applied to b (solvers.py:222-255): normalised power
    basis, Householder TSQR with the 1e-13 rank cut, Σ c_i K^i b."""
    if dim < 1:
        raise ValueError("Krylov dimension must be at least 1")
    ta, tb = _dev.dev_f64(a), _dev.dev_f64(b)
    out = _dev.empty(grid.num_dofs)
    call("bsp_krylov_apply", grid_handle(grid), ta.data_ptr(), tb.data_ptr(), int(dim), out.data_ptr(),
         None, _dev.stream())
    return _dev.like(b, out)


def low_level_step(grid: GridModel, a, u, config: SolverConfig, beta: float, residual=None,
                   threads: int = 1):
    """One damped displacement update (solvers.py:258-281)."""
    config = as_solver_config(config)
    algo = config.algorithm
    if algo not in ("fbto", "pfbto_jacobi", "cpfbto_krylov") + APPROX_INVERSES:
        raise ValueError(f"low_level_step does not apply to algorithm {algo!r}")
    if algo in APPROX_INVERSES:
        steps = config.resolved_inner_steps()
        if algo == "pcg_jacobi" and steps < 1:
            raise ValueError("pcg_jacobi needs inner_steps >= 1")
        r = residual if residual is not None else residual_reduce(grid, _dev.dev_f64(a),
                                                                  _dev.dev_f64(u))[0]
        mg = None
        if algo != "pcg_jacobi":
            mg = Multigrid(grid, config.mg_levels)
        out = pcg_apply(grid, a, r, steps, mg, config.mg_omega, config.resolved_mg_smooth(),
                        base=_dev.dev_f64(u), beta=float(beta))
        return _dev.like(u, out)
    ta, tu = _dev.dev_f64(a), _dev.dev_f64(u)
    tr = None if residual is None else _dev.dev_f64(residual)
    out = _dev.empty(grid.num_dofs)
    call("bsp_low_level_step", grid_handle(grid), ALGO[algo], ta.data_ptr(), tu.data_ptr(),
         float(beta), _dev.ptr(tr), int(config.krylov_dim), out.data_ptr(), _dev.stream())
    return _dev.like(u, out)


def high_level_step(v, g, alpha_k: float, bounds: SimplexBounds, active=None,
                    mean_projection: bool = True):
    """P_X(v + α_k·ĝ) with optional mean removal; passive entries pinned (solvers.py:284-302)."""
    n = int(_dev.shape_of(v)[0])
    tv, tg = _dev.dev_f64(v), _dev.dev_f64(g)
    ta = None if active is None else _dev.dev_u8(active)
    if active is None:
        bounds.validate(n)
    else:
        bounds.validate(int(np.count_nonzero(_dev.host_f64(active) if _dev.is_tensor(active)
                                             else np.asarray(active))))
    out = _dev.empty(n)
    call("bsp_high_level_step", tv.data_ptr(), tg.data_ptr(), n, float(alpha_k),
         float(bounds.v_lo), float(bounds.v_hi), float(bounds.v_bar), _dev.ptr(ta),
         1 if mean_projection else 0, out.data_ptr(), _dev.stream())
    return _dev.like(v, out)


# ------------------------------------------------------------------ setup ---

@dataclass
class _Workspace:
    """Resolved operators and parameters of one run (solvers.py:305-316)."""

    grid: GridModel
    filter_spec: FilterSpec
    eta: float
    active: np.ndarray | None
    bounds: SimplexBounds
    v_init: np.ndarray
    beta: float | None  # None: to be estimated on the row slabs


def _squared_jacobi_rho(grid: GridModel, v, eta, filter_spec, seed, iters=50) -> float:
    """Power iteration on K M⁻² K at the initial design (solvers.py:348-364), on device."""
    _, a = apply_filter_and_activation(_dev.dev_f64(v), grid.nx, grid.ny, filter_spec, eta)
    x0 = start_vector(grid, seed)
    rho = C.c_double()
    call("bsp_estimate_sqjacobi_rho", grid_handle(grid), a.data_ptr(), x0.data_ptr(), int(iters),
         C.addressof(rho), _dev.stream())
    return float(rho.value)


def _prepare(problem: ProblemSpec, config: SolverConfig, with_beta: bool = True) -> _Workspace:
    """Grid, bounds, initial design and β (solvers.py:319-345).  Large grids
    are resolved as index lists and scattered on the device
    (problems.resolve_device), and β's seeded start vector is generated on the
    device (fea.start_vector): no O(n) host work.  with_beta=False leaves a
    power-iteration β (fbto / pfbto without config.beta) as None: the row-slab
    loop estimates it on the slabs (distributed.SlabLoop)."""
    grid = resolve_device(problem) if problem.nx * problem.ny >= _DEVICE_RESOLVE_CELLS \
        else resolve(problem)
    eta = config.eta if config.eta is not None else problem.eta
    passive = problem.passive_mask()
    active = None if not passive.any() else ~passive
    n_active = problem.num_elements if active is None else int(active.sum())
    bounds = SimplexBounds(problem.v_lo, 1.0, problem.volume_fraction * n_active)
    v = np.full(problem.num_elements, problem.v_lo)
    level = min(max(problem.volume_fraction, problem.v_lo), 1.0)
    if active is None:
        v[:] = level
    else:
        v[active] = level
    beta = config.beta
    if beta is None and not with_beta and config.algorithm in ("fbto", "pfbto_jacobi"):
        return _Workspace(grid, problem.filter, eta, active, bounds, v, None)
    if beta is None:
        if config.algorithm == "fbto":
            beta = 1.0 / estimate_rho_max(grid, np.ones(grid.num_elements), 50,
                                          config.seed).rho_max
        elif config.algorithm == "pfbto_jacobi":
            beta = 1.0 / _squared_jacobi_rho(grid, v, eta, problem.filter, config.seed)
        else:
            beta = config.resolved_beta()
    return _Workspace(grid, problem.filter, eta, active, bounds, v, float(beta))


# ------------------------------------------------------------- device loop ---

class DeviceLoop:
    """Owner of a `bsp_solver` (device-resident outer loop, include/bisimp_b200.h)."""

    FIELDS = {"u": 0, "v": 1, "v_phys": 2, "activation": 3, "u_next": 4, "v_next": 5}

    def __init__(self, ws: _Workspace, config: SolverConfig, max_batch: int = _MAX_BATCH):
        _dev.require_cuda()
        self.ws = ws
        self.config = config
        self.max_batch = int(max_batch)
        grid = ws.grid
        cfg = config_c(ws, config, self.max_batch)
        act = None
        if ws.active is not None:
            act = np.ascontiguousarray(ws.active, dtype=np.uint8)
        v0 = np.ascontiguousarray(ws.v_init, dtype=np.float64)
        h = C.c_void_p()
        call("bsp_solver_create", grid_handle(grid), C.byref(cfg),
             None if act is None else act.ctypes.data, v0.ctypes.data, C.byref(h))
        self._h = h.value
        self._rec = np.zeros((self.max_batch, 4))
        self._alphas = np.zeros(self.max_batch)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                load().bsp_solver_destroy(h)
            except Exception:
                pass
            self._h = None

    def run(self, k_first: int, alphas) -> tuple[int, int, np.ndarray]:
        n = len(alphas)
        self._alphas[:n] = alphas
        done, status = C.c_int(), C.c_int()
        call("bsp_solver_run", self._h, int(k_first), n, self._alphas.ctypes.data,
             self._rec.ctypes.data, C.byref(done), C.byref(status))
        return done.value, status.value, self._rec[:n].copy()

    def stamps(self, n: int) -> np.ndarray:
        """Device-clock stamps (ns) of the rows returned by the last run()."""
        out = np.zeros(n, dtype=np.int64)
        call("bsp_solver_stamps", self._h, int(n), out.ctypes.data)
        return out

    def read(self, name: str) -> np.ndarray:
        grid = self.ws.grid
        size = grid.num_dofs if name in ("u", "u_next") else grid.num_elements
        out = np.empty(size)
        call("bsp_solver_read", self._h, self.FIELDS[name], out.ctypes.data)
        return out

    def read_state(self):
        """(u, v, v_phys, activation) of the last completed iteration, one device sync."""
        grid = self.ws.grid
        u, v = np.empty(grid.num_dofs), np.empty(grid.num_elements)
        vp, a = np.empty(grid.num_elements), np.empty(grid.num_elements)
        call("bsp_solver_read_state", self._h, u.ctypes.data, v.ctypes.data, vp.ctypes.data,
             a.ctypes.data)
        return u, v, vp, a

    def step_host(self, k: int, alpha: float, v: np.ndarray, u: np.ndarray,
                  v_next: np.ndarray, u_next: np.ndarray) -> np.ndarray:
        """One iteration through host buffers (the e2e drop-in call)."""
        rec = np.empty(4)
        call("bsp_solver_step_host", self._h, int(k), float(alpha), v.ctypes.data, u.ctypes.data,
             v_next.ctypes.data, u_next.ctypes.data, rec.ctypes.data)
        return rec

    def read_frame(self, kind: str = "f32") -> bytes:
        """v_phys of the last completed iteration as the service's float32 payload
        ("f32") or PGM pixels ("pgm"), converted on the device."""
        from .outputs import FRAME_KINDS
        E = self.ws.grid.num_elements
        out = np.empty(E, dtype="<f4" if kind == "f32" else np.uint8)
        call("bsp_solver_read_frame", self._h, FRAME_KINDS[kind], out.ctypes.data)
        return out.tobytes()

    def info(self) -> dict:
        out = np.zeros(4)
        call("bsp_solver_info", self._h, out.ctypes.data)
        return {"graphs": bool(out[0]), "kernels_per_iter": int(out[1]),
                "lambda_rounds": int(out[2]), "krylov_rank": int(out[3])}

    def stream(self) -> int:
        return load().bsp_solver_stream(self._h)


# Clocks that tell real time: iterations are stamped on the device and mapped
# onto them, so a run with clock= still executes in batches.  Any other
# callable is called once per completed iteration, as the reference does
# (solvers.py:466), which needs one host synchronisation per iteration.
_REALTIME_CLOCKS = (time.perf_counter, time.monotonic, time.time)


class _StampClock:
    """Maps the device's %globaltimer stamps of the record rows onto the
    caller's real-time clock.  Calibrated at every batch start: one host
    reading on each side of a one-thread kernel that reads the device timer
    (error about half a launch round trip, a few microseconds)."""

    def __init__(self, clk, stream: int):
        self.clk, self.stream = clk, stream
        self.ns0, self.h0 = 0, 0.0

    def calibrate(self) -> None:
        ns = C.c_longlong()
        h0 = self.clk()
        call("bsp_device_clock", self.stream, C.byref(ns))
        h1 = self.clk()
        self.ns0, self.h0 = int(ns.value), 0.5 * (h0 + h1)

    def at(self, ns: int) -> float:
        return self.h0 + (int(ns) - self.ns0) * 1e-9


def _make_state(k, u, v, v_phys, a, residual_inf, compliance, dv_inf, fresh=False) -> SolverState:
    """SolverState with host copies (solvers.py:367-378); `fresh` arrays are owned already."""
    cp = not fresh
    v = np.array(v, dtype=float, copy=cp)
    return SolverState(iter=k, u=np.array(u, dtype=float, copy=cp), v=DensityField(v),
                       v_phys=np.array(v_phys, dtype=float, copy=cp),
                       activation=np.array(a, dtype=float, copy=cp),
                       residual_inf=residual_inf, compliance=compliance,
                       volume=float(v.sum()), last_dv_inf=dv_inf)


def _divergence(k, residual_inf, compliance, alpha0, algorithm):
    return DivergenceError(
        f"non-finite iterate at iteration {k} "
        f"(residual_inf={residual_inf}, compliance={compliance}); "
        f"alpha0={alpha0} is likely too large for {algorithm}")


def run(problem: ProblemSpec, config: SolverConfig, sink: Callable[[SolverState], None] | None = None,
        control: RunControl | None = None, threads: int = 1,
        clock: Callable[[], float] | None = None, *,
        frame_sink: Callable | None = None, frame_kind: str = "f32",
        slabs: int | str | None = None) -> RunResult:
    """Iterate until both termination tolerances hold ("converged") or the budget runs out
    ("budget"); "stopped" on a STOP command (solvers.py:381-484).

    Extension: `frame_sink(outputs.Frame)` is called at the
    sink's cadence (every `snapshot_every` iterations and on the final state)
    with v_phys converted ON THE DEVICE to the service's float32 payload
    (`frame_kind="f32"`, service/sessions.py:97) or to PGM pixels
    (`"pgm"`, outputs.py:27); it works with or without `sink`.

    Extension: `slabs` runs the same loop with the grid split
    into row slabs (distributed.SlabLoop): "nccl" puts one slab on each rank of
    the initialised torch.distributed group (one GPU per process, NCCL halo
    exchanges and all-gathers; every rank calls run() and gets the same
    RunResult, sinks run on every rank with the gathered state); an int G
    puts G slabs on this GPU (the same kernels and exchange pattern, device
    copies as the transport).  None: one GPU."""
    config = as_solver_config(config)
    from .outputs import FRAME_KINDS
    if frame_kind not in FRAME_KINDS:
        raise ValueError(f"unknown frame kind {frame_kind!r}; expected one of {sorted(FRAME_KINDS)}")
    emit = _Emitter(sink, frame_sink, frame_kind, problem.nx, problem.ny)
    if slabs is not None and config.max_iters > 0:
        from .distributed import slab_loop
        loop = slab_loop(problem, config, slabs)
        return _drive(loop.ws, config, loop, emit, control, clock)
    ws = _prepare(problem, config)
    if config.algorithm == "pgd_exact":
        return _run_pgd(ws, config, emit, control, clock)
    loop = DeviceLoop(ws, config) if config.max_iters > 0 else None
    return _drive(ws, config, loop, emit, control, clock)


def _drive(ws: _Workspace, config: SolverConfig, loop, emit: "_Emitter", control, clock) -> RunResult:
    """run()'s outer loop over a device-resident loop (DeviceLoop or
    distributed.SlabLoop): batches, control, sink cadence, clock, record."""
    grid = ws.grid
    clk = clock if clock is not None else (lambda: 0.0)
    alpha0 = config.resolved_alpha0()
    snapshot_every = config.snapshot_every
    record = ConvergenceRecord()
    reason = "budget"
    last = None  # (k, residual_inf, compliance, dv_inf) of the latest completed iteration
    emitted_iter = -1
    stamped = (clock is not None and clock in _REALTIME_CLOCKS and loop is not None
               and hasattr(loop, "stamps"))
    stamp_clock = _StampClock(clock, loop.stream()) if stamped else None
    t0 = clk()
    last_elapsed = 0.0
    k = 1
    while k <= config.max_iters:
        if control is not None:
            stop = False
            paused = False
            commands = control.drain()
            while True:
                for cmd in commands:
                    if cmd == RunControl.PAUSE:
                        paused = True
                    elif cmd == RunControl.RESUME:
                        paused = False
                    elif cmd == RunControl.STOP:
                        stop = True
                    elif isinstance(cmd, dict):
                        if "alpha0" in cmd:
                            alpha0 = float(cmd["alpha0"])
                        if "snapshot_every" in cmd:
                            snapshot_every = int(cmd["snapshot_every"])
                    else:
                        raise ValueError(f"unknown control command {cmd!r}")
                if stop or not paused:
                    break
                commands = [control.wait()]
            if stop:
                reason = "stopped"
                break
        n = min(loop.max_batch, config.max_iters - k + 1)
        if emit and snapshot_every > 0:
            n = min(n, snapshot_every - (k - 1) % snapshot_every)
        if control is not None:
            n = min(n, _CONTROL_BATCH)
        if clock is not None and not stamped:
            n = 1
        alphas = [config.step_size(j, alpha0) for j in range(k, k + n)]
        if stamped:
            stamp_clock.calibrate()
        done, status, rows = loop.run(k, alphas)
        stamps = loop.stamps(done) if stamped else None
        for i in range(done):
            c, r, dv, vol = (float(t) for t in rows[i])
            if stamped:  # device stamp on the caller's clock; monotone like the clock itself
                last_elapsed = max(last_elapsed, stamp_clock.at(stamps[i]) - t0)
                elapsed = last_elapsed
            else:
                elapsed = clk() - t0
            record.append(k + i, elapsed, c, r, dv, vol)
        if done:
            kk = k + done - 1
            last = (kk, float(rows[done - 1][1]), float(rows[done - 1][0]),
                    float(rows[done - 1][2]), float(rows[done - 1][3]))
            if emit and snapshot_every > 0 and kk % snapshot_every == 0:
                emit.from_loop(loop, last)
                emitted_iter = kk
        if status == 4:
            raise NotImplementedError(
                f"krylov_dim={config.krylov_dim}: the Krylov basis is numerically full rank "
                "past the 63 powers the device TSQR holds (see csrc/krylov.cu)")
        if status == 2:  # diverged at iteration k + done
            raise _divergence(k + done, float(rows[done][1]), float(rows[done][0]), alpha0,
                              config.algorithm)
        k += done
        if status == 1:
            reason = "converged"
            break
    if last is None:  # zero-iteration budget or immediate stop: initial design
        v = ws.v_init
        v_phys, a = apply_filter_and_activation(v, grid.nx, grid.ny, ws.filter_spec, ws.eta)
        state = _make_state(0, np.zeros(grid.num_dofs), v, v_phys, a,
                            float(np.abs(grid.load).max()), 0.0, 0.0)
    else:
        state = _loop_state(loop, last)
    if emitted_iter != state.iter:
        if last is None:
            emit.from_state(state)
        else:
            emit.from_loop(loop, last, state)
    return RunResult(state=state, record=record, reason=reason)


def _loop_state(loop: DeviceLoop, last) -> SolverState:
    k, res, comp, dv = last[:4]
    u, v, vp, a = loop.read_state()
    return _make_state(k, u, v, vp, a, res, comp, dv, fresh=True)


class _Emitter:
    """Snapshot fan-out: the reference's `sink(SolverState)` and/or the device
    frame sink (`frame_sink(Frame)`)."""

    def __init__(self, sink, frame_sink, kind, nx, ny):
        self.sink, self.frame_sink, self.kind, self.nx, self.ny = sink, frame_sink, kind, nx, ny

    def __bool__(self):
        return self.sink is not None or self.frame_sink is not None

    def _frame(self, k, comp, res, vol, payload):
        from .outputs import Frame
        return Frame(iter=k, compliance=comp, residual_inf=res, volume=vol, nx=self.nx,
                     ny=self.ny, payload=payload, kind=self.kind)

    def from_loop(self, loop: DeviceLoop, last, state: SolverState | None = None):
        """Iterate `last` = (k, res, comp, dv, volume) still resident in the device loop."""
        if self.sink is not None:
            self.sink(state if state is not None else _loop_state(loop, last))
        if self.frame_sink is not None:
            k, res, comp, _, vol = last
            self.frame_sink(self._frame(k, comp, res, vol, loop.read_frame(self.kind)))

    def from_state(self, state: SolverState, v_phys_dev=None):
        """A host (or host + device v_phys) state outside the device loop."""
        if self.sink is not None:
            self.sink(state)
        if self.frame_sink is not None:
            from .outputs import density_pixels, frame_payload
            vp = state.v_phys if v_phys_dev is None else v_phys_dev
            if self.kind == "f32":
                payload = frame_payload(vp)
            else:
                px = density_pixels(vp)
                payload = (px.cpu().numpy() if _dev.is_tensor(px) else px).tobytes()
            self.frame_sink(self._frame(state.iter, state.compliance, state.residual_inf,
                                        state.volume, payload))


def _run_pgd(ws: _Workspace, config: SolverConfig, emit: _Emitter, control, clock) -> RunResult:
    """Exact-inversion baseline (solvers.py:445-446): host-driven loop of device ops."""
    grid = ws.grid
    clk = clock if clock is not None else (lambda: 0.0)
    alpha0 = config.resolved_alpha0()
    snapshot_every = config.snapshot_every
    u = _dev.zeros(grid.num_dofs)
    v = _dev.dev_f64(ws.v_init)
    act = None if ws.active is None else _dev.dev_u8(ws.active)
    record = ConvergenceRecord()
    reason = "budget"
    last = None
    emitted_iter = -1
    t0 = clk()
    for k in range(1, config.max_iters + 1):
        if control is not None:
            stop = False
            paused = False
            commands = control.drain()
            while True:
                for cmd in commands:
                    if cmd == RunControl.PAUSE:
                        paused = True
                    elif cmd == RunControl.RESUME:
                        paused = False
                    elif cmd == RunControl.STOP:
                        stop = True
                    elif isinstance(cmd, dict):
                        if "alpha0" in cmd:
                            alpha0 = float(cmd["alpha0"])
                        if "snapshot_every" in cmd:
                            snapshot_every = int(cmd["snapshot_every"])
                    else:
                        raise ValueError(f"unknown control command {cmd!r}")
                if stop or not paused:
                    break
                commands = [control.wait()]
            if stop:
                reason = "stopped"
                break
        v_phys, a = apply_filter_and_activation(v, grid.nx, grid.ny, ws.filter_spec, ws.eta)
        u = exact_solve(grid, a, _EXACT_SOLVE_TOL, x0=u)
        _, uku, residual_inf = residual_reduce(grid, a, u)
        compliance = 0.5 * uku
        if not (np.isfinite(residual_inf) and np.isfinite(compliance)):
            raise _divergence(k, residual_inf, compliance, alpha0, config.algorithm)
        g = sensitivity(grid, v_phys, u, ws.eta, ws.filter_spec)
        alpha_k = config.step_size(k, alpha0)
        v_next = high_level_step(v, g, alpha_k, ws.bounds, act, config.mean_projection)
        dv_inf = float(torch.max(torch.abs(v_next - v)).item())
        record.append(k, clk() - t0, compliance, residual_inf, dv_inf, float(v.sum().item()))
        last = (k, u, v, v_phys, a, residual_inf, compliance, dv_inf)
        if emit and snapshot_every > 0 and k % snapshot_every == 0:
            emit.from_state(_make_state(*(t.cpu().numpy() if torch.is_tensor(t) else t
                                          for t in last)), v_phys_dev=v_phys)
            emitted_iter = k
        v = v_next
        if dv_inf < config.tol_dv and residual_inf < config.tol_res:
            reason = "converged"
            break
    if last is None:
        v_phys, a = apply_filter_and_activation(v, grid.nx, grid.ny, ws.filter_spec, ws.eta)
        last = (0, u, v, v_phys, a, float(np.abs(grid.load).max()), 0.0, 0.0)
    state = _make_state(*(t.cpu().numpy() if torch.is_tensor(t) else t for t in last))
    if emitted_iter != state.iter:
        emit.from_state(state, v_phys_dev=last[3])
    return RunResult(state=state, record=record, reason=reason)


def pgd_step(grid: GridModel, v, u_prev, config: SolverConfig, k: int, filter_spec: FilterSpec,
             eta: float, bounds: SimplexBounds, active=None, threads: int = 1):
    """One exact-inversion step (solvers.py:487-506)."""
    config = as_solver_config(config)
    v_phys, a = apply_filter_and_activation(_dev.dev_f64(v), grid.nx, grid.ny, filter_spec, eta)
    u = exact_solve(grid, a, _EXACT_SOLVE_TOL, x0=u_prev)
    g = sensitivity(grid, v_phys, u, eta, filter_spec)
    v_next = high_level_step(_dev.dev_f64(v), g, config.step_size(k), bounds, active,
                             config.mean_projection)
    return _dev.like(v, u), _dev.like(v, v_next)


def diagnostics_projection_error(problem: ProblemSpec, state: SolverState, config: SolverConfig,
                                 k: int, grid: GridModel | None = None,
                                 exact: bool = False) -> float:
    """‖P_X(v + α_k·g) − v‖²/α_k² (solvers.py:509-538)."""
    config = as_solver_config(config)
    if k < 1:
        raise ValueError("k must be at least 1")
    if grid is None:
        grid = resolve(problem)
    eta = config.eta if config.eta is not None else problem.eta
    passive = problem.passive_mask()
    active = None if not passive.any() else ~passive
    n_active = problem.num_elements if active is None else int(active.sum())
    bounds = SimplexBounds(problem.v_lo, 1.0, problem.volume_fraction * n_active)
    v = _dev.dev_f64(state.v.values)
    v_phys, a = apply_filter_and_activation(v, grid.nx, grid.ny, problem.filter, eta)
    u = exact_solve(grid, a, 1e-12, x0=state.u) if exact else _dev.dev_f64(state.u)
    g = sensitivity(grid, v_phys, u, eta, problem.filter)
    alpha_k = config.step_size(k)
    moved = high_level_step(v, g, alpha_k, bounds, active, mean_projection=False)
    return float(torch.sum((moved - v) ** 2).item()) / alpha_k ** 2
