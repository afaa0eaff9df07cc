"""Matrix-free Q4 finite elements on the GPU — drop-in for `bisimp.fea`.

Same names, signatures, defaults and exceptions as the reference module
(`/root/reference/pkg/src/bisimp/fea.py`); the arithmetic runs in the sm_100a
library through the C ABI (`include/bisimp_b200.h`).

Grid conventions (reference fea.py:8-11): element e = ey*nx+ex, node
n = y*(nx+1)+x with DOFs 2n (x) and 2n+1 (y); row 0 is the top of the image.
`threads` arguments are accepted for API compatibility and ignored (the
reference's CPU chunking knob, fea.py:167-179, has no GPU meaning).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _dev
from ._native import call, load


class LinearSolveError(RuntimeError):
    """Raised when the iterative linear solver fails to reach tolerance (fea.py:23-24)."""


@dataclass(frozen=True)
class Material:
    """Plane-stress constitutive parameters (fea.py:27-38)."""

    young_modulus: float = 1.0
    poisson_ratio: float = 0.3

    def __post_init__(self):
        if not self.young_modulus > 0:
            raise ValueError(f"young_modulus must be > 0, got {self.young_modulus}")
        if not 0.0 <= self.poisson_ratio < 0.5:
            raise ValueError(f"poisson_ratio must be in [0, 0.5), got {self.poisson_ratio}")


@dataclass
class DensityField:
    """Per-element infill levels, row-major (fea.py:41-50)."""

    values: np.ndarray

    def validate(self, v_lo: float) -> None:
        v = self.values
        lo, hi = float(v.min()), float(v.max())
        if lo < v_lo - 1e-12 or hi > 1.0 + 1e-12:
            raise ValueError(f"density outside [{v_lo}, 1]: min {lo}, max {hi}")


@dataclass
class SpectrumEstimate:
    """Power-iteration spectrum estimate (fea.py:53-58)."""

    rho_max: float
    rho_min_hint: float | None = None


def element_stiffness(material: Material) -> np.ndarray:
    """8x8 unit bilinear quad, plane stress (fea.py:61-87).

    Closed form of the exactly integrated element; local nodes (0,0), (1,0),
    (1,1), (0,1), DOFs interleaved (ux, uy)."""
    nu = material.poisson_ratio
    c = material.young_modulus / (1.0 - nu * nu)
    k = np.array([0.5 - nu / 6.0, 0.125 + nu / 8.0, -0.25 - nu / 12.0, -0.125 + 3.0 * nu / 8.0,
                  -0.25 + nu / 12.0, -0.125 - nu / 8.0, nu / 6.0, 0.125 - 3.0 * nu / 8.0])
    # index pattern of the Q4 element: row r, column s -> k[_KIDX[r][s]]
    return c * k[_KIDX]


_KIDX = np.array([
    [0, 1, 2, 3, 4, 5, 6, 7],
    [1, 0, 7, 6, 5, 4, 3, 2],
    [2, 7, 0, 5, 6, 3, 4, 1],
    [3, 6, 5, 0, 7, 2, 1, 4],
    [4, 5, 6, 7, 0, 1, 2, 3],
    [5, 4, 3, 2, 1, 0, 7, 6],
    [6, 3, 4, 1, 2, 7, 0, 5],
    [7, 2, 1, 4, 3, 6, 5, 0],
])


def element_dof_map(nx: int, ny: int) -> np.ndarray:
    """(E, 8) global DOFs per element in element_stiffness order (fea.py:90-101)."""
    e = np.arange(nx * ny)
    base = (e // nx) * (nx + 1) + e % nx
    nodes = np.stack([base, base + 1, base + nx + 2, base + nx + 1], axis=1)
    out = np.empty((nx * ny, 8), dtype=np.int64)
    out[:, 0::2] = 2 * nodes
    out[:, 1::2] = 2 * nodes + 1
    return out


@dataclass
class GridModel:
    """Discretised problem (fea.py:104-143), mirrored into HBM on first use.

    The device copy (fixed-DOF bitmask, load, Hadamard-mode element
    constants) is built lazily by `native()` and freed with the object.
    `edof` is computed on demand (the kernels never need it)."""

    nx: int
    ny: int
    ke: np.ndarray
    fixed_dofs: np.ndarray
    load: np.ndarray
    _handle: object = field(default=None, init=False, repr=False, compare=False)
    _edof: object = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError("grid must have at least one element per axis")
        n = self.num_dofs
        fixed = np.asarray(self.fixed_dofs)
        if fixed.shape != (n,) or fixed.dtype != bool:
            raise ValueError("fixed_dofs must be a boolean mask over all DOFs")
        if np.shape(self.load) != (n,):
            raise ValueError("load length must equal the DOF count")
        ke = np.asarray(self.ke, dtype=float)
        if not np.allclose(ke, ke.T, atol=1e-12):
            raise ValueError("element stiffness must be symmetric")
        if int(fixed.sum()) < 3:
            raise ValueError("at least 3 DOFs must be fixed (rigid modes)")
        if np.any(np.asarray(self.load)[fixed] != 0.0):
            raise ValueError("load must be zero on fixed DOFs")

    @property
    def edof(self) -> np.ndarray:
        if self._edof is None:
            self._edof = element_dof_map(self.nx, self.ny)
        return self._edof

    @property
    def num_elements(self) -> int:
        return self.nx * self.ny

    @property
    def num_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1)

    @property
    def num_dofs(self) -> int:
        return 2 * self.num_nodes

    def native(self):
        """Handle of the device-resident grid (bsp_grid*)."""
        if self._handle is None:
            _dev.require_cuda()
            ke = np.ascontiguousarray(self.ke, dtype=np.float64)
            fixed = np.ascontiguousarray(self.fixed_dofs, dtype=np.uint8)
            load_ = np.ascontiguousarray(self.load, dtype=np.float64)
            h = C.c_void_p()
            call("bsp_grid_create", self.nx, self.ny, ke.ctypes.data, fixed.ctypes.data,
                 load_.ctypes.data, C.byref(h))
            self._handle = _GridHandle(h.value)
        return self._handle.ptr

    def native_flags(self) -> int:
        flags = C.c_int()
        call("bsp_grid_info", self.native(), None, None, C.byref(flags))
        return flags.value


class SparseGridModel(GridModel):
    """A GridModel held as index lists (problems.resolve_device): the device
    copy is built by scattering them (bsp_grid_create_sparse), so a 268M-DOF
    grid costs no O(n) host work; `fixed_dofs` / `load` materialise the dense
    host arrays (once) only when read."""

    def __init__(self, nx, ny, ke, fixed_idx, load_idx, load_vals):
        if nx < 1 or ny < 1:
            raise ValueError("grid must have at least one element per axis")
        ke = np.asarray(ke, dtype=float)
        if not np.allclose(ke, ke.T, atol=1e-12):
            raise ValueError("element stiffness must be symmetric")
        if np.unique(fixed_idx).size < 3:
            raise ValueError("at least 3 DOFs must be fixed (rigid modes)")
        if np.isin(load_idx, fixed_idx).any():
            raise ValueError("load must be zero on fixed DOFs")
        object.__setattr__(self, "nx", int(nx))
        object.__setattr__(self, "ny", int(ny))
        object.__setattr__(self, "ke", ke)
        self._fixed_idx = np.ascontiguousarray(fixed_idx, dtype=np.int64)
        self._load_idx = np.ascontiguousarray(load_idx, dtype=np.int64)
        self._load_vals = np.ascontiguousarray(load_vals, dtype=np.float64)
        self._dense = None
        self._handle = None
        self._edof = None

    def _materialise(self):
        if self._dense is None:
            fixed = np.zeros(self.num_dofs, dtype=bool)
            fixed[self._fixed_idx] = True
            load = np.zeros(self.num_dofs)
            load[self._load_idx] = self._load_vals
            self._dense = (fixed, load)
        return self._dense

    @property
    def fixed_dofs(self):
        return self._materialise()[0]

    @property
    def load(self):
        return self._materialise()[1]

    def native(self):
        if self._handle is None:
            _dev.require_cuda()
            ke = np.ascontiguousarray(self.ke, dtype=np.float64)
            h = C.c_void_p()
            call("bsp_grid_create_sparse", self.nx, self.ny, ke.ctypes.data,
                 int(self._fixed_idx.size), self._fixed_idx.ctypes.data,
                 int(self._load_idx.size), self._load_idx.ctypes.data,
                 self._load_vals.ctypes.data, C.byref(h))
            self._handle = _GridHandle(h.value)
        return self._handle.ptr


_FOREIGN: dict = {}  # id(grid) -> (weakref to the caller's grid, mirror GridModel)


def grid_handle(grid) -> int:
    """Device handle (bsp_grid*) for any grid-like object.

    This module's GridModel owns its handle.  Any other object with the
    reference GridModel's fields (nx, ny, ke, fixed_dofs, load; fea.py:104-143)
    -- in particular the reference's own GridModel, which the reference's
    callers build through `problems.resolve` -- is validated once through a
    mirror GridModel whose device copy lives as long as the caller's object
    (the cache entry is dropped by a weakref callback when it dies).  Like the
    reference's own `_assembly_cache` / `_lu_cache` (fea.py:113-114), the
    device copy assumes the grid's arrays are not mutated in place."""
    if isinstance(grid, GridModel):
        return grid.native()
    key = id(grid)
    ent = _FOREIGN.get(key)
    if ent is not None and ent[0]() is grid:
        return ent[1].native()
    mirror = GridModel(nx=int(grid.nx), ny=int(grid.ny), ke=np.asarray(grid.ke, dtype=float),
                       fixed_dofs=np.asarray(grid.fixed_dofs), load=np.asarray(grid.load))
    try:
        ref = weakref.ref(grid, lambda _r, key=key: _FOREIGN.pop(key, None))
    except TypeError:  # not weak-referenceable: key the mirror by the object itself
        ref = (lambda g=grid: g)
    _FOREIGN[key] = (ref, mirror)
    return mirror.native()


class _GridHandle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            load().bsp_grid_destroy(self.ptr)
        except Exception:
            pass


def _check_shapes(grid: GridModel, a=None, u=None):
    if u is not None and _dev.shape_of(u) != (grid.num_dofs,):
        raise ValueError(f"u has length {_dev.shape_of(u)}, expected {grid.num_dofs}")
    if a is not None and _dev.shape_of(a) != (grid.num_elements,):
        raise ValueError(f"a has length {_dev.shape_of(a)}, expected {grid.num_elements}")


def apply_stiffness(grid: GridModel, a, u, threads: int = 1):
    """K(a)·u, fixed DOFs of u read as zero and zeroed in the result (fea.py:150-181)."""
    _check_shapes(grid, a=a, u=u)
    ta, tu = _dev.dev_f64(a), _dev.dev_f64(u)
    y = _dev.empty(grid.num_dofs)
    call("bsp_apply_stiffness", grid_handle(grid), ta.data_ptr(), tu.data_ptr(), y.data_ptr(),
         _dev.stream())
    return _dev.like(u, y)


def stiffness_diagonal(grid: GridModel, a):
    """diag(K(a)) with ones at fixed DOFs (fea.py:184-189)."""
    _check_shapes(grid, a=a)
    ta = _dev.dev_f64(a)
    d = _dev.empty(grid.num_dofs)
    call("bsp_stiffness_diagonal", grid_handle(grid), ta.data_ptr(), d.data_ptr(), _dev.stream())
    return _dev.like(a, d)


def residual_reduce(grid: GridModel, a, u):
    """(r = K(a)u − f, u·K(a)u, max|r|) in one fused pass (solvers.py:447-449)."""
    ta, tu = _dev.dev_f64(a), _dev.dev_f64(u)
    r = _dev.empty(grid.num_dofs)
    out = (C.c_double * 4)()
    call("bsp_residual", grid_handle(grid), ta.data_ptr(), tu.data_ptr(), r.data_ptr(),
         C.addressof(out), _dev.stream())
    return r, float(out[0]), float(out[3])


def compliance_energy(grid: GridModel, a, u) -> float:
    """½ uᵀK(a)u (fea.py:192-194)."""
    _check_shapes(grid, a=a, u=u)
    _, uku, _ = residual_reduce(grid, a, u)
    return 0.5 * uku


def element_energies(grid: GridModel, u):
    """½ u_eᵀ ke u_e per element, fixed DOFs of u read as zero (fea.py:197-201)."""
    _check_shapes(grid, u=u)
    tu = _dev.dev_f64(u)
    e = _dev.empty(grid.num_elements)
    call("bsp_element_energies", grid_handle(grid), tu.data_ptr(), e.data_ptr(), _dev.stream())
    return _dev.like(u, e)


def exact_solve(grid: GridModel, a, tol: float, x0=None, max_iters: int = 30, threads: int = 1):
    """Solve K(a)u = f to ‖K u − f‖∞ ≤ tol (contract of fea.py:230-275).

    The reference factors the free block with SuperLU and refines; on the GPU
    this is restarted multigrid-preconditioned CG (8 steps per restart, one
    V-cycle per step) with a true-residual check per restart.  The
    postcondition is the reference's; `max_iters` scales the CG budget
    (max_iters · max(200, n_dofs) steps).  Raises LinearSolveError when the
    budget cannot reach tol or the residual stalls at the rounding floor."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    _check_shapes(grid, a=a)
    ta = _dev.dev_f64(a)
    tx0 = None if x0 is None else _dev.dev_f64(x0)
    out = _dev.empty(grid.num_dofs)
    budget = int(max_iters) * max(200, grid.num_dofs)
    call("bsp_exact_solve", grid_handle(grid), ta.data_ptr(), float(tol), _dev.ptr(tx0), budget,
         out.data_ptr(), _dev.stream())
    return _dev.like(a, out)


def pcg64_state(seed: int) -> np.ndarray:
    """numpy's PCG64 state after seeding `default_rng(seed)` (SeedSequence
    hashing, host, O(1)) as {state lo, state hi, inc lo, inc hi}."""
    st = np.random.PCG64(np.random.SeedSequence(seed)).state["state"]
    m = (1 << 64) - 1
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s & m, s >> 64, inc & m, inc >> 64], dtype=np.uint64)


def standard_normal(seed: int, n: int):
    """np.random.default_rng(seed).standard_normal(n), generated ON THE DEVICE
    (csrc/rng.cu: PCG64 + numpy's ziggurat; a CUDA tensor)."""
    out = _dev.empty(n)
    st = pcg64_state(seed)
    call("bsp_standard_normal", st.ctypes.data, int(n), out.data_ptr(), _dev.stream())
    return out


def start_vector(grid: GridModel, seed: int):
    """The reference's seeded, masked, normalised power-iteration start
    (fea.py:289-292), generated on the device: numpy's normal stream bit for
    bit (csrc/rng.cu), the norm by a device tree sum.  A CUDA tensor."""
    out = _dev.empty(grid.num_dofs)
    st = pcg64_state(seed)
    call("bsp_start_vector", grid_handle(grid), st.ctypes.data, out.data_ptr(), _dev.stream())
    return out


def estimate_rho_max(grid: GridModel, a, iters: int, seed: int = 0) -> SpectrumEstimate:
    """Largest eigenvalue of the masked K(a) by seeded power iteration (fea.py:278-301)."""
    if iters < 5:
        raise ValueError("iters must be >= 5")
    _check_shapes(grid, a=a)
    ta = _dev.dev_f64(a)
    x0 = start_vector(grid, seed)
    rho = C.c_double()
    call("bsp_estimate_rho_max", grid_handle(grid), ta.data_ptr(), x0.data_ptr(), int(iters),
         C.addressof(rho), _dev.stream())
    return SpectrumEstimate(rho_max=float(rho.value))
