"""Separable Gaussian density filter on the GPU — drop-in for `bisimp.filtering`.

The taps are computed on the host exactly as the reference does
(filtering.py:30-35, numpy exp + pairwise sum) and passed to the sm_100a
shared-memory stencil kernels (`csrc/filter.cu`); boundary masses
(filtering.py:38-43) are evaluated in-kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev
from ._native import call


@dataclass(frozen=True)
class FilterSpec:
    """Odd kernel width `size`, standard deviation `sigma` in elements (filtering.py:17-27)."""

    size: int = 7
    sigma: float = 1.5

    def __post_init__(self):
        if self.size < 1 or self.size % 2 == 0:
            raise ValueError(f"kernel size must be odd and >= 1, got {self.size}")
        if not self.sigma > 0:
            raise ValueError(f"sigma must be positive, got {self.sigma}")


def gaussian_weights(spec: FilterSpec) -> np.ndarray:
    """Symmetric 1-D taps normalised to sum 1 (filtering.py:30-35)."""
    r = spec.size // 2
    t = np.exp(-0.5 * (np.arange(-r, r + 1, dtype=float) / spec.sigma) ** 2)
    return t / t.sum()


def _taps(spec: FilterSpec) -> np.ndarray:
    return np.ascontiguousarray(gaussian_weights(spec), dtype=np.float64)


def _run(field, nx: int, ny: int, spec: FilterSpec, adjoint: bool, act_eta=None):
    if _dev.shape_of(field) != (nx * ny,):
        raise ValueError(f"field has length {_dev.shape_of(field)}, expected {nx * ny}")
    t = _dev.dev_f64(field)
    out = _dev.empty(nx * ny)
    act = _dev.empty(nx * ny) if act_eta is not None else None
    w = _taps(spec)
    call("bsp_filter", t.data_ptr(), out.data_ptr(), _dev.ptr(act),
         float(act_eta if act_eta is not None else 1.0), int(nx), int(ny), w.ctypes.data,
         int(spec.size), 1 if adjoint else 0, _dev.stream())
    return out, act


def apply_filter(field, nx: int, ny: int, spec: FilterSpec):
    """Physical densities C(v): x pass then y pass, renormalised (filtering.py:46-55)."""
    out, _ = _run(field, nx, ny, spec, False)
    return _dev.like(field, out)


def apply_filter_and_activation(field, nx: int, ny: int, spec: FilterSpec, eta: float):
    """(C(v), C(v)**eta) in one kernel (filtering.py:46-55 + solvers.py:443)."""
    out, act = _run(field, nx, ny, spec, False, act_eta=eta)
    return _dev.like(field, out), _dev.like(field, act)


def apply_filter_adjoint(field, nx: int, ny: int, spec: FilterSpec):
    """Exact transpose Cᵀ, boundary renormalisation included (filtering.py:58-72)."""
    out, _ = _run(field, nx, ny, spec, True)
    return _dev.like(field, out)
