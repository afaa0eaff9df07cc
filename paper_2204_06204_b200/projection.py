"""Bounded-simplex projection on the GPU — drop-in for `bisimp.projection`.

`project_simplex` runs the cooperative projection kernel (`csrc/highlevel.cu`):
box early exit, otherwise a deterministic regime-Newton search for λ with
Σ clamp(v − λ, lo, hi) = budget (same solution as the reference's
sorted-breakpoint sweep, projection.py:50-91).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _dev
from ._native import call


@dataclass(frozen=True)
class SimplexBounds:
    """Box [v_lo, v_hi] and total budget v_bar (projection.py:14-28)."""

    v_lo: float
    v_hi: float
    v_bar: float

    def validate(self, n: int) -> None:
        if not 0.0 < self.v_lo < self.v_hi:
            raise ValueError(f"need 0 < v_lo < v_hi, got [{self.v_lo}, {self.v_hi}]")
        if not n * self.v_lo <= self.v_bar <= n * self.v_hi:
            raise ValueError(
                f"budget {self.v_bar} infeasible for {n} elements in [{self.v_lo}, {self.v_hi}]")


def project_box(v, lo: float, hi: float):
    """Elementwise clamp to [lo, hi] (projection.py:31-35)."""
    if not lo < hi:
        raise ValueError(f"need lo < hi, got [{lo}, {hi}]")
    t = _dev.dev_f64(v)
    return _dev.like(v, torch.clamp(t, min=lo, max=hi))


def project_simplex(v, bounds: SimplexBounds):
    """argmin ½‖x − v‖² over {lo ≤ x ≤ hi, Σx ≤ v_bar} (projection.py:50-91)."""
    n = int(_dev.shape_of(v)[0])
    bounds.validate(n)
    t = _dev.dev_f64(v)
    out = _dev.empty(n)
    call("bsp_project_simplex", t.data_ptr(), n, float(bounds.v_lo), float(bounds.v_hi),
         float(bounds.v_bar), out.data_ptr(), _dev.stream())
    return _dev.like(v, out)
