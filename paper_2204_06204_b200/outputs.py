"""Density frames produced on the device.

The reference converts `state.v_phys` on the host at every snapshot: the
service streams it as little-endian float32 (`service/sessions.py:90-97`)
and the CLI writes it as a binary PGM (`outputs.py:21-30`, called from
`cli.py:66-69,75`).  Here both conversions run on the GPU
(`csrc/frames.cu`), byte-identical to the reference's, so a snapshot of a
134M-cell design moves 4 or 1 bytes per cell over PCIe instead of the 8·(n+3E)
bytes of a full `SolverState`.

* `frame_payload(v_phys)` — the service payload bytes;
* `density_pixels(v_phys)` — the PGM pixel array (numpy in → numpy out, CUDA
  tensor in → CUDA tensor out);
* `write_snapshot(v_phys, nx, ny, path)` — `outputs.write_snapshot`, same
  header, validation order and messages;
* `Frame` — the service's frame record (`service/sessions.py:25-35`), which
  `solvers.run(..., frame_sink=...)` emits straight from the device loop.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._native import call

FRAME_KINDS = {"f32": 0, "pgm": 1}


@dataclass
class Frame:
    """One density snapshot plus its scalar diagnostics (service/sessions.py:25-35).

    `payload` is v_phys as row-major little-endian float32 for kind "f32"
    (sessions.py:97) or the PGM pixel bytes for kind "pgm" (outputs.py:27)."""

    iter: int
    compliance: float
    residual_inf: float
    volume: float
    nx: int
    ny: int
    payload: bytes
    kind: str = "f32"


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _flat(v_phys) -> torch.Tensor:
    t = _dev.dev_f64(v_phys)
    if t.dim() != 1:
        t = t.reshape(-1)
    return t


def frame_payload(v_phys) -> bytes:
    """`v_phys.astype("<f4").tobytes()` (service/sessions.py:97), converted on the GPU."""
    t = _flat(v_phys)
    out = torch.empty(t.numel(), dtype=torch.float32, device=t.device)
    call("bsp_density_frame", _dev.ptr(t), t.numel(), _dev.ptr(out), _stream())
    return out.cpu().numpy().astype("<f4", copy=False).tobytes()


def density_pixels(v_phys):
    """PGM pixels `floor(255·(1 − v) + 0.5)` as uint8 (outputs.py:27), on the GPU.

    Raises ValueError("density values must lie in [0, 1]") like outputs.py:25-26."""
    t = _flat(v_phys)
    if t.numel() == 0:  # numpy's min() of an empty field raises ValueError (outputs.py:25)
        raise ValueError("zero-size density field")
    out = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    bad = torch.zeros(1, dtype=torch.int32, device=t.device)
    call("bsp_density_pixels", _dev.ptr(t), t.numel(), _dev.ptr(out), _dev.ptr(bad), _stream())
    if int(bad.item()):
        raise ValueError("density values must lie in [0, 1]")
    return out if _dev.is_tensor(v_phys) else out.cpu().numpy()


def pgm_header(nx: int, ny: int) -> bytes:
    return f"P5\n{nx} {ny}\n255\n".encode("ascii")


def write_snapshot(v_phys, nx: int, ny: int, path) -> None:
    """Binary PGM (P5, maxval 255), rows top to bottom, solid = black (outputs.py:21-30)."""
    shape = _dev.shape_of(v_phys) if _dev.is_tensor(v_phys) else np.shape(v_phys)
    if tuple(shape) != (nx * ny,):
        raise ValueError(f"field has length {tuple(shape)}, expected {nx * ny}")
    pixels = density_pixels(v_phys)
    if _dev.is_tensor(pixels):
        pixels = pixels.cpu().numpy()
    with open(path, "wb") as fh:
        fh.write(pgm_header(nx, ny))
        fh.write(pixels.tobytes())


def write_frame_pgm(frame: Frame, path) -> None:
    """A "pgm" Frame from `run(..., frame_sink=..., frame_kind="pgm")` as a PGM file."""
    if frame.kind != "pgm":
        raise ValueError(f"frame kind is {frame.kind!r}, expected 'pgm'")
    with open(path, "wb") as fh:
        fh.write(pgm_header(frame.nx, frame.ny))
        fh.write(frame.payload)
