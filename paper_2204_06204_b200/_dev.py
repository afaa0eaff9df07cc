"""Device plumbing: numpy <-> CUDA tensors, raw pointers and the current stream.

Public functions accept numpy arrays (the reference's types) or CUDA torch
tensors.  Results come back in the caller's kind: numpy in -> numpy out
(computed on the GPU), CUDA tensor in -> CUDA tensor out (no host copy).
"""
from __future__ import annotations

import numpy as np
import torch

from ._native import NativeUnavailable, load

_F64 = torch.float64


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def shape_of(x) -> tuple:
    return tuple(x.shape)


def dev_f64(x) -> torch.Tensor:
    """CUDA, float64, contiguous view/copy of x (numpy or tensor)."""
    d = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device=d, dtype=_F64)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(a).to(d, non_blocking=False)


def dev_u8(x) -> torch.Tensor:
    d = require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=d, dtype=torch.uint8).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint8))
    return torch.from_numpy(a).to(d)


def empty(n: int) -> torch.Tensor:
    return torch.empty(int(n), dtype=_F64, device=require_cuda())


def zeros(n: int) -> torch.Tensor:
    return torch.zeros(int(n), dtype=_F64, device=require_cuda())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def like(ref, t: torch.Tensor):
    """Return t in the kind of `ref` (numpy -> host ndarray)."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.cpu().numpy()


def host_f64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().to("cpu", torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)
