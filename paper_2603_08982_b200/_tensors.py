"""Input validation and device plumbing shared by the host-side mirror modules.

Validation mirrors routedattn.linalg.as_token_matrix (linalg.py:21-32): token data must be 2-D
(one instance) — the batched form [bh, n, d] is this package's extension — and finite.  Validation
happens BEFORE the CUDA requirement is checked so argument errors surface identically on any box;
a valid call without a CUDA device raises (there is no CPU fallback).
"""

from __future__ import annotations

import numpy as np
import torch


class ShapeError(ValueError):
    """Operand dimensions do not line up (same role as routedattn.linalg.ShapeError)."""


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2603_08982_b200 needs a CUDA device (B200, sm_100a): the operator has no CPU "
            "fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_tokens(data, name="token matrix", check_finite=True):
    """-> (bf16 CUDA tensor [bh, n, d], was_2d).  numpy / torch, any float dtype."""
    if isinstance(data, torch.Tensor):
        t = data
    else:
        arr = np.asarray(data)
        if arr.dtype == object or not np.issubdtype(arr.dtype, np.number):
            raise ValueError(f"{name} must be numeric")
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32 if arr.dtype != np.float64 else np.float64))
    if t.ndim not in (2, 3):
        raise ShapeError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if check_finite and not bool(torch.isfinite(t).all()):
        raise ValueError(f"{name} contains non-finite entries")
    if t.shape[-1] not in (64, 128):
        raise ShapeError(f"{name}: head dimension must be 64 or 128 on the B200 path, got {t.shape[-1]}")
    dev = require_cuda()
    was_2d = t.ndim == 2
    t = t.to(device=dev, dtype=torch.bfloat16).contiguous()
    return (t.unsqueeze(0) if was_2d else t), was_2d


def as_f32(data, shape, name):
    dev = require_cuda()
    t = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
    t = t.to(device=dev, dtype=torch.float32).contiguous()
    if tuple(t.shape) != tuple(shape):
        if t.ndim == len(shape) - 1 and tuple(t.shape) == tuple(shape[1:]) and shape[0] == 1:
            t = t.unsqueeze(0)
        else:
            raise ShapeError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def as_i32(data, shape, name):
    dev = require_cuda()
    t = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
    t = t.to(device=dev, dtype=torch.int32).contiguous()
    if tuple(t.shape) != tuple(shape):
        if tuple(t.shape) == tuple(shape[1:]) and shape[0] == 1:
            t = t.unsqueeze(0)
        else:
            raise ShapeError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def workspace(nbytes, device):
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device)
