"""The DiT attention block around the operator.

    x [B,S,dim] --QKV projection (library GEMM)--> qkv [B,S,3,H,d]
      --svgear_qkv_prologue (q/k RMSNorm + rotary embedding + head-major layout, one pass)-->
      q,k,v [B,H,S,d] --SVG-EAR attention (or dense, per the warm-up schedule)--> [B,H,S,d]
      --svgear_heads_to_tokens--> [B,S,H*d] --output projection (library GEMM)--> [B,S,dim]

The reference has no module of this kind (it stops at single (Q,K,V) matrices); the layout follows
the paper's two deployments: Wan2.2 (q/k RMSNorm over the whole token, 3-D rotary embedding on
interleaved pairs, all tokens are video tokens) and HunyuanVideo (per-head q/k RMSNorm, text tokens
appended after the video tokens and not rotated).  No CPU path: the two layout kernels live in
libsvgear.so and raise when the library or the device is missing.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from ._tensors import ShapeError, require_cuda, stream_ptr
from .schedule import SvgEarStack

_NORM = {"none": _lib.NORM_NONE, "head": _lib.NORM_HEAD, "token": _lib.NORM_TOKEN}
_ROPE = {"none": _lib.ROPE_NONE, "interleaved": _lib.ROPE_INTERLEAVED, "half_split": _lib.ROPE_HALF_SPLIT}


def rope_table_3d(grid, d, theta=10000.0, device=None):
    """(cos, sin) float32 [T*Hh*W, d/2] for a (T, Hh, W) latent grid, tokens in row-major (t, h, w)
    order.  The d/2 rotation frequencies are split over the three axes as Wan2.2 does: the time axis
    gets d/2 - 2*(d/2 // 3) of them, height and width d/2 // 3 each; inside an axis of n frequencies
    the i-th one is theta^(-i/n)."""
    t, hh, w = (int(g) for g in grid)
    half = d // 2
    n_hw = half // 3
    n_t = half - 2 * n_hw
    ang = []
    for size, nf in ((t, n_t), (hh, n_hw), (w, n_hw)):
        freq = theta ** (-torch.arange(nf, dtype=torch.float64) / nf)
        ang.append(torch.arange(size, dtype=torch.float64)[:, None] * freq[None, :])
    a = torch.cat([ang[0][:, None, None, :].expand(t, hh, w, n_t),
                   ang[1][None, :, None, :].expand(t, hh, w, n_hw),
                   ang[2][None, None, :, :].expand(t, hh, w, n_hw)], dim=-1).reshape(t * hh * w, half)
    cos, sin = a.cos().float(), a.sin().float()
    if device is not None:
        cos, sin = cos.to(device), sin.to(device)
    return cos.contiguous(), sin.contiguous()


def qkv_prologue(qkv, n_heads, *, norm="none", q_weight=None, k_weight=None, eps=1e-6, rope=None,
                 rope_mode="interleaved"):
    """qkv [B, S, 3*H*d] (or [B,S,3,H,d]) bf16 CUDA -> (q, k, v), each [B, H, S, d] bf16.

    norm : "none" | "head" (RMS over d) | "token" (RMS over H*d); weights float32 [H*d].
    rope : None or (cos, sin) float32 [L, d/2], L <= S: the first L tokens are rotated, the rest
           (appended text tokens) are not.  rope_mode: "interleaved" pairs (2i, 2i+1) or
           "half_split" pairs (i, i + d/2).
    """
    if norm not in _NORM:
        raise ValueError(f"unknown norm mode {norm!r}")
    if rope is not None and rope_mode not in ("interleaved", "half_split"):
        raise ValueError(f"unknown rope mode {rope_mode!r}")
    if qkv.ndim == 3:
        b, s, w = qkv.shape
        if w % (3 * n_heads):
            raise ShapeError(f"qkv width {w} is not 3 * {n_heads} heads * d")
        d = w // (3 * n_heads)
    elif qkv.ndim == 5 and qkv.shape[2] == 3 and qkv.shape[3] == n_heads:
        b, s, _, _, d = qkv.shape
    else:
        raise ShapeError(f"qkv must be [B,S,3*H*d] or [B,S,3,H,d], got {tuple(qkv.shape)}")
    if d not in (64, 128):
        raise ShapeError(f"head dimension must be 64 or 128 on the B200 path, got {d}")
    if n_heads * d > 8192:
        raise ShapeError(f"H*d = {n_heads * d} exceeds 8192")
    dev = require_cuda()
    x = qkv.to(dev, torch.bfloat16).contiguous()
    wq = wk = None
    if norm != "none":
        if q_weight is None or k_weight is None:
            raise ValueError("q_weight and k_weight are required with a norm")
        wq = q_weight.to(dev, torch.float32).reshape(-1).contiguous()
        wk = k_weight.to(dev, torch.float32).reshape(-1).contiguous()
        if wq.numel() != n_heads * d or wk.numel() != n_heads * d:
            raise ShapeError(f"norm weights must have {n_heads * d} entries")
    cos = sin = None
    rope_len = 0
    if rope is not None:
        cos = rope[0].to(dev, torch.float32).contiguous()
        sin = rope[1].to(dev, torch.float32).contiguous()
        if cos.shape != sin.shape or cos.ndim != 2 or cos.shape[1] != d // 2:
            raise ShapeError(f"rope tables must both be [L, {d // 2}], got {tuple(cos.shape)} / {tuple(sin.shape)}")
        rope_len = int(cos.shape[0])
        if rope_len > s:
            raise ShapeError(f"rope table has {rope_len} positions for {s} tokens")
    q = torch.empty((b, n_heads, s, d), dtype=torch.bfloat16, device=dev)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    ptr = lambda t: t.data_ptr() if t is not None else None
    rc = _lib.lib().svgear_qkv_prologue(
        b, s, n_heads, d, x.data_ptr(), _NORM[norm], ptr(wq), ptr(wk), float(eps),
        _ROPE[rope_mode] if rope is not None else _lib.ROPE_NONE, rope_len, ptr(cos), ptr(sin),
        q.data_ptr(), k.data_ptr(), v.data_ptr(), stream_ptr())
    _lib.check("svgear_qkv_prologue", rc)
    return q, k, v


def heads_to_tokens(x):
    """[B, H, S, d] bf16 -> [B, S, H*d] bf16."""
    if x.ndim != 4:
        raise ShapeError(f"expected [B,H,S,d], got {tuple(x.shape)}")
    b, h, s, d = x.shape
    if d not in (64, 128):
        raise ShapeError(f"head dimension must be 64 or 128 on the B200 path, got {d}")
    dev = require_cuda()
    xb = x.to(dev, torch.bfloat16).contiguous()
    out = torch.empty((b, s, h * d), dtype=torch.bfloat16, device=dev)
    rc = _lib.lib().svgear_heads_to_tokens(b, s, h, d, xb.data_ptr(), out.data_ptr(), stream_ptr())
    _lib.check("svgear_heads_to_tokens", rc)
    return out


class SvgEarSelfAttention(torch.nn.Module):
    """Self-attention block of a video DiT with SVG-EAR as the attention operator.

    dim = n_heads * head_dim.  `norm`: "token" (Wan2.2), "head" (HunyuanVideo) or "none".
    forward(x, stack, layer, step, rope=None) -> [B, S, dim]; `stack` (schedule.SvgEarStack)
    decides dense / cold / warm-started SVG-EAR for this (layer, step) and keeps the centroids.
    Inference only (the operator has no backward).
    """

    def __init__(self, dim, n_heads, *, norm="token", eps=1e-6, rope_mode="interleaved", bias=True,
                 device=None, dtype=torch.bfloat16):
        super().__init__()
        if dim % n_heads or dim // n_heads not in (64, 128):
            raise ShapeError(f"dim {dim} / heads {n_heads} must give a head dimension of 64 or 128")
        if norm not in _NORM:
            raise ValueError(f"unknown norm mode {norm!r}")
        self.dim, self.n_heads, self.head_dim = dim, n_heads, dim // n_heads
        self.norm, self.eps, self.rope_mode = norm, eps, rope_mode
        self.qkv = torch.nn.Linear(dim, 3 * dim, bias=bias, device=device, dtype=dtype)
        self.proj = torch.nn.Linear(dim, dim, bias=bias, device=device, dtype=dtype)
        self.q_norm_weight = torch.nn.Parameter(torch.ones(dim, device=device, dtype=torch.float32))
        self.k_norm_weight = torch.nn.Parameter(torch.ones(dim, device=device, dtype=torch.float32))
        with torch.no_grad():
            for lin in (self.qkv, self.proj):
                lin.weight.normal_(0.0, 1.0 / math.sqrt(dim))
                if bias:
                    lin.bias.zero_()

    @torch.no_grad()
    def forward(self, x, stack: SvgEarStack, layer=0, step=0, rope=None):
        if x.ndim != 3 or x.shape[-1] != self.dim:
            raise ShapeError(f"x must be [B, S, {self.dim}], got {tuple(x.shape)}")
        qkv = self.qkv(x)
        q, k, v = qkv_prologue(qkv, self.n_heads, norm=self.norm, q_weight=self.q_norm_weight,
                               k_weight=self.k_norm_weight, eps=self.eps, rope=rope,
                               rope_mode=self.rope_mode)
        o = stack.attend(layer, step, q, k, v)
        return self.proj(heads_to_tokens(o))
