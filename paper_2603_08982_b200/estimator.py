"""Block error tables on the GPU — host mirror of routedattn.estimator (estimator.py:50-253)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import as_tokens, stream_ptr, workspace
from .clustering import ClusterModel, segment_means


def plain_key_flops(d: int) -> int:  # estimator.py:38-39
    return 2 * d + 4


def value_aware_key_flops(d: int) -> int:  # estimator.py:42-43
    return 6 * d + 4


@dataclass(frozen=True)
class BlockErrorTable:
    """Per-block stabilised error sums plus the sizes routing needs (estimator.py:50-73)."""

    error_sum: torch.Tensor    # (C_q, C_k) float64, all >= 0
    q_sizes: torch.Tensor      # (C_q,) int32
    k_sizes: torch.Tensor      # (C_k,) int32
    stabilizers: torch.Tensor  # (C_q,) float32
    mode: str
    flops: int

    @property
    def block_sizes(self):
        return self.q_sizes.long().unsqueeze(-1) * self.k_sizes.long().unsqueeze(-2)

    @property
    def total_entries(self) -> int:
        q = self.q_sizes.long().sum(dim=-1)
        k = self.k_sizes.long().sum(dim=-1)
        return int((q * k).flatten()[0])

    @property
    def raw_error_sum(self):
        return self.error_sum * torch.exp(2.0 * self.stabilizers.double()).unsqueeze(-1)


def _run(q_model: ClusterModel, k_model: ClusterModel, k, v, mode, fp32_check=False, v_centroids=None):
    kp, was_2d = as_tokens(k, "k", check_finite=False)
    bh, n_k, d = kp.shape
    vp = None
    if mode == "valueAware":
        vp, _ = as_tokens(v, "v", check_finite=False)
        if vp.shape != kp.shape:
            raise ValueError(f"key/value shapes differ: {tuple(kp.shape)} vs {tuple(vp.shape)}")
    c_q, c_k = q_model.num_clusters, k_model.num_clusters
    dev = kp.device
    qc = q_model.centroids.view(bh, c_q, d).contiguous()
    kc = k_model.centroids.view(bh, c_k, d).contiguous()
    qs = q_model.sizes.view(bh, c_q).contiguous()
    ks = k_model.sizes.view(bh, c_k).contiguous()
    ko = k_model.offsets.view(bh, c_k).contiguous()
    vc = None
    if vp is not None:  # v̄ (clustering.segment_means): computed here unless the caller already has it
        vc = v_centroids.view(bh, c_k, d).float().contiguous() if v_centroids is not None else \
            segment_means(vp, ClusterModel(c_k, k_model.assignments, kc, ks, k_model.permutation, ko))
    err = torch.empty((bh, c_q, c_k), dtype=torch.float64, device=dev)
    stab = torch.empty((bh, c_q), dtype=torch.float32, device=dev)
    n_q = int(qs[0].sum())
    shape = _lib.Shape(bh, max(n_q, c_q), n_k, d, c_q, c_k)
    ws = workspace(_lib.workspace_bytes(shape), dev)
    rc = _lib.lib().svgear_error_table(
        C.byref(shape), _lib.EXEC_FP32_CHECK if fp32_check else _lib.EXEC_BF16_TENSOR,
        _lib.EST_VALUE_AWARE if mode == "valueAware" else _lib.EST_PLAIN,
        qc.data_ptr(), kc.data_ptr(), vc.data_ptr() if vc is not None else None, kp.data_ptr(),
        vp.data_ptr() if vp is not None else None, qs.data_ptr(), ks.data_ptr(), ko.data_ptr(),
        err.data_ptr(), stab.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_error_table", rc)
    per_key = value_aware_key_flops(d) if mode == "valueAware" else plain_key_flops(d)
    sq = (lambda t: t[0]) if was_2d else (lambda t: t)
    return BlockErrorTable(error_sum=sq(err), q_sizes=sq(qs), k_sizes=sq(ks), stabilizers=sq(stab),
                           mode=mode, flops=c_q * n_k * per_key)


def estimate_errors_streaming(q_model, k_model, k, v, *, tile_size: int = 64, fp32_check=False, v_centroids=None):
    """Value-aware table (estimator.py:187-253).  `k`, `v` cluster-contiguous for k_model.  The
    result does not depend on the tile size (the kernel streams 32-key tiles).  `v_centroids`
    (optional, [.., C_k, d] float32 = segment_means(v, k_model)) saves recomputing them."""
    if tile_size < 1:
        raise ValueError(f"tile_size must be >= 1, got {tile_size}")
    return _run(q_model, k_model, k, v, "valueAware", fp32_check, v_centroids)


def estimate_errors_value_aware(q_model, k_model, k, v):
    """Same quantity as the streaming route (estimator.py:151-184)."""
    return _run(q_model, k_model, k, v, "valueAware")


def estimate_errors(q_model, k_model, k):
    """Plain-mode table (estimator.py:120-148)."""
    return _run(q_model, k_model, k, None, "plain")
