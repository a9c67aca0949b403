"""Block-sparse executor on the GPU — host mirror of routedattn.attention (attention.py:37-219).

One fused kernel does the exact pass over the selected blocks and the centroid compensation of all
unselected blocks in a single online softmax (see csrc/attend_tc.cu, csrc/attend_ref.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import as_tokens, stream_ptr, workspace
from .clustering import ClusterModel, segment_means
from .router import BlockMask


@dataclass
class FlopCounters:  # attention.py:37-46
    exact_block: int = 0
    compensation: int = 0
    estimation: int = 0
    clustering: int = 0

    @property
    def total(self) -> int:
        return self.exact_block + self.compensation + self.estimation + self.clustering


@dataclass
class AttentionResult:  # attention.py:48-54
    output: torch.Tensor  # (N_q, d) in permuted row order (as the reference)
    lse: torch.Tensor     # (N_q,)
    flops: FlopCounters = field(default_factory=FlopCounters)
    density_used: object = 1.0


def exact_block_flops(d: int, density_entries: int) -> int:  # attention.py:212-214
    return 4 * d * density_entries


def compensation_flops(d: int, q_sizes, compensated_per_row) -> int:  # attention.py:217-219
    return int(4 * d * (np.asarray(q_sizes) * np.asarray(compensated_per_row)).sum())


def sparse_attend(q, k, v, q_model: ClusterModel, k_model: ClusterModel, mask: BlockMask, *,
                  dtype=torch.bfloat16, v_centroids=None, unpermute=False, variant=None) -> AttentionResult:
    """Full executor (attention.py:160-192).  Inputs cluster-contiguous for their models.

    dtype=torch.bfloat16 -> tcgen05 tensor-core executor (bf16 output);
    dtype=torch.float32  -> CUDA-core fp32 executor (the fp32 check mode).
    `unpermute=True` scatters rows back to original token order (inverse_permute_rows).
    `variant` (bf16 only) selects a measured alternative of the fused kernel instead of the default
    (two threads per query row, 64-key tiles): "one_thread_per_row" or "tile128".
    """
    if variant not in (None, "one_thread_per_row", "tile128"):
        raise ValueError(f"unknown executor variant {variant!r}")
    if variant is not None and dtype != torch.bfloat16:
        raise ValueError("executor variants exist for the bf16 tensor-core executor only")
    if mask.selected.shape[-1] == 0:
        raise ValueError("no key clusters: softmax over an empty set is undefined")
    if dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("dtype must be torch.bfloat16 or torch.float32")
    qp, was_2d = as_tokens(q, "q", check_finite=False)
    kp, _ = as_tokens(k, "k", check_finite=False)
    vp, _ = as_tokens(v, "v", check_finite=False)
    bh, n_q, d = qp.shape
    n_k = kp.shape[1]
    if vp.shape != kp.shape:
        raise ValueError(f"key/value row counts differ: {kp.shape[1]} vs {vp.shape[1]}")
    c_q, c_k = q_model.num_clusters, k_model.num_clusters
    dev = qp.device
    qs = q_model.sizes.view(bh, c_q).contiguous()
    qo = q_model.offsets.view(bh, c_q).contiguous()
    ks = k_model.sizes.view(bh, c_k).contiguous()
    ko = k_model.offsets.view(bh, c_k).contiguous()
    kc = k_model.centroids.view(bh, c_k, d).contiguous()
    vc = (segment_means(vp, ClusterModel(c_k, k_model.assignments, kc, ks, k_model.permutation, ko))
          if v_centroids is None else v_centroids.view(bh, c_k, d).contiguous())
    sel = mask.selected.to(dev).view(bh, c_q, c_k).to(torch.uint8).contiguous()
    out = torch.empty((bh, n_q, d), dtype=dtype, device=dev)
    lse = torch.empty((bh, n_q), dtype=torch.float32, device=dev)
    perm = q_model.permutation.view(bh, n_q).contiguous() if unpermute else None
    shape = _lib.Shape(bh, n_q, n_k, d, c_q, c_k)
    ws = workspace(_lib.workspace_bytes(shape), dev)
    rc = _lib.lib().svgear_sparse_attend(
        C.byref(shape), _lib.EXEC_FP32_CHECK if dtype == torch.float32 else (_lib.EXEC_BF16_TENSOR | {
            None: 0, "one_thread_per_row": _lib.ATTEND_ONE_THREAD_PER_ROW, "tile128": _lib.ATTEND_TILE128}[variant]),
        qp.data_ptr(), kp.data_ptr(), vp.data_ptr(), perm.data_ptr() if perm is not None else None,
        qs.data_ptr(), qo.data_ptr(), ks.data_ptr(), ko.data_ptr(), kc.data_ptr(), vc.data_ptr(),
        sel.data_ptr(), out.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_sparse_attend", rc)
    block = qs.long().unsqueeze(-1) * ks.long().unsqueeze(-2)
    ent = (block * sel.long()).sum(dim=(1, 2))
    n_comp = (c_k - sel.long().sum(dim=2))
    counters = FlopCounters(exact_block=exact_block_flops(d, int(ent.sum())),
                            compensation=int(4 * d * (qs.long() * n_comp).sum()))
    sq = (lambda t: t[0]) if was_2d else (lambda t: t)
    return AttentionResult(output=sq(out), lse=sq(lse), flops=counters, density_used=mask.density)
