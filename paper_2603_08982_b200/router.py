"""Budgeted block routing on the GPU — host mirror of routedattn.router (router.py:33-280)."""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._tensors import require_cuda, stream_ptr, workspace
from .estimator import BlockErrorTable

FILL_REMAINDER = "fillRemainder"
STOP_AT_FIRST_OVERFLOW = "stopAtFirstOverflow"
_OVERSHOOT = {FILL_REMAINDER: _lib.FILL_REMAINDER, STOP_AT_FIRST_OVERFLOW: _lib.STOP_AT_FIRST_OVERFLOW}


@dataclass(frozen=True)
class DensityBudget:
    """Compute budget for routing (router.py:33-65)."""

    mode: str
    rho: Optional[float] = None
    p: Optional[float] = None
    overshoot: str = FILL_REMAINDER

    def __post_init__(self):
        if self.mode == "globalDensity":
            if self.rho is None or not (0.0 <= self.rho <= 1.0):
                raise ValueError(f"globalDensity budget needs rho in [0, 1], got {self.rho}")
        elif self.mode == "perClusterTopP":
            if self.p is None or not (0.0 < self.p <= 1.0):
                raise ValueError(f"perClusterTopP budget needs p in (0, 1], got {self.p}")
        else:
            raise ValueError(f"unknown budget mode {self.mode!r}")
        if self.overshoot not in _OVERSHOOT:
            raise ValueError(f"unknown overshoot policy {self.overshoot!r}")

    @staticmethod
    def global_density(rho: float, overshoot: str = FILL_REMAINDER) -> "DensityBudget":
        return DensityBudget(mode="globalDensity", rho=rho, overshoot=overshoot)

    @staticmethod
    def top_p(p: float, overshoot: str = FILL_REMAINDER) -> "DensityBudget":
        return DensityBudget(mode="perClusterTopP", p=p, overshoot=overshoot)


@dataclass(frozen=True)
class BlockMask:
    """Boolean routing decision per block (router.py:68-78).  True = computed exactly."""

    selected: torch.Tensor  # (C_q, C_k) bool
    density_entries: object  # int (one instance) or int64 tensor [bh]
    density: object


def entry_capacity(rho: float, total_entries: int) -> int:
    """Entry budget implied by a target density (router.py:93-97) — same float64 arithmetic."""
    return int(math.floor(rho * total_entries + 1e-9))


def mask_from_selected(selected, block_sizes) -> BlockMask:  # router.py:81-85
    selected = torch.as_tensor(selected, dtype=torch.bool)
    sizes = torch.as_tensor(block_sizes).to(selected.device).long()
    ent = (sizes * selected).sum(dim=(-2, -1))
    tot = sizes.sum(dim=(-2, -1))
    if selected.ndim == 2:
        return BlockMask(selected, int(ent), int(ent) / int(tot))
    return BlockMask(selected, ent, ent.double() / tot.double())


def _finish(mask_u8, entries, total, was_2d):
    sel = mask_u8.bool()
    if was_2d:
        e = int(entries[0])
        return BlockMask(sel[0], e, e / total)
    return BlockMask(sel, entries, entries.double() / float(total))


def route_error_aware_entries(table: BlockErrorTable, capacity_entries: int, *,
                              overshoot: str = FILL_REMAINDER,
                              single_item_fallback: bool = True) -> BlockMask:
    """Greedy error-to-cost routing under an explicit entry budget (router.py:124-142)."""
    if overshoot not in _OVERSHOOT:
        raise ValueError(f"unknown overshoot policy {overshoot!r}")
    dev = require_cuda()
    err = torch.as_tensor(table.error_sum).to(dev, torch.float64).contiguous()
    was_2d = err.ndim == 2
    if was_2d:
        err = err.unsqueeze(0)
    bh, c_q, c_k = err.shape
    qs = torch.as_tensor(table.q_sizes).to(dev, torch.int32).view(bh, c_q).contiguous()
    ks = torch.as_tensor(table.k_sizes).to(dev, torch.int32).view(bh, c_k).contiguous()
    mask = torch.empty((bh, c_q, c_k), dtype=torch.uint8, device=dev)
    entries = torch.empty((bh,), dtype=torch.int64, device=dev)
    ws = workspace(bh * c_q * c_k * 8 + 1024, dev)
    rc = _lib.lib().svgear_route_error_aware(
        bh, c_q, c_k, err.data_ptr(), qs.data_ptr(), ks.data_ptr(), int(capacity_entries),
        _OVERSHOOT[overshoot], 1 if single_item_fallback else 0, mask.data_ptr(), entries.data_ptr(),
        ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_route_error_aware", rc)
    total = int(qs[0].long().sum()) * int(ks[0].long().sum())
    return _finish(mask, entries, total, was_2d)


def route_error_aware(table: BlockErrorTable, budget: DensityBudget, *, q_centroids=None,
                      k_centroids=None, single_item_fallback: bool = True,
                      size_weighted_scores: bool = True) -> BlockMask:
    """Greedy error-to-cost routing under the given budget (router.py:145-190)."""
    if budget.mode == "globalDensity":
        return route_error_aware_entries(
            table, entry_capacity(budget.rho, table.total_entries), overshoot=budget.overshoot,
            single_item_fallback=single_item_fallback)
    if q_centroids is None or k_centroids is None:
        raise ValueError("perClusterTopP routing needs q_centroids and k_centroids")
    if not size_weighted_scores:
        raise NotImplementedError("only size-weighted scores run on the GPU path")
    if budget.overshoot not in _OVERSHOOT:
        raise ValueError(f"unknown overshoot policy {budget.overshoot!r}")
    dev = require_cuda()
    err = torch.as_tensor(table.error_sum).to(dev, torch.float64).contiguous()
    qc = torch.as_tensor(q_centroids).to(dev, torch.float32).contiguous()
    kc = torch.as_tensor(k_centroids).to(dev, torch.float32).contiguous()
    was_2d = err.ndim == 2
    if was_2d:
        err, qc, kc = err.unsqueeze(0), qc.unsqueeze(0), kc.unsqueeze(0)
    bh, c_q, c_k = err.shape
    d = qc.shape[-1]
    qs = torch.as_tensor(table.q_sizes).to(dev, torch.int32).view(bh, c_q).contiguous()
    ks = torch.as_tensor(table.k_sizes).to(dev, torch.int32).view(bh, c_k).contiguous()
    n_q, n_k = int(qs[0].long().sum()), int(ks[0].long().sum())
    shape = _lib.Shape(bh, n_q, n_k, d, c_q, c_k)
    mask = torch.empty((bh, c_q, c_k), dtype=torch.uint8, device=dev)
    entries = torch.empty((bh,), dtype=torch.int64, device=dev)
    ws = workspace(bh * c_q * c_k * 8 + 1024, dev)
    rc = _lib.lib().svgear_route_error_aware_top_p(
        C.byref(shape), err.data_ptr(), qc.data_ptr(), kc.data_ptr(), qs.data_ptr(), ks.data_ptr(),
        float(budget.p), _OVERSHOOT[budget.overshoot], 1 if single_item_fallback else 0, mask.data_ptr(),
        entries.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_route_error_aware_top_p", rc)
    return _finish(mask, entries, n_q * n_k, was_2d)


def route_score(q_centroids, k_centroids, q_sizes, k_sizes, budget: DensityBudget, *,
                size_weighted: bool = True) -> BlockMask:
    """Cluster-mass (SVG2-style) routing at a global density (router.py:253-280)."""
    if budget.mode != "globalDensity":
        raise ValueError("route_score is defined for the globalDensity budget")
    if not size_weighted:
        raise NotImplementedError("only size-weighted scores run on the GPU path")
    dev = require_cuda()
    qc = torch.as_tensor(q_centroids).to(dev, torch.float32).contiguous()
    kc = torch.as_tensor(k_centroids).to(dev, torch.float32).contiguous()
    was_2d = qc.ndim == 2
    if was_2d:
        qc, kc = qc.unsqueeze(0), kc.unsqueeze(0)
    bh, c_q, d = qc.shape
    c_k = kc.shape[1]
    qs = torch.as_tensor(q_sizes).to(dev, torch.int32).view(bh, c_q).contiguous()
    ks = torch.as_tensor(k_sizes).to(dev, torch.int32).view(bh, c_k).contiguous()
    n_q, n_k = int(qs[0].long().sum()), int(ks[0].long().sum())
    shape = _lib.Shape(bh, n_q, n_k, d, c_q, c_k)
    ws = workspace(_lib.workspace_bytes(shape), dev)
    mask = torch.empty((bh, c_q, c_k), dtype=torch.uint8, device=dev)
    entries = torch.empty((bh,), dtype=torch.int64, device=dev)
    rc = _lib.lib().svgear_route_score(
        C.byref(shape), qc.data_ptr(), kc.data_ptr(), qs.data_ptr(), ks.data_ptr(),
        entry_capacity(budget.rho, n_q * n_k), _OVERSHOOT[budget.overshoot], mask.data_ptr(),
        entries.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_route_score", rc)
    return _finish(mask, entries, n_q * n_k, was_2d)


def score_top_p(q_centroids, k_centroids, q_sizes, k_sizes, p: float, *, size_weighted: bool = True) -> BlockMask:
    """Per-row minimal prefix of cluster mass reaching cumulative p (router.py:209-236): each
    query-cluster row softmaxes q̄·k̄/sqrt(d) + ln|k_c|; blocks are taken in descending mass order
    (ties to the lower key-cluster index) until the cumulative mass reaches p; p = 1 selects all."""
    if not (0.0 < p <= 1.0):
        raise ValueError(f"p must be in (0, 1], got {p}")
    if not size_weighted:
        raise NotImplementedError("only size-weighted scores run on the GPU path")
    dev = require_cuda()
    qc = torch.as_tensor(q_centroids).to(dev, torch.float32).contiguous()
    kc = torch.as_tensor(k_centroids).to(dev, torch.float32).contiguous()
    was_2d = qc.ndim == 2
    if was_2d:
        qc, kc = qc.unsqueeze(0), kc.unsqueeze(0)
    bh, c_q, d = qc.shape
    c_k = kc.shape[1]
    qs = torch.as_tensor(q_sizes).to(dev, torch.int32).view(bh, c_q).contiguous()
    ks = torch.as_tensor(k_sizes).to(dev, torch.int32).view(bh, c_k).contiguous()
    n_q, n_k = int(qs[0].long().sum()), int(ks[0].long().sum())
    shape = _lib.Shape(bh, n_q, n_k, d, c_q, c_k)
    mask = torch.empty((bh, c_q, c_k), dtype=torch.uint8, device=dev)
    entries = torch.empty((bh,), dtype=torch.int64, device=dev)
    ws = workspace(bh * c_q * c_k * 8 + 1024, dev)
    rc = _lib.lib().svgear_route_score_top_p(
        C.byref(shape), qc.data_ptr(), kc.data_ptr(), qs.data_ptr(), ks.data_ptr(), float(p), mask.data_ptr(),
        entries.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_route_score_top_p", rc)
    return _finish(mask, entries, n_q * n_k, was_2d)


def relaxed_objective(table: BlockErrorTable, mask: BlockMask) -> float:  # router.py:297-299
    return float(table.error_sum[~mask.selected].sum())
