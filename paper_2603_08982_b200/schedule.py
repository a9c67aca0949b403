"""Denoising-run schedules around the operator: dense warm-up and warm-started,
few-iteration k-means across denoising steps.

* Dense warm-up (Table `config`): the first `time_warm` of
  `total_steps` diffusion steps and the first `layer_warm` of `total_layers` layers run dense
  attention; every other (layer, step) runs SVG-EAR.  Wan2.2 / HunyuanVideo: 10/50 and 1/40.
* Warm start (clustering.py:158-163, `kmeans(..., init_centroids=...)`): Lloyd at step t of a layer
  starts from the centroids that layer produced at step t-1, with a small iteration cap.  The
  reference adds the warm start as one more run of its restart pool; here it REPLACES the seeded
  run (one Lloyd run per side per call), i.e. it is exactly `_lloyd(tokens, k, warm_iters,
  previous_centroids)` (clustering.py:104-141) — the parity test hands the same centres to the
  oracle's `lloyd`.

`SvgEarStack` holds the per-layer centroid cache and one workspace for all layers; it has no CPU
path (dense steps go through the library SDPA exactly as the paper runs FlashAttention there).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .operator import operator_workspace_bytes, svg_ear_attention


@dataclass(frozen=True)
class WarmupSchedule:
    """Which (layer, step) pairs run dense attention (PAPER.md Table `config`)."""

    total_steps: int = 50
    time_warm: int = 10
    total_layers: int = 40
    layer_warm: int = 1

    def __post_init__(self):
        if self.total_steps < 1 or self.total_layers < 1:
            raise ValueError("total_steps and total_layers must be >= 1")
        if not (0 <= self.time_warm <= self.total_steps):
            raise ValueError(f"time_warm must be in [0, {self.total_steps}], got {self.time_warm}")
        if not (0 <= self.layer_warm <= self.total_layers):
            raise ValueError(f"layer_warm must be in [0, {self.total_layers}], got {self.layer_warm}")

    @classmethod
    def wan22(cls):
        return cls(50, 10, 40, 1)

    @classmethod
    def hunyuan(cls, total_layers=60):
        return cls(50, 10, total_layers, 1)

    @classmethod
    def none(cls, total_steps=50, total_layers=40):
        return cls(total_steps, 0, total_layers, 0)

    def is_dense(self, layer: int, step: int) -> bool:
        if not (0 <= layer < self.total_layers):
            raise IndexError(f"layer {layer} outside [0, {self.total_layers})")
        if not (0 <= step < self.total_steps):
            raise IndexError(f"step {step} outside [0, {self.total_steps})")
        return step < self.time_warm or layer < self.layer_warm

    @property
    def sparse_calls(self) -> int:
        return (self.total_steps - self.time_warm) * (self.total_layers - self.layer_warm)

    @property
    def dense_calls(self) -> int:
        return self.total_steps * self.total_layers - self.sparse_calls


@dataclass
class _LayerState:
    q_centroids: torch.Tensor | None = None
    k_centroids: torch.Tensor | None = None
    last_step: int = -1
    q_iters: torch.Tensor | None = None
    k_iters: torch.Tensor | None = None


@dataclass
class SvgEarStack:
    """SVG-EAR attention for every layer of a denoising run.

    `attend(layer, step, q, k, v)` returns the attention output [B, H, S, d] (original token
    order).  Sparse calls start k-means from the layer's previous centroids when `warm_start` is
    on and the previous sparse call of that layer was step-1 with the same shape; otherwise they
    seed on the device (`init`) and run up to `cold_iters` Lloyd iterations.

    Classifier-free guidance runs every layer twice per step (conditional and unconditional
    branch): pass `branch=0` / `branch=1` so that each branch keeps its own centroid cache and
    warm-starts from ITS previous step (one cache per (layer, branch); a single cache would see
    the second call of a step as "not step-1" and fall back to a cold start every time).
    """

    n_q_clusters: int
    n_k_clusters: int
    budget: float
    budget_mode: str = "globalDensity"
    schedule: WarmupSchedule = field(default_factory=WarmupSchedule.wan22)
    warm_start: bool = True
    cold_iters: int = 25
    warm_iters: int = 4
    init: str = "device"
    seed: int = 0
    estimator: str = "valueAware"
    _layers: dict = field(default_factory=dict, repr=False)
    _ws: torch.Tensor | None = field(default=None, repr=False)
    calls: dict = field(default_factory=lambda: {"dense": 0, "cold": 0, "warm": 0}, repr=False)

    def __post_init__(self):
        if self.cold_iters < 1 or self.warm_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {min(self.cold_iters, self.warm_iters)}")

    def reset(self, release_workspace=False):
        """Forget every layer's centroids (start of a new denoising run); optionally also drop the
        cached workspace buffer."""
        self._layers.clear()
        self.calls = {"dense": 0, "cold": 0, "warm": 0}
        if release_workspace:
            self._ws = None

    def plan(self, layer: int, step: int, q=None, k=None, branch: int = 0) -> str:
        """'dense' | 'cold' | 'warm' — what `attend(layer, step, ...)` does now.  A warm start needs
        the (layer, branch)'s centroids from step - 1 and, when q and k are given, centroids of their
        shape."""
        if self.schedule.is_dense(layer, step):
            return "dense"
        st = self._layers.get((layer, branch))
        if not (self.warm_start and st is not None and st.q_centroids is not None and st.last_step == step - 1):
            return "cold"
        if q is not None and k is not None:
            want_q = tuple(q.shape[:-2]) + (self.n_q_clusters, q.shape[-1])
            want_k = tuple(k.shape[:-2]) + (self.n_k_clusters, k.shape[-1])
            if tuple(st.q_centroids.shape) != want_q or tuple(st.k_centroids.shape) != want_k:
                return "cold"  # the layer's shape changed: its cached centres are meaningless
        return "warm"

    def _workspace(self, bh, n_q, n_k, d, device):
        need = operator_workspace_bytes(bh, n_q, n_k, d, self.n_q_clusters, self.n_k_clusters)
        if self._ws is None or self._ws.numel() < need or self._ws.device != device:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def attend(self, layer, step, q, k, v, *, return_mask=False, branch: int = 0):
        mode = self.plan(layer, step, q, k, branch)
        self.calls[mode] += 1
        if mode == "dense":
            out = torch.nn.functional.scaled_dot_product_attention(q, k, v)
            return (out, None) if return_mask else out
        st = self._layers.setdefault((layer, branch), _LayerState())
        if mode == "warm":
            kw = dict(q_init=st.q_centroids, k_init=st.k_centroids, kmeans_iters=self.warm_iters)
        else:
            kw = dict(init=self.init, kmeans_iters=self.cold_iters)
        lead = q.shape[:-2]
        bh = 1
        for x in lead:
            bh *= int(x)
        out, mask, aux = svg_ear_attention(
            q, k, v, self.n_q_clusters, self.n_k_clusters, self.budget, budget_mode=self.budget_mode,
            seed=self.seed + layer, estimator=self.estimator, return_aux=True,
            workspace_buffer=self._workspace(bh, q.shape[-2], k.shape[-2], q.shape[-1], q.device), **kw)
        st.q_centroids, st.k_centroids = aux["q_centroids"], aux["k_centroids"]
        st.q_iters, st.k_iters = aux["q_iters"], aux["k_iters"]
        st.last_step = step
        return (out, mask) if return_mask else out

    def lloyd_iterations(self, layer, branch: int = 0):
        """(query-side, key-side) Lloyd iteration counts [bh] of the (layer, branch)'s last sparse call."""
        st = self._layers.get((layer, branch))
        return (None, None) if st is None else (st.q_iters, st.k_iters)
