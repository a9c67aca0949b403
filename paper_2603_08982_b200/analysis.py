"""prepare / build_error_table — host mirror of the hot-path part of routedattn.analysis
(analysis.py:181-249)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._tensors import as_tokens
from .clustering import ClusterModel, kmeans, permute_rows
from .estimator import BlockErrorTable, estimate_errors, estimate_errors_streaming


@dataclass(frozen=True)
class Prepared:
    """Clustered, permuted instance ready for the sparse path (analysis.py:181-204)."""

    q_raw: torch.Tensor
    k_raw: torch.Tensor
    v_raw: torch.Tensor
    q_model: ClusterModel
    k_model: ClusterModel
    q: torch.Tensor  # cluster-contiguous
    k: torch.Tensor
    v: torch.Tensor

    @property
    def n_q(self) -> int:
        return self.q.shape[-2]

    @property
    def n_k(self) -> int:
        return self.k.shape[-2]

    @property
    def d(self) -> int:
        return self.q.shape[-1]


def side_seeds(seed):
    """(q_seed, k_seed) = SeedSequence(seed).generate_state(2)  (analysis.py:227)."""
    s = np.random.SeedSequence(seed).generate_state(2)
    return int(s[0]), int(s[1])


def prepare(q_raw, k_raw, v_raw, c_q: int, c_k: int, *, seed: int = 0, restarts: int = 1,
            q_init_centroids=None, k_init_centroids=None, max_iters: int = 25) -> Prepared:
    """Cluster both sides and permute the instance cluster-contiguous (analysis.py:207-239)."""
    q, q2 = as_tokens(q_raw, "q")
    k, _ = as_tokens(k_raw, "k")
    v, _ = as_tokens(v_raw, "v")
    if k.shape[1] != v.shape[1]:
        raise ValueError(f"key/value row counts differ: {k.shape[1]} vs {v.shape[1]}")
    if q2:
        q, k, v = q[0], k[0], v[0]
    # instance b of a batch is seeded like the operator seeds it: side_seeds(seed + b)
    bh = 1 if q2 else q.shape[0]
    seeds = [side_seeds(seed + b) for b in range(bh)]
    q_model = kmeans(q, c_q, seed=[s_[0] for s_ in seeds], restarts=restarts, init_centroids=q_init_centroids,
                     max_iters=max_iters)
    k_model = kmeans(k, c_k, seed=[s_[1] for s_ in seeds], restarts=restarts, init_centroids=k_init_centroids,
                     max_iters=max_iters)
    return Prepared(q_raw=q, k_raw=k, v_raw=v, q_model=q_model, k_model=k_model,
                    q=permute_rows(q, q_model), k=permute_rows(k, k_model), v=permute_rows(v, k_model))


def build_error_table(prep: Prepared, mode: str = "valueAware", tile_size: int = 64) -> BlockErrorTable:
    """Mode dispatch (analysis.py:242-249)."""
    if mode == "valueAware":
        return estimate_errors_streaming(prep.q_model, prep.k_model, prep.k, prep.v, tile_size=tile_size)
    if mode == "plain":
        return estimate_errors(prep.q_model, prep.k_model, prep.k)
    raise ValueError(f"unknown estimator mode {mode!r}")
