"""Head-parallel sharding (subsystem 4): one process per GPU, contiguous head ranges, one
all_gather of the per-rank output slab.  The reference has no multi-device path;
heads are independent instances (analysis.py:207-239), so there is no data-path exchange before
the gather.  Host logic is backend-agnostic (NCCL on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(n_heads: int, world_size: int, rank: int):
    """Contiguous head range [lo, hi) owned by `rank`; the first n_heads % world_size ranks take
    one extra head.  world_size > n_heads leaves the surplus ranks with an empty range."""
    if n_heads < 0 or world_size < 1 or not (0 <= rank < world_size):
        raise ValueError(f"bad partition request: heads={n_heads} world={world_size} rank={rank}")
    base, extra = divmod(n_heads, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def head_seed(base_seed: int, batch_index: int, head_index: int, n_heads: int) -> int:
    """Seed of instance (b, h): independent of the world size, so results do not depend on how
    heads are sharded."""
    return base_seed + batch_index * n_heads + head_index


def gather_heads(local: torch.Tensor, n_heads: int, group=None, head_dim: int = 1):
    """All-gather per-rank slabs [B, H_local, ...] along the head dimension into [B, H, ...].

    Ranks may own different head counts (n_heads not divisible by the world size): slabs are
    padded to the largest count for the collective and trimmed afterwards.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    counts = [head_range(n_heads, world, r) for r in range(world)]
    widest = max(hi - lo for lo, hi in counts)
    pad_shape = list(local.shape)
    pad_shape[head_dim] = widest
    send = local
    if local.shape[head_dim] != widest:
        send = torch.zeros(pad_shape, dtype=local.dtype, device=local.device)
        send.narrow(head_dim, 0, local.shape[head_dim]).copy_(local)
    send = send.contiguous()
    if local.dtype == torch.bool:
        send = send.to(torch.uint8)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    parts = [p.narrow(head_dim, 0, hi - lo) for p, (lo, hi) in zip(parts, counts)]
    full = torch.cat(parts, dim=head_dim)
    return full.bool() if local.dtype == torch.bool else full


def sharded_svg_ear_attention(q, k, v, n_q_clusters, n_k_clusters, budget, *, group=None,
                              gather=True, op=None, **kwargs):
    """Run the operator on this rank's head range of replicated [B, H, S, d] inputs and gather
    the outputs (and masks) over the group.  `op` is injectable for CPU tests."""
    if op is None:
        from .operator import svg_ear_attention as op
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_heads = q.shape[1]
    lo, hi = head_range(n_heads, world, rank)
    seed = kwargs.pop("seed", 0)
    if hi > lo:
        out, mask = op(q[:, lo:hi], k[:, lo:hi], v[:, lo:hi], n_q_clusters, n_k_clusters, budget,
                       seed=seed + lo, **kwargs)[:2]
    else:
        out = q.new_zeros((q.shape[0], 0, q.shape[2], q.shape[3]))
        mask = torch.zeros((q.shape[0], 0, n_q_clusters, n_k_clusters), dtype=torch.bool, device=q.device)
    if not gather:
        return out, mask
    return gather_heads(out, n_heads, group), gather_heads(mask, n_heads, group)
