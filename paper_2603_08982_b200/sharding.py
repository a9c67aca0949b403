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
    """Seed of instance (b, h) = base_seed + its GLOBAL instance index b * n_heads + h: independent
    of the world size, so results do not depend on how heads are sharded.  This is the rule the
    operator applies when it is told which heads it holds (head_offset, total_heads)."""
    return base_seed + batch_index * n_heads + head_index


def _padded(local, widest, head_dim):
    if local.shape[head_dim] == widest:
        return local.contiguous()
    shape = list(local.shape)
    shape[head_dim] = widest
    send = torch.zeros(shape, dtype=local.dtype, device=local.device)
    send.narrow(head_dim, 0, local.shape[head_dim]).copy_(local)
    return send


def gather_heads(local: torch.Tensor, n_heads: int, group=None, head_dim: int = 1, out=None):
    """All-gather per-rank slabs [B, H_local, ...] along the head dimension into [B, H, ...].

    When every rank owns the same head count and B == 1 (the layout of a head-parallel attention
    layer) the slabs land directly in the final buffer with ONE all_gather_into_tensor — rank r's
    heads are the contiguous range r of `out`, no staging copy.  Otherwise (uneven head counts, or a
    batch dimension outside the head dimension) slabs are padded to the largest count, gathered,
    trimmed and concatenated.  `out` (optional) is the preallocated [B, H, ...] result.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        if out is not None:
            out.copy_(local)
            return out
        return local
    as_bool = local.dtype == torch.bool
    counts = [head_range(n_heads, world, r) for r in range(world)]
    widest = max(hi - lo for lo, hi in counts)
    even = all(hi - lo == widest for lo, hi in counts)
    lead = 1
    for s_ in local.shape[:head_dim]:
        lead *= s_
    shape = list(local.shape)
    shape[head_dim] = n_heads
    if even and lead == 1:
        send = local.contiguous()
        full = out if out is not None else torch.empty(shape, dtype=local.dtype, device=local.device)
        if as_bool:
            send, recv = send.view(torch.uint8), full.view(torch.uint8)
        else:
            recv = full
        dist.all_gather_into_tensor(recv.view(-1), send.view(-1), group=group)  # flat: rank r -> range r
        return full
    send = _padded(local, widest, head_dim)
    if as_bool:
        send = send.to(torch.uint8)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    parts = [p.narrow(head_dim, 0, hi - lo) for p, (lo, hi) in zip(parts, counts)]
    full = torch.cat(parts, dim=head_dim)
    full = full.bool() if as_bool else full
    if out is not None:
        out.copy_(full)
        return out
    return full


def sharded_svg_ear_attention(q, k, v, n_q_clusters, n_k_clusters, budget, *, group=None,
                              gather=True, op=None, **kwargs):
    """Run the operator on this rank's head range of replicated [B, H, S, d] inputs and gather
    the outputs (and masks) over the group.  Every instance is seeded by its global (batch, head)
    index (`head_offset`, `total_heads` of the operator), so the result equals the unsharded call
    for every world size.  `op` is injectable for CPU tests."""
    if op is None:
        from .operator import svg_ear_attention as op
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n_heads = q.shape[1]
    lo, hi = head_range(n_heads, world, rank)
    if hi > lo:
        out, mask = op(q[:, lo:hi], k[:, lo:hi], v[:, lo:hi], n_q_clusters, n_k_clusters, budget,
                       head_offset=lo, total_heads=n_heads, **kwargs)[:2]
    else:
        out = q.new_zeros((q.shape[0], 0, q.shape[2], q.shape[3]))
        mask = torch.zeros((q.shape[0], 0, n_q_clusters, n_k_clusters), dtype=torch.bool, device=q.device)
    if not gather:
        return out, mask
    return gather_heads(out, n_heads, group), gather_heads(mask, n_heads, group)
