"""world_size-2 gloo test of the head-parallel path (host logic only; the operator is injected)."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08982_b200.sharding import gather_heads, head_range, sharded_svg_ear_attention


def _fake_op(q, k, v, cq, ck, rho, *, seed=0, **kw):
    # deterministic function of (inputs, per-head seed) so any sharding must reproduce it
    h = q.shape[1]
    tag = torch.arange(seed, seed + h, dtype=q.dtype).view(1, h, 1, 1)
    out = q * 2 + k.mean(dim=2, keepdim=True) + v.sum(dim=(2, 3), keepdim=True) * 0 + tag
    mask = (torch.arange(cq * ck).view(1, 1, cq, ck) + torch.arange(seed, seed + h).view(1, h, 1, 1)) % 3 == 0
    return out, mask.expand(q.shape[0], h, cq, ck)


def _worker(rank, world, port, heads, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(1)
        q = torch.randn(2, heads, 6, 4, generator=g)
        k = torch.randn(2, heads, 6, 4, generator=g)
        v = torch.randn(2, heads, 6, 4, generator=g)
        out, mask = sharded_svg_ear_attention(q, k, v, 2, 3, 0.25, op=_fake_op, seed=10)
        want_out, want_mask = _fake_op(q, k, v, 2, 3, 0.25, seed=10)
        lo, hi = head_range(heads, world, rank)
        local = torch.full((2, hi - lo, 1), float(rank))
        ranks = gather_heads(local, heads)
        ok = (torch.equal(out, want_out) and torch.equal(mask, want_mask)
              and ranks.shape == (2, heads, 1)
              and all(float(ranks[0, h, 0]) == r for r in range(world)
                      for h in range(*head_range(heads, world, r))))
        ret[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(heads):
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, heads, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert ret.get(0) is True and ret.get(1) is True


def test_two_ranks_even_heads():
    _run(4)


def test_two_ranks_uneven_heads():
    _run(5)
