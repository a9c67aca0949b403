"""world_size-2 gloo test of the head-parallel path (host logic only; the operator is injected)."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08982_b200.sharding import gather_heads, head_range, head_seed, sharded_svg_ear_attention


def _fake_op(q, k, v, cq, ck, rho, *, seed=0, head_offset=0, total_heads=None, **kw):
    # deterministic function of (inputs, seed of the GLOBAL (batch, head) index), the operator's rule:
    # any sharding must reproduce it, including the batch rows beyond the first
    b, h = q.shape[0], q.shape[1]
    total = h if total_heads is None else total_heads
    ids = torch.stack([torch.tensor([head_seed(seed, bi, head_offset + hi, total) for hi in range(h)])
                       for bi in range(b)])
    tag = ids.to(q.dtype).view(b, h, 1, 1)
    out = q * 2 + k.mean(dim=2, keepdim=True) + v.sum(dim=(2, 3), keepdim=True) * 0 + tag
    mask = (torch.arange(cq * ck).view(1, 1, cq, ck) + ids.view(b, h, 1, 1)) % 3 == 0
    return out, mask


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
        # B = 1 with even head counts takes the zero-copy all_gather_into_tensor path, also into a
        # caller-provided buffer and for bool masks
        o1, m1 = sharded_svg_ear_attention(q[:1], k[:1], v[:1], 2, 3, 0.25, op=_fake_op, seed=10)
        w1, wm1 = _fake_op(q[:1], k[:1], v[:1], 2, 3, 0.25, seed=10)
        ok = ok and torch.equal(o1, w1) and torch.equal(m1, wm1)
        buf = torch.empty_like(w1)
        part = _fake_op(q[:1, lo:hi], k[:1, lo:hi], v[:1, lo:hi], 2, 3, 0.25, seed=10, head_offset=lo,
                        total_heads=heads)[0]
        got = gather_heads(part, heads, out=buf)
        ok = ok and got.data_ptr() == buf.data_ptr() and torch.equal(buf, w1)
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
