"""Two-GPU NCCL check of the head-parallel path with the REAL operator: the sharded result must
equal the single-GPU result bit for bit.  Skipped when fewer than two devices are
visible (the driver's GPU box has one)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_2603_08982_b200 as P
        g = torch.Generator().manual_seed(3)
        H, S, d, cq, ck = 6, 1536, 64, 12, 30
        q, k, v = (torch.randn(1, H, S, d, generator=g).to("cuda", torch.bfloat16) for _ in range(3))
        ok = True
        for init in ("device", "reference"):
            want = P.svg_ear_attention(q, k, v, cq, ck, 0.3, seed=4, init=init)
            got = P.sharded_svg_ear_attention(q, k, v, cq, ck, 0.3, seed=4, init=init)
            ok = ok and torch.equal(got[0], want[0]) and torch.equal(got[1], want[1])
        ret[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_gpus_equal_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert ret.get(0) is True and ret.get(1) is True
