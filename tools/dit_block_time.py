"""Times the two layout kernels of the DiT attention block (svgear_qkv_prologue, svgear_heads_to_tokens)
at a workload shape against the HBM roofline (algorithmic bytes = one read + one write of q, k, v /
of the output), and one whole SvgEarSelfAttention block (projections are library GEMMs).

    python tools/dit_block_time.py [--workload wan2.2-720p] [--block]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_08982_b200 import dit, schedule

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--block", action="store_true", help="also time one whole attention block (cold SVG-EAR)")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--blobs", action="store_true",
                help="block input = blob mixture (1000 blobs, sigma 0.1) and no rotary embedding, so q and k keep "
                     "a cluster structure behind the random projection; default is iid input, on which Lloyd "
                     "never converges (all 25 iterations, no bound skipping)")
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
    if os.path.exists("MEASURED_PEAKS.json") else {}
g = torch.Generator(device=dev).manual_seed(1)
qkv = torch.randn(1, S, 3 * H * d, generator=g, device=dev).to(torch.bfloat16)
w = torch.ones(H * d, device=dev)
if a.workload.startswith("wan"):
    grid, norm = (21, 45, 80), "token"
else:
    grid, norm = (33, 45, 80), "head"
rope = dit.rope_table_3d(grid, d, device=dev)
assert rope[0].shape[0] <= S


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {"workload": a.workload, "heads": H, "tokens": S, "d": d}
ms = timed(lambda: dit.qkv_prologue(qkv, H, norm=norm, q_weight=w, k_weight=w, rope=rope))
byt = 2 * qkv.numel() * 2
res["qkv_prologue"] = {"ms": ms, "algorithmic_GB": byt / 1e9, "GB_per_s": byt / ms / 1e6}
q, k, v = dit.qkv_prologue(qkv, H, norm=norm, q_weight=w, k_weight=w, rope=rope)
ms = timed(lambda: dit.heads_to_tokens(q))
byt = 2 * q.numel() * 2
res["heads_to_tokens"] = {"ms": ms, "algorithmic_GB": byt / 1e9, "GB_per_s": byt / ms / 1e6}
del qkv, q, k, v
if a.block:
    blk = dit.SvgEarSelfAttention(H * d, H, norm=norm, device=dev)
    if a.blobs:
        cen = torch.randn(1000, H * d, generator=g, device=dev)
        lab = torch.randint(1000, (S,), generator=g, device=dev)
        x = (cen[lab] + 0.1 * torch.randn(S, H * d, generator=g, device=dev)).to(torch.bfloat16).unsqueeze(0)
        rope = None
    else:
        x = torch.randn(1, S, H * d, generator=g, device=dev).to(torch.bfloat16)
    res["block_input"] = "blobs, no rope" if a.blobs else "iid"
    stack = schedule.SvgEarStack(cq, ck, 0.25, schedule=schedule.WarmupSchedule.none(1, 1), warm_start=False)
    res["block_cold_ms"] = timed(lambda: blk(x, stack, 0, 0, rope=rope))
    qi, ki = stack.lloyd_iterations(0)
    res["lloyd_iters_q_k"] = [qi.float().mean().item(), ki.float().mean().item()]
    dense = schedule.SvgEarStack(cq, ck, 0.25, schedule=schedule.WarmupSchedule(1, 1, 1, 1))
    res["block_dense_ms"] = timed(lambda: blk(x, dense, 0, 0, rope=rope))
print(json.dumps(res))
