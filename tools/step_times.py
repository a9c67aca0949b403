"""Per-step times of the fused operator (resident inputs) — shows run-to-run spread."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib
H, S, d, cq, ck = bench.WORKLOADS["wan2.2-720p"]
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
ws = torch.empty(_lib.workspace_bytes(_lib.Shape(H, S, S, d, cq, ck)), dtype=torch.uint8, device="cuda")
def run():
    return P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", workspace_buffer=ws)
for mode in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for _ in range(2): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(mode, " ".join(f"{t:.1f}" for t in ts), flush=True)
