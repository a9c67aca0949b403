"""Capture the fused operator in a CUDA graph (the library's internal fork/join onto its helper
streams is event based), replay it, and compare with the eager result; report replay time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib
H, S, d, cq, ck = bench.WORKLOADS["wan2.2-720p"]
H = int(os.environ.get("HEADS", 40))
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
ws = torch.empty(_lib.workspace_bytes(_lib.Shape(H, S, S, d, cq, ck)), dtype=torch.uint8, device="cuda")
run = lambda: P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", workspace_buffer=ws)
for _ in range(3):
    eager_out, eager_mask = run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out, mask = run()
torch.cuda.synchronize()
ts = []
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("graph replay ms:", " ".join(f"{t:.1f}" for t in ts))
print("replay == eager:", bool(torch.equal(out, eager_out)), bool(torch.equal(mask, eager_mask)))
