"""Run the operator once (after one warm-up call) at a bench workload — for ncu launch lists."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--heads", type=int, default=0)
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--kmeans-iters", type=int, default=25)
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
for _ in range(a.calls):
    out, mask = P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", kmeans_iters=a.kmeans_iters)
torch.cuda.synchronize()
print("ok", float(mask.float().mean()))
