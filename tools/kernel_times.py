"""Per-kernel GPU time of one operator call via torch.profiler (CUPTI) — quick, no replay."""
import argparse, sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench
import paper_2603_08982_b200 as P
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--heads", type=int, default=0)
ap.add_argument("--kmeans-iters", type=int, default=25)
ap.add_argument("--rho", type=float, default=0.25)
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
run = lambda: P.svg_ear_attention(q, k, v, cq, ck, a.rho, init="strided", kmeans_iters=a.kmeans_iters)
run(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run(); torch.cuda.synchronize()
agg = collections.OrderedDict()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        n = e.name.split("(")[0].replace("void ", "")
        x = agg.setdefault(n, [0, 0.0]); x[0] += 1; x[1] += e.device_time / 1e3
tot = sum(x[1] for x in agg.values())
print(f"{'kernel':64s} {'n':>5s} {'ms':>9s} {'share':>6s}")
for n, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:28]:
    print(f"{n[:64]:64s} {c:5d} {ms:9.3f} {100*ms/tot:5.1f}%")
print(f"{'TOTAL':64s} {sum(x[0] for x in agg.values()):5d} {tot:9.3f}")
