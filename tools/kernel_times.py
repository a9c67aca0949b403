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
ap.add_argument("--init", default="device")
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
run = lambda: P.svg_ear_attention(q, k, v, cq, ck, a.rho, init=a.init, kmeans_iters=a.kmeans_iters, return_aux=True)
run(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run(); torch.cuda.synchronize()
agg = collections.OrderedDict()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        n = e.name.split("(")[0].replace("void ", "")
        x = agg.setdefault(n, [0, 0.0]); x[0] += 1; x[1] += e.device_time / 1e3
seq = [(e.name.split("(")[0].replace("void ", "").replace("svg::", ""), e.device_time / 1e3) for e in prof.events()
       if e.device_type == torch.autograd.DeviceType.CUDA and "svg::" in e.name]
import os as _os
if _os.environ.get("SEQ"):
    names = _os.environ["SEQ"].split(",")
    for nm in names:
        print(nm, " ".join(f"{ms:.3f}" for n_, ms in seq if nm in n_))
tot = sum(x[1] for x in agg.values())
print(f"{'kernel':64s} {'n':>5s} {'ms':>9s} {'share':>6s}")
for n, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:28]:
    print(f"{n[:64]:64s} {c:5d} {ms:9.3f} {100*ms/tot:5.1f}%")
aux = run()[2]
print("kmeans iters q/k max:", int(aux["q_iters"].max()), int(aux["k_iters"].max()), "mean:", float(aux["q_iters"].float().mean()), float(aux["k_iters"].float().mean()))
print(f"{'TOTAL':64s} {sum(x[0] for x in agg.values()):5d} {tot:9.3f}")
