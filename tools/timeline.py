"""Timeline of ONE operator call at a bench workload (torch profiler / CUPTI): per kernel family the
first start, last end and summed duration, relative to the first kernel of the call — shows what is
on the critical path and how the head groups / the two k-means sides overlap."""
import argparse, collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench
import paper_2603_08982_b200 as P
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--heads", type=int, default=0)
ap.add_argument("--head-groups", type=int, default=None)
ap.add_argument("--inputs", default="blobs")
ap.add_argument("--stagger", action="store_true")
ap.add_argument("--brief", action="store_true")
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0), a.inputs)
ws = torch.empty(P.operator_workspace_bytes(H, S, S, d, cq, ck, a.head_groups), dtype=torch.uint8, device="cuda")
run = lambda: P.svg_ear_attention(q, k, v, cq, ck, 0.25, workspace_buffer=ws, head_groups=a.head_groups,
                                  stagger_groups=a.stagger)
for _ in range(2):
    run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run(); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
fam = collections.OrderedDict()
for e in sorted(evs, key=lambda e: e.time_range.start):
    n = e.name.split("(")[0].replace("void ", "").replace("svg::", "").replace("<unnamed>::", "")[:44]
    f = fam.setdefault(n, [1e18, 0, 0.0, 0])
    f[0] = min(f[0], e.time_range.start - t0); f[1] = max(f[1], e.time_range.end - t0); f[2] += e.device_time; f[3] += 1
if not a.brief:
    print(f"{'kernel':46s} {'n':>5s} {'first start':>12s} {'last end':>10s} {'busy ms':>9s}")
    for n, (s0, e1, busy, cnt) in fam.items():
        print(f"{n:46s} {cnt:5d} {s0 / 1e3:12.3f} {e1 / 1e3:10.3f} {busy / 1e3:9.3f}")
# wall time of the call measured with events, without the profiler
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("eager call ms (5 runs):", " ".join(f"{t:.2f}" for t in ts))
print("call span ms:", (max(e.time_range.end for e in evs) - t0) / 1e3)
