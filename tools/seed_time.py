"""Times the device-side k-means++ seeding alone (svgear_kmeans_seed through clustering.device_start)
at the Wan2.2 shape, key side (1000 centres) and query side (300 centres)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_08982_b200.clustering import device_start
H, S, d, cq, ck = bench.WORKLOADS["wan2.2-720p"]
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
out = {}
for name, x, c in (("key_side_1000", k[0], ck), ("query_side_300", q[0], cq)):
    device_start(x, c); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        device_start(x, c)
    e1.record(); torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / 10, 4)
print(json.dumps(out))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    device_start(k[0], ck); device_start(q[0], cq); torch.cuda.synchronize()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        print(f"{e.device_time / 1e3:8.3f} ms  {e.name[:90]}")
