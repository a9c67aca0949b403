"""Fused Lloyd step (lloyd_step.cu) against a reference run of the same library in full-evaluation
mode: assignments, permutation, sizes, offsets, centroids, iteration counts must be bit-identical
(the bound-based skipping and the fused step change the work, never a result).  Also times the
k-means stage alone.  Usage: python tools/lloyd_ab.py [--workload wan2.2-720p] [--heads 8]"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_08982_b200 import clustering as CL, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--heads", type=int, default=8)
ap.add_argument("--inputs", default="blobs")
ap.add_argument("--iters", type=int, default=25)
ap.add_argument("--start", default="strided", choices=["strided", "device"])
ap.add_argument("--no-inertia", action="store_true", help="the one-launch-per-iteration path svgear_forward uses")
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
dev = torch.device("cuda", 0)
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, dev, kind=a.inputs)


def run(x, c, full_eval=False):
    init = CL.strided_start(x[0], c) if a.start == "strided" else CL.device_start(x[0], c, seed=0)
    go = lambda: CL.run_lloyd(x[0], init, a.iters, full_eval=full_eval, want_inertia=not a.no_inertia)
    go()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    m = go()
    t1.record(); torch.cuda.synchronize()
    return m, t0.elapsed_time(t1)


for name, x, c in (("query", q, cq), ("key", k, ck)):
    new, t_new = run(x, c)
    ref, t_ref = run(x, c, full_eval=True)
    same = {f: bool(torch.equal(new[f], ref[f])) for f in ("assign", "perm", "sizes", "offsets", "centroids", "iters")}
    it_new = new["iters"]
    rel = float(((new["inertia"] - ref["inertia"]).abs() / ref["inertia"].abs().clamp_min(1e-30)).max())
    same["inertia<=1e-6"] = a.no_inertia or rel <= 1e-6
    print(f"{name}: fused {t_new:.3f} ms, full-eval {t_ref:.3f} ms, "
          f"iters max {int(it_new.max())} mean {float(it_new.float().mean()):.1f}, identical: {same}", flush=True)
    assert all(same.values()), same
print("OK")

if os.environ.get("PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    for name, x, c in (("query", q, cq), ("key", k, ck)):
        init = CL.device_start(x[0], c, seed=0)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            CL.run_lloyd(x[0], init, a.iters, want_inertia=False)
            torch.cuda.synchronize()
        evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                     key=lambda e: e.time_range.start)
        t0 = evs[0].time_range.start
        print(name)
        for e in evs:
            print(f"  {(e.time_range.start - t0) / 1e3:8.3f} ms  +{e.device_time / 1e3:7.3f} ms  {e.name.split('(')[0][:60]}")
