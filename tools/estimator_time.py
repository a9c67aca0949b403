"""Times the block error table alone (svgear_error_table through estimate_errors_streaming: key
statistics + centroid logits + the tcgen05 table kernel) at the Wan2.2 shape; prints a checksum of the
table so that two builds can be compared for identical results."""
import sys, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200.clustering import device_start, run_lloyd, ClusterModel
H, S, d, cq, ck = bench.WORKLOADS["wan2.2-720p"]
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
qb, kb, vb = q[0], k[0], v[0]
rq = run_lloyd(qb, device_start(qb, cq), 25); rk = run_lloyd(kb, device_start(kb, ck), 25)
qm = ClusterModel(cq, rq["assign"], rq["centroids"], rq["sizes"], rq["perm"], rq["offsets"])
km = ClusterModel(ck, rk["assign"], rk["centroids"], rk["sizes"], rk["perm"], rk["offsets"])
kp, vp = P.permute_rows(kb, km), P.permute_rows(vb, km)
t = P.estimate_errors_streaming(qm, km, kp, vp); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): t2 = P.estimate_errors_streaming(qm, km, kp, vp)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"estimator_ms": e0.elapsed_time(e1) / 10, "checksum": float(t2.error_sum.sum())}))
if os.environ.get("PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.estimate_errors_streaming(qm, km, kp, vp); torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            print(f"{e.device_time / 1e3:8.3f} ms  {e.name[:90]}")
    # against the fp32 check kernel (same quantity on CUDA cores): largest deviation relative to the table's maximum
    t32 = P.estimate_errors_streaming(qm, km, kp, vp, fp32_check=True)
    dev = float(((t2.error_sum - t32.error_sum).abs().amax(dim=(1, 2)) / t32.error_sum.amax(dim=(1, 2))).max())
    print(json.dumps({"max_dev_vs_fp32_check_rel_to_table_max": dev}))
