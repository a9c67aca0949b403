"""Time the fused attention kernel alone (staged API, CUDA events) at a bench workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import router as R
from paper_2603_08982_b200.clustering import ClusterModel, device_start, run_lloyd

H, S, d, cq, ck = bench.WORKLOADS[os.environ.get("WORKLOAD", "wan2.2-720p")]
H = int(os.environ.get("HEADS", 8))
rho = float(os.environ.get("RHO", 0.25))
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0))
qb, kb, vb = q[0], k[0], v[0]
rq = run_lloyd(qb, device_start(qb, cq, 0), 25)
rk = run_lloyd(kb, device_start(kb, ck, 0x9E37), 25)
qm = ClusterModel(cq, rq["assign"], rq["centroids"], rq["sizes"], rq["perm"], rq["offsets"])
km = ClusterModel(ck, rk["assign"], rk["centroids"], rk["sizes"], rk["perm"], rk["offsets"])
qp, kp, vp = P.permute_rows(qb, qm), P.permute_rows(kb, km), P.permute_rows(vb, km)
vc = P.segment_means(vp, km)
table = P.estimate_errors_streaming(qm, km, kp, vp)
mask = R.route_error_aware(table, R.DensityBudget.global_density(rho))
ts = []
for rep in range(int(os.environ.get("REPS", 5))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = P.sparse_attend(qp, kp, vp, qm, km, mask, v_centroids=vc, unpermute=True, dtype=torch.bfloat16)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
fl = float(res.flops.exact_block + res.flops.compensation)
t = min(ts[1:])
print(f"heads={H} attend {t:8.3f} ms  ({fl / t / 1e9:7.1f} TFLOP/s algorithmic)", flush=True)
