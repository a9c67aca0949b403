"""BASELINE config 4: exact-budget sweep, error-aware routing vs SVG2 score-magnitude routing on the
SAME clustering; metric = relative L2 of the sparse output against dense bf16 attention
(reference analogue: analysis.sweep_one_seed / evaluate_policy, analysis.py:308-368).

    python tools/budget_sweep.py [--heads 2] [--seq 75600] [--cq 300] [--ck 1000] [--sigma 0.1]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import router as R
from paper_2603_08982_b200.clustering import ClusterModel, device_start_pair, run_lloyd

ap = argparse.ArgumentParser()
ap.add_argument("--heads", type=int, default=2)
ap.add_argument("--seq", type=int, default=75600)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--cq", type=int, default=300)
ap.add_argument("--ck", type=int, default=1000)
ap.add_argument("--sigma", type=float, default=0.1)
ap.add_argument("--rhos", default="0.05,0.1,0.15,0.2,0.25,0.3,0.4,0.5")
a = ap.parse_args()
dev = torch.device("cuda", 0)
q, k, v = bench.make_heads(torch, 0, a.heads, a.seq, a.d, a.cq, a.ck, a.sigma, dev)
qb, kb, vb = q[0], k[0], v[0]
qi, ki = device_start_pair(qb, a.cq, kb, a.ck, 0)
rq, rk = run_lloyd(qb, qi, 25), run_lloyd(kb, ki, 25)
qm = ClusterModel(a.cq, rq["assign"], rq["centroids"], rq["sizes"], rq["perm"], rq["offsets"])
km = ClusterModel(a.ck, rk["assign"], rk["centroids"], rk["sizes"], rk["perm"], rk["offsets"])
qp, kp, vp = P.permute_rows(qb, qm), P.permute_rows(kb, km), P.permute_rows(vb, km)
vc = P.segment_means(vp, km)
table = P.estimate_errors_streaming(qm, km, kp, vp)
dense = torch.nn.functional.scaled_dot_product_attention(q, k, v)[0].float()
dn = dense.norm(dim=(1, 2))
rows = []
for rho in [float(x) for x in a.rhos.split(",")]:
    budget = R.DensityBudget.global_density(rho)
    out = {}
    for name, mask in (("error_aware", R.route_error_aware(table, budget)),
                       ("score", R.route_score(qm.centroids, km.centroids, qm.sizes, km.sizes, budget))):
        res = P.sparse_attend(qp, kp, vp, qm, km, mask, v_centroids=vc, unpermute=True, dtype=torch.bfloat16)
        err = ((res.output.float() - dense).norm(dim=(1, 2)) / dn).mean()
        out[name] = float(err)
        out[name + "_density"] = float(mask.density.double().mean())
    rows.append({"rho": rho, **out})
    print(json.dumps(rows[-1]), flush=True)
wins = sum(r["error_aware"] <= r["score"] for r in rows)
print(json.dumps({"workload": vars(a), "error_aware_wins": wins, "of": len(rows)}))
