"""Times svgear_route_error_aware alone on random Wan2.2-sized tables (300 x 1000 blocks per head)
for several head counts: the routing stage is latency bound, so its time barely depends on the
number of heads.   python tools/route_time.py [--heads 40,20,10,5]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08982_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--heads", default="40,20,10,5")
ap.add_argument("--cq", type=int, default=300)
ap.add_argument("--ck", type=int, default=1000)
ap.add_argument("--rho", type=float, default=0.25)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
rng = np.random.default_rng(0)
out = {}
for bh in [int(x) for x in a.heads.split(",")]:
    qs = rng.multinomial(75600 - a.cq, np.ones(a.cq) / a.cq, size=bh) + 1
    ks = rng.multinomial(75600 - a.ck, np.ones(a.ck) / a.ck, size=bh) + 1
    err = rng.random((bh, a.cq, a.ck)) ** 4 * (qs[:, :, None] * ks[:, None, :])
    t = P.BlockErrorTable(error_sum=torch.from_numpy(err).cuda(), q_sizes=torch.from_numpy(qs).int().cuda(),
                          k_sizes=torch.from_numpy(ks).int().cuda(), stabilizers=None, mode="valueAware", flops=0)
    cap = P.entry_capacity(a.rho, 75600 * 75600)
    for ov in (P.FILL_REMAINDER, P.STOP_AT_FIRST_OVERFLOW):
        P.route_error_aware_entries(t, cap, overshoot=ov)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            P.route_error_aware_entries(t, cap, overshoot=ov)
        e1.record()
        torch.cuda.synchronize()
        out[f"heads={bh},{ov}"] = round(e0.elapsed_time(e1) / a.reps, 4)
print(json.dumps(out))
