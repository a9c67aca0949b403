"""Run the fused operator several times on the same inputs at a bench workload and compare every
output bit for bit (the library uses no floating-point atomics; k-means sides and the two attention
kernels run concurrently, so a race would show up here)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
wl = os.environ.get("WORKLOAD", "wan2.2-720p")
H, S, d, cq, ck = bench.WORKLOADS[wl]
H = int(os.environ.get("HEADS", H))
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, float(os.environ.get("SIGMA", 0.1)), torch.device("cuda", 0))
ref = None
for rep in range(int(os.environ.get("REPS", 4))):
    out, mask, aux = P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", return_aux=True)
    torch.cuda.synchronize()
    cur = dict(out=out, mask=mask, **{n: aux[n] for n in ("q_perm", "k_perm", "q_centroids", "k_centroids", "error_table", "lse", "q_iters", "k_iters")})
    if ref is None:
        ref = {n: t.clone() for n, t in cur.items()}
        print("rep 0: reference taken; finite:", bool(torch.isfinite(out.float()).all()))
    else:
        bad = [n for n, t in cur.items() if not torch.equal(t, ref[n])]
        print(f"rep {rep}:", "bit-identical" if not bad else f"DIFFERS in {bad}")
