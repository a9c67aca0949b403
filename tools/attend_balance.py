"""How much of the attention kernel's time is tail / imbalance?  Takes the routing mask of a bench
workload, derives every query tile's number of 64-key steps, and list-schedules the tiles onto the
SMs (one CTA per SM) in three orders: launch order (tile-major inside a head, heads in turn), longest
first inside each head, and globally longest first."""
import os, sys, json, heapq
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2603_08982_b200 as P
w = os.environ.get("WORKLOAD", "wan2.2-720p"); kind = os.environ.get("INPUTS", "blobs")
H, S, d, cq, ck = bench.WORKLOADS[w]
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, torch.device("cuda", 0), kind)
out, mask, aux = P.svg_ear_attention(q, k, v, cq, ck, 0.25, return_aux=True, kmeans_iters=25 if kind == "blobs" else 8)
ks, qs = aux["k_sizes"][0].long(), aux["q_sizes"][0].long()          # [H, ck], [H, cq]
sel = (mask[0].long() * ks[:, None, :]).sum(-1)                      # selected keys per (head, q cluster)
steps = (sel + 63) // 64 + (ck + 63) // 64                           # exact tiles + centroid tiles
tiles = []                                                           # (head, steps) per 256-row tile, launch order
for h in range(H):
    for i in range(cq):
        n = int(qs[h, i]); t = int(steps[h, i])
        full, rem = divmod(n, 256)
        tiles += [(h, t)] * full
        if rem > 128: tiles.append((h, t))
        elif rem > 0: tiles.append((h, t * 0.5))                     # remainder kernel: two CTAs per SM
def makespan(order, sms=148):
    heap = [0.0] * sms
    for _, t in order:
        heapq.heappush(heap, heapq.heappop(heap) + t)
    return max(heap)
total = sum(t for _, t in tiles)
res = {"workload": w, "inputs": kind, "tiles": len(tiles), "ideal_steps_per_sm": total / 148,
       "longest_tile_steps": max(t for _, t in tiles), "mean_tile_steps": total / len(tiles),
       "launch_order": makespan(tiles),
       "longest_first_per_head": makespan(sorted(tiles, key=lambda x: (x[0], -x[1]))),
       "longest_first_global": makespan(sorted(tiles, key=lambda x: -x[1]))}
for key in ("launch_order", "longest_first_per_head", "longest_first_global"):
    res[key + "_over_ideal"] = res[key] / res["ideal_steps_per_sm"]
print(json.dumps(res))
