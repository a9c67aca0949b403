"""Probe: one Wan2.2 layer as G head groups, each group's svg_ear_attention on its own stream
(latency-bound phases of one group overlap throughput-bound phases of another) vs one call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib

H, S, d, cq, ck = bench.WORKLOADS["wan2.2-720p"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
q, k, v = bench.make_heads(torch, 0, H, S, d, cq, ck, 0.1, dev)



def timed(fn, reps=5, graph=True):
    for _ in range(2):
        fn()
    if graph:  # replay from a captured graph: host launch latency must not decide the comparison
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        fn = g.replay
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
ws = torch.empty(_lib.workspace_bytes(_lib.Shape(H, S, S, d, cq, ck)), dtype=torch.uint8, device=dev)
ref = P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", workspace_buffer=ws)
res["one_call"] = timed(lambda: P.svg_ear_attention(q, k, v, cq, ck, 0.25, init="device", workspace_buffer=ws))
del ws
for G in (2, 3, 4):
    bounds = [H * g // G for g in range(G + 1)]
    wss = [torch.empty(_lib.workspace_bytes(_lib.Shape(bounds[g + 1] - bounds[g], S, S, d, cq, ck)), dtype=torch.uint8,
                       device=dev) for g in range(G)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(G)]
    outs = [None] * G

    def run():
        cur = torch.cuda.current_stream(dev)
        for g in range(G):
            a, b = bounds[g], bounds[g + 1]
            streams[g].wait_stream(cur)
            with torch.cuda.stream(streams[g]):
                outs[g] = P.svg_ear_attention(q[:, a:b], k[:, a:b], v[:, a:b], cq, ck, 0.25, init="device", seed=a,
                                              workspace_buffer=wss[g])
        for g in range(G):
            cur.wait_stream(streams[g])

    res[f"groups_{G}"] = timed(run)
    same = all(torch.equal(outs[g][0], ref[0][:, bounds[g]:bounds[g + 1]]) for g in range(G))
    res[f"groups_{G}_same_as_one_call"] = same
    del wss
print(json.dumps(res))
