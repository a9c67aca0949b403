"""BASELINE config 5: the attention stack of a denoising run — L layers x T steps of SVG-EAR
attention at a workload shape, on synthetic latents that drift slowly from step to step (per layer a
fixed blob mixture whose centres random-walk by `--drift` per step, fresh token noise every step).

Two schedules are timed (CUDA events around the whole run, inputs resident):
  cold : every (layer, step) seeds its k-means on the device (svgear_kmeans_seed_gram);
  warm : step t of a layer starts Lloyd from the centroids of step t-1 of the same layer
         (the reference's warm start, clustering.py:158-163) with the iteration
         cap --warm-iters (the first step of a layer is cold).
With --gpus N (torchrun) the heads are sharded as in bench.py.

    python tools/stack_bench.py --layers 4 --steps 6          # quick
    python tools/stack_bench.py --layers 40 --steps 50        # the full config-5 stack
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="wan2.2-720p")
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--heads", type=int, default=0)
ap.add_argument("--rho", type=float, default=0.25)
ap.add_argument("--sigma", type=float, default=0.1)
ap.add_argument("--drift", type=float, default=0.02)
ap.add_argument("--warm-iters", type=int, default=4, help="Lloyd iteration cap of a warm-started step")
a = ap.parse_args()
H, S, d, cq, ck = bench.WORKLOADS[a.workload]
H = a.heads or H
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
g = torch.Generator(device=dev).manual_seed(7)


class Layer:
    """Slowly drifting blob mixture for one layer (labels fixed, centres random-walk)."""
    def __init__(self):
        mk = lambda nb: (torch.randn(H, nb, d, generator=g, device=dev),
                         torch.stack([torch.arange(S, device=dev).remainder(nb)[torch.randperm(S, generator=g, device=dev)]
                                      for _ in range(H)]))
        (self.qc, self.ql), (self.kc, self.kl) = mk(cq), mk(ck)
        self.vc = torch.randn(H, ck, d, generator=g, device=dev)
        self.q_cent = self.k_cent = None

    def sample(self):
        for c in (self.qc, self.kc, self.vc):
            c.add_(a.drift * torch.randn(c.shape, generator=g, device=dev))
        tok = lambda c, l: (torch.gather(c, 1, l.unsqueeze(-1).expand(-1, -1, d)) +
                            a.sigma * torch.randn(H, S, d, generator=g, device=dev)).to(torch.bfloat16).unsqueeze(0)
        return tok(self.qc, self.ql), tok(self.kc, self.kl), tok(self.vc, self.kl)


layers = [Layer() for _ in range(a.layers)]
ws = torch.empty(_lib.workspace_bytes(_lib.Shape(H, S, S, d, cq, ck)), dtype=torch.uint8, device=dev)


def run(warm):
    for L in layers:
        L.q_cent = L.k_cent = None
    iters = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gen_ms = 0.0
    e0.record()
    for t in range(a.steps):
        for L in layers:
            q, k, v = L.sample()
            kw = {}
            if warm and L.q_cent is not None:
                kw = dict(q_init=L.q_cent, k_init=L.k_cent, kmeans_iters=a.warm_iters)
            out, mask, aux = P.svg_ear_attention(q, k, v, cq, ck, a.rho, init="device", return_aux=True,
                                                 workspace_buffer=ws, **kw)
            L.q_cent, L.k_cent = aux["q_centroids"][0], aux["k_centroids"][0]
            iters.append((aux["q_iters"], aux["k_iters"]))
    e1.record()
    torch.cuda.synchronize()
    qi = torch.stack([i[0].float().mean() for i in iters]).mean().item()
    ki = torch.stack([i[1].float().mean() for i in iters]).mean().item()
    return e0.elapsed_time(e1), qi, ki


# input generation is inside the timed loop; time it alone and subtract
torch.cuda.synchronize()
g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g0.record()
for t in range(a.steps):
    for L in layers:
        L.sample()
g1.record()
torch.cuda.synchronize()
gen = g0.elapsed_time(g1)
run(False)  # warm-up
res = {}
for name, warm in (("cold", False), ("warm", True)):
    ms, qi, ki = run(warm)
    n = a.layers * a.steps
    res[name] = {"total_ms": ms - gen, "ms_per_layer": (ms - gen) / n, "mean_lloyd_iters_q": qi, "mean_lloyd_iters_k": ki}
print(json.dumps({"workload": a.workload, "heads": H, "layers": a.layers, "steps": a.steps, "rho": a.rho,
                  "drift": a.drift, "warm_iters": a.warm_iters, "input_generation_ms": gen, **res}))
