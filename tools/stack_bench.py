"""BASELINE config 5: the attention stack of a denoising run — L layers x T steps of SVG-EAR
attention at a workload shape, on synthetic latents that drift slowly from step to step (per layer a
fixed blob mixture whose centres random-walk by `--drift` per step, fresh token noise every step).

Three schedules are timed (CUDA events around the whole run, inputs resident), all through the
product scheduler `schedule.SvgEarStack`:
  cold : every (layer, step) seeds its k-means on the device (svgear_kmeans_seed);
  warm : step t of a layer starts Lloyd from the centroids of step t-1 of the same layer
         (the reference's warm start, clustering.py:158-163) with the iteration
         cap --warm-iters (the first step of a layer is cold);
  warm_paper_schedule : as warm, plus the paper's dense warm-up (first 20 % of the steps and layer 0
         run dense attention).
With --gpus N (torchrun) the heads are sharded as in bench.py.

    python tools/stack_bench.py --layers 4 --steps 6          # quick
    python tools/stack_bench.py --layers 40 --steps 50        # the full config-5 stack
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib, schedule

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


def run(warm, dense_warmup=False):
    """One denoising run through the product scheduler (schedule.SvgEarStack)."""
    sched = (schedule.WarmupSchedule(a.steps, max(1, a.steps // 5), a.layers, min(1, a.layers - 1))
             if dense_warmup else schedule.WarmupSchedule.none(a.steps, a.layers))
    stack = schedule.SvgEarStack(cq, ck, a.rho, schedule=sched, warm_start=warm, warm_iters=a.warm_iters)
    iters = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.steps):
        for li, L in enumerate(layers):
            q, k, v = L.sample()
            stack.attend(li, t, q, k, v)
            if not sched.is_dense(li, t):
                iters.append(stack.lloyd_iterations(li))
    e1.record()
    torch.cuda.synchronize()
    qi = torch.stack([i[0].float().mean() for i in iters]).mean().item() if iters else 0.0
    ki = torch.stack([i[1].float().mean() for i in iters]).mean().item() if iters else 0.0
    return e0.elapsed_time(e1), qi, ki, dict(stack.calls)


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
_q, _k, _v = layers[0].sample()
torch.nn.functional.scaled_dot_product_attention(_q, _k, _v)  # builds the library's dense plan outside the timing
del _q, _k, _v
torch.cuda.synchronize()
res = {}
n = a.layers * a.steps
for name, warm, dense in (("cold", False, False), ("warm", True, False), ("warm_paper_schedule", True, True)):
    ms, qi, ki, calls = run(warm, dense)
    res[name] = {"total_ms": ms - gen, "ms_per_layer": (ms - gen) / n, "mean_lloyd_iters_q": qi, "mean_lloyd_iters_k": ki,
                 "calls": calls}
print(json.dumps({"workload": a.workload, "heads": H, "layers": a.layers, "steps": a.steps, "rho": a.rho,
                  "drift": a.drift, "warm_iters": a.warm_iters, "input_generation_ms": gen,
                  "paper_schedule": "dense for the first 20% of the steps and for layer 0 (PAPER.md Table config)", **res}))
