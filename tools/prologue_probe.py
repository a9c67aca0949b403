import sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_2603_08982_b200 import dit
H, S, d = 40, 75600, 128
dev = "cuda"
qkv = torch.randn(1, S, 3 * H * d, device=dev).to(torch.bfloat16)
w = torch.ones(H * d, device=dev)
rope = dit.rope_table_3d((21, 45, 80), d, device=dev)
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
for norm in ("none", "head", "token"):
    for r in (None, rope):
        ms = timed(lambda: dit.qkv_prologue(qkv, H, norm=norm, q_weight=w, k_weight=w, rope=r))
        out[f"{norm},{'rope' if r is not None else 'norope'}"] = round(2 * qkv.numel() * 2 / ms / 1e6)
print(json.dumps(out))
