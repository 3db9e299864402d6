"""Time the attention kernels at the config shapes (CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api

def t(fn, iters=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for name, b, s, a, d in [("c2", 6, 1024, 24, 96), ("c3", 3, 1024, 32, 128), ("c5", 1, 1024, 48, 128)]:
    h = a * d
    qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
    o = torch.empty(b * s, h, device="cuda").bfloat16()
    lse = torch.empty(b, a, s, device="cuda")
    do = torch.randn(b * s, h, device="cuda").bfloat16()
    dq = torch.empty_like(qkv); dl = torch.empty_like(lse)
    fwd = t(lambda: api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d))
    bwd = t(lambda: api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d))
    flops_f = 4 * b * a * s * s * d / 2   # causal
    flops_b = 10 * b * a * s * s * d / 2  # 5 matmuls (dkdv + dq recompute counted once as algorithmic)
    print(json.dumps({"cfg": name, "fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
                      "fwd_tflops": round(flops_f / fwd / 1e9, 1), "bwd_tflops_alg": round(flops_b / bwd / 1e9, 1)}))
