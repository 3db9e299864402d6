"""W-grouping at the b = 1 configs (14.6B h 5120, 28.3B h 6144; T = 1024 tokens per
microbatch): the W contraction dW += dY^T X over k microbatches as ONE GEMM with K = k T
(zb_dbg_gemm_wgroup, with the bias column sums) vs k separate W GEMMs.  TFLOP/s from CUDA
events over 10 repetitions (f32 gradient accumulation, beta = 1)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api


def run(M, N, T, k, grouped, iters=10):
    As = [torch.randn(T, M, device="cuda").bfloat16() for _ in range(k)]
    Bs = [torch.randn(T, N, device="cuda").bfloat16() for _ in range(k)]
    C = torch.zeros(M, N, device="cuda")
    db = torch.zeros(M, device="cuda")

    def once():
        if grouped:
            api.dbg_gemm_wgroup(As, Bs, C, M=M, N=N, bias=db, beta=1)
        else:
            for a, b in zip(As, Bs):
                api.dbg_gemm_wgroup([a], [b], C, M=M, N=N, bias=db, beta=1)
    for _ in range(2):
        once()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        once()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return round(2.0 * M * N * T * k / ms / 1e9, 1)


for name, h in (("14.6B", 5120), ("28.3B", 6144)):
    for lin, (M, N) in (("fc1", (4 * h, h)), ("fc2", (h, 4 * h)), ("proj", (h, h)), ("qkv", (3 * h, h))):
        r = {"cfg": name, "linear": lin, "MN": [M, N], "T": 1024}
        for k in (2, 4):
            r[f"k{k}_separate_tflops"] = run(M, N, 1024, k, False)
            r[f"k{k}_grouped_tflops"] = run(M, N, 1024, k, True)
        print(json.dumps(r), flush=True)
