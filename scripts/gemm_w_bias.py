"""W GEMM (dW += dY^T X, f32 reduce-add) with and without the in-kernel bias column sums
(gemm.h bias_out) at the 1.5B / 6.2B W shapes: TFLOP/s (CUDA events, 20 launches)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api


def bench(M, N, K, bias, iters=20):
    A = torch.randn(K, M, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    C = torch.zeros(M, N, device="cuda")
    db = torch.zeros(M, device="cuda") if bias else None
    for _ in range(3):
        api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, beta=1, bias=db)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, beta=1, bias=db)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return round(2.0 * M * N * K / ms / 1e9, 1), round(ms * 1e3, 1)


for T, h in ((6144, 2304), (3072, 4096)):
    for (M, N) in ((h, 4 * h), (4 * h, h), (h, h), (3 * h, h)):
        r = {"MNK": (M, N, T), "no_bias": bench(M, N, T, False), "bias": bench(M, N, T, True)}
        print(json.dumps(r), flush=True)
