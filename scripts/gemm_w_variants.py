import json, sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/scripts')
import torch
from paper_2401_10241_b200 import api
def bench(M, N, K, a_mn, b_mn, epi, beta, iters=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    Cb = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (4, 5) else torch.bfloat16)
    for _ in range(3): api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi, beta=beta)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi, beta=beta)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return round(2.0 * M * N * K / ms / 1e9, 1)
for (M, N, K) in [(2304, 9216, 6144), (9216, 2304, 6144), (2304, 2304, 6144), (6912, 2304, 6144)]:
    r = {"MNK": (M, N, K)}
    r["W_acc_beta1"] = bench(M, N, K, True, True, 4, 1)
    r["W_acc_beta0"] = bench(M, N, K, True, True, 4, 0)
    r["W_bf16store"] = bench(M, N, K, True, True, 0, 0)
    r["Kmajor_bf16store"] = bench(M, N, K, False, False, 0, 0)
    r["Kmajor_f32acc"] = bench(M, N, K, False, False, 4, 1)
    print(os.environ.get("ZB_GEMM_NO_SPLITK", "0"), json.dumps(r))
