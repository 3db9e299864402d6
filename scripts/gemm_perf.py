"""Time the tcgen05 GEMM at the config shapes (CUDA events, warm-up, L2-sized inputs)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api

def bench(M, N, K, a_mn, b_mn, epi, iters=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    Cb = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi in (4, 5) else torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in (1, 2, 3) else None
    for _ in range(3):
        api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi, bias=bias if epi < 3 else None, aux=aux, beta=1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi, bias=bias if epi < 3 else None, aux=aux, beta=1)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return ms, 2.0 * M * N * K / ms / 1e9

shapes = [
  ("c2 F qkv", 6144, 6912, 2304, False, False, 0),
  ("c2 F proj", 6144, 2304, 2304, False, False, 2),
  ("c2 F fc1", 6144, 9216, 2304, False, False, 1),
  ("c2 F fc2", 6144, 2304, 9216, False, False, 2),
  ("c2 B qkv", 6144, 2304, 6912, False, True, 0),
  ("c2 B proj", 6144, 2304, 2304, False, True, 0),
  ("c2 B fc1", 6144, 2304, 9216, False, True, 0),
  ("c2 B fc2", 6144, 9216, 2304, False, True, 3),
  ("c2 W qkv", 6912, 2304, 6144, True, True, 4),
  ("c2 W proj", 2304, 2304, 6144, True, True, 4),
  ("c2 W fc1", 9216, 2304, 6144, True, True, 4),
  ("c2 W fc2", 2304, 9216, 6144, True, True, 4),
  ("c2 head", 6144, 50304, 2304, False, False, 5),
  ("c5 W fc1", 24576, 6144, 1024, True, True, 4),
  ("8192^3", 8192, 8192, 8192, False, False, 0),
]


def cublas(M, N, K, a_mn, b_mn, iters=20):
    """torch.matmul (cuBLAS) on the same operand layouts, bf16 out (context only)."""
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    a = A.t() if a_mn else A
    b = B if b_mn else B.t()
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): a @ b
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return ms, 2.0 * M * N * K / ms / 1e9


for name, *sh in shapes:
    ms, tf = bench(*sh)
    cms, ctf = cublas(*sh[:5])
    print(json.dumps({"shape": name, "MNK": sh[:3], "ms": round(ms, 4), "tflops": round(tf, 1),
                      "cublas_ms": round(cms, 4), "cublas_tflops": round(ctf, 1)}))
