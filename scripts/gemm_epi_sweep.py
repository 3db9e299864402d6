"""The same GEMM shape under every epilogue (0 store, 1 bias+GeLU, 2 residual, 3 GeLU-bwd,
5 f32 store) and both B majornesses: separates epilogue cost from mainloop cost."""
import os, sys
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


M, N, K = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (6144, 9216, 2304)
for b_mn in (False, True):
    for epi in (0, 1, 2, 3, 5):
        ms, tf = bench(M, N, K, False, b_mn, epi)
        print(f"M{M} N{N} K{K} b_mn={int(b_mn)} epi={epi}: {ms * 1e3:7.1f} us  {tf:7.1f} TF/s")
