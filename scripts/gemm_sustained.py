"""Sustained (power-capped) throughput of the tcgen05 GEMM vs cuBLAS on the
1.5B step's shapes: each kernel runs back-to-back for --secs seconds after a
warm-up, ours and cuBLAS alternated (A/B/A) so both see the same clocks.
cuBLAS gets the same operand majorness (transposed views), plain bf16 output."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api

ap = argparse.ArgumentParser(); ap.add_argument("--secs", type=float, default=2.0)
ap.add_argument("--model", default="1.5B", choices=["1.5B", "6.2B"]); a = ap.parse_args()

def timed_loop(fn, secs):
    fn(); torch.cuda.synchronize()
    # calibrate the iteration count
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    n = max(3, int(secs * 1000 / max(s.elapsed_time(e), 1e-3)))
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n

def case(name, M, N, K, a_mn, b_mn, epi):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    Cb = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi in (4, 5) else torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in (1, 2, 3) else None
    ours = lambda: api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi,
                                bias=bias if epi < 3 else None, aux=aux, beta=1)
    At = A.t() if a_mn else A            # [M, K] view
    Bt = B if b_mn else B.t()            # [K, N] view
    Co = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cub = lambda: torch.matmul(At, Bt, out=Co)
    fl = 2.0 * M * N * K
    t1 = timed_loop(ours, a.secs); t2 = timed_loop(cub, a.secs); t3 = timed_loop(ours, a.secs)
    o = fl / ((t1 + t3) / 2) / 1e9; c = fl / t2 / 1e9
    print(json.dumps({"shape": name, "MNK": [M, N, K], "epi": epi, "ours_tflops": round(o, 1),
                      "cublas_tflops": round(c, 1), "ratio": round(o / c, 3)}), flush=True)

T, h, V = (6144, 2304, 50304) if a.model == "1.5B" else (3072, 4096, 50304)
for sh in [("F qkv", T, 3 * h, h, False, False, 0), ("F proj+resid", T, h, h, False, False, 2),
           ("F fc1+gelu", T, 4 * h, h, False, False, 1), ("F fc2+resid", T, h, 4 * h, False, False, 2),
           ("B fc2 (gelu bwd)", T, 4 * h, h, False, True, 3), ("B fc1 (f32 out)", T, h, 4 * h, False, True, 5),
           ("B qkv", T, h, 3 * h, False, True, 5), ("B proj", T, h, h, False, True, 0),
           ("W qkv", 3 * h, h, T, True, True, 4), ("W proj", h, h, T, True, True, 4),
           ("W fc1", 4 * h, h, T, True, True, 4), ("W fc2", h, 4 * h, T, True, True, 4),
           ("head F", T, V, h, False, False, 5), ("8192^3", 8192, 8192, 8192, False, False, 0)]:
    case(*sh)
