"""Where the W GEMM loses to F at the 6.2B shapes (round 2): the same M x N x K (K = T =
3072) as the production W (MN-major A and B, f32 TMA reduce-add, bias column sums), then
without the column sums, with a bf16 store instead of the f32 reduce-add, and with both
operands K-major (the F layout); cuBLAS (bf16 out) beside.  Each variant runs back to back
for --secs seconds (power-capped clocks, like the step)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api

ap = argparse.ArgumentParser(); ap.add_argument("--secs", type=float, default=1.0); a = ap.parse_args()


def timed(fn):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    n = max(3, int(a.secs * 1000 / max(s.elapsed_time(e), 1e-3)))
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n


T, h = 3072, 4096
for name, M, N in [("qkv", 3 * h, h), ("proj", h, h), ("fc1", 4 * h, h), ("fc2", h, 4 * h)]:
    K = T
    dY = torch.randn(K, M, device="cuda").bfloat16()      # [T, n_out]: MN-major A of W
    X = torch.randn(K, N, device="cuda").bfloat16()       # [T, n_in]:  MN-major B of W
    dYt, Xt = dY.t().contiguous(), X.t().contiguous()     # K-major copies (F-like layout)
    C32 = torch.zeros(M, N, device="cuda")
    C16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(M, device="cuda")
    fl = 2.0 * M * N * K
    v = {
        "W_cs": lambda: api.dbg_gemm_wgroup([dY], [X], C32, M=M, N=N, bias=bias, beta=1),
        "W_acc": lambda: api.dbg_gemm(dY, X, C32, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, beta=1),
        "W_bf16": lambda: api.dbg_gemm(dY, X, C16, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=0),
        "Kmaj_acc": lambda: api.dbg_gemm(dYt, Xt, C32, M=M, N=N, K=K, epi=4, beta=1),
        "Kmaj_bf16": lambda: api.dbg_gemm(dYt, Xt, C16, M=M, N=N, K=K, epi=0),
        "W_acc_beta0": lambda: api.dbg_gemm(dY, X, C32, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, beta=0),
        "cublas": lambda: torch.matmul(dY.t(), X, out=C16),
    }
    r = {"shape": f"W {name}", "MNK": [M, N, K]}
    for k, fn in v.items():
        r[k] = round(fl / timed(fn) / 1e9, 1)
    # the same reduce-add epilogue behind twice the mainloop per tile (K = 2T)
    dY2, X2 = torch.cat([dY, dY]), torch.cat([X, X])
    r["W_acc_K2T"] = round(2 * fl / timed(lambda: api.dbg_gemm(dY2, X2, C32, M=M, N=N, K=2 * K, a_mn=True, b_mn=True,
                                                               epi=4, beta=1)) / 1e9, 1)
    print(json.dumps(r), flush=True)
