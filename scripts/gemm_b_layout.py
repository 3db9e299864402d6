"""The B (dgrad) GEMMs at the 6.2B shapes with the weight operand as stored (MN-major: W is
[n_out, n_in] and B needs W with n_in contiguous) against a K-major copy (W^T stored), plain
bf16 store and the production epilogues; power-capped loops of --secs seconds each.  Decides
whether a transposed bf16 weight shadow for the B pass would pay."""
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
for name, n_out, n_in in [("qkv", 3 * h, h), ("proj", h, h), ("fc1", 4 * h, h), ("fc2", h, 4 * h)]:
    M, N, K = T, n_in, n_out                     # dX[T, n_in] = dY[T, n_out] W[n_out, n_in]
    dY = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(n_out, n_in, device="cuda") * 0.02).bfloat16()
    Wt = W.t().contiguous()                       # [n_in, n_out]: K-major B
    C16 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    C32 = torch.empty(M, N, device="cuda")
    fl = 2.0 * M * N * K
    v = {
        "mn_bf16": lambda: api.dbg_gemm(dY, W, C16, M=M, N=N, K=K, b_mn=True, epi=0),
        "kmaj_bf16": lambda: api.dbg_gemm(dY, Wt, C16, M=M, N=N, K=K, epi=0),
        "mn_f32": lambda: api.dbg_gemm(dY, W, C32, M=M, N=N, K=K, b_mn=True, epi=5),
        "kmaj_f32": lambda: api.dbg_gemm(dY, Wt, C32, M=M, N=N, K=K, epi=5),
    }
    r = {"shape": f"B {name}", "MNK": [M, N, K]}
    for k, fn in v.items():
        r[k] = round(fl / timed(fn) / 1e9, 1)
    print(json.dumps(r), flush=True)
