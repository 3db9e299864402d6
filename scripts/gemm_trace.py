"""Timeline of CTA 0 of the 2-CTA GEMM (ZB_GEMM_TRACE build, libzb_gtrace.so): per tile of
pair 0, when the MMA warp got the accumulator, issued the tile's last MMA, and when epilogue
warps 4 / 11 got / released it (microseconds from the first event).  argv: M N K b_mn epi [a_mn]
(a_mn = 1 with b_mn = 1, epi = 4: the W GEMM layout)."""
import ctypes as C, os, sys
os.environ.setdefault("ZB_LIB", "libzb_gtrace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib
M, N, K, b_mn, epi = [int(x) for x in sys.argv[1:6]] if len(sys.argv) > 5 else (6144, 9216, 2304, 1, 3)
a_mn = int(sys.argv[6]) if len(sys.argv) > 6 else 0
A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
Cb = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi in (4, 5) else torch.bfloat16)
bias = torch.zeros(N, device="cuda")
aux = torch.randn(M, N, device="cuda").bfloat16() if epi in (1, 2, 3) else None
for _ in range(5):
    api.dbg_gemm(A, B, Cb, M=M, N=N, K=K, a_mn=bool(a_mn), b_mn=bool(b_mn), epi=epi, bias=bias if epi < 3 else None,
                 aux=aux, beta=1)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 64))()
lib.zb_dbg_gemm_trace(buf)
t0 = min(buf[r * 64 + j] for r in range(5) for j in range(64) if buf[r * 64 + j])
names = ["mma_has_acc", "mma_last_issued", "epi4_has_acc", "epi4_released", "epi11_released"]
print(f"M{M} N{N} K{K} a_mn={a_mn} b_mn={b_mn} epi={epi}")
print("tile " + " ".join(f"{n:>16s}" for n in names))
for j in range(64):
    if not buf[j]:
        break
    print(f"{j:4d} " + " ".join(f"{(buf[r * 64 + j] - t0) / 1e3 if buf[r * 64 + j] else float('nan'):16.2f}" for r in range(5)))
