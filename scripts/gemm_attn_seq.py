"""QKV GEMM (EPI_STORE + bias) -> attention forward on its output, repeated, host-timed
(debugging aid): python scripts/gemm_attn_seq.py b s a d"""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(50, exit=True)
import torch
from paper_2401_10241_b200 import api
b, s, a, d = (int(x) for x in sys.argv[1:5])
h = a * d; T = b * s
x = (torch.randn(T, h, device="cuda") * 0.5).bfloat16()
w = (torch.randn(3 * h, h, device="cuda") * 0.02).bfloat16()
bias = torch.zeros(3 * h, device="cuda")
qkv = torch.empty(T, 3 * h, device="cuda").bfloat16()
o = torch.empty(T, h, device="cuda").bfloat16(); lse = torch.empty(b, a, s, device="cuda")
for i in range(4):
    t0 = time.time()
    api.dbg_gemm(x, w, qkv, M=T, N=3 * h, K=h, epi=0, bias=bias); torch.cuda.synchronize(); t1 = time.time()
    api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d); torch.cuda.synchronize(); t2 = time.time()
    print(i, "gemm", round((t1 - t0) * 1e3, 2), "attn", round((t2 - t1) * 1e3, 2), flush=True)
