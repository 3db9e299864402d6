"""Timeline of one k_dkdv_tc CTA (kb = 0: 16 query steps) from the ZB_ATTN_TRACE build
(libzb_trace.so): per step the TMA issue, Q/dO arrival, S-buffer free, elementwise start /
end and the dS -> grad MMA issue, in microseconds from the CTA start."""
import ctypes as C, os, sys
os.environ.setdefault("ZB_LIB", "libzb_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib
b, s, a, d = 6, 1024, 24, 96
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
o = torch.randn(b * s, h, device="cuda").bfloat16()
lse = torch.zeros(b, a, s, device="cuda")
do = torch.randn(b * s, h, device="cuda").bfloat16()
dq = torch.empty_like(qkv); dl = torch.empty_like(lse)
api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
for _ in range(3):
    api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (12 * 64))()
lib.zb_dbg_attn_trace(buf)
t0 = buf[6 * 64 + 0]
names = ["tma_issue", "qdo_arrived", "sbuf_free", "ds_ready(grad issue)", "ew_start", "ew_end", "-", "ew_loaded", "ew_computed", "grad_done", "grad_issued", "st_issued"]
print("end (o_final) at us", (buf[6 * 64 + 1] - t0) / 1e3)
print("step " + " ".join(f"{n:>12s}" for n in names if n != "-"))
for n in range(16):
    print(f"{n:4d} " + " ".join(f"{(buf[r * 64 + n] - t0) / 1e3:12.2f}" for r in range(12) if r != 6))
