"""Timeline of the heaviest k_fwd_tc CTA (query tiles 6, 7: 8 key blocks) from the ZB_ATTN_TRACE
build (libzb_trace.so): per key block the PV issue of each tile (P ready at the MMA warp) and,
per tile, the softmax start (S ready), S loaded from TMEM, P stored; microseconds from the
first event."""
import ctypes as C, os, sys
os.environ["ZB_LIB"] = "libzb_trace.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib
b, s, a, d = 6, 1024, 24, 96
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
o = torch.empty(b * s, h, device="cuda").bfloat16()
lse = torch.zeros(b, a, s, device="cuda")
for _ in range(3):
    api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (12 * 64))()
lib.zb_dbg_attn_fwd_trace(buf)
n = s // 128
t0 = min(buf[r * 64 + j] for r in range(12) for j in range(n) if buf[r * 64 + j])
names = ["pv0_issue", "pv1_issue", "t0_s_ready", "t0_s_loaded", "t0_p_stored", "t1_s_ready", "t1_s_loaded",
         "t1_p_stored", "t0_exp_go", "t1_exp_go", "t0_exp_end", "t1_exp_end"]
print("blk " + " ".join(f"{x:>11s}" for x in names))
for j in range(n):
    print(f"{j:3d} " + " ".join(f"{(buf[r * 64 + j] - t0) / 1e3 if buf[r * 64 + j] else float('nan'):11.2f}"
                             for r in range(12)))
