"""Per-item timeline of CTA 0 of the persistent attention forward (ZB_ATTN_TRACE build,
libzb_trace.so): for each item the CTA walks, the first S issue, tile 0 / 1 first S ready,
last P stored, O final seen and O stored, and the last PV issue (microseconds from the
CTA's first event).  Shapes: 6.2B (b 3, a 32, d 128) and 1.5B (b 6, a 24, d 96)."""
import ctypes as C, os, sys
os.environ["ZB_LIB"] = "libzb_trace.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib
names = ["S_issue0", "PV_issue_last", "t0_S0_ready", "t1_S0_ready", "t0_lastP", "t1_lastP", "t0_Ofinal",
         "t1_Ofinal", "t0_Ostored", "t1_Ostored"]
for tag, b, s, a, d in (("6.2B", 3, 1024, 32, 128), ("1.5B", 6, 1024, 24, 96)):
    h = a * d
    qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
    o = torch.empty(b * s, h, device="cuda").bfloat16()
    lse = torch.zeros(b, a, s, device="cuda")
    for _ in range(3):
        api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (10 * 16))()
    lib.zb_dbg_attn_fwd_item_trace(buf)
    vals = [buf[i] for i in range(160) if buf[i]]
    t0 = min(vals)
    print(f"# {tag}: item rows, us from the first event")
    print("item " + " ".join(f"{x:>13s}" for x in names))
    for r in range(16):
        row = [buf[e * 16 + r] for e in range(10)]
        if not any(row):
            continue
        print(f"{r:4d} " + " ".join(f"{(v - t0) / 1e3 if v else float('nan'):13.2f}" for v in row))
