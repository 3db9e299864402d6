"""Per-item timeline of CTA 0 of the persistent attention backward (ZB_ATTN_TRACE build,
libzb_trace.so), elementwise warp 4: for each dK/dV item and each dQ item the CTA walks, the
item start (K / V resp. Q / dO resident), first step's S ready, last step published, final
accumulator seen and epilogue stored (microseconds from the first event)."""
import ctypes as C, os, sys
os.environ["ZB_LIB"] = "libzb_trace.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib
names = ["start", "S0_ready", "last_pub", "acc_final", "stored"]
for tag, b, s, a, d in (("6.2B", 3, 1024, 32, 128), ("1.5B", 6, 1024, 24, 96)):
    h = a * d
    qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
    o = torch.randn(b * s, h, device="cuda").bfloat16()
    lse = torch.zeros(b, a, s, device="cuda")
    api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
    do = torch.randn(b * s, h, device="cuda").bfloat16()
    dq = torch.empty_like(qkv)
    dl = torch.empty_like(lse)
    for _ in range(3):
        api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (10 * 16))()
    lib.zb_dbg_attn_bwd_item_trace(buf)
    t0 = min(buf[i] for i in range(160) if buf[i])
    for body, off in (("dK/dV", 0), ("dQ", 5)):
        print(f"# {tag} {body}: us from the CTA's first event")
        print("item " + " ".join(f"{x:>10s}" for x in names))
        for r in range(16):
            row = [buf[(off + e) * 16 + r] for e in range(5)]
            if any(row):
                print(f"{r:4d} " + " ".join(f"{(v - t0) / 1e3 if v else float('nan'):10.2f}" for v in row))
