"""One attention forward + backward at a config shape (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
b, s, a, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (6, 1024, 24, 96))]
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
o = torch.empty(b * s, h, device="cuda").bfloat16()
lse = torch.empty(b, a, s, device="cuda")
do = torch.randn(b * s, h, device="cuda").bfloat16()
dq = torch.empty_like(qkv); dl = torch.empty_like(lse)
for _ in range(2):
    api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
    api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
