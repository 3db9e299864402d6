import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2401_10241_b200 import api
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
