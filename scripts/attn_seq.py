"""fwd -> bwd -> fwd ... sequences of the tcgen05 attention kernels at a shape, each call
host-timed (debugging aid for shape-dependent stalls): python scripts/attn_seq.py b s a d"""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(60, exit=True)
import torch
from paper_2401_10241_b200 import api
b, s, a, d = (int(x) for x in sys.argv[1:5])
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
o = torch.empty(b * s, h, device="cuda").bfloat16()
lse = torch.empty(b, a, s, device="cuda")
do = torch.randn(b * s, h, device="cuda").bfloat16()
dq = torch.empty_like(qkv); dl = torch.empty_like(lse)
for i in range(3):
    for name, fn in (("fwd", lambda: api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)),
                     ("bwd", lambda: api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d))):
        t0 = time.time(); fn(); torch.cuda.synchronize()
        print(i, name, round((time.time() - t0) * 1e3, 2), "ms", flush=True)
