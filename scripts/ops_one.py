"""The HBM-bound stage kernels once at the 1.5B microbatch shape (for ncu):
LN forward, LN backward (dx + gamma/beta grads), bias grads of widths h, 3h, 4h."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
rows, h = 6144, 2304
x = torch.randn(rows, h, device="cuda").bfloat16()
g = torch.ones(h, device="cuda"); b = torch.zeros(h, device="cuda")
y = torch.empty_like(x); mean = torch.empty(rows, device="cuda"); rs = torch.empty(rows, device="cuda")
dy = torch.randn(rows, h, device="cuda"); resid = torch.randn(rows, h, device="cuda")
dx32 = torch.empty(rows, h, device="cuda"); dx = torch.empty_like(x)
gg = torch.empty(h, device="cuda"); gb = torch.empty(h, device="cuda")
u = torch.randn(rows, 4 * h, device="cuda").bfloat16(); out = torch.empty(4 * h, device="cuda")
for _ in range(2):
    api.dbg_layernorm_fwd(x, g, b, y, mean, rs, rows=rows, h=h)
    api.dbg_layernorm_bwd(dy, x, mean, rs, g, dx, gg, gb, rows=rows, h=h, resid=resid, dx32=dx32)
    api.dbg_bias_grad(u, out, rows=rows, n=4 * h)
    api.dbg_bias_grad(x, out, rows=rows, n=h)
torch.cuda.synchronize()
