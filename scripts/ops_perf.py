"""CUDA-event timing of the HBM-bound stage kernels at the 1.5B microbatch shape,
next to torch copies moving the same number of bytes (the achievable bandwidth
for a transfer of that size; inputs rotate over buffers larger than L2)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api
rows, h = 6144, 2304
NB = 8   # rotate inputs so the working set (> 126 MB L2) comes from HBM

def timeit(fn, iters=40):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters): fn(i)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1000.0   # us

xs = [torch.randn(rows, h, device="cuda").bfloat16() for _ in range(NB)]
g = torch.ones(h, device="cuda"); b = torch.zeros(h, device="cuda")
ys = [torch.empty(rows, h, device="cuda").bfloat16() for _ in range(NB)]
mean = torch.empty(rows, device="cuda"); rs = torch.empty(rows, device="cuda")
dys = [torch.randn(rows, h, device="cuda") for _ in range(NB)]
res = [torch.randn(rows, h, device="cuda") for _ in range(NB)]
dx32 = [torch.empty(rows, h, device="cuda") for _ in range(NB)]
gg = torch.empty(h, device="cuda"); gb = torch.empty(h, device="cuda")
us = [torch.randn(rows, 4 * h, device="cuda").bfloat16() for _ in range(4)]
out = torch.empty(4 * h, device="cuda")
f32 = [torch.randn(rows, h, device="cuda") for _ in range(NB)]
res_ = {}
res_["ln_fwd"] = (timeit(lambda i: api.dbg_layernorm_fwd(xs[i % NB], g, b, ys[i % NB], mean, rs, rows=rows, h=h)), 2 * rows * h * 2)
res_["copy_bf16_x"] = (timeit(lambda i: ys[i % NB].copy_(xs[i % NB])), 2 * rows * h * 2)
res_["ln_bwd_total"] = (timeit(lambda i: api.dbg_layernorm_bwd(dys[i % NB], xs[i % NB], mean, rs, g, ys[i % NB], gg, gb, rows=rows, h=h,
                                                               resid=res[i % NB], dx32=dx32[i % NB])), rows * h * (4 + 2 + 4 + 4 + 2 + 4 + 2))
res_["bias_h"] = (timeit(lambda i: api.dbg_bias_grad(xs[i % NB], out, rows=rows, n=h)), rows * h * 2)
res_["bias_4h"] = (timeit(lambda i: api.dbg_bias_grad(us[i % 4], out, rows=rows, n=4 * h)), rows * 4 * h * 2)
res_["copy_f32_x"] = (timeit(lambda i: dx32[i % NB].copy_(f32[i % NB])), 2 * rows * h * 4)
res_["sum_torch_4h"] = (timeit(lambda i: torch.sum(us[i % 4], dim=0, dtype=torch.float32, out=out)), rows * 4 * h * 2)
for k, (t, byt) in res_.items():
    print(json.dumps({"op": k, "us": round(t, 2), "GBs": round(byt / t / 1e3, 1)}))
