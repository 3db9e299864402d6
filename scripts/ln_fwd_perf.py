"""LayerNorm forward (bf16) at the 6.2B / 1.5B microbatch shapes: CUDA-event time per call
with inputs rotating over buffers larger than L2, next to a torch copy moving the same bytes
(the achievable bandwidth for a transfer of that size), and the LayerNorm backward
(gamma/beta + dx passes).  (The ZB_LN_FWD variant switch belonged to a bulk-staged LN forward
that measured no faster — profiles/r02_ln_fwd_bulk_rejected.jsonl — and was removed.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_10241_b200 import api


def timeit(fn, iters=50):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1000.0


for rows, h in ((3072, 4096), (6144, 2304), (3072, 5120)):
    nb = max(4, int(300e6 // (rows * h * 4)) + 1)
    xs = [torch.randn(rows, h, device="cuda").bfloat16() for _ in range(nb)]
    ys = [torch.empty(rows, h, device="cuda").bfloat16() for _ in range(nb)]
    g = torch.ones(h, device="cuda")
    b = torch.zeros(h, device="cuda")
    mean = torch.empty(rows, device="cuda")
    rs = torch.empty(rows, device="cuda")
    byt = 2 * rows * h * 2
    t_ln = timeit(lambda i: api.dbg_layernorm_fwd(xs[i % nb], g, b, ys[i % nb], mean, rs, rows=rows, h=h))
    t_cp = timeit(lambda i: ys[i % nb].copy_(xs[i % nb]))
    dys = [torch.randn(rows, h, device="cuda") for _ in range(max(2, nb // 2))]
    nd = len(dys)
    res = torch.randn(rows, h, device="cuda")
    dx32 = torch.empty(rows, h, device="cuda")
    gg = torch.empty(h, device="cuda")
    gb = torch.empty(h, device="cuda")
    t_bwd = timeit(lambda i: api.dbg_layernorm_bwd(dys[i % nd], xs[i % nb], mean, rs, g, ys[i % nb], gg, gb, rows=rows,
                                                   h=h, resid=res, dx32=dx32))
    byt_bwd = rows * h * (4 + 2) + rows * h * (4 + 2 + 4 + 4 + 2)  # gamma/beta pass + dx pass
    print(json.dumps({"variant": os.environ.get("ZB_LN_FWD", "1"), "rows": rows, "h": h, "ln_us": round(t_ln, 2),
                      "ln_GBs": round(byt / t_ln / 1e3, 1), "copy_us": round(t_cp, 2),
                      "copy_GBs": round(byt / t_cp / 1e3, 1), "ln_bwd_us": round(t_bwd, 2),
                      "ln_bwd_GBs": round(byt_bwd / t_bwd / 1e3, 1)}))
