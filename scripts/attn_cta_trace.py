"""Per-CTA timeline of the attention kernels from the ZB_ATTN_TRACE build (libzb_trace.so):
every CTA's SM, start and end (globaltimer).  Reports the kernel span, per-SM busy time
(sum of its CTAs' durations) and gaps between consecutive CTAs on an SM, and (for grids of
one CTA per work item, as in the first round-2 measurement) a fit of CTA duration =
c0 + c1 * work — c0 the fixed per-CTA cost (prologue, fill, drain, epilogue).  Both kernels
are persistent now (one CTA per SM): the busy / span figures are the meaningful ones."""
import ctypes as C, json, os, sys
os.environ["ZB_LIB"] = "libzb_trace.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2401_10241_b200 import api
from paper_2401_10241_b200._lib import lib

b, s, a, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (3, 1024, 32, 128))]
h = a * d
qkv = torch.randn(b * s, 3 * h, device="cuda").bfloat16()
o = torch.empty(b * s, h, device="cuda").bfloat16()
lse = torch.zeros(b, a, s, device="cuda")
do = torch.randn(b * s, h, device="cuda").bfloat16()
dq = torch.empty_like(qkv); dl = torch.empty_like(lse)


def analyse(name, buf, n, work):
    x = np.array(buf[:3 * n], dtype=np.float64).reshape(n, 3)
    sm, t0, t1 = x[:, 0].astype(int), x[:, 1], x[:, 2]
    base = t0.min()
    t0, t1 = (t0 - base) / 1e3, (t1 - base) / 1e3
    dur = t1 - t0
    span = t1.max()
    busy = np.zeros(sm.max() + 1)
    gaps = []
    for k in np.unique(sm):
        idx = np.where(sm == k)[0]
        idx = idx[np.argsort(t0[idx])]
        busy[k] = dur[idx].sum()
        gaps += list(t0[idx[1:]] - t1[idx[:-1]])
    A = np.vstack([np.ones(n), work]).T
    c0, c1 = np.linalg.lstsq(A, dur, rcond=None)[0]
    print(json.dumps({"kernel": name, "shape": [b, s, a, d], "ctas": n, "span_us": round(span, 2),
                      "busy_mean_us": round(busy[busy > 0].mean(), 2), "busy_max_us": round(busy.max(), 2),
                      "gap_mean_us": round(float(np.mean(gaps)), 3) if gaps else None,
                      "fit_cta_us": {"fixed": round(c0, 3), "per_unit": round(c1, 4)},
                      "last_start_us": round(t0.max(), 2)}))


for _ in range(3):
    api.dbg_attention_fwd(qkv, o, lse, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
# the forward is persistent (one CTA per SM, min(items, SMs) CTAs): per-CTA busy time / span only
items = (s // 128 + 1) // 2 * a * b
nf = min(items, torch.cuda.get_device_properties(0).multi_processor_count)
buf = (C.c_ulonglong * (8192 * 3))()
lib.zb_dbg_attn_fwd_cta_trace(buf)
analyse("fwd (persistent)", buf, nf, np.ones(nf))
for _ in range(3):
    api.dbg_attention_bwd(qkv, o, do, lse, dq, dl, b=b, s=s, a=a, d=d)
torch.cuda.synchronize()
nb = min(2 * (s // 128) * a * b, torch.cuda.get_device_properties(0).multi_processor_count)  # persistent too
buf = (C.c_ulonglong * (16384 * 3))()
lib.zb_dbg_attn_bwd_cta_trace(buf)
analyse("bwd (persistent)", buf, nb, np.ones(nb))
