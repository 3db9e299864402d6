"""Diagnostic: error structure of the QKV weight gradient at the 6.2B width (b 2, m 2,
p 2 virtual stages) against the fp64 oracle: per Q / K / V block normwise error and the
worst elements relative to the bf16 C15 bound (tests/zbtest_util.close_report)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import zb_synth
from test_gpu_stage import gpu_run, oracle_grads
from zbtest_util import close_report

name = sys.argv[1] if len(sys.argv) > 1 else "6.2B"
cfg = zb_synth.CONFIGS[name].with_(L=2, b=2, m=2)
ref_loss, ref = oracle_grads(cfg, "bf16")
loss, g, _ = gpu_run(cfg, 2, "bf16")
out = {}
for k in ref:
    nrm, worst = close_report(g[k], ref[k], 2e-2, bf16=True, exact_zero_rows=True)
    out[k] = {"normwise": nrm, "worst": worst}
    if k.endswith("qkv_w") or worst > 0.7:
        x = g[k].astype(np.float64); r = ref[k]
        h = cfg.h
        if k.endswith("qkv_w"):
            for i, part in enumerate("QKV"):
                xb, rb = x[i * h:(i + 1) * h], r[i * h:(i + 1) * h]
                out[k][part] = close_report(xb, rb, 2e-2, bf16=True)
        d = np.abs(x - r)
        rows = np.sqrt(np.mean(r * r, axis=1)) if r.ndim == 2 else None
        idx = np.argsort(d.ravel())[-8:][::-1]
        top = []
        for f in idx:
            at = np.unravel_index(f, d.shape)
            top.append({"at": [int(a) for a in at], "ref": float(r[at]), "got": float(x[at]),
                        "row_rms": float(rows[at[0]]) if rows is not None else None})
        out[k]["top_abs_err"] = top
        out[k]["rms"] = float(np.sqrt(np.mean(r * r)))
        z = (x - r).ravel() / max(out[k]["rms"], 1e-30)
        out[k]["err_std_over_rms"] = float(np.std(z))
        out[k]["err_kurtosis"] = float(np.mean(z ** 4) / max(np.mean(z ** 2) ** 2, 1e-300))
print(json.dumps(out, indent=1))
