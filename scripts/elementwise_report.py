"""Elementwise error structure of the bf16 path against the fp64 oracle (diagnostic for
the SURVEY C15 elementwise bound): per gradient tensor the normwise error, the worst
|x - ref| / (rtol |ref| + rtol rms(ref)) with the global rms floor, with a structured
floor s_oi = rowrms_o * colrms_i / rms (the scale of a dW = dY^T X element), and the
location of the worst element."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import zb_synth
from test_gpu_stage import gpu_run, oracle_grads, SHAPES


def report(x, ref, rtol=2e-2):
    x = np.asarray(x, np.float64); ref = np.asarray(ref, np.float64)
    d = np.abs(x - ref)
    nrm = float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-30))
    rms = float(np.sqrt(np.mean(ref * ref)))
    r1 = d / (rtol * np.abs(ref) + rtol * rms + 1e-300)
    out = {"normwise": nrm, "global_floor": float(r1.max())}
    if ref.ndim == 2:
        rr = np.sqrt(np.mean(ref * ref, axis=1, keepdims=True))
        cr = np.sqrt(np.mean(ref * ref, axis=0, keepdims=True))
        s = rr * cr / max(rms, 1e-300)
        r2 = d / (rtol * np.abs(ref) + rtol * s + 1e-300)
        zero_rows = rr[:, 0] == 0
        out["struct_floor"] = float(np.where(np.isfinite(r2), r2, 0).max())
        out["zero_ref_rows"] = int(zero_rows.sum())
        out["max_abs_on_zero_rows"] = float(d[zero_rows].max()) if zero_rows.any() else 0.0
        i = np.unravel_index(np.argmax(r1), r1.shape)
        out["worst_global"] = {"at": [int(i[0]), int(i[1])], "ref": float(ref[i]), "err": float(d[i]),
                               "row_rms": float(rr[i[0], 0]), "rms": rms}
        # error std relative to the structured scale
        z = (x - ref) / np.where(s > 0, s, 1)
        out["err_over_scale_std"] = float(np.std(z[~zero_rows])) if (~zero_rows).any() else 0.0
        out["n"] = int(ref.size)
    return out


cases = {"1.5B_L1": zb_synth.CONFIGS["1.5B"].with_(L=1, b=1, m=1), "d96": SHAPES["d96"], "d64": SHAPES["d64"],
         "tiny": zb_synth.CONFIGS["tiny"]}
res = {}
for name, cfg in cases.items():
    p = 4 if name == "tiny" else 1
    ref_loss, ref = oracle_grads(cfg, "bf16")
    loss, grads, _ = gpu_run(cfg, p, "bf16")
    res[name] = {k: report(grads[k], ref[k]) for k in ref}
    worst = sorted(res[name].items(), key=lambda kv: -kv[1].get("global_floor", 0))[:6]
    print(name, json.dumps(worst, indent=0)[:4000], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/elementwise_report.json", "w"), indent=1)
