"""Predicted p = 8 bubble rates of every BASELINE config on B200-measured pass times
(§5.3's method: profiled T_F, T_B, T_W into the simulator).

Per config: one microbatch's F / B / W of a 2-layer and of a 4-layer model are timed with
CUDA events (after warm-up) at the config's h, heads, b, s, V; the difference gives the
per-layer times, the rest the embedding + LM-head edge.  A stage of the p = 8 partition
(P:169 rule) then takes L_s x per-layer (+ the head edge on the last stage), and the
schedulers run with T_comm = 20 us, M_B = M_W = this build's stash bytes of a middle
stage, and the BASELINE memory rules (c4: M_limit = 1F1B peak, c5: 2 x 1F1B peak)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import zb_synth
from paper_2401_10241_b200 import api


def pass_ms(cfg, L, reps=5):
    c = cfg.with_(m=1, L=L)
    ctx = api.Context(c, 1, 0, 1, 1, dtype="bf16")
    prm = zb_synth.make_stage_params(c, 1, 0)
    ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(c, 1, 0)])
    tok = zb_synth.make_tokens(c, 0)
    t = torch.from_numpy(np.ascontiguousarray(tok[0, ..., :c.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[0, ..., 1:])).cuda()
    out = {"F": [], "B": [], "W": []}
    for r in range(reps + 2):
        ctx.begin_iteration()
        for k, fn in (("F", lambda: ctx.forward(0, 0, t.data_ptr(), None, lab.data_ptr())),
                      ("B", lambda: ctx.backward_input(0, 0)), ("W", lambda: ctx.backward_weight(0, 0))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(); fn(); e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                out[k].append(e0.elapsed_time(e1))
    ctx.close()
    del prm
    torch.cuda.empty_cache()
    return {k: float(np.median(v)) for k, v in out.items()}


res = {}
for name in ("1.5B", "6.2B", "14.6B", "28.3B"):
    cfg = zb_synth.CONFIGS[name]
    t2, t4 = pass_ms(cfg, 2), pass_ms(cfg, 4)
    layer = {k: (t4[k] - t2[k]) / 2 for k in "FBW"}
    edge = {k: t2[k] - 2 * layer[k] for k in "FBW"}
    p, m = 8, cfg.m
    Lmid = (cfg.L + 2) // p if (cfg.L + 2) % p == 0 else -(-cfg.L // p)
    us = {k: int(round(layer[k] * Lmid * 1000)) for k in "FBW"}
    MB = api.slot_bytes(api.model_cfg(cfg, p, 1, m, 1))
    row = {"per_layer_ms": layer, "edge_ms": edge, "layers_per_stage": Lmid, "T_us": us, "m": m,
           "M_B_bytes": MB}
    for fam in ("1f1b", "zbh1", "zbh2"):
        if fam == "zbh2" and m < 2 * p - 1:
            continue
        _, sim = api.schedule(fam, p, m, us["F"], us["B"], us["W"], 20, M_B=MB, M_W=MB)
        row[fam] = round(sim.bubble_rate, 4)
    for mult in (1, 2):
        _, sim = api.schedule("auto", p, m, us["F"], us["B"], us["W"], 20, M_limit=mult * p * MB, M_B=MB, M_W=MB)
        row[f"auto_{mult}pMB"] = round(sim.bubble_rate, 4)
    _, sim = api.schedule_chunked("zbv", p, m, 2, us["F"] // 2, us["B"] // 2, us["W"] // 2, 20, M_B=MB // 2,
                                  M_W=MB // 2)
    row["zbv_pMB"] = round(sim.bubble_rate, 4)
    res[name] = row
    print(name, json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/predicted_configs.json", "w"), indent=1)
