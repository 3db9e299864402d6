"""Memory-limit sweep (§5.4 / Fig. 5 and §6 Fig. 7 analogues, P:300-302, P:436;
App. B) on B200-measured inputs: the per-layer F / B / W times of the
latest N=1 bench line (profiles/*bench*final.json, scaled to a p = 8 stage of the
1.5B model), M_B = M_W = this build's stash bytes per stage (zb_ctx_slot_bytes),
T_comm assumed 20 us (NVLink P2P of a 28 MB activation at ~770 GB/s + latency).
For M_limit in [M_B, 3p M_B]: the AUTO schedule's simulated bubble rate
(zb_schedule) and ZB-V's with the W right-shift under the same per-worker limit
(zb_schedule_chunked, two chunks of half a stage each), next to App. B's plateau
threshold k* M_B and zero-bubble memory.  Host-only (no GPU)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import zb_synth
from paper_2401_10241_b200 import api
from oracle import schedule as osch   # closed forms of App. B only (the schedules come from libzb)

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bench = json.load(open(os.path.join(root, "profiles", "r01_bench_1p5b_n1_final.json")))
us = bench["bubble"]["T_us"]                     # one 3-layer stage of 1.5B at p = 8
TF, TB, TW, TC = us["F"], us["B"], us["W"], 20
cfg = zb_synth.CONFIGS["1.5B"]
p, m = 8, cfg.m
MB = api.slot_bytes(api.model_cfg(cfg, p, 1, m, 1))   # a middle stage (3 layers)
MW = MB
ab = osch.appendix_b(p, TF, TB, TC, MB)
rows = []
for k in range(2, 3 * 2 * p + 1):                # M_limit = k/2 M_B
    lim = k * MB // 2
    if lim < MB:
        continue
    _, sim = api.schedule("auto", p, m, TF, TB, TW, TC, M_limit=lim, M_B=MB, M_W=MW)
    try:
        _, simv = api.schedule_chunked("zbv", p, m, 2, TF // 2, TB // 2, TW // 2, TC, M_limit=lim, M_B=MB // 2,
                                       M_W=MW // 2)
        zbv = round(simv.bubble_rate, 4)
    except Exception:   # ZB_ELIMIT: below ZB-V's own p M_B
        zbv = None
    rows.append({"M_limit_over_MB": k / 2, "auto_bubble": round(sim.bubble_rate, 4), "auto_chosen": sim.chosen,
                 "auto_peak_over_MB": round(max(sim.peak_bytes[:p]) / MB, 2), "zbv_bubble": zbv})
out = {"inputs": {"T_F_us": TF, "T_B_us": TB, "T_W_us": TW, "T_comm_us": TC, "M_B_bytes": MB, "p": p, "m": m,
                  "source": "profiles/r01_bench_1p5b_n1_final.json (per-layer pass times x 3 layers)"},
       "appendix_b": {"k_star": ab["k_star"], "plateau_M_over_MB": ab["k_star"],
                      "zero_bubble_M_over_MB": ab["m_zero"] // MB, "paper_rule_of_thumb": "2p M_B = 16 M_B"},
       "sweep": rows}
path = os.path.join(root, "profiles", "r01_memory_sweep_1p5b_p8.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out["appendix_b"]))
for r in rows:
    print(r)
