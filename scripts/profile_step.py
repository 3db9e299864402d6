"""One microbatch F/B/W (+ optimizer) of a config at p=1, bracketed by
cudaProfilerStart/Stop for `ncu --profile-from-start off` launch lists."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import zb_synth
from paper_2401_10241_b200 import api

ap = argparse.ArgumentParser(); ap.add_argument("--config", default="1.5B"); ap.add_argument("--m", type=int, default=1)
ap.add_argument("--layers", type=int, default=2)
a = ap.parse_args()
cfg = zb_synth.CONFIGS[a.config].with_(m=a.m, L=a.layers)
passes, sim = api.schedule("zbh1", 1, cfg.m, 1, 1, 1)
ctx = api.Context(cfg, 1, 0, cfg.m, sim.n_slots[0], dtype="bf16")
prm = zb_synth.make_stage_params(cfg, 1, 0)
ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, 1, 0)])
tok = zb_synth.make_tokens(cfg, 0)
t = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda(); l = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
opt = api.optim_cfg(mode="pv")
for i in range(2):
    if i == 1: torch.cuda.synchronize(); torch.cuda.profiler.start()
    ctx.run_iteration(passes, t, l); ctx.post_validate_step(opt); ctx.post_validate_finish(opt)
    torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("loss", ctx.loss())
