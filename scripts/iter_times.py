"""Host-timed iterations / post-validation of a truncated config (debugging aid): python scripts/iter_times.py <config> <layers> <m>"""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("IT_TIMEOUT", "200")), exit=True)
import numpy as np, torch
import zb_synth
from paper_2401_10241_b200 import api
name, L, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = zb_synth.CONFIGS[name].with_(m=m, L=L)
for kv in sys.argv[4:]:            # overrides, e.g. a=18 b=1
    k, v = kv.split("=")
    cfg = cfg.with_(**{k: int(v)})
print(cfg, flush=True)
passes, sim = api.schedule("zbh1", 1, cfg.m, 1, 1, 1)
ctx = api.Context(cfg, 1, 0, cfg.m, sim.n_slots[0], dtype="bf16")
prm = zb_synth.make_stage_params(cfg, 1, 0)
ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, 1, 0)])
tok = zb_synth.make_tokens(cfg, 0)
t = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda(); l = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
opt = api.optim_cfg(mode="pv")
for i in range(int(os.environ.get("IT_ITERS", "3"))):
    t0 = time.time(); ctx.run_iteration(passes, t, l); torch.cuda.synchronize(); t1 = time.time()
    ctx.post_validate_step(opt); torch.cuda.synchronize(); t2 = time.time()
    ctx.post_validate_finish(opt); torch.cuda.synchronize(); t3 = time.time()
    print(i, "iter", round((t1-t0)*1e3,1), "pv_step", round((t2-t1)*1e3,1), "finish", round((t3-t2)*1e3,1), "loss", ctx.loss(), flush=True)
