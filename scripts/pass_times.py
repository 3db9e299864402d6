"""Time F, B, W of one microbatch separately (host-synchronised) for a config:
python scripts/pass_times.py <config> <layers> — a debugging aid for new shapes."""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("PT_TIMEOUT", "240")), exit=True)
import numpy as np, torch
import zb_synth
from paper_2401_10241_b200 import api
cfg = zb_synth.CONFIGS[sys.argv[1]].with_(m=1, L=int(sys.argv[2]))
ctx = api.Context(cfg, 1, 0, 1, 1, dtype="bf16")
prm = zb_synth.make_stage_params(cfg, 1, 0)
ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, 1, 0)])
tok = zb_synth.make_tokens(cfg, 0)
t = torch.from_numpy(np.ascontiguousarray(tok[0, ..., :cfg.s])).cuda()
l = torch.from_numpy(np.ascontiguousarray(tok[0, ..., 1:])).cuda()
ctx.begin_iteration()
torch.cuda.synchronize()
for name, fn in (("F", lambda: ctx.forward(0, 0, t.data_ptr(), None, l.data_ptr())),
                 ("B", lambda: ctx.backward_input(0, 0)), ("W", lambda: ctx.backward_weight(0, 0))):
    t0 = time.time(); fn(); torch.cuda.synchronize(); print(name, round((time.time() - t0) * 1000, 2), "ms", flush=True)
