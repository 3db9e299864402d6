"""Per-tensor normwise errors of the bf16 path vs the fp64 oracle (tiny c1 config)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import zb_synth
import test_gpu_stage as t
cfg = zb_synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
ref_loss, ref = t.oracle_grads(cfg, "bf16")
loss, grads, _ = t.gpu_run(cfg, 4, "bf16", "zbh1")
errs = sorted(((t.rel(grads[k], ref[k]), k) for k in ref), reverse=True)
print("loss", loss, ref_loss, "mean err", np.mean([e for e, _ in errs]))
for e, k in errs[:15]: print(f"{e:.4e} {k}")
