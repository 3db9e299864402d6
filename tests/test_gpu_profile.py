"""SURVEY §8(a) a1 "Profile" -> a2 "Schedule" on the GPU ("we first
conducted a specific number of iterations for profiling, collecting ... T_F, T_B,
T_W ... fed them into our automatic pipeline scheduling algorithm").

Per-stage pass times measured through zb_ctx_profile (CUDA events, median int64 ns)
on p virtual stages feed zb_schedule_per_stage; the AUTO pass lists it returns must
be IDENTICAL to the oracle's AUTO (oracle/schedule.py) on the same integers, and
executing them gives gradients bitwise equal to ZB-H1's."""
import numpy as np
import pytest

import zb_synth
from zbtest_util import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


def _ctxs(cfg, p, n_slots, dtype="bf16"):
    from paper_2401_10241_b200 import api
    out = []
    for s in range(p):
        c = api.Context(cfg, p, s, cfg.m, n_slots, dtype=dtype)
        prm = zb_synth.make_stage_params(cfg, p, s)
        c.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
        out.append(c)
    return out


def _grads(ctxs, cfg, p):
    g = {}
    for s, c in enumerate(ctxs):
        for (name, shape, _), x in zip(zb_synth.param_specs(cfg, p, s), c.get_grads()):
            g[name] = x.reshape(shape)
    return g


def test_profiled_times_drive_auto_schedule_identical_to_oracle():
    import torch
    from oracle import schedule as osch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.ModelConfig("prof", h=256, a=2, L=6, s=256, b=2, V=512, p=3, m=6, family="auto")
    p, m = 3, cfg.m
    tok = zb_synth.make_tokens(cfg, 0)
    tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
    base, _ = api.schedule("zbh1", p, m, 1, 1, 1)
    ctxs = _ctxs(cfg, p, 2 * p)
    for c in ctxs:
        c.profile(reset=True)
    for _ in range(3):                      # profiling iterations
        api.run_local(ctxs, base, tin, lab, timing=True)
        for c in ctxs:
            c.profile()
    prof = [c.profile() for c in ctxs]
    TF = [t[0] for t, _ in prof]
    TB = [t[1] for t, _ in prof]
    TW = [t[2] for t, _ in prof]
    assert all(n == [3 * m] * 3 for _, n in prof), prof
    assert min(TF + TB + TW) > 0
    slot_b = api.slot_bytes(ctxs[1].mc)
    lim = 2 * p * slot_b
    passes, sim = api.schedule_per_stage("auto", p, m, TF, TB, TW, 0, M_limit=lim, M_B=slot_b, M_W=slot_b)
    lists, maps, counts, osim, chosen = osch.schedule("auto", p, m, TF, TB, TW, 0, MB=slot_b, MW=slot_b, Mlimit=lim)
    assert api.stage_lists(passes, p) == [list(o) for o in lists]
    assert sim.cost == osim["cost"] and sim.chosen == chosen
    assert list(sim.n_slots[:p]) == counts
    # the last stage carries the LM head in its B (DESIGN.md R-head)
    assert TB[-1] > TB[1]
    # the profiled AUTO schedule runs and reproduces ZB-H1's gradients bitwise
    ref = _grads(ctxs, cfg, p)
    ctxs2 = _ctxs(cfg, p, max(2 * p, max(sim.n_slots[:p])))
    api.run_local(ctxs2, passes, tin, lab)
    got = _grads(ctxs2, cfg, p)
    for k in ref:
        assert np.array_equal(got[k], ref[k]), k


def test_profile_reset_and_single_collection():
    import torch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.ModelConfig("prof1", h=128, a=2, L=2, s=128, b=1, V=256, p=1, m=3, family="zbh1")
    passes, _ = api.schedule("zbh1", 1, cfg.m, 1, 1, 1)
    ctx = _ctxs(cfg, 1, 1)[0]
    tok = zb_synth.make_tokens(cfg, 0)
    tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
    ctx.profile(reset=True)
    ctx.run_iteration(passes, tin, lab, timing=True)
    t1, n1 = ctx.profile()
    t2, n2 = ctx.profile()                  # the same run is not collected twice
    assert n1 == n2 == [cfg.m] * 3 and t1 == t2
    starts, ends = ctx.stats()              # read_stats still sees the run
    assert len(starts) == 3 * cfg.m
    ctx.run_iteration(passes, tin, lab, timing=True)
    _, n3 = ctx.profile()
    assert n3 == [2 * cfg.m] * 3
    ctx.profile(reset=True)
    _, n4 = ctx.profile()
    assert n4 == [0, 0, 0]
