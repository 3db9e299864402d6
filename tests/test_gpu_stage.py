"""GPU parity of whole stage passes F / B / W and iterations through the C-ABI
against the fp64 oracle (oracle/model.py) on the same seeded inputs.

Tolerances (BASELINE.json north_star): f32 mode normwise relative
error <= 1e-5 for the loss and every gradient; bf16 mode (bf16 operands,
f32 accumulation) <= 2e-2 per tensor and <= 1e-2 mean over tensors.  Schedules
must produce bitwise-identical gradients."""
import numpy as np
import pytest

import zb_synth
from zbtest_util import close_report, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

SHAPES = {
    "d64": zb_synth.ModelConfig("d64", h=64, a=1, L=4, s=256, b=2, V=512, p=4, m=3, family="zbh1"),
    "d96": zb_synth.ModelConfig("d96", h=192, a=2, L=2, s=128, b=2, V=264, p=2, m=2, family="zbh1"),
    "d128": zb_synth.ModelConfig("d128", h=256, a=2, L=2, s=192, b=1, V=512, p=2, m=2, family="zbh1"),
}
MATRICES = ("qkv_w", "proj_w", "fc1_w", "fc2_w", "head_w")


def rel(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / max(np.linalg.norm(ref), 1e-30))


def inputs(cfg, it=0):
    tok = zb_synth.make_tokens(cfg, it)
    return np.ascontiguousarray(tok[..., :cfg.s]), np.ascontiguousarray(tok[..., 1:])


def make_ctxs(cfg, p, dtype, family="zbh1", n_slots=None):
    from paper_2401_10241_b200 import api
    passes, sim = api.schedule(family, p, cfg.m, 10, 11, 6, 0, M_limit=2 * p * 10 if family == "auto" else 0,
                               M_B=10, M_W=10)
    ctxs = []
    for s in range(p):
        c = api.Context(cfg, p, s, cfg.m, max(1, sim.n_slots[s]), dtype=dtype)
        params = zb_synth.make_stage_params(cfg, p, s)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
        ctxs.append(c)
    return ctxs, passes


def oracle_grads(cfg, dtype):
    from oracle import model as om
    params = zb_synth.make_model_params(cfg)
    if dtype == "bf16":
        params = {k: (zb_synth.round_to_bf16(v) if k.endswith(MATRICES) else v) for k, v in params.items()}
    tok = zb_synth.make_tokens(cfg, 0)
    return om.reference_iteration(cfg, params, tok)


def gpu_run(cfg, p, dtype, family="zbh1"):
    import torch
    from paper_2401_10241_b200 import api
    ctxs, passes = make_ctxs(cfg, p, dtype, family)
    tok, lab = inputs(cfg)
    tok_d = torch.from_numpy(tok).cuda()
    lab_d = torch.from_numpy(lab).cuda()
    if p == 1:
        ctxs[0].run_iteration(passes, tok_d, lab_d)
    else:
        api.run_local(ctxs, passes, tok_d, lab_d)
    loss = ctxs[-1].loss()
    grads = {}
    for s, c in enumerate(ctxs):
        for (name, shape, _), g in zip(zb_synth.param_specs(cfg, p, s), c.get_grads()):
            grads[name] = g.reshape(shape)
    return loss, grads, ctxs


def check_tolerance(loss, grads, ref_loss, ref_grads, dtype):
    """per tensor the normwise relative error AND the elementwise
    bound (zbtest_util.close_report: f32 |x - ref| <= rtol*|ref| + rtol*rms(ref);
    bf16 the row-aware floor with kappa = sqrt(2 ln N), DESIGN R-tol); f32 rtol 1e-5, bf16
    rtol 2e-2 per tensor and normwise mean over tensors <= 1e-2."""
    rtol = 1e-5 if dtype == "f32" else 2e-2
    rep = {k: close_report(grads[k], ref_grads[k], rtol, bf16=dtype != "f32", exact_zero_rows=True) for k in ref_grads}
    errs = {k: r[0] for k, r in rep.items()}
    assert abs(loss - ref_loss) <= rtol * abs(ref_loss), (loss, ref_loss)
    bad = {k: e for k, e in errs.items() if e > rtol}
    assert not bad, bad
    bad_el = {k: round(r[1], 3) for k, r in rep.items() if r[1] > 1.0}
    assert not bad_el, f"elementwise bound exceeded (x bound): {bad_el}"
    if dtype != "f32":
        assert np.mean(list(errs.values())) <= 1e-2
    return errs


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", list(SHAPES))
def test_single_stage_iteration_vs_oracle(shape, dtype):
    cfg = SHAPES[shape]
    ref_loss, ref = oracle_grads(cfg, dtype)
    loss, grads, _ = gpu_run(cfg, 1, dtype)
    check_tolerance(loss, grads, ref_loss, ref, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_virtual_stages_bitwise_across_schedules(dtype):
    """identical results across 1F1B / ZB-H1 / ZB-H2 / AUTO (and p = 1)."""
    cfg = SHAPES["d64"].with_(m=5)
    base_loss, base, _ = gpu_run(cfg, 1, dtype)
    for fam in ("1f1b", "zbh1", "zbh2", "auto"):
        loss, grads, _ = gpu_run(cfg, 4, dtype, fam)
        assert loss == base_loss, fam
        for k in base:
            assert np.array_equal(grads[k], base[k]), (fam, k)


def test_tiny_config_c1_vs_oracle_f32():
    """BASELINE.json configs[0]: tiny 8-layer stack, h 64, p 4, m 8, ZB-H1 vs 1F1B."""
    cfg = zb_synth.CONFIGS["tiny"]
    ref_loss, ref = oracle_grads(cfg, "f32")
    for fam in ("zbh1", "1f1b"):
        loss, grads, _ = gpu_run(cfg, 4, "f32", fam)
        check_tolerance(loss, grads, ref_loss, ref, "f32")


def test_tiny_config_c1_vs_oracle_bf16():
    cfg = zb_synth.CONFIGS["tiny"]
    ref_loss, ref = oracle_grads(cfg, "bf16")
    loss, grads, _ = gpu_run(cfg, 4, "bf16", "zbh1")
    check_tolerance(loss, grads, ref_loss, ref, "bf16")


def test_pass_api_and_input_copies():
    """zb_stage_forward / backward_input / backward_weight called directly with
    caller buffers (copied into the slot) equal the runner (zb_run_iteration_local)."""
    import torch
    from paper_2401_10241_b200 import api
    cfg = SHAPES["d64"].with_(m=2)
    _, ref, _ = gpu_run(cfg, 2, "f32")
    ctxs, passes = make_ctxs(cfg, 2, "f32")
    tok, lab = inputs(cfg)
    tok_d = torch.from_numpy(tok).cuda()
    lab_d = torch.from_numpy(lab).cuda()
    T, h = cfg.T, cfg.h
    act = torch.empty(T, h, device="cuda")
    grad = torch.empty(T, h, device="cuda")
    for c in ctxs:
        c.begin_iteration()
    slot = [{q.microbatch: q.slot for q in passes if q.stage == s and q.kind == 0} for s in range(2)]
    for j in range(cfg.m):
        ctxs[0].forward(j, slot[0][j], tok_d[j].data_ptr(), act.data_ptr())
        ctxs[1].forward(j, slot[1][j], act.data_ptr(), None, lab_d[j].data_ptr())
        ctxs[1].backward_input(j, slot[1][j], None, grad.data_ptr())
        ctxs[0].backward_input(j, slot[0][j], grad.data_ptr(), None)
        ctxs[1].backward_weight(j, slot[1][j])
        ctxs[0].backward_weight(j, slot[0][j])
    for s, c in enumerate(ctxs):
        for (name, shape, _), g in zip(zb_synth.param_specs(cfg, 2, s), c.get_grads()):
            assert np.array_equal(g.reshape(shape), ref[name]), name


def test_host_inputs_equal_device_inputs():
    from paper_2401_10241_b200 import api
    cfg = SHAPES["d64"].with_(m=2)
    loss_d, ref, _ = gpu_run(cfg, 1, "bf16")
    ctxs, passes = make_ctxs(cfg, 1, "bf16")
    tok, lab = inputs(cfg)
    ctxs[0].run_iteration(passes, tok, lab, host_inputs=True)
    assert ctxs[0].loss() == loss_d
    for (name, shape, _), g in zip(zb_synth.param_specs(cfg, 1, 0), ctxs[0].get_grads()):
        assert np.array_equal(g.reshape(shape), ref[name])


# ------------------------------------------------------------------ optimizer + post-validation

def _params_of(ctxs, cfg, p):
    out = {}
    for s, c in enumerate(ctxs):
        for (name, shape, _), v in zip(zb_synth.param_specs(cfg, p, s), c.get_params()):
            out[name] = v.reshape(shape)
    return out


@pytest.mark.parametrize("clip_mode", ["none", "stage0-rollback", "all-defer"])
def test_post_validation_vs_sync_and_oracle(clip_mode):
    from oracle import optim as oo
    from paper_2401_10241_b200 import api
    cfg = SHAPES["d64"]
    p = 4
    _, g_all, ctx_sync = gpu_run(cfg, p, "f32")
    _, _, ctx_pv = gpu_run(cfg, p, "f32")
    # stage-local squared norms decide which path each stage takes
    loc = [sum(float(np.sum(g.astype(np.float64) ** 2)) for g in c.get_grads()) for c in ctx_sync]
    clip = {"none": 1e6, "stage0-rollback": float(np.sqrt(loc[0])) * 1.001,
            "all-defer": float(np.sqrt(loc[0])) * 0.5}[clip_mode]
    hyp = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, clip=clip)
    api.post_validate_local(ctx_sync, api.optim_cfg(mode="sync", **hyp))
    api.post_validate_local(ctx_pv, api.optim_cfg(mode="pv", **hyp))
    reps = [c.pv_report() for c in ctx_pv]
    if clip_mode == "none":
        assert [r["first"] for r in reps] == ["step"] * p and [r["final"] for r in reps] == ["none"] * p
    elif clip_mode == "stage0-rollback":
        assert reps[0]["first"] == "step" and reps[0]["final"] == "rollback+redo"
        assert all(r["first"] == "defer" and r["final"] == "deferred-step" for r in reps[1:])
    else:
        assert all(r["first"] == "defer" and r["final"] == "deferred-step" for r in reps)
    assert all(r["t"] == 1 for r in reps)
    ps, pp = _params_of(ctx_sync, cfg, p), _params_of(ctx_pv, cfg, p)
    for k in ps:
        if clip_mode == "stage0-rollback" and k in {n for n, _, _ in zb_synth.param_specs(cfg, p, 0)}:
            assert rel(pp[k], ps[k]) < 1e-6, k       # rounding of the f32 inverse step
        else:
            assert np.array_equal(pp[k], ps[k]), k   # clean / deferred paths: bitwise
    # the synchronous GPU step against Algorithm 1 in fp64 on the same gradients
    theta0 = zb_synth.make_model_params(cfg)
    S = sum(loc)
    coef = min(1.0, clip / (np.sqrt(S) + 1e-6))
    for k, v in ps.items():
        wd = 0.1 if theta0[k].ndim >= 2 else 0.0
        want, _, _, _ = oo.adamw_step(theta0[k].astype(np.float64), 0.0, 0.0, 0, g_all[k].astype(np.float64) * coef,
                                      1e-3, 0.9, 0.95, 1e-8, wd)
        assert rel(v, want) < 1e-6, k


def test_nan_skips_step_everywhere():
    from paper_2401_10241_b200 import api
    cfg = SHAPES["d64"]
    p = 2
    ctxs, passes = make_ctxs(cfg, p, "f32")
    params = zb_synth.make_stage_params(cfg, p, 1)
    lst = [params[n] for n, _, _ in zb_synth.param_specs(cfg, p, 1)]
    lst[0] = lst[0].copy()
    lst[0][0] = np.nan                      # stage 1's first LayerNorm gain
    ctxs[1].set_params(lst)
    import torch
    tok, lab = inputs(cfg)
    api.run_local(ctxs, passes, torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda())
    before = [c.get_params() for c in ctxs]
    api.post_validate_local(ctxs, api.optim_cfg(mode="pv", lr=1e-3))
    for c, b in zip(ctxs, before):
        r = c.pv_report()
        assert r["full_nonfinite"] == 1 and r["t"] == 0
        for x, y in zip(c.get_params(), b):
            assert np.array_equal(x, y, equal_nan=True)


def gpu_run_chunked(cfg, p, chunks, family, dtype):
    """p workers holding `chunks` model chunks each (ZB-V / 1F1B-I) run as
    chunks*p virtual-stage contexts in one process (zb_run_iteration_local)."""
    import torch
    from paper_2401_10241_b200 import api
    nv = chunks * p
    passes, sim = api.schedule_chunked(family, p, cfg.m, chunks, 10, 11, 6, 1, M_B=10, M_W=10)
    ctxs = []
    for v in range(nv):
        c = api.Context(cfg, nv, v, cfg.m, max(1, sim.n_slots[v]), dtype=dtype)
        params = zb_synth.make_stage_params(cfg, nv, v)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, nv, v)])
        ctxs.append(c)
    tok, lab = inputs(cfg)
    api.run_local(ctxs, passes, torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda())
    grads = {}
    for v, c in enumerate(ctxs):
        for (name, shape, _), g in zip(zb_synth.param_specs(cfg, nv, v), c.get_grads()):
            grads[name] = g.reshape(shape)
    return ctxs[-1].loss(), grads


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_chunked_schedules_vs_oracle_and_bitwise(dtype):
    """ZB-V and 1F1B-I on BASELINE configs[0] (8 layers,
    p = 4 workers x 2 chunks of one layer): within tolerance of the oracle and
    bitwise equal to 1F1B over the same 8 chunks."""
    cfg = zb_synth.CONFIGS["tiny"]
    ref_loss, ref = oracle_grads(cfg, dtype)
    base_loss, base, _ = gpu_run(cfg, 8, dtype, "1f1b")
    for fam in ("zbv", "1f1bi"):
        loss, grads = gpu_run_chunked(cfg, 4, 2, fam, dtype)
        check_tolerance(loss, grads, ref_loss, ref, dtype)
        assert loss == base_loss, fam
        for k in base:
            assert np.array_equal(grads[k], base[k]), (fam, k)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_head_weight_gradient_in_w_equals_eager(dtype):
    """DESIGN R-head: the LM head's dW runs in the last stage's W pass (dlogits kept in the
    slot) by default; ZB_CFG_HEAD_W_EAGER runs it inside B.  Same per-microbatch order ->
    bitwise identical gradients; the deferred mode's last-stage slot holds 2 T V more bytes."""
    import torch
    from paper_2401_10241_b200 import api
    cfg = SHAPES["d96"].with_(m=3)
    p = 2
    passes, sim = api.schedule("zbh1", p, cfg.m, 10, 11, 6)
    tok, lab = inputs(cfg)
    tin, tl = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
    out = []
    for eager in (False, True):
        ctxs = []
        for s in range(p):
            c = api.Context(cfg, p, s, cfg.m, max(1, sim.n_slots[s]), dtype=dtype, head_w_eager=eager)
            prm = zb_synth.make_stage_params(cfg, p, s)
            c.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
            ctxs.append(c)
        api.run_local(ctxs, passes, tin, tl)
        out.append((ctxs[-1].loss(), [c.get_grads() for c in ctxs], [api.slot_bytes(c.mc) for c in ctxs]))
    (l0, g0, b0), (l1, g1, b1) = out
    assert l0 == l1
    for a, b in zip(g0, g1):
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
    esz = 2 if dtype == "bf16" else 4
    assert b0[0] == b1[0] and b0[-1] - b1[-1] >= cfg.T * cfg.V * esz


# ------------------------------------------------------------------ CUDA-graph replay (ZB_RUN_GRAPH)

def test_graph_replay_bitwise_equals_eager():
    """zb_run_iteration with ZB_RUN_GRAPH: eager on a new key, captured on the second call,
    replayed after that — loss, gradients and post-validated parameters bitwise equal to the
    eager context's over several iterations with per-step device input buffers (staged into
    the context), ordered split-K W GEMMs inside the graph (T = 2048: the W launches split K),
    and a re-key when the pass list changes."""
    import torch
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import lib
    import ctypes as C
    cfg = zb_synth.ModelConfig("graph", h=256, a=2, L=2, s=1024, b=2, V=512, p=1, m=3, family="zbh1")
    opt = api.optim_cfg(lr=1e-3, mode="pv", clip=1.0)
    runs = []
    passes, sim = api.schedule("zbh1", 1, cfg.m, 10, 11, 6, 0, M_B=10, M_W=10)
    passes_h2, sim2 = api.schedule("zbh2", 1, cfg.m, 10, 11, 6, 0, M_B=10, M_W=10)
    for graph in (False, True):
        stream = torch.cuda.Stream()  # a capturable stream (the legacy default stream is not)
        c = api.Context(cfg, 1, 0, cfg.m, max(sim.n_slots[0], sim2.n_slots[0]), dtype="bf16", stream=stream)
        params = zb_synth.make_stage_params(cfg, 1, 0)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, 1, 0)])
        out = []
        for it in range(5):
            q = passes if it < 4 else passes_h2
            tok, lab = inputs(cfg, it)
            with torch.cuda.stream(stream):
                tok_d = torch.from_numpy(tok).cuda()
                lab_d = torch.from_numpy(lab).cuda()
            n0 = C.c_int64()
            lib.zb_dbg_launch_count(1, C.byref(n0))
            c.run_iteration(q, tok_d, lab_d, graph=graph)
            n1 = C.c_int64()
            lib.zb_dbg_launch_count(0, C.byref(n1))
            loss = c.loss()
            grads = [g.copy() for g in c.get_grads()]
            c.post_validate_step(opt)
            c.post_validate_finish(opt)
            out.append((loss, grads, [v.copy() for v in c.get_params()], int(n1.value)))
        runs.append(out)
        c.close()
    for it, (e, g) in enumerate(zip(*runs)):
        assert e[0] == g[0], (it, e[0], g[0])
        for a, b in zip(e[1], g[1]):
            assert np.array_equal(a, b), it
        for a, b in zip(e[2], g[2]):
            assert np.array_equal(a, b), it
        assert e[3] == g[3] > 0, (it, e[3], g[3])  # a replay counts its kernel nodes
