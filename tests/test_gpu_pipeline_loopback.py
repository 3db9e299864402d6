"""The multi-stage runner (comm.cu: plan.cpp's op lists with P2P sends /
receives, post-validation chains, speculative Fs and replays) executed on one
GPU: p stage contexts of one process, each driven by its own host thread and
CUDA stream, exchange messages through the in-process loopback transport
(zb_ctx_attach_loopback) instead of NCCL.  Everything except the NCCL calls
themselves is the code path a p-GPU run takes.

Reference: the same contexts driven by zb_run_iteration_local (virtual stages,
P2P replaced by device copies) and zb_post_validate_local, which the other
GPU tests pin to the fp64 oracle.  Results must be bitwise identical: the
same kernels run on the same data in the same per-stage order."""
import threading

import numpy as np
import pytest

import zb_synth
from zbtest_util import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

CFG = zb_synth.ModelConfig("lb", h=64, a=1, L=6, s=256, b=2, V=512, p=4, m=6, family="zbh1")


@pytest.fixture(autouse=True)
def _short_timeout(monkeypatch):
    monkeypatch.setenv("ZB_LOOPBACK_TIMEOUT_S", "60")


def _inputs(cfg, it):
    import torch
    tok = zb_synth.make_tokens(cfg, it)
    return (torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda(),
            torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda())


def _contexts(cfg, p, dtype, family, own_streams):
    import torch
    from paper_2401_10241_b200 import api
    passes, sim = api.schedule(family, p, cfg.m, 10, 11, 6, 0, M_limit=2 * p * 10 if family == "auto" else 0,
                               M_B=10, M_W=10)
    ctxs = []
    for s in range(p):
        st = torch.cuda.Stream() if own_streams else None
        c = api.Context(cfg, p, s, cfg.m, max(1, sim.n_slots[s]), dtype=dtype, stream=st)
        params = zb_synth.make_stage_params(cfg, p, s)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
        ctxs.append(c)
    return ctxs, passes


def _threads(ctxs, fn):
    """Run fn(rank, ctx) on one host thread per stage; re-raise the first error."""
    errs = [None] * len(ctxs)

    def body(r):
        try:
            fn(r, ctxs[r])
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a stage thread did not finish"
    for e in errs:
        if e is not None:
            raise e


def _state(ctxs):
    for c in ctxs:
        c.sync()
    return ctxs[-1].loss(), [c.get_grads() for c in ctxs], [c.get_params() for c in ctxs]


def _assert_same(a, b, what):
    la, ga, pa = a
    lb, gb, pb = b
    assert la == lb or (np.isnan(la) and np.isnan(lb)), (what, la, lb)
    for s, (x, y) in enumerate(zip(ga, gb)):
        for i, (u, v) in enumerate(zip(x, y)):
            assert np.array_equal(u, v, equal_nan=True), (what, "grad", s, i)
    for s, (x, y) in enumerate(zip(pa, pb)):
        for i, (u, v) in enumerate(zip(x, y)):
            assert np.array_equal(u, v, equal_nan=True), (what, "param", s, i)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("family", ["zbh1", "zbh2", "auto", "1f1b"])
def test_loopback_iteration_equals_virtual_stages(family, dtype):
    import torch
    from paper_2401_10241_b200 import api
    p = CFG.p
    tok, lab = _inputs(CFG, 0)
    ref, passes = _contexts(CFG, p, dtype, family, own_streams=False)
    api.run_local(ref, passes, tok, lab)
    want = _state(ref)

    ctxs, passes = _contexts(CFG, p, dtype, family, own_streams=True)
    group = api.Loopback(p)
    for c in ctxs:
        c.attach_loopback(group)
    torch.cuda.synchronize()
    _threads(ctxs, lambda r, c: c.run_iteration(passes, tok if r == 0 else None, lab if r == p - 1 else None,
                                                fused=(family == "1f1b")))
    _assert_same(_state(ctxs), want, family)


@pytest.mark.parametrize("case", ["clean", "rollback", "nan"])
def test_loopback_post_validation_with_speculation(case):
    """Two iterations with the post-validated step in between: the
    loopback pipeline validates INSIDE iteration 2 after each stage's
    speculative warm-up Fs (replayed when the step is amended: clip or NaN);
    the reference validates before iteration 2 starts (zb_post_validate_local)."""
    import torch
    from paper_2401_10241_b200 import api
    p, dtype, family = CFG.p, "f32", "zbh1"
    tok1, lab1 = _inputs(CFG, 0)
    tok2, lab2 = _inputs(CFG, 1)

    def setup(own_streams):
        ctxs, passes = _contexts(CFG, p, dtype, family, own_streams)
        if case == "nan":
            params = zb_synth.make_stage_params(CFG, p, 2)
            lst = [params[n] for n, _, _ in zb_synth.param_specs(CFG, p, 2)]
            lst[0] = lst[0].copy()
            lst[0][0] = np.nan
            ctxs[2].set_params(lst)
        return ctxs, passes

    ref, passes = setup(False)
    api.run_local(ref, passes, tok1, lab1)
    if case == "rollback":   # clip just above stage 0's own norm: stage 0 steps optimistically, then rolls back
        loc0 = sum(float(np.sum(g.astype(np.float64) ** 2)) for g in ref[0].get_grads())
        clip = float(np.sqrt(loc0)) * 1.001
    else:
        clip = 1e6
    opt = api.optim_cfg(mode="pv", lr=1e-3, clip=clip)
    api.post_validate_local(ref, opt)
    rep_ref = [c.pv_report() for c in ref]
    api.run_local(ref, passes, tok2, lab2)
    want = _state(ref)

    ctxs, passes = setup(True)
    group = api.Loopback(p)
    for c in ctxs:
        c.attach_loopback(group)
    torch.cuda.synchronize()

    def stage(r, c):
        c.run_iteration(passes, tok1 if r == 0 else None, lab1 if r == p - 1 else None)
        c.post_validate_step(opt)
        c.run_iteration(passes, tok2 if r == 0 else None, lab2 if r == p - 1 else None)
        c.post_validate_finish(opt)   # nothing pending: validated inside iteration 2
    _threads(ctxs, stage)
    got = _state(ctxs)
    reps = [c.pv_report() for c in ctxs]
    for a, b in zip(reps, rep_ref):
        assert (a["first"], a["final"], a["t"]) == (b["first"], b["final"], b["t"]), (a, b)
    if case == "rollback":
        assert reps[0]["final"] == "rollback+redo"
    if case == "nan":
        assert all(r["final"] in ("skip", "none") and r["t"] == 0 for r in reps), reps
        assert np.isnan(got[0])
    _assert_same(got, want, case)


# ---------------------------------------------------------------- chunked schedules (ZB-V, 1F1B-I)
CFG_V = zb_synth.ModelConfig("lbv", h=64, a=1, L=8, s=256, b=2, V=512, p=4, m=8, family="zbh1")


def _chunk_contexts(cfg, p, family, dtype, own_streams):
    import torch
    from paper_2401_10241_b200 import api
    nv = 2 * p
    passes, sim = api.schedule_chunked(family, p, cfg.m, 2, 10, 11, 6, 1, M_B=10, M_W=10)
    ctxs = []
    for v in range(nv):
        st = torch.cuda.Stream() if own_streams else None
        c = api.Context(cfg, nv, v, cfg.m, max(1, sim.n_slots[v]), dtype=dtype, stream=st)
        params = zb_synth.make_stage_params(cfg, nv, v)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, nv, v)])
        ctxs.append(c)
    per = 3 * 2 * cfg.m
    workers = [sorted({passes[i].stage for i in range(w * per, (w + 1) * per)}) for w in range(p)]
    return ctxs, passes, workers


@pytest.mark.parametrize("family", ["zbv", "1f1bi"])
def test_loopback_chunked_workers_equal_virtual_stages(family):
    """p = 4 workers x 2 chunks (P:318 V placement / cyclic 1F1B-I), each worker
    one host thread running zb_run_iteration_worker in its own pass order over
    the loopback transport; two iterations with the post-validated step between
    (steps in ascending v, finishes in descending v per worker).  Reference: the
    same 8 chunk contexts under zb_run_iteration_local / zb_post_validate_local."""
    import torch
    from paper_2401_10241_b200 import api
    p, dtype = CFG_V.p, "bf16"
    nv = 2 * p
    tok1, lab1 = _inputs(CFG_V, 0)
    tok2, lab2 = _inputs(CFG_V, 1)
    opt = api.optim_cfg(mode="pv", lr=1e-3, clip=1e6)
    ref, passes, workers = _chunk_contexts(CFG_V, p, family, dtype, own_streams=False)
    api.run_local(ref, passes, tok1, lab1)
    api.post_validate_local(ref, opt)
    api.run_local(ref, passes, tok2, lab2)
    want = _state(ref)

    ctxs, passes, workers = _chunk_contexts(CFG_V, p, family, dtype, own_streams=True)
    group = api.Loopback(nv)
    for c in ctxs:
        c.attach_loopback(group)
    torch.cuda.synchronize()
    fused = family == "1f1bi"

    def worker(w, _):
        mine = [ctxs[v] for v in workers[w]]
        for it, (tok, lab) in enumerate(((tok1, lab1), (tok2, lab2))):
            api.run_worker(mine, passes, tok if 0 in workers[w] else None, lab if nv - 1 in workers[w] else None,
                           fused=fused)
            if it == 0:
                for c in sorted(mine, key=lambda c: c.stage):
                    c.post_validate_step(opt)
                for c in sorted(mine, key=lambda c: -c.stage):
                    c.post_validate_finish(opt)
    _threads(list(range(p)), worker)
    _assert_same(_state(ctxs), want, family)


def test_hybrid_attach_single_worker_zbv():
    """zb_ctx_attach_nccl_chunks on a worker whose every link is local (ZB-V with
    p = 1: chunks v = 0, 1 on worker 0, the V turn is the in-process channel):
    the hybrid transport path without NCCL, bitwise equal to virtual stages."""
    import torch
    from paper_2401_10241_b200 import api
    cfg = CFG_V.with_(L=4, m=3)
    tok, lab = _inputs(cfg, 0)
    ref, passes, workers = _chunk_contexts(cfg, 1, "zbv", "bf16", own_streams=False)
    api.run_local(ref, passes, tok, lab)
    want = _state(ref)
    ctxs, passes, workers = _chunk_contexts(cfg, 1, "zbv", "bf16", own_streams=True)
    api.attach_nccl_chunks(ctxs, b"\0" * 128 * 2, 2, [0, 0], 0)
    torch.cuda.synchronize()
    api.run_worker(ctxs, passes, tok, lab)
    _assert_same(_state(ctxs), want, "hybrid")
