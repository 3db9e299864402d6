"""W-grouping (W "can be scheduled anywhere after the
corresponding B"): adjacent W passes of a stage run as ONE contraction per linear with
K = k T (ZB_RUN_GROUP_W), so at b = 1 the f32 gradient read-modify-write is paid once
for k microbatches.

* the grouped contraction itself (zb_dbg_gemm_wgroup) against the plain definition;
* grouped iterations against the fp64 oracle (normwise + elementwise, C15);
* bitwise equality between runtimes with the same grouping (the single-stage runner,
  the virtual-stage runner and the loopback multi-stage runner), and identity with the
  ungrouped run when no two W passes are adjacent."""
import threading

import numpy as np
import pytest

import zb_synth
from zbtest_util import assert_close, cuda_available
from test_gpu_stage import check_tolerance, oracle_grads

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


@pytest.mark.parametrize("M,N,T,k", [(2304, 2304, 1024, 4), (5120, 1280, 1024, 2), (768, 512, 512, 3)])
def test_grouped_w_contraction(M, N, T, k):
    import torch
    from paper_2401_10241_b200 import api
    g = torch.Generator(device="cpu").manual_seed(M + k)
    As = [(torch.randn(T, M, generator=g) * 0.5).bfloat16().cuda() for _ in range(k)]
    Bs = [(torch.randn(T, N, generator=g) * 0.5).bfloat16().cuda() for _ in range(k)]
    C = torch.randn(M, N, generator=g).cuda()
    C0 = C.double().cpu().numpy()
    db = torch.zeros(M).cuda()
    api.dbg_gemm_wgroup(As, Bs, C, M=M, N=N, bias=db, beta=1)
    torch.cuda.synchronize()
    want = C0 + sum(a.double().cpu().numpy().T @ b.double().cpu().numpy() for a, b in zip(As, Bs))
    wb = sum(a.double().cpu().numpy().sum(0) for a in As)
    assert_close(C.double().cpu().numpy(), want, 1e-5, "dW", bf16=True)
    assert_close(db.double().cpu().numpy(), wb, 1e-5, "db", bf16=True)


def _ctx1(cfg, n_slots, dtype):
    from paper_2401_10241_b200 import api
    c = api.Context(cfg, 1, 0, cfg.m, n_slots, dtype=dtype)
    prm = zb_synth.make_stage_params(cfg, 1, 0)
    c.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, 1, 0)])
    return c


def _deferred_list(m):
    """p = 1 list with every W deferred to the end (F0 B0 F1 B1 ... W0 .. W_{m-1}): all Ws adjacent."""
    from paper_2401_10241_b200._lib import zb_pass_t
    arr = (zb_pass_t * (3 * m))()
    k = 0
    for j in range(m):
        for kind in (0, 1):
            arr[k].stage, arr[k].microbatch, arr[k].kind, arr[k].slot = 0, j, kind, j
            k += 1
    for j in range(m):
        arr[k].stage, arr[k].microbatch, arr[k].kind, arr[k].slot = 0, j, 2, j
        k += 1
    return arr


def _grads(c, cfg, p=1, s=0):
    return {n: g.reshape(sh) for (n, sh, _), g in zip(zb_synth.param_specs(cfg, p, s), c.get_grads())}


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_grouped_iteration_vs_oracle_and_runtimes(dtype):
    import torch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.ModelConfig("wg", h=256, a=2, L=2, s=256, b=2, V=512, p=1, m=6, family="zbh1")
    ref_loss, ref = oracle_grads(cfg, dtype)
    tok = zb_synth.make_tokens(cfg, 0)
    tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
    passes = _deferred_list(cfg.m)          # 6 adjacent Ws -> groups of 4 and 2
    c = _ctx1(cfg, cfg.m, dtype)
    c.run_iteration(passes, tin, lab, group_w=True)
    loss, g = c.loss(), _grads(c, cfg)
    check_tolerance(loss, g, ref_loss, ref, dtype)
    c2 = _ctx1(cfg, cfg.m, dtype)           # the virtual-stage runner, same grouping: bitwise
    api.run_local([c2], passes, tin, lab, group_w=True)
    g2 = _grads(c2, cfg)
    assert c2.loss() == loss and all(np.array_equal(g[k], g2[k]) for k in g)
    # ZB-H1 at p = 1 has no adjacent Ws: grouping changes nothing
    p1, sim = api.schedule("zbh1", 1, cfg.m, 1, 1, 1)
    c3, c4 = _ctx1(cfg, sim.n_slots[0], dtype), _ctx1(cfg, sim.n_slots[0], dtype)
    c3.run_iteration(p1, tin, lab)
    c4.run_iteration(p1, tin, lab, group_w=True)
    g3, g4 = _grads(c3, cfg), _grads(c4, cfg)
    assert all(np.array_equal(g3[k], g4[k]) for k in g3)


def test_grouped_loopback_runner_equals_virtual_stages():
    """ZB-H2 over p = 2 stages (its cool-down has adjacent Ws on every stage): the
    multi-stage runner (plan ops, loopback transport, one thread per stage) with
    grouping is bitwise equal to the virtual-stage runner with grouping."""
    import torch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.ModelConfig("wg2", h=128, a=2, L=4, s=256, b=2, V=512, p=2, m=5, family="zbh2")
    p = 2
    passes, sim = api.schedule("zbh2", p, cfg.m, 10, 11, 6)
    lists = api.stage_lists(passes, p)
    assert any(a[0] == "W" and b[0] == "W" for o in lists for a, b in zip(o, o[1:]))
    tok = zb_synth.make_tokens(cfg, 0)
    tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()

    def make(own_streams):
        out = []
        for s in range(p):
            st = torch.cuda.Stream() if own_streams else None
            c = api.Context(cfg, p, s, cfg.m, max(1, sim.n_slots[s]), dtype="bf16", stream=st)
            prm = zb_synth.make_stage_params(cfg, p, s)
            c.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
            out.append(c)
        return out

    ref = make(False)
    api.run_local(ref, passes, tin, lab, group_w=True)
    lb = make(True)
    grp = api.Loopback(p)
    for c in lb:
        c.attach_loopback(grp)
    errs = []

    def body(r):
        try:
            lb[r].run_iteration(api.stage_passes(passes, r), tin if r == 0 else None, lab if r == p - 1 else None,
                                group_w=True)
            lb[r].sync()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    assert lb[-1].loss() == ref[-1].loss()
    for s in range(p):
        a, b = _grads(ref[s], cfg, p, s), _grads(lb[s], cfg, p, s)
        assert all(np.array_equal(a[k], b[k]) for k in a), s
