"""Parity at the bench workload's full widths (BASELINE configs[1], 1.5B: h 2304,
24 heads of d = 96, seq 1024, vocab 50304; and configs[2], 6.2B: h 4096, 32 heads of
d = 128) on one sequence and one layer, in the
launch configuration bench.py times (tcgen05 GEMMs with split-K W, tcgen05 attention,
two-phase column reductions): loss and every gradient against the fp64 oracle within
the bf16 tolerances, and bitwise repeatability of the whole iteration."""
import numpy as np
import pytest

import zb_synth
from zbtest_util import cuda_available
from test_gpu_stage import check_tolerance, gpu_run, oracle_grads

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


@pytest.mark.parametrize("name", ["1.5B", "6.2B"])
def test_full_width_layer_vs_oracle_and_repeatable(name):
    cfg = zb_synth.CONFIGS[name].with_(L=1, b=1, m=1)
    ref_loss, ref = oracle_grads(cfg, "bf16")
    loss, grads, _ = gpu_run(cfg, 1, "bf16")
    errs = check_tolerance(loss, grads, ref_loss, ref, "bf16")
    assert max(errs.values()) < 2e-2
    loss2, grads2, _ = gpu_run(cfg, 1, "bf16")
    assert loss2 == loss
    assert all(np.array_equal(grads[k], grads2[k]) for k in grads)


@pytest.mark.parametrize("name", ["1.5B", "6.2B"])
def test_full_width_multi_microbatch_two_stages_vs_oracle(name):
    """The bench widths with b = 2 sequences per microbatch (b-batched attention),
    m = 2 microbatches (the second W accumulates into the f32 grads with beta = 1
    through the ordered split-K reduce-add) and p = 2 virtual stages (the f32
    stage-boundary gradient, R-grad32), ZB-H1: loss and every gradient against
    the fp64 oracle (normwise and elementwise)."""
    cfg = zb_synth.CONFIGS[name].with_(L=2, b=2, m=2)
    ref_loss, ref = oracle_grads(cfg, "bf16")
    loss, grads, _ = gpu_run(cfg, 2, "bf16")
    check_tolerance(loss, grads, ref_loss, ref, "bf16")


@pytest.mark.parametrize("name", ["14.6B", "28.3B"])
def test_c4_c5_widths_grouped_w_vs_oracle(name):
    """BASELINE configs[3] / [4] widths (14.6B: h 5120, 40 heads; 28.3B: h 6144, 48 heads;
    d = 128, b = 1 so T = 1024 — the W GEMM at the HBM ridge): one layer, two
    microbatches whose Ws are deferred and run as ONE grouped contraction per linear
    (W-grouping, K = 2T), against the fp64 oracle (normwise + elementwise)."""
    import torch
    from test_gpu_wgroup import _ctx1, _deferred_list, _grads
    cfg = zb_synth.CONFIGS[name].with_(L=1, b=1, m=2)
    ref_loss, ref = oracle_grads(cfg, "bf16")
    tok = zb_synth.make_tokens(cfg, 0)
    tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
    c = _ctx1(cfg, cfg.m, "bf16")
    c.run_iteration(_deferred_list(cfg.m), tin, lab, group_w=True)
    check_tolerance(c.loss(), _grads(c, cfg), ref_loss, ref, "bf16")


def test_bench_config_6p2b_graph_and_schedules_bitwise():
    """The bench's headline workload itself (BASELINE configs[2]: 6.2B, 30 layers, b 3, m 32,
    p = 1) — too large for the oracle, so checked by properties that hold at any size:
    the CUDA-graph replay (ZB_RUN_GRAPH: eager, capture, replay) reproduces the eager
    iteration bitwise; ZB-H1 and 1F1B pass orders give bitwise the same loss and gradients
    as ZB-H2 (P:196 — the W sums run in microbatch order whatever the placement, R-splitk);
    the loss at initialisation matches its closed form and every sampled gradient is
    finite.  Closed form: LN_f's output rows have mean 0 and mean square gamma^2 + beta^2
    (gamma = 1 + 0.02 z, beta = 0.02 z: 1 + 8e-4 in expectation), the head rows are
    N(0, 0.02^2) (zb_synth), so each logit is ~N(0, sigma^2) with sigma^2 = h 0.02^2 (1 + 8e-4)
    and the cross-entropy of V Gaussian logits is ln V + sigma^2 / 2 (E[ln sum_v e^z_v] for
    large V; the label logit has mean 0).  Gradients sampled: embedding, first and last layer,
    LN_f, head."""
    import math
    import torch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.CONFIGS["6.2B"]
    p, m = 1, cfg.m
    mc = api.model_cfg(cfg, p, 0, m, 1, "bf16")
    slot_b = api.slot_bytes(mc)
    fam = {f: api.schedule(f, p, m, 1, 1, 1, 0, M_B=slot_b, M_W=slot_b) for f in ("zbh2", "zbh1", "1f1b")}
    n_slots = max(max(1, sim.n_slots[0]) for _, sim in fam.values())
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, 0, m, n_slots, dtype="bf16", stream=stream)
    names = [n for n, _, _ in zb_synth.param_specs(cfg, p, 0)]
    params = zb_synth.make_stage_params(cfg, p, 0)
    ctx.set_params([params[n] for n in names])
    del params
    only = {i for i, n in enumerate(names) if not n.startswith("l") or n.startswith(("l0.", f"l{cfg.L - 1}.", "lnf"))}
    tok = zb_synth.make_tokens(cfg, 0)
    with torch.cuda.stream(stream):
        tok_d = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
        lab_d = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()

    def run(family, graph):
        ctx.run_iteration(fam[family][0], tok_d, lab_d, graph=graph)
        return ctx.loss(), ctx.get_grads(only)

    try:
        loss0, g0 = run("zbh2", False)
        sigma2 = cfg.h * 0.02 ** 2 * (1 + 8e-4)
        expect = math.log(cfg.V) + sigma2 / 2  # 11.6454 at h 4096, V 50304
        assert math.isfinite(loss0) and abs(loss0 - expect) < 0.02, (loss0, expect)
        for i in only:
            assert np.isfinite(g0[i]).all(), names[i]
        for family, graph in (("zbh2", True), ("zbh2", True), ("zbh2", True), ("zbh1", False), ("1f1b", False)):
            loss, g = run(family, graph)
            assert loss == loss0, (family, graph, loss, loss0)
            for i in only:
                assert np.array_equal(g[i], g0[i]), (family, graph, names[i])
    finally:
        ctx.close()
