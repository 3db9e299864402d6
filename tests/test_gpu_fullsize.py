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
