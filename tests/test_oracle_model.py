"""Pins for oracle/model.py against things other than itself.

* CPU torch float64 autograd (an independent library: F.layer_norm,
  F.gelu(approximate='tanh'), F.scaled_dot_product_attention(is_causal),
  F.cross_entropy) on the same weights: loss and every gradient.
* central finite differences on a tiny model.
* special cases with closed forms (LayerNorm moments, GeLU values, attention
  at s=1 and with uniform scores).
* B + W == unsplit backward bitwise (P:46 regrouping).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import zb_synth
from oracle import model as om

SMALL = zb_synth.ModelConfig("small", h=32, a=2, L=2, s=16, b=2, V=64, p=2, m=2, family="zbh1")


def torch_reference(cfg, params, tokens):
    """Independent fp64 autograd implementation of the same GPT block stack."""
    P = {k: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=True) for k, v in params.items()}
    m = tokens.shape[0]
    total = 0.0
    h, a, s, b = cfg.h, cfg.a, cfg.s, cfg.b
    d = h // a
    for j in range(m):
        tok = torch.tensor(tokens[j, :, :s].astype(np.int64))
        lab = torch.tensor(tokens[j, :, 1:].astype(np.int64))
        x = P["wte"][tok] + P["wpe"][:s][None]
        for l in range(cfg.L):
            q = lambda n: P[f"l{l}.{n}"]
            ln1 = F.layer_norm(x, (h,), q("ln1_g"), q("ln1_b"), eps=1e-5)
            qkv = ln1 @ q("qkv_w").T + q("qkv_b")
            Q, K, Vv = qkv.split(h, dim=-1)
            sh = lambda t: t.view(b, s, a, d).transpose(1, 2)
            o = F.scaled_dot_product_attention(sh(Q), sh(K), sh(Vv), is_causal=True)
            o = o.transpose(1, 2).reshape(b, s, h)
            x = x + o @ q("proj_w").T + q("proj_b")
            ln2 = F.layer_norm(x, (h,), q("ln2_g"), q("ln2_b"), eps=1e-5)
            u = ln2 @ q("fc1_w").T + q("fc1_b")
            x = x + F.gelu(u, approximate="tanh") @ q("fc2_w").T + q("fc2_b")
        lnf = F.layer_norm(x, (h,), P["lnf_g"], P["lnf_b"], eps=1e-5)
        logits = lnf @ P["head_w"].T
        total = total + F.cross_entropy(logits.reshape(-1, cfg.V), lab.reshape(-1)) / m
    total.backward()
    return float(total.detach()), {k: v.grad.numpy() for k, v in P.items()}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_against_torch_fp64_autograd():
    params = zb_synth.make_model_params(SMALL)
    tokens = zb_synth.make_tokens(SMALL, 0)
    loss, grads = om.reference_iteration(SMALL, params, tokens)
    tl, tg = torch_reference(SMALL, params, tokens)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    for k in params:
        assert rel(grads[k], tg[k]) <= 1e-10, k


def test_finite_differences():
    cfg = SMALL.with_(L=1, s=8, b=1, V=32, h=16, a=2, m=1)
    params = {k: v.astype(np.float64) for k, v in zb_synth.make_model_params(cfg).items()}
    tokens = zb_synth.make_tokens(cfg, 3)
    _, grads = om.reference_iteration(cfg, params, tokens)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for name in ["wte", "wpe", "l0.qkv_w", "l0.proj_b", "l0.ln1_g", "l0.fc1_w", "l0.fc2_w", "lnf_b", "head_w"]:
        idx = tuple(int(rng.integers(0, n)) for n in params[name].shape)
        if name == "wte":
            idx = (int(tokens[0, 0, 2]), idx[1])
        pp = {k: v.copy() for k, v in params.items()}
        pp[name][idx] += eps
        lp, _ = om.reference_iteration(cfg, pp, tokens)
        pp[name][idx] -= 2 * eps
        lm, _ = om.reference_iteration(cfg, pp, tokens)
        fd = (lp - lm) / (2 * eps)
        assert abs(fd - grads[name][idx]) <= 1e-6 * max(1e-3, abs(fd)), (name, fd, grads[name][idx])


def test_split_equals_unsplit_bitwise():
    """B then W reproduce the unsplit backward exactly (same fp64 ops)."""
    cfg = SMALL
    params = zb_synth.make_model_params(cfg)
    tokens = zb_synth.make_tokens(cfg, 1)
    a = om.Stage(cfg, 1, 0, params, cfg.m)
    b = om.Stage(cfg, 1, 0, params, cfg.m)
    for j in range(cfg.m):
        a.forward(j, tokens[j, :, :cfg.s], tokens[j, :, 1:])
        a.backward_unsplit(j)
        b.forward(j, tokens[j, :, :cfg.s], tokens[j, :, 1:])
        b.backward_input(j)
        b.backward_weight(j)
    for k in a.grads:
        assert np.array_equal(a.grads[k], b.grads[k]), k


def test_loss_at_init_close_to_log_vocab():
    cfg = SMALL.with_(V=512)
    params = zb_synth.make_model_params(cfg)
    loss, _ = om.reference_iteration(cfg, params, zb_synth.make_tokens(cfg, 0))
    assert abs(loss - math.log(cfg.V)) < 0.1


def test_layernorm_moments_and_grad_orthogonality():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((7, 33)) * 3 + 1
    y, (xh, rs) = om.layernorm_fwd(x, np.ones(33), np.zeros(33), eps=0.0)
    assert np.allclose(y.mean(-1), 0, atol=1e-13) and np.allclose(y.var(-1), 1, atol=1e-12)
    dy = rng.standard_normal((7, 33))
    dx = om.layernorm_bwd_input(dy, xh, rs, np.ones(33))
    # LN is invariant to x -> x + c and x -> k x: dx sums to 0 and is orthogonal to xhat
    assert np.allclose(dx.sum(-1), 0, atol=1e-12)
    assert np.allclose((dx * xh).sum(-1), 0, atol=1e-12)


def test_gelu_special_values():
    assert om.gelu(np.array(0.0)) == 0.0
    assert abs(om.gelu_grad(np.array(0.0)) - 0.5) < 1e-15
    assert abs(om.gelu(np.array(10.0)) - 10.0) < 1e-12
    assert abs(om.gelu(np.array(-10.0))) < 1e-12
    x = np.linspace(-4, 4, 101)
    fd = (om.gelu(x + 1e-6) - om.gelu(x - 1e-6)) / 2e-6
    assert np.allclose(fd, om.gelu_grad(x), atol=1e-8)


def test_attention_special_cases():
    rng = np.random.default_rng(2)
    b, s, a, d = 2, 5, 3, 4
    h = a * d
    qkv = rng.standard_normal((b * s, 3 * h))
    # s = 1: softmax over one key -> O = V
    one = rng.standard_normal((b, 3 * h))
    O, _ = om.causal_attention_fwd(one, b, 1, a)
    assert np.allclose(O, one[:, 2 * h:])
    # zero queries -> uniform weights over the causal prefix -> running mean of V
    z = qkv.copy()
    z[:, :h] = 0
    O, _ = om.causal_attention_fwd(z, b, s, a)
    V = z[:, 2 * h:].reshape(b, s, h)
    run = np.cumsum(V, axis=1) / np.arange(1, s + 1)[None, :, None]
    assert np.allclose(O.reshape(b, s, h), run)


def test_schedules_produce_bitwise_identical_grads():
    """fixed seed, identical losses across schedules -> here: identical
    gradients from 1F1B, ZB-H1, ZB-H2 and AUTO pass lists (W FIFO order)."""
    from oracle import schedule as osch
    cfg = SMALL.with_(L=4, m=5)
    p = 4
    params = zb_synth.make_model_params(cfg)
    tokens = zb_synth.make_tokens(cfg, 2)
    ref_loss, ref = om.reference_iteration(cfg, params, tokens)
    fam = {
        "1f1b": (osch.build_1f1b(p, cfg.m), True),
        "zbh1": (osch.build_zbh1(p, cfg.m), False),
        "zbh2": (osch.build_zbh2(p, cfg.m), False),
        "auto": (osch.auto_schedule(p, cfg.m, 10, 11, 6, 1, 3, 2, 2 * p * 3)[0], False),
    }
    for name, (lists, fused) in fam.items():
        loss, g, _ = om.run_pass_lists(cfg, p, params, tokens, [[(k, j) for k, j in o] for o in lists],
                                       fused_backward=fused)
        assert abs(loss - ref_loss) <= 1e-14 * ref_loss, name
        for k in ref:
            assert np.array_equal(g[k], ref[k]), (name, k)
