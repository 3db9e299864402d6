"""Pins for oracle/optim.py.

* Algorithm 1 hand example (evaluated by hand) and the
  zero-gradient case (theta (1 - lr wd)).
* ROLLBACK o STEP = identity to rounding ("arithmetically reversible").
* errors: t = 0, lr*wd = 1.
* post-validation vs the synchronous baseline over a
  fault corpus: clean / deferred paths bitwise equal, rollback paths within
  1e-12; partial state at stage k = sum over stages < k; no
  rollbacks on clean runs.
"""
import zlib

import numpy as np
import pytest

from oracle import optim as oo


def test_hand_example():
    th, m, v, t = oo.adamw_step(np.array(2.0), np.array(0.0), np.array(0.0), 0, np.array(1.0),
                                0.1, 0.9, 0.999, 1e-8, 0.0)
    assert t == 1
    assert abs(m - 0.1) < 1e-16 and abs(v - 0.001) < 1e-18
    # m' = 0.1 / (1 - 0.9) = 1, v' = 0.001 / (1 - 0.999) = 1  -> theta - 0.1 / (1 + 1e-8)
    assert abs(th - (2.0 - 0.1 / (1.0 + 1e-8))) < 1e-15


def test_zero_gradient():
    th0 = np.array([1.5, -2.0])
    th, m, v, t = oo.adamw_step(th0, np.zeros(2), np.zeros(2), 0, np.zeros(2), 1e-3, 0.9, 0.95, 1e-8, 0.1)
    assert np.array_equal(m, np.zeros(2)) and np.array_equal(v, np.zeros(2)) and t == 1
    assert np.allclose(th, th0 * (1 - 1e-3 * 0.1), rtol=0, atol=1e-16)


def test_rollback_roundtrip_random():
    rng = np.random.default_rng(0)
    worst = [0.0, 0.0, 0.0]
    for _ in range(1000):
        n = 64
        th = rng.standard_normal(n)
        m = rng.standard_normal(n) * 1e-2
        v = rng.random(n) * 1e-4 + 1e-8
        t = int(rng.integers(0, 50))
        g = rng.standard_normal(n) * 1e-2
        lr, wd = 1e-3, 0.1
        s = oo.adamw_step(th, m, v, t, g, lr, 0.9, 0.95, 1e-8, wd)
        r = oo.adamw_rollback(*s, g, lr, 0.9, 0.95, 1e-8, wd)
        assert r[3] == t
        worst[0] = max(worst[0], np.max(np.abs(r[0] - th) / np.abs(th)))
        # m and v are measured against the scale of the terms that cancel
        worst[1] = max(worst[1], np.max(np.abs(r[1] - m) / np.maximum(np.abs(m), 0.1 * np.abs(g))))
        worst[2] = max(worst[2], np.max(np.abs(r[2] - v) / np.maximum(v, 0.05 * g * g)))
    assert worst[0] <= 1e-12 and worst[1] <= 1e-12 and worst[2] <= 1e-12, worst


def test_rollback_errors():
    with pytest.raises(ValueError):
        oo.adamw_rollback(np.ones(1), np.ones(1), np.ones(1), 0, np.ones(1), 1e-3, 0.9, 0.95, 1e-8, 0.0)
    with pytest.raises(ValueError):
        oo.adamw_rollback(np.ones(1), np.ones(1), np.ones(1), 1, np.ones(1), 0.5, 0.9, 0.95, 1e-8, 2.0)


# ------------------------------------------------------------------ fault corpus

def _make_stage_params(p, rng):
    shapes = [("w", (6, 5)), ("b", (5,)), ("e", (3, 4))]
    return [{f"s{i}.{n}": rng.standard_normal(sh) for n, sh in shapes} for i in range(p)]


def _grads(params, rng, scale):
    return [{k: rng.standard_normal(v.shape) * scale for k, v in st.items()} for st in params]


FAULTS = []
# (name, p, iterations, {(iteration, stage): ("nan" | "inf" | "big", factor)}, base scale)
FAULTS.append(("clean", 4, 3, {}, 0.05))
FAULTS.append(("clean-p1", 1, 3, {}, 0.05))
FAULTS.append(("clean-p8", 8, 2, {}, 0.02))
for st in range(4):
    FAULTS.append((f"nan-it1-s{st}", 4, 3, {(1, st): ("nan", 0)}, 0.05))
    FAULTS.append((f"inf-it0-s{st}", 4, 2, {(0, st): ("inf", 0)}, 0.05))
    FAULTS.append((f"clip-it1-s{st}", 4, 3, {(1, st): ("big", 100.0)}, 0.05))
FAULTS.append(("clip-all", 4, 3, {}, 5.0))
FAULTS.append(("clip-then-nan", 4, 3, {(0, 3): ("big", 50.0), (1, 0): ("nan", 0)}, 0.05))
FAULTS.append(("nan-then-clip", 4, 3, {(0, 2): ("nan", 0), (1, 1): ("big", 50.0)}, 0.05))
FAULTS.append(("consecutive-clip", 3, 4, {(1, 2): ("big", 40.0), (2, 0): ("big", 40.0)}, 0.05))
FAULTS.append(("nan-and-clip-same-iter", 4, 2, {(0, 0): ("big", 80.0), (0, 3): ("nan", 0)}, 0.05))


@pytest.mark.parametrize("name,p,iters,faults,scale", FAULTS, ids=[f[0] for f in FAULTS])
def test_post_validation_equals_sync(name, p, iters, faults, scale):
    assert len(FAULTS) >= 20
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    params = _make_stage_params(p, rng)
    hyp = oo.AdamWHyper(lr=1e-3, clip=1.0)
    sync = [oo.StageOptimizer(pp, hyp) for pp in params]
    pv = [oo.StageOptimizer(pp, hyp) for pp in params]
    exact = True
    for it in range(iters):
        grads = _grads(params, rng, scale)
        for (fi, fs), (kind, fac) in faults.items():
            if fi == it:
                k = next(iter(grads[fs]))
                if kind == "nan":
                    grads[fs][k][0, 0] = np.nan
                elif kind == "inf":
                    grads[fs][k][0, 0] = np.inf
                else:
                    for kk in grads[fs]:
                        grads[fs][kk] = grads[fs][kk] * fac
        oo.sync_step(sync, grads)
        tr = oo.pv_step(pv, grads)
        # partial state received by stage k = sum over stages before k
        acc = 0.0
        for i in range(p):
            got = tr["partial_in"][i][0]
            assert got == acc or (np.isnan(got) and np.isnan(acc))
            acc += oo.local_state(grads[i])[0]
        if any(a in ("rollback", "rollback+redo") for a in tr["final"]):
            exact = False
        if not faults and scale < 1:
            assert all(a == "none" for a in tr["final"]) and all(a == "step" for a in tr["first"])
    for a, b in zip(sync, pv):
        assert a.t == b.t
        for k in a.theta:
            if exact:
                assert np.array_equal(a.theta[k], b.theta[k]) and np.array_equal(a.m[k], b.m[k]), k
            else:
                assert np.allclose(b.theta[k], a.theta[k], rtol=1e-12, atol=1e-15), k
                assert np.allclose(b.m[k], a.m[k], rtol=1e-12, atol=1e-15)
                assert np.allclose(b.v[k], a.v[k], rtol=1e-12, atol=1e-18)


# ------------------------------------------------------------------ independent pins of the global state
# local_state / clip_coef / sync_step ("gradient clipping ... global norm ... NaN/INF
# check") are pinned against torch's own implementations — torch.nn.utils.clip_grad_norm_
# (global 2-norm, coef = max_norm / (norm + 1e-6) clamped to 1) and torch.optim.AdamW
# (decoupled weight decay, bias-corrected moments) — an independent library, not a retyping.

def _torch_sync_reference(params, grads, hyp, wd_of):
    """torch CPU fp64: clip_grad_norm_ over ALL stages' grads, skip on a
    non-finite norm, else torch.optim.AdamW.step() with per-tensor weight decay."""
    import torch
    names = [k for st in params for k in st]
    flat_p = {k: v for st in params for k, v in st.items()}
    flat_g = {k: v for st in grads for k, v in st.items()}
    tp = {k: torch.nn.Parameter(torch.tensor(flat_p[k], dtype=torch.float64)) for k in names}
    for k in names:
        tp[k].grad = torch.tensor(flat_g[k], dtype=torch.float64)
    norm = torch.nn.utils.clip_grad_norm_([tp[k] for k in names], max_norm=hyp.clip, error_if_nonfinite=False,
                                          foreach=False)
    groups = {}
    for k in names:
        groups.setdefault(wd_of(k, flat_p[k].shape), []).append(tp[k])
    opt = torch.optim.AdamW([{"params": v, "weight_decay": w} for w, v in groups.items()], lr=hyp.lr,
                            betas=(hyp.beta1, hyp.beta2), eps=hyp.eps, foreach=False)
    stepped = bool(torch.isfinite(norm))
    if stepped:
        opt.step()
    out = {}
    for k in names:
        st = opt.state.get(tp[k], {})
        out[k] = (tp[k].detach().numpy(), st.get("exp_avg"), st.get("exp_avg_sq"))
    return float(norm), stepped, out


@pytest.mark.parametrize("case", ["clean", "clip", "nan", "inf"])
def test_sync_step_matches_torch_clip_and_adamw(case):
    rng = np.random.default_rng({"clean": 1, "clip": 2, "nan": 3, "inf": 4}[case])
    p = 3
    params = _make_stage_params(p, rng)
    grads = _grads(params, rng, 0.05 if case != "clip" else 3.0)
    if case == "nan":
        grads[1]["s1.b"][2] = np.nan
    if case == "inf":
        grads[2]["s2.e"][0, 1] = -np.inf
    hyp = oo.AdamWHyper(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, clip=1.0)
    opts = [oo.StageOptimizer(pp, hyp) for pp in params]
    action = oo.sync_step(opts, grads)
    norm, stepped, ref = _torch_sync_reference(params, grads, hyp, lambda k, sh: oo.default_weight_decay(k, sh, 0.1))
    # the oracle's global state against torch's total norm
    S = sum(oo.local_state(g)[0] for g in grads)
    nan = any(oo.local_state(g)[1] for g in grads)
    assert nan == (not np.isfinite(norm))
    if not nan:
        assert abs(np.sqrt(S) - norm) <= 1e-13 * norm
        assert (action == "clip") == (hyp.clip / (norm + 1e-6) < 1.0)
        assert action == ("clip" if case == "clip" else "step")
    else:
        assert action == "skip" and not stepped
    for o in opts:
        assert o.t == (1 if stepped else 0)
        for k in o.theta:
            th, m, v = ref[k]
            assert np.allclose(o.theta[k], th, rtol=1e-13, atol=1e-16), k
            if stepped:
                assert np.allclose(o.m[k], m.numpy(), rtol=1e-13, atol=1e-18), k
                assert np.allclose(o.v[k], v.numpy(), rtol=1e-13, atol=1e-20), k
            else:
                assert np.array_equal(o.theta[k], params[[i for i in range(p) if k in params[i]][0]][k])


def test_global_norm_hand_example():
    """Gradients (3, 4) on one stage and (12,) on another: global norm 13
    (P:149 'global gradient norm'); clip 1 -> coef 1 / (13 + 1e-6); clip 100 -> no clipping."""
    g = [{"a": np.array([3.0, 4.0])}, {"b": np.array([12.0])}]
    s = [oo.local_state(x) for x in g]
    assert s[0] == (25.0, False) and s[1] == (144.0, False)
    S = s[0][0] + s[1][0]
    assert S == 169.0
    assert oo.clip_coef(S, 1.0) == 1.0 / (13.0 + 1e-6)
    assert oo.clip_coef(S, 100.0) > 1.0
    assert oo.local_state({"a": np.array([1.0, np.nan])})[1] is True
    assert oo.local_state({"a": np.array([np.inf])})[1] is True
    # a sum of squares, not of absolute values or norms: (3,4) -> 25 (not 7, not 5)
    assert oo.local_state({"a": np.array([3.0, -4.0])})[0] == 25.0


def test_sync_step_clip_scales_gradient_by_coef():
    """With lr small and fresh AdamW state, the first step's m = (1-b1) * coef * g:
    the clipped gradient is recoverable and must equal clip_grad_norm_'s output."""
    import torch
    rng = np.random.default_rng(9)
    g = {"w": rng.standard_normal((4, 3)) * 10.0}
    hyp = oo.AdamWHyper(lr=1e-6, weight_decay=0.0, clip=1.0)
    o = oo.StageOptimizer({"w": np.zeros((4, 3))}, hyp)
    assert oo.sync_step([o], [g]) == "clip"
    tg = torch.nn.Parameter(torch.zeros(4, 3, dtype=torch.float64))
    tg.grad = torch.tensor(g["w"])
    torch.nn.utils.clip_grad_norm_([tg], 1.0, foreach=False)
    assert np.allclose(o.m["w"] / (1 - hyp.beta1), tg.grad.numpy(), rtol=1e-14, atol=0)
