"""Oracle optimizer: AdamW step / in-place rollback and post-validation
(test infrastructure only; see oracle/__init__).

Algorithm 1 (App. C) written out literally:
    STEP(g):     t = t+1; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
                 m' = m/(1-b1^t); v' = v/(1-b2^t);
                 theta = theta - lr*wd*theta - lr*m'/(sqrt(v')+eps)
    ROLLBACK(g): m' = m/(1-b1^t); v' = v/(1-b2^t);
                 theta = (theta + lr*m'/(sqrt(v')+eps)) / (1 - lr*wd);
                 m = (m - (1-b1) g)/b1; v = (v - (1-b2) g^2)/b2; t = t-1

Post-validation (section 4) in the SURVEY C12 readings:
  * local state of stage i: s_i = sum of squared grads, nan_i = any non-finite;
  * partial state P_i = (s_1+...+s_i, nan_1 or ... or nan_i) flows 1 -> p;
  * stage i: P_i.nan -> skip; clip/(sqrt(P_i.s)+1e-6) < 1 -> defer;
    else optimistic unclipped step (g retained for rollback);
  * the full state F = P_p flows back p -> 1; each stage validates:
    F.nan -> roll back if it stepped; F needs clipping -> roll back if it
    stepped, then step with g*coef(F) (a deferred stage just steps);
    clean -> nothing.
Synchronous baseline: all-reduce (here: stage-order sum) first,
then skip on NaN or step with clipped g.  "skip" never advances t.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

Array = np.ndarray


@dataclass
class AdamWHyper:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    clip: float = 1.0


def adamw_step(theta: Array, m: Array, v: Array, t: int, g: Array, lr, b1, b2, eps, wd):
    """Algorithm 1 STEP.  Returns (theta, m, v, t)."""
    t = t + 1
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    theta = theta - lr * wd * theta - lr * mh / (np.sqrt(vh) + eps)
    return theta, m, v, t


def adamw_rollback(theta: Array, m: Array, v: Array, t: int, g: Array, lr, b1, b2, eps, wd):
    """Algorithm 1 ROLLBACK.  Errors on t == 0 and lr*wd == 1
    (division by zero)."""
    if t <= 0:
        raise ValueError("rollback at t = 0")
    if lr * wd == 1:
        raise ValueError("rollback undefined for lr * weight_decay == 1")
    if b1 == 0 or b2 == 0:
        raise ValueError("rollback undefined for beta == 0")
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    theta = (theta + lr * mh / (np.sqrt(vh) + eps)) / (1 - lr * wd)
    m = (m - (1 - b1) * g) / b1
    v = (v - (1 - b2) * g * g) / b2
    return theta, m, v, t - 1


def default_weight_decay(name: str, shape: Tuple[int, ...], wd: float) -> float:
    """Reading (DESIGN.md R-opt): decay matrices and embeddings (ndim >= 2),
    not biases or LayerNorm parameters (Megatron-like; the paper is silent)."""
    return wd if len(shape) >= 2 else 0.0


class StageOptimizer:
    """AdamW state of one pipeline stage (D8 of SURVEY §2.4)."""

    def __init__(self, params: Dict[str, Array], hyper: AdamWHyper):
        self.h = hyper
        self.theta = {k: np.array(v, dtype=np.float64) for k, v in params.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.theta.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.theta.items()}
        self.wd = {k: default_weight_decay(k, v.shape, hyper.weight_decay) for k, v in self.theta.items()}
        self.t = 0

    def step(self, grads: Dict[str, Array], coef: float = 1.0) -> None:
        h = self.h
        t_new = self.t
        for k in self.theta:
            g = grads[k] * coef if coef != 1.0 else grads[k]
            self.theta[k], self.m[k], self.v[k], t_new = adamw_step(
                self.theta[k], self.m[k], self.v[k], self.t, g, h.lr, h.beta1, h.beta2, h.eps, self.wd[k])
        self.t = t_new

    def rollback(self, grads: Dict[str, Array], coef: float = 1.0) -> None:
        h = self.h
        t_new = self.t
        for k in self.theta:
            g = grads[k] * coef if coef != 1.0 else grads[k]
            self.theta[k], self.m[k], self.v[k], t_new = adamw_rollback(
                self.theta[k], self.m[k], self.v[k], self.t, g, h.lr, h.beta1, h.beta2, h.eps, self.wd[k])
        self.t = t_new


def local_state(grads: Dict[str, Array], order: Optional[Sequence[str]] = None) -> Tuple[float, bool]:
    """(sum of squared gradients, any non-finite) of one stage, summed in the
    canonical parameter order."""
    keys = list(order) if order is not None else list(grads)
    s = 0.0
    nan = False
    for k in keys:
        g = grads[k]
        if not np.all(np.isfinite(g)):
            nan = True
        s += float(np.sum(g * g))
    return s, nan


def clip_coef(sumsq: float, clip: float) -> float:
    """clip / (sqrt(S) + 1e-6) (global-norm clipping)."""
    return clip / (np.sqrt(sumsq) + 1e-6)


def sync_step(opts: List[StageOptimizer], grads: List[Dict[str, Array]]) -> str:
    """Synchronous baseline: global state first, then the step."""
    S, N = 0.0, False
    for g in grads:
        s, n = local_state(g)
        S += s
        N = N or n
    if N:
        return "skip"
    coef = clip_coef(S, opts[0].h.clip)
    c = coef if coef < 1.0 else 1.0
    for o, g in zip(opts, grads):
        o.step(g, c)
    return "clip" if coef < 1.0 else "step"


def pv_step(opts: List[StageOptimizer], grads: List[Dict[str, Array]]) -> Dict:
    """Post-validation protocol for one iteration.  Returns a
    transcript: partial states received per stage, the optimistic action
    and the validation action of every stage."""
    p = len(opts)
    clip = opts[0].h.clip
    partial_in: List[Tuple[float, bool]] = []
    acc = (0.0, False)
    first_action: List[str] = []
    for i in range(p):                          # 1 -> p before each step
        partial_in.append(acc)
        s, n = local_state(grads[i])
        acc = (acc[0] + s, acc[1] or n)
        if acc[1]:
            first_action.append("skip")
        elif clip_coef(acc[0], clip) < 1.0:
            first_action.append("defer")
        else:
            opts[i].step(grads[i])
            first_action.append("step")
    full = acc
    final_action: List[str] = []
    for i in reversed(range(p)):                # p -> 1 during the next warm-up
        a = first_action[i]
        if full[1]:
            if a == "step":
                opts[i].rollback(grads[i])
                final_action.append("rollback")
            else:
                final_action.append("none")
            continue
        coef = clip_coef(full[0], clip)
        if coef < 1.0:
            if a == "step":
                opts[i].rollback(grads[i])
                opts[i].step(grads[i], coef)
                final_action.append("rollback+redo")
            elif a == "defer":
                opts[i].step(grads[i], coef)
                final_action.append("deferred-step")
            else:
                final_action.append("none")
        else:
            final_action.append("none")
    final_action.reverse()
    return dict(partial_in=partial_in, full=full, first=first_action, final=final_action)
