"""Oracle stage math in float64 (test infrastructure only; see oracle/__init__).

The layer is the GPT-3-like pre-LN transformer block PAPER.md describes at
P:89 ("a typical setting similar to GPT-3 ... feedforward 4h ... head h/a"),
with the readings of SURVEY.md C1 (listed in DESIGN.md): pre-LN, biases on,
tanh-GeLU, dropout 0, LN eps 1e-5, learned absolute position embeddings,
untied input / output embeddings.

    x1 = x  + Attn(LN1(x)) W_proj^T + b_proj
    x2 = x1 + GeLU(LN2(x1) W_fc1^T + b_fc1) W_fc2^T + b_fc2

The backward is split as P:46 defines it: for a layer y = f(x, W),
    B = grad_x f(x, W)^T dl/dy        (input gradient; attention is all B)
    W = grad_W f(x, W)^T dl/dy        (every parameter gradient)
and the unsplit backward computes both together, layer by layer (the
"traditional" single backward function).  Loss:
    loss = (1/m) sum_j mean_{t in microbatch j} (lse(logits_t) - logits_t[label_t]).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import numpy as np

Array = np.ndarray
EPS = 1e-5
GELU_C = np.sqrt(2.0 / np.pi)


# --------------------------------------------------------------------------
# primitive layers (definitions written out)
# --------------------------------------------------------------------------

def layernorm_fwd(x: Array, g: Array, b: Array, eps: float = EPS):
    """y = g * (x - mean) / sqrt(var + eps) + b, over the last axis."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * rstd
    return xhat * g + b, (xhat, rstd)


def layernorm_bwd_input(dy: Array, xhat: Array, rstd: Array, g: Array) -> Array:
    """dx of LayerNorm (B part): rstd * (gh - mean(gh) - xhat * mean(gh * xhat)), gh = dy*g."""
    gh = dy * g
    return rstd * (gh - gh.mean(axis=-1, keepdims=True) - xhat * (gh * xhat).mean(axis=-1, keepdims=True))


def layernorm_bwd_weight(dy: Array, xhat: Array) -> Tuple[Array, Array]:
    """(dg, db) of LayerNorm (W part): column sums of dy*xhat and dy."""
    return (dy * xhat).sum(axis=0), dy.sum(axis=0)


def gelu(x: Array) -> Array:
    """tanh-GeLU: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + 0.044715 * x ** 3)))


def gelu_grad(x: Array) -> Array:
    """d/dx of the tanh-GeLU above."""
    t = np.tanh(GELU_C * (x + 0.044715 * x ** 3))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * 0.044715 * x * x)


def linear_fwd(x: Array, w: Array, bias: Optional[Array]) -> Array:
    """y = x W^T + b with W stored [n_out, n_in]."""
    y = x @ w.T
    return y if bias is None else y + bias


def linear_bwd_input(dy: Array, w: Array) -> Array:
    """B of a linear layer: dX = dY W."""
    return dy @ w


def linear_bwd_weight(dy: Array, x: Array) -> Tuple[Array, Array]:
    """W of a linear layer: dW = dY^T X, db = sum_t dY."""
    return dy.T @ x, dy.sum(axis=0)


def causal_attention_fwd(qkv: Array, b: int, s: int, a: int):
    """Causal multi-head attention.  qkv [b*s, 3h]; Q/K/V are column blocks
    [0,h), [h,2h), [2h,3h); head k uses columns k*d..(k+1)*d of each block.
    O = softmax(Q K^T / sqrt(d) + causal mask) V, heads concatenated."""
    h = qkv.shape[1] // 3
    d = h // a
    q = qkv[:, :h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    k = qkv[:, h:2 * h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    v = qkv[:, 2 * h:].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    scale = 1.0 / np.sqrt(d)
    S = (q @ k.transpose(0, 1, 3, 2)) * scale            # [b, a, s, s]
    mask = np.triu(np.ones((s, s), dtype=bool), 1)
    S = np.where(mask, -np.inf, S)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=-1, keepdims=True)
    o = P @ v                                            # [b, a, s, d]
    O = o.transpose(0, 2, 1, 3).reshape(b * s, h)
    return O, P


def causal_attention_bwd(dO: Array, qkv: Array, P: Array, b: int, s: int, a: int) -> Array:
    """dQKV from dO: dV = P^T dO, dP = dO V^T, dS = P * (dP - rowsum(dP*P)),
    dQ = dS K / sqrt(d), dK = dS^T Q / sqrt(d)."""
    h = qkv.shape[1] // 3
    d = h // a
    q = qkv[:, :h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    k = qkv[:, h:2 * h].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    v = qkv[:, 2 * h:].reshape(b, s, a, d).transpose(0, 2, 1, 3)
    do = dO.reshape(b, s, a, d).transpose(0, 2, 1, 3)
    scale = 1.0 / np.sqrt(d)
    dv = P.transpose(0, 1, 3, 2) @ do
    dP = do @ v.transpose(0, 1, 3, 2)
    dS = P * (dP - (dP * P).sum(axis=-1, keepdims=True))
    dq = (dS @ k) * scale
    dk = (dS.transpose(0, 1, 3, 2) @ q) * scale
    back = lambda t: t.transpose(0, 2, 1, 3).reshape(b * s, h)
    return np.concatenate([back(dq), back(dk), back(dv)], axis=1)


# --------------------------------------------------------------------------
# transformer layer: F, B, W, unsplit
# --------------------------------------------------------------------------

def layer_forward(x: Array, p: Dict[str, Array], b: int, s: int, a: int):
    """F of one layer ("forward pass").  Returns x2 and the cache B needs."""
    ln1, (xh1, rs1) = layernorm_fwd(x, p["ln1_g"], p["ln1_b"])
    qkv = linear_fwd(ln1, p["qkv_w"], p["qkv_b"])
    O, P = causal_attention_fwd(qkv, b, s, a)
    x1 = x + linear_fwd(O, p["proj_w"], p["proj_b"])
    ln2, (xh2, rs2) = layernorm_fwd(x1, p["ln2_g"], p["ln2_b"])
    u = linear_fwd(ln2, p["fc1_w"], p["fc1_b"])
    g = gelu(u)
    x2 = x1 + linear_fwd(g, p["fc2_w"], p["fc2_b"])
    cache = dict(xh1=xh1, rs1=rs1, ln1=ln1, qkv=qkv, P=P, O=O, xh2=xh2, rs2=rs2, ln2=ln2, u=u, g=g)
    return x2, cache


def layer_backward_input(dx2: Array, c: Dict[str, Array], p: Dict[str, Array], b: int, s: int, a: int):
    """B of one layer: every input gradient, in reverse order; returns dx and
    the (input, output-gradient) pairs W needs ("keeps some extra
    gradients for W")."""
    dg = linear_bwd_input(dx2, p["fc2_w"])
    du = dg * gelu_grad(c["u"])
    dln2 = linear_bwd_input(du, p["fc1_w"])
    dx1 = dx2 + layernorm_bwd_input(dln2, c["xh2"], c["rs2"], p["ln2_g"])
    dO = linear_bwd_input(dx1, p["proj_w"])
    dqkv = causal_attention_bwd(dO, c["qkv"], c["P"], b, s, a)
    dln1 = linear_bwd_input(dqkv, p["qkv_w"])
    dx = dx1 + layernorm_bwd_input(dln1, c["xh1"], c["rs1"], p["ln1_g"])
    wstash = dict(fc2=(dx2, c["g"]), fc1=(du, c["ln2"]), proj=(dx1, c["O"]), qkv=(dqkv, c["ln1"]),
                  ln2=(dln2, c["xh2"]), ln1=(dln1, c["xh1"]))
    return dx, wstash


def layer_backward_weight(ws: Dict[str, Tuple[Array, Array]]) -> Dict[str, Array]:
    """W of one layer: every parameter gradient from the stashed pairs."""
    g: Dict[str, Array] = {}
    for lin in ("qkv", "proj", "fc1", "fc2"):
        dy, x = ws[lin]
        g[lin + "_w"], g[lin + "_b"] = linear_bwd_weight(dy, x)
    for ln in ("ln1", "ln2"):
        dy, xh = ws[ln]
        g[ln + "_g"], g[ln + "_b"] = layernorm_bwd_weight(dy, xh)
    return g


def layer_backward_unsplit(dx2: Array, c: Dict[str, Array], p: Dict[str, Array], b: int, s: int, a: int):
    """The traditional fused backward: dX and dW together, op by op."""
    g: Dict[str, Array] = {}
    g["fc2_w"], g["fc2_b"] = linear_bwd_weight(dx2, c["g"])
    dg = linear_bwd_input(dx2, p["fc2_w"])
    du = dg * gelu_grad(c["u"])
    g["fc1_w"], g["fc1_b"] = linear_bwd_weight(du, c["ln2"])
    dln2 = linear_bwd_input(du, p["fc1_w"])
    g["ln2_g"], g["ln2_b"] = layernorm_bwd_weight(dln2, c["xh2"])
    dx1 = dx2 + layernorm_bwd_input(dln2, c["xh2"], c["rs2"], p["ln2_g"])
    g["proj_w"], g["proj_b"] = linear_bwd_weight(dx1, c["O"])
    dO = linear_bwd_input(dx1, p["proj_w"])
    dqkv = causal_attention_bwd(dO, c["qkv"], c["P"], b, s, a)
    g["qkv_w"], g["qkv_b"] = linear_bwd_weight(dqkv, c["ln1"])
    dln1 = linear_bwd_input(dqkv, p["qkv_w"])
    g["ln1_g"], g["ln1_b"] = layernorm_bwd_weight(dln1, c["xh1"])
    dx = dx1 + layernorm_bwd_input(dln1, c["xh1"], c["rs1"], p["ln1_g"])
    return dx, g


# --------------------------------------------------------------------------
# embedding and head
# --------------------------------------------------------------------------

def embed_forward(tok: Array, wte: Array, wpe: Array) -> Array:
    """x0[b, t] = W_te[tok[b, t]] + W_pe[t]; tok [b, s] -> x0 [b*s, h]."""
    b, s = tok.shape
    return (wte[tok] + wpe[None, :s]).reshape(b * s, -1)


def embed_backward_weight(tok: Array, dx0: Array, V: int, s_max: int) -> Tuple[Array, Array]:
    """dW_te[v] = sum over positions with tok == v of dx0; dW_pe[t] = sum_b dx0[b, t]."""
    b, s = tok.shape
    h = dx0.shape[1]
    dwte = np.zeros((V, h))
    np.add.at(dwte, tok.reshape(-1), dx0)
    dwpe = np.zeros((s_max, h))
    dwpe[:s] = dx0.reshape(b, s, h).sum(axis=0)
    return dwte, dwpe


def head_forward(x: Array, lnf_g: Array, lnf_b: Array, head_w: Array, labels: Array, m: int):
    """Last stage: LN_f -> logits = ln W_out^T -> per-microbatch CE contribution
    (1/m) mean_t (lse - logit[label])."""
    lnf, (xh, rs) = layernorm_fwd(x, lnf_g, lnf_b)
    logits = lnf @ head_w.T
    mx = logits.max(axis=1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(axis=1))
    lab = labels.reshape(-1)
    T = logits.shape[0]
    loss = (lse - logits[np.arange(T), lab]).mean() / m
    cache = dict(lnf=lnf, xh=xh, rs=rs, logits=logits, lse=lse, lab=lab, m=m)
    return loss, cache


def head_backward_input(c: Dict[str, Array], lnf_g: Array, head_w: Array):
    """dlogits = (softmax - onehot) / (T m); dx through W_out and LN_f."""
    T = c["logits"].shape[0]
    dlog = np.exp(c["logits"] - c["lse"][:, None])
    dlog[np.arange(T), c["lab"]] -= 1.0
    dlog /= (T * c["m"])
    dlnf = dlog @ head_w
    dx = layernorm_bwd_input(dlnf, c["xh"], c["rs"], lnf_g)
    return dx, dict(head=(dlog, c["lnf"]), lnf=(dlnf, c["xh"]))


def head_backward_weight(ws) -> Dict[str, Array]:
    dlog, lnf = ws["head"]
    dlnf, xh = ws["lnf"]
    g_lnf, b_lnf = layernorm_bwd_weight(dlnf, xh)
    return {"head_w": dlog.T @ lnf, "lnf_g": g_lnf, "lnf_b": b_lnf}


# --------------------------------------------------------------------------
# one pipeline stage: F / B / W passes over microbatches
# --------------------------------------------------------------------------

class Stage:
    """Stage `stage` of p: layers [first, last) plus the embedding (stage 0)
    and the head (stage p-1).  Passes keep per-microbatch stashes; grads are
    accumulated in fp64 in the order W passes are called (C4)."""

    def __init__(self, cfg, p: int, stage: int, params: Dict[str, Array], m: int):
        from zb_synth import stage_layers
        self.cfg, self.p, self.stage, self.m = cfg, p, stage, m
        self.first, self.last = stage_layers(cfg.L, p, stage)
        self.params = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
        self.grads = {k: np.zeros_like(v) for k, v in self.params.items()}
        self.fstash: Dict[int, dict] = {}
        self.wstash: Dict[int, dict] = {}
        self.losses: Dict[int, float] = {}

    def _lp(self, l: int) -> Dict[str, Array]:
        pre = f"l{l}."
        return {k[len(pre):]: v for k, v in self.params.items() if k.startswith(pre)}

    def _acc(self, name: str, g: Array) -> None:
        self.grads[name] += g

    # F ---------------------------------------------------------------
    def forward(self, j: int, inp: Array, labels: Optional[Array] = None):
        c, b, s, a = self.cfg, self.cfg.b, self.cfg.s, self.cfg.a
        st = {}
        if self.stage == 0:
            st["tok"] = inp
            x = embed_forward(inp, self.params["wte"], self.params["wpe"])
        else:
            x = np.asarray(inp, dtype=np.float64)
        caches = []
        for l in range(self.first, self.last):
            x, cl = layer_forward(x, self._lp(l), b, s, a)
            caches.append(cl)
        st["layers"] = caches
        out = x
        if self.stage == self.p - 1:
            loss, hc = head_forward(x, self.params["lnf_g"], self.params["lnf_b"], self.params["head_w"],
                                    labels, self.m)
            st["head"] = hc
            self.losses[j] = loss
            out = loss
        self.fstash[j] = st
        return out

    # B ---------------------------------------------------------------
    def backward_input(self, j: int, dy: Optional[Array] = None):
        b, s, a = self.cfg.b, self.cfg.s, self.cfg.a
        st = self.fstash.pop(j)
        ws = {}
        if self.stage == self.p - 1:
            dy, ws["head"] = head_backward_input(st["head"], self.params["lnf_g"], self.params["head_w"])
        ls = []
        for idx in reversed(range(self.last - self.first)):
            l = self.first + idx
            dy, w = layer_backward_input(dy, st["layers"][idx], self._lp(l), b, s, a)
            ls.append((l, w))
        ws["layers"] = ls
        if self.stage == 0:
            ws["embed"] = (st["tok"], dy)
            dy = None
        self.wstash[j] = ws
        return dy

    # W ---------------------------------------------------------------
    def backward_weight(self, j: int) -> None:
        ws = self.wstash.pop(j)
        if "head" in ws:
            for k, g in head_backward_weight(ws["head"]).items():
                self._acc(k, g)
        for l, w in ws["layers"]:
            for k, g in layer_backward_weight(w).items():
                self._acc(f"l{l}.{k}", g)
        if "embed" in ws:
            tok, dx0 = ws["embed"]
            dwte, dwpe = embed_backward_weight(tok, dx0, self.cfg.V, self.cfg.s)
            self._acc("wte", dwte)
            self._acc("wpe", dwpe)

    # unsplit B+W (the traditional backward) ---------------------------
    def backward_unsplit(self, j: int, dy: Optional[Array] = None):
        b, s, a = self.cfg.b, self.cfg.s, self.cfg.a
        st = self.fstash.pop(j)
        if self.stage == self.p - 1:
            dy, ws = head_backward_input(st["head"], self.params["lnf_g"], self.params["head_w"])
            for k, g in head_backward_weight(ws).items():
                self._acc(k, g)
        for idx in reversed(range(self.last - self.first)):
            l = self.first + idx
            dy, g = layer_backward_unsplit(dy, st["layers"][idx], self._lp(l), b, s, a)
            for k, v in g.items():
                self._acc(f"l{l}.{k}", v)
        if self.stage == 0:
            dwte, dwpe = embed_backward_weight(st["tok"], dy, self.cfg.V, self.cfg.s)
            self._acc("wte", dwte)
            self._acc("wpe", dwpe)
            return None
        return dy


def reference_iteration(cfg, params: Dict[str, Array], tokens: Array, p: int = 1, m: Optional[int] = None):
    """Plain definition of one training iteration's loss and gradients: all
    microbatches in order, each F then the unsplit backward, grads summed in
    microbatch order.  `params` holds the whole model (p=1 names); returns
    (loss, grads)."""
    m = tokens.shape[0] if m is None else m
    st = Stage(cfg, 1, 0, params, m)
    loss = 0.0
    for j in range(m):
        loss += st.forward(j, tokens[j, :, :cfg.s], tokens[j, :, 1:])
        st.backward_unsplit(j)
    return loss, st.grads


def run_pass_lists(cfg, p: int, params: Dict[str, Array], tokens: Array, lists, fused_backward: bool = False):
    """Execute per-stage pass lists (as produced by oracle.schedule) serially
    in a global order consistent with every dependency: a pass runs when it is
    next in its stage's list and its cross-stage inputs exist.  Passing
    activations / gradients between Stage objects stands in for P2P.
    Returns (loss, merged grads, execution order)."""
    from zb_synth import param_specs
    m = tokens.shape[0]
    stages = []
    for sidx in range(p):
        names = [n for n, _, _ in param_specs(cfg, p, sidx)]
        stages.append(Stage(cfg, p, sidx, {n: params[n] for n in names}, m))
    acts: Dict[Tuple[int, int], Array] = {}
    grads_in: Dict[Tuple[int, int], Array] = {}
    pos = [0] * p
    order = []
    total = sum(len(x) for x in lists)
    done = 0
    while done < total:
        progressed = False
        for sidx in range(p):
            if pos[sidx] >= len(lists[sidx]):
                continue
            kind, j = lists[sidx][pos[sidx]]
            st = stages[sidx]
            if kind == "F":
                lab = tokens[j, :, 1:] if sidx == p - 1 else None
                if sidx == 0:
                    out = st.forward(j, tokens[j, :, :cfg.s], lab)
                elif (sidx, j) in acts:
                    out = st.forward(j, acts.pop((sidx, j)), lab)
                else:
                    continue
                if sidx < p - 1:
                    acts[(sidx + 1, j)] = out
            elif kind == "B":
                if sidx == p - 1:
                    dy = None
                elif (sidx, j) in grads_in:
                    dy = grads_in.pop((sidx, j))
                else:
                    continue
                dx = st.backward_unsplit(j, dy) if fused_backward else st.backward_input(j, dy)
                if sidx > 0:
                    grads_in[(sidx - 1, j)] = dx
            else:  # W
                if not fused_backward:
                    st.backward_weight(j)
            order.append((sidx, kind, j))
            pos[sidx] += 1
            done += 1
            progressed = True
        if not progressed:
            raise RuntimeError("pass lists deadlock (invalid schedule)")
    loss = sum(stages[-1].losses.values())
    grads: Dict[str, Array] = {}
    for st in stages:
        grads.update(st.grads)
    return loss, grads, order
