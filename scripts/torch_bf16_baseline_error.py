"""Diagnostic: how far does standard torch bf16 mixed precision (autocast,
flash SDPA) land from the fp64 oracle on the same config?  Context for the
bf16 tolerance (DESIGN.md R-tol) — not part of the product path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import numpy as np, torch, torch.nn.functional as F
import zb_synth
from oracle import model as om

def run(cfg):
    params = zb_synth.make_model_params(cfg)
    MAT = ("qkv_w", "proj_w", "fc1_w", "fc2_w", "head_w")
    params_r = {k: (zb_synth.round_to_bf16(v) if k.endswith(MAT) else v) for k, v in params.items()}
    tok = zb_synth.make_tokens(cfg, 0)
    ref_loss, ref = om.reference_iteration(cfg, params_r, tok)
    P = {k: torch.tensor(v, device="cuda", dtype=torch.float32, requires_grad=True) for k, v in params_r.items()}
    h, a, s, b = cfg.h, cfg.a, cfg.s, cfg.b; d = h // a
    total = 0.0
    with torch.autocast("cuda", dtype=torch.bfloat16):
        for j in range(tok.shape[0]):
            t = torch.tensor(tok[j, :, :s].astype(np.int64), device="cuda"); lab = torch.tensor(tok[j, :, 1:].astype(np.int64), device="cuda")
            x = P["wte"][t] + P["wpe"][:s][None]
            for l in range(cfg.L):
                q = lambda n: P[f"l{l}.{n}"]
                ln1 = F.layer_norm(x, (h,), q("ln1_g"), q("ln1_b"), eps=1e-5)
                qkv = F.linear(ln1, q("qkv_w"), q("qkv_b"))
                Q, K, V = qkv.split(h, -1)
                sh = lambda z: z.reshape(b, s, a, d).transpose(1, 2)
                o = F.scaled_dot_product_attention(sh(Q), sh(K), sh(V), is_causal=True).transpose(1, 2).reshape(b, s, h)
                x = x + F.linear(o, q("proj_w"), q("proj_b"))
                ln2 = F.layer_norm(x, (h,), q("ln2_g"), q("ln2_b"), eps=1e-5)
                x = x + F.linear(F.gelu(F.linear(ln2, q("fc1_w"), q("fc1_b")), approximate="tanh"), q("fc2_w"), q("fc2_b"))
            lnf = F.layer_norm(x, (h,), P["lnf_g"], P["lnf_b"], eps=1e-5)
            logits = F.linear(lnf, P["head_w"]).float()
            total = total + F.cross_entropy(logits.reshape(-1, cfg.V), lab.reshape(-1)) / tok.shape[0]
    total.backward()
    errs = {k: float(np.linalg.norm(P[k].grad.double().cpu().numpy() - ref[k]) / np.linalg.norm(ref[k])) for k in ref}
    e = sorted(errs.values(), reverse=True)
    print(cfg.name, "torch-bf16 loss", float(total), "oracle", ref_loss, "mean", np.mean(e), "max", e[0])
    blocks = {}
    for k in ref:
        if k.endswith("qkv_w"):
            g = P[k].grad.double().cpu().numpy()
            for i, part in enumerate("QKV"):
                r = ref[k][i * h:(i + 1) * h]
                blocks[f"{k}.{part}"] = float(np.linalg.norm(g[i * h:(i + 1) * h] - r) / np.linalg.norm(r))
    print(cfg.name, "torch-bf16 per-tensor", json.dumps({k: round(v, 4) for k, v in errs.items()}))
    print(cfg.name, "torch-bf16 qkv blocks", json.dumps({k: round(v, 4) for k, v in blocks.items()}))

if len(sys.argv) > 1:
    run(zb_synth.CONFIGS[sys.argv[1]].with_(L=2, b=2, m=2))
else:
    run(zb_synth.CONFIGS["tiny"])
    run(zb_synth.ModelConfig("d64", h=64, a=1, L=4, s=256, b=2, V=512, p=4, m=3, family="zbh1"))
