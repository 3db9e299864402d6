"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path.

This module holds DATA ONLY: model-shape tables, the layer partition rule,
parameter names/shapes in the canonical order, and seeded random draws.  It
contains none of the method's arithmetic (no layer math, no schedules, no
optimizer), so that `oracle/` and `paper_2401_10241_b200/` can both consume
identical inputs while sharing no code (DESIGN.md §"Inputs").

Recipe (DESIGN.md §"Input recipe"):
  * every parameter tensor has its own numpy PCG64 stream seeded with
    SeedSequence([weight_seed, crc32(name)]) so a stage can be generated
    without generating the whole model;
  * matrices and embeddings ~ N(0, 0.02^2); the two residual-output
    projections (proj_w, fc2_w) ~ N(0, (0.02/sqrt(2L))^2);
  * biases ~ N(0, 0.02^2), LayerNorm gains 1 + N(0, 0.02^2), LayerNorm
    biases N(0, 0.02^2) (non-trivial so the bias / LN-grad paths are tested);
  * tokens: PCG64(data_seed + iteration), uniform integers in [0, V), shape
    [m, b, s+1]; inputs are [..., :s], labels are [..., 1:].

Model shapes follow PAPER.md Table "experiment_model"; the tiny
config is BASELINE.json configs[0].  Vocabulary V = 50304 is the SURVEY.md
C1 reading (the paper is silent).
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field, replace
from typing import Dict, List, Sequence, Tuple

import numpy as np

WEIGHT_SEED = 1234
DATA_SEED = 1000


@dataclass(frozen=True)
class ModelConfig:
    name: str
    h: int          # hidden size
    a: int          # attention heads
    L: int          # total transformer layers
    s: int          # sequence length
    b: int          # microbatch size (sequences)
    V: int          # vocabulary
    p: int          # pipeline stages of the named config
    m: int          # microbatches per iteration
    family: str     # schedule family the config is quoted on
    mem_factor: int = 1   # AUTO: M_limit = mem_factor * (1F1B peak)
    post_validation: bool = False

    @property
    def d(self) -> int:
        return self.h // self.a

    @property
    def T(self) -> int:
        return self.b * self.s

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


# BASELINE.json configs[0..4]; b from PAPER.md P:177-180.
CONFIGS: Dict[str, ModelConfig] = {
    "tiny": ModelConfig("tiny", h=64, a=1, L=8, s=1024, b=1, V=512, p=4, m=8, family="zbh1"),
    "1.5B": ModelConfig("1.5B", h=2304, a=24, L=22, s=1024, b=6, V=50304, p=8, m=24, family="zbh1"),
    "6.2B": ModelConfig("6.2B", h=4096, a=32, L=30, s=1024, b=3, V=50304, p=8, m=32, family="zbh2"),
    "14.6B": ModelConfig("14.6B", h=5120, a=40, L=46, s=1024, b=1, V=50304, p=8, m=48, family="auto",
                         mem_factor=1),
    "28.3B": ModelConfig("28.3B", h=6144, a=48, L=62, s=1024, b=1, V=50304, p=8, m=64, family="auto",
                         mem_factor=2, post_validation=True),
}


def partition(L: int, p: int) -> List[int]:
    """Layers per stage.  PAPER.md P:169: the first and last stage hold one
    fewer layer than the middle stages.  Applied when (L+2) % p == 0 and
    p >= 2; otherwise an even split (remainder to the middle stages), which
    is the tiny config's [2,2,2,2]."""
    if p <= 0 or L < p:
        raise ValueError(f"cannot partition {L} layers over {p} stages")
    if p == 1:
        return [L]
    if (L + 2) % p == 0 and (L + 2) // p >= 2:
        mid = (L + 2) // p
        return [mid - 1] + [mid] * (p - 2) + [mid - 1]
    base, rem = divmod(L, p)
    out = [base] * p
    # remainder to the middle stages first (stage order 1, 2, ..., then 0, p-1)
    order = list(range(1, p - 1)) + [0, p - 1]
    for i in range(rem):
        out[order[i % p]] += 1
    return out


def stage_layers(L: int, p: int, stage: int) -> Tuple[int, int]:
    """[first, last) global layer indices of `stage`."""
    parts = partition(L, p)
    first = sum(parts[:stage])
    return first, first + parts[stage]


LAYER_PARAMS: Sequence[Tuple[str, str]] = (
    ("ln1_g", "ln_gain"), ("ln1_b", "ln_bias"),
    ("qkv_w", "matrix"), ("qkv_b", "bias"),
    ("proj_w", "matrix_out"), ("proj_b", "bias"),
    ("ln2_g", "ln_gain"), ("ln2_b", "ln_bias"),
    ("fc1_w", "matrix"), ("fc1_b", "bias"),
    ("fc2_w", "matrix_out"), ("fc2_b", "bias"),
)


def _layer_shape(short: str, h: int) -> Tuple[int, ...]:
    return {
        "ln1_g": (h,), "ln1_b": (h,), "qkv_w": (3 * h, h), "qkv_b": (3 * h,),
        "proj_w": (h, h), "proj_b": (h,), "ln2_g": (h,), "ln2_b": (h,),
        "fc1_w": (4 * h, h), "fc1_b": (4 * h,), "fc2_w": (h, 4 * h), "fc2_b": (h,),
    }[short]


def param_specs(cfg: ModelConfig, p: int, stage: int) -> List[Tuple[str, Tuple[int, ...], str]]:
    """Canonical ordered (name, shape, kind) list of the parameters owned by
    `stage` when the model is split over p stages.  This order is the one
    zb_ctx_set_params() expects (include/zb.h)."""
    first, last = stage_layers(cfg.L, p, stage)
    specs: List[Tuple[str, Tuple[int, ...], str]] = []
    if stage == 0:
        specs.append(("wte", (cfg.V, cfg.h), "embedding"))
        specs.append(("wpe", (cfg.s, cfg.h), "embedding"))
    for l in range(first, last):
        for short, kind in LAYER_PARAMS:
            specs.append((f"l{l}.{short}", _layer_shape(short, cfg.h), kind))
    if stage == p - 1:
        specs.append(("lnf_g", (cfg.h,), "ln_gain"))
        specs.append(("lnf_b", (cfg.h,), "ln_bias"))
        specs.append(("head_w", (cfg.V, cfg.h), "matrix"))
    return specs


def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, zlib.crc32(name.encode())])))


def make_param(cfg: ModelConfig, name: str, shape: Tuple[int, ...], kind: str,
               seed: int = WEIGHT_SEED) -> np.ndarray:
    """One parameter tensor, float32, from its own seeded stream."""
    g = _rng(seed, name)
    z = g.standard_normal(shape, dtype=np.float32)
    std = np.float32(0.02)
    if kind == "matrix_out":
        std = np.float32(0.02 / np.sqrt(2.0 * cfg.L))
    z *= std
    if kind == "ln_gain":
        z += np.float32(1.0)
    return z


def make_stage_params(cfg: ModelConfig, p: int, stage: int, seed: int = WEIGHT_SEED) -> Dict[str, np.ndarray]:
    return {n: make_param(cfg, n, sh, k, seed) for n, sh, k in param_specs(cfg, p, stage)}


def make_model_params(cfg: ModelConfig, seed: int = WEIGHT_SEED) -> Dict[str, np.ndarray]:
    out: Dict[str, np.ndarray] = {}
    for n, sh, k in param_specs(cfg, 1, 0):
        out[n] = make_param(cfg, n, sh, k, seed)
    return out


def make_tokens(cfg: ModelConfig, iteration: int = 0, m: int | None = None,
                seed: int = DATA_SEED) -> np.ndarray:
    """int32 [m, b, s+1] token ids; inputs tok[..., :s], labels tok[..., 1:]."""
    m = cfg.m if m is None else m
    g = np.random.Generator(np.random.PCG64(seed + iteration))
    return g.integers(0, cfg.V, size=(m, cfg.b, cfg.s + 1), dtype=np.int64).astype(np.int32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even) and return
    them as float32.  Data preparation only: the bf16-mode parity tests give
    the oracle the same bf16-rounded weights the GPU computes with, so weight
    quantisation is not counted as kernel error."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out.reshape(x.shape)
