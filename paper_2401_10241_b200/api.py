"""Thin Python wrappers over include/zb.h (marshalling only; no compute here)."""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import (FAMILY, ZB_DTYPE_BF16, ZB_DTYPE_F32, check, lib, zb_model_cfg_t, zb_optim_cfg_t, zb_pass_t,
                   zb_pv_report_t, zb_sim_t, zb_iter_stats_t)

KIND_NAME = {0: "F", 1: "B", 2: "W"}


# ------------------------------------------------------------------ schedules

def schedule(family: str, p: int, m: int, T_F: int, T_B: int, T_W: int, T_comm: int = 0,
             M_limit: int = 0, M_B: int = 1, M_W: int = 1):
    """zb_schedule -> (passes array, sim).  passes are grouped by stage."""
    n = 3 * p * m
    out = (zb_pass_t * n)()
    sim = zb_sim_t()
    check(lib.zb_schedule(p, m, int(T_F), int(T_B), int(T_W), int(T_comm), int(M_limit), int(M_B), int(M_W),
                          FAMILY[family], out, n, C.byref(sim)))
    return out, sim


def stage_lists(passes, p: int) -> List[List[Tuple[str, int]]]:
    lists: List[List[Tuple[str, int]]] = [[] for _ in range(p)]
    for q in passes:
        lists[q.stage].append((KIND_NAME[q.kind], q.microbatch))
    return lists


def simulate(p: int, m: int, lists: Sequence[Sequence[Tuple[str, int]]], T_F, T_B, T_W, T_comm: int = 0,
             M_B: int = 1, M_W: int = 1, fused: bool = False):
    kinds = {"F": 0, "B": 1, "W": 2}
    n = 3 * p * m
    arr = (zb_pass_t * n)()
    k = 0
    for s, o in enumerate(lists):
        for kind, j in o:
            arr[k].stage, arr[k].microbatch, arr[k].kind, arr[k].slot = s, j, kinds[kind], -1
            k += 1
    per = lambda x: (C.c_int64 * p)(*([int(x)] * p if isinstance(x, (int, float)) else [int(v) for v in x]))
    sim = zb_sim_t()
    check(lib.zb_simulate(p, m, arr, n, per(T_F), per(T_B), per(T_W), int(T_comm), int(M_B), int(M_W),
                          1 if fused else 0, C.byref(sim)))
    return arr, sim


# ------------------------------------------------------------------ kernels (debug entry points)

def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream


def dbg_gemm(A, B, C_out, *, M, N, K, a_mn=False, b_mn=False, epi=0, bias=None, aux=None, beta=0,
             lda=None, ldb=None, ldc=None, ldaux=None, stream=None):
    dtype = ZB_DTYPE_F32 if A.dtype.is_floating_point and A.element_size() == 4 else ZB_DTYPE_BF16
    lda = lda if lda is not None else A.shape[-1]
    ldb = ldb if ldb is not None else B.shape[-1]
    ldc = ldc if ldc is not None else C_out.shape[-1]
    ldaux = ldaux if ldaux is not None else (aux.shape[-1] if aux is not None else 0)
    check(lib.zb_dbg_gemm(dtype, M, N, K, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn), epi, _ptr(C_out), ldc,
                          _ptr(bias), _ptr(aux), ldaux, beta, _stream(stream)))


def dbg_attention_fwd(qkv, o, lse, *, b, s, a, d, stream=None):
    dtype = ZB_DTYPE_F32 if qkv.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_attention_fwd(dtype, b, s, a, d, _ptr(qkv), _ptr(o), _ptr(lse), _stream(stream)))


def dbg_attention_bwd(qkv, o, dout, lse, dqkv, delta, *, b, s, a, d, stream=None):
    dtype = ZB_DTYPE_F32 if qkv.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_attention_bwd(dtype, b, s, a, d, _ptr(qkv), _ptr(o), _ptr(dout), _ptr(lse), _ptr(dqkv),
                                   _ptr(delta), _stream(stream)))
