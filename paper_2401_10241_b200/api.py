"""Thin Python wrappers over include/zb.h (marshalling only; no compute here).

torch provides device memory (the context arena) and streams; every step of
the hot path runs in libzb.so's kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from ._lib import (CHUNKED_FAMILY, FAMILY, ZB_DTYPE_BF16, ZB_DTYPE_F32, ZB_OPT_PV, ZB_OPT_SYNC, ZB_RUN_FUSED_BW,
                   ZB_RUN_DP_REORDER, ZB_RUN_GRAPH, ZB_RUN_GROUP_W, ZB_RUN_HOST_INPUTS, ZB_RUN_TIMING, ZB_CFG_HEAD_W_EAGER,
                   ACTIONS, check, lib, zb_iter_stats_t, zb_model_cfg_t, zb_optim_cfg_t, zb_pass_t, zb_pv_report_t,
                   zb_sim_t)

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


def schedule_per_stage(family: str, p: int, m: int, T_F: Sequence[int], T_B: Sequence[int], T_W: Sequence[int],
                       T_comm: int = 0, M_limit: int = 0, M_B: int = 1, M_W: int = 1):
    """zb_schedule_per_stage (per-stage profiled times) -> (passes, sim)."""
    n = 3 * p * m
    out = (zb_pass_t * n)()
    sim = zb_sim_t()
    arr = lambda x: (C.c_int64 * p)(*[int(v) for v in x])
    check(lib.zb_schedule_per_stage(p, m, arr(T_F), arr(T_B), arr(T_W), int(T_comm), int(M_limit), int(M_B),
                                    int(M_W), FAMILY[family], out, n, C.byref(sim)))
    return out, sim


def partition(L: int, p: int) -> List[int]:
    """zb_partition: layers per stage."""
    out = (C.c_int32 * p)()
    check(lib.zb_partition(L, p, out))
    return list(out)


def stage_layers(L: int, p: int, stage: int) -> Tuple[int, int]:
    parts = partition(L, p)
    first = sum(parts[:stage])
    return first, first + parts[stage]


def schedule_chunked(family: str, p: int, m: int, chunks: int, T_F: int, T_B: int, T_W: int, T_comm: int = 0,
                     M_limit: int = 0, M_B: int = 1, M_W: int = 1):
    """zb_schedule_chunked ("zbv" | "1f1bi") -> (passes, sim).  passes are
    grouped by WORKER; each pass's `stage` is its virtual stage (chunk)."""
    n = 3 * chunks * p * m
    out = (zb_pass_t * n)()
    sim = zb_sim_t()
    check(lib.zb_schedule_chunked(p, m, chunks, int(T_F), int(T_B), int(T_W), int(T_comm), int(M_limit), int(M_B),
                                  int(M_W), CHUNKED_FAMILY[family], out, n, C.byref(sim)))
    return out, sim


def worker_lists(passes, p: int, m: int, chunks: int) -> List[List[Tuple[str, int, int]]]:
    """Split a zb_schedule_chunked output into per-worker (kind, v, j) lists."""
    per = 3 * chunks * m
    return [[(KIND_NAME[q.kind], q.stage, q.microbatch) for q in passes[w * per:(w + 1) * per]] for w in range(p)]


def stage_lists(passes, p: int) -> List[List[Tuple[str, int]]]:
    lists: List[List[Tuple[str, int]]] = [[] for _ in range(p)]
    for q in passes:
        lists[q.stage].append((KIND_NAME[q.kind], q.microbatch))
    return lists


def stage_passes(passes, stage: int):
    sel = [q for q in passes if q.stage == stage]
    arr = (zb_pass_t * len(sel))()
    for i, q in enumerate(sel):
        arr[i] = q
    return arr


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


# ------------------------------------------------------------------ helpers

def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream


# ------------------------------------------------------------------ stage context

def model_cfg(cfg, p: int, stage: int, m: int, n_slots: int, dtype: str = "bf16",
              head_w_eager: bool = False) -> zb_model_cfg_t:
    first, last = stage_layers(cfg.L, p, stage)
    return zb_model_cfg_t(cfg.h, cfg.a, cfg.L, cfg.s, cfg.b, cfg.V, p, stage, first, last, m, n_slots,
                          ZB_DTYPE_BF16 if dtype == "bf16" else ZB_DTYPE_F32, 1 if head_w_eager else 0)


def arena_bytes(mc: zb_model_cfg_t) -> int:
    n = C.c_size_t()
    check(lib.zb_ctx_arena_bytes(C.byref(mc), C.byref(n)))
    return n.value


def slot_bytes(mc: zb_model_cfg_t) -> int:
    n = C.c_size_t()
    check(lib.zb_ctx_slot_bytes(C.byref(mc), C.byref(n)))
    return n.value


class Context:
    """One pipeline stage (zb_ctx_t) with a torch-allocated device arena."""

    def __init__(self, cfg, p: int, stage: int, m: int, n_slots: int, dtype: str = "bf16", stream=None,
                 head_w_eager: bool = False):
        import torch
        self.cfg, self.p, self.stage, self.m, self.dtype = cfg, p, stage, m, dtype
        self.mc = model_cfg(cfg, p, stage, m, n_slots, dtype, head_w_eager)
        self.nbytes = arena_bytes(self.mc)
        self.arena = torch.empty(self.nbytes, dtype=torch.uint8, device="cuda")
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = C.c_void_p()
        check(lib.zb_ctx_create(C.byref(self.mc), self.arena.data_ptr(), self.nbytes, self.stream.cuda_stream,
                                C.byref(h)))
        self.h = h
        n = C.c_int32()
        check(lib.zb_ctx_param_count(self.h, C.byref(n)))
        self.n_params = n.value
        numel = (C.c_int64 * self.n_params)()
        check(lib.zb_ctx_param_numel(self.h, numel))
        self.numel = list(numel)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib.zb_ctx_destroy(self.h)       # drains the context's stream before freeing
            self.h = C.c_void_p()
            # the arena was allocated on torch's current stream but written on self.stream
            try:
                if hasattr(self.stream, "wait_stream"):
                    self.arena.record_stream(self.stream)
            except Exception:
                pass

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # parameters -------------------------------------------------------------
    def set_params(self, arrays: Sequence[np.ndarray]):
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in arrays]
        assert len(arrs) == self.n_params, (len(arrs), self.n_params)
        for a, n in zip(arrs, self.numel):
            assert a.size == n, (a.shape, n)
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        check(lib.zb_ctx_set_params(self.h, ptrs, len(arrs)))

    def _get(self, fn, only=None) -> List[Optional[np.ndarray]]:
        """All tensors, or (only = indices) just those; the others come back as None."""
        outs = [np.empty(n, dtype=np.float32) if only is None or i in only else None
                for i, n in enumerate(self.numel)]
        ptrs = (C.c_void_p * len(outs))(*[a.ctypes.data if a is not None else None for a in outs])
        check(fn(self.h, ptrs, len(outs)))
        return outs

    def get_params(self, only=None):
        return self._get(lib.zb_ctx_get_params, only)

    def get_grads(self, only=None):
        return self._get(lib.zb_ctx_get_grads, only)

    def get_moments(self):
        ms = [np.empty(n, dtype=np.float32) for n in self.numel]
        vs = [np.empty(n, dtype=np.float32) for n in self.numel]
        pm = (C.c_void_p * len(ms))(*[a.ctypes.data for a in ms])
        pv = (C.c_void_p * len(vs))(*[a.ctypes.data for a in vs])
        check(lib.zb_ctx_get_moments(self.h, pm, pv, len(ms)))
        return ms, vs

    # passes -----------------------------------------------------------------
    def begin_iteration(self):
        check(lib.zb_ctx_begin_iteration(self.h))

    def slot_ptr(self, slot: int, which: int) -> int:
        p = C.c_void_p()
        check(lib.zb_ctx_slot_ptr(self.h, slot, which, C.byref(p)))
        return p.value

    def forward(self, mb, slot, inp: int, out: Optional[int] = None, labels: Optional[int] = None):
        check(lib.zb_stage_forward(self.h, mb, slot, inp, out, labels))

    def backward_input(self, mb, slot, dy: Optional[int] = None, dx: Optional[int] = None):
        check(lib.zb_stage_backward_input(self.h, mb, slot, dy, dx))

    def backward_weight(self, mb, slot):
        check(lib.zb_stage_backward_weight(self.h, mb, slot))

    def attach_nccl(self, ids: bytes, rank: int, world: int):
        """ids: 2*(world-1) x 128-byte NCCL unique ids, identical on every rank."""
        buf = C.create_string_buffer(ids, len(ids))
        check(lib.zb_ctx_attach_nccl(self.h, buf, rank, world))

    def attach_dp(self, id128: bytes, dp_rank: int, dp_world: int):
        """zb_ctx_attach_dp: the D-rank gradient all-reduce communicator of this stage's
        replicas (after attach_nccl when p > 1)."""
        buf = C.create_string_buffer(id128, 128) if id128 else None
        check(lib.zb_ctx_attach_dp(self.h, buf, dp_rank, dp_world))

    def w_units(self):
        """(W units of this stage's W pass, data-parallel all-reduces issued so far)."""
        n, r = C.c_int32(), C.c_int64()
        check(lib.zb_dbg_w_units(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def comm_probe(self, nbytes: int, iters: int = 10) -> int:
        """zb_ctx_comm_probe: median round trip (ns) of one message to stage+1 and back
        (collective over the pipeline; 0 on the last stage)."""
        v = C.c_int64()
        check(lib.zb_ctx_comm_probe(self.h, int(nbytes), int(iters), C.byref(v)))
        return v.value

    def attach_loopback(self, group: "Loopback"):
        """Attach to an in-process loopback group (rank = this context's stage)."""
        check(lib.zb_ctx_attach_loopback(self.h, group.h, self.stage))
        self._group = group

    def run_iteration(self, passes, tokens=None, labels=None, host_inputs=False, timing=False, fused=False,
                      group_w=False, dp_reorder=False, graph=False):
        flags = (ZB_RUN_HOST_INPUTS if host_inputs else 0) | (ZB_RUN_TIMING if timing else 0) | \
            (ZB_RUN_FUSED_BW if fused else 0) | (ZB_RUN_GROUP_W if group_w else 0) | \
            (ZB_RUN_DP_REORDER if dp_reorder else 0) | (ZB_RUN_GRAPH if graph else 0)
        tp = tokens.ctypes.data if host_inputs and tokens is not None else _ptr(tokens)
        lp = labels.ctypes.data if host_inputs and labels is not None else _ptr(labels)
        check(lib.zb_run_iteration(self.h, passes, len(passes), tp, lp, flags))

    def sync(self):
        check(lib.zb_ctx_sync(self.h))

    def loss(self) -> float:
        v = C.c_double()
        check(lib.zb_ctx_read_loss(self.h, C.byref(v)))
        return v.value

    def stats(self):
        st = zb_iter_stats_t()
        check(lib.zb_ctx_read_stats(self.h, C.byref(st)))
        n = st.n_passes
        return list(st.pass_start_ms[:n]), list(st.pass_end_ms[:n])

    def profile(self, reset: bool = False):
        """zb_ctx_profile: median (T_F, T_B, T_W) in ns over the timed runs since the
        last reset, and the sample counts (P:169 profiling iterations)."""
        t = (C.c_int64 * 3)()
        n = (C.c_int32 * 3)()
        check(lib.zb_ctx_profile(self.h, 1 if reset else 0, t, n))
        return list(t), list(n)

    # optimizer --------------------------------------------------------------
    def post_validate_step(self, opt: zb_optim_cfg_t):
        check(lib.zb_post_validate_step(self.h, C.byref(opt)))

    def post_validate_finish(self, opt: zb_optim_cfg_t):
        check(lib.zb_post_validate_finish(self.h, C.byref(opt)))

    def pv_report(self) -> Dict:
        r = zb_pv_report_t()
        check(lib.zb_ctx_read_pv_report(self.h, C.byref(r)))
        return dict(local_sumsq=r.local_sumsq, partial_sumsq=r.partial_sumsq, full_sumsq=r.full_sumsq,
                    local_nonfinite=r.local_nonfinite, partial_nonfinite=r.partial_nonfinite,
                    full_nonfinite=r.full_nonfinite, first=ACTIONS[r.first_action], final=ACTIONS[r.final_action],
                    t=r.t)


class Loopback:
    """In-process loopback transport group (zb_loopback_t) for p stage contexts on one GPU."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib.zb_loopback_create(world, C.byref(h)))
        self.h, self.world = h, world

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib.zb_loopback_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_ids(n: int) -> bytes:
    out = b""
    for _ in range(n):
        buf = C.create_string_buffer(128)
        check(lib.zb_nccl_unique_id(buf))
        out += buf.raw
    return out


def optim_cfg(lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, clip=1.0, mode="pv") -> zb_optim_cfg_t:
    return zb_optim_cfg_t(lr, beta1, beta2, eps, weight_decay, clip, ZB_OPT_PV if mode == "pv" else ZB_OPT_SYNC)


def run_local(ctxs: Sequence[Context], passes, tokens, labels, host_inputs=False, timing=False, group_w=False):
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    flags = (ZB_RUN_HOST_INPUTS if host_inputs else 0) | (ZB_RUN_TIMING if timing else 0) | \
        (ZB_RUN_GROUP_W if group_w else 0)
    tp = tokens.ctypes.data if host_inputs else _ptr(tokens)
    lp = labels.ctypes.data if host_inputs else _ptr(labels)
    check(lib.zb_run_iteration_local(arr, len(ctxs), passes, len(passes), tp, lp, flags))


def run_worker(chunks: Sequence[Context], passes, tokens=None, labels=None, fused=False, timing=False):
    """zb_run_iteration_worker: one worker's chunk contexts (virtual stages of a
    zb_schedule_chunked schedule), executed in the worker's pass order."""
    arr = (C.c_void_p * len(chunks))(*[c.h.value for c in chunks])
    flags = (ZB_RUN_TIMING if timing else 0) | (4 if fused else 0)
    check(lib.zb_run_iteration_worker(arr, len(chunks), passes, len(passes), _ptr(tokens), _ptr(labels), flags))


def attach_nccl_chunks(chunks: Sequence[Context], ids: bytes, nv: int, worker_of: Sequence[int], worker: int):
    """zb_ctx_attach_nccl_chunks: NCCL links to other workers, loopback inside this worker."""
    arr = (C.c_void_p * len(chunks))(*[c.h.value for c in chunks])
    buf = C.create_string_buffer(ids, len(ids))
    wo = (C.c_int32 * nv)(*worker_of)
    check(lib.zb_ctx_attach_nccl_chunks(arr, len(chunks), buf, nv, wo, worker))


def dp_plan(passes, p: int, m: int, stage: int, n_units: int, reorder: bool, pending=False, amend=False,
            fused=False):
    """zb_dbg_dp_plan -> [(type, microbatch, msg, slot)] (10 WP: msg = W unit; 11 ALLREDUCE)."""
    cap = 8 * len(passes) * (n_units + 1) + 64
    buf = (C.c_int32 * (4 * cap))()
    n = C.c_int32()
    check(lib.zb_dbg_dp_plan(passes, len(passes), p, m, stage, int(pending), int(amend), int(fused), n_units,
                             int(reorder), buf, cap, C.byref(n)))
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n.value)]


def worker_plan(passes, nv: int, m: int, worker: int, worker_of: Sequence[int], fused: bool = False):
    """zb_dbg_worker_plan -> [(type, microbatch, msg, slot, chunk)]."""
    cap = 16 * len(passes) + 64
    buf = (C.c_int32 * (5 * cap))()
    wo = (C.c_int32 * nv)(*worker_of)
    n = C.c_int32()
    check(lib.zb_dbg_worker_plan(passes, len(passes), nv, m, worker, wo, int(fused), buf, cap, C.byref(n)))
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]


def post_validate_local(ctxs: Sequence[Context], opt: zb_optim_cfg_t):
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    check(lib.zb_post_validate_local(arr, len(ctxs), C.byref(opt)))


# ------------------------------------------------------------------ kernels (debug entry points)

def dbg_gemm(A, B, C_out, *, M, N, K, a_mn=False, b_mn=False, epi=0, bias=None, aux=None, beta=0,
             lda=None, ldb=None, ldc=None, ldaux=None, stream=None):
    dtype = ZB_DTYPE_F32 if A.element_size() == 4 else ZB_DTYPE_BF16
    lda = lda if lda is not None else A.shape[-1]
    ldb = ldb if ldb is not None else B.shape[-1]
    ldc = ldc if ldc is not None else C_out.shape[-1]
    ldaux = ldaux if ldaux is not None else (aux.shape[-1] if aux is not None else 0)
    check(lib.zb_dbg_gemm(dtype, M, N, K, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn), epi, _ptr(C_out), ldc,
                          _ptr(bias), _ptr(aux), ldaux, beta, _stream(stream)))


def dbg_gemm_wgroup(A_segs, B_segs, C_out, *, M, N, bias=None, beta=0, stream=None):
    """zb_dbg_gemm_wgroup: C (+)= sum_s A_s^T B_s over nseg = len(A_segs) segments."""
    n = len(A_segs)
    K = sum(int(a.shape[0]) for a in A_segs)
    ap = (C.c_void_p * n)(*[a.data_ptr() for a in A_segs])
    bp = (C.c_void_p * n)(*[b.data_ptr() for b in B_segs])
    check(lib.zb_dbg_gemm_wgroup(M, N, K, n, ap, bp, _ptr(C_out), _ptr(bias), beta, _stream(stream)))


def dbg_layernorm_fwd(x, g, b, y, mean, rstd, *, rows, h, eps=1e-5, stream=None):
    dtype = ZB_DTYPE_F32 if x.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_layernorm_fwd(dtype, _ptr(x), _ptr(g), _ptr(b), _ptr(y), _ptr(mean), _ptr(rstd), rows, h,
                                   float(eps), _stream(stream)))


def dbg_layernorm_bwd(dy, x, mean, rstd, g, dx, gg, gb, *, rows, h, resid=None, dx32=None, beta=0, stream=None):
    dtype = ZB_DTYPE_F32 if x.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_layernorm_bwd(dtype, _ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(g), _ptr(resid), _ptr(dx32),
                                   _ptr(dx), _ptr(gg), _ptr(gb), beta, rows, h, _stream(stream)))


def dbg_bias_grad(y, out, *, rows, n, ldy=None, beta=0, stream=None):
    dtype = ZB_DTYPE_F32 if y.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_bias_grad(dtype, _ptr(y), ldy if ldy is not None else y.shape[-1], _ptr(out), rows, n, beta,
                               _stream(stream)))


def dbg_attention_fwd(qkv, o, lse, *, b, s, a, d, stream=None):
    dtype = ZB_DTYPE_F32 if qkv.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_attention_fwd(dtype, b, s, a, d, _ptr(qkv), _ptr(o), _ptr(lse), _stream(stream)))


def dbg_attention_bwd(qkv, o, dout, lse, dqkv, delta, *, b, s, a, d, stream=None):
    dtype = ZB_DTYPE_F32 if qkv.element_size() == 4 else ZB_DTYPE_BF16
    check(lib.zb_dbg_attention_bwd(dtype, b, s, a, d, _ptr(qkv), _ptr(o), _ptr(dout), _ptr(lse), _ptr(dqkv),
                                   _ptr(delta), _stream(stream)))
