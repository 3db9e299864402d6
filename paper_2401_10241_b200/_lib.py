"""ctypes binding of libzb.so (include/zb.h, include/zb_debug.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Importing this module loads the in-tree libzb.so and raises
immediately if it is missing or stale — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ZB_LIB: alternative in-tree build of the same library (debug variants, e.g. libzb_v1.so)
LIB_PATH = os.path.join(_HERE, os.environ.get("ZB_LIB", "libzb.so"))

ZB_OK, ZB_EINVAL, ZB_ELIMIT, ZB_ECAP, ZB_ECUDA, ZB_ENCCL, ZB_ESTATE, ZB_ETIMEOUT = 0, -1, -2, -3, -4, -5, -6, -7
ZB_F, ZB_B, ZB_W = 0, 1, 2
ZB_1F1B, ZB_H1, ZB_H2, ZB_AUTO = 0, 1, 2, 3
FAMILY = {"1f1b": ZB_1F1B, "zbh1": ZB_H1, "zbh2": ZB_H2, "auto": ZB_AUTO}
ZB_V, ZB_1F1B_I = 4, 5
CHUNKED_FAMILY = {"zbv": ZB_V, "1f1bi": ZB_1F1B_I}
ZB_DTYPE_BF16, ZB_DTYPE_F32 = 0, 1
ZB_RUN_HOST_INPUTS, ZB_RUN_TIMING, ZB_RUN_FUSED_BW, ZB_RUN_GROUP_W, ZB_RUN_DP_REORDER, ZB_RUN_GRAPH = 1, 2, 4, 8, 16, 32
ZB_OPT_SYNC, ZB_OPT_PV = 0, 1
ZB_CFG_HEAD_W_EAGER = 1
ZB_MAX_STAGES = 64

ACTIONS = {0: "none", 1: "step", 2: "skip", 3: "defer", 4: "rollback", 5: "rollback+redo", 6: "deferred-step",
           7: "clipped-step"}


class ZbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"zb error {code}: {msg}")
        self.code = code


class zb_pass_t(C.Structure):
    _fields_ = [("stage", C.c_int32), ("microbatch", C.c_int32), ("kind", C.c_int32), ("slot", C.c_int32),
                ("start", C.c_int64), ("end", C.c_int64)]


class zb_sim_t(C.Structure):
    _fields_ = [("cost", C.c_int64), ("work", C.c_int64), ("bubble_rate", C.c_double),
                ("peak_bytes", C.c_int64 * ZB_MAX_STAGES), ("n_slots", C.c_int32 * ZB_MAX_STAGES),
                ("chosen", C.c_int32), ("n_passes", C.c_int32)]


class zb_model_cfg_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("h", "a", "L", "s", "b", "V", "p", "stage", "layer_first", "layer_last",
                                         "m", "n_slots", "dtype", "flags")]


class zb_iter_stats_t(C.Structure):
    _fields_ = [("n_passes", C.c_int32), ("pass_start_ms", C.c_float * 3072), ("pass_end_ms", C.c_float * 3072),
                ("loss", C.c_double)]


class zb_optim_cfg_t(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("clip", C.c_float), ("mode", C.c_int32)]


class zb_pv_report_t(C.Structure):
    _fields_ = [("local_sumsq", C.c_double), ("partial_sumsq", C.c_double), ("full_sumsq", C.c_double),
                ("local_nonfinite", C.c_int32), ("partial_nonfinite", C.c_int32), ("full_nonfinite", C.c_int32),
                ("first_action", C.c_int32), ("final_action", C.c_int32), ("t", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          f"(make -C paper_2401_10241_b200)")
    return C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)


lib = _load()

_P = C.c_void_p
_I32, _I64 = C.c_int32, C.c_int64
_SIGS = {
    "zb_last_error": ([], C.c_char_p),
    "zb_version": ([], C.c_char_p),
    "zb_schedule": ([_I32, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, C.POINTER(zb_pass_t), _I32,
                     C.POINTER(zb_sim_t)], _I32),
    "zb_schedule_chunked": ([_I32, _I32, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I32, C.POINTER(zb_pass_t),
                             _I32, C.POINTER(zb_sim_t)], _I32),
    "zb_schedule_per_stage": ([_I32, _I32, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64), _I64, _I64, _I64, _I64,
                               _I32, C.POINTER(zb_pass_t), _I32, C.POINTER(zb_sim_t)], _I32),
    "zb_partition": ([_I32, _I32, C.POINTER(_I32)], _I32),
    "zb_simulate": ([_I32, _I32, C.POINTER(zb_pass_t), _I32, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64),
                     _I64, _I64, _I64, _I32, C.POINTER(zb_sim_t)], _I32),
    "zb_dbg_gemm": ([_I32, _I32, _I32, _I32, _P, _I64, _I32, _P, _I64, _I32, _I32, _P, _I64, _P, _P, _I64, _I32, _P],
                    _I32),
    "zb_dbg_gemm_wgroup": ([_I32, _I32, _I32, _I32, C.POINTER(_P), C.POINTER(_P), _P, _P, _I32, _P], _I32),
    "zb_dbg_layernorm_fwd": ([_I32, _P, _P, _P, _P, _P, _P, _I32, _I32, C.c_float, _P], _I32),
    "zb_dbg_layernorm_bwd": ([_I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P], _I32),
    "zb_dbg_bias_grad": ([_I32, _P, _I64, _P, _I32, _I32, _I32, _P], _I32),
    "zb_dbg_attention_fwd": ([_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P], _I32),
    "zb_dbg_attention_bwd": ([_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P], _I32),
    "zb_dbg_stage_plan": ([C.POINTER(zb_pass_t), _I32, _I32, _I32, _I32, _I32, _I32, _I32, C.POINTER(_I32), _I32,
                           C.POINTER(_I32)], _I32),
    "zb_dbg_dp_plan": ([C.POINTER(zb_pass_t), _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                        C.POINTER(_I32), _I32, C.POINTER(_I32)], _I32),
    "zb_dbg_w_units": ([_P, C.POINTER(_I32), C.POINTER(_I64)], _I32),
    "zb_ctx_attach_dp": ([_P, _P, _I32, _I32], _I32),
    "zb_dbg_worker_plan": ([C.POINTER(zb_pass_t), _I32, _I32, _I32, _I32, C.POINTER(_I32), _I32, C.POINTER(_I32),
                            _I32, C.POINTER(_I32)], _I32),
    "zb_ctx_attach_nccl_chunks": ([C.POINTER(_P), _I32, _P, _I32, C.POINTER(_I32), _I32], _I32),
    "zb_run_iteration_worker": ([C.POINTER(_P), _I32, C.POINTER(zb_pass_t), _I32, _P, _P, _I32], _I32),
    "zb_dbg_speculative_counts": ([C.POINTER(zb_pass_t), _I32, _I32, C.POINTER(_I32)], _I32),
    "zb_dbg_kernel_timing": ([_I32, _I32], _I32),
    "zb_dbg_launch_count": ([_I32, C.POINTER(_I64)], _I32),
    "zb_dbg_kernel_timing_read": ([_I32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(_I64)], _I32),
    "zb_ctx_arena_bytes": ([C.POINTER(zb_model_cfg_t), C.POINTER(C.c_size_t)], _I32),
    "zb_ctx_slot_bytes": ([C.POINTER(zb_model_cfg_t), C.POINTER(C.c_size_t)], _I32),
    "zb_ctx_create": ([C.POINTER(zb_model_cfg_t), _P, C.c_size_t, _P, C.POINTER(_P)], _I32),
    "zb_ctx_destroy": ([_P], _I32),
    "zb_ctx_sync": ([_P], _I32),
    "zb_ctx_param_count": ([_P, C.POINTER(_I32)], _I32),
    "zb_ctx_param_numel": ([_P, C.POINTER(_I64)], _I32),
    "zb_ctx_set_params": ([_P, C.POINTER(_P), _I32], _I32),
    "zb_ctx_get_params": ([_P, C.POINTER(_P), _I32], _I32),
    "zb_ctx_get_grads": ([_P, C.POINTER(_P), _I32], _I32),
    "zb_ctx_get_moments": ([_P, C.POINTER(_P), C.POINTER(_P), _I32], _I32),
    "zb_ctx_begin_iteration": ([_P], _I32),
    "zb_ctx_read_loss": ([_P, C.POINTER(C.c_double)], _I32),
    "zb_ctx_slot_ptr": ([_P, _I32, _I32, C.POINTER(_P)], _I32),
    "zb_stage_forward": ([_P, _I32, _I32, _P, _P, _P], _I32),
    "zb_stage_backward_input": ([_P, _I32, _I32, _P, _P], _I32),
    "zb_stage_backward_weight": ([_P, _I32, _I32], _I32),
    "zb_run_iteration": ([_P, C.POINTER(zb_pass_t), _I32, _P, _P, _I32], _I32),
    "zb_run_iteration_local": ([C.POINTER(_P), _I32, C.POINTER(zb_pass_t), _I32, _P, _P, _I32], _I32),
    "zb_ctx_read_stats": ([_P, C.POINTER(zb_iter_stats_t)], _I32),
    "zb_ctx_profile": ([_P, _I32, C.POINTER(_I64), C.POINTER(_I32)], _I32),
    "zb_post_validate_step": ([_P, C.POINTER(zb_optim_cfg_t)], _I32),
    "zb_post_validate_finish": ([_P, C.POINTER(zb_optim_cfg_t)], _I32),
    "zb_post_validate_local": ([C.POINTER(_P), _I32, C.POINTER(zb_optim_cfg_t)], _I32),
    "zb_ctx_read_pv_report": ([_P, C.POINTER(zb_pv_report_t)], _I32),
    "zb_nccl_unique_id": ([_P], _I32),
    "zb_ctx_attach_nccl": ([_P, _P, _I32, _I32], _I32),
    "zb_ctx_comm_probe": ([_P, C.c_size_t, _I32, C.POINTER(_I64)], _I32),
    "zb_loopback_create": ([_I32, C.POINTER(_P)], _I32),
    "zb_loopback_destroy": ([_P], _I32),
    "zb_ctx_attach_loopback": ([_P, _P, _I32], _I32),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name, None)
    if _f is None:
        continue   # reported by tests/test_abi.py (every header symbol must be exported)
    _f.argtypes = _args
    _f.restype = _res


def check(code: int) -> None:
    if code != ZB_OK:
        raise ZbError(code, lib.zb_last_error().decode(errors="replace"))


def exported_symbols():
    return [n for n in _SIGS if getattr(lib, n, None) is not None]
