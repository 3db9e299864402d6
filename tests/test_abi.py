"""The C-ABI library loads and exports every function include/*.h declares
(no compute calls: runs without a GPU), and the Python binding declares a
signature for each of them."""
import glob
import os
import re

from zbtest_util import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(hdr).read()
        names |= set(re.findall(r"\b(zb_\w+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_t"))


def test_every_declared_symbol_is_exported():
    from paper_2401_10241_b200 import _lib
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if getattr(_lib.lib, n, None) is None]
    assert not missing, missing
    unbound = [n for n in names if n not in _lib._SIGS]
    assert not unbound, unbound


def test_version_and_error_plumbing():
    from paper_2401_10241_b200 import _lib
    assert b"sm_100a" in _lib.lib.zb_version()
    # a failing call sets a message and returns a negative status
    rc = _lib.lib.zb_schedule(0, 1, 1, 1, 1, 0, 0, 1, 1, 0, None, 0, None)
    assert rc == _lib.ZB_EINVAL
    assert b"p" in _lib.lib.zb_last_error()


def test_arena_sizing_cpu_only():
    """zb_ctx_arena_bytes / zb_ctx_slot_bytes are pure host computations:
    slot bytes equal the stash layout of SURVEY §8(a) a6 (16 T h activations
    per layer + per-slot buffers)."""
    import zb_synth
    from paper_2401_10241_b200 import api
    cfg = zb_synth.CONFIGS["1.5B"]
    mc = api.model_cfg(cfg, 8, 3, cfg.m, 8, "bf16")
    sb = api.slot_bytes(mc)
    T, h, L = cfg.T, cfg.h, 3
    per_layer = 16 * T * h * 2 + 4 * T * 4 + cfg.a * T * 4
    # + per slot: received gradient in bf16 (GEMM operand) and f32 (residual chain)
    assert per_layer * L <= sb <= per_layer * L + T * h * (2 + 4) + 64 * 1024
    assert sb / 1e9 > 1.3     # SURVEY: c2 1.36 GB per slot per stage
    total = api.arena_bytes(mc)
    assert total > 8 * sb


def test_python_constants_match_the_header_enums():
    """Every ZB_* enum constant the binding re-declares (flags, kinds, families, status codes)
    has the header's value: the binding must not drift from include/zb.h."""
    from paper_2401_10241_b200 import _lib
    src = open(os.path.join(ROOT, "include", "zb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    header = {}
    for body in re.findall(r"enum\s*\{([^}]*)\}", src):
        for name, val in re.findall(r"\b(ZB_\w+)\s*=\s*(-?\d+)", body):
            header[name] = int(val)
    assert {"ZB_RUN_GRAPH", "ZB_RUN_GROUP_W", "ZB_EINVAL", "ZB_W"} <= set(header)
    checked = 0
    for name, val in header.items():
        if hasattr(_lib, name):
            assert getattr(_lib, name) == val, (name, getattr(_lib, name), val)
            checked += 1
    assert checked >= 8, checked
