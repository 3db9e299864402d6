#!/usr/bin/env python
"""bench.py — Zero Bubble Pipeline Parallelism hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl zb|reference]

A step is one training iteration of BASELINE.json's configs[1] workload: the
GPT-style 1.5B model (h 2304, 24 heads, 22 layers, seq 1024), microbatch 6,
m = 24 microbatches, scheduled ZB-H1 over p = N pipeline stages (one per GPU;
at N = 1 one stage holds all 22 layers), bf16 operands / f32 accumulation,
followed by the post-validated AdamW step.  Synthetic seeded data and weights
(zb_synth).  Prints ONE JSON line on rank 0.

The reference arm (--impl reference) times the fp64 CPU oracle (oracle/) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import zb_synth  # noqa: E402

METRIC = "tokens/s per box (training iterations, ZB pipeline schedule)"


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except Exception:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- reference arm (CPU oracle)

def oracle_sample(cfg, seconds_hint=True):
    """Time the oracle on a bounded sample: one transformer layer F+B+W and the
    LM head + embedding for ONE sequence (1024 tokens) at the config's width;
    extrapolate tokens/s = tokens / (L * t_layer + t_edges)."""
    import numpy as np
    from oracle import model as om
    one = cfg.with_(b=1, L=1)
    params = zb_synth.make_model_params(one)
    tok = zb_synth.make_tokens(one, 0, m=1)
    st = om.Stage(one, 1, 0, params, 1)
    t0 = time.perf_counter()
    st.forward(0, tok[0, :, :one.s], tok[0, :, 1:])
    st.backward_input(0)
    st.backward_weight(0)
    t_total = time.perf_counter() - t0
    # split: time the layer alone
    x = np.random.default_rng(0).standard_normal((one.T, one.h)) * 0.5
    lp = {k[len("l0."):]: v.astype(np.float64) for k, v in params.items() if k.startswith("l0.")}
    t1 = time.perf_counter()
    y, cache = om.layer_forward(x, lp, 1, one.s, one.a)
    dx, ws = om.layer_backward_input(np.ones_like(y) * 1e-3, cache, lp, 1, one.s, one.a)
    om.layer_backward_weight(ws)
    t_layer = time.perf_counter() - t1
    t_edges = max(t_total - t_layer, 0.0)
    t_seq = cfg.L * t_layer + t_edges
    return one.T / t_seq, dict(t_layer_s=round(t_layer, 3), t_edges_s=round(t_edges, 3), tokens=one.T,
                               work_s=round(t_total + t_layer, 3))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    cfg = zb_synth.CONFIGS[args.config]
    cores = os.cpu_count()
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        v, info = oracle_sample(cfg)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    sample = (f"oracle (numpy fp64) one {cfg.name} layer F+B+W + head/embedding on 1 x {cfg.s} tokens, "
              f"extrapolated to {cfg.L} layers")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg.T * cfg.m / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args.gpus, args.family),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "detail": info},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, n, family):
    return {"workload": f"GPT {cfg.name} ({cfg.L} layers, h {cfg.h}, {cfg.a} heads, seq {cfg.s}), "
                        f"microbatch {cfg.b}, m={cfg.m}, {family.upper()} over p={n} stage(s)",
            "model": cfg.name, "global_batch": cfg.b * cfg.m, "seq_len": cfg.s, "microbatch": cfg.b,
            "microbatches": cfg.m, "stages": n, "schedule": family, "parallelism": f"pp{n}",
            "l2": "inputs larger than L2 (weights alone 3+ GB bf16)"}


# --------------------------------------------------------------------------- our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="zb", choices=["zb", "reference"])
    ap.add_argument("--config", default="1.5B")
    ap.add_argument("--family", default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = zb_synth.CONFIGS[args.config]
    if args.m:
        cfg = cfg.with_(m=args.m)
    args.family = args.family or cfg.family
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        _start_watchdog(rank)
        if args.family in ("zbv", "1f1bi"):
            return run_pipeline_chunked(args, cfg, rank, world, local)
        return run_pipeline(args, cfg, rank, world, local)
    if args.family in ("zbv", "1f1bi"):
        raise SystemExit("--family zbv / 1f1bi needs --gpus >= 2 (two model chunks per GPU)")
    return run_single(args, cfg)


def _start_watchdog(rank):
    """Multi-GPU runs only: the NCCL P2P path cannot be exercised on the one-GPU
    development boxes, so a hang there ends the process with a message instead of
    holding the node until the driver's own limit (ZB_BENCH_WATCHDOG_S, default 1200 s)."""
    import threading
    limit = float(os.environ.get("ZB_BENCH_WATCHDOG_S", "1200"))

    def fire():
        sys.stderr.write(f"bench.py rank {rank}: no result after {limit:.0f} s (watchdog), exiting\n")
        sys.stderr.flush()
        os._exit(3)

    t = threading.Timer(limit, fire)
    t.daemon = True
    t.start()


def run_single(args, cfg):
    import numpy as np
    import torch
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import lib
    import ctypes as C  # noqa: F811

    p = 1
    m = cfg.m
    passes, sim = api.schedule(args.family, p, m, 10, 10, 10, 0, M_limit=0 if args.family != "auto" else 10,
                               M_B=10, M_W=10)
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, 0, m, max(1, sim.n_slots[0]), dtype="bf16", stream=stream)
    params = zb_synth.make_stage_params(cfg, p, 0)
    ctx.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, 0)])
    del params
    n_steps = args.warmup + args.steps
    toks = [zb_synth.make_tokens(cfg, i) for i in range(n_steps)]
    tok_h = [np.ascontiguousarray(t[..., :cfg.s]) for t in toks]
    lab_h = [np.ascontiguousarray(t[..., 1:]) for t in toks]
    tok_d = [torch.from_numpy(t).cuda() for t in tok_h]
    lab_d = [torch.from_numpy(t).cuda() for t in lab_h]
    opt = api.optim_cfg(lr=1e-4, mode="pv", clip=1.0)

    def step(i, host=False, timing=False):
        if host:
            ctx.run_iteration(passes, tok_pin[i], lab_pin[i], host_inputs=True, timing=timing)
        else:
            ctx.run_iteration(passes, tok_d[i], lab_d[i], timing=timing)
        ctx.post_validate_step(opt)
        ctx.post_validate_finish(opt)

    torch.cuda.synchronize()
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # ---- device-resident timed region (value): no per-kernel events inside
    nl = C.c_int64()
    lib.zb_dbg_launch_count(1, C.byref(nl))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.warmup, n_steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    lib.zb_dbg_launch_count(0, C.byref(nl))
    launches = int(nl.value)
    ms = ev0.elapsed_time(ev1) / args.steps
    tokens_per_step = cfg.T * m
    value = tokens_per_step / (ms / 1000.0)
    # ---- the same K steps again with CUDA events around every GEMM / attention
    # launch (on the launching stream) for the per-kernel-class roofline
    lib.zb_dbg_kernel_timing(1, 1)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev2.record(stream)
    for i in range(args.warmup, n_steps):
        step(i)
    ev3.record(stream)
    torch.cuda.synchronize()
    lib.zb_dbg_kernel_timing(0, 0)
    ms_ev = ev2.elapsed_time(ev3) / args.steps
    kstats = {}
    for cls, name in ((0, "gemm"), (3, "gemm_F"), (4, "gemm_B"), (5, "gemm_W"), (1, "attn_fwd"), (2, "attn_bwd")):
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        lib.zb_dbg_kernel_timing_read(cls, C.byref(a), C.byref(b), C.byref(n))
        kstats[name] = {"ms_total": a.value / args.steps, "tflops": (b.value / (a.value / 1e3) / 1e12) if a.value else 0,
                        "launches_per_step": n.value / args.steps,
                        "share_of_step": (a.value / args.steps) / ms_ev if ms_ev else 0}
    hbm = hbm_classes(lib, args.steps, ms_ev)
    loss = ctx.loss()
    # ---- per-pass times -> predicted bubbles at p=8 (Table 8 analog on B200)
    step(args.warmup, timing=True)
    starts, ends = ctx.stats()
    torch.cuda.synchronize()
    durs = {"F": [], "B": [], "W": []}
    for q, s0, s1 in zip(list(passes), starts, ends):
        durs["FBW"[q.kind]].append(s1 - s0)
    t_pass = {k: statistics.median(v) for k, v in durs.items()}
    bubble = predicted_bubbles(cfg, t_pass)
    # ---- end-to-end through the C-ABI with host buffers (e2e)
    e2e = None
    if not args.no_e2e:
        tok_pin = [torch.from_numpy(t).pin_memory().numpy() for t in tok_h]
        lab_pin = [torch.from_numpy(t).pin_memory().numpy() for t in lab_h]
        step(0, host=True)
        ctx.loss()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.warmup, n_steps):
            step(i, host=True)
            ctx.loss()          # D2H of the step's result
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.steps
        e2e = {"value": tokens_per_step / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(tok_h[0].nbytes + lab_h[0].nbytes), "d2h_bytes_per_step": 8,
               "ms_per_step": e_ms, "wall_ms_per_step": (time.perf_counter() - t0) * 1000.0 / args.steps}
    # ---- roofline of the dominant kernel (the GEMM family)
    peaks, src = read_peaks()
    g = kstats["gemm"]
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    roof = {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (F/B/W, all launches)",
            "achieved": round(g["tflops"], 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(g["tflops"] / peak, 4) if peak else None, "traffic": None,
            "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)",
            "timing": f"CUDA events around every launch over a second region of the same {args.steps} steps "
                      f"({ms_ev:.1f} ms/step with the events)",
            "per_class": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in kstats.items()},
            "hbm_kernels": hbm}
    roof["traffic"], roof["traffic_source"] = gemm_traffic()
    accounted = sum(v["ms_total"] for k, v in kstats.items() if k in ("gemm", "attn_fwd", "attn_bwd")) + \
        sum(v["ms_total"] for v in hbm["classes"].values())
    roof["unaccounted_ms_per_step"] = round(ms_ev - accounted, 3)
    flops_token = cfg.L * (72 * cfg.h ** 2 + 12 * cfg.s * cfg.h) + 6 * cfg.h * cfg.V
    mfu = value * flops_token / (peaks.get("bf16_tflops", 1680.3) * 1e12)
    line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (zb_synth seeded weights and tokens)",
            "config": workload_config(cfg, 1, args.family),
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "model_flops_utilization": round(mfu, 4), "loss": loss,
            "bubble": bubble, "pass_ms": t_pass}
    if not args.no_cpu_baseline:
        v, info = oracle_sample(cfg)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                                "sample": f"one {cfg.name} layer F+B+W + head on {cfg.s} tokens, extrapolated",
                                "detail": info}
    print(json.dumps(line), flush=True)


HBM_CLASSES = ((6, "ln_fwd"), (7, "ln_bwd_dx"), (8, "ln_param_grads"), (9, "bias_grads"), (10, "cross_entropy"),
               (11, "optimizer"), (12, "embed_convert"))


def hbm_classes(lib, steps, ms_ev):
    """Per-class CUDA-event totals of the HBM-bound kernels (ktimer classes 6-12:
    algorithmic bytes / time) against the measured copy bandwidth."""
    peaks, src = read_peaks()
    peak = peaks.get("hbm_gbs")
    out = {}
    for cls, name in HBM_CLASSES:
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        lib.zb_dbg_kernel_timing_read(cls, C.byref(a), C.byref(b), C.byref(n))
        if not n.value:
            continue
        gbs = b.value / (a.value / 1e3) / 1e9 if a.value else 0.0
        out[name] = {"ms_total": round(a.value / steps, 4), "gbs": round(gbs, 1),
                     "frac": round(gbs / peak, 4) if peak else None,
                     "launches_per_step": n.value / steps, "share_of_step": round((a.value / steps) / ms_ev, 4)}
    return {"unit": "GB/s (algorithmic bytes / event time)", "peak": peak, "peak_source": f"{src} hbm_gbs",
            "classes": out}


def gemm_traffic():
    """DRAM bytes per GEMM launch from the committed ncu capture (profiles/), if any."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "gemm_dram_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["dram_bytes_per_launch"], d["source"]
    except (OSError, KeyError, ValueError):
        return None, None


def predicted_bubbles(cfg, t_pass):
    """Feed measured per-pass times (scaled from one all-layer stage to the
    paper's p = 8 partition) to the simulator: predicted bubble rates of 1F1B,
    ZB-H1, ZB-H2 at p = 8 for this workload (§5.3 method)."""
    from paper_2401_10241_b200 import api
    p = 8
    per_layer = {k: v / cfg.L for k, v in t_pass.items()}
    Lmid = (cfg.L + 2) // p
    us = {k: int(round(per_layer[k] * Lmid * 1000)) for k in "FBW"}
    out = {"p": p, "layers_per_stage": Lmid, "T_us": us}
    for fam in ("1f1b", "zbh1", "zbh2"):
        if fam == "zbh2" and cfg.m < 2 * p - 1:
            continue
        _, sim = api.schedule(fam, p, cfg.m, us["F"], us["B"], us["W"], 20)
        out[fam] = round(sim.bubble_rate, 4)
    # chunked schedules on the same per-layer times: ZB-V (2 chunks of Lmid/2 layers) and
    # 1F1B-I with one layer per chunk (the Table 4 baseline); per-chunk pass times
    half = {k: per_layer[k] * Lmid / 2 * 1000 for k in "FBW"}
    _, sim = api.schedule_chunked("zbv", p, cfg.m, 2, int(round(half["F"])), int(round(half["B"])),
                                  int(round(half["W"])), 20)
    out["zbv"] = round(sim.bubble_rate, 4)
    if cfg.m % p == 0:
        one = {k: int(round(per_layer[k] * 1000)) for k in "FBW"}
        _, sim = api.schedule_chunked("1f1bi", p, cfg.m, Lmid, one["F"], one["B"], one["W"], 20)
        out["1f1bi"] = round(sim.bubble_rate, 4)
    out["measured_p1"] = 0.0
    return out


def run_pipeline(args, cfg, rank, world, local):
    """p = N stages, one per GPU, NCCL P2P (zb_ctx_attach_nccl).  Times are
    taken on each rank with CUDA events and the MAX over ranks is reported."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import lib
    import ctypes as C

    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, m = world, cfg.m
    mc = api.model_cfg(cfg, p, rank, m, 1, "bf16")
    slot_b = api.slot_bytes(mc)
    passes, sim = api.schedule(args.family, p, m, 10, 10, 10, 0,
                               M_limit=(cfg.mem_factor * p * slot_b if args.family == "auto" else 0),
                               M_B=slot_b, M_W=slot_b)
    ids = [api.nccl_unique_ids(2 * (p - 1)) if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, rank, m, max(1, sim.n_slots[rank]), dtype="bf16", stream=stream)
    params = zb_synth.make_stage_params(cfg, p, rank)
    ctx.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, rank)])
    del params
    ctx.attach_nccl(ids[0], rank, p)
    n_steps = args.warmup + args.steps
    toks = [zb_synth.make_tokens(cfg, i) for i in range(n_steps)]
    tok_d = [torch.from_numpy(np.ascontiguousarray(t[..., :cfg.s])).cuda() for t in toks]
    lab_d = [torch.from_numpy(np.ascontiguousarray(t[..., 1:])).cuda() for t in toks]
    opt = api.optim_cfg(lr=1e-4, mode="pv", clip=1.0)

    tok_pin = [torch.from_numpy(np.ascontiguousarray(t[..., :cfg.s])).pin_memory().numpy() for t in toks]
    lab_pin = [torch.from_numpy(np.ascontiguousarray(t[..., 1:])).pin_memory().numpy() for t in toks]

    def run(family_passes, fused, steps, first, timing=False, host=False):
        for i in range(first, first + steps):
            if host:   # e2e: pinned host inputs copied inside the call, loss read back every step
                ctx.run_iteration(family_passes, tok_pin[i % n_steps] if rank == 0 else None,
                                  lab_pin[i % n_steps] if rank == p - 1 else None, host_inputs=True, fused=fused)
            else:
                ctx.run_iteration(family_passes, tok_d[i % n_steps] if rank == 0 else None,
                                  lab_d[i % n_steps] if rank == p - 1 else None, timing=timing, fused=fused)
            ctx.post_validate_step(opt)
            if host and rank == p - 1:
                ctx.loss()

    def timed(family_passes, fused, host=False):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(family_passes, fused, args.steps, args.warmup, host=host)
        ctx.post_validate_finish(opt)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    run(passes, False, args.warmup, 0)
    ctx.post_validate_finish(opt)
    torch.cuda.synchronize()
    nl = C.c_int64()
    lib.zb_dbg_launch_count(1, C.byref(nl))
    with ClockSampler(local) as clk:
        ms = timed(passes, False)
    lib.zb_dbg_launch_count(0, C.byref(nl))
    nlt = torch.tensor([nl.value], device="cuda", dtype=torch.int64)
    dist.all_reduce(nlt)                       # kernels launched by all ranks
    tokens_per_step = cfg.T * m
    value = tokens_per_step / (ms / 1000.0)
    # per-kernel-class timing over a second region of the same steps (roofline)
    lib.zb_dbg_kernel_timing(1, 1)
    ms_ev = timed(passes, False)
    lib.zb_dbg_kernel_timing(0, 0)
    a, b, n = C.c_double(), C.c_double(), C.c_int64()
    lib.zb_dbg_kernel_timing_read(0, C.byref(a), C.byref(b), C.byref(n))
    gt = torch.tensor([a.value, b.value], device="cuda", dtype=torch.float64)
    dist.all_reduce(gt)                        # GEMM ms and FLOPs summed over ranks
    # e2e: host inputs through the public call, loss read back every step
    e2e_ms = timed(passes, False, host=True)
    # measured per-stage busy / span of one iteration (scheduling bubble)
    run(passes, False, 1, 0, timing=True)
    ctx.post_validate_finish(opt)
    starts, ends = ctx.stats()
    busy = sum(e - s for s, e in zip(starts, ends))
    span = ends[-1] - starts[0] if starts else 0.0
    stat = torch.tensor([busy, span], device="cuda")
    gathered = [torch.zeros_like(stat) for _ in range(p)]
    dist.all_gather(gathered, stat)
    busys = [float(g[0]) for g in gathered]
    spans = [float(g[1]) for g in gathered]
    cost = max(spans)
    bubble = {"measured_scheduling": (cost - max(busys)) / cost if cost else None,
              "imbalance": 1 - (sum(busys) / len(busys)) / max(busys) if busys else None,
              "stage_busy_ms": busys, "stage_span_ms": spans, "predicted": sim.bubble_rate}
    # 1F1B on the same kernels ("vs 1F1B")
    p1, s1 = api.schedule("1f1b", p, m, 10, 10, 10, 0)
    ms_1f1b = None
    if args.family != "1f1b" and s1.n_slots[rank] <= max(1, sim.n_slots[rank]):
        run(p1, True, 1, 0)
        ctx.post_validate_finish(opt)
        ms_1f1b = timed(p1, True)
    if rank == 0:
        peaks, src = read_peaks()
        flops_token = cfg.L * (72 * cfg.h ** 2 + 12 * cfg.s * cfg.h) + 6 * cfg.h * cfg.V
        g_tf = float(gt[1]) / (float(gt[0]) / 1e3) / 1e12 if float(gt[0]) else 0.0
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        roof = {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (F/B/W, all launches, all ranks)",
                "achieved": round(g_tf, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(g_tf / peak, 4) if peak else None, "traffic": None,
                "peak_source": f"{src} bf16_tflops_sustained",
                "timing": f"CUDA events around every GEMM launch over a second region of {args.steps} steps "
                          f"({ms_ev:.1f} ms/step max over ranks with the events)",
                "share_of_step": round(float(gt[0]) / p / args.steps / ms_ev, 4) if ms_ev else None}
        e2e = {"value": tokens_per_step / (e2e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(2 * m * cfg.T * 4), "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms}
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": p, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (zb_synth seeded weights and tokens)",
                "config": workload_config(cfg, p, args.family), "clocks": clk.summary(), "e2e": e2e,
                "gpu_launches": int(nlt.item()), "roofline": roof,
                "bubble": bubble,
                "vs_1f1b": {"tokens_per_s_1f1b": tokens_per_step / (ms_1f1b / 1000.0) if ms_1f1b else None,
                            "speedup": ms_1f1b / ms if ms_1f1b else None},
                "model_flops_utilization": round(value * flops_token / (p * peaks.get("bf16_tflops", 1680.3) * 1e12), 4)}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_pipeline_chunked(args, cfg, rank, world, local):
    """ZB-V / 1F1B-I over N GPUs (section 6): two model chunks per GPU (virtual
    stages v of 2N, V placement for ZB-V, cyclic for 1F1B-I), NCCL links between GPUs
    and an in-process link for ZB-V's turn (zb_ctx_attach_nccl_chunks), each GPU running
    its merged pass list (zb_run_iteration_worker); max-over-ranks CUDA-event timing."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2401_10241_b200 import api

    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, m, chunks = world, cfg.m, 2
    nv = chunks * p
    fused = args.family == "1f1bi"
    slot_b = api.slot_bytes(api.model_cfg(cfg, nv, 1, m, 1, "bf16"))
    passes, sim = api.schedule_chunked(args.family, p, m, chunks, 10, 10, 10, 0, M_B=slot_b, M_W=slot_b)
    per = 3 * chunks * m
    worker_of = [0] * nv
    for i in range(len(passes)):
        worker_of[passes[i].stage] = i // per
    mine = [v for v in range(nv) if worker_of[v] == rank]
    ids = [api.nccl_unique_ids(2 * (nv - 1)) if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    stream = torch.cuda.Stream()
    ctxs = []
    for v in mine:
        c = api.Context(cfg, nv, v, m, max(1, sim.n_slots[v]), dtype="bf16", stream=stream)
        params = zb_synth.make_stage_params(cfg, nv, v)
        c.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, nv, v)])
        del params
        ctxs.append(c)
    api.attach_nccl_chunks(ctxs, ids[0], nv, worker_of, rank)
    n_steps = args.warmup + args.steps
    toks = [zb_synth.make_tokens(cfg, i) for i in range(n_steps)]
    tok_d = [torch.from_numpy(np.ascontiguousarray(t[..., :cfg.s])).cuda() for t in toks]
    lab_d = [torch.from_numpy(np.ascontiguousarray(t[..., 1:])).cuda() for t in toks]
    opt = api.optim_cfg(lr=1e-4, mode="pv", clip=1.0)

    def run(steps, first):
        for i in range(first, first + steps):
            api.run_worker(ctxs, passes, tok_d[i % n_steps] if 0 in mine else None,
                           lab_d[i % n_steps] if nv - 1 in mine else None, fused=fused)
            for c in sorted(ctxs, key=lambda c: c.stage):      # partial chain: ascending v
                c.post_validate_step(opt)
            for c in sorted(ctxs, key=lambda c: -c.stage):     # full chain: descending v
                c.post_validate_finish(opt)

    run(args.warmup, 0)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(args.steps, args.warmup)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t)
    value = cfg.T * m / (ms / 1000.0)
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": p, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (zb_synth seeded weights and tokens)",
                "config": dict(workload_config(cfg, p, args.family), chunks_per_gpu=chunks),
                "clocks": clk.summary(), "e2e": None, "roofline": None,
                "bubble": {"predicted": sim.bubble_rate}}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
