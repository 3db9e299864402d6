#!/usr/bin/env python
"""bench.py — Zero Bubble Pipeline Parallelism hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl zb|reference]
                    [--config 6.2B|1.5B|...] [--family ...] [--opt pv|sync]

A step is one training iteration of a BASELINE.json workload: the GPT-style model
(seq 1024, V 50304) over m microbatches, scheduled over p = N pipeline stages (one
per GPU; at N = 1 one stage holds all layers), bf16 operands / f32 accumulation,
followed by the post-validated AdamW step.  Synthetic seeded data and weights
(zb_synth).  The headline at N = 1 is configs[2] — 6.2B (h 4096, 32 heads, 30 layers,
b 3, m 32, ZB-H2), the largest config that fits one GPU; configs[1] (1.5B, b 6,
m 24, ZB-H1) is measured in the same run and nested under "second_config".
Rank 0 prints ONE JSON line.

Profiling: warm-up iterations are timed per pass
(zb_ctx_profile, median int64 ns) and the timed schedule is built from those
measured times (zb_schedule_per_stage); at N > 1 every stage contributes its own
T's and T_comm is measured by a P2P ping-pong of one boundary message.

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
SECOND = {"6.2B": "1.5B", "1.5B": "6.2B"}


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

def _oracle_layer_seconds(cfg):
    """One transformer layer F + B + W (oracle layer math) on ONE sequence at the
    config's width."""
    import numpy as np
    from oracle import model as om
    one = cfg.with_(b=1, L=1, m=1)
    params = zb_synth.make_model_params(one)
    x = np.random.default_rng(0).standard_normal((one.T, one.h)) * 0.5
    lp = {k[len("l0."):]: v.astype(np.float64) for k, v in params.items() if k.startswith("l0.")}
    t1 = time.perf_counter()
    y, cache = om.layer_forward(x, lp, 1, one.s, one.a)
    dx, ws = om.layer_backward_input(np.ones_like(y) * 1e-3, cache, lp, 1, one.s, one.a)
    om.layer_backward_weight(ws)
    return time.perf_counter() - t1


def _oracle_edges_seconds(cfg):
    """Embedding + LM head + loss (forward and backward) of ONE sequence: a full
    oracle iteration of a 1-layer, 1-sequence model minus one layer."""
    from oracle import model as om
    one = cfg.with_(b=1, L=1, m=1)
    params = zb_synth.make_model_params(one)
    tok = zb_synth.make_tokens(one, 0, m=1)
    t0 = time.perf_counter()
    om.reference_iteration(one, params, tok)
    total = time.perf_counter() - t0
    return max(total - _oracle_layer_seconds(cfg), 0.0)


def _oracle_full_iteration_seconds(cfg):
    from oracle import model as om
    params = zb_synth.make_model_params(cfg)
    tok = zb_synth.make_tokens(cfg, 0)
    t0 = time.perf_counter()
    om.reference_iteration(cfg, params, tok)
    return time.perf_counter() - t0


def oracle_extrapolation_check():
    """SURVEY §8(d) / BASELINE.md: validate the per-layer extrapolation with FULL timed
    oracle iterations — configs[0] (tiny, 8 layers, m 8) and a 2-layer, m = 2, b = 1
    truncation of configs[1] (1.5B width) — against L * t_layer + t_edges per sequence."""
    out = {}
    for name, cfg in (("c1_tiny_full", zb_synth.CONFIGS["tiny"]),
                      ("c2_1.5B_L2_m2_b1", zb_synth.CONFIGS["1.5B"].with_(L=2, m=2, b=1))):
        t_layer = _oracle_layer_seconds(cfg)
        t_edges = _oracle_edges_seconds(cfg)
        predicted = cfg.m * cfg.b * (cfg.L * t_layer + t_edges)
        measured = _oracle_full_iteration_seconds(cfg)
        out[name] = {"predicted_s": round(predicted, 3), "measured_s": round(measured, 3),
                     "measured_over_predicted": round(measured / predicted, 4) if predicted else None}
    return out


def oracle_sample(cfg, t_edges=None):
    """Bounded sample of the oracle on the workload: one layer F+B+W on one sequence
    (the steps) plus the embedding/head edges (once); tokens/s extrapolated as
    T_seq / (L * t_layer + t_edges)."""
    t_layer = _oracle_layer_seconds(cfg)
    if t_edges is None:
        t_edges = _oracle_edges_seconds(cfg)
    t_seq = cfg.L * t_layer + t_edges
    return cfg.s / t_seq, dict(t_layer_s=round(t_layer, 3), t_edges_s=round(t_edges, 3), tokens_per_sequence=cfg.s)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = zb_synth.CONFIGS[args.config]
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.environ.get("OMP_NUM_THREADS", os.cpu_count())))
    t0 = time.perf_counter()
    t_edges = _oracle_edges_seconds(cfg)
    layer_s = []
    step_ms = []
    for i in range(args.warmup + args.steps):
        s0 = time.perf_counter()
        t = _oracle_layer_seconds(cfg)
        if i >= args.warmup:
            layer_s.append(t)
            step_ms.append((time.perf_counter() - s0) * 1e3)
    t_layer = statistics.median(layer_s)
    value = cfg.s / (cfg.L * t_layer + t_edges)
    check = oracle_extrapolation_check() if not args.no_validate else None
    sample = (f"oracle (numpy fp64): each step = one {cfg.name} layer F+B+W on one {cfg.s}-token sequence; "
              f"embedding + LM head timed once; tokens/s extrapolated to {cfg.L} layers x {cfg.b * cfg.m} sequences")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(step_ms),
            "ms_per_step_is": "wall time of one bounded sample (one layer, one sequence), not of an iteration",
            "extrapolated": True,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args.gpus, args.family),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle", "sample": sample,
                             "extrapolated": True,
                             "detail": {"t_layer_s": round(t_layer, 3), "t_edges_s": round(t_edges, 3),
                                        "wall_s": round(time.perf_counter() - t0, 1)},
                             "extrapolation_check": check},
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
    ap.add_argument("--config", default="6.2B")
    ap.add_argument("--second-config", default=None, help="N = 1: config measured after the headline ('none' = skip)")
    ap.add_argument("--family", default=None)
    ap.add_argument("--opt", default="pv", choices=["pv", "sync"])
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N = 1: launch every kernel eagerly instead of replaying the iteration's CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-validate", action="store_true", help="reference arm: skip the extrapolation check")
    ap.add_argument("--no-profile-p8", action="store_true")
    ap.add_argument("--dp", type=int, default=1,
                    help="data-parallel replicas (SURVEY §8(f)4): p = gpus / dp stages each, the global batch "
                         "(m microbatches) split over the replicas, gradient all-reduces with App. A reordering")
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
    torch.cuda.set_device(0 if os.environ.get("ZB_SAME_DEVICE") == "1" else local)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dp > 1 and (world % args.dp or cfg.m % args.dp or args.family in ("zbv", "1f1bi")):
        raise SystemExit("--dp must divide --gpus and m (and is not for the chunked families)")
    if world > 1:
        _start_watchdog(rank)
        if args.family in ("zbv", "1f1bi"):
            return run_pipeline_chunked(args, cfg, rank, world, local)
        return run_pipeline(args, cfg, rank, world, local)
    if args.family in ("zbv", "1f1bi"):
        raise SystemExit("--family zbv / 1f1bi needs --gpus >= 2 (two model chunks per GPU)")
    line = run_single(args, cfg, headline=True)
    second = args.second_config if args.second_config is not None else SECOND.get(args.config)
    if second and second != "none" and args.m is None and args.family == cfg.family:
        torch.cuda.empty_cache()
        c2 = zb_synth.CONFIGS[second]
        a2 = argparse.Namespace(**vars(args))
        a2.family = c2.family
        a2.no_cpu_baseline = True
        line["second_config"] = run_single(a2, c2, headline=False)
    print(json.dumps(line), flush=True)


def _start_watchdog(rank):
    """Multi-GPU runs only: a hang in the NCCL exchange ends the process with a
    message instead of holding the node until the driver's own limit
    (ZB_BENCH_WATCHDOG_S, default 1200 s)."""
    import threading
    limit = float(os.environ.get("ZB_BENCH_WATCHDOG_S", "1200"))

    def fire():
        sys.stderr.write(f"bench.py rank {rank}: no result after {limit:.0f} s (watchdog), exiting\n")
        sys.stderr.flush()
        os._exit(3)

    t = threading.Timer(limit, fire)
    t.daemon = True
    t.start()


def _mem_limit(cfg, family, p, slot_b):
    """AUTO's memory rule of the config (BASELINE: c4 M_limit = 1F1B peak = p M_B,
    c5 2x): per-stage activation budget in bytes."""
    return cfg.mem_factor * p * slot_b if family == "auto" else 0


def run_single(args, cfg, headline=True):
    """N = 1: one stage holding every layer.  Returns the JSON line (dict)."""
    import numpy as np
    import torch
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import lib
    import ctypes as C  # noqa: F811

    p = 1
    m = cfg.m
    mc = api.model_cfg(cfg, p, 0, m, 1, "bf16")
    slot_b = api.slot_bytes(mc)
    lim = _mem_limit(cfg, args.family, p, slot_b)
    # provisional schedule (unit times) only sizes the stash; the timed schedule comes from
    # the profiled pass times below
    passes, sim = api.schedule(args.family, p, m, 1, 1, 1, 0, M_limit=lim, M_B=slot_b, M_W=slot_b)
    n_slots = max(1, sim.n_slots[0]) if args.family != "auto" else max(1, lim // slot_b)
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, 0, m, n_slots, dtype="bf16", stream=stream)
    params = zb_synth.make_stage_params(cfg, p, 0)
    ctx.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, 0)])
    del params
    n_steps = args.warmup + args.steps
    toks = [zb_synth.make_tokens(cfg, i) for i in range(n_steps)]
    tok_h = [np.ascontiguousarray(t[..., :cfg.s]) for t in toks]
    lab_h = [np.ascontiguousarray(t[..., 1:]) for t in toks]
    tok_d = [torch.from_numpy(t).cuda() for t in tok_h]
    lab_d = [torch.from_numpy(t).cuda() for t in lab_h]
    opt = api.optim_cfg(lr=1e-4, mode=args.opt, clip=1.0)
    sched = {"passes": passes}

    graph = not args.no_graph  # ZB_RUN_GRAPH: captured once, replayed (eager while kernel timing is on)

    def step(i, host=False, timing=False):
        q = sched["passes"]
        if host:
            ctx.run_iteration(q, tok_pin[i], lab_pin[i], host_inputs=True, timing=timing, graph=graph)
        else:
            ctx.run_iteration(q, tok_d[i], lab_d[i], timing=timing, graph=graph)
        ctx.post_validate_step(opt)
        ctx.post_validate_finish(opt)

    # ---- warm-up: profiling iterations (per-pass CUDA events), then the schedule from the
    # measured medians (zb_ctx_profile -> zb_schedule_per_stage)
    torch.cuda.synchronize()
    ctx.profile(reset=True)
    for i in range(args.warmup):
        step(i, timing=True)
        ctx.profile()
    t_ns, n_samp = ctx.profile()
    passes, sim = api.schedule_per_stage(args.family, p, m, [t_ns[0]], [t_ns[1]], [t_ns[2]], 0, M_limit=lim,
                                         M_B=slot_b, M_W=slot_b)
    if max(1, sim.n_slots[0]) > n_slots:
        raise SystemExit("profiled schedule needs more stash slots than allocated")
    sched["passes"] = passes
    step(0)
    step(1 % n_steps)  # graph mode: the first call with the final pass list runs eagerly, this one captures
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
    loss = ctx.loss()
    # ---- the same workload again with CUDA events around every GEMM / attention / HBM-kernel
    # launch (on the launching stream) for the per-kernel-class roofline
    k_steps = min(args.steps, 5)
    lib.zb_dbg_kernel_timing(1, 1)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev2.record(stream)
    for i in range(args.warmup, args.warmup + k_steps):
        step(i)
    ev3.record(stream)
    torch.cuda.synchronize()
    lib.zb_dbg_kernel_timing(0, 0)
    ms_ev = ev2.elapsed_time(ev3) / k_steps
    kstats = {}
    for cls, name in ((0, "gemm"), (3, "gemm_F"), (4, "gemm_B"), (5, "gemm_W"), (1, "attn_fwd"), (2, "attn_bwd")):
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        lib.zb_dbg_kernel_timing_read(cls, C.byref(a), C.byref(b), C.byref(n))
        kstats[name] = {"ms_total": a.value / k_steps, "tflops": (b.value / (a.value / 1e3) / 1e12) if a.value else 0,
                        "launches_per_step": n.value / k_steps,
                        "share_of_step": (a.value / k_steps) / ms_ev if ms_ev else 0}
    hbm = hbm_classes(lib, k_steps, ms_ev)
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
        for i in range(args.warmup, args.warmup + k_steps):
            step(i, host=True)
            ctx.loss()          # D2H of the step's result
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / k_steps
        e2e = {"value": tokens_per_step / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(tok_h[0].nbytes + lab_h[0].nbytes), "d2h_bytes_per_step": 8,
               "ms_per_step": e_ms, "steps": k_steps,
               "wall_ms_per_step": (time.perf_counter() - t0) * 1000.0 / k_steps}
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
    # ---- size context for the HBM classes: a same-size copy's bandwidth per launch
    for v in hbm["classes"].values():
        if v.get("launches_per_step") and v.get("bytes_per_step"):
            cg = same_size_copy_gbs(v["bytes_per_step"] / v["launches_per_step"])
            v["bytes_per_launch"] = round(v["bytes_per_step"] / v["launches_per_step"])
            v["same_size_copy_gbs"] = round(cg, 1)
            v["frac_of_same_size_copy"] = round(v["gbs"] / cg, 4) if cg else None
    torch.cuda.empty_cache()
    # ---- roofline of the dominant kernel (the GEMM family)
    peaks, src = read_peaks()
    g = kstats["gemm"]
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    roof = {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (F/B/W, all launches)",
            "achieved": round(g["tflops"], 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(g["tflops"] / peak, 4) if peak else None, "traffic": None,
            "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)",
            "timing": f"CUDA events around every launch over a second region of {k_steps} steps "
                      f"({ms_ev:.1f} ms/step with the events)",
            "per_class": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in kstats.items()},
            "hbm_kernels": hbm}
    roof["traffic"], roof["traffic_source"] = gemm_traffic(cfg.name)
    accounted = sum(v["ms_total"] for k, v in kstats.items() if k in ("gemm", "attn_fwd", "attn_bwd")) + \
        sum(v["ms_total"] for v in hbm["classes"].values())
    roof["unaccounted_ms_per_step"] = round(ms_ev - accounted, 3)
    # the same against the value region's step (CUDA-graph replay, no per-launch events): the
    # per-class times are measured with events around every launch (eager), which inflate each
    # bracketed kernel, so a value near or below 0 means no time is left outside the kernels
    roof["value_region_minus_kernels_ms_per_step"] = round(ms - accounted, 3)
    roof["unaccounted_note"] = ("unaccounted_ms_per_step: eager timing region minus the event-timed classes "
                                "(mostly the events' own cost); value_region_minus_kernels: the graph-replayed "
                                "step minus the same class times")
    flops_token = cfg.L * (72 * cfg.h ** 2 + 12 * cfg.s * cfg.h) + 6 * cfg.h * cfg.V
    mfu = value * flops_token / (peaks.get("bf16_tflops", 1680.3) * 1e12)
    line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (zb_synth seeded weights and tokens)",
            "config": dict(workload_config(cfg, 1, args.family), optimizer=f"AdamW, {args.opt}",
                           launch="one CUDA graph per iteration (ZB_RUN_GRAPH), optimizer eager" if graph
                           else "eager"),
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "model_flops_utilization": round(mfu, 4), "loss": loss,
            "profile": {"T_ns": {"F": t_ns[0], "B": t_ns[1], "W": t_ns[2]}, "samples": n_samp,
                        "schedule_from": "zb_schedule_per_stage on the profiled medians (P:169)"}}
    if not args.no_profile_p8:
        line["bubble_p8_predicted"] = profile_p8(cfg, stream)
    if headline and not args.no_cpu_baseline:
        v, info = oracle_sample(cfg)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                                "sample": f"one {cfg.name} layer F+B+W on one {cfg.s}-token sequence + embedding/"
                                          f"head once, extrapolated to {cfg.L} layers",
                                "extrapolated": True, "detail": info}
    return line


def profile_p8(cfg, stream, reps=4):
    """PAPER.md §5.3 / P:169: per-stage T_F, T_B, T_W of the paper's p = 8 partition,
    measured on real stage contexts (stage 0 with the embedding, a middle stage, the
    last stage with LN_f + LM head) through the pass API with CUDA events (median of
    `reps` microbatches after one warm-up), then every schedule family simulated on
    those per-stage times (zb_schedule_per_stage / zb_schedule_chunked), T_comm = the
    P2P time of one [T, h] f32 gradient message at the measured NVLink rate
    (ZB_TCOMM_US, default 20 us)."""
    import numpy as np
    import torch
    from paper_2401_10241_b200 import api
    p = 8
    parts = api.partition(cfg.L, p)
    tcomm_us = int(os.environ.get("ZB_TCOMM_US", "20"))
    per_stage = {}
    slot_b = {}
    for s in sorted({0, 1, p - 1}):
        ctx = api.Context(cfg, p, s, reps + 1, 1, dtype="bf16", stream=stream)
        prm = zb_synth.make_stage_params(cfg, p, s)
        ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
        del prm
        slot_b[s] = api.slot_bytes(ctx.mc)
        tok = zb_synth.make_tokens(cfg, 0, m=1)
        t = torch.from_numpy(np.ascontiguousarray(tok[0, ..., :cfg.s])).cuda()
        lab = torch.from_numpy(np.ascontiguousarray(tok[0, ..., 1:])).cuda()
        g = torch.Generator(device="cuda").manual_seed(s)
        x_in = (torch.randn(cfg.T, cfg.h, device="cuda", generator=g) * 0.5).bfloat16()
        act_out = torch.empty(cfg.T, cfg.h, device="cuda", dtype=torch.bfloat16)
        dy = torch.randn(cfg.T, cfg.h, device="cuda", generator=g) * 1e-4
        dx = torch.empty(cfg.T, cfg.h, device="cuda")
        torch.cuda.synchronize()
        out = {"F": [], "B": [], "W": []}
        ctx.begin_iteration()
        for r in range(reps + 1):
            calls = (("F", lambda: ctx.forward(r, 0, t.data_ptr() if s == 0 else x_in.data_ptr(),
                                               act_out.data_ptr() if s < p - 1 else None,
                                               lab.data_ptr() if s == p - 1 else None)),
                     ("B", lambda: ctx.backward_input(r, 0, dy.data_ptr() if s < p - 1 else None,
                                                      dx.data_ptr() if s > 0 else None)),
                     ("W", lambda: ctx.backward_weight(r, 0)))
            for k, fn in calls:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                torch.cuda.synchronize()
                if r >= 1:
                    out[k].append(e0.elapsed_time(e1))
        per_stage[s] = {k: int(round(float(np.median(v)) * 1000)) for k, v in out.items()}   # us
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    Ts = [per_stage[0]] + [per_stage[1]] * (p - 2) + [per_stage[p - 1]]
    TF, TB, TW = ([x[k] for x in Ts] for k in "FBW")
    mb = slot_b[1]
    res = {"p": p, "layers_per_stage": parts, "T_comm_us": tcomm_us, "M_B_bytes_mid_stage": mb,
           "T_us": {"stage0": per_stage[0], "middle": per_stage[1], "last": per_stage[p - 1]},
           "method": "stage contexts of the p = 8 partition timed per pass (CUDA events, median), "
                     "families simulated on the per-stage times (zb_schedule_per_stage)"}
    for fam in ("1f1b", "zbh1", "zbh2"):
        if fam == "zbh2" and cfg.m < 2 * p - 1:
            continue
        _, sim = api.schedule_per_stage(fam, p, cfg.m, TF, TB, TW, tcomm_us)
        res[fam] = round(sim.bubble_rate, 4)
    for f in (1, 2):
        _, sim = api.schedule_per_stage("auto", p, cfg.m, TF, TB, TW, tcomm_us, M_limit=f * p * mb, M_B=mb, M_W=mb)
        res[f"auto_{f}pMB"] = round(sim.bubble_rate, 4)
    # ZB-V: two chunks of half a middle stage per worker, per-chunk times
    half = {k: per_stage[1][k] // 2 for k in "FBW"}
    _, sim = api.schedule_chunked("zbv", p, cfg.m, 2, half["F"], half["B"], half["W"], tcomm_us)
    res["zbv"] = round(sim.bubble_rate, 4)
    res["ratios_middle"] = {"T_B/T_F": round(per_stage[1]["B"] / per_stage[1]["F"], 3),
                            "T_W/T_F": round(per_stage[1]["W"] / per_stage[1]["F"], 3)}
    return res


HBM_CLASSES = ((6, "ln_fwd"), (7, "ln_bwd_dx"), (8, "ln_param_grads"), (9, "bias_grads"), (10, "cross_entropy"),
               (11, "optimizer"), (12, "embed_convert"))


def hbm_classes(lib, steps, ms_ev):
    """Per-class CUDA-event totals of the HBM-bound kernels (ktimer classes 6-12:
    algorithmic bytes / time) against the measured copy bandwidth.  The optimizer
    class counts the grad-norm read (4 B/param) and the step that runs (28 B/param +
    2 B per bf16 shadow element); the validation launch of post-validation, which is
    predicated off on a clean step, is reported separately with its time only."""
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
                     "frac": round(gbs / peak, 4) if peak else None, "bytes_per_step": b.value / steps,
                     "launches_per_step": n.value / steps, "share_of_step": round((a.value / steps) / ms_ev, 4)}
    a, b, n = C.c_double(), C.c_double(), C.c_int64()
    lib.zb_dbg_kernel_timing_read(13, C.byref(a), C.byref(b), C.byref(n))
    if n.value:
        out["optimizer_validation"] = {"ms_total": round(a.value / steps, 4), "launches_per_step": n.value / steps,
                                       "note": "post-validation launch, predicated off on clean steps (no bytes)"}
    return {"unit": "GB/s (algorithmic bytes / event time)", "peak": peak, "peak_source": f"{src} hbm_gbs",
            "classes": out}


def same_size_copy_gbs(nbytes, iters=20):
    """Bandwidth of a torch device copy moving the same bytes per launch as an HBM-class
    kernel (half read, half written; rotating over buffers larger than L2): the achievable
    rate for a transfer of that size, reported beside the fraction of the 2 GB-copy peak."""
    import torch
    half = max(1 << 20, min(int(nbytes // 2), 1 << 30))
    nb = max(2, -(-(320 << 20) // half))
    src = [torch.empty(half, dtype=torch.uint8, device="cuda") for _ in range(nb)]
    dst = [torch.empty(half, dtype=torch.uint8, device="cuda") for _ in range(nb)]
    for i in range(3):
        dst[i % nb].copy_(src[i % nb])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(iters):
        dst[i % nb].copy_(src[i % nb])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    del src, dst
    return 2 * half / (ms / 1e3) / 1e9


def gemm_traffic(model):
    """DRAM bytes per GEMM launch from the committed ncu capture (profiles/), if any."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "gemm_dram_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        d = d[model] if model in d else (d if d.get("model", "1.5B") == model else None)
        if d is None:
            return None, None
        return d["dram_bytes_per_launch"], d["source"]
    except (OSError, KeyError, ValueError, AttributeError):
        return None, None


def dist_setup(local):
    """torch.distributed plumbing: NCCL across GPUs; ZB_DIST_BACKEND=gloo (with
    ZB_SAME_DEVICE=1 and ZB_NCCL_LIB = the 2-process / 1-GPU shim) runs N stages as N
    processes on ONE device (tests/test_gpu_nccl_shim.py) — then the small collectives
    of the bench move CPU tensors."""
    import torch
    import torch.distributed as dist
    backend = os.environ.get("ZB_DIST_BACKEND", "nccl")
    dev = 0 if os.environ.get("ZB_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        return "cuda"
    dist.init_process_group(backend)
    return "cpu"


def run_pipeline(args, cfg, rank, world, local):
    """p = N stages, one per GPU, NCCL P2P (zb_ctx_attach_nccl).  Times are
    taken on each rank with CUDA events and the MAX over ranks is reported."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2401_10241_b200 import api
    from paper_2401_10241_b200._lib import lib
    import ctypes as C

    cdev = dist_setup(local)
    D = args.dp                              # data-parallel replicas (1: pipeline only)
    p, m = world // D, cfg.m // D            # stages per replica, microbatches per replica
    rep, rank = divmod(rank, p)              # replica, stage (rank below = the stage)
    grank = rep * p + rank
    # every process creates every group in the same order
    pgroups = [dist.new_group(list(range(r * p, r * p + p))) for r in range(D)] if D > 1 else [None]
    pg = pgroups[rep]                        # this replica's pipeline
    mc = api.model_cfg(cfg, p, rank, m, 1, "bf16")
    sb = torch.tensor([api.slot_bytes(mc)], device=cdev, dtype=torch.int64)
    dist.all_reduce(sb, op=dist.ReduceOp.MAX)
    slot_b = int(sb.item())
    lim = _mem_limit(cfg, args.family, p, slot_b)
    # provisional schedule (unit times): sizes the stash and drives the profiling iterations
    passes, sim = api.schedule(args.family, p, m, 1, 1, 1, 0, M_limit=lim, M_B=slot_b, M_W=slot_b)
    p1f, s1f = api.schedule("1f1b", p, m, 1, 1, 1, 0)
    n_slots = max(1, sim.n_slots[rank], s1f.n_slots[rank])
    if args.family == "auto":
        n_slots = max(n_slots, lim // slot_b)
    ids = [([api.nccl_unique_ids(2 * (p - 1)) if p > 1 else b"" for _ in range(D)],
            [api.nccl_unique_ids(1) for _ in range(p)] if D > 1 else None) if grank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, rank, m, n_slots, dtype="bf16", stream=stream)
    params = zb_synth.make_stage_params(cfg, p, rank)
    ctx.set_params([params[n] for n, _, _ in zb_synth.param_specs(cfg, p, rank)])
    del params
    if p > 1:
        ctx.attach_nccl(ids[0][0][rep], rank, p)
    if D > 1:   # the stage's replicas sum their gradients (App. A reordered tail)
        ctx.attach_dp(ids[0][1][rank], rep, D)
    n_steps = args.warmup + args.steps
    toks = [zb_synth.make_tokens(cfg, i)[rep * m:(rep + 1) * m] for i in range(n_steps)]
    tok_d = [torch.from_numpy(np.ascontiguousarray(t[..., :cfg.s])).cuda() for t in toks]
    lab_d = [torch.from_numpy(np.ascontiguousarray(t[..., 1:])).cuda() for t in toks]
    opt = api.optim_cfg(lr=1e-4, mode=args.opt, clip=1.0)
    opt_other = api.optim_cfg(lr=1e-4, mode="sync" if args.opt == "pv" else "pv", clip=1.0)

    tok_pin = [torch.from_numpy(np.ascontiguousarray(t[..., :cfg.s])).pin_memory().numpy() for t in toks]
    lab_pin = [torch.from_numpy(np.ascontiguousarray(t[..., 1:])).pin_memory().numpy() for t in toks]
    fused_main = args.family == "1f1b"

    dp_reorder = D > 1

    def run(family_passes, fused, steps, first, timing=False, host=False, o=None):
        o = o or opt
        for i in range(first, first + steps):
            if host:   # e2e: pinned host inputs copied inside the call, loss read back every step
                ctx.run_iteration(family_passes, tok_pin[i % n_steps] if rank == 0 else None,
                                  lab_pin[i % n_steps] if rank == p - 1 else None, host_inputs=True, fused=fused,
                                  dp_reorder=dp_reorder)
            else:
                ctx.run_iteration(family_passes, tok_d[i % n_steps] if rank == 0 else None,
                                  lab_d[i % n_steps] if rank == p - 1 else None, timing=timing, fused=fused,
                                  dp_reorder=dp_reorder)
            ctx.post_validate_step(o)
            if host and rank == p - 1:
                ctx.loss()

    def timed(family_passes, fused, host=False, steps=None, o=None):
        o = o or opt
        steps = steps or args.steps
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(family_passes, fused, steps, args.warmup, host=host, o=o)
        ctx.post_validate_finish(o)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    # ---- profiling warm-up: per-pass times of every stage + T_comm, then the schedule
    ctx.profile(reset=True)
    for i in range(args.warmup):
        run(passes, fused_main, 1, i, timing=True)
        ctx.post_validate_finish(opt)
        ctx.profile()
    t_ns, _ = ctx.profile()
    mine = torch.tensor(t_ns, device=cdev, dtype=torch.int64)
    allT = [torch.zeros_like(mine) for _ in range(p)]
    dist.all_gather(allT, mine, group=pg)
    TF, TB, TW = ([int(x[k]) for x in allT] for k in range(3))
    # T_comm: one f32 [T, h] boundary-gradient message, round trip / 2, max over pairs (zb_ctx_comm_probe)
    rt = torch.tensor([ctx.comm_probe(4 * cfg.T * cfg.h, 10)], device=cdev, dtype=torch.int64)
    dist.all_reduce(rt, op=dist.ReduceOp.MAX)
    tcomm = int(rt.item()) // 2
    passes, sim = api.schedule_per_stage(args.family, p, m, TF, TB, TW, tcomm, M_limit=lim, M_B=slot_b, M_W=slot_b)
    if max(1, sim.n_slots[rank]) > n_slots:
        raise SystemExit("profiled schedule needs more stash slots than allocated")
    run(passes, fused_main, 1, 0)
    ctx.post_validate_finish(opt)
    torch.cuda.synchronize()
    nl = C.c_int64()
    lib.zb_dbg_launch_count(1, C.byref(nl))
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms = timed(passes, fused_main)
    lib.zb_dbg_launch_count(0, C.byref(nl))
    nlt = torch.tensor([nl.value], device=cdev, dtype=torch.int64)
    dist.all_reduce(nlt)                       # kernels launched by all ranks
    tokens_per_step = cfg.T * m * D          # all replicas
    value = tokens_per_step / (ms / 1000.0)
    k_steps = min(args.steps, 5)
    # per-kernel-class timing over a second region (roofline)
    lib.zb_dbg_kernel_timing(1, 1)
    ms_ev = timed(passes, fused_main, steps=k_steps)
    lib.zb_dbg_kernel_timing(0, 0)
    a, b, n = C.c_double(), C.c_double(), C.c_int64()
    lib.zb_dbg_kernel_timing_read(0, C.byref(a), C.byref(b), C.byref(n))
    gt = torch.tensor([a.value, b.value], device=cdev, dtype=torch.float64)
    dist.all_reduce(gt)                        # GEMM ms and FLOPs summed over ranks
    # e2e: host inputs through the public call, loss read back every step
    e2e_ms = timed(passes, fused_main, host=True, steps=k_steps)
    # measured per-stage busy / span of one iteration (scheduling bubble)
    run(passes, fused_main, 1, 0, timing=True)
    ctx.post_validate_finish(opt)
    starts, ends = ctx.stats()
    busy = sum(e - s for s, e in zip(starts, ends))
    span = ends[-1] - starts[0] if starts else 0.0
    stat = torch.tensor([busy, span], device=cdev)
    gathered = [torch.zeros_like(stat) for _ in range(p)]
    dist.all_gather(gathered, stat, group=pg)
    busys = [float(g[0]) for g in gathered]
    spans = [float(g[1]) for g in gathered]
    cost = max(spans)
    _, sim_pred = api.schedule_per_stage(args.family, p, m, TF, TB, TW, tcomm, M_limit=lim, M_B=slot_b, M_W=slot_b)
    bubble = {"measured_scheduling": (cost - max(busys)) / cost if cost else None,
              "imbalance": 1 - (sum(busys) / len(busys)) / max(busys) if busys else None,
              "stage_busy_ms": busys, "stage_span_ms": spans, "predicted_from_profile": sim_pred.bubble_rate}
    # 1F1B on the same kernels ("vs 1F1B"), same profiled times
    p1, s1 = api.schedule_per_stage("1f1b", p, m, TF, TB, TW, tcomm)
    ms_1f1b = None
    if args.family != "1f1b" and s1.n_slots[rank] <= n_slots:
        run(p1, True, 1, 0)
        ctx.post_validate_finish(opt)
        ms_1f1b = timed(p1, True)
    # post-validation vs the synchronous all-reduce-style optimizer (Table 7 ablation)
    run(passes, fused_main, 1, 0, o=opt_other)
    ctx.post_validate_finish(opt_other)
    ms_other = timed(passes, fused_main, o=opt_other)
    ms_noreorder = None
    if D > 1:   # App. A ablation: the tail Ws in their W-major order (all-reduces start late)
        dp_reorder = False
        run(passes, fused_main, 1, 0)
        ctx.post_validate_finish(opt)
        ms_noreorder = timed(passes, fused_main)
        dp_reorder = True
    if grank == 0:
        peaks, src = read_peaks()
        flops_token = cfg.L * (72 * cfg.h ** 2 + 12 * cfg.s * cfg.h) + 6 * cfg.h * cfg.V
        g_tf = float(gt[1]) / (float(gt[0]) / 1e3) / 1e12 if float(gt[0]) else 0.0
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        roof = {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (F/B/W, all launches, all ranks)",
                "achieved": round(g_tf, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(g_tf / peak, 4) if peak else None, "traffic": None,
                "peak_source": f"{src} bf16_tflops_sustained",
                "timing": f"CUDA events around every GEMM launch over a second region of {k_steps} steps "
                          f"({ms_ev:.1f} ms/step max over ranks with the events)",
                "share_of_step": round(float(gt[0]) / p / k_steps / ms_ev, 4) if ms_ev else None}
        roof["traffic"], roof["traffic_source"] = gemm_traffic(cfg.name)
        e2e = {"value": tokens_per_step / (e2e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(2 * m * D * cfg.T * 4), "d2h_bytes_per_step": 8 * D, "ms_per_step": e2e_ms,
               "steps": k_steps}
        pv_ms, sync_ms = (ms, ms_other) if args.opt == "pv" else (ms_other, ms)
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": p, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (zb_synth seeded weights and tokens)",
                "config": dict(workload_config(cfg, p, args.family), optimizer=f"AdamW, {args.opt}"),
                "clocks": clk.summary(), "e2e": e2e,
                "gpu_launches": int(nlt.item()), "roofline": roof,
                "bubble": bubble,
                "profile": {"T_F_ns": TF, "T_B_ns": TB, "T_W_ns": TW, "T_comm_ns": tcomm,
                            "schedule_from": "zb_schedule_per_stage on the profiled per-stage medians (P:169)"},
                "vs_1f1b": {"tokens_per_s_1f1b": tokens_per_step / (ms_1f1b / 1000.0) if ms_1f1b else None,
                            "speedup": ms_1f1b / ms if ms_1f1b else None},
                "pv_vs_sync": {"ms_per_step_pv": pv_ms, "ms_per_step_sync": sync_ms,
                               "speedup_pv": sync_ms / pv_ms if pv_ms else None},
                "model_flops_utilization": round(value * flops_token / (p * D * peaks.get("bf16_tflops", 1680.3) * 1e12), 4)}
        if D > 1:
            line["n_gpus"] = p * D
            line["config"].update(parallelism=f"pp{p}dp{D}", replicas=D, microbatches_per_replica=m)
            line["dp"] = {"replicas": D, "ms_per_step_app_a": ms, "ms_per_step_w_major_tail": ms_noreorder,
                          "speedup_app_a": ms_noreorder / ms if ms_noreorder else None,
                          "note": "gradient all-reduce per W unit on a side stream; App. A reorders the tail Ws "
                                  "per parameter (P:452-454)"}
        print(json.dumps(line), flush=True)
    dist.barrier()
    ctx.close()
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

    cdev = dist_setup(local)
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
    opt = api.optim_cfg(lr=1e-4, mode=args.opt, clip=1.0)

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
    with ClockSampler(torch.cuda.current_device()) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(args.steps, args.warmup)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=cdev)
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
    for c in ctxs:
        c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
