"""The NCCL transport of libzb.so (comm.cu: zb_ctx_attach_nccl, zb_run_iteration over
2-rank communicators on per-channel streams, the post-validation chains, the
speculative warm-up F replay, zb_ctx_comm_probe) across REAL processes on one GPU:
libnccl is replaced by the CUDA-IPC shim (tests/shim/nccl_ipc.cu, ZB_NCCL_LIB) since
NCCL refuses two ranks on one device.  Every rank is a separate process driven
exactly as bench.py drives a GPU; the results must be BITWISE equal to the
virtual-stage runner (zb_run_iteration_local + zb_post_validate_local), which the
other GPU tests pin to the oracle.  The bench's multi-GPU code (run_pipeline /
run_pipeline_chunked) is run the same way on the tiny config."""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import zb_synth
from zbtest_util import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "shim", "libzbnccl_ipc.so")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _env(world, rank, port, **kw):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(port), ZB_NCCL_LIB=SHIM, ZB_SAME_DEVICE="1", ZB_DIST_BACKEND="gloo",
               ZB_LOOPBACK_TIMEOUT_S="120")
    env.update({k: str(v) for k, v in kw.items()})
    return env


def _run_ranks(world, **kw):
    out = tempfile.mkdtemp(prefix="zbshim")
    port = _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shim", "worker.py")],
                              env=_env(world, r, port, ZB_OUT=out, **kw), stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)[-4000:]
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(world)]


def _local_reference(world, family, dtype, iters, clip, opt_mode="pv"):
    import torch
    from paper_2401_10241_b200 import api
    cfg = zb_synth.ModelConfig("shim", h=128, a=2, L=4, s=256, b=2, V=512, p=world, m=5, family=family)
    passes, sim = api.schedule(family, world, cfg.m, 10, 11, 6, 0)
    ctxs = []
    for s in range(world):
        c = api.Context(cfg, world, s, cfg.m, max(1, sim.n_slots[s]), dtype=dtype)
        prm = zb_synth.make_stage_params(cfg, world, s)
        c.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, world, s)])
        ctxs.append(c)
    opt = api.optim_cfg(lr=1e-3, mode=opt_mode, clip=clip)
    for it in range(iters):
        tok = zb_synth.make_tokens(cfg, it)
        tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
        lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
        api.run_local(ctxs, passes, tin, lab)
        loss = ctxs[-1].loss()
        grads = [c.get_grads() for c in ctxs]
        api.post_validate_local(ctxs, opt)
    params = [c.get_params() for c in ctxs]
    moments = [c.get_moments() for c in ctxs]
    t = [c.pv_report()["t"] for c in ctxs]
    return loss, grads, params, moments, t


@pytest.mark.parametrize("family,dtype,clip", [("zbh1", "bf16", 1.0), ("zbh2", "f32", 1.0), ("1f1b", "bf16", 1.0),
                                               ("zbh1", "bf16", 0.05)])
def test_nccl_transport_two_processes_bitwise_equal_to_virtual_stages(family, dtype, clip):
    """clip 0.05: every iteration needs clipping -> stage 0 steps optimistically, the
    full state forces rollback + redo inside the NEXT iteration (after its speculative
    warm-up Fs, which are then replayed) — the whole P:153 protocol over the transport."""
    world, iters = 2, 3
    res = _run_ranks(world, ZB_FAMILY=family, ZB_DTYPE=dtype, ZB_ITERS=iters, ZB_CLIP=clip)
    loss, grads, params, moments, t = _local_reference(world, family, dtype, iters, clip)
    assert float(res[-1]["loss"]) == loss
    for r in range(world):
        n = len(grads[r])
        for i in range(n):
            assert np.array_equal(res[r][f"g{i}"], grads[r][i]), (r, i, "grad")
            assert np.array_equal(res[r][f"p{i}"], params[r][i]), (r, i, "param")
            assert np.array_equal(res[r][f"m{i}"], moments[r][0][i]), (r, i, "m")
            assert np.array_equal(res[r][f"v{i}"], moments[r][1][i]), (r, i, "v")
        assert int(res[r]["t"]) == t[r]
    assert int(res[0]["rt"]) > 0 and int(res[-1]["rt"]) == 0


def test_nccl_transport_three_stages_sync_optimizer():
    world, iters = 3, 2
    res = _run_ranks(world, ZB_FAMILY="zbh1", ZB_DTYPE="bf16", ZB_ITERS=iters, ZB_CLIP=1.0, ZB_OPT="sync")
    loss, grads, params, _, _ = _local_reference(world, "zbh1", "bf16", iters, 1.0, opt_mode="sync")
    assert float(res[-1]["loss"]) == loss
    for r in range(world):
        for i in range(len(grads[r])):
            assert np.array_equal(res[r][f"g{i}"], grads[r][i])
            assert np.array_equal(res[r][f"p{i}"], params[r][i])


@pytest.mark.parametrize("family", ["zbh1", "zbv"])
def test_bench_multi_gpu_code_path_under_the_shim(family):
    """bench.py --gpus 2 (torchrun, one process per stage) on the tiny config: the
    multi-GPU bench code runs end to end and prints the measured bubble, the 1F1B
    comparison and the PV-vs-sync ablation (numbers meaningless on one shared GPU)."""
    port = _port()
    env = dict(os.environ, ZB_NCCL_LIB=SHIM, ZB_SAME_DEVICE="1", ZB_DIST_BACKEND="gloo", ZB_BENCH_WATCHDOG_S="500")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--config", "tiny", "--family", family]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    if family == "zbh1":
        assert d["bubble"]["measured_scheduling"] is not None
        assert d["vs_1f1b"]["speedup"] is not None and d["pv_vs_sync"]["speedup_pv"] is not None
        assert len(d["profile"]["T_F_ns"]) == 2 and d["profile"]["T_comm_ns"] > 0
