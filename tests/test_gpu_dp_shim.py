"""Data parallelism (App. A) across real processes on
one GPU: D = 2 replicas of a p-stage pipeline, every rank its own process, libnccl replaced
by the CUDA-IPC shim (tests/shim/nccl_ipc.cu, ZB_NCCL_LIB; its 2-rank ncclAllReduce adds
a + b on rank 0 and b + a on rank 1, the same bits).  Checks:
* the replicas hold bitwise-identical gradients after the iteration and identical
  parameters after the post-validated steps;
* the gradients equal the fp64 oracle over all D m microbatches (f32 parity mode, 1e-5):
  the all-reduce sums the replicas' microbatch ranges and the loss mean runs over T m D;
* App. A's per-parameter reordering of the tail Ws changes only WHEN each all-reduce
  starts, not the sums (bitwise equal to the W-major order);
* one all-reduce per W unit plus the vector region per iteration."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import zb_synth
from oracle import model as om
from zbtest_util import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "shim", "libzbnccl_ipc.so")
M = 4


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(D, p, **kw):
    out = tempfile.mkdtemp(prefix="zbdp")
    port = _port()
    world = D * p
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), ZB_NCCL_LIB=SHIM, ZB_OUT=out, ZB_DP=str(D), ZB_PP=str(p), ZB_M=str(M))
        env.update({k: str(v) for k, v in kw.items()})
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shim", "worker_dp.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for q in procs:
        try:
            o, _ = q.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for x in procs:
                x.kill()
            raise
        logs.append(o)
    assert all(q.returncode == 0 for q in procs), "\n".join(logs)[-4000:]
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(world)]


def _oracle(p):
    cfg = zb_synth.ModelConfig("dp", h=128, a=2, L=4, s=256, b=2, V=512, p=p, m=2 * M, family="zbh1")
    return om.reference_iteration(cfg, zb_synth.make_model_params(cfg), zb_synth.make_tokens(cfg, 0)), cfg


@pytest.mark.parametrize("p,family", [(1, "zbh1"), (2, "zbh1"), (2, "1f1b")])
def test_dp_two_replicas_match_oracle_and_each_other(p, family):
    D = 2
    res = _run(D, p, ZB_FAMILY=family, ZB_DTYPE="f32", ZB_ITERS=2, ZB_DP_REORDER=1)
    (ref_loss, ref), cfg = _oracle(p)
    for s in range(p):
        a, b = res[s], res[p + s]   # replica 0 / 1 of stage s
        specs = zb_synth.param_specs(cfg, p, s)
        for i, (name, shape, _) in enumerate(specs):
            assert np.array_equal(a[f"g{i}"], b[f"g{i}"]), (s, name, "replica grads differ")
            assert np.array_equal(a[f"p{i}"], b[f"p{i}"]), (s, name, "replica params differ")
            g, r = a[f"g{i}"].reshape(shape), ref[name]
            err = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
            assert err <= 1e-5, (s, name, err)
        n_units = int(a["n_units"])
        assert int(a["reduces"]) == 2 * (n_units + 1), (int(a["reduces"]), n_units)   # per iteration
    loss = sum(float(res[r * p + p - 1]["loss"]) for r in range(D))   # each replica's share of the mean
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss), (loss, ref_loss)


def test_dp_reordered_tail_is_bitwise_equal_to_w_major_order():
    kw = dict(ZB_FAMILY="zbh1", ZB_DTYPE="bf16", ZB_ITERS=2)
    a = _run(2, 2, ZB_DP_REORDER=1, **kw)
    b = _run(2, 2, ZB_DP_REORDER=0, **kw)
    for ra, rb in zip(a, b):
        keys = [k for k in ra if k.startswith(("g", "p"))]
        assert keys and all(np.array_equal(ra[k], rb[k]) for k in keys)


def test_dp_grouped_tail_within_tolerance():
    """ZB_RUN_GROUP_W with the reordered tail: each parameter's tail contributions form one
    multi-segment contraction (different f32 grouping: tolerance, not bits)."""
    a = _run(2, 1, ZB_FAMILY="zbh1", ZB_DTYPE="bf16", ZB_ITERS=1, ZB_DP_REORDER=1, ZB_GROUP_W=1)
    b = _run(2, 1, ZB_FAMILY="zbh1", ZB_DTYPE="bf16", ZB_ITERS=1, ZB_DP_REORDER=1, ZB_GROUP_W=0)
    for ra, rb in zip(a, b):
        for k in ra:
            if k.startswith("g"):
                err = np.linalg.norm(ra[k] - rb[k]) / max(np.linalg.norm(rb[k]), 1e-30)
                assert err <= 1e-3, (k, err)


def test_bench_dp_code_path_under_the_shim():
    """bench.py --gpus 2 --dp 2 (two replicas of a 1-stage pipeline, one process each, on
    one GPU through the shim): the data-parallel bench path runs end to end and prints the
    App. A ablation (numbers meaningless on one shared GPU)."""
    import json
    port = _port()
    env = dict(os.environ, ZB_NCCL_LIB=SHIM, ZB_SAME_DEVICE="1", ZB_DIST_BACKEND="gloo", ZB_BENCH_WATCHDOG_S="500")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dp", "2",
           "--steps", "2", "--warmup", "3", "--config", "tiny"]
    q = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert q.returncode == 0, q.stdout[-3000:] + q.stderr[-3000:]
    lines = [x for x in q.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, q.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "pp1dp2"
    assert d["dp"]["speedup_app_a"] is not None
