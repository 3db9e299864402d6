"""Worker plans of chunked schedules (ZB-V P:318-324, 1F1B-I P:193): the op list
comm.cu's worker runner executes (plan.h worker_plan — every chunk's
per-virtual-stage plan merged in the worker's pass order), checked on CPU:

* an interpreter steps all workers (one op list each) with FIFO channels per
  virtual link (activations v -> v+1, gradients v+1 -> v): every receive gets
  the microbatch its plan expects, the passes of each worker run in exactly
  the order zb_schedule_chunked emitted, and the run completes (no deadlock);
* the same plans across processes with gloo (one process per worker; links
  inside a worker — ZB-V's v = p-1 -> p turn — stay in-process).
"""
import collections
import multiprocessing as mp
import os
import socket
import traceback

import pytest

try:
    from paper_2401_10241_b200 import api
    LIB = True
except ImportError:
    LIB = False

pytestmark = pytest.mark.skipif(not LIB, reason="libzb.so not built")
RECV_ACT, SEND_ACT, RECV_GRAD, SEND_GRAD = 3, 4, 5, 6
KIND = {0: "F", 1: "B", 2: "W"}


def _sched(family, p, m, chunks):
    passes, _ = api.schedule_chunked(family, p, m, chunks, 10, 11, 6, 1, M_B=3, M_W=3)
    nv = chunks * p
    per = 3 * chunks * m
    worker_of = [0] * nv
    for i in range(len(passes)):
        worker_of[passes[i].stage] = i // per
    return passes, nv, worker_of


def _link(op, v):
    """(channel key, peer virtual stage) of a communication op of chunk v."""
    t = op[0]
    if t == SEND_ACT:
        return ("act", v, v + 1)
    if t == RECV_ACT:
        return ("act", v - 1, v)
    if t == SEND_GRAD:
        return ("grad", v, v - 1)
    return ("grad", v + 1, v)


CASES = [("zbv", 2, 3, 2), ("zbv", 4, 8, 2), ("zbv", 4, 5, 2), ("zbv", 8, 24, 2), ("zbv", 3, 9, 2),
         ("1f1bi", 2, 4, 2), ("1f1bi", 4, 8, 2), ("1f1bi", 4, 12, 3), ("1f1bi", 8, 16, 2)]


@pytest.mark.parametrize("family,p,m,chunks", CASES, ids=[f"{c[0]}-p{c[1]}-m{c[2]}-c{c[3]}" for c in CASES])
def test_worker_plans_interpret(family, p, m, chunks):
    passes, nv, worker_of = _sched(family, p, m, chunks)
    fused = family == "1f1bi"
    plans = [api.worker_plan(passes, nv, m, w, worker_of, fused) for w in range(p)]
    # the compute ops of each worker, in order, are exactly its scheduled passes
    per = 3 * chunks * m
    for w in range(p):
        got = [(KIND[t], c, j) for (t, j, _, _, c) in plans[w] if t in (0, 1, 2)]
        want = [(KIND[q.kind], q.stage, q.microbatch) for q in passes[w * per:(w + 1) * per]]
        assert got == want
    queues = collections.defaultdict(collections.deque)
    pos = [0] * p
    seen_b0 = set()
    while any(pos[w] < len(plans[w]) for w in range(p)):
        progressed = False
        for w in range(p):
            while pos[w] < len(plans[w]):
                t, j, msg, slot, v = plans[w][pos[w]]
                if t in (RECV_ACT, RECV_GRAD):
                    key = _link((t,), v)
                    if not queues[key]:
                        break
                    jj = queues[key].popleft()
                    assert jj == j, (family, w, v, t, j, jj)
                elif t in (SEND_ACT, SEND_GRAD):
                    queues[_link((t,), v)].append(j)
                elif t == 1 and v == 0:
                    seen_b0.add(j)
                pos[w] += 1
                progressed = True
        assert progressed, f"deadlock at {pos}"
    assert seen_b0 == set(range(m))
    assert all(not q for q in queues.values())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, family, m, chunks, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        passes, nv, worker_of = _sched(family, world, m, chunks)
        plan = api.worker_plan(passes, nv, m, rank, worker_of, family == "1f1bi")
        local = collections.defaultdict(collections.deque)
        sends = []
        b0 = []
        for (t, j, msg, slot, v) in plan:
            if t in (SEND_ACT, SEND_GRAD):
                key = _link((t,), v)
                dst = worker_of[key[2]]
                if dst == rank:
                    local[key].append(j)
                else:   # tag = link id: 2 * lower virtual stage (+1 for gradients)
                    tag = 2 * min(key[1], key[2]) + (1 if key[0] == "grad" else 0)
                    sends.append(dist.isend(torch.tensor([j], dtype=torch.int64), dst=dst, tag=tag))
            elif t in (RECV_ACT, RECV_GRAD):
                key = _link((t,), v)
                src = worker_of[key[1]]
                if src == rank:
                    jj = local[key].popleft()
                else:
                    buf = torch.zeros(1, dtype=torch.int64)
                    dist.recv(buf, src=src, tag=2 * min(key[1], key[2]) + (1 if key[0] == "grad" else 0))
                    jj = int(buf[0])
                assert jj == j, (rank, v, t, j, jj)
            elif t == 1 and v == 0:
                b0.append(j)
        for r in sends:
            r.wait()
        dist.barrier()
        q.put((rank, "ok", b0))
    except Exception:
        q.put((rank, "err", traceback.format_exc()))


@pytest.mark.parametrize("family,world,m", [("zbv", 2, 4), ("zbv", 4, 8), ("1f1bi", 4, 8)])
def test_worker_plans_gloo(family, world, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, family, m, 2, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    try:
        for _ in range(world):
            rank, status, payload = q.get(timeout=120)
            res[rank] = (status, payload)
    finally:
        for pr in procs:
            pr.join(timeout=10)
            if pr.is_alive():
                pr.kill()
    errs = {r: v[1] for r, v in res.items() if v[0] != "ok"}
    assert not errs, errs
    assert sorted(res[0][1]) == list(range(m))      # v = 0 lives on worker 0 in both placements
