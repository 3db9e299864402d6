"""Multi-process (gloo, CPU) test of the P2P protocol the NCCL runner executes.

Each rank asks libzb.so for its stage plan (zb_dbg_stage_plan: the exact op
sequence comm.cu runs) for two iterations — the second with a pending
post-validation whose outcome does or does not amend the weights —
and executes it with torch.distributed send / recv: tag 0 = activation
channel (s -> s+1), tag 1 = gradient channel (s+1 -> s).  Messages carry
(microbatch, code) where code accumulates, stage by stage, the weight version
each forward used.  Checks: every receive gets the microbatch the plan
expects (message matching and the replay index mapping), stale speculative
messages are drained, no rank deadlocks, and every gradient that reaches
stage 0 in iteration 2 was computed from forwards that used the validated
weights on every stage.
"""
import ctypes as C
import multiprocessing as mp
import os
import socket
import traceback

import pytest

try:
    from paper_2401_10241_b200 import api  # noqa: F401
    LIB = True
except ImportError:
    LIB = False

pytestmark = pytest.mark.skipif(not LIB, reason="libzb.so not built")

ACT, GRAD = 0, 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan(passes, p, m, stage, pending, amend, fused):
    from paper_2401_10241_b200._lib import lib, check
    cap = 64 * p * m + 64
    buf = (C.c_int32 * (4 * cap))()
    n = C.c_int32()
    check(lib.zb_dbg_stage_plan(passes, len(passes), p, m, stage, int(pending), int(amend), int(fused), buf, cap,
                                C.byref(n)))
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n.value)]


def _worker(rank, world, port, family, m, amend, fused, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2401_10241_b200 import api
        p = world
        passes, _ = api.schedule(family, p, m, 10, 11, 6, 1, M_limit=2 * p * 3 if family == "auto" else 0,
                                 M_B=3, M_W=3)
        pending_sends = []

        def send(j, code, dst, tag):
            pending_sends.append(dist.isend(torch.tensor([j, code], dtype=torch.int64), dst=dst, tag=tag))

        def recv(src, tag):
            t = torch.zeros(2, dtype=torch.int64)
            dist.recv(t, src=src, tag=tag)
            return int(t[0]), int(t[1])

        weight = 1          # version of this stage's weights during iteration 1
        out_code, grad_code, final_grads = {}, {}, {}
        for it, (pending, am) in enumerate(((False, False), (True, amend))):
            inputs = {}
            for (typ, j, msg, slot) in _plan(passes, p, m, rank, pending, am, fused):
                if typ == 3:       # RECV_ACT
                    jj, code = recv(rank - 1, ACT)
                    assert jj == j, (rank, it, "act mismatch", j, jj, msg)
                    inputs[j] = code
                elif typ == 8:     # DISCARD_ACT (stale speculative message)
                    jj, code = recv(rank - 1, ACT)
                    assert am and code % 10 == 2, ("discarded a non-stale message", rank, jj, code)
                elif typ in (0, 9):  # F / REPLAY_F
                    base = 0 if rank == 0 else inputs[j]
                    out_code[j] = base * 10 + weight
                elif typ == 4:     # SEND_ACT
                    send(j, out_code[j], rank + 1, ACT)
                elif typ == 5:     # RECV_GRAD
                    jj, code = recv(rank + 1, GRAD)
                    assert jj == j, (rank, it, "grad mismatch", j, jj)
                    grad_code[j] = code
                elif typ == 1:     # B: the gradient carries the last stage's forward code
                    grad_code[j] = out_code[j] if rank == p - 1 else grad_code[j]
                    if it == 1:
                        final_grads[j] = grad_code[j]
                elif typ == 6:     # SEND_GRAD
                    send(j, grad_code[j], rank - 1, GRAD)
                elif typ == 2:     # W
                    pass
                elif typ == 7:     # VALIDATE: full state from stage+1, forwarded to stage-1
                    if rank < p - 1:
                        jj, code = recv(rank + 1, GRAD)
                        assert jj == -7, "full-state message out of order"
                    if rank > 0:
                        send(-7, 0, rank - 1, GRAD)
                    weight = 3 if am else 2
                else:
                    raise AssertionError(f"unknown op {typ}")
            if it == 0:            # post-validation step: partial chain 1 -> p on ACT, optimistic step
                if rank > 0:
                    jj, _ = recv(rank - 1, ACT)
                    assert jj == -5, "partial-state message out of order"
                if rank < p - 1:
                    send(-5, 0, rank + 1, ACT)
                weight = 2         # optimistic (not yet validated) weights
        for r in pending_sends:
            r.wait()
        dist.barrier()
        q.put((rank, "ok", final_grads if rank == 0 else None))
    except Exception:
        q.put((rank, "err", traceback.format_exc()))


CASES = [("zbh1", 2, 4, True, False), ("zbh1", 2, 4, False, False), ("zbh2", 3, 6, True, False),
         ("zbh1", 4, 8, True, False), ("auto", 4, 8, True, False), ("1f1b", 4, 6, True, True),
         ("zbh2", 4, 8, False, False)]


@pytest.mark.parametrize("family,world,m,amend,fused", CASES,
                         ids=[f"{c[0]}-p{c[1]}-m{c[2]}-{'amend' if c[3] else 'clean'}" for c in CASES])
def test_plans_execute_across_ranks(family, world, m, amend, fused):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, family, m, amend, fused, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = {}
    try:
        for _ in range(world):
            rank, status, payload = q.get(timeout=120)
            results[rank] = (status, payload)
    finally:
        for pr in procs:
            pr.join(timeout=10)
            if pr.is_alive():
                pr.kill()
    errs = {r: v[1] for r, v in results.items() if v[0] != "ok"}
    assert not errs, errs
    grads = results[0][1]
    assert sorted(grads) == list(range(m))
    want_version = 3 if amend else 2
    expect = int(str(want_version) * world)       # every stage's forward used the validated weights
    assert all(v == expect for v in grads.values()), grads
