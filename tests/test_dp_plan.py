"""Data-parallel tail plans (plan.h dp_tail, App. A),
host only.

* Structure: only the trailing run of W ops (with 1F1B's fused gradient sends) changes; each tail W becomes one WP op per W
  unit; every unit's ALLREDUCE comes right after its LAST sub-computation; the vector
  region is reduced last.  reorder = True clusters the sub-computations of each parameter
  (App. A: "reorder all of these computations to cluster those calculating the gradients
  for the same parameter"), so unit u's all-reduce is issued after (u + 1) k
  sub-computations instead of after (k - 1) n_units + u + 1 of them (W-major order).
* Multi-process (gloo, CPU): D = 2 replicas x p = 2 stages execute their plans — P2P
  messages on the pipeline, all-reduces on the stage's DP group — with stand-in
  "gradients" (unit u of microbatch j of replica r contributes (r m + j + 1) (u + 1));
  every all-reduce must meet the same unit on the other replica (a mismatch shows up in
  the reduced unit tag) and carry that unit's complete sum over both replicas.
"""
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

OP_F, OP_B, OP_W, OP_RECV_ACT, OP_SEND_ACT, OP_RECV_GRAD, OP_SEND_GRAD, OP_VALIDATE = range(8)
OP_WP, OP_ALLREDUCE = 10, 11


@pytest.mark.parametrize("family,p,m", [("zbh1", 4, 8), ("zbh2", 4, 8), ("1f1b", 4, 8), ("zbh1", 1, 3),
                                        ("auto", 3, 6)])
@pytest.mark.parametrize("reorder", [False, True])
def test_dp_tail_structure(family, p, m, reorder):
    kw = {"M_limit": 2 * p * 3} if family == "auto" else {}
    passes, _ = api.schedule(family, p, m, 10, 11, 6, 1, **kw)
    U = 9
    for s in range(p):
        dp = api.dp_plan(passes, p, m, s, U, reorder, fused=family == "1f1b")
        # the base plan is the dp plan with the tail restored
        first_wp = next(i for i, o in enumerate(dp) if o[0] in (OP_WP, OP_ALLREDUCE))
        prefix = dp[:first_wp]
        tail = dp[first_wp:]
        assert all(o[0] in (OP_WP, OP_ALLREDUCE, OP_SEND_GRAD) for o in tail)
        for i, o in enumerate(tail):   # 1F1B's fused backward: a gradient leaves after its whole W
            if o[0] == OP_SEND_GRAD:
                assert [x for x in tail[i:] if x[0] == OP_WP and x[1] == o[1]] == []
                assert len([x for x in tail[:i] if x[0] == OP_WP and x[1] == o[1]]) == U
        tail = [o for o in tail if o[0] != OP_SEND_GRAD]
        assert tail[-1] == (OP_ALLREDUCE, -1, -1, -1)
        wps = [o for o in tail if o[0] == OP_WP]
        k = len(wps) // U
        assert k >= 1 and len(wps) == k * U
        tail_mbs = [o[1] for o in wps if o[2] == 0]
        assert len(tail_mbs) == k and len(set(tail_mbs)) == k
        # W ops of the prefix + tail microbatches = every microbatch exactly once
        w_pre = [o[1] for o in prefix if o[0] == OP_W]
        assert sorted(w_pre + tail_mbs) == list(range(m))
        assert all(o[0] != OP_W for o in tail)
        # every unit reduced once, right after its last sub-computation
        ar = [i for i, o in enumerate(tail) if o[0] == OP_ALLREDUCE and o[2] >= 0]
        assert sorted(tail[i][2] for i in ar) == list(range(U))
        for i in ar:
            u = tail[i][2]
            last = max(j for j, o in enumerate(tail) if o[0] == OP_WP and o[2] == u)
            assert last < i
            assert all(not (o[0] == OP_WP and o[2] == u) for o in tail[i:])
        # position of each unit's all-reduce, counted in sub-computations issued before it
        issued = {tail[i][2]: sum(1 for o in tail[:i] if o[0] == OP_WP) for i in ar}
        for u in range(U):
            assert issued[u] == ((u + 1) * k if reorder else (k - 1) * U + u + 1)
        if reorder:   # unit-major clusters in the tail microbatch order
            assert [(o[2], o[1]) for o in wps] == [(u, j) for u in range(U) for j in tail_mbs]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, D, p, m, U, port, reorder, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=D * p)
        r, s = divmod(rank, p)
        dp_groups = [dist.new_group([rr * p + ss for rr in range(D)]) for ss in range(p)]
        passes, _ = api.schedule("zbh1", p, m, 10, 11, 6, 1)
        plan = api.dp_plan(passes, p, m, s, U, reorder)
        grad = torch.zeros(U + 1, dtype=torch.float64)     # [unit] partial sums, [U] vector region
        act = torch.zeros(1, dtype=torch.int64)
        ev, pending = [], []

        def contrib(j, u):
            return float((r * m + j + 1) * (u + 1))
        for op in plan:
            t, j, msg, _ = op
            me = r * p + s
            if t == OP_RECV_ACT:
                dist.recv(act, src=me - 1, tag=0)
                assert int(act) == j
            elif t == OP_SEND_ACT:
                pending.append(dist.isend(torch.tensor([j]), dst=me + 1, tag=0))   # NCCL: never blocks the host
            elif t == OP_RECV_GRAD:
                dist.recv(act, src=me + 1, tag=1)
                assert int(act) == j
            elif t == OP_SEND_GRAD:
                pending.append(dist.isend(torch.tensor([j]), dst=me - 1, tag=1))
            elif t == OP_B:
                grad[U] += j + 1            # LayerNorm-style vector grads formed in B
            elif t == OP_W:
                for u in range(U):
                    grad[u] += contrib(j, u)
            elif t == OP_WP:
                grad[msg] += contrib(j, msg)
            elif t == OP_ALLREDUCE:
                u = U if msg < 0 else msg
                x = torch.tensor([float(u), grad[u].item()], dtype=torch.float64)
                dist.all_reduce(x, group=dp_groups[s])
                assert x[0].item() == D * u, ("all-reduce met a different unit", x[0].item(), u)
                grad[u] = x[1]
                ev.append(u)
        for w in pending:
            w.wait()
        want = [sum((rr * m + j + 1) * (u + 1) for rr in range(D) for j in range(m)) for u in range(U)]
        want.append(sum(j + 1 for j in range(m)) * D)
        assert [grad[u].item() for u in range(U + 1)] == [float(w) for w in want]
        assert sorted(ev) == list(range(U + 1))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("reorder", [False, True])
def test_dp_plans_across_gloo_processes(reorder):
    D, p, m, U = 2, 2, 6, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(rk, D, p, m, U, port, reorder, q)) for rk in range(D * p)]
    for x in procs:
        x.start()
    res = [q.get(timeout=240) for _ in procs]
    for x in procs:
        x.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad
