"""One rank of the data-parallel test (tests/test_gpu_dp_shim.py): D replicas of a
p-stage pipeline, rank = replica * p + stage, all processes on one GPU with the CUDA-IPC
libnccl shim (ZB_NCCL_LIB).  Replica r trains on microbatches [r m, (r + 1) m) of an
iteration's D m microbatches; the stage's gradients are summed over the replicas by
zb_run_iteration's all-reduces (zb_ctx_attach_dp; ZB_DP_REORDER=1 reorders the tail Ws per
parameter, App. A).  Writes the first iteration's gradients and loss, the final
parameters and the all-reduce count to OUT/rank<r>.npz."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import zb_synth  # noqa: E402
from paper_2401_10241_b200 import api  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    D, p = int(os.environ["ZB_DP"]), int(os.environ["ZB_PP"])
    assert world == D * p
    r, s = divmod(rank, p)
    out, family, dtype = os.environ["ZB_OUT"], os.environ["ZB_FAMILY"], os.environ["ZB_DTYPE"]
    iters = int(os.environ.get("ZB_ITERS", "2"))
    reorder = os.environ.get("ZB_DP_REORDER", "0") == "1"
    group_w = os.environ.get("ZB_GROUP_W", "0") == "1"
    m = int(os.environ.get("ZB_M", "4"))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    cfg = zb_synth.ModelConfig("dp", h=128, a=2, L=4, s=256, b=2, V=512, p=p, m=m, family=family)
    cfg_all = cfg.with_(m=D * m)
    passes, sim = api.schedule(family, p, m, 10, 11, 6, 0)
    ids = [None]
    if rank == 0:
        ids = [{"p2p": [api.nccl_unique_ids(2 * (p - 1)) if p > 1 else b"" for _ in range(D)],
                "dp": [api.nccl_unique_ids(1) for _ in range(p)]}]
    dist.broadcast_object_list(ids, src=0)
    ids = ids[0]
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, p, s, m, max(1, sim.n_slots[s]), dtype=dtype, stream=stream)
    prm = zb_synth.make_stage_params(cfg, p, s)
    ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, p, s)])
    if p > 1:
        ctx.attach_nccl(ids["p2p"][r], s, p)
    ctx.attach_dp(ids["dp"][s], r, D)
    opt = api.optim_cfg(lr=1e-3, mode=os.environ.get("ZB_OPT", "pv"), clip=1.0)
    fused = family == "1f1b"
    grads0, loss0 = None, 0.0
    for it in range(iters):
        tok = zb_synth.make_tokens(cfg_all, it)[r * m:(r + 1) * m]
        tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
        lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
        ctx.run_iteration(passes, tin if s == 0 else None, lab if s == p - 1 else None, fused=fused,
                          group_w=group_w, dp_reorder=reorder)
        if it == 0:
            loss0 = ctx.loss() if s == p - 1 else 0.0
            grads0 = ctx.get_grads()
        ctx.post_validate_step(opt)
    ctx.post_validate_finish(opt)
    ctx.sync()
    params = ctx.get_params()
    n_units, reduces = ctx.w_units()
    np.savez(os.path.join(out, f"rank{rank}.npz"), loss=loss0, n_units=n_units, reduces=reduces,
             **{f"g{i}": g for i, g in enumerate(grads0)}, **{f"p{i}": x for i, x in enumerate(params)})
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
