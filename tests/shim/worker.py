"""One rank of the 2-process / 1-GPU NCCL-path test (tests/test_gpu_nccl_shim.py).

Runs stage RANK of a p = WORLD_SIZE pipeline through zb_ctx_attach_nccl +
zb_run_iteration + zb_post_validate_step / _finish (libnccl = the IPC shim named by
ZB_NCCL_LIB), ITERS iterations, then writes its gradients, parameters, AdamW
moments, loss and the T_comm probe to OUT/rank<r>.npz."""
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
    out, family, dtype = os.environ["ZB_OUT"], os.environ["ZB_FAMILY"], os.environ["ZB_DTYPE"]
    iters = int(os.environ.get("ZB_ITERS", "2"))
    clip = float(os.environ.get("ZB_CLIP", "1.0"))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    cfg = zb_synth.ModelConfig("shim", h=128, a=2, L=4, s=256, b=2, V=512, p=world, m=5, family=family)
    passes, sim = api.schedule(family, world, cfg.m, 10, 11, 6, 0)
    ids = [api.nccl_unique_ids(2 * (world - 1)) if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    stream = torch.cuda.Stream()
    ctx = api.Context(cfg, world, rank, cfg.m, max(1, sim.n_slots[rank]), dtype=dtype, stream=stream)
    prm = zb_synth.make_stage_params(cfg, world, rank)
    ctx.set_params([prm[n] for n, _, _ in zb_synth.param_specs(cfg, world, rank)])
    ctx.attach_nccl(ids[0], rank, world)
    opt = api.optim_cfg(lr=1e-3, mode=os.environ.get("ZB_OPT", "pv"), clip=clip)
    fused = family == "1f1b"
    for it in range(iters):
        tok = zb_synth.make_tokens(cfg, it)
        tin = torch.from_numpy(np.ascontiguousarray(tok[..., :cfg.s])).cuda()
        lab = torch.from_numpy(np.ascontiguousarray(tok[..., 1:])).cuda()
        ctx.run_iteration(passes, tin if rank == 0 else None, lab if rank == world - 1 else None, fused=fused)
        loss = ctx.loss() if rank == world - 1 else 0.0
        grads = ctx.get_grads()
        ctx.post_validate_step(opt)
    ctx.post_validate_finish(opt)
    rt = ctx.comm_probe(4 * cfg.T * cfg.h, 5)
    ctx.sync()
    params = ctx.get_params()
    ms, vs = ctx.get_moments()
    rep = ctx.pv_report()
    np.savez(os.path.join(out, f"rank{rank}.npz"), loss=loss, rt=rt, t=rep["t"],
             **{f"g{i}": g for i, g in enumerate(grads)}, **{f"p{i}": x for i, x in enumerate(params)},
             **{f"m{i}": x for i, x in enumerate(ms)}, **{f"v{i}": x for i, x in enumerate(vs)})
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
