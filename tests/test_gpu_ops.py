"""GPU parity of the HBM-bound row / column kernels (ops.h) against the
oracle's written-out definitions (oracle/model.py: layernorm_fwd,
layernorm_bwd_input, layernorm_bwd_weight; bias grads = column sums, P:46's W
of a bias) in fp64 on the same (dtype-rounded) inputs — at the bench shape
(1.5B microbatch: 6144 rows x 2304, and the 4h = 9216 / 3h = 6912 bias widths)
and at small ragged shapes; plus bitwise repeatability of the deterministic
two-phase column reductions."""
import numpy as np
import pytest

from zbtest_util import assert_close, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]



LN_SHAPES = [(6144, 2304), (3072, 4096), (1024, 6144), (37, 64), (2000, 264), (300, 2304), (5, 4096), (149, 1024),
             (3001, 3072)]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("rows,h", LN_SHAPES)
def test_layernorm_fwd_bwd(rows, h, dtype):
    import torch
    from oracle import model as om
    from paper_2401_10241_b200 import api
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    gen = torch.Generator().manual_seed(rows + h)
    x = (torch.randn(rows, h, generator=gen) * 2 + 0.5).to(tdt)
    g = 1 + 0.1 * torch.randn(h, generator=gen)
    b = 0.1 * torch.randn(h, generator=gen)
    dy = torch.randn(rows, h, generator=gen)
    resid = torch.randn(rows, h, generator=gen)
    xd, gd, bd, dyd, rd = (t.double().numpy() for t in (x, g, b, dy, resid))
    y_ref, (xhat, rstd) = om.layernorm_fwd(xd, gd, bd)
    dx_ref = rd + om.layernorm_bwd_input(dyd, xhat, rstd, gd)
    gg_ref, gb_ref = om.layernorm_bwd_weight(dyd, xhat)
    X, G, B, DY, R = (t.cuda() for t in (x, g, b, dy, resid))
    Y = torch.empty_like(X)
    mean = torch.empty(rows, device="cuda")
    rs = torch.empty(rows, device="cuda")
    api.dbg_layernorm_fwd(X, G, B, Y, mean, rs, rows=rows, h=h)
    gg = torch.full((h,), 3.0, device="cuda")
    gb = torch.full((h,), -2.0, device="cuda")
    dx32 = torch.empty(rows, h, device="cuda")
    dx = torch.empty_like(X)
    api.dbg_layernorm_bwd(DY, X, mean, rs, G, dx, gg, gb, rows=rows, h=h, resid=R, dx32=dx32, beta=1)
    torch.cuda.synchronize()
    ftol = 1e-5 if dtype == "f32" else 8e-3
    assert_close(Y.double().cpu().numpy(), y_ref, ftol, "LN y")
    assert_close(rs.double().cpu().numpy(), rstd[:, 0], 1e-5, "LN rstd")
    assert_close(dx32.double().cpu().numpy(), dx_ref, 1e-5, "LN dx f32")
    assert_close(dx.double().cpu().numpy(), dx_ref, ftol, "LN dx")
    assert_close(gg.double().cpu().numpy(), gg_ref + 3.0, 1e-5, "LN dgamma")
    assert_close(gb.double().cpu().numpy(), gb_ref - 2.0, 1e-5, "LN dbeta")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("rows,n,ld", [(6144, 2304, 2304), (6144, 9216, 9216), (6144, 2304, 6912), (6144, 6912, 6912),
                                       (100, 64, 64), (1, 8, 8), (777, 264, 1000)])
def test_bias_grad(rows, n, ld, dtype):
    import torch
    from paper_2401_10241_b200 import api
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    gen = torch.Generator().manual_seed(rows * 3 + n)
    y = torch.randn(rows, ld, generator=gen).to(tdt)
    ref = y[:, :n].double().sum(0).numpy()
    Y = y.cuda()
    out = torch.full((n,), 1.5, device="cuda")
    api.dbg_bias_grad(Y, out, rows=rows, n=n, ldy=ld, beta=1)
    o1 = out.clone()
    api.dbg_bias_grad(Y, out, rows=rows, n=n, ldy=ld, beta=0)
    torch.cuda.synchronize()
    assert_close(o1.double().cpu().numpy(), ref + 1.5, 1e-5, "bias grad beta=1")
    assert_close(out.double().cpu().numpy(), ref, 1e-5, "bias grad beta=0")
    again = torch.empty_like(out)
    api.dbg_bias_grad(Y, again, rows=rows, n=n, ldy=ld, beta=0)
    torch.cuda.synchronize()
    assert torch.equal(again, out)          # fixed partition and order: bitwise repeatable
