"""GPU parity of the F / B / W GEMM kernels (tcgen05 bf16 and SIMT f32) against
the plain definition C = A(m,k) B(n,k) summed in fp64 on the same (bf16-rounded)
inputs.  Shapes span several 128 x 256 tiles, ragged M / N / K tails, and every
operand-major combination the stage passes use (gemm.h)."""
import numpy as np
import pytest

from zbtest_util import assert_close, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


def _gelu(x):
    return 0.5 * x * (1 + np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3)))


def _gelu_grad(x):
    t = np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * np.sqrt(2 / np.pi) * (1 + 3 * 0.044715 * x * x)



CASES = [
    # (M, N, K, a_mn, b_mn, epi)
    (1024, 192, 64, False, False, 0),     # tiny qkv F
    (300, 264, 200, False, False, 0),     # ragged everything, F
    (640, 512, 384, False, False, 1),     # bias + GeLU (fc1 F)
    (384, 256, 520, False, False, 2),     # residual (proj / fc2 F)
    (300, 136, 520, False, True, 0),      # B variant dX = dY W
    (512, 640, 256, False, True, 3),      # GeLU backward epilogue (fc2 dgrad)
    (264, 200, 1000, True, True, 4),      # W variant dW += dY^T X, ragged T
    (768, 512, 1024, True, True, 4),
    (512, 512, 4096, True, True, 4),      # ordered split-K: 4 tiles -> 4 splits of 16 k-blocks
    (2304, 2304, 6144, True, True, 4),    # 1.5B proj W: 81 tiles for 74 CTA pairs -> 4 splits
    (256, 512, 320, False, False, 5),     # f32 logits
]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}x{c[2]}-{int(c[3])}{int(c[4])}-e{c[5]}" for c in CASES])
def test_gemm_parity(case, dtype):
    import torch
    from paper_2401_10241_b200 import api
    M, N, K, a_mn, b_mn, epi = case
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K + epi)
    A = (torch.randn((K, M) if a_mn else (M, K), generator=g) * 0.5).to(tdt).cuda()
    B = (torch.randn((K, N) if b_mn else (N, K), generator=g) * 0.5).to(tdt).cuda()
    bias = (torch.randn(N, generator=g) * 0.1).float().cuda()
    Ad = A.double().cpu().numpy()
    Bd = B.double().cpu().numpy()
    Am = Ad.T if a_mn else Ad
    Bm = Bd.T if b_mn else Bd
    acc = Am @ Bm.T
    use_bias = epi in (0, 1, 2)
    f32_out = epi in (4, 5)
    out_dt = torch.float32 if f32_out else tdt
    Cbuf = torch.randn(M, N, generator=g).to(out_dt).cuda()
    aux = None
    ref = acc + (bias.double().cpu().numpy() if use_bias else 0)
    if epi == 1:
        aux = torch.zeros(M, N, dtype=tdt).cuda()
    elif epi == 2:
        aux = torch.randn(M, N, generator=g).to(tdt).cuda()
        ref = ref + aux.double().cpu().numpy()
    elif epi == 3:
        aux = torch.randn(M, N, generator=g).to(tdt).cuda()
        ref = acc * _gelu_grad(aux.double().cpu().numpy())
    for beta in ((0, 1) if epi == 4 else (0,)):
        C0 = Cbuf.double().cpu().numpy()
        api.dbg_gemm(A, B, Cbuf, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn, epi=epi,
                     bias=bias if use_bias else None, aux=aux, beta=beta)
        torch.cuda.synchronize()
        got = Cbuf.double().cpu().numpy()
        want = ref + (C0 if (epi == 4 and beta) else 0)
        tol = 1e-5 if (dtype == "f32" or f32_out) else 6e-3
        assert_close(got, want, tol, f"C beta={beta}")
        if epi == 1:
            gg = aux.double().cpu().numpy()
            assert_close(gg, _gelu(ref), 1e-5 if dtype == "f32" else 6e-3, "GeLU aux")


@pytest.mark.parametrize("M,N,K", [(2304, 2304, 6144), (9216, 2304, 6144), (768, 512, 1000), (264, 200, 1000),
                                   (6912, 2304, 3072), (512, 512, 4096)])
def test_w_gemm_bias_column_sums(M, N, K):
    """W's bias gradient formed inside the W GEMM (column-sum warps over the dY tiles,
    gemm.h bias_out) against the plain column sums in fp64; split-K shapes (partials
    summed in order) and ragged tails; beta = 0 overwrites, beta = 1 accumulates; bitwise
    repeatable.  The dW output is unchanged by the fused sums."""
    import torch
    from paper_2401_10241_b200 import api
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = (torch.randn(K, M, generator=g) * 0.5).bfloat16().cuda()
    B = (torch.randn(K, N, generator=g) * 0.5).bfloat16().cuda()
    Ad, Bd = A.double().cpu().numpy(), B.double().cpu().numpy()
    want_c = Ad.T @ Bd
    want_b = Ad.sum(0)
    C = torch.zeros(M, N, dtype=torch.float32).cuda()
    db = torch.full((M,), 7.0, dtype=torch.float32).cuda()
    api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, bias=db, beta=0)
    torch.cuda.synchronize()
    # f32 accumulation over K up to 6144 in TMEM: the statistical elementwise form (R-tol)
    assert_close(C.double().cpu().numpy(), want_c, 1e-5, "dW", bf16=True)
    assert_close(db.double().cpu().numpy(), want_b, 1e-5, "db beta=0")
    first = db.clone()
    api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, bias=db, beta=1)
    torch.cuda.synchronize()
    assert_close(db.double().cpu().numpy(), 2 * want_b, 1e-5, "db beta=1")
    again = torch.zeros_like(db)
    api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, bias=again, beta=0)
    torch.cuda.synchronize()
    assert torch.equal(again, first)


def test_split_k_w_is_deterministic():
    """The ordered split-K of W (gemm.cu split_k_plan) sums in one fixed order:
    repeated accumulations are bitwise identical (P:196 needs this across schedules)."""
    import torch
    from paper_2401_10241_b200 import api
    M, N, K = 2304, 2304, 6144
    g = torch.Generator(device="cpu").manual_seed(7)
    A = torch.randn(K, M, generator=g).bfloat16().cuda()
    B = torch.randn(K, N, generator=g).bfloat16().cuda()
    outs = []
    for _ in range(3):
        C = torch.zeros(M, N, dtype=torch.float32).cuda()
        for beta in (0, 1, 1):
            api.dbg_gemm(A, B, C, M=M, N=N, K=K, a_mn=True, b_mn=True, epi=4, beta=beta)
        torch.cuda.synchronize()
        outs.append(C.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
