// Kernel-level extern "C" entry points (include/zb_debug.h) for the parity tests.
#include "abi_util.h"
#include "gemm.h"
#include "zb_debug.h"

using namespace zb;

extern "C" zb_status_t zb_dbg_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                                   int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn, int32_t epi, void* C,
                                   int64_t ldc, const float* bias, void* aux, int64_t ldaux, int32_t beta,
                                   void* stream) {
  ZB_TRY {
    if (dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) return set_error(ZB_EINVAL, "bad dtype");
    if (epi < EPI_STORE || epi > EPI_F32_STORE) return set_error(ZB_EINVAL, "bad epilogue");
    if (M < 0 || N < 0 || K < 0 || !A || !B || !C) return set_error(ZB_EINVAL, "bad gemm operands");
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_mn = a_mn != 0;
    g.B = B; g.ldb = ldb; g.b_mn = b_mn != 0;
    g.epi = epi;
    g.ep = EpiArgs{C, ldc, bias, aux, ldaux, beta};
    gemm(g, static_cast<DType>(dtype), static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

