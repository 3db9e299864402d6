// Kernel-level extern "C" entry points (include/zb_debug.h) for the parity tests.
#include "abi_util.h"
#include "attention.h"
#include "gemm.h"
#include "ktimer.h"
#include "ops.h"
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
    if (epi == EPI_F32_ACC && bias != nullptr) {  // W: `bias` receives the column sums of A (bias_out)
      if (!a_mn) return set_error(ZB_EINVAL, "bias_out needs an MN-major A (the W contraction)");
      g.ep.bias = nullptr;
      g.ep.bias_out = const_cast<float*>(bias);
    }
    gemm(g, static_cast<DType>(dtype), static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}


extern "C" zb_status_t zb_dbg_gemm_wgroup(int32_t M, int32_t N, int32_t K, int32_t nseg, const void* const* A_seg,
                                          const void* const* B_seg, float* C, float* bias_out, int32_t beta,
                                          void* stream) {
  ZB_TRY {
    if (M <= 0 || N <= 0 || K <= 0 || nseg < 1 || nseg > kMaxSeg || !A_seg || !B_seg || !C)
      return set_error(ZB_EINVAL, "bad grouped W arguments");
    GemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = A_seg[0]; g.lda = M; g.a_mn = true;
    g.B = B_seg[0]; g.ldb = N; g.b_mn = true;
    g.epi = EPI_F32_ACC;
    g.ep = EpiArgs{C, N, nullptr, nullptr, 0, beta};
    g.ep.bias_out = bias_out;
    g.nseg = nseg;
    for (int i = 0; i < nseg; ++i) {
      g.A_seg[i] = A_seg[i];
      g.B_seg[i] = B_seg[i];
    }
    gemm(g, DT_BF16, static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_attention_fwd(int32_t dtype, int32_t b, int32_t s, int32_t a, int32_t d,
                                            const void* qkv, void* o, float* lse, void* stream) {
  ZB_TRY {
    if (dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) return set_error(ZB_EINVAL, "bad dtype");
    AttnShape sh{b, s, a, d};
    attention_fwd(sh, static_cast<DType>(dtype), qkv, o, lse, static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_attention_bwd(int32_t dtype, int32_t b, int32_t s, int32_t a, int32_t d,
                                            const void* qkv, const void* o, const void* dout, const float* lse,
                                            void* dqkv, float* delta, void* stream) {
  ZB_TRY {
    if (dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) return set_error(ZB_EINVAL, "bad dtype");
    AttnShape sh{b, s, a, d};
    attention_bwd(sh, static_cast<DType>(dtype), qkv, o, dout, lse, dqkv, delta, static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_kernel_timing(int32_t enable, int32_t reset) {
  ZB_TRY {
    if (reset) ktimer::reset();
    ktimer::set_enabled(enable != 0);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_launch_count(int32_t reset, int64_t* count) {
  ZB_TRY {
    if (!count) return set_error(ZB_EINVAL, "null count");
    *count = launch_count(reset != 0);
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_kernel_timing_read(int32_t cls, double* total_ms, double* total_flops,
                                                 int64_t* launches) {
  ZB_TRY {
    if (cls < 0 || cls >= ktimer::N_CLASSES || !total_ms || !total_flops || !launches)
      return set_error(ZB_EINVAL, "bad kernel timing query");
    if (cls == 0) {  // all GEMMs = F + B + W classes
      double ms = 0, fl = 0;
      int64_t n = 0;
      for (int c : {ktimer::GEMM_F, ktimer::GEMM_B, ktimer::GEMM_W}) {
        double a, b;
        int64_t k;
        ktimer::read(c, &a, &b, &k);
        ms += a; fl += b; n += k;
      }
      *total_ms = ms; *total_flops = fl; *launches = n;
    } else {
      ktimer::read(cls, total_ms, total_flops, launches);
    }
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_layernorm_fwd(int32_t dtype, const void* x, const float* g, const float* b, void* y,
                                            float* mean, float* rstd, int32_t rows, int32_t h, float eps,
                                            void* stream) {
  ZB_TRY {
    if ((dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) || !x || !g || !b || !y || !mean || !rstd || rows < 0 ||
        h <= 0)
      return set_error(ZB_EINVAL, "zb_dbg_layernorm_fwd: bad arguments");
    layernorm_fwd(static_cast<DType>(dtype), x, g, b, y, mean, rstd, rows, h, eps, static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_layernorm_bwd(int32_t dtype, const float* dy, const void* x, const float* mean,
                                            const float* rstd, const float* g, const float* resid, float* dx32,
                                            void* dx, float* gg, float* gb, int32_t beta, int32_t rows, int32_t h,
                                            void* stream) {
  ZB_TRY {
    if ((dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) || !dy || !x || !mean || !rstd || !g || !dx || !gg ||
        !gb || rows < 0 || h <= 0)
      return set_error(ZB_EINVAL, "zb_dbg_layernorm_bwd: bad arguments");
    layernorm_bwd(static_cast<DType>(dtype), dy, x, mean, rstd, g, resid, dx32, dx, gg, gb, beta, rows, h,
                  static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}

extern "C" zb_status_t zb_dbg_bias_grad(int32_t dtype, const void* y, int64_t ldy, float* out, int32_t rows,
                                        int32_t n, int32_t beta, void* stream) {
  ZB_TRY {
    if ((dtype != ZB_DTYPE_BF16 && dtype != ZB_DTYPE_F32) || !y || !out || rows < 0 || n <= 0 || ldy < n)
      return set_error(ZB_EINVAL, "zb_dbg_bias_grad: bad arguments");
    bias_grad(static_cast<DType>(dtype), y, ldy, out, rows, n, beta, static_cast<cudaStream_t>(stream));
    return ZB_OK;
  }
  ZB_CATCH
}
