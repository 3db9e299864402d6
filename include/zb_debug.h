/*
 * zb_debug.h — kernel-level entry points of libzb used by the parity tests
 * (tests/test_gpu_kernels.py).  Same conventions as zb.h: device pointers,
 * the caller owns every buffer, work is enqueued on `stream` (cudaStream_t,
 * NULL = default), errors are returned as zb_status_t with zb_last_error().
 * They expose the exact kernels the stage passes launch, so each can be
 * checked against the oracle in isolation.
 */
#ifndef ZB_DEBUG_H
#define ZB_DEBUG_H
#include "zb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM of the F / B / W contractions:
 *   C[m,n] (op)= sum_k A(m,k) B(n,k),
 *   A(m,k) = a_mn ? A[k*lda + m] : A[m*lda + k]   (a_mn: A stored [K, M])
 *   B(n,k) = b_mn ? B[k*ldb + n] : B[n*ldb + k]   (b_mn: B stored [K, N])
 * dtype ZB_DTYPE_BF16: A, B bf16 (tcgen05 kernel), activation outputs bf16;
 * ZB_DTYPE_F32: everything f32 (SIMT kernel).
 * epi: 0 C = acc (+bias); 1 C = acc + bias, aux = GeLU(C); 2 C = aux + acc (+bias);
 *      3 C = acc * GeLU'(aux); 4 C(f32) = acc + (beta ? C : 0); 5 C(f32) = acc.
 * epi 4 (W) with a_mn: a non-NULL `bias` is an OUTPUT, f32 [M]: (beta ? += : =) the
 *      column sums sum_k A(m,k) (W's bias gradient, formed inside the GEMM). 
 * N and ldc must be multiples of 8; operands 16-byte aligned. */
zb_status_t zb_dbg_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_mn,
                        const void* B, int64_t ldb, int32_t b_mn, int32_t epi, void* C, int64_t ldc,
                        const float* bias, void* aux, int64_t ldaux, int32_t beta, void* stream);

/* W-grouping contraction (bf16): C[M,N] (beta ? += : =) sum over the nseg
 * segments s of A_s^T B_s with A_s = dY_s [K/nseg, M] and B_s = X_s [K/nseg, N] (dev,
 * row-major, MN-major operands, K/nseg a multiple of 64); bias_out (nullable, f32 [M]) gets
 * the column sums of all A_s the same way.  nseg in 1..4. */
zb_status_t zb_dbg_gemm_wgroup(int32_t M, int32_t N, int32_t K, int32_t nseg, const void* const* A_seg,
                               const void* const* B_seg, float* C, float* bias_out, int32_t beta, void* stream);

/* Causal multi-head attention forward on a packed qkv [b*s, 3h] (Q, K, V
 * column blocks, head k at columns k*d of each): o [b*s, h], lse [b, a, s] f32. */
zb_status_t zb_dbg_attention_fwd(int32_t dtype, int32_t b, int32_t s, int32_t a, int32_t d, const void* qkv,
                                 void* o, float* lse, void* stream);
/* Attention backward: dqkv [b*s, 3h] from qkv, o, do, lse; delta: f32 scratch [b, a, s]. */
zb_status_t zb_dbg_attention_bwd(int32_t dtype, int32_t b, int32_t s, int32_t a, int32_t d, const void* qkv,
                                 const void* o, const void* dout, const float* lse, void* dqkv, float* delta,
                                 void* stream);

/* The HBM-bound row / column kernels of the stage passes (ops.h), for the
 * parity tests (all device pointers, row-major, f32 statistics):
 *  layernorm_fwd: y[rows,h] = g * (x - mean) * rstd + b; mean, rstd [rows] written.
 *  layernorm_bwd: dx = resid + rstd * (gh - mean(gh) - xhat * mean(gh*xhat)),
 *      gh = dy * g (dy f32; resid, dx32 f32 and nullable; dx in the dtype, may alias x);
 *      gg (+)= colsum(dy * xhat), gb (+)= colsum(dy) (beta != 0: accumulate).
 *  bias_grad: out[n] (+)= colsum(y[rows, n] with leading dimension ldy). */
zb_status_t zb_dbg_layernorm_fwd(int32_t dtype, const void* x, const float* g, const float* b, void* y, float* mean,
                                 float* rstd, int32_t rows, int32_t h, float eps, void* stream);
zb_status_t zb_dbg_layernorm_bwd(int32_t dtype, const float* dy, const void* x, const float* mean, const float* rstd,
                                 const float* g, const float* resid, float* dx32, void* dx, float* gg, float* gb,
                                 int32_t beta, int32_t rows, int32_t h, void* stream);
zb_status_t zb_dbg_bias_grad(int32_t dtype, const void* y, int64_t ldy, float* out, int32_t rows, int32_t n,
                             int32_t beta, void* stream);

/* Kernel-class timing used by bench.py for the live roofline numbers: when
 * enabled, every GEMM / attention / HBM-bound op launch is bracketed by CUDA
 * events on its stream and its algorithmic work is recorded (FLOPs for
 * classes 0-5, BYTES for 6-12).  Classes: 0 all GEMMs, 1 attention forward,
 * 2 attention backward, 3 F GEMMs (X W^T), 4 B GEMMs (dY W), 5 W GEMMs
 * (dY^T X), 6 LayerNorm forward, 7 LayerNorm backward dx, 8 LayerNorm
 * gamma/beta grads, 9 bias grads (column sums), 10 cross-entropy, 11 grad
 * norm + AdamW, 12 embedding / conversions.  read() synchronises the
 * pending events. */
zb_status_t zb_dbg_kernel_timing(int32_t enable, int32_t reset);
zb_status_t zb_dbg_kernel_timing_read(int32_t cls, double* total_ms, double* total_flops, int64_t* launches);

/* The host-side P2P plan the NCCL runner executes for `stage` in one
 * iteration (csrc/plan.h): out_ops[4*i .. 4*i+3] = {type, microbatch,
 * message index, slot}; types 0 F, 1 B, 2 W, 3 RECV_ACT, 4 SEND_ACT,
 * 5 RECV_GRAD, 6 SEND_GRAD, 7 VALIDATE, 8 DISCARD_ACT, 9 REPLAY_F.
 * passes: zb_schedule output of every stage.  Pure host code (no GPU). */
zb_status_t zb_dbg_stage_plan(const zb_pass_t* passes, int32_t n, int32_t p, int32_t m, int32_t stage,
                              int32_t pv_pending, int32_t amend, int32_t fused, int32_t* out_ops, int32_t cap,
                              int32_t* n_out);
/* The same plan with the data-parallel tail (plan.h dp_tail, SURVEY §8(f)4 /
 * App. A): the trailing W ops become types 10 WP {microbatch, unit (message
 * index field), slot} and 11 ALLREDUCE {-1, unit or -1 for the vector region,
 * -1}; n_units W units per pass (zb_dbg_w_units), reorder != 0 clusters them
 * per unit (ZB_RUN_DP_REORDER). */
zb_status_t zb_dbg_dp_plan(const zb_pass_t* passes, int32_t n, int32_t p, int32_t m, int32_t stage,
                           int32_t pv_pending, int32_t amend, int32_t fused, int32_t n_units, int32_t reorder,
                           int32_t* out_ops, int32_t cap, int32_t* n_out);
/* W units of a context's W pass and the all-reduce calls its DP communicator issued. */
zb_status_t zb_dbg_w_units(zb_ctx_t* ctx, int32_t* n_units, int64_t* dp_reduces);
/* n'_s, the number of speculative warm-up Fs of each stage (plan.h). */
/* Merged op list of one worker of a chunked schedule (plan.h worker_plan):
 * 5 ints per op: type, microbatch, message index, slot, chunk (virtual stage).
 * worker_of[nv]: the worker of every virtual stage. */
zb_status_t zb_dbg_worker_plan(const zb_pass_t* passes, int32_t n, int32_t nv, int32_t m, int32_t worker,
                               const int32_t* worker_of, int32_t fused, int32_t* out_ops, int32_t cap,
                               int32_t* n_out);
zb_status_t zb_dbg_speculative_counts(const zb_pass_t* passes, int32_t n, int32_t p, int32_t* out);

/* Measurement builds only (not exported by the default libzb.so, so not declared here):
 * `make BUILD=build_trace OUT=libzb_trace.so EXTRA=-DZB_ATTN_TRACE` adds the dK/dV and the
 * forward CTA timelines (12 x 64 globaltimer stamps each), `make BUILD=build_gtrace
 * OUT=libzb_gtrace.so EXTRA=-DZB_GEMM_TRACE` the 2-CTA GEMM's CTA-0 timeline (8 x 64);
 * their readers are scripts/attn_trace.py, scripts/attn_fwd_trace.py and
 * scripts/gemm_trace.py. */

#ifdef __cplusplus
}
#endif
#endif
