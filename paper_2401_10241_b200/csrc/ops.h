// Row-wise / elementwise kernels of the stage passes (HBM-bound; ops.cu).
// All reductions are deterministic: fixed partitions, fixed summation order,
// no floating-point atomics (bitwise-reproducible gradients).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace zb {

// LayerNorm forward: y = g * (x - mean) * rstd + b; mean / rstd saved (f32).
void layernorm_fwd(DType dt, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                   int rows, int h, float eps, cudaStream_t st);
// LayerNorm backward (B) and its parameter grads:
//   dx = resid + rstd * (gh - mean(gh) - xhat * mean(gh * xhat)), gh = dy * g
// dy is f32 in both modes; x is in the activation dtype; dx may alias x.
// The residual-gradient stream is f32 (resid, dx32; either may be null) and dx
// (activation dtype) receives the copy the GEMMs consume (DESIGN.md R-grad32).
// gg / gb (+)= column sums of dy * xhat / dy (beta: accumulate), deterministic
// (fixed row partition and fixed reduction tree).
void layernorm_bwd(DType dt, const float* dy, const void* x, const float* mean, const float* rstd, const float* g,
                   const float* resid, float* dx32, void* dx, float* gg, float* gb, int beta, int rows, int h,
                   cudaStream_t st);
// f32 -> activation dtype row copy (received stage-boundary gradients)
void convert_rows(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st);
// out[n] (+)= column sums of y [rows, n] (activation dtype), deterministic (fixed order).
void bias_grad(DType dt, const void* y, int64_t ldy, float* out, int rows, int n, int beta, cudaStream_t st);

// Embedding: x0[t] = wte[tok[t]] + wpe[t % s]  (wte / wpe f32 master copies)
void embed_fwd(DType dt, const int32_t* tok, const float* wte, const float* wpe, void* x0, int rows, int s, int h,
               cudaStream_t st);
// dW_te[v] += sum over positions with tok == v (in position order); dW_pe[t] += sum_b dx0[b, t].
// keys: scratch u32 [8192]; rows <= 8192 and V * rows < 2^32.
void embed_bwd(DType dt, const int32_t* tok, const void* dx0, float* dwte, float* dwpe, uint32_t* keys, int rows,
               int s, int h, cudaStream_t st);

// Softmax cross-entropy of logits [rows, V] f32 with labels: writes
//   dlogits = (softmax - onehot) * inv_scale (activation dtype), loss_rows[t] = lse - logit[label]
// and adds inv_scale * sum_t loss_rows[t] to *loss_acc (double, fixed order).
void cross_entropy(DType dt, const float* logits, const int32_t* labels, void* dlogits, float* loss_rows,
                   double* loss_acc, int rows, int V, float inv_scale, cudaStream_t st);

// f32 -> activation-dtype copy (bf16 shadow refresh) of n elements.
void convert_f32(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st);

// ---- optimizer (K12 / K13) -------------------------------------------------------------------
// Device-side post-validation state of one stage (§4).
struct PvState {
  double local_sumsq, partial_in_sumsq, partial_sumsq, full_sumsq;
  int32_t local_nf, partial_in_nf, partial_nf, full_nf;
  int32_t first_action, final_action;  // ZB_ACT_* of zb.h
  int32_t t;                           // AdamW time stamp
  int32_t adam_mode;                   // action of the next adamw launch: 0 none, 1 step, 2 rollback, 3 rollback+step
  float coef_step, coef_rollback;      // gradient multipliers of the step / of the undone step
  float coef_first;                    // coefficient the optimistic step used
  int32_t pad;
};

// sum of squares (f64) and non-finite flag of g[0..n) -> st->local_*; part: f64 scratch [kNormBlocks]
constexpr int kNormBlocks = 296;
void grad_norm(const float* g, int64_t n, double* part, int32_t* nf_part, PvState* st, cudaStream_t st_);
// partial = partial_in + local (single thread)
void pv_combine(PvState* st, cudaStream_t s);
// decisions (single thread): mode 0 = sync (full == partial), 1 = post-validation first step
void pv_decide_first(PvState* st, float clip, int sync_mode, cudaStream_t s);
void pv_decide_final(PvState* st, float clip, cudaStream_t s);
// Algorithm 1 over the flat parameter space, predicated on st->adam_mode.
// Elements [0, n_wd) decay with weight_decay; [n_shadow) also refresh the bf16 shadow.
// validation: the launch of the validation pass (zb_post_validate_finish) — timed separately.
void adamw_apply(float* theta, float* m, float* v, const float* g, bf16* shadow, int64_t n, int64_t n_wd,
                 int64_t n_shadow, float lr, float b1, float b2, float eps, float wd, const PvState* st,
                 bool validation, cudaStream_t s);
void pv_finish_apply(PvState* st, cudaStream_t s);  // advance t per the applied mode

}  // namespace zb
