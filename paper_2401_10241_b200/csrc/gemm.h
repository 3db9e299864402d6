// GEMM entry used by the stage passes (F, B and W contractions).
//
//   C[m, n] (op)= sum_k A(m, k) * B(n, k)
//   A(m, k) = a_mn ? A[k * lda + m] : A[m * lda + k]
//   B(n, k) = b_mn ? B[k * ldb + n] : B[n * ldb + k]
//
// F:  Y  = X  W^T   A = X  [T, n_in]  K-major,  B = W [n_out, n_in] K-major
// B:  dX = dY W     A = dY [T, n_out] K-major,  B = W [n_out, n_in] MN-major
// W:  dW += dY^T X  A = dY [T, n_out] MN-major, B = X [T, n_in]     MN-major
//
// bf16 mode runs the tcgen05 / TMEM / TMA kernel (gemm.cu); f32 mode (the
// 1e-5 parity mode of BASELINE.json) runs a SIMT FFMA kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace zb {

enum Epi : int32_t {
  EPI_STORE = 0,      // C = acc (+ bias)                       (activation dtype)
  EPI_BIAS_GELU = 1,  // C = acc + bias; aux = GeLU(acc + bias) (activation dtype)
  EPI_RESID = 2,      // C = aux + acc (+ bias)                 (activation dtype)
  EPI_GELU_BWD = 3,   // C = acc * GeLU'(aux)                   (activation dtype; C may alias aux)
  EPI_F32_ACC = 4,    // C(f32) = acc + (beta ? C : 0)
  EPI_F32_STORE = 5,  // C(f32) = acc
};

struct EpiArgs {
  void* C;
  int64_t ldc;
  const float* bias;
  void* aux;
  int64_t ldaux;
  int32_t beta;
  // ordered split-K of EPI_F32_ACC (set by gemm(), not by callers): K is cut into `splits`
  // ranges; split s of a tile reduce-adds into C only after split s-1 of the same tile
  // (per 32-row epilogue-warp region) has completed, so the f32 sums are formed in one
  // fixed order (bitwise reproducible).  flags[tile * 16 + region] is a monotone counter:
  // split s waits for >= flag_base + s and then stores flag_base + s + 1.
  int32_t splits = 1;
  int32_t flag_base = 0;
  int32_t* flags = nullptr;
  // W's bias gradient (EPI_F32_ACC only): bias_out[m] (beta ? += : =) sum_k A(m, k), the
  // column sums of dY (P:46's W of a bias).  The 2-CTA kernel forms them from the A tiles it
  // already streams (column-sum warps, gemm.cu); other paths fall back to ops.h bias_grad.
  float* bias_out = nullptr;
  float* bias_part = nullptr;  // set by gemm(): partial sums [splits * n-tiles, M]
  // set by gemm(): one arrival counter per 128-row block of M (zero between launches): the
  // column-sum warps that write the LAST partial of a block sum all of its partials in order
  int32_t* bias_tickets = nullptr;
  // set by gemm(): L2 cache hints of the 2-CTA kernel (ZB_GEMM_CHINT bits, measurement):
  // 1 = W's f32 output (unsplit) evict-first, 2 = operand tiles evict-last
  int32_t cache_hints = 0;
};

constexpr int kMaxSeg = 4;

struct GemmArgs {
  int32_t M, N, K;
  const void* A;
  int64_t lda;
  bool a_mn;
  const void* B;
  int64_t ldb;
  bool b_mn;
  int32_t epi;
  EpiArgs ep;
  // W-grouping: the K = T tokens of nseg microbatches as ONE
  // contraction — segment s covers K rows [s K/nseg, (s+1) K/nseg) of A and B at
  // A_seg[s] / B_seg[s] (same lda / ldb; MN-major W operands only; K/nseg % 64 == 0).
  // nseg <= 1: A / B as above.
  int32_t nseg = 1;
  const void* A_seg[kMaxSeg] = {nullptr, nullptr, nullptr, nullptr};
  const void* B_seg[kMaxSeg] = {nullptr, nullptr, nullptr, nullptr};
};

// Throws zb::CudaError on launch failure / unsupported shapes.
void gemm(const GemmArgs& g, DType dt, cudaStream_t stream);

// a CUDA-graph capture of launches on stream starts (ZB_RUN_GRAPH): restart the ordered
// split-K flag counters of that stream inside the graph
void gemm_graph_begin(cudaStream_t stream);

// number of SMs of the current device (cached)
int num_sms();

// 2-D bf16 (or f32) TMA descriptor (128B swizzle) over a row-major [outer, inner]
// view with leading dimension ld elements and box {box_inner, box_outer}.
CUtensorMap make_tmap(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                      uint32_t box_outer, bool f32 = false,
                      int swizzle = 128 /* 128 or 64 (bytes) */);

}  // namespace zb
