// Causal multi-head attention forward / backward (the attention part of F and
// B; attention has no weights, so it has no W part — SURVEY C3 reading).
//
// qkv  [b*s, 3h]: Q, K, V column blocks, head k at columns k*d of each block
// o    [b*s, h]   heads concatenated
// lse  [b, a, s]  f32 natural-log sum-exp of the scaled scores (saved by F for B)
// dqkv [b*s, 3h]  written (not accumulated) by attention_bwd
// delta[b, a, s]  f32 scratch: rowsum(dO * O)
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace zb {

struct AttnShape {
  int b, s, a, d;
};

void attention_fwd(const AttnShape& sh, DType dt, const void* qkv, void* o, float* lse, cudaStream_t st);
void attention_bwd(const AttnShape& sh, DType dt, const void* qkv, const void* o, const void* dout, const float* lse,
                   void* dqkv, float* delta, cudaStream_t st);

}  // namespace zb
