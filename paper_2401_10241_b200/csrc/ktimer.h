// Optional per-kernel-class CUDA-event timing (zb_dbg_kernel_timing): when on,
// every GEMM / attention / HBM-bound op launch is bracketed by events on its own stream and
// its algorithmic FLOPs are recorded; bench.py reads the totals after the
// timed region to report the dominant kernel's achieved TFLOP/s live.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace zb {

// kernel launches of the library since the last reset (common.cuh launch())
int64_t launch_count(bool reset);
// kernel nodes of a replayed CUDA graph (counted like launches)
void add_launches(int64_t n);

namespace ktimer {

// GEMM / attention classes carry algorithmic FLOPs; the HBM-bound classes (LN_*,
// BIAS_GRAD, CE, OPT, MISC) carry algorithmic BYTES in the same field.
enum Class : int {
  GEMM = 0, ATTN_FWD = 1, ATTN_BWD = 2, GEMM_F = 3, GEMM_B = 4, GEMM_W = 5,
  LN_FWD = 6, LN_BWD = 7, LN_PARAM = 8, BIAS_GRAD = 9, CE = 10, OPT = 11, MISC = 12, OPT_VALIDATE = 13,
  N_CLASSES = 14
};

bool enabled();
void set_enabled(bool on);
// returns an index to pass to stop(), or -1 when timing is off
int start(int cls, double flops, cudaStream_t s);
void stop(int idx, cudaStream_t s);
// synchronises pending events and accumulates; then returns totals of a class
void read(int cls, double* ms, double* flops, int64_t* launches);
void reset();

}  // namespace ktimer
}  // namespace zb
