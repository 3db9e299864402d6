// Microbenchmark: MUFU ex2 throughput per SM sub-partition (FFMA + ex2.approx.ftz per element,
// 32 independent chains per thread), for 1, 2 and 4 warps per sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int MODE>
__global__ void k(int iters, float a, float b, float* out, long long* clk) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-2f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0) v[i] = ex2(fmaf(v[i], a, b));
      else v[i] = fmaf(v[i], a, b);  // FFMA only (the issue floor)
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int w : {4, 8, 16}) {
      const int iters = 2048;
      if (mode == 0) k<0><<<148, 32 * w>>>(iters, 0.5f, -1.f, o, c); else k<1><<<148, 32 * w>>>(iters, 0.5f, -1.f, o, c);
      if (mode == 0) k<0><<<148, 32 * w>>>(iters, 0.5f, -1.f, o, c); else k<1><<<148, 32 * w>>>(iters, 0.5f, -1.f, o, c);
      cudaDeviceSynchronize();
      long long clk; cudaMemcpy(&clk, c, 8, cudaMemcpyDeviceToHost);
      const double per_smsp = double(w) / 4 * iters * 32;  // warp-instructions of the measured kind per SMSP
      printf("%s warps/SMSP=%d: %.2f clk per warp-instr per SMSP -> %.1f lanes/clk/SM\n", mode ? "FFMA" : "FFMA+EX2",
             w / 4, clk / per_smsp, 4 * 32 * per_smsp / clk);
    }
  return 0;
}
