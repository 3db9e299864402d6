// Microbenchmark: tcgen05.mma issue cost when the issuing warp shares its SM sub-partition
// with busy ALU warps (the attention kernels' situation).  M=128, N=64, TS, K=16.
//   MODE 0: lane 0 alone issues (if (lane == 0) { ... })
//   MODE 1: the whole warp runs the loop, descriptors warp-uniform, elect.sync per MMA
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace zb;
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\tselp.u32 %0, 1, 0, q;\n\t}" : "=r"(p));
  return p != 0;
}
template <int MODE, int BUSY>
__global__ void __launch_bounds__(384, 1) k(int iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); stop = 0; }
  if (warp == 0) sm100::tmem_alloc<512>(&tslot);
  sm100::fence_proxy_async();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tb = tslot;
  constexpr uint32_t idesc = sm100::idesc_bf16(128, 64, false, false);
  if (warp == 1) {
    const uint32_t sa = sm100::smem_addr(smem);
    if (MODE == 0) {
      if (lane == 0) {
        const uint64_t bd = sm100::smem_desc(sa + 32768, 16, 1024, sm100::kSwizzle128B);
        long long t0 = clock64();
        for (int it = 0; it < iters; it += 8) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            sm100::mma_bf16_ts(tb + (it & 8) * 8, tb + 256 + kk * 8, sm100::desc_adv(bd, (kk & 3) * 32), idesc, 1u);
        }
        sm100::mma_commit(&bar);
        sm100::mbar_wait(&bar, 0);
        if (blockIdx.x == 0) out[0] = clock64() - t0;
        stop = 1;
      }
    } else {
      const uint64_t bd = sm100::smem_desc(sa + 32768, 16, 1024, sm100::kSwizzle128B);
      long long t0 = clock64();
      for (int it = 0; it < iters; it += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          if (elect_one())
            sm100::mma_bf16_ts(tb + (it & 8) * 8, tb + 256 + kk * 8, sm100::desc_adv(bd, (kk & 3) * 32), idesc, 1u);
        __syncwarp();
      }
      if (elect_one()) sm100::mma_commit(&bar);
      __syncwarp();
      sm100::mbar_wait(&bar, 0);
      if (blockIdx.x == 0 && lane == 0) out[0] = clock64() - t0;
      if (lane == 0) stop = 1;
    }
  } else if (warp >= 4 && warp < 4 + BUSY) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
    while (!*reinterpret_cast<volatile int*>(&stop)) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaf(v[i], 0.999f, 0.5f);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
    sink[blockIdx.x * 384 + threadIdx.x] = s;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tb);
}
template <int MODE, int BUSY>
void run() {
  long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 148 * 384 * 4);
  auto kk = k<MODE, BUSY>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int rep = 0; rep < 2; ++rep) kk<<<148, 384, 65536 + 1024>>>(4096, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long clk; cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
  printf("MODE %d (%s) busy warps %d: %.1f clk/mma  %s\n", MODE, MODE ? "warp+elect" : "lane0", BUSY, clk / 4096.0,
         cudaGetErrorString(e));
  cudaFree(d); cudaFree(s);
}
int main() {
  run<0, 0>(); run<1, 0>();
  run<0, 8>(); run<1, 8>();
  return 0;
}
