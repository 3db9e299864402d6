// Microbenchmark: issue-to-completion cost of back-to-back tcgen05.mma (cta_group::1, bf16,
// K = 16) per instruction, by shape and operand source, one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2401_10241_b200/csrc mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace zb;

// BMN: B operand MN-major (the dK/dV "grads" products: B = Q_i / dO_i, K = queries);
// LDW: warps 4..7 stream tcgen05.ld of 64 columns per loop from TMEM while the MMAs run
template <int N, bool TS, bool BMN, bool LDW, bool LDW_ST = false>
__global__ void __launch_bounds__(256, 1) k_rate(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  if (warp == 0) sm100::tmem_alloc<512>(&tslot);
  sm100::fence_proxy_async();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = sm100::idesc_bf16(128, N, false, BMN);
    const uint32_t sa = sm100::smem_addr(smem);
    const uint64_t ad = sm100::smem_desc(sa, 16, 1024, sm100::kSwizzle128B);
    const uint64_t bd = BMN ? sm100::smem_desc(sa + 32768, 8192, 1024, sm100::kSwizzle128B)
                            : sm100::smem_desc(sa + 32768, 16, 1024, sm100::kSwizzle128B);
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = BMN ? (k & 3) * 2048 : (k & 3) * 32;
        if constexpr (TS)
          sm100::mma_bf16_ts(tb, tb + 256 + k * 8, sm100::desc_adv(bd, off), idesc, 1u);
        else
          sm100::mma_bf16_ss(tb, sm100::desc_adv(ad, off), sm100::desc_adv(bd, off), idesc, 1u);
      }
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    *reinterpret_cast<volatile uint32_t*>(&tslot + 0) = tb;  // keep
    stop = 1;
  }
  if (LDW && warp >= 4) {
    const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!*reinterpret_cast<volatile int*>(&stop)) {
      uint32_t r[32];
      sm100::tmem_ld32(tb + lo + 384, r);
      sm100::tmem_ld32(tb + lo + 416, r + 0);
      sm100::tmem_ld_wait();
      acc += r[0] + r[31];
      if (LDW_ST) {
        sm100::tmem_st16(tb + lo + 448, r);
        sm100::tmem_st16(tb + lo + 464, r + 16);
        sm100::tmem_st_wait();
      }
    }
    if (acc == 12345) out[1] = acc;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tb);
}

template <int N, bool TS, bool BMN = false, bool LDW = false, bool LDW_ST = false>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = k_rate<N, TS, BMN, LDW, LDW_ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int iters = 8192;
  k<<<148, 256, 65536 + 1024>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 256, 65536 + 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long clk; cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 128.0 * N * 16 * iters * 148;
  printf("%-10s N=%3d  %6.1f clk/mma (floor %5.1f)  %7.1f TFLOP/s  %s\n", name, N, double(clk) / iters,
         128.0 * N / 256, 2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<64, false>("SS");
  run<96, false>("SS");
  run<128, false>("SS");
  run<256, false>("SS");
  run<64, true>("TS");
  run<96, true>("TS");
  run<128, true>("TS");
  run<256, true>("TS");
  run<96, true, true>("TS-Bmn");
  run<64, true, true>("TS-Bmn");
  run<96, true, true, true>("TS-Bmn+ld");
  run<64, true, false, true>("TS+ld");
  run<64, false, false, true>("SS+ld");
  run<96, true, true, true, true>("TS-Bmn+ldst");
  run<64, false, false, true, true>("SS+ldst");
  return 0;
}
