// Shared device/host helpers for the zb library (sm_100a only).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a only"
#endif

namespace zb {

typedef __nv_bfloat16 bf16;

enum DType : int32_t { DT_BF16 = 0, DT_F32 = 1 };

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define ZB_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t e__ = (x);                                                              \
    if (e__ != cudaSuccess)                                                             \
      throw ::zb::CudaError(std::string(#x) + " -> " + cudaGetErrorString(e__) + " @ " + \
                            __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

#define ZB_LAUNCH_CHECK() ZB_CUDA(cudaGetLastError())

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- launches ----------------------------------------------------------------
// Every kernel of the library is launched through launch(): counted
// (zb_dbg_launch_count) and, when enabled for its class, launched with
// programmatic dependent launch (PDL) so its prologue can overlap the tail of
// the previous kernel on the stream.  Contract of every kernel: pdl_wait()
// before its first global-memory access (griddepcontrol.wait returns once the
// previous grid has completed and its writes are visible; a no-op without
// PDL).  Only the TMEM kernels (GEMM, attention) trigger early, and only AFTER
// their TMEM allocation, so a dependent CTA can never hold TMEM that a CTA of
// an earlier grid still has to allocate; the HBM-bound kernels trigger
// implicitly at exit.  (Early triggers in the HBM-bound kernels deadlocked the
// 1.5B step on B200 — cause not identified.)  PDL of the TMEM classes measured
// no gain in round 1; with the persistent attention kernels of round 2 it gives
// +0.7% on the 6.2B step (28.2k -> 28.4k tokens/s) and the GPU suite passes with
// it, so the default is GEMM | attention.
// ZB_PDL=<mask>: PDL for kernel classes (1 GEMM, 2 attention, 4 others); 0 = off.
// ZB_TRACE_LAUNCH=1 prints every kernel when the stream reaches it (debugging;
// serialises).
enum PdlClass : int { PDL_GEMM = 1, PDL_ATTN = 2, PDL_OPS = 4 };
void note_launch();
bool pdl_enabled(int cls);
void trace_launch(const void* kern, cudaStream_t st);

template <typename... KArgs, typename... Args>
inline void launch(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(cls) ? 1 : 0;
  ZB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  note_launch();
  trace_launch(reinterpret_cast<const void*>(kern), st);
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- element conversion ----------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// 8-element vector load/store in float registers (16 B for bf16, 32 B for f32).
template <typename T> struct Vec8;
template <> struct Vec8<bf16> {
  static __device__ __forceinline__ void load(const bf16* p, float* v) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void store(bf16* p, const float* v) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// tanh-GeLU (SURVEY C1 reading) and its derivative, fp32.
__device__ __forceinline__ float gelu_f(float x) {
  const float c = 0.7978845608028654f;
  float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * x * (1.f + t);
}
// Hardware tanh (MUFU.TANH, |rel err| ~ 2^-11): used only where the result is
// rounded to bf16 (2^-9) anyway; the f32 parity mode keeps tanhf.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.f + tanh_approx(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanh_approx(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * x * x);
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c = 0.7978845608028654f;
  float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * x * x);
}

}  // namespace zb
