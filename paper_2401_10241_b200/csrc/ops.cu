// Row-wise / elementwise kernels (see ops.h).  HBM-bound: 16-byte vector
// loads, one CTA per row (or row chunk), warp-shuffle reductions, and
// deterministic two-level column reductions instead of atomics.
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "ops.h"
#include "zb.h"

namespace zb {

namespace {

constexpr int LN_THREADS = 256;

template <int NW>
__device__ __forceinline__ void block_sum2(float& a, float& b, float* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // protect red from the previous use
  if (l == 0) {
    red[w] = a;
    red[NW + w] = b;
  }
  __syncthreads();
  a = 0.f;
  b = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    a += red[i];
    b += red[NW + i];
  }
}

// ---------------------------------------------------------------- LayerNorm forward
template <typename T, int VPT>
__global__ void __launch_bounds__(LN_THREADS) k_ln_fwd(const T* __restrict__ x, const float* __restrict__ g,
                                                      const float* __restrict__ b, T* __restrict__ y,
                                                      float* __restrict__ mean, float* __restrict__ rstd, int h,
                                                      float eps) {
  pdl_wait();
  constexpr int NW = LN_THREADS / 32;
  __shared__ float red[2 * NW];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * h;
  const int nv = h / 8;
  float v[VPT][8];
  float s = 0.f, dummy = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * LN_THREADS;
    if (vi < nv) {
      Vec8<T>::load(xr + vi * 8, v[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[k][i];
    }
  }
  block_sum2<NW>(s, dummy, red);
  const float mu = s / h;
  float q = 0.f;
  dummy = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * LN_THREADS;
    if (vi < nv) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[k][i] - mu;
        q += d * d;
      }
    }
  }
  block_sum2<NW>(q, dummy, red);
  const float rs = rsqrtf(q / h + eps);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * LN_THREADS;
    if (vi < nv) {
      float gg[8], bb[8], o[8];
      Vec8<float>::load(g + vi * 8, gg);
      Vec8<float>::load(b + vi * 8, bb);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (v[k][i] - mu) * rs * gg[i] + bb[i];
      Vec8<T>::store(y + row * h + vi * 8, o);
    }
  }
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// warp-per-row variant for h <= 3072: no block barriers, 4 rows per 128-thread CTA
template <typename T, int VPL>
__global__ void __launch_bounds__(128) k_ln_fwd_warp(const T* __restrict__ x, const float* __restrict__ g,
                                                    const float* __restrict__ b, T* __restrict__ y,
                                                    float* __restrict__ mean, float* __restrict__ rstd, int rows, int h,
                                                    float eps) {
  pdl_wait();
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nv = h / 8;
  float v[VPL][8];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
      Vec8<T>::load(x + row * h + vi * 8, v[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += v[k][i];
    }
  }
  const float mu = warp_sum(sum) / h;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    if (lane + 32 * k < nv) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[k][i] - mu;
        q += d * d;
      }
    }
  }
  const float rs = rsqrtf(warp_sum(q) / h + eps);
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int vi = lane + 32 * k;
    if (vi < nv) {
      float gg[8], bb[8], o[8];
      Vec8<float>::load(g + vi * 8, gg);
      Vec8<float>::load(b + vi * 8, bb);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (v[k][i] - mu) * rs * gg[i] + bb[i];
      Vec8<T>::store(y + row * h + vi * 8, o);
    }
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// ---------------------------------------------------------------- LayerNorm backward
// dx only, one CTA per row (full parallelism over rows).  The residual-gradient
// stream stays f32 (resid and dx32, may be null); dx (activation dtype, may
// alias x) is the copy the dgrad / wgrad GEMMs consume.
template <typename T, int VPT>
__global__ void __launch_bounds__(LN_THREADS) k_ln_bwd_dx(const float* __restrict__ dy, const T* x,
                                                         const float* __restrict__ mean, const float* __restrict__ rstd,
                                                         const float* __restrict__ g, const float* resid, float* dx32,
                                                         T* dx, int h) {
  pdl_wait();
  constexpr int NW = LN_THREADS / 32;
  __shared__ float red[2 * NW];
  const int64_t r = blockIdx.x;
  const int nv = h / 8;
  const float mu = mean[r], rs = rstd[r];
  float xh[VPT][8], gh[VPT][8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * LN_THREADS;
    if (vi < nv) {
      float d[8], gw[8];
      Vec8<float>::load(dy + r * h + vi * 8, d);
      Vec8<T>::load(x + r * h + vi * 8, xh[k]);
      Vec8<float>::load(g + vi * 8, gw);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xh[k][i] = (xh[k][i] - mu) * rs;
        gh[k][i] = d[i] * gw[i];
        s1 += gh[k][i];
        s2 += gh[k][i] * xh[k][i];
      }
    }
  }
  block_sum2<NW>(s1, s2, red);  // orders every read of row r before the in-place writes
  const float m1 = s1 / h, m2 = s2 / h;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * LN_THREADS;
    if (vi < nv) {
      float o[8];
      if (resid != nullptr) {
        Vec8<float>::load(resid + r * h + vi * 8, o);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] += rs * (gh[k][i] - m1 - xh[k][i] * m2);
      if (dx32 != nullptr) Vec8<float>::store(dx32 + r * h + vi * 8, o);
      Vec8<T>::store(dx + r * h + vi * 8, o);
    }
  }
}

// Column reductions in one pass: a CTA owns VPC 8-column groups over ALL rows
// (kColThreads / VPC row lanes, each summing rows lane, lane + RL, ... in order),
// then a fixed binary tree over the row lanes in shared memory. Deterministic
// (fixed partition and order), no partial buffers, one launch. VPC is chosen so
// the grid covers the SMs (colred_vpc).
constexpr int kColThreads = 512;

template <int VPC, int NACC>
__device__ __forceinline__ void colred_tree(float (&acc)[NACC][8], float* sm) {
  constexpr int RL = kColThreads / VPC, W = VPC * 8 + 4;  // +4: spread banks
  const int vec = threadIdx.x % VPC, rl = threadIdx.x / VPC;
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[(q * RL + rl) * W + vec * 8 + i] = acc[q][i];
  __syncthreads();
#pragma unroll
  for (int stride = RL / 2; stride > 0; stride >>= 1) {
    if (rl < stride) {
#pragma unroll
      for (int q = 0; q < NACC; ++q)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[q][i] += sm[(q * RL + rl + stride) * W + vec * 8 + i];
          sm[(q * RL + rl) * W + vec * 8 + i] = acc[q][i];
        }
    }
    __syncthreads();
  }
}

// gamma / beta: gg (+)= sum_r dy * xhat, gb (+)= sum_r dy
template <typename T, int VPC>
__global__ void __launch_bounds__(kColThreads) k_ln_param_grads(const float* __restrict__ dy, const T* __restrict__ x,
                                                                const float* __restrict__ mean,
                                                                const float* __restrict__ rstd, float* __restrict__ gg,
                                                                float* __restrict__ gb, int rows, int h, int beta) {
  pdl_wait();
  constexpr int RL = kColThreads / VPC;
  extern __shared__ float colsm[];
  const int vec = threadIdx.x % VPC, rl = threadIdx.x / VPC;
  const int col = (blockIdx.x * VPC + vec) * 8;
  const bool valid = col < h;
  float acc[2][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[0][i] = acc[1][i] = 0.f;
  if (valid) {
    int r = rl;
    for (; r + 3 * RL < rows; r += 4 * RL) {  // four rows of loads in flight per thread
      float d[4][8], xv[4][8], mu[4], rs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + u * RL;
        Vec8<float>::load(dy + rr * h + col, d[u]);
        Vec8<T>::load(x + rr * h + col, xv[u]);
        mu[u] = mean[rr];
        rs[u] = rstd[rr];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[0][i] += d[u][i] * ((xv[u][i] - mu[u]) * rs[u]);
          acc[1][i] += d[u][i];
        }
    }
    for (; r < rows; r += RL) {
      float d[8], xv[8];
      Vec8<float>::load(dy + static_cast<int64_t>(r) * h + col, d);
      Vec8<T>::load(x + static_cast<int64_t>(r) * h + col, xv);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[0][i] += d[i] * ((xv[i] - mu) * rs);
        acc[1][i] += d[i];
      }
    }
  }
  colred_tree<VPC, 2>(acc, colsm);
  if (rl == 0 && valid) {
    if (beta) {
      float o[8];
      Vec8<float>::load(gg + col, o);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0][i] += o[i];
      Vec8<float>::load(gb + col, o);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[1][i] += o[i];
    }
    Vec8<float>::store(gg + col, acc[0]);
    Vec8<float>::store(gb + col, acc[1]);
  }
}

template <typename T, int VPC>
__global__ void __launch_bounds__(kColThreads) k_colsum(const T* __restrict__ y, int64_t ldy, float* __restrict__ out,
                                                        int rows, int n, int beta) {
  pdl_wait();
  constexpr int RL = kColThreads / VPC;
  extern __shared__ float colsm[];
  const int vec = threadIdx.x % VPC, rl = threadIdx.x / VPC;
  const int col = (blockIdx.x * VPC + vec) * 8;
  const bool valid = col < n;
  float acc[1][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[0][i] = 0.f;
  if (valid) {
    int r = rl;
    for (; r + 7 * RL < rows; r += 8 * RL) {
      float v[8][8];
#pragma unroll
      for (int u = 0; u < 8; ++u) Vec8<T>::load(y + static_cast<int64_t>(r + u * RL) * ldy + col, v[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[0][i] += v[u][i];
    }
    for (; r < rows; r += RL) {
      float v[8];
      Vec8<T>::load(y + static_cast<int64_t>(r) * ldy + col, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0][i] += v[i];
    }
  }
  colred_tree<VPC, 1>(acc, colsm);
  if (rl == 0 && valid) {
    if (beta) {
      float o[8];
      Vec8<float>::load(out + col, o);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0][i] += o[i];
    }
    Vec8<float>::store(out + col, acc[0]);
  }
}

// ---------------------------------------------------------------- embedding
template <typename T>
__global__ void k_embed_fwd(const int32_t* __restrict__ tok, const float* __restrict__ wte,
                            const float* __restrict__ wpe, T* __restrict__ x0, int s, int h) {
  pdl_wait();
  const int64_t row = blockIdx.x;
  const int64_t t = tok[row];
  const int pos = static_cast<int>(row % s);
  for (int vi = threadIdx.x; vi < h / 8; vi += blockDim.x) {
    float a[8], b[8];
    Vec8<float>::load(wte + t * h + vi * 8, a);
    Vec8<float>::load(wpe + static_cast<int64_t>(pos) * h + vi * 8, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] += b[i];
    Vec8<T>::store(x0 + row * h + vi * 8, a);
  }
}

// One-block bitonic sort of keys = tok * rows + pos (<= 8192 keys, padded with UINT32_MAX).
__global__ void __launch_bounds__(1024) k_sort_tokens(const int32_t* __restrict__ tok, uint32_t* __restrict__ keys,
                                                     int rows) {
  pdl_wait();
  constexpr int N = 8192;
  __shared__ uint32_t sk[N];
  for (int i = threadIdx.x; i < N; i += blockDim.x)
    sk[i] = i < rows ? static_cast<uint32_t>(tok[i]) * static_cast<uint32_t>(rows) + static_cast<uint32_t>(i)
                     : 0xFFFFFFFFu;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const uint32_t a = sk[i], b = sk[ixj];
          if ((a > b) == up) {
            sk[i] = b;
            sk[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < rows; i += blockDim.x) keys[i] = sk[i];
}

// One warp per sorted position that starts a segment: dwte[tok] += rows of the segment in position order.
template <typename T>
__global__ void k_embed_bwd_wte(const uint32_t* __restrict__ keys, const T* __restrict__ dx0, float* __restrict__ dwte,
                                int rows, int h) {
  pdl_wait();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  const uint32_t R = static_cast<uint32_t>(rows);
  const uint32_t tokw = keys[w] / R;
  if (w > 0 && keys[w - 1] / R == tokw) return;
  int end = w + 1;
  while (end < rows && keys[end] / R == tokw) ++end;
  for (int vi = lane; vi < h / 8; vi += 32) {
    float acc[8];
    Vec8<float>::load(dwte + static_cast<int64_t>(tokw) * h + vi * 8, acc);
    for (int i = w; i < end; ++i) {
      const int64_t pos = keys[i] % R;
      float v[8];
      Vec8<T>::load(dx0 + pos * h + vi * 8, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
    Vec8<float>::store(dwte + static_cast<int64_t>(tokw) * h + vi * 8, acc);
  }
}

template <typename T>
__global__ void k_embed_bwd_wpe(const T* __restrict__ dx0, float* __restrict__ dwpe, int rows, int s, int h) {
  pdl_wait();
  const int t = blockIdx.x;
  for (int vi = threadIdx.x; vi < h / 8; vi += blockDim.x) {
    float acc[8];
    Vec8<float>::load(dwpe + static_cast<int64_t>(t) * h + vi * 8, acc);
    for (int bi = 0; bi * s + t < rows; ++bi) {
      float v[8];
      Vec8<T>::load(dx0 + (static_cast<int64_t>(bi) * s + t) * h + vi * 8, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
    Vec8<float>::store(dwpe + static_cast<int64_t>(t) * h + vi * 8, acc);
  }
}

// ---------------------------------------------------------------- cross-entropy
template <typename T>
__global__ void __launch_bounds__(1024) k_ce(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                                            T* __restrict__ dlogits, float* __restrict__ loss_rows, int V,
                                            float inv_scale) {
  pdl_wait();
  __shared__ float red[32];
  __shared__ float bc;
  const int64_t row = blockIdx.x;
  const float* lr = logits + row * V;
  const int nv = V / 8;
  float mx = -INFINITY;
  for (int vi = threadIdx.x; vi < nv; vi += blockDim.x) {
    float v[8];
    Vec8<float>::load(lr + vi * 8, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) mx = fmaxf(mx, v[i]);
  }
  mx = warp_max(mx);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int i = 0; i < nw; ++i) m = fmaxf(m, red[i]);
    bc = m;
  }
  __syncthreads();
  mx = bc;
  float sum = 0.f;
  for (int vi = threadIdx.x; vi < nv; vi += blockDim.x) {
    float v[8];
    Vec8<float>::load(lr + vi * 8, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) sum += expf(v[i] - mx);
  }
  sum = warp_sum(sum);
  __syncthreads();
  if (l == 0) red[w] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < nw; ++i) s += red[i];
    bc = mx + logf(s);
  }
  __syncthreads();
  const float lse = bc;
  const int lab = labels[row];
  for (int vi = threadIdx.x; vi < nv; vi += blockDim.x) {
    float v[8];
    Vec8<float>::load(lr + vi * 8, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float pr = expf(v[i] - lse);
      v[i] = (pr - (vi * 8 + i == lab ? 1.f : 0.f)) * inv_scale;
    }
    Vec8<T>::store(dlogits + row * V + vi * 8, v);
  }
  if (threadIdx.x == 0) loss_rows[row] = lse - lr[lab];
}

__global__ void k_loss_reduce(const float* __restrict__ loss_rows, double* __restrict__ acc, int rows,
                              float inv_scale) {
  pdl_wait();
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) s += static_cast<double>(loss_rows[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
    *acc += t * static_cast<double>(inv_scale);
  }
}

template <typename T>
__global__ void k_convert(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  pdl_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

// ---------------------------------------------------------------- optimizer
__global__ void k_sumsq(const float* __restrict__ g, int64_t n, double* __restrict__ part, int32_t* __restrict__ nfp) {
  pdl_wait();
  __shared__ double red[32];
  __shared__ int nfr[32];
  double s = 0.0;
  int nf = 0;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = g4[i];
    float ls = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    nf |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    s += static_cast<double>(ls);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    s += static_cast<double>(g[i]) * g[i];
    nf |= !isfinite(g[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    nf |= __shfl_xor_sync(0xffffffffu, nf, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red[w] = s;
    nfr[w] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    int f = 0;
    for (int i = 0; i < (blockDim.x >> 5); ++i) {
      t += red[i];
      f |= nfr[i];
    }
    part[blockIdx.x] = t;
    nfp[blockIdx.x] = f;
  }
}

__global__ void k_sumsq_final(const double* __restrict__ part, const int32_t* __restrict__ nfp, int nb, PvState* st) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  double t = 0.0;
  int f = 0;
  for (int i = 0; i < nb; ++i) {
    t += part[i];
    f |= nfp[i];
  }
  st->local_sumsq = t;
  st->local_nf = f;
}

__global__ void k_pv_combine(PvState* st) {
  pdl_wait();
  st->partial_sumsq = st->partial_in_sumsq + st->local_sumsq;
  st->partial_nf = st->partial_in_nf | st->local_nf;
}

__device__ __forceinline__ double clip_coef(double sumsq, float clip) { return clip / (sqrt(sumsq) + 1e-6); }

// Optimistic decision on the partial state: skip on NaN, defer if the
// partial norm already needs clipping, else an unclipped step.  In sync mode
// the partial IS the full state and a clipped step is taken directly.
__global__ void k_pv_decide_first(PvState* st, float clip, int sync_mode) {
  pdl_wait();
  st->coef_rollback = 0.f;
  if (st->partial_nf) {
    st->first_action = ZB_ACT_SKIP;
    st->adam_mode = 0;
    st->coef_step = 0.f;
  } else {
    const double c = clip_coef(st->partial_sumsq, clip);
    if (c < 1.0) {
      if (sync_mode) {
        st->first_action = ZB_ACT_CLIPPED_STEP;
        st->adam_mode = 1;
        st->coef_step = static_cast<float>(c);
      } else {
        st->first_action = ZB_ACT_DEFER;
        st->adam_mode = 0;
        st->coef_step = 0.f;
      }
    } else {
      st->first_action = ZB_ACT_STEP;
      st->adam_mode = 1;
      st->coef_step = 1.f;
    }
  }
  st->coef_first = st->coef_step;
  st->final_action = ZB_ACT_NONE;
}

// Validation with the fully reduced state: roll back, redo, or take the deferred step.
__global__ void k_pv_decide_final(PvState* st, float clip) {
  pdl_wait();
  const int a = st->first_action;
  st->adam_mode = 0;
  st->final_action = ZB_ACT_NONE;
  if (st->full_nf) {
    if (a == ZB_ACT_STEP) {
      st->adam_mode = 2;
      st->coef_rollback = st->coef_first;
      st->final_action = ZB_ACT_ROLLBACK;
    }
    return;
  }
  const double c = clip_coef(st->full_sumsq, clip);
  if (c < 1.0) {
    if (a == ZB_ACT_STEP) {
      st->adam_mode = 3;
      st->coef_rollback = st->coef_first;
      st->coef_step = static_cast<float>(c);
      st->final_action = ZB_ACT_ROLLBACK_REDO;
    } else if (a == ZB_ACT_DEFER) {
      st->adam_mode = 1;
      st->coef_step = static_cast<float>(c);
      st->final_action = ZB_ACT_DEFERRED_STEP;
    }
  }
}

__global__ void k_pv_finish(PvState* st) {
  pdl_wait();
  const int mode = st->adam_mode;
  if (mode == 1) st->t += 1;
  if (mode == 2) st->t -= 1;
  st->adam_mode = 0;
}

// Algorithm 1, in f32 on the master copy.
__global__ void k_adamw(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
                        const float* __restrict__ g, bf16* __restrict__ shadow, int64_t n, int64_t n_wd,
                        int64_t n_shadow, float lr, float b1, float b2, float eps, float wd,
                        const PvState* __restrict__ st) {
  pdl_wait();
  const int mode = st->adam_mode;
  if (mode == 0) return;
  const int t0 = st->t;
  const float cs = st->coef_step, cr = st->coef_rollback;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float th = theta[i], mm = m[i], vv = v[i];
    const float gi = g[i];
    const float lw = i < n_wd ? lr * wd : 0.f;
    int t = t0;
    if (mode >= 2) {  // ROLLBACK(g * cr) at time stamp t
      const float gr = gi * cr;
      const float mh = mm / (1.f - powf(b1, static_cast<float>(t)));
      const float vh = vv / (1.f - powf(b2, static_cast<float>(t)));
      th = (th + lr * mh / (sqrtf(vh) + eps)) / (1.f - lw);
      mm = (mm - (1.f - b1) * gr) / b1;
      vv = (vv - (1.f - b2) * gr * gr) / b2;
      t -= 1;
    }
    if (mode == 1 || mode == 3) {  // STEP(g * cs)
      const float gs = gi * cs;
      t += 1;
      mm = b1 * mm + (1.f - b1) * gs;
      vv = b2 * vv + (1.f - b2) * gs * gs;
      const float mh = mm / (1.f - powf(b1, static_cast<float>(t)));
      const float vh = vv / (1.f - powf(b2, static_cast<float>(t)));
      th = th - lw * th - lr * mh / (sqrtf(vh) + eps);
    }
    theta[i] = th;
    m[i] = mm;
    v[i] = vv;
    if (i < n_shadow) shadow[i] = __float2bfloat16_rn(th);
  }
}

template <int VPT, typename F>
void ln_dispatch(int h, F&& f) {
  (void)VPT;
  const int vpt = (h / 8 + LN_THREADS - 1) / LN_THREADS;
  if (vpt <= 1) f(std::integral_constant<int, 1>());
  else if (vpt <= 2) f(std::integral_constant<int, 2>());
  else if (vpt <= 3) f(std::integral_constant<int, 3>());
  else if (vpt <= 4) f(std::integral_constant<int, 4>());
  else throw CudaError("layernorm: h > 8192 unsupported");
}

}  // namespace

// ---------------------------------------------------------------- host wrappers
template <int VPL>
static void ln_fwd_warp(DType dt, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                        int rows, int h, float eps, cudaStream_t st) {
  const int blocks = (rows + 3) / 4;
  if (dt == DT_BF16)
    launch(PDL_OPS, k_ln_fwd_warp<bf16, VPL>, blocks, 128, 0, st, static_cast<const bf16*>(x), g, b, static_cast<bf16*>(y), mean,
                                                     rstd, rows, h, eps);
  else
    launch(PDL_OPS, k_ln_fwd_warp<float, VPL>, blocks, 128, 0, st, static_cast<const float*>(x), g, b, static_cast<float*>(y),
                                                      mean, rstd, rows, h, eps);
}

void layernorm_fwd(DType dt, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                   int rows, int h, float eps, cudaStream_t st) {
  if (rows <= 0) return;
  if (h % 8) throw CudaError("layernorm: h must be a multiple of 8");
  const int vpl = (h / 8 + 31) / 32;
  if (vpl <= 2) {
    ln_fwd_warp<2>(dt, x, g, b, y, mean, rstd, rows, h, eps, st);
  } else if (vpl <= 6) {
    ln_fwd_warp<6>(dt, x, g, b, y, mean, rstd, rows, h, eps, st);
  } else if (vpl <= 9) {
    ln_fwd_warp<9>(dt, x, g, b, y, mean, rstd, rows, h, eps, st);
  } else if (vpl <= 12) {
    ln_fwd_warp<12>(dt, x, g, b, y, mean, rstd, rows, h, eps, st);
  } else {
    ln_dispatch<0>(h, [&](auto V) {
      constexpr int VPT = decltype(V)::value;
      if (dt == DT_BF16)
        launch(PDL_OPS, k_ln_fwd<bf16, VPT>, rows, LN_THREADS, 0, st, static_cast<const bf16*>(x), g, b, static_cast<bf16*>(y),
                                                         mean, rstd, h, eps);
      else
        launch(PDL_OPS, k_ln_fwd<float, VPT>, rows, LN_THREADS, 0, st, static_cast<const float*>(x), g, b, static_cast<float*>(y),
                                                          mean, rstd, h, eps);
    });
  }
  ZB_LAUNCH_CHECK();
}

// 8-column groups per CTA: the widest of 1, 2, 4, 8 that still gives >= ~1 CTA per SM
static int colred_vpc(int n) {
  const int groups = n / 8;
  int vpc = 8;
  while (vpc > 1 && groups / vpc < 140) vpc >>= 1;
  return vpc;
}

template <int VPC>
static size_t colred_smem(int nacc) {
  return static_cast<size_t>(nacc) * (kColThreads / VPC) * (VPC * 8 + 4) * sizeof(float);
}

template <typename F>
static void colred_dispatch(int vpc, F&& f) {
  switch (vpc) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 4: return f(std::integral_constant<int, 4>{});
    default: return f(std::integral_constant<int, 8>{});
  }
}

template <typename K>
static void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) ZB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void layernorm_bwd(DType dt, const float* dy, const void* x, const float* mean, const float* rstd, const float* g,
                   const float* resid, float* dx32, void* dx, float* gg, float* gb, int beta, int rows, int h,
                   cudaStream_t st) {
  if (rows <= 0) return;
  // 1) gamma / beta grads (reads x before step 2 may overwrite it in place)
  const int vpc = colred_vpc(h);
  colred_dispatch(vpc, [&](auto V) {
    constexpr int VPC = decltype(V)::value;
    const int grid = (h / 8 + VPC - 1) / VPC;
    const size_t sm = colred_smem<VPC>(2);
    if (dt == DT_BF16) {
      allow_smem(k_ln_param_grads<bf16, VPC>, sm);
      launch(PDL_OPS, k_ln_param_grads<bf16, VPC>, grid, kColThreads, sm, st, dy, static_cast<const bf16*>(x), mean, rstd, gg, gb,
                                                                 rows, h, beta);
    } else {
      allow_smem(k_ln_param_grads<float, VPC>, sm);
      launch(PDL_OPS, k_ln_param_grads<float, VPC>, grid, kColThreads, sm, st, dy, static_cast<const float*>(x), mean, rstd, gg,
                                                                  gb, rows, h, beta);
    }
  });
  ZB_LAUNCH_CHECK();
  // 2) dx, one CTA per row (dy arrives in f32: the dLN GEMM epilogue keeps full precision)
  ln_dispatch<0>(h, [&](auto V) {
    constexpr int VPT = decltype(V)::value;
    if (dt == DT_BF16)
      launch(PDL_OPS, k_ln_bwd_dx<bf16, VPT>, rows, LN_THREADS, 0, st, dy, static_cast<const bf16*>(x), mean, rstd, g, resid, dx32,
                                                          static_cast<bf16*>(dx), h);
    else
      launch(PDL_OPS, k_ln_bwd_dx<float, VPT>, rows, LN_THREADS, 0, st, dy, static_cast<const float*>(x), mean, rstd, g, resid,
                                                           dx32, static_cast<float*>(dx), h);
  });
  ZB_LAUNCH_CHECK();
}

void bias_grad(DType dt, const void* y, int64_t ldy, float* out, int rows, int n, int beta, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return;
  colred_dispatch(colred_vpc(n), [&](auto V) {
    constexpr int VPC = decltype(V)::value;
    const int grid = (n / 8 + VPC - 1) / VPC;
    const size_t sm = colred_smem<VPC>(1);
    if (dt == DT_BF16) {
      allow_smem(k_colsum<bf16, VPC>, sm);
      launch(PDL_OPS, k_colsum<bf16, VPC>, grid, kColThreads, sm, st, static_cast<const bf16*>(y), ldy, out, rows, n, beta);
    } else {
      allow_smem(k_colsum<float, VPC>, sm);
      launch(PDL_OPS, k_colsum<float, VPC>, grid, kColThreads, sm, st, static_cast<const float*>(y), ldy, out, rows, n, beta);
    }
  });
  ZB_LAUNCH_CHECK();
}

void embed_fwd(DType dt, const int32_t* tok, const float* wte, const float* wpe, void* x0, int rows, int s, int h,
               cudaStream_t st) {
  if (rows <= 0) return;
  const int thr = h / 8 < 256 ? ((h / 8 + 31) / 32) * 32 : 256;
  if (dt == DT_BF16)
    launch(PDL_OPS, k_embed_fwd<bf16>, rows, thr, 0, st, tok, wte, wpe, static_cast<bf16*>(x0), s, h);
  else
    launch(PDL_OPS, k_embed_fwd<float>, rows, thr, 0, st, tok, wte, wpe, static_cast<float*>(x0), s, h);
  ZB_LAUNCH_CHECK();
}

void embed_bwd(DType dt, const int32_t* tok, const void* dx0, float* dwte, float* dwpe, uint32_t* keys, int rows,
               int s, int h, cudaStream_t st) {
  if (rows <= 0) return;
  if (rows > 8192) throw CudaError("embed_bwd: at most 8192 tokens per microbatch");
  launch(PDL_OPS, k_sort_tokens, 1, 1024, 0, st, tok, keys, rows);
  ZB_LAUNCH_CHECK();
  const int blocks = (rows * 32 + 255) / 256;
  const int thr = h / 8 < 256 ? ((h / 8 + 31) / 32) * 32 : 256;
  if (dt == DT_BF16) {
    launch(PDL_OPS, k_embed_bwd_wte<bf16>, blocks, 256, 0, st, keys, static_cast<const bf16*>(dx0), dwte, rows, h);
    launch(PDL_OPS, k_embed_bwd_wpe<bf16>, s < rows ? s : rows, thr, 0, st, static_cast<const bf16*>(dx0), dwpe, rows, s, h);
  } else {
    launch(PDL_OPS, k_embed_bwd_wte<float>, blocks, 256, 0, st, keys, static_cast<const float*>(dx0), dwte, rows, h);
    launch(PDL_OPS, k_embed_bwd_wpe<float>, s < rows ? s : rows, thr, 0, st, static_cast<const float*>(dx0), dwpe, rows, s, h);
  }
  ZB_LAUNCH_CHECK();
}

void cross_entropy(DType dt, const float* logits, const int32_t* labels, void* dlogits, float* loss_rows,
                   double* loss_acc, int rows, int V, float inv_scale, cudaStream_t st) {
  if (rows <= 0) return;
  if (V % 8) throw CudaError("cross_entropy: V must be a multiple of 8");
  if (dt == DT_BF16)
    launch(PDL_OPS, k_ce<bf16>, rows, 1024, 0, st, logits, labels, static_cast<bf16*>(dlogits), loss_rows, V, inv_scale);
  else
    launch(PDL_OPS, k_ce<float>, rows, 1024, 0, st, logits, labels, static_cast<float*>(dlogits), loss_rows, V, inv_scale);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_loss_reduce, 1, 1024, 0, st, loss_rows, loss_acc, rows, inv_scale);
  ZB_LAUNCH_CHECK();
}

void convert_rows(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st) {
  convert_f32(dt, src, dst, n, st);
}

void convert_f32(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  if (dt == DT_BF16) launch(PDL_OPS, k_convert<bf16>, blocks, 256, 0, st, src, static_cast<bf16*>(dst), n);
  else launch(PDL_OPS, k_convert<float>, blocks, 256, 0, st, src, static_cast<float*>(dst), n);
  ZB_LAUNCH_CHECK();
}

void grad_norm(const float* g, int64_t n, double* part, int32_t* nf_part, PvState* pst, cudaStream_t st) {
  launch(PDL_OPS, k_sumsq, kNormBlocks, 512, 0, st, g, n, part, nf_part);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_sumsq_final, 1, 32, 0, st, part, nf_part, kNormBlocks, pst);
  ZB_LAUNCH_CHECK();
}

void pv_combine(PvState* pst, cudaStream_t st) {
  launch(PDL_OPS, k_pv_combine, 1, 1, 0, st, pst);
  ZB_LAUNCH_CHECK();
}
void pv_decide_first(PvState* pst, float clip, int sync_mode, cudaStream_t st) {
  launch(PDL_OPS, k_pv_decide_first, 1, 1, 0, st, pst, clip, sync_mode);
  ZB_LAUNCH_CHECK();
}
void pv_decide_final(PvState* pst, float clip, cudaStream_t st) {
  launch(PDL_OPS, k_pv_decide_final, 1, 1, 0, st, pst, clip);
  ZB_LAUNCH_CHECK();
}
void pv_finish_apply(PvState* pst, cudaStream_t st) {
  launch(PDL_OPS, k_pv_finish, 1, 1, 0, st, pst);
  ZB_LAUNCH_CHECK();
}
void adamw_apply(float* theta, float* m, float* v, const float* g, bf16* shadow, int64_t n, int64_t n_wd,
                 int64_t n_shadow, float lr, float b1, float b2, float eps, float wd, const PvState* pst,
                 cudaStream_t st) {
  const int blocks = static_cast<int>(std::min<int64_t>((n + 511) / 512, 148 * 8));
  launch(PDL_OPS, k_adamw, blocks, 512, 0, st, theta, m, v, g, shadow, n, n_wd, n_shadow, lr, b1, b2, eps, wd, pst);
  ZB_LAUNCH_CHECK();
}

}  // namespace zb
