// Row-wise / elementwise kernels (see ops.h).  HBM-bound: 16-byte vector
// loads, one CTA per row (or row chunk), warp-shuffle reductions, and
// deterministic two-level column reductions instead of atomics.
#include <math.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <type_traits>

#include "ktimer.h"
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
template <typename T, int VPT, int NT = LN_THREADS>
__global__ void __launch_bounds__(NT) k_ln_fwd(const T* __restrict__ x, const float* __restrict__ g,
                                                      const float* __restrict__ b, T* __restrict__ y,
                                                      float* __restrict__ mean, float* __restrict__ rstd, int h,
                                                      float eps) {
  pdl_wait();
  constexpr int NW = NT / 32;
  __shared__ float red[2 * NW];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * h;
  const int nv = h / 8;
  float v[VPT][8];
  float s = 0.f, dummy = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int vi = threadIdx.x + k * NT;
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
    const int vi = threadIdx.x + k * NT;
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
    const int vi = threadIdx.x + k * NT;
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

// bf16, persistent warp-per-row with a one-row prefetch: each warp walks rows
// w, w + W, ... (W = all warps of the grid) and issues the loads of its next row before
// reducing / normalising / storing the current one, so every warp keeps a row of loads
// in flight for the whole kernel (the one-row-per-warp kernel was latency-bound:
// load -> reduce -> store with nothing outstanding in between, 33% of HBM bandwidth).
// Rows are held packed (16 B per 8 columns); gamma / beta come through L1.
template <int VPL>
__global__ void __launch_bounds__(128, 4) k_ln_fwd_rows(const bf16* __restrict__ x, const float* __restrict__ g,
                                                    const float* __restrict__ b, bf16* __restrict__ y,
                                                    float* __restrict__ mean, float* __restrict__ rstd, int rows, int h,
                                                    float eps) {
  pdl_wait();
  // gamma / beta staged once per (persistent) CTA: read from shared memory per row instead of
  // L2 (the dependent global loads of the output loop were the long-scoreboard stalls)
  extern __shared__ float gb_sm[];  // [2][h]
  for (int i = threadIdx.x; i < h / 4; i += blockDim.x) {
    reinterpret_cast<float4*>(gb_sm)[i] = reinterpret_cast<const float4*>(g)[i];
    reinterpret_cast<float4*>(gb_sm + h)[i] = reinterpret_cast<const float4*>(b)[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 4;
  int64_t row = static_cast<int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int nv = h / 8;
  uint4 cur[VPL], nxt[VPL];
  auto load = [&](int64_t r, uint4* dst) {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int vi = lane + 32 * k;
      dst[k] = vi < nv ? __ldcs(reinterpret_cast<const uint4*>(x + r * h + vi * 8)) : make_uint4(0, 0, 0, 0);
    }
  };
  if (row < rows) load(row, cur);
  for (; row < rows; row += stride) {
    if (row + stride < rows) load(row + stride, nxt);
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(hv[i]);
        sum += f.x + f.y;
      }
    }
    const float mu = warp_sum(sum) / h;
    float sq = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (lane + 32 * k < nv) {
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(hv[i]);
          sq += (f.x - mu) * (f.x - mu) + (f.y - mu) * (f.y - mu);
        }
      }
    }
    const float rs = rsqrtf(warp_sum(sq) / h + eps);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int vi = lane + 32 * k;
      if (vi < nv) {
        float gg[8], bb[8], o[8];
        Vec8<float>::load(gb_sm + vi * 8, gg);
        Vec8<float>::load(gb_sm + h + vi * 8, bb);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[k]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(hv[i]);
          o[2 * i] = (f.x - mu) * rs * gg[2 * i] + bb[2 * i];
          o[2 * i + 1] = (f.y - mu) * rs * gg[2 * i + 1] + bb[2 * i + 1];
        }
        Vec8<bf16>::store(y + row * h + vi * 8, o);
      }
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) cur[k] = nxt[k];
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

// Coalesced two-phase column reductions (bias grads, LayerNorm gamma / beta grads).
// CTA (ct, rb) owns a 256-column tile ct (lane l of every warp: columns 8l..8l+7, so a
// warp reads 512 contiguous bytes of a bf16 row) over row block rb; its 8 warps take rows
// w, w+8, ... with 4 rows of loads in flight.  Warp partials meet in shared memory (fixed
// order), the CTA's partial row goes to scratch, and the LAST CTA of the column tile
// (atomic ticket) sums the RB partial rows in row-block order and applies beta.  The
// result is deterministic (fixed partition, fixed summation order) and needs one launch.
// MODE 0: out0 (+)= sum_r y[r];  MODE 1: out0 (+)= sum_r dy[r] * xhat[r], out1 (+)= sum_r dy[r].
constexpr int kCR_THREADS = 256, kCR_COLS = 256;

template <int MODE, typename T>
__global__ void __launch_bounds__(kCR_THREADS) k_colred2(const T* __restrict__ y, int64_t ldy,
                                                         const float* __restrict__ dy, const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, float* __restrict__ out0,
                                                         float* __restrict__ out1, float* __restrict__ part,
                                                         int32_t* __restrict__ tickets, int rows, int n, int rpb,
                                                         int beta) {
  pdl_wait();
  constexpr int NACC = MODE == 0 ? 1 : 2;
  constexpr int U = MODE == 0 ? 8 : 4;  // rows of loads in flight per thread (128 / 192 B)
  __shared__ float sm[NACC][8][kCR_COLS];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ct = blockIdx.x, rb = blockIdx.y, RB = gridDim.y;
  const int col = ct * kCR_COLS + lane * 8;
  const bool valid = col < n;
  const int r0 = rb * rpb, r1 = min(rows, r0 + rpb);
  float acc[NACC][8];
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[q][i] = 0.f;
  if (valid) {
    for (int r = r0 + warp; r < r1; r += 8 * U) {  // U rows per batch, tail rows masked (loads stay batched)
      float v[U][8], d[U][8], mu[U], rs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + 8 * u;
        if (rr < r1) {
          Vec8<T>::load(y + rr * ldy + col, v[u]);
          if (MODE == 1) {
            Vec8<float>::load(dy + rr * ldy + col, d[u]);
            mu[u] = mean[rr];
            rs[u] = rstd[rr];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[u][i] = d[u][i] = 0.f;
          mu[u] = rs[u] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (MODE == 0) {
            acc[0][i] += v[u][i];
          } else {
            acc[0][i] += d[u][i] * ((v[u][i] - mu[u]) * rs[u]);
            acc[1][i] += d[u][i];
          }
        }
    }
  }
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[q][warp][lane * 8 + i] = acc[q][i];
  __syncthreads();
  const int c = ct * kCR_COLS + threadIdx.x;  // thread t writes column t of the CTA's partial row
  if (c < n) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += sm[q][w][threadIdx.x];
      part[(static_cast<int64_t>(q) * RB + rb) * n + c] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&tickets[ct], 1) == RB - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA of the tile: warp w sums partial rows w, w+8, ... of lane's 8 columns (all its
  // loads in flight at once), then the 8 warp sums meet in shared memory in warp order
  float fin[NACC][8];
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) fin[q][i] = 0.f;
  if (valid) {
#pragma unroll 4
    for (int bb = warp; bb < RB; bb += 8)
#pragma unroll
      for (int q = 0; q < NACC; ++q) {
        const float* src = part + (static_cast<int64_t>(q) * RB + bb) * n + col;
        const float4 lo = __ldcg(reinterpret_cast<const float4*>(src));
        const float4 hi = __ldcg(reinterpret_cast<const float4*>(src + 4));
        fin[q][0] += lo.x; fin[q][1] += lo.y; fin[q][2] += lo.z; fin[q][3] += lo.w;
        fin[q][4] += hi.x; fin[q][5] += hi.y; fin[q][6] += hi.z; fin[q][7] += hi.w;
      }
  }
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[q][warp][lane * 8 + i] = fin[q][i];
  __syncthreads();
  if (c < n) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += sm[q][w][threadIdx.x];
      float* o = q == 0 ? out0 : out1;
      o[c] = beta ? o[c] + t : t;
    }
  }
  if (threadIdx.x == 0) tickets[ct] = 0;  // ready for the next launch on this stream
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

// Algorithm 1, in f32 on the master copy.  Four elements per
// thread (16-B loads / stores; the flat regions [0, n_wd) and [0, n_shadow) start at
// 64-element aligned offsets, so a float4 never straddles a boundary); the bias
// corrections 1 - beta^t are computed once per thread (the same f32 values the
// per-element form computed, so results are unchanged bit for bit).
__global__ void k_adamw(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
                        const float* __restrict__ g, bf16* __restrict__ shadow, int64_t n, int64_t n_wd,
                        int64_t n_shadow, float lr, float b1, float b2, float eps, float wd,
                        const PvState* __restrict__ st) {
  pdl_wait();
  const int mode = st->adam_mode;
  if (mode == 0) return;  // predicated off: no traffic
  const int t0 = st->t;
  const float cs = st->coef_step, cr = st->coef_rollback;
  // rollback at stamp t0, step at stamp t0 (mode 1) or t0 after the rollback's t0 - 1 (mode 3)
  const float rb1 = 1.f - powf(b1, static_cast<float>(t0)), rb2 = 1.f - powf(b2, static_cast<float>(t0));
  const int ts = mode == 3 ? t0 : t0 + 1;
  const float sb1 = 1.f - powf(b1, static_cast<float>(ts)), sb2 = 1.f - powf(b2, static_cast<float>(ts));
  const int64_t n4 = n / 4;
  float4* th4 = reinterpret_cast<float4*>(theta);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n4;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = 4 * q;
    float4 TH = th4[q], MM = m4[q], VV = v4[q];
    const float4 G = g4[q];
    const float lw = i < n_wd ? lr * wd : 0.f;
    float* th = &TH.x;
    float* mm = &MM.x;
    float* vv = &VV.x;
    const float* gi = &G.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (mode >= 2) {  // ROLLBACK(g * cr) at time stamp t0
        const float gr = gi[e] * cr;
        const float mh = mm[e] / rb1;
        const float vh = vv[e] / rb2;
        th[e] = (th[e] + lr * mh / (sqrtf(vh) + eps)) / (1.f - lw);
        mm[e] = (mm[e] - (1.f - b1) * gr) / b1;
        vv[e] = (vv[e] - (1.f - b2) * gr * gr) / b2;
      }
      if (mode == 1 || mode == 3) {  // STEP(g * cs)
        const float gs = gi[e] * cs;
        mm[e] = b1 * mm[e] + (1.f - b1) * gs;
        vv[e] = b2 * vv[e] + (1.f - b2) * gs * gs;
        const float mh = mm[e] / sb1;
        const float vh = vv[e] / sb2;
        th[e] = th[e] - lw * th[e] - lr * mh / (sqrtf(vh) + eps);
      }
    }
    th4[q] = TH;
    m4[q] = MM;
    v4[q] = VV;
    if (i < n_shadow) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(TH.x, TH.y), hi = __floats2bfloat162_rn(TH.z, TH.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(shadow + i) = pk;
    }
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
// Per-stream scratch of the two-phase column reductions (partial rows + column-tile
// tickets, zeroed once; the last CTA of a tile re-zeroes its ticket), so concurrent
// streams never share tickets.
struct ColredScratch {
  float* part = nullptr;
  int32_t* tickets = nullptr;
};
static constexpr int64_t kColredPartFloats = 4 << 20;  // 16 MB
static constexpr int kColredTickets = 4096;
static ColredScratch colred_scratch(cudaStream_t st) {
  static std::mutex mu;
  static std::map<cudaStream_t, ColredScratch> bufs;
  std::lock_guard<std::mutex> lock(mu);
  ColredScratch& c = bufs[st];
  if (!c.part) {
    ZB_CUDA(cudaMalloc(&c.part, sizeof(float) * kColredPartFloats));
    ZB_CUDA(cudaMalloc(&c.tickets, sizeof(int32_t) * kColredTickets));
    // on the stream itself: a legacy-stream cudaMemset is not ordered before work on a
    // non-blocking stream (the first launch could read uninitialised tickets)
    ZB_CUDA(cudaMemsetAsync(c.tickets, 0, sizeof(int32_t) * kColredTickets, st));
  }
  return c;
}

// grid of the two-phase reduction: ~2 CTAs per SM (warps keep 8 / 4 rows of loads in
// flight), a multiple of 64 rows per CTA
static void colred2_grid(int rows, int n, int nacc, int& ntiles, int& rb, int& rpb) {
  ntiles = (n + kCR_COLS - 1) / kCR_COLS;
  rb = std::max(1, std::min((2 * 148 + ntiles - 1) / ntiles, (rows + 63) / 64));
  while (static_cast<int64_t>(nacc) * rb * n > kColredPartFloats && rb > 1) rb >>= 1;
  if (static_cast<int64_t>(nacc) * rb * n > kColredPartFloats || ntiles > kColredTickets)
    throw CudaError("column reduction: n too large for the scratch");
  rpb = (rows + rb - 1) / rb;
  rpb = (rpb + 63) / 64 * 64;  // whole 8-warp x 8-row batches per CTA
  rb = (rows + rpb - 1) / rpb;
}

template <int VPL>
static void ln_fwd_warp(DType dt, const void* x, const float* g, const float* b, void* y, float* mean, float* rstd,
                        int rows, int h, float eps, cudaStream_t st) {
  if (dt == DT_BF16) {  // persistent: 4 CTAs of 4 warps per SM (or fewer for small inputs)
    const int blocks = std::min((rows + 3) / 4, 4 * 148);
    const size_t sm = 2 * sizeof(float) * static_cast<size_t>(h);
    static bool attr = false;
    if (!attr) {  // h <= 3072 here: at most 24 KB
      ZB_CUDA(cudaFuncSetAttribute(k_ln_fwd_rows<VPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
      attr = true;
    }
    launch(PDL_OPS, k_ln_fwd_rows<VPL>, blocks, 128, sm, st, static_cast<const bf16*>(x), g, b, static_cast<bf16*>(y),
           mean, rstd, rows, h, eps);
    return;
  }
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
  const int tk__ = ktimer::start(ktimer::LN_FWD, static_cast<double>(rows) * h * 2 * (dt == DT_BF16 ? 2.0 : 4.0) + 8.0 * h + 8.0 * rows, st);
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
    // h in (3072, 4096] (bf16): 128 threads of 4 vectors per row measured 15.8 vs 16.7 us
    // for 256 x 2 at 3072 x 4096 (512 threads: 20.8); wider rows stay at 256 threads
    // (h = 5120: 19.2 vs 20.7 us for 128 threads) — profiles/r02_ln_fwd_threads_per_row.jsonl
    if (dt == DT_BF16 && h / 8 <= 128 * 4) {
      launch(PDL_OPS, k_ln_fwd<bf16, 4, 128>, rows, 128, 0, st, static_cast<const bf16*>(x), g, b, static_cast<bf16*>(y),
             mean, rstd, h, eps);
    } else
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
  ktimer::stop(tk__, st);
}

void layernorm_bwd(DType dt, const float* dy, const void* x, const float* mean, const float* rstd, const float* g,
                   const float* resid, float* dx32, void* dx, float* gg, float* gb, int beta, int rows, int h,
                   cudaStream_t st) {
  if (rows <= 0) return;
  const double esz = dt == DT_BF16 ? 2.0 : 4.0, elems = static_cast<double>(rows) * h;
  // 1) gamma / beta grads (reads x before step 2 may overwrite it in place)
  int tk = ktimer::start(ktimer::LN_PARAM, elems * (4.0 + esz) + 8.0 * rows + 8.0 * h, st);
  {
    int ntiles, rb, rpb;
    colred2_grid(rows, h, 2, ntiles, rb, rpb);
    const ColredScratch sc = colred_scratch(st);
    const dim3 grid(ntiles, rb);
    if (dt == DT_BF16)
      launch(PDL_OPS, k_colred2<1, bf16>, grid, kCR_THREADS, 0, st, static_cast<const bf16*>(x), static_cast<int64_t>(h),
             dy, mean, rstd, gg, gb, sc.part, sc.tickets, rows, h, rpb, beta);
    else
      launch(PDL_OPS, k_colred2<1, float>, grid, kCR_THREADS, 0, st, static_cast<const float*>(x), static_cast<int64_t>(h),
             dy, mean, rstd, gg, gb, sc.part, sc.tickets, rows, h, rpb, beta);
  }
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk, st);
  // 2) dx, one CTA per row (dy arrives in f32: the dLN GEMM epilogue keeps full precision)
  tk = ktimer::start(ktimer::LN_BWD,
                     elems * (4.0 + 2 * esz + (resid ? 4.0 : 0.0) + (dx32 ? 4.0 : 0.0)) + 8.0 * rows + 4.0 * h, st);
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
  ktimer::stop(tk, st);
}

void bias_grad(DType dt, const void* y, int64_t ldy, float* out, int rows, int n, int beta, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return;
  const int tk__ = ktimer::start(ktimer::BIAS_GRAD, static_cast<double>(rows) * n * (dt == DT_BF16 ? 2.0 : 4.0) + 4.0 * n, st);
  int ntiles, rb, rpb;
  colred2_grid(rows, n, 1, ntiles, rb, rpb);
  const ColredScratch sc = colred_scratch(st);
  const dim3 grid(ntiles, rb);
  if (dt == DT_BF16)
    launch(PDL_OPS, k_colred2<0, bf16>, grid, kCR_THREADS, 0, st, static_cast<const bf16*>(y), ldy, nullptr, nullptr,
           nullptr, out, nullptr, sc.part, sc.tickets, rows, n, rpb, beta);
  else
    launch(PDL_OPS, k_colred2<0, float>, grid, kCR_THREADS, 0, st, static_cast<const float*>(y), ldy, nullptr, nullptr,
           nullptr, out, nullptr, sc.part, sc.tickets, rows, n, rpb, beta);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk__, st);
}

void embed_fwd(DType dt, const int32_t* tok, const float* wte, const float* wpe, void* x0, int rows, int s, int h,
               cudaStream_t st) {
  if (rows <= 0) return;
  const int tk__ = ktimer::start(ktimer::MISC, static_cast<double>(rows) * h * (8.0 + (dt == DT_BF16 ? 2.0 : 4.0)) + 4.0 * rows, st);
  const int thr = h / 8 < 256 ? ((h / 8 + 31) / 32) * 32 : 256;
  if (dt == DT_BF16)
    launch(PDL_OPS, k_embed_fwd<bf16>, rows, thr, 0, st, tok, wte, wpe, static_cast<bf16*>(x0), s, h);
  else
    launch(PDL_OPS, k_embed_fwd<float>, rows, thr, 0, st, tok, wte, wpe, static_cast<float*>(x0), s, h);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk__, st);
}

void embed_bwd(DType dt, const int32_t* tok, const void* dx0, float* dwte, float* dwpe, uint32_t* keys, int rows,
               int s, int h, cudaStream_t st) {
  if (rows <= 0) return;
  if (rows > 8192) throw CudaError("embed_bwd: at most 8192 tokens per microbatch");
  const int tk__ = ktimer::start(ktimer::MISC, static_cast<double>(rows) * h * (2 * (dt == DT_BF16 ? 2.0 : 4.0) + 8.0) + 8.0 * rows, st);
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
  ktimer::stop(tk__, st);
}

void cross_entropy(DType dt, const float* logits, const int32_t* labels, void* dlogits, float* loss_rows,
                   double* loss_acc, int rows, int V, float inv_scale, cudaStream_t st) {
  if (rows <= 0) return;
  if (V % 8) throw CudaError("cross_entropy: V must be a multiple of 8");
  const int tk__ = ktimer::start(ktimer::CE, static_cast<double>(rows) * V * (4.0 + (dt == DT_BF16 ? 2.0 : 4.0)), st);
  if (dt == DT_BF16)
    launch(PDL_OPS, k_ce<bf16>, rows, 1024, 0, st, logits, labels, static_cast<bf16*>(dlogits), loss_rows, V, inv_scale);
  else
    launch(PDL_OPS, k_ce<float>, rows, 1024, 0, st, logits, labels, static_cast<float*>(dlogits), loss_rows, V, inv_scale);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_loss_reduce, 1, 1024, 0, st, loss_rows, loss_acc, rows, inv_scale);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk__, st);
}

void convert_rows(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st) {
  convert_f32(dt, src, dst, n, st);
}

void convert_f32(DType dt, const float* src, void* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int tk__ = ktimer::start(ktimer::MISC, static_cast<double>(n) * (4.0 + (dt == DT_BF16 ? 2.0 : 4.0)), st);
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  if (dt == DT_BF16) launch(PDL_OPS, k_convert<bf16>, blocks, 256, 0, st, src, static_cast<bf16*>(dst), n);
  else launch(PDL_OPS, k_convert<float>, blocks, 256, 0, st, src, static_cast<float*>(dst), n);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk__, st);
}

void grad_norm(const float* g, int64_t n, double* part, int32_t* nf_part, PvState* pst, cudaStream_t st) {
  const int tk = ktimer::start(ktimer::OPT, 4.0 * static_cast<double>(n), st);
  launch(PDL_OPS, k_sumsq, kNormBlocks, 512, 0, st, g, n, part, nf_part);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_sumsq_final, 1, 32, 0, st, part, nf_part, kNormBlocks, pst);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk, st);
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
                 bool validation, cudaStream_t st) {
  if (n % 4) throw CudaError("adamw_apply: n must be a multiple of 4");
  const int blocks = static_cast<int>(std::min<int64_t>((n / 4 + 511) / 512, 148 * 8));
  // The first (optimistic / synchronous) step: theta, m, v, g read + theta, m, v written (f32) + the bf16
  // shadow.  The validation launch works only on a rollback / deferred step and is otherwise
  // predicated off on the device, so it is timed in its own class with no algorithmic bytes.
  const int tk = validation ? ktimer::start(ktimer::OPT_VALIDATE, 0.0, st)
                            : ktimer::start(ktimer::OPT, 28.0 * static_cast<double>(n) +
                                                             2.0 * static_cast<double>(n_shadow), st);
  launch(PDL_OPS, k_adamw, blocks, 512, 0, st, theta, m, v, g, shadow, n, n_wd, n_shadow, lr, b1, b2, eps, wd, pst);
  ZB_LAUNCH_CHECK();
  ktimer::stop(tk, st);
}

}  // namespace zb
