// Causal flash attention, forward and backward (see attention.h).
//
// bf16 path: FlashAttention-2 style tiling with mma.sync.m16n8k16 (bf16 in,
// f32 accumulate), ldmatrix and cp.async double buffering; 64x64 tiles, one
// warp per 16 rows.  Backward is deterministic: one kernel owns dK/dV of a key
// block (loop over query blocks), another owns dQ of a query block (loop over
// key blocks) — no atomics, so gradients are bitwise reproducible.
// f32 path (1e-5 parity mode): one thread per row, online softmax in f32.
//
// softmax(Q K^T / sqrt(d) + causal mask) V per head; lse is saved by F and
// P is recomputed in B (Table 1 counts the 4s / 8s attention terms
// of F / B).
#include <math.h>

#include "attention.h"
#include "ktimer.h"

namespace zb {
void attention_bwd_impl(const AttnShape& sh, DType dt, const void* qkv, const void* o, const void* dout,
                        const float* lse, void* dqkv, float* delta, cudaStream_t st);
bool attention_fwd_tc(const AttnShape& sh, const void* qkv, void* o, float* lse, cudaStream_t st);
bool attention_bwd_tc(const AttnShape& sh, const void* qkv, const void* dout, const float* lse, void* dqkv,
                      const float* delta, cudaStream_t st);
// ZB_ATTN_LEGACY=1 selects the mma.sync kernels (comparison / debugging)
static bool legacy_attention() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZB_ATTN_LEGACY");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
namespace attn {

constexpr int TILE = 64;
constexpr int NT = 128;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 64 x D tile of rows [row0, row0+64) of a column block with row pitch ld; rows >= s are zero-filled.
template <int D>
__device__ __forceinline__ void load_tile(bf16* sdst, const bf16* g, int row0, int s, int64_t ld) {
  constexpr int CH = D / 8, LDS = D + 8;
  for (int c = threadIdx.x; c < TILE * CH; c += NT) {
    const int r = c / CH, cc = c % CH;
    const int gr = row0 + r;
    const bf16* src = g + static_cast<int64_t>(gr < s ? gr : s - 1) * ld + cc * 8;
    cp_async16(saddr(sdst + r * LDS + cc * 8), src, gr < s ? 16 : 0);
  }
}

// A fragment (16 x 16) of rows r0.., cols c0.. from a row-major smem tile.
template <int LDS>
__device__ __forceinline__ void frag_a(uint32_t* a, const bf16* t, int r0, int c0) {
  const int l = threadIdx.x & 31;
  ldsm4(a, saddr(t + (r0 + (l & 15)) * LDS + c0 + (l >> 4) * 8));
}
// B fragments for two n-tiles (n0, n0+8) x k16 from storage [n][k] (non-transposed).
template <int LDS>
__device__ __forceinline__ void frag_b_nk(uint32_t* b, const bf16* t, int n0, int k0) {
  const int l = threadIdx.x & 31;
  ldsm4(b, saddr(t + (n0 + (l & 7) + (l >> 4) * 8) * LDS + k0 + ((l >> 3) & 1) * 8));
}
// B fragments for two n-tiles (n0, n0+8) x k16 from storage [k][n] (transposed load).
template <int LDS>
__device__ __forceinline__ void frag_b_kn(uint32_t* b, const bf16* t, int k0, int n0) {
  const int l = threadIdx.x & 31;
  ldsm4t(b, saddr(t + (k0 + (l & 7) + ((l >> 3) & 1) * 8) * LDS + n0 + (l >> 4) * 8));
}

// acc[8][4] (16 x 64) = A_tile(rows r0 of sa, D) * B_tile(64 rows of sb, D)^T
template <int D>
__device__ __forceinline__ void gemm_rows_x64(float (*acc)[4], const bf16* sa, int r0, const bf16* sb) {
  constexpr int LDS = D + 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    uint32_t a[4];
    frag_a<LDS>(a, sa, r0, kk * 16);
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      frag_b_nk<LDS>(b, sb, np * 16, kk * 16);
      mma16816(acc[2 * np], a, b[0], b[1]);
      mma16816(acc[2 * np + 1], a, b[2], b[3]);
    }
  }
}

// out[D/8][4] += P(16 x 64, C-fragment layout in p) * T(64 rows of st, D) where st is [k][n].
template <int D>
__device__ __forceinline__ void gemm_p_x_tile(float (*out)[4], float (*p)[4], const bf16* st) {
  constexpr int LDS = D + 8;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    uint32_t a[4] = {pack2(p[2 * t][0], p[2 * t][1]), pack2(p[2 * t][2], p[2 * t][3]),
                     pack2(p[2 * t + 1][0], p[2 * t + 1][1]), pack2(p[2 * t + 1][2], p[2 * t + 1][3])};
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      uint32_t b[4];
      frag_b_kn<LDS>(b, st, t * 16, dp * 16);
      mma16816(out[2 * dp], a, b[0], b[1]);
      mma16816(out[2 * dp + 1], a, b[2], b[3]);
    }
  }
}

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(NT) k_fwd_bf16(const bf16* __restrict__ qkv, bf16* __restrict__ o,
                                                 float* __restrict__ lse, int s, int a, float scale_log2) {
  pdl_wait();
  constexpr int LDS = D + 8, TS = TILE * LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = reinterpret_cast<bf16*>(smraw);
  bf16* sK = sQ + TS;       // 2 buffers
  bf16* sV = sK + 2 * TS;   // 2 buffers
  const int nqb = (s + TILE - 1) / TILE;
  const int qb = nqb - 1 - blockIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const bf16* base = qkv + static_cast<int64_t>(bb) * s * ld;
  const bf16* Qg = base + hd * D;
  const bf16* Kg = base + h + hd * D;
  const bf16* Vg = base + 2 * h + hd * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  load_tile<D>(sQ, Qg, qb * TILE, s, ld);
  load_tile<D>(sK, Kg, 0, s, ld);
  load_tile<D>(sV, Vg, 0, s, ld);
  cp_commit();

  float oacc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int q0 = qb * TILE + warp * 16 + (lane >> 2);

  for (int j = 0; j <= qb; ++j) {
    const int cur = j & 1;
    if (j < qb) {
      load_tile<D>(sK + (cur ^ 1) * TS, Kg, (j + 1) * TILE, s, ld);
      load_tile<D>(sV + (cur ^ 1) * TS, Vg, (j + 1) * TILE, s, ld);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    float sacc[8][4];
    gemm_rows_x64<D>(sacc, sQ, warp * 16, sK + cur * TS);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = sacc[nt][e] * scale_log2;
        const int key = j * TILE + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = q0 + (e >= 2 ? 8 : 0);
        if (j == qb && key > q) v = -INFINITY;
        sacc[nt][e] = v;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(sacc[nt][2 * r], sacc[nt][2 * r + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mnew = fmaxf(mrow[r], mx);
      const float corr = exp2f(mrow[r] - mnew);
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = exp2f(sacc[nt][2 * r] - mnew), p1 = exp2f(sacc[nt][2 * r + 1] - mnew);
        sacc[nt][2 * r] = p0;
        sacc[nt][2 * r + 1] = p1;
        sum += p0 + p1;
      }
      lrow[r] = lrow[r] * corr + sum;
      mrow[r] = mnew;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        oacc[i][2 * r] *= corr;
        oacc[i][2 * r + 1] *= corr;
      }
    }
    gemm_p_x_tile<D>(oacc, sacc, sV + cur * TS);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float l = lrow[r];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const int q = q0 + r * 8;
    if (q < s) {
      const float inv = 1.f / l;
      bf16* orow = o + (static_cast<int64_t>(bb) * s + q) * h + hd * D + (lane & 3) * 2;
#pragma unroll
      for (int i = 0; i < D / 8; ++i)
        *reinterpret_cast<uint32_t*>(orow + i * 8) = pack2(oacc[i][2 * r] * inv, oacc[i][2 * r + 1] * inv);
      if ((lane & 3) == 0) lse[(static_cast<int64_t>(bb) * a + hd) * s + q] = (mrow[r] + log2f(l)) * LN2;
    }
  }
}

// ------------------------------------------------------------------ backward: delta = rowsum(dO * O)
template <typename T, int DC>
__global__ void k_delta(const T* __restrict__ o, const T* __restrict__ dout, float* __restrict__ delta, int s, int a,
                        int d_rt, int rows) {
  pdl_wait();
  // one thread per (row, head): d/8 vector loads of each operand summed in order (DC > 0: the
  // head dim at compile time, every load of the thread in flight at once)
  const int d = DC > 0 ? DC : d_rt;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(rows) * a) return;
  const int row = static_cast<int>(t / a), hd = static_cast<int>(t % a);  // row in [0, b*s)
  const int64_t off = t * d;
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < d; i += 8) {
    float x[8], y[8];
    Vec8<T>::load(o + off + i, x);
    Vec8<T>::load(dout + off + i, y);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += x[k] * y[k];
  }
  const int bb = row / s, q = row % s;
  delta[(static_cast<int64_t>(bb) * a + hd) * s + q] = acc;
}

// ------------------------------------------------------------------ backward: dQ
template <int D>
__global__ void __launch_bounds__(NT) k_bwd_dq_bf16(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                    const float* __restrict__ lse, const float* __restrict__ delta,
                                                    bf16* __restrict__ dqkv, int s, int a, float scale,
                                                    float scale_log2) {
  pdl_wait();
  constexpr int LDS = D + 8, TS = TILE * LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = reinterpret_cast<bf16*>(smraw);
  bf16* sdO = sQ + TS;
  bf16* sK = sdO + TS;      // 2 buffers
  bf16* sV = sK + 2 * TS;   // 2 buffers
  const int nqb = (s + TILE - 1) / TILE;
  const int qb = nqb - 1 - blockIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const bf16* base = qkv + static_cast<int64_t>(bb) * s * ld;
  const bf16* Kg = base + h + hd * D;
  const bf16* Vg = base + 2 * h + hd * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  load_tile<D>(sQ, base + hd * D, qb * TILE, s, ld);
  load_tile<D>(sdO, dout + static_cast<int64_t>(bb) * s * h + hd * D, qb * TILE, s, h);
  load_tile<D>(sK, Kg, 0, s, ld);
  load_tile<D>(sV, Vg, 0, s, ld);
  cp_commit();

  const int q0 = qb * TILE + warp * 16 + (lane >> 2);
  float Lr[2], Dr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = q0 + 8 * r;
    const int64_t idx = (static_cast<int64_t>(bb) * a + hd) * s + q;
    Lr[r] = q < s ? lse[idx] * LOG2E : 0.f;
    Dr[r] = q < s ? delta[idx] : 0.f;
  }
  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int j = 0; j <= qb; ++j) {
    const int cur = j & 1;
    if (j < qb) {
      load_tile<D>(sK + (cur ^ 1) * TS, Kg, (j + 1) * TILE, s, ld);
      load_tile<D>(sV + (cur ^ 1) * TS, Vg, (j + 1) * TILE, s, ld);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    float p[8][4], dp[8][4];
    gemm_rows_x64<D>(p, sQ, warp * 16, sK + cur * TS);
    gemm_rows_x64<D>(dp, sdO, warp * 16, sV + cur * TS);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const int key = j * TILE + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = q0 + 8 * r;
        float pv = exp2f(p[nt][e] * scale_log2 - Lr[r]);
        if (j == qb && key > q) pv = 0.f;
        p[nt][e] = pv * (dp[nt][e] - Dr[r]);  // dS
      }
    gemm_p_x_tile<D>(dq, p, sK + cur * TS);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = q0 + 8 * r;
    if (q >= s) continue;
    bf16* row = dqkv + (static_cast<int64_t>(bb) * s + q) * ld + hd * D + (lane & 3) * 2;
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
      *reinterpret_cast<uint32_t*>(row + i * 8) = pack2(dq[i][2 * r] * scale, dq[i][2 * r + 1] * scale);
  }
}

// ------------------------------------------------------------------ backward: dK, dV
template <int D>
__global__ void __launch_bounds__(NT) k_bwd_dkdv_bf16(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                      const float* __restrict__ lse, const float* __restrict__ delta,
                                                      bf16* __restrict__ dqkv, int s, int a, float scale,
                                                      float scale_log2) {
  pdl_wait();
  constexpr int LDS = D + 8, TS = TILE * LDS;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sK = reinterpret_cast<bf16*>(smraw);
  bf16* sV = sK + TS;
  bf16* sQ = sV + TS;       // 2 buffers
  bf16* sdO = sQ + 2 * TS;  // 2 buffers
  float* sL = reinterpret_cast<float*>(sdO + 2 * TS);  // [2][64]
  float* sD = sL + 2 * TILE;                           // [2][64]
  const int nqb = (s + TILE - 1) / TILE;
  const int kb = blockIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const bf16* base = qkv + static_cast<int64_t>(bb) * s * ld;
  const bf16* Qg = base + hd * D;
  const bf16* dOg = dout + static_cast<int64_t>(bb) * s * h + hd * D;
  const float* Lg = lse + (static_cast<int64_t>(bb) * a + hd) * s;
  const float* Dg = delta + (static_cast<int64_t>(bb) * a + hd) * s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto load_q = [&](int i, int buf) {
    load_tile<D>(sQ + buf * TS, Qg, i * TILE, s, ld);
    load_tile<D>(sdO + buf * TS, dOg, i * TILE, s, h);
    if (threadIdx.x < TILE) {
      const int q = i * TILE + threadIdx.x;
      sL[buf * TILE + threadIdx.x] = q < s ? Lg[q] * LOG2E : 0.f;
      sD[buf * TILE + threadIdx.x] = q < s ? Dg[q] : 0.f;
    }
  };
  load_tile<D>(sK, base + h + hd * D, kb * TILE, s, ld);
  load_tile<D>(sV, base + 2 * h + hd * D, kb * TILE, s, ld);
  load_q(kb, 0);
  cp_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = 0.f;
    dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
  }
  const int k0 = kb * TILE + warp * 16 + (lane >> 2);

  for (int i = kb; i < nqb; ++i) {
    const int cur = (i - kb) & 1;
    if (i + 1 < nqb) {
      load_q(i + 1, cur ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* q_t = sQ + cur * TS;
    const bf16* do_t = sdO + cur * TS;
    const float* Lc = sL + cur * TILE;
    const float* Dc = sD + cur * TILE;
    float pt[8][4], dpt[8][4];
    gemm_rows_x64<D>(pt, sK, warp * 16, q_t);    // S^T: keys x queries
    gemm_rows_x64<D>(dpt, sV, warp * 16, do_t);  // dP^T = V dO^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = i * TILE + ql;
        const int key = k0 + (e >= 2 ? 8 : 0);
        float pv = exp2f(pt[nt][e] * scale_log2 - Lc[ql]);
        if (q < key) pv = 0.f;
        pt[nt][e] = pv;
        dpt[nt][e] = pv * (dpt[nt][e] - Dc[ql]);  // dS^T
      }
    gemm_p_x_tile<D>(dv, pt, do_t);   // dV += P^T dO
    gemm_p_x_tile<D>(dk, dpt, q_t);   // dK += dS^T Q
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = k0 + 8 * r;
    if (key >= s) continue;
    bf16* row = dqkv + (static_cast<int64_t>(bb) * s + key) * ld + hd * D + (lane & 3) * 2;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      *reinterpret_cast<uint32_t*>(row + h + i * 8) = pack2(dk[i][2 * r] * scale, dk[i][2 * r + 1] * scale);
      *reinterpret_cast<uint32_t*>(row + 2 * h + i * 8) = pack2(dv[i][2 * r], dv[i][2 * r + 1]);
    }
  }
}

// ------------------------------------------------------------------ f32 parity kernels
template <int D>
__global__ void k_fwd_f32(const float* __restrict__ qkv, float* __restrict__ o, float* __restrict__ lse, int s, int a,
                          float scale) {
  pdl_wait();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  if (q >= s) return;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const float* base = qkv + static_cast<int64_t>(bb) * s * ld;
  float qv[D], acc[D];
  for (int i = 0; i < D; ++i) {
    qv[i] = base[static_cast<int64_t>(q) * ld + hd * D + i] * scale;
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int k = 0; k <= q; ++k) {
    const float* kr = base + static_cast<int64_t>(k) * ld + h + hd * D;
    const float* vr = kr + h;
    float sc = 0.f;
    for (int i = 0; i < D; ++i) sc = fmaf(qv[i], kr[i], sc);
    const float mn = fmaxf(m, sc);
    const float corr = expf(m - mn), pv = expf(sc - mn);
    l = l * corr + pv;
    for (int i = 0; i < D; ++i) acc[i] = acc[i] * corr + pv * vr[i];
    m = mn;
  }
  float* orow = o + (static_cast<int64_t>(bb) * s + q) * h + hd * D;
  for (int i = 0; i < D; ++i) orow[i] = acc[i] / l;
  lse[(static_cast<int64_t>(bb) * a + hd) * s + q] = m + logf(l);
}

template <int D>
__global__ void k_bwd_dq_f32(const float* __restrict__ qkv, const float* __restrict__ dout,
                             const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ dqkv,
                             int s, int a, float scale) {
  pdl_wait();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  if (q >= s) return;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const float* base = qkv + static_cast<int64_t>(bb) * s * ld;
  const float* qr = base + static_cast<int64_t>(q) * ld + hd * D;
  const float* dor = dout + (static_cast<int64_t>(bb) * s + q) * h + hd * D;
  const int64_t li = (static_cast<int64_t>(bb) * a + hd) * s + q;
  const float L = lse[li], Dl = delta[li];
  float dq[D];
  for (int i = 0; i < D; ++i) dq[i] = 0.f;
  for (int k = 0; k <= q; ++k) {
    const float* kr = base + static_cast<int64_t>(k) * ld + h + hd * D;
    const float* vr = kr + h;
    float sc = 0.f, dp = 0.f;
    for (int i = 0; i < D; ++i) {
      sc = fmaf(qr[i], kr[i], sc);
      dp = fmaf(dor[i], vr[i], dp);
    }
    const float ds = expf(sc * scale - L) * (dp - Dl);
    for (int i = 0; i < D; ++i) dq[i] = fmaf(ds, kr[i], dq[i]);
  }
  float* out = dqkv + (static_cast<int64_t>(bb) * s + q) * ld + hd * D;
  for (int i = 0; i < D; ++i) out[i] = dq[i] * scale;
}

template <int D>
__global__ void k_bwd_dkdv_f32(const float* __restrict__ qkv, const float* __restrict__ dout,
                               const float* __restrict__ lse, const float* __restrict__ delta,
                               float* __restrict__ dqkv, int s, int a, float scale) {
  pdl_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int hd = blockIdx.y, bb = blockIdx.z;
  if (k >= s) return;
  const int h = a * D;
  const int64_t ld = 3LL * h;
  const float* base = qkv + static_cast<int64_t>(bb) * s * ld;
  const float* kr = base + static_cast<int64_t>(k) * ld + h + hd * D;
  const float* vr = kr + h;
  float dk[D], dv[D];
  for (int i = 0; i < D; ++i) dk[i] = dv[i] = 0.f;
  for (int q = k; q < s; ++q) {
    const float* qr = base + static_cast<int64_t>(q) * ld + hd * D;
    const float* dor = dout + (static_cast<int64_t>(bb) * s + q) * h + hd * D;
    const int64_t li = (static_cast<int64_t>(bb) * a + hd) * s + q;
    float sc = 0.f, dp = 0.f;
    for (int i = 0; i < D; ++i) {
      sc = fmaf(qr[i], kr[i], sc);
      dp = fmaf(dor[i], vr[i], dp);
    }
    const float pv = expf(sc * scale - lse[li]);
    const float ds = pv * (dp - delta[li]);
    for (int i = 0; i < D; ++i) {
      dv[i] = fmaf(pv, dor[i], dv[i]);
      dk[i] = fmaf(ds, qr[i], dk[i]);
    }
  }
  float* out = dqkv + (static_cast<int64_t>(bb) * s + k) * ld + hd * D;
  for (int i = 0; i < D; ++i) {
    out[h + i] = dk[i] * scale;
    out[2 * h + i] = dv[i];
  }
}

template <int D>
static void fwd_bf16(const AttnShape& sh, const void* qkv, void* o, float* lse, cudaStream_t st) {
  constexpr int TS = TILE * (D + 8);
  const int smem = 5 * TS * 2;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(k_fwd_bf16<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dim3 grid((sh.s + TILE - 1) / TILE, sh.a, sh.b);
  launch(PDL_OPS, k_fwd_bf16<D>, grid, NT, smem, st, static_cast<const bf16*>(qkv), static_cast<bf16*>(o), lse, sh.s, sh.a,
                                        LOG2E / sqrtf(static_cast<float>(D)));
  ZB_LAUNCH_CHECK();
}

template <int D>
static void bwd_bf16(const AttnShape& sh, const void* qkv, const void* dout, const float* lse, void* dqkv,
                     const float* delta, cudaStream_t st) {
  constexpr int TS = TILE * (D + 8);
  const int smem_dq = 6 * TS * 2;
  const int smem_kv = 6 * TS * 2 + 4 * TILE * 4;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(k_bwd_dq_bf16<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dq));
    ZB_CUDA(cudaFuncSetAttribute(k_bwd_dkdv_bf16<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    attr = true;
  }
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  dim3 grid((sh.s + TILE - 1) / TILE, sh.a, sh.b);
  launch(PDL_OPS, k_bwd_dkdv_bf16<D>, grid, NT, smem_kv, st, static_cast<const bf16*>(qkv), static_cast<const bf16*>(dout), lse,
                                                delta, static_cast<bf16*>(dqkv), sh.s, sh.a, scale, scale * LOG2E);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_bwd_dq_bf16<D>, grid, NT, smem_dq, st, static_cast<const bf16*>(qkv), static_cast<const bf16*>(dout), lse,
                                              delta, static_cast<bf16*>(dqkv), sh.s, sh.a, scale, scale * LOG2E);
  ZB_LAUNCH_CHECK();
}

template <int D>
static void fwd_f32(const AttnShape& sh, const void* qkv, void* o, float* lse, cudaStream_t st) {
  dim3 grid((sh.s + 63) / 64, sh.a, sh.b);
  launch(PDL_OPS, k_fwd_f32<D>, grid, 64, 0, st, static_cast<const float*>(qkv), static_cast<float*>(o), lse, sh.s, sh.a,
                                    1.f / sqrtf(static_cast<float>(D)));
  ZB_LAUNCH_CHECK();
}

template <int D>
static void bwd_f32(const AttnShape& sh, const void* qkv, const void* dout, const float* lse, void* dqkv,
                    const float* delta, cudaStream_t st) {
  dim3 grid((sh.s + 63) / 64, sh.a, sh.b);
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  launch(PDL_OPS, k_bwd_dkdv_f32<D>, grid, 64, 0, st, static_cast<const float*>(qkv), static_cast<const float*>(dout), lse, delta,
                                         static_cast<float*>(dqkv), sh.s, sh.a, scale);
  ZB_LAUNCH_CHECK();
  launch(PDL_OPS, k_bwd_dq_f32<D>, grid, 64, 0, st, static_cast<const float*>(qkv), static_cast<const float*>(dout), lse, delta,
                                       static_cast<float*>(dqkv), sh.s, sh.a, scale);
  ZB_LAUNCH_CHECK();
}

}  // namespace attn

void attention_fwd(const AttnShape& sh, DType dt, const void* qkv, void* o, float* lse, cudaStream_t st) {
  if (sh.b <= 0 || sh.s <= 0 || sh.a <= 0) return;
  // algorithmic causal FLOPs: Q K^T and P V over the lower triangle
  const int tk = ktimer::start(ktimer::ATTN_FWD, 2.0 * sh.b * sh.a * static_cast<double>(sh.s) * sh.s * sh.d, st);
  if (dt == DT_BF16 && !legacy_attention() && attention_fwd_tc(sh, qkv, o, lse, st)) {
    ktimer::stop(tk, st);
    return;
  }
  switch (sh.d) {
    case 64: dt == DT_BF16 ? attn::fwd_bf16<64>(sh, qkv, o, lse, st) : attn::fwd_f32<64>(sh, qkv, o, lse, st); break;
    case 96: dt == DT_BF16 ? attn::fwd_bf16<96>(sh, qkv, o, lse, st) : attn::fwd_f32<96>(sh, qkv, o, lse, st); break;
    case 128:
      dt == DT_BF16 ? attn::fwd_bf16<128>(sh, qkv, o, lse, st) : attn::fwd_f32<128>(sh, qkv, o, lse, st);
      break;
    default: throw CudaError("attention: head dim must be 64, 96 or 128");
  }
  ktimer::stop(tk, st);
}

void attention_bwd(const AttnShape& sh, DType dt, const void* qkv, const void* o, const void* dout, const float* lse,
                   void* dqkv, float* delta, cudaStream_t st) {
  if (sh.b <= 0 || sh.s <= 0 || sh.a <= 0) return;
  // algorithmic causal FLOPs of the five backward products (recomputation not counted)
  const int tk = ktimer::start(ktimer::ATTN_BWD, 5.0 * sh.b * sh.a * static_cast<double>(sh.s) * sh.s * sh.d, st);
  attention_bwd_impl(sh, dt, qkv, o, dout, lse, dqkv, delta, st);
  ktimer::stop(tk, st);
}

void attention_bwd_impl(const AttnShape& sh, DType dt, const void* qkv, const void* o, const void* dout,
                        const float* lse, void* dqkv, float* delta, cudaStream_t st) {
  const int rows = sh.b * sh.s;
  // 128 threads per CTA (more, smaller CTAs per SM): 28.3B backward 70.7-71.6 -> 68.6 us,
  // 6.2B -0.5% against 256 (profiles/r02_attn_delta_block_size.jsonl)
  constexpr int dnt = 128;
  const int blocks = static_cast<int>((static_cast<int64_t>(rows) * sh.a + 255) / 256);
  if (dt == DT_BF16) {
    auto kern = sh.d == 64 ? attn::k_delta<bf16, 64> : sh.d == 96 ? attn::k_delta<bf16, 96>
              : sh.d == 128 ? attn::k_delta<bf16, 128> : attn::k_delta<bf16, 0>;
    launch(PDL_OPS, kern, static_cast<int>((static_cast<int64_t>(rows) * sh.a + dnt - 1) / dnt), dnt, 0, st, static_cast<const bf16*>(o), static_cast<const bf16*>(dout), delta, sh.s,
           sh.a, sh.d, rows);
  } else {
    launch(PDL_OPS, attn::k_delta<float, 0>, blocks, 256, 0, st, static_cast<const float*>(o),
           static_cast<const float*>(dout), delta, sh.s, sh.a, sh.d, rows);
  }
  ZB_LAUNCH_CHECK();
  if (dt == DT_BF16 && !legacy_attention() && attention_bwd_tc(sh, qkv, dout, lse, dqkv, delta, st)) return;
  switch (sh.d) {
    case 64:
      return dt == DT_BF16 ? attn::bwd_bf16<64>(sh, qkv, dout, lse, dqkv, delta, st)
                           : attn::bwd_f32<64>(sh, qkv, dout, lse, dqkv, delta, st);
    case 96:
      return dt == DT_BF16 ? attn::bwd_bf16<96>(sh, qkv, dout, lse, dqkv, delta, st)
                           : attn::bwd_f32<96>(sh, qkv, dout, lse, dqkv, delta, st);
    case 128:
      return dt == DT_BF16 ? attn::bwd_bf16<128>(sh, qkv, dout, lse, dqkv, delta, st)
                           : attn::bwd_f32<128>(sh, qkv, dout, lse, dqkv, delta, st);
  }
  throw CudaError("attention: head dim must be 64, 96 or 128");
}

}  // namespace zb
