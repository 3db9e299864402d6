// Causal flash-attention FORWARD on tcgen05 (bf16, s % 128 == 0).
//
// One CTA per (pair of 128-query tiles, head, sequence), heaviest pairs first.
//   warp 0      TMA: Q_0, Q_1 once; K_j, V_j in 2-stage rings (boxes {64 cols, 128 rows} of the
//               packed qkv [b*s, 3h], 128B swizzle), shared by both query tiles
//   warp 1      MMA: S_t = Q_t K_j^T (SS) and O_t += P_t V_j (TS, P from TMEM), ping-ponging
//               between the two tiles so one tile's softmax overlaps the other tile's products
//   warp 2      TMEM allocator (512 columns)
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: one row per thread (TMEM lane =
//               row), all 128 keys of a block in registers: causal mask, row max, lazy O rescale
//               (only when the max grows by > 8 in log2 units), exp2, bf16 P written into TMEM
//               over S; finally O / l -> bf16 rows and the log-sum-exp.
// Operand layouts: Q, K are K-major SW128 (atoms of 64 elements x 8 rows);
// V is the MN-major B operand of PV (d contiguous), read from the same TMA boxes.
#include <math.h>

#include "attention.h"
#include "gemm.h"
#include "sm100.cuh"

namespace zb {
namespace attn_tc {

#ifdef ZB_ATTN_TRACE
// timeline of CTA (0, 0, 0) (the heaviest query-tile pair), globaltimer ns (measurement build only)
__device__ unsigned long long g_trace_fwd[12][64];
__device__ __forceinline__ void trf(int row, int n) {
  if (blockIdx.x == 0 && n < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace_fwd[row][n] = t;
  }
}
#define TRF(row, n) trf(row, n)
#else
#define TRF(row, n)
#endif

constexpr int BQ = 128, BKV = 128;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// 2^x on the FMA pipe for x in [-126, 9): round-to-nearest split x = j + f (f in [-1/2, 1/2]) with
// the 1.5 * 2^23 shifter, a cubic for 2^f (max relative error 8e-5, far below bf16's 2^-9), and
// j added to the exponent field.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05516014f, f, 0.24258275f), f, 0.69326056f), f, 0.99993022f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

constexpr bool kAlternate = false;
// P of a key block is published to the MMA warp in PQ parts (2: halves of 64 keys, 4: quarters
// of 32) so the PV products of the first parts overlap the exponentials of the later ones
#ifndef ZB_ATTN_PQ
#define ZB_ATTN_PQ 2  // 4 measured equal (73.9 vs 74.1 us)
#endif
constexpr int PQ = ZB_ATTN_PQ;
constexpr bool kPolyExp = false;  // measured slower on B200 twice (75.6 -> 89 us; with the elect-style MMA issue 77.6 -> 91.6 us)

template <int D> struct FwdCfg {
  static constexpr int ATOMS = (D + 63) / 64;           // 64-column TMA boxes per tile
  static constexpr int TILE = ATOMS * 128 * 128;        // bytes of one 128-row tile (Q, K or V)
  static constexpr int KST = 2, VST = 2;                // K ring (freed after S0_j, S1_j), V ring (after PV0_j, PV1_j)
  static constexpr int OFF_Q = 0;                       // Q0, Q1
  static constexpr int OFF_K = 2 * TILE;
  static constexpr int OFF_V = (2 + KST) * TILE;
  static constexpr int OFF_BAR = (2 + KST + VST) * TILE;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
};

// One CTA per (pair of 128-query tiles {2t, 2t+1}, head, sequence), heaviest pairs first
// (1-D grid in that order).
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256, 256+D), O_1 [384, 384+D);
// P_t (bf16 pairs) is written over the first 64 columns of S_t.
// MMA issue order per key block j:  PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) — the tensor core
// runs one tile's products while the other tile's softmax warps work.  S_t(j+1) overwrites the
// P_t(j) that PV_t(j), issued just before it, reads: tcgen05.mma of one thread execute in issue
// order.  The commit after S_t(j+1) also covers PV_t(j), so the softmax warps may rescale O_t
// as soon as they see S_t(j+1).
template <int D>
__global__ void __launch_bounds__(384, 1) k_fwd_tc(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ o,
                                                   float* __restrict__ lse, int s, int a, float scale_log2) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;     // [2]
  uint64_t* k_empty = bar + 3;    // [2]
  uint64_t* v_full = bar + 5;     // [2]
  uint64_t* v_empty = bar + 7;    // [2]
  uint64_t* s_full = bar + 9;     // [2] per tile
  uint64_t* p_full = bar + 11;    // [2] per tile
  uint64_t* o_final = bar + 13;   // [2] per tile
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 15);
  uint64_t* tok = bar + 16;       // [2] per tile: the other tile's exponential phase is done
  uint64_t* p_part = bar + 18;    // [2][PQ - 1] per tile: P of keys [0, 32 (q + 1)) stored (PV may start)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / BQ;
  const int npair = (nqb + 1) / 2;
  // 1-D grid in work order: every (head, sequence) of the heaviest pair first, so the
  // hardware's in-order block dispatch is a longest-first list schedule (a 3-D grid
  // dispatched x fastest interleaved heavy and light pairs and left heavy CTAs for the tail)
  const int per = static_cast<int>(gridDim.x) / npair;  // a * b
  const int pr = npair - 1 - static_cast<int>(blockIdx.x) / per;
  const int hd = static_cast<int>(blockIdx.x) % per % a, bb = static_cast<int>(blockIdx.x) % per / a;
  const int h = a * D;
  const int q0 = 2 * pr;
  const bool two = q0 + 1 < nqb;
  const int nkv0 = q0 + 1, nkv1 = two ? q0 + 2 : 0;
  const int nkv = two ? nkv1 : nkv0;

  if (threadIdx.x == 0) {
    sm100::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 4);  // one arrival per softmax warp
      sm100::mbar_init(&o_final[i], 1);
      sm100::mbar_init(&tok[i], 4);
      for (int q = 0; q < PQ - 1; ++q) sm100::mbar_init(&p_part[i * (PQ - 1) + q], 4);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) sm100::tma_prefetch(&tm);
  if (warp == 2) sm100::tmem_alloc<512>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see launch() in common.cuh)
  pdl_wait();
  const uint32_t tbase = *tslot;
  const int row0 = bb * s;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA
      sm100::mbar_arrive_expect_tx(q_full, (two ? 2 : 1) * C::TILE);
      for (int t = 0; t < (two ? 2 : 1); ++t)
        for (int at = 0; at < C::ATOMS; ++at)
          sm100::tma_load_2d(smem + C::OFF_Q + t * C::TILE + at * 16384, &tm, q_full, hd * D + 64 * at,
                             row0 + (q0 + t) * BQ);
      auto load_k = [&](int j) {
        const int st = j & 1;
        sm100::mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&k_full[st], C::TILE);
        for (int at = 0; at < C::ATOMS; ++at)
          sm100::tma_load_2d(smem + C::OFF_K + st * C::TILE + at * 16384, &tm, &k_full[st], h + hd * D + 64 * at,
                             row0 + j * BKV);
      };
      auto load_v = [&](int j) {
        const int st = j & 1;
        sm100::mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&v_full[st], C::TILE);
        for (int at = 0; at < C::ATOMS; ++at)
          sm100::tma_load_2d(smem + C::OFF_V + st * C::TILE + at * 16384, &tm, &v_full[st], 2 * h + hd * D + 64 * at,
                             row0 + j * BKV);
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {  // K runs one block ahead of V
        if (j + 1 < nkv) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA
      constexpr uint32_t idesc_s = sm100::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = sm100::idesc_bf16(128, D, false, true);
      const uint32_t sq = sm100::smem_addr(smem + C::OFF_Q);
      auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
        const uint32_t sk = sm100::smem_addr(smem + C::OFF_K + (j & 1) * C::TILE);
        const uint64_t qd = sm100::smem_desc(sq + t * C::TILE, 16, 1024, sm100::kSwizzle128B);
        const uint64_t kd = sm100::smem_desc(sk, 16, 1024, sm100::kSwizzle128B);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          if (sm100::elect_one()) sm100::mma_bf16_ss(tbase + t * 128, sm100::desc_adv(qd, off), sm100::desc_adv(kd, off), idesc_s,
                             kk != 0 ? 1u : 0u);
        }
        if (sm100::elect_one()) sm100::mma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j, the first 64 keys as soon as their P is stored
        const uint32_t sv = sm100::smem_addr(smem + C::OFF_V + (j & 1) * C::TILE);
        const uint64_t vd = sm100::smem_desc(sv, 16384, 1024, sm100::kSwizzle128B);
#pragma unroll
        for (int q = 0; q < PQ; ++q) {
          constexpr int KQ = BKV / 16 / PQ;  // K-steps per published part of P
          sm100::mbar_wait_warp(q + 1 < PQ ? &p_part[t * (PQ - 1) + q] : &p_full[t], j & 1);
          if (q + 1 == PQ) TRF(t, j);
          sm100::tc_fence_after();
          if (sm100::elect_one()) {
#pragma unroll
            for (int kk = KQ * q; kk < KQ * q + KQ; ++kk)
              sm100::mma_bf16_ts(tbase + 256 + t * 128, tbase + t * 128 + kk * 8, sm100::desc_adv(vd, kk * 2048),
                                 idesc_o, (j | kk) != 0 ? 1u : 0u);
          }
          __syncwarp();
        }
      };
      sm100::mbar_wait_warp(q_full, 0);
      sm100::mbar_wait_warp(&k_full[0], 0);
      sm100::tc_fence_after();
      issue_s(0, 0);
      if (two) issue_s(1, 0);
      if (sm100::elect_one()) sm100::mma_commit(&k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const bool more = j + 1 < nkv;
        sm100::mbar_wait_warp(&v_full[j & 1], (j >> 1) & 1);
        if (more) sm100::mbar_wait_warp(&k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
        sm100::tc_fence_after();
        if (j < nkv0) {
          issue_pv(0, j);
          if (j == nkv0 - 1) { if (sm100::elect_one()) sm100::mma_commit(&o_final[0]); }
        }
        if (j + 1 < nkv0) issue_s(0, j + 1);
        if (j < nkv1) {
          issue_pv(1, j);
          if (j == nkv1 - 1) { if (sm100::elect_one()) sm100::mma_commit(&o_final[1]); }
        }
        if (sm100::elect_one()) sm100::mma_commit(&v_empty[j & 1]);
        if (j + 1 < nkv1) issue_s(1, j + 1);
        if (more) { if (sm100::elect_one()) sm100::mma_commit(&k_empty[(j + 1) & 1]); }
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax: 4 warps per tile, one row per thread
    const int t = (warp - 4) >> 2;
    const int nk = t == 0 ? nkv0 : nkv1;
    const int r = (warp & 3) * 32 + lane;  // row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tbase + t * 128 + lane_off, t_o = tbase + 256 + t * 128 + lane_off;
    const int qt = q0 + t;
    float m = -INFINITY, l = 0.f;  // m: reference max (log2 units), l: running sum relative to m
    for (int j = 0; j < nk; ++j) {
      sm100::mbar_wait(&s_full[t], j & 1);
      if ((warp & 3) == 0 && lane == 0) TRF(2 + 3 * t, j);
      sm100::tc_fence_after();
      float sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) sm100::tmem_ld32(t_s + c * 32, reinterpret_cast<uint32_t*>(sv + 32 * c));
      sm100::tmem_ld_wait();
      if ((warp & 3) == 0 && lane == 0) TRF(3 + 3 * t, j);
      if (j == qt) {
#pragma unroll
        for (int k = 0; k < 128; ++k)
          if (k > r) sv[k] = -INFINITY;
      }
      float mx;
      {  // 8 independent chains, then a tree (a single 128-long chain is pure latency)
        float m8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m8[i] = sv[i];
#pragma unroll
        for (int k = 8; k < 128; ++k) m8[k & 7] = fmaxf(m8[k & 7], sv[k]);
        mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      }
      mx *= scale_log2;
      // lazy rescaling: keep the old reference max unless it grew by more than 8 (p <= 2^8).
      // The decision is per row, but tcgen05.ld / st are warp-collective (.sync.aligned):
      // the whole warp enters the rescale when any of its rows needs it (corr = 1 elsewhere).
      const bool grow = mx > m + 8.f;
      if (__any_sync(0xffffffffu, grow)) {
        const float corr = grow ? sm100::ex2(m - mx) : 1.f;
        if (grow) {
          m = mx;
          l *= corr;
        }
        if (j > 0) {  // O_t holds blocks < j (PV_t(j-1) completed before S_t(j) was committed)
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            sm100::tmem_ld32(t_o + c * 32, ov);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
            sm100::tmem_st32(t_o + c * 32, ov);
          }
          sm100::tmem_st_wait();
        }
      }
      // kAlternate: the two tiles' exponential phases strictly alternate (token passing), so
      // each runs alone on the MUFU while the other tile's PV and next S use the tensor core.
      // Measured: no faster than free-running (the per-tile chain exp -> PV, S -> exp, not
      // the MUFU, sets the period: scripts/attn_fwd_trace.py), so it is off.
      const bool alt = kAlternate && two && j < nkv0;
      if (alt) sm100::mbar_wait(&tok[t], t == 0 ? ((j & 1) ^ 1) : (j & 1));
      if ((warp & 3) == 0 && lane == 0) TRF(8 + t, j);
      const float mneg = -m;
      const bool poly = kPolyExp && j != qt;  // masked (-inf) scores only on the diagonal block: MUFU there
      float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < PQ; ++q) {  // keys [KP q, KP q + KP) -> P columns [KP q / 2, KP (q + 1) / 2)
        constexpr int KP = BKV / PQ;
        uint32_t pk[KP / 2];
#pragma unroll
        for (int k = 0; k < KP; k += 2) {
          const float x0 = fmaf(sv[KP * q + k], scale_log2, mneg), x1 = fmaf(sv[KP * q + k + 1], scale_log2, mneg);
          float p0, p1;
          if ((k & 6) == 6 && poly) {  // a quarter of the exponentials on the FMA pipe (MUFU is the bottleneck)
            p0 = ex2_poly(x0);
            p1 = ex2_poly(x1);
          } else {
            p0 = sm100::ex2(x0);
            p1 = sm100::ex2(x1);
          }
          sum4[(k >> 1) & 3] += p0 + p1;
          __nv_bfloat162 v2 = __floats2bfloat162_rn(p0, p1);
          pk[k >> 1] = *reinterpret_cast<uint32_t*>(&v2);
        }
        if constexpr (KP == 64)
          sm100::tmem_st32(t_s + KP / 2 * q, pk);
        else
          sm100::tmem_st16(t_s + KP / 2 * q, pk);
        if (q + 1 < PQ) {  // publish this part of P: its PV products overlap the next part here
          sm100::tmem_st_wait();
          sm100::tc_fence_before();
          sm100::mbar_arrive_warp(&p_part[t * (PQ - 1) + q]);
        }
      }
      l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
      if ((warp & 3) == 0 && lane == 0) TRF(10 + t, j);
      if (alt) sm100::mbar_arrive_warp(&tok[t ^ 1]);
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      if ((warp & 3) == 0 && lane == 0) TRF(4 + 3 * t, j);
      sm100::mbar_arrive_warp(&p_full[t]);
    }
    if (nk > 0) {
      sm100::mbar_wait(&o_final[t], 0);
      sm100::tc_fence_after();
      const int q = qt * BQ + r;
      const float inv = 1.f / l;
      bf16* orow = o + (static_cast<int64_t>(bb) * s + q) * h + hd * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        sm100::tmem_ld32(t_o + c * 32, ov);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 u;
          __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            hv[e] = __floats2bfloat162_rn(__uint_as_float(ov[8 * g + 2 * e]) * inv,
                                          __uint_as_float(ov[8 * g + 2 * e + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + g * 8) = u;
        }
      }
      lse[(static_cast<int64_t>(bb) * a + hd) * s + q] = (m + log2f(l)) * LN2;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc<512>(tbase);
}

}  // namespace attn_tc

static CUtensorMap make_qkv_tmap(const void* qkv, int rows, int cols3h) {
  return make_tmap(qkv, static_cast<uint64_t>(cols3h), static_cast<uint64_t>(rows), static_cast<uint64_t>(cols3h), 64,
                   128);
}

template <int D>
static void fwd_tc_launch(const AttnShape& sh, const void* qkv, void* o, float* lse, cudaStream_t st) {
  using C = attn_tc::FwdCfg<D>;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(attn_tc::k_fwd_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int h = sh.a * D;
  CUtensorMap tm = make_qkv_tmap(qkv, sh.b * sh.s, 3 * h);
  const int grid = (sh.s / attn_tc::BQ + 1) / 2 * sh.a * sh.b;
  launch(PDL_ATTN, attn_tc::k_fwd_tc<D>, grid, 384, C::SMEM, st, tm, static_cast<bf16*>(o), lse, sh.s, sh.a,
                                                   attn_tc::LOG2E / sqrtf(static_cast<float>(D)));
  ZB_LAUNCH_CHECK();
}

bool attention_fwd_tc(const AttnShape& sh, const void* qkv, void* o, float* lse, cudaStream_t st) {
  if (sh.s % attn_tc::BQ != 0) return false;
  switch (sh.d) {
    case 64: fwd_tc_launch<64>(sh, qkv, o, lse, st); return true;
    case 96: fwd_tc_launch<96>(sh, qkv, o, lse, st); return true;
    case 128: fwd_tc_launch<128>(sh, qkv, o, lse, st); return true;
  }
  return false;
}

}  // namespace zb

#ifdef ZB_ATTN_TRACE
extern "C" int zb_dbg_attn_fwd_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_tc::g_trace_fwd, sizeof(unsigned long long) * 12 * 64));
}
#endif
