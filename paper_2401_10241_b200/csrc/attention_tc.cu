// Causal flash-attention FORWARD on tcgen05 (bf16, s % 128 == 0).
//
// One CTA per (128-query block, head, sequence), heavy blocks first.
//   warp 0      TMA: Q once; K_j (3-stage ring, one block ahead), V_j (2-stage ring) (boxes {64 cols, 128 rows}
//               of the packed qkv [b*s, 3h], 128B swizzle)
//   warp 1      MMA: S_j = Q K_j^T into one of two TMEM S buffers (128 cols each),
//               O += P_j V_j into the TMEM O accumulator (D cols); S_{j+1} is issued
//               before PV_j so the next QK^T overlaps this block's softmax
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  softmax, a row per thread pair (TMEM lane = row, one key half each): tcgen05.ld S,
//               causal mask, online max / sum in base 2, O rescale in TMEM
//               (tcgen05.ld/st, lazy: only when a row max grows by > 8), bf16 P written
//               into TMEM over its S buffer (tcgen05.st) and consumed by a TS MMA (A from
//               TMEM); finally O / l -> bf16 rows and the log-sum-exp.
// Operand layouts: Q, K are K-major SW128 (atoms of 64 elements x 8 rows);
// V is the MN-major B operand of PV (d contiguous), read from the same TMA boxes.
#include <math.h>

#include "attention.h"
#include "gemm.h"
#include "sm100.cuh"

namespace zb {
namespace attn_tc {

constexpr int BQ = 128, BKV = 128;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// barrier among the softmax warps only (ids 1+; 0 is __syncthreads)
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int D> struct FwdCfg {
  static constexpr int ATOMS = (D + 63) / 64;           // 64-column TMA boxes per tile
  static constexpr int TILE = ATOMS * 128 * 128;        // bytes of one 128-row tile (Q, K or V)
  static constexpr int KST = 3, VST = 2;                // K ring (freed after S_j), V ring (freed after PV_j)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = TILE;
  static constexpr int OFF_V = (1 + KST) * TILE;
  static constexpr int OFF_BAR = (1 + KST + VST) * TILE;
  static constexpr int OFF_RED = OFF_BAR + 256;          // 768 f32
  static constexpr int SMEM = OFF_RED + 3072 + 1024;
};

template <int D>
__global__ void __launch_bounds__(384, 1) k_fwd_tc(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ o,
                                                   float* __restrict__ lse, int s, int a, float scale_log2) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;     // [3]
  uint64_t* k_empty = bar + 4;    // [3]
  uint64_t* v_full = bar + 7;     // [2]
  uint64_t* v_empty = bar + 9;    // [2]
  uint64_t* s_full = bar + 11;    // [2]
  uint64_t* s_empty = bar + 13;   // [2]
  uint64_t* p_full = bar + 15;
  uint64_t* o_done = bar + 16;
  uint64_t* o_final = bar + 17;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / BQ;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x);
  const int hd = blockIdx.y, bb = blockIdx.z;
  const int h = a * D;
  const int nkv = qb + 1;

  if (threadIdx.x == 0) {
    sm100::mbar_init(q_full, 1);
    for (int i = 0; i < C::KST; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&s_empty[i], 1);  // released by the PV that consumed the P aliased over S
    }
    sm100::mbar_init(p_full, 256);
    sm100::mbar_init(o_done, 1);
    sm100::mbar_init(o_final, 1);
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
  const uint32_t t_s0 = tbase, t_o = tbase + 256;
  const int row0 = bb * s;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA
      sm100::mbar_arrive_expect_tx(q_full, C::TILE);
      for (int at = 0; at < C::ATOMS; ++at)
        sm100::tma_load_2d(smem + C::OFF_Q + at * 16384, &tm, q_full, hd * D + 64 * at, row0 + qb * BQ);
      auto load_k = [&](int j) {
        const int st = j % C::KST;
        sm100::mbar_wait(&k_empty[st], ((j / C::KST) & 1) ^ 1);
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
    if (lane == 0) {  // ---------------- MMA
      constexpr uint32_t idesc_s = sm100::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = sm100::idesc_bf16(128, D, false, true);
      const uint32_t sq = sm100::smem_addr(smem + C::OFF_Q);
      auto issue_pv = [&](int j, bool last) {
        const int st = j & 1;
        sm100::mbar_wait(&v_full[st], (j >> 1) & 1);
        sm100::mbar_wait(p_full, j & 1);
        sm100::tc_fence_after();
        const uint32_t sv = sm100::smem_addr(smem + C::OFF_V + st * C::TILE);
        const uint32_t tp = t_s0 + st * 128;  // P_j (bf16 pairs) aliased over S_j
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint64_t bd = sm100::smem_desc(sv + kk * 2048, 16384, 1024, sm100::kSwizzle128B);
          sm100::mma_bf16_ts(t_o, tp + kk * 8, bd, idesc_o, (j | kk) != 0 ? 1u : 0u);
        }
        sm100::mma_commit(o_done);
        sm100::mma_commit(&s_empty[st]);
        sm100::mma_commit(&v_empty[st]);
        if (last) sm100::mma_commit(o_final);
      };
      sm100::mbar_wait(q_full, 0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::KST, sb = j & 1;
        sm100::mbar_wait(&k_full[st], (j / C::KST) & 1);
        sm100::mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t sk = sm100::smem_addr(smem + C::OFF_K + st * C::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          sm100::mma_bf16_ss(t_s0 + sb * 128, sm100::smem_desc(sq + off, 16, 1024, sm100::kSwizzle128B),
                             sm100::smem_desc(sk + off, 16, 1024, sm100::kSwizzle128B), idesc_s, kk != 0 ? 1u : 0u);
        }
        sm100::mma_commit(&s_full[sb]);
        sm100::mma_commit(&k_empty[st]);
        if (j > 0) issue_pv(j - 1, false);
      }
      issue_pv(nkv - 1, true);
    }
  } else if (warp >= 4) {  // ---------------- softmax: two warps per row group, one key half each
    const int qw = warp & 3, hf = (warp - 4) >> 2;
    const int r = qw * 32 + lane;  // row within the block = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [2 parity][2][128] maxima, [2][128] sums
    float m = -INFINITY, l = 0.f;  // m: running max (log2 units) shared by both halves; l: this half's sum
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      sm100::mbar_wait(&s_full[sb], (j >> 1) & 1);
      sm100::tc_fence_after();
      float sv[64];
#pragma unroll
      for (int c = 0; c < 2; ++c)
        sm100::tmem_ld32(t_s0 + sb * 128 + hf * 64 + lane_off + c * 32, reinterpret_cast<uint32_t*>(sv + 32 * c));
      sm100::tmem_ld_wait();
      float mx = -INFINITY;
      const bool diag = j == qb;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        float x = sv[k] * scale_log2;
        if (diag && hf * 64 + k > r) x = -INFINITY;
        sv[k] = x;
        mx = fmaxf(mx, x);
      }
      float* rj = red + (j & 1) * 256;  // double-buffered by block parity: no write-after-read race
      rj[hf * 128 + r] = mx;
      named_sync(1, 256);
      mx = fmaxf(mx, rj[(hf ^ 1) * 128 + r]);
      // lazy rescaling: keep the old reference max unless it grew by more than 8 (p <= 2^8)
      float corr = 1.f;
      if (mx > m + 8.f) {
        corr = sm100::ex2(m - mx);
        m = mx;
      }
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const float pv = sm100::ex2(sv[k] - m);
        sv[k] = pv;
        sum += pv;
      }
      l = l * corr + sum;
      if (j > 0) {  // PV_{j-1} has finished: O may be rescaled and the P buffer is free
        sm100::mbar_wait(o_done, (j - 1) & 1);
        sm100::tc_fence_after();
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int c = hf; c < D / 32; c += 2) {
            uint32_t ov[32];
            sm100::tmem_ld32(t_o + lane_off + c * 32, ov);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
            sm100::tmem_st32(t_o + lane_off + c * 32, ov);
          }
          sm100::tmem_st_wait();
        }
      }
      // P row half -> TMEM over this S buffer: keys [64 hf, 64 hf + 64) -> columns [32 hf, 32 hf + 32)
      // (both halves finished reading S before the max exchange above)
      uint32_t pk[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        __nv_bfloat162 v2 = __floats2bfloat162_rn(sv[2 * i], sv[2 * i + 1]);
        pk[i] = *reinterpret_cast<uint32_t*>(&v2);
      }
      sm100::tmem_st32(t_s0 + sb * 128 + hf * 32 + lane_off, pk);
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(p_full);
    }
    red[512 + hf * 128 + r] = l;
    named_sync(1, 256);
    l += red[512 + (hf ^ 1) * 128 + r];
    sm100::mbar_wait(o_final, 0);
    sm100::tc_fence_after();
    const int q = qb * BQ + r;
    const float inv = 1.f / l;
    bf16* orow = o + (static_cast<int64_t>(bb) * s + q) * h + hd * D;
#pragma unroll 1
    for (int c = hf; c < D / 32; c += 2) {
      uint32_t ov[32];
      sm100::tmem_ld32(t_o + lane_off + c * 32, ov);
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
    if (hf == 0) lse[(static_cast<int64_t>(bb) * a + hd) * s + q] = (m + log2f(l)) * LN2;
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
  dim3 grid(sh.s / attn_tc::BQ, sh.a, sh.b);
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
