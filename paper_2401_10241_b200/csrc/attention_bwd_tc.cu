// Causal flash-attention BACKWARD on tcgen05 (bf16, s % 128 == 0), deterministic:
// one kernel owns dK / dV of a 128-key block, another owns dQ of a 128-query block.
//
// dK/dV kernel (per key block kb, loop over 64-query blocks i >= 2 kb):
//   MMA   S^T = K Q_i^T, dP^T = V dO_i^T             (M = 128 keys, N = 64 queries; K (and V
//         when the TMEM columns allow, d <= 64) copied once into TMEM: TS, else SS)
//   warps 4-11 (key row per thread pair, one query half each):
//         P^T = exp2(S^T c - lse_q log2 e) (causal), dS^T = P^T (dP^T - D_q),
//         both written back as bf16 into TMEM over their own S^T / dP^T columns
//   MMA   dV += P^T dO_i, dK += dS^T Q_i              (TS: A from TMEM, B = dO_i / Q_i MN-major)
//   S^T / dP^T are double-buffered (2 x 128 columns) so block i+1's products overlap
//   block i's elementwise work; dK, dV accumulate in TMEM (2 x D columns).
// dQ kernel (per query block, loop over 64-key blocks j <= 2 qb + 1):
//   MMA   S = Q K_j^T, dP = dO V_j^T (TS: Q, dO copied once into TMEM);
//         dS = P (dP - D) -> TMEM;  dQ += dS K_j (TS).
// Q, dO, L, D of a query block arrive by TMA / bulk copy in a 3-stage ring.
#include <math.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>
#include <type_traits>
#include <vector>

#include "attention.h"
#include "gemm.h"
#include "sm100.cuh"

namespace zb {
namespace attn_bwd_tc {

constexpr float LOG2E = 1.4426950408889634f;

#ifdef ZB_ATTN_TRACE
// timeline of one CTA (blockIdx (TR_BX, 0, 0)) of k_dkdv_tc, globaltimer ns (measurement build only)
__device__ unsigned long long g_trace[12][64];
#ifndef TR_BX
#define TR_BX 0
#endif
__device__ __forceinline__ void tr(int row, int n) {
  if (blockIdx.x == TR_BX && blockIdx.y == 0 && blockIdx.z == 0 && n < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[row][n] = t;
  }
}
#define TR(row, n) tr(row, n)
__device__ unsigned long long g_cta_bwd[16384][3];  // every CTA: {smid, start, end}
// per-item events of CTA 0, warp 4 lane 0 (row = body * 5 + event, column = item of the body):
// 0 item start (K / V or Q / dO resident), 1 first step's S ready, 2 last step published,
// 3 final accumulator seen, 4 epilogue stored
__device__ unsigned long long g_item_bwd[10][16];
__device__ __forceinline__ void tri_b(int e, int r) {
  if (blockIdx.x == 0 && r < 16) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_item_bwd[e][r] = t;
  }
}
#define TRB(e, r) tri_b(e, r)
__device__ __forceinline__ unsigned long long gtime_b() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define TR(row, n)
#define TRB(e, r)
#endif

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// One 32-column chunk of the calling warp's 32 rows (v: this thread's row, f32, times mul) to
// global memory by a TMA tensor store (box 32 rows x 64 B, SWIZZLE_64B: 16-B piece k of row i
// at piece k ^ ((i >> 1) & 3)) from one of the warp's two 2 KB staging buffers (stg, stg +
// 2048, alternating with nbuf).  The warp only writes shared memory and waits for the store
// issued two chunks earlier to have READ its buffer; the global writes drain asynchronously
// while the warp moves on to the next item.  (Row-per-thread 16-B global stores touched 32
// lines per instruction; row-contiguous stores from the warp itself made the epilogue
// write-bandwidth-bound when every CTA reached it at once: ~2 us per dK/dV item.)
// Lane 0 issues and owns the bulk groups.
__device__ __forceinline__ void store_chunk_tma(uint32_t stg, int& nbuf, const uint32_t* v, float mul,
                                                const CUtensorMap* tm, int col, int row, int lane) {
  const uint32_t buf = stg + (nbuf & 1) * 2048;
  if (lane == 0) sm100::bulk_wait_read<1>();  // this buffer's previous store has read it
  __syncwarp();
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint32_t x = pack_bf16(__uint_as_float(v[8 * g]) * mul, __uint_as_float(v[8 * g + 1]) * mul);
    const uint32_t y = pack_bf16(__uint_as_float(v[8 * g + 2]) * mul, __uint_as_float(v[8 * g + 3]) * mul);
    const uint32_t z = pack_bf16(__uint_as_float(v[8 * g + 4]) * mul, __uint_as_float(v[8 * g + 5]) * mul);
    const uint32_t w = pack_bf16(__uint_as_float(v[8 * g + 6]) * mul, __uint_as_float(v[8 * g + 7]) * mul);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4)),
                 "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
  }
  sm100::fence_proxy_async();  // generic-proxy shared writes -> visible to the TMA (async proxy)
  __syncwarp();
  if (lane == 0) {
    sm100::tma_store_2d_sa(tm, buf, col, row);
    sm100::bulk_commit();
  }
  ++nbuf;
}

// Row r (0..127) of a 128-row SWIZZLE_128B bf16 tile (D columns in 64-column atoms 16 KB apart,
// 16-byte chunk c of row r stored at chunk c ^ (r & 7)) into TMEM lane r, columns
// [taddr, taddr + D/2) as packed bf16 pairs (low half = even column): the A-operand layout of a
// TS tcgen05.mma, so a CTA-constant A tile is read from TMEM by every product instead of from
// shared memory (an SS product streams A AND B through the shared-memory port; the A read is
// what bounds the small-N products of these kernels).  Warp-collective: the calling warp
// (warp % 4 == r / 32) owns TMEM lanes 32 (warp % 4) ..; taddr carries that lane offset.
template <int D>
__device__ __forceinline__ void tile_row_to_tmem(const uint8_t* tile, int r, uint32_t taddr) {
  static_assert(D % 32 == 0, "head dim");
#pragma unroll
  for (int g = 0; g < D / 32; ++g) {
    uint32_t w[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int gc = g * 4 + c;
      const uint4 u = *reinterpret_cast<const uint4*>(tile + (gc >> 3) * 16384 + r * 128 + (((gc & 7) ^ (r & 7)) << 4));
      w[4 * c] = u.x;
      w[4 * c + 1] = u.y;
      w[4 * c + 2] = u.z;
      w[4 * c + 3] = u.w;
    }
    sm100::tmem_st16(taddr + g * 16, w);
  }
}

// item (level, head, sequence) of a level-major list (per = a b items per level)
__device__ __forceinline__ void decode_item(int it, int a, int per, int& level, int& hd, int& bb) {
  level = it / per;
  hd = it % per % a;
  bb = it % per / a;
}

// ================================================================== dK / dV
template <int D> struct DkdvCfg {
  // TMEM: S^T / dP^T x 2 buffers (256 columns), dK, dV (D each), then the CTA-constant A
  // operands K (and V) as packed bf16 (D/2 each) where the 512 columns allow it
  static constexpr bool KT = 256 + 2 * D + D / 2 <= 512;
  static constexpr bool VT = 256 + 2 * D + D <= 512;
  static constexpr int ATOMS = (D + 63) / 64;
  static constexpr int KV_TILE = ATOMS * 16384;  // 128 rows
  static constexpr int Q_TILE = ATOMS * 8192;    // 64 rows
  // Q_i / dO_i ring depth.  The globaltimer trace (scripts/attn_trace.py) shows ~1.1 us per
  // 64-query step with Q_i / dO_i arriving ~1.1 us after issue; ST = 4 moved the issue 2.3 us
  // ahead without shortening the step (arrivals stay ~1.1 us apart), so 3 stages suffice
  static constexpr int ST = 3;
  static constexpr int STAGE = 2 * Q_TILE + 1024;  // Q_i, dO_i, L_i[64], D_i[64] (1024-aligned)
  static constexpr int OFF_K = 0, OFF_V = KV_TILE, OFF_ST = 2 * KV_TILE;
  static constexpr int OFF_BAR = OFF_ST + ST * STAGE;
  static constexpr int OFF_OST = OFF_BAR + 1024;  // epilogue staging: 8 elementwise warps x 2 x 2 KB
  static constexpr int SMEM = OFF_OST + 8 * 4096 + 1024;
};

// Persistent over this CTA's dK/dV items (key block kb = level, head, sequence): barriers,
// TMEM and the Q_i / dO_i ring stay live across items, barrier parities come from running
// counters (items `ri`, query steps `gn`).  Per item the next item's K / V load waits only
// for the last S^T / dP^T products of the current item (kv_empty), and its first dV / dK
// products only for the softmax warps having read the current dK / dV (o_empty), so one
// item's epilogue overlaps the next item's first steps.  (The tensor maps are references to
// the launching kernel's __grid_constant__ parameters.)
template <int D, typename ItemOf>
__device__ __forceinline__ void dkdv_run(const CUtensorMap& tmKV, const CUtensorMap& tmQ, const CUtensorMap& tmDO,
                                         const CUtensorMap& tmOut, const float* __restrict__ lse,
                                         const float* __restrict__ delta, bf16* __restrict__ dqkv, int s, int a,
                                         int per, float scale,
                                         float scale_log2, uint32_t tbase, ItemOf item_of) {
  using C = DkdvCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* st_full = bar + 1;                 // [ST]
  uint64_t* st_empty = st_full + C::ST;        // [ST]
  uint64_t* sp_full = st_empty + C::ST;        // [2]
  uint64_t* sp_empty = sp_full + 2;            // [2]
  uint64_t* ds_full = sp_empty + 2;            // [2]
  uint64_t* o_final = ds_full + 2;
  uint64_t* at_full = o_final + 1;  // K (V) resident in TMEM
  uint64_t* ds_part = bar + 16;  // [2]: the first 16 queries / keys of each half are in TMEM
  uint64_t* kv_empty = bar + 18;  // the item's last S^T / dP^T products have read K / V
  uint64_t* o_empty = bar + 19;   // the elementwise warps have read dK / dV of their item
  constexpr int NBAR = 20;
  static_assert((NBAR + 1) * 8 <= 256, "barrier area");
  static_assert((1 + 2 * C::ST + 8) <= 16, "barrier layout");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = a * D;
  if (threadIdx.x == 0) {
    sm100::mbar_init(kv_full, 1);
    for (int i = 0; i < C::ST; ++i) {
      sm100::mbar_init(&st_full[i], 1);
      sm100::mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&sp_full[i], 1);
      sm100::mbar_init(&sp_empty[i], 1);
      sm100::mbar_init(&ds_full[i], 8);  // one arrival per elementwise warp
      sm100::mbar_init(&ds_part[i], 8);
    }
    sm100::mbar_init(o_final, 1);
    sm100::mbar_init(at_full, 8);
    sm100::mbar_init(kv_empty, 1);
    sm100::mbar_init(o_empty, 8);
#ifdef ZB_ATTN_TRACE
    sm100::mbar_init(bar + 20, 1);
#endif
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t t_dk = tbase + 256, t_dv = tbase + 256 + D;
  const uint32_t t_kt = tbase + 256 + 2 * D, t_vt = t_kt + D / 2;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA / bulk copies
      int gn = 0;  // query steps issued (ring position)
      for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
        int kb, hd, bb;
        decode_item(it, a, per, kb, hd, bb);
        const int i0 = 2 * kb, nq = s / 64 - i0, row0 = bb * s;
        const int64_t stat0 = (static_cast<int64_t>(bb) * a + hd) * s;
        sm100::mbar_wait(kv_empty, (ri & 1) ^ 1);  // the previous item's S^T / dP^T are done with K / V
        sm100::mbar_arrive_expect_tx(kv_full, 2 * C::KV_TILE);
        for (int at = 0; at < C::ATOMS; ++at) {
          sm100::tma_load_2d(smem + C::OFF_K + at * 16384, &tmKV, kv_full, h + hd * D + 64 * at, row0 + kb * 128);
          sm100::tma_load_2d(smem + C::OFF_V + at * 16384, &tmKV, kv_full, 2 * h + hd * D + 64 * at, row0 + kb * 128);
        }
        for (int n = 0; n < nq; ++n, ++gn) {
          const int i = i0 + n, st = gn % C::ST;
          sm100::mbar_wait(&st_empty[st], ((gn / C::ST) & 1) ^ 1);
          if (ri == 0) TR(0, n);
          uint8_t* sg = smem + C::OFF_ST + st * C::STAGE;
          sm100::mbar_arrive_expect_tx(&st_full[st], 2 * C::Q_TILE + 512);
          for (int at = 0; at < C::ATOMS; ++at) {
            sm100::tma_load_2d(sg + at * 8192, &tmQ, &st_full[st], hd * D + 64 * at, row0 + i * 64);
            sm100::tma_load_2d(sg + C::Q_TILE + at * 8192, &tmDO, &st_full[st], hd * D + 64 * at, row0 + i * 64);
          }
          sm100::bulk_load(sg + 2 * C::Q_TILE, lse + stat0 + i * 64, 256, &st_full[st]);
          sm100::bulk_load(sg + 2 * C::Q_TILE + 256, delta + stat0 + i * 64, 256, &st_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA
      constexpr uint32_t idesc_s = sm100::idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_g = sm100::idesc_bf16(128, D, false, true);
      const uint32_t sk = sm100::smem_addr(smem + C::OFF_K), sv = sm100::smem_addr(smem + C::OFF_V);
      int gn = 0;  // query steps whose S^T / dP^T were issued
      for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
        int kb, hd, bb;
        decode_item(it, a, per, kb, hd, bb);
        const int nq = s / 64 - 2 * kb;
        const int g0 = gn;  // first step of the item
        auto issue_grad = [&](int g) {  // step g (global count) of this item
          const int n = g - g0;
          const int b = g & 1, st = g % C::ST;
          const uint32_t sq = sm100::smem_addr(smem + C::OFF_ST + st * C::STAGE);
          const uint32_t sdo = sq + C::Q_TILE;
          const uint32_t tp = tbase + b * 128;
          const uint64_t dod = sm100::smem_desc(sdo, 8192, 1024, sm100::kSwizzle128B);
          const uint64_t qd = sm100::smem_desc(sq, 8192, 1024, sm100::kSwizzle128B);
          if (n == 0) sm100::mbar_wait_warp(o_empty, (ri & 1) ^ 1);  // dK / dV of the previous item read
          // K = 64 queries: halves live at columns [0,16) and [32,48); each half's first 16 queries
          // (K-steps 0 and 2) are published before its last 16 (K-steps 1 and 3)
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            sm100::mbar_wait_warp(part == 0 ? &ds_part[b] : &ds_full[b], (g >> 1) & 1);
            if (part == 1 && ri == 0) TR(3, n);
            sm100::tc_fence_after();
            if (sm100::elect_one()) {
#pragma unroll
              for (int kh = 0; kh < 2; ++kh) {
                const int kk = 2 * kh + part;
                const uint32_t acol = kh * 32 + part * 8;
                sm100::mma_bf16_ts(t_dv, tp + acol, sm100::desc_adv(dod, kk * 2048), idesc_g, (n | kk) != 0 ? 1u : 0u);
                sm100::mma_bf16_ts(t_dk, tp + 64 + acol, sm100::desc_adv(qd, kk * 2048), idesc_g, (n | kk) != 0 ? 1u : 0u);
              }
            }
            __syncwarp();
          }
          if (ri == 0) TR(10, n);
          if (sm100::elect_one()) sm100::mma_commit(&sp_empty[b]);
          if (sm100::elect_one()) sm100::mma_commit(&st_empty[st]);
#ifdef ZB_ATTN_TRACE
          if (ri == 0) { if (sm100::elect_one()) sm100::mma_commit(bar + 20); }
#endif
          if (n == nq - 1) { if (sm100::elect_one()) sm100::mma_commit(o_final); }
        };
        sm100::mbar_wait_warp(kv_full, ri & 1);
        if constexpr (C::KT) {
          sm100::mbar_wait_warp(at_full, ri & 1);
          sm100::tc_fence_after();
        }
        for (int n = 0; n < nq; ++n, ++gn) {
          const int b = gn & 1, st = gn % C::ST;
          sm100::mbar_wait_warp(&st_full[st], (gn / C::ST) & 1);
          if (ri == 0) TR(1, n);
          sm100::mbar_wait_warp(&sp_empty[b], ((gn >> 1) & 1) ^ 1);
          if (ri == 0) TR(2, n);
          sm100::tc_fence_after();
          const uint32_t sq = sm100::smem_addr(smem + C::OFF_ST + st * C::STAGE);
          const uint32_t sdo = sq + C::Q_TILE;
          const uint32_t tp = tbase + b * 128;
          const uint64_t kd = sm100::smem_desc(sk, 16, 1024, sm100::kSwizzle128B);
          const uint64_t vd = sm100::smem_desc(sv, 16, 1024, sm100::kSwizzle128B);
          const uint64_t qd = sm100::smem_desc(sq, 16, 1024, sm100::kSwizzle128B);
          const uint64_t dod = sm100::smem_desc(sdo, 16, 1024, sm100::kSwizzle128B);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * 16384 + (kk & 3) * 32, ob = (kk >> 2) * 8192 + (kk & 3) * 32;
            if (sm100::elect_one()) {
              if constexpr (C::KT)
                sm100::mma_bf16_ts(tp, t_kt + kk * 8, sm100::desc_adv(qd, ob), idesc_s, kk != 0 ? 1u : 0u);
              else
                sm100::mma_bf16_ss(tp, sm100::desc_adv(kd, oa), sm100::desc_adv(qd, ob), idesc_s, kk != 0 ? 1u : 0u);
              if constexpr (C::VT)
                sm100::mma_bf16_ts(tp + 64, t_vt + kk * 8, sm100::desc_adv(dod, ob), idesc_s, kk != 0 ? 1u : 0u);
              else
                sm100::mma_bf16_ss(tp + 64, sm100::desc_adv(vd, oa), sm100::desc_adv(dod, ob), idesc_s, kk != 0 ? 1u : 0u);
            }
          }
          if (ri == 0) TR(11, n);
          if (sm100::elect_one()) sm100::mma_commit(&sp_full[b]);
          if (n == nq - 1) { if (sm100::elect_one()) sm100::mma_commit(kv_empty); }  // last reads of K / V
          if (n > 0) issue_grad(gn - 1);
        }
        issue_grad(gn - 1);
      }
    }
#ifdef ZB_ATTN_TRACE
  } else if (warp == 3) {  // trace observer (first item): completion of each step's dV / dK products
    const int it0 = item_of(0);
    if (lane == 0 && it0 >= 0) {
      int kb, hd, bb;
      decode_item(it0, a, per, kb, hd, bb);
      for (int n = 0; n < s / 64 - 2 * kb; ++n) {
        sm100::mbar_wait(bar + 20, n & 1);
        TR(9, n);
      }
    }
#endif
  } else if (warp >= 4) {  // ---------------- elementwise: P^T, dS^T
    const int qw = warp & 3, hf = (warp - 4) >> 2;
    const int r = qw * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    const uint32_t stg = sm100::smem_addr(smem + C::OFF_OST) + (warp - 4) * 4096;  // epilogue staging (2 x 2 KB)
    int nbuf = 0;
    int gn = 0;
    // K (and V) of item ri into TMEM (TS A operands, d <= 96): waits for the tiles in shared
    // memory and for the previous item's products to be done with the TMEM copies
    auto copy_kv = [&](int ri_) {
      if constexpr (C::KT) {
        sm100::mbar_wait(kv_full, ri_ & 1);
        sm100::mbar_wait(kv_empty, (ri_ & 1) ^ 1);
        if (hf == 0) tile_row_to_tmem<D>(smem + C::OFF_K, r, t_kt + lane_off);
        if (C::VT && hf == 1) tile_row_to_tmem<D>(smem + C::OFF_V, r, t_vt + lane_off);
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive_warp(at_full);
      }
    };
    if (item_of(0) >= 0) copy_kv(0);
    for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
      int kb, hd, bb;
      decode_item(it, a, per, kb, hd, bb);
      const int i0 = 2 * kb, nq = s / 64 - i0, row0 = bb * s;
      const int key = kb * 128 + r;
      if (warp == 4 && lane == 0) TRB(0, ri);
      for (int n = 0; n < nq; ++n, ++gn) {
        const int i = i0 + n, b = gn & 1, st = gn % C::ST;
        sm100::mbar_wait(&sp_full[b], (gn >> 1) & 1);
        if (warp == 4 && lane == 0 && n == 0) TRB(1, ri);
        if (warp == 4 && lane == 0 && ri == 0) TR(4, n);
        sm100::tc_fence_after();
        uint32_t sr[32], dr[32];
        const uint32_t tp = tbase + b * 128 + lane_off;
        sm100::tmem_ld32(tp + 32 * hf, sr);
        sm100::tmem_ld32(tp + 64 + 32 * hf, dr);
        sm100::tmem_ld_wait();
        // this half's 32 L_q and D_q (warp-uniform: broadcast loads), L in log2 units
        float nl[32], dd[32];
        {
          const uint32_t sl = sm100::smem_addr(smem + C::OFF_ST + st * C::STAGE + 2 * C::Q_TILE) + 128 * hf;
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 l4 = sm100::lds128(sl + 4 * c), d4 = sm100::lds128(sl + 256 + 4 * c);
            nl[c] = -l4.x * LOG2E, nl[c + 1] = -l4.y * LOG2E, nl[c + 2] = -l4.z * LOG2E, nl[c + 3] = -l4.w * LOG2E;
            dd[c] = d4.x, dd[c + 1] = d4.y, dd[c + 2] = d4.z, dd[c + 3] = d4.w;
          }
        }
        if (warp == 4 && lane == 0 && ri == 0) TR(7, n);
        // queries of this half: i*64 + 32 hf + c; the causal mask (q >= key) only bites on blocks
        // that reach below the diagonal of this key block
        const int qlo = i * 64 + 32 * hf;
        const bool diag = qlo < kb * 128 + 128;
        uint32_t pk[16], dk[16];
        // the mask test only on the (warp-uniform) diagonal steps: off the diagonal the
        // compare / select / index arithmetic was a third of the loop's instructions
        auto elementwise = [&](auto masked, int c0) {
#pragma unroll
          for (int c = c0; c < c0 + 16; c += 2) {
            float pv[2], dv[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float p = sm100::ex2(fmaf(__uint_as_float(sr[c + e]), scale_log2, nl[c + e]));
              if constexpr (decltype(masked)::value)
                if (qlo + c + e < key) p = 0.f;
              pv[e] = p;
              dv[e] = p * (__uint_as_float(dr[c + e]) - dd[c + e]);
            }
            pk[c >> 1] = pack_bf16(pv[0], pv[1]);
            dk[c >> 1] = pack_bf16(dv[0], dv[1]);
          }
        };
        // two parts of 16 queries: the grad products of the first overlap the second's exponentials
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          if (diag)
            elementwise(std::true_type{}, 16 * part);
          else
            elementwise(std::false_type{}, 16 * part);
          sm100::tmem_st8(tp + 32 * hf + 8 * part, pk + 8 * part);       // P^T over this half's S^T columns
          sm100::tmem_st8(tp + 64 + 32 * hf + 8 * part, dk + 8 * part);  // dS^T over this half's dP^T columns
          if (part == 0) {
            sm100::tmem_st_wait();
            sm100::tc_fence_before();
            sm100::mbar_arrive_warp(&ds_part[b]);
          }
        }
        if (warp == 4 && lane == 0 && ri == 0) TR(8, n);
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        if (warp == 4 && lane == 0 && ri == 0) TR(5, n);
        sm100::mbar_arrive_warp(&ds_full[b]);
      }
      if (warp == 4 && lane == 0) TRB(2, ri);
      // the next item's K / V copies before this item's epilogue (its first S^T / dP^T products
      // then run while the dK / dV stores are prepared)
      if (item_of(ri + 1) >= 0) copy_kv(ri + 1);
      sm100::mbar_wait(o_final, ri & 1);
      if (warp == 4 && lane == 0) TRB(3, ri);
      if (warp == 4 && lane == 0 && ri == 0) TR(6, 1);
      sm100::tc_fence_after();
      (void)key;
      const int wr = row0 + kb * 128 + qw * 32;  // the warp's first row of dqkv
#pragma unroll 1
      for (int c = hf; c < D / 32; c += 2) {
        uint32_t v[32];
        sm100::tmem_ld32(t_dk + lane_off + c * 32, v);
        sm100::tmem_ld_wait();
        store_chunk_tma(stg, nbuf, v, scale, &tmOut, h + hd * D + c * 32, wr, lane);
        sm100::tmem_ld32(t_dv + lane_off + c * 32, v);
        sm100::tmem_ld_wait();
        store_chunk_tma(stg, nbuf, v, 1.f, &tmOut, 2 * h + hd * D + c * 32, wr, lane);
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive_warp(o_empty);  // dK / dV may be overwritten by the next item
      if (warp == 4 && lane == 0) TRB(4, ri);
    }
    if (lane == 0) sm100::bulk_wait<0>();  // epilogue stores complete (staging reused by the next body / exit)
  }
  // every role is done (all commits observed by their waiters): the barrier memory may be reused
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBAR; ++i)
      if (i != 15) sm100::mbar_inval(bar + i);  // 15: unused
#ifdef ZB_ATTN_TRACE
    sm100::mbar_inval(bar + 20);
#endif
  }
  __syncthreads();
}

// ================================================================== dQ
template <int D> struct DqCfg {
  static constexpr int ATOMS = (D + 63) / 64;
  static constexpr int Q_TILE = ATOMS * 16384;   // 128 rows
  static constexpr int KV_TILE = ATOMS * 8192;   // 64 rows
  static constexpr int ST = 3;  // K_j / V_j ring depth (see DkdvCfg)
  static constexpr int STAGE = 2 * KV_TILE;      // K_j, V_j
  static constexpr int OFF_Q = 0, OFF_DO = Q_TILE, OFF_ST = 2 * Q_TILE;
  static constexpr int OFF_BAR = OFF_ST + ST * STAGE;
  static constexpr int OFF_OST = OFF_BAR + 1024;  // epilogue staging: 8 elementwise warps x 2 x 2 KB
  static constexpr int SMEM = OFF_OST + 8 * 4096 + 1024;
};

// Persistent over this CTA's dQ items (query block nqb-1-level, head, sequence); running
// counters as in dkdv_run.  Q / dO of an item are only read by their copies into TMEM (the
// products are TS), so the next item's Q / dO load waits for those copies (at_full), the next
// copies for the current item's last S / dP products (qt_empty), and the next item's first dQ
// product for the current dQ having been read (o_empty).
template <int D, typename ItemOf>
__device__ __forceinline__ void dq_run(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const CUtensorMap& tmDO,
                                       const CUtensorMap& tmOut, const float* __restrict__ lse,
                                       const float* __restrict__ delta,
                                       bf16* __restrict__ dqkv, int s, int a, int per, float scale, float scale_log2,
                                       uint32_t tbase, ItemOf item_of) {
  using C = DqCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* st_full = bar + 1;                 // [ST]
  uint64_t* st_empty = st_full + C::ST;        // [ST]
  uint64_t* sp_full = st_empty + C::ST;        // [2]
  uint64_t* sp_empty = sp_full + 2;            // [2]
  uint64_t* ds_full = sp_empty + 2;            // [2]
  uint64_t* o_final = ds_full + 2;
  uint64_t* at_full = o_final + 1;  // Q, dO resident in TMEM
  uint64_t* ds_part = bar + 16;  // [2]: the first 16 queries / keys of each half are in TMEM
  uint64_t* qt_empty = bar + 18;  // the item's last S / dP products have read Q / dO in TMEM
  uint64_t* o_empty = bar + 19;   // the elementwise warps have read dQ of their item
  constexpr int NBAR = 20;
  static_assert((NBAR + 1) * 8 <= 256, "barrier area");
  static_assert(256 + 2 * D <= 512, "TMEM: S/dP x 2, dQ, Q and dO as packed bf16");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / 128;
  const int h = a * D;
  if (threadIdx.x == 0) {
    sm100::mbar_init(q_full, 1);
    for (int i = 0; i < C::ST; ++i) {
      sm100::mbar_init(&st_full[i], 1);
      sm100::mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&sp_full[i], 1);
      sm100::mbar_init(&sp_empty[i], 1);
      sm100::mbar_init(&ds_full[i], 8);  // one arrival per elementwise warp
      sm100::mbar_init(&ds_part[i], 8);
    }
    sm100::mbar_init(o_final, 1);
    sm100::mbar_init(at_full, 8);
    sm100::mbar_init(qt_empty, 1);
    sm100::mbar_init(o_empty, 8);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t t_dq = tbase + 256;
  const uint32_t t_qt = tbase + 256 + D, t_dot = t_qt + D / 2;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA
      int gj = 0;  // key steps issued (ring position)
      for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
        int level, hd, bb;
        decode_item(it, a, per, level, hd, bb);
        const int qb = nqb - 1 - level, nkv = 2 * qb + 2, row0 = bb * s;
        sm100::mbar_wait(at_full, (ri & 1) ^ 1);  // the previous item's Q / dO were copied into TMEM
        sm100::mbar_arrive_expect_tx(q_full, 2 * C::Q_TILE);
        for (int at = 0; at < C::ATOMS; ++at) {
          sm100::tma_load_2d(smem + C::OFF_Q + at * 16384, &tmQ, q_full, hd * D + 64 * at, row0 + qb * 128);
          sm100::tma_load_2d(smem + C::OFF_DO + at * 16384, &tmDO, q_full, hd * D + 64 * at, row0 + qb * 128);
        }
        for (int j = 0; j < nkv; ++j, ++gj) {
          const int st = gj % C::ST;
          sm100::mbar_wait(&st_empty[st], ((gj / C::ST) & 1) ^ 1);
          uint8_t* sg = smem + C::OFF_ST + st * C::STAGE;
          sm100::mbar_arrive_expect_tx(&st_full[st], 2 * C::KV_TILE);
          for (int at = 0; at < C::ATOMS; ++at) {
            sm100::tma_load_2d(sg + at * 8192, &tmKV, &st_full[st], h + hd * D + 64 * at, row0 + j * 64);
            sm100::tma_load_2d(sg + C::KV_TILE + at * 8192, &tmKV, &st_full[st], 2 * h + hd * D + 64 * at,
                               row0 + j * 64);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA
      constexpr uint32_t idesc_s = sm100::idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_g = sm100::idesc_bf16(128, D, false, true);
      int gj = 0;
      for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
        int level, hd, bb;
        decode_item(it, a, per, level, hd, bb);
        const int nkv = 2 * (nqb - 1 - level) + 2;
        const int g0 = gj;
        auto issue_dq = [&](int g) {
          const int j = g - g0;
          const int b = g & 1, st = g % C::ST;
          const uint32_t skj = sm100::smem_addr(smem + C::OFF_ST + st * C::STAGE);
          const uint32_t tp = tbase + b * 128;
          const uint64_t kjd = sm100::smem_desc(skj, 8192, 1024, sm100::kSwizzle128B);
          if (j == 0) sm100::mbar_wait_warp(o_empty, (ri & 1) ^ 1);  // dQ of the previous item read
#pragma unroll
          for (int part = 0; part < 2; ++part) {  // see dkdv_run
            sm100::mbar_wait_warp(part == 0 ? &ds_part[b] : &ds_full[b], (g >> 1) & 1);
            sm100::tc_fence_after();
            if (sm100::elect_one()) {
#pragma unroll
              for (int kh = 0; kh < 2; ++kh) {
                const int kk = 2 * kh + part;
                sm100::mma_bf16_ts(t_dq, tp + kh * 32 + part * 8, sm100::desc_adv(kjd, kk * 2048), idesc_g,
                                   (j | kk) != 0 ? 1u : 0u);
              }
            }
            __syncwarp();
          }
          if (sm100::elect_one()) sm100::mma_commit(&sp_empty[b]);
          if (sm100::elect_one()) sm100::mma_commit(&st_empty[st]);
          if (j == nkv - 1) { if (sm100::elect_one()) sm100::mma_commit(o_final); }
        };
        sm100::mbar_wait_warp(at_full, ri & 1);
        sm100::tc_fence_after();
        for (int j = 0; j < nkv; ++j, ++gj) {
          const int b = gj & 1, st = gj % C::ST;
          sm100::mbar_wait_warp(&st_full[st], (gj / C::ST) & 1);
          sm100::mbar_wait_warp(&sp_empty[b], ((gj >> 1) & 1) ^ 1);
          sm100::tc_fence_after();
          const uint32_t skj = sm100::smem_addr(smem + C::OFF_ST + st * C::STAGE);
          const uint32_t svj = skj + C::KV_TILE;
          const uint32_t tp = tbase + b * 128;
          const uint64_t kjd = sm100::smem_desc(skj, 16, 1024, sm100::kSwizzle128B);
          const uint64_t vjd = sm100::smem_desc(svj, 16, 1024, sm100::kSwizzle128B);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ob = (kk >> 2) * 8192 + (kk & 3) * 32;
            if (sm100::elect_one()) {
              sm100::mma_bf16_ts(tp, t_qt + kk * 8, sm100::desc_adv(kjd, ob), idesc_s, kk != 0 ? 1u : 0u);
              sm100::mma_bf16_ts(tp + 64, t_dot + kk * 8, sm100::desc_adv(vjd, ob), idesc_s, kk != 0 ? 1u : 0u);
            }
          }
          if (sm100::elect_one()) sm100::mma_commit(&sp_full[b]);
          if (j == nkv - 1) { if (sm100::elect_one()) sm100::mma_commit(qt_empty); }  // last reads of Q / dO
          if (j > 0) issue_dq(gj - 1);
        }
        issue_dq(gj - 1);
      }
    }
  } else if (warp >= 4) {  // ---------------- elementwise: dS
    const int qw = warp & 3, hf = (warp - 4) >> 2;
    const int r = qw * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    const uint32_t stg = sm100::smem_addr(smem + C::OFF_OST) + (warp - 4) * 4096;  // epilogue staging (2 x 2 KB)
    int nbuf = 0;
    int gj = 0;
    // Q / dO of item ri into TMEM (the TS A operands): waits for the tile in shared memory and
    // for the previous item's last S / dP products to be done with the TMEM copies
    auto copy_qdo = [&](int ri_) {
      sm100::mbar_wait(q_full, ri_ & 1);
      sm100::mbar_wait(qt_empty, (ri_ & 1) ^ 1);
      tile_row_to_tmem<D>(smem + (hf == 0 ? C::OFF_Q : C::OFF_DO), r, (hf == 0 ? t_qt : t_dot) + lane_off);
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive_warp(at_full);
    };
    if (item_of(0) >= 0) copy_qdo(0);
    for (int ri = 0, it; (it = item_of(ri)) >= 0; ++ri) {
      int level, hd, bb;
      decode_item(it, a, per, level, hd, bb);
      const int qb = nqb - 1 - level, nkv = 2 * qb + 2;
      const int q = qb * 128 + r;
      const int64_t si = (static_cast<int64_t>(bb) * a + hd) * s + q;
      const float L2 = lse[si] * LOG2E, Dq = delta[si];
      for (int j = 0; j < nkv; ++j, ++gj) {
        const int b = gj & 1;
        if (warp == 4 && lane == 0 && j == 0) TRB(5, ri);
        sm100::mbar_wait(&sp_full[b], (gj >> 1) & 1);
        if (warp == 4 && lane == 0 && j == 0) TRB(6, ri);
        sm100::tc_fence_after();
        uint32_t sr[32], dr[32];
        const uint32_t tp = tbase + b * 128 + lane_off;
        sm100::tmem_ld32(tp + 32 * hf, sr);
        sm100::tmem_ld32(tp + 64 + 32 * hf, dr);
        sm100::tmem_ld_wait();
        uint32_t dk[16];
        const int klo = j * 64 + 32 * hf;
        auto elementwise = [&](auto masked, int c0) {
#pragma unroll
          for (int c = c0; c < c0 + 16; c += 2) {
            float dv[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float p = sm100::ex2(fmaf(__uint_as_float(sr[c + e]), scale_log2, -L2));
              if constexpr (decltype(masked)::value)
                if (klo + c + e > q) p = 0.f;
              dv[e] = p * (__uint_as_float(dr[c + e]) - Dq);
            }
            dk[c >> 1] = pack_bf16(dv[0], dv[1]);
          }
        };
        // keys of this half reach above the warp's first query only near the diagonal
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          if (klo + 31 > qb * 128 + qw * 32)
            elementwise(std::true_type{}, 16 * part);
          else
            elementwise(std::false_type{}, 16 * part);
          sm100::tmem_st8(tp + 32 * hf + 8 * part, dk + 8 * part);  // dS over this half's S columns
          if (part == 0) {
            sm100::tmem_st_wait();
            sm100::tc_fence_before();
            sm100::mbar_arrive_warp(&ds_part[b]);
          }
        }
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive_warp(&ds_full[b]);
      }
      if (warp == 4 && lane == 0) TRB(7, ri);
      // the next item's Q / dO copies before this item's epilogue: its first S / dP products then
      // run while the dQ stores are prepared
      if (item_of(ri + 1) >= 0) copy_qdo(ri + 1);
      sm100::mbar_wait(o_final, ri & 1);
      if (warp == 4 && lane == 0) TRB(8, ri);
      sm100::tc_fence_after();
      const int wr = bb * s + qb * 128 + qw * 32;  // the warp's first row of dqkv
#pragma unroll 1
      for (int c = hf; c < D / 32; c += 2) {
        uint32_t v[32];
        sm100::tmem_ld32(t_dq + lane_off + c * 32, v);
        sm100::tmem_ld_wait();
        store_chunk_tma(stg, nbuf, v, scale, &tmOut, hd * D + c * 32, wr, lane);
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive_warp(o_empty);  // dQ may be overwritten by the next item
      if (warp == 4 && lane == 0) TRB(9, ri);
    }
    if (lane == 0) sm100::bulk_wait<0>();  // epilogue stores complete before the CTA exits
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (threadIdx.x == 0)
    for (int i = 0; i < NBAR; ++i)
      if (i != 15) sm100::mbar_inval(bar + i);  // 15: unused
  __syncthreads();
}

// One persistent launch for both halves of the backward.  Items: the dK/dV items of every
// level, heaviest (level 0) first, then the dQ items likewise; CTA c of G takes the items
// r G + c (even rounds r) and r G + G-1-c (odd rounds) — its dK/dV items come first, then its
// dQ items, so a CTA switches body (barrier layout) at most once.  TMEM (512 columns) is
// allocated once for the CTA.
template <int D>
__global__ void __launch_bounds__(384, 1)
    k_bwd_tc(const __grid_constant__ CUtensorMap kv128, const __grid_constant__ CUtensorMap kv64,
             const __grid_constant__ CUtensorMap do64, const __grid_constant__ CUtensorMap do128,
             const __grid_constant__ CUtensorMap tmOut, const int32_t* __restrict__ table,
             const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv, int s, int a,
             int b, float scale, float scale_log2) {
#ifdef ZB_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 16384) {
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_cta_bwd[blockIdx.x][0] = sm;
    g_cta_bwd[blockIdx.x][1] = gtime_b();
  }
#endif
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    sm100::tma_prefetch(&kv128);
    sm100::tma_prefetch(&kv64);
    sm100::tma_prefetch(&do64);
    sm100::tma_prefetch(&do128);
    sm100::tma_prefetch(&tmOut);
  }
  if (warp == 2) sm100::tmem_alloc<512>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see launch() in common.cuh)
  pdl_wait();
  const uint32_t tbase = tslot;
  const int per = a * b;
  const int n_items = s / 128 * per;  // per half (dK/dV or dQ)
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  // this CTA's items from the host-built LPT table (bwd_item_table): table[c] .. table[c + 1]
  // index ids in table[G + 1 ..]; an id < n_items is a dK/dV item, else a dQ item (id - n_items)
  const int t_lo = __ldg(table + c), t_hi = __ldg(table + c + 1);
  (void)G;
  auto nth = [&](int r) {  // r-th item of this CTA (dK/dV items first), or -1
    return t_lo + r < t_hi ? __ldg(table + G + 1 + t_lo + r) : -1;
  };
  int r_q = 0;  // first round whose item is a dQ item
  while (nth(r_q) >= 0 && nth(r_q) < n_items) ++r_q;
  dkdv_run<D>(kv128, kv64, do64, tmOut, lse, delta, dqkv, s, a, per, scale, scale_log2, tbase,
              [&](int r) { return r < r_q ? nth(r) : -1; });
  dq_run<D>(kv128, kv64, do128, tmOut, lse, delta, dqkv, s, a, per, scale, scale_log2, tbase, [&](int r) {
    const int it = nth(r_q + r);
    return it >= 0 ? it - n_items : -1;
  });
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc<512>(tbase);
#ifdef ZB_ATTN_TRACE
  if (threadIdx.x == 64 && blockIdx.x < 16384) g_cta_bwd[blockIdx.x][2] = gtime_b();
#endif
}

}  // namespace attn_bwd_tc

// Static LPT assignment of the backward's items to the G persistent CTAs (cached per shape):
// cost of a dK/dV item of key block kb = its s/64 - 2 kb query steps + 1.5 (epilogue of two
// tiles), of a dQ item of query block qb = its 2 qb + 2 key steps + 1 — the per-item trace of
// the kernel (scripts/attn_bwd_item_trace.py) puts a step at ~1 us and the epilogues at
// ~1.3 / 0.6 us.  Items go heaviest first to the least-loaded CTA (ties: lowest index); each
// CTA then runs its dK/dV items before its dQ items, each group in id order.  The snake order
// this replaces left the busiest CTA 9.5% above the mean (scripts/attn_cta_trace.py).  Which
// CTA computes an item does not change its result (no cross-item accumulation).
static const int32_t* bwd_item_table(int s, int a, int b, int G) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, int32_t*> cache;
  std::lock_guard<std::mutex> lock(mu);
  int dev_id = 0;
  ZB_CUDA(cudaGetDevice(&dev_id));
  auto key = std::make_tuple(dev_id, s, a, b, G);  // per device: the table is device memory
  auto f = cache.find(key);
  if (f != cache.end()) return f->second;
  const int per = a * b, nqb = s / 128, n_items = nqb * per;
  std::vector<std::pair<double, int>> items;  // (cost, combined id)
  items.reserve(2 * n_items);
  for (int id = 0; id < n_items; ++id) {
    const int kb = id / per;                  // dK/dV: level = key block, heaviest first
    items.push_back({(s / 64 - 2 * kb) + 1.5, id});
  }
  for (int id = 0; id < n_items; ++id) {
    const int qb = nqb - 1 - id / per;        // dQ: level 0 = the last query block
    items.push_back({(2 * qb + 2) + 1.0, n_items + id});
  }
  std::stable_sort(items.begin(), items.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<double> load(G, 0.0);
  std::vector<std::vector<int>> mine(G);
  using E = std::pair<double, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;  // (load, cta): least load, lowest index
  for (int c = 0; c < G; ++c) heap.push({0.0, c});
  for (const auto& it : items) {
    E e = heap.top();
    heap.pop();
    mine[e.second].push_back(it.second);
    heap.push({e.first + it.first, e.second});
  }
  std::vector<int32_t> host(G + 1 + 2 * n_items);
  int pos = 0;
  for (int c = 0; c < G; ++c) {
    std::sort(mine[c].begin(), mine[c].end());  // dK/dV ids (< n_items) first, heaviest first
    host[c] = pos;
    for (int id : mine[c]) host[G + 1 + pos++] = id;
  }
  host[G] = pos;
  int32_t* dev = nullptr;
  ZB_CUDA(cudaMalloc(&dev, sizeof(int32_t) * host.size()));
  ZB_CUDA(cudaMemcpy(dev, host.data(), sizeof(int32_t) * host.size(), cudaMemcpyHostToDevice));
  cache[key] = dev;
  return dev;
}

template <int D>
static void bwd_tc_launch(const AttnShape& sh, const void* qkv, const void* dout, const float* lse, void* dqkv,
                          const float* delta, cudaStream_t st) {
  using C1 = attn_bwd_tc::DkdvCfg<D>;
  using C2 = attn_bwd_tc::DqCfg<D>;
  constexpr int SMEM = C1::SMEM > C2::SMEM ? C1::SMEM : C2::SMEM;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(attn_bwd_tc::k_bwd_tc<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  const int h = sh.a * D, rows = sh.b * sh.s;
  const CUtensorMap kv128 = make_tmap(qkv, 3 * h, rows, 3 * h, 64, 128);
  const CUtensorMap kv64 = make_tmap(qkv, 3 * h, rows, 3 * h, 64, 64);
  const CUtensorMap do64 = make_tmap(dout, h, rows, h, 64, 64);
  const CUtensorMap do128 = make_tmap(dout, h, rows, h, 64, 128);
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const int items = 2 * (sh.s / 128) * sh.a * sh.b;
  const int grid = items < num_sms() ? items : num_sms();  // persistent: one CTA per SM
  // dK / dV / dQ epilogue stores: box 32 rows x 32 columns (64 B), 64-byte swizzle
  const CUtensorMap out32 = make_tmap(dqkv, 3 * h, rows, 3 * h, 32, 32, false, 64);
  const int32_t* table = bwd_item_table(sh.s, sh.a, sh.b, grid);
  launch(PDL_ATTN, attn_bwd_tc::k_bwd_tc<D>, grid, 384, SMEM, st, kv128, kv64, do64, do128, out32, table, lse, delta,
         static_cast<bf16*>(dqkv), sh.s, sh.a, sh.b, scale, scale * attn_bwd_tc::LOG2E);
  ZB_LAUNCH_CHECK();
}

bool attention_bwd_tc(const AttnShape& sh, const void* qkv, const void* dout, const float* lse, void* dqkv,
                      const float* delta, cudaStream_t st) {
  if (sh.s % 128 != 0) return false;
  switch (sh.d) {
    case 64: bwd_tc_launch<64>(sh, qkv, dout, lse, dqkv, delta, st); return true;
    case 96: bwd_tc_launch<96>(sh, qkv, dout, lse, dqkv, delta, st); return true;
    case 128: bwd_tc_launch<128>(sh, qkv, dout, lse, dqkv, delta, st); return true;
  }
  return false;
}

}  // namespace zb

#ifdef ZB_ATTN_TRACE
extern "C" int zb_dbg_attn_bwd_item_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_bwd_tc::g_item_bwd, sizeof(unsigned long long) * 10 * 16));
}
extern "C" int zb_dbg_attn_bwd_cta_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_bwd_tc::g_cta_bwd, sizeof(unsigned long long) * 16384 * 3));
}
extern "C" int zb_dbg_attn_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_bwd_tc::g_trace, sizeof(unsigned long long) * 12 * 64));
}
#endif
