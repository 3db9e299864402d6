// Causal flash-attention FORWARD on tcgen05 (bf16, s % 128 == 0).
//
// Persistent CTAs (one per SM) over work items (pair of 128-query tiles, head, sequence),
// heaviest pairs first.
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
// per-item events of CTA 0 (persistent walk): row e, column = item index r of the CTA
//  0 MMA: first S issued   1 MMA: last PV issued   2/3 tile 0/1 softmax: S(0) ready
//  4/5 tile 0/1: last P stored   6/7 tile 0/1: O final seen   8/9 tile 0/1: O stored
__device__ unsigned long long g_item_fwd[10][16];
__device__ __forceinline__ void tri(int e, int r) {
  if (blockIdx.x == 0 && r < 16) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_item_fwd[e][r] = t;
  }
}
#define TRI(e, r) tri(e, r)
// every CTA: {smid, start, end} (globaltimer ns) — CTA durations and per-SM gaps
__device__ unsigned long long g_cta_fwd[8192][3];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#else
#define TRF(row, n)
#define TRI(e, r)
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
  static constexpr int OFF_OST = OFF_BAR + 1024;        // O epilogue staging: 8 softmax warps x 4 KB
  static constexpr int SMEM = OFF_OST + 8 * 4096 + 1024;
  static_assert((18 + 2 * (PQ - 1) + 3) * 8 <= 256, "barrier area");
};

// Persistent: one CTA per SM walks work items (pair of 128-query tiles {2t, 2t+1}, head,
// sequence), numbered heaviest pair first; CTA c takes items r G + c (even rounds r) and
// r G + G-1-c (odd rounds) of G = gridDim.x CTAs — a snake order that evens out the
// triangular per-pair work.  Across items the TMEM allocation, barriers and K/V rings stay
// live: the next item's Q is loaded as soon as the current item's last S product has read
// Q (q_empty), its first S products run while the softmax warps still write the current
// item's O (o_empty gates only the next item's first PV per tile), so the per-item
// prologue / epilogue of the former one-CTA-per-item grid (~6.6 us per CTA at the 6.2B
// shape, scripts/attn_cta_trace.py) overlaps compute.
// TMEM (512 columns): S_0 [0,128), S_1 [128,256), O_0 [256, 256+D), O_1 [384, 384+D);
// P_t (bf16 pairs) is written over the first 64 columns of S_t.
// MMA issue order per key block j:  PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) — the tensor core
// runs one tile's products while the other tile's softmax warps work.  S_t(j+1) overwrites the
// P_t(j) that PV_t(j), issued just before it, reads: tcgen05.mma of one thread execute in issue
// order.  The commit after S_t(j+1) also covers PV_t(j), so the softmax warps may rescale O_t
// as soon as they see S_t(j+1).
// Barrier parities come from running counters of the CTA (blocks per tile, items per tile,
// K/V ring position), not from the block index of the current item.
// One 32-column chunk of the calling warp's 32 O rows (v: this thread's row, f32, times inv) to
// global memory by a TMA tensor store (box 32 rows x 64 B, SWIZZLE_64B: 16-B piece k of row i
// at k ^ ((i >> 1) & 3)) from one of the warp's two 2 KB staging buffers (alternating with
// nbuf); the warp waits only for the store issued two chunks earlier to have read its buffer,
// the global writes drain while it moves on.  Lane 0 issues and owns the bulk groups.
__device__ __forceinline__ void store_o_chunk(uint32_t stg, int& nbuf, const uint32_t* v, float inv,
                                              const CUtensorMap* tm, int col, int row, int lane) {
  const uint32_t buf = stg + (nbuf & 1) * 2048;
  if (lane == 0) sm100::bulk_wait_read<1>();
  __syncwarp();
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[8 * g + 2 * e]) * inv,
                                                __uint_as_float(v[8 * g + 2 * e + 1]) * inv);
      w[e] = *reinterpret_cast<uint32_t*>(&b2);
    }
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4)),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
  sm100::fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    sm100::tma_store_2d_sa(tm, buf, col, row);
    sm100::bulk_commit();
  }
  ++nbuf;
}

template <int D>
__global__ void __launch_bounds__(384, 1) k_fwd_tc(const __grid_constant__ CUtensorMap tm,
                                                   const __grid_constant__ CUtensorMap tmO, bf16* __restrict__ o,
                                                   float* __restrict__ lse, int s, int a, int items,
                                                   float scale_log2) {
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
  uint64_t* o_empty = bar + 16;   // [2] per tile: the softmax warps have read O_t of their item
  uint64_t* p_part = bar + 18;    // [2][PQ - 1] per tile: P of keys [0, 32 (q + 1)) stored (PV may start)
  // per tile t: q_full[t] Q_t landed; q_empty[t] the item's last S_t product has read Q_t (tile 0's
  // buffer is refilled for the next item while tile 1 still runs its last block)
  uint64_t* q_empty0 = bar + 18 + 2 * (PQ - 1);
  uint64_t* q_full1 = q_empty0 + 1;
  uint64_t* q_empty1 = q_empty0 + 2;
  uint64_t* q_fulls[2] = {q_full, q_full1};
  uint64_t* q_empties[2] = {q_empty0, q_empty1};

#ifdef ZB_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 8192) {
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_cta_fwd[blockIdx.x][0] = sm;
    g_cta_fwd[blockIdx.x][1] = gtime();
  }
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / BQ;
  const int npair = (nqb + 1) / 2;
  const int per = items / npair;  // a * b
  const int h = a * D;
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  // r-th item of this CTA (snake order), or -1
  auto item_of = [&](int r) {
    const int it = r * G + ((r & 1) ? G - 1 - c : c);
    return it < items ? it : -1;
  };
  struct Item {
    int q0, hd, bb, nkv0, nkv1;
    bool two;
  };
  auto decode = [&](int it) {
    Item w;
    const int pr = npair - 1 - it / per;
    w.hd = it % per % a;
    w.bb = it % per / a;
    w.q0 = 2 * pr;
    w.two = w.q0 + 1 < nqb;
    w.nkv0 = w.q0 + 1;
    w.nkv1 = w.two ? w.q0 + 2 : 0;
    return w;
  };

  if (threadIdx.x == 0) {
    for (int t = 0; t < 2; ++t) {
      sm100::mbar_init(q_fulls[t], 1);
      sm100::mbar_init(q_empties[t], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&k_full[i], 1);
      sm100::mbar_init(&k_empty[i], 1);
      sm100::mbar_init(&v_full[i], 1);
      sm100::mbar_init(&v_empty[i], 1);
      sm100::mbar_init(&s_full[i], 1);
      sm100::mbar_init(&p_full[i], 4);  // one arrival per softmax warp
      sm100::mbar_init(&o_final[i], 1);
      sm100::mbar_init(&o_empty[i], 4);
      for (int q = 0; q < PQ - 1; ++q) sm100::mbar_init(&p_part[i * (PQ - 1) + q], 4);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm);
    sm100::tma_prefetch(&tmO);
  }
  if (warp == 2) sm100::tmem_alloc<512>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see launch() in common.cuh)
  pdl_wait();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA
      int kn = 0, vn = 0;  // K / V ring positions (continuous over items)
      int qn[2] = {0, 0};  // Q_t loads issued
      for (int r = 0, it; (it = item_of(r)) >= 0; ++r) {
        const Item w = decode(it);
        const int row0 = w.bb * s;
        const int nkv = w.two ? w.nkv1 : w.nkv0;
        auto load_q = [&](int t) {  // Q_t of this item once the previous item's last S_t has read it
          sm100::mbar_wait(q_empties[t], (qn[t] & 1) ^ 1);
          sm100::mbar_arrive_expect_tx(q_fulls[t], C::TILE);
          for (int at = 0; at < C::ATOMS; ++at)
            sm100::tma_load_2d(smem + C::OFF_Q + t * C::TILE + at * 16384, &tm, q_fulls[t], w.hd * D + 64 * at,
                               row0 + (w.q0 + t) * BQ);
          ++qn[t];
        };
        auto load_k = [&](int j) {
          const int st = kn & 1;
          sm100::mbar_wait(&k_empty[st], ((kn >> 1) & 1) ^ 1);
          sm100::mbar_arrive_expect_tx(&k_full[st], C::TILE);
          for (int at = 0; at < C::ATOMS; ++at)
            sm100::tma_load_2d(smem + C::OFF_K + st * C::TILE + at * 16384, &tm, &k_full[st],
                               h + w.hd * D + 64 * at, row0 + j * BKV);
          ++kn;
        };
        auto load_v = [&](int j) {
          const int st = vn & 1;
          sm100::mbar_wait(&v_empty[st], ((vn >> 1) & 1) ^ 1);
          sm100::mbar_arrive_expect_tx(&v_full[st], C::TILE);
          for (int at = 0; at < C::ATOMS; ++at)
            sm100::tma_load_2d(smem + C::OFF_V + st * C::TILE + at * 16384, &tm, &v_full[st],
                               2 * h + w.hd * D + 64 * at, row0 + j * BKV);
          ++vn;
        };
        // Q_0, K(0) first: the MMA warp issues this item's S_0(0) while the previous item's tile 1
        // still finishes its last block; Q_1 waits for that block's S_1
        load_q(0);
        load_k(0);
        if (w.two) load_q(1);
        for (int j = 0; j < nkv; ++j) {  // K runs one block ahead of V
          if (j + 1 < nkv) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA
      constexpr uint32_t idesc_s = sm100::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = sm100::idesc_bf16(128, D, false, true);
      const uint32_t sq = sm100::smem_addr(smem + C::OFF_Q);
      int kn = 0, vn = 0;              // K / V ring positions
      int pb[2] = {0, 0};              // PV blocks issued per tile (P barrier parity)
      int ti[2] = {0, 0};              // items started per tile (o_empty parity)
      int qm[2] = {0, 0};              // Q_t loads consumed (q_full parity)
      bool pre = false;                // this item's S_0(0) was issued in the previous item's tail
      int pre_left0 = 0;               // its remaining S_0 products after that
      for (int r = 0, it; (it = item_of(r)) >= 0; ++r) {
        const Item w = decode(it);
        const int nkv = w.two ? w.nkv1 : w.nkv0;
        // S_t products of the item still to issue; the last one commits q_empty[t]
        int s_left[2] = {pre ? pre_left0 : w.nkv0, w.nkv1};
        auto issue_s = [&](int t, int stage, int& left) {  // S_t = Q_t K^T (K in ring stage `stage`)
          const uint32_t sk = sm100::smem_addr(smem + C::OFF_K + stage * C::TILE);
          const uint64_t qd = sm100::smem_desc(sq + t * C::TILE, 16, 1024, sm100::kSwizzle128B);
          const uint64_t kd = sm100::smem_desc(sk, 16, 1024, sm100::kSwizzle128B);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            if (sm100::elect_one()) sm100::mma_bf16_ss(tbase + t * 128, sm100::desc_adv(qd, off), sm100::desc_adv(kd, off), idesc_s,
                               kk != 0 ? 1u : 0u);
          }
          if (sm100::elect_one()) sm100::mma_commit(&s_full[t]);
          if (--left == 0) { if (sm100::elect_one()) sm100::mma_commit(q_empties[t]); }
        };
        auto issue_pv = [&](int t, int j, int stage) {  // O_t += P_t V_j, the first keys as soon as their P is stored
          const uint32_t sv = sm100::smem_addr(smem + C::OFF_V + stage * C::TILE);
          const uint64_t vd = sm100::smem_desc(sv, 16384, 1024, sm100::kSwizzle128B);
          if (j == 0) {  // the softmax warps have read O_t of the tile's previous item
            sm100::mbar_wait_warp(&o_empty[t], (ti[t] & 1) ^ 1);
            ++ti[t];
          }
          const uint32_t par = pb[t] & 1;
#pragma unroll
          for (int q = 0; q < PQ; ++q) {
            constexpr int KQ = BKV / 16 / PQ;  // K-steps per published part of P
            sm100::mbar_wait_warp(q + 1 < PQ ? &p_part[t * (PQ - 1) + q] : &p_full[t], par);
            if (q + 1 == PQ && r == 0) TRF(t, j);
            sm100::tc_fence_after();
            if (sm100::elect_one()) {
#pragma unroll
              for (int kk = KQ * q; kk < KQ * q + KQ; ++kk)
                sm100::mma_bf16_ts(tbase + 256 + t * 128, tbase + t * 128 + kk * 8, sm100::desc_adv(vd, kk * 2048),
                                   idesc_o, (j | kk) != 0 ? 1u : 0u);
            }
            __syncwarp();
          }
          ++pb[t];
        };
        if (!pre) {
          sm100::mbar_wait_warp(q_fulls[0], qm[0] & 1);
          ++qm[0];
          sm100::mbar_wait_warp(&k_full[kn & 1], (kn >> 1) & 1);
          sm100::tc_fence_after();
          if (lane == 0) TRI(0, r);
          issue_s(0, kn & 1, s_left[0]);
        }
        pre = false;
        if (w.two) {
          sm100::mbar_wait_warp(q_fulls[1], qm[1] & 1);
          ++qm[1];
          sm100::tc_fence_after();
          issue_s(1, kn & 1, s_left[1]);
        }
        if (sm100::elect_one()) sm100::mma_commit(&k_empty[kn & 1]);  // after both S(0) products
        ++kn;
        for (int j = 0; j < nkv; ++j) {
          const bool more = j + 1 < nkv;
          const int vst = vn & 1;
          sm100::mbar_wait_warp(&v_full[vst], (vn >> 1) & 1);
          if (more) sm100::mbar_wait_warp(&k_full[kn & 1], (kn >> 1) & 1);
          sm100::tc_fence_after();
          if (j < w.nkv0) {
            issue_pv(0, j, vst);
            if (j == w.nkv0 - 1) { if (sm100::elect_one()) sm100::mma_commit(&o_final[0]); }
          }
          if (j + 1 < w.nkv0) issue_s(0, kn & 1, s_left[0]);
          if (j + 1 == nkv && lane == 0) TRI(1, r);
          if (j + 1 == nkv && w.two) {
            // item tail: tile 0 is done (PV_0 of its last block issued, so S_0's TMEM is free in
            // issue order) while tile 1's last softmax runs — issue the NEXT item's S_0(0) now, so
            // its tile-0 softmax overlaps this block instead of following it
            const int it2 = item_of(r + 1);
            if (it2 >= 0) {
              const Item w2 = decode(it2);
              sm100::mbar_wait_warp(q_fulls[0], qm[0] & 1);
              ++qm[0];
              sm100::mbar_wait_warp(&k_full[kn & 1], (kn >> 1) & 1);
              sm100::tc_fence_after();
              if (lane == 0) TRI(0, r + 1);
              pre_left0 = w2.nkv0;
              issue_s(0, kn & 1, pre_left0);
              pre = true;
            }
          }
          if (j < w.nkv1) {
            issue_pv(1, j, vst);
            if (j == w.nkv1 - 1) { if (sm100::elect_one()) sm100::mma_commit(&o_final[1]); }
          }
          if (sm100::elect_one()) sm100::mma_commit(&v_empty[vst]);
          ++vn;
          if (j + 1 < w.nkv1) issue_s(1, kn & 1, s_left[1]);
          if (more) {
            if (sm100::elect_one()) sm100::mma_commit(&k_empty[kn & 1]);
            ++kn;
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- softmax: 4 warps per tile, one row per thread
    const int t = (warp - 4) >> 2;
    const int r_ = (warp & 3) * 32 + lane;  // row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t t_s = tbase + t * 128 + lane_off, t_o = tbase + 256 + t * 128 + lane_off;
    const uint32_t stg = sm100::smem_addr(smem + C::OFF_OST) + (warp - 4) * 4096;  // O staging (2 x 2 KB)
    int nbuf = 0;
    int sb = 0;  // S blocks consumed by this tile (s_full / p barrier parity)
    int ni = 0;  // items finished by this tile (o_final parity)
    for (int rr = 0, it; (it = item_of(rr)) >= 0; ++rr) {
      const Item w = decode(it);
      const int nk = t == 0 ? w.nkv0 : w.nkv1;
      const int qt = w.q0 + t;
      float m = -INFINITY, l = 0.f;  // m: reference max (log2 units), l: running sum relative to m
      for (int j = 0; j < nk; ++j, ++sb) {
        sm100::mbar_wait(&s_full[t], sb & 1);
        if ((warp & 3) == 0 && lane == 0 && j == 0) TRI(2 + t, rr);
        if ((warp & 3) == 0 && lane == 0 && rr == 0) TRF(2 + 3 * t, j);
        sm100::tc_fence_after();
        float sv[128];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) sm100::tmem_ld32(t_s + c4 * 32, reinterpret_cast<uint32_t*>(sv + 32 * c4));
        sm100::tmem_ld_wait();
        if ((warp & 3) == 0 && lane == 0 && rr == 0) TRF(3 + 3 * t, j);
        if (j == qt) {
#pragma unroll
          for (int k = 0; k < 128; ++k)
            if (k > r_) sv[k] = -INFINITY;
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
            for (int c4 = 0; c4 < D / 32; ++c4) {
              uint32_t ov[32];
              sm100::tmem_ld32(t_o + c4 * 32, ov);
              sm100::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
              sm100::tmem_st32(t_o + c4 * 32, ov);
            }
            sm100::tmem_st_wait();
          }
        }
        if ((warp & 3) == 0 && lane == 0 && rr == 0) TRF(8 + t, j);
        const float mneg = -m;
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < PQ; ++q) {  // keys [KP q, KP q + KP) -> P columns [KP q / 2, KP (q + 1) / 2)
          constexpr int KP = BKV / PQ;
          uint32_t pk[KP / 2];
#pragma unroll
          for (int k = 0; k < KP; k += 2) {
            const float x0 = fmaf(sv[KP * q + k], scale_log2, mneg), x1 = fmaf(sv[KP * q + k + 1], scale_log2, mneg);
            float p0, p1;
            if ((k & 6) == 6 && kPolyExp && j != qt) {  // a quarter on the FMA pipe (measured slower: off)
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
        if ((warp & 3) == 0 && lane == 0 && rr == 0) TRF(10 + t, j);
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        if ((warp & 3) == 0 && lane == 0 && rr == 0) TRF(4 + 3 * t, j);
        sm100::mbar_arrive_warp(&p_full[t]);
        if ((warp & 3) == 0 && lane == 0 && j + 1 == nk) TRI(4 + t, rr);
      }
      if (nk > 0) {
        sm100::mbar_wait(&o_final[t], ni & 1);
        if ((warp & 3) == 0 && lane == 0) TRI(6 + t, rr);
        ++ni;
        sm100::tc_fence_after();
        const int q = qt * BQ + r_;
        const float inv = 1.f / l;
        // O rows leave by TMA tensor stores from warp-private staging (store_o_chunk): the warp
        // writes shared memory only, the global writes drain while it starts the next item
        // (row-per-thread 16-B stores touched 32 lines per instruction: ~2 us per tile,
        // profiles/r02_attn_fwd_item_trace_before.txt)
        const int wr = w.bb * s + qt * BQ + (warp & 3) * 32;  // the warp's first O row
#pragma unroll 1
        for (int c4 = 0; c4 < D / 32; ++c4) {
          uint32_t ov[32];
          sm100::tmem_ld32(t_o + c4 * 32, ov);
          sm100::tmem_ld_wait();
          store_o_chunk(stg, nbuf, ov, inv, &tmO, w.hd * D + c4 * 32, wr, lane);
        }
        sm100::tc_fence_before();
        sm100::mbar_arrive_warp(&o_empty[t]);  // O_t may be overwritten by the next item's PV
        if ((warp & 3) == 0 && lane == 0) TRI(8 + t, rr);
        lse[(static_cast<int64_t>(w.bb) * a + w.hd) * s + q] = (m + log2f(l)) * LN2;
      }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // O stores complete before the CTA exits
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc<512>(tbase);
#ifdef ZB_ATTN_TRACE
  if (threadIdx.x == 64 && blockIdx.x < 8192) g_cta_fwd[blockIdx.x][2] = gtime();
#endif
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
  const int items = (sh.s / attn_tc::BQ + 1) / 2 * sh.a * sh.b;
  const int grid = items < num_sms() ? items : num_sms();  // persistent: one CTA per SM
  const CUtensorMap tmO = make_tmap(o, h, sh.b * sh.s, h, 32, 32, false, 64);  // O stores: 32 x 32, 64-B swizzle
  launch(PDL_ATTN, attn_tc::k_fwd_tc<D>, grid, 384, C::SMEM, st, tm, tmO, static_cast<bf16*>(o), lse, sh.s, sh.a, items,
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
extern "C" int zb_dbg_attn_fwd_cta_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_tc::g_cta_fwd, sizeof(unsigned long long) * 8192 * 3));
}
extern "C" int zb_dbg_attn_fwd_item_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_tc::g_item_fwd, sizeof(unsigned long long) * 10 * 16));
}
extern "C" int zb_dbg_attn_fwd_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::attn_tc::g_trace_fwd, sizeof(unsigned long long) * 12 * 64));
}
#endif
