// tcgen05 / TMEM / TMA bf16 GEMM for the F, B and W contractions, plus the
// SIMT f32 GEMM of the parity mode.  See gemm.h for the operand conventions.
//
// bf16 kernel (one CTA per SM, persistent, warp-specialised):
//   warp 0     TMA producer: 128x64 A tile + BNx64 B tile per stage, 128B swizzle,
//              K-major boxes {64, rows} or MN-major boxes {64, 64}
//   warp 1     MMA issuer: tcgen05.mma.cta_group::1.kind::f16 128xBNx16, f32
//              accumulator in TMEM, double-buffered (2 x BN columns)
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld 32x32b.x32 -> fused epilogue -> global
// The smem ring (full/empty mbarriers) overlaps TMA with MMA; the TMEM ring
// (tfull/tempty) overlaps a tile's epilogue with the next tile's MMAs.
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <type_traits>

#include "gemm.h"
#include "ktimer.h"
#include "ops.h"
#include "sm100.cuh"

namespace zb {

// ------------------------------------------------------------------ epilogue
template <int EPI, typename TO>
__device__ __forceinline__ void epi8(const EpiArgs& e, int64_t row, int col, float* v) {
  if (EPI == EPI_F32_STORE || EPI == EPI_F32_ACC) {
    float* c = reinterpret_cast<float*>(e.C) + row * e.ldc + col;
    if (EPI == EPI_F32_ACC && e.beta) {
      float o[8];
      Vec8<float>::load(c, o);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += o[i];
    }
    Vec8<float>::store(c, v);
    return;
  }
  if (EPI != EPI_GELU_BWD && e.bias != nullptr) {
    float b[8];
    Vec8<float>::load(e.bias + col, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += b[i];
  }
  TO* c = reinterpret_cast<TO*>(e.C) + row * e.ldc + col;
  if (EPI == EPI_STORE) {
    Vec8<TO>::store(c, v);
  } else if (EPI == EPI_BIAS_GELU) {
    Vec8<TO>::store(c, v);
    float g[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = std::is_same<TO, bf16>::value ? gelu_fast(v[i]) : gelu_f(v[i]);
    Vec8<TO>::store(reinterpret_cast<TO*>(e.aux) + row * e.ldaux + col, g);
  } else if (EPI == EPI_RESID) {
    float r[8];
    Vec8<TO>::load(reinterpret_cast<const TO*>(e.aux) + row * e.ldaux + col, r);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += r[i];
    Vec8<TO>::store(c, v);
  } else if (EPI == EPI_GELU_BWD) {
    float u[8];
    Vec8<TO>::load(reinterpret_cast<const TO*>(e.aux) + row * e.ldaux + col, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] *= std::is_same<TO, bf16>::value ? gelu_grad_fast(u[i]) : gelu_grad_f(u[i]);
    Vec8<TO>::store(c, v);
  }
}

// ------------------------------------------------------------------ ordered split-K flags
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// order generic-proxy flag accesses with async-proxy (TMA) global writes
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05 kernel
namespace tc {
constexpr int BM = 128, BK = 64;
constexpr int kThreads = 384;     // warps 0-3: TMA, MMA, TMEM alloc, idle; warps 4-11: epilogue
constexpr int kEpiWarps = 8;     // 256 epilogue threads
constexpr int kStageBytes = 4096;  // epilogue staging per warp: a 32-row x 128-byte TMA box
constexpr int A_BYTES = BM * BK * 2;
template <int BN> struct Cfg {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : 6;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int EPI_OFF = STAGES * STAGE;
  static constexpr int BAR_OFF = EPI_OFF + kEpiWarps * kStageBytes;
  static constexpr int SMEM = BAR_OFF + 1024 /*align slack*/ + 256 /*barriers*/;
};

// output element type of an epilogue
template <int EPI> using OutT = typename std::conditional<(EPI == EPI_F32_ACC || EPI == EPI_F32_STORE), float, bf16>::type;

#ifdef ZB_GEMM_TRACE
// timeline of CTA 0 (leader of pair 0) of k_gemm_tc2, globaltimer ns (measurement build only):
// row 0 MMA warp has the accumulator (tempty), 1 last MMA of the tile issued, 2 epilogue warp 4
// has the accumulator (tfull), 3 epilogue warp 4 released it, 4 epilogue warp 11 released it
__device__ unsigned long long g_gtrace[8][64];
__device__ __forceinline__ void gtr(int row, int n) {
  if (blockIdx.x == 0 && n < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gtrace[row][n] = t;
  }
}
#define GTR(row, n) gtr(row, n)
#else
#define GTR(row, n)
#endif

// byte offset of 16-byte piece j of row `lane` in a 32 x 128 B box, TMA 128B-swizzle layout
__device__ __forceinline__ int swz(int lane, int j) { return lane * 128 + ((j ^ (lane & 7)) << 4); }

// TMA epilogue of one warp: 32 rows (the warp's TMEM lane quadrant) x ncols columns
// starting at global (row0, col0); taddr = TMEM address of the first column.  Per chunk
// of 128 B per row (64 bf16 / 32 f32 columns): tcgen05.ld, fused epilogue in f32,
// write the 32 x 128 B box into the warp's staging buffer in the 128B-swizzled layout,
// TMA-store it (coalesced, asynchronous, M / N tails clipped by the tensor map).  W's
// f32 accumulation (EPI_F32_ACC, beta) is a TMA reduce-add: the L2 adds the tile, nothing
// is read back into the SM.  RESID / GELU_BWD read their bf16 operand through the same
// staging buffer (TMA load on the warp's mbarrier), BIAS_GELU stores C then GeLU(C).
template <int EPI>
__device__ __forceinline__ void epilogue_chunks(const EpiArgs& ep, const CUtensorMap* tmC, const CUtensorMap* tmX,
                                                uint32_t taddr, uint8_t* buf, uint64_t* xbar, uint32_t& xph,
                                                int row0, int col0, int ncols, int N, int lane, bool reduce,
                                                bool pre = false, bool stream_out = false) {
  using TO = OutT<EPI>;
  constexpr int CC = 128 / static_cast<int>(sizeof(TO));
  constexpr bool kAuxIn = EPI == EPI_RESID || EPI == EPI_GELU_BWD;
  constexpr bool kBias = EPI == EPI_STORE || EPI == EPI_BIAS_GELU || EPI == EPI_RESID;
  // the epilogue's activation traffic streams through L2 once: evict it first so it does not
  // push the A / B operand tiles (re-read by other CTAs) out of L2.  W's f32 reduce-adds keep
  // the default policy (split-K re-touches the same gradient tile).
  const uint64_t pol = sm100::l2_evict_first();
#pragma unroll 1
  for (int ch = 0; ch < ncols / CC; ++ch) {
    const int col = col0 + ch * CC;
    if (lane == 0 && !(pre && ch == 0)) {  // pre: chunk 0's aux tile was requested by the caller
      sm100::bulk_wait_read<0>();  // the previous chunk's store has read the staging buffer
      if (kAuxIn) {
        sm100::mbar_arrive_expect_tx(xbar, kStageBytes);
        sm100::tma_load_2d_hint(buf, tmX, xbar, col, row0, pol);
      }
    }
    __syncwarp();
    uint32_t r[CC];
    sm100::tmem_ld32(taddr + ch * CC, r);
    if (CC == 64) sm100::tmem_ld32(taddr + ch * CC + 32, r + 32);
    sm100::tmem_ld_wait();
    float* v = reinterpret_cast<float*>(r);
    if (kBias && ep.bias != nullptr) {
#pragma unroll
      for (int g = 0; g < CC / 8; ++g) {
        if (col + 8 * g < N) {
          float b[8];
          Vec8<float>::load(ep.bias + col + 8 * g, b);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[8 * g + i] += b[i];
        }
      }
    }
    if (kAuxIn) {
      sm100::mbar_wait(xbar, xph);
      xph ^= 1;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4* p = reinterpret_cast<uint4*>(buf + swz(lane, j));
      if (sizeof(TO) == 4) {
        *p = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
      } else {
        float* x = v + 8 * j;
        if (kAuxIn) {
          float u[8];
          Vec8<bf16>::load(reinterpret_cast<const bf16*>(p), u);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = (EPI == EPI_RESID) ? x[i] + u[i] : x[i] * gelu_grad_fast(u[i]);
        }
        Vec8<bf16>::store(reinterpret_cast<bf16*>(p), x);
      }
    }
    sm100::fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if (EPI == EPI_F32_ACC && reduce && stream_out)
        sm100::tma_reduce_add_2d_hint(tmC, buf, col, row0, pol);
      else if (EPI == EPI_F32_ACC && reduce)
        sm100::tma_reduce_add_2d(tmC, buf, col, row0);
      else if (EPI == EPI_F32_ACC && stream_out)
        sm100::tma_store_2d_hint(tmC, buf, col, row0, pol);
      else if (EPI == EPI_F32_ACC)
        sm100::tma_store_2d(tmC, buf, col, row0);
      else
        sm100::tma_store_2d_hint(tmC, buf, col, row0, pol);
      sm100::bulk_commit();
    }
    if (EPI == EPI_BIAS_GELU) {  // second output: GeLU of the same f32 values
      if (lane == 0) sm100::bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float g[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) g[i] = gelu_fast(v[8 * j + i]);
        Vec8<bf16>::store(reinterpret_cast<bf16*>(buf + swz(lane, j)), g);
      }
      sm100::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        sm100::tma_store_2d_hint(tmX, buf, col, row0, pol);
        sm100::bulk_commit();
      }
    }
  }
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mt, int& nt) {
  constexpr int G = 8;  // group of 8 M-tiles swept across N for L2 reuse
  int per_group = G * num_n;
  int group = t / per_group;
  int first_m = group * G;
  int gm = min(num_m - first_m, G);
  int r = t % per_group;
  mt = first_m + r % gm;
  nt = r / gm;
}

template <int BN, bool A_MN, bool B_MN, int EPI, typename TO>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX, const EpiArgs ep,
              int M, int N, int K) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbar = tempty + 2;  // [kEpiWarps]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xbar + kEpiWarps);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      sm100::mbar_init(&full[i], 1);
      sm100::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], kEpiWarps);  // one arrival per epilogue warp
    }
    for (int i = 0; i < kEpiWarps; ++i) sm100::mbar_init(&xbar[i], 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    sm100::tma_prefetch(&tmC);
    sm100::tma_prefetch(&tmX);
  }
  if (warp == 2) sm100::tmem_alloc<C::TMEM_COLS>(tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see launch() in common.cuh)
  pdl_wait();
  const uint32_t tbase = *tslot;

  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n, nk = (K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mt, nt;
        tile_coords(t, num_m, num_n, mt, nt);
        const int m0 = mt * BM, n0 = nt * BN;
        for (int kb = 0; kb < nk; ++kb) {
          sm100::mbar_wait(&empty[stage], ph ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE);
          uint8_t* sa = smem + stage * C::STAGE;
          uint8_t* sb = sa + A_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            sm100::tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          } else {
            sm100::tma_load_2d(sa, &tmA, &full[stage], m0, k0);
            sm100::tma_load_2d(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!B_MN) {
            sm100::tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) sm100::tma_load_2d(sb + i * 8192, &tmB, &full[stage], n0 + 64 * i, k0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (whole warp, one elected lane issues)
      constexpr uint32_t idesc = sm100::idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        sm100::mbar_wait_warp(&tempty[acc], aph ^ 1);
        sm100::tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          sm100::mbar_wait_warp(&full[stage], ph);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_addr(smem + stage * C::STAGE);
          const uint32_t sb = sa + A_BYTES;
          const uint64_t ad0 = A_MN ? sm100::smem_desc(sa, 8192, 1024, sm100::kSwizzle128B)
                                    : sm100::smem_desc(sa, 16, 1024, sm100::kSwizzle128B);
          const uint64_t bd0 = B_MN ? sm100::smem_desc(sb, 8192, 1024, sm100::kSwizzle128B)
                                    : sm100::smem_desc(sb, 16, 1024, sm100::kSwizzle128B);
          if (sm100::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              sm100::mma_bf16_ss(d, sm100::desc_adv(ad0, A_MN ? kk * 2048 : kk * 32),
                                 sm100::desc_adv(bd0, B_MN ? kk * 2048 : kk * 32), idesc, (kb | kk) != 0 ? 1u : 0u);
            sm100::mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            ph ^= 1;
          }
        }
        if (sm100::elect_one()) sm100::mma_commit(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    // 8 epilogue warps: warp w reads TMEM lanes 32*(w%4).. (hardware lane quadrant) and
    // one half of the tile's columns, so two warps per SMSP hide each other's latency
    const int ew = (warp - 4) & 3, half = (warp - 4) >> 2;
    uint8_t* buf = smem + C::EPI_OFF + (warp - 4) * kStageBytes;
    uint32_t xph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int mt, nt;
      tile_coords(t, num_m, num_n, mt, nt);
      sm100::mbar_wait(&tfull[acc], aph);
      sm100::tc_fence_after();
      epilogue_chunks<EPI>(ep, &tmC, &tmX,
                           tbase + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + half * (BN / 2), buf,
                           &xbar[warp - 4], xph, mt * BM + ew * 32, nt * BN + half * (BN / 2), BN / 2, N, lane, ep.beta != 0);
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // stores complete before the CTA exits
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc<C::TMEM_COLS>(tbase);
}

// ------------------------------------------------------------------ tcgen05 kernel, CTA pair
// Two CTAs of a cluster (one TPC) compute a 256 x BN tile with tcgen05.mma.cta_group::2:
// CTA r holds rows [128r, 128r+128) of A and D and columns [r BN/2, (r+1) BN/2) of B,
// so each SM stages only half of the B tile (32 KB / stage at BN = 256, 6 stages) and
// L2 -> SM traffic per output element drops by a third versus the 1-CTA kernel.
// The leader (rank 0) issues every MMA; both CTAs' TMA transactions land on the
// leader's full barrier; the leader's commits multicast to both CTAs' barriers; both
// CTAs' epilogues release the accumulator on the leader's tempty barrier.
template <int BN> struct Cfg2 {
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 6 : 8;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int EPI_OFF = STAGES * STAGE;
  static constexpr int BAR_OFF = EPI_OFF + kEpiWarps * kStageBytes;
  static constexpr int CS_OFF = BAR_OFF + 512;  // column-sum combine buffer (16 x 8 floats)
  static constexpr int SMEM = BAR_OFF + 1024 + 512 + 512 + 16;  // + the column sums' last-arrival flag
};

// Column sums of the A operand (W's bias gradient, A = dY MN-major) by warps 2-3 of each
// CTA of the pair.  A stage holds the CTA's 128 M values x 64 K rows as two 64 x 64 boxes
// (box b = M [64b, 64b+64), row r = k, 128 B per row, 16-B chunk j of row r at
// r*128 + ((j ^ (r & 7)) << 4)).  Thread t (of 64) owns chunk c = t % 16 (8 M values) and
// the rows r = t/16 (mod 4): per quarter-warp the 8 lanes read 8 distinct chunks of one
// row (conflict-free).  The k-blocks of an M block are shared out over its num_n tiles
// (tile nt reads k-blocks kb = nt mod num_n), so every tile delays only ~1/num_n of its
// stages: for those the leader's MMA commit lands on mdone, the warps read the stage and
// release it to the producer (empty); the other stages go straight back.  Each tile writes
// its partial sums (zeros if it read nothing); the tile completing a 128-row block adds the
// block's (split, n-tile) partials in a fixed order (deterministic, no second launch).
__device__ __forceinline__ void colsum_stage(const uint8_t* sa, int t, float* acc) {
  const int c = t & 15, g = t >> 4;
  // shared-window address: a generic pointer after the alignment arithmetic would compile to LD.E
  const uint32_t base = sm100::smem_addr(sa) + (c >> 3) * 8192;
  const int j = c & 7;
#pragma unroll 4
  for (int r = g; r < 64; r += 4) {
    uint32_t w[4];
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "r"(base + r * 128 + ((j ^ (r & 7)) << 4)));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += __uint_as_float(w[i] << 16);
      acc[2 * i + 1] += __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}

// W-grouping: per-segment A / B tensor maps (segment s = k-blocks [s kbseg, (s+1) kbseg))
struct SegMaps {
  CUtensorMap a[kMaxSeg], b[kMaxSeg];
  int nseg, kbseg;
};

template <int BN, bool A_MN, bool B_MN, int EPI, typename TO, bool CS = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX, const EpiArgs ep,
               int M, int N, int K, const __grid_constant__ SegMaps sg) {
  static_assert(!CS || (A_MN && EPI == EPI_F32_ACC), "column sums: W's A operand only");
  using C = Cfg2<BN>;
  constexpr int BM2 = 2 * BM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbar = tempty + 2;  // [kEpiWarps]
  uint64_t* mdone = xbar + kEpiWarps;  // [STAGES] CS: MMAs of a stage the column sums read completed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mdone + C::STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      sm100::mbar_init(&full[i], 2);  // one arrival per CTA (+ both CTAs' TMA bytes)
      // one arrival: the MMA commit, or (CS, a stage the column sums read) the column-sum warps
      sm100::mbar_init(&empty[i], 1);
      sm100::mbar_init(&mdone[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], 2 * kEpiWarps);  // one arrival per epilogue warp of both CTAs
    }
    for (int i = 0; i < kEpiWarps; ++i) sm100::mbar_init(&xbar[i], 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
    sm100::tma_prefetch(&tmC);
    sm100::tma_prefetch(&tmX);
    for (int i = 0; i < sg.nseg; ++i) {
      sm100::tma_prefetch(&sg.a[i]);
      sm100::tma_prefetch(&sg.b[i]);
    }
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tslot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  pdl_trigger();  // after the TMEM allocation (see launch() in common.cuh)
  pdl_wait();
  const uint32_t tbase = *tslot;

  const int num_m = (M + BM2 - 1) / BM2, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n, nk = (K + BK - 1) / BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // work item t = split (t / tiles) of tile (t % tiles): every split-s item precedes every
  // split-(s+1) item, and each CTA pair walks its items in increasing t, so the ordered
  // split-K waits below cannot deadlock (all CTAs are resident: grid <= #SMs)
  const int splits = EPI == EPI_F32_ACC ? ep.splits : 1;
  const int items = tiles * splits;
  auto kb_begin = [&](int sp) { return static_cast<int>((static_cast<int64_t>(nk) * sp) / splits); };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t ph = 0;
      const uint64_t pol_ops = sm100::l2_evict_last();
      for (int t = cid; t < items; t += ncl) {
        int mt, nt;
        tile_coords(t % tiles, num_m, num_n, mt, nt);
        const int sp = t / tiles;
        const int m0 = mt * BM2 + static_cast<int>(rank) * BM, n0 = nt * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = kb_begin(sp); kb < kb_begin(sp + 1); ++kb) {
          sm100::mbar_wait(&empty[stage], ph ^ 1);
          const uint32_t fbar = sm100::map_to_cta(&full[stage], 0);
          if (leader)
            sm100::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE);
          else
            sm100::mbar_arrive_cluster(fbar);
          uint8_t* sa = smem + stage * C::STAGE;
          uint8_t* sb = sa + A_BYTES;
          int k0 = kb * BK;
          const CUtensorMap* mA = &tmA;
          const CUtensorMap* mB = &tmB;
          if (sg.nseg > 1) {  // W-grouping: the k-block's microbatch segment
            const int sgi = kb / sg.kbseg;
            mA = &sg.a[sgi];
            mB = &sg.b[sgi];
            k0 = (kb - sgi * sg.kbseg) * BK;
          }
          if (ep.cache_hints & 2) {  // operands re-read by other CTAs: keep them in L2
            if (!A_MN) {
              sm100::tma_load_2d_pair_hint(sa, mA, fbar, k0, m0, pol_ops);
            } else {
              sm100::tma_load_2d_pair_hint(sa, mA, fbar, m0, k0, pol_ops);
              sm100::tma_load_2d_pair_hint(sa + 8192, mA, fbar, m0 + 64, k0, pol_ops);
            }
            if (!B_MN) {
              sm100::tma_load_2d_pair_hint(sb, mB, fbar, k0, n0, pol_ops);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 128; ++i)
                sm100::tma_load_2d_pair_hint(sb + i * 8192, mB, fbar, n0 + 64 * i, k0, pol_ops);
            }
          } else {
            if (!A_MN) {
              sm100::tma_load_2d_pair(sa, mA, fbar, k0, m0);
            } else {
              sm100::tma_load_2d_pair(sa, mA, fbar, m0, k0);
              sm100::tma_load_2d_pair(sa + 8192, mA, fbar, m0 + 64, k0);
            }
            if (!B_MN) {
              sm100::tma_load_2d_pair(sb, mB, fbar, k0, n0);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 128; ++i) sm100::tma_load_2d_pair(sb + i * 8192, mB, fbar, n0 + 64 * i, k0);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ---------------- MMA issuer (leader only; whole warp, one elected lane issues)
      constexpr uint32_t idesc = sm100::idesc_bf16(BM2, BN, A_MN, B_MN);
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int t = cid; t < items; t += ncl) {
        sm100::mbar_wait_warp(&tempty[acc], aph ^ 1);
        if (lane == 0) GTR(0, (t - cid) / ncl);
        sm100::tc_fence_after();
        const uint32_t d = tbase + acc * BN;
        const int kb0 = kb_begin(t / tiles);
        int mt_, nt_;
        tile_coords(t % tiles, num_m, num_n, mt_, nt_);
        for (int kb = kb0; kb < kb_begin(t / tiles + 1); ++kb) {
          sm100::mbar_wait_warp(&full[stage], ph);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_addr(smem + stage * C::STAGE);
          const uint32_t sb = sa + A_BYTES;
          const uint64_t ad0 = A_MN ? sm100::smem_desc(sa, 8192, 1024, sm100::kSwizzle128B)
                                    : sm100::smem_desc(sa, 16, 1024, sm100::kSwizzle128B);
          const uint64_t bd0 = B_MN ? sm100::smem_desc(sb, 8192, 1024, sm100::kSwizzle128B)
                                    : sm100::smem_desc(sb, 16, 1024, sm100::kSwizzle128B);
          if (sm100::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              sm100::mma_bf16_ss_pair(d, sm100::desc_adv(ad0, A_MN ? kk * 2048 : kk * 32),
                                      sm100::desc_adv(bd0, B_MN ? kk * 2048 : kk * 32), idesc,
                                      (kb != kb0 || kk != 0) ? 1u : 0u);
            // CS: the stages whose column sums this tile forms (kb = nt mod num_n) go through the
            // column-sum warps, which release them to the producer; the others straight back
            sm100::mma_commit_pair(CS && kb % num_n == nt_ ? &mdone[stage] : &empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            ph ^= 1;
          }
        }
        if (lane == 0) GTR(1, (t - cid) / ncl);
        if (sm100::elect_one()) sm100::mma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else if (CS && (warp == 2 || warp == 3)) {  // ---------------- column sums of A (both CTAs)
    const int t = threadIdx.x - 64;
    const uint32_t xs = sm100::smem_addr(smem + C::CS_OFF);
    int stage = 0;
    uint32_t mph = 0;  // per-stage parity of mdone (a stage completes mdone phases only when read)
    for (int it = cid; it < items; it += ncl) {
      int mt, nt;
      tile_coords(it % tiles, num_m, num_n, mt, nt);
      const int sp = it / tiles;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int kb = kb_begin(sp); kb < kb_begin(sp + 1); ++kb) {
        if (kb % num_n == nt) {  // this tile's share of the M block's column sums
          sm100::mbar_wait(&mdone[stage], (mph >> stage) & 1u);
          mph ^= 1u << stage;
          colsum_stage(smem + stage * C::STAGE, t, acc);
          asm volatile("bar.sync 1, 64;" ::: "memory");  // both warps have read the stage
          if (t == 0) sm100::mbar_arrive(&empty[stage]);
        }
        if (++stage == C::STAGES) stage = 0;
      }
      // combine the four row groups: (g0 + g1) in warp 2, (g2 + g3) in warp 3, then the warps
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
      if (warp == 3 && lane < 16)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(xs + (lane * 8 + i) * 4), "f"(acc[i]) : "memory");
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (warp == 2 && lane < 16) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float o;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(xs + (lane * 8 + i) * 4) : "memory");
          acc[i] += o;
        }
        const int m = mt * BM2 + static_cast<int>(rank) * BM + (lane >> 3) * 64 + (lane & 7) * 8;
        float* dst = ep.bias_part + static_cast<int64_t>(sp * num_n + nt) * M;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (m + i < M) dst[m + i] = acc[i];
        __threadfence();  // the partial is visible before this tile's arrival is counted
      }
      // the tile whose partial completes its 128-row block (all splits x n-tiles arrived) sums
      // the block's partials in (split, n-tile) order — the order of the former separate
      // finalize kernel, so the bias gradient is bitwise the same whichever CTA finishes last
      uint32_t* last = reinterpret_cast<uint32_t*>(smem + C::CS_OFF + 512);
      asm volatile("bar.sync 1, 64;" ::: "memory");  // xbuf is reused by the next tile; partial written
      const int blk = mt * 2 + static_cast<int>(rank);
      const int parts = splits * num_n;
      if (t == 0) *last = atomicAdd(&ep.bias_tickets[blk], 1) == parts - 1 ? 1u : 0u;
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (*last) {
        __threadfence();
        const int mb = mt * BM2 + static_cast<int>(rank) * BM;
#pragma unroll
        for (int hrow = 0; hrow < 2; ++hrow) {
          const int m = mb + hrow * 64 + t;
          if (m < M) {
            float v = __ldcg(ep.bias_part + m);
            for (int q = 1; q < parts; ++q) v += __ldcg(ep.bias_part + static_cast<int64_t>(q) * M + m);
            ep.bias_out[m] = ep.beta ? ep.bias_out[m] + v : v;
          }
        }
        if (t == 0) ep.bias_tickets[blk] = 0;  // ready for the next launch on this stream
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs, own 128 rows)
    const int ew = (warp - 4) & 3, half = (warp - 4) >> 2;  // see the 1-CTA kernel
    const uint32_t te0 = sm100::map_to_cta(&tempty[0], 0), te1 = sm100::map_to_cta(&tempty[1], 0);
    uint8_t* buf = smem + C::EPI_OFF + (warp - 4) * kStageBytes;
    uint32_t xph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = cid; t < items; t += ncl) {
      int mt, nt;
      const int tile = t % tiles, sp = t / tiles;
      tile_coords(tile, num_m, num_n, mt, nt);
      int32_t* flag = ep.flags + tile * 16 + static_cast<int>(rank) * 8 + (warp - 4);
      if (sp > 0 && lane == 0) {  // split sp-1 of this region has landed in C
        while (ld_acquire(flag) < ep.flag_base + sp) {
        }
        fence_proxy_async_global();
      }
      __syncwarp();
      const int erow = mt * BM2 + static_cast<int>(rank) * BM + ew * 32, ecol = nt * BN + half * (BN / 2);
      constexpr bool kAuxIn = EPI == EPI_RESID || EPI == EPI_GELU_BWD;
      if (kAuxIn && lane == 0) {  // request chunk 0's aux tile while this tile's MMAs still run
        sm100::bulk_wait_read<0>();
        sm100::mbar_arrive_expect_tx(&xbar[warp - 4], kStageBytes);
        sm100::tma_load_2d_hint(buf, &tmX, &xbar[warp - 4], ecol, erow, sm100::l2_evict_first());
      }
      sm100::mbar_wait(&tfull[acc], aph);
      if (warp == 4 && lane == 0) GTR(2, (t - cid) / ncl);
      sm100::tc_fence_after();
      epilogue_chunks<EPI>(ep, &tmC, &tmX,
                           tbase + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + half * (BN / 2), buf,
                           &xbar[warp - 4], xph, erow, ecol, BN / 2, N, lane, ep.beta != 0 || sp > 0, kAuxIn,
                           EPI == EPI_F32_ACC && splits == 1 && (ep.cache_hints & 1));
      if (sp + 1 < splits && lane == 0) {  // publish: this region's reduce-adds are complete
        sm100::bulk_wait<0>();
        fence_proxy_async_global();
        st_release(flag, ep.flag_base + sp + 1);
      }
      sm100::tc_fence_before();
      __syncwarp();  // the warp's TMEM reads are complete (tmem_ld_wait + fence above): one remote arrival
      if (lane == 0) sm100::mbar_arrive_cluster(acc == 0 ? te0 : te1);
      if (lane == 0 && (warp == 4 || warp == 11)) GTR(warp == 4 ? 3 : 4, (t - cid) / ncl);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // stores complete before the CTA exits
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  if (warp == 2) sm100::tmem_dealloc_pair<C::TMEM_COLS>(tbase);
}
}  // namespace tc

// ------------------------------------------------------------------ SIMT f32 kernel
namespace simt {
constexpr int BT = 64, BKK = 16;
template <bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(64) k_gemm_f32(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                                                 int64_t ldb, const EpiArgs ep, int M, int N, int K) {
  pdl_wait();
  __shared__ float As[BKK][BT + 4];
  __shared__ float Bs[BKK][BT + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BT, n0 = blockIdx.x * BT;
  const int tr = tid / 8, tcol = tid % 8;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += BKK) {
    for (int e = tid; e < BT * BKK; e += 64) {
      int mm, kk;
      if (A_MN) { mm = e % BT; kk = e / BT; } else { kk = e % BKK; mm = e / BKK; }
      int gm = m0 + mm, gk = k0 + kk;
      float a = 0.f;
      if (gm < M && gk < K) a = A_MN ? A[static_cast<int64_t>(gk) * lda + gm] : A[static_cast<int64_t>(gm) * lda + gk];
      As[kk][mm] = a;
      int nn;
      if (B_MN) { nn = e % BT; kk = e / BT; } else { kk = e % BKK; nn = e / BKK; }
      int gn = n0 + nn;
      gk = k0 + kk;
      float b = 0.f;
      if (gn < N && gk < K) b = B_MN ? B[static_cast<int64_t>(gk) * ldb + gn] : B[static_cast<int64_t>(gn) * ldb + gk];
      Bs[kk][nn] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BKK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][tr * 8 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tcol * 8 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int col = n0 + tcol * 8;
  if (col >= N) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t row = m0 + tr * 8 + i;
    if (row < M) epi8<EPI, float>(ep, row, col, acc[i]);
  }
}
}  // namespace simt

// ------------------------------------------------------------------ host side
int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    ZB_CUDA(cudaGetDevice(&dev));
    ZB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D bf16 tensor map over a row-major [outer, inner] view with leading dim ld.
CUtensorMap make_tmap(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                      uint32_t box_outer, bool f32, int swizzle) {
  const uint64_t esz = f32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * esz) & 15))
    throw CudaError("gemm: operand must be 16-byte aligned with a 16-byte multiple row pitch");
  CUtensorMap tm;
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstride[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstride, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return tm;
}

// epilogue tensor maps: C (output, box 32 rows x 128 B) and X (the bf16 aux operand:
// GeLU output of BIAS_GELU, residual / pre-activation input of RESID / GELU_BWD)
template <int EPI>
static void epi_tmaps(const GemmArgs& g, CUtensorMap& tc_, CUtensorMap& tx) {
  constexpr bool f32 = EPI == EPI_F32_ACC || EPI == EPI_F32_STORE;
  tc_ = make_tmap(g.ep.C, g.N, g.M, g.ep.ldc, f32 ? 32 : 64, 32, f32);
  if (EPI == EPI_BIAS_GELU || EPI == EPI_RESID || EPI == EPI_GELU_BWD) {
    if (!g.ep.aux) throw CudaError("gemm: epilogue needs its aux operand");
    tx = make_tmap(g.ep.aux, g.N, g.M, g.ep.ldaux, 64, 32);
  } else {
    tx = tc_;
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static void launch_tc(const GemmArgs& g, cudaStream_t st) {
  using C = tc::Cfg<BN>;
  auto kern = tc::k_gemm_tc<BN, A_MN, B_MN, EPI, bf16>;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CUtensorMap ta = A_MN ? make_tmap(g.A, g.M, g.K, g.lda, 64, 64) : make_tmap(g.A, g.K, g.M, g.lda, 64, tc::BM);
  CUtensorMap tb = B_MN ? make_tmap(g.B, g.N, g.K, g.ldb, 64, 64) : make_tmap(g.B, g.K, g.N, g.ldb, 64, BN);
  const int tiles = static_cast<int>(ceil_div(g.M, tc::BM) * ceil_div(g.N, BN));
  const int grid = tiles < num_sms() ? tiles : num_sms();
  CUtensorMap tcm, txm;
  epi_tmaps<EPI>(g, tcm, txm);
  launch(PDL_GEMM, kern, grid, tc::kThreads, C::SMEM, st, ta, tb, tcm, txm, g.ep, g.M, g.N, g.K);
  ZB_LAUNCH_CHECK();
}

// Ordered split-K of the W contraction (EPI_F32_ACC, K = T tokens): W's M x N (weight
// shape) often gives few 256 x 256 tiles for 74 CTA pairs (proj 2304 x 2304: 81 tiles =
// 2 rounds at 55% occupancy).  Pick the split count S <= 4 (>= 16 k-blocks per split)
// minimising ceil(S tiles / pairs) / S x (1 + 0.15 (S - 1)), smallest S on ties.  The flag counters live in a
// per-stream device buffer (zeroed once) with a per-stream launch base, so concurrent
// streams (loopback stages) never share counters.
struct SplitFlags {
  int32_t* dev = nullptr;
  int32_t base = 0;
  float* part = nullptr;  // bias partial sums [splits * n-tiles, M] (column-sum W GEMMs)
  size_t part_cap = 0;
  int32_t* tick = nullptr;  // per-128-row-block arrival counters of the column sums
  int tick_cap = 0;
};
static std::mutex g_split_mu;
static std::map<cudaStream_t, SplitFlags> g_split_bufs;
static constexpr int kMaxFlagTiles = 4096;
static void split_k_plan(int tiles, int nk, int pairs, cudaStream_t st, EpiArgs& ep) {
  static int disabled = -1;
  if (disabled < 0) {
    const char* e = getenv("ZB_GEMM_NO_SPLITK");
    disabled = (e && e[0] == '1') ? 1 : 0;
  }
  ep.splits = 1;
  if (disabled || tiles > kMaxFlagTiles) return;
  int best = 1;
  double best_t = static_cast<double>(ceil_div(tiles, pairs));
  for (int sk = 2; sk <= 4 && nk / sk >= 16; ++sk) {
    // each extra split costs ~15% (measured on the 1.5B W shapes: 81 tiles -> S = 2 is
    // 1.52x S = 1 but S = 4 only 1.30x; 243 / 324 tiles: S = 1 within 2% of the best)
    const double t = static_cast<double>(ceil_div(static_cast<int64_t>(tiles) * sk, pairs)) / sk * (1.0 + 0.15 * (sk - 1));
    if (t < best_t - 1e-9) {
      best_t = t;
      best = sk;
    }
  }
  static int force = -1;  // ZB_GEMM_SPLITK=<S>: fixed split count (measurement only)
  if (force < 0) {
    const char* e = getenv("ZB_GEMM_SPLITK");
    force = e ? std::max(1, std::min(4, atoi(e))) : 0;
  }
  if (force) best = force;
  if (best == 1) return;
  std::lock_guard<std::mutex> lock(g_split_mu);
  SplitFlags& f = g_split_bufs[st];
  if (!f.dev) {
    ZB_CUDA(cudaMalloc(&f.dev, sizeof(int32_t) * 16 * kMaxFlagTiles));
    ZB_CUDA(cudaMemsetAsync(f.dev, 0, sizeof(int32_t) * 16 * kMaxFlagTiles, st));  // ordered on st
  }
  if (f.base > (1 << 30)) {  // counters would overflow: reset (ordered after earlier work on st)
    ZB_CUDA(cudaMemsetAsync(f.dev, 0, sizeof(int32_t) * 16 * kMaxFlagTiles, st));
    f.base = 0;
  }
  ep.splits = best;
  ep.flags = f.dev;
  ep.flag_base = f.base;
  f.base += best;
}

// start of a CUDA-graph capture on st (ZB_RUN_GRAPH): the ordered split-K counters restart
// from 0 inside the graph (a memset node), so every replay sees the flag bases it was captured
// with; eager launches after it continue above the captured bases
void gemm_graph_begin(cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_split_mu);
  SplitFlags& f = g_split_bufs[st];
  if (!f.dev) return;  // no split-K launch has run on st yet: the capture never allocates (eager first)
  ZB_CUDA(cudaMemsetAsync(f.dev, 0, sizeof(int32_t) * 16 * kMaxFlagTiles, st));
  f.base = 0;
}

// per-split bias partials of a column-sum W GEMM (stream-private, grown on demand; the
// previous user on the same stream has finished before the next GEMM reads / writes it)
static float* bias_partials(cudaStream_t st, size_t n, int32_t** tickets, int blocks) {
  std::lock_guard<std::mutex> lock(g_split_mu);
  SplitFlags& f = g_split_bufs[st];
  if (f.tick_cap < blocks) {
    if (f.tick) {
      ZB_CUDA(cudaStreamSynchronize(st));
      ZB_CUDA(cudaFree(f.tick));
    }
    ZB_CUDA(cudaMalloc(&f.tick, static_cast<size_t>(blocks) * sizeof(int32_t)));
    ZB_CUDA(cudaMemsetAsync(f.tick, 0, static_cast<size_t>(blocks) * sizeof(int32_t), st));  // kernels reset them
    f.tick_cap = blocks;
  }
  *tickets = f.tick;
  if (f.part_cap < n) {
    if (f.part) {
      ZB_CUDA(cudaStreamSynchronize(st));
      ZB_CUDA(cudaFree(f.part));
    }
    ZB_CUDA(cudaMalloc(&f.part, n * sizeof(float)));
    f.part_cap = n;
  }
  return f.part;
}

template <int BN, bool A_MN, bool B_MN, int EPI, bool CS = false>
static void launch_tc2(const GemmArgs& g, cudaStream_t st) {
  using C = tc::Cfg2<BN>;
  auto kern = tc::k_gemm_tc2<BN, A_MN, B_MN, EPI, bf16, CS>;
  static bool attr = false;
  if (!attr) {
    ZB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  tc::SegMaps sg{};
  sg.nseg = g.nseg > 1 ? g.nseg : 1;
  CUtensorMap ta, tb;
  if (sg.nseg > 1) {  // W-grouping: one map pair per microbatch segment (MN-major W operands)
    const int kseg = g.K / sg.nseg;
    sg.kbseg = kseg / tc::BK;
    for (int i = 0; i < sg.nseg; ++i) {
      sg.a[i] = make_tmap(g.A_seg[i], g.M, kseg, g.lda, 64, 64);
      sg.b[i] = make_tmap(g.B_seg[i], g.N, kseg, g.ldb, 64, 64);
    }
    ta = sg.a[0];
    tb = sg.b[0];
  } else {
    ta = A_MN ? make_tmap(g.A, g.M, g.K, g.lda, 64, 64) : make_tmap(g.A, g.K, g.M, g.lda, 64, tc::BM);
    tb = B_MN ? make_tmap(g.B, g.N, g.K, g.ldb, 64, 64) : make_tmap(g.B, g.K, g.N, g.ldb, 64, BN / 2);
  }
  const int tiles = static_cast<int>(ceil_div(g.M, 2 * tc::BM) * ceil_div(g.N, BN));
  const int pairs = num_sms() / 2;
  EpiArgs ep = g.ep;
  if (EPI == EPI_F32_ACC) split_k_plan(tiles, static_cast<int>(ceil_div(g.K, tc::BK)), pairs, st, ep);
  static const int chint = [] {  // ZB_GEMM_CHINT: L2 cache-hint bits (gemm.h EpiArgs::cache_hints)
    const char* e = getenv("ZB_GEMM_CHINT");
    return e ? atoi(e) : 0;
  }();
  ep.cache_hints = chint;
  const int items = tiles * ep.splits;
  const int grid = 2 * (items < pairs ? items : pairs);
  const int num_n = static_cast<int>(ceil_div(g.N, BN));
  if (CS)
    ep.bias_part = bias_partials(st, static_cast<size_t>(ep.splits) * num_n * g.M, &ep.bias_tickets,
                                 static_cast<int>(ceil_div(g.M, tc::BM)));
  CUtensorMap tcm, txm;
  epi_tmaps<EPI>(g, tcm, txm);
  launch(PDL_GEMM, kern, grid, tc::kThreads, C::SMEM, st, ta, tb, tcm, txm, ep, g.M, g.N, g.K, sg);
  ZB_LAUNCH_CHECK();
}

// 2-CTA tiles when the problem fills at least one 256 x 256 pair tile; env ZB_GEMM_1CTA=1 forces 1-CTA.
static bool use_pair(const GemmArgs& g) {
  static int force1 = -1;
  if (force1 < 0) {
    const char* e = getenv("ZB_GEMM_1CTA");
    force1 = (e && e[0] == '1') ? 1 : 0;
  }
  return !force1 && g.M >= 256 && g.N >= 256;
}

// returns true when the kernel also formed W's bias gradient (ep.bias_out)
template <int BN, bool A_MN, bool B_MN, int EPI>
static bool launch_any(const GemmArgs& g, cudaStream_t st) {
  constexpr bool kCS = A_MN && EPI == EPI_F32_ACC && BN == 256;
  if (BN == 256 && use_pair(g)) {
    if (kCS && g.ep.bias_out != nullptr) {
      launch_tc2<BN, A_MN, B_MN, EPI, kCS>(g, st);
      return true;
    }
    launch_tc2<BN, A_MN, B_MN, EPI>(g, st);
  } else {
    launch_tc<BN, A_MN, B_MN, EPI>(g, st);
  }
  return false;
}

template <int BN, bool A_MN, bool B_MN>
static bool dispatch_epi_tc(const GemmArgs& g, cudaStream_t st) {
  switch (g.epi) {
    case EPI_STORE: return launch_any<BN, A_MN, B_MN, EPI_STORE>(g, st);
    case EPI_BIAS_GELU: return launch_any<BN, A_MN, B_MN, EPI_BIAS_GELU>(g, st);
    case EPI_RESID: return launch_any<BN, A_MN, B_MN, EPI_RESID>(g, st);
    case EPI_GELU_BWD: return launch_any<BN, A_MN, B_MN, EPI_GELU_BWD>(g, st);
    case EPI_F32_ACC: return launch_any<BN, A_MN, B_MN, EPI_F32_ACC>(g, st);
    case EPI_F32_STORE: return launch_any<BN, A_MN, B_MN, EPI_F32_STORE>(g, st);
  }
  throw CudaError("gemm: bad epilogue");
}

template <int BN>
static bool dispatch_major_tc(const GemmArgs& g, cudaStream_t st) {
  if (!g.a_mn && !g.b_mn) return dispatch_epi_tc<BN, false, false>(g, st);
  if (!g.a_mn && g.b_mn) return dispatch_epi_tc<BN, false, true>(g, st);
  if (g.a_mn && g.b_mn) return dispatch_epi_tc<BN, true, true>(g, st);
  return dispatch_epi_tc<BN, true, false>(g, st);
}

template <bool A_MN, bool B_MN>
static void dispatch_epi_f32(const GemmArgs& g, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div(g.N, simt::BT)), static_cast<unsigned>(ceil_div(g.M, simt::BT)));
  const float* A = static_cast<const float*>(g.A);
  const float* B = static_cast<const float*>(g.B);
  switch (g.epi) {
#define ZB_F32_CASE(E) \
  case E: launch(PDL_GEMM, simt::k_gemm_f32<A_MN, B_MN, E>, grid, 64, 0, st, A, g.lda, B, g.ldb, g.ep, g.M, g.N, g.K); break;
    ZB_F32_CASE(EPI_STORE)
    ZB_F32_CASE(EPI_BIAS_GELU)
    ZB_F32_CASE(EPI_RESID)
    ZB_F32_CASE(EPI_GELU_BWD)
    ZB_F32_CASE(EPI_F32_ACC)
    ZB_F32_CASE(EPI_F32_STORE)
#undef ZB_F32_CASE
    default: throw CudaError("gemm: bad epilogue");
  }
  ZB_LAUNCH_CHECK();
}

void gemm(const GemmArgs& g, DType dt, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return;
  if (g.nseg > 1) {
    if (g.nseg > kMaxSeg || !g.a_mn || !g.b_mn || g.epi != EPI_F32_ACC || g.K % g.nseg || (g.K / g.nseg) % 64)
      throw CudaError("gemm: W-grouping needs the W contraction, <= 4 segments of a multiple of 64 tokens");
    // the 2-CTA tcgen05 kernel walks the segments inside one accumulation; elsewhere (f32 parity
    // mode, small 1-CTA shapes) the segments are accumulated one after the other
    if (dt == DT_F32 || g.N <= 128 || !use_pair(g)) {
      const int kseg = g.K / g.nseg;
      for (int i = 0; i < g.nseg; ++i) {
        GemmArgs s1 = g;
        s1.nseg = 1;
        s1.K = kseg;
        s1.A = g.A_seg[i];
        s1.B = g.B_seg[i];
        if (i > 0) s1.ep.beta = 1;
        gemm(s1, dt, st);
      }
      return;
    }
  }
  if (g.N % 8 != 0 || g.ep.ldc % 8 != 0) throw CudaError("gemm: N and ldc must be multiples of 8");
  if (g.ep.bias_out != nullptr && (g.epi != EPI_F32_ACC || !g.a_mn))
    throw CudaError("gemm: bias_out is W's bias gradient (EPI_F32_ACC, MN-major A)");
  const int cls = g.a_mn ? ktimer::GEMM_W : (g.b_mn ? ktimer::GEMM_B : ktimer::GEMM_F);
  const int tk = ktimer::start(cls, 2.0 * g.M * g.N * static_cast<double>(g.K), st);
  bool bias_done = false;
  if (dt == DT_F32) {
    if (!g.a_mn && !g.b_mn) dispatch_epi_f32<false, false>(g, st);
    else if (!g.a_mn && g.b_mn) dispatch_epi_f32<false, true>(g, st);
    else if (g.a_mn && g.b_mn) dispatch_epi_f32<true, true>(g, st);
    else dispatch_epi_f32<true, false>(g, st);
  } else if (g.N <= 128) {
    bias_done = dispatch_major_tc<128>(g, st);
  } else {
    bias_done = dispatch_major_tc<256>(g, st);
  }
  ktimer::stop(tk, st);
  // paths without the in-kernel column sums (f32 parity mode, 1-CTA tiles): separate kernel
  if (g.ep.bias_out != nullptr && !bias_done)
    bias_grad(dt, g.A, g.lda, g.ep.bias_out, g.K, g.M, g.ep.beta, st);
}

}  // namespace zb

#ifdef ZB_GEMM_TRACE
extern "C" int zb_dbg_gemm_trace(unsigned long long* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, zb::tc::g_gtrace, sizeof(unsigned long long) * 8 * 64));
}
#endif
