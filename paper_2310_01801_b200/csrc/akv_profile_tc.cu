// K1 on the 5th-generation tensor cores: tcgen05.mma + TMA + TMEM passes of
// the prompt profiler for bf16 Q/K/V with head dim 128 (akv_profile routes
// here; the SIMT passes in akv_profile.cu serve fp32 and other head dims).
//
// Pass 1 (query-major) — per (head, 128-query tile): S = Q_i K_j^T for key
//   tiles j <= i, 128x128x128 per tcgen05.mma group into a double-buffered
//   TMEM accumulator; the epilogue warps (one TMEM lane = one query row)
//   fold each tile into the row's online (max, sum) in the exp2 domain and
//   finally write lse_i (attention.py:64-89 normaliser).
// Pass 2 (key-major, recomputed) — per (head, 128-key tile): S^T = K_j Q_i^T
//   for query tiles i >= j, so a TMEM lane is a key and the column sums are
//   per-thread register reductions (no shuffles, no atomics):
//   colsum_j = sum_i exp(s_ij - lse_i) (engine.py:196), its square sum
//   (profiler.py:148-161 cosine), the prompt's last row A[N-1, :] and the
//   last-row output partial A[N-1, tile] @ V[tile] (engine.py:248,255).
// Warp roles per CTA (320 threads): warp 0 TMA producer, warp 1 TMEM owner
// and single-thread MMA issuer, warps 2-9 epilogue in kGroups = 2 column
// groups of 64 accumulator columns (a group's 4 warps cover the 128 TMEM
// lanes; the groups merge their per-row / per-key results at the end).
// Measured at config 4: 4 groups (16 epilogue warps per CTA, 56 registers)
// is slower (column pass 6.3 -> 7.8 ms).  The fixed operand (Q
// tile in pass 1, K tile in pass 2) is loaded once; the streamed operand
// goes through a 2-stage ring.  Grid blocks are ordered heaviest first.

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"
#include "akv_tc.cuh"

namespace akv {

constexpr int kTT = 128;                   // tile edge (queries / keys)
constexpr int kBoxB = 128 * 128;           // one 128-row x 64-col bf16 box (16 KB)
constexpr int kTileB = 2 * kBoxB;          // 128 x 128 bf16 tile (32 KB)
#ifndef AKV_K1_RING
#define AKV_K1_RING 2
#endif
#ifndef AKV_K1_CTAS_PER_SM
#define AKV_K1_CTAS_PER_SM 2
#endif
constexpr int kRing = AKV_K1_RING;         // streamed-operand stages
#ifndef AKV_K1_GROUPS
#define AKV_K1_GROUPS 2
#endif
constexpr int kGroups = AKV_K1_GROUPS;     // epilogue column groups (4 warps = 128 TMEM lanes each)
constexpr int kCols = 128 / kGroups;       // accumulator columns per epilogue thread and tile
constexpr int kEpiWarps = 4 * kGroups;
constexpr int kTcThreads = 64 + 32 * kEpiWarps;  // warp0 TMA, warp1 MMA/TMEM, then the epilogue
constexpr uint32_t kTmemCols = 256;        // two 128-column fp32 accumulators
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr size_t kTcSmem = 1024 + (size_t)(1 + kRing) * kTileB;

struct TcParams {
  int H, N;
  int64_t ld;
  const uint8_t* cls;
  int64_t cls_ld;
  const float* slope;
  const float* sink;
  const __nv_bfloat16* v;
  float* lse;
  double* colsum;
  double* colsq;
  float* lastp;
  float* out_part;  // [G, ntiles, 128]
  float scale;
};

using EpiSync = NamedSync<32 * kEpiWarps, 1, 64>;

// kCols consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
  if constexpr (kCols == 128) tmem_ld128(taddr, v);
  else if constexpr (kCols == 64) tmem_ld64(taddr, v);
  else tmem_ld32(taddr, v);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// issue the 8 K=16 steps of one 128x128x128 tile product
__device__ __forceinline__ void mma_tile(uint32_t tmem_d, const uint8_t* a_tile,
                                         const uint8_t* b_tile) {
  constexpr uint32_t idesc = umma_idesc_bf16(128, 128);
  const uint32_t a0 = smem_u32(a_tile), b0 = smem_u32(b_tile);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t off = (k >> 2) * kBoxB + (k & 3) * 32;
    umma_bf16_ss(tmem_d, umma_desc_sw128(a0 + off), umma_desc_sw128(b0 + off), idesc, k > 0);
  }
}

// online (max, sum) update of a row with kCols logits already in the log2
// domain (masked entries -inf)
__device__ __forceinline__ void row_update_scaled(const float* v, float& m, float& l) {
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < kCols; ++c) mx[c & 3] = fmaxf(mx[c & 3], v[c]);
  const float mn = fmaxf(fmaxf(m, fmaxf(mx[0], mx[1])), fmaxf(mx[2], mx[3]));
  if (mn == -INFINITY) return;
  float sm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    const float x = v[c] - mn;
    sm[c & 3] += exp2_mixed(x, c);
  }
  l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + ((sm[0] + sm[1]) + (sm[2] + sm[3]));
  m = mn;
}

// the same on raw accumulator values: the max is taken before scaling
// (scale > 0) and the scale folds into one FFMA per exponential
__device__ __forceinline__ void row_update_raw(const float* v, float sl2, float& m, float& l) {
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < kCols; ++c) mx[c & 3] = fmaxf(mx[c & 3], v[c]);
  const float mn = fmaxf(m, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2);
  // packed pairs: one FFMA2 and one FADD2 per two exponentials
  const uint64_t s2 = f2_pack(sl2, sl2), nb2 = f2_pack(-mn, -mn);
  uint64_t acc[2] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < kCols; c += 2) {
    const uint64_t x = f2_fma(f2_pack(v[c], v[c + 1]), s2, nb2);
    const bool poly = kPolyEvery > 0 && (c >> 1) % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1;
    acc[(c >> 1) & 1] = f2_add(acc[(c >> 1) & 1], poly ? f2_exp2_fma(x) : f2_exp2(x));
  }
  float a0, a1, a2, a3;
  f2_unpack(acc[0], a0, a1);
  f2_unpack(acc[1], a2, a3);
  l = (m == -INFINITY ? 0.f : l * fast_exp2(m - mn)) + ((a0 + a1) + (a2 + a3));
  m = mn;
}

// Work pairing: CTA (x, g) processes query tiles x and ntiles-1-x of head g
// (one when they coincide), so every CTA carries ntiles+1 key tiles of the
// triangle - uniform work, half the CTA setups.  TMEM, the barriers and the
// tensor-map prefetch serve both items, the second item's Q tile loads as
// soon as the first item's last MMA has read sQ, and all ring / accumulator
// phases run on per-CTA counters.
__global__ void __launch_bounds__(kTcThreads, AKV_K1_CTAS_PER_SM)
    k1tc_rowlse(const __grid_constant__ TcParams p, const __grid_constant__ CUtensorMap tmQ,
                const __grid_constant__ CUtensorMap tmK) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTileB;
  __shared__ __align__(8) uint64_t q_full, q_empty, k_full[kRing], k_empty[kRing], acc_full[2],
      acc_empty[2];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(16) float s_col[2][kTT];
  const int ntiles = (p.N + kTT - 1) / kTT;
  const int g = blockIdx.y, h = g % p.H, b = g / p.H;
  const int x = blockIdx.x;
  const int nitems = (ntiles - 1 - x == x) ? 1 : 2;
  // the column pass may launch now; it reads lse only after griddepcontrol.wait
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  auto item_qt = [&](int j) { return j == 0 ? ntiles - 1 - x : x; };  // heavier first
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    for (int s = 0; s < kRing; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&acc_full[a], 1); mbar_init(&acc_empty[a], kEpiWarps); }
    mbar_fence_init();
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
  }
  if (warp == 1) tmem_alloc(&s_tmem, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first(), pol_k = policy_evict_last();
      int t = 0;
      for (int j = 0; j < nitems; ++j) {
        const int qt = item_qt(j);
        const int rq = (int)((int64_t)g * p.ld + (int64_t)qt * kTT);
        mbar_wait(&q_empty, (j & 1) ^ 1);  // the previous item's MMAs have read sQ
        mbar_arrive_expect_tx(&q_full, kTileB);
        tma_load_2d(sQ, &tmQ, 0, rq, &q_full, pol_q);
        tma_load_2d(sQ + kBoxB, &tmQ, 64, rq, &q_full, pol_q);
        for (int kt = 0; kt <= qt; ++kt, ++t) {
          const int s = t % kRing;
          mbar_wait(&k_empty[s], ((t / kRing) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[s], kTileB);
          const int rk = (int)((int64_t)g * p.ld + (int64_t)kt * kTT);
          tma_load_2d(sK + s * kTileB, &tmK, 0, rk, &k_full[s], pol_k);
          tma_load_2d(sK + s * kTileB + kBoxB, &tmK, 64, rk, &k_full[s], pol_k);
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int t = 0;
      for (int j = 0; j < nitems; ++j) {
        const int qt = item_qt(j);
        mbar_wait(&q_full, j & 1);
        for (int kt = 0; kt <= qt; ++kt, ++t) {
          const int s = t % kRing, a = t & 1;
          mbar_wait(&k_full[s], (t / kRing) & 1);
          mbar_wait(&acc_empty[a], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          mma_tile(tmem + a * kTT, sQ, sK + s * kTileB);
          umma_commit(&k_empty[s]);
          umma_commit(&acc_full[a]);
        }
        umma_commit(&q_empty);
      }
    }
  } else {  // ---------------- epilogue (warps 2-9) ----------------
    __shared__ float s_ml[2][kGroups][kTT][2];
    const int quarter = warp & 3;
    const int et = threadIdx.x - 64;
    const int half = et >> 7;  // column group: accumulator columns [kCols*half, kCols*(half+1))
    const int rl = quarter * 32 + lane;
    const float sl2 = p.scale * kLog2e;
    const float slope_l2 = (p.slope ? p.slope[h] : 0.f) * kLog2e;
    const float sink_l2 = (p.sink ? p.sink[h] : 0.f) * kLog2e;
    const bool bias = slope_l2 != 0.f || sink_l2 != 0.f;
    const uint8_t* cls = p.cls + (size_t)b * p.cls_ld;
    int t = 0;
    for (int j = 0; j < nitems; ++j) {
      const int qt = item_qt(j);
      const int nk = qt + 1;
      const int row = qt * kTT + rl;
      // logits in the log2 domain without the row term -slope*row, which is
      // constant along a row and joins the lse at the end
      float m = -INFINITY, l = 0.f;
      uint8_t cnext = 0;
      if (bias && et < kTT) cnext = et < p.N ? cls[et] : 0;
      for (int kt = 0; kt < nk; ++kt, ++t) {
        const int a = t & 1;
        if (bias) {  // per-column bias of this key tile: sink on special keys + slope * col
          if (et < kTT) {
            const int col = kt * kTT + et;
            s_col[a][et] = (cnext == AKV_CLS_SPECIAL ? sink_l2 : 0.f) + slope_l2 * (float)col;
            const int nc = col + kTT;
            cnext = (kt + 1 < nk && nc < p.N) ? cls[nc] : 0;
          }
          EpiSync::sync();
        }
        mbar_wait(&acc_full[a], (t >> 1) & 1);
        tc_fence_after();
        float v[kCols];
        tmem_ld_cols(tmem + ((uint32_t)(quarter * 32) << 16) + a * kTT + half * kCols, v);
        // the values are in registers: hand the accumulator back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
        const bool masked = (kt == qt) || ((kt + 1) * kTT > p.N);
        const float* ct = &s_col[a][half * kCols];
        if (masked) {  // diagonal / ragged tile: causal and length masks
          const int c0 = kt * kTT + half * kCols;
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            float y = bias ? fmaf(v[c], sl2, ct[c]) : v[c] * sl2;
            if (c0 + c > row || c0 + c >= p.N) y = -INFINITY;
            v[c] = y;
          }
          row_update_scaled(v, m, l);
        } else if (bias) {
#pragma unroll
          for (int c = 0; c < kCols; c += 4) {
            const float4 tt = *reinterpret_cast<const float4*>(ct + c);
            v[c] = fmaf(v[c], sl2, tt.x);
            v[c + 1] = fmaf(v[c + 1], sl2, tt.y);
            v[c + 2] = fmaf(v[c + 2], sl2, tt.z);
            v[c + 3] = fmaf(v[c + 3], sl2, tt.w);
          }
          row_update_scaled(v, m, l);
        } else {
          row_update_raw(v, sl2, m, l);
        }
      }
      // merge the column groups of every row (double-buffered by item)
      float(*ml)[kTT][2] = s_ml[j & 1];
      ml[half][rl][0] = m;
      ml[half][rl][1] = l;
      EpiSync::sync();
      if (half == 0) {
        float mm = -INFINITY;
#pragma unroll
        for (int gq = 0; gq < kGroups; ++gq) mm = fmaxf(mm, ml[gq][rl][0]);
        float ll = 0.f;
#pragma unroll
        for (int gq = 0; gq < kGroups; ++gq) {
          const float m2 = ml[gq][rl][0];
          if (m2 != -INFINITY) ll += ml[gq][rl][1] * fast_exp2(m2 - mm);
        }
        const float rowterm = -slope_l2 * (float)row;
        if (row < p.N) p.lse[(size_t)g * p.N + row] = (mm + rowterm + __log2f(ll)) * kLn2;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Pass 2, paired like pass 1: CTA (x, g) processes key tiles x and
// ntiles-1-x of head g (one when they coincide), ntiles+1 query tiles in
// all - uniform work per CTA, half the CTA setups (TMEM allocation,
// barriers, descriptor prefetch, first TMA round trip).  The first item
// (key tile x, ntiles-x query tiles) is the heavier one.
constexpr size_t kTcSmemCol = kTcSmem + (size_t)(32 * kEpiWarps / 16) * 128 * 4;  // + out_part scratch

__global__ void __launch_bounds__(kTcThreads, AKV_K1_CTAS_PER_SM)
    k1tc_colsum(const __grid_constant__ TcParams p, const __grid_constant__ CUtensorMap tmQ,
                const __grid_constant__ CUtensorMap tmK) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sQ = smem + kTileB;
  float* s_red = reinterpret_cast<float*>(smem + (1 + kRing) * kTileB);  // [RG][128]
  __shared__ __align__(8) uint64_t k_full, k_empty, q_full[kRing], q_empty[kRing], acc_full[2],
      acc_empty[2];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(16) float s_col[2][kTT];
  __shared__ float s_lastp[kTT];
  const int ntiles = (p.N + kTT - 1) / kTT;
  const int g = blockIdx.y, h = g % p.H, b = g / p.H;
  const int x = blockIdx.x;
  const int nitems = (ntiles - 1 - x == x) ? 1 : 2;
  auto item_kt = [&](int j) { return j == 0 ? x : ntiles - 1 - x; };  // heavier first
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&k_full, 1);
    mbar_init(&k_empty, 1);
    for (int s = 0; s < kRing; ++s) { mbar_init(&q_full[s], 1); mbar_init(&q_empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&acc_full[a], 1); mbar_init(&acc_empty[a], kEpiWarps); }
    mbar_fence_init();
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
  }
  if (warp == 1) tmem_alloc(&s_tmem, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_k = policy_evict_first(), pol_q = policy_evict_last();
      int t = 0;
      for (int j = 0; j < nitems; ++j) {
        const int kt = item_kt(j), nq = ntiles - kt;
        const int rk = (int)((int64_t)g * p.ld + (int64_t)kt * kTT);
        // the key tile's V rows, read by the epilogue's last-row partial at
        // the item's end: into L2 now
        bulk_prefetch_l2(p.v + ((size_t)g * p.ld + (size_t)kt * kTT) * 128,
                         (uint32_t)min(kTT, p.N - kt * kTT) * 256u);
        mbar_wait(&k_empty, (j & 1) ^ 1);  // the previous item's MMAs have read sK
        mbar_arrive_expect_tx(&k_full, kTileB);
        tma_load_2d(sK, &tmK, 0, rk, &k_full, pol_k);
        tma_load_2d(sK + kBoxB, &tmK, 64, rk, &k_full, pol_k);
        for (int i = 0; i < nq; ++i, ++t) {
          const int s = t % kRing;
          mbar_wait(&q_empty[s], ((t / kRing) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[s], kTileB);
          const int rq = (int)((int64_t)g * p.ld + (int64_t)(kt + i) * kTT);
          tma_load_2d(sQ + s * kTileB, &tmQ, 0, rq, &q_full[s], pol_q);
          tma_load_2d(sQ + s * kTileB + kBoxB, &tmQ, 64, rq, &q_full[s], pol_q);
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int t = 0;
      for (int j = 0; j < nitems; ++j) {
        const int nq = ntiles - item_kt(j);
        mbar_wait(&k_full, j & 1);
        for (int i = 0; i < nq; ++i, ++t) {
          const int s = t % kRing, a = t & 1;
          mbar_wait(&q_full[s], (t / kRing) & 1);
          mbar_wait(&acc_empty[a], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          mma_tile(tmem + a * kTT, sK, sQ + s * kTileB);  // S^T: keys on TMEM lanes
          umma_commit(&q_empty[s]);
          umma_commit(&acc_full[a]);
        }
        umma_commit(&k_empty);
      }
    }
  } else {  // ---------------- epilogue (warps 2-9) ----------------
    __shared__ double s_part[2][kGroups][kTT];
    __shared__ float s_plast[kGroups][kTT];
    const int quarter = warp & 3;
    const int et = threadIdx.x - 64;
    const int half = et >> 7;  // column group: query columns [kCols*half, kCols*(half+1)) of a tile
    const int kl = quarter * 32 + lane;
    const float sl2 = p.scale * kLog2e;
    const float slope_l2 = (p.slope ? p.slope[h] : 0.f) * kLog2e;
    const float sink_l2 = (p.sink ? p.sink[h] : 0.f) * kLog2e;
    const uint8_t* cls = p.cls + (size_t)b * p.cls_ld;
    const float* lse = p.lse + (size_t)g * p.N;
    const bool slope_on = slope_l2 != 0.f;
    const int qlast = p.N - 1;
    // the row pass (programmatic predecessor) must be complete before lse is
    // read; the producer and MMA warps run ahead meanwhile
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int t = 0;
    for (int j = 0; j < nitems; ++j) {
      const int kt = item_kt(j), nq = ntiles - kt;
      const int key = kt * kTT + kl;
      // per-key term: sink on a special key, + slope * key.  Without a slope
      // the key term is a constant factor of the key's column and is applied
      // to the tile sums (kfac) instead of inside every exponential.
      const float ksink = key < p.N && cls[key] == AKV_CLS_SPECIAL ? sink_l2 : 0.f;
      const float kterm = ksink + slope_l2 * (float)key;
      const float kfac = fast_exp2(ksink);
      double dsum = 0.0, dsq = 0.0;
      float lastp = 0.f;
      float lnext = 0.f;
      if (et < kTT) lnext = kt * kTT + et < p.N ? lse[kt * kTT + et] : 0.f;
      for (int i = 0; i < nq; ++i, ++t) {
        const int a = t & 1;
        const int qt = kt + i;
        if (et < kTT) {  // per-query term of this tile: -lse_q * log2e - slope * q
          const int q = qt * kTT + et;
          s_col[a][et] = -lnext * kLog2e - slope_l2 * (float)q;
          const int qn = q + kTT;
          lnext = (i + 1 < nq && qn < p.N) ? lse[qn] : 0.f;
        }
        EpiSync::sync();
        mbar_wait(&acc_full[a], (t >> 1) & 1);
        tc_fence_after();
        float v[kCols];
        tmem_ld_cols(tmem + ((uint32_t)(quarter * 32) << 16) + a * kTT + half * kCols, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
        // diagonal tile (causal mask), ragged tail (q >= N) and the tile holding row N-1
        const bool masked = (i == 0) || ((qt + 1) * kTT > p.N) || (qt == qlast / kTT);
        const float* ct = &s_col[a][half * kCols];
        float ts[4] = {0.f, 0.f, 0.f, 0.f}, tq[4] = {0.f, 0.f, 0.f, 0.f};
        if (masked) {
          const int q0 = qt * kTT + half * kCols;
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            float pr = fast_exp2(fmaf(v[c], sl2, kterm + ct[c]));
            const int q = q0 + c;
            if (q < key || q >= p.N) pr = 0.f;
            if (q == qlast) lastp = pr;
            ts[c & 3] += pr;
            tq[c & 3] = fmaf(pr, pr, tq[c & 3]);
          }
          dsum += (double)((ts[0] + ts[1]) + (ts[2] + ts[3]));
          dsq += (double)((tq[0] + tq[1]) + (tq[2] + tq[3]));
        } else if (slope_on) {
#pragma unroll
          for (int c = 0; c < kCols; c += 4) {
            const float4 tt4 = *reinterpret_cast<const float4*>(ct + c);
            const float tt[4] = {tt4.x, tt4.y, tt4.z, tt4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float xx = fmaf(v[c + u], sl2, kterm + tt[u]);
              const float pr = exp2_mixed(xx, u);
              ts[u] += pr;
              tq[u] = fmaf(pr, pr, tq[u]);
            }
          }
          dsum += (double)((ts[0] + ts[1]) + (ts[2] + ts[3]));
          dsq += (double)((tq[0] + tq[1]) + (tq[2] + tq[3]));
        } else {
          // packed pairs: FFMA2 for the logits, FADD2 / FFMA2 for the two sums
          const uint64_t s2x = f2_pack(sl2, sl2);
          uint64_t as = f2_pack(0.f, 0.f), aq = f2_pack(0.f, 0.f);
          uint64_t bs = f2_pack(0.f, 0.f), bq = f2_pack(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < kCols; c += 4) {
            const float4 tt4 = *reinterpret_cast<const float4*>(ct + c);
            const uint64_t p0 = f2_exp2(f2_fma(f2_pack(v[c], v[c + 1]), s2x, f2_pack(tt4.x, tt4.y)));
            const uint64_t x1 = f2_fma(f2_pack(v[c + 2], v[c + 3]), s2x, f2_pack(tt4.z, tt4.w));
            // all on MUFU: a quarter on the FMA pipe measured 1.6 % slower here
            // (config 4), while it gains 5 % in the row pass
            const uint64_t p1 = f2_exp2(x1);
            as = f2_add(as, p0);
            aq = f2_fma(p0, p0, aq);
            bs = f2_add(bs, p1);
            bq = f2_fma(p1, p1, bq);
          }
          float x0, x1, x2, x3, y0, y1, y2, y3;
          f2_unpack(as, x0, x1);
          f2_unpack(bs, x2, x3);
          f2_unpack(aq, y0, y1);
          f2_unpack(bq, y2, y3);
          const float s1 = (x0 + x1) + (x2 + x3);
          const float s2 = (y0 + y1) + (y2 + y3);
          dsum += (double)(s1 * kfac);
          dsq += (double)(s2 * (kfac * kfac));
        }
      }
      // the last query row lies in the last (masked) tile; merge the groups
      if (half > 0) { s_part[0][half][kl] = dsum; s_part[1][half][kl] = dsq; s_plast[half][kl] = lastp; }
      EpiSync::sync();
      if (half == 0) {
#pragma unroll
        for (int gq = 1; gq < kGroups; ++gq) {
          dsum += s_part[0][gq][kl];
          dsq += s_part[1][gq][kl];
          lastp += s_plast[gq][kl];
        }
        if (key >= p.N) lastp = 0.f;
        if (key < p.N) {
          p.colsum[(size_t)g * p.N + key] = dsum;
          p.colsq[(size_t)g * p.N + key] = dsq;
          p.lastp[(size_t)g * p.N + key] = lastp;
        }
        s_lastp[kl] = lastp;
      }
      EpiSync::sync();
      {
        // last-row output partial of this key tile, sum_j lastp_j V_j, by all
        // epilogue threads: 16-byte loads of 8 dims, every load in flight at
        // once (a per-dimension loop here was a chain of ~30 L2/DRAM round
        // trips at the end of every CTA); partials meet in s_red
        constexpr int RG = 32 * kEpiWarps / 16;  // row groups (16 threads cover a 128-dim row)
        static_assert(kTT % RG == 0, "row groups tile the key tile");
        const __nv_bfloat16* vt = p.v + ((size_t)g * p.ld + (size_t)kt * kTT) * 128;
        const int nrow = min(kTT, p.N - kt * kTT);
        const int c = et & 15, r0 = et >> 4;
        uint4 raw[kTT / RG];
#pragma unroll
        for (int k = 0; k < kTT / RG; ++k) {
          const int jr = r0 + RG * k;
          raw[k] = jr < nrow ? ld_nc_v4(vt + (size_t)jr * 128 + c * 8) : make_uint4(0u, 0u, 0u, 0u);
        }
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < kTT / RG; ++k) {
          const int jr = r0 + RG * k;
          const float w = jr < nrow ? s_lastp[jr] : 0.f;
          float f[8];
          Elem<__nv_bfloat16>::unpack(raw[k], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaf(w, f[e], acc[e]);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) s_red[r0 * 128 + c * 8 + e] = acc[e];
        EpiSync::sync();
        if (half == 0) {
          float o = 0.f;
#pragma unroll
          for (int r = 0; r < RG; ++r) o += s_red[r * 128 + et];
          p.out_part[((size_t)g * ntiles + kt) * 128 + et] = o;
        }
        EpiSync::sync();  // s_red / s_lastp / s_part are reused by the next item
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

bool tc_profile_supported(int N) { return !g_disable_tc && N >= 1; }

int tc_tiles(int N) { return (N + kTT - 1) / kTT; }

cudaError_t launch_tc_passes(const void* q, const void* k, const void* v, int B, int H, int N,
                             int64_t ld, const uint8_t* cls, int64_t cls_ld, const float* slope,
                             const float* sink, float* lse, double* colsum, double* colsq,
                             float* lastp, float* out_part, cudaStream_t st) {
  const int G = B * H;
  const uint64_t rows = (uint64_t)G * (uint64_t)ld;
  if (rows >= (1ull << 31)) return cudaErrorInvalidValue;
  CUtensorMap tmQ, tmK;
  if (!encode_tmap_2d_bf16(&tmQ, q, rows, 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_2d_bf16(&tmK, k, rows, 128, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static PerDeviceOnce attr;
  cudaError_t e = attr.run([](int) {
    cudaError_t r = cudaFuncSetAttribute(k1tc_rowlse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTcSmem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(k1tc_colsum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmemCol);
    return r;
  });
  if (e != cudaSuccess) return e;
  TcParams p{H, N, ld, cls, cls_ld, slope, sink, static_cast<const __nv_bfloat16*>(v), lse, colsum,
             colsq, lastp, out_part, (float)(1.0 / sqrt(128.0))};
  const dim3 pairs((tc_tiles(N) + 1) / 2, G);  // tiles x and ntiles-1-x share a CTA
  k1tc_rowlse<<<pairs, kTcThreads, kTcSmem, st>>>(p, tmQ, tmK);
  if ((e = cudaGetLastError())) return e;
  {  // programmatic dependent launch: setup, K/Q loads and the first MMAs
     // overlap the row pass's tail
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = pairs;  // key tiles x and ntiles-1-x share a CTA
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = kTcSmemCol;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if ((e = cudaLaunchKernelEx(&cfg, k1tc_colsum, p, tmQ, tmK))) return e;
  }
  return cudaGetLastError();
}

}  // namespace akv
