// K3: one decode step over the ragged compressed cache, with fused insert
// and evict (sm_100a).
//
// Replaces the reference's generate_step per-head body (engine.py:303-350):
//   append k/v of the new token (engine.py:315-317)
//   attend over the live rows + the new row (engine.py:93-97, softmax over L+1)
//   FREQUENT heads: score[live] += p[:-1], score[new] = 0
//                   (policies.py:332-360, engine.py:320-330)
//   re-apply the frozen policy over candidates = live + new with
//   current_len = pos+1 (policies.py:214-267, engine.py:332-338)
//   drop the rows it no longer keeps (evicted rows never return).
//
// Layout: head g owns arena slots [seg_off[g], seg_off[g]+seg_cap[g]);
// slots [0, live) hold live rows (any order): d elements of K (kc) and V
// (vc), meta = position | class<<24 | inF<<30, score = float64 cumulative
// attention (FREQUENT heads).
//
// Kernel structure (one launch per step for all heads): a persistent grid
// of 2 CTAs per SM.  The step's work is cut into 16 KB "pages" of K and V
// (64 slots of bf16 d=128); every CTA computes the per-head page counts
// from live_in and takes one contiguous, equal share of the flattened page
// list.  The last warp is the producer: one elected lane streams each
// page's K rows, V rows, slot metadata and the head's q (plus the new
// token's k/v for the page holding slot `live`) into a 2-stage shared
// memory ring (TMA, mbarrier transaction counts; 3 stages for the SIMT
// variant and as a tuning option).  The other warps consume:
// logits with the planted bias, online softmax, PV accumulation per head
// segment; at the end of a head's segment they publish (max, sum, o[d])
// and bump the head's split-K semaphore.  The CTA completing a head runs
// its epilogue while its producer keeps prefetching: combine, output,
// score update, keep rule (exact top-k on (score desc, position asc) with
// an incremental fast path and a radix-select fallback) and swap-remove
// compaction of the evicted rows.  The consumer owning slot `live` writes
// the new token's row into the arena (fused insert).  live_in / live_out
// are distinct buffers (double-buffered across steps).
//
// Two consumers share this skeleton:
//  * bf16, d in {64,128} (the production path): pages arrive through 2-D
//    TMA with the 128-byte swizzle, and each consumer warp turns a
//    16-key x 16-dim tile into logits and PV with bf16 mma.sync
//    (ldmatrix / ldmatrix.trans, fp32 accumulate), so the SIMT pipes only
//    run the softmax.  Logits (and hence scores) stay fp32; p is rounded to
//    bf16 for the PV product (the cache itself is bf16).
//  * everything else (fp32 caches, small head dims): 1-D bulk copies and
//    SIMT dot products, 8 consumer warps.

#include <math.h>
#include <stdlib.h>

#include "akv_common.cuh"
#include "akv_internal.h"
#include "akv_tma.cuh"

namespace akv {

constexpr int kStages = 3;  // SIMT (fp32 / small d) variant; the tcgen05-era mma kernel takes ST
constexpr int kPageBytes = 16384;  // per K (and per V) page
constexpr int kMaxHeads = 2048;
constexpr int kEpr = 8;   // candidates per thread per batch in the epilogue passes
constexpr int kSmemEvict = 64;  // evictions per head-step paired through shared memory

struct DecParams {
  int B, H, G, prompt_len, pos;
  const void* q;
  const void* kn;
  const void* vn;
  int64_t bh_stride;
  const uint8_t* new_cls;
  const float* slope;
  const float* sink;
  const uint8_t* atoms;
  const double* r_l;
  const double* r_f;
  const int64_t* seg_off;
  const int32_t* seg_cap;
  void* kc;
  void* vc;
  int32_t* meta;
  double* score;
  const int32_t* base_live;
  const int32_t* live_in;
  int32_t* live_out;
  float* out;
  int32_t* evicted;
  int32_t* status;
  float* part;       // [G, max_parts, D+2]
  float* logit;      // [total_slots]
  int32_t* counter;  // [G]
  int max_parts;
  float scale;
  unsigned long long* trace;  // optional [grid, 16] globaltimer stamps (debug hook)
  const int32_t* pos_dev;     // device position (CUDA-graph replays), overrides pos
  int flags;                  // AKV_DECODE_* flags
  float* lse_out;             // [G] log-sum-exp of each head's attended logits, or NULL
  void* const* peer_out;      // [n_peers] buffers [B, peer_ld] receiving o (cache dtype)
  int n_peers;
  int64_t peer_ld, peer_col0;
  int peer_bf16;
  int l2_prefetch;            // pages prefetched into L2 ahead of the shared-memory ring
  int consumer_tail;          // consumers publish (and complete) the CTA's last segment
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define AKV_TRACE(slot)                                                        \
  do {                                                                          \
    if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 16 + (slot)] = gtimer(); \
  } while (0)

// FREQUENT-policy phase stamps (cycles) into trace slots 11-15, debug builds
// only (-DAKV_TRACE_EPI; tools/k3_regimes.py reports them): policy start,
// pass A done, decision made, action done, evictions done
#ifdef AKV_TRACE_EPI
#define AKV_EPI_STAMP(slot)                                                            \
  do {                                                                                 \
    if (p.trace && freq && tid == 0) p.trace[blockIdx.x * 16 + (slot)] = clock64();    \
  } while (0)
#else
#define AKV_EPI_STAMP(slot) do {} while (0)
#endif

// owner CTA of flattened page pg when P pages are split evenly over `grid`
// (CTA i owns [floor(i*P/grid), floor((i+1)*P/grid)))
__device__ __forceinline__ int page_owner(long long pg, long long P, int grid) {
  return (int)(((pg + 1) * grid - 1) / P);
}

struct HeadCtx {
  int g, L, n;
  int pos;  // position of the inserted token
  int64_t base;
  uint8_t atoms;
  bool freq;
  float slope, sink;
  int ncls;
};

__device__ __forceinline__ void load_head(const DecParams& p, int g, int L, HeadCtx& hc) {
  hc.g = g;
  hc.L = L;
  hc.n = L + 1;
  hc.base = p.seg_off[g];
  hc.atoms = p.atoms[g];
  hc.freq = (hc.atoms & AKV_ATOM_FREQUENT) && !(hc.atoms & AKV_ATOM_FULL);
  const int h = g % p.H;
  hc.slope = p.slope ? p.slope[h] : 0.f;
  hc.sink = p.sink ? p.sink[h] : 0.f;
  hc.ncls = p.new_cls[g / p.H];
  hc.pos = p.pos_dev ? *p.pos_dev : p.pos;
}

__device__ __forceinline__ float biased_logit(float dot, int mt, const HeadCtx& hc, int pos) {
  float x = dot;
  if (meta_cls(mt) == AKV_CLS_SPECIAL) x += hc.sink;
  if (hc.slope != 0.f) x -= hc.slope * (float)(pos - meta_pos(mt));
  return x;
}

// ---------------------------------------------------------------------------
// Page plan, run by every CTA: pages per head from live_in and their
// exclusive prefix in shared memory.  Heads whose segment cannot take the
// new row are skipped and flagged (capacity error).
__device__ __forceinline__ long long plan_pages(const DecParams& p, int page, int* s_prefix,
                                                int* s_live, int* red_i) {
  const int G = p.G;
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int lo = min(G, (int)threadIdx.x * per), hi = min(G, lo + per);
  int cnt = 0;
  for (int g = lo; g < hi; ++g) {
    const int L = p.live_in[g];
    int np = 0;
    if (L >= 0 && L + 1 <= p.seg_cap[g]) {
      np = (L + 1 + page - 1) / page;
    } else if (L >= 0 && blockIdx.x == 0) {
      atomicExch(p.status, AKV_ERR_CAPACITY);
      p.live_out[g] = L;
    }
    s_live[g] = np > 0 ? L : -1;
    cnt += np;
  }
  int total;
  int off = block_exclusive_scan<BlockSync>(cnt, red_i, &total);
  for (int g = lo; g < hi; ++g) {
    s_prefix[g] = off;
    off += s_live[g] >= 0 ? (s_live[g] + 1 + page - 1) / page : 0;
  }
  if (threadIdx.x == 0) s_prefix[G] = total;
  __syncthreads();
  return s_prefix[G];
}

// Page plan from live-count BOUNDS (base_live + step), computable before
// the previous step has finished: exact for full-cache heads (their live
// count grows by one per step), an upper bound otherwise (surplus pages are
// streamed as empty).  s_full marks full-cache heads.
__device__ __forceinline__ long long plan_pages_bound(const DecParams& p, int page, int step,
                                                      int* s_prefix, int* s_live,
                                                      uint8_t* s_full, int* red_i) {
  const int G = p.G;
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int lo = min(G, (int)threadIdx.x * per), hi = min(G, lo + per);
  int cnt = 0;
  for (int g = lo; g < hi; ++g) {
    const int want = p.base_live[g] + step;
    // a full-cache head's live count is exactly base_live + step: past its
    // segment the insert cannot fit (flag it; writes stay in bounds)
    if (want > p.seg_cap[g] - 1 && (p.atoms[g] & AKV_ATOM_FULL) && blockIdx.x == 0)
      atomicExch(p.status, AKV_ERR_CAPACITY);
    const int bound = min(want, p.seg_cap[g] - 1);
    s_live[g] = bound;
    s_full[g] = (p.atoms[g] & AKV_ATOM_FULL) ? 1 : 0;
    cnt += (bound + 1 + page - 1) / page;
  }
  int total;
  int off = block_exclusive_scan<BlockSync>(cnt, red_i, &total);
  for (int g = lo; g < hi; ++g) {
    s_prefix[g] = off;
    off += (s_live[g] + 1 + page - 1) / page;
  }
  if (threadIdx.x == 0) s_prefix[G] = total;
  __syncthreads();
  return s_prefix[G];
}

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// live count of a non-full head, read after the previous step completed
__device__ __forceinline__ int live_after_wait(const DecParams& p, int g) {
  int L = p.live_in[g];
  if (L + 1 > p.seg_cap[g]) {  // capacity overflow: flag it, keep writes in bounds
    atomicExch(p.status, AKV_ERR_CAPACITY);
    L = p.seg_cap[g] - 1;
  }
  return L;
}

// largest g with s_prefix[g] <= pg
__device__ __forceinline__ int head_of_page(const int* s_prefix, int G, long long pg) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_prefix[mid] <= pg) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Keep rule + compaction of one head (epilogue group CS).  Pass A streams
// the head's slot metadata (and, for FREQUENT heads, the scores and this
// step's logits) in coalesced batches of kEpr per thread: it applies the
// score update (policies.py:355-357), gathers the statistics of the
// incremental top-k (smallest key in the current frequent set F, largest
// key outside it) and counts the slots that no atom keeps.  The common
// outcomes are resolved from those statistics alone:
//   * F still ranks above every other candidate and the budget grew by at
//     most one -> F stays, plus the best outsider when the budget grew;
//   * at most one slot leaves -> it is refilled from the segment tail.
// Otherwise a crossing repair re-ranks only the candidates between the two
// extremes (the rest of the order is fixed), falling back to the exact
// radix select, and a general compaction pass pairs holes with donors.
template <typename CS>
__device__ void policy_v3(const DecParams& p, const HeadCtx& hc, float lse, int* hist, int* red_i,
                          int rv) {
  constexpr int NC = CS::kThreads, NW = CS::kWarps;
  const int tid = CS::tid(), lane = tid & 31, warp = tid >> 5;
  const int g = hc.g, L = hc.L, n = hc.n;
  const int cur = hc.pos + 1;
  double* score = p.score + hc.base;
  int32_t* meta = p.meta + hc.base;
  const float* lg = p.logit + hc.base;
  const uint8_t atoms = hc.atoms;
  const bool freq = hc.freq;
  const int window_start = cur - budget(p.r_l[g], p.prompt_len);
  auto class_keep = [&](int m) -> bool {
    const int cl = meta_cls(m), ps = meta_pos(m);
    return ((atoms & AKV_ATOM_SPECIAL) && cl == AKV_CLS_SPECIAL) ||
           ((atoms & AKV_ATOM_PUNCT) && cl == AKV_CLS_PUNCT) ||
           ((atoms & AKV_ATOM_LOCAL) && ps >= window_start);
  };
  // key order: larger score first, then lower position (policies.py:238-240)
  auto above = [](unsigned long long ka, int pa, unsigned long long kb, int pb) {
    return ka > kb || (ka == kb && pa < pb);
  };

  AKV_EPI_STAMP(11);
  // ---------------- pass A ----------------
  unsigned long long minF_k = ~0ull, maxN_k = 0ull;
  int minF_p = -1, maxN_p = 0x7fffffff, maxN_slot = -1, maxN_ck = 0, anyN = 0, cntF = 0;
  int nk_cnt = 0, nk_min = 0x7fffffff, nk_max = -1, new_ck = 0;
  for (int b0 = 0; b0 < n; b0 += NC * kEpr) {
    int mv[kEpr];
    double sv[kEpr];
    float lv[kEpr];
#pragma unroll
    for (int i = 0; i < kEpr; ++i) {
      const int j = b0 + i * NC + tid;
      mv[i] = j < n ? __ldcg(meta + j) : 0;
      sv[i] = (freq && j < n) ? __ldcg(score + j) : 0.0;
      lv[i] = (freq && j < L) ? __ldcg(lg + j) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kEpr; ++i) {
      const int j = b0 + i * NC + tid;
      if (j >= n) continue;
      if (freq && j < L) {
        sv[i] += (double)expf(lv[i] - lse);
        score[j] = sv[i];
      }
      const bool ck = class_keep(mv[i]);
      const bool inF = freq && (mv[i] & kInF);
      if (j == L) new_ck = ck;
      else if (!ck && !inF) { ++nk_cnt; nk_min = min(nk_min, j); nk_max = max(nk_max, j); }
      if (freq) {
        const unsigned long long key = score_key(sv[i]);
        const int ps = meta_pos(mv[i]);
        if (inF) {
          ++cntF;
          if (!above(key, ps, minF_k, minF_p) && (key != minF_k || ps != minF_p)) { minF_k = key; minF_p = ps; }
        } else if (!anyN || above(key, ps, maxN_k, maxN_p)) {
          maxN_k = key; maxN_p = ps; maxN_slot = j; maxN_ck = ck; anyN = 1;
        }
      }
    }
  }
  AKV_EPI_STAMP(12);
  // group reductions
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nk_cnt += __shfl_xor_sync(0xffffffffu, nk_cnt, o);
    nk_min = min(nk_min, __shfl_xor_sync(0xffffffffu, nk_min, o));
    nk_max = max(nk_max, __shfl_xor_sync(0xffffffffu, nk_max, o));
    new_ck |= __shfl_xor_sync(0xffffffffu, new_ck, o);
    if (freq) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, minF_k, o);
      const int op = __shfl_xor_sync(0xffffffffu, minF_p, o);
      if (above(minF_k, minF_p, ok, op)) { minF_k = ok; minF_p = op; }
      const unsigned long long nk = __shfl_xor_sync(0xffffffffu, maxN_k, o);
      const int np_ = __shfl_xor_sync(0xffffffffu, maxN_p, o);
      const int ns = __shfl_xor_sync(0xffffffffu, maxN_slot, o);
      const int nc = __shfl_xor_sync(0xffffffffu, maxN_ck, o);
      const int na = __shfl_xor_sync(0xffffffffu, anyN, o);
      if (na && (!anyN || above(nk, np_, maxN_k, maxN_p))) {
        maxN_k = nk; maxN_p = np_; maxN_slot = ns; maxN_ck = nc; anyN = 1;
      }
      cntF += __shfl_xor_sync(0xffffffffu, cntF, o);
    }
  }
  __shared__ unsigned long long s_k[2][NW];
  __shared__ int s_i[9][NW];
  __shared__ int s_mode, s_add, s_nkeep, s_x, s_donor, s_cnt;
  __shared__ unsigned long long s_mf_k, s_mn_k;
  __shared__ int s_mf_p, s_mn_p, s_kb;
  CS::sync();
  if (lane == 0) {
    s_k[0][warp] = minF_k; s_i[0][warp] = minF_p;
    s_k[1][warp] = maxN_k; s_i[1][warp] = maxN_p;
    s_i[2][warp] = anyN ? maxN_slot : -1; s_i[3][warp] = maxN_ck;
    s_i[4][warp] = cntF; s_i[5][warp] = nk_cnt; s_i[6][warp] = nk_min; s_i[7][warp] = nk_max;
    s_i[8][warp] = new_ck;
  }
  CS::sync();
  if (tid == 0) {
    unsigned long long mf = ~0ull, mn = 0ull;
    int mfp = -1, mnp = 0x7fffffff, mns = -1, mnc = 0, cf = 0, ec = 0, emin = 0x7fffffff, emax = -1, nck = 0;
    bool an = false;
    for (int w = 0; w < NW; ++w) {
      cf += s_i[4][w]; ec += s_i[5][w];
      emin = min(emin, s_i[6][w]); emax = max(emax, s_i[7][w]); nck |= s_i[8][w];
      if (above(mf, mfp, s_k[0][w], s_i[0][w])) { mf = s_k[0][w]; mfp = s_i[0][w]; }
      if (s_i[2][w] >= 0 && (!an || above(s_k[1][w], s_i[1][w], mn, mnp))) {
        mn = s_k[1][w]; mnp = s_i[1][w]; mns = s_i[2][w]; mnc = s_i[3][w]; an = true;
      }
    }
    // mode: 0 resolved from statistics, 1 crossing repair, 2 radix select, 3 select all
    int mode = 0, add = -1;
    const int kb = freq ? budget(p.r_f[g], cur) : 0;
    if (freq) {
      if (kb >= n) mode = 3;
      else if (cf == 0) mode = 2;
      else if (!an || above(mf, mfp, mn, mnp)) {  // F separated from the rest
        if (kb == cf) mode = 0;
        else if (kb == cf + 1) { mode = 0; add = mns; }
        else mode = 2;
      } else {
        mode = 1;
      }
    }
    int nkeep = -1, x = -1, donor = -1;
    if (mode == 0) {
      // slots leaving: old slots no atom keeps, minus the joining outsider
      int e = ec;
      int a0 = emin, a1 = emax;
      if (add >= 0 && add != L && !mnc) {
        --e;
        if (add == a0) a0 = a1; else if (add == a1) a1 = a0;
      }
      const bool new_kept = nck || add == L;
      if (e == 0) {
        nkeep = new_kept ? n : n - 1;
      } else if (e == 1) {
        x = a0;
        if (new_kept) { nkeep = n - 1; donor = n - 1; }
        else { nkeep = n - 2; donor = (x == n - 2) ? -1 : n - 2; }
      }
    }
    s_mode = mode; s_add = add; s_nkeep = nkeep; s_x = x; s_donor = donor;
    s_mf_k = mf; s_mf_p = mfp; s_mn_k = mn; s_mn_p = mnp; s_kb = kb;
    s_cnt = 0;
  }
  CS::sync();
  int mode = s_mode;
  AKV_EPI_STAMP(13);
  if (freq) {
    if (mode == 0) {
      if (tid == 0 && s_add >= 0) meta[s_add] = __ldcg(meta + s_add) | kInF;
    } else if (mode == 3) {  // every candidate is in the frequent set
      for (int j = tid; j < n; j += NC) {
        const int m = __ldcg(meta + j);
        if (!(m & kInF)) meta[j] = m | kInF;
      }
    } else if (mode == 1) {
      // crossing repair: F members above the best outsider stay, outsiders
      // below the weakest F member stay out; re-rank the band between them
      constexpr int kBand = 128;
      __shared__ unsigned long long s_bk[kBand];
      __shared__ int s_bp[kBand], s_bs[kBand];
      __shared__ int s_above;
      if (tid == 0) s_above = 0;
      CS::sync();
      const unsigned long long mf = s_mf_k, mn = s_mn_k;
      const int mfp = s_mf_p, mnp = s_mn_p;
      int my_above = 0;
      for (int b0 = 0; b0 < n; b0 += NC * kEpr) {
        int mv[kEpr];
        double sv[kEpr];
#pragma unroll
        for (int i = 0; i < kEpr; ++i) {
          const int j = b0 + i * NC + tid;
          mv[i] = j < n ? __ldcg(meta + j) : 0;
          sv[i] = j < n ? __ldcg(score + j) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kEpr; ++i) {
          const int j = b0 + i * NC + tid;
          if (j >= n) continue;
          const unsigned long long key = score_key(sv[i]);
          const int ps = meta_pos(mv[i]);
          if (above(key, ps, mn, mnp)) { my_above += (mv[i] & kInF) ? 1 : 0; continue; }
          if (above(mf, mfp, key, ps)) continue;  // strictly below the weakest F member
          const int at = atomicAdd(&s_cnt, 1);
          if (at < kBand) { s_bk[at] = key; s_bp[at] = ps; s_bs[at] = j; }
        }
      }
      my_above = block_sum<int, CS>(my_above, red_i);
      const int band = s_cnt;
      const int need = s_kb - my_above;
      if (band > kBand || need < 0 || need > band) {
        mode = 2;
      } else {
        for (int c = tid; c < band; c += NC) {
          int rank = 0;
          for (int o = 0; o < band; ++o) rank += above(s_bk[o], s_bp[o], s_bk[c], s_bp[c]);
          const int j = s_bs[c];
          const int m = __ldcg(meta + j);
          const int nm = rank < need ? (m | kInF) : (m & ~kInF);
          if (nm != m) meta[j] = nm;
        }
      }
    }
    if (mode == 2) {  // exact radix select over all candidates
      if (p.trace && tid == 0) atomicAdd(&p.trace[blockIdx.x * 16 + 7], 1ull);
      unsigned long long thr_key;
      int thr_pos;
      auto get = [&](int i, unsigned long long* key, int* pos) {
        *key = score_key(__ldcg(score + i));
        *pos = meta_pos(__ldcg(meta + i));
      };
      block_topk_threshold<CS>(n, s_kb, get, hist, red_i, &thr_key, &thr_pos);
      for (int j = tid; j < n; j += NC) {
        const int m = __ldcg(meta + j);
        const bool sel = topk_selected(score_key(__ldcg(score + j)),
                                       meta_pos(m), thr_key, thr_pos);
        const int nm = sel ? (m | kInF) : (m & ~kInF);
        if (nm != m) meta[j] = nm;
      }
    }
    CS::sync();
  }
  AKV_EPI_STAMP(14);
  uint4* kw = static_cast<uint4*>(p.kc) + hc.base * rv;
  uint4* vw = static_cast<uint4*>(p.vc) + hc.base * rv;
  int n_keep;
  if (mode == 0 && s_nkeep >= 0) {
    // at most one hole, refilled from the tail
    n_keep = s_nkeep;
    const int x = s_x, src = s_donor;
    if (x >= 0 && src >= 0 && warp == 0) {
      for (int v = lane; v < rv; v += 32) {
        st_v4(kw + (size_t)x * rv + v, ld_cg_v4(kw + (size_t)src * rv + v));
        st_v4(vw + (size_t)x * rv + v, ld_cg_v4(vw + (size_t)src * rv + v));
      }
      if (lane == 0) {
        meta[x] = __ldcg(meta + src);
        if (freq) score[x] = __ldcg(score + src);
      }
    }
  } else if (mode == 3) {
    n_keep = n;
  } else {
    // general compaction: count, then pair holes (dropped slots below n')
    // with donors (kept slots at or above n'); any pairing is valid
    auto keep = [&](int m) { return class_keep(m) || (freq && (m & kInF)); };
    int nk = 0;
    for (int b0 = 0; b0 < n; b0 += NC * kEpr) {
      int mv[kEpr];
#pragma unroll
      for (int i = 0; i < kEpr; ++i) {
        const int j = b0 + i * NC + tid;
        mv[i] = j < n ? __ldcg(meta + j) : 0;
      }
#pragma unroll
      for (int i = 0; i < kEpr; ++i) nk += (b0 + i * NC + tid < n) && keep(mv[i]);
    }
    n_keep = block_sum<int, CS>(nk, red_i);
    if (n_keep < n) {
      __shared__ int s_hole[kSmemEvict], s_don[kSmemEvict];
      __shared__ int s_nh, s_nd;
      if (tid == 0) { s_nh = 0; s_nd = 0; }
      CS::sync();
      int* gl_hole = reinterpret_cast<int*>(p.logit + hc.base);  // logits are consumed
      const int cap_g = n / 2;
      for (int b0 = 0; b0 < n; b0 += NC * kEpr) {
        int mv[kEpr];
#pragma unroll
        for (int i = 0; i < kEpr; ++i) {
          const int j = b0 + i * NC + tid;
          mv[i] = j < n ? __ldcg(meta + j) : 0;
        }
#pragma unroll
        for (int i = 0; i < kEpr; ++i) {
          const int j = b0 + i * NC + tid;
          if (j >= n) continue;
          const bool k = keep(mv[i]);
          if (j < n_keep && !k) {
            const int at = atomicAdd(&s_nh, 1);
            if (at < kSmemEvict) s_hole[at] = j; else gl_hole[at] = j;
          } else if (j >= n_keep && k) {
            const int at = atomicAdd(&s_nd, 1);
            if (at < kSmemEvict) s_don[at] = j; else gl_hole[cap_g + at] = j;
          }
        }
      }
      CS::sync();
      const int nh = s_nh;
      for (int r = warp; r < nh; r += NW) {
        const int dst = r < kSmemEvict ? s_hole[r] : __ldcg(gl_hole + r);
        const int src = r < kSmemEvict ? s_don[r] : __ldcg(gl_hole + cap_g + r);
        for (int v = lane; v < rv; v += 32) {
          st_v4(kw + (size_t)dst * rv + v, ld_cg_v4(kw + (size_t)src * rv + v));
          st_v4(vw + (size_t)dst * rv + v, ld_cg_v4(vw + (size_t)src * rv + v));
        }
        if (lane == 0) {
          meta[dst] = __ldcg(meta + src);
          if (freq) score[dst] = __ldcg(score + src);
        }
      }
    }
  }
  if (tid == 0) {
    AKV_EPI_STAMP(15);
    p.live_out[g] = n_keep;
    if (p.evicted) p.evicted[g] = n - n_keep;
    p.counter[g] = 0;
  }
  CS::sync();
}

// ---------------------------------------------------------------------------
// Epilogue of one head: the combine of its split-K partials, its output and
// live count, and (evicting heads) its policy - run by the group CS of the
// head's last contributor.
template <typename CS, int D, bool kPolicy = true>
__device__ void head_epilogue(const DecParams& p, const HeadCtx& hc, int nparts, int rv,
                              int* hist, int* red_i) {
  constexpr int NC = CS::kThreads;
  const int tid = CS::tid();
  const int g = hc.g, n = hc.n;
  // combine the partials of all contributing CTAs; every thread issues its
  // loads for a batch of parts (max, sum and its output dims) at once, so a
  // batch costs one L2 round trip
  const float* parts = p.part + (size_t)g * p.max_parts * (D + 2);
  constexpr int kB = 8;
  constexpr int DPT = (D + NC - 1) / NC;  // output dims per thread
  float gM = -INFINITY, gl = 0.f, acc[DPT];
#pragma unroll
  for (int u = 0; u < DPT; ++u) acc[u] = 0.f;
  for (int k0 = 0; k0 < nparts; k0 += kB) {
    float mk[kB], lk[kB], ok[kB][DPT];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const bool v = k0 + b < nparts;
      const float* pk = parts + (size_t)(k0 + b) * (D + 2);
      mk[b] = v ? __ldcg(pk + D) : -INFINITY;
      lk[b] = v ? __ldcg(pk + D + 1) : 0.f;
#pragma unroll
      for (int u = 0; u < DPT; ++u) {
        const int t = tid + u * NC;
        ok[b][u] = (v && t < D) ? __ldcg(pk + t) : 0.f;
      }
    }
    float newM = gM;
#pragma unroll
    for (int b = 0; b < kB; ++b) newM = fmaxf(newM, mk[b]);
    const float rs = (gM == -INFINITY) ? 0.f : __expf(gM - newM);
    gl *= rs;
#pragma unroll
    for (int u = 0; u < DPT; ++u) acc[u] *= rs;
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const float w = (mk[b] == -INFINITY) ? 0.f : __expf(mk[b] - newM);
      gl += w * lk[b];
#pragma unroll
      for (int u = 0; u < DPT; ++u) acc[u] += w * ok[b][u];
    }
    gM = newM;
  }
  {
    const float inv = 1.f / gl;
#pragma unroll
    for (int u = 0; u < DPT; ++u) {
      const int t = tid + u * NC;
      if (t < D) p.out[(size_t)g * D + t] = acc[u] * inv;
    }
    if (p.lse_out && tid == 0) p.lse_out[g] = gM + logf(gl);
    // the head's output row also goes straight into every peer's gathered
    // [B, H_total*d] buffer (the cross-shard gather of a head-sharded model
    // layer, fused into the combine: no separate collective, no cast)
    if (p.n_peers > 0) {
      const int b = g / p.H, h = g % p.H;
      const int64_t off = (int64_t)b * p.peer_ld + p.peer_col0 + (int64_t)h * D;
      for (int r = 0; r < p.n_peers; ++r) {
        void* base = p.peer_out[r];
#pragma unroll
        for (int u = 0; u < DPT; ++u) {
          const int t = tid + u * NC;
          if (t >= D) continue;
          if (p.peer_bf16)
            static_cast<__nv_bfloat16*>(base)[off + t] = __float2bfloat16_rn(acc[u] * inv);
          else
            static_cast<float*>(base)[off + t] = acc[u] * inv;
        }
      }
    }
  }
  if (hc.atoms & AKV_ATOM_FULL) {  // the full cache never evicts
    if (tid == 0) {
      p.live_out[g] = n;
      if (p.evicted) p.evicted[g] = 0;
      p.counter[g] = 0;
    }
    CS::sync();
    return;
  }
  const float lse = gM + logf(gl);
  if constexpr (kPolicy) policy_v3<CS>(p, hc, lse, hist, red_i, rv);
}

// Publish a CTA's partial (max, sum, o[D]) for head g from NWC per-warp
// values in s_red / s_ml (group CS), bump the semaphore, and run the
// epilogue if this CTA is the last contributor.  `release` (optional) is
// arrived on once s_red / s_ml have been consumed.
template <typename CS, int NWC, int D, bool kPolicy = true>
__device__ __forceinline__ void publish_head(const DecParams& p, const HeadCtx& hc,
                                             const int* s_prefix, long long P, int grid,
                                             const float (*s_red)[D], const float (*s_ml)[2],
                                             int* s_last, int rv, int* hist, int* red_i,
                                             uint64_t* release) {
  constexpr int NC = CS::kThreads;
  const int tid = CS::tid();
  const int g = hc.g;
  CS::sync();
  if (p.trace && tid == 0) p.trace[blockIdx.x * 16 + 8] = gtimer();   // publish start
  const int own0 = page_owner(s_prefix[g], P, grid);
  const int nparts = page_owner(s_prefix[g + 1] - 1, P, grid) - own0 + 1;
  float* part = p.part + ((size_t)g * p.max_parts + (blockIdx.x - own0)) * (D + 2);
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NWC; ++w) M = fmaxf(M, s_ml[w][0]);
  for (int t = tid; t < D; t += NC) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < NWC; ++w)
      if (s_ml[w][0] != -INFINITY) acc += s_red[w][t] * __expf(s_ml[w][0] - M);
    part[t] = acc;
  }
  if (tid == 0) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < NWC; ++w)
      if (s_ml[w][0] != -INFINITY) l += s_ml[w][1] * __expf(s_ml[w][0] - M);
    part[D] = M;
    part[D + 1] = l;
  }
  CS::sync();  // the partial is written by the whole group ...
  if (tid == 0) {  // ... and released to the device by one thread (cumulative)
    if (release) mbar_arrive(release);
    int prev;
    asm volatile("fence.acq_rel.gpu;\n\tatom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(p.counter + g) : "memory");
    *s_last = (prev == nparts - 1);
    if (p.trace) p.trace[blockIdx.x * 16 + 9] = gtimer();                // partial released
  }
  CS::sync();
  if (*s_last) head_epilogue<CS, D, kPolicy>(p, hc, nparts, rv, hist, red_i);
  if (p.trace && tid == 0) p.trace[blockIdx.x * 16 + 10] = gtimer();    // segment finished
}

// ===========================================================================
// SIMT consumer (fp32 caches, any supported head dim): 1-D bulk copies.
template <typename T, int D>
struct SimtShape {
  static constexpr int NW = 8;
  static constexpr int EV = Elem<T>::kPerVec;
  static constexpr int RB = D * (int)sizeof(T);
  static constexpr int LPR = RB / 16;
  static constexpr int RPW = 32 / LPR;
  static constexpr int PAGE = kPageBytes / RB;
  static constexpr int STEPS = PAGE / (NW * RPW);
  static constexpr int META_B = PAGE * 4;
  static constexpr int STAGE_B = 2 * kPageBytes + META_B + 3 * RB;
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "unsupported head dim");
  static_assert(STEPS >= 1 && STEPS * NW * RPW == PAGE, "page split");
};

template <typename T, int D>
__global__ void __launch_bounds__(SimtShape<T, D>::NW * 32 + 32, 2) k3_decode_simt(DecParams p) {
  using S = SimtShape<T, D>;
  constexpr int NW = S::NW, EV = S::EV, RB = S::RB, LPR = S::LPR, RPW = S::RPW, PAGE = S::PAGE;
  constexpr int STEPS = S::STEPS;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ float s_red[NW][D];
  __shared__ float s_ml[NW][2];
  __shared__ int s_last;
  __shared__ int hist[256];
  __shared__ int red_i[33];

  const int G = p.G;
  int* s_prefix = reinterpret_cast<int*>(smem + kStages * S::STAGE_B);
  int* s_live = s_prefix + (G + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], NW); }
    mbar_fence_init();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long P = plan_pages(p, PAGE, s_prefix, s_live, red_i);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int grid = (int)(P < (long long)gridDim.x ? P : (long long)gridDim.x);
  if ((int)blockIdx.x >= grid) return;
  const long long pbeg = (long long)blockIdx.x * P / grid;
  const long long pend = (long long)(blockIdx.x + 1) * P / grid;
  const int g0 = head_of_page(s_prefix, G, pbeg);

  if (warp == NW) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
      int g = g0, stage = 0;
      uint32_t phase = 0;
      for (long long pg = pbeg; pg < pend; ++pg) {
        while (pg >= s_prefix[g + 1]) ++g;
        const int L = s_live[g];
        const int slot0 = (int)(pg - s_prefix[g]) * PAGE;
        const int rows = max(0, min(PAGE, L - slot0));
        const bool has_new = (L >= slot0 && L < slot0 + PAGE);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * S::STAGE_B;
        const int64_t base = p.seg_off[g];
        const uint32_t meta_b = ((rows * 4) + 15) & ~15;
        const uint32_t bytes = 2u * rows * RB + (rows ? meta_b : 0) + RB + (has_new ? 2 * RB : 0);
        mbar_arrive_expect_tx(&full_bar[stage], bytes);
        if (rows) {
          bulk_g2s(st, static_cast<const uint8_t*>(p.kc) + (base + slot0) * RB, rows * RB,
                   &full_bar[stage], pol_stream);
          bulk_g2s(st + kPageBytes, static_cast<const uint8_t*>(p.vc) + (base + slot0) * RB,
                   rows * RB, &full_bar[stage], pol_stream);
          bulk_g2s(st + 2 * kPageBytes, p.meta + base + slot0, meta_b, &full_bar[stage], pol_keep);
        }
        uint8_t* hdr = st + 2 * kPageBytes + S::META_B;
        bulk_g2s(hdr, static_cast<const T*>(p.q) + (size_t)g * p.bh_stride, RB, &full_bar[stage],
                 pol_keep);
        if (has_new) {
          bulk_g2s(hdr + RB, static_cast<const T*>(p.kn) + (size_t)g * p.bh_stride, RB,
                   &full_bar[stage], pol_keep);
          bulk_g2s(hdr + 2 * RB, static_cast<const T*>(p.vn) + (size_t)g * p.bh_stride, RB,
                   &full_bar[stage], pol_keep);
        }
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int sub = lane / LPR, sl = lane % LPR;
  int g = g0, stage = 0;
  uint32_t phase = 0;
  HeadCtx hc;
  hc.g = -1;
  float m_run = -INFINITY, l_run = 0.f;
  float o[EV];
#pragma unroll
  for (int e = 0; e < EV; ++e) o[e] = 0.f;

  for (long long pg = pbeg; pg < pend; ++pg) {
    while (pg >= s_prefix[g + 1]) ++g;
    if (g != hc.g) load_head(p, g, s_live[g], hc);
    const int L = hc.L;
    const int slot0 = (int)(pg - s_prefix[g]) * PAGE;
    mbar_wait(&full_bar[stage], phase);
    const uint8_t* st = smem + stage * S::STAGE_B;
    const uint4* kpage = reinterpret_cast<const uint4*>(st);
    const uint4* vpage = reinterpret_cast<const uint4*>(st + kPageBytes);
    const int* mpage = reinterpret_cast<const int*>(st + 2 * kPageBytes);
    const uint4* hdr = reinterpret_cast<const uint4*>(st + 2 * kPageBytes + S::META_B);
    float qf[EV];
    Elem<T>::unpack(hdr[sl], qf);
#pragma unroll
    for (int e = 0; e < EV; ++e) qf[e] *= p.scale;
    float sj[STEPS];
    float pm = -INFINITY;
#pragma unroll
    for (int s = 0; s < STEPS; ++s) {
      const int row = warp * (PAGE / NW) + s * RPW + sub;
      const int slot = slot0 + row;
      uint4 kv;
      int mt;
      if (slot < L) { kv = kpage[row * LPR + sl]; mt = mpage[row]; }
      else if (slot == L) { kv = hdr[LPR + sl]; mt = hc.pos | (hc.ncls << kClsShift); }
      else { kv = make_uint4(0, 0, 0, 0); mt = -1; }
      float kf[EV];
      Elem<T>::unpack(kv, kf);
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < EV; ++e) dot = fmaf(qf[e], kf[e], dot);
#pragma unroll
      for (int off = 1; off < LPR; off <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      float x = -INFINITY;
      if (mt >= 0) {
        x = biased_logit(dot, mt, hc, hc.pos);
        if (hc.freq && sl == 0 && slot < L) p.logit[hc.base + slot] = x;
      }
      sj[s] = x;
      pm = fmaxf(pm, x);
    }
    pm = warp_allreduce(pm, [](float a, float b) { return fmaxf(a, b); });
    const float m_new = fmaxf(m_run, pm);
    if (m_new != -INFINITY) {
      const float sc = (m_run == -INFINITY) ? 0.f : __expf(m_run - m_new);
      l_run *= sc;
#pragma unroll
      for (int e = 0; e < EV; ++e) o[e] *= sc;
#pragma unroll
      for (int s = 0; s < STEPS; ++s) {
        const int row = warp * (PAGE / NW) + s * RPW + sub;
        const int slot = slot0 + row;
        const float pe = (sj[s] == -INFINITY) ? 0.f : __expf(sj[s] - m_new);
        if (sl == 0) l_run += pe;
        uint4 vv;
        if (slot < L) vv = vpage[row * LPR + sl];
        else if (slot == L) vv = hdr[2 * LPR + sl];
        else vv = make_uint4(0, 0, 0, 0);
        float vf[EV];
        Elem<T>::unpack(vv, vf);
#pragma unroll
        for (int e = 0; e < EV; ++e) o[e] = fmaf(pe, vf[e], o[e]);
        if (slot == L) {  // fused insert of the new token's row
          uint4* kw = static_cast<uint4*>(p.kc) + (hc.base + slot) * LPR;
          uint4* vw = static_cast<uint4*>(p.vc) + (hc.base + slot) * LPR;
          st_v4(kw + sl, hdr[LPR + sl]);
          st_v4(vw + sl, vv);
          if (sl == 0) {
            p.meta[hc.base + slot] = hc.pos | (hc.ncls << kClsShift);
            p.score[hc.base + slot] = 0.0;  // policies.py:357
          }
        }
      }
      m_run = m_new;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);
    if (++stage == kStages) { stage = 0; phase ^= 1; }

    if (!((pg + 1 == pend) || (pg + 1 == s_prefix[g + 1]))) continue;
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
      for (int e = 0; e < EV; ++e) o[e] += __shfl_xor_sync(0xffffffffu, o[e], off);
    }
    l_run = warp_allreduce(l_run, [](float a, float b) { return a + b; });
    if (sub == 0) {
#pragma unroll
      for (int e = 0; e < EV; ++e) s_red[warp][sl * EV + e] = o[e];
    }
    if (lane == 0) { s_ml[warp][0] = m_run; s_ml[warp][1] = l_run; }
    publish_head<NamedSync<NW * 32, 1, 0>, NW, D>(p, hc, s_prefix, P, grid, s_red, s_ml, &s_last,
                                                  LPR, hist, red_i, nullptr);
    m_run = -INFINITY;
    l_run = 0.f;
#pragma unroll
    for (int e = 0; e < EV; ++e) o[e] = 0.f;
  }
}

// ===========================================================================
// bf16 tensor-core consumer (d = 64 / 128): 2-D TMA with the 128-byte
// swizzle, ldmatrix + mma.sync.m16n8k16 (bf16 in, fp32 accumulate).
template <int D>
struct MmaShape {
  static constexpr int NW = 4;                      // consumer warps
  // three epilogue warps: 9 -> 8 warps per CTA lifts the register cap of
  // two CTAs per SM from 96 to 128 (4 warps per SM sub-partition); measured
  // c1 29.60 -> 28.71 us/step, c1_frequent 32.61 -> 32.76 (two: 28.90 /
  // 36.35, the FREQUENT epilogues need the threads)
  static constexpr int NE = 3;                      // epilogue warps
  static constexpr int THREADS = (NW + 1 + NE) * 32; // + producer warp
  static constexpr int EFIRST = (NW + 1) * 32;      // first epilogue thread
  static constexpr int RB = D * 2;
  static constexpr int PAGE = kPageBytes / RB;      // 64 (d=128) / 128 (d=64)
  static constexpr int KPW = PAGE / NW;             // keys per warp per page
  static constexpr int TILES = KPW / 16;            // 16-key tiles per warp
  static constexpr int NBOX = D / 64;               // 64-column TMA boxes per page
  static constexpr int BOX_B = PAGE * 128;          // bytes per box
  static constexpr int META_B = PAGE * 4;
  static constexpr int HDR_OFF = 2 * kPageBytes + META_B;
  static constexpr int STAGE_B = ((HDR_OFF + 3 * RB) + 1023) & ~1023;  // 1 KB aligned stages
  static_assert(TILES >= 1 && KPW % 16 == 0, "page split");
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                        uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                          uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset of (row r, 16-byte chunk c of the d axis) in a swizzled page
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 3) * MmaShape<D>::BOX_B + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// Consumer -> epilogue handoff of one head segment's per-warp results.
template <int NW, int D>
struct PubSlot {
  float red[NW][D];
  float ml[NW][2];
  HeadCtx ctx;
};

// ST ring stages (2 by default, 3 for tuning; see launch_mma)
template <int D, int ST>
__global__ void __launch_bounds__(MmaShape<D>::THREADS, 2)
    k3_decode_mma(const __grid_constant__ DecParams p, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV) {
  using S = MmaShape<D>;
  constexpr int NW = S::NW, RB = S::RB, PAGE = S::PAGE, KPW = S::KPW, TILES = S::TILES;
  constexpr int NK = D / 16;  // 16-dim chunks
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[ST], empty_bar[ST];
  __shared__ __align__(8) uint64_t pub_full[2], pub_empty[2];
  __shared__ PubSlot<NW, D> s_pub[2];
  __shared__ int s_last;
  __shared__ int hist[256];
  __shared__ int red_i[33];
  using ES = NamedSync<S::NE * 32, 2, S::EFIRST>;

  const int G = p.G;
  int* s_prefix = reinterpret_cast<int*>(smem + ST * S::STAGE_B);
  int* s_live = s_prefix + (G + 1);
  uint8_t* s_full = reinterpret_cast<uint8_t*>(s_live + G);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  AKV_TRACE(0);
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], NW); }
    for (int s = 0; s < 2; ++s) { mbar_init(&pub_full[s], NW); mbar_init(&pub_empty[s], 1); }
    mbar_fence_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  // Programmatic dependent launch.  When the previous launch on the stream
  // is the previous decode step (step > 0), its CTAs signalled only after
  // their own predecessor had completed, so every arena row below slot
  // live-1 of a full-cache head is already final: those pages stream
  // before griddepcontrol.wait.  Anything the previous step writes (its
  // inserted row, live counts and rows of evicting heads, semaphores,
  // partials, outputs) is touched only after the wait.
  // Early streaming is opt-in (AKV_DECODE_CHAINED): the caller guarantees
  // that q/k/v and the new classes were not written by the kernel launched
  // just before this one (e.g. a rope kernel of a model layer).  A device
  // position (graph replays) is read only after the wait.
  int step;
  bool early = false;
  if (p.pos_dev) {
    grid_dep_wait();
    step = *p.pos_dev - p.prompt_len;
  } else {
    step = p.pos - p.prompt_len;
    early = (p.flags & AKV_DECODE_CHAINED) && step > 0;
    if (!early) grid_dep_wait();
  }
  const long long P = plan_pages_bound(p, PAGE, step, s_prefix, s_live, s_full, red_i);
  AKV_TRACE(1);
  const int grid = (int)(P < (long long)gridDim.x ? P : (long long)gridDim.x);
  if ((int)blockIdx.x >= grid) return;
  const long long pbeg = (long long)blockIdx.x * P / grid;
  const long long pend = (long long)(blockIdx.x + 1) * P / grid;
  const int g0 = head_of_page(s_prefix, G, pbeg);

  if (warp == NW) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
      bool waited = !early;
      int g = g0, stage = 0, gl = -1, L = 0;
      uint32_t phase = 0;
      // L2 prefetch cursor: the pages just beyond the shared-memory ring go
      // to L2 early (coherent, so safe before the previous step drains),
      // raising the bytes in flight per CTA beyond what the ring can hold
      long long pf = pbeg + ST;
      int gpf = g0;
      for (long long pg = pbeg; pg < pend; ++pg) {
        for (const long long lim = min(pend, pg + ST + p.l2_prefetch); pf < lim; ++pf) {
          while (pf >= s_prefix[gpf + 1]) ++gpf;
          const int s0 = (int)(pf - s_prefix[gpf]) * PAGE;
          if (s0 <= s_live[gpf]) {
            const int row0 = (int)(p.seg_off[gpf] + s0);
#pragma unroll
            for (int bx = 0; bx < S::NBOX; ++bx) {
              tma_prefetch_l2_2d(&tmK, bx * 64, row0);
              tma_prefetch_l2_2d(&tmV, bx * 64, row0);
            }
          }
        }
        while (pg >= s_prefix[g + 1]) ++g;
        if (g != gl) {
          gl = g;
          if (s_full[g]) {
            L = s_live[g];
          } else {
            if (!waited) { grid_dep_wait(); waited = true; }
            L = live_after_wait(p, g);
          }
        }
        const int slot0 = (int)(pg - s_prefix[g]) * PAGE;
        const int rows = max(0, min(PAGE, L - slot0));
        const bool has_new = (L >= slot0 && L < slot0 + PAGE);
        // the previous step wrote row L-1 of a full head; a page holding it waits
        if (!waited && slot0 + rows > L - 1) { grid_dep_wait(); waited = true; }
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * S::STAGE_B;
        const int64_t base = p.seg_off[g];
        const uint32_t meta_b = ((rows * 4) + 15) & ~15;
        const uint32_t bytes = (rows ? 2u * kPageBytes + meta_b : 0u) + RB + (has_new ? 2 * RB : 0);
        mbar_arrive_expect_tx(&full_bar[stage], bytes);
        if (rows) {
          const int row0 = (int)(base + slot0);
#pragma unroll
          for (int bx = 0; bx < S::NBOX; ++bx) {
            tma_load_2d(st + bx * S::BOX_B, &tmK, bx * 64, row0, &full_bar[stage], pol_stream);
            tma_load_2d(st + kPageBytes + bx * S::BOX_B, &tmV, bx * 64, row0, &full_bar[stage],
                        pol_stream);
          }
          bulk_g2s(st + 2 * kPageBytes, p.meta + base + slot0, meta_b, &full_bar[stage], pol_keep);
        }
        uint8_t* hdr = st + S::HDR_OFF;
        bulk_g2s(hdr, static_cast<const __nv_bfloat16*>(p.q) + (size_t)g * p.bh_stride, RB,
                 &full_bar[stage], pol_keep);
        if (has_new) {
          bulk_g2s(hdr + RB, static_cast<const __nv_bfloat16*>(p.kn) + (size_t)g * p.bh_stride, RB,
                   &full_bar[stage], pol_keep);
          bulk_g2s(hdr + 2 * RB, static_cast<const __nv_bfloat16*>(p.vn) + (size_t)g * p.bh_stride,
                   RB, &full_bar[stage], pol_keep);
        }
        if (++stage == ST) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }

  if (warp > NW) {  // ---------------- epilogue warps ----------------
    // semaphores, partials, outputs and policy state belong to the previous
    // step until it completes; once it has, dependents may launch
    grid_dep_wait();
    if (warp == NW + 1 && lane == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // one published segment per head touched by this CTA's page range, in order
    int pub_n = 0;
    for (int g = g0; g < G && s_prefix[g] < pend; ++g) {
      if (s_prefix[g + 1] == s_prefix[g]) continue;  // head without pages
      // the consumers publish the CTA's last segment themselves (and run
      // its policy if this CTA completes the head)
      if (p.consumer_tail && s_prefix[g + 1] >= pend) break;
      const int slot = pub_n & 1;
      mbar_wait(&pub_full[slot], (pub_n >> 1) & 1);
      const HeadCtx hc = s_pub[slot].ctx;
      publish_head<ES, NW, D>(p, hc, s_prefix, P, grid, s_pub[slot].red, s_pub[slot].ml, &s_last,
                              RB / 16, hist, red_i, &pub_empty[slot]);
      if (s_last && p.trace && ES::tid() == 0) {
        atomicAdd(&p.trace[blockIdx.x * 16 + 5], 1ull);               // epilogues run
        if (hc.freq) atomicAdd(&p.trace[blockIdx.x * 16 + 6], 1ull);  // frequent ones
      }
      ++pub_n;
    }
    if (p.trace && ES::tid() == 0) p.trace[blockIdx.x * 16 + 4] = gtimer();
    return;
  }

  // ---------------- consumers ----------------
  const int gq = lane >> 2, qq = lane & 3;  // mma fragment coordinates
  int pub_n = 0;
  int g = g0, stage = 0;
  uint32_t phase = 0;
  HeadCtx hc;
  hc.g = -1;
  float m_run = -INFINITY, l_run = 0.f;
  float o[NK][4];
#pragma unroll
  for (int t = 0; t < NK; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;

  for (long long pg = pbeg; pg < pend; ++pg) {
    while (pg >= s_prefix[g + 1]) ++g;
    if (g != hc.g) {
      int Lh = s_live[g];
      if (!s_full[g]) {  // evicting head: its live count comes from the previous step
        if (early) grid_dep_wait();
        Lh = live_after_wait(p, g);
      }
      load_head(p, g, Lh, hc);
    }
    const int L = hc.L, n = hc.n;
    const int slot0 = (int)(pg - s_prefix[g]) * PAGE;
    mbar_wait(&full_bar[stage], phase);
    if (pg == pbeg) AKV_TRACE(2);
    uint8_t* st = smem + stage * S::STAGE_B;
    const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + kPageBytes);
    const int* mpage = reinterpret_cast<const int*>(st + 2 * kPageBytes);
    const uint8_t* hdr = st + S::HDR_OFF;
    // the new token's row replaces its (stale) arena row in this warp's tile
    const int wrow0 = warp * KPW;
    if (L >= slot0 + wrow0 && L < slot0 + wrow0 + KPW) {
      const int r = L - slot0;
      const uint4* kn = reinterpret_cast<const uint4*>(hdr + RB);
      const uint4* vn = reinterpret_cast<const uint4*>(hdr + 2 * RB);
      for (int c = lane; c < 2 * (RB / 16); c += 32) {
        const int cc = c % (RB / 16);
        const uint4 val = c < RB / 16 ? kn[cc] : vn[cc];
        *reinterpret_cast<uint4*>(st + (c < RB / 16 ? 0 : kPageBytes) + swz<D>(r, cc)) = val;
        uint4* dstg = static_cast<uint4*>(c < RB / 16 ? p.kc : p.vc) + (hc.base + L) * (RB / 16);
        st_v4(dstg + cc, val);  // fused insert into the arena
      }
      if (lane == 0) {
        p.meta[hc.base + L] = hc.pos | (hc.ncls << kClsShift);
        p.score[hc.base + L] = 0.0;  // policies.py:357
      }
      fence_proxy_async_smem();  // generic writes precede the next TMA into this stage
      __syncwarp();
    }
    // q as the B operand: column 0 of a 16x8 tile per 16-dim chunk
    uint32_t qb[NK][2];
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      if (gq == 0) {
        qb[kk][0] = *reinterpret_cast<const uint32_t*>(hdr + (kk * 16 + 2 * qq) * 2);
        qb[kk][1] = *reinterpret_cast<const uint32_t*>(hdr + (kk * 16 + 2 * qq + 8) * 2);
      } else {
        qb[kk][0] = qb[kk][1] = 0u;
      }
    }
    // logits: lanes with qq == 0 own keys (gq) and (gq + 8) of each tile
    float sx[TILES][2];
    float pm = -INFINITY;
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      const int r0 = wrow0 + t * 16;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int lr = r0 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kbase + swz<D>(lr, kk * 2 + (lane >> 4)), a0, a1, a2, a3);
        mma_bf16(acc, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
      }
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int row = r0 + gq + 8 * h2;
        const int slot = slot0 + row;
        float x = -INFINITY;
        if (qq == 0 && slot < n) {
          const int mt = slot < L ? mpage[row] : (hc.pos | (hc.ncls << kClsShift));
          x = biased_logit(acc[2 * h2] * p.scale, mt, hc, hc.pos);
          if (hc.freq && slot < L) p.logit[hc.base + slot] = x;
        }
        sx[t][h2] = x;
        pm = fmaxf(pm, x);
      }
    }
    pm = warp_allreduce(pm, [](float a, float b) { return fmaxf(a, b); });
    const float m_new = fmaxf(m_run, pm);
    if (m_new != -INFINITY) {
      const float sc = (m_run == -INFINITY) ? 0.f : __expf(m_run - m_new);
      l_run *= sc;
#pragma unroll
      for (int t = 0; t < NK; ++t) {
        o[t][0] *= sc; o[t][1] *= sc; o[t][2] *= sc; o[t][3] *= sc;
      }
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        const int r0 = wrow0 + t * 16;
        // p in bf16 for the PV product, packed (key gq | key gq+8) on the
        // owning lanes; the softmax sum takes the fp32 values, so the lse the
        // score update divides by carries fp32 (not bf16) rounding
        const float e0 = sx[t][0] == -INFINITY ? 0.f : __expf(sx[t][0] - m_new);
        const float e1 = sx[t][1] == -INFINITY ? 0.f : __expf(sx[t][1] - m_new);
        const __nv_bfloat16 p0 = __float2bfloat16_rn(e0);
        const __nv_bfloat16 p1 = __float2bfloat16_rn(e1);
        if (qq == 0) l_run += e0 + e1;
        const uint32_t pk = (uint32_t)__bfloat16_as_ushort(p0) | ((uint32_t)__bfloat16_as_ushort(p1) << 16);
        const uint32_t u = __shfl_sync(0xffffffffu, pk, 8 * qq);      // keys 2qq, 2qq+8
        const uint32_t v = __shfl_sync(0xffffffffu, pk, 8 * qq + 4);  // keys 2qq+1, 2qq+9
        const uint32_t b0 = gq == 0 ? __byte_perm(u, v, 0x5410) : 0u;
        const uint32_t b1 = gq == 0 ? __byte_perm(u, v, 0x7632) : 0u;
        const bool partial = slot0 + r0 + 16 > n;  // rows past the live tail hold stale data
        const int lr = r0 + (lane >> 4) * 8 + (lane & 7);
#pragma unroll
        for (int tt = 0; tt < NK; ++tt) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(vbase + swz<D>(lr, tt * 2 + ((lane >> 3) & 1)), a0, a1, a2, a3);
          if (partial) {  // zero V of keys >= n (0 * NaN would poison the sum)
            const int k0 = slot0 + r0 + 2 * qq;
            const uint32_t m0 = (k0 < n ? 0xffffu : 0u) | (k0 + 1 < n ? 0xffff0000u : 0u);
            const uint32_t m8 = (k0 + 8 < n ? 0xffffu : 0u) | (k0 + 9 < n ? 0xffff0000u : 0u);
            a0 &= m0; a1 &= m0; a2 &= m8; a3 &= m8;
          }
          mma_bf16(o[tt], a0, a1, a2, a3, b0, b1);
        }
      }
      m_run = m_new;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);
    if (++stage == ST) { stage = 0; phase ^= 1; }

    if (!((pg + 1 == pend) || (pg + 1 == s_prefix[g + 1]))) continue;
    l_run = warp_allreduce(l_run, [](float a, float b) { return a + b; });
    if (p.consumer_tail && pg + 1 == pend) {
      // The CTA's last segment: publish it from the consumer warps - and,
      // if this CTA completes the head, run its combine and eviction
      // policy - in parallel with the epilogue warps finishing the previous
      // segments (that serialisation was the step's tail; measured:
      // FREQUENT-heavy c1_frequent 32.7 -> 29.5 us/step, headline c1
      // unchanged, T=0.99 with 16 FREQUENT heads 31.9 -> 33.2).  Every page
      // has been consumed, so stage 0 holds the handoff and policy scratch.
      // The split-K partials, semaphore, output and live counts belong to
      // the previous step until it completes: a chained step whose pages
      // all streamed early waits for it here (the head's other parts may
      // sit in CTAs whose producer never had to wait).
      if (early) grid_dep_wait();
      using CSync = NamedSync<NW * 32, 3, 0>;
      CSync::sync();  // all consumer warps are past the last page
      float(*red)[D] = reinterpret_cast<float(*)[D]>(smem);
      float(*mls)[2] = reinterpret_cast<float(*)[2]>(smem + NW * D * 4);
      int* scratch_i = reinterpret_cast<int*>(smem + NW * D * 4 + 64);
      if (qq == 0) {
#pragma unroll
        for (int tt = 0; tt < NK; ++tt) {
          red[warp][tt * 16 + gq] = o[tt][0];
          red[warp][tt * 16 + gq + 8] = o[tt][2];
        }
      }
      if (lane == 0) { mls[warp][0] = m_run; mls[warp][1] = l_run; }
      AKV_TRACE(3);
      publish_head<CSync, NW, D, true>(p, hc, s_prefix, P, grid, red, mls, scratch_i + 300,
                                       RB / 16, scratch_i, scratch_i + 256, nullptr);
      if (scratch_i[300] && p.trace && CSync::tid() == 0) {
        atomicAdd(&p.trace[blockIdx.x * 16 + 5], 1ull);               // epilogues run
        if (hc.freq) atomicAdd(&p.trace[blockIdx.x * 16 + 6], 1ull);  // frequent ones
      }
      return;
    }
    // hand the segment to the epilogue warps and keep streaming
    {
      const int slot = pub_n & 1;
      mbar_wait(&pub_empty[slot], ((pub_n >> 1) & 1) ^ 1);
      PubSlot<NW, D>& ps = s_pub[slot];
      if (qq == 0) {
#pragma unroll
        for (int tt = 0; tt < NK; ++tt) {
          ps.red[warp][tt * 16 + gq] = o[tt][0];
          ps.red[warp][tt * 16 + gq + 8] = o[tt][2];
        }
      }
      if (lane == 0) {
        ps.ml[warp][0] = m_run;
        ps.ml[warp][1] = l_run;
        if (warp == 0) ps.ctx = hc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pub_full[slot]);
      ++pub_n;
    }
    if (pg + 1 == pend) AKV_TRACE(3);
    m_run = -INFINITY;
    l_run = 0.f;
#pragma unroll
    for (int t = 0; t < NK; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  }
}

// ===========================================================================
// Tuning knobs read from the environment once per process (thread-safe
// static initialisation).
static int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}
// Decode grid: AKV_K3_GRID CTAs if set (tuning), else 2 per SM
static int k3_grid(int sms) {
  static const int v = env_int("AKV_K3_GRID", 0);
  return v > 0 ? v : 2 * sms;
}
unsigned long long* g_dec_trace = nullptr;  // set by akv_debug_set_decode_trace
int g_dec_trace_ring = 1;                    // consecutive steps to keep apart (trace ring)
// consumers publish the CTA's last segment (AKV_K3_CONSUMER_TAIL, tuning)
static int k3_consumer_tail() {
  static const int v = env_int("AKV_K3_CONSUMER_TAIL", 1) != 0;
  return v;
}
// pages of L2 prefetch ahead of the ring (AKV_K3_L2_PREFETCH, tuning)
static int k3_l2_prefetch() {
  // measured at config 1: 0 best (2: +0.6 us, 4: +1.4, 8: +4.1)
  static const int v = env_int("AKV_K3_L2_PREFETCH", 0) > 0 ? env_int("AKV_K3_L2_PREFETCH", 0) : 0;
  return v;
}

static std::atomic<int> g_num_sms[kMaxDevices];

}  // namespace akv

cudaError_t akv::current_sm_count(int* out) {
  int dev;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev))) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  int v = g_num_sms[dev].load(std::memory_order_relaxed);
  if (!v) {
    if ((e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev))) return e;
    g_num_sms[dev].store(v, std::memory_order_relaxed);
  }
  *out = v;
  return cudaSuccess;
}

namespace akv {

static cudaError_t num_sms(int* out) { return current_sm_count(out); }

// Launch with programmatic dependent launch: the next step's CTAs start
// their prologue while this step drains (griddepcontrol in the kernels).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename T, int D>
static cudaError_t launch_simt(const DecParams& p, cudaStream_t st) {
  using S = SimtShape<T, D>;
  auto kern = k3_decode_simt<T, D>;
  static PerDeviceOnce attr;
  cudaError_t e = attr.run([&](int) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kStages * S::STAGE_B + (2 * kMaxHeads + 1) * 4));
  });
  if (e != cudaSuccess) return e;
  int sms;
  if ((e = num_sms(&sms))) return e;
  const size_t smem = (size_t)kStages * S::STAGE_B + (size_t)(2 * p.G + 1) * 4;
  return launch_pdl(kern, k3_grid(sms), S::NW * 32 + 32, smem, st, p);
}

// tensor maps of the arena, cached per (base, slots) so steady-state steps
// (and CUDA-graph capture) do no host-side encoding
struct TmapCache {
  const void* kc = nullptr;
  const void* vc = nullptr;
  int64_t slots = -1;
  int d = 0;
  CUtensorMap k, v;
};
constexpr int kTmapSlots = 256;  // one per (layer) cache of a multi-layer model
static thread_local TmapCache g_tmap_slots[kTmapSlots];
static thread_local int g_tmap_next = 0;

static TmapCache* tmap_lookup(const void* kc, const void* vc, int64_t slots, int d) {
  for (int i = 0; i < kTmapSlots; ++i) {
    TmapCache& c = g_tmap_slots[i];
    if (c.kc == kc && c.vc == vc && c.slots == slots && c.d == d) return &c;
  }
  return nullptr;
}

template <int D>
static cudaError_t launch_mma(const DecParams& p, int64_t total_slots, cudaStream_t st) {
  using S = MmaShape<D>;
  TmapCache* tm = tmap_lookup(p.kc, p.vc, total_slots, D);
  if (!tm) {
    tm = &g_tmap_slots[g_tmap_next];
    g_tmap_next = (g_tmap_next + 1) % kTmapSlots;
    tm->kc = nullptr;
    if (!encode_tmap_2d_bf16(&tm->k, p.kc, (uint64_t)total_slots, D, 64, S::PAGE, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_tmap_2d_bf16(&tm->v, p.vc, (uint64_t)total_slots, D, 64, S::PAGE, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    tm->kc = p.kc; tm->vc = p.vc; tm->slots = total_slots; tm->d = D;
  }
  auto k3 = k3_decode_mma<D, 3>;
  auto k2 = k3_decode_mma<D, 2>;
  const size_t plan = (size_t)(2 * kMaxHeads + 1) * 4 + kMaxHeads;
  // per-device launch facts: the attribute opt-ins and the shared-memory
  // budget that decides whether a 3-stage ring keeps two CTAs per SM
  struct Facts { size_t static3, per_sm, reserve; };
  static Facts facts[kMaxDevices];
  static PerDeviceOnce attr;
  cudaError_t e = attr.run([&](int dev) {
    cudaError_t r;
    if ((r = cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 + 3 * S::STAGE_B + plan))) ||
        (r = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 + 2 * S::STAGE_B + plan))))
      return r;
    cudaFuncAttributes fa;
    if ((r = cudaFuncGetAttributes(&fa, k3))) return r;
    Facts f;
    f.static3 = fa.sharedSizeBytes;
    int v = 0;
    if ((r = cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev))) return r;
    f.per_sm = (size_t)v;
    if ((r = cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, dev))) return r;
    f.reserve = (size_t)v;
    facts[dev] = f;
    return cudaSuccess;
  });
  if (e != cudaSuccess) return e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev))) return e;
  const Facts& f = facts[dev];
  int sms;
  if ((e = num_sms(&sms))) return e;
  const size_t plan_g = (size_t)(2 * p.G + 1) * 4 + p.G;
  const size_t smem3 = 1024 + (size_t)3 * S::STAGE_B + plan_g;
  // Two ring stages by default: measured at least as fast as three at every
  // size (c1 29.44 -> 29.26 us/step; B*H 128..512 likewise) and they keep two
  // CTAs per SM up to 2048 heads per launch, where a 3-stage ring drops to
  // one CTA per SM beyond 512 heads (3.5 vs 5.9 TB/s).  AKV_K3_STAGES=3
  // selects the 3-stage ring where two CTAs still fit (tuning).
  static const int stages = env_int("AKV_K3_STAGES", 2);
  if (stages == 3 && 2 * (smem3 + f.static3 + f.reserve) <= f.per_sm)
    return launch_pdl(k3, k3_grid(sms), S::THREADS, smem3, st, p, tm->k, tm->v);
  const size_t smem2 = 1024 + (size_t)2 * S::STAGE_B + plan_g;
  return launch_pdl(k2, k3_grid(sms), S::THREADS, smem2, st, p, tm->k, tm->v);
}

struct DecWs {
  float* part;
  float* logit;
  int32_t* counter;
  int32_t* status;
  size_t bytes;
  int max_parts;
};

// partial slots per head: one per contributing CTA, bounded by the head's
// page count (smallest page over dtypes for this head dim: fp32 rows)
static inline int max_parts_for(int d, int max_cap) {
  const int page = kPageBytes / (d * 4);
  return (max_cap + page - 1) / page + 1;
}

static DecWs carve(void* ws, int B, int H, int d, int max_cap, int64_t total_slots) {
  DecWs w;
  const int G = B * H;
  w.max_parts = max_parts_for(d, max_cap);
  char* c = static_cast<char*>(ws);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = c + off; off += (bytes + 255) & ~size_t(255); return r; };
  w.counter = reinterpret_cast<int32_t*>(take((size_t)G * 4));
  w.status = reinterpret_cast<int32_t*>(take(4));
  w.part = reinterpret_cast<float*>(take((size_t)G * w.max_parts * (d + 2) * 4));
  w.logit = reinterpret_cast<float*>(take((size_t)total_slots * 4));
  w.bytes = off;
  return w;
}

}  // namespace akv

using namespace akv;

// Debug hook (not part of the ABI header): record per-CTA timestamps of
// the next decode launches into a device buffer of [2*SMs, 16] uint64.
extern "C" void akv_debug_set_decode_trace(void* buf) {
  g_dec_trace = static_cast<unsigned long long*>(buf);
  g_dec_trace_ring = 1;
}

// The same, for n consecutive steps kept apart: step s records into block
// (s mod n) of a buffer of n x [2*SMs, 16] uint64 (decode_steps runs).
extern "C" void akv_debug_set_decode_trace_ring(void* buf, int n) {
  g_dec_trace = static_cast<unsigned long long*>(buf);
  g_dec_trace_ring = n > 1 ? n : 1;
}

extern "C" size_t akv_decode_workspace_size(int32_t B, int32_t H, int32_t d, int32_t max_cap,
                                           int64_t total_slots) {
  return carve(nullptr, B, H, d, max_cap, total_slots).bytes;
}

extern "C" int akv_decode_workspace_init(void* ws, size_t bytes, int32_t B, int32_t H, int32_t d,
                                         int32_t max_cap, int64_t total_slots, void* stream) {
  DecWs w = carve(ws, B, H, d, max_cap, total_slots);
  if (bytes < w.bytes) return set_error(AKV_ERR_CAPACITY, "akv_decode_workspace_init: workspace too small");
  cudaError_t e = cudaMemsetAsync(ws, 0, reinterpret_cast<char*>(w.part) - static_cast<char*>(ws),
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_workspace_init: %s", cudaGetErrorString(e));
  return AKV_OK;
}

static unsigned long long* trace_for(const akv_decode_args* a) {
  if (!g_dec_trace) return nullptr;
  int sms = 0;
  if (current_sm_count(&sms) != cudaSuccess) return nullptr;
  // the trace buffers hold [2*SMs, 16] stamps: a larger grid (AKV_K3_GRID) is not traced
  if (k3_grid(sms) > 2 * sms) return nullptr;
  if (g_dec_trace_ring <= 1) return g_dec_trace;
  const int slot = (a->pos - a->prompt_len) % g_dec_trace_ring;
  return g_dec_trace + (size_t)slot * 2 * sms * 16;
}

extern "C" int akv_decode_step(const akv_decode_args* a, void* stream) {
  if (!a) return set_error(AKV_ERR_INVALID, "akv_decode_step: null args");
  if (a->B < 1 || a->H < 1) return set_error(AKV_ERR_INVALID, "akv_decode_step: empty input");
  if (a->H > kMaxHeads)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_step: more than %d heads per batch row", kMaxHeads);
  if ((!a->pos_dev && a->pos < a->prompt_len) || a->prompt_len < 1)
    return set_error(AKV_ERR_INVALID, "akv_decode_step: need pos >= prompt_len >= 1");
  if (a->pos_dev && (a->flags & AKV_DECODE_CHAINED))
    return set_error(AKV_ERR_INVALID, "akv_decode_step: AKV_DECODE_CHAINED needs a host position");
  if (a->pos > kPosMask) return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_step: position too large");
  if (a->live_in_dev == a->live_out_dev)
    return set_error(AKV_ERR_INVALID, "akv_decode_step: live_in and live_out must be distinct buffers");
  if (a->bh_stride < a->d) return set_error(AKV_ERR_INVALID, "akv_decode_step: bh_stride < d");
  if (a->n_peers < 0 || (a->n_peers > 0 && (!a->peer_out_dev || a->peer_ld < a->peer_col0 +
                                                                    (int64_t)a->H * a->d)))
    return set_error(AKV_ERR_INVALID, "akv_decode_step: bad peer output (n_peers %d, ld %lld)",
                     a->n_peers, (long long)a->peer_ld);
  DecWs w = carve(a->workspace_dev, a->B, a->H, a->d, a->max_cap, a->total_slots);
  if (a->workspace_bytes < w.bytes) return set_error(AKV_ERR_CAPACITY, "akv_decode_step: workspace too small");
  const float scale = (float)(1.0 / sqrt((double)a->d));
  const size_t es = a->dtype == AKV_DTYPE_BF16 ? 2 : 4;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  bool ok = true;
  // Heads are independent: batches beyond kMaxHeads heads per launch (the
  // page plan lives in shared memory) run as consecutive launches over
  // whole batch rows.  Each launch depends programmatically only on the one
  // before it, and every launch's CTAs wait for their predecessor before
  // signalling, so the chained-step invariant (only the immediately
  // preceding launch may still be writing) holds for every chunk.
  const int rows_per = kMaxHeads / a->H;
  for (int b0 = 0; b0 < a->B && ok && e == cudaSuccess; b0 += rows_per) {
    const int nb = min(rows_per, a->B - b0);
    const int64_t g0 = (int64_t)b0 * a->H;
    const int64_t qoff = g0 * a->bh_stride * (int64_t)es;
    auto at = [&](auto* ptr, int64_t n) { return ptr ? ptr + n : ptr; };
    DecParams p{nb, a->H, nb * a->H, a->prompt_len, a->pos,
                static_cast<const char*>(a->q_dev) + qoff, static_cast<const char*>(a->k_dev) + qoff,
                static_cast<const char*>(a->v_dev) + qoff, a->bh_stride, a->new_cls_dev + b0,
                a->slope_dev, a->sink_dev, a->head_atoms_dev + g0, a->head_r_l_dev + g0,
                a->head_r_f_dev + g0, a->seg_off_dev + g0, a->seg_cap_dev + g0, a->kc_dev, a->vc_dev,
                a->meta_dev, a->score_dev, a->base_live_dev + g0, a->live_in_dev + g0,
                a->live_out_dev + g0, a->out_dev + g0 * a->d, at(a->evicted_dev, g0),
                a->status_dev ? a->status_dev : w.status,
                w.part + g0 * w.max_parts * (a->d + 2), w.logit, w.counter + g0, w.max_parts, scale,
                trace_for(a), a->pos_dev, a->flags, at(a->lse_out_dev, g0), a->peer_out_dev,
                a->n_peers, a->peer_ld, a->peer_col0 + (int64_t)b0 * a->peer_ld,
                a->dtype == AKV_DTYPE_BF16, k3_l2_prefetch(), k3_consumer_tail()};
    if (a->dtype == AKV_DTYPE_BF16) {
      switch (a->d) {
        case 16: e = launch_simt<__nv_bfloat16, 16>(p, st); break;
        case 32: e = launch_simt<__nv_bfloat16, 32>(p, st); break;
        case 64: e = g_disable_tc ? launch_simt<__nv_bfloat16, 64>(p, st) : launch_mma<64>(p, a->total_slots, st); break;
        case 128: e = g_disable_tc ? launch_simt<__nv_bfloat16, 128>(p, st) : launch_mma<128>(p, a->total_slots, st); break;
        default: ok = false;
      }
    } else if (a->dtype == AKV_DTYPE_F32) {
      switch (a->d) {
        case 16: e = launch_simt<float, 16>(p, st); break;
        case 32: e = launch_simt<float, 32>(p, st); break;
        case 64: e = launch_simt<float, 64>(p, st); break;
        case 128: e = launch_simt<float, 128>(p, st); break;
        default: ok = false;
      }
    } else {
      ok = false;
    }
  }
  if (!ok) return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_step: unsupported dtype %d / head dim %d", a->dtype, a->d);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_step: %s", cudaGetErrorString(e));
  return AKV_OK;
}

// n consecutive teacher-forced decode steps in one call (the host loop in
// C++: a launch costs ~2-3 us of host time instead of a Python call's
// ~10-13 us, which bounds small batches).  Step s inserts position pos + s,
// reads q/k/v at q_dev/k_dev/v_dev + s*step_stride elements and the classes
// at new_cls_dev + s*cls_step_stride; the live counts alternate between
// live_in_dev and live_out_dev (after the call they are in live_out_dev for
// odd n, live_in_dev for even n); step s writes its output to
// out_steps + s*out_step_stride, or to out_dev when out_steps is NULL.
// `flags` apply to step 0; later steps are chained (their predecessor is the
// previous step and their inputs were resident before the call).
extern "C" int akv_decode_steps(const akv_decode_args* a, int32_t n_steps, int64_t step_stride,
                                int64_t cls_step_stride, float* out_steps, int64_t out_step_stride,
                                void* stream) {
  if (!a) return set_error(AKV_ERR_INVALID, "akv_decode_steps: null args");
  if (n_steps < 0) return set_error(AKV_ERR_INVALID, "akv_decode_steps: n_steps < 0");
  if (a->pos_dev) return set_error(AKV_ERR_INVALID, "akv_decode_steps: needs host positions (pos_dev is set)");
  const size_t es = a->dtype == AKV_DTYPE_BF16 ? 2 : 4;
  akv_decode_args s = *a;
  for (int i = 0; i < n_steps; ++i) {
    s.pos = a->pos + i;
    s.q_dev = static_cast<const char*>(a->q_dev) + (int64_t)i * step_stride * (int64_t)es;
    s.k_dev = static_cast<const char*>(a->k_dev) + (int64_t)i * step_stride * (int64_t)es;
    s.v_dev = static_cast<const char*>(a->v_dev) + (int64_t)i * step_stride * (int64_t)es;
    s.new_cls_dev = a->new_cls_dev + (int64_t)i * cls_step_stride;
    s.live_in_dev = (i & 1) ? a->live_out_dev : a->live_in_dev;
    s.live_out_dev = (i & 1) ? const_cast<int32_t*>(a->live_in_dev) : a->live_out_dev;
    s.out_dev = out_steps ? out_steps + (int64_t)i * out_step_stride : a->out_dev;
    s.flags = i == 0 ? a->flags : (a->flags | AKV_DECODE_CHAINED);
    const int rc = akv_decode_step(&s, stream);
    if (rc != AKV_OK) return rc;
  }
  return AKV_OK;
}
