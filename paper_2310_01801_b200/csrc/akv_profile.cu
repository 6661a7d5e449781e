// K1: prompt profiling for FastGen's adaptive KV cache (sm_100a).
//
// Replaces, per head, the reference's
//   engine.py:161-200  prompt_head_data: causal_attention + A.sum(axis=0)
//   attention.py:102-127 causal_attention (logits q.k/sqrt(d), causal softmax)
//   profiler.py:70-87   recovery_ratio    (= sum_{j in S} colsum_j / N)
//   profiler.py:135-145 select_policy     (first family member with R >= T)
//   profiler.py:148-178 cosine selector   (||A[:,S]||_F / ||A||_F)
//   policies.py:214-267 retained_indices  (union of atom position sets)
//   engine.py:248,255   pending_output = A[N-1] @ V
// without ever materialising A:
//   pass 1 (query-major) computes the row log-sum-exp,
//   pass 2 (key-major, recompute) accumulates per-key attention mass
//   colsum_j = sum_i exp(s_ij - lse_i), its square sum, the last row and the
//   last row's output partials;
//   the policy epilogue runs the exact top-k and the family search per head.
// This file holds the SIMT (FFMA) passes used for fp32 inputs and any head
// dim; bf16 d=128 prompts take the tcgen05 passes in akv_profile_tc.cu.

#include <math.h>
#include <stdio.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kTile = 64;      // query and key tile edge
constexpr int kThreads = 256;  // 16 x 16 threads, 4x4 logits each

struct ProfParams {
  int B, H, N;
  const void* q;
  const void* k;
  const void* v;
  int64_t ld;
  const uint8_t* cls;
  int64_t cls_ld;
  const float* slope;
  const float* sink;
  float scale;  // 1/sqrt(d)
  float* lse;
  double* colsum;
  double* colsq;
  float* lastp;
  float* out_part;  // [G, ntiles, d]
};

// Load a 64-row tile of a [rows, D] head matrix into smem transposed
// (dst[c*kTile + r]) as fp32, scaled.  Rows >= n are zero.
template <typename T, int D>
__device__ __forceinline__ void load_tile_T(float* dst, const T* src, int row0, int n, float scale) {
  constexpr int EV = Elem<T>::kPerVec;
  constexpr int NV = D / EV;  // vectors per row
  // thread -> (row r = idx % 64, vec = idx / 64): a warp covers 32 rows of
  // one column group, so the transposed smem stores are conflict-free.
  for (int idx = threadIdx.x; idx < kTile * NV; idx += blockDim.x) {
    const int r = idx % kTile, vg = idx / kTile;
    const int row = row0 + r;
    float f[EV];
    if (row < n) {
      uint4 u = *reinterpret_cast<const uint4*>(src + (size_t)row * D + vg * EV);
      Elem<T>::unpack(u, f);
    } else {
#pragma unroll
      for (int e = 0; e < EV; ++e) f[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < EV; ++e) dst[(vg * EV + e) * kTile + r] = f[e] * scale;
  }
}

template <int D>
__device__ __forceinline__ void tile_dot(const float* Qs, const float* Ks, int r0, int j0,
                                         float s[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
  for (int c = 0; c < D; ++c) {
    const float4 a = *reinterpret_cast<const float4*>(Qs + c * kTile + r0);
    const float4 b = *reinterpret_cast<const float4*>(Ks + c * kTile + j0);
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = fmaf(av[i], bv[j], s[i][j]);
  }
}

// Pass 1: row log-sum-exp.  grid (ntiles, G), 256 threads.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) k1_rowlse(ProfParams p) {
  extern __shared__ __align__(16) float smem[];
  float* Qs = smem;
  float* Ks = smem + D * kTile;
  __shared__ float s_sinkbias[kTile];
  const int g = blockIdx.y, qt = blockIdx.x;
  const int b = g / p.H, h = g % p.H;
  const T* qh = static_cast<const T*>(p.q) + (size_t)g * p.ld * D;
  const T* kh = static_cast<const T*>(p.k) + (size_t)g * p.ld * D;
  const uint8_t* cls = p.cls + (size_t)b * p.cls_ld;
  const float slope = p.slope ? p.slope[h] : 0.f;
  const float sink = p.sink ? p.sink[h] : 0.f;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = ty * 4, j0 = tx * 4;

  load_tile_T<T, D>(Qs, qh, qt * kTile, p.N, p.scale);
  float m[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { m[i] = -INFINITY; l[i] = 0.f; }

  for (int kt = 0; kt <= qt; ++kt) {
    __syncthreads();
    load_tile_T<T, D>(Ks, kh, kt * kTile, p.N, 1.f);
    if (threadIdx.x < kTile) {
      const int col = kt * kTile + threadIdx.x;
      s_sinkbias[threadIdx.x] = (col < p.N && cls[col] == AKV_CLS_SPECIAL) ? sink : 0.f;
    }
    __syncthreads();
    float s[4][4];
    tile_dot<D>(Qs, Ks, r0, j0, s);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = qt * kTile + r0 + i;
      float tmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = kt * kTile + j0 + j;
        float x = s[i][j] + s_sinkbias[j0 + j];
        if (slope != 0.f) x -= slope * (float)(row - col);
        x = (col <= row && row < p.N) ? x : -INFINITY;
        s[i][j] = x;
        tmax = fmaxf(tmax, x);
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      const float mnew = fmaxf(m[i], tmax);
      float sum = 0.f;
      if (mnew != -INFINITY) {
#pragma unroll
        for (int j = 0; j < 4; ++j) sum += (s[i][j] == -INFINITY) ? 0.f : expf(s[i][j] - mnew);
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (mnew != -INFINITY) {
        l[i] = (m[i] == -INFINITY ? 0.f : l[i] * expf(m[i] - mnew)) + sum;
        m[i] = mnew;
      }
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = qt * kTile + r0 + i;
      if (row < p.N) p.lse[(size_t)g * p.N + row] = m[i] + logf(l[i]);
    }
  }
}

// Pass 2: per-key attention mass.  grid (ntiles, G), 256 threads.  Key tile
// 0 carries the most query tiles; blocks are dispatched in blockIdx order,
// so the heaviest tiles start first.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) k1_colsum(ProfParams p) {
  extern __shared__ __align__(16) float smem[];
  float* Qs = smem;
  float* Ks = smem + D * kTile;
  __shared__ float s_sinkbias[kTile];
  __shared__ float s_lse[kTile];
  __shared__ float s_lastp[kTile];
  __shared__ double s_red[16][kTile];
  const int ntiles = (p.N + kTile - 1) / kTile;
  const int g = blockIdx.y, kt = blockIdx.x;
  const int b = g / p.H, h = g % p.H;
  const T* qh = static_cast<const T*>(p.q) + (size_t)g * p.ld * D;
  const T* kh = static_cast<const T*>(p.k) + (size_t)g * p.ld * D;
  const T* vh = static_cast<const T*>(p.v) + (size_t)g * p.ld * D;
  const uint8_t* cls = p.cls + (size_t)b * p.cls_ld;
  const float slope = p.slope ? p.slope[h] : 0.f;
  const float sink = p.sink ? p.sink[h] : 0.f;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = ty * 4, j0 = tx * 4;

  load_tile_T<T, D>(Ks, kh, kt * kTile, p.N, 1.f);
  if (threadIdx.x < kTile) {
    const int col = kt * kTile + threadIdx.x;
    s_sinkbias[threadIdx.x] = (col < p.N && cls[col] == AKV_CLS_SPECIAL) ? sink : 0.f;
    s_lastp[threadIdx.x] = 0.f;
  }
  double acc[4] = {0, 0, 0, 0}, accsq[4] = {0, 0, 0, 0};
  for (int qt = kt; qt < ntiles; ++qt) {
    __syncthreads();
    load_tile_T<T, D>(Qs, qh, qt * kTile, p.N, p.scale);
    if (threadIdx.x < kTile) {
      const int row = qt * kTile + threadIdx.x;
      s_lse[threadIdx.x] = row < p.N ? p.lse[(size_t)g * p.N + row] : 0.f;
    }
    __syncthreads();
    float s[4][4];
    tile_dot<D>(Qs, Ks, r0, j0, s);
    float ps[4] = {0, 0, 0, 0}, pq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = qt * kTile + r0 + i;
      const float lse = s_lse[r0 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = kt * kTile + j0 + j;
        float x = s[i][j] + s_sinkbias[j0 + j];
        if (slope != 0.f) x -= slope * (float)(row - col);
        const float pr = (col <= row && row < p.N && col < p.N) ? expf(x - lse) : 0.f;
        ps[j] += pr;
        pq[j] = fmaf(pr, pr, pq[j]);
        if (row == p.N - 1 && col < p.N) s_lastp[j0 + j] = pr;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[j] += (double)ps[j]; accsq[j] += (double)pq[j]; }
  }
  // reduce over the 16 row groups (fixed order -> deterministic)
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) s_red[ty][j0 + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < kTile) {
    double t = 0.0;
    for (int i = 0; i < 16; ++i) t += s_red[i][threadIdx.x];
    const int col = kt * kTile + threadIdx.x;
    if (col < p.N) {
      p.colsum[(size_t)g * p.N + col] = t;
      p.lastp[(size_t)g * p.N + col] = s_lastp[threadIdx.x];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) s_red[ty][j0 + j] = accsq[j];
  __syncthreads();
  if (threadIdx.x < kTile) {
    double t = 0.0;
    for (int i = 0; i < 16; ++i) t += s_red[i][threadIdx.x];
    const int col = kt * kTile + threadIdx.x;
    if (col < p.N) p.colsq[(size_t)g * p.N + col] = t;
  }
  // last-row output partial over this key tile: sum_j lastp_j V_j
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float o = 0.f;
    const int nj = min(kTile, p.N - kt * kTile);
    for (int j = 0; j < nj; ++j)
      o = fmaf(s_lastp[j], Elem<T>::to_f(vh[(size_t)(kt * kTile + j) * D + c]), o);
    p.out_part[((size_t)g * ntiles + kt) * D + c] = o;
  }
}

// ---------------------------------------------------------------------------
// Policy epilogue: one CTA per head.
struct PolicyParams {
  int B, H, N, d;
  int ntiles;  // out_last partials per head
  const uint8_t* cls;
  int64_t cls_ld;
  const double* colsum;
  const double* colsq;
  const float* lastp;
  const float* out_part;
  int n_family;
  uint8_t atoms[AKV_MAX_FAMILY];
  double r_l[AKV_MAX_FAMILY];
  double r_f[AKV_MAX_FAMILY];
  int n_thr;
  double thr[AKV_MAX_THRESHOLDS];
  int rows, criterion;
  int local_len;  // prompt length anchoring the local budget (policies.py:209-211)
  float* out_last;
  double* recovery;
  int32_t* cost;
  double* cosine;
  int8_t* choice;
  int32_t* kept_pos;
  int32_t* kept_count;
  double* last_row_recovery;
  double* topk_gap;
  unsigned long long* thr_key;
  int32_t* thr_pos;
};

constexpr int kPolicyThreads = 512;
#ifdef AKV_TRACE_POL
__device__ unsigned long long g_pol_trace[4096][8];
#define POL_STAMP(i) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_pol_trace[blockIdx.x][i] = clock64(); } while (0)
extern "C" int akv_debug_pol_trace(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_pol_trace, sizeof(g_pol_trace));
}
#else
#define POL_STAMP(i) do {} while (0)
#endif
// per-key bytes staged in shared memory (score key, colsq, lastp, class) and
// the largest prompt staged; longer prompts read the global arrays
constexpr int kPolicyStageBytes = 8 + 8 + 4 + 1;
constexpr int kPolicyStageMaxN = 7680;

// One CTA per head.  The head's per-key inputs are staged in shared memory
// once, so the top-k radix passes and the member passes touch no global
// memory; every family member's recovery, cost and cosine come from ONE pass
// over the keys with per-member register accumulators and one combined
// reduction (the per-thread strided sums and the warp-tree / warp-order
// combine are those of block_sum, so the results are unchanged bit for bit).
__global__ void __launch_bounds__(kPolicyThreads, 2) k1_policy(PolicyParams p) {
  extern __shared__ __align__(16) uint8_t s_stage[];
  __shared__ int hist[256];
  __shared__ int red_i[33];
  __shared__ double red_d[kPolicyThreads / 32];
  __shared__ unsigned long long s_thr_key[AKV_MAX_FAMILY];
  __shared__ int s_thr_pos[AKV_MAX_FAMILY];
  __shared__ int s_loc[AKV_MAX_FAMILY];
  __shared__ int s_choice[AKV_MAX_THRESHOLDS];
  __shared__ double s_rs[kPolicyThreads / 32][AKV_MAX_FAMILY + 1], s_qs[kPolicyThreads / 32][AKV_MAX_FAMILY];
  __shared__ int s_cn[kPolicyThreads / 32][AKV_MAX_FAMILY];
  __shared__ double s_R[AKV_MAX_FAMILY], s_cs[AKV_MAX_FAMILY];
  // launched programmatically after the tensor-core passes: their outputs
  // are complete past this point (a no-op after an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int g = blockIdx.x;
  const int b = g / p.H;
  const int N = p.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWP = kPolicyThreads / 32;
  const uint8_t* cls_g = p.cls + (size_t)b * p.cls_ld;
  const double* colsum_g = p.colsum + (size_t)g * N;
  const double* colsq_g = p.colsq + (size_t)g * N;
  const float* lastp_g = p.lastp + (size_t)g * N;
  const bool staged = N <= kPolicyStageMaxN;
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_stage);
  double* s_sq = reinterpret_cast<double*>(s_key + N);
  float* s_lp = reinterpret_cast<float*>(s_sq + N);
  uint8_t* s_cls = reinterpret_cast<uint8_t*>(s_lp + N);
  POL_STAMP(0);
  if (staged) {
    for (int j = tid; j < N; j += kPolicyThreads) {
      s_key[j] = score_key(colsum_g[j]);
      s_sq[j] = colsq_g[j];
      s_lp[j] = lastp_g[j];
      s_cls[j] = cls_g[j];
    }
  }
  if (tid < p.n_family) s_loc[tid] = N - budget(p.r_l[tid], p.local_len);
  __syncthreads();
  POL_STAMP(1);
  auto key_at = [&](int j) { return staged ? s_key[j] : score_key(colsum_g[j]); };
  auto sq_at = [&](int j) { return staged ? s_sq[j] : colsq_g[j]; };
  auto lp_at = [&](int j) { return staged ? s_lp[j] : lastp_g[j]; };
  auto cls_at = [&](int j) { return staged ? (int)s_cls[j] : (int)cls_g[j]; };
  // the staged key is the score with -0.0 folded onto +0.0: the same sums
  auto cs_at = [&](int j) { return staged ? __longlong_as_double((long long)s_key[j]) : colsum_g[j]; };

  auto get = [&](int i, unsigned long long* key, int* pos) {
    *key = key_at(i);
    *pos = i;
  };
  // exact frequent top-k thresholds (one per member with FREQUENT), and the
  // min relative gap at each boundary (k-th vs (k+1)-th largest score)
  // One radix select per distinct frequent budget (members sharing r_f share
  // the threshold); the (k+1)-th largest key for the gap is the largest key
  // outside the selected set - a block max, not a second select.
  __shared__ unsigned long long s_next[NWP];
  double min_gap = INFINITY;
  int have = -1;  // a member whose threshold is already in s_thr_*
  for (int f = 0; f < p.n_family; ++f) {
    if (!(p.atoms[f] & AKV_ATOM_FREQUENT) || (p.atoms[f] & AKV_ATOM_FULL)) continue;
    if (have >= 0 && p.r_f[have] == p.r_f[f]) {
      if (tid == 0) { s_thr_key[f] = s_thr_key[have]; s_thr_pos[f] = s_thr_pos[have]; }
      __syncthreads();
      continue;
    }
    const int kb = budget(p.r_f[f], N);
    unsigned long long tk; int tp;
    block_topk_threshold(N, kb, get, hist, red_i, &tk, &tp);
    if (tid == 0) { s_thr_key[f] = tk; s_thr_pos[f] = tp; }
    if (kb < N) {
      unsigned long long nk = 0ull;
      for (int j = tid; j < N; j += kPolicyThreads) {
        const unsigned long long key = key_at(j);
        if (!topk_selected(key, j, tk, tp) && key > nk) nk = key;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, nk, o);
        nk = other > nk ? other : nk;
      }
      if (lane == 0) s_next[warp] = nk;
      __syncthreads();
      nk = 0ull;
      for (int w = 0; w < NWP; ++w) nk = s_next[w] > nk ? s_next[w] : nk;
      const double a = __longlong_as_double(tk), c = __longlong_as_double(nk);
      const double gap = a > 0.0 ? (a - c) / a : 0.0;
      min_gap = fmin(min_gap, gap);
    }
    have = f;
    __syncthreads();
  }
  __syncthreads();

  POL_STAMP(2);
  auto kept = [&](int f, int j, unsigned long long key, int c) -> bool {
    const uint8_t at = p.atoms[f];
    if (at & AKV_ATOM_FULL) return true;
    bool k = ((at & AKV_ATOM_SPECIAL) && c == AKV_CLS_SPECIAL) ||
             ((at & AKV_ATOM_PUNCT) && c == AKV_CLS_PUNCT);
    if (at & AKV_ATOM_LOCAL) k |= j >= s_loc[f];
    if (at & AKV_ATOM_FREQUENT) k |= topk_selected(key, j, s_thr_key[f], s_thr_pos[f]);
    return k;
  };

  // every member's kept mass (colsum or last row), colsq mass and count, and
  // the colsq total for the cosine criterion: per member one pass over the
  // staged keys and a warp reduction, then ONE block barrier for them all
  {
    const bool last = p.rows == AKV_ROWS_LAST;
    double tot = 0.0;
    for (int j = tid; j < N; j += kPolicyThreads) tot += sq_at(j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) s_rs[warp][AKV_MAX_FAMILY] = tot;
    for (int f = 0; f < p.n_family; ++f) {
      double rs = 0.0, qs = 0.0;
      int cn = 0;
      for (int j = tid; j < N; j += kPolicyThreads) {
        if (kept(f, j, key_at(j), cls_at(j))) {
          rs += last ? (double)lp_at(j) : cs_at(j);
          qs += sq_at(j);
          ++cn;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rs += __shfl_xor_sync(0xffffffffu, rs, o);
        qs += __shfl_xor_sync(0xffffffffu, qs, o);
        cn += __shfl_xor_sync(0xffffffffu, cn, o);
      }
      if (lane == 0) { s_rs[warp][f] = rs; s_qs[warp][f] = qs; s_cn[warp][f] = cn; }
    }
    __syncthreads();
    if (tid < p.n_family) {
      const int f = tid;
      double rsum = 0.0, qsum = 0.0, tot_sq = 0.0;
      int cnt = 0;
      for (int w = 0; w < NWP; ++w) {
        rsum += s_rs[w][f];
        qsum += s_qs[w][f];
        cnt += s_cn[w][f];
        tot_sq += s_rs[w][AKV_MAX_FAMILY];
      }
      double R;
      if (p.atoms[f] & AKV_ATOM_FULL) R = 1.0;  // A's rows sum to 1 exactly
      else if (cnt == 0) R = 0.0;               // profiler.py:82-83
      else R = last ? rsum : rsum / (double)N;
      p.recovery[(size_t)g * p.n_family + f] = R;
      s_R[f] = R;
      p.cost[(size_t)g * p.n_family + f] = cnt;
      const double cs = (p.atoms[f] & AKV_ATOM_FULL) ? 1.0 : (qsum == 0.0 ? 0.0 : sqrt(qsum) / sqrt(tot_sq));
      p.cosine[(size_t)g * p.n_family + f] = cs;
      s_cs[f] = cs;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double* R = s_R;  // this block's values: no global round trip per member
    const double* cs = s_cs;
    for (int t = 0; t < p.n_thr; ++t) {
      int c = -1;
      if (p.criterion == AKV_CRIT_COSINE) {
        double best = -1.0;
        for (int f = 0; f < p.n_family; ++f)
          if (cs[f] > best) { best = cs[f]; c = f; }  // strict >, profiler.py:176
      } else {
        for (int f = 0; f < p.n_family; ++f)
          if (R[f] >= p.thr[t]) { c = f; break; }   // profiler.py:142
      }
      s_choice[t] = c;
      p.choice[(size_t)g * p.n_thr + t] = (int8_t)c;
    }
    p.topk_gap[g] = min_gap;
  }
  __syncthreads();
  POL_STAMP(3);
  const int f0 = s_choice[0];
  // ordered kept positions of the primary choice: each thread owns a
  // contiguous range of positions
  const int per = (N + kPolicyThreads - 1) / kPolicyThreads;
  const int lo = min(N, tid * per), hi = min(N, lo + per);
  int mine = 0;
  double lr = 0.0;
  if (f0 >= 0)
    for (int j = lo; j < hi; ++j)
      if (kept(f0, j, key_at(j), cls_at(j))) { ++mine; lr += (double)lp_at(j); }
  int total;
  int off = block_exclusive_scan(mine, red_i, &total);
  if (f0 >= 0)
    for (int j = lo; j < hi; ++j)
      if (kept(f0, j, key_at(j), cls_at(j))) p.kept_pos[(size_t)g * N + off++] = j;
  POL_STAMP(4);
  lr = block_sum(lr, red_d);
  if (tid == 0) {
    p.kept_count[g] = f0 >= 0 ? total : 0;
    p.last_row_recovery[g] = f0 >= 0 ? lr : 0.0;
    // initial frequent set of the chosen policy (decode's incremental top-k)
    const bool fr = f0 >= 0 && (p.atoms[f0] & AKV_ATOM_FREQUENT) && !(p.atoms[f0] & AKV_ATOM_FULL);
    p.thr_key[g] = fr ? s_thr_key[f0] : ~0ull;
    p.thr_pos[g] = fr ? s_thr_pos[f0] : -1;
  }
  POL_STAMP(5);
  // pending output A[N-1] @ V = sum of the per-key-tile partials
  for (int c = tid; c < p.d; c += kPolicyThreads) {
    float o = 0.f;
    for (int t = 0; t < p.ntiles; ++t) o += p.out_part[((size_t)g * p.ntiles + t) * p.d + c];
    p.out_last[(size_t)g * p.d + c] = o;
  }
  POL_STAMP(6);
}

template <typename T, int D>
static cudaError_t launch_simt_passes(const ProfParams& pp, int G, int ntiles, cudaStream_t st) {
  const size_t smem = 2 * D * kTile * sizeof(float);
  auto k1 = k1_rowlse<T, D>;
  auto k2 = k1_colsum<T, D>;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if ((e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  dim3 grid(ntiles, G);
  k1<<<grid, kThreads, smem, st>>>(pp);
  if ((e = cudaGetLastError())) return e;
  k2<<<grid, kThreads, smem, st>>>(pp);
  return cudaGetLastError();
}

}  // namespace akv

using namespace akv;

// the policy epilogue launches programmatically (AKV_K1_POLICY_PDL=0: ordinary launch, A/B)
static bool k1_policy_pdl() {
  static const bool v = [] { const char* e = getenv("AKV_K1_POLICY_PDL"); return !e || atoi(e) != 0; }();
  return v;
}

extern "C" size_t akv_profile_workspace_size(int32_t B, int32_t H, int32_t N, int32_t d) {
  const size_t ntiles = (size_t)(N + kTile - 1) / kTile;
  return (size_t)B * H * ntiles * d * sizeof(float) + 256;
}

extern "C" int akv_profile(const akv_profile_args* a, void* stream) {
  if (!a) return set_error(AKV_ERR_INVALID, "akv_profile: null args");
  if (a->B < 1 || a->H < 1 || a->N < 1)
    return set_error(AKV_ERR_INVALID, "akv_profile: empty input (B=%d H=%d N=%d)", a->B, a->H, a->N);
  if (a->N > kPosMask) return set_error(AKV_ERR_UNSUPPORTED, "akv_profile: N=%d too large", a->N);
  if (a->ld < a->N) return set_error(AKV_ERR_INVALID, "akv_profile: ld %lld < N %d", (long long)a->ld, a->N);
  if (a->n_family < 1 || a->n_family > AKV_MAX_FAMILY)
    return set_error(AKV_ERR_INVALID, "akv_profile: feasible set is empty or too large (%d)", a->n_family);
  if (a->n_thresholds < 1 || a->n_thresholds > AKV_MAX_THRESHOLDS)
    return set_error(AKV_ERR_INVALID, "akv_profile: need 1..%d thresholds", AKV_MAX_THRESHOLDS);
  if (a->workspace_bytes < akv_profile_workspace_size(a->B, a->H, a->N, a->d))
    return set_error(AKV_ERR_CAPACITY, "akv_profile: workspace too small");
  const int G = a->B * a->H;
  const int ntiles = (a->N + kTile - 1) / kTile;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ProfParams pp{a->B, a->H, a->N, a->q_dev, a->k_dev, a->v_dev, a->ld, a->cls_dev, a->cls_ld,
                a->slope_dev, a->sink_dev, (float)(1.0 / sqrt((double)a->d)), a->lse_dev,
                a->colsum_dev, a->colsq_dev, a->lastp_dev,
                static_cast<float*>(a->workspace_dev)};
  cudaError_t e = cudaErrorInvalidValue;
  bool done = false;
  int part_tiles = ntiles;  // out_part rows per head (64-key SIMT tiles / 128-key TC tiles)
  if (a->dtype == AKV_DTYPE_BF16 && a->d == 128 && tc_profile_supported(a->N)) {
    part_tiles = tc_tiles(a->N);
    e = launch_tc_passes(pp.q, pp.k, pp.v, a->B, a->H, a->N, a->ld, a->cls_dev, a->cls_ld,
                         a->slope_dev, a->sink_dev, a->lse_dev, a->colsum_dev, a->colsq_dev,
                         a->lastp_dev, pp.out_part, st);
    done = true;
  }
#define AKV_SIMT(T, D) e = launch_simt_passes<T, D>(pp, G, ntiles, st); done = true;
  if (!done) {
    if (a->dtype == AKV_DTYPE_F32) {
      switch (a->d) {
        case 16: AKV_SIMT(float, 16) break;
        case 32: AKV_SIMT(float, 32) break;
        case 64: AKV_SIMT(float, 64) break;
        case 128: AKV_SIMT(float, 128) break;
        default: break;
      }
    } else if (a->dtype == AKV_DTYPE_BF16) {
      switch (a->d) {
        case 16: AKV_SIMT(__nv_bfloat16, 16) break;
        case 32: AKV_SIMT(__nv_bfloat16, 32) break;
        case 64: AKV_SIMT(__nv_bfloat16, 64) break;
        case 128: AKV_SIMT(__nv_bfloat16, 128) break;
        default: break;
      }
    }
  }
#undef AKV_SIMT
  if (!done) return set_error(AKV_ERR_UNSUPPORTED, "akv_profile: unsupported dtype %d / head dim %d", a->dtype, a->d);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_profile: %s", cudaGetErrorString(e));

  PolicyParams pol{};
  pol.B = a->B; pol.H = a->H; pol.N = a->N; pol.d = a->d; pol.ntiles = part_tiles;
  pol.cls = a->cls_dev; pol.cls_ld = a->cls_ld;
  pol.colsum = a->colsum_dev; pol.colsq = a->colsq_dev; pol.lastp = a->lastp_dev;
  pol.out_part = pp.out_part;
  pol.n_family = a->n_family;
  for (int f = 0; f < a->n_family; ++f) {
    pol.atoms[f] = a->family_atoms[f]; pol.r_l[f] = a->family_r_l[f]; pol.r_f[f] = a->family_r_f[f];
  }
  pol.n_thr = a->n_thresholds;
  for (int t = 0; t < a->n_thresholds; ++t) pol.thr[t] = a->thresholds[t];
  pol.rows = a->rows; pol.criterion = a->criterion;
  pol.local_len = a->local_len > 0 ? a->local_len : a->N;
  if (pol.local_len > a->N)
    return set_error(AKV_ERR_INVALID, "akv_profile: local_len %d exceeds N %d", a->local_len, a->N);
  pol.out_last = a->out_last_dev; pol.recovery = a->recovery_dev; pol.cost = a->cost_dev;
  pol.cosine = a->cosine_dev; pol.choice = a->choice_dev; pol.kept_pos = a->kept_pos_dev;
  pol.kept_count = a->kept_count_dev; pol.last_row_recovery = a->last_row_recovery_dev;
  pol.topk_gap = a->topk_gap_dev;
  pol.thr_key = reinterpret_cast<unsigned long long*>(a->topk_thr_key_dev);
  pol.thr_pos = a->topk_thr_pos_dev;
  if (!pol.thr_key || !pol.thr_pos)
    return set_error(AKV_ERR_INVALID, "akv_profile: topk threshold outputs are required");
  static PerDeviceOnce pol_attr;
  e = pol_attr.run([](int) {
    return cudaFuncSetAttribute(k1_policy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kPolicyStageMaxN * kPolicyStageBytes);
  });
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_profile policy: %s", cudaGetErrorString(e));
  const size_t pol_smem = a->N <= kPolicyStageMaxN ? (size_t)a->N * kPolicyStageBytes : 0;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kPolicyThreads);
    cfg.dynamicSmemBytes = pol_smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = k1_policy_pdl() ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, k1_policy, pol);
    if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_profile policy: %s", cudaGetErrorString(e));
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_profile policy: %s", cudaGetErrorString(e));
  return AKV_OK;
}
