// Shared device helpers for the sm_100a adaptive-KV kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/akv.h"

namespace akv {

constexpr int kClsShift = 24;          // meta = position | class << 24 | inF << 30
constexpr int kPosMask = (1 << kClsShift) - 1;
constexpr int kInF = 1 << 30;          // slot is in the frequent top-k set

__device__ __forceinline__ int meta_pos(int m) { return m & kPosMask; }
__device__ __forceinline__ int meta_cls(int m) { return (m >> kClsShift) & 0x3f; }

// Thread-group synchronisation policies for the block-level helpers: the
// whole CTA (barrier 0) or a named barrier over a warp-aligned subset.
struct BlockSync {
  static constexpr int kThreads = 0;  // dynamic (blockDim.x)
  __device__ __forceinline__ static void sync() { __syncthreads(); }
  __device__ __forceinline__ static int tid() { return threadIdx.x; }
  __device__ __forceinline__ static int nthreads() { return blockDim.x; }
};
template <int NT, int ID, int FIRST>
struct NamedSync {
  static constexpr int kThreads = NT;
  static constexpr int kWarps = NT / 32;
  __device__ __forceinline__ static void sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NT) : "memory"); }
  __device__ __forceinline__ static int tid() { return threadIdx.x - FIRST; }
  __device__ __forceinline__ static int nthreads() { return NT; }
};

// policies.py:205-206: max(1, ceil(r*L - 1e-9)) in IEEE float64, with the
// product and the subtraction rounded separately (no FMA contraction), so
// the budget is bit-identical to the reference's Python float arithmetic.
__device__ __forceinline__ int budget(double r, int len) {
  double x = __dsub_rn(__dmul_rn(r, (double)len), 1e-9);
  int b = (int)ceil(x);
  return b < 1 ? 1 : b;
}

template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kPerVec = 4;  // elements per 16-byte vector
  __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ __forceinline__ static float to_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kPerVec = 8;
  __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
};

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

template <typename F>
__device__ __forceinline__ float warp_allreduce(float v, F op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Group-wide sum (deterministic tree order); `red` needs nthreads/32 slots.
template <typename V, typename Sync = BlockSync>
__device__ __forceinline__ V block_sum(V v, V* red) {
  const int lane = Sync::tid() & 31, warp = Sync::tid() >> 5, nw = Sync::nthreads() >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  Sync::sync();
  if (lane == 0) red[warp] = v;
  Sync::sync();
  V t = V(0);
  for (int i = 0; i < nw; ++i) t += red[i];
  Sync::sync();
  return t;
}

// Exclusive group scan of small ints; returns the exclusive prefix of this
// thread and writes the group total to *total.  `red` needs nthreads/32+1.
template <typename Sync = BlockSync>
__device__ __forceinline__ int block_exclusive_scan(int v, int* red, int* total) {
  const int lane = Sync::tid() & 31, warp = Sync::tid() >> 5, nw = Sync::nthreads() >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  Sync::sync();
  if (lane == 31) red[warp] = x;
  Sync::sync();
  if (Sync::tid() == 0) {
    int acc = 0;
    for (int i = 0; i < nw; ++i) { int t = red[i]; red[i] = acc; acc += t; }
    red[nw] = acc;
  }
  Sync::sync();
  int ex = red[warp] + x - v;
  *total = red[nw];
  Sync::sync();
  return ex;
}

// Histogram increment with warp aggregation: the lanes of a warp that hit
// the same bin (bin < 0: none) add once, by their lowest lane.  Scores of one
// head share their leading key bytes, so without it every lane of every warp
// serialises on one shared-memory address in the first radix passes.
__device__ __forceinline__ void hist_add_agg(int* hist, int bin) {
  const unsigned peers = __match_any_sync(__activemask(), bin);
  if (bin >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
}

// ---------------------------------------------------------------------------
// Exact block-wide top-k over candidates keyed by (score desc, position asc),
// the order of the reference's stable argsort on -scores (policies.py:238-240).
// Scores are non-negative float64, so their IEEE bit patterns order like
// unsigned integers.  Radix select on the 64-bit score keys (8-bit digits)
// finds the k-th largest value v*; elements equal to v* are then taken in
// ascending position order until k are selected (second radix select on
// the 24-bit position when more than the remaining count tie).
//
// get(i, &key, &pos) reads candidate i (0 <= i < n).  Returns, through
// *thr_key / *thr_pos, the smallest selected (key, pos): candidate i is in the
// top-k iff key > thr_key || (key == thr_key && pos <= thr_pos).  If k >= n
// everything is selected (thr_key = 0, thr_pos = INT_MAX).
// Once the bucket holding the k-th candidate has at most 64 members (after
// two or three passes for one head's scores, instead of eight), one warp
// ranks them exactly.
// `hist` needs 256 ints of shared memory, `red` 33 ints.
template <typename Sync = BlockSync, typename Get>
__device__ void block_topk_threshold(int n, int k, Get get, int* hist, int* red,
                                     unsigned long long* thr_key, int* thr_pos) {
  const int tid = Sync::tid(), nth = Sync::nthreads();
  if (k >= n) {
    *thr_key = 0ull;
    *thr_pos = 0x7fffffff;
    return;
  }
  constexpr int kSmall = 64;
  __shared__ unsigned long long s_prefix, s_ck[kSmall], s_tk;
  __shared__ int s_remain, s_digit, s_bucket, s_cn, s_cp[kSmall], s_tp;
  if (tid == 0) { s_prefix = 0ull; s_remain = k; }
  Sync::sync();
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nth) hist[i] = 0;
    Sync::sync();
    const unsigned long long prefix = s_prefix;
    for (int i = tid; i < n; i += nth) {
      unsigned long long key; int pos;
      get(i, &key, &pos);
      hist_add_agg(hist, (key & mask) == prefix ? (int)((key >> shift) & 0xff) : -1);
    }
    Sync::sync();
    if (tid < 32) {
      // suffix scan over 256 bins (descending digit): lane owns 8 bins
      const int lane = tid;
      int c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c[j] = hist[255 - (lane * 8 + j)]; s += c[j]; }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int before = incl - s;  // elements with larger digits than my first bin
      const int remain = s_remain;
      int found = -1, above = 0, fcnt = 0;
      int run = before;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (found < 0 && run < remain && run + c[j] >= remain) { found = 255 - (lane * 8 + j); above = run; fcnt = c[j]; }
        run += c[j];
      }
      unsigned ball = __ballot_sync(0xffffffffu, found >= 0);
      int src = __ffs(ball) - 1;
      int dg = __shfl_sync(0xffffffffu, found, src);
      int ab = __shfl_sync(0xffffffffu, above, src);
      int bc = __shfl_sync(0xffffffffu, fcnt, src);
      if (lane == 0) {
        s_digit = dg;
        s_remain = remain - ab;
        s_prefix = prefix | ((unsigned long long)dg << shift);
        s_bucket = bc;
        s_cn = 0;
      }
    }
    Sync::sync();
    mask |= (0xffull << shift);
    if (s_bucket <= kSmall) break;
  }
  if (s_bucket <= kSmall) {
    // gather the bucket, rank it in one warp: the candidate ranked need-1
    // (key desc, position asc) is the smallest selected one
    const unsigned long long bp = s_prefix;
    for (int i = tid; i < n; i += nth) {
      unsigned long long key; int pos;
      get(i, &key, &pos);
      if ((key & mask) == bp) {
        const int slot = atomicAdd(&s_cn, 1);
        s_ck[slot] = key;
        s_cp[slot] = pos;
      }
    }
    Sync::sync();
    if (tid < 32) {
      const int lane = tid, m = s_cn, need = s_remain;
      const unsigned long long k0 = lane < m ? s_ck[lane] : 0ull, k1 = lane + 32 < m ? s_ck[lane + 32] : 0ull;
      const int p0 = lane < m ? s_cp[lane] : 0, p1 = lane + 32 < m ? s_cp[lane + 32] : 0;
      int r0 = 0, r1 = 0;
      for (int o = 0; o < m; ++o) {
        const unsigned long long ko = s_ck[o];
        const int po = s_cp[o];
        r0 += (ko > k0 || (ko == k0 && po < p0));
        r1 += (ko > k1 || (ko == k1 && po < p1));
      }
      const unsigned b0 = __ballot_sync(0xffffffffu, lane < m && r0 == need - 1);
      const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < m && r1 == need - 1);
      const int src = b0 ? __ffs(b0) - 1 : __ffs(b1) - 1;
      const unsigned long long tk = __shfl_sync(0xffffffffu, b0 ? k0 : k1, src);
      const int tp = __shfl_sync(0xffffffffu, b0 ? p0 : p1, src);
      // every candidate equal to the threshold value selected: open position bound
      const bool more = (lane < m && k0 == tk && p0 > tp) || (lane + 32 < m && k1 == tk && p1 > tp);
      const bool any = __any_sync(0xffffffffu, more);
      if (lane == 0) { s_tk = tk; s_tp = any ? tp : 0x7fffffff; }
    }
    Sync::sync();
    *thr_key = s_tk;
    *thr_pos = s_tp;
    return;
  }
  const unsigned long long vstar = s_prefix;
  const int need_eq = s_remain;  // how many elements equal to v* are selected (>= 1)
  // count elements equal to v*
  int cnt = 0;
  for (int i = tid; i < n; i += nth) {
    unsigned long long key; int pos;
    get(i, &key, &pos);
    cnt += (key == vstar);
  }
  cnt = warp_sum_i(cnt);
  Sync::sync();
  if ((tid & 31) == 0) red[tid >> 5] = cnt;
  Sync::sync();
  int n_eq = 0;
  for (int i = 0; i < (nth >> 5); ++i) n_eq += red[i];
  Sync::sync();
  if (n_eq == need_eq) {
    *thr_key = vstar;
    *thr_pos = 0x7fffffff;
    return;
  }
  // ties: select the need_eq smallest positions among key == v* (radix on
  // inverted 24-bit positions, largest inverted == smallest position).
  __shared__ int s_pprefix, s_premain;
  if (tid == 0) { s_pprefix = 0; s_premain = need_eq; }
  Sync::sync();
  int pmask = 0;
  for (int shift = 16; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nth) hist[i] = 0;
    Sync::sync();
    const int prefix = s_pprefix;
    for (int i = tid; i < n; i += nth) {
      unsigned long long key; int pos;
      get(i, &key, &pos);
      int ip = kPosMask - pos;
      hist_add_agg(hist, (key == vstar && (ip & pmask) == prefix) ? ((ip >> shift) & 0xff) : -1);
    }
    Sync::sync();
    if (tid == 0) {
      int remain = s_premain, run = 0;
      for (int dg = 255; dg >= 0; --dg) {
        if (run + hist[dg] >= remain) {
          s_premain = remain - run;
          s_pprefix = prefix | (dg << shift);
          break;
        }
        run += hist[dg];
      }
    }
    Sync::sync();
    pmask |= (0xff << shift);
  }
  *thr_key = vstar;
  *thr_pos = kPosMask - s_pprefix;
}

// Radix key of a (finite, >= 0) float64 score: its bit pattern, which orders
// like the value.  -0.0 is folded onto +0.0 first (the reference's stable
// argsort ties them, policies.py:238-240; their raw bits would rank -0.0
// above every positive score).
__device__ __forceinline__ unsigned long long score_key(double s) {
  return (unsigned long long)__double_as_longlong(__dadd_rn(s, 0.0));
}

__device__ __forceinline__ bool topk_selected(unsigned long long key, int pos,
                                              unsigned long long thr_key, int thr_pos) {
  return key > thr_key || (key == thr_key && pos <= thr_pos);
}

}  // namespace akv

namespace akv {

// Register-resident variant of block_topk_threshold: thread t holds up to
// EPT candidates in key[]/pos[] (the first `cnt` are valid).  Same result
// contract (threshold (key, pos) of the k-th largest under (key desc, pos
// asc)); every pass is a shared-memory histogram over registers.
template <typename Sync, int EPT>
__device__ void regs_topk_threshold(int n, int k, const unsigned long long* key, const int* pos,
                                    int cnt, int* hist, unsigned long long* thr_key, int* thr_pos) {
  const int tid = Sync::tid(), nth = Sync::nthreads();
  if (k >= n) {
    *thr_key = 0ull;
    *thr_pos = 0x7fffffff;
    return;
  }
  __shared__ unsigned long long s_prefix;
  __shared__ int s_remain, s_neq;
  if (tid == 0) { s_prefix = 0ull; s_remain = k; s_neq = 0; }
  Sync::sync();
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nth) hist[i] = 0;
    Sync::sync();
    const unsigned long long prefix = s_prefix;
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      if (i < cnt && (key[i] & mask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 0xff], 1);
    Sync::sync();
    if (tid < 32) {
      const int lane = tid;
      int c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c[j] = hist[255 - (lane * 8 + j)]; s += c[j]; }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int remain = s_remain;
      int found = -1, above = 0, run = incl - s;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (found < 0 && run < remain && run + c[j] >= remain) { found = 255 - (lane * 8 + j); above = run; }
        run += c[j];
      }
      const unsigned ball = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(ball) - 1;
      const int dg = __shfl_sync(0xffffffffu, found, src);
      const int ab = __shfl_sync(0xffffffffu, above, src);
      if (lane == 0) {
        s_remain = remain - ab;
        s_prefix = prefix | ((unsigned long long)dg << shift);
      }
    }
    Sync::sync();
    mask |= (0xffull << shift);
  }
  const unsigned long long vstar = s_prefix;
  const int need_eq = s_remain;
  int mine = 0;
#pragma unroll
  for (int i = 0; i < EPT; ++i) mine += (i < cnt && key[i] == vstar);
  if (mine) atomicAdd(&s_neq, mine);
  Sync::sync();
  if (s_neq == need_eq) {
    *thr_key = vstar;
    *thr_pos = 0x7fffffff;
    return;
  }
  // ties on the value: the need_eq smallest positions win (inverted-position radix)
  __shared__ int s_pp, s_pr;
  if (tid == 0) { s_pp = 0; s_pr = need_eq; }
  Sync::sync();
  int pmask = 0;
  for (int shift = 16; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nth) hist[i] = 0;
    Sync::sync();
    const int prefix = s_pp;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int ip = kPosMask - pos[i];
      if (i < cnt && key[i] == vstar && (ip & pmask) == prefix) atomicAdd(&hist[(ip >> shift) & 0xff], 1);
    }
    Sync::sync();
    if (tid == 0) {
      int remain = s_pr, run = 0;
      for (int dg = 255; dg >= 0; --dg) {
        if (run + hist[dg] >= remain) { s_pr = remain - run; s_pp = prefix | (dg << shift); break; }
        run += hist[dg];
      }
    }
    Sync::sync();
    pmask |= (0xff << shift);
  }
  *thr_key = vstar;
  *thr_pos = kPosMask - s_pp;
}

}  // namespace akv
