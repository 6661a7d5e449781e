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
// Layout: each head g owns arena slots [seg_off[g], seg_off[g]+seg_cap[g]);
// slots [0, live) are live rows (any order), row = d elements of K (kc) and
// V (vc), meta = position | class<<24, score = float64 cumulative attention.
//
// One launch = one step for all B*H heads.  grid = (max chunks, B*H); CTA
// (c, g) streams C consecutive slots of head g with 16-byte non-allocating
// loads (all of the chunk's K and V rows are in flight before the first
// FMA), computes logits, a chunk-local softmax and the PV partial, and
// publishes (max, sum, o[d]) to the workspace.  The last CTA of a head to
// finish (split-K semaphore) combines the partials, writes the output and
// runs the policy epilogue: score update, keep rule (exact top-k on
// (score desc, position asc)), and swap-remove compaction of evicted rows
// (only the few evicted holes are filled, from the segment tail).  The
// chunk that holds slot `live` reads the new row from the inputs and
// stores it into the cache (fused insert).  live_in/live_out are distinct
// buffers so CTAs that exit early never see this step's update.

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kDecWarps = 4;
constexpr int kDecSteps = 8;  // row steps per warp per chunk

template <typename T, int D>
struct DecShape {
  static constexpr int EV = Elem<T>::kPerVec;  // elements per 16-byte vector
  static constexpr int LPR = D / EV;           // lanes per row
  static constexpr int RPW = 32 / LPR;         // rows per warp step
  static constexpr int C = kDecSteps * kDecWarps * RPW;  // slots per chunk
  static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "unsupported head dim");
};

// smallest chunk over dtypes for a head dim (sizes the workspace)
static inline int min_chunk(int d) { return kDecSteps * kDecWarps * (32 / (d * 4 / 16)); }

struct DecParams {
  int B, H, prompt_len, pos;
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
  const int32_t* live_in;
  int32_t* live_out;
  float* out;
  int32_t* evicted;
  int32_t* status;
  float* part;       // [G, max_chunks, D+2]
  float* logit;      // [total_slots]
  int32_t* counter;  // [G]
  int max_chunks;
  float scale;
};

template <typename T, int D>
__global__ void __launch_bounds__(kDecWarps * 32) k3_decode(DecParams p) {
  using S = DecShape<T, D>;
  constexpr int EV = S::EV, LPR = S::LPR, RPW = S::RPW, C = S::C;
  constexpr int RV = D * sizeof(T) / 16;  // 16-byte vectors per row (== LPR)
  __shared__ float s_red[kDecWarps][D];
  __shared__ float s_m[kDecWarps], s_l[kDecWarps];
  __shared__ int s_last;
  __shared__ int hist[256];
  __shared__ int red_i[33];

  const int g = blockIdx.y, c = blockIdx.x;
  const int L = p.live_in[g];
  const int n = L + 1;
  const int start = c * C;
  if (L < 0 || start >= n) return;
  if (n > p.seg_cap[g]) {  // capacity: every CTA of the head agrees and bails
    if (c == 0 && threadIdx.x == 0) atomicExch(p.status, AKV_ERR_CAPACITY);
    return;
  }
  const int nchunks = (n + C - 1) / C;
  const int b = g / p.H, h = g % p.H;
  const int64_t base = p.seg_off[g];
  const uint8_t atoms = p.atoms[g];
  const bool freq = (atoms & AKV_ATOM_FREQUENT) && !(atoms & AKV_ATOM_FULL);
  const int posq = p.pos;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, sl = lane % LPR;
  const float slope = p.slope ? p.slope[h] : 0.f;
  const float sink = p.sink ? p.sink[h] : 0.f;
  const int new_cls = p.new_cls[b];

  const uint4* kc = static_cast<const uint4*>(p.kc) + base * RV;
  const uint4* vc = static_cast<const uint4*>(p.vc) + base * RV;
  const uint4* kn = reinterpret_cast<const uint4*>(static_cast<const T*>(p.kn) + (size_t)g * p.bh_stride);
  const uint4* vn = reinterpret_cast<const uint4*>(static_cast<const T*>(p.vn) + (size_t)g * p.bh_stride);
  const uint4* qv = reinterpret_cast<const uint4*>(static_cast<const T*>(p.q) + (size_t)g * p.bh_stride);

  // issue every K/V load of the chunk before using any of them
  uint4 kr[kDecSteps], vr[kDecSteps];
  int mt[kDecSteps];
#pragma unroll
  for (int s = 0; s < kDecSteps; ++s) {
    const int slot = start + (s * kDecWarps + warp) * RPW + sub;
    if (slot < L) {
      kr[s] = ld_nc_v4(kc + (size_t)slot * RV + sl);
      vr[s] = ld_nc_v4(vc + (size_t)slot * RV + sl);
      mt[s] = p.meta[base + slot];
    } else if (slot == L) {  // fused insert of the new token
      kr[s] = kn[sl];
      vr[s] = vn[sl];
      mt[s] = posq | (new_cls << kClsShift);
      uint4* kw = static_cast<uint4*>(p.kc) + (base + slot) * RV;
      uint4* vw = static_cast<uint4*>(p.vc) + (base + slot) * RV;
      st_v4(kw + sl, kr[s]);
      st_v4(vw + sl, vr[s]);
      if (sl == 0) {
        p.meta[base + slot] = mt[s];
        p.score[base + slot] = 0.0;  // policies.py:357
      }
    } else {
      kr[s] = make_uint4(0, 0, 0, 0);
      vr[s] = make_uint4(0, 0, 0, 0);
      mt[s] = -1;
    }
  }
  float qf[EV];
  Elem<T>::unpack(qv[sl], qf);
#pragma unroll
  for (int e = 0; e < EV; ++e) qf[e] *= p.scale;

  // logits (engine.py:95) + planted head bias
  float sj[kDecSteps];
  float mx = -INFINITY;
#pragma unroll
  for (int s = 0; s < kDecSteps; ++s) {
    float kf[EV];
    Elem<T>::unpack(kr[s], kf);
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < EV; ++e) dot = fmaf(qf[e], kf[e], dot);
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    float x = -INFINITY;
    if (mt[s] >= 0) {
      x = dot;
      if (meta_cls(mt[s]) == AKV_CLS_SPECIAL) x += sink;
      if (slope != 0.f) x -= slope * (float)(posq - meta_pos(mt[s]));
    }
    sj[s] = x;
    mx = fmaxf(mx, x);
  }
  if (freq && sl == 0) {
#pragma unroll
    for (int s = 0; s < kDecSteps; ++s) {
      const int slot = start + (s * kDecWarps + warp) * RPW + sub;
      if (slot < L) p.logit[base + slot] = sj[s];
    }
  }
  mx = warp_allreduce(mx, [](float a, float b) { return fmaxf(a, b); });
  if (lane == 0) s_m[warp] = mx;
  __syncthreads();
  float M = s_m[0];
#pragma unroll
  for (int w = 1; w < kDecWarps; ++w) M = fmaxf(M, s_m[w]);

  // chunk-local softmax numerator and PV partial
  float o[EV];
#pragma unroll
  for (int e = 0; e < EV; ++e) o[e] = 0.f;
  float lsum = 0.f;
#pragma unroll
  for (int s = 0; s < kDecSteps; ++s) {
    const float pe = (sj[s] == -INFINITY) ? 0.f : __expf(sj[s] - M);
    if (sl == 0) lsum += pe;
    float vf[EV];
    Elem<T>::unpack(vr[s], vf);
#pragma unroll
    for (int e = 0; e < EV; ++e) o[e] = fmaf(pe, vf[e], o[e]);
  }
  // reduce over the RPW rows of a warp step (lanes with equal sl)
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
    for (int e = 0; e < EV; ++e) o[e] += __shfl_xor_sync(0xffffffffu, o[e], off);
  }
  lsum = warp_allreduce(lsum, [](float a, float b) { return a + b; });
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < EV; ++e) s_red[warp][sl * EV + e] = o[e];
  }
  if (lane == 0) s_l[warp] = lsum;
  __syncthreads();
  float* part = p.part + ((size_t)g * p.max_chunks + c) * (D + 2);
  for (int t = threadIdx.x; t < D; t += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) acc += s_red[w][t];
    part[t] = acc;
  }
  if (threadIdx.x == 0) {
    float l = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) l += s_l[w];
    part[D] = M;
    part[D + 1] = l;
  }
  // split-K semaphore: the last CTA of this head runs the epilogue
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&p.counter[g], 1) == nchunks - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- epilogue (one CTA per head) ----
  const float* parts = p.part + (size_t)g * p.max_chunks * (D + 2);
  float gM = -INFINITY;
  for (int k = 0; k < nchunks; ++k) gM = fmaxf(gM, __ldcg(parts + (size_t)k * (D + 2) + D));
  float gl = 0.f;
  for (int k = 0; k < nchunks; ++k) {
    const float* pk = parts + (size_t)k * (D + 2);
    gl += __ldcg(pk + D + 1) * __expf(__ldcg(pk + D) - gM);
  }
  const float inv = 1.f / gl;
  for (int t = threadIdx.x; t < D; t += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < nchunks; ++k) {
      const float* pk = parts + (size_t)k * (D + 2);
      acc += __ldcg(pk + t) * __expf(__ldcg(pk + D) - gM);
    }
    p.out[(size_t)g * D + t] = acc * inv;
  }
  if (atoms & AKV_ATOM_FULL) {  // full cache: nothing is ever evicted
    if (threadIdx.x == 0) {
      p.live_out[g] = n;
      if (p.evicted) p.evicted[g] = 0;
      p.counter[g] = 0;
    }
    return;
  }
  const float lse = gM + logf(gl);
  const int cur = posq + 1;
  double* score = p.score + base;
  const int32_t* meta = p.meta + base;
  if (freq) {  // engine.py:320-330 / policies.py:355-357 (score[new] is 0)
    const float* lg = p.logit + base;
    for (int j = threadIdx.x; j < L; j += blockDim.x)
      score[j] += (double)expf(__ldcg(lg + j) - lse);
  }
  __syncthreads();
  unsigned long long thr_key = 0ull;
  int thr_pos = 0x7fffffff;
  if (freq) {
    const int kb = budget(p.r_f[g], cur);
    auto get = [&](int i, unsigned long long* key, int* pos) {
      *key = (unsigned long long)__double_as_longlong(__ldcg(score + i));
      *pos = meta_pos(__ldcg(meta + i));
    };
    block_topk_threshold(n, kb, get, hist, red_i, &thr_key, &thr_pos);
  }
  const int window_start = cur - budget(p.r_l[g], p.prompt_len);
  auto keep = [&](int j) -> bool {
    const int m = __ldcg(meta + j);
    const int cl = meta_cls(m), ps = meta_pos(m);
    bool k = ((atoms & AKV_ATOM_SPECIAL) && cl == AKV_CLS_SPECIAL) ||
             ((atoms & AKV_ATOM_PUNCT) && cl == AKV_CLS_PUNCT) ||
             ((atoms & AKV_ATOM_LOCAL) && ps >= window_start);
    if (freq && !k)
      k = topk_selected((unsigned long long)__double_as_longlong(__ldcg(score + j)), ps, thr_key, thr_pos);
    return k;
  };
  // count kept, then pair holes (evicted slots below n') with donors (kept
  // slots at or above n'), both in slot order
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int nk = 0;
  for (int j = lo; j < hi; ++j) nk += keep(j);
  const int n_keep = block_sum(nk, red_i);
  int holes = 0, donors = 0;
  for (int j = lo; j < hi; ++j) {
    const bool k = keep(j);
    holes += (j < n_keep && !k);
    donors += (j >= n_keep && k);
  }
  int n_holes, n_donors;
  int hole_off = block_exclusive_scan(holes, red_i, &n_holes);
  int donor_off = block_exclusive_scan(donors, red_i, &n_donors);
  int* hole_list = reinterpret_cast<int*>(p.logit + base);  // logits are consumed
  int* donor_list = hole_list + n_holes;
  __syncthreads();
  for (int j = lo; j < hi; ++j) {
    const bool k = keep(j);
    if (j < n_keep && !k) hole_list[hole_off++] = j;
    if (j >= n_keep && k) donor_list[donor_off++] = j;
  }
  __syncthreads();
  uint4* kw = static_cast<uint4*>(p.kc) + base * RV;
  uint4* vw = static_cast<uint4*>(p.vc) + base * RV;
  for (int r = warp; r < n_holes; r += kDecWarps) {
    const int dst = hole_list[r], src = donor_list[r];
    for (int v = lane; v < RV; v += 32) {
      st_v4(kw + (size_t)dst * RV + v, ld_cg_v4(kw + (size_t)src * RV + v));
      st_v4(vw + (size_t)dst * RV + v, ld_cg_v4(vw + (size_t)src * RV + v));
    }
    if (lane == 0) {
      p.meta[base + dst] = __ldcg(meta + src);
      score[dst] = __ldcg(score + src);
    }
  }
  if (threadIdx.x == 0) {
    p.live_out[g] = n_keep;
    if (p.evicted) p.evicted[g] = n - n_keep;
    p.counter[g] = 0;
  }
}

template <typename T, int D>
static cudaError_t launch_decode(const DecParams& p, int G, cudaStream_t st) {
  dim3 grid(p.max_chunks, G);
  k3_decode<T, D><<<grid, kDecWarps * 32, 0, st>>>(p);
  return cudaGetLastError();
}

struct DecWs {
  float* part;
  float* logit;
  int32_t* counter;
  int32_t* status;
  size_t bytes;
  int max_chunks;
};

static DecWs carve(void* ws, int B, int H, int d, int max_cap, int64_t total_slots) {
  DecWs w;
  const int G = B * H;
  w.max_chunks = (max_cap + min_chunk(d) - 1) / min_chunk(d);
  char* c = static_cast<char*>(ws);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = c + off; off += (bytes + 255) & ~size_t(255); return r; };
  w.counter = reinterpret_cast<int32_t*>(take((size_t)G * 4));
  w.status = reinterpret_cast<int32_t*>(take(4));
  w.part = reinterpret_cast<float*>(take((size_t)G * w.max_chunks * (d + 2) * 4));
  w.logit = reinterpret_cast<float*>(take((size_t)total_slots * 4));
  w.bytes = off;
  return w;
}

}  // namespace akv

using namespace akv;

extern "C" size_t akv_decode_workspace_size(int32_t B, int32_t H, int32_t d, int32_t max_cap,
                                           int64_t total_slots) {
  return carve(nullptr, B, H, d, max_cap, total_slots).bytes;
}

extern "C" int akv_decode_workspace_init(void* ws, size_t bytes, int32_t B, int32_t H, int32_t d,
                                         int32_t max_cap, int64_t total_slots, void* stream) {
  DecWs w = carve(ws, B, H, d, max_cap, total_slots);
  if (bytes < w.bytes) return set_error(AKV_ERR_CAPACITY, "akv_decode_workspace_init: workspace too small");
  // counters + status are contiguous at the start
  cudaError_t e = cudaMemsetAsync(ws, 0, reinterpret_cast<char*>(w.part) - static_cast<char*>(ws),
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_workspace_init: %s", cudaGetErrorString(e));
  return AKV_OK;
}

extern "C" int akv_decode_step(const akv_decode_args* a, void* stream) {
  if (!a) return set_error(AKV_ERR_INVALID, "akv_decode_step: null args");
  if (a->B < 1 || a->H < 1) return set_error(AKV_ERR_INVALID, "akv_decode_step: empty input");
  if (a->pos < a->prompt_len || a->prompt_len < 1)
    return set_error(AKV_ERR_INVALID, "akv_decode_step: need pos >= prompt_len >= 1");
  if (a->pos > kPosMask) return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_step: position too large");
  if (a->live_in_dev == a->live_out_dev)
    return set_error(AKV_ERR_INVALID, "akv_decode_step: live_in and live_out must be distinct buffers");
  if (a->bh_stride < a->d) return set_error(AKV_ERR_INVALID, "akv_decode_step: bh_stride < d");
  DecWs w = carve(a->workspace_dev, a->B, a->H, a->d, a->max_cap, a->total_slots);
  if (a->workspace_bytes < w.bytes) return set_error(AKV_ERR_CAPACITY, "akv_decode_step: workspace too small");
  DecParams p{a->B, a->H, a->prompt_len, a->pos, a->q_dev, a->k_dev, a->v_dev, a->bh_stride,
              a->new_cls_dev, a->slope_dev, a->sink_dev, a->head_atoms_dev, a->head_r_l_dev,
              a->head_r_f_dev, a->seg_off_dev, a->seg_cap_dev, a->kc_dev, a->vc_dev, a->meta_dev,
              a->score_dev, a->live_in_dev, a->live_out_dev, a->out_dev, a->evicted_dev,
              a->status_dev ? a->status_dev : w.status, w.part, w.logit, w.counter, 0,
              (float)(1.0 / sqrt((double)a->d))};
  const int G = a->B * a->H;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaErrorInvalidValue;
  bool ok = true;
#define AKV_DEC(T, DD)                                              \
  p.max_chunks = (a->max_cap + DecShape<T, DD>::C - 1) / DecShape<T, DD>::C; \
  e = launch_decode<T, DD>(p, G, st);
  if (a->dtype == AKV_DTYPE_BF16) {
    switch (a->d) {
      case 16: AKV_DEC(__nv_bfloat16, 16) break;
      case 32: AKV_DEC(__nv_bfloat16, 32) break;
      case 64: AKV_DEC(__nv_bfloat16, 64) break;
      case 128: AKV_DEC(__nv_bfloat16, 128) break;
      default: ok = false;
    }
  } else if (a->dtype == AKV_DTYPE_F32) {
    switch (a->d) {
      case 16: AKV_DEC(float, 16) break;
      case 32: AKV_DEC(float, 32) break;
      case 64: AKV_DEC(float, 64) break;
      case 128: AKV_DEC(float, 128) break;
      default: ok = false;
    }
  } else {
    ok = false;
  }
#undef AKV_DEC
  if (!ok) return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_step: unsupported dtype %d / head dim %d", a->dtype, a->d);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_step: %s", cudaGetErrorString(e));
  return AKV_OK;
}
