// Diagnostics mode of a decode step (reference engine.py:341-349): the
// recovery of each head's attended set against uncompressed attention.
//
// The reference keeps every key of every head ("shadow keys",
// engine.py:260-261), appends the new key each step, and reports
//   recovery = sum_{j in attended} softmax(K_full q / sqrt(d))_j
// where attended = the positions live before this step's eviction plus the
// new position (engine.py:317, 345-347).  StepRecord.mean_recovery is the
// mean over heads (engine.py:365).
//
// One CTA per head, launched BEFORE the decode step (so the live slots are
// still the pre-eviction set): the attended positions become a bitmap in
// shared memory, the new key row is appended to the head's shadow rows
// (position-indexed, [G, shadow_ld, d]), and one streaming pass over the
// shadow keys keeps a running (max, total mass, attended mass) per row group
// (16-byte vector loads, q in registers).  HBM-bound: (pos+1)*d*es bytes
// per head.

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kDiagThreads = 256;

template <typename T>
__device__ __forceinline__ void load16(const T* p, float* f) {
  Elem<T>::unpack(*reinterpret_cast<const uint4*>(p), f);
}

struct Online {
  float m, all, att;
};

__device__ __forceinline__ Online merge(Online a, Online b) {
  const float m = fmaxf(a.m, b.m);
  if (m == -INFINITY) return a;
  const float ea = __expf(a.m - m), eb = __expf(b.m - m);
  return {m, a.all * ea + b.all * eb, a.att * ea + b.att * eb};
}

template <typename T, int D>
__global__ void __launch_bounds__(kDiagThreads) k_decode_recovery(akv_diag_args a) {
  extern __shared__ uint32_t s_bits[];
  __shared__ Online s_red[kDiagThreads / 32];
  constexpr int PER = Elem<T>::kPerVec;   // elements per 16-byte vector
  constexpr int LPR = D / PER;            // lanes per key row
  constexpr int RPW = 32 / LPR;           // rows per warp per iteration
  static_assert(LPR >= 1 && LPR <= 32 && 32 % LPR == 0, "head dim");
  const int g = blockIdx.x;
  const int b = g / a.H, h = g % a.H;
  const int pos = a.pos_dev ? *a.pos_dev : a.pos;
  const int n = pos + 1;
  const int words = (n + 31) >> 5;
  for (int w = threadIdx.x; w < words; w += blockDim.x) s_bits[w] = 0u;
  __syncthreads();
  const int L = a.live_in_dev[g];
  const int32_t* meta = a.meta_dev + a.seg_off_dev[g];
  for (int s = threadIdx.x; s < L; s += blockDim.x) {
    const int p = meta_pos(meta[s]);
    if (p < n) atomicOr(&s_bits[p >> 5], 1u << (p & 31));
  }
  if (threadIdx.x == 0) atomicOr(&s_bits[pos >> 5], 1u << (pos & 31));
  const uint8_t new_cls = a.new_cls_dev[b];
  T* shadow = reinterpret_cast<T*>(a.shadow_dev) + (int64_t)g * a.shadow_ld * D;
  const T* knew = reinterpret_cast<const T*>(a.k_dev) + (int64_t)g * a.bh_stride;
  // append the new key row (engine.py:342) and the new class (head 0 of the row)
  for (int c = threadIdx.x; c < D / PER; c += blockDim.x)
    reinterpret_cast<uint4*>(shadow + (int64_t)pos * D)[c] = reinterpret_cast<const uint4*>(knew)[c];
  if (h == 0 && threadIdx.x == 0 && a.cls_hist_dev) a.cls_hist_dev[(int64_t)b * a.cls_ld + pos] = new_cls;
  __syncthreads();

  const float slope = a.slope_dev ? a.slope_dev[h] : 0.f;
  const float sink = a.sink_dev ? a.sink_dev[h] : 0.f;
  const float scale = rsqrtf((float)D);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, sl = lane % LPR;
  float qf[PER];
  load16(reinterpret_cast<const T*>(a.q_dev) + (int64_t)g * a.bh_stride + sl * PER, qf);
  Online acc{-INFINITY, 0.f, 0.f};
  const int nw = blockDim.x >> 5;
  for (int j0 = warp * RPW; j0 < n; j0 += nw * RPW) {
    const int j = j0 + sub;
    float dot = 0.f;
    if (j < n) {
      float kf[PER];
      load16((j == pos ? knew : shadow + (int64_t)j * D) + sl * PER, kf);
#pragma unroll
      for (int e = 0; e < PER; ++e) dot = fmaf(qf[e], kf[e], dot);
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (j < n && sl == 0) {
      float x = dot * scale;
      const int cl = j == pos ? new_cls
                              : (a.cls_hist_dev ? a.cls_hist_dev[(int64_t)b * a.cls_ld + j] : 0);
      if (cl == AKV_CLS_SPECIAL) x += sink;
      if (slope != 0.f) x -= slope * (float)(pos - j);
      const bool in = (s_bits[j >> 5] >> (j & 31)) & 1u;
      if (x > acc.m) {
        const float r = __expf(acc.m - x);
        acc.all *= r;
        acc.att *= r;
        acc.m = x;
      }
      const float e = __expf(x - acc.m);
      acc.all += e;
      if (in) acc.att += e;
    }
  }
  // combine the row groups of the warp, then the warps
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Online other{__shfl_xor_sync(0xffffffffu, acc.m, o), __shfl_xor_sync(0xffffffffu, acc.all, o),
                 __shfl_xor_sync(0xffffffffu, acc.att, o)};
    acc = merge(acc, other);
  }
  if (lane == 0) s_red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Online t = s_red[0];
    for (int w = 1; w < nw; ++w) t = merge(t, s_red[w]);
    a.recovery_dev[g] = t.all > 0.f ? (double)t.att / (double)t.all : 0.0;
  }
}

template <typename T>
static cudaError_t launch_diag(const akv_diag_args& a, int max_pos, cudaStream_t st) {
  const size_t smem = (size_t)((max_pos + 1 + 31) / 32) * 4;
  const int G = a.B * a.H;
  switch (a.d) {
    case 16: k_decode_recovery<T, 16><<<G, kDiagThreads, smem, st>>>(a); break;
    case 32: k_decode_recovery<T, 32><<<G, kDiagThreads, smem, st>>>(a); break;
    case 64: k_decode_recovery<T, 64><<<G, kDiagThreads, smem, st>>>(a); break;
    case 128: k_decode_recovery<T, 128><<<G, kDiagThreads, smem, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace akv

using namespace akv;

extern "C" int akv_decode_recovery(const akv_diag_args* a, void* stream) {
  if (!a || a->B < 1 || a->H < 1 || !a->q_dev || !a->k_dev || !a->new_cls_dev ||
      !a->seg_off_dev || !a->live_in_dev || !a->meta_dev || !a->shadow_dev || !a->recovery_dev)
    return set_error(AKV_ERR_INVALID, "akv_decode_recovery: bad arguments");
  if (a->d != 16 && a->d != 32 && a->d != 64 && a->d != 128)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_recovery: head dim %d", a->d);
  if (a->bh_stride < a->d) return set_error(AKV_ERR_INVALID, "akv_decode_recovery: bh_stride < d");
  // the device position is bounded by the shadow capacity (the caller checks
  // the host-side step count against it)
  const int max_pos = a->pos_dev ? (int)a->shadow_ld - 1 : a->pos;
  if (max_pos < 0 || max_pos >= a->shadow_ld || (a->cls_hist_dev && max_pos >= a->cls_ld))
    return set_error(AKV_ERR_CAPACITY, "akv_decode_recovery: position %d beyond the shadow "
                     "capacity %lld", max_pos, (long long)a->shadow_ld);
  if ((max_pos + 32) / 32 * 4 > 48 * 1024)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_recovery: context too long");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (a->dtype == AKV_DTYPE_F32)
    e = launch_diag<float>(*a, max_pos, st);
  else if (a->dtype == AKV_DTYPE_BF16)
    e = launch_diag<__nv_bfloat16>(*a, max_pos, st);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_recovery: dtype %d", a->dtype);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_recovery: %s", cudaGetErrorString(e));
  return AKV_OK;
}
