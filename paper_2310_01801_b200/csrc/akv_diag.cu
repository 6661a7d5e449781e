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
// Launched BEFORE the decode step of the same position (the live slots are
// still the pre-eviction set), grid (chunk, head): each CTA takes a chunk of
// kChunk positions, marks which of them are attended (live slots' positions
// + the new one) in a shared-memory bitmap, and streams the chunk's shadow
// keys with 16-byte vector loads and q in registers, keeping an online
// (max, total mass, attended mass) per row group - the same arithmetic for
// both sums, so a head that attends to everything reports 1 exactly.  The
// chunk partials meet in a workspace and the last CTA of a head (semaphore)
// combines them into the recovery.  The CTA whose chunk holds the new
// position appends the new key row (and the new class) to the shadow.
// HBM-bound: (pos+1)*d*es bytes per head.

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kDiagThreads = 256;
constexpr int kChunk = 128;  // positions per CTA

struct DiagWs {
  float4* part;     // [G, max_chunks] (max, total mass, attended mass, -)
  int32_t* counter; // [G]
  size_t bytes;
  int max_chunks;
};

static DiagWs diag_carve(void* ws, int G, int64_t shadow_ld) {
  DiagWs w;
  w.max_chunks = (int)((shadow_ld + kChunk - 1) / kChunk);
  char* c = static_cast<char*>(ws);
  size_t off = 0;
  auto take = [&](size_t b) { char* r = c + off; off += (b + 255) & ~size_t(255); return r; };
  w.counter = reinterpret_cast<int32_t*>(take((size_t)G * 4));
  w.part = reinterpret_cast<float4*>(take((size_t)G * w.max_chunks * sizeof(float4)));
  w.bytes = off;
  return w;
}

// running (max, total, attended) in natural-log units
struct Mass {
  float m, all, att;
};

__device__ __forceinline__ void mass_add(Mass& s, float x, bool in) {
  if (x > s.m) {
    const float r = __expf(s.m - x);
    s.all = s.all * r + 1.f;
    s.att = s.att * r + (in ? 1.f : 0.f);
    s.m = x;
  } else {
    const float e = __expf(x - s.m);
    s.all += e;
    if (in) s.att += e;
  }
}

__device__ __forceinline__ void mass_merge(Mass& s, const Mass& o) {
  const float mm = fmaxf(s.m, o.m);
  if (mm == -INFINITY) return;
  const float a = s.m == -INFINITY ? 0.f : __expf(s.m - mm);
  const float b = o.m == -INFINITY ? 0.f : __expf(o.m - mm);
  s = {mm, s.all * a + o.all * b, s.att * a + o.att * b};
}

template <typename T, int D>
__global__ void __launch_bounds__(kDiagThreads, 4) k_decode_recovery(akv_diag_args a, DiagWs w) {
  __shared__ Mass s_red[kDiagThreads / 32];
  __shared__ uint32_t s_bits[kChunk / 32];
  constexpr int PER = Elem<T>::kPerVec;   // elements per 16-byte vector
  constexpr int LPR = D / PER;            // lanes per key row
  constexpr int RPW = 32 / LPR;           // rows per warp per iteration
  constexpr int U = 4;                    // iterations whose loads are in flight together
  static_assert(LPR >= 1 && LPR <= 32 && 32 % LPR == 0, "head dim");
  const int g = blockIdx.y, chunk = blockIdx.x;
  const int b = g / a.H, h = g % a.H;
  // a full-cache head attends to every position: its recovery is exactly 1
  // and its shadow keys are never needed (policies are frozen per session)
  if (a.head_atoms_dev && (a.head_atoms_dev[g] & AKV_ATOM_FULL)) {
    if (chunk == 0 && threadIdx.x == 0) a.recovery_dev[g] = 1.0;
    return;
  }
  const int pos = a.pos_dev ? *a.pos_dev : a.pos;
  const int n = pos + 1;
  const int nchunks = (n + kChunk - 1) / kChunk;
  if (chunk >= nchunks) return;
  const int j0 = chunk * kChunk, j1 = min(n, j0 + kChunk);
  T* shadow = reinterpret_cast<T*>(a.shadow_dev) + (int64_t)g * a.shadow_ld * D;
  const T* knew = reinterpret_cast<const T*>(a.k_dev) + (int64_t)g * a.bh_stride;
  const uint8_t new_cls = a.new_cls_dev[b];
  // attended positions of this chunk: the live slots (pre-eviction) + the new one
  for (int i = threadIdx.x; i < kChunk / 32; i += blockDim.x) s_bits[i] = 0u;
  __syncthreads();
  {
    const int L = a.live_in_dev[g];
    const int32_t* meta = a.meta_dev + a.seg_off_dev[g];
    for (int sl = threadIdx.x; sl < L; sl += blockDim.x) {
      const int p = meta_pos(__ldg(meta + sl)) - j0;
      if (p >= 0 && p < kChunk) atomicOr(&s_bits[p >> 5], 1u << (p & 31));
    }
    if (threadIdx.x == 0 && pos >= j0 && pos < j1)
      atomicOr(&s_bits[(pos - j0) >> 5], 1u << ((pos - j0) & 31));
  }
  if (pos >= j0 && pos < j1) {  // append the new key row (engine.py:342) and class
    for (int c = threadIdx.x; c < D / PER; c += blockDim.x)
      reinterpret_cast<uint4*>(shadow + (int64_t)pos * D)[c] = reinterpret_cast<const uint4*>(knew)[c];
    if (h == 0 && threadIdx.x == 0 && a.cls_hist_dev) a.cls_hist_dev[(int64_t)b * a.cls_ld + pos] = new_cls;
  }
  const float slope = a.slope_dev ? a.slope_dev[h] : 0.f;
  const float sink = a.sink_dev ? a.sink_dev[h] : 0.f;
  const float scale = rsqrtf((float)D);
  const uint8_t* cls = a.cls_hist_dev ? a.cls_hist_dev + (int64_t)b * a.cls_ld : nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sub = lane / LPR, sl = lane % LPR;
  float qf[PER];
  Elem<T>::unpack(*reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(a.q_dev) +
                                                  (int64_t)g * a.bh_stride + sl * PER), qf);
#pragma unroll
  for (int e = 0; e < PER; ++e) qf[e] *= scale;
  __syncthreads();  // bitmap complete
  Mass acc{-INFINITY, 0.f, 0.f};
  const int stride = nw * RPW;
  // the loop bound is warp-uniform (the row groups of a warp shuffle together)
  for (int jw = j0 + warp * RPW; jw < j1; jw += U * stride) {
    const int jb = jw + sub;
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u * stride;
      if (j < j1)
        raw[u] = j == pos ? *reinterpret_cast<const uint4*>(knew + sl * PER)
                          : ld_nc_v4(shadow + (int64_t)j * D + sl * PER);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u * stride;
      float kf[PER];
      Elem<T>::unpack(raw[u], kf);
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < PER; ++e) dot = fmaf(qf[e], kf[e], dot);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (j < j1 && sl == 0) {
        float x = dot;
        const int cl = j == pos ? new_cls : (cls ? cls[j] : 0);
        if (cl == AKV_CLS_SPECIAL) x += sink;
        if (slope != 0.f) x -= slope * (float)(pos - j);
        const int r = j - j0;
        mass_add(acc, x, (s_bits[r >> 5] >> (r & 31)) & 1u);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Mass other{__shfl_xor_sync(0xffffffffu, acc.m, o), __shfl_xor_sync(0xffffffffu, acc.all, o),
                     __shfl_xor_sync(0xffffffffu, acc.att, o)};
    mass_merge(acc, other);
  }
  if (lane == 0) s_red[warp] = acc;
  __syncthreads();
  if (threadIdx.x != 0) return;
  Mass t = s_red[0];
  for (int i = 1; i < nw; ++i) mass_merge(t, s_red[i]);
  w.part[(size_t)g * w.max_chunks + chunk] = make_float4(t.m, t.all, t.att, 0.f);
  __threadfence();
  const int prev = atomicAdd(&w.counter[g], 1);
  if (prev != nchunks - 1) return;
  __threadfence();  // every chunk's partial of this head is visible
  double M = -INFINITY;
  for (int c = 0; c < nchunks; ++c) M = fmax(M, (double)__ldcg(&w.part[(size_t)g * w.max_chunks + c]).x);
  double all = 0.0, att = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const float4 pc = __ldcg(&w.part[(size_t)g * w.max_chunks + c]);
    if (pc.x == -INFINITY) continue;
    const double e = exp((double)pc.x - M);
    all += e * pc.y;
    att += e * pc.z;
  }
  w.counter[g] = 0;
  a.recovery_dev[g] = all > 0.0 ? att / all : 0.0;
}

template <typename T>
static cudaError_t launch_diag(const akv_diag_args& a, const DiagWs& w, int max_pos,
                               cudaStream_t st) {
  const dim3 grid((max_pos + 1 + kChunk - 1) / kChunk, a.B * a.H);
  switch (a.d) {
    case 16: k_decode_recovery<T, 16><<<grid, kDiagThreads, 0, st>>>(a, w); break;
    case 32: k_decode_recovery<T, 32><<<grid, kDiagThreads, 0, st>>>(a, w); break;
    case 64: k_decode_recovery<T, 64><<<grid, kDiagThreads, 0, st>>>(a, w); break;
    case 128: k_decode_recovery<T, 128><<<grid, kDiagThreads, 0, st>>>(a, w); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace akv

using namespace akv;

extern "C" size_t akv_decode_recovery_workspace_size(int32_t B, int32_t H, int64_t shadow_ld) {
  return diag_carve(nullptr, B * H, shadow_ld).bytes;
}

extern "C" int akv_decode_recovery_workspace_init(void* ws, size_t bytes, int32_t B, int32_t H,
                                                  int64_t shadow_ld, void* stream) {
  DiagWs w = diag_carve(ws, B * H, shadow_ld);
  if (!ws || bytes < w.bytes)
    return set_error(AKV_ERR_CAPACITY, "akv_decode_recovery_workspace_init: workspace too small");
  cudaError_t e = cudaMemsetAsync(w.counter, 0, (size_t)B * H * 4, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(AKV_ERR_CUDA, "akv_decode_recovery_workspace_init: %s", cudaGetErrorString(e));
  return AKV_OK;
}

extern "C" int akv_decode_recovery(const akv_diag_args* a, void* stream) {
  if (!a || a->B < 1 || a->H < 1 || !a->q_dev || !a->k_dev || !a->new_cls_dev ||
      !a->seg_off_dev || !a->live_in_dev || !a->meta_dev || !a->shadow_dev || !a->recovery_dev ||
      !a->workspace_dev)
    return set_error(AKV_ERR_INVALID, "akv_decode_recovery: bad arguments");
  if (a->d != 16 && a->d != 32 && a->d != 64 && a->d != 128)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_recovery: head dim %d", a->d);
  if (a->bh_stride < a->d) return set_error(AKV_ERR_INVALID, "akv_decode_recovery: bh_stride < d");
  DiagWs w = diag_carve(a->workspace_dev, a->B * a->H, a->shadow_ld);
  if (a->workspace_bytes < w.bytes)
    return set_error(AKV_ERR_CAPACITY, "akv_decode_recovery: workspace too small");
  // a device position is bounded by the shadow capacity (the caller checks
  // the host-side step count against it); the grid covers that bound
  const int max_pos = a->pos_dev ? (int)a->shadow_ld - 1 : a->pos;
  if (max_pos < 0 || max_pos >= a->shadow_ld || (a->cls_hist_dev && max_pos >= a->cls_ld))
    return set_error(AKV_ERR_CAPACITY, "akv_decode_recovery: position %d beyond the shadow "
                     "capacity %lld", max_pos, (long long)a->shadow_ld);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (a->dtype == AKV_DTYPE_F32)
    e = launch_diag<float>(*a, w, max_pos, st);
  else if (a->dtype == AKV_DTYPE_BF16)
    e = launch_diag<__nv_bfloat16>(*a, w, max_pos, st);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_decode_recovery: dtype %d", a->dtype);
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_decode_recovery: %s", cudaGetErrorString(e));
  return AKV_OK;
}
