// Model-caller kernels around the adaptive-KV path: the per-layer glue a
// multi-layer decoder needs between the cuBLAS projections and K1/K2/K3
// (the reference's consumer is the concat + linear
// head of engine.py:354-357 and the per-layer row producers of
// model.py:219-286).  All are HBM-bound elementwise / row kernels:
//
//   akv_embed_classify  token ids -> embedding rows + token classes
//                       (tokens.py:28-44 classify_id via a uint8 LUT)
//   akv_add_rmsnorm     residual += x; out = rmsnorm(residual) * w
//   akv_rope_scatter    RoPE on q/k of a fused QKV projection and scatter of
//                       q/k/v into the head-major [B, H, ld, d] layout the
//                       profiling / decode kernels read
//   akv_swiglu          out = silu(gate) * up of a fused gate|up projection
//   akv_greedy_next     argmax over the vocab (np.argmax tie rule: first
//                       index, engine.py:79-80) -> next token id, its class
//                       and its embedding row, all on the device (no host
//                       round trip per decode step)

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

template <typename T> struct Vec16;
template <> struct Vec16<float> {
  static constexpr int n = 4;
  __device__ __forceinline__ static void load(const float* p, float* f) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
};
template <> struct Vec16<__nv_bfloat16> {
  static constexpr int n = 8;
  __device__ __forceinline__ static void load(const __nv_bfloat16* p, float* f) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    Elem<__nv_bfloat16>::unpack(u, f);
  }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

constexpr int kRowThreads = 256;
constexpr int kMaxVecPerThread = 8;

// one CTA per token: embedding row copy (16-byte vectors) + class lookup
template <typename T>
__global__ void __launch_bounds__(kRowThreads) k_embed_classify(const int64_t* ids, int vocab,
                                                                const uint8_t* lut, const T* emb,
                                                                int dm, T* x, uint8_t* cls) {
  const int t = blockIdx.x;
  int64_t id = ids[t];
  id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);  // host validates the prompt range
  if (threadIdx.x == 0 && cls) cls[t] = lut[id];
  if (!emb) return;
  constexpr int n = Vec16<T>::n;
  const T* src = emb + id * (int64_t)dm;
  T* dst = x + (int64_t)t * dm;
  for (int c = threadIdx.x * n; c < dm; c += blockDim.x * n)
    *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
}

// one CTA per row; the row stays in registers between the two passes
template <typename T>
__global__ void __launch_bounds__(kRowThreads) k_add_rmsnorm(int dim, const T* x, T* res,
                                                             const T* w, float eps, T* out) {
  __shared__ float red[kRowThreads / 32];
  constexpr int n = Vec16<T>::n;
  const int64_t base = (int64_t)blockIdx.x * dim;
  const int nv = dim / n;
  float v[kMaxVecPerThread][n];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxVecPerThread; ++j) {
    const int iv = threadIdx.x + j * kRowThreads;
    if (iv < nv) {
      Vec16<T>::load(res + base + iv * n, v[j]);
      if (x) {
        float a[n];
        Vec16<T>::load(x + base + iv * n, a);
#pragma unroll
        for (int e = 0; e < n; ++e) v[j][e] = to_f(from_f<T>(v[j][e] + a[e]));
        Vec16<T>::store(res + base + iv * n, v[j]);
      }
#pragma unroll
      for (int e = 0; e < n; ++e) ss = fmaf(v[j][e], v[j][e], ss);
    }
  }
  ss = block_sum(ss, red);
  const float rs = rsqrtf(ss / (float)dim + eps);
#pragma unroll
  for (int j = 0; j < kMaxVecPerThread; ++j) {
    const int iv = threadIdx.x + j * kRowThreads;
    if (iv < nv) {
      float g[n];
      Vec16<T>::load(w + iv * n, g);
#pragma unroll
      for (int e = 0; e < n; ++e) g[e] *= v[j][e] * rs;
      Vec16<T>::store(out + base + iv * n, g);
    }
  }
}

// Tensor-parallel reduction fused with the residual add and the RMSNorm
// that consumes it: row `row` of every rank's row-parallel partial product
// is read straight from that rank's (symmetric, peer-mapped) buffer - NVLink
// loads - and summed in rank order in fp32, so every rank computes the same
// bits; then residual += sum (rounded to T like the NCCL all-reduce result)
// and out = rmsnorm(residual) * w.  Replaces all_reduce + akv_add_rmsnorm.
template <typename T>
__global__ void __launch_bounds__(kRowThreads) k_peer_add_rmsnorm(int dim, const uint64_t* peers,
                                                                  int n_peers, int64_t peer_ld,
                                                                  T* res, const T* w, float eps,
                                                                  T* out) {
  __shared__ float red[kRowThreads / 32];
  constexpr int n = Vec16<T>::n;
  const int64_t base = (int64_t)blockIdx.x * dim;
  const int nv = dim / n;
  float v[kMaxVecPerThread][n];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxVecPerThread; ++j) {
    const int iv = threadIdx.x + j * kRowThreads;
    if (iv < nv) {
      float a[n];
#pragma unroll
      for (int e = 0; e < n; ++e) a[e] = 0.f;
      for (int r = 0; r < n_peers; ++r) {
        const T* src = reinterpret_cast<const T*>(peers[r]) + (int64_t)blockIdx.x * peer_ld;
        // another GPU wrote it: fetch past any cached copy (ld.global.cv)
        const uint4 u = __ldcv(reinterpret_cast<const uint4*>(src + iv * n));
        float f[n];
        if constexpr (n == 4) {
          f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
          f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
        } else {
          Elem<__nv_bfloat16>::unpack(u, f);
        }
#pragma unroll
        for (int e = 0; e < n; ++e) a[e] += f[e];
      }
      Vec16<T>::load(res + base + iv * n, v[j]);
#pragma unroll
      for (int e = 0; e < n; ++e) v[j][e] = to_f(from_f<T>(v[j][e] + to_f(from_f<T>(a[e]))));
      Vec16<T>::store(res + base + iv * n, v[j]);
#pragma unroll
      for (int e = 0; e < n; ++e) ss = fmaf(v[j][e], v[j][e], ss);
    }
  }
  ss = block_sum(ss, red);
  const float rs = rsqrtf(ss / (float)dim + eps);
#pragma unroll
  for (int j = 0; j < kMaxVecPerThread; ++j) {
    const int iv = threadIdx.x + j * kRowThreads;
    if (iv < nv) {
      float g[n];
      Vec16<T>::load(w + iv * n, g);
#pragma unroll
      for (int e = 0; e < n; ++e) g[e] *= v[j][e] * rs;
      Vec16<T>::store(out + base + iv * n, g);
    }
  }
}

// RoPE (rotate-half pairing c <-> c + d/2) of q and k, copy of v; token t =
// b*n + i sits at position pos0 + i and lands in row row0 + i of head h of
// batch row b.  128 threads = (128 / (d/2)) heads x d/2 pairs.
template <typename T>
__global__ void __launch_bounds__(128) k_rope_scatter(akv_rope_args a) {
  const int half = a.d / 2;
  const int hpb = 128 / half;
  const int t = blockIdx.x;  // tokens on x: up to 2^31-1 (y is capped at 65535)
  const int h = blockIdx.y * hpb + threadIdx.x / half;
  const int c = threadIdx.x % half;
  if (h >= a.Hl) return;
  const int b = t / a.n, i = t % a.n;
  int pos = a.pos0 + i + (a.pos_dev ? *a.pos_dev : 0);
  pos = pos < a.max_pos ? pos : a.max_pos - 1;
  const T* row = reinterpret_cast<const T*>(a.qkv_dev) + (int64_t)t * a.qkv_ld;
  const int64_t hd = (int64_t)a.Hl * a.d;
  const float cs = a.cos_dev[(int64_t)pos * half + c];
  const float sn = a.sin_dev[(int64_t)pos * half + c];
  const int64_t dst = (((int64_t)b * a.Hl + h) * a.out_ld + a.row0 + i) * a.d;
  const int64_t src = (int64_t)h * a.d;
  {
    const float x1 = to_f(row[src + c]), x2 = to_f(row[src + c + half]);
    T* q = reinterpret_cast<T*>(a.q_dev) + dst;
    q[c] = from_f<T>(x1 * cs - x2 * sn);
    q[c + half] = from_f<T>(x2 * cs + x1 * sn);
  }
  {
    const float x1 = to_f(row[hd + src + c]), x2 = to_f(row[hd + src + c + half]);
    T* k = reinterpret_cast<T*>(a.k_dev) + dst;
    k[c] = from_f<T>(x1 * cs - x2 * sn);
    k[c + half] = from_f<T>(x2 * cs + x1 * sn);
  }
  T* v = reinterpret_cast<T*>(a.v_dev) + dst;
  v[c] = row[2 * hd + src + c];
  v[c + half] = row[2 * hd + src + c + half];
}

template <typename T>
__global__ void k_swiglu(int64_t total, int F, const T* gu, T* out) {
  constexpr int n = Vec16<T>::n;
  const int64_t nvec = total / n;
  for (int64_t iv = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; iv < nvec;
       iv += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = iv * n;
    const int64_t r = e0 / F, c = e0 % F;
    float g[n], u[n];
    Vec16<T>::load(gu + r * 2 * F + c, g);
    Vec16<T>::load(gu + r * 2 * F + F + c, u);
#pragma unroll
    for (int e = 0; e < n; ++e) g[e] = g[e] / (1.f + __expf(-g[e])) * u[e];
    Vec16<T>::store(out + e0, g);
  }
}

constexpr int kArgmaxThreads = 1024;

// one CTA per batch row: first-index argmax, class, embedding of the token
template <typename T>
__global__ void __launch_bounds__(kArgmaxThreads) k_greedy_next(int V, const T* logits, int64_t ld,
                                                                const uint8_t* lut, const T* emb,
                                                                int dm, int64_t* tokens,
                                                                uint8_t* cls, T* x) {
  __shared__ float sv[kArgmaxThreads / 32];
  __shared__ int si[kArgmaxThreads / 32];
  __shared__ int tok;
  const int b = blockIdx.x;
  const T* row = logits + (int64_t)b * ld;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float s = to_f(row[j]);
    if (s > bv) { bv = s; bi = j; }  // ascending j per thread: first max kept
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float v0 = sv[0];
    int i0 = si[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > v0 || (sv[w] == v0 && si[w] < i0)) { v0 = sv[w]; i0 = si[w]; }
    if (i0 == 0x7fffffff) i0 = 0;  // all -inf/NaN: np.argmax would return 0
    tok = i0;
    tokens[b] = i0;
    if (cls) cls[b] = lut[i0];
  }
  __syncthreads();
  if (!emb) return;
  constexpr int n = Vec16<T>::n;
  const T* src = emb + (int64_t)tok * dm;
  T* dst = x + (int64_t)b * dm;
  for (int c = threadIdx.x * n; c < dm; c += blockDim.x * n)
    *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
}

static int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return AKV_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace akv

using namespace akv;

extern "C" int akv_embed_classify(int32_t n, const int64_t* ids_dev, int32_t vocab,
                                  const uint8_t* lut_dev, const void* emb_dev, int32_t dm,
                                  int32_t dtype, void* x_out_dev, uint8_t* cls_out_dev,
                                  void* stream) {
  if (n < 0 || vocab < 1 || !ids_dev || (!emb_dev && !cls_out_dev) || (cls_out_dev && !lut_dev))
    return set_error(AKV_ERR_INVALID, "akv_embed_classify: bad arguments");
  if (n == 0) return AKV_OK;
  const int vec = dtype == AKV_DTYPE_F32 ? 4 : 8;
  if (emb_dev && (dm % vec || !aligned16(emb_dev) || !aligned16(x_out_dev)))
    return set_error(AKV_ERR_UNSUPPORTED, "akv_embed_classify: dm %d must be a multiple of %d and "
                     "rows 16-byte aligned", dm, vec);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == AKV_DTYPE_F32)
    k_embed_classify<float><<<n, kRowThreads, 0, st>>>(ids_dev, vocab, lut_dev, (const float*)emb_dev,
                                                       dm, (float*)x_out_dev, cls_out_dev);
  else if (dtype == AKV_DTYPE_BF16)
    k_embed_classify<__nv_bfloat16><<<n, kRowThreads, 0, st>>>(
        ids_dev, vocab, lut_dev, (const __nv_bfloat16*)emb_dev, dm, (__nv_bfloat16*)x_out_dev,
        cls_out_dev);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_embed_classify: dtype %d", dtype);
  return launch_status("akv_embed_classify");
}

extern "C" int akv_add_rmsnorm(int32_t rows, int32_t dim, int32_t dtype, const void* x_dev,
                               void* residual_dev, const void* w_dev, float eps, void* out_dev,
                               void* stream) {
  if (rows < 0 || dim < 1 || !residual_dev || !w_dev || !out_dev)
    return set_error(AKV_ERR_INVALID, "akv_add_rmsnorm: bad arguments");
  if (rows == 0) return AKV_OK;
  const int vec = dtype == AKV_DTYPE_F32 ? 4 : 8;
  if (dim % vec || dim > vec * kRowThreads * kMaxVecPerThread || !aligned16(residual_dev) ||
      !aligned16(out_dev) || !aligned16(w_dev) || (x_dev && !aligned16(x_dev)))
    return set_error(AKV_ERR_UNSUPPORTED, "akv_add_rmsnorm: dim %d unsupported for dtype %d", dim,
                     dtype);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == AKV_DTYPE_F32)
    k_add_rmsnorm<float><<<rows, kRowThreads, 0, st>>>(dim, (const float*)x_dev, (float*)residual_dev,
                                                       (const float*)w_dev, eps, (float*)out_dev);
  else if (dtype == AKV_DTYPE_BF16)
    k_add_rmsnorm<__nv_bfloat16><<<rows, kRowThreads, 0, st>>>(
        dim, (const __nv_bfloat16*)x_dev, (__nv_bfloat16*)residual_dev, (const __nv_bfloat16*)w_dev,
        eps, (__nv_bfloat16*)out_dev);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_add_rmsnorm: dtype %d", dtype);
  return launch_status("akv_add_rmsnorm");
}

extern "C" int akv_add_rmsnorm_peers(int32_t rows, int32_t dim, int32_t dtype,
                                     const uint64_t* peer_ptrs_dev, int32_t n_peers,
                                     int64_t peer_ld, void* residual_dev, const void* w_dev,
                                     float eps, void* out_dev, void* stream) {
  if (rows < 0 || dim < 1 || n_peers < 1 || peer_ld < dim || !peer_ptrs_dev || !residual_dev ||
      !w_dev || !out_dev)
    return set_error(AKV_ERR_INVALID, "akv_add_rmsnorm_peers: bad arguments");
  if (rows == 0) return AKV_OK;
  const int vec = dtype == AKV_DTYPE_F32 ? 4 : 8;
  if (dim % vec || peer_ld % vec || dim > vec * kRowThreads * kMaxVecPerThread ||
      !aligned16(residual_dev) || !aligned16(out_dev) || !aligned16(w_dev))
    return set_error(AKV_ERR_UNSUPPORTED, "akv_add_rmsnorm_peers: dim %d unsupported for dtype %d",
                     dim, dtype);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == AKV_DTYPE_F32)
    k_peer_add_rmsnorm<float><<<rows, kRowThreads, 0, st>>>(
        dim, peer_ptrs_dev, n_peers, peer_ld, (float*)residual_dev, (const float*)w_dev, eps,
        (float*)out_dev);
  else if (dtype == AKV_DTYPE_BF16)
    k_peer_add_rmsnorm<__nv_bfloat16><<<rows, kRowThreads, 0, st>>>(
        dim, peer_ptrs_dev, n_peers, peer_ld, (__nv_bfloat16*)residual_dev,
        (const __nv_bfloat16*)w_dev, eps, (__nv_bfloat16*)out_dev);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_add_rmsnorm_peers: dtype %d", dtype);
  return launch_status("akv_add_rmsnorm_peers");
}

extern "C" int akv_rope_scatter(const akv_rope_args* a, void* stream) {
  if (!a || a->T < 0 || a->n < 1 || a->Hl < 1 || !a->qkv_dev || !a->cos_dev || !a->sin_dev ||
      !a->q_dev || !a->k_dev || !a->v_dev || a->out_ld < 1 || a->row0 < 0)
    return set_error(AKV_ERR_INVALID, "akv_rope_scatter: bad arguments");
  if (a->d < 2 || a->d % 2 || 128 % (a->d / 2) || a->d > 256)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_rope_scatter: head dim %d", a->d);
  if (a->pos0 < 0 || (!a->pos_dev && a->pos0 + a->n > a->max_pos))
    return set_error(AKV_ERR_INVALID, "akv_rope_scatter: positions %d..%d out of range for a "
                     "%d-position table", a->pos0, a->pos0 + a->n - 1, a->max_pos);
  if (a->T == 0) return AKV_OK;
  if (a->T % a->n || a->row0 + a->n > a->out_ld)
    return set_error(AKV_ERR_INVALID, "akv_rope_scatter: T %% n != 0 or rows exceed out_ld");
  const int hpb = 128 / (a->d / 2);
  dim3 grid(a->T, (a->Hl + hpb - 1) / hpb);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a->dtype == AKV_DTYPE_F32)
    k_rope_scatter<float><<<grid, 128, 0, st>>>(*a);
  else if (a->dtype == AKV_DTYPE_BF16)
    k_rope_scatter<__nv_bfloat16><<<grid, 128, 0, st>>>(*a);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_rope_scatter: dtype %d", a->dtype);
  return launch_status("akv_rope_scatter");
}

extern "C" int akv_swiglu(int32_t rows, int32_t F, int32_t dtype, const void* gu_dev, void* out_dev,
                          void* stream) {
  if (rows < 0 || F < 1 || !gu_dev || !out_dev)
    return set_error(AKV_ERR_INVALID, "akv_swiglu: bad arguments");
  if (rows == 0) return AKV_OK;
  const int vec = dtype == AKV_DTYPE_F32 ? 4 : 8;
  if (F % vec || !aligned16(gu_dev) || !aligned16(out_dev))
    return set_error(AKV_ERR_UNSUPPORTED, "akv_swiglu: F %d must be a multiple of %d", F, vec);
  const int64_t total = (int64_t)rows * F;
  const int64_t nvec = total / vec;
  const int threads = 256;
  int blocks = (int)((nvec + threads - 1) / threads);
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == AKV_DTYPE_F32)
    k_swiglu<float><<<blocks, threads, 0, st>>>(total, F, (const float*)gu_dev, (float*)out_dev);
  else if (dtype == AKV_DTYPE_BF16)
    k_swiglu<__nv_bfloat16><<<blocks, threads, 0, st>>>(total, F, (const __nv_bfloat16*)gu_dev,
                                                         (__nv_bfloat16*)out_dev);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_swiglu: dtype %d", dtype);
  return launch_status("akv_swiglu");
}

extern "C" int akv_greedy_next(int32_t B, int32_t V, int32_t dtype, const void* logits_dev,
                               int64_t ld, const uint8_t* lut_dev, const void* emb_dev, int32_t dm,
                               int64_t* tokens_dev, uint8_t* cls_dev, void* x_out_dev,
                               void* stream) {
  if (B < 0 || V < 1 || ld < V || !logits_dev || !tokens_dev || (cls_dev && !lut_dev) ||
      (emb_dev && !x_out_dev))
    return set_error(AKV_ERR_INVALID, "akv_greedy_next: bad arguments");
  if (B == 0) return AKV_OK;
  const int vec = dtype == AKV_DTYPE_F32 ? 4 : 8;
  if (emb_dev && (dm % vec || !aligned16(emb_dev) || !aligned16(x_out_dev)))
    return set_error(AKV_ERR_UNSUPPORTED, "akv_greedy_next: dm %d", dm);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == AKV_DTYPE_F32)
    k_greedy_next<float><<<B, kArgmaxThreads, 0, st>>>(V, (const float*)logits_dev, ld, lut_dev,
                                                       (const float*)emb_dev, dm, tokens_dev,
                                                       cls_dev, (float*)x_out_dev);
  else if (dtype == AKV_DTYPE_BF16)
    k_greedy_next<__nv_bfloat16><<<B, kArgmaxThreads, 0, st>>>(
        V, (const __nv_bfloat16*)logits_dev, ld, lut_dev, (const __nv_bfloat16*)emb_dev, dm,
        tokens_dev, cls_dev, (__nv_bfloat16*)x_out_dev);
  else
    return set_error(AKV_ERR_UNSUPPORTED, "akv_greedy_next: dtype %d", dtype);
  return launch_status("akv_greedy_next");
}
