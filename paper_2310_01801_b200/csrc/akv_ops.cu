// Reference single-context operations on the GPU (float64): the building
// blocks the reference exposes besides the fused session path, batched over
// contexts so profile_model/select_policy run as one launch each.
//
//   akv_softmax_rows_f64      <- attention.py:64-89  softmax_rows (+causal lengths)
//   akv_causal_attention_f64  <- attention.py:102-127 causal_attention
//   akv_keep_mask             <- policies.py:214-267 _atom_indices / retained_indices,
//                                policies.py:291-293 cache_memory_cost
//   akv_map_recovery_f64      <- profiler.py:70-87 recovery_ratio,
//                                profiler.py:148-161 masked_cosine_similarity
//   akv_update_scores_f64     <- policies.py:332-360 update_cumulative_scores
//   akv_gather_rows_f64       <- policies.py:270-288 apply_policy
//   akv_tv_distance_f64       <- profiler.py:51-67 tv_distance_row

#include <math.h>

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kOpsThreads = 256;

template <typename V>
__device__ __forceinline__ V block_max(V v, V* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  V t = red[0];
  for (int i = 1; i < nw; ++i) t = fmax(t, red[i]);
  __syncthreads();
  return t;
}

// one CTA per row: max-subtract, exp, normalise over the first `len` cols
__global__ void __launch_bounds__(kOpsThreads) ops_softmax_rows(int cols, const double* in,
                                                                const int32_t* lengths, double* out) {
  __shared__ double red[kOpsThreads / 32];
  const int r = blockIdx.x;
  const int len = lengths ? lengths[r] : cols;
  const double* x = in + (size_t)r * cols;
  double* y = out + (size_t)r * cols;
  double m = -INFINITY;
  for (int c = threadIdx.x; c < len; c += blockDim.x) m = fmax(m, x[c]);
  m = block_max(m, red);
  double s = 0.0;
  for (int c = threadIdx.x; c < len; c += blockDim.x) s += exp(x[c] - m);
  s = block_sum(s, red);
  for (int c = threadIdx.x; c < cols; c += blockDim.x) y[c] = c < len ? exp(x[c] - m) / s : 0.0;
}

// one CTA per query row i: logits over keys j <= i, softmax, A row, O row
__global__ void __launch_bounds__(kOpsThreads) ops_causal_attention(int n, int dq, int dv,
                                                                    const double* q, const double* k,
                                                                    const double* v, double scale,
                                                                    double* A, double* O) {
  __shared__ double red[kOpsThreads / 32];
  const int i = blockIdx.x;
  double* a = A + (size_t)i * n;
  const double* qi = q + (size_t)i * dq;
  double m = -INFINITY;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) {
    const double* kj = k + (size_t)j * dq;
    double s = 0.0;
    for (int c = 0; c < dq; ++c) s += qi[c] * kj[c];
    s *= scale;
    a[j] = s;
    m = fmax(m, s);
  }
  m = block_max(m, red);
  double sum = 0.0;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) sum += exp(a[j] - m);
  sum = block_sum(sum, red);
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) a[j] = j <= i ? exp(a[j] - m) / sum : 0.0;
  __syncthreads();
  for (int c = threadIdx.x; c < dv; c += blockDim.x) {
    double o = 0.0;
    for (int j = 0; j <= i; ++j) o += a[j] * v[(size_t)j * dv + c];
    O[(size_t)i * dv + c] = o;
  }
}

struct KeepParams {
  int stride;
  const int32_t* prompt_len;
  const int32_t* current_len;
  const uint8_t* cls;
  const double* score;
  const uint8_t* cand;
  const uint8_t* atoms;
  const double* r_l;
  const double* r_f;
  uint8_t* keep;
  int32_t* count;
  int32_t* scratch;
};

// one CTA per context: union of the policy's atoms over the candidates;
// FREQUENT = exact top-budget of the candidates by (score desc, pos asc)
__global__ void __launch_bounds__(kOpsThreads) ops_keep_mask(KeepParams p) {
  __shared__ int hist[256];
  __shared__ int red[33];
  const int g = blockIdx.x;
  const int cur = p.current_len[g], plen = p.prompt_len[g];
  const uint8_t at = p.atoms[g];
  const uint8_t* cls = p.cls + (size_t)g * p.stride;
  const double* sc = p.score + (size_t)g * p.stride;
  const uint8_t* cand = p.cand ? p.cand + (size_t)g * p.stride : nullptr;
  uint8_t* keep = p.keep + (size_t)g * p.stride;
  int32_t* list = p.scratch + (size_t)g * p.stride;
  // compact candidate list (ascending positions)
  const int per = (cur + blockDim.x - 1) / blockDim.x;
  const int lo = min(cur, (int)threadIdx.x * per), hi = min(cur, lo + per);
  int mine = 0;
  for (int j = lo; j < hi; ++j) mine += cand ? (cand[j] != 0) : 1;
  int total;
  int off = block_exclusive_scan(mine, red, &total);
  for (int j = lo; j < hi; ++j)
    if (!cand || cand[j]) list[off++] = j;
  __syncthreads();
  unsigned long long tk = ~0ull;
  int tp = -1;
  const bool freq = (at & AKV_ATOM_FREQUENT) && !(at & AKV_ATOM_FULL);
  if (freq && total > 0) {
    const int kb = budget(p.r_f[g], cur);
    auto get = [&](int i, unsigned long long* key, int* pos) {
      const int j = list[i];
      *key = score_key(sc[j]);
      *pos = j;
    };
    block_topk_threshold(total, kb, get, hist, red, &tk, &tp);
  }
  const int ws = cur - budget(p.r_l[g], plen);
  int cnt = 0;
  for (int j = threadIdx.x; j < p.stride; j += blockDim.x) {
    bool k = false;
    if (j < cur && (!cand || cand[j])) {
      if (at & AKV_ATOM_FULL) k = true;
      const int c = cls[j];
      k |= (at & AKV_ATOM_SPECIAL) && c == AKV_CLS_SPECIAL;
      k |= (at & AKV_ATOM_PUNCT) && c == AKV_CLS_PUNCT;
      k |= (at & AKV_ATOM_LOCAL) && j >= ws;
      if (freq) k |= topk_selected(score_key(sc[j]), j, tk, tp);
    }
    keep[j] = k;
    cnt += k;
  }
  cnt = block_sum(cnt, red);
  if (threadIdx.x == 0) p.count[g] = cnt;
}

// one CTA per map: column sums / square sums of A (or its last row), then
// the masked recovery and cosine of every mask
__global__ void __launch_bounds__(kOpsThreads) ops_map_recovery(int n, const double* A, int F,
                                                                const uint8_t* masks, int rows,
                                                                double* col, double* colsq,
                                                                double* recovery, double* cosine) {
  __shared__ double red[kOpsThreads / 32];
  const int g = blockIdx.x;
  const double* a = A + (size_t)g * n * n;
  double* cs = col + (size_t)g * n;
  double* cq = colsq + (size_t)g * n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0, q = 0.0;
    for (int i = 0; i < n; ++i) {
      const double x = a[(size_t)i * n + j];
      s += x;
      q += x * x;
    }
    cs[j] = rows == AKV_ROWS_LAST ? a[(size_t)(n - 1) * n + j] : s;
    cq[j] = q;
  }
  __syncthreads();
  double tq = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) tq += cq[j];
  tq = block_sum(tq, red);
  for (int f = 0; f < F; ++f) {
    const uint8_t* m = masks + ((size_t)g * F + f) * n;
    double s = 0.0, q = 0.0;
    int c = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x)
      if (m[j]) { s += cs[j]; q += cq[j]; ++c; }
    s = block_sum(s, red);
    q = block_sum(q, red);
    c = block_sum(c, reinterpret_cast<int*>(red));
    if (threadIdx.x == 0) {
      recovery[(size_t)g * F + f] = c == 0 ? 0.0 : (rows == AKV_ROWS_LAST ? s : s / n);
      cosine[(size_t)g * F + f] = (c == 0 || q == 0.0) ? 0.0 : sqrt(q) / sqrt(tq);
    }
  }
}

__global__ void ops_update_scores(int L, const double* in, int m, const int32_t* idx,
                                  const double* row, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= L; j += gridDim.x * blockDim.x)
    out[j] = j < L ? in[j] : 0.0;
  // single pass is enough: idx are distinct, but the copy above must land first
}
__global__ void ops_update_scores_add(int m, const int32_t* idx, const double* row, double* out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
    out[idx[t]] += row[t];
}

__global__ void ops_gather_rows(int dk, int dv, const double* K, const double* V, int m,
                                const int32_t* idx, double* Kc, double* Vc) {
  const int r = blockIdx.x;
  const int src = idx[r];
  for (int c = threadIdx.x; c < dk; c += blockDim.x) Kc[(size_t)r * dk + c] = K[(size_t)src * dk + c];
  for (int c = threadIdx.x; c < dv; c += blockDim.x) Vc[(size_t)r * dv + c] = V[(size_t)src * dv + c];
}

__global__ void __launch_bounds__(kOpsThreads) ops_tv_distance(int n, const double* pr,
                                                               const uint8_t* mask, double* out) {
  __shared__ double red[kOpsThreads / 32];
  double mass = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (mask[j]) mass += pr[j];
  mass = block_sum(mass, red);
  if (mass <= 0.0) {
    if (threadIdx.x == 0) *out = 1.0;
    return;
  }
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s += fabs(pr[j] - (mask[j] ? pr[j] / mass : 0.0));
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = 0.5 * s;
}

static int launch_result(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return AKV_OK;
}

}  // namespace akv

using namespace akv;

extern "C" int akv_softmax_rows_f64(int32_t rows, int32_t cols, const double* in,
                                    const int32_t* lengths, double* out, void* stream) {
  if (rows < 1 || cols < 1) return set_error(AKV_ERR_INVALID, "empty input");
  ops_softmax_rows<<<rows, kOpsThreads, 0, static_cast<cudaStream_t>(stream)>>>(cols, in, lengths, out);
  return launch_result("akv_softmax_rows_f64");
}

extern "C" int akv_causal_attention_f64(int32_t n, int32_t dq, int32_t dv, const double* q,
                                        const double* k, const double* v, double scale, double* A,
                                        double* O, void* stream) {
  if (n < 1 || dq < 1 || dv < 1) return set_error(AKV_ERR_INVALID, "empty input");
  ops_causal_attention<<<n, kOpsThreads, 0, static_cast<cudaStream_t>(stream)>>>(n, dq, dv, q, k, v,
                                                                                 scale, A, O);
  return launch_result("akv_causal_attention_f64");
}

extern "C" int akv_keep_mask(const akv_keep_args* a, void* stream) {
  if (!a || a->G < 1 || a->stride < 1) return set_error(AKV_ERR_INVALID, "akv_keep_mask: empty input");
  if (a->stride > kPosMask) return set_error(AKV_ERR_UNSUPPORTED, "akv_keep_mask: context too long");
  KeepParams p{a->stride, a->prompt_len_dev, a->current_len_dev, a->cls_dev, a->score_dev,
               a->cand_dev, a->atoms_dev, a->r_l_dev, a->r_f_dev, a->keep_dev, a->count_dev,
               a->scratch_dev};
  ops_keep_mask<<<a->G, kOpsThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return launch_result("akv_keep_mask");
}

extern "C" int akv_map_recovery_f64(int32_t G, int32_t n, const double* A, int32_t F,
                                    const uint8_t* masks, int32_t rows, double* colsum_ws,
                                    double* colsq_ws, double* recovery, double* cosine,
                                    void* stream) {
  if (G < 1 || n < 1 || F < 1) return set_error(AKV_ERR_INVALID, "empty input");
  ops_map_recovery<<<G, kOpsThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      n, A, F, masks, rows, colsum_ws, colsq_ws, recovery, cosine);
  return launch_result("akv_map_recovery_f64");
}

extern "C" int akv_update_scores_f64(int32_t L, const double* scores_in, int32_t m,
                                     const int32_t* retained, const double* row, double* scores_out,
                                     void* stream) {
  if (L < 0 || m < 0 || m > L) return set_error(AKV_ERR_INVALID, "akv_update_scores_f64: bad sizes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ops_update_scores<<<(L + 256) / 256, 256, 0, st>>>(L, scores_in, m, retained, row, scores_out);
  if (m > 0) ops_update_scores_add<<<(m + 255) / 256, 256, 0, st>>>(m, retained, row, scores_out);
  return launch_result("akv_update_scores_f64");
}

extern "C" int akv_gather_rows_f64(int32_t dk, int32_t dv, const double* K, const double* V,
                                   int32_t m, const int32_t* idx, double* Kc, double* Vc,
                                   void* stream) {
  if (m < 0 || dk < 1 || dv < 1) return set_error(AKV_ERR_INVALID, "akv_gather_rows_f64: bad sizes");
  if (m == 0) return AKV_OK;
  ops_gather_rows<<<m, 128, 0, static_cast<cudaStream_t>(stream)>>>(dk, dv, K, V, m, idx, Kc, Vc);
  return launch_result("akv_gather_rows_f64");
}

extern "C" int akv_tv_distance_f64(int32_t n, const double* p, const uint8_t* mask, double* out,
                                   void* stream) {
  if (n < 1) return set_error(AKV_ERR_INVALID, "empty input");
  ops_tv_distance<<<1, kOpsThreads, 0, static_cast<cudaStream_t>(stream)>>>(n, p, mask, out);
  return launch_result("akv_tv_distance_f64");
}
