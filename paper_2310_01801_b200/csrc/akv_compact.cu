// K2: per-head KV compaction into the ragged, head-major compressed cache.
//
// Replaces the reference's encode_prompt compaction loop (engine.py:236-259):
// retained_indices -> apply_policy (policies.py:270-288, rows gathered in
// ascending position order) and the FREQUENT-only score copy
// (engine.py:243-247).  Each head g owns slots [seg_off[g], seg_off[g] +
// seg_cap[g]) of the arena; the kept rows fill the first kept_count[g]
// slots and decode appends after them.  Rows move as 16-byte vectors,
// a warp covering whole rows so loads and stores stay coalesced.

#include "akv_common.cuh"
#include "akv_internal.h"

namespace akv {

constexpr int kCompactRows = 32;

struct CompactParams {
  int H, N, row_vecs;  // 16-byte vectors per row
  const uint4* k;
  const uint4* v;
  int64_t ld;
  const uint8_t* cls;
  int64_t cls_ld;
  const int32_t* kept_pos;
  const int32_t* kept_count;
  const double* colsum;
  const int8_t* choice;
  const unsigned long long* thr_key;
  const int32_t* thr_pos;
  int choice_stride;
  int n_family;
  uint8_t fam_atoms[AKV_MAX_FAMILY];
  double fam_r_l[AKV_MAX_FAMILY];
  double fam_r_f[AKV_MAX_FAMILY];
  uint8_t* atoms;
  double* r_l;
  double* r_f;
  const int64_t* seg_off;
  const int32_t* seg_cap;
  uint4* kc;
  uint4* vc;
  int32_t* meta;
  double* score;
  int32_t* live;
};

__global__ void __launch_bounds__(128) k2_compact(CompactParams p) {
  const int g = blockIdx.y;
  const int kept = p.kept_count[g];
  const int cap = p.seg_cap[g];
  const int i0 = blockIdx.x * kCompactRows;
  int c = p.choice[(size_t)g * p.choice_stride];
  c = (c >= 0 && c < p.n_family) ? c : p.n_family - 1;
  const uint8_t at = p.fam_atoms[c];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // a segment too small for its kept rows is reported as live = -1
    p.live[g] = kept > cap ? -1 : kept;
    p.atoms[g] = at;  // per-head policy table for decode
    p.r_l[g] = p.fam_r_l[c];
    p.r_f[g] = p.fam_r_f[c];
  }
  if (i0 >= kept || kept > cap) return;
  const int nrows = min(kCompactRows, kept - i0);
  const int64_t base = p.seg_off[g];
  const int b = g / p.H;
  const int32_t* kp = p.kept_pos + (size_t)g * p.N;
  const uint4* ksrc = p.k + (size_t)g * p.ld * p.row_vecs;
  const uint4* vsrc = p.v + (size_t)g * p.ld * p.row_vecs;
  for (int idx = threadIdx.x; idx < nrows * p.row_vecs; idx += blockDim.x) {
    const int r = idx / p.row_vecs, c = idx % p.row_vecs;
    const int pos = kp[i0 + r];
    const size_t dst = (size_t)(base + i0 + r) * p.row_vecs + c;
    const uint4 kv = ld_nc_v4(ksrc + (size_t)pos * p.row_vecs + c);
    const uint4 vv = ld_nc_v4(vsrc + (size_t)pos * p.row_vecs + c);
    st_v4(p.kc + dst, kv);
    st_v4(p.vc + dst, vv);
  }
  const bool freq = (at & AKV_ATOM_FREQUENT) && !(at & AKV_ATOM_FULL);
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    const int pos = kp[i0 + r];
    const int64_t slot = base + i0 + r;
    const double sc = freq ? p.colsum[(size_t)g * p.N + pos] : 0.0;
    const bool inF = freq && topk_selected(score_key(sc), pos,
                                           p.thr_key[g], p.thr_pos[g]);
    p.meta[slot] = pos | ((int)p.cls[(size_t)b * p.cls_ld + pos] << kClsShift) | (inF ? kInF : 0);
    p.score[slot] = sc;
  }
}

constexpr int kPlanThreads = 1024;

// one CTA: each thread owns a contiguous run of heads; block scan of the
// run totals (8-slot aligned segments)
__global__ void __launch_bounds__(kPlanThreads) k2_plan(int G, const int32_t* kept, int32_t extra,
                                                        int32_t* cap, int64_t* off, int64_t* total) {
  __shared__ int red[kPlanThreads / 32 + 1];
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int lo = min(G, (int)threadIdx.x * per), hi = min(G, lo + per);
  int mine = 0;
  for (int g = lo; g < hi; ++g) mine += ((kept[g] + extra + 7) / 8) * 8;
  int tot;
  int acc = block_exclusive_scan(mine, red, &tot);
  for (int g = lo; g < hi; ++g) {
    const int c = ((kept[g] + extra + 7) / 8) * 8;
    cap[g] = c;
    off[g] = acc;
    acc += c;
  }
  if (threadIdx.x == 0) *total = tot;
}

// The same plan carved from a device-side arena pool (bump allocator): the
// segments of this call start at base = atomicAdd(pool_used, total), so no
// host read is needed before the compaction.  A pool that cannot hold them
// zeroes every capacity (compaction and decode then skip the heads) and
// flags AKV_ERR_CAPACITY.
__global__ void __launch_bounds__(kPlanThreads) k2_plan_pool(int G, const int32_t* kept,
                                                             int32_t extra, int32_t* cap,
                                                             int64_t* off, int64_t* total,
                                                             unsigned long long* pool_used,
                                                             int64_t pool_slots, int32_t* status) {
  __shared__ int red[kPlanThreads / 32 + 1];
  __shared__ long long s_base;
  const int per = (G + blockDim.x - 1) / blockDim.x;
  const int lo = min(G, (int)threadIdx.x * per), hi = min(G, lo + per);
  int mine = 0;
  for (int g = lo; g < hi; ++g) mine += ((kept[g] + extra + 7) / 8) * 8;
  int tot;
  int acc = block_exclusive_scan(mine, red, &tot);
  if (threadIdx.x == 0) {
    const unsigned long long b = atomicAdd(pool_used, (unsigned long long)tot);
    if ((long long)(b + tot) > pool_slots) {
      atomicExch(status, AKV_ERR_CAPACITY);
      s_base = -1;
    } else {
      s_base = (long long)b;
    }
    *total = tot;
  }
  __syncthreads();
  const long long base = s_base;
  for (int g = lo; g < hi; ++g) {
    const int c = ((kept[g] + extra + 7) / 8) * 8;
    cap[g] = base < 0 ? 0 : c;
    off[g] = base < 0 ? 0 : base + acc;
    acc += c;
  }
}

}  // namespace akv

using namespace akv;

extern "C" int akv_plan_segments_pool(int32_t G, const int32_t* kept_count_dev, int32_t extra,
                                      int32_t* seg_cap_dev, int64_t* seg_off_dev,
                                      int64_t* total_dev, unsigned long long* pool_used_dev,
                                      int64_t pool_slots, int32_t* status_dev, void* stream) {
  if (G < 1 || extra < 0 || !pool_used_dev || !status_dev || pool_slots < 1)
    return set_error(AKV_ERR_INVALID, "akv_plan_segments_pool: bad arguments");
  k2_plan_pool<<<1, kPlanThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      G, kept_count_dev, extra, seg_cap_dev, seg_off_dev, total_dev, pool_used_dev, pool_slots,
      status_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_plan_segments_pool: %s", cudaGetErrorString(e));
  return AKV_OK;
}

extern "C" int akv_plan_segments(int32_t G, const int32_t* kept_count_dev, int32_t extra,
                                 int32_t* seg_cap_dev, int64_t* seg_off_dev, int64_t* total_dev,
                                 void* stream) {
  if (G < 1 || extra < 0) return set_error(AKV_ERR_INVALID, "akv_plan_segments: bad G/extra");
  k2_plan<<<1, kPlanThreads, 0, static_cast<cudaStream_t>(stream)>>>(G, kept_count_dev, extra,
                                                                    seg_cap_dev, seg_off_dev,
                                                                    total_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_plan_segments: %s", cudaGetErrorString(e));
  return AKV_OK;
}

extern "C" int akv_compact(const akv_compact_args* a, void* stream) {
  if (!a) return set_error(AKV_ERR_INVALID, "akv_compact: null args");
  if (a->B < 1 || a->H < 1 || a->N < 1) return set_error(AKV_ERR_INVALID, "akv_compact: empty input");
  const int es = a->dtype == AKV_DTYPE_BF16 ? 2 : a->dtype == AKV_DTYPE_F32 ? 4 : 0;
  if (!es || (a->d * es) % 16 || a->d * es > 512)
    return set_error(AKV_ERR_UNSUPPORTED, "akv_compact: unsupported dtype %d / head dim %d", a->dtype, a->d);
  if (a->n_family < 1 || a->n_family > AKV_MAX_FAMILY || a->choice_stride < 1)
    return set_error(AKV_ERR_INVALID, "akv_compact: bad family / choice stride");
  CompactParams p{};
  p.H = a->H; p.N = a->N; p.row_vecs = a->d * es / 16;
  p.k = static_cast<const uint4*>(a->k_dev); p.v = static_cast<const uint4*>(a->v_dev); p.ld = a->ld;
  p.cls = a->cls_dev; p.cls_ld = a->cls_ld;
  p.kept_pos = a->kept_pos_dev; p.kept_count = a->kept_count_dev; p.colsum = a->colsum_dev;
  p.choice = a->choice_dev; p.choice_stride = a->choice_stride; p.n_family = a->n_family;
  p.thr_key = reinterpret_cast<const unsigned long long*>(a->topk_thr_key_dev);
  p.thr_pos = a->topk_thr_pos_dev;
  if (!p.thr_key || !p.thr_pos)
    return set_error(AKV_ERR_INVALID, "akv_compact: topk threshold inputs are required");
  for (int f = 0; f < a->n_family; ++f) {
    p.fam_atoms[f] = a->family_atoms[f]; p.fam_r_l[f] = a->family_r_l[f]; p.fam_r_f[f] = a->family_r_f[f];
  }
  p.atoms = a->head_atoms_dev; p.r_l = a->head_r_l_dev; p.r_f = a->head_r_f_dev;
  p.seg_off = a->seg_off_dev; p.seg_cap = a->seg_cap_dev;
  p.kc = static_cast<uint4*>(a->kc_dev); p.vc = static_cast<uint4*>(a->vc_dev);
  p.meta = a->meta_dev; p.score = a->score_dev; p.live = a->live_dev;
  dim3 grid((a->N + kCompactRows - 1) / kCompactRows, a->B * a->H);
  k2_compact<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(AKV_ERR_CUDA, "akv_compact: %s", cudaGetErrorString(e));
  return AKV_OK;
}
