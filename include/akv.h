/*
 * akv.h — C ABI of libakv_sm100a.so, the B200 (sm_100a) implementation of
 * FastGen's adaptive-KV hot path: prompt profiling (K1), per-head KV
 * compaction (K2) and compressed decode with fused insert/evict (K3).
 *
 * The reference (arxiv/paper_2310_01801, /root/reference/pkg/src/adaptive_kv)
 * is a pure-Python/numpy package with no FFI; each entry point below replaces
 * the per-head numpy loops of one reference function and is bound from the
 * Python host layer with ctypes:
 *
 *   akv_profile      <- engine.py:161-200  prompt_head_data (causal_attention,
 *                                          A.sum(axis=0)),
 *                       profiler.py:70-87  recovery_ratio,
 *                       profiler.py:135-145 select_policy,
 *                       profiler.py:148-178 select_policy_by_similarity,
 *                       policies.py:244-267 retained_indices (candidates=None),
 *                       engine.py:248,255  pending_output = A[n-1] @ V
 *   akv_compact      <- engine.py:236-259  encode_prompt compaction loop,
 *                       policies.py:270-288 apply_policy
 *   akv_decode_step  <- engine.py:303-350  generate_step per-head body,
 *                       engine.py:93-97    _attend_row,
 *                       policies.py:332-360 update_cumulative_scores,
 *                       policies.py:244-267 retained_indices (candidates=live)
 *
 * Conventions: plain pointers and sizes only.  All pointers named *_dev are
 * device pointers; calls are stream-ordered with no implicit host sync and
 * are reentrant across streams (each call's scratch lives in the caller's
 * workspace).  The caller owns all memory.  Heads are flattened
 * g = b*H + h.  Status codes are returned; akv_last_error() gives a
 * thread-local message.
 */
#ifndef AKV_H
#define AKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define AKV_OK 0
#define AKV_ERR_INVALID 1     /* invalid argument (maps to PolicyError/ProfilerError/EngineError) */
#define AKV_ERR_CAPACITY 2    /* cache segment capacity exceeded / workspace too small */
#define AKV_ERR_UNSUPPORTED 3 /* unsupported shape or dtype */
#define AKV_ERR_CUDA 4        /* CUDA runtime error */

/* element types of Q/K/V and of the compressed cache */
#define AKV_DTYPE_F32 0
#define AKV_DTYPE_BF16 1

/* policy atoms (policies.py:29-34) as bit flags; FULL excludes the others */
#define AKV_ATOM_SPECIAL 1
#define AKV_ATOM_PUNCT 2
#define AKV_ATOM_FREQUENT 4
#define AKV_ATOM_LOCAL 8
#define AKV_ATOM_FULL 16

/* token classes (tokens.py:15-18) */
#define AKV_CLS_OTHER 0
#define AKV_CLS_SPECIAL 1
#define AKV_CLS_PUNCT 2

/* profiler.py:41-48 */
#define AKV_ROWS_ALL 0
#define AKV_ROWS_LAST 1
#define AKV_CRIT_RECOVERY 0
#define AKV_CRIT_COSINE 1

#define AKV_MAX_FAMILY 8
#define AKV_MAX_THRESHOLDS 8

/* ---- K1: prompt profiling ------------------------------------------- */
typedef struct akv_profile_args {
  int32_t B, H, N, d;            /* batch rows, heads, prompt length, head dim (16,32,64,128) */
  int32_t dtype;                 /* AKV_DTYPE_* of q/k/v */
  const void* q_dev;             /* [B,H,ld,d]; rows 0..N-1 of each head are the prompt */
  const void* k_dev;
  const void* v_dev;
  int64_t ld;                    /* rows per head in q/k/v (>= N) */
  const uint8_t* cls_dev;        /* [B,cls_ld] class of every position */
  int64_t cls_ld;
  const float* slope_dev;        /* [H] planted -slope*|i-j| bias, or NULL */
  const float* sink_dev;         /* [H] planted +sink on special keys, or NULL */
  int32_t n_family;              /* feasible family (policies.py:304-329), last usually FULL */
  uint8_t family_atoms[AKV_MAX_FAMILY];
  double family_r_l[AKV_MAX_FAMILY];
  double family_r_f[AKV_MAX_FAMILY];
  int32_t n_thresholds;          /* thresholds[0] drives keep_mask/kept_pos */
  double thresholds[AKV_MAX_THRESHOLDS];
  int32_t rows;                  /* AKV_ROWS_* */
  int32_t criterion;             /* AKV_CRIT_* */
  /* outputs (device, all [B*H,...]) */
  float* lse_dev;                /* [B*H,N] row log-sum-exp */
  double* colsum_dev;            /* [B*H,N] attention mass per key (frequency signal) */
  double* colsq_dev;             /* [B*H,N] sum of squared weights per key (cosine) */
  float* lastp_dev;              /* [B*H,N] A[N-1,:] */
  float* out_last_dev;           /* [B*H,d] A[N-1,:] @ V (pending output) */
  double* recovery_dev;          /* [B*H,n_family] */
  int32_t* cost_dev;             /* [B*H,n_family] retained tokens */
  double* cosine_dev;            /* [B*H,n_family] */
  int8_t* choice_dev;            /* [B*H,n_thresholds] family index, -1 if none met T */
  int32_t* kept_pos_dev;         /* [B*H,N] ascending kept positions of the chosen policy */
  int32_t* kept_count_dev;       /* [B*H] */
  double* last_row_recovery_dev; /* [B*H] A[N-1, kept].sum() */
  double* topk_gap_dev;          /* [B*H] min relative score gap at any frequent boundary */
  uint64_t* topk_thr_key_dev;    /* [B*H] frequent top-k threshold of the primary choice: */
  int32_t* topk_thr_pos_dev;     /*   position p is in the set iff (bits(colsum[p]), -p) >= (key, -pos) */
  void* workspace_dev;
  size_t workspace_bytes;
  int32_t local_len;             /* prompt length anchoring the local budget (0 = N); re-profiling a
                                    prompt plus generated tokens passes the true prompt length
                                    (engine.py:161-176, metrics.py:140-187) */
} akv_profile_args;

size_t akv_profile_workspace_size(int32_t B, int32_t H, int32_t N, int32_t d);
int akv_profile(const akv_profile_args* a, void* stream);

/* ---- K2: compaction into the ragged head-major cache ----------------- */
typedef struct akv_compact_args {
  int32_t B, H, N, d;
  int32_t dtype;
  const void* k_dev;             /* [B,H,ld,d] */
  const void* v_dev;
  int64_t ld;
  const uint8_t* cls_dev;        /* [B,cls_ld] */
  int64_t cls_ld;
  const int32_t* kept_pos_dev;   /* [B*H,N] from akv_profile */
  const int32_t* kept_count_dev; /* [B*H] */
  const double* colsum_dev;      /* [B*H,N] scores copied for FREQUENT heads */
  const int8_t* choice_dev;      /* [B*H,choice_stride] from akv_profile; column 0 is used */
  const uint64_t* topk_thr_key_dev; /* [B*H] from akv_profile: marks the initial frequent set */
  const int32_t* topk_thr_pos_dev;
  int32_t choice_stride;
  int32_t n_family;              /* the family akv_profile chose from */
  uint8_t family_atoms[AKV_MAX_FAMILY];
  double family_r_l[AKV_MAX_FAMILY];
  double family_r_f[AKV_MAX_FAMILY];
  uint8_t* head_atoms_dev;       /* [B*H] out: atoms of each head's chosen policy */
  double* head_r_l_dev;          /* [B*H] out: its r_l */
  double* head_r_f_dev;          /* [B*H] out: its r_f */
  const int64_t* seg_off_dev;    /* [B*H] first slot of each head's segment */
  const int32_t* seg_cap_dev;    /* [B*H] segment capacity (slots) */
  void* kc_dev;                  /* [total_slots,d] compressed K (dtype) */
  void* vc_dev;                  /* [total_slots,d] compressed V */
  int32_t* meta_dev;             /* [total_slots] position | class << 24 */
  double* score_dev;             /* [total_slots] cumulative score (FREQUENT heads) */
  int32_t* live_dev;             /* [B*H] out: live slots */
} akv_compact_args;

int akv_compact(const akv_compact_args* a, void* stream);
/* Device prefix sum of capacities: seg_cap[g] = round_up(kept_count[g] + extra, 8),
 * seg_off = exclusive scan; *total_dev = sum (int64).  Lets the host size the
 * arena with a single 8-byte device->host read. */
int akv_plan_segments(int32_t G, const int32_t* kept_count_dev, int32_t extra,
                      int32_t* seg_cap_dev, int64_t* seg_off_dev, int64_t* total_dev,
                      void* stream);

/* The same plan carved from a device-side arena pool (bump allocator over
 * [0, pool_slots) slots of caller-owned kc/vc/meta/score arrays): this call's
 * segments start at base = atomicAdd(*pool_used_dev, total), so the
 * compaction can follow without any host read.  If the pool cannot hold them,
 * every seg_cap is 0 (compaction and decode skip the heads) and *status_dev =
 * AKV_ERR_CAPACITY.  Resetting *pool_used_dev (stream-ordered) frees the
 * pool. */
int akv_plan_segments_pool(int32_t G, const int32_t* kept_count_dev, int32_t extra,
                           int32_t* seg_cap_dev, int64_t* seg_off_dev, int64_t* total_dev,
                           unsigned long long* pool_used_dev, int64_t pool_slots,
                           int32_t* status_dev, void* stream);

/* ---- K3: one decode step over the compressed cache ------------------- */
typedef struct akv_decode_args {
  int32_t B, H, d;
  int32_t dtype;
  int32_t prompt_len;            /* local budget anchor (policies.py:209-211) */
  int32_t pos;                   /* position of the inserted token; current_len = pos+1 */
  const void* q_dev;             /* [B,H,d] query of the new token */
  const void* k_dev;             /* [B,H,d] key/value rows of the new token (inserted) */
  const void* v_dev;
  int64_t bh_stride;             /* elements between consecutive heads of q/k/v (>= d) */
  const uint8_t* new_cls_dev;    /* [B] class of the new token */
  const float* slope_dev;        /* [H] or NULL */
  const float* sink_dev;         /* [H] or NULL */
  const uint8_t* head_atoms_dev; /* [B*H] */
  const double* head_r_l_dev;    /* [B*H] */
  const double* head_r_f_dev;    /* [B*H] */
  const int64_t* seg_off_dev;    /* [B*H] */
  const int32_t* seg_cap_dev;    /* [B*H] */
  void* kc_dev;
  void* vc_dev;
  int32_t* meta_dev;
  double* score_dev;
  const int32_t* base_live_dev;  /* [B*H] live slots right after compaction (akv_compact's live):
                                    base_live + (pos - prompt_len) bounds live_in and equals it
                                    for full-cache heads, which lets a step start streaming
                                    before the previous step has drained */
  const int32_t* live_in_dev;    /* [B*H] live slots before the step */
  int32_t* live_out_dev;         /* [B*H] live slots after insert+evict (distinct buffer) */
  float* out_dev;                /* [B,H,d] attention output (fp32) */
  int32_t* evicted_dev;          /* [B*H] evictions this step (optional, may be NULL) */
  int32_t* status_dev;           /* [1] sticky device status (capacity overflow), may be NULL */
  int32_t max_cap;               /* max over heads of seg_cap (sizes the grid) */
  int64_t total_slots;           /* arena slots (sizes the logit scratch) */
  void* workspace_dev;
  size_t workspace_bytes;
  const int32_t* pos_dev;        /* optional device position of the inserted token; when set it
                                    replaces pos (so a captured CUDA graph can be replayed for
                                    successive steps) */
  int32_t flags;                 /* AKV_DECODE_* */
  float* lse_out_dev;            /* optional [B*H] natural-log log-sum-exp of each head's attended
                                    logits (live slots + the new token), for diagnostics */
  void* const* peer_out_dev;     /* optional device array of n_peers pointers, each to a
                                    [B, peer_ld] buffer (cache dtype) that receives this call's
                                    head outputs at columns peer_col0 + h*d: the cross-shard
                                    gather of a head-sharded layer fused into the combine
                                    (peer pointers from CUDA IPC / symmetric memory; the caller
                                    barriers before reading) */
  int32_t n_peers;
  int64_t peer_ld;
  int64_t peer_col0;
} akv_decode_args;

/* akv_decode_args.flags: the previous kernel on the stream is this cache's
 * previous decode step and q/k/v/new_cls were complete before it started, so
 * the step may stream settled full-cache pages before that kernel drains
 * (programmatic dependent launch).  Without it the step waits for its
 * predecessor before reading anything. */
#define AKV_DECODE_CHAINED 1

size_t akv_decode_workspace_size(int32_t B, int32_t H, int32_t d, int32_t max_cap, int64_t total_slots);
int akv_decode_step(const akv_decode_args* a, void* stream);
/* n_steps consecutive teacher-forced decode steps in one call (engine.py:283-371
 * applied n times with known tokens: trace replay, benchmarks, prompt-extension
 * checks): step s inserts position pos + s, reads q/k/v at *_dev + s*step_stride
 * elements and classes at new_cls_dev + s*cls_step_stride; live counts
 * alternate between live_in_dev and live_out_dev (after the call they are in
 * live_out_dev for odd n_steps, live_in_dev for even); step s writes its output
 * to out_steps + s*out_step_stride (fp32), or to out_dev when out_steps is
 * NULL.  `flags` apply to step 0; later steps are chained.  pos_dev must be
 * NULL. */
int akv_decode_steps(const akv_decode_args* a, int32_t n_steps, int64_t step_stride,
                     int64_t cls_step_stride, float* out_steps, int64_t out_step_stride,
                     void* stream);
/* Zero the decode workspace counters (call once after allocating it). */
int akv_decode_workspace_init(void* workspace_dev, size_t workspace_bytes, int32_t B, int32_t H,
                              int32_t d, int32_t max_cap, int64_t total_slots, void* stream);


/* ---- diagnostics: per-step recovery against uncompressed attention -----
 * Replaces engine.py:341-349 (shadow keys, full softmax of the new query,
 * recovery = mass on the attended positions).  Launch BEFORE
 * akv_decode_step of the same position (live_in is the pre-eviction live set
 * whose positions plus the new one are "attended"); it appends the new key
 * to the position-indexed shadow rows (and the class to cls_hist), streams
 * every shadow key once and writes the per-head recovery. */
typedef struct akv_diag_args {
  int32_t B, H, d, dtype;
  int32_t pos;                   /* position of the new token (ignored when pos_dev is set) */
  const int32_t* pos_dev;        /* optional device position (graph replays) */
  const void* q_dev;             /* [B,H,d] rows of the new token, head stride bh_stride */
  const void* k_dev;
  int64_t bh_stride;
  const uint8_t* new_cls_dev;    /* [B] */
  const float* slope_dev;        /* [H] or NULL (planted bias, as in the decode step) */
  const float* sink_dev;         /* [H] or NULL */
  const int64_t* seg_off_dev;    /* the cache's segments, live counts and slot metadata */
  const int32_t* live_in_dev;
  const int32_t* meta_dev;
  void* shadow_dev;              /* [B*H, shadow_ld, d] every key by position (in/out) */
  int64_t shadow_ld;
  uint8_t* cls_hist_dev;         /* [B, cls_ld] class of every position (in/out), or NULL */
  int64_t cls_ld;
  double* recovery_dev;          /* [B*H] out */
  const uint8_t* head_atoms_dev; /* optional [B*H] policy atoms (akv_compact): full-cache heads
                                    report 1 exactly and skip the shadow stream */
  void* workspace_dev;           /* akv_decode_recovery_workspace_size bytes, initialised once */
  size_t workspace_bytes;
} akv_diag_args;
size_t akv_decode_recovery_workspace_size(int32_t B, int32_t H, int64_t shadow_ld);
int akv_decode_recovery_workspace_init(void* workspace_dev, size_t workspace_bytes, int32_t B,
                                       int32_t H, int64_t shadow_ld, void* stream);
int akv_decode_recovery(const akv_diag_args* a, void* stream);

/* ---- reference single-context operations (float64, batched) ----------
 * The reference's building blocks besides the fused session path, so the
 * Python mirror of attention.py / policies.py / profiler.py runs on the GPU.
 */
/* attention.py:64-89 softmax_rows: row r normalised over its first lengths[r]
 * columns (all columns when lengths is NULL), the rest exactly 0 */
int akv_softmax_rows_f64(int32_t rows, int32_t cols, const double* in_dev,
                         const int32_t* lengths_dev, double* out_dev, void* stream);
/* attention.py:102-127 causal_attention: A = causal softmax(q k^T * scale), O = A v */
int akv_causal_attention_f64(int32_t n, int32_t dq, int32_t dv, const double* q_dev,
                             const double* k_dev, const double* v_dev, double scale,
                             double* A_dev, double* O_dev, void* stream);

/* policies.py:214-267 retained_indices over G independent contexts (one
 * policy each); count = cache_memory_cost (policies.py:291-293) */
typedef struct akv_keep_args {
  int32_t G;
  int32_t stride;                 /* positions per context row (>= every current_len) */
  const int32_t* prompt_len_dev;  /* [G] */
  const int32_t* current_len_dev; /* [G] */
  const uint8_t* cls_dev;         /* [G,stride] class per position */
  const double* score_dev;        /* [G,stride] cumulative scores */
  const uint8_t* cand_dev;        /* [G,stride] candidate flags, or NULL (all < current_len) */
  const uint8_t* atoms_dev;       /* [G] policy atoms */
  const double* r_l_dev;          /* [G] */
  const double* r_f_dev;          /* [G] */
  uint8_t* keep_dev;              /* [G,stride] out */
  int32_t* count_dev;             /* [G] out */
  int32_t* scratch_dev;           /* [G,stride] workspace */
} akv_keep_args;
int akv_keep_mask(const akv_keep_args* a, void* stream);

/* profiler.py:70-87 recovery_ratio and :148-161 masked_cosine_similarity of
 * F retained masks on each of G dense maps A [G,n,n] */
int akv_map_recovery_f64(int32_t G, int32_t n, const double* A_dev, int32_t F,
                         const uint8_t* masks_dev, int32_t rows, double* colsum_ws_dev,
                         double* colsq_ws_dev, double* recovery_dev, double* cosine_dev,
                         void* stream);
/* policies.py:332-360 update_cumulative_scores: out[:L] = in, out[L] = 0,
 * out[retained[t]] += row[t] */
int akv_update_scores_f64(int32_t L, const double* scores_in_dev, int32_t m,
                          const int32_t* retained_dev, const double* row_dev,
                          double* scores_out_dev, void* stream);
/* policies.py:270-288 apply_policy: Kc[r] = K[idx[r]], Vc[r] = V[idx[r]] */
int akv_gather_rows_f64(int32_t dk, int32_t dv, const double* K_dev, const double* V_dev,
                        int32_t m, const int32_t* idx_dev, double* Kc_dev, double* Vc_dev,
                        void* stream);
/* profiler.py:51-67 tv_distance_row */
int akv_tv_distance_f64(int32_t n, const double* p_dev, const uint8_t* mask_dev, double* out_dev,
                        void* stream);

/* ---- model caller (multi-layer decoder around K1-K3) ------------------
 * The per-layer glue of a Llama-style decoder that produces the q/k/v rows
 * the reference's model protocol hands to the engine (model.py:219-286)
 * and consumes the concatenated head outputs (engine.py:354-357).  dtype is
 * AKV_DTYPE_F32 or AKV_DTYPE_BF16 for every tensor of a call; rows are
 * contiguous and 16-byte aligned. */
/* x_out[t] = emb[ids[t]] (emb may be NULL), cls_out[t] = lut[ids[t]] (may be NULL) */
int akv_embed_classify(int32_t n, const int64_t* ids_dev, int32_t vocab, const uint8_t* lut_dev,
                       const void* emb_dev, int32_t dm, int32_t dtype, void* x_out_dev,
                       uint8_t* cls_out_dev, void* stream);
/* residual += x (x may be NULL); out = residual * rsqrt(mean(residual^2) + eps) * w */
int akv_add_rmsnorm(int32_t rows, int32_t dim, int32_t dtype, const void* x_dev,
                    void* residual_dev, const void* w_dev, float eps, void* out_dev,
                    void* stream);
/* Tensor-parallel decode: the all-reduce of row-parallel partial products
 * fused with its consumer.  peer_ptrs_dev[r] (device array of n_peers
 * addresses, rank order) points at rank r's [rows, peer_ld] partial -
 * symmetric memory mapped over NVLink; the caller runs a cross-rank barrier
 * after the partials are written.  residual += sum_r partial_r (fp32 sum in
 * rank order, rounded to dtype: identical bits on every rank); out =
 * residual * rsqrt(mean(residual^2) + eps) * w.  Replaces an all_reduce
 * followed by akv_add_rmsnorm. */
int akv_add_rmsnorm_peers(int32_t rows, int32_t dim, int32_t dtype, const uint64_t* peer_ptrs_dev,
                          int32_t n_peers, int64_t peer_ld, void* residual_dev, const void* w_dev,
                          float eps, void* out_dev, void* stream);
typedef struct akv_rope_args {
  int32_t T;                  /* token rows of qkv; T % n == 0 */
  int32_t n;                  /* rows per sequence: token t = b*n + i */
  int32_t Hl, d, dtype;       /* heads in this projection, head dim */
  const void* qkv_dev;        /* row t: [q heads Hl*d | k heads Hl*d | v heads Hl*d] */
  int64_t qkv_ld;             /* elements between rows of qkv */
  int32_t pos0;               /* RoPE position of i = 0 */
  int32_t max_pos;            /* rows of the cos/sin tables */
  const float* cos_dev;       /* [max_pos, d/2] */
  const float* sin_dev;
  void* q_dev;                /* out [B, Hl, out_ld, d]: token (b, i) -> row row0 + i */
  void* k_dev;
  void* v_dev;
  int64_t out_ld;
  int32_t row0;
  const int32_t* pos_dev;     /* optional device base added to pos0 (graph replays); positions
                                 past the table are clamped to its last row */
} akv_rope_args;
/* rotate-half RoPE of q and k, copy of v, scattered head-major */
int akv_rope_scatter(const akv_rope_args* a, void* stream);
/* out[r, c] = silu(gu[r, c]) * gu[r, F + c] */
int akv_swiglu(int32_t rows, int32_t F, int32_t dtype, const void* gu_dev, void* out_dev,
               void* stream);
/* tokens[b] = first argmax of logits[b, :V]; cls[b] = lut[token] (may be NULL);
 * x_out[b] = emb[token] (emb may be NULL) */
int akv_greedy_next(int32_t B, int32_t V, int32_t dtype, const void* logits_dev, int64_t ld,
                    const uint8_t* lut_dev, const void* emb_dev, int32_t dm, int64_t* tokens_dev,
                    uint8_t* cls_dev, void* x_out_dev, void* stream);

/* ---- misc ------------------------------------------------------------ */
const char* akv_last_error(void);
const char* akv_version(void);
int akv_device_check(void);   /* AKV_OK iff a sm_100 device is current */

#ifdef __cplusplus
}
#endif
#endif /* AKV_H */
