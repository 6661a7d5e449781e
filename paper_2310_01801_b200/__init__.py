"""B200-native FastGen adaptive KV cache (arXiv 2310.01801).

Drop-in for the reference package's profiling / policy / cache hot path
(``adaptive_kv``: encode_prompt, generate_step, ...), backed by hand-written
sm_100a kernels in ``libakv_sm100a.so`` (include/akv.h).  Importing the
package loads the library and fails if it has not been built; compute
calls fail unless an sm_100 device is present.  There is no CPU fallback.
"""

from ._lib import AkvError, lib as _lib_handle  # noqa: F401  (loads the .so)
from .attention import (AttentionError, AttentionMap, causal_attention, softmax_rows,
                        softmax_vector)
from .engine import (ArenaPool, CompressedCache, EngineError, GenerationConfig, GenerationResult,
                     HeadCacheState,
                     GreedyArgmax, Nucleus, ProfileResult, StepRecord, decode_step_tensors,
                     decode_steps_tensors,
                     encode_prompt, encode_prompt_tensors, generate, generate_fixed_baseline,
                     generate_step, grow_cache, records_to_ndjson, reference_generate)
from .policies import (DEFAULT_FEASIBLE_ORDER, DEFAULT_RATIO, CompressionPolicy, PolicyAtom,
                       PolicyContext, PolicyError, RetainedSet, apply_policy, cache_memory_cost,
                       feasible_set, format_policy, full_policy, local_budget, parse_policy,
                       retained_indices, update_cumulative_scores)
from .profiler import (HeadDecision, HeadProfile, ProfilerConfig, ProfilerError, RecoveryReport,
                       RowAveraging, SelectionCriterion, evaluate_policy, masked_cosine_similarity,
                       profile_model, recovery_ratio, select_policy, select_policy_by_similarity,
                       tv_distance_row)
from .tokens import TokenAnnotation, TokenClass, VocabMetadata, classify_tokens
from .metrics import (MemoryModel, MetricsError, TradeoffPoint, compare_adaptive_vs_fixed,
                      consistency_report, full_cache_bytes, layer_distribution_report,
                      pruned_ratio, sidecar_overhead_fraction, tradeoff_curve)
from .trace import (AttentionTrace, ModelConfig, ModelError, TraceBlock, TraceDimensionError,
                    TraceError, TraceHeaderError, TraceModel, TraceTruncatedError, read_trace,
                    replay_tensors, trace_tensors, write_trace, write_trace_ndjson)

__version__ = "0.1.0"
