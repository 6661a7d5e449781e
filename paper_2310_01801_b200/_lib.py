"""ctypes binding of libakv_sm100a.so (include/akv.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the shared object is missing the import fails, and compute
entry points raise when no sm_100 device is present.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AKV_LIB (experiments only): load another build of the library, e.g. an
# A/B variant built by tools/build_variant.sh
LIB_PATH = os.environ.get("AKV_LIB") or os.path.join(_HERE, "libakv_sm100a.so")

AKV_OK, AKV_ERR_INVALID, AKV_ERR_CAPACITY, AKV_ERR_UNSUPPORTED, AKV_ERR_CUDA = range(5)
DTYPE_F32, DTYPE_BF16 = 0, 1
ATOM_SPECIAL, ATOM_PUNCT, ATOM_FREQUENT, ATOM_LOCAL, ATOM_FULL = 1, 2, 4, 8, 16
ROWS_ALL, ROWS_LAST = 0, 1
CRIT_RECOVERY, CRIT_COSINE = 0, 1
MAX_FAMILY = 8
MAX_THRESHOLDS = 8
DECODE_CHAINED = 1

P = C.c_void_p
i32, i64, f64, sz = C.c_int32, C.c_int64, C.c_double, C.c_size_t


class ProfileArgs(C.Structure):
    _fields_ = [
        ("B", i32), ("H", i32), ("N", i32), ("d", i32), ("dtype", i32),
        ("q_dev", P), ("k_dev", P), ("v_dev", P), ("ld", i64),
        ("cls_dev", P), ("cls_ld", i64), ("slope_dev", P), ("sink_dev", P),
        ("n_family", i32), ("family_atoms", C.c_uint8 * MAX_FAMILY),
        ("family_r_l", f64 * MAX_FAMILY), ("family_r_f", f64 * MAX_FAMILY),
        ("n_thresholds", i32), ("thresholds", f64 * MAX_THRESHOLDS),
        ("rows", i32), ("criterion", i32),
        ("lse_dev", P), ("colsum_dev", P), ("colsq_dev", P), ("lastp_dev", P),
        ("out_last_dev", P), ("recovery_dev", P), ("cost_dev", P), ("cosine_dev", P),
        ("choice_dev", P), ("kept_pos_dev", P), ("kept_count_dev", P),
        ("last_row_recovery_dev", P), ("topk_gap_dev", P), ("topk_thr_key_dev", P),
        ("topk_thr_pos_dev", P), ("workspace_dev", P), ("workspace_bytes", sz),
        ("local_len", i32),
    ]


class CompactArgs(C.Structure):
    _fields_ = [
        ("B", i32), ("H", i32), ("N", i32), ("d", i32), ("dtype", i32),
        ("k_dev", P), ("v_dev", P), ("ld", i64), ("cls_dev", P), ("cls_ld", i64),
        ("kept_pos_dev", P), ("kept_count_dev", P), ("colsum_dev", P), ("choice_dev", P),
        ("topk_thr_key_dev", P), ("topk_thr_pos_dev", P), ("choice_stride", i32), ("n_family", i32), ("family_atoms", C.c_uint8 * MAX_FAMILY),
        ("family_r_l", f64 * MAX_FAMILY), ("family_r_f", f64 * MAX_FAMILY),
        ("head_atoms_dev", P), ("head_r_l_dev", P), ("head_r_f_dev", P),
        ("seg_off_dev", P), ("seg_cap_dev", P), ("kc_dev", P), ("vc_dev", P),
        ("meta_dev", P), ("score_dev", P), ("live_dev", P),
    ]


class DecodeArgs(C.Structure):
    _fields_ = [
        ("B", i32), ("H", i32), ("d", i32), ("dtype", i32), ("prompt_len", i32), ("pos", i32),
        ("q_dev", P), ("k_dev", P), ("v_dev", P), ("bh_stride", i64), ("new_cls_dev", P),
        ("slope_dev", P), ("sink_dev", P), ("head_atoms_dev", P), ("head_r_l_dev", P),
        ("head_r_f_dev", P), ("seg_off_dev", P), ("seg_cap_dev", P), ("kc_dev", P),
        ("vc_dev", P), ("meta_dev", P), ("score_dev", P), ("base_live_dev", P), ("live_in_dev", P),
        ("live_out_dev", P), ("out_dev", P), ("evicted_dev", P), ("status_dev", P),
        ("max_cap", i32), ("total_slots", i64), ("workspace_dev", P), ("workspace_bytes", sz),
        ("pos_dev", P), ("flags", i32), ("lse_out_dev", P), ("peer_out_dev", P),
        ("n_peers", i32), ("peer_ld", i64), ("peer_col0", i64),
    ]


class KeepArgs(C.Structure):
    _fields_ = [
        ("G", i32), ("stride", i32), ("prompt_len_dev", P), ("current_len_dev", P),
        ("cls_dev", P), ("score_dev", P), ("cand_dev", P), ("atoms_dev", P), ("r_l_dev", P),
        ("r_f_dev", P), ("keep_dev", P), ("count_dev", P), ("scratch_dev", P),
    ]


class RopeArgs(C.Structure):
    _fields_ = [
        ("T", i32), ("n", i32), ("Hl", i32), ("d", i32), ("dtype", i32), ("qkv_dev", P),
        ("qkv_ld", i64), ("pos0", i32), ("max_pos", i32), ("cos_dev", P), ("sin_dev", P),
        ("q_dev", P), ("k_dev", P), ("v_dev", P), ("out_ld", i64), ("row0", i32),
        ("pos_dev", P),
    ]


class DiagArgs(C.Structure):
    _fields_ = [
        ("B", i32), ("H", i32), ("d", i32), ("dtype", i32), ("pos", i32), ("pos_dev", P),
        ("q_dev", P), ("k_dev", P), ("bh_stride", i64), ("new_cls_dev", P), ("slope_dev", P),
        ("sink_dev", P), ("seg_off_dev", P), ("live_in_dev", P), ("meta_dev", P),
        ("shadow_dev", P), ("shadow_ld", i64), ("cls_hist_dev", P), ("cls_ld", i64),
        ("recovery_dev", P), ("head_atoms_dev", P), ("workspace_dev", P), ("workspace_bytes", sz),
    ]


# every symbol include/akv.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "akv_profile_workspace_size", "akv_profile", "akv_compact", "akv_plan_segments",
    "akv_plan_segments_pool",
    "akv_decode_workspace_size", "akv_decode_step", "akv_decode_steps", "akv_decode_workspace_init",
    "akv_decode_recovery", "akv_decode_recovery_workspace_size",
    "akv_decode_recovery_workspace_init",
    "akv_softmax_rows_f64", "akv_causal_attention_f64", "akv_keep_mask", "akv_map_recovery_f64",
    "akv_update_scores_f64", "akv_gather_rows_f64", "akv_tv_distance_f64",
    "akv_embed_classify", "akv_add_rmsnorm", "akv_add_rmsnorm_peers", "akv_rope_scatter",
    "akv_swiglu", "akv_greedy_next", "akv_last_error", "akv_version", "akv_device_check",
)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
            "(nvcc -gencode arch=compute_100a,code=sm_100a); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    lib.akv_profile_workspace_size.restype = sz
    lib.akv_profile_workspace_size.argtypes = [i32, i32, i32, i32]
    lib.akv_profile.restype = C.c_int
    lib.akv_profile.argtypes = [C.POINTER(ProfileArgs), P]
    lib.akv_compact.restype = C.c_int
    lib.akv_compact.argtypes = [C.POINTER(CompactArgs), P]
    lib.akv_plan_segments.restype = C.c_int
    lib.akv_plan_segments.argtypes = [i32, P, i32, P, P, P, P]
    lib.akv_plan_segments_pool.restype = C.c_int
    lib.akv_plan_segments_pool.argtypes = [i32, P, i32, P, P, P, P, i64, P, P]
    lib.akv_decode_workspace_size.restype = sz
    lib.akv_decode_workspace_size.argtypes = [i32, i32, i32, i32, i64]
    lib.akv_decode_step.restype = C.c_int
    lib.akv_decode_step.argtypes = [C.POINTER(DecodeArgs), P]
    lib.akv_decode_steps.restype = C.c_int
    lib.akv_decode_steps.argtypes = [C.POINTER(DecodeArgs), i32, i64, i64, P, i64, P]
    lib.akv_decode_workspace_init.restype = C.c_int
    lib.akv_decode_workspace_init.argtypes = [P, sz, i32, i32, i32, i32, i64, P]
    lib.akv_softmax_rows_f64.argtypes = [i32, i32, P, P, P, P]
    lib.akv_causal_attention_f64.argtypes = [i32, i32, i32, P, P, P, f64, P, P, P]
    lib.akv_keep_mask.argtypes = [C.POINTER(KeepArgs), P]
    lib.akv_map_recovery_f64.argtypes = [i32, i32, P, i32, P, i32, P, P, P, P, P]
    lib.akv_update_scores_f64.argtypes = [i32, P, i32, P, P, P, P]
    lib.akv_gather_rows_f64.argtypes = [i32, i32, P, P, i32, P, P, P, P]
    lib.akv_tv_distance_f64.argtypes = [i32, P, P, P, P]
    lib.akv_decode_recovery.argtypes = [C.POINTER(DiagArgs), P]
    lib.akv_decode_recovery.restype = C.c_int
    lib.akv_decode_recovery_workspace_size.argtypes = [i32, i32, i64]
    lib.akv_decode_recovery_workspace_size.restype = sz
    lib.akv_decode_recovery_workspace_init.argtypes = [P, sz, i32, i32, i64, P]
    lib.akv_decode_recovery_workspace_init.restype = C.c_int
    lib.akv_embed_classify.argtypes = [i32, P, i32, P, P, i32, i32, P, P, P]
    lib.akv_add_rmsnorm.argtypes = [i32, i32, i32, P, P, P, C.c_float, P, P]
    lib.akv_add_rmsnorm_peers.argtypes = [i32, i32, i32, P, i32, i64, P, P, C.c_float, P, P]
    lib.akv_add_rmsnorm_peers.restype = C.c_int
    lib.akv_rope_scatter.argtypes = [C.POINTER(RopeArgs), P]
    lib.akv_swiglu.argtypes = [i32, i32, i32, P, P, P]
    lib.akv_greedy_next.argtypes = [i32, i32, i32, P, i64, P, P, i32, P, P, P, P]
    for fn in ("akv_embed_classify", "akv_add_rmsnorm", "akv_rope_scatter", "akv_swiglu",
               "akv_greedy_next", "akv_softmax_rows_f64", "akv_causal_attention_f64", "akv_keep_mask",
               "akv_map_recovery_f64", "akv_update_scores_f64", "akv_gather_rows_f64",
               "akv_tv_distance_f64"):
        getattr(lib, fn).restype = C.c_int
    lib.akv_last_error.restype = C.c_char_p
    lib.akv_version.restype = C.c_char_p
    lib.akv_device_check.restype = C.c_int
    return lib


lib = _load()


class AkvError(RuntimeError):
    """Raised for CUDA / capacity / unsupported-shape failures of the library."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[akv status {code}] {message}")
        self.code = code


def check(rc: int, exc_invalid=None):
    """Map a status code to an exception.  AKV_ERR_INVALID raises
    ``exc_invalid`` (the reference's PolicyError/ProfilerError/EngineError)
    when given."""
    if rc == AKV_OK:
        return
    msg = lib.akv_last_error().decode(errors="replace")
    if rc == AKV_ERR_INVALID and exc_invalid is not None:
        raise exc_invalid(msg)
    raise AkvError(rc, msg)


_checked_devices = set()


def require_device():
    """Fail loudly unless a sm_100 device is current (no CPU fallback).
    Checked once per device per process."""
    import torch

    if not torch.cuda.is_available():
        check(lib.akv_device_check())
    dev = torch.cuda.current_device()
    if dev not in _checked_devices:
        check(lib.akv_device_check())
        _checked_devices.add(dev)
