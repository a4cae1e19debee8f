"""ctypes loader for libsrt.so (the C ABI in include/srt.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
libsrt.so.  There is no CPU fallback — if the library or a CUDA device is
missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libsrt.so"
# development A/B runs load another build of the same ABI (tools/*_probe*)
if os.environ.get("SRT_LIB"):
    LIB_PATH = Path(os.environ["SRT_LIB"]).resolve()

SRT_OK, SRT_ERR_INVALID_CONFIG, SRT_ERR_INVALID_ARG, SRT_ERR_CUDA, SRT_ERR_DEVICE = range(5)
STATUS_NAMES = {0: "SRT_OK", 1: "SRT_ERR_INVALID_CONFIG", 2: "SRT_ERR_INVALID_ARG",
                3: "SRT_ERR_CUDA", 4: "SRT_ERR_DEVICE"}
SRT_DEV_OOV, SRT_DEV_CAPACITY, SRT_DEV_BAD_PROMPT, SRT_DEV_NONFINITE_LOGIT = 1, 2, 4, 8
SRT_DEV_INCONSISTENT = 0x10
SRT_BF16, SRT_F32 = 0, 1

# Every symbol include/srt.h declares (tests check the export table).
EXPORTS = ["srt_abi_version", "srt_error_string", "srt_cache_create", "srt_cache_destroy",
           "srt_insert", "srt_insert_cursor", "srt_draft", "srt_draft_cursor", "srt_verify", "srt_verify_path", "srt_verify_insert_cursor", "srt_verify_insert_draft_cursor", "srt_verify_lmhead", "srt_verify_lmhead_insert_cursor", "srt_cache_dump",
           "srt_cache_prune", "srt_cache_evict", "srt_cache_load", "srt_cache_status",
           "srt_cache_clear_errors", "srt_noise_table", "srt_log_det_range", "srt_row_noise", "srt_stream_read", "srt_sample_rows_reference",
           "srt_profile_enable", "srt_profile_read", "srt_profile_peek", "srt_debug_draft_profile", "srt_debug_insert_profile",
           "srt_pack_drafts", "srt_unpack_drafts", "srt_pack_spans", "srt_apply_spans",
           "srt_cache_set_step_overlap"]
KERNEL_NAMES = {0: "insert_plan", 1: "insert_walk", 2: "draft", 3: "row_offsets", 4: "scan",
                5: "accept", 6: "insert_cursor",
                7: "hub_refresh", 8: "accept_insert", 9: "lmhead",
                10: "tree_step"}


class SrtConfig(ctypes.Structure):
    _fields_ = [("vocab_size", ctypes.c_int32), ("max_prompts", ctypes.c_int32),
                ("max_depth", ctypes.c_int32), ("max_match_len", ctypes.c_int32),
                ("budget_max", ctypes.c_int32), ("budget_base", ctypes.c_int32),
                ("budget_slope_num", ctypes.c_int32), ("budget_slope_den", ctypes.c_int32),
                ("min_path_score", ctypes.c_double), ("node_capacity", ctypes.c_int64),
                ("hash_capacity", ctypes.c_int64), ("slot_capacity", ctypes.c_int64),
                ("logits_dtype", ctypes.c_int)]


class SrtCacheStats(ctypes.Structure):
    _fields_ = [("nodes_used", ctypes.c_uint64), ("node_capacity", ctypes.c_uint64),
                ("slots_used", ctypes.c_uint64), ("slot_capacity", ctypes.c_uint64),
                ("hash_capacity", ctypes.c_uint64)]


class SrtDumpRecord(ctypes.Structure):
    _fields_ = [("token", ctypes.c_int32), ("n_children", ctypes.c_int32),
                ("count", ctypes.c_uint64)]


class SrtProfileRecord(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("ms", ctypes.c_float)]


class SrtError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    """Load libsrt.so; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise SrtError(f"{LIB_PATH} is missing: run `python -m paper_2601_09083_b200.build` "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i32, i64, u64, f32 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                              ctypes.c_float)
    L.srt_abi_version.restype = ctypes.c_int
    L.srt_error_string.restype = ctypes.c_char_p
    L.srt_cache_create.argtypes = [ctypes.POINTER(SrtConfig), vp, ctypes.POINTER(vp)]
    L.srt_cache_destroy.argtypes = [vp, vp]
    L.srt_insert.argtypes = [vp, i32, vp, vp, i64, vp, vp, vp, vp, vp]
    L.srt_insert_cursor.argtypes = [vp, i32, vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.srt_pack_drafts.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.srt_unpack_drafts.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.srt_pack_spans.argtypes = [i32, i32, vp, vp, vp, vp]
    L.srt_apply_spans.argtypes = [i32, i32, vp, vp, vp, i64, vp, vp, vp, vp]
    L.srt_draft.argtypes = [vp, i32, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.srt_draft_cursor.argtypes = [vp, i32, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                   vp]
    L.srt_verify.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, u64, f32, i32, vp, vp, i64,
                             vp, vp, vp, vp, vp, vp, vp, vp]
    L.srt_verify_insert_cursor.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, u64, f32, i32, vp,
                                           vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                           vp]
    L.srt_verify_insert_draft_cursor.argtypes = (L.srt_verify_insert_cursor.argtypes[:-1] +
                                                  [vp] * 9 + [vp])  # pos_base, 8 outputs, stream
    _lm = [vp, i32, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, u64, f32, i32, vp, vp, i64, vp,
           vp, vp, vp, vp, vp, vp]
    L.srt_verify_lmhead.argtypes = _lm + [vp]
    L.srt_verify_lmhead_insert_cursor.argtypes = _lm + [vp, vp, vp, vp, vp]
    L.srt_verify_path.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, u64, f32, i32, vp, vp,
                                  i64, vp, vp, vp, vp, vp, vp, vp, vp]
    L.srt_cache_prune.argtypes = [vp, i32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_int64), vp]
    L.srt_cache_evict.argtypes = [vp, i64, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_uint32), vp]
    L.srt_cache_load.argtypes = [vp, i32, ctypes.POINTER(SrtDumpRecord), i64, vp]
    L.srt_cache_dump.argtypes = [vp, i32, ctypes.POINTER(SrtDumpRecord), i64,
                                 ctypes.POINTER(ctypes.c_int64), vp]
    L.srt_cache_status.argtypes = [vp, ctypes.POINTER(ctypes.c_uint32),
                                   ctypes.POINTER(SrtCacheStats), vp]
    L.srt_cache_clear_errors.argtypes = [vp, vp]
    L.srt_noise_table.argtypes = [vp, vp]
    L.srt_log_det_range.argtypes = [ctypes.c_uint32, i64, vp, vp]
    L.srt_row_noise.argtypes = [i32, u64, i32, vp, vp, vp, vp]
    L.srt_stream_read.argtypes = [vp, i64, i32, i32, i32, vp, vp]
    L.srt_sample_rows_reference.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, f32, vp, vp]
    L.srt_profile_enable.argtypes = [vp, i64]
    L.srt_cache_set_step_overlap.argtypes = [vp, i32]
    L.srt_debug_draft_profile.argtypes = [vp]
    L.srt_debug_insert_profile.argtypes = [vp]
    L.srt_profile_read.argtypes = [vp, ctypes.POINTER(SrtProfileRecord), i64,
                                   ctypes.POINTER(ctypes.c_int64), vp]
    L.srt_profile_peek.argtypes = L.srt_profile_read.argtypes
    for name in EXPORTS:
        if name not in ("srt_abi_version", "srt_error_string"):
            getattr(L, name).restype = ctypes.c_int
    if L.srt_abi_version() != 1:
        raise SrtError("libsrt ABI version mismatch")
    _lib = L
    return L


def check(status: int, what: str) -> None:
    if status != SRT_OK:
        msg = STATUS_NAMES.get(status, str(status))
        if status == SRT_ERR_CUDA:
            msg += ": " + load().srt_error_string().decode()
        raise SrtError(f"{what} failed: {msg}")
