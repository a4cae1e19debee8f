"""SRT CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow CPU implementation of SRT's per-step hot path (arXiv 2601.09083,
PAPER.md §3 "Method").  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2601_09083_b200`` never imports it, and
the two share no code: the arithmetic lives in ``srt_oracle.cpp`` (restated from
the paper and the DESIGN.md readings), this module only marshals numpy arrays.

Every function is pinned by ``-m "not gpu"`` tests against something other than
itself (see tests/test_oracle_*.py): the paper's Fig. 3 worked example
(P:L125-132), SPEC's insert examples, brute-force enumeration of substrings /
suffixes / draft orders on tiny inputs, the published Philox4x32-10 KAT vectors,
fp64 libm accuracy bounds for ``log_det``, closed-form count invariants and the
losslessness property (speculative == plain decoding).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "srt_oracle.cpp"
_LIB = _HERE / "liboracle.so"

__all__ = ["build", "lib", "Oracle", "philox4x32_10", "log_det", "gumbel_from_word",
           "noise_table", "sample_row", "log_det_array", "row_noise_many", "sample_rows"]


def build(force: bool = False) -> Path:
    """Compile the oracle with plain IEEE semantics (no contraction, no fast-math)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", str(_SRC), "-o", str(_LIB) + ".tmp"]
        subprocess.run(cmd, check=True)
        os.replace(str(_LIB) + ".tmp", _LIB)
    return _LIB


_lib = None

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.orc_log_det.argtypes = [ctypes.c_float]
        L.orc_log_det.restype = ctypes.c_float
        L.orc_log_det_array.argtypes = [_f32p, _f32p, ctypes.c_int64]
        L.orc_gumbel_from_word.argtypes = [ctypes.c_uint32]
        L.orc_gumbel_from_word.restype = ctypes.c_float
        L.orc_noise_table.argtypes = [_f32p]
        L.orc_row_noise.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_int32, _f32p]
        L.orc_sample_row.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_int32, ctypes.c_float,
                                     ctypes.POINTER(ctypes.c_int)]
        L.orc_sample_row.restype = ctypes.c_int32
        L.orc_row_noise_many.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, _u64p,
                                         _i32p, _f32p]
        L.orc_sample_rows.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.c_uint64, _u64p, _i32p, ctypes.c_float, _i32p, _i32p,
                                      _i32p]
        L.orc_cache_create.argtypes = [ctypes.c_int32] * 8 + [ctypes.c_double]
        L.orc_cache_create.restype = ctypes.c_void_p
        L.orc_cache_destroy.argtypes = [ctypes.c_void_p]
        L.orc_error_bits.argtypes = [ctypes.c_void_p]
        L.orc_error_bits.restype = ctypes.c_uint32
        L.orc_node_count.argtypes = [ctypes.c_void_p]
        L.orc_node_count.restype = ctypes.c_uint64
        L.orc_insert.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p, _i32p, ctypes.c_int64,
                                 _i32p, _i32p, _i32p]
        L.orc_draft.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p, _i32p, ctypes.c_int64,
                                _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _u64p,
                                _i64p]
        L.orc_verify.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int,
                                 _i64p, _i32p, _i32p, _i32p, _i32p, _u64p, ctypes.c_uint64,
                                 ctypes.c_float, ctypes.c_int32, _i32p, _i32p, ctypes.c_int64,
                                 _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _u8p, _i32p]
        L.orc_verify.restype = ctypes.c_int
        L.orc_dump.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p, _u64p, _i32p, ctypes.c_int64]
        L.orc_dump.restype = ctypes.c_int64
        L.orc_prune.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64]
        L.orc_prune.restype = ctypes.c_int64
        L.orc_load.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p, _u64p, _i32p, ctypes.c_int64]
        L.orc_load.restype = ctypes.c_int32
        L.orc_count_of.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p, ctypes.c_int32]
        L.orc_count_of.restype = ctypes.c_uint64
        _lib = L
    return _lib


def philox4x32_10(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def log_det(x: float) -> np.float32:
    return np.float32(lib().orc_log_det(float(x)))


def log_det_array(x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().orc_log_det_array(x.ravel(), out.ravel(), x.size)
    return out


def gumbel_from_word(w: int) -> np.float32:
    return np.float32(lib().orc_gumbel_from_word(int(w)))


def noise_table() -> np.ndarray:
    out = np.empty(1 << 23, np.float32)
    lib().orc_noise_table(out)
    return out


def row_noise(V: int, seed: int, seq_id: int, pos: int) -> np.ndarray:
    """The sampler's Gumbel noise g_v for every v of one row key (O11)."""
    out = np.empty(V, np.float32)
    lib().orc_row_noise(V, seed, seq_id, pos, out)
    return out


def row_noise_many(V: int, seed: int, seq_id, pos) -> np.ndarray:
    """row_noise for n keys at once (OpenMP over keys): [n, V] float32."""
    seq_id = np.ascontiguousarray(seq_id, np.uint64)
    pos = np.ascontiguousarray(pos, np.int32)
    out = np.empty((len(seq_id), V), np.float32)
    lib().orc_row_noise_many(V, seed, len(seq_id), seq_id, pos, out.reshape(-1))
    return out


def sample_rows(rows: np.ndarray, seed: int, seq_id, pos, temperature: float = 1.0):
    """sample_row over n rows [n, V] (float32 or bf16 bits as uint16), OpenMP
    over rows.  Returns (tokens, ties, nan): ties[k] = number of indices whose
    z equals row k's maximum (>= 2 means the smallest-index rule decided)."""
    rows = np.ascontiguousarray(rows)
    n, V = rows.shape
    tok = np.empty(n, np.int32)
    ties = np.empty(n, np.int32)
    nan = np.empty(n, np.int32)
    lib().orc_sample_rows(rows.ctypes.data, _dtype_code(rows), V, n, seed,
                          np.ascontiguousarray(seq_id, np.uint64),
                          np.ascontiguousarray(pos, np.int32), temperature, tok, ties, nan)
    return tok, ties, nan.astype(bool)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 1
    if a.dtype == np.uint16:  # bf16 bit patterns
        return 0
    raise TypeError("logits must be float32 or uint16 (bf16 bits)")


def sample_row(row: np.ndarray, seed: int, seq_id: int, pos: int, temperature: float = 1.0):
    row = np.ascontiguousarray(row)
    nan = ctypes.c_int(0)
    tok = lib().orc_sample_row(row.ctypes.data, _dtype_code(row), row.shape[-1], seed, seq_id, pos,
                               temperature, ctypes.byref(nan))
    return tok, bool(nan.value)


class Oracle:
    """One oracle cache (all prompts' trees).  Arrays are numpy, host memory."""

    def __init__(self, vocab_size, max_prompts, max_depth, max_match_len, budget_max,
                 budget_base=None, slope_num=0, slope_den=1, min_path_score=0.0):
        if budget_base is None:
            budget_base = budget_max
        self.V, self.P, self.D, self.L = vocab_size, max_prompts, max_depth, max_match_len
        self.Bmax = budget_max
        self.h = lib().orc_cache_create(vocab_size, max_prompts, max_depth, max_match_len,
                                        budget_max, budget_base, slope_num, slope_den,
                                        float(min_path_score))
        if not self.h:
            raise ValueError("invalid oracle config")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_cache_destroy(h)
            self.h = None

    @property
    def error_bits(self) -> int:
        return int(lib().orc_error_bits(self.h))

    @property
    def node_count(self) -> int:
        return int(lib().orc_node_count(self.h))

    def insert(self, prompt_id, seq_tok, frm, to, floor=None):
        prompt_id = np.ascontiguousarray(prompt_id, np.int32)
        seq_tok = np.ascontiguousarray(seq_tok, np.int32)
        n = prompt_id.shape[0]
        floor = np.zeros(n, np.int32) if floor is None else np.ascontiguousarray(floor, np.int32)
        lib().orc_insert(self.h, n, prompt_id, seq_tok, seq_tok.shape[1],
                         np.ascontiguousarray(frm, np.int32), np.ascontiguousarray(to, np.int32),
                         floor)

    def insert_sequence(self, p, tokens):
        """SPEC insert_sequence: the whole token list as one span from 0."""
        t = np.asarray(tokens, np.int32)[None, :]
        self.insert([p], t, [0], [t.shape[1]])

    def draft(self, prompt_id, seq_tok, seq_len, pos_base=None):
        prompt_id = np.ascontiguousarray(prompt_id, np.int32)
        seq_tok = np.ascontiguousarray(seq_tok, np.int32)
        seq_len = np.ascontiguousarray(seq_len, np.int32)
        n = prompt_id.shape[0]
        B = self.Bmax
        pos_base = np.zeros(n, np.int32) if pos_base is None else np.ascontiguousarray(pos_base, np.int32)
        out = dict(match_len=np.zeros(n, np.int32), draft_len=np.zeros(n, np.int32),
                   draft_tok=np.zeros((n, B), np.int32), draft_parent=np.zeros((n, B), np.int32),
                   draft_depth=np.zeros((n, B), np.int32), draft_pos=np.zeros((n, B), np.int32),
                   draft_mask=np.zeros((n, B), np.uint64), row_offsets=np.zeros(n + 1, np.int64))
        lib().orc_draft(self.h, n, prompt_id, seq_tok, seq_tok.shape[1], seq_len, pos_base,
                        out["match_len"], out["draft_len"], out["draft_tok"], out["draft_parent"],
                        out["draft_depth"], out["draft_pos"], out["draft_mask"], out["row_offsets"])
        return out

    def verify(self, logits, row_offsets, draft_len, draft_tok, draft_parent, draft_depth, seq_id,
               seed, seq_tok, seq_len, max_new, temperature=1.0, eos_id=-1):
        """Mutates seq_tok / seq_len in place (like the GPU call).  Returns a dict."""
        logits = np.ascontiguousarray(logits)
        assert seq_tok.flags["C_CONTIGUOUS"] and seq_tok.dtype == np.int32
        assert seq_len.flags["C_CONTIGUOUS"] and seq_len.dtype == np.int32
        n = seq_len.shape[0]
        B = self.Bmax
        rows = int(row_offsets[n])
        assert logits.shape[0] >= rows and logits.shape[-1] == self.V
        out = dict(sampled=np.zeros(rows, np.int32), accept_len=np.zeros(n, np.int32),
                   n_commit=np.zeros(n, np.int32), commit_tok=np.zeros((n, B + 1), np.int32),
                   accepted_nodes=np.zeros((n, B), np.int32), finished=np.zeros(n, np.uint8),
                   ties=np.zeros(rows, np.int32))
        nan = lib().orc_verify(self.h, n, logits.ctypes.data, _dtype_code(logits),
                               np.ascontiguousarray(row_offsets, np.int64),
                               np.ascontiguousarray(draft_len, np.int32),
                               np.ascontiguousarray(draft_tok, np.int32),
                               np.ascontiguousarray(draft_parent, np.int32),
                               np.ascontiguousarray(draft_depth, np.int32),
                               np.ascontiguousarray(seq_id, np.uint64), seed, temperature, eos_id,
                               np.ascontiguousarray(max_new, np.int32), seq_tok, seq_tok.shape[1],
                               seq_len, out["sampled"], out["accept_len"], out["n_commit"],
                               out["commit_tok"], out["accepted_nodes"], out["finished"],
                               out["ties"])
        out["nan_seen"] = bool(nan)
        return out

    def dump(self, p):
        cap = 1 << 16
        while True:
            tok = np.zeros(cap, np.int32)
            cnt = np.zeros(cap, np.uint64)
            nch = np.zeros(cap, np.int32)
            k = lib().orc_dump(self.h, p, tok, cnt, nch, cap)
            if k < 0:
                raise ValueError("bad prompt id")
            if k <= cap:
                return np.stack([tok[:k].astype(np.int64), cnt[:k].astype(np.int64),
                                 nch[:k].astype(np.int64)], axis=1)
            cap = int(k)

    def prune(self, p, theta) -> int:
        """Remove every non-root node of T_p (all prompts if p < 0) with count < theta."""
        r = lib().orc_prune(self.h, int(p), int(theta))
        if r < 0:
            raise ValueError("bad prompt id")
        return int(r)

    def load(self, p, records):
        """Merge dump records [(token, count, n_children), ...] (preorder) into T_p."""
        r = np.asarray(records, np.int64).reshape(-1, 3)
        tok = np.ascontiguousarray(r[:, 0], np.int32)
        cnt = np.ascontiguousarray(r[:, 1], np.uint64)
        nch = np.ascontiguousarray(r[:, 2], np.int32)
        if lib().orc_load(self.h, int(p), tok, cnt, nch, r.shape[0]) != 0:
            raise ValueError("malformed dump records")

    def count_of(self, p, tokens) -> int:
        t = np.ascontiguousarray(tokens, np.int32)
        return int(lib().orc_count_of(self.h, p, t, t.shape[0]))
