"""Thin Python binding of libsrt's C ABI (include/srt.h) over torch tensors.

torch is used for device memory and streams only: this module allocates
output tensors (torch.empty) and passes data pointers + the current stream to
the C ABI; every step of the SRT path runs inside libsrt's CUDA kernels.
Names follow the paper: insert, draft, verify.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import SrtCacheStats, SrtConfig, SrtDumpRecord, SrtError, check

__all__ = ["SrtCache", "DraftOut", "VerifyOut", "config", "noise_table", "log_det_range", "row_noise", "stream_read", "SrtError",
           "pack_drafts", "unpack_drafts", "pack_spans", "apply_spans", "draft_record_words",
           "span_record_words"]

_DT = {torch.bfloat16: _lib.SRT_BF16, torch.float32: _lib.SRT_F32}


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None, dtype=None, name: str = "") -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_cuda:
        raise SrtError(f"{name}: expected a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise SrtError(f"{name}: expected a contiguous tensor")
    if dtype is not None and t.dtype != dtype:
        raise SrtError(f"{name}: expected {dtype}, got {t.dtype}")
    return ctypes.c_void_p(t.data_ptr())


def config(vocab_size: int, max_prompts: int, max_depth: int, max_match_len: int,
           budget_max: int, budget_base: int | None = None, slope_num: int = 0,
           slope_den: int = 1, min_path_score: float = 0.0, node_capacity: int = 1 << 20,
           hash_capacity: int | None = None, slot_capacity: int | None = None,
           logits_dtype: torch.dtype = torch.bfloat16) -> SrtConfig:
    if budget_base is None:
        budget_base = budget_max
    if hash_capacity is None:
        hash_capacity = 1 << max(1, (2 * node_capacity - 1).bit_length())
    if slot_capacity is None:
        slot_capacity = 2 * node_capacity
    return SrtConfig(vocab_size, max_prompts, max_depth, max_match_len, budget_max, budget_base,
                     slope_num, slope_den, float(min_path_score), node_capacity, hash_capacity,
                     slot_capacity, _DT[logits_dtype])


@dataclass
class DraftOut:
    match_len: torch.Tensor      # [n] i32
    draft_len: torch.Tensor      # [n] i32
    draft_tok: torch.Tensor      # [n, Bmax] i32
    draft_parent: torch.Tensor   # [n, Bmax] i32
    draft_depth: torch.Tensor    # [n, Bmax] i32
    draft_pos: torch.Tensor      # [n, Bmax] i32
    draft_mask: torch.Tensor     # [n, Bmax] i64 (u64 bit patterns)
    row_offsets: torch.Tensor    # [n+1] i64

    @staticmethod
    def empty(n: int, Bmax: int, device) -> "DraftOut":
        i32 = dict(dtype=torch.int32, device=device)
        return DraftOut(torch.empty(n, **i32), torch.empty(n, **i32), torch.empty(n, Bmax, **i32),
                        torch.empty(n, Bmax, **i32), torch.empty(n, Bmax, **i32),
                        torch.empty(n, Bmax, **i32),
                        torch.empty(n, Bmax, dtype=torch.int64, device=device),
                        torch.empty(n + 1, dtype=torch.int64, device=device))


@dataclass
class VerifyOut:
    sampled: torch.Tensor         # [rows] i32
    accept_len: torch.Tensor      # [n] i32
    n_commit: torch.Tensor        # [n] i32
    commit_tok: torch.Tensor      # [n, Bmax+1] i32
    accepted_nodes: torch.Tensor  # [n, Bmax] i32
    finished: torch.Tensor        # [n] u8

    @staticmethod
    def empty(n: int, rows: int, Bmax: int, device) -> "VerifyOut":
        i32 = dict(dtype=torch.int32, device=device)
        return VerifyOut(torch.empty(rows, **i32), torch.empty(n, **i32), torch.empty(n, **i32),
                         torch.empty(n, Bmax + 1, **i32), torch.empty(n, Bmax, **i32),
                         torch.empty(n, dtype=torch.uint8, device=device))


class SrtCache:
    """The per-prompt tree caches T_p of P prompts, resident in HBM."""

    def __init__(self, cfg: SrtConfig, device: int | torch.device | None = None):
        self.L = _lib.load()
        if not torch.cuda.is_available():
            raise SrtError("SRT needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.cfg = cfg
        self.V, self.P, self.Bmax = cfg.vocab_size, cfg.max_prompts, cfg.budget_max
        self.logits_dtype = torch.bfloat16 if cfg.logits_dtype == _lib.SRT_BF16 else torch.float32
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.L.srt_cache_create(ctypes.byref(cfg), _stream(), ctypes.byref(self._h)),
                  "srt_cache_create")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            with torch.cuda.device(self.device):
                self.L.srt_cache_destroy(self._h, _stream())
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the hot path -------------------------------------------------------
    def insert(self, prompt_id, seq_tok, frm, to, floor=None, stats=None, cursor=None) -> None:
        """srt_insert, or srt_insert_cursor when `cursor` (see new_cursors) is given."""
        n = prompt_id.shape[0]
        i32 = torch.int32
        args = [self._h, n, _ptr(prompt_id, i32, "prompt_id"), _ptr(seq_tok, i32, "seq_tok"),
                seq_tok.shape[1], _ptr(frm, i32, "from"), _ptr(to, i32, "to"),
                _ptr(floor, i32, "floor")]
        if cursor is None:
            check(self.L.srt_insert(*args, _ptr(stats, torch.int64, "stats"), _stream()),
                  "srt_insert")
        else:
            if cursor.shape != (n, self.cfg.max_depth + 4):
                raise ValueError(f"cursor must be ({n}, D + 4) int32")
            check(self.L.srt_insert_cursor(*args, _ptr(cursor, i32, "cursor"),
                                           _ptr(stats, torch.int64, "stats"), _stream()),
                  "srt_insert_cursor")

    def new_cursors(self, n: int, device="cuda"):
        """Zero-filled (= invalid, rebuilt on first use) insert cursors for n sequences."""
        return torch.zeros((n, self.cfg.max_depth + 4), dtype=torch.int32, device=device)

    def draft(self, prompt_id, seq_tok, seq_len, pos_base=None, out: DraftOut | None = None,
              cursor=None) -> DraftOut:
        """srt_draft, or srt_draft_cursor when the insert cursors are given."""
        n = prompt_id.shape[0]
        if out is None:
            out = DraftOut.empty(n, self.Bmax, seq_tok.device)
        i32 = torch.int32
        head = (self._h, n, _ptr(prompt_id, i32, "prompt_id"), _ptr(seq_tok, i32, "seq_tok"),
                seq_tok.shape[1], _ptr(seq_len, i32, "seq_len"), _ptr(pos_base, i32, "pos_base"))
        tail = (_ptr(out.match_len, i32), _ptr(out.draft_len, i32), _ptr(out.draft_tok, i32),
                _ptr(out.draft_parent, i32), _ptr(out.draft_depth, i32), _ptr(out.draft_pos, i32),
                _ptr(out.draft_mask, torch.int64), _ptr(out.row_offsets, torch.int64), _stream())
        if cursor is None:
            check(self.L.srt_draft(*head, *tail), "srt_draft")
        else:
            check(self.L.srt_draft_cursor(*head, _ptr(cursor, torch.int32, "cursor"), *tail),
                  "srt_draft_cursor")
        return out

    def verify(self, logits, d: DraftOut, seq_id, seed: int, seq_tok, seq_len, max_new,
               temperature: float = 1.0, eos_id: int = -1, out: VerifyOut | None = None,
               rows: int | None = None, path_rounds: int | None = None) -> VerifyOut:
        """Mutates seq_tok / seq_len (appends the committed tokens).  path_rounds
        = R selects srt_verify_path (only the accepted path's rows sampled)."""
        n = seq_len.shape[0]
        if logits.dtype != self.logits_dtype:
            raise SrtError(f"logits dtype {logits.dtype} != cache's {self.logits_dtype}")
        if logits.shape[-1] != self.V:
            raise SrtError("logits row length != V")
        if out is None:
            out = VerifyOut.empty(n, logits.shape[0] if rows is None else rows, self.Bmax,
                                  seq_tok.device)
        i32 = torch.int32
        fn, head = self.L.srt_verify, (self._h, n)
        if path_rounds is not None:
            fn, head = self.L.srt_verify_path, (self._h, n, int(path_rounds))
        check(fn(*head, _ptr(logits, None, "logits"),
                                _ptr(d.row_offsets, torch.int64), _ptr(d.draft_len, i32),
                                _ptr(d.draft_tok, i32), _ptr(d.draft_parent, i32),
                                _ptr(d.draft_depth, i32), _ptr(seq_id, torch.int64, "seq_id"),
                                ctypes.c_uint64(seed & (2 ** 64 - 1)), float(temperature),
                                int(eos_id), _ptr(max_new, i32, "max_new"),
                                _ptr(seq_tok, i32, "seq_tok"), seq_tok.shape[1],
                                _ptr(seq_len, i32, "seq_len"), _ptr(out.sampled, i32),
                                _ptr(out.accept_len, i32), _ptr(out.n_commit, i32),
                                _ptr(out.commit_tok, i32), _ptr(out.accepted_nodes, i32),
                                _ptr(out.finished, torch.uint8), _stream()), "srt_verify")
        return out

    def verify_insert(self, logits, d: DraftOut, seq_id, seed: int, seq_tok, seq_len, max_new,
                      prompt_id, cursor, floor=None, stats=None, temperature: float = 1.0,
                      eos_id: int = -1, out: VerifyOut | None = None,
                      rows: int | None = None) -> VerifyOut:
        """srt_verify_insert_cursor: verify, then insert each sequence's committed
        span through its cursor, fused (same results as verify() then
        insert(..., cursor=cursor) from the old to the new seq_len)."""
        n = seq_len.shape[0]
        if logits.dtype != self.logits_dtype:
            raise SrtError(f"logits dtype {logits.dtype} != cache's {self.logits_dtype}")
        if logits.shape[-1] != self.V:
            raise SrtError("logits row length != V")
        if cursor.shape != (n, self.cfg.max_depth + 4):
            raise ValueError(f"cursor must be ({n}, D + 4) int32")
        if out is None:
            out = VerifyOut.empty(n, logits.shape[0] if rows is None else rows, self.Bmax,
                                  seq_tok.device)
        i32 = torch.int32
        check(self.L.srt_verify_insert_cursor(
            self._h, n, _ptr(logits, None, "logits"), _ptr(d.row_offsets, torch.int64),
            _ptr(d.draft_len, i32), _ptr(d.draft_tok, i32), _ptr(d.draft_parent, i32),
            _ptr(d.draft_depth, i32), _ptr(seq_id, torch.int64, "seq_id"),
            ctypes.c_uint64(seed & (2 ** 64 - 1)), float(temperature), int(eos_id),
            _ptr(max_new, i32, "max_new"), _ptr(seq_tok, i32, "seq_tok"), seq_tok.shape[1],
            _ptr(seq_len, i32, "seq_len"), _ptr(out.sampled, i32), _ptr(out.accept_len, i32),
            _ptr(out.n_commit, i32), _ptr(out.commit_tok, i32), _ptr(out.accepted_nodes, i32),
            _ptr(out.finished, torch.uint8), _ptr(prompt_id, i32, "prompt_id"),
            _ptr(floor, i32, "floor"), _ptr(cursor, i32, "cursor"),
            _ptr(stats, torch.int64, "stats"), _stream()), "srt_verify_insert_cursor")
        return out

    def verify_insert_draft(self, logits, d: DraftOut, seq_id, seed: int, seq_tok, seq_len,
                            max_new, prompt_id, cursor, pos_base=None, next_d: DraftOut | None = None,
                            floor=None, stats=None, temperature: float = 1.0, eos_id: int = -1,
                            out: VerifyOut | None = None, rows: int | None = None) -> VerifyOut:
        """srt_verify_insert_draft_cursor: verify_insert() then the next step's
        draft_cursor(prompt_id, seq_tok, seq_len, pos_base) in one persistent
        kernel ordered per prompt.  next_d may be d itself (the draft buffers
        are reused); pos_base may be seq_len (read after the commit)."""
        n = seq_len.shape[0]
        if logits.dtype != self.logits_dtype:
            raise SrtError(f"logits dtype {logits.dtype} != cache's {self.logits_dtype}")
        if logits.shape[-1] != self.V:
            raise SrtError("logits row length != V")
        if cursor.shape != (n, self.cfg.max_depth + 4):
            raise ValueError(f"cursor must be ({n}, D + 4) int32")
        if next_d is None:
            next_d = d
        if out is None:
            out = VerifyOut.empty(n, logits.shape[0] if rows is None else rows, self.Bmax,
                                  seq_tok.device)
        i32 = torch.int32
        check(self.L.srt_verify_insert_draft_cursor(
            self._h, n, _ptr(logits, None, "logits"), _ptr(d.row_offsets, torch.int64),
            _ptr(d.draft_len, i32), _ptr(d.draft_tok, i32), _ptr(d.draft_parent, i32),
            _ptr(d.draft_depth, i32), _ptr(seq_id, torch.int64, "seq_id"),
            ctypes.c_uint64(seed & (2 ** 64 - 1)), float(temperature), int(eos_id),
            _ptr(max_new, i32, "max_new"), _ptr(seq_tok, i32, "seq_tok"), seq_tok.shape[1],
            _ptr(seq_len, i32, "seq_len"), _ptr(out.sampled, i32), _ptr(out.accept_len, i32),
            _ptr(out.n_commit, i32), _ptr(out.commit_tok, i32), _ptr(out.accepted_nodes, i32),
            _ptr(out.finished, torch.uint8), _ptr(prompt_id, i32, "prompt_id"),
            _ptr(floor, i32, "floor"), _ptr(cursor, i32, "cursor"),
            _ptr(stats, torch.int64, "stats"), _ptr(pos_base, i32, "pos_base"),
            _ptr(next_d.match_len, i32), _ptr(next_d.draft_len, i32), _ptr(next_d.draft_tok, i32),
            _ptr(next_d.draft_parent, i32), _ptr(next_d.draft_depth, i32),
            _ptr(next_d.draft_pos, i32), _ptr(next_d.draft_mask, torch.int64),
            _ptr(next_d.row_offsets, torch.int64), _stream()), "srt_verify_insert_draft_cursor")
        return out

    def verify_lmhead(self, hidden, weight, d: DraftOut, seq_id, seed: int, seq_tok, seq_len,
                      max_new, prompt_id=None, cursor=None, floor=None, stats=None,
                      temperature: float = 1.0, eos_id: int = -1, out: VerifyOut | None = None,
                      rows: int | None = None, logits_out=None) -> VerifyOut:
        """srt_verify_lmhead (or srt_verify_lmhead_insert_cursor when `cursor` is
        given): the verify pass with the LM-head GEMM fused in front of the
        sampler -- hidden [hidden_rows, K] bf16 (row r = logits row r),
        weight [V, K] bf16; the logits are never written unless logits_out
        ([rows, V], the cache's logits dtype) is given."""
        n = seq_len.shape[0]
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
            raise SrtError("hidden and weight must be bfloat16")
        if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
            raise SrtError("hidden [rows, K] and weight [V, K] expected")
        if weight.shape[0] != self.V:
            raise SrtError("weight rows != V")
        if logits_out is not None and (logits_out.dtype != self.logits_dtype
                                       or logits_out.shape[-1] != self.V):
            raise SrtError("logits_out must be [rows, V] of the cache's logits dtype")
        if out is None:
            out = VerifyOut.empty(n, hidden.shape[0] if rows is None else rows, self.Bmax,
                                  seq_tok.device)
        i32 = torch.int32
        args = [self._h, n, _ptr(hidden, torch.bfloat16, "hidden"), hidden.shape[0],
                hidden.shape[1], _ptr(weight, torch.bfloat16, "weight"),
                _ptr(logits_out, None, "logits_out"), _ptr(d.row_offsets, torch.int64),
                _ptr(d.draft_len, i32), _ptr(d.draft_tok, i32), _ptr(d.draft_parent, i32),
                _ptr(d.draft_depth, i32), _ptr(seq_id, torch.int64, "seq_id"),
                ctypes.c_uint64(seed & (2 ** 64 - 1)), float(temperature), int(eos_id),
                _ptr(max_new, i32, "max_new"), _ptr(seq_tok, i32, "seq_tok"), seq_tok.shape[1],
                _ptr(seq_len, i32, "seq_len"), _ptr(out.sampled, i32), _ptr(out.accept_len, i32),
                _ptr(out.n_commit, i32), _ptr(out.commit_tok, i32),
                _ptr(out.accepted_nodes, i32), _ptr(out.finished, torch.uint8)]
        if cursor is None:
            check(self.L.srt_verify_lmhead(*args, _stream()), "srt_verify_lmhead")
        else:
            if cursor.shape != (n, self.cfg.max_depth + 4):
                raise ValueError(f"cursor must be ({n}, D + 4) int32")
            check(self.L.srt_verify_lmhead_insert_cursor(
                *args, _ptr(prompt_id, i32, "prompt_id"), _ptr(floor, i32, "floor"),
                _ptr(cursor, i32, "cursor"), _ptr(stats, torch.int64, "stats"), _stream()),
                "srt_verify_lmhead_insert_cursor")
        return out

    # ---- test / inspection support -----------------------------------------
    def sample_rows_reference(self, logits, d: DraftOut, seq_len, seq_id, seed: int,
                              temperature: float = 1.0, out=None) -> torch.Tensor:
        n = seq_len.shape[0]
        if out is None:
            out = torch.empty(logits.shape[0], dtype=torch.int32, device=logits.device)
        check(self.L.srt_sample_rows_reference(
            self._h, n, _ptr(logits, None, "logits"), _ptr(d.row_offsets, torch.int64),
            _ptr(d.draft_depth, torch.int32), _ptr(seq_len, torch.int32),
            _ptr(seq_id, torch.int64), ctypes.c_uint64(seed & (2 ** 64 - 1)), float(temperature),
            _ptr(out, torch.int32), _stream()), "srt_sample_rows_reference")
        return out

    def status(self):
        bits = ctypes.c_uint32(0)
        st = SrtCacheStats()
        r = self.L.srt_cache_status(self._h, ctypes.byref(bits), ctypes.byref(st), _stream())
        if r not in (_lib.SRT_OK, _lib.SRT_ERR_DEVICE):
            check(r, "srt_cache_status")
        return int(bits.value), {k: int(getattr(st, k)) for k, _ in SrtCacheStats._fields_}

    def set_step_overlap(self, sms: int) -> None:
        """srt_cache_set_step_overlap: the fused tree step of verify_insert_draft
        on `sms` SMs beside the scan (0: after it on every SM, -1: default)."""
        check(self.L.srt_cache_set_step_overlap(self._h, int(sms)), "srt_cache_set_step_overlap")

    def profile_enable(self, capacity: int) -> None:
        check(self.L.srt_profile_enable(self._h, int(capacity)), "srt_profile_enable")

    def profile_read(self):
        """[(kernel name, ms), ...] for every timed launch since the last read (blocking)."""
        n = ctypes.c_int64(0)
        cap = 1 << 16
        buf = (_lib.SrtProfileRecord * cap)()
        check(self.L.srt_profile_read(self._h, buf, cap, ctypes.byref(n), _stream()),
              "srt_profile_read")
        return [(_lib.KERNEL_NAMES.get(buf[i].kernel, str(buf[i].kernel)), float(buf[i].ms))
                for i in range(min(n.value, cap))]

    def profile_peek(self):
        """profile_read without clearing (blocking): after a CUDA-graph replay,
        the replay's per-kernel times of the captured launches."""
        n = ctypes.c_int64(0)
        cap = 256
        buf = (_lib.SrtProfileRecord * cap)()
        check(self.L.srt_profile_peek(self._h, buf, cap, ctypes.byref(n), _stream()),
              "srt_profile_peek")
        return [(_lib.KERNEL_NAMES.get(buf[i].kernel, str(buf[i].kernel)), float(buf[i].ms))
                for i in range(min(n.value, cap))]

    def clear_errors(self):
        check(self.L.srt_cache_clear_errors(self._h, _stream()), "srt_cache_clear_errors")

    def dump(self, prompt_id: int):
        """Canonical preorder records [(token, count, n_children), ...] (blocking)."""
        n = ctypes.c_int64(0)
        check(self.L.srt_cache_dump(self._h, prompt_id, None, 0, ctypes.byref(n), _stream()),
              "srt_cache_dump")
        buf = (SrtDumpRecord * max(1, n.value))()
        check(self.L.srt_cache_dump(self._h, prompt_id, buf, n.value, ctypes.byref(n), _stream()),
              "srt_cache_dump")
        return [(buf[i].token, int(buf[i].count), buf[i].n_children) for i in range(n.value)]


    # ---- capacity management and persistence (include/srt.h; O17) --
    def prune(self, prompt_id: int, theta: int) -> int:
        """Remove every non-root node of T_p (all prompts if -1) with count < theta
        (blocking); returns the number removed.  Invalidates the insert cursors."""
        r = ctypes.c_int64(0)
        check(self.L.srt_cache_prune(self._h, prompt_id, theta, ctypes.byref(r), _stream()),
              "srt_cache_prune")
        return r.value

    def reset(self, prompt_id: int) -> int:
        """Empty T_p (blocking)."""
        return self.prune(prompt_id, 0xFFFFFFFF)

    def evict(self, max_nodes: int):
        """Prune every tree to <= 0.9 * max_nodes nodes if more than max_nodes are
        live (blocking); returns (removed, theta)."""
        r, th = ctypes.c_int64(0), ctypes.c_uint32(0)
        check(self.L.srt_cache_evict(self._h, max_nodes, ctypes.byref(r), ctypes.byref(th),
                                     _stream()), "srt_cache_evict")
        return r.value, th.value

    def load(self, prompt_id: int, records) -> None:
        """Merge canonical dump records [(token, count, n_children), ...] into T_p."""
        n = len(records)
        buf = (SrtDumpRecord * max(1, n))()
        for i, (t, cnt, nch) in enumerate(records):
            buf[i].token, buf[i].count, buf[i].n_children = int(t), int(cnt), int(nch)
        check(self.L.srt_cache_load(self._h, prompt_id, buf, n, _stream()), "srt_cache_load")


# ---- multi-GPU exchange records (include/srt.h) ----------------
def draft_record_words(Bmax: int) -> int:
    return 2 + 5 * Bmax


def span_record_words(Bmax: int) -> int:
    return Bmax + 2


def pack_drafts(d: DraftOut, Bmax: int, out: torch.Tensor) -> torch.Tensor:
    """out[s] <- draft record of sequence s (out: [>= n, draft_record_words] int32)."""
    n = d.draft_len.shape[0]
    i32 = torch.int32
    check(_lib.load().srt_pack_drafts(n, Bmax, _ptr(d.match_len, i32), _ptr(d.draft_len, i32),
                                      _ptr(d.draft_tok, i32), _ptr(d.draft_parent, i32),
                                      _ptr(d.draft_depth, i32), _ptr(d.draft_mask, torch.int64),
                                      _ptr(out, i32, "records"), _stream()), "srt_pack_drafts")
    return out


def unpack_drafts(records: torch.Tensor, src: torch.Tensor, Bmax: int, out: DraftOut,
                  pos_base=None) -> DraftOut:
    n = out.draft_len.shape[0]
    i32 = torch.int32
    check(_lib.load().srt_unpack_drafts(n, Bmax, _ptr(records, i32, "records"), _ptr(src, i32, "src"),
                                        _ptr(pos_base, i32, "pos_base"), _ptr(out.match_len, i32),
                                        _ptr(out.draft_len, i32), _ptr(out.draft_tok, i32),
                                        _ptr(out.draft_parent, i32), _ptr(out.draft_depth, i32),
                                        _ptr(out.draft_pos, i32), _ptr(out.draft_mask, torch.int64),
                                        _ptr(out.row_offsets, torch.int64), _stream()),
          "srt_unpack_drafts")
    return out


def pack_spans(v: VerifyOut, Bmax: int, out: torch.Tensor) -> torch.Tensor:
    n = v.n_commit.shape[0]
    i32 = torch.int32
    check(_lib.load().srt_pack_spans(n, Bmax, _ptr(v.n_commit, i32), _ptr(v.commit_tok, i32),
                                     _ptr(out, i32, "records"), _stream()), "srt_pack_spans")
    return out


def apply_spans(records: torch.Tensor, src: torch.Tensor, Bmax: int, seq_tok: torch.Tensor,
                seq_len: torch.Tensor, frm: torch.Tensor, to: torch.Tensor) -> None:
    n = seq_len.shape[0]
    i32 = torch.int32
    check(_lib.load().srt_apply_spans(n, Bmax, _ptr(records, i32, "records"), _ptr(src, i32, "src"),
                                      _ptr(seq_tok, i32, "seq_tok"), seq_tok.shape[1],
                                      _ptr(seq_len, i32, "seq_len"), _ptr(frm, i32, "from"),
                                      _ptr(to, i32, "to"), _stream()), "srt_apply_spans")


def noise_table(device=None) -> torch.Tensor:
    L = _lib.load()
    out = torch.empty(1 << 23, dtype=torch.float32, device=device or "cuda")
    check(L.srt_noise_table(_ptr(out, torch.float32, "out"), _stream()), "srt_noise_table")
    return out


def log_det_range(first_bits: int, n: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """srt_log_det_range (test hook): log_det of the floats with bit patterns
    first_bits .. first_bits + n - 1, on the device."""
    L = _lib.load()
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device="cuda")
    check(L.srt_log_det_range(first_bits, n, _ptr(out[:n], torch.float32, "out"), _stream()),
          "srt_log_det_range")
    return out[:n]


def row_noise(vocab_size: int, seed: int, seq_id: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """srt_row_noise (test hook): the sampler's noise g_v, [n, V] float32."""
    L = _lib.load()
    n = seq_id.shape[0]
    out = torch.empty(n, vocab_size, dtype=torch.float32, device=seq_id.device)
    check(L.srt_row_noise(vocab_size, seed & (2**64 - 1), n, _ptr(seq_id, torch.int64, "seq_id"),
                          _ptr(pos, torch.int32, "pos"), _ptr(out, torch.float32, "out"),
                          _stream()), "srt_row_noise")
    return out


def stream_read(buf: torch.Tensor, chunk: int = 32768, nbuf: int = 6, ctas_per_sm: int = 1,
                sink: torch.Tensor | None = None) -> None:
    """srt_stream_read (measurement hook): read `buf` once through a TMA ring."""
    L = _lib.load()
    if sink is None:
        sink = torch.empty(1, dtype=torch.int64, device=buf.device)
    check(L.srt_stream_read(_ptr(buf, None, "buf"), buf.numel() * buf.element_size(), chunk, nbuf,
                            ctas_per_sm, _ptr(sink, torch.int64, "sink"), _stream()),
          "srt_stream_read")
