"""rollout.py — the rollout loop around the SRT step: slots, bubbles and
run-ahead generation.

P:L50-51 (§1): "when only a few long sequences remain, GPUs sit idle; SRT
uses these bubbles to generate rollouts for prompts that will be sampled
soon"; P:L151 (§3, cache update strategy): the tree of a prompt is updated
online from its running rollouts and from run-ahead rollouts of look-ahead
prompts, which are "never used for learning targets"; P:L196-204 (§4, Fig. 5):
history-only (cache updated with completed responses only) vs online vs
online + run-ahead, compared by mean accepted tokens.  SPEC's `scheduler`
module is followed for the interface only: discrete ticks, one
engine step per occupied slot and tick, K samples per prompt enqueued at the
start of a training step, freed slots filled first by queued real sequences,
then by run-ahead sequences of the look-ahead window, round robin (SPEC's
preemption of run-ahead occupants by newly enqueued real sequences cannot
occur: every real sequence of a step is queued when the step starts, and
run-ahead starts only once the queue is empty).  Run-ahead occupants are
discarded when the step's last real sequence completes.

This module is host logic only: every tick is ONE batched SRT step (draft ->
policy stand-in -> verify -> insert) through an engine.  `GpuEngine` drives
libsrt (the C ABI kernels) with device-resident slot tables; the tests drive
the same scheduler with an oracle engine and require identical per-tick
results.  The policy is a synthetic stand-in passed in by the caller
(`synth.SimPolicy`: head = the rollout's ground-truth token at the row's
position, sparse edits of an all-zero logits row), keyed by
(sequence, position) only, so every mode commits the same rollouts
(losslessness) and only the schedule and acceptance differ.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

MODES = ("baseline", "history_only", "srt")


@dataclass
class SimConfig:
    V: int
    D: int
    L: int
    Bmax: int
    prompts_per_step: int          # training batch B (prompts per training step)
    samples: int                   # K rollouts per prompt
    steps: int                     # training steps simulated
    slots: int = 0                 # concurrent sequences (0 = B * K)
    mode: str = "srt"              # baseline | history_only | srt
    run_ahead: bool = False
    lookahead: int = 0             # prompts in the look-ahead window (0 = next step's B)
    ra_per_prompt: int = 4         # run-ahead rollouts per look-ahead prompt and step
    epoch: int = 1                 # the epoch being decoded (epoch 0 = the warm history)
    warm: bool = True              # epoch-0 rollouts of every prompt inserted first
    median: int = 64
    cap: int = 256
    profile: str = "rl-mix"
    seed: int = 0
    node_capacity: int = 1 << 22   # GpuEngine's cache size

    def validate(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.run_ahead and self.mode != "srt":
            raise ValueError("run-ahead needs online insertion (mode 'srt')")
        if min(self.prompts_per_step, self.samples, self.steps) < 1:
            raise ValueError("prompts_per_step, samples and steps must be >= 1")
        if self.n_slots < 1 or self.lookahead < 0 or self.ra_per_prompt < 0:
            raise ValueError("bad slot / look-ahead configuration")

    @property
    def n_slots(self) -> int:
        return self.slots or self.prompts_per_step * self.samples

    @property
    def n_prompts(self) -> int:
        return self.prompts_per_step * (self.steps + 1)  # + the last step's look-ahead

    def window(self) -> int:
        return self.lookahead or self.prompts_per_step


RA_BIT = 1 << 63


def seq_key(step: int, prompt: int, j: int, run_ahead: bool = False) -> int:
    """u64 sequence id (the Philox key of its rows): step, prompt, sample."""
    return (RA_BIT if run_ahead else 0) | (step << 44) | (prompt << 16) | j


@dataclass
class Seq:
    key: int
    prompt: int
    truth: np.ndarray
    real: bool
    slot: int = -1
    length: int = 0
    tokens: list = field(default_factory=list)

    @property
    def max_new(self) -> int:
        return len(self.truth)

    @property
    def done(self) -> bool:
        return self.length >= self.max_new


@dataclass
class StepReport:
    step: int
    ticks: int                     # simulated time (one engine step per tick)
    tokens: int                    # tokens committed by real sequences
    seq_ticks: int                 # engine steps of real sequences
    accepted: int                  # accepted draft tokens of real sequences
    mean_accepted: float           # accepted / seq_ticks (Fig. 5's metric)
    mean_committed: float          # tokens / seq_ticks
    bubble_slot_ticks: int         # slot-ticks with no real sequence
    run_ahead_seqs: int
    run_ahead_tokens: int

    def as_dict(self) -> dict:
        return dict(self.__dict__)


class RolloutSim:
    """Simulates `cfg.steps` training steps of rollout generation through an
    engine (see GpuEngine for the interface)."""

    def __init__(self, cfg: SimConfig, engine, streams):
        cfg.validate()
        self.cfg, self.eng, self.streams = cfg, engine, streams
        self.trace = []          # per tick: dict (busy, free, real, run_ahead, accepted, ...)
        self.rollouts = {}       # key -> committed tokens of each real sequence
        self.reports = []

    def _warm(self):
        c = self.cfg
        if c.mode == "baseline" or not c.warm or c.epoch < 1:
            return
        ps, st = [], []
        for p in range(c.n_prompts):
            for j in range(c.samples):
                ps.append(p)
                st.append(self.streams.stream(p, c.epoch - 1, j))
        self.eng.insert_streams(ps, st)

    def run(self):
        self._warm()
        for k in range(self.cfg.steps):
            self.reports.append(self._step(k))
        return self.reports

    def _step(self, k: int) -> StepReport:
        c, eng = self.cfg, self.eng
        S, B, K = c.n_slots, c.prompts_per_step, c.samples
        batch = list(range(k * B, (k + 1) * B))
        queue = deque(Seq(seq_key(k, p, j), p, self.streams.stream(p, c.epoch, j), True)
                      for p in batch for j in range(K))
        window = [p for p in range((k + 1) * B, (k + 1) * B + c.window()) if p < c.n_prompts]
        ra_made = {p: 0 for p in window}
        rr = 0
        slots: list = [None] * S
        live_real = 0
        completed = []
        ticks = tokens = seq_ticks = accepted = bubbles = ra_seqs = ra_tokens = 0
        while queue or live_real:
            # ---- tick boundary: finished sequences leave, queued real ones enter
            for i in range(S):
                q = slots[i]
                if q is not None and q.done:
                    slots[i] = None
            free = [i for i in range(S) if slots[i] is None]
            while queue and free:
                self._place(slots, free.pop(0), queue.popleft())
                live_real += 1
            # ---- bubbles: run-ahead rollouts of the look-ahead prompts
            if c.run_ahead and window:
                free = [i for i in range(S) if slots[i] is None]
                for i in free:
                    for _ in range(len(window)):
                        p = window[rr % len(window)]
                        rr += 1
                        if ra_made[p] < c.ra_per_prompt:
                            j = K + ra_made[p]
                            ra_made[p] += 1
                            self._place(slots, i, Seq(seq_key(k, p, j, True), p,
                                                      self.streams.stream(p, c.epoch, j), False))
                            ra_seqs += 1
                            break
            occ = [q for q in slots if q is not None]
            n_real = sum(q.real for q in occ)
            assert len(occ) + sum(q is None for q in slots) == S  # slot conservation
            bubbles += S - n_real
            # ---- one engine step over every occupied slot (ascending slot order)
            occ.sort(key=lambda q: q.slot)
            res = eng.tick(np.array([q.slot for q in occ], np.int32), c.mode == "srt")
            t_acc = t_com = 0
            for q, a, n, ct in zip(occ, res["accept_len"], res["n_commit"], res["commit_tok"]):
                q.tokens.extend(int(x) for x in ct[:n])
                q.length += int(n)
                if q.real:
                    t_acc += int(min(a, max(n - 1, 0)))
                    t_com += int(n)
                    if q.done:
                        live_real -= 1
                        completed.append(q)
                        self.rollouts[q.key] = np.asarray(q.tokens, np.int32)
                else:
                    ra_tokens += int(n)
            ticks += 1
            tokens += t_com
            seq_ticks += n_real
            accepted += t_acc
            self.trace.append(dict(step=k, tick=ticks, busy=len(occ), free=S - len(occ),
                                   real=n_real, run_ahead=len(occ) - n_real, accepted=t_acc,
                                   committed=t_com))
        if c.mode == "history_only":  # completed responses enter the cache at step end
            completed.sort(key=lambda q: q.key)
            eng.insert_streams([q.prompt for q in completed],
                               [np.asarray(q.tokens, np.int32) for q in completed])
        for i in range(S):  # run-ahead occupants are discarded (never learning targets)
            slots[i] = None
        return StepReport(step=k, ticks=ticks, tokens=tokens, seq_ticks=seq_ticks,
                          accepted=accepted, mean_accepted=accepted / max(seq_ticks, 1),
                          mean_committed=tokens / max(seq_ticks, 1), bubble_slot_ticks=bubbles,
                          run_ahead_seqs=ra_seqs, run_ahead_tokens=ra_tokens)

    def _place(self, slots, i: int, q: Seq):
        q.slot = i
        slots[i] = q
        self.eng.place(i, q.prompt, q.key, q.truth)


class GpuEngine:
    """The SRT step on the GPU through libsrt: per tick srt_draft over the
    occupied slots, the policy stand-in written into a bf16 logits buffer,
    srt_verify, and srt_insert of the committed spans (online modes).  Slot
    tables (response tokens, lengths, prompt, key, max_new) stay on the
    device; the host sees only each tick's draft layout (for the stand-in)
    and commits."""

    def __init__(self, cfg: SimConfig, policy, device=None):
        import torch
        from . import srt
        self.torch, self.cfg, self.policy = torch, cfg, policy
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        S, W = cfg.n_slots, cfg.cap + cfg.Bmax + 1
        self.cache = srt.SrtCache(srt.config(cfg.V, cfg.n_prompts, cfg.D, cfg.L, cfg.Bmax,
                                             node_capacity=cfg.node_capacity, logits_dtype=torch.bfloat16),
                                  self.dev)
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.tok = torch.zeros((S, W), **i32)
        self.len = torch.zeros(S, **i32)
        self.prompt = torch.zeros(S, **i32)
        self.maxn = torch.zeros(S, **i32)
        self.key = torch.zeros(S, dtype=torch.int64, device=self.dev)
        self.h_len = np.zeros(S, np.int64)
        self.h_key = np.zeros(S, np.uint64)
        self.h_truth = np.zeros((S, cfg.cap), np.int32)
        self.h_tlen = np.zeros(S, np.int64)
        self.rows_cap = S * (cfg.Bmax + 1)
        self.logits = torch.zeros((self.rows_cap, cfg.V), dtype=torch.bfloat16, device=self.dev)
        self.seed = (cfg.seed * 0x9E3779B97F4A7C15 + 17) & (2 ** 64 - 1)

    def place(self, slot: int, prompt: int, key: int, truth: np.ndarray):
        self.len[slot] = 0
        self.prompt[slot] = prompt
        self.maxn[slot] = len(truth)
        self.key[slot] = int(np.uint64(key).view(np.int64))
        self.h_len[slot] = 0
        self.h_key[slot] = key
        self.h_truth[slot, :len(truth)] = truth
        self.h_tlen[slot] = len(truth)

    def insert_streams(self, prompts, streams):
        if not streams:
            return
        torch = self.torch
        W = max(len(s) for s in streams)
        tab = np.zeros((len(streams), W), np.int32)
        for i, s in enumerate(streams):
            tab[i, :len(s)] = s
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(self.dev)
        self.cache.insert(t(prompts), t(tab), t(np.zeros(len(streams))),
                          t([len(s) for s in streams]))

    def tick(self, slots: np.ndarray, insert: bool) -> dict:
        torch = self.torch
        idx = torch.from_numpy(slots.astype(np.int64)).to(self.dev)
        tok = self.tok.index_select(0, idx)
        ln = self.len.index_select(0, idx)
        t0 = ln.clone()
        prompt = self.prompt.index_select(0, idx)
        d = self.cache.draft(prompt, tok, ln, ln)
        ro = d.row_offsets.cpu().numpy()
        dl = d.draft_len.cpu().numpy()
        dd = d.draft_depth.cpu().numpy()
        rows = int(ro[-1])
        et, ev = self.policy(slots, ro, dl, dd, self.h_len, self.h_key, self.h_truth,
                             self.h_tlen)
        lin = torch.from_numpy((np.arange(rows)[:, None] * self.cfg.V + et).reshape(-1)).to(self.dev)
        flat = self.logits.view(-1)
        flat[lin] = torch.from_numpy(ev.reshape(-1)).to(self.dev).to(torch.bfloat16)
        v = self.cache.verify(self.logits, d, self.key.index_select(0, idx), self.seed, tok, ln,
                              self.maxn.index_select(0, idx), rows=max(rows, 1))
        flat[lin] = 0
        if insert:
            self.cache.insert(prompt, tok, t0, ln)
        self.tok.index_copy_(0, idx, tok)
        self.len.index_copy_(0, idx, ln)
        out = {"accept_len": v.accept_len.cpu().numpy(), "n_commit": v.n_commit.cpu().numpy(),
               "commit_tok": v.commit_tok.cpu().numpy(), "draft_len": dl,
               "match_len": d.match_len.cpu().numpy()}
        self.h_len[slots] += out["n_commit"]
        bits, _ = self.cache.status()
        if bits:
            raise RuntimeError(f"libsrt device error bits {bits:#x}")
        return out

    def dump(self, p: int):
        return self.cache.dump(p)


def summarize(reports) -> dict:
    """Totals over the simulated training steps."""
    st = sum(r.seq_ticks for r in reports)
    return {"ticks": sum(r.ticks for r in reports),
            "tokens": sum(r.tokens for r in reports),
            "mean_accepted": sum(r.accepted for r in reports) / max(st, 1),
            "mean_committed": sum(r.tokens for r in reports) / max(st, 1),
            "bubble_slot_ticks": sum(r.bubble_slot_ticks for r in reports),
            "run_ahead_seqs": sum(r.run_ahead_seqs for r in reports),
            "run_ahead_tokens": sum(r.run_ahead_tokens for r in reports),
            "per_step": [r.as_dict() for r in reports]}
