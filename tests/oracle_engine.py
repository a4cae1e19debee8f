"""The rollout simulation's engine on the CPU oracle (test infrastructure):
the same interface as paper_2601_09083_b200.rollout.GpuEngine -- per tick the
oracle's draft over the occupied slots, the policy stand-in as dense bf16
rows, the oracle's verify, and the oracle's insert of the committed spans."""
from __future__ import annotations

import numpy as np

import oracle
from synth import bf16_bits


class OracleEngine:
    def __init__(self, cfg, policy):
        self.cfg, self.policy = cfg, policy
        S, W = cfg.n_slots, cfg.cap + cfg.Bmax + 1
        self.orc = oracle.Oracle(cfg.V, cfg.n_prompts, cfg.D, cfg.L, cfg.Bmax)
        self.tok = np.zeros((S, W), np.int32)
        self.len = np.zeros(S, np.int32)
        self.prompt = np.zeros(S, np.int32)
        self.maxn = np.zeros(S, np.int32)
        self.key = np.zeros(S, np.uint64)
        self.truth = np.zeros((S, cfg.cap), np.int32)
        self.tlen = np.zeros(S, np.int64)
        self.seed = (cfg.seed * 0x9E3779B97F4A7C15 + 17) & (2 ** 64 - 1)

    def place(self, slot, prompt, key, truth):
        self.len[slot] = 0
        self.prompt[slot] = prompt
        self.maxn[slot] = len(truth)
        self.key[slot] = key
        self.truth[slot, :len(truth)] = truth
        self.tlen[slot] = len(truth)

    def insert_streams(self, prompts, streams):
        if not streams:
            return
        W = max(len(s) for s in streams)
        tab = np.zeros((len(streams), W), np.int32)
        for i, s in enumerate(streams):
            tab[i, :len(s)] = s
        self.orc.insert(np.asarray(prompts, np.int32), tab, np.zeros(len(streams), np.int32),
                        np.asarray([len(s) for s in streams], np.int32))

    def tick(self, slots, insert):
        tok = np.ascontiguousarray(self.tok[slots])
        ln = np.ascontiguousarray(self.len[slots])
        t0 = ln.copy()
        prompt = self.prompt[slots]
        d = self.orc.draft(prompt, tok, ln, ln)
        rows = int(d["row_offsets"][-1])
        et, ev = self.policy(slots, d["row_offsets"], d["draft_len"], d["draft_depth"],
                             self.len, self.key, self.truth, self.tlen)
        x = np.zeros((rows, self.cfg.V), np.float32)
        np.put_along_axis(x, et, ev, axis=1)
        v = self.orc.verify(bf16_bits(x), d["row_offsets"], d["draft_len"], d["draft_tok"],
                            d["draft_parent"], d["draft_depth"], self.key[slots], self.seed, tok,
                            ln, self.maxn[slots])
        if insert:
            self.orc.insert(prompt, tok, t0, ln)
        self.tok[slots] = tok
        self.len[slots] = ln
        assert self.orc.error_bits == 0
        return {"accept_len": v["accept_len"], "n_commit": v["n_commit"],
                "commit_tok": v["commit_tok"], "draft_len": d["draft_len"],
                "match_len": d["match_len"]}

    def dump(self, p):
        return [tuple(int(x) for x in r) for r in self.orc.dump(p)]
