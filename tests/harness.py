"""Test harness: drive the CUDA path (paper_2601_09083_b200, via the C ABI) and
the oracle on the SAME seeded inputs and compare every output element.
Only the inputs are shared; each side computes independently."""
from __future__ import annotations

import numpy as np


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


class Pair:
    """A GPU cache and an oracle cache with the same configuration."""

    def __init__(self, orc, V, P, D, L, Bmax, b0=None, num=0, den=1, min_score=0.0,
                 node_capacity=1 << 16, dtype="bf16"):
        import torch
        import paper_2601_09083_b200 as srt
        self.torch = torch
        self.V, self.P, self.D, self.L, self.Bmax = V, P, D, L, Bmax
        self.dtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        cfg = srt.config(V, P, D, L, Bmax, budget_base=b0, slope_num=num, slope_den=den,
                         min_path_score=min_score, node_capacity=node_capacity,
                         logits_dtype=self.dtype)
        self.gpu = srt.SrtCache(cfg)
        self.orc = orc.Oracle(V, P, D, L, Bmax, budget_base=b0, slope_num=num, slope_den=den,
                              min_path_score=min_score)

    def t(self, a, dtype=None):
        x = self.torch.from_numpy(np.ascontiguousarray(a))
        if dtype is not None:
            x = x.to(dtype)
        return x.cuda()

    # -- insert on both ------------------------------------------------------
    def insert(self, prompt_id, seq_tok, frm, to, floor=None, cursor=None, stats=None):
        n = len(prompt_id)
        fl = np.zeros(n, np.int32) if floor is None else np.asarray(floor, np.int32)
        self.orc.insert(prompt_id, seq_tok, frm, to, fl)
        self.gpu.insert(self.t(np.asarray(prompt_id, np.int32)), self.t(np.asarray(seq_tok, np.int32)),
                        self.t(np.asarray(frm, np.int32)), self.t(np.asarray(to, np.int32)),
                        self.t(fl), cursor=cursor, stats=stats)

    def compare_trees(self):
        for p in range(self.P):
            g = self.gpu.dump(p)
            o = [tuple(int(v) for v in r) for r in self.orc.dump(p)]
            g = [(t, c, n) for (t, c, n) in g]
            assert g == o, f"tree of prompt {p} differs ({len(g)} vs {len(o)} records)"
        bits, _ = self.gpu.status()
        assert not bits & 0x10, "child-slot mirrors disagree with the node arrays"

    # -- draft on both -------------------------------------------------------
    def draft(self, prompt_id, seq_tok, seq_len, pos_base=None):
        n = len(prompt_id)
        pb = np.zeros(n, np.int32) if pos_base is None else np.asarray(pos_base, np.int32)
        od = self.orc.draft(prompt_id, seq_tok, seq_len, pb)
        gd = self.gpu.draft(self.t(np.asarray(prompt_id, np.int32)),
                            self.t(np.asarray(seq_tok, np.int32)),
                            self.t(np.asarray(seq_len, np.int32)), self.t(pb))
        return od, gd

    @staticmethod
    def compare_drafts(od, gd):
        for k in ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth",
                  "draft_pos", "row_offsets"):
            g = getattr(gd, k).cpu().numpy()
            assert np.array_equal(g, od[k].astype(g.dtype)), k
        gm = gd.draft_mask.cpu().numpy().view(np.uint64)
        assert np.array_equal(gm, od["draft_mask"]), "draft_mask"

    # -- verify on both --------------------------------------------------------
    def verify(self, logits_f32, od, gd, seq_id, seed, seq_tok, seq_len, max_new,
               temperature=1.0, eos=-1):
        """logits_f32: float32 numpy rows; converted to the cache dtype for
        both sides identically (bf16 = round-to-nearest-even bits)."""
        from synth import bf16_bits
        torch = self.torch
        if self.dtype == torch.bfloat16:
            bits = bf16_bits(logits_f32)
            host = bits
            dev = self.t(bits.view(np.int16)).view(torch.bfloat16)
        else:
            host = np.ascontiguousarray(logits_f32, np.float32)
            dev = self.t(host)
        o_tok = np.array(seq_tok, np.int32, copy=True)
        o_len = np.array(seq_len, np.int32, copy=True)
        ov = self.orc.verify(host, od["row_offsets"], od["draft_len"], od["draft_tok"],
                             od["draft_parent"], od["draft_depth"], np.asarray(seq_id, np.uint64),
                             seed, o_tok, o_len, np.asarray(max_new, np.int32),
                             temperature=temperature, eos_id=eos)
        g_tok = self.t(np.asarray(seq_tok, np.int32))
        g_len = self.t(np.asarray(seq_len, np.int32))
        gv = self.gpu.verify(dev, gd, self.t(np.asarray(seq_id, np.uint64).view(np.int64)), seed,
                             g_tok, g_len, self.t(np.asarray(max_new, np.int32)),
                             temperature=temperature, eos_id=eos,
                             rows=int(od["row_offsets"][-1]))
        return ov, gv, (o_tok, o_len), (g_tok, g_len), dev

    @staticmethod
    def compare_verify(ov, gv, o_seq, g_seq):
        for k in ("sampled", "accept_len", "n_commit", "commit_tok", "accepted_nodes", "finished"):
            g = getattr(gv, k).cpu().numpy()
            assert np.array_equal(g, ov[k].astype(g.dtype)), k
        assert np.array_equal(g_seq[0].cpu().numpy(), o_seq[0]), "seq_tok"
        assert np.array_equal(g_seq[1].cpu().numpy(), o_seq[1]), "seq_len"
