"""Multi-GPU exchange protocol (paper_2601_09083_b200.dist) on
CPU: world_size 2 over gloo, with the oracle standing in for libsrt's kernels
(tests only).  Each rank owns the trees of its hash-sharded prompts, drafts
for their mirrored sequences, returns the drafts by all-to-all, verifies its
own contiguous share of the sequences and all-gathers the committed spans to
the owners.  G-invariance: every rank's committed tokens and owned trees must
equal a single-process run of the same workload, bit for bit."""
import os
import socket

import numpy as np
import pytest

V, D, L, B = 40, 6, 4, 6
STEPS = 6


def _workload():
    from synth import make_workload
    w = make_workload(11, V, n_prompts=5, samples=3, median=40, cap=64, prior_epochs=1)
    S = len(w.truth)
    t0 = np.array([min(4 + (s * 7) % 13, len(w.truth[s]) - 1) for s in range(S)], np.int32)
    max_new = np.array([len(t) for t in w.truth], np.int32)
    return w, t0, max_new


def _row_logits(seq, pos, tok, truth):
    """Deterministic stand-in forward: a function of (sequence, position,
    node token) only, so it does not depend on where the row is computed."""
    rng = np.random.default_rng([seq, pos, tok + 1])
    x = rng.normal(0.0, 2.0, V).astype(np.float32)
    x[truth[min(pos, len(truth) - 1)]] += 7.0
    return x


def _logits(seqs, d, seq_len, w):
    rows = int(d["row_offsets"][-1])
    out = np.zeros((rows, V), np.float32)
    for j, s in enumerate(seqs):
        r0 = int(d["row_offsets"][j])
        out[r0] = _row_logits(s, int(seq_len[j]), -1, w.truth[s])
        for i in range(int(d["draft_len"][j])):
            out[r0 + 1 + i] = _row_logits(s, int(seq_len[j] + d["draft_depth"][j, i]),
                                          int(d["draft_tok"][j, i]), w.truth[s])
    return out


def _tables(w, seqs, t0, stride):
    tab = np.zeros((len(seqs), stride), np.int32)
    for j, s in enumerate(seqs):
        tab[j, :t0[s]] = w.truth[s][:t0[s]]
    return tab, t0[seqs].astype(np.int32).copy()


def _reference(orc_mod):
    """Single process, all prompts in one oracle cache."""
    w, t0, max_new = _workload()
    S = len(w.truth)
    o = orc_mod.Oracle(V, w.n_prompts, D, L, B)
    for p, tk in w.prior:
        o.insert_sequence(p, tk)
    seqs = np.arange(S)
    tab, ln = _tables(w, seqs, t0, 64 + B + 2)
    o.insert(w.seq_prompt, tab, np.zeros(S, np.int32), ln)
    for k in range(STEPS):
        d = o.draft(w.seq_prompt, tab, ln, ln)
        x = _logits(seqs, d, ln, w)
        before = ln.copy()
        o.verify(x, d["row_offsets"], d["draft_len"], d["draft_tok"], d["draft_parent"],
                 d["draft_depth"], w.seq_id, 1234, tab, ln, max_new)
        o.insert(w.seq_prompt, tab, before, ln)
    return tab, ln, o, w


class OracleOps:
    """ShardedStep ops with the oracle as the engine (numpy)."""

    def __init__(self, o, w, plan, rank, t0, max_new):
        self.o, self.w, self.plan, self.rank = o, w, plan, rank
        self.mirror = plan.mirror[rank]
        self.mprompt = plan.mirror_prompt[rank]
        self.local = plan.local[rank]
        stride = 64 + B + 2
        self.mtab, self.mlen = _tables(w, self.mirror, t0, stride)
        self.ltab, self.llen = _tables(w, self.local, t0, stride)
        self.max_new = max_new[self.local]
        self.md = None

    def draft_mirror(self):
        self.md = self.o.draft(self.mprompt, self.mtab, self.mlen, self.mlen)

    def pack_drafts(self, send):
        a = send.numpy()
        n = len(self.mirror)
        a[:n, 0] = self.md["match_len"]
        a[:n, 1] = self.md["draft_len"]
        a[:n, 2:2 + B] = self.md["draft_tok"]
        a[:n, 2 + B:2 + 2 * B] = self.md["draft_parent"]
        a[:n, 2 + 2 * B:2 + 3 * B] = self.md["draft_depth"]
        m = self.md["draft_mask"]
        a[:n, 2 + 3 * B:2 + 4 * B] = (m & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
        a[:n, 2 + 4 * B:2 + 5 * B] = (m >> np.uint64(32)).astype(np.uint32).view(np.int32)

    def unpack_drafts(self, recv, src):
        r = recv.numpy()[src.numpy()]
        dl = r[:, 1].astype(np.int32)
        self.ld = dict(match_len=r[:, 0].copy(), draft_len=dl,
                       draft_tok=r[:, 2:2 + B].copy(), draft_parent=r[:, 2 + B:2 + 2 * B].copy(),
                       draft_depth=r[:, 2 + 2 * B:2 + 3 * B].copy(),
                       row_offsets=np.concatenate([[0], np.cumsum(dl.astype(np.int64) + 1)]))

    def verify(self):
        x = _logits(self.local, self.ld, self.llen, self.w)
        self.v = self.o_verify(x)

    def o_verify(self, x):
        d = self.ld
        return self.o.verify(x, d["row_offsets"], d["draft_len"], d["draft_tok"],
                             d["draft_parent"], d["draft_depth"], self.w.seq_id[self.local], 1234,
                             self.ltab, self.llen, self.max_new)

    def pack_spans(self, send):
        a = send.numpy()
        n = len(self.local)
        a[:n, 0] = self.v["n_commit"]
        a[:n, 1:] = self.v["commit_tok"]

    def apply_and_insert(self, recv, src):
        r = recv.numpy()[src.numpy()]
        frm = self.mlen.copy()
        for j in range(len(self.mirror)):
            k = int(r[j, 0])
            self.mtab[j, frm[j]:frm[j] + k] = r[j, 1:1 + k]
        self.mlen = (frm + r[:, 0]).astype(np.int32)
        self.o.insert(self.mprompt, self.mtab, frm, self.mlen)


def _worker(rank, world, port, result_dir):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2601_09083_b200.dist import ShardPlan, ShardedStep, all_gather_rows, all_to_all_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ref_tab, ref_len, ref_o, w = _reference(oracle)
        _, t0, max_new = _workload()
        plan = ShardPlan.build(w.seq_prompt, world)
        mine = plan.prompts[rank]
        o = oracle.Oracle(V, max(1, len(mine)), D, L, B)
        for p, tk in w.prior:
            if p in mine:
                o.insert_sequence(int(np.searchsorted(mine, p)), tk)
        ops = OracleOps(o, w, plan, rank, t0, max_new)
        if len(ops.mirror):
            o.insert(ops.mprompt, ops.mtab, np.zeros(len(ops.mirror), np.int32), ops.mlen)
        step = ShardedStep(plan, rank, ops, all_gather_rows, B, a2a=all_to_all_rows)
        for k in range(STEPS):
            step.draft()
            ops.verify()
            step.commit()
        # G-invariance: local commits and owned trees equal the single-process run
        assert np.array_equal(ops.llen, ref_len[plan.local[rank]])
        assert np.array_equal(ops.ltab, ref_tab[plan.local[rank]])
        assert np.array_equal(ops.mlen, ref_len[plan.mirror[rank]])
        for i, p in enumerate(mine):
            assert np.array_equal(np.asarray(o.dump(i)), np.asarray(ref_o.dump(int(p)))), f"tree {p}"
        assert (ref_len > t0).all()
        with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
            f.write(f"{len(plan.local[rank])} local, {len(plan.mirror[rank])} mirror")
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_routing_is_a_bijection():
    from paper_2601_09083_b200.dist import ShardPlan, owner_of
    seq_prompt = np.repeat(np.arange(37), 4)
    for G in (1, 2, 3, 8):
        plan = ShardPlan.build(seq_prompt, G)
        S = len(seq_prompt)
        assert sorted(np.concatenate(plan.local).tolist()) == list(range(S))
        assert sorted(np.concatenate(plan.mirror).tolist()) == list(range(S))
        for r in range(G):
            assert all(owner_of(int(seq_prompt[s]), G) == r for s in plan.mirror[r])
            # the draft of local[r][i] comes from its owner's mirror slot: rank
            # r's all-to-all receive buffer is, owner by owner, the slice of
            # each owner's mirror records that r decodes
            recv = []
            for o in range(G):
                offs = np.concatenate([[0], np.cumsum(plan.draft_send[o])])
                recv += list(plan.mirror[o][offs[r]:offs[r + 1]])
                assert plan.draft_recv[r][o] == plan.draft_send[o][r]
            assert len(recv) == len(plan.local[r]) == sum(plan.draft_recv[r])
            for i, s in enumerate(plan.local[r]):
                assert recv[int(plan.draft_src[r][i])] == s
            for j, s in enumerate(plan.mirror[r]):
                src = int(plan.span_src[r][j])
                dr = src // plan.n_local_max
                assert plan.local[dr][src % plan.n_local_max] == s
            assert (plan.prompts[r][plan.mirror_prompt[r]] == seq_prompt[plan.mirror[r]]).all()


def test_gloo_world2_matches_single_process(orc, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()
