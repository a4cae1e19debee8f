"""srt_verify_path: sampling only the rows the commit needs
must commit exactly what srt_verify / the oracle commit, for every number of
path rounds (0 = every row, then 1, 2, 3 rounds before the subtree tail, and
more rounds than any path is long), and its samples on the path are the
oracle's.  Logits put a large head on a draft child's token with high
probability, so walks go deep and every round and the tail are exercised."""
import numpy as np
import pytest

from harness import Pair

pytestmark = pytest.mark.gpu


def _insert_all(pair, seqs, width=80):
    tab = np.zeros((len(seqs), width), np.int32)
    for i, (_, t) in enumerate(seqs):
        tab[i, :len(t)] = t
    pair.insert(np.array([p for p, _ in seqs], np.int32), tab, np.zeros(len(seqs), np.int32),
                np.array([len(t) for _, t in seqs], np.int32))


def _deep_logits(rng, od, V, B, p_follow=0.85, gap=40.0):
    rows = int(od["row_offsets"][-1])
    x = rng.normal(0, 2, (rows, V)).astype(np.float32)
    n = len(od["draft_len"])
    for s in range(n):
        r0, ns = int(od["row_offsets"][s]), int(od["draft_len"][s])
        par = od["draft_parent"][s, :ns]
        tok = od["draft_tok"][s, :ns]
        for node in range(-1, ns):
            kids = np.nonzero(par == node)[0]
            if len(kids) and rng.random() < p_follow:
                head = int(tok[rng.choice(kids)])
            else:
                head = int(rng.integers(0, V))
            x[r0 + 1 + node, head] = gap
    return x


@pytest.mark.parametrize("V", [1000, 151936])
def test_path_verify_matches_oracle(orc, V):
    import torch
    rng = np.random.default_rng(V)
    D, L, Bmax = 16, 6, 32
    pair = Pair(orc, V, 2, D, L, Bmax, node_capacity=1 << 18)
    base = rng.integers(0, 40, 70).astype(np.int32)
    seqs = [(k % 2, np.where(rng.random(70) < 0.05, rng.integers(0, 40, 70), base).astype(np.int32))
            for k in range(16)]
    _insert_all(pair, seqs)
    n = 48 if V < 100000 else 24
    ctx = np.zeros((n, 70 + Bmax + 2), np.int32)
    ctx[:, :70] = base
    seq_len = rng.integers(2, 40, n).astype(np.int32)
    prompts = rng.integers(0, 2, n).astype(np.int32)
    od, gd = pair.draft(prompts, ctx, seq_len)
    pair.compare_drafts(od, gd)
    logits = _deep_logits(rng, od, V, Bmax)
    max_new = np.full(n, 200, np.int32)
    sid = rng.integers(0, 2 ** 62, n).astype(np.uint64)
    ov, gv, o_seq, g_seq, dev = pair.verify(logits, od, gd, sid, 77, ctx, seq_len, max_new)
    pair.compare_verify(ov, gv, o_seq, g_seq)
    assert ov["accept_len"].max() >= 4, "walks too shallow to exercise the rounds"
    rows = int(od["row_offsets"][-1])
    for R in (0, 1, 2, 3, 40):
        g_tok = pair.t(ctx)
        g_len = pair.t(seq_len)
        pv = pair.gpu.verify(dev, gd, pair.t(sid.view(np.int64)), 77, g_tok, g_len,
                             pair.t(max_new), rows=rows, path_rounds=R)
        for k in ("accept_len", "n_commit", "commit_tok", "accepted_nodes", "finished"):
            g = getattr(pv, k).cpu().numpy()
            assert np.array_equal(g, ov[k].astype(g.dtype)), (R, k)
        assert np.array_equal(g_tok.cpu().numpy(), o_seq[0]), R
        assert np.array_equal(g_len.cpu().numpy(), o_seq[1]), R
        sm = pv.sampled[:rows].cpu().numpy()
        done = sm >= 0
        assert np.array_equal(sm[done], ov["sampled"][done]), R
        for s in range(n):  # the root and every accepted node's row were sampled
            r0 = int(od["row_offsets"][s])
            assert done[r0]
            for a in range(int(ov["accept_len"][s])):
                assert done[r0 + 1 + int(ov["accepted_nodes"][s, a])], (R, s, a)
        if R == 0:
            assert done.all()
        else:
            assert done.sum() < rows  # fewer rows read than srt_verify
    torch.cuda.synchronize()
