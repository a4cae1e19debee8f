"""Pins for the oracle's verify (sample at every draft row + first-mismatch
walk + commit; O9-O14).

P8   losslessness: speculative decoding with drafts from warm trees produces the
     token stream of plain decoding (empty drafts), token for token, under the
     position-keyed sampler; a mis-keyed position (negative control) diverges.
P10  empty draft: the root's sample is the plain decode token at position t.
P11  the accepted nodes form a root path of the draft; committed[k] = the
     sample at path node k; a <= n_s.
Forced-logit closed forms for the walk, EOS and length truncation.
"""
import numpy as np
import pytest

from synth import splitmix64

M64 = (1 << 64) - 1


def policy_row(ctx, V, k=2, seed=0):
    """A context-keyed synthetic policy: logits depend on the last k tokens."""
    h = seed
    for t in ctx[-k:] if k else []:
        h = splitmix64((h ^ (int(t) + 1)) & M64)
    rng = np.random.default_rng(h)
    x = rng.normal(0.0, 1.0, V).astype(np.float32)
    x[int(rng.integers(0, V))] += 5.0
    return x


def _empty_draft(n, B):
    return dict(draft_len=np.zeros(n, np.int32), draft_tok=np.full((n, B), -1, np.int32),
                draft_parent=np.full((n, B), -1, np.int32), draft_depth=np.zeros((n, B), np.int32),
                row_offsets=np.arange(n + 1, dtype=np.int64))


def _node_ctx(y, d, i):
    path = []
    while i >= 0:
        path.append(int(d["draft_tok"][0, i]))
        i = int(d["draft_parent"][0, i])
    return list(y) + path[::-1]


def rollout(orc, o, p, sid, seed, V, max_new, speculative, k=2, pos_shift=0, eos=-1):
    """Decode one sequence to completion; returns (tokens, n_steps, accepted)."""
    B = o.Bmax
    seq_tok = np.zeros((1, max_new + B + 2), np.int32)
    seq_len = np.zeros(1, np.int32)
    steps = acc_total = 0
    while True:
        t = int(seq_len[0])
        if speculative:
            d = o.draft([p], seq_tok, seq_len, pos_base=[t])
        else:
            d = _empty_draft(1, B)
        n = int(d["draft_len"][0])
        rows = [policy_row(seq_tok[0, :t].tolist(), V, k)]
        for i in range(n):
            rows.append(policy_row(_node_ctx(seq_tok[0, :t].tolist(), d, i), V, k))
        depth = d["draft_depth"].copy()
        depth[0, :n] += pos_shift  # negative control: mis-keyed positions
        r = o.verify(np.stack(rows), d["row_offsets"], d["draft_len"], d["draft_tok"],
                     d["draft_parent"], depth, np.array([sid], np.uint64), seed, seq_tok,
                     seq_len, np.array([max_new], np.int32), eos_id=eos)
        nc = int(r["n_commit"][0])
        a = int(r["accept_len"][0])
        assert 0 <= a <= n
        assert nc == a + 1 or r["finished"][0]
        # online insertion of the freshly decoded span
        o.insert([p], seq_tok, [t], [t + nc])
        steps += 1
        acc_total += a
        if r["finished"][0]:
            return seq_tok[0, :int(seq_len[0])].tolist(), steps, acc_total


@pytest.mark.parametrize("trial", range(60))
def test_losslessness(orc, trial):
    """P8 (S:L554 analog): speculative == plain decoding, token for token."""
    rng = np.random.default_rng(trial)
    V = int(rng.integers(6, 14))
    D = int(rng.integers(3, 9))
    L = int(rng.integers(1, D + 1))
    Bmax = int(rng.integers(1, 10))
    o_spec = orc.Oracle(V, 1, D, L, Bmax)
    o_warm = orc.Oracle(V, 1, D, L, Bmax)  # unused tree for the baseline runs
    seed = int(rng.integers(0, 1 << 62))
    max_new = int(rng.integers(5, 40))
    eos = int(rng.integers(0, V)) if trial % 3 == 0 else -1
    # warm the tree with sibling rollouts of the same policy (other seq ids)
    for sib in range(3):
        toks, _, _ = rollout(orc, o_warm, 0, 1000 + sib, seed, V, max_new, False, eos=eos)
        if toks:
            o_spec.insert_sequence(0, np.asarray(toks, np.int32))
    spec, spec_steps, acc = rollout(orc, o_spec, 0, 7, seed, V, max_new, True, eos=eos)
    base, base_steps, _ = rollout(orc, o_warm, 0, 7, seed, V, max_new, False, eos=eos)
    assert spec == base
    assert spec_steps <= base_steps  # step-count dominance
    assert spec_steps + acc >= len(spec) if spec else True


def test_losslessness_accepts_something(orc):
    """The test above is not vacuous: warm trees make drafts get accepted."""
    V, D, L, Bmax = 8, 8, 4, 8
    seed = 99
    total_acc = 0
    for trial in range(10):
        o = orc.Oracle(V, 1, D, L, Bmax)
        w = orc.Oracle(V, 1, D, L, Bmax)
        for sib in range(4):
            toks, _, _ = rollout(orc, w, 0, 500 + sib, seed + trial, V, 30, False)
            o.insert_sequence(0, np.asarray(toks, np.int32))
        _, _, acc = rollout(orc, o, 0, 1, seed + trial, V, 30, True)
        total_acc += acc
    assert total_acc > 20


def test_negative_control_miskeyed_position(orc):
    """shifting the position key of draft rows must break exactness."""
    diverged = 0
    for trial in range(20):
        V, D, L, Bmax = 8, 8, 4, 8
        seed = 1234 + trial
        o = orc.Oracle(V, 1, D, L, Bmax)
        w = orc.Oracle(V, 1, D, L, Bmax)
        for sib in range(3):
            toks, _, _ = rollout(orc, w, 0, 800 + sib, seed, V, 30, False)
            o.insert_sequence(0, np.asarray(toks, np.int32))
        w2 = orc.Oracle(V, 1, D, L, Bmax)
        base, _, _ = rollout(orc, w2, 0, 3, seed, V, 30, False)
        bad, _, _ = rollout(orc, o, 0, 3, seed, V, 30, True, pos_shift=1)
        diverged += bad != base
    assert diverged > 0


def test_empty_draft_root_sample(orc):
    """P10: with n_s = 0 the root sample is the plain decode token at t."""
    rng = np.random.default_rng(0)
    V, n = 97, 5
    o = orc.Oracle(V, 1, 4, 2, 4)
    d = _empty_draft(n, 4)
    logits = rng.normal(0, 2, (n, V)).astype(np.float32)
    seq_tok = np.zeros((n, 32), np.int32)
    seq_len = np.array([0, 3, 7, 1, 20], np.int32)
    t0 = seq_len.copy()
    sid = np.array([11, 12, 13, 14, 15], np.uint64)
    r = o.verify(logits, d["row_offsets"], d["draft_len"], d["draft_tok"], d["draft_parent"],
                 d["draft_depth"], sid, 5, seq_tok, seq_len, np.full(n, 100, np.int32))
    for s in range(n):
        want, _ = orc.sample_row(logits[s], 5, int(sid[s]), int(t0[s]))
        assert r["sampled"][s] == want
        assert r["accept_len"][s] == 0 and r["n_commit"][s] == 1
        assert seq_tok[s, t0[s]] == want and seq_len[s] == t0[s] + 1


def _forced_rows(tokens, V):
    """Rows whose sample is forced: +inf at the wanted token (O11: +inf wins)."""
    x = np.zeros((len(tokens), V), np.float32)
    for i, t in enumerate(tokens):
        x[i, t] = np.inf
    return x


def _draft_arrays(B, toks, parents, depths):
    n = len(toks)
    d = dict(draft_len=np.array([n], np.int32), draft_tok=np.full((1, B), -1, np.int32),
             draft_parent=np.full((1, B), -1, np.int32), draft_depth=np.zeros((1, B), np.int32),
             row_offsets=np.array([0, n + 1], np.int64))
    d["draft_tok"][0, :n] = toks
    d["draft_parent"][0, :n] = parents
    d["draft_depth"][0, :n] = depths
    return d


def _run_forced(orc, d, forced, max_new=100, eos=-1, t=5, B=8, V=10):
    o = orc.Oracle(V, 1, 4, 2, B)
    seq_tok = np.zeros((1, 64), np.int32)
    seq_len = np.array([t], np.int32)
    r = o.verify(_forced_rows(forced, V), d["row_offsets"], d["draft_len"], d["draft_tok"],
                 d["draft_parent"], d["draft_depth"], np.array([1], np.uint64), 3, seq_tok,
                 seq_len, np.array([max_new], np.int32), eos_id=eos)
    return r, seq_tok, seq_len


def test_walk_forced_tree(orc):
    """Draft tree: 0:a(root child) 1:b(root child) 2:c(under 0) 3:d(under 0) 4:e(under 3).
    Tokens a=1,b=2,c=3,d=4,e=5.  Forced samples per row [root,0,1,2,3,4]."""
    d = _draft_arrays(8, [1, 2, 3, 4, 5], [-1, -1, 0, 0, 3], [1, 1, 2, 2, 3])
    # rows are [root, n0, n1, n2, n3, n4]; root samples 1 (= node 0), node 0
    # samples 7 (no draft child 7): stop, 7 is the bonus
    r, st, sl = _run_forced(orc, d, [1, 7, 7, 7, 4, 9])
    assert r["accept_len"][0] == 1 and list(r["commit_tok"][0, :2]) == [1, 7]
    r, st, sl = _run_forced(orc, d, [1, 4, 7, 7, 5, 9])
    # root->a(node0); node0 samples 4=d(node3); node3 samples 5=e(node4); node4 samples 9 -> bonus
    assert r["accept_len"][0] == 3
    assert list(r["accepted_nodes"][0, :3]) == [0, 3, 4]
    assert list(r["commit_tok"][0, :4]) == [1, 4, 5, 9]
    assert r["n_commit"][0] == 4 and sl[0] == 9 and list(st[0, 5:9]) == [1, 4, 5, 9]
    # immediate mismatch at the root: only the bonus token
    r, st, sl = _run_forced(orc, d, [6, 4, 7, 7, 5, 9])
    assert r["accept_len"][0] == 0 and r["n_commit"][0] == 1 and r["commit_tok"][0, 0] == 6
    # sampled[] holds the forced token of every row
    assert list(r["sampled"]) == [6, 4, 7, 7, 5, 9]


def test_truncation_eos_and_length(orc):
    d = _draft_arrays(8, [1, 4, 5], [-1, 0, 1], [1, 2, 3])
    # full acceptance would commit [1,4,5,9]
    r, st, sl = _run_forced(orc, d, [1, 4, 5, 9], eos=4)
    assert r["n_commit"][0] == 2 and list(r["commit_tok"][0, :2]) == [1, 4] and r["finished"][0]
    assert r["accept_len"][0] == 3  # the walk result itself is not truncated
    r, st, sl = _run_forced(orc, d, [1, 4, 5, 9], max_new=7, t=5)
    assert r["n_commit"][0] == 2 and sl[0] == 7 and r["finished"][0]
    r, st, sl = _run_forced(orc, d, [1, 4, 5, 9], max_new=5, t=5)
    assert r["n_commit"][0] == 0 and sl[0] == 5 and r["finished"][0]
    r, st, sl = _run_forced(orc, d, [1, 4, 5, 9], max_new=100)
    assert r["n_commit"][0] == 4 and not r["finished"][0]


@pytest.mark.parametrize("seed", range(10))
def test_acceptance_is_a_prefix(orc, seed):
    """P11 on random drafts and random logits."""
    rng = np.random.default_rng(seed)
    V, B, n_seq = 6, 12, 8
    o = orc.Oracle(V, 1, 16, 4, B)
    for _ in range(4):
        o.insert_sequence(0, rng.integers(0, V, 40).astype(np.int32))
    seq_tok = rng.integers(0, V, (n_seq, 80)).astype(np.int32)
    seq_len = rng.integers(1, 30, n_seq).astype(np.int32)
    d = o.draft(np.zeros(n_seq, np.int32), seq_tok, seq_len, pos_base=seq_len)
    rows = int(d["row_offsets"][-1])
    logits = rng.normal(0, 0.5, (rows, V)).astype(np.float32)
    t0 = seq_len.copy()
    r = o.verify(logits, d["row_offsets"], d["draft_len"], d["draft_tok"], d["draft_parent"],
                 d["draft_depth"], np.arange(n_seq, dtype=np.uint64), seed, seq_tok, seq_len,
                 np.full(n_seq, 1000, np.int32))
    for s in range(n_seq):
        a = r["accept_len"][s]
        assert a <= d["draft_len"][s]
        path = list(r["accepted_nodes"][s, :a])
        prev = -1
        for k, node in enumerate(path):
            assert d["draft_parent"][s, node] == prev
            assert d["draft_tok"][s, node] == r["sampled"][d["row_offsets"][s] + 1 + prev]
            prev = node
        rows_on_path = [-1] + path
        for k in range(a + 1):
            assert r["commit_tok"][s, k] == r["sampled"][d["row_offsets"][s] + 1 + rows_on_path[k]]
        assert seq_len[s] == t0[s] + a + 1
