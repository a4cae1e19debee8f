"""Pins for the oracle's tree, match and draft (O1-O9).

P1  the paper's Fig. 3 worked example (tests/golden/fig3.txt)
P2  SPEC's insert examples
P3  brute-force substring counting on tiny random inputs, incremental == batch
P4  brute-force longest qualifying suffix
P5  brute-force full sort of all descendants under the recursive total order
P6  layout invariants (masks, parents, positions)
"""
import os
from collections import Counter

import numpy as np
import pytest

from bruteforce import (canonical_from_counts, draft_bruteforce, longest_match, node_set,
                        substring_counts)
from synth import FIG3_VOCAB, fig3_sentences

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _mk(orc, V=8, P=1, D=8, L=8, B=16, **kw):
    return orc.Oracle(V, P, D, L, B, **kw)


def _fig3_tree(orc, B=16):
    o = _mk(orc, V=8, D=8, L=8, B=B)
    for s in fig3_sentences():
        o.insert_sequence(0, s)
    return o


def _words(ws):
    return [FIG3_VOCAB[w] for w in ws.split(",")]


def test_fig3_worked_example(orc):
    o = _fig3_tree(orc)
    for line in open(os.path.join(GOLD, "fig3.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        if f[0] == "count":
            assert o.count_of(0, _words(f[1])) == int(f[2]), line
        elif f[0] == "cond":
            parent = _words(f[1])
            child = parent + [FIG3_VOCAB[f[2]]]
            # C(v) from the tree's counts equals the figure's fraction
            kids = [o.count_of(0, parent + [t]) for t in range(8)]
            assert o.count_of(0, child) / sum(kids) == int(f[3]) / int(f[4])
        elif f[0] == "match":
            ctx = np.asarray(_words(f[1]), np.int32)[None, :]
            d = o.draft([0], ctx, [ctx.shape[1]])
            assert d["match_len"][0] == int(f[2])
        elif f[0] == "draft":
            ob = _fig3_tree(orc, B=int(f[1]))
            ctx = np.asarray(_words("the,cat"), np.int32)[None, :]
            d = ob.draft([0], ctx, [2])
            n = d["draft_len"][0]
            assert list(d["draft_tok"][0, :n]) == _words(f[2])
            # a chain: each node's parent is the previous one
            assert list(d["draft_parent"][0, :n]) == list(range(-1, n - 1))


def test_fig3_full_draft_order(orc):
    """Best-first order of every descendant of 'the cat' (O8) with fp64 path
    products evaluated in the O6 operation order from the figure's counts."""
    o = _fig3_tree(orc, B=16)
    ctx = np.asarray(_words("the,cat"), np.int32)[None, :]
    d = o.draft([0], ctx, [2])
    n = d["draft_len"][0]
    toks = [k for k, v in sorted(FIG3_VOCAB.items(), key=lambda kv: kv[1])]
    got = [toks[t] for t in d["draft_tok"][0, :n]]
    assert got == ["sit", "on", "the", "mat", "eat", "the", "fish", "sofa"]
    assert list(d["draft_parent"][0, :n]) == [-1, 0, 1, 2, -1, 4, 5, 2]
    assert list(d["draft_depth"][0, :n]) == [1, 2, 3, 4, 1, 2, 3, 4]
    # RN(RN(5/7) * RN(4/5)) is 4/7 + 1 ulp: the draft uses the O6 op order
    assert (5 / 7) * (4 / 5) != 4 / 7


def test_spec_insert_examples(orc):
    a, b = 0, 1
    o = _mk(orc, V=4, D=2, L=2, B=4)
    o.insert_sequence(0, [a, b])
    assert o.count_of(0, [a]) == 1 and o.count_of(0, [a, b]) == 1 and o.count_of(0, [b]) == 1
    assert o.node_count == 3
    o = _mk(orc, V=4, D=2, L=2, B=4)
    o.insert_sequence(0, [a, a, a, a])
    assert o.count_of(0, [a]) == 4 and o.count_of(0, [a, a]) == 3
    assert o.node_count == 2


def test_spec_create_validation(orc):
    with pytest.raises(ValueError):
        orc.Oracle(8, 1, 8, 9, 4)        # L > D
    with pytest.raises(ValueError):
        orc.Oracle(8, 1, 8, 8, 65)       # Bmax > 64 (one u64 mask word)
    with pytest.raises(ValueError):
        orc.Oracle(1, 1, 8, 8, 4)        # V < 2


def _random_spans(rng, n_prompts, V, n_seqs, max_len, max_chunks=4, floor_max=0):
    """Contiguous incremental spans per sequence (how rollouts grow)."""
    seqs = []
    for s in range(n_seqs):
        p = int(rng.integers(0, n_prompts))
        n = int(rng.integers(1, max_len + 1))
        toks = rng.integers(0, V, n).astype(np.int32)
        floor = int(rng.integers(0, min(floor_max, n - 1) + 1)) if floor_max else 0
        cuts = sorted(set([floor, n] + list(rng.integers(floor, n + 1, int(rng.integers(0, max_chunks))))))
        spans = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
        seqs.append((p, toks, floor, spans))
    return seqs


def _apply(o, seqs):
    """Insert every span, one call per 'step' with one span per sequence."""
    maxlen = max(len(t) for _, t, _, _ in seqs)
    table = np.zeros((len(seqs), maxlen), np.int32)
    for i, (_, t, _, _) in enumerate(seqs):
        table[i, :len(t)] = t
    k = 0
    while True:
        idx = [i for i, s in enumerate(seqs) if k < len(s[3])]
        if not idx:
            break
        o.insert([seqs[i][0] for i in idx], table[idx],
                 [seqs[i][3][k][0] for i in idx], [seqs[i][3][k][1] for i in idx],
                 [seqs[i][2] for i in idx])
        k += 1


@pytest.mark.parametrize("seed", range(40))
def test_insert_matches_bruteforce(orc, seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(2, 5))
    D = int(rng.integers(1, 6))
    P = 2
    seqs = _random_spans(rng, P, V, int(rng.integers(1, 5)), 12, floor_max=3 if seed % 2 else 0)
    o = orc.Oracle(V, P, D, min(D, 3), 8)
    _apply(o, seqs)
    spans = [(p, t.tolist(), a, b, fl) for p, t, fl, sp in seqs for a, b in sp]
    want = substring_counts(spans, D)
    for p in range(P):
        got = [tuple(r) for r in o.dump(p).tolist()]
        assert got == canonical_from_counts(want.get(p, Counter())), (seed, p)
    assert o.node_count == sum(len(node_set(c)) for c in want.values())
    assert o.error_bits == 0


def test_count_closed_forms(orc):
    """P3: sum of depth-d counts = number of inserted windows of length >= d."""
    rng = np.random.default_rng(7)
    V, D = 6, 5
    o = orc.Oracle(V, 1, D, 3, 8)
    seqs = [rng.integers(0, V, int(rng.integers(1, 30))).astype(np.int32) for _ in range(10)]
    for s in seqs:
        o.insert_sequence(0, s)
    dump = o.dump(0)
    # depth-d sums via an explicit preorder parser
    def parse(i, d, acc):
        tok, cnt, nch = dump[i]
        acc[d] += int(cnt)
        j = i + 1
        for _ in range(int(nch)):
            j = parse(j, d + 1, acc)
        return j
    acc = Counter()
    assert parse(0, 0, acc) == len(dump)
    for d in range(1, D + 1):
        want = sum(max(0, len(s) - d + 1) for s in seqs)
        assert acc[d] == want
    assert acc[0] == sum(len(s) for s in seqs)  # root record = # window starts


@pytest.mark.parametrize("seed", range(40))
def test_match_matches_bruteforce(orc, seed):
    rng = np.random.default_rng(100 + seed)
    V = int(rng.integers(2, 4))
    D = int(rng.integers(2, 6))
    L = int(rng.integers(1, D + 1))
    o = orc.Oracle(V, 1, D, L, 8)
    text = rng.integers(0, V, 20).astype(np.int32)
    o.insert_sequence(0, text)
    nodes = node_set(substring_counts([(0, text.tolist(), 0, len(text), 0)], D)[0])
    ctxs = [rng.integers(0, V, int(rng.integers(0, 8))).astype(np.int32) for _ in range(30)]
    tbl = np.zeros((len(ctxs), 8), np.int32)
    for i, c in enumerate(ctxs):
        tbl[i, :len(c)] = c
    d = o.draft(np.zeros(len(ctxs), np.int32), tbl, [len(c) for c in ctxs])
    for i, c in enumerate(ctxs):
        assert d["match_len"][i] == longest_match(nodes, c.tolist(), L), (seed, c)
        if d["match_len"][i] == 0:
            assert d["draft_len"][i] == 0 and d["row_offsets"][i + 1] - d["row_offsets"][i] == 1


@pytest.mark.parametrize("seed", range(60))
def test_draft_matches_bruteforce(orc, seed):
    """P5 on random trees with <= ~50 nodes (S:L556 scale)."""
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.integers(2, 4))
    D = int(rng.integers(3, 6))
    L = int(rng.integers(1, 3))
    Bmax = int(rng.integers(1, 12))
    min_score = [0.0, 0.0, 0.05, 0.3][seed % 4]
    o = orc.Oracle(V, 1, D, L, Bmax, min_path_score=min_score)
    texts = [rng.integers(0, V, int(rng.integers(3, 10))).astype(np.int32) for _ in range(3)]
    for t in texts:
        o.insert_sequence(0, t)
    cnt = substring_counts([(0, t.tolist(), 0, len(t), 0) for t in texts], D)[0]
    nodes = node_set(cnt)
    ctx = rng.integers(0, V, 6).astype(np.int32)
    d = o.draft([0], ctx[None, :], [6], pos_base=[100])
    q = d["match_len"][0]
    assert q == longest_match(nodes, ctx.tolist(), L)
    n = d["draft_len"][0]
    if q == 0:
        assert n == 0
        return
    uq = tuple(ctx[6 - q:].tolist())
    want = draft_bruteforce(cnt, uq, Bmax, min_score)
    assert n == len(want)
    # reconstruct each drafted node's full path from tokens + parents
    paths = []
    for i in range(n):
        par = d["draft_parent"][0, i]
        base = uq if par < 0 else paths[par]
        paths.append(base + (int(d["draft_tok"][0, i]),))
    assert paths == [w for w, _ in want], seed
    # P6 layout invariants
    for i in range(n):
        par = int(d["draft_parent"][0, i])
        assert par < i
        m = int(d["draft_mask"][0, i])
        pm = int(d["draft_mask"][0, par]) if par >= 0 else 0
        assert m == pm | (1 << i)
        assert bin(m).count("1") == d["draft_depth"][0, i] == len(paths[i]) - q
        assert d["draft_pos"][0, i] == 100 + d["draft_depth"][0, i]
    assert list(d["row_offsets"]) == [0, n + 1]
    # unused entries are padding
    assert np.all(d["draft_tok"][0, n:] == -1) and np.all(d["draft_mask"][0, n:] == 0)


def test_conditional_normalisation(orc):
    """sum over siblings of C = 1 within k ulps."""
    rng = np.random.default_rng(3)
    o = orc.Oracle(5, 1, 4, 2, 64)
    for _ in range(20):
        o.insert_sequence(0, rng.integers(0, 5, 15).astype(np.int32))
    for ctx in ([0], [1, 2], [3]):
        kids = [o.count_of(0, ctx + [t]) for t in range(5)]
        tot = sum(kids)
        if tot:
            cs = [k / tot for k in kids if k]
            assert abs(sum(cs) - 1.0) <= len(cs) * np.finfo(np.float64).eps


def test_budget_function(orc):
    """B(q) = min(Bmax, b0 + floor(q*num/den)) (O5; SPEC S:L112 defaults 4 + 2q, cap 32).
    A periodic text gives every u_q a unary subtree of exactly D - q nodes, so the
    draft length is min(B(q), D - q)."""
    D = 16
    chain = np.array([0, 1, 2] * 12, np.int32)
    for (b0, num, den, Bmax) in [(4, 2, 1, 32), (1, 1, 2, 8), (3, 0, 1, 5), (0, 3, 1, 64)]:
        o = orc.Oracle(3, 1, D, 8, Bmax, budget_base=b0, slope_num=num, slope_den=den)
        o.insert_sequence(0, chain)
        for q in range(1, 9):
            d = o.draft([0], chain[None, :], [q])
            assert d["match_len"][0] == q
            assert d["draft_len"][0] == min(Bmax, b0 + (q * num) // den, D - q)
