"""Capacity management in the oracle (O17): prune by
count threshold (SPEC's lowest-count-subtree eviction) and the
dump/load round trip (persistence).  Pinned against independent
definitions written here: a filter over the canonical preorder dump, brute-force
substring counts, and the paper's Fig. 3 tree."""
import numpy as np
import pytest

from synth import fig3_sentences


def _tree(orc, seqs, D=6, V=8):
    o = orc.Oracle(V, 1, D, min(D, 4), 8)
    for t in seqs:
        o.insert_sequence(0, t)
    return o


def _filter_dump(records, theta):
    """Expected dump after removing every non-root node with count < theta:
    drop such a record with its whole subtree (preorder + child counts), reduce
    its parent's child count, recompute the root count."""
    out, removed = [], 0

    def walk(k, parent):
        nonlocal removed
        tok, cnt, nch = records[k]
        if k > 0 and cnt < theta:
            nxt = _skip(records, k)
            removed += nxt - k
            return nxt
        out.append([tok, cnt, 0])
        me = len(out) - 1
        if parent is not None:
            out[parent][2] += 1
        k += 1
        for _ in range(nch):
            k = walk(k, me)
        return k

    walk(0, None)
    out[0][1] = sum(r[1] for r in _children_of_root(out))
    return [tuple(r) for r in out], removed


def _children_of_root(recs):
    res, k = [], 1
    for _ in range(recs[0][2]):
        res.append(recs[k])
        k = _skip(recs, k)
    return res


def _skip(recs, k):
    n = recs[k][2]
    k += 1
    for _ in range(n):
        k = _skip(recs, k)
    return k


def _dump(o):
    return [tuple(int(v) for v in r) for r in o.dump(0)]


@pytest.mark.parametrize("theta", [1, 2, 3, 5, 8, 1 << 40])
def test_prune_matches_dump_filter_random(orc, theta):
    rng = np.random.default_rng(theta % 1000)
    for trial in range(40):
        seqs = [rng.integers(0, 4, rng.integers(1, 14)).astype(np.int32) for _ in range(4)]
        o = _tree(orc, seqs)
        before = _dump(o)
        n_before = o.node_count
        want, removed = _filter_dump(before, theta)
        got_removed = o.prune(0, theta)
        assert got_removed == removed
        assert _dump(o) == want
        assert o.node_count == n_before - removed


def test_prune_keeps_exact_counts_bruteforce(orc):
    """After prune(theta) the tree is exactly the set of windowed substrings
    (depth <= D) whose occurrence count is >= theta, with those counts."""
    rng = np.random.default_rng(7)
    D = 5
    for trial in range(30):
        seqs = [rng.integers(0, 3, rng.integers(2, 12)).astype(np.int32) for _ in range(3)]
        o = _tree(orc, seqs, D=D)
        theta = int(rng.integers(1, 5))
        o.prune(0, theta)
        counts = {}
        for t in seqs:
            t = list(t)
            for i in range(len(t)):
                for d in range(1, D + 1):
                    if i + d > len(t):
                        break
                    key = tuple(t[i:i + d])
                    counts[key] = counts.get(key, 0) + 1
        for key, cnt in counts.items():
            assert o.count_of(0, list(key)) == (cnt if cnt >= theta else 0), (key, cnt, theta)


def test_prune_fig3(orc):
    """'on the' -> mat:4, sofa:1; 'the cat' -> sit:5, eat:2.
    theta = 2 removes sofa (count 1) and keeps the rest; theta = 3 also drops
    the eat branch (count 2)."""
    s = fig3_sentences()
    o = orc.Oracle(16, 1, 8, 8, 8)
    for t in s:
        o.insert_sequence(0, t)
    the, cat, sit, on, mat, sofa, eat = (int(x) for x in
                                         (s[0][0], s[0][1], s[0][2], s[0][3], s[0][5],
                                          s[4][5], s[5][2]))
    assert o.count_of(0, [on, the, sofa]) == 1
    o.prune(0, 2)
    assert o.count_of(0, [on, the, sofa]) == 0
    assert o.count_of(0, [on, the, mat]) == 4
    assert o.count_of(0, [the, cat, eat]) == 2
    o.prune(0, 3)
    assert o.count_of(0, [the, cat, eat]) == 0
    assert o.count_of(0, [the, cat, sit]) == 5
    assert o.count_of(0, [the, cat]) == 7  # the parent keeps its own count (O1)


def test_load_round_trip_and_merge(orc):
    rng = np.random.default_rng(11)
    for trial in range(20):
        seqs = [rng.integers(0, 5, rng.integers(1, 16)).astype(np.int32) for _ in range(5)]
        a = _tree(orc, seqs)
        recs = _dump(a)
        b = _tree(orc, [])
        b.load(0, recs)
        assert _dump(b) == recs
        assert b.node_count == a.node_count
        b.load(0, recs)  # merge: every count doubles, same shape
        assert _dump(b) == [(t, 2 * c, n) for (t, c, n) in recs]


def test_load_rejects_malformed(orc):
    o = _tree(orc, [])
    with pytest.raises(ValueError):
        o.load(0, [(5, 1, 0)])  # no root record
    with pytest.raises(ValueError):
        o.load(0, [(-1, 1, 1), (3, 1, 0), (4, 1, 0)])  # more records than children
