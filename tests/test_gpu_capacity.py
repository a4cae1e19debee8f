"""GPU parity of capacity management and persistence (DESIGN.md
O17): srt_cache_prune / reset / evict and srt_cache_load against the oracle's
prune and load, bit-exact on canonical dumps, and the trees stay fully usable
afterwards (tombstones, compacted child lists, invalidated cursors): further
inserts (walk and cursor paths) and drafts keep matching the oracle."""
import numpy as np
import pytest

from harness import Pair

pytestmark = pytest.mark.gpu


def _seqs(rng, n, V, lo=20, hi=160):
    base = rng.integers(0, V, 400).astype(np.int32)
    out = []
    for _ in range(n):  # siblings share a template (fan-out at the forks)
        t = base[: int(rng.integers(lo, hi))].copy()
        forks = rng.random(len(t)) < 0.08
        t[forks] = rng.integers(0, V, int(forks.sum()))
        out.append(t)
    return out


def _table(seqs, width):
    tab = np.zeros((len(seqs), width), np.int32)
    for i, t in enumerate(seqs):
        tab[i, :len(t)] = t
    return tab


def _fill(pair, rng, P, V, per=6, width=256):
    seqs, prompts = [], []
    for p in range(P):
        for t in _seqs(rng, per, V):
            seqs.append(t)
            prompts.append(p)
    tab = _table(seqs, width)
    pair.insert(np.array(prompts, np.int32), tab, np.zeros(len(seqs), np.int32),
                np.array([len(t) for t in seqs], np.int32))
    return tab, np.array(prompts, np.int32), np.array([len(t) for t in seqs], np.int32)


def _continue(pair, rng, tab, prompts, lens, V, steps=4, cursor=None):
    """More tokens on every sequence (cursor or walk insert), then drafts."""
    import torch
    for _ in range(steps):
        t0 = lens.copy()
        add = rng.integers(1, 6, len(lens))
        for i in range(len(lens)):
            e = min(tab.shape[1], lens[i] + add[i])
            tab[i, lens[i]:e] = rng.integers(0, V, e - lens[i])
            lens[i] = e
        pair.insert(prompts, tab, t0, lens, cursor=cursor)
        pair.compare_trees()
        od, gd = pair.draft(prompts, tab, lens, pos_base=lens)
        pair.compare_drafts(od, gd)
    torch.cuda.synchronize()


@pytest.mark.parametrize("theta", [2, 3, 6])
def test_prune_parity_then_keep_working(orc, theta):
    import torch
    rng = np.random.default_rng(theta)
    P, V = 3, 40
    pair = Pair(orc, V, P, 12, 6, 16, node_capacity=1 << 16)
    tab, prompts, lens = _fill(pair, rng, P, V)
    pair.compare_trees()
    cur = pair.gpu.new_cursors(len(lens), "cuda")
    pair.insert(prompts, tab, lens, lens, cursor=cur)  # (empty spans: cursors untouched)
    for p in (1, -1):
        n_o = pair.orc.prune(p, theta)
        n_g = pair.gpu.prune(p, theta)
        assert n_g == n_o and n_o > 0
        pair.compare_trees()
        st = pair.gpu.status()
        assert st[0] == 0
    _continue(pair, rng, tab, prompts, lens, V, cursor=cur)
    _continue(pair, rng, tab, prompts, lens, V, cursor=None)


def test_reset_and_refill(orc):
    rng = np.random.default_rng(5)
    P, V = 3, 30
    pair = Pair(orc, V, P, 10, 6, 16, node_capacity=1 << 16)
    tab, prompts, lens = _fill(pair, rng, P, V)
    nodes_before = pair.gpu.status()[1]["nodes_used"]
    removed = pair.gpu.reset(1)
    pair.orc.prune(1, 1 << 40)
    assert pair.gpu.dump(1) == [(-1, 0, 0)]
    pair.compare_trees()
    assert pair.gpu.status()[1]["nodes_used"] == nodes_before - removed
    # the same rollouts again: prompt 1's tree is rebuilt exactly
    sel = prompts == 1
    pair.insert(prompts[sel], tab[sel], np.zeros(int(sel.sum()), np.int32), lens[sel])
    pair.compare_trees()
    _continue(pair, rng, tab, prompts, lens, V)


def test_evict_hysteresis(orc):
    rng = np.random.default_rng(9)
    P, V = 4, 50
    pair = Pair(orc, V, P, 12, 6, 16, node_capacity=1 << 16)
    tab, prompts, lens = _fill(pair, rng, P, V)
    live = pair.gpu.status()[1]["nodes_used"] - P
    assert pair.gpu.evict(live + 10) == (0, 0)  # under capacity: nothing
    cap = live // 2
    removed, theta = pair.gpu.evict(cap)
    assert theta >= 2 and removed > 0
    assert pair.orc.prune(-1, theta) == removed
    pair.compare_trees()
    assert pair.gpu.status()[1]["nodes_used"] - P <= 0.9 * cap
    # theta is the smallest such threshold: theta - 1 would keep too many
    o2 = orc.Oracle(V, P, 12, 6, 16)
    o2.insert(prompts, tab, np.zeros(len(lens), np.int32), lens)
    o2.prune(-1, theta - 1)
    assert o2.node_count > 0.9 * cap
    _continue(pair, rng, tab, prompts, lens, V)


def test_load_restores_exactly(orc):
    import paper_2601_09083_b200 as srt
    rng = np.random.default_rng(13)
    P, V = 2, 60
    pair = Pair(orc, V, P, 12, 6, 16, node_capacity=1 << 16)
    tab, prompts, lens = _fill(pair, rng, P, V, per=8)
    pair.gpu.prune(0, 2)
    pair.orc.prune(0, 2)
    dumps = [pair.gpu.dump(p) for p in range(P)]
    # a new cache (another process / training step) restored from the dumps
    fresh = Pair(orc, V, P, 12, 6, 16, node_capacity=1 << 16)
    for p in range(P):
        fresh.gpu.load(p, dumps[p])
        fresh.orc.load(p, [(t, c, n) for (t, c, n) in dumps[p]])
        assert fresh.gpu.dump(p) == dumps[p]
    fresh.compare_trees()
    # merge semantics: loading again doubles every count
    fresh.gpu.load(1, dumps[1])
    fresh.orc.load(1, [(t, c, n) for (t, c, n) in dumps[1]])
    assert fresh.gpu.dump(1) == [(t, 2 * c, n) for (t, c, n) in dumps[1]]
    fresh.compare_trees()
    # the restored cache drafts like the original (same trees)
    od, gd = pair.draft(prompts, tab, lens, pos_base=lens)
    fresh.gpu.reset(1)
    fresh.orc.prune(1, 1 << 40)
    fresh.gpu.load(1, dumps[1])
    fresh.orc.load(1, [(t, c, n) for (t, c, n) in dumps[1]])
    od2, gd2 = fresh.draft(prompts, tab, lens, pos_base=lens)
    Pair.compare_drafts(od2, gd2)
    Pair.compare_drafts(od, gd2)
    with pytest.raises(srt.SrtError):
        fresh.gpu.load(0, [(5, 1, 0)])
