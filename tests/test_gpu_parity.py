"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by
element, on the same seeded inputs.  Integer / token / tree outputs must be
bit-exact; sampled tokens too (identical Philox keys and IEEE arithmetic,
BJ:north_star), with the number of rows whose GPU sample differs = 0."""
import numpy as np
import pytest

from harness import Pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2601_09083_b200 import build
    build.build()


def test_noise_table_bitwise(orc):
    """P9: the whole 2^23-point noise domain, GPU == oracle bit for bit."""
    import paper_2601_09083_b200 as srt
    g = srt.noise_table().cpu().numpy()
    o = orc.noise_table()
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def _spans(rng, P, V, n_seq, max_len, chunks=4):
    seqs = []
    for s in range(n_seq):
        p = int(rng.integers(0, P))
        n = int(rng.integers(1, max_len + 1))
        toks = rng.integers(0, V, n).astype(np.int32)
        cuts = sorted(set([0, n] + list(rng.integers(0, n + 1, int(rng.integers(0, chunks))))))
        seqs.append((p, toks, [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]))
    return seqs


def _insert_all(pair, seqs):
    maxlen = max(len(t) for _, t, _ in seqs)
    table = np.zeros((len(seqs), maxlen), np.int32)
    for i, (_, t, _) in enumerate(seqs):
        table[i, :len(t)] = t
    k = 0
    while True:
        idx = [i for i, s in enumerate(seqs) if k < len(s[2])]
        if not idx:
            break
        pair.insert([seqs[i][0] for i in idx], table[idx], [seqs[i][2][k][0] for i in idx],
                    [seqs[i][2][k][1] for i in idx])
        k += 1
    return table


@pytest.mark.parametrize("seed", range(12))
def test_insert_parity(orc, seed):
    rng = np.random.default_rng(seed)
    V = [3, 5, 50, 1000][seed % 4]
    D = int(rng.integers(1, 12))
    P = 3
    pair = Pair(orc, V, P, D, min(D, 4), 8)
    # many sibling spans of the same prompt in one call: concurrent creation
    _insert_all(pair, _spans(rng, P, V, 40, 60))
    pair.compare_trees()
    bits, st = pair.gpu.status()
    assert bits == 0
    assert st["nodes_used"] == P + pair.orc.node_count


@pytest.mark.parametrize("seed", range(6))
def test_insert_cursor_parity(orc, seed):
    """srt_insert_cursor builds the same tree as the oracle (and the same stats
    as srt_insert) over many lockstep steps, including spans longer than D (walk
    path), skipped positions, floors that change, records handed to another
    prompt, garbage records and D > 32 (several lane groups)."""
    import torch
    import paper_2601_09083_b200 as srt
    rng = np.random.default_rng(300 + seed)
    V = [4, 30, 500][seed % 3]
    D = [1, 3, 8, 16, 40, 70][seed]
    P, n, T = 3, 24, 260
    pair = Pair(orc, V, P, D, min(D, 4), 8, node_capacity=1 << 18)
    plain = srt.SrtCache(srt.config(V, P, D, min(D, 4), 8, node_capacity=1 << 18))
    toks = rng.integers(0, V, (n, T)).astype(np.int32)
    tk = torch.from_numpy(toks).cuda()
    prompt = rng.integers(0, P, n).astype(np.int32)
    floor = np.where(rng.random(n) < 0.3, rng.integers(0, 6, n), 0).astype(np.int32)
    cur = pair.gpu.new_cursors(n)
    pos = np.zeros(n, np.int32)
    st_c = torch.zeros(3, dtype=torch.int64, device="cuda")
    st_p = torch.zeros(3, dtype=torch.int64, device="cuda")
    for step in range(40):
        grow = rng.choice([0, 1, 1, 2, 3, 5], n)
        if step % 9 == 4:
            grow[rng.integers(0, n)] = D + 1 + int(rng.integers(0, 5))  # long span: walk path
        frm = pos.copy()
        if step % 7 == 3:
            k = rng.integers(0, n)
            frm[k] = min(pos[k] + 2, T)  # skipped positions: the record no longer matches
        if step % 11 == 5:
            k = rng.integers(0, n)
            prompt[k] = (prompt[k] + 1) % P  # record handed to another prompt
        if step % 13 == 6:
            k = rng.integers(0, n)
            floor[k] = min(frm[k], floor[k] + 3)
        if step % 17 == 8:
            cur[rng.integers(0, n)] = torch.randint(-2**31, 2**31 - 1, (D + 4,), dtype=torch.int32)
        to = np.minimum(frm + grow, T).astype(np.int32)
        pair.insert(prompt, toks, frm, to, floor, cursor=cur, stats=st_c)
        plain.insert(torch.from_numpy(prompt).cuda(), tk, torch.from_numpy(frm).cuda(),
                     torch.from_numpy(to).cuda(), torch.from_numpy(floor).cuda(), stats=st_p)
        pos = np.maximum(pos, to)
    pair.compare_trees()
    bits, _ = pair.gpu.status()
    assert bits == 0
    assert st_c.tolist() == st_p.tolist()
    for p in range(P):
        assert plain.dump(p) == pair.gpu.dump(p)


@pytest.mark.parametrize("D,V", [(64, 8), (128, 8), (128, 3)])
def test_insert_cursor_deep_siblings_midspan_flush(orc, D, V):
    """D > 32 (one CTA of D/32 warps per sequence) with many sibling
    sequences of the same prompts inserting spans of ~D new positions at once:
    each warp creates up to 32 nodes per position, so its log passes the
    mid-span flush threshold after ~12 positions, while siblings on other CTAs
    wait for each other's node publications (the flush decision is
    block-wide).  Trees equal the oracle's; the call terminates."""
    rng = np.random.default_rng(D + V)
    P, n, T = 2, 64, 4 * D
    # nearly every window of length > log_V(n T) is a new node: up to n T D
    pair = Pair(orc, V, P, D, 8, 8, node_capacity=1 << 20 if D <= 64 else 1 << 23)
    base = rng.integers(0, V, (P, T)).astype(np.int32)
    prompt = (np.arange(n) % P).astype(np.int32)
    # siblings share their prompt's template with 30% substitutions: nodes
    # created by one CTA are met (pending) by others in the same call
    toks = np.where(rng.random((n, T)) < 0.3, rng.integers(0, V, (n, T)), base[prompt]).astype(np.int32)
    cur = pair.gpu.new_cursors(n)
    pos = np.zeros(n, np.int32)
    for step in range(4):
        grow = rng.integers(D - 8, D + 1, n)  # <= D: the cursor path
        to = np.minimum(pos + grow, T).astype(np.int32)
        pair.insert(prompt, toks, pos, to, cursor=cur)
        pos = to
        pair.compare_trees()
    bits, _ = pair.gpu.status()
    assert bits == 0


def test_insert_repeat_is_deterministic(orc):
    """Concurrent CAS/atomics: the logical tree is identical across runs."""
    rng = np.random.default_rng(5)
    seqs = _spans(rng, 1, 4, 64, 80)
    dumps = []
    for _ in range(3):
        pair = Pair(orc, 4, 1, 10, 4, 8)
        _insert_all(pair, seqs)
        dumps.append(pair.gpu.dump(0))
    assert dumps[0] == dumps[1] == dumps[2]


def test_insert_long_spans_and_floor(orc):
    """Run-ahead style long spans (2k tokens) and a non-zero floor."""
    rng = np.random.default_rng(9)
    V, D = 64, 16
    pair = Pair(orc, V, 2, D, 8, 16, node_capacity=1 << 18)
    toks = rng.integers(0, V, (4, 2048)).astype(np.int32)
    pair.insert([0, 1, 0, 1], toks, [0, 0, 100, 5], [2048, 1500, 2048, 2000], [0, 0, 100, 5])
    pair.compare_trees()


@pytest.mark.parametrize("seed", range(10))
def test_draft_parity(orc, seed):
    rng = np.random.default_rng(100 + seed)
    V = [4, 8, 300][seed % 3]
    D = int(rng.integers(3, 14))
    L = int(rng.integers(1, min(D, 8) + 1))
    Bmax = [1, 5, 8, 32, 64][seed % 5]
    b0, num, den = [(Bmax, 0, 1), (1, 1, 1), (2, 3, 2)][seed % 3]
    b0 = min(b0, Bmax)
    ms = [0.0, 0.0, 0.01][seed % 3]
    pair = Pair(orc, V, 2, D, L, Bmax, b0=b0, num=num, den=den, min_score=ms)
    # a repetitive corpus so drafts are deep and bushy
    base = rng.integers(0, V, 40).astype(np.int32)
    seqs = []
    for k in range(30):
        s = np.where(rng.random(40) < 0.15, rng.integers(0, V, 40), base).astype(np.int32)
        seqs.append((k % 2, s, [(0, 40)]))
    _insert_all(pair, seqs)
    n = 64
    ctx = np.stack([base if i % 3 else rng.integers(0, V, 40).astype(np.int32) for i in range(n)])
    seq_len = rng.integers(0, 41, n).astype(np.int32)
    od, gd = pair.draft(rng.integers(0, 2, n).astype(np.int32), ctx, seq_len,
                        pos_base=seq_len + 7)
    pair.compare_drafts(od, gd)
    assert od["draft_len"].sum() > 0


@pytest.mark.parametrize("Bmax", [7, 32, 64])
def test_draft_parity_hubs(orc, Bmax):
    """Hub nodes with thousands of children (several 256-child enumeration
    rounds), Zipf counts with many ties (resolved by token, O8), and both the
    register top-K path (budget <= 32) and the serial path (> 32)."""
    from synth import zipf_tokens
    rng = np.random.default_rng(7000 + Bmax)
    V, D, L = 6000, 6, 3
    pair = Pair(orc, V, 2, D, L, Bmax, node_capacity=1 << 20)
    perm = rng.permutation(V).astype(np.int32)
    seqs = [(k % 2, zipf_tokens(rng, 400, V, perm, s=1.05), [(0, 400)]) for k in range(60)]
    _insert_all(pair, seqs)
    n = 96
    ctx = zipf_tokens(rng, n * 20, V, perm, s=1.05).reshape(n, 20)
    seq_len = rng.integers(1, 21, n).astype(np.int32)
    od, gd = pair.draft(rng.integers(0, 2, n).astype(np.int32), ctx, seq_len)
    pair.compare_drafts(od, gd)
    assert od["draft_len"].sum() > n


@pytest.mark.parametrize("Bmax", [32, 64])
def test_draft_parity_hub_lists_across_inserts(orc, Bmax):
    """Hub child lists over alternating drafts and inserts: lists built after
    the bulk insert, lists gone stale (an insert changed the hub's csum) and
    rebuilt, hubs first met by a draft without a list (logged, built after
    the next insert), and frontier merges of listed children (Bmax 64: two
    32-entry chunks into a 64-entry frontier).  Drafts equal the oracle's at
    every step."""
    from synth import zipf_tokens
    rng = np.random.default_rng(7100 + Bmax)
    V, D, L = 3000, 5, 3
    pair = Pair(orc, V, 2, D, L, Bmax, node_capacity=1 << 20)
    perm = rng.permutation(V).astype(np.int32)
    seqs = [(k % 2, zipf_tokens(rng, 300, V, perm, s=1.1), [(0, 300)]) for k in range(40)]
    _insert_all(pair, seqs)
    n = 64
    for step in range(5):
        ctx = zipf_tokens(rng, n * 16, V, perm, s=1.1).reshape(n, 16)
        seq_len = rng.integers(1, 17, n).astype(np.int32)
        prompts = rng.integers(0, 2, n).astype(np.int32)
        od, gd = pair.draft(prompts, ctx, seq_len)
        pair.compare_drafts(od, gd)
        assert od["draft_len"].sum() > n
        # a few more rollouts: shallow hubs change csum (their lists go stale)
        more = [(k % 2, zipf_tokens(rng, 40, V, perm, s=1.1), [(0, 40)]) for k in range(6)]
        _insert_all(pair, more)
    pair.compare_trees()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("seed", range(4))
def test_verify_parity_random(orc, dtype, seed):
    """Random drafts from real trees, logits with the rl-mix head profile,
    temperature 1 and != 1, EOS and length caps."""
    from synth import random_logits_np
    rng = np.random.default_rng(200 + seed)
    V = [1000, 4096, 151936, 1003 if dtype == "f32" else 1001][seed]
    D, L, Bmax = 12, 4, 16
    pair = Pair(orc, V, 2, D, L, Bmax, dtype=dtype)
    base = rng.integers(0, min(V, 50), 60).astype(np.int32)
    seqs = [(k % 2, np.where(rng.random(60) < 0.1, rng.integers(0, min(V, 50), 60), base).astype(np.int32),
             [(0, 60)]) for k in range(12)]
    _insert_all(pair, seqs)
    n = 24 if V > 100000 else 48
    ctx = np.zeros((n, 60 + Bmax + 2), np.int32)
    ctx[:, :60] = base
    seq_len = rng.integers(1, 50, n).astype(np.int32)
    od, gd = pair.draft(rng.integers(0, 2, n).astype(np.int32), ctx, seq_len)
    pair.compare_drafts(od, gd)
    rows = int(od["row_offsets"][-1])
    logits = random_logits_np(rng, rows, V)
    T = [1.0, 0.7, 1.0, 1.3][seed]
    eos = [-1, 3, int(base[5]), -1][seed]
    max_new = rng.integers(10, 60, n).astype(np.int32)
    sid = rng.integers(0, 2 ** 62, n).astype(np.uint64)
    ov, gv, o_seq, g_seq, dev = pair.verify(logits, od, gd, sid, 0xC0FFEE + seed, ctx, seq_len,
                                            max_new, temperature=T, eos=eos)
    pair.compare_verify(ov, gv, o_seq, g_seq)
    # the pruned product scan and the unpruned reference scan agree bitwise
    import torch
    ref = pair.gpu.sample_rows_reference(dev, gd, pair.t(seq_len), pair.t(sid.view(np.int64)),
                                         0xC0FFEE + seed, temperature=T)
    assert torch.equal(ref[:rows].cpu(), gv.sampled[:rows].cpu())


@pytest.mark.parametrize("profile", ["peaked", "moderate", "flat"])
def test_verify_profiles(orc, profile):
    """Every logits profile (prune rate from ~100% to 0%) gives the oracle's tokens."""
    from synth import random_logits_np
    rng = np.random.default_rng(7)
    V = 151936
    pair = Pair(orc, V, 1, 8, 4, 8)
    n = 16
    ctx = np.zeros((n, 32), np.int32)
    seq_len = np.zeros(n, np.int32)
    od, gd = pair.draft(np.zeros(n, np.int32), ctx, seq_len)
    logits = random_logits_np(rng, n, V, profile=profile)
    ov, gv, o_seq, g_seq, _ = pair.verify(logits, od, gd, np.arange(n, dtype=np.uint64), 42, ctx,
                                          seq_len, np.full(n, 100, np.int32))
    pair.compare_verify(ov, gv, o_seq, g_seq)


def test_verify_special_rows(orc):
    """All -inf rows, +inf ties, NaN (flagged, never chosen), ties at the max."""
    V = 4096
    pair = Pair(orc, V, 1, 4, 2, 4, dtype="f32")
    n = 6
    ctx = np.zeros((n, 16), np.int32)
    seq_len = np.zeros(n, np.int32)
    od, gd = pair.draft(np.zeros(n, np.int32), ctx, seq_len)
    x = np.random.default_rng(1).normal(0, 1, (n, V)).astype(np.float32)
    x[0] = -np.inf
    x[1, [5, 900, 3000]] = np.inf
    x[2, 17] = np.nan
    x[2, 4000] = 30.0
    x[3, :] = 0.0                       # every element ties in x: noise decides
    x[4, [10, 20]] = 40.0               # two equal maxima far above the bulk
    x[5, :] = -np.inf
    x[5, 3] = np.nan
    x[5, 4095] = -np.inf
    ov, gv, o_seq, g_seq, _ = pair.verify(x, od, gd, np.arange(n, dtype=np.uint64), 9, ctx,
                                          seq_len, np.full(n, 100, np.int32))
    pair.compare_verify(ov, gv, o_seq, g_seq)
    assert ov["nan_seen"]
    bits, _ = pair.gpu.status()
    assert bits & 8  # SRT_DEV_NONFINITE_LOGIT
    assert gv.sampled[0].item() == 0 and gv.sampled[1].item() == 5


def test_error_flags(orc):
    import torch
    pair = Pair(orc, 50, 2, 4, 2, 4)
    toks = np.array([[1, 2, 60, 3]], np.int32)  # 60 is out of vocabulary
    pair.insert([0], toks, [0], [4])
    pair.compare_trees()  # both sides stop the window at the OOV token
    bits, _ = pair.gpu.status()
    assert bits & 1
    pair.gpu.clear_errors()
    assert pair.gpu.status()[0] == 0
    pair.gpu.insert(pair.t(np.array([5], np.int32)), pair.t(toks), pair.t(np.array([0], np.int32)),
                    pair.t(np.array([2], np.int32)))
    assert pair.gpu.status()[0] & 4  # bad prompt id


def test_capacity_overflow_is_sticky(orc):
    import paper_2601_09083_b200 as srt
    import torch
    cfg = srt.config(100, 1, 8, 4, 8, node_capacity=64)
    c = srt.SrtCache(cfg)
    toks = torch.arange(100, dtype=torch.int32, device="cuda").remainder(97).reshape(1, 100)
    z = torch.zeros(1, dtype=torch.int32, device="cuda")
    c.insert(z, toks, z, torch.full((1,), 100, dtype=torch.int32, device="cuda"))
    bits, st = c.status()
    assert bits & 2 and st["nodes_used"] == 64
    with pytest.raises(srt.SrtError):
        c.dump(0)


def test_empty_batches(orc):
    import torch
    pair = Pair(orc, 100, 1, 4, 2, 4)
    e = torch.zeros(0, dtype=torch.int32, device="cuda")
    pair.gpu.insert(e, torch.zeros(0, 4, dtype=torch.int32, device="cuda"), e, e)
    d = pair.gpu.draft(e, torch.zeros(0, 4, dtype=torch.int32, device="cuda"), e)
    assert d.row_offsets.cpu().tolist() == [0]
    assert pair.gpu.status()[0] == 0


def test_tiny_config_lockstep(orc):
    """BJ:configs[0] end to end: 1 prompt, 8 cached rollouts x 64 tokens,
    V = 1000, 4 active sequences, Bmax = 8.  Draft -> verify -> insert every
    step on both sides; every output and the tree compared at every step."""
    from synth import make_workload, random_logits_np
    w = make_workload(seed=0, V=1000, n_prompts=1, samples=8, median=64, cap=64, active=4)
    pair = Pair(orc, 1000, 1, 16, 8, 8)
    prior = np.zeros((8, 64), np.int32)
    lens = []
    for i, (p, t) in enumerate(w.prior):
        prior[i, :len(t)] = t
        lens.append(len(t))
    pair.insert([0] * 8, prior, [0] * 8, lens)
    pair.compare_trees()
    n, cap = 4, 256
    rng = np.random.default_rng(1)
    seq_tok = np.zeros((n, cap + 16), np.int32)
    seq_len = np.zeros(n, np.int32)
    max_new = np.full(n, cap, np.int32)
    total_acc = 0
    for step in range(40):
        t0 = seq_len.copy()
        od, gd = pair.draft(np.zeros(n, np.int32), seq_tok, seq_len, pos_base=seq_len)
        pair.compare_drafts(od, gd)
        rows = int(od["row_offsets"][-1])
        # forward stand-in: head = ground-truth next token of each row's context
        heads = np.empty(rows, np.int64)
        for s in range(n):
            r0 = od["row_offsets"][s]
            truth = w.truth[s]
            heads[r0] = truth[min(t0[s], len(truth) - 1)]
            for i in range(od["draft_len"][s]):
                d = od["draft_depth"][s, i]
                heads[r0 + 1 + i] = truth[min(t0[s] + d, len(truth) - 1)]
        logits = random_logits_np(rng, rows, 1000, heads=heads)
        ov, gv, o_seq, g_seq, _ = pair.verify(logits, od, gd, w.seq_id, 1234 + step, seq_tok,
                                              seq_len, max_new)
        pair.compare_verify(ov, gv, o_seq, g_seq)
        seq_tok, seq_len = o_seq
        total_acc += int(ov["accept_len"].sum())
        pair.insert(np.zeros(n, np.int32), seq_tok, t0, seq_len)
        pair.compare_trees()
    assert total_acc > 0
