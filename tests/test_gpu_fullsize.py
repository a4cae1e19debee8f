"""Full-size parity: BASELINE.json's configurations at their full sizes, in the
launch configuration bench.py times (bench.GpuRun: the same caches, kernels,
workload recipe and forward stand-in), checked against the oracle on SAMPLED
outputs the oracle can compute one by one:

* the trees of sampled prompts — the oracle re-inserts each sampled prompt's
  whole history (prior-epoch rollouts + every active sequence's committed
  tokens) and its canonical dump must equal the GPU's (before and after a
  step's insert, which runs through srt_verify_insert_cursor: the fused
  accept + cursor-insert kernel bench.py times);
* the drafts of every sequence of the sampled prompts (match, tokens, parents,
  depths, positions, masks) from that tree;
* verify/commit of those sequences on the bench's own logits rows (sampled
  tokens of every row, accepted lengths, commits, sequence tables);
* randomly sampled rows of the whole batch: the oracle's full-V Gumbel-max
  (orc_sample_row) on the same row and key must equal sampled[row].

Everything is bit-exact (north_star).  The oracle runs on the host cores; the
samples are sized to keep each config to well under a minute of CPU work.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _history_tree(orc, wl, cfg, p, seq_tok, seq_len, gr):
    """Oracle cache (1 prompt) holding prompt p's whole inserted history:
    prior-epoch rollouts, run-ahead spans so far, active sequences."""
    o = orc.Oracle(cfg["V"], 1, cfg["D"], cfg["L"], cfg["Bmax"])
    prior = [tk for q, tk in wl.w.prior if q == p]
    if gr.ra is not None:
        done = gr.runahead_inserted()
        prior += [tk[:done[i]] for i, (q, tk) in enumerate(wl.w.runahead)
                  if q == p and done[i] > 0]
    if prior:
        m = max(len(t) for t in prior)
        tab = np.zeros((len(prior), m), np.int32)
        for i, t in enumerate(prior):
            tab[i, :len(t)] = t
        o.insert(np.zeros(len(prior), np.int32), tab, np.zeros(len(prior), np.int32),
                 np.array([len(t) for t in prior], np.int32))
    seqs = np.nonzero(wl.seq_prompt == p)[0]
    o.insert(np.zeros(len(seqs), np.int32), seq_tok[seqs], np.zeros(len(seqs), np.int32),
             seq_len[seqs])
    return o, seqs


def _dump_equal(cache, p, o):
    g = [tuple(r) for r in cache.dump(p)]
    want = [tuple(int(v) for v in r) for r in o.dump(0)]
    assert g == want, f"tree of prompt {p}: {len(g)} vs {len(want)} records"
    return len(g)


@pytest.mark.parametrize("config,steps,n_prompts,n_rows", [
    ("grpo", 3, 2, 48),
    ("ppo", 3, 4, 32),
    ("dapo", 3, 2, 32),
])
def test_fullsize_sampled_parity(orc, config, steps, n_prompts, n_rows):
    import torch
    import bench

    cfg = bench.CONFIGS[config]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    gr = run.groups[0]
    # the launch configuration: every D <= 128 here runs the fused tree step
    # (srt_verify_insert_draft_cursor: commit + insert + refresh + next draft)
    gr.fused_step = cfg["D"] <= 128
    for k in range(steps):
        run.step(bench.step_seed(0, k))
    torch.cuda.synchronize()
    assert run.status()[0] == 0

    rng = np.random.default_rng(17)
    # prompts of the active sequences (+ one look-ahead prompt with run-ahead spans)
    active_prompts = np.unique(wl.seq_prompt)
    prompts = list(rng.choice(active_prompts, size=n_prompts, replace=False))
    if gr.ra is not None:
        prompts.append(cfg["runahead"]["first"] + 3)
    seq_tok = gr.seq_tok.cpu().numpy()
    seq_len = gr.seq_len.cpu().numpy()

    # ---- the step under test: draft -> stand-in -> fused verify + insert -----
    # (gr.verify_insert = srt_verify_insert_draft_cursor for D <= 32, else
    # srt_verify_insert_cursor -- the kernels bench.py times -- plus DAPO's
    # run-ahead spans; with the fused step this draft is the previous call's)
    gr.draft_if_needed()
    gr.standin()
    seed = bench.step_seed(0, steps)
    torch.cuda.synchronize()
    d = gr.d
    g_draft = {k: getattr(d, k).cpu().numpy() for k in
               ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth", "draft_pos")}
    g_draft["draft_mask"] = d.draft_mask.cpu().numpy().view(np.uint64)
    row_off = d.row_offsets.cpu().numpy()
    logits = gr.logits  # bf16 [rows_max + 1, V]
    seq_id = wl.seq_id
    max_new = wl.max_new

    # trees before the step's insert, and the drafts drawn from them
    drafted = 0
    trees = []
    for p in prompts:
        o, seqs = _history_tree(orc, wl, cfg, int(p), seq_tok, seq_len, gr)
        _dump_equal(gr.cache, int(p), o)
        if len(seqs):
            od = o.draft(np.zeros(len(seqs), np.int32), seq_tok[seqs], seq_len[seqs],
                         seq_len[seqs])
            for k, v in g_draft.items():
                assert np.array_equal(v[seqs], od[k].astype(v.dtype)), (config, p, k)
            drafted += int(od["draft_len"].sum())
        else:  # a look-ahead prompt: only run-ahead spans reach its tree
            od = None
        trees.append((int(p), o, seqs, od))
    assert drafted > 0, "the sampled prompts drafted nothing: the check is vacuous"

    ra_before = gr.runahead_inserted().copy() if gr.ra is not None else None
    gr.verify_insert(seed)
    torch.cuda.synchronize()
    sampled = gr.v.sampled.cpu().numpy()
    g_v = {k: getattr(gr.v, k).cpu().numpy() for k in
           ("accept_len", "n_commit", "commit_tok", "accepted_nodes", "finished")}
    g_tok_after = gr.seq_tok.cpu().numpy()
    g_len_after = gr.seq_len.cpu().numpy()

    for p, o, seqs, od in trees:
        if od is not None:
            # verify/commit of p's sequences on the bench's own logits rows
            rows = np.concatenate([np.arange(row_off[s], row_off[s + 1]) for s in seqs])
            bits = logits[torch.from_numpy(rows).to(logits.device)].view(torch.int16).cpu().numpy()
            bits = bits.view(np.uint16)
            o_tok = np.ascontiguousarray(seq_tok[seqs])
            o_len = np.ascontiguousarray(seq_len[seqs])
            ov = o.verify(bits, od["row_offsets"], od["draft_len"], od["draft_tok"],
                          od["draft_parent"], od["draft_depth"], seq_id[seqs], seed, o_tok, o_len,
                          max_new[seqs])
            assert np.array_equal(sampled[rows], ov["sampled"]), (config, p, "sampled")
            for k, v in g_v.items():
                w = ov[k] if v.ndim == 1 else ov[k].reshape(v[seqs].shape)
                assert np.array_equal(v[seqs], w.astype(v.dtype)), (config, p, k)
            assert np.array_equal(g_tok_after[seqs], o_tok), (config, p, "seq_tok")
            assert np.array_equal(g_len_after[seqs], o_len), (config, p, "seq_len")
            # the step's insert (committed spans), oracle side
            o.insert(np.zeros(len(seqs), np.int32), o_tok, seq_len[seqs], o_len)
        if gr.ra is not None:  # this step's run-ahead spans (walk insertion)
            after = gr.runahead_inserted()
            sel = [i for i, (q, _) in enumerate(wl.w.runahead)
                   if q == p and after[i] > ra_before[i]]
            if sel:
                m = max(int(after[i]) for i in sel)
                tab = np.zeros((len(sel), m), np.int32)
                for j, i in enumerate(sel):
                    t = wl.w.runahead[i][1]
                    tab[j, :after[i]] = t[:after[i]]
                o.insert(np.zeros(len(sel), np.int32), tab, ra_before[sel], after[sel])
    # trees after the fused kernel's insert
    for p, o, _, _ in trees:
        _dump_equal(gr.cache, p, o)
    if gr.fused_step:
        # the NEXT drafts the fused call made from those trees, and the row offsets
        torch.cuda.synchronize()
        nd = {k: getattr(gr.d, k).cpu().numpy() for k in
              ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth", "draft_pos")}
        nd["draft_mask"] = gr.d.draft_mask.cpu().numpy().view(np.uint64)
        nro = gr.d.row_offsets.cpu().numpy()
        assert nro[0] == 0 and np.array_equal(np.diff(nro), nd["draft_len"].astype(np.int64) + 1)
        for p, o, seqs, _ in trees:
            if not len(seqs):
                continue
            od2 = o.draft(np.zeros(len(seqs), np.int32), g_tok_after[seqs], g_len_after[seqs],
                          g_len_after[seqs])
            for k, v in nd.items():
                assert np.array_equal(v[seqs], od2[k].astype(v.dtype)), (config, p, "next", k)

    # ---- random rows of the whole batch: full-V oracle Gumbel-max ------------
    total = int(row_off[-1])
    seq_of_row = np.searchsorted(row_off, np.arange(total), side="right") - 1
    pick = rng.choice(total, size=min(n_rows, total), replace=False)
    bits = logits[torch.from_numpy(pick).to(logits.device)].view(torch.int16).cpu().numpy()
    bits = bits.view(np.uint16)
    for i, r in enumerate(pick):
        s = int(seq_of_row[r])
        j = int(r - row_off[s])  # 0 = root row, else draft node j-1
        pos = int(seq_len[s]) + (0 if j == 0 else int(g_draft["draft_depth"][s, j - 1]))
        tok, nan = orc.sample_row(bits[i], seed, int(seq_id[s]), pos)
        assert not nan
        assert tok == sampled[r], (config, int(r), tok, int(sampled[r]))
    assert run.status()[0] == 0


def test_fullsize_grpo_first_step_every_row(orc):
    """BJ's headline configuration (GRPO, 1024 sequences, V = 151,936), the
    first step in full: the oracle engine holds all 128 prompts' trees (the
    same prior-epoch rollouts and committed prefixes), and EVERY output of
    the GPU step bench.py times -- every draft, every sampled row (~20K full-V
    Gumbel-max rows), every accept/commit and sequence table, the node count
    of every tree after the fused insert -- equals the oracle's.  Rows whose
    maximum z is a float tie are counted (the smallest-index rule decided
    them); divergent rows must be 0."""
    import torch
    import bench

    cfg = bench.CONFIGS["grpo"]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    gr = run.groups[0]
    n, B = gr.n, cfg["Bmax"]
    o = orc.Oracle(cfg["V"], cfg["prompts"], cfg["D"], cfg["L"], B)
    prior = wl.w.prior
    for i0 in range(0, len(prior), 1024):
        part = prior[i0:i0 + 1024]
        tab = np.zeros((len(part), max(len(t) for _, t in part)), np.int32)
        for i, (_, t) in enumerate(part):
            tab[i, :len(t)] = t
        o.insert([p for p, _ in part], tab, np.zeros(len(part), np.int32),
                 [len(t) for _, t in part])
    prompt = wl.seq_prompt.astype(np.int32)
    seq_tok = gr.seq_tok.cpu().numpy()
    seq_len = gr.seq_len.cpu().numpy()
    assert np.array_equal(seq_len, wl.t0)
    o.insert(prompt, seq_tok, np.zeros(n, np.int32), seq_len)
    assert run.status()[1]["nodes_used"] == cfg["prompts"] + o.node_count

    gr.draft()
    gr.standin()
    torch.cuda.synchronize()
    od = o.draft(prompt, seq_tok, seq_len, seq_len)
    d = gr.d
    for k in ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth", "draft_pos",
              "row_offsets"):
        assert np.array_equal(getattr(d, k).cpu().numpy(), od[k].astype(np.int64
                              if k == "row_offsets" else np.int32)), k
    assert np.array_equal(d.draft_mask.cpu().numpy().view(np.uint64), od["draft_mask"])
    row_off = od["row_offsets"]
    total = int(row_off[-1])
    assert total > 10 * n, "the step drafted almost nothing"

    seed = bench.step_seed(0, 0)
    gr.verify_insert(seed)  # srt_verify_insert_cursor: scan + fused accept + cursor insert
    torch.cuda.synchronize()
    sampled = gr.v.sampled.cpu().numpy()[:total]
    g_v = {k: getattr(gr.v, k).cpu().numpy() for k in
           ("accept_len", "n_commit", "commit_tok", "accepted_nodes", "finished")}
    o_tok, o_len = seq_tok.copy(), seq_len.copy()
    o_sampled = np.empty(total, np.int32)
    ties = np.empty(total, np.int32)
    o_v = {k: [] for k in g_v}
    step = 64  # sequences per oracle chunk (~1.3K rows, 0.4 GB of host logits)
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        r0, r1 = int(row_off[s0]), int(row_off[s1])
        bits = gr.logits[r0:r1].view(torch.int16).cpu().numpy().view(np.uint16)
        t_chunk, l_chunk = o_tok[s0:s1].copy(), o_len[s0:s1].copy()
        ov = o.verify(bits, row_off[s0:s1 + 1] - r0, od["draft_len"][s0:s1], od["draft_tok"][s0:s1],
                      od["draft_parent"][s0:s1], od["draft_depth"][s0:s1], wl.seq_id[s0:s1],
                      seed, t_chunk, l_chunk, wl.max_new[s0:s1])
        o_tok[s0:s1], o_len[s0:s1] = t_chunk, l_chunk
        o_sampled[r0:r1] = ov["sampled"]
        ties[r0:r1] = ov["ties"]
        for k in o_v:
            o_v[k].append(ov[k])
    divergent = int(np.count_nonzero(sampled != o_sampled))
    tie_rows = int(np.count_nonzero(ties >= 2))
    print(f"[every-row parity] rows {total}, tie rows {tie_rows}, divergent rows {divergent}")
    assert divergent == 0
    for k, v in g_v.items():
        w = np.concatenate(o_v[k]).reshape(v.shape)
        assert np.array_equal(v, w.astype(v.dtype)), k
    assert np.array_equal(gr.seq_tok.cpu().numpy(), o_tok)
    assert np.array_equal(gr.seq_len.cpu().numpy(), o_len)
    # the committed spans into the oracle trees; every tree's node count and a
    # few whole trees equal the fused kernel's insert
    o.insert(prompt, o_tok, seq_len, o_len)
    bits, st = run.status()
    assert bits == 0
    assert st["nodes_used"] == cfg["prompts"] + o.node_count
    for p in np.random.default_rng(3).choice(cfg["prompts"], 3, replace=False):
        _dump_equal(gr.cache, int(p), _OracleView(o, int(p)))


class _OracleView:
    """o.dump(0) of a one-prompt oracle == dump(p) of the whole-batch oracle."""

    def __init__(self, o, p):
        self.o, self.p = o, p

    def dump(self, _):
        return self.o.dump(self.p)


def test_fullsize_b200x8_sharded_rank(orc):
    """BJ:configs[4] per rank at full size through the hash-sharded path
    bench.py times (bench.ShardedRun at N = 1: owner drafts over the mirror
    tables, the draft-return all-to-all, verify, the span all-gather, the
    owner's cursor insert; 4096 sequences of 256 prompts x 16): after 2 steps
    the trees of sampled prompts, the next drafts of their sequences and their
    verify / commit on the bench's own logits equal the oracle's."""
    import torch
    import bench

    cfg = dict(bench.CONFIGS["b200x8"])
    run = bench.ShardedRun(cfg, 0, 0, 1, "bf16", "rl-mix", gather=lambda t: t)
    for k in range(2):
        run.step(bench.step_seed(0, k))
    torch.cuda.synchronize()
    assert run.status()[0] == 0
    wl = bench.Workload(cfg, 0, prompt_ids=range(0, cfg["prompts"]))  # block 0 = every prompt
    rng = np.random.default_rng(23)
    prompts = [int(p) for p in rng.choice(np.unique(wl.seq_prompt), size=2, replace=False)]
    # the owner's mirror tables (at N = 1: mirror j = local sequence j)
    seq_tok = run.m_tok.cpu().numpy()
    seq_len = run.m_len.cpu().numpy()
    assert np.array_equal(seq_len, run.seq_len.cpu().numpy())
    trees = []
    for p in prompts:
        o, seqs = _history_tree(orc, wl, cfg, p, seq_tok, seq_len, run)
        _dump_equal(run.cache, p, o)
        trees.append((p, o, seqs))
    # the step under test
    run.draft()
    run.standin()
    seed = bench.step_seed(0, 2)
    torch.cuda.synchronize()
    d = run.d
    g_draft = {k: getattr(d, k).cpu().numpy() for k in
               ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth", "draft_pos")}
    row_off = d.row_offsets.cpu().numpy()
    run.verify_insert(seed)
    torch.cuda.synchronize()
    sampled = run.v.sampled.cpu().numpy()
    n_commit = run.v.n_commit.cpu().numpy()
    drafted = 0
    for p, o, seqs in trees:
        od = o.draft(np.zeros(len(seqs), np.int32), seq_tok[seqs], seq_len[seqs], seq_len[seqs])
        for k, v in g_draft.items():
            assert np.array_equal(v[seqs], od[k].astype(v.dtype)), (p, k)
        drafted += int(od["draft_len"].sum())
        rows = np.concatenate([np.arange(row_off[s], row_off[s + 1]) for s in seqs])
        bits = run.logits[torch.from_numpy(rows).to(run.logits.device)].view(torch.int16)
        bits = bits.cpu().numpy().view(np.uint16)
        o_tok = np.ascontiguousarray(seq_tok[seqs])
        o_len = np.ascontiguousarray(seq_len[seqs])
        ov = o.verify(bits, od["row_offsets"], od["draft_len"], od["draft_tok"], od["draft_parent"],
                      od["draft_depth"], wl.seq_id[seqs], seed, o_tok, o_len, wl.max_new[seqs])
        assert np.array_equal(sampled[rows], ov["sampled"]), (p, "sampled")
        assert np.array_equal(n_commit[seqs], ov["n_commit"]), (p, "n_commit")
        # the owner inserted the spans: its tree equals the oracle's after the commit
        o.insert(np.zeros(len(seqs), np.int32), o_tok, seq_len[seqs], o_len)
        _dump_equal(run.cache, p, o)
    assert drafted > 0
    assert run.status()[0] == 0
