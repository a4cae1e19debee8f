"""Full-size parity: BASELINE.json's configurations at their full sizes, in the
launch configuration bench.py times (bench.GpuRun: the same caches, kernels,
workload recipe and forward stand-in), checked against the oracle on SAMPLED
outputs the oracle can compute one by one:

* the trees of sampled prompts — the oracle re-inserts each sampled prompt's
  whole history (prior-epoch rollouts + every active sequence's committed
  tokens) and its canonical dump must equal the GPU's (before and after a
  step's insert);
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

    # ---- the step under test: draft -> stand-in -> verify -> insert ----------
    gr.draft()
    gr.standin()
    seed = bench.step_seed(0, steps)
    torch.cuda.synchronize()
    d = gr.d
    g_draft = {k: getattr(d, k).cpu().numpy() for k in
               ("match_len", "draft_len", "draft_tok", "draft_parent", "draft_depth", "draft_pos")}
    g_draft["draft_mask"] = d.draft_mask.cpu().numpy().view(np.uint64)
    row_off = d.row_offsets.cpu().numpy()
    logits = gr.logits  # bf16 [rows_max + 1, V]
    gr.cache.verify(logits, d, gr.seq_id, seed, gr.seq_tok, gr.seq_len, gr.max_new, out=gr.v,
                    rows=gr.rows_max)
    torch.cuda.synchronize()
    sampled = gr.v.sampled.cpu().numpy()
    g_v = {k: getattr(gr.v, k).cpu().numpy() for k in
           ("accept_len", "n_commit", "commit_tok", "accepted_nodes", "finished")}
    g_tok_after = gr.seq_tok.cpu().numpy()
    g_len_after = gr.seq_len.cpu().numpy()
    seq_id = wl.seq_id
    max_new = wl.max_new

    drafted = 0
    trees = []
    for p in prompts:
        o, seqs = _history_tree(orc, wl, cfg, int(p), seq_tok, seq_len, gr)
        _dump_equal(gr.cache, int(p), o)
        if len(seqs) == 0:  # a look-ahead prompt: only run-ahead spans reach its tree
            trees.append((int(p), o))
            continue
        # drafts of p's sequences from the full-size tree
        od = o.draft(np.zeros(len(seqs), np.int32), seq_tok[seqs], seq_len[seqs], seq_len[seqs])
        for k, v in g_draft.items():
            assert np.array_equal(v[seqs], od[k].astype(v.dtype)), (config, p, k)
        drafted += int(od["draft_len"].sum())
        # verify/commit of p's sequences on the bench's own logits rows
        rows = np.concatenate([np.arange(row_off[s], row_off[s + 1]) for s in seqs])
        bits = logits[torch.from_numpy(rows).to(logits.device)].view(torch.int16).cpu().numpy()
        bits = bits.view(np.uint16)
        o_tok = np.ascontiguousarray(seq_tok[seqs])
        o_len = np.ascontiguousarray(seq_len[seqs])
        ov = o.verify(bits, od["row_offsets"], od["draft_len"], od["draft_tok"], od["draft_parent"],
                      od["draft_depth"], seq_id[seqs], seed, o_tok, o_len, max_new[seqs])
        assert np.array_equal(sampled[rows], ov["sampled"]), (config, p, "sampled")
        for k, v in g_v.items():
            w = ov[k] if v.ndim == 1 else ov[k].reshape(v[seqs].shape)
            assert np.array_equal(v[seqs], w.astype(v.dtype)), (config, p, k)
        assert np.array_equal(g_tok_after[seqs], o_tok), (config, p, "seq_tok")
        assert np.array_equal(g_len_after[seqs], o_len), (config, p, "seq_len")
        # the step's insert (committed spans), oracle side
        o.insert(np.zeros(len(seqs), np.int32), o_tok, seq_len[seqs], o_len)
        trees.append((int(p), o))
    assert drafted > 0, "the sampled prompts drafted nothing: the check is vacuous"
    # the step's insert, GPU side (cursor kernel, as bench.py times it)
    gr.cache.insert(gr.prompt_id, gr.seq_tok, gr.t_before, gr.seq_len, cursor=gr.cursor)
    if gr.ra is not None:  # and this step's run-ahead spans (walk insertion)
        before = gr.runahead_inserted().copy()
        gr.runahead_insert()
        after = gr.runahead_inserted()
        for p, o in trees:
            sel = [i for i, (q, _) in enumerate(wl.w.runahead) if q == p and after[i] > before[i]]
            if sel:
                m = max(int(after[i]) for i in sel)
                tab = np.zeros((len(sel), m), np.int32)
                for j, i in enumerate(sel):
                    t = wl.w.runahead[i][1]
                    tab[j, :after[i]] = t[:after[i]]
                o.insert(np.zeros(len(sel), np.int32), tab, before[sel], after[sel])
    torch.cuda.synchronize()
    for p, o in trees:
        _dump_equal(gr.cache, p, o)

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
