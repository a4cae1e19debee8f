"""bench.py's pipelined schedule (prompt groups, each with its own cache, on
separate streams with no host sync) must commit exactly what the sequential
schedule of the same groups on one stream commits: groups own disjoint
prompts and the library keeps no state shared between caches.
(The forward stand-in's synthetic logits depend on the row layout, so the
comparison is between schedules of the same grouping.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(groups, pipelined, steps=6):
    import torch
    import bench
    cfg = dict(bench.CONFIGS["grpo"])
    cfg.update(prompts=6, active=48, V=5000, cap=1024, act_cap=1024, median=300,
               node_capacity=1 << 20)
    wl = bench.Workload(cfg, 1)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 1, groups=groups)
    seed = bench.step_seed(1, 0)
    for _ in range(steps):
        if pipelined:
            run.step_pipelined(seed)
        else:
            run.step(seed)
    torch.cuda.synchronize()
    bits, _ = run.status()
    assert bits == 0
    n = cfg["active"]
    toks = np.zeros((n, run.groups[0].seq_tok.shape[1]), np.int32)
    lens = np.zeros(n, np.int32)
    for gr in run.groups:
        toks[gr.seqs] = gr.seq_tok.cpu().numpy()
        lens[gr.seqs] = gr.seq_len.cpu().numpy()
    return toks, lens, wl


def test_pipelined_groups_match_sequential():
    t1, l1, wl = _run(3, False)
    t3, l3, _ = _run(3, True)
    assert np.array_equal(l1, l3)
    assert np.array_equal(t1, t3)
    assert (l1 > wl.t0).all()  # every sequence advanced


@pytest.mark.parametrize("D", [32, 64, 128])
def test_fused_verify_insert_matches_separate_calls(D):
    """srt_verify_insert_cursor (accept + cursor insert fused; one warp per
    sequence at D = 32, one CTA of D/32 warps at D = 64 and 128) leaves
    exactly what srt_verify then srt_insert_cursor leave: sequence tables,
    commits, sampled tokens, trees, the next drafts, and the cursors -- the
    same position / prompt / floor and the same existing suffix nodes wherever
    the separate call's record is valid (a span longer than D goes through
    the walk path there and invalidates it; the fused record must then sit at
    the new length)."""
    import torch
    import bench
    cfg = dict(bench.CONFIGS["grpo"])
    cfg.update(prompts=6, active=48, V=5000, cap=1024, act_cap=1024, median=300,
               node_capacity={32: 1 << 20, 64: 1 << 23, 128: 1 << 24}[D], D=D, L=8)
    out = []
    for fused in (False, True):
        wl = bench.Workload(cfg, 2)
        run = bench.GpuRun(wl, "bf16", "rl-mix", 2)
        gr = run.groups[0]
        gr.fused = fused
        rec = []
        for k in range(6):
            run.step(bench.step_seed(2, k))
            R = int(gr.d.row_offsets[-1].item())  # (rows past R are not written)
            rec.append((gr.v.sampled[:R].cpu().numpy().copy(), gr.v.n_commit.cpu().numpy().copy(),
                        gr.v.commit_tok.cpu().numpy().copy(), gr.d.draft_tok.cpu().numpy().copy()))
        torch.cuda.synchronize()
        assert run.status()[0] == 0
        out.append((rec, gr.seq_tok.cpu().numpy(), gr.seq_len.cpu().numpy(),
                    gr.cursor.cpu().numpy(), [gr.cache.dump(p) for p in range(3)]))
    (ra, ta, la, ca, da), (rb, tb, lb, cb, db) = out
    for x, y in zip(ra, rb):
        for u, v in zip(x, y):
            np.testing.assert_array_equal(u, v)
    np.testing.assert_array_equal(ta, tb)
    np.testing.assert_array_equal(la, lb)
    assert da == db
    assert (la > 0).all() and sum(int(r[1].sum()) for r in ra) > 48
    # cursor records: word 0 is the cache's tag and words 4.. are node ids
    # (hash slots, which depend on the order racing inserts claimed them), so
    # the two caches' records agree on position / prompt / floor and on which
    # suffix nodes exist
    NONE = np.uint32(0xFFFFFFFF).view(np.int32)
    valid = ca[:, 1] != NONE  # separate record valid
    np.testing.assert_array_equal(ca[valid, 1:4], cb[valid, 1:4])
    np.testing.assert_array_equal(ca[valid, 4:] == NONE, cb[valid, 4:] == NONE)
    assert np.array_equal(cb[~valid, 1], lb[~valid])  # fused record at the new length
    assert valid.sum() > len(valid) // 2


def test_graph_replay_matches_eager():
    """bench.py's CUDA-graph step (draft segment + verify/insert segment
    captured once, replayed) commits exactly what the eager step commits."""
    import torch
    import bench
    cfg = dict(bench.CONFIGS["grpo"])
    cfg.update(prompts=6, active=48, V=5000, cap=1024, act_cap=1024, median=300,
               node_capacity=1 << 20)
    seed = bench.step_seed(1, 0)
    out = []
    for graph in (False, True):
        wl = bench.Workload(cfg, 1)
        run = bench.GpuRun(wl, "bf16", "rl-mix", 1)
        gr = run.groups[0]
        run.step(seed)  # warm (allocations happen outside any capture)
        if graph:
            g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                gr.draft()
            with torch.cuda.graph(g2):
                gr.verify_insert(seed)
            for _ in range(6):
                g1.replay()
                gr.standin()
                g2.replay()
        else:
            for _ in range(6):
                run.step(seed)
        torch.cuda.synchronize()
        assert run.status()[0] == 0
        out.append((gr.seq_tok.cpu().numpy(), gr.seq_len.cpu().numpy(), gr.cache.dump(0)))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("D", [16, 32, 64, 128])
def test_fused_tree_step_matches_separate_calls(D):
    """srt_verify_insert_draft_cursor (commit + cursor insert + per-prompt hub
    refresh + the next draft in one persistent kernel) leaves exactly what
    srt_verify_insert_cursor then srt_draft_cursor leave, step after step:
    sampled rows, commits, sequence tables, trees, the next drafts and row
    offsets (both from the same buffers the next step reads)."""
    import torch
    import bench
    cfg = dict(bench.CONFIGS["grpo"])
    cfg.update(prompts=12, active=96, V=5000, cap=1024, act_cap=1024, median=300,
               node_capacity={16: 1 << 21, 32: 1 << 21, 64: 1 << 23, 128: 1 << 24}[D], D=D, L=8)
    out = []
    for fused_step in (False, True):
        wl = bench.Workload(cfg, 3)
        run = bench.GpuRun(wl, "bf16", "rl-mix", 3)
        gr = run.groups[0]
        gr.fused_step = fused_step
        rec = []
        for k in range(8):
            run.step(bench.step_seed(3, k))
            if not fused_step:
                gr.draft()  # the next step's draft, as the fused call makes it
            torch.cuda.synchronize()
            rec.append(tuple(getattr(gr.d, k).cpu().numpy().copy() for k in
                             ("match_len", "draft_len", "draft_tok", "draft_parent",
                              "draft_depth", "draft_pos", "draft_mask", "row_offsets")) +
                       (gr.v.n_commit.cpu().numpy().copy(), gr.v.commit_tok.cpu().numpy().copy(),
                        gr.v.accept_len.cpu().numpy().copy()))
        torch.cuda.synchronize()
        assert run.status()[0] == 0
        out.append((rec, gr.seq_tok.cpu().numpy(), gr.seq_len.cpu().numpy(),
                    [gr.cache.dump(p) for p in range(cfg["prompts"])]))
    (ra, ta, la, da), (rb, tb, lb, db) = out
    for x, y in zip(ra, rb):
        for u, v in zip(x, y):
            np.testing.assert_array_equal(u, v)
    np.testing.assert_array_equal(ta, tb)
    np.testing.assert_array_equal(la, lb)
    assert da == db
    assert sum(int(r[1].sum()) for r in ra) > 0 and sum(int(r[8].sum()) for r in ra) > 96 * 8


@pytest.mark.parametrize("D", [16, 32])
def test_fused_tree_step_beside_scan_matches(D):
    """The fused tree step run BESIDE the scan (srt_cache_set_step_overlap:
    the step kernel on a few SMs, committing each sequence as the scan
    finishes its rows) leaves exactly what the step after the scan leaves,
    step after step: sampled rows, commits, sequence tables, trees, the next
    drafts and row offsets -- for several SM splits, including one SM (every
    sequence's work serialised behind the scan's progress)."""
    import torch
    import bench
    cfg = dict(bench.CONFIGS["grpo"])
    cfg.update(prompts=12, active=96, V=5000, cap=1024, act_cap=1024, median=300,
               node_capacity=1 << 21, D=D, L=8)
    out = []
    for sms in (0, 1, 8, 40):
        wl = bench.Workload(cfg, 5)
        run = bench.GpuRun(wl, "bf16", "rl-mix", 5)
        gr = run.groups[0]
        gr.fused_step = True
        gr.cache.set_step_overlap(sms)
        rec = []
        for k in range(8):
            rows = int(gr.d.row_offsets[gr.n].item()) if k else None  # (the rows this step verifies)
            run.step(bench.step_seed(5, k))
            torch.cuda.synchronize()
            rec.append(tuple(getattr(gr.d, k).cpu().numpy().copy() for k in
                             ("match_len", "draft_len", "draft_tok", "draft_parent",
                              "draft_depth", "draft_pos", "draft_mask", "row_offsets")) +
                       (gr.v.n_commit.cpu().numpy().copy(), gr.v.commit_tok.cpu().numpy().copy(),
                        gr.v.accept_len.cpu().numpy().copy(),
                        gr.v.sampled[:rows].cpu().numpy().copy() if rows else np.zeros(0)))
        torch.cuda.synchronize()
        assert run.status()[0] == 0
        out.append((rec, gr.seq_tok.cpu().numpy(), gr.seq_len.cpu().numpy(),
                    [gr.cache.dump(p) for p in range(cfg["prompts"])]))
    ra, ta, la, da = out[0]
    for rb, tb, lb, db in out[1:]:
        for x, y in zip(ra, rb):
            for u, v in zip(x, y):
                np.testing.assert_array_equal(u, v)
        np.testing.assert_array_equal(ta, tb)
        np.testing.assert_array_equal(la, lb)
        assert da == db
    assert sum(int(r[1].sum()) for r in ra) > 0 and sum(int(r[8].sum()) for r in ra) > 96 * 8


@pytest.mark.parametrize("extra", [[], ["--sharded"], ["--fused-step", "0"], ["--verify", "path"],
                                   ["--graph", "0"]])
def test_bench_cli_runs(extra):
    """bench.py's control flow end to end on the tiny configuration (the
    driver runs it; the single-rank, sharded, unfused, path-only and eager
    variants): one parseable JSON line with the contract's keys."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "tiny",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1",
                        *extra], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "roofline", "e2e", "gpu_launches", "config"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0
