"""Insert-kernel probe (development tool): how srt_insert_cursor time depends
on the span length m (every sequence appends m ground-truth tokens), and the
commit-length distribution of real steps.

    python tools/insert_probe.py [--config grpo]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="grpo")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    for k in range(4):
        run.step(bench.step_seed(0, k))
        nc = run.v.n_commit.cpu().numpy()
        print(f"step {k}: n_commit mean {nc.mean():.2f} p90 {np.percentile(nc, 90):.0f} "
              f"p99 {np.percentile(nc, 99):.0f} max {nc.max()}")
    n = run.n
    # per-sequence cycle profile of the cursor kernel inside real steps
    import ctypes
    from paper_2601_09083_b200 import _lib
    L = _lib.load()
    prof = torch.zeros(n, 8, dtype=torch.int64, device=run.dev)
    L.srt_debug_insert_profile(ctypes.c_void_p(prof.data_ptr()))
    for k in range(3):
        prof.zero_()
        run.step(bench.step_seed(0, 10 + k))
        torch.cuda.synchronize()
        p = prof.cpu().numpy()
        tot = p[:, 0]
        act = tot > 0
        print(f"profiled step {k}: active {act.sum()} total cycles p50 {np.percentile(tot[act], 50):.0f} "
              f"p90 {np.percentile(tot[act], 90):.0f} p99 {np.percentile(tot[act], 99):.0f} max {tot.max()}; "
              f"cursor-phase p50 {np.percentile(p[act, 1], 50):.0f} max {p[:, 1].max()}; "
              f"invalid cursors {(act & (p[:, 5] == 0)).sum()}")
        for s_ in np.argsort(-tot)[:6]:
            print(f"   slow seq {s_}: cycles {p[s_, 0]} cursor {p[s_, 1]} positions {p[s_, 2]} "
                  f"created {p[s_, 3]} slowest position {p[s_, 4]} valid {p[s_, 5]} batch {p[s_, 6]} "
                  f"resolve {p[s_, 7] >> 32} counts {p[s_, 7] & 0xFFFFFFFF}")
    # the longest span alone (every other sequence's span empty), then the rest
    for k in range(2):
        run.draft()
        run.standin()
        run.cache.verify(run.logits, run.d, run.seq_id, bench.step_seed(0, 20 + k), run.seq_tok,
                         run.seq_len, run.max_new, out=run.v, rows=run.rows_max)
        torch.cuda.synchronize()
        nc = run.v.n_commit
        big = int(torch.argmax(nc).item())
        to1 = run.t_before.clone()
        to1[big] = run.seq_len[big]
        prof.zero_()
        us1 = timed(lambda: run.cache.insert(run.prompt_id, run.seq_tok, run.t_before, to1,
                                             cursor=run.cursor))
        p1 = prof[big].cpu().numpy()
        fr2 = run.t_before.clone()
        fr2[big] = run.seq_len[big]
        us2 = timed(lambda: run.cache.insert(run.prompt_id, run.seq_tok, fr2, run.seq_len,
                                             cursor=run.cursor))
        print(f"alone: seq {big} span {int(nc[big])}: insert {us1:.1f} us, cycles {p1[0]} "
              f"slowest position {p1[4]} created {p1[3]} batch {p1[6] >> 20} rounds {p1[6] & 0xFFFFF} resolve {p1[7] >> 32} "
              f"counts {p1[7] & 0xFFFFFFFF}; the other 1023 spans: {us2:.1f} us")
    L.srt_debug_insert_profile(ctypes.c_void_p(0))
    ar = torch.arange(n, device=run.dev)
    for m in (1, 2, 4, 8, 16, 24, 32):
        for mode in ("cursor", "walk"):
            tok = run.seq_tok.clone()
            t0 = run.seq_len.clone()
            cur = run.cursor.clone()
            pos = t0.to(torch.int64)[:, None] + torch.arange(m, device=run.dev)[None, :]
            src = torch.minimum(pos, run.truth_last[:, None])
            tok[ar[:, None], pos.clamp(max=tok.shape[1] - 1)] = torch.gather(run.truth, 1, src)
            to = (t0 + m).clamp(max=tok.shape[1])
            if mode == "cursor":
                us = timed(lambda: run.cache.insert(run.prompt_id, tok, t0, to, cursor=cur))
            else:
                us = timed(lambda: run.cache.insert(run.prompt_id, tok, t0, to))
            print(f"m={m:2d} {mode:6s}: {us:8.1f} us")
    bits, st = run.cache.status()
    print("status", bits, st)


if __name__ == "__main__":
    main()
