"""Draft-kernel probe (development tool): per-sequence cycle profile of
srt_draft on the bench workload (srt_debug_draft_profile), to see whether the
slow warps are long pop chains or hub expansions.

    python tools/draft_probe.py [--config grpo] [--steps 3]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_09083_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="grpo")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    for k in range(3):
        run.step(bench.step_seed(0, k))
    n = run.n
    prof = torch.zeros(n, 8, dtype=torch.int64, device="cuda")
    L = _lib.load()
    L.srt_debug_draft_profile(ctypes.c_void_p(prof.data_ptr()))
    for k in range(a.steps):
        torch.cuda.synchronize()
        run.cache.draft(run.prompt_id, run.seq_tok, run.seq_len, run.seq_len, out=run.d,
                        cursor=run.cursor)
        torch.cuda.synchronize()
        p = prof.cpu().numpy()
        q = run.d.match_len.cpu().numpy()
        dl = run.d.draft_len.cpu().numpy()
        tot, mt, sc, mx = p[:, 1], p[:, 0], p[:, 2], p[:, 3]
        print(f"step {k}: total cycles p50 {np.percentile(tot, 50):.0f} p90 {np.percentile(tot, 90):.0f} "
              f"p99 {np.percentile(tot, 99):.0f} max {tot.max()}; match p50 {np.percentile(mt, 50):.0f} "
              f"max {mt.max()}")
        print(f"   q hist {np.bincount(q, minlength=9).tolist()}  draft_len mean {dl.mean():.1f}")
        print(f"   children scanned p50 {np.percentile(sc, 50):.0f} p99 {np.percentile(sc, 99):.0f} "
              f"max {sc.max()}; max fan-out p50 {np.percentile(mx, 50):.0f} p99 {np.percentile(mx, 99):.0f} max {mx.max()}")
        nsing = p[:, 7] & ((1 << 20) - 1)
        nmul = p[:, 7] >> 20
        full = dl == cfg["Bmax"]
        if full.any():
            f = full
            print(f"   full drafts: {f.sum()} seqs; per seq mean: single pops {nsing[f].mean():.1f}, "
                  f"multi pops {nmul[f].mean():.1f}; cycles: total {tot[f].mean():.0f}, match "
                  f"{mt[f].mean():.0f}, rec waits {p[f, 4].mean():.0f} "
                  f"({p[f, 4].sum() / max(1, (nsing[f] + nmul[f]).sum()):.0f}/pop), block lookups "
                  f"{p[f, 5].mean():.0f} ({p[f, 5].sum() / max(1, nmul[f].sum()):.0f}/multi), "
                  f"child rounds {p[f, 6].mean():.0f} ({p[f, 6].sum() / max(1, nmul[f].sum()):.0f}/multi)")
        for lo, hi in ((0, 64), (64, 256), (256, 1024), (1024, 1 << 30)):
            sel = (sc >= lo) & (sc < hi)
            if sel.any():
                print(f"   scanned in [{lo},{hi}): {sel.sum()} seqs, cycles p50 "
                      f"{np.percentile(tot[sel], 50):.0f} p90 {np.percentile(tot[sel], 90):.0f} "
                      f"max {tot[sel].max()}; draft_len mean {dl[sel].mean():.1f}")
        slow = np.argsort(-tot)[:8]
        for s in slow:
            print(f"   slow seq {s}: cycles {tot[s]} match {mt[s]} q {q[s]} len {dl[s]} scanned {sc[s]} "
                  f"maxfan {mx[s]} rec {p[s,4]} blk {p[s,5]} rounds {p[s,6]} single/multi {nsing[s]}/{nmul[s]}")
        run.standin()
        run.cache.verify(run.logits, run.d, run.seq_id, bench.step_seed(0, 100 + k), run.seq_tok,
                         run.seq_len, run.max_new, out=run.v)
        run.cache.insert(run.prompt_id, run.seq_tok, run.t_before, run.seq_len, cursor=run.cursor)
    L.srt_debug_draft_profile(ctypes.c_void_p(0))


if __name__ == "__main__":
    main()
