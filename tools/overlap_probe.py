"""Overlap probe (development tool): does a latency-bound tree kernel of one
prompt group run concurrently with the HBM-bound verify scan of another?

    python tools/overlap_probe.py [--config grpo]

Times group 0's verify (scan + accept) alone, group 1's draft alone, and both
launched on two streams at once.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="grpo")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0, groups=2)
    g0, g1 = run.groups
    s0, s1 = run.streams
    seed = bench.step_seed(0, 0)
    for _ in range(3):
        run.step(seed)
    torch.cuda.synchronize()
    g0.draft()
    g0.standin()
    torch.cuda.synchronize()

    def verify0():
        g0.cache.verify(g0.logits, g0.d, g0.seq_id, seed, g0.seq_tok.clone(), g0.seq_len.clone(),
                        g0.max_new, out=g0.v, rows=g0.rows_max)

    def draft1():
        g1.draft()

    for name, fns in (("verify0 alone", [verify0]), ("draft1 alone", [draft1]),
                      ("both", [verify0, draft1])):
        for rep in range(3):
            e0, e1 = ev(), ev()
            torch.cuda.synchronize()
            e0.record()
            for st in (s0, s1):
                st.wait_event(e0)
            for fn, st in zip(fns, (s0, s1)):
                with torch.cuda.stream(st):
                    fn()
            for st in (s0, s1):
                torch.cuda.current_stream().wait_stream(st)
            e1.record()
            torch.cuda.synchronize()
            print(f"{name:14s} rep {rep}: {e0.elapsed_time(e1) * 1000:8.1f} us")


if __name__ == "__main__":
    main()
