"""Scan time in context (development probe): the GRPO step's scan right after
the fused tree step (as the bench times it) vs the same rows scanned again
right after a scan (no tree work in between), vs after an L2 flush.

    python tools/scan_context_probe.py [--config grpo]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="grpo")
    a = ap.parse_args()
    wl = bench.Workload(bench.CONFIGS[a.config], 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    gr = run.groups[0]
    gr.fused_step = True
    for k in range(4):
        run.step(bench.step_seed(0, k))
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    c = gr.cache
    c.profile_enable(4096)
    res = {"after_tree_step": [], "after_scan": [], "after_flush": []}
    rows = {k: [] for k in res}
    for k in range(6):
        rows["after_tree_step"].append(int(gr.d.row_offsets[gr.n].item()))
        run.step(bench.step_seed(0, 10 + k))  # scan + fused tree step (this step's scan: after a tree step)
        torch.cuda.synchronize()
        recs = c.profile_read()
        res["after_tree_step"] += [ms for n, ms in recs if n == "scan"]
        # the same rows again, twice: a scan after a scan; then after an L2 flush
        sl, st = gr.seq_len.clone(), gr.seq_tok.clone()
        for mode in ("after_scan", "after_flush"):
            if mode == "after_flush":
                flush.add_(1)
            gr.seq_len.copy_(sl)
            rows[mode].append(int(gr.d.row_offsets[gr.n].item()))
            c.verify(run.logits, gr.d, gr.seq_id, bench.step_seed(0, 10 + k), gr.seq_tok, gr.seq_len,
                     gr.max_new, out=gr.v, rows=gr.rows_max)
            torch.cuda.synchronize()
            res[mode] += [ms for n, ms in c.profile_read() if n == "scan"]
        gr.seq_len.copy_(sl)
        gr.seq_tok.copy_(st)
    for k, v in res.items():
        v, r = v[1:], rows[k][1:]
        gbs = sum(r) * wl.cfg["V"] * 2 / (sum(v) / 1000) / 1e9
        print(f"{k:16s} scan mean {1000 * sum(v) / len(v):8.1f} us, rows mean {sum(r) / len(r):8.0f}, "
              f"{gbs:7.1f} GB/s over {len(v)}")


if __name__ == "__main__":
    main()
