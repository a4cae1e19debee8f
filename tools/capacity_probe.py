"""Capacity-management probe (development tool): on the GRPO bench cache
(72M nodes), time srt_cache_evict to 90 % / 50 % of the live nodes and the
dump + load round trip of one prompt's tree into a fresh cache, then run a
few steps to show the pruned cache keeps drafting (accepted tokens per step).

    python tools/capacity_probe.py [--config grpo]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_09083_b200 as srt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="grpo")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    out = {}

    def acc(k):
        tot = 0
        for i in range(k):
            run.step(bench.step_seed(0, 100 + i))
            tot += int(run.v.accept_len.sum().item())
        return tot / (k * run.n)

    out["accepted_per_seq_step_before"] = acc(3)
    live = run.status()[1]["nodes_used"]
    for frac in (0.9, 0.5):
        torch.cuda.synchronize()
        t = time.time()
        removed, theta = run.cache.evict(int(live * frac))
        dt = time.time() - t
        live2 = run.status()[1]["nodes_used"]
        out[f"evict_to_{frac}"] = {"seconds": dt, "theta": theta, "removed": removed,
                                  "live_before": live, "live_after": live2}
        out[f"accepted_per_seq_step_after_evict_{frac}"] = acc(3)
        live = live2
    p = int(run.prompt_id[0].item())
    t = time.time()
    recs = run.cache.dump(p)
    t_dump = time.time() - t
    fresh = srt.SrtCache(srt.config(cfg["V"], cfg["prompts"], cfg["D"], cfg["L"], cfg["Bmax"],
                                    node_capacity=1 << 22))
    t = time.time()
    fresh.load(p, recs)
    t_load = time.time() - t
    assert fresh.dump(p) == recs
    out["dump_load_one_prompt"] = {"records": len(recs), "dump_s": t_dump, "load_s": t_load,
                                   "round_trip_equal": True}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
