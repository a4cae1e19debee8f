"""Synthetic Fig. 5 through the libsrt kernels,
with the rollout loop's slot scheduler (paper_2601_09083_b200/rollout.py):
a DAPO-shaped run of several training steps (B prompts x K samples per step,
one slot per real sequence, long-tailed rollout lengths), each tick one SRT
step (draft -> policy stand-in -> verify -> insert) over the occupied slots,
for the paper's three cache-maintenance strategies:

  history-only     the cache gets completed responses at the end of each
                   training step only (the paper's comparison);
  online (SRT)     every tick's committed tokens are inserted;
  online+run-ahead + the slots freed by finished sequences (the bubbles of
                   the long tail) decode rollouts of the next step's
                   prompts (the look-ahead window), inserted online and
                   discarded at step end.

Plain decoding's step time is the longest rollout of the step (one token per
tick; tests/test_rollout_sim.py pins this on the oracle engine), reported as
the baseline.  Only the ORDERING of the strategies is comparable with the
paper (its values are absent, O16).

    python tools/fig5_sim.py [--steps 3] > profiles/r02_fig5_sim.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2601_09083_b200.rollout import GpuEngine, RolloutSim, SimConfig, summarize  # noqa: E402


def run_mode(mode, ra, a):
    cfg = SimConfig(V=151936, D=a.depth, L=8, Bmax=32, prompts_per_step=a.prompts,
                    samples=a.samples, steps=a.steps, mode=mode, run_ahead=ra, median=a.median,
                    cap=a.cap, seed=a.seed, ra_per_prompt=a.ra_per_prompt,
                    node_capacity=1 << 29)
    t = time.time()
    sim = RolloutSim(cfg, GpuEngine(cfg, synth.SimPolicy(cfg.seed, cfg.V)),
                     synth.RolloutStreams(cfg.seed, cfg.V, cfg.median, cfg.cap))
    sim.run()
    out = summarize(sim.reports)
    out["wall_s"] = round(time.time() - t, 1)
    out["baseline_ticks_per_step"] = [
        max(len(v) for k, v in sim.rollouts.items() if (k >> 44) & 0xFFFFF == s)
        for s in range(cfg.steps)]
    del sim
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--prompts", type=int, default=64)
    ap.add_argument("--samples", type=int, default=16)
    ap.add_argument("--median", type=int, default=1000)
    ap.add_argument("--cap", type=int, default=4000)
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--ra-per-prompt", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    out = {"workload": f"fig5-sim: {a.steps} training steps x {a.prompts} prompts x {a.samples} "
                       f"samples (one slot per real sequence), V=151936, Bmax=32, D={a.depth}, "
                       f"L=8, rollout length LogNormal(median {a.median}, 0.9) <= {a.cap}, one "
                       f"warm epoch; run-ahead: <= {a.ra_per_prompt} rollouts per look-ahead "
                       f"prompt (the next step's batch)",
           "modes": {}}
    for mode, ra, name in (("history_only", False, "history-only"), ("srt", False, "online"),
                           ("srt", True, "online+runahead")):
        out["modes"][name] = run_mode(mode, ra, a)
        print(f"[fig5] {name}: {out['modes'][name]['mean_accepted']:.3f} accepted/step, "
              f"{out['modes'][name]['ticks']} ticks, {out['modes'][name]['wall_s']} s",
              file=sys.stderr, flush=True)
    m = out["modes"]
    acc = {k: v["mean_accepted"] for k, v in m.items()}
    out["ordering_holds"] = acc["history-only"] < acc["online"] < acc["online+runahead"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
