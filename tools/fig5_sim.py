"""Synthetic Fig. 5: mean accepted tokens per
decoding step for three cache-maintenance strategies, driven through the
libsrt kernels on a DAPO-shaped synthetic batch (1024 fresh rollouts of 64
prompts x 16 samples, V = 151,936, Bmax = 32, D = 32):

  history-only   the cache holds only completed responses of the previous
                 epoch; nothing is inserted while the batch decodes
                 (He et al. 2025, the paper's comparison);
  online (SRT)   + every step's committed tokens are inserted (P:L151 first
                 source: running rollouts);
  online + run-ahead  + before the batch starts, run-ahead rollouts of the same
                 prompts (generated in an earlier batch's bubbles, P:L151
                 second source) were inserted.

Only the ORDERING is comparable with the paper (its values are absent, O16);
the logits are the bench stand-in (the ground-truth continuation is the
policy's preferred token, rl-mix gaps), so acceptance measures how often the
tree predicts the rollout.

    python tools/fig5_sim.py [--steps 48] [--runahead 2] > profiles/r01_fig5_sim.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

CFG = dict(V=151936, prompts=64, samples=16, active=1024, Bmax=32, D=32, L=8, median=3000,
           cap=8192, act_cap=8192, prior_epochs=1, node_capacity=1 << 27)


def run_mode(mode: str, steps: int, runahead: int, seed: int):
    cfg = dict(CFG)
    if mode == "online+runahead":
        cfg["runahead"] = dict(first=0, prompts=cfg["prompts"], per=runahead, spans=0, lo=1, hi=1)
    wl = bench.Workload(cfg, seed)
    wl.t0[:] = 0  # fresh rollouts: nothing of this epoch is in the cache yet
    run = bench.GpuRun(wl, "bf16", "rl-mix", seed)
    gr = run.groups[0]
    gr.ra = None  # run-ahead rollouts go in once, before the batch (below)
    if mode == "online+runahead":
        streams = wl.w.runahead
        m = max(len(t) for _, t in streams)
        tab = np.zeros((len(streams), m), np.int32)
        for i, (_, t) in enumerate(streams):
            tab[i, :len(t)] = t
        dev = gr.dev
        gr.cache.insert(torch.tensor([p for p, _ in streams], dtype=torch.int32, device=dev),
                        torch.from_numpy(tab).to(dev),
                        torch.zeros(len(streams), dtype=torch.int32, device=dev),
                        torch.tensor([len(t) for _, t in streams], dtype=torch.int32, device=dev))
    acc, com, match = [], [], []
    seed_k = bench.step_seed(seed, 0)
    for k in range(steps):
        gr.draft()
        gr.standin()
        gr.cache.verify(gr.logits, gr.d, gr.seq_id, seed_k, gr.seq_tok, gr.seq_len, gr.max_new,
                        out=gr.v, rows=gr.rows_max)
        if mode != "history-only":
            gr.cache.insert(gr.prompt_id, gr.seq_tok, gr.t_before, gr.seq_len, cursor=gr.cursor)
        acc.append(float(gr.v.accept_len.float().mean().item()))
        com.append(float(gr.v.n_commit.float().mean().item()))
        match.append(float((gr.d.match_len > 0).float().mean().item()))
    bits, st = run.status()
    assert bits == 0, bits
    del run, gr
    torch.cuda.empty_cache()
    return {"mean_accepted_per_step": float(np.mean(acc)),
            "mean_committed_per_step": float(np.mean(com)),
            "fraction_of_steps_with_a_match": float(np.mean(match)),
            "accepted_per_step_curve": [round(a, 4) for a in acc]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--runahead", type=int, default=2, help="run-ahead rollouts per prompt")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    out = {"workload": "fig5-sim: 64 prompts x 16 samples (1024 fresh rollouts), V=151936, "
                       f"Bmax=32, D=32, L=8, median 3000 tokens, {a.steps} decoding steps, "
                       f"{a.runahead} run-ahead rollouts per prompt",
           "modes": {}}
    for mode in ("history-only", "online", "online+runahead"):
        out["modes"][mode] = run_mode(mode, a.steps, a.runahead, a.seed)
        print(f"[fig5] {mode}: {out['modes'][mode]['mean_accepted_per_step']:.3f} accepted/step",
              file=sys.stderr, flush=True)
    m = out["modes"]
    out["ordering_holds"] = (m["history-only"]["mean_accepted_per_step"]
                             < m["online"]["mean_accepted_per_step"]
                             < m["online+runahead"]["mean_accepted_per_step"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
