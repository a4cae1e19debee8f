"""Development check of bench.py's forward stand-in: head logit placement."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
cfg = dict(bench.CONFIGS["grpo"]); cfg["prompts"] = 4; cfg["active"] = 32; cfg["node_capacity"] = 1 << 24
wl = bench.Workload(cfg, 0)
run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
for k in range(2):
    run.cache.draft(run.prompt_id, run.seq_tok, run.seq_len, run.seq_len, out=run.d)
    run.standin()
    torch.cuda.synchronize()
    rows = run.d.row_offsets.cpu().numpy(); t = run.seq_len.cpu().numpy()
    for s in range(4):
        r = rows[s]
        x = run.logits[r].float().cpu().numpy()
        h = wl.truth[s][min(t[s], len(wl.truth[s]) - 1)]
        top = np.argsort(-x)[:5]
        lse = np.log(np.exp(x.astype(np.float64) - x.max()).sum()) + x.max()
        print(f"step {k} seq {s} row {r}: head {h} x[head] {x[h]:.2f} top5 {top.tolist()} {x[top].round(2).tolist()} p_head {np.exp(x[h]-lse):.3f} gap {run.gaps[r].item():.2f}")
    run.cache.verify(run.logits, run.d, run.seq_id, bench.step_seed(0, k), run.seq_tok, run.seq_len, run.max_new, out=run.v)
    run.cache.insert(run.prompt_id, run.seq_tok, run.t_before, run.seq_len)
