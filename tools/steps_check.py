import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
cfg = dict(bench.CONFIGS["grpo"]); cfg["prompts"] = 4; cfg["active"] = 32; cfg["node_capacity"] = 1 << 24
wl = bench.Workload(cfg, 0)
run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
for k in range(6):
    t_before = run.seq_len.clone()
    run.step(bench.step_seed(0, k))
    torch.cuda.synchronize()
    q = run.d.match_len.cpu().numpy(); dl = run.d.draft_len.cpu().numpy()
    nc = run.v.n_commit.cpu().numpy(); acc = run.v.accept_len.cpu().numpy()
    st = run.seq_tok.cpu().numpy(); tb = t_before.cpu().numpy()
    eq = []; 
    for s in range(run.n):
        tr = wl.truth[s]
        for i in range(nc[s]):
            pos = tb[s] + i
            eq.append(st[s, pos] == tr[min(pos, len(tr)-1)])
    # sampled root token vs head
    rows = run.d.row_offsets.cpu().numpy()
    smp = run.v.sampled.cpu().numpy()
    root_eq = np.mean([smp[rows[s]] == wl.truth[s][min(tb[s], len(wl.truth[s])-1)] for s in range(run.n)])
    print(f"step {k}: q hist {np.bincount(q, minlength=9).tolist()} draft mean {dl.mean():.1f} acc mean {acc.mean():.2f} commit==truth {np.mean(eq):.2f} root sample==truth {root_eq:.2f}")
