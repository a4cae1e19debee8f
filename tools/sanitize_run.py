"""compute-sanitizer driver (SURVEY §5.2 race / memory evidence): a few eager
steps of a small GRPO-shaped configuration (V = 151,936, 48 sequences, the
same kernels bench.py times: cursor draft, scan, fused accept + cursor insert,
hub refresh, walk insertion; then the same with the fused tree step
srt_verify_insert_draft_cursor), the tiny configuration, the LM-head fused
sampler, and a D = 128 multi-warp cursor insert with sibling spans.
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2601_09083_b200 as srt  # noqa: E402


def small(name, fused_step=False, **over):
    cfg = dict(bench.CONFIGS[name])
    cfg.update(over)
    wl = bench.Workload(cfg, 1)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 1)
    run.groups[0].fused_step = fused_step
    for k in range(3):
        run.step(bench.step_seed(1, k))
    torch.cuda.synchronize()
    bits, _ = run.status()
    print(f"[sanitize] {name} {cfg['active']} seqs{' (fused tree step)' if fused_step else ''}: "
          f"3 steps, error bits {bits}", flush=True)
    return run


small("grpo", prompts=6, active=48, cap=1024, act_cap=1024, median=300, node_capacity=1 << 20)
small("grpo", True, prompts=6, active=48, cap=1024, act_cap=1024, median=300,
      node_capacity=1 << 20)
small("tiny")
run = small("grpo", prompts=4, active=32, cap=512, act_cap=512, median=200, node_capacity=1 << 20)
run.enable_lmhead(256, 1)
for k in range(2):
    run.step(bench.step_seed(1, 10 + k))
torch.cuda.synchronize()
print(f"[sanitize] lmhead 2 steps, error bits {run.status()[0]}", flush=True)
# D = 128: one CTA of 4 warps per sequence, sibling spans of ~D positions
D, V, n = 128, 8, 32
c = srt.SrtCache(srt.config(V, 2, D, 8, 8, node_capacity=1 << 22))
rng = np.random.default_rng(0)
toks = torch.from_numpy(rng.integers(0, V, (n, 4 * D)).astype(np.int32)).cuda()
prompt = torch.from_numpy((np.arange(n) % 2).astype(np.int32)).cuda()
cur = c.new_cursors(n)
pos = torch.zeros(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    to = torch.clamp(pos + D - 4, max=4 * D)
    c.insert(prompt, toks, pos, to, cursor=cur)
    pos = to
torch.cuda.synchronize()
print(f"[sanitize] D=128 cursor inserts, error bits {c.status()[0]}", flush=True)
