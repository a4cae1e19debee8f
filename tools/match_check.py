"""Development check: does srt_draft's match length agree with a host-side
brute force on the bench workload (small prompt count, full V)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    prompts = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = dict(bench.CONFIGS["grpo"])
    cfg["prompts"] = prompts
    cfg["active"] = prompts * 8
    cfg["node_capacity"] = 1 << 24
    wl = bench.Workload(cfg, 0)
    run = bench.GpuRun(wl, "bf16", "rl-mix", 0)
    run.cache.draft(run.prompt_id, run.seq_tok, run.seq_len, run.seq_len, out=run.d)
    torch.cuda.synchronize()
    q = run.d.match_len.cpu().numpy()
    print("gpu q hist", np.bincount(q, minlength=9).tolist())
    # host brute force: largest q <= L with y[t-q:t] followed by some token in a
    # window of an inserted text (prior rollouts + the active prefixes)
    texts = {}
    for p, t in wl.w.prior:
        texts.setdefault(p, []).append(np.asarray(t))
    for s in range(len(wl.truth)):
        texts.setdefault(int(wl.seq_prompt[s]), []).append(np.asarray(wl.truth[s][:wl.t0[s]]))
    bad = 0
    for s in range(len(wl.truth)):
        p = int(wl.seq_prompt[s])
        t0 = int(wl.t0[s])
        y = wl.truth[s][:t0]
        best = 0
        for qq in range(1, min(cfg["L"], t0) + 1):
            suf = y[t0 - qq:]
            found = False
            for tx in texts[p]:
                n = len(tx)
                if n <= qq:
                    continue
                win = np.lib.stride_tricks.sliding_window_view(tx[:-1], qq)
                if np.any(np.all(win == suf, axis=1)):
                    found = True
                    break
            if found:
                best = qq
        if best != q[s]:
            bad += 1
            if bad <= 5:
                print(f"seq {s}: gpu q {q[s]} host q {best} (t0 {t0})")
    print("mismatches", bad, "of", len(wl.truth))


if __name__ == "__main__":
    main()
