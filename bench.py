"""bench.py — SRT draft + verify + insert step throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config grpo|tiny|ppo|dapo]
                    [--impl srt|reference] [--dtype bf16|f32] [--profile rl-mix|...]

One "step" = one pass of the whole hot path over one batch (BASELINE.json
north_star): srt_draft (match + best-first draft + layout) -> [forward
stand-in, NOT timed] -> srt_verify (Philox Gumbel-max scan of every drafted
row + first-mismatch walk + commit) -> srt_insert (commit spans into the
trees).  Inputs are seeded and synthetic (synth/ recipe) and
resident in HBM when the timed region starts; the logits buffer (10.3 GB for
GRPO bf16) is far larger than L2, so no flush is needed between steps.

Timing: CUDA events on the launching stream around the draft segment and the
verify+insert segment of every step (the forward stand-in between them is
excluded), barrier + synchronize on both sides, max over ranks.  Per-kernel
device times come from libsrt's own event pairs (srt_profile_*).
N > 1: prompts are hash-sharded (owner(p) = splitmix64(p) mod N) and each
rank decodes a contiguous block of 1024 sequences (weak scaling); every step
the owners' drafts go back to the decoding ranks (all-to-all of draft
records) and the committed spans go to the owners (NCCL all-gather of span
records) before insertion.
`--impl reference` times the CPU oracle on a bounded sample of the same
workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BJ:configs[0]
    "tiny": dict(V=1000, prompts=1, samples=8, active=4, Bmax=8, D=16, L=8, median=64, cap=64,
                 act_cap=256, prior_epochs=1, node_capacity=1 << 16),
    # BJ:configs[1] (headline)
    "grpo": dict(V=151936, prompts=128, samples=8, active=1024, Bmax=32, D=32, L=8, median=1200,
                 cap=8192, act_cap=8192, prior_epochs=1, node_capacity=1 << 27, hidden=1536),
    # BJ:configs[3]
    "ppo": dict(V=152064, prompts=256, samples=1, active=256, Bmax=64, D=128, L=16, median=1200,
                cap=4096, act_cap=4096, prior_epochs=3, node_capacity=1 << 28, hidden=3584),
    # BJ:configs[4] per rank: 8 ranks x 256 prompts x 16 samples = 2048 x 16, 4096
    # sequences decoded per rank, trees hash-sharded, span all-gather + draft
    # return every step (run with torchrun --nproc-per-node 8, or --sharded at N=1)
    "b200x8": dict(V=151936, prompts=256, samples=16, active=4096, Bmax=32, D=32, L=8,
                   median=1200, cap=8192, act_cap=8192, prior_epochs=1, node_capacity=1 << 29,
                   slot_capacity=1 << 29),
    # BJ:configs[2] (1024 of the 8192 sequences concurrently).  D = 16: the warm
    # cache (8192 prior rollouts, 57M tokens) has > 1.07B distinct windows at
    # D = 32 (measured: node capacity 2^30 overflowed during the warm-up); at
    # D = 16 it has 483M nodes, within 2^29
    "dapo": dict(V=151936, prompts=512, samples=16, active=1024, Bmax=32, D=16, L=8, median=3000,
                 cap=20000, act_cap=20000, prior_epochs=1, node_capacity=1 << 29,
                 slot_capacity=1 << 29,
                 # run-ahead generation: rollouts of the next 64 prompts (the
                 # look-ahead window) are inserted as spans of 512-2048 tokens, 8 per step
                 runahead=dict(first=64, prompts=64, per=4, spans=8, lo=512, hi=2048),
                 # measured: the fused tree step is slower here (16 sequences per prompt,
                 # deeper hubs: 316-326 us vs 270 us for the separate kernels)
                 fused_step=False),
}

KERNELS_PER_STEP = 9  # timed segments per group and step (an upper bound, for the profile buffer)
SEGMENT_KERNELS = {"scan": 2, "hub_refresh": 2, "tree_step": 2}  # segments of two kernels
                      # (+ insert_plan/walk of the run-ahead spans)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_tensor_peak():
    """Dense bf16 tensor peak: the driver's sustained cuBLAS measurement (the
    kernel runs inside a long step)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops_sustained"]), "measured (cuBLAS bf16, sustained)"
    except Exception:
        return 1400.0, "fallback (sustained)"


def lmhead_comparison(run, seed: int, args, reps: int = 5) -> dict:
    """The fused LM-head verify against the unfused pipeline it replaces, on
    the last step's drafted rows (state cloned, nothing committed): cuBLAS
    bf16 GEMM writing [rows, V] logits (torch.matmul) + srt_verify's HBM
    scan, versus srt_verify_lmhead.  Also a parity check: the fused kernel's
    debug dump of the logits it sampled from, re-sampled by srt_verify, must
    give the same tokens on every row."""
    torch = run.torch
    gr = run.groups[0]
    lm = gr.lm
    rows = int(gr.d.row_offsets[-1].item())
    H, W = lm["H"], lm["W"]
    logits = gr.logits[:rows]
    tok0, len0 = gr.seq_tok.clone(), gr.seq_len.clone()

    def clone_state():
        return tok0.clone(), len0.clone()

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = {"gemm": [], "scan": [], "fused": []}
    for _ in range(reps + 1):
        tk, ln = clone_state()
        ev[0].record()
        torch.matmul(H[:rows], W.T, out=logits)
        ev[1].record()
        gr.cache.verify(gr.logits, gr.d, gr.seq_id, seed, tk, ln, gr.max_new, out=gr.v,
                        rows=gr.rows_max)
        ev[2].record()
        tk, ln = clone_state()
        gr.cache.verify_lmhead(H, W, gr.d, gr.seq_id, seed, tk, ln, gr.max_new, out=gr.v,
                               rows=gr.rows_max)
        ev[3].record()
        torch.cuda.synchronize()
        t["gemm"].append(ev[0].elapsed_time(ev[1]))
        t["scan"].append(ev[1].elapsed_time(ev[2]))
        t["fused"].append(ev[2].elapsed_time(ev[3]))
    med = {k: float(np.median(v[1:])) for k, v in t.items()}
    # parity: the fused kernel's dumped logits through srt_verify
    tk, ln = clone_state()
    gr.cache.verify_lmhead(H, W, gr.d, gr.seq_id, seed, tk, ln, gr.max_new, out=gr.v,
                           rows=gr.rows_max, logits_out=gr.logits)
    fused_s = gr.v.sampled[:rows].clone()
    tk, ln = clone_state()
    gr.cache.verify(gr.logits, gr.d, gr.seq_id, seed, tk, ln, gr.max_new, out=gr.v,
                    rows=gr.rows_max)
    div = int((gr.v.sampled[:rows] != fused_s).sum().item())
    flops = 2.0 * rows * run.V * lm["K"]
    return {"rows": rows, "cublas_gemm_ms": med["gemm"], "srt_verify_ms": med["scan"],
            "unfused_ms": med["gemm"] + med["scan"], "fused_ms": med["fused"],
            "speedup": (med["gemm"] + med["scan"]) / med["fused"],
            "fused_tflops": flops / (med["fused"] / 1000) / 1e12,
            "cublas_tflops": flops / (med["gemm"] / 1000) / 1e12,
            "dump_rescan_divergent_rows": div,
            "note": "verify only (accept included, insert excluded), state cloned; median of "
                    f"{reps} after 1 warm-up"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # block until the sampler is live (its first line), so that a short
            # timed region still gets samples at the 20 ms cadence
            self.first = self.p.stdout.readline()
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
            if not self.lines and getattr(self, "first", "").strip():
                self.lines = [self.first]  # region shorter than one period: the sample at its start

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# the workload (seeded, synthetic)
# ---------------------------------------------------------------------------
def owned_prompts(rank: int, world: int, count: int):
    """Hash sharding: global prompt g is owned by splitmix64(g) mod world."""
    from paper_2601_09083_b200.dist import owner_of
    out, g = [], 0
    while len(out) < count:
        if owner_of(g, world) == rank:
            out.append(g)
        g += 1
    return out


class Workload:
    def __init__(self, cfg: dict, seed: int, rank: int = 0, world: int = 1, prompt_ids=None):
        from synth import make_workload
        self.cfg = cfg
        t = time.time()
        gp = list(prompt_ids) if prompt_ids is not None else owned_prompts(rank, world, cfg["prompts"])
        self.global_prompts = gp
        ra = cfg.get("runahead")
        w = make_workload(seed + 1000003 * gp[0], cfg["V"], cfg["prompts"], cfg["samples"],
                          cfg["median"], cfg["cap"], prior_epochs=cfg["prior_epochs"],
                          active=cfg["active"],
                          runahead=(ra["first"], ra["prompts"], ra["per"]) if ra else None)
        self.w = w
        rng = np.random.default_rng(seed + 7 + gp[0])
        # every active sequence starts part-way into its rollout (steady state):
        # t0 ~ U[0, len/2], its prefix already committed and inserted online
        self.truth = w.truth
        self.t0 = np.array([int(rng.integers(0, max(1, len(t) // 2))) for t in w.truth], np.int32)
        self.max_new = np.array([len(t) for t in w.truth], np.int32)
        self.seq_prompt = w.seq_prompt
        gpa = np.asarray(gp, np.uint64)
        self.seq_id = ((np.uint64(cfg["prior_epochs"]) << np.uint64(40))
                       | (gpa[w.seq_prompt].astype(np.uint64) << np.uint64(8))
                       | (np.arange(len(w.truth)) % cfg["samples"]).astype(np.uint64))
        log(f"[bench] workload: {len(w.prior)} prior rollouts ({sum(len(t) for _, t in w.prior)} "
            f"tokens), {len(w.truth)} active, generated in {time.time() - t:.1f}s")


class Group:
    """Device state of one prompt group: its own cache (the trees of the
    prompts p with p % G == g), sequence tables, draft/verify outputs and a
    slice of the shared logits buffer.  Groups share no tree, so their steps
    may run concurrently on different streams with results identical to one
    cache processing everything in order."""

    def __init__(self, wl: Workload, dtype: str, profile: str, seed: int, g: int, G: int,
                 logits, gaps, offs, row0: int):
        import torch
        import paper_2601_09083_b200 as srt
        self.torch = torch
        cfg = wl.cfg
        self.cfg = cfg
        dev = logits.device
        self.dev = dev
        seqs = np.nonzero(wl.seq_prompt % G == g)[0]
        self.seqs = seqs
        self.n = n = len(seqs)
        self.V, self.Bmax = V, B = cfg["V"], cfg["Bmax"]
        self.ldtype = logits.dtype
        n_prompts = len(range(g, cfg["prompts"], G))
        c = srt.config(V, n_prompts, cfg["D"], cfg["L"], B,
                       node_capacity=max(1 << 16, cfg["node_capacity"] // G),
                       slot_capacity=(max(1 << 16, cfg["slot_capacity"] // G)
                                      if "slot_capacity" in cfg else None),
                       logits_dtype=self.ldtype)
        self.cache = srt.SrtCache(c)
        # ---- warm trees: prior-epoch rollouts ("carries signal across steps")
        prior = [(p // G, tk) for p, tk in wl.w.prior if p % G == g]
        cap = cfg["cap"]
        chunk = 4096
        for i0 in range(0, len(prior), chunk):
            part = prior[i0:i0 + chunk]
            tab = np.zeros((len(part), cap), np.int32)
            for i, (_, tk) in enumerate(part):
                tab[i, :len(tk)] = tk
            self.cache.insert(torch.tensor([p for p, _ in part], dtype=torch.int32, device=dev),
                              torch.from_numpy(tab).to(dev),
                              torch.zeros(len(part), dtype=torch.int32, device=dev),
                              torch.tensor([len(tk) for _, tk in part], dtype=torch.int32, device=dev))
        # ---- active sequences: committed prefixes, inserted online
        stride = cfg["act_cap"] + B + 2
        tab = np.zeros((n, stride), np.int32)
        truth = np.zeros((n, cfg["act_cap"]), np.int32)
        for j, s in enumerate(seqs):
            tr = wl.truth[s]
            tab[j, :wl.t0[s]] = tr[:wl.t0[s]]
            truth[j, :len(tr)] = tr
            truth[j, len(tr):] = tr[-1]
        i32 = dict(dtype=torch.int32, device=dev)
        self.prompt_id = torch.from_numpy((wl.seq_prompt[seqs] // G).astype(np.int32)).to(dev)
        self.seq_tok = torch.from_numpy(tab).to(dev)
        self.seq_len = torch.from_numpy(wl.t0[seqs].copy()).to(dev)
        self.t_before = self.seq_len.clone()
        self.truth = torch.from_numpy(truth).to(dev)
        self.truth_last = torch.from_numpy(np.maximum(wl.max_new[seqs] - 1, 0)).to(dev).to(torch.int64)
        self.max_new = torch.from_numpy(wl.max_new[seqs].copy()).to(dev)
        self.seq_id = torch.from_numpy(wl.seq_id[seqs].view(np.int64)).to(dev)
        # per-sequence suffix cursors (srt_insert_cursor): one hop per window end
        self.cursor = self.cache.new_cursors(n, dev)
        self.cache.insert(self.prompt_id, self.seq_tok, torch.zeros(n, **i32), self.seq_len,
                          cursor=self.cursor)
        bits, st = self.cache.status()
        if bits:
            raise RuntimeError(f"cache error bits {bits} after warm-up inserts ({st})")
        self.tree_stats = st
        self.path_rounds = None  # srt_verify_path rounds (bench --verify path)
        self.fused = True  # srt_verify_insert_cursor (accept + cursor insert in one kernel)
        # srt_verify_insert_draft_cursor: commit + insert + hub refresh + the NEXT
        # draft in one persistent kernel (GpuRun sets it; D <= 32, full verify)
        self.fused_step = False
        self.need_draft = True  # no draft of the current step in self.d yet
        self.snap = None        # (row_offsets, draft_depth) of the last verified draft
        # ---- run-ahead spans (DAPO): a fixed schedule, uploaded once
        self.ra = None
        if wl.w.runahead and cfg.get("runahead"):
            if G != 1:
                raise ValueError("run-ahead spans need --groups 1")
            self.ra = runahead_schedule(wl.w.runahead, cfg["runahead"], cfg["cap"], seed, dev)
            self.ra_k = torch.zeros(1, dtype=torch.int64, device=dev)
            self.ra_cur = torch.zeros(2, self.ra["frm"].shape[1], dtype=torch.int32, device=dev)
        # ---- this group's rows of the logits buffer: rows_max + 1 dummy row
        self.rows_max = n * (B + 1)
        self.logits = logits[row0:row0 + self.rows_max + 1]
        self.gaps = gaps[row0:row0 + self.rows_max + 1]
        self.offs = offs[row0:row0 + self.rows_max + 1]
        self.profile = profile
        self.flat_logits = self.logits.view(-1)
        self.lm = None  # --verify lmhead: hidden states + LM-head weight (GpuRun.enable_lmhead)
        self.d = srt.DraftOut.empty(n, B, dev)
        self.v = srt.VerifyOut.empty(n, self.rows_max, B, dev)
        self.slot = torch.arange(B + 1, device=dev, dtype=torch.int64)
        # stand-in edits of the previous step (static buffers: restored in place)
        self.mod_idx = torch.zeros(n * (B + 1) * 4, dtype=torch.int64, device=dev)
        self.mod_val = self.flat_logits[self.mod_idx].clone()

    # ---- forward stand-in (NOT part of the SRT path) -----------------------
    def standin(self):
        """Write each drafted row's head logit: the policy's preferred next
        token is the ground-truth token at that row's position (the rollout
        re-joins its template after a divergence), bulk mean 0, gap from the
        row's profile, 3 distractors below it.  Previous step's edits are
        restored first.  Also snapshots seq_len (the insert span start)."""
        torch = self.torch
        if self.profile == "flat":
            self.t_before.copy_(self.seq_len)
            return
        d, n, B, V = self.d, self.n, self.Bmax, self.V
        self.flat_logits[self.mod_idx] = self.mod_val
        depth = torch.cat([torch.zeros(n, 1, dtype=torch.int32, device=self.dev), d.draft_depth],
                          dim=1).to(torch.int64)                                   # [n, B+1]
        pos = self.seq_len.to(torch.int64)[:, None] + depth
        pos = torch.minimum(pos, self.truth_last[:, None])
        head = torch.gather(self.truth, 1, pos).to(torch.int64)                    # [n, B+1]
        valid = self.slot[None, :] <= d.draft_len.to(torch.int64)[:, None]
        row = d.row_offsets[:-1, None] + self.slot[None, :]
        row = torch.where(valid, row, torch.full_like(row, self.rows_max))         # dummy row
        gap = self.gaps[row]
        off = self.offs[row]  # [n, B+1, 3]
        idx = [row * V + head]
        val = [gap]
        for k in range(3):
            idx.append(row * V + (head + 1 + 7919 * (k + 1) + row * 31) % V)
            val.append(gap - off[..., k])
        idx = torch.stack(idx, -1).reshape(-1)
        val = torch.stack(val, -1).reshape(-1).to(self.ldtype)
        self.mod_idx.copy_(idx)
        self.mod_val.copy_(self.flat_logits[idx])
        self.flat_logits[idx] = val
        self.t_before.copy_(self.seq_len)

    def standin_lmhead(self):
        """The forward stand-in of --verify lmhead: each drafted row's final
        hidden state h_r = z_r + gap_r W[head_r] + sum_k (gap_r - off_rk) W[d_rk]
        with z_r ~ N(0, 2^2 I) (fixed per row) and W ~ N(0, 1/K): the LM head
        then yields bulk logits ~ N(0, 2^2), the head at ~gap and 3 distractors
        below it -- the rl-mix rows of the logits stand-in, produced by the GEMM."""
        torch = self.torch
        lm, d, n, B, V = self.lm, self.d, self.n, self.Bmax, self.V
        depth = torch.cat([torch.zeros(n, 1, dtype=torch.int32, device=self.dev), d.draft_depth],
                          dim=1).to(torch.int64)
        pos = torch.minimum(self.seq_len.to(torch.int64)[:, None] + depth, self.truth_last[:, None])
        head = torch.gather(self.truth, 1, pos).to(torch.int64).reshape(-1)
        valid = (self.slot[None, :] <= d.draft_len.to(torch.int64)[:, None]).reshape(-1)
        row = (d.row_offsets[:-1, None] + self.slot[None, :]).reshape(-1)
        row = torch.where(valid, row, torch.full_like(row, self.rows_max))
        gap = torch.where(valid, self.gaps[row], torch.zeros_like(self.gaps[row]))
        W = lm["W"]
        h = lm["Z"][row].float() + gap[:, None] * W[head].float()
        off = self.offs[row]
        for k in range(3):
            dk = (head + 1 + 7919 * (k + 1) + row * 31) % V
            h += torch.where(valid, gap - off[:, k], torch.zeros_like(gap))[:, None] * W[dk].float()
        lm["H"][row] = h.to(torch.bfloat16)
        self.t_before.copy_(self.seq_len)

    def draft(self):
        self.cache.draft(self.prompt_id, self.seq_tok, self.seq_len, self.seq_len, out=self.d,
                         cursor=self.cursor)
        self.need_draft = False

    def draft_if_needed(self):
        """The fused step drafted this step already (inside the previous
        verify); otherwise srt_draft_cursor."""
        if not (self.fused_step and not self.need_draft):
            self.draft()

    def snapshot_layout(self):
        """Keep the verified draft's row layout (the fused step overwrites
        self.d with the next draft; the parity sample maps rows to positions)."""
        self.snap = (self.d.row_offsets.clone(), self.d.draft_depth.clone())

    def verify_insert(self, seed: int, logits=None):
        c = self.cache
        lg = self.logits if logits is None else logits
        if (self.fused_step and self.lm is None and self.path_rounds is None
                and self.cache.cfg.max_depth <= 128):
            # run-ahead spans target look-ahead prompts (no active sequence's
            # tree); inserts commute (O14), so they go first and the next draft,
            # inside the fused call, sees them as it would after the unfused step
            if self.ra is not None:
                self.runahead_insert()
            c.verify_insert_draft(lg, self.d, self.seq_id, seed, self.seq_tok, self.seq_len,
                                  self.max_new, self.prompt_id, self.cursor, pos_base=self.seq_len,
                                  next_d=self.d, out=self.v, rows=self.rows_max)
            self.need_draft = False
            return
        self.need_draft = True
        if self.lm is not None and logits is None:  # the LM head fused into the sampler
            c.verify_lmhead(self.lm["H"], self.lm["W"], self.d, self.seq_id, seed, self.seq_tok,
                            self.seq_len, self.max_new, prompt_id=self.prompt_id,
                            cursor=self.cursor, out=self.v, rows=self.rows_max)
        elif self.fused and self.path_rounds is None:
            c.verify_insert(lg, self.d, self.seq_id, seed, self.seq_tok, self.seq_len, self.max_new,
                            self.prompt_id, self.cursor, out=self.v, rows=self.rows_max)
        else:
            c.verify(lg, self.d, self.seq_id, seed, self.seq_tok, self.seq_len, self.max_new,
                     out=self.v, rows=self.rows_max, path_rounds=self.path_rounds)
            c.insert(self.prompt_id, self.seq_tok, self.t_before, self.seq_len, cursor=self.cursor)
        if self.ra is not None:
            self.runahead_insert()

    def runahead_inserted(self):
        """Host view: tokens of each look-ahead rollout inserted so far."""
        ra = self.ra
        k = min(int(self.ra_k.item()), ra["frm"].shape[0]) - 1
        return ra["to_host"][k] if k >= 0 else np.zeros(len(ra["prompt_host"]), np.int32)

    def runahead_insert(self):
        """This step's run-ahead spans: [frm, to) of each look-ahead rollout
        (empty for the rollouts not scheduled this step), walk insertion.  The
        step index lives on the device, so the step can be a CUDA graph."""
        torch = self.torch
        ra = self.ra
        k = torch.clamp(self.ra_k, max=ra["frm"].shape[0] - 1)  # past the schedule: empty spans
        torch.index_select(ra["frm"], 0, k, out=self.ra_cur[0:1])
        torch.index_select(ra["to"], 0, k, out=self.ra_cur[1:2])
        self.cache.insert(ra["prompt"], ra["tok"], self.ra_cur[0], self.ra_cur[1])
        self.ra_k += 1


def runahead_schedule(streams, rc: dict, cap: int, seed: int, dev, steps: int = 512):
    """Run-ahead spans for `steps` steps: each step the next rc["spans"]
    unfinished look-ahead rollouts (round robin) advance by U[lo, hi] tokens.
    Row k of frm/to holds every rollout's span of step k (empty = not
    scheduled); after the rollouts run out every span is empty."""
    import torch
    R = len(streams)
    lens = np.array([len(t) for _, t in streams], np.int64)
    tab = np.zeros((R, cap), np.int32)
    for i, (_, t) in enumerate(streams):
        tab[i, :len(t)] = t
    rng = np.random.default_rng(seed + 99991)
    pos = np.zeros(R, np.int64)
    frm = np.zeros((steps + 1, R), np.int32)  # the last row: all empty
    to = np.zeros((steps + 1, R), np.int32)
    ptr = 0
    for k in range(steps):
        nxt = pos.copy()
        picked = tries = 0
        while picked < rc["spans"] and tries < R:
            r = ptr % R
            ptr += 1
            tries += 1
            if pos[r] >= lens[r]:
                continue
            nxt[r] = min(lens[r], pos[r] + int(rng.integers(rc["lo"], rc["hi"] + 1)))
            picked += 1
        frm[k], to[k] = pos, nxt
        pos = nxt
    frm[steps], to[steps] = pos, pos
    prompt = np.array([p for p, _ in streams], np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    return {"tok": t(tab), "prompt": t(prompt), "frm": t(frm), "to": t(to),
            "frm_host": frm, "to_host": to, "tok_host": tab, "prompt_host": prompt}


class GpuRun:
    """Device state for one rank: G prompt groups (each its own cache and
    stream) over one shared logits buffer."""

    def __init__(self, wl: Workload, dtype: str, profile: str, seed: int, groups: int = 1):
        import torch
        self.torch = torch
        cfg = wl.cfg
        self.cfg = cfg
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.n = n = cfg["active"]
        self.V, self.Bmax = V, B = cfg["V"], cfg["Bmax"]
        self.ldtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        t = time.time()
        G = max(1, min(groups, cfg["prompts"]))
        self.G = G
        # ---- logits buffer: every group's rows_max + 1 dummy row, bulk N(0, 2^2)
        counts = [int(np.sum(wl.seq_prompt % G == g)) for g in range(G)]
        total_rows = sum(c * (B + 1) + 1 for c in counts)
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.logits = torch.empty(total_rows, V, dtype=self.ldtype, device=dev)
        step = 2048
        for r0 in range(0, total_rows, step):
            r1 = min(total_rows, r0 + step)
            if profile == "flat":
                self.logits[r0:r1].uniform_(0, 1, generator=gen)
            else:
                self.logits[r0:r1].normal_(0.0, 2.0, generator=gen)
        rg = np.random.default_rng(seed + 3)
        from synth import head_profile
        gaps, offs = head_profile(rg, total_rows, profile if profile != "flat" else "moderate")
        gaps = torch.from_numpy(gaps.astype(np.float32)).to(dev)
        offs = torch.from_numpy(offs.astype(np.float32)).to(dev)  # [rows, 3]
        self.groups = []
        row0 = 0
        for g in range(G):
            self.groups.append(Group(wl, dtype, profile, seed, g, G, self.logits, gaps, offs, row0))
            row0 += counts[g] * (B + 1) + 1
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(G)]
        self.rows_max = sum(gr.rows_max for gr in self.groups)
        torch.cuda.synchronize()
        self.tree_stats = {k: sum(gr.tree_stats[k] for gr in self.groups)
                           for k in self.groups[0].tree_stats}
        log(f"[bench] device setup {time.time() - t:.1f}s; {G} group(s); tree nodes "
            f"{self.tree_stats['nodes_used']:,} (cap {self.tree_stats['node_capacity']:,}); logits "
            f"{self.logits.numel() * self.logits.element_size() / 1e9:.2f} GB")

    def enable_lmhead(self, K: int, seed: int):
        """--verify lmhead: a bf16 LM-head weight [V, K] (random init of the
        configuration's shape, W ~ N(0, 1/K)) and per-row hidden states; the
        logits buffer is then used only by the unfused comparison."""
        torch = self.torch
        gen = torch.Generator(device=self.dev)
        gen.manual_seed(seed + 4242)
        W = torch.empty(self.V, K, dtype=torch.bfloat16, device=self.dev)
        for v0 in range(0, self.V, 16384):
            W[v0:v0 + 16384].normal_(0.0, 1.0 / K ** 0.5, generator=gen)
        for gr in self.groups:
            Z = torch.empty(gr.rows_max + 1, K, dtype=torch.bfloat16, device=self.dev)
            Z.normal_(0.0, 2.0, generator=gen)
            gr.lm = {"W": W, "Z": Z, "H": Z.clone(), "K": K}
            gr.standin = gr.standin_lmhead
        self.lm_K = K

    def __getattr__(self, name):
        # single-group convenience for the development probes (tools/)
        groups = self.__dict__.get("groups")
        if groups is not None and len(groups) == 1:
            return getattr(groups[0], name)
        raise AttributeError(name)

    def step(self, seed: int, ev=None, rows_out=None):
        """Sequential step on the current stream: draft -> [stand-in] ->
        verify -> insert for every group (with --fused-step the draft of this
        step was made by the previous step's fused call).  ev = 4 CUDA events
        bracketing the draft segment and the verify+insert segment (stand-in
        excluded); rows_out (1-element device tensor) <- this step's rows."""
        if ev:
            ev[0].record()
        for gr in self.groups:
            gr.draft_if_needed()
        if ev:
            ev[1].record()
        for gr in self.groups:
            gr.standin()
        if rows_out is not None:
            rows_out.copy_(sum(gr.d.row_offsets[-1:] for gr in self.groups))
        for gr in self.groups:
            if gr.fused_step:
                gr.snapshot_layout()  # (the fused call overwrites self.d with the next draft)
        if ev:
            ev[2].record()
        for gr in self.groups:
            gr.verify_insert(seed)
        if ev:
            ev[3].record()

    def step_pipelined(self, seed: int):
        """One step of every group, each on its own stream, no host sync:
        verify+insert of one group overlap the draft / stand-in of the next
        and the HBM-bound scans of the others.  Stand-in included."""
        torch = self.torch
        for gr, st in zip(self.groups, self.streams):
            with torch.cuda.stream(st):
                gr.draft()
                gr.standin()
                gr.verify_insert(seed)

    def status(self):
        bits, tot = 0, None
        for gr in self.groups:
            b, st = gr.cache.status()
            bits |= b
            tot = st if tot is None else {k: tot[k] + st[k] for k in tot}
        return bits, tot


class ShardedRun:
    """One rank of the hash-sharded multi-GPU step (SURVEY
    §8(e)): global prompt blocks of cfg["prompts"] prompts, block b decoded by
    rank b (contiguous, prompt-major); prompt p's tree on owner(p) =
    splitmix64(p) mod G with a mirror of its sequences; drafts returned and
    committed spans sent to the owners by NCCL all-gathers every step."""

    def __init__(self, cfg: dict, seed: int, rank: int, world: int, dtype: str, profile: str,
                 gather=None):
        import torch
        import paper_2601_09083_b200 as srt
        from paper_2601_09083_b200.dist import (GpuOps, ShardPlan, ShardedStep, all_gather_rows,
                                                 all_to_all_rows)
        self.torch = torch
        self.cfg = cfg
        t = time.time()
        npb = cfg["prompts"]
        blocks = [Workload(cfg, seed, prompt_ids=range(b * npb, (b + 1) * npb)) for b in range(world)]
        S_b = cfg["active"]
        seq_prompt = np.concatenate([b.seq_prompt.astype(np.int64) + i * npb
                                     for i, b in enumerate(blocks)])
        plan = ShardPlan.build(seq_prompt, world)
        self.plan = plan
        assert all(len(plan.local[r]) == S_b for r in range(world))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        V, B = cfg["V"], cfg["Bmax"]
        self.V, self.Bmax = V, B
        self.ldtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        i32 = dict(dtype=torch.int32, device=dev)

        def seq_data(g):  # global sequence g -> (block, index in block)
            return blocks[g // S_b], g % S_b

        # ---- owner side: trees of the owned prompts + mirror of their sequences
        owned = plan.prompts[rank]
        c = srt.config(V, max(1, len(owned)), cfg["D"], cfg["L"], B,
                       node_capacity=cfg["node_capacity"], logits_dtype=self.ldtype)
        self.cache = srt.SrtCache(c)
        cap = cfg["cap"]
        prior = [(int(np.searchsorted(owned, b * npb + p)), tk)
                 for b, blk in enumerate(blocks) for p, tk in blk.w.prior
                 if owner_of_global(b * npb + p, world) == rank]
        for i0 in range(0, len(prior), 4096):
            part = prior[i0:i0 + 4096]
            tab = np.zeros((len(part), cap), np.int32)
            for i, (_, tk) in enumerate(part):
                tab[i, :len(tk)] = tk
            self.cache.insert(torch.tensor([p for p, _ in part], **i32), torch.from_numpy(tab).to(dev),
                              torch.zeros(len(part), **i32),
                              torch.tensor([len(tk) for _, tk in part], **i32))
        stride = cfg["act_cap"] + B + 2
        mirror = plan.mirror[rank]
        nm = len(mirror)
        mtab = np.zeros((max(1, nm), stride), np.int32)
        mlen = np.zeros(max(1, nm), np.int32)
        for j, g in enumerate(mirror):
            blk, i = seq_data(g)
            mtab[j, :blk.t0[i]] = blk.truth[i][:blk.t0[i]]
            mlen[j] = blk.t0[i]
        self.m_tok = torch.from_numpy(mtab[:nm]).to(dev)
        self.m_len = torch.from_numpy(mlen[:nm]).to(dev)
        self.m_prompt = torch.from_numpy(plan.mirror_prompt[rank]).to(dev)
        self.m_cursor = self.cache.new_cursors(nm, dev)
        self.m_draft = srt.DraftOut.empty(nm, B, dev)
        if nm:
            self.cache.insert(self.m_prompt, self.m_tok, torch.zeros(nm, **i32), self.m_len,
                              cursor=self.m_cursor)
        # ---- decode side: the local block's sequences (same layout as Group)
        blk = blocks[rank]
        n = S_b
        self.n = n
        tab = np.zeros((n, stride), np.int32)
        truth = np.zeros((n, cfg["act_cap"]), np.int32)
        for j in range(n):
            tr = blk.truth[j]
            tab[j, :blk.t0[j]] = tr[:blk.t0[j]]
            truth[j, :len(tr)] = tr
            truth[j, len(tr):] = tr[-1]
        self.seq_tok = torch.from_numpy(tab).to(dev)
        self.seq_len = torch.from_numpy(blk.t0.copy()).to(dev)
        self.t_before = self.seq_len.clone()
        self.truth = torch.from_numpy(truth).to(dev)
        self.truth_last = torch.from_numpy(np.maximum(blk.max_new - 1, 0)).to(dev).to(torch.int64)
        self.max_new = torch.from_numpy(blk.max_new).to(dev)
        self.seq_id = torch.from_numpy(blk.seq_id.view(np.int64)).to(dev)
        self.rows_max = n * (B + 1)
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed + rank)
        self.logits = torch.empty(self.rows_max + 1, V, dtype=self.ldtype, device=dev)
        for r0 in range(0, self.rows_max + 1, 2048):
            r1 = min(self.rows_max + 1, r0 + 2048)
            if profile == "flat":
                self.logits[r0:r1].uniform_(0, 1, generator=gen)
            else:
                self.logits[r0:r1].normal_(0.0, 2.0, generator=gen)
        from synth import head_profile
        gaps, offs = head_profile(np.random.default_rng(seed + 3 + rank), self.rows_max + 1,
                                  profile if profile != "flat" else "moderate")
        self.gaps = torch.from_numpy(gaps.astype(np.float32)).to(dev)
        self.offs = torch.from_numpy(offs.astype(np.float32)).to(dev)
        self.profile = profile
        self.flat_logits = self.logits.view(-1)
        self.lm = None  # --verify lmhead: hidden states + LM-head weight (GpuRun.enable_lmhead)
        self.d = srt.DraftOut.empty(n, B, dev)
        self.v = srt.VerifyOut.empty(n, self.rows_max, B, dev)
        self.slot = torch.arange(B + 1, device=dev, dtype=torch.int64)
        self.mod_idx = torch.zeros(n * (B + 1) * 4, dtype=torch.int64, device=dev)
        self.mod_val = self.flat_logits[self.mod_idx].clone()
        # ---- the exchange
        ops = GpuOps(self.cache, B, self.m_prompt, self.m_tok, self.m_len, self.m_cursor,
                     self.m_draft, self.d, self.seq_len, self.v)
        a2a = ((lambda t, sc, rc: t[:int(sum(sc))]) if world == 1 and gather is not None
               else all_to_all_rows)
        self.ex = ShardedStep(plan, rank, ops, gather or all_gather_rows, B, device=dev, a2a=a2a)
        bits, st = self.cache.status()
        if bits:
            raise RuntimeError(f"cache error bits {bits} after warm-up inserts ({st})")
        self.tree_stats = st
        torch.cuda.synchronize()
        log(f"[bench] rank {rank}/{world}: {len(owned)} owned prompts, {nm} mirror / {n} local "
            f"sequences, tree nodes {st['nodes_used']:,}; setup {time.time() - t:.1f}s")

    standin = Group.standin

    def draft(self):
        self.ex.draft()

    def verify_insert(self, seed: int, logits=None):
        self.cache.verify(self.logits if logits is None else logits, self.d, self.seq_id, seed,
                          self.seq_tok, self.seq_len, self.max_new, out=self.v, rows=self.rows_max)
        self.ex.commit()

    fused_step = False  # (the fused tree step needs verify and insert on one cache)
    snap = None
    ra = None  # (no run-ahead spans in the sharded configuration)

    def draft_if_needed(self):
        self.draft()

    def snapshot_layout(self):
        self.snap = (self.d.row_offsets.clone(), self.d.draft_depth.clone())

    def step(self, seed: int, ev=None, rows_out=None):
        """draft (owner) -> draft return -> [stand-in] -> verify -> span
        all-gather -> owner insert.  ev = 4 events (stand-in excluded);
        rows_out (1-element device tensor) <- this step's rows."""
        if ev:
            ev[0].record()
        self.draft()
        if ev:
            ev[1].record()
        self.standin()
        if rows_out is not None:
            rows_out.copy_(self.d.row_offsets[-1:])
        if ev:
            ev[2].record()
        self.verify_insert(seed)
        if ev:
            ev[3].record()

    @property
    def groups(self):
        return [self]

    def status(self):
        return self.cache.status()


def spawn_ranks(n: int) -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    log(f"[bench] spawning {n} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def owner_of_global(p: int, world: int) -> int:
    from paper_2601_09083_b200.dist import owner_of
    return owner_of(p, world)


def step_seed(run_seed: int, k: int) -> int:
    from synth import splitmix64
    return splitmix64(run_seed ^ k)


# ---------------------------------------------------------------------------
# CPU oracle on a bounded sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_sample_steps(wl: Workload, dtype: str, steps: int, n_prompts_sample: int, seed: int,
                        bulk_rows=None):
    """Run the oracle's draft -> verify -> insert for the sequences of the
    first n_prompts_sample prompts, `steps` steps; returns (seconds per step,
    sequences in the sample, accepted per step)."""
    import oracle
    from synth import bf16_bits
    cfg = wl.cfg
    V, B = cfg["V"], cfg["Bmax"]
    o = oracle.Oracle(V, cfg["prompts"], cfg["D"], cfg["L"], B)
    keep = [i for i, (p, _) in enumerate(wl.w.prior) if p < n_prompts_sample]
    cap = cfg["cap"]
    tab = np.zeros((len(keep), cap), np.int32)
    for j, i in enumerate(keep):
        tab[j, :len(wl.w.prior[i][1])] = wl.w.prior[i][1]
    o.insert([wl.w.prior[i][0] for i in keep], tab, [0] * len(keep),
             [len(wl.w.prior[i][1]) for i in keep])
    seqs = [s for s in range(len(wl.truth)) if wl.seq_prompt[s] < n_prompts_sample]
    n = len(seqs)
    stride = cfg["act_cap"] + B + 2
    seq_tok = np.zeros((n, stride), np.int32)
    for j, s in enumerate(seqs):
        seq_tok[j, :wl.t0[s]] = wl.truth[s][:wl.t0[s]]
    seq_len = wl.t0[seqs].copy()
    prompt = wl.seq_prompt[seqs].astype(np.int32)
    o.insert(prompt, seq_tok, np.zeros(n, np.int32), seq_len)
    rng = np.random.default_rng(seed)
    total = 0.0
    acc = 0
    for k in range(steps):
        t_a = time.perf_counter()
        d = o.draft(prompt, seq_tok, seq_len, seq_len)
        t_b = time.perf_counter()
        rows = int(d["row_offsets"][-1])
        # forward stand-in (untimed): bulk N(0,4) rows, head = truth at the row's position
        if bulk_rows is not None and bulk_rows.shape[0] >= rows:
            x = bulk_rows[:rows].astype(np.float32)
        else:
            x = rng.normal(0, 2, (rows, V)).astype(np.float32)
        for j, s in enumerate(seqs):
            r0 = d["row_offsets"][j]
            tr = wl.truth[s]
            for i in range(d["draft_len"][j] + 1):
                dep = 0 if i == 0 else d["draft_depth"][j, i - 1]
                x[r0 + i, tr[min(seq_len[j] + dep, len(tr) - 1)]] = 20.0
        host = bf16_bits(x) if dtype == "bf16" else x
        t_c = time.perf_counter()
        t0 = seq_len.copy()
        v = o.verify(host, d["row_offsets"], d["draft_len"], d["draft_tok"], d["draft_parent"],
                     d["draft_depth"], wl.seq_id[seqs], step_seed(seed, 0), seq_tok, seq_len,
                     wl.max_new[seqs])
        o.insert(prompt, seq_tok, t0, seq_len)
        t_d = time.perf_counter()
        total += (t_b - t_a) + (t_d - t_c)
        acc += int(v["accept_len"].sum())
    return total / steps, n, acc / steps


def cpu_cores_used(n_units: int) -> int:
    return max(1, min(int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), n_units))


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="grpo", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="srt", choices=["srt", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--profile", default="rl-mix", choices=["rl-mix", "peaked", "moderate", "flat"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-prompts", type=int, default=0, help="oracle sample size in prompts")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--parity-rows", type=int, default=1024,
                    help="rows of the last timed step the oracle re-samples after the run "
                         "(tie-break divergence count; 0 = off)")
    ap.add_argument("--sharded", action="store_true",
                    help="N=1: run the multi-GPU exchange path (owner draft, draft return, span "
                         "all-gather) on one rank")
    ap.add_argument("--verify", default="full", choices=["full", "path", "lmhead"],
                    help="full = srt_verify (every draft row sampled, the headline); path = "
                         "srt_verify_path (only the accepted path's rows, SURVEY f3b); lmhead = "
                         "srt_verify_lmhead_insert_cursor (the LM-head GEMM fused with the "
                         "sampler, SURVEY f3a: the step then includes the LM head)")
    ap.add_argument("--path-rounds", type=int, default=3)
    ap.add_argument("--fused-step", type=int, default=-1,
                    help="1: srt_verify_insert_draft_cursor (commit + insert + hub refresh + the "
                         "next draft in one persistent kernel; D <= 128, --verify full, 1 group); "
                         "0: the separate kernels; -1: the configuration's measured choice")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: each step's draft segment and verify+insert segment replay as CUDA "
                         "graphs (no launch gaps); the per-kernel breakdown then comes from a "
                         "separate profiled eager pass")
    ap.add_argument("--step-overlap", type=int, default=-1,
                    help="SMs the fused tree step runs on BESIDE the scan (srt_cache_set_step_overlap; "
                         "0 = after the scan on every SM, -1 = the library's default)")
    ap.add_argument("--groups", type=int, default=1,
                    help="prompt groups pipelined on separate streams (1 = sequential; >1 measured slower: the latency-bound tree kernels stall behind the scan's HBM traffic)")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-run this command under
        # torchrun, one process per GPU (rank 0 prints the JSON line)
        sys.exit(spawn_ranks(args.gpus))
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "draft+verify+insert steps/sec"
    workload = f"{args.config}:{cfg['prompts']}x{cfg['samples']} prompts x samples, " \
               f"{cfg['active']} active seqs, V={cfg['V']}, Bmax={cfg['Bmax']}, D={cfg['D']}, L={cfg['L']}"

    if args.impl == "reference":
        if rank != 0:
            return
        wl = Workload(cfg, args.seed)
        npr = args.cpu_prompts or max(1, min(cfg["prompts"], 64 // cfg["samples"]))
        oracle_sample_steps(wl, args.dtype, 1, npr, args.seed)  # warm
        t_wall = time.perf_counter()
        t_step, n_s, acc = oracle_sample_steps(wl, args.dtype, max(1, args.steps), npr, args.seed)
        t_wall = time.perf_counter() - t_wall
        frac = n_s / cfg["active"]
        value = frac / t_step
        cores = cpu_cores_used(n_s)
        sample = (f"{n_s} of {cfg['active']} sequences ({npr} prompts) per step, full V rows; "
                  f"value = (sample steps/s) x {n_s}/{cfg['active']}, i.e. extrapolated "
                  f"linearly in sequences; the sample's measured oracle time is "
                  f"{t_step:.2f} s per step ({t_wall:.1f} s wall for {max(1, args.steps)} "
                  f"steps incl. the untimed forward stand-in)")
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": workload, "profile": args.profile},
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "sample_s_per_step": t_step,
                             "sample_wall_s": t_wall, "extrapolated": True},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }), flush=True)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_2601_09083_b200 import build
    if rank == 0 or world == 1:
        build.build()
    if world > 1:
        dist.barrier()
    if world > 1 or args.sharded:
        # hash-sharded trees + draft return / span all-gather
        run = ShardedRun(cfg, args.seed, rank, world, args.dtype, args.profile,
                         gather=None if world > 1 else (lambda t: t))
        wl = None
        G = 1
    else:
        wl = Workload(cfg, args.seed, rank, world)
        run = GpuRun(wl, args.dtype, args.profile, args.seed + rank, groups=args.groups)
        if args.verify == "path":
            for gr in run.groups:
                gr.path_rounds = args.path_rounds
        if args.verify == "lmhead":
            run.enable_lmhead(cfg.get("hidden", 1536), args.seed)
        G = run.G
        fused = cfg.get("fused_step", True) if args.fused_step < 0 else bool(args.fused_step)
        if fused and args.verify == "full" and cfg["D"] <= 128 and G == 1:
            for gr in run.groups:
                gr.fused_step = True
                if args.step_overlap >= 0:
                    gr.cache.set_step_overlap(args.step_overlap)
    pipelined = G > 1
    K, W = args.steps, args.warmup
    seed = step_seed(args.seed, 0)
    for k in range(W):
        if pipelined:
            run.step_pipelined(seed)
        else:
            run.step(seed)
        if os.environ.get("BENCH_ROWS_LOG"):  # profiling support: rows of each warm-up scan
            log(f"[bench] warm-up step {k}: rows "
                f"{[int(gr.d.row_offsets[-1].item()) for gr in run.groups]}")
    torch.cuda.synchronize()
    bits, _ = run.status()
    if bits:
        raise RuntimeError(f"device error bits {bits} during warm-up")
    # ---- timed region
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows_log = torch.zeros(K, dtype=torch.int64, device=run.dev)
    smp_log = torch.zeros(K, dtype=torch.int64, device=run.dev)
    acc_log = torch.zeros(K, dtype=torch.int64, device=run.dev)
    com_log = torch.zeros(K, dtype=torch.int64, device=run.dev)
    logs = [torch.zeros(3, K, dtype=torch.int64, device=run.dev) for _ in range(G)]
    use_graph = bool(args.graph) and not pipelined and G == 1
    step_prof = []
    if use_graph:
        # capture one step's two segments (the stand-in stays eager between
        # them); the sharded path's segments include its NCCL collectives
        gr0 = run.groups[0]
        try:
            g_draft, g_vi = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            if not gr0.fused_step:  # (fused: the previous step's call drafts this one)
                with torch.cuda.graph(g_draft):
                    gr0.draft()
            with torch.cuda.graph(g_vi):
                gr0.verify_insert(seed)
            for _ in range(2):  # graph warm-up steps
                if not gr0.fused_step:
                    g_draft.replay()
                gr0.standin()
                g_vi.replay()
            torch.cuda.synchronize()
        except Exception as e:  # capture unsupported here: time the eager step instead
            log(f"[bench] CUDA-graph capture failed ({e!r}); timing eager steps")
            use_graph = False
            torch.cuda.synchronize()
    if not use_graph:
        for gr in run.groups:
            gr.cache.profile_enable(K * KERNELS_PER_STEP)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        if pipelined:
            # every group on its own stream, no host sync inside the region;
            # the forward stand-in and the bookkeeping are INSIDE the timing
            ev_a.record()
            for st in run.streams:
                st.wait_event(ev_a)
            for k in range(K):
                for g, (gr, st) in enumerate(zip(run.groups, run.streams)):
                    with torch.cuda.stream(st):
                        gr.draft()
                        gr.standin()
                        gr.verify_insert(seed)
                        logs[g][0, k] = gr.d.row_offsets[-1]
                        logs[g][1, k] = gr.v.accept_len.sum()
                        logs[g][2, k] = gr.v.n_commit.sum()
            for st in run.streams:
                torch.cuda.current_stream().wait_stream(st)
            ev_b.record()
        else:
            for k in range(K):
                if use_graph:
                    e = evs[k]
                    e[0].record()
                    if not gr0.fused_step:  # (fused: the previous step drafted this one)
                        g_draft.replay()
                    e[1].record()
                    gr0.standin()
                    rows_log[k] = gr0.d.row_offsets[-1]  # (outside the timed segments)
                    if k == K - 1:
                        gr0.snapshot_layout()
                    e[2].record()
                    g_vi.replay()
                    e[3].record()
                else:
                    run.step(seed, evs[k], rows_out=rows_log[k:k + 1])
                # bookkeeping outside the event-bracketed segments
                if args.verify == "path":  # rows srt_verify_path actually sampled
                    nr = run.d.row_offsets[-1]
                    smp_log[k] = ((run.v.sampled[:run.rows_max] >= 0)
                                  & (torch.arange(run.rows_max, device=run.dev) < nr)).sum()
                acc_log[k] = run.v.accept_len.sum()
                com_log[k] = run.v.n_commit.sum()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    psample = None
    if not pipelined and rank == 0 and args.parity_rows > 0 and args.verify != "lmhead":
        psample = capture_parity_sample(run, args.parity_rows, args.seed + 12345)
    if pipelined:
        my_ms = float(ev_a.elapsed_time(ev_b))
        tot_log = sum(logs)
        rows_log, acc_log, com_log = tot_log[0], tot_log[1], tot_log[2]
    else:
        my_ms = float(sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in evs))
    KP = K
    prof_rows = None
    if use_graph:
        # per-kernel breakdown: the same two segments captured again with the
        # library's event pairs inside (every replay re-records them; read after
        # each step with srt_profile_peek), KP more graph-replayed steps with
        # their rows logged -- the timed graphs carry no profiling nodes
        KP = min(K, 20)
        gr0.cache.profile_enable(4 * KERNELS_PER_STEP)
        gp_draft, gp_vi = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        if not gr0.fused_step:
            with torch.cuda.graph(gp_draft):
                gr0.draft()
        with torch.cuda.graph(gp_vi):
            gr0.verify_insert(seed)
        prof_rows = torch.zeros(KP, dtype=torch.int64, device=run.dev)
        for k in range(KP):
            if not gr0.fused_step:
                gp_draft.replay()
            gr0.standin()
            prof_rows[k] = gr0.d.row_offsets[-1]
            gp_vi.replay()
            step_prof.append(gr0.cache.profile_peek())
        torch.cuda.synchronize()
        prof = [x for sp in step_prof for x in sp]
        prof_rows = prof_rows.cpu().numpy()
        del gp_draft, gp_vi
        gr0.cache.profile_enable(0)
    else:
        prof = [x for gr in run.groups for x in gr.cache.profile_read()]
    bits, st = run.status()
    if bits:
        raise RuntimeError(f"device error bits {bits} in the timed region")
    tot = torch.tensor([my_ms], dtype=torch.float64, device=run.dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    max_ms = float(tot.item())
    rows = rows_log.cpu().numpy()
    acc = int(acc_log.sum().item())
    com = int(com_log.sum().item())
    per_kernel = {}
    for name, ms in prof:
        per_kernel.setdefault(name, []).append(ms)
    # ---- e2e: same steps through the public API with host-resident logits
    e2e = e2e_leg(run, args, min(args.e2e_steps, K)) if args.e2e_steps > 0 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    esz = 2 if args.dtype == "bf16" else 4
    scan_ms = per_kernel.get("scan", [])
    path_mode = args.verify == "path" and wl is not None
    smp = smp_log.cpu().numpy() if path_mode else None
    # bytes the scan reads: every drafted row (srt_verify) or the sampled ones (srt_verify_path)
    scan_bytes = float((smp if path_mode else rows).sum()) * cfg["V"] * esz
    peak, peak_kind = load_peaks()
    # per launch: the algorithmic bytes of the SAME launches the per-kernel
    # times come from (the timed steps in eager mode; the profiled eager
    # steps, whose rows are logged, in graph mode) over their mean time
    prof_bytes = (float(np.mean(prof_rows)) * cfg["V"] * esz
                  if prof_rows is not None and not path_mode else scan_bytes / K)
    achieved = prof_bytes / (float(np.mean(scan_ms)) / 1000.0) / 1e9 if scan_ms else None
    traffic = traffic_ratio = None
    tf = os.path.join(ROOT, "profiles", f"scan_traffic_{args.config}_{args.dtype}.json")
    if os.path.exists(tf):
        tj = json.load(open(tf))
        traffic = tj.get("bytes_per_launch")
        if tj.get("algorithmic_bytes_same_launch"):
            traffic_ratio = traffic / tj["algorithmic_bytes_same_launch"]
    value = world * K / (max_ms / 1000.0)
    kern = {k: {"launches": len(v), "mean_us": 1000 * float(np.mean(v)),
                "share": float(sum(v) / sum(sum(x) for x in per_kernel.values()))}
            for k, v in per_kernel.items()}
    out = {
        "metric": metric, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": workload, "profile": args.profile, "parallelism": f"dp{world}",
                   "global_batch": cfg["active"] * world, "seqs_per_rank": cfg["active"],
                   "l2": "inputs larger than L2 (logits buffer "
                         f"{run.logits.numel() * esz / 1e9:.1f} GB)",
                   "groups": G,
                   "placement": ("hash-sharded trees (owner = splitmix64(p) mod N), sequences "
                                 "decoded on a contiguous split; per step an all-to-all of draft "
                                 "records (draft return) and an all-gather of span records "
                                 "(before insertion)"
                                 if (world > 1 or args.sharded) else "single rank"),
                   "timed": (f"whole step loop on the device (CUDA events, {G} prompt groups "
                             f"pipelined on {G} streams); forward stand-in and bookkeeping "
                             f"INCLUDED" if pipelined else
                             ("draft + verify + insert device time (CUDA events around the two "
                              "CUDA-graph replays per step; per-kernel breakdown from the same "
                              "segments re-captured with the library's event pairs and replayed "
                              "after the timed region, rows logged); forward stand-in excluded"
                              if use_graph else
                              "draft + verify + insert device time (CUDA events); forward "
                              "stand-in excluded")),
                   "seed": "one run seed for every step (the Philox counter carries the "
                           "position, so every (sequence, position) draws fresh noise)"},
        "accepted_tokens_per_s": world * acc / (max_ms / 1000.0),
        "committed_tokens_per_s": world * com / (max_ms / 1000.0),
        "mean_accepted_per_seq_step": acc / (K * cfg["active"]),
        "mean_rows_per_step": float(rows.mean()),
        **({"verify": f"path-only (srt_verify_path, {args.path_rounds} rounds + subtree tail)",
            "mean_rows_sampled_per_step": float(smp.mean())} if path_mode else {}),
        "roofline": {"bound": "hbm", "kernel": ("path verify (all rounds of k_scan_rows + "
                                                "k_path_*)" if path_mode else
                                                "scan (k_scan_rows + k_rowinfo)"),
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_over_algorithmic": traffic_ratio,
                     "traffic_source": "one ncu --set full capture of k_scan_rows "
                                       "(profiles/scan_traffic_*.json; its launch's rows differ "
                                       "from this run's mean)",
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": prof_bytes,
                     "algorithmic_bytes_per_timed_step": scan_bytes / K,
                     "frac_of_8TBps_spec": (achieved / 8000.0) if achieved else None},
        "kernels": kern,
        "tree_stage_us_per_batch": {k: kern[k]["mean_us"] for k in
                                    ("draft", "row_offsets", "insert_plan", "insert_walk",
                                     "insert_cursor", "accept", "accept_insert", "hub_refresh",
                                     "tree_step")
                                    if k in kern},
        # kernels per timed segment: the scan segment launches k_rowinfo + k_scan_rows,
        # the hub refresh k_hub_pick + k_hub_refresh; every other segment one kernel
        "gpu_launches": int(round(sum(SEGMENT_KERNELS.get(name, 1) for name, _ in prof) / KP * K)),
        "launches_per_step": sum(SEGMENT_KERNELS.get(name, 1) for name, _ in prof) / KP,
        "tree_nodes": st["nodes_used"],
    }
    cs = clk.summary()
    if cs:
        out["clocks"] = cs
    lm_mode = args.verify == "lmhead" and wl is not None
    if lm_mode:
        lm_ms = per_kernel.get("lmhead", [])
        K_h = run.lm_K
        rows_prof = (float(np.mean(prof_rows)) if prof_rows is not None else float(rows.mean()))
        flops = 2.0 * rows_prof * cfg["V"] * K_h
        ach_tf = flops / (float(np.mean(lm_ms)) / 1000.0) / 1e12 if lm_ms else None
        pk, pk_kind = load_tensor_peak()
        out["verify"] = ("lmhead: srt_verify_lmhead_insert_cursor (LM-head GEMM on tcgen05 + the "
                         "Gumbel-max sampler as its epilogue; logits never written)")
        out["config"]["hidden"] = K_h
        out["roofline"] = {"bound": "tensor", "kernel": "k_lmhead_sample (+k_rowinfo)",
                           "achieved": ach_tf, "peak": pk, "unit": "TFLOP/s",
                           "frac": ach_tf / pk if ach_tf else None, "traffic": None,
                           "peak_kind": pk_kind,
                           "algorithmic_flops_per_launch": flops}
        achieved = None  # (no HBM read-only comparison for this kernel)
        try:
            out["lmhead_vs_unfused"] = lmhead_comparison(run, seed, args)
        except Exception as e:
            out["lmhead_vs_unfused"] = {"error": repr(e)[:300]}
    if achieved:
        try:
            ro = readonly_stream_gbs(run.logits)
            out["roofline"]["readonly_stream"] = ro
            out["roofline"]["frac_of_readonly_stream"] = achieved / ro["gbs"]
        except Exception as e:  # never lose the GPU line over the probe
            out["roofline"]["readonly_stream"] = {"error": repr(e)[:200]}
    if psample is not None and not args.no_cpu_baseline:
        try:
            out["parity"] = check_parity_sample(psample, seed)
        except Exception as e:
            out["parity"] = {"error": repr(e)[:200]}
    if e2e:
        out["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1 and wl is not None:
        try:
            npr = args.cpu_prompts or max(1, min(cfg["prompts"], 64 // cfg["samples"]))
            bulk = run.logits[:npr * cfg["samples"] * (cfg["Bmax"] + 1)].float().cpu().numpy()
            t_step, n_s, _ = oracle_sample_steps(wl, args.dtype, 2, npr, args.seed, bulk)
            cores = cpu_cores_used(n_s)
            out["cpu_baseline"] = {
                "value": (n_s / cfg["active"]) / t_step, "unit": "steps/s", "cores": cores,
                "kind": "oracle",
                "sample": f"{n_s} of {cfg['active']} sequences ({npr} prompts), 2 steps, "
                          f"full-V rows; value scaled by {n_s}/{cfg['active']}"}
        except Exception as e:  # never lose the GPU line over the baseline
            out["cpu_baseline"] = {"value": None, "error": repr(e)[:200]}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def capture_parity_sample(run, n_rows: int, seed_rows: int):
    """Right after the timed region: a bounded random sample of the LAST timed
    step's logits rows with their sampler keys and the GPU's samples (device ->
    host, untimed).  The oracle checks them later (cpu leg): north_star's
    tie-break divergence count."""
    torch = run.torch
    gr = run.groups[0]
    ro_t, dep_t = gr.snap if gr.snap is not None else (gr.d.row_offsets, gr.d.draft_depth)
    total = int(ro_t[-1].item())
    if total <= 0 or n_rows <= 0:
        return None
    rng = np.random.default_rng(seed_rows)
    pick = np.sort(rng.choice(total, size=min(n_rows, total), replace=False))
    row_off = ro_t.cpu().numpy()
    s_of = np.searchsorted(row_off, pick, side="right") - 1
    j = pick - row_off[s_of]  # 0 = root row, else draft node j - 1
    depth = dep_t.cpu().numpy()
    t_before = gr.t_before.cpu().numpy()
    pos = t_before[s_of] + np.where(j == 0, 0, depth[s_of, np.maximum(j - 1, 0)])
    idx = torch.from_numpy(pick).to(gr.logits.device)
    rows = gr.logits[idx]
    if rows.dtype == torch.bfloat16:
        host = rows.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        host = rows.cpu().numpy()
    return {"rows": host, "seq_id": gr.seq_id.cpu().numpy().view(np.uint64)[s_of],
            "pos": pos.astype(np.int32), "gpu": gr.v.sampled[idx].cpu().numpy(),
            "of_rows": total}


def check_parity_sample(ps, seed: int):
    """The oracle's full-V Gumbel-max on the captured rows (same Philox keys):
    rows whose maximum z is shared by >= 2 indices (decided by the smallest-
    index rule) and rows where the GPU differs (north_star: must be 0)."""
    import oracle
    t = time.perf_counter()
    tok, ties, nan = oracle.sample_rows(ps["rows"], seed, ps["seq_id"], ps["pos"])
    return {"checked_rows": int(len(tok)), "of_rows_in_step": ps["of_rows"],
            "tie_rows": int(np.count_nonzero(ties >= 2)),
            "divergent_rows": int(np.count_nonzero(tok != ps["gpu"])),
            "nan_rows": int(np.count_nonzero(nan)),
            "oracle_s": round(time.perf_counter() - t, 2),
            "sample": "random rows of the last timed step, full V, oracle sample_row on the "
                      "same (seed, sequence, position) keys"}


def readonly_stream_gbs(buf) -> dict:
    """The read-only HBM stream (srt_stream_read: persistent TMA ring, one CTA
    per SM) over the bench's logits buffer, CUDA events, best of 3 shapes."""
    import torch
    import paper_2601_09083_b200 as srt
    nbytes = buf.numel() * buf.element_size()
    sink = torch.empty(1, dtype=torch.int64, device=buf.device)
    best = {"gbs": 0.0}
    for chunk, nbuf in ((32768, 6), (32768, 4), (16384, 12)):
        srt.stream_read(buf, chunk, nbuf, 1, sink)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            srt.stream_read(buf, chunk, nbuf, 1, sink)
        e1.record()
        torch.cuda.synchronize()
        gbs = 3 * (nbytes // chunk) * chunk / (e0.elapsed_time(e1) / 1000.0) / 1e9
        if gbs > best["gbs"]:
            best = {"gbs": gbs, "chunk": chunk, "stages": nbuf, "bytes": nbytes}
    return best


def e2e_leg(run: GpuRun, args, steps: int):
    """Same metric through the public API with HOST buffers: every step copies
    that step's logits rows from pinned host memory (H2D) and reads the step's
    results back (D2H) inside the timed region (groups one after another)."""
    torch = run.torch
    if steps <= 0:
        return None
    seed = step_seed(args.seed, 0)
    rows_max = max(gr.rows_max for gr in run.groups)
    lm = run.groups[0].lm if args.verify == "lmhead" else None
    src = lm["H"] if lm is not None else run.logits
    host = torch.empty(src[:rows_max].shape, dtype=src.dtype, pin_memory=True)
    host.copy_(src[:rows_max])
    dev_rows = lm["H"] if lm is not None else torch.empty_like(run.logits[:rows_max])
    nmax = max(gr.n for gr in run.groups)
    out_n = torch.empty(nmax, dtype=torch.int32).pin_memory()
    out_a = torch.empty(nmax, dtype=torch.int32).pin_memory()
    out_c = torch.empty(nmax, run.Bmax + 1, dtype=torch.int32).pin_memory()
    h2d = d2h = 0
    total_ms = 0.0
    for k in range(steps):
        for gr in run.groups:
            n = gr.n
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record()
            gr.draft_if_needed()
            rows_t = gr.d.row_offsets[-1:].to("cpu", non_blocking=True)
            e[1].record()
            torch.cuda.synchronize()
            rows = int(rows_t.item())
            gr.t_before.copy_(gr.seq_len)
            e[2].record()
            dev_rows[:rows].copy_(host[:rows], non_blocking=True)
            gr.verify_insert(seed, None if lm is not None else dev_rows)
            out_n[:n].copy_(gr.v.n_commit, non_blocking=True)
            out_a[:n].copy_(gr.v.accept_len, non_blocking=True)
            out_c[:n].copy_(gr.v.commit_tok, non_blocking=True)
            e[3].record()
            torch.cuda.synchronize()
            total_ms += e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3])
            h2d += rows * host.shape[1] * host.element_size()
            d2h += 8 + n * 4 * 2 + n * (run.Bmax + 1) * 4
    return {"value": steps / (total_ms / 1000.0), "unit": "steps/s",
            "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
            "steps": steps}


if __name__ == "__main__":
    main()
