"""Scan-kernel probe: time srt_verify's scan alone on R synthetic rows (one
row per sequence, empty drafts) for several logit profiles, with libsrt's own
per-kernel CUDA-event timing.  Development tool, not part of the product.

    python tools/scan_probe.py [--rows 16384] [--dtype bf16] [--profiles peaked,rl-mix,flat]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2601_09083_b200 as srt  # noqa: E402


def make_rows(R, V, profile, dtype, gen):
    x = torch.empty(R, V, dtype=dtype, device="cuda")
    if profile == "flat":
        x.uniform_(0, 1, generator=gen)
        return x
    x.normal_(0, 2, generator=gen)
    heads = torch.randint(0, V, (R,), device="cuda", generator=gen)
    if profile == "peaked":
        gap = torch.full((R,), 26.0, device="cuda")
    elif profile == "moderate":
        gap = torch.full((R,), 18.0, device="cuda")
    elif profile == "gap15":
        gap = torch.full((R,), 15.0, device="cuda")
    else:  # rl-mix (rl-mix-d: with the bench stand-in's 3 distractors below the head)
        u = torch.rand(R, device="cuda", generator=gen)
        hi = torch.rand(R, device="cuda", generator=gen) < 0.7
        gap = torch.where(hi, 18 + 6 * u, 12 + 6 * u)
        if profile == "rl-mix-d":
            ar = torch.arange(R, device="cuda")
            for k in range(3):
                off = torch.where(hi, 5 + 4 * torch.rand(R, device="cuda", generator=gen),
                                  0.5 + 3.5 * torch.rand(R, device="cuda", generator=gen))
                dk = torch.randint(0, V, (R,), device="cuda", generator=gen)
                x[ar, dk] = (gap - off).to(dtype)
    x[torch.arange(R, device="cuda"), heads] = gap.to(dtype)
    return x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--V", type=int, default=151936)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--profiles", default="peaked,rl-mix,gap15,flat")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--prealloc-gb", type=float, default=0.0,
                    help="allocate this much device memory first (placement experiments)")
    ap.add_argument("--padrows", type=int, default=0, help="extra rows after the scanned ones")
    a = ap.parse_args()
    dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    R, V = a.rows, a.V
    hold = torch.empty(int(a.prealloc_gb * 2**30), dtype=torch.uint8, device="cuda") if a.prealloc_gb else None
    cache = srt.SrtCache(srt.config(V, 1, 4, 2, 4, node_capacity=1024, logits_dtype=dt))
    n = R
    d = srt.DraftOut.empty(n, 4, "cuda")
    z = torch.zeros(n, dtype=torch.int32, device="cuda")
    seq_tok = torch.zeros(n, 16, dtype=torch.int32, device="cuda")
    cache.draft(z, seq_tok, z, out=d)  # empty tree -> empty drafts, rows = n
    seq_id = torch.arange(n, dtype=torch.int64, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    out = {}
    for prof in a.profiles.split(","):
        x = make_rows(R, V, prof, dt, gen)
        cache.profile_enable(64)
        for it in range(a.iters):
            seq_len = torch.zeros(n, dtype=torch.int32, device="cuda")
            cache.verify(x, d, seq_id, 1234 + it, seq_tok, seq_len,
                         torch.full((n,), 8, dtype=torch.int32, device="cuda"))
        recs = cache.profile_read()
        scan = [ms for k, ms in recs if k == "scan"][1:]
        ms = sum(scan) / len(scan)
        gbs = R * V * x.element_size() / (ms / 1000) / 1e9
        out[prof] = {"scan_ms": ms, "GB/s": gbs}
        print(f"{prof:9s} scan {ms:8.3f} ms  {gbs:8.1f} GB/s", flush=True)
        del x
    print(json.dumps(out))


if __name__ == "__main__":
    main()
