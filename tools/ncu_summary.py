"""Summarise ncu outputs for profiles/ (development tool).

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel time shares
    python tools/ncu_summary.py full <report.ncu-rep>        # key metrics of a --set full capture
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def kname(s: str) -> str:
    m = re.findall(r"(k_\w+|[a-z_]+elementwise_kernel|reduce_kernel|[A-Za-z_]\w*kernel\w*)", s)
    return m[0] if m else s[:40]


def launches(path, tail=None):
    """Per-kernel device time; tail=K keeps each kernel's last K launches (the
    timed steps; earlier ones are setup such as the warm-tree inserts)."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in data:
        if len(r) <= vi or not r[vi]:
            continue
        agg[kname(r[ki])].append(float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0))
    setup = {}
    if tail:
        # kernels with fewer launches than the timed steps ran only during setup
        # (warm-tree build, noise tables): listed apart, not in the shares
        setup = {k: v for k, v in agg.items() if len(v) < int(tail)}
        agg = {k: v[-int(tail):] for k, v in agg.items() if len(v) >= int(tail)}
    tot = sum(sum(v) for k, v in agg.items() if k.startswith("k_"))
    print("| kernel | launches | total us | mean us | share of libsrt time |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot:.1f}%" if k.startswith("k_") else "(torch, bench stand-in)"
        print(f"| {k} | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {share} |")
    if setup:
        print("\nSetup-only launches (before the timed steps, excluded above): " +
              ", ".join(f"{k} x{len(v)} ({sum(v):.0f} us)" for k, v in sorted(setup.items())))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for vals in rows[2:]:
        print(f"### {kname(vals[ki])}")
        print("| metric | value | unit |")
        print("|---|---|---|")
        for i, h in enumerate(hdr):
            if h in KEYS or (h.startswith("smsp__average_warps_issue_stalled") and
                             vals[i] and float(vals[i]) > 0.25):
                print(f"| {h} | {vals[i]} | {units[i]} |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
