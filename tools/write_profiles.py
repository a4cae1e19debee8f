"""Write profiles/r01_<tag>_* from a tools/final_round.sh pass (development tool).

    python tools/write_profiles.py <tag> "<what changed since the last tag>"
"""
import json
import re
import shutil
import subprocess
import sys

tag, note = sys.argv[1], sys.argv[2]
G = "gpurun_out"
rows = int(re.search(r"warm-up step 3: rows \[(\d+)\]", open(f"{G}/rows_{tag}.log").read()).group(1))
alg = rows * 151936 * 2


def summary(*args):
    return subprocess.run([sys.executable, "tools/ncu_summary.py", *args], capture_output=True,
                          text=True, check=True).stdout


s = summary("full", f"{G}/scan_{tag}.ncu-rep")
rd = float(re.search(r"dram__bytes_read.sum \| ([\d.]+) \| Gbyte", s).group(1)) * 1e9
wv, wu = re.search(r"dram__bytes_write.sum \| ([\d.]+) \| (\w+)", s).groups()
wr = float(wv) * (1e6 if wu == "Mbyte" else 1e3 if wu == "Kbyte" else 1e9)
t = float(re.search(r"gpu__time_duration.sum \| ([\d.]+)", s).group(1))
pk = re.search(r"dram_throughput.avg.pct_of_peak_sustained_elapsed \| ([\d.]+)", s).group(1)
open(f"profiles/r01_{tag}_ncu_scan.md", "w").write(
    f"# r01 {tag} — ncu --set full, k_scan_rows (GRPO bf16, warm-up step 3: {rows:,} rows)\n\n"
    f"Algorithmic bytes of this launch: {rows:,} rows x 151,936 x 2 B = {alg/1e9:.4f} GB; measured "
    f"DRAM read {rd/1e9:.4f} GB ({(rd/alg-1)*100:+.2f} %), write {wv} {wu}.  {t:.1f} us under ncu "
    f"(cold, serialised) = {alg/t/1e6:.2f} TB/s; DRAM throughput {pk} % of ncu's peak.\n\n"
    "Command: `ncu --set full --import-source on --clock-control none -k regex:k_scan_rows -s 3 -c 1 "
    "python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4` "
    f"(tools/profile_round.sh {tag}).\n\n" + s)
open(f"profiles/r01_{tag}_ncu_tree.md", "w").write(
    f"# r01 {tag} — ncu --set full, tree kernels (GRPO bf16, one timed step)\n\n"
    "Latency-bound pointer work (a few % warps active, long-scoreboard stalls dominate).  "
    f"{note}  Analysis of the slowest warps (tools/draft_probe.py, tools/insert_probe.py, "
    "tools/latency_probe.cu) in DESIGN.md §5 and §11.\n\n" + summary("full", f"{G}/tree_{tag}.ncu-rep"))
b = json.loads(open(f"{G}/bench_{tag}.log").read().strip().splitlines()[-1])
sh = {k: v.get("share") or 0.0 for k, v in b["kernels"].items()}
parts = ", ".join(f"{k} {sh[k]*100:.1f} %" for k in ("scan", "draft", "accept_insert", "insert_cursor",
                                                      "hub_refresh") if k in sh)
open(f"profiles/r01_{tag}_launches.md", "w").write(
    f"# r01 {tag} — ncu launch list, GRPO bf16 (bench.py --steps 3 --warmup 3, CUDA-graph step replay)\n\n"
    "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py "
    "--no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3`.  Per-launch times are cold-cache and "
    "serialised; the last 3 launches of each kernel are kept.  Live bench line of the same commit: "
    f"profiles/r01_bench_grpo_{tag}.json, {b['value']:.1f} steps/s ({parts}).\n\n{note}\n\n"
    + summary("launches", f"{G}/launches_{tag}.csv", "3"))
shutil.copy(f"{G}/launches_{tag}.csv", f"profiles/r01_{tag}_launches_grpo.csv")
json.dump({"bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
           "algorithmic_bytes_same_launch": alg, "rows": rows,
           "source": f"ncu --set full -k k_scan_rows, bench.py GRPO bf16 warm-up step 3 "
                     f"(profiles/r01_{tag}_ncu_scan.md)"},
          open("profiles/scan_traffic_grpo_bf16.json", "w"))
for src, dst in ((f"bench_{tag}", "grpo"), (f"bench_grpo_path_{tag}", "grpo_path"),
                 (f"bench_ppo_{tag}", "ppo"), (f"bench_dapo_{tag}", "dapo")):
    line = open(f"{G}/{src}.log").read().strip().splitlines()[-1]
    open(f"profiles/r01_bench_{dst}_{tag}.json", "w").write(line + "\n")
print("ok", rows, f"{rd/alg-1:+.4f}")
