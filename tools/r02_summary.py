"""Write profiles/r02_<tag>_* from a tools/profile_r02.sh pass (development tool).

    python tools/r02_summary.py <tag> "<what changed since the last tag>"

Copies every bench line of gpurun_out/<tag>/bench_<config>.log to
profiles/r02_<tag>_<config>.json and writes profiles/r02_<tag>_summary.md
(the bench table, the GPU-suite tail, the full-draft scan stress, the ncu
launch list and the key metrics of each ncu --set full capture).
"""
import glob
import json
import os
import subprocess
import sys

tag, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
G = f"gpurun_out/{tag}"
TREE = ("tree_step", "draft", "row_offsets", "accept_insert", "accept", "insert_plan", "insert_walk",
        "insert_cursor", "hub_refresh")


def last_json(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def sh(*args):
    r = subprocess.run([sys.executable, "tools/ncu_summary.py", *args], capture_output=True, text=True)
    return r.stdout if r.returncode == 0 else f"(ncu_summary failed: {r.stderr.strip()[-200:]})\n"


out = [f"# r02 {tag} — measurement pass (tools/profile_r02.sh {tag}, one B200)\n"]
if note:
    out.append(note + "\n")
for f, what in ((f"{G}/pytest_gpu.log", "`pytest -m gpu`"), (f"{G}/smoke.log", "smoke")):
    if os.path.exists(f):
        lines = [l for l in open(f).read().splitlines() if l.strip()]
        out.append(f"{what}: `{lines[-1] if lines else '(empty)'}`\n")
out.append("| config | steps/s | us/step | rows/step | roofline achieved | frac (copy peak) | "
           "frac (read-only stream) | scan us | tree us (share) | SM MHz |")
out.append("|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(f"{G}/bench_*.log")):
    cfg = os.path.basename(f)[len("bench_"):-len(".log")]
    d = last_json(f)
    if not d or "value" not in d:
        out.append(f"| {cfg} | (no bench line) |||||||||")
        continue
    json.dump(d, open(f"profiles/r02_{tag}_{cfg}.json", "w"), indent=1)
    r, k = d.get("roofline", {}), d.get("kernels", {})
    main = k.get("scan") or k.get("lmhead") or {}
    tree = sum(v["mean_us"] for n, v in k.items() if n in TREE)
    tshare = sum(v["share"] for n, v in k.items() if n in TREE)
    ach = f"{r.get('bound')} {r.get('achieved', 0):.0f} {r.get('unit')}"
    out.append(f"| {cfg} | {d['value']:.1f} | {d['ms_per_step'] * 1000:.0f} | "
               f"{d.get('mean_rows_per_step', 0):,.0f} | {ach} | {r.get('frac', 0):.3f} | "
               f"{r.get('frac_of_readonly_stream', 0):.3f} | {main.get('mean_us', 0):.0f} | "
               f"{tree:.0f} ({100 * tshare:.0f}%) | {d.get('clocks', {}).get('sm_mhz')} |")
g = last_json(f"{G}/bench_grpo.log") if os.path.exists(f"{G}/bench_grpo.log") else None
if g and "parity" in g:
    p = g["parity"]
    out.append(f"\nGRPO parity sample: divergent_rows {p['divergent_rows']} of {p['checked_rows']} "
               f"full-V rows (tie_rows {p['tie_rows']}).\n")
for f, title in ((f"{G}/scan_fulldraft.txt", "Full-draft scan stress (33,792 rows bf16)"),
                 (f"{G}/scan_fulldraft_f32.txt", "Full-draft scan stress (16,896 rows f32)")):
    if os.path.exists(f):
        out.append(f"## {title}\n```\n{open(f).read().strip()}\n```\n")
if os.path.exists(f"{G}/launches.csv"):
    out.append("## ncu launch list (last 3 launches per kernel)\n")
    out.append(sh("launches", f"{G}/launches.csv", "3"))
for rep in sorted(glob.glob(f"{G}/*.ncu-rep")):
    out.append(f"## ncu --set full: {os.path.basename(rep)[:-8]}\n")
    out.append(sh("full", rep))
open(f"profiles/r02_{tag}_summary.md", "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
