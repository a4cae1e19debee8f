"""Aggregate an ncu report's SASS-level warp-stall samples and executed
instructions per CUDA source line (development aid; needs -lineinfo and
--import-source on).  python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, agg, src, hdr = None, collections.Counter(), {}, None
    inst = collections.Counter()
    stall_cols = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            iI = hdr.index("Instructions Executed")
            continue
        if hdr is None or r[0] in ("Function Name",):
            continue
        if r[0].isdigit() and len(r) > iS:
            key = (fname, int(r[0]))
            src[key] = r[1].strip()
            try:
                agg[key] += int(r[iS] or 0)
                inst[key] += int(r[iI] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    ti = sum(inst.values()) or 1
    print(f"total stall samples {tot}, instructions {ti}")
    for key, v in agg.most_common(top):
        print(f"{100 * v / tot:5.1f}% samp {100 * inst[key] / ti:5.1f}% inst  {key[0]}:{key[1]:<4} {src[key][:100]}")


if __name__ == "__main__":
    main()
