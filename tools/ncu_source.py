#!/usr/bin/env python3
"""Top stall lines (SASS) of one kernel in an ncu report: ncu_source.py rep regex [N]."""
import csv, subprocess, sys

def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
start = rows.index(hdr) + 1
data = [r for r in rows[start:] if len(r) == len(hdr) and r[0] != "Address"]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(f(r[i_s]) for r in data) or 1.0
for r in sorted(data, key=lambda r: -f(r[i_s]))[:n]:
    print(f"{f(r[i_s]) / tot * 100:5.1f}%  {r[0]:>6}  {r[i_src][:110]}")
