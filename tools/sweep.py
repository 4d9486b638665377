#!/usr/bin/env python3
"""BASELINE.json's other configs at one GPU (and emulated n): the C4 density
sweep (0.1% .. 10%), C2 (1M x 16, 0.5%, Zipf rows) and C3 (800K x 1024, 1%),
each through bench.py (same timing rules), one JSON object per config.

  python tools/sweep.py [--out gpurun_out/sweep.json] [--quick]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFIGS = [
    # name, rows, width, density, emulate
    ("C4 1M x 64, 0.1%", 1_000_000, 64, 0.001, 8),
    ("C4 1M x 64, 1%", 1_000_000, 64, 0.01, 8),
    ("C4 1M x 64, 3%", 1_000_000, 64, 0.03, 0),
    ("C4 1M x 64, 10%", 1_000_000, 64, 0.10, 0),
    ("C2 1M x 16, 0.5% (Zipf rows)", 1_000_000, 16, 0.005, 8),
    ("C3 800K x 1024, 1%", 800_000, 1024, 0.01, 0),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    res = []
    for name, rows, width, dens, emu in CONFIGS:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--rows", str(rows), "--width",
               str(width), "--density", str(dens), "--no-e2e", "--no-extras", "--no-cpu",
               "--steps", "20" if args.quick else "100", "--warmup", "5"]
        if emu:
            cmd += ["--emulate", str(emu)]
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=1200)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            res.append({"config": name, "error": (r.stderr or r.stdout)[-500:]})
            continue
        m = rows * width
        z = d["config"]["nnz_per_worker"]
        hash_ms = d["stage_ms"]["hash_push"]
        entry = {"config": name, "M": m, "nnz_per_worker": z, "ms_per_sync_n1": d["value"],
                 "stage_ms": d["stage_ms"], "extract_roofline_frac": d["roofline"]["frac"],
                 "hash_stage": d["hash_stage"],
                 "throughput_mnnz_per_s": d["throughput_mnnz_per_s"]}
        if d.get("emulated_local"):
            entry["emulated"] = d["emulated_local"]
        res.append(entry)
        print(json.dumps(entry), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
