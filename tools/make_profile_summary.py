#!/usr/bin/env python3
"""Turn one tools/profile_round.sh output directory (gpurun_out/<tag>) into the
tracked evidence under profiles/<tag>/:

  launches.csv          ncu --metrics gpu__time_duration.sum launch list (raw)
  launch_summary.md     per-kernel mean launch time and share of one sync
  ncu_full_summary.txt  --set full: time, DRAM bytes, occupancy, top stalls
  ncu_full_raw.csv      selected raw metrics of the --set full capture
  bench.json / bench_ref.json / pytest_gpu.log / compat_test.log (copies)

and refresh profiles/ncu_traffic.json (DRAM bytes per launch of the
roofline kernel, read by bench.py)."""
import collections
import re
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def short(name):
    for junk in ("(anonymous namespace)::", "<unnamed>::", "unnamed>::", "void "):
        name = name.replace(junk, "")
    return name.split("(")[0]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = {k: j for j, k in enumerate(rows[start])}
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[h["Metric Unit"]]
        v = float(r[h["Metric Value"]].replace(",", ""))
        v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        per.setdefault(short(r[h["Kernel Name"]]), []).append(v)
    return per


def raw_full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {k: j for j, k in enumerate(hdr)}
    recs = []
    for r in data:
        rec = {"kernel": short(r[ix["Kernel Name"]])}
        for k in RAW_KEYS:
            if k in ix:
                rec[k] = r[ix[k]] + ("" if not units[ix[k]] else " " + units[ix[k]])
        recs.append(rec)
    return recs, hdr, units, data, ix


def to_bytes(s):
    v, u = s.split(" ") if " " in s else (s, "byte")
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main(tag):
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    for f in ["launches.csv", "bench.json", "bench_ref.json", "pytest_gpu.log", "compat_test.log",
              "status", "short.json"]:
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    lines = []
    if os.path.exists(os.path.join(src, "launches.csv")):
        per = launch_table(os.path.join(src, "launches.csv"))
        extra = re.compile(r"k_topk|MagnitudeAtLeast|at_cuda_detail|at::|k_check_canonical|"
                           r"k_coo_|k_tb_|CUB_|k_tables")
        steady = {k: v for k, v in per.items() if not extra.search(k)}
        counts = sorted(len(v) for v in steady.values())
        nsync = counts[len(counts) // 2] if counts else 0
        step = sum(sum(v) / len(v) for v in steady.values())
        lines += [f"# Launch list ({tag}): ncu --metrics gpu__time_duration.sum --clock-control none",
                  "", "Cold-cache, serialised per-launch times (ncu replays each launch); "
                  "the SHARE of the sync is what compares with bench.py's live numbers.", "",
                  f"syncs captured: {nsync}; one sync = sum of per-kernel means: {step:.1f} us "
                  "(k_place[_tiles]/k_depth[_scan]/k_serial_*/k_fallback run on the forked side stream, "
                  "overlapped with the data path in the live run)", "",
                  "| kernel | launches | mean us | share of sync |", "|---|---|---|---|"]
        for k, v in per.items():
            m = sum(v) / len(v)
            share = (f"{100 * m / step:.1f}%" if k in steady else
                     "setup (once)" if "k_tables" in k else "not in the sync")
            lines.append(f"| {k} | {len(v)} | {m:.2f} | {share} |")
        open(os.path.join(dst, "launch_summary.md"), "w").write("\n".join(lines) + "\n")
    rep = os.path.join(src, "full.ncu-rep")
    if os.path.exists(rep):
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                              capture_output=True, text=True).stdout
        open(os.path.join(dst, "ncu_full_summary.txt"), "w").write(
            f"# ncu --set full --clock-control none --import-source on ({tag})\n" + summ)
        recs, hdr, units, data, ix = raw_full(rep)
        with open(os.path.join(dst, "ncu_full_raw.csv"), "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=["kernel"] + RAW_KEYS)
            w.writeheader()
            for r in recs:
                w.writerow(r)
        traffic = {}
        for r in recs:
            if r["kernel"].startswith("k_extract_tiles") and "dram__bytes_read.sum" in r:
                traffic["k_extract"] = int(to_bytes(r["dram__bytes_read.sum"]) +
                                           to_bytes(r["dram__bytes_write.sum"]))
        if traffic:
            traffic["source"] = f"profiles/{tag}/ncu_full_raw.csv (k_extract_tiles, one launch)"
            json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"),
                      indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
