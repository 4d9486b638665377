#!/usr/bin/env python3
"""Summarise an ncu --set full report: time, DRAM bytes, occupancy, top stalls per kernel."""
import csv, subprocess, sys

def main(rep, top=5):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
    if not stall:
        stall = [h for h in hdr if "warps_issue_stalled" in h and h.endswith(".ratio")]
    def g(r, k):
        try:
            return float(r[idx[k]])
        except Exception:
            return float("nan")
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")[-40:]
        t = g(r, "gpu__time_duration.sum")
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        ur, uw = units[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_write.sum"]]
        occ = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        ipc = g(r, "smsp__issue_active.avg.pct_of_peak_sustained_active") if "smsp__issue_active.avg.pct_of_peak_sustained_active" in idx else float("nan")
        st = sorted(((g(r, h), h.split("stalled_")[1].split(".")[0]) for h in stall), reverse=True)[:top]
        print(f"{name:40s} t={t:8.2f}{units[idx['gpu__time_duration.sum']]} dram r={rd:.2f}{ur} w={wr:.2f}{uw} "
              f"occ={occ:.0f}% issue={ipc:.0f}% regs={r[idx['launch__registers_per_thread']]} grid={r[idx['launch__grid_size']]}")
        print("     stalls(cycles/inst): " + ", ".join(f"{n}={v:.1f}" for v, n in st))

if __name__ == "__main__":
    main(sys.argv[1])
