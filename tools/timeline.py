#!/usr/bin/env python3
"""Warm-run kernel timeline of BP syncs (CUPTI via torch.profiler): per-kernel
start/end relative to each sync's first kernel, stream id, and the gaps on
the critical stream.  Diagnostic only (numbers taken under a profiler are
never bench values).

  python tools/timeline.py [--workers 1] [--syncs 3] [--out gpurun_out/tl.txt]
"""
import argparse
import collections
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--syncs", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--scheme", default="bp", choices=["bp", "hc"],
                    help="hc: Hierarchical Centralization (rank mode, torchrun)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import paper_2309_13254_b200 as zen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:  # rank mode under torchrun: one worker per GPU
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        args.workers = world
    torch.cuda.set_stream(torch.cuda.Stream())
    n = args.workers
    per = int(np.ceil(args.density * args.rows))
    rows = bench.live_rows(args.rows, per, n, 0.5, 1.05, 1)
    mine = [rank] if dist else list(range(n))
    dd = [torch.from_numpy(bench.dense_gradient(args.rows, args.width, rows[w], 1 + w)).cuda()
          for w in mine]
    m = args.rows * args.width
    z = per * args.width
    if args.scheme == "hc":
        hc = zen.HCSynchronizer(n, m, rank, max_nnz=int(z * 1.25) + 4096)
        hc.connect_process_group() if dist else hc.connect([hc.ipc_handle()])

        def run():
            hc.sync_dense(dd[0])
        first, last = "k_hc_begin", None
    else:
        bp = zen.BPSynchronizer(n, m, max_nnz=int(z * 1.25) + 4096, params=zen.HashParams(seed=1),
                                rank=rank if dist else None)
        if dist:
            bp.connect_process_group()

        def run():
            bp.sync_dense(dd)
        first, last = "k_bp_begin", "k_decode"
    for _ in range(10):
        run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    if dist:
        dist.barrier()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.syncs):
            run()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
        if args.out:
            args.out = args.out.replace(".txt", f"_r{rank}.txt")
    tmp = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(tmp)
    ev = json.load(open(tmp))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    # split into syncs at each extraction kernel
    syncs, cur = [], []
    for e in ks:
        if first in e["name"] and cur and (last is None or any(last in x["name"] for x in cur)):
            syncs.append(cur)
            cur = []
        cur.append(e)
    if cur:
        syncs.append(cur)
    lines = []
    agg = collections.OrderedDict()
    for si, s in enumerate(syncs):
        t0 = s[0]["ts"]
        end = max(e["ts"] + e["dur"] for e in s)
        lines.append(f"--- sync {si}: {end - t0:.1f} us, {len(s)} kernels")
        prev_end = {}
        for e in s:
            nm = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:44]
            st = e["args"].get("stream", -1)
            gap = e["ts"] - prev_end.get(st, e["ts"])
            prev_end[st] = e["ts"] + e["dur"]
            lines.append(f"  {e['ts'] - t0:8.1f} +{e['dur']:7.1f}  gap {gap:6.1f}  s{st:<4} {nm}")
            if si > 0:
                agg.setdefault(nm, []).append(e["dur"])
    lines.append("--- mean warm duration per kernel (syncs 1..):")
    for k, v in agg.items():
        lines.append(f"  {sum(v) / len(v):8.2f} us  {k}")
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        open(args.out, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
