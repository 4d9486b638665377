#!/usr/bin/env python3
"""NVLink evidence for the BP exchange (rank mode, one process per GPU).

The push (k_push_scatter: NVLink stores into the owners' inboxes) and the pull
(k_agg_union + k_agg_values, or k_agg_fused from 4 workers up: NVLink stores of the HashBitmap, the values and
the per-chunk bases into every receiver) have no kernel of their own, so
their link rate is measured on the kernels that carry them:

  * bytes: the GPU's NVLink hardware counters (NVML field values
    NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, summed over the links; KiB)
    read before and after K syncs, per sync;
  * time: the warm durations of those kernels from a CUPTI trace
    (torch.profiler) of the same K syncs.

achieved = TX bytes per sync / (push + pull kernel time), against the
900 GB/s per direction NVLink 5 nominal and the 770 GB/s measured peer copy
(B200_PROFILING.md).  The counters see every NVLink byte of the GPU (the
data path only: the library makes no NCCL call during a sync).
Diagnostic only -- numbers taken under a profiler are never bench values.

  torchrun --nproc-per-node N tools/nvlink_profile.py [--syncs 20] [--out f.json]
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PUSH = ("k_push_scatter",)
PULL = ("k_agg_union", "k_agg_values", "k_agg_fused")


def nvlink_kib(handle, pynvml):
    """(tx, rx) data KiB summed over the GPU's NVLinks, or None if unsupported."""
    tx = rx = 0
    ok = False
    for link in range(18):
        try:
            fv = pynvml.nvmlDeviceGetFieldValues(
                handle, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                         (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
        except Exception:  # noqa: BLE001
            continue
        for f, acc in zip(fv, ("tx", "rx")):
            if f.nvmlReturn == 0:
                ok = True
                v = f.value.ullVal
                if acc == "tx":
                    tx += v
                else:
                    rx += v
    return (tx, rx) if ok else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--syncs", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    import bench
    import paper_2309_13254_b200 as zen
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    torch.cuda.set_stream(torch.cuda.Stream())
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rows, d = args.rows, 64
    per = int(np.ceil(args.density * rows))
    live = bench.live_rows(rows, per, world, 0.5, 1.05, 1)
    g = torch.from_numpy(bench.dense_gradient(rows, d, live[rank], 1 + rank)).cuda()
    bp = zen.BPSynchronizer(world, rows * d, max_nnz=int(per * d * 1.25) + 4096, rank=rank)
    bp.connect_process_group()
    for _ in range(5):
        bp.sync_dense([g])
    bp.wait()
    led, counts, agg = bp.ledger()
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    dist.barrier()
    torch.cuda.synchronize()
    c0 = nvlink_kib(h, pynvml)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.syncs):
            bp.sync_dense([g])
        torch.cuda.synchronize()
    c1 = nvlink_kib(h, pynvml)
    dist.barrier()
    tmp = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(tmp)
    ev = [e for e in json.load(open(tmp))["traceEvents"] if e.get("cat") == "kernel"]
    dur = {}
    for e in ev:
        nm = e["name"].replace("(anonymous namespace)::", "")
        for k in PUSH + PULL:
            if k in nm:
                dur.setdefault(k, []).append(e["dur"])
    mean_us = {k: float(np.mean(v)) for k, v in dur.items()}
    push_us = sum(mean_us.get(k, 0.0) for k in PUSH)
    pull_us = sum(mean_us.get(k, 0.0) for k in PULL)
    # exchange bytes each rank stores to its peers (the library's wire format:
    # u32 index + f32 value per pushed entry; the pulled bitmap words, values
    # and per-chunk bases per receiver), from the device counts
    n = world
    push_entries = int(sum(counts[rank][s] for s in range(n) if s != rank))
    res = {"rank": rank, "n": n, "syncs": args.syncs, "kernel_us": mean_us,
           "push_kernel_us": round(push_us, 2), "pull_kernel_us": round(pull_us, 2),
           "push_entries_per_sync": push_entries,
           "ledger_push_sent_bits": int(led[0, 0, rank]), "ledger_pull_sent_bits": int(led[1, 0, rank])}
    if c0 is not None and c1 is not None:
        tx = (c1[0] - c0[0]) * 1024 / args.syncs
        rx = (c1[1] - c0[1]) * 1024 / args.syncs
        t = (push_us + pull_us) * 1e-6
        res.update({"nvlink_tx_bytes_per_sync": tx, "nvlink_rx_bytes_per_sync": rx,
                    "achieved_tx_GBps": round(tx / t / 1e9, 1) if t else None,
                    "frac_of_900": round(tx / t / 900e9, 4) if t else None,
                    "frac_of_770_measured": round(tx / t / 770e9, 4) if t else None,
                    "counter": "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB, all links)"})
    else:
        res["counter"] = "NVML NVLink throughput fields unsupported here"
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        txt = json.dumps(allr, indent=1)
        print(txt, flush=True)
        if args.out:
            open(args.out, "w").write(txt + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
