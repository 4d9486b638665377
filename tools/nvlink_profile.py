#!/usr/bin/env python3
"""NVLink evidence for the BP exchange (rank mode, one process per GPU).

The push (k_push_scatter, NVLink stores into the owners' inboxes) and the
pull (k_agg_union + k_agg_values, NVLink stores of the HashBitmap and the
values into every receiver) have no kernel of their own, so their link rate
is measured on the kernels that carry them: ncu's NVLink counters
(nvltx__bytes / nvlrx__bytes, 32-B granularity, all links of the GPU) and the
kernel's duration, collected on rank 0 only with a metric set that fits one
pass (no replay), while the other ranks run unprofiled.

  python tools/nvlink_profile.py --gpus 2 [--out gpurun_out/nvl]

Launches the ranks itself (not torchrun): rank 0 as `ncu ... python
tools/nvlink_profile.py --worker`, the others plain, plumbing over gloo on
127.0.0.1.  Every peer wait in the library has a 30 s watchdog, so a slow
profiled rank cannot hang the others.  Diagnostic only: no number taken under
ncu is a bench value.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ("gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,"
           "nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum")
KERNELS = "regex:k_push_scatter|k_agg_union|k_agg_values|k_decode|k_agg_mark"


def worker(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import bench
    import paper_2309_13254_b200 as zen
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    torch.cuda.set_stream(torch.cuda.Stream())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, d = args.rows, 64
    per = int(np.ceil(args.density * rows))
    live = bench.live_rows(rows, per, world, 0.5, 1.05, 1)
    g = torch.from_numpy(bench.dense_gradient(rows, d, live[rank], 1 + rank)).cuda()
    bp = zen.BPSynchronizer(world, rows * d, max_nnz=int(per * d * 1.25) + 4096, rank=rank)
    bp.connect_process_group()
    for _ in range(args.syncs):
        bp.sync_dense([g])
        bp.wait()
        dist.barrier()
    led, counts, agg = bp.ledger()
    if rank == 0:
        print(json.dumps({"ledger_push_sent_bits": int(led[0, 0, 0]),
                          "ledger_pull_sent_bits": int(led[1, 0, 0]),
                          "counts_row0": [int(x) for x in counts[0]],
                          "agg": [int(x) for x in agg]}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--syncs", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/nvl")
    ap.add_argument("--worker", action="store_true")
    args = ap.parse_args()
    if args.worker:
        return worker(args)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + os.getpid() % 300),
               WORLD_SIZE=str(args.gpus))
    me = [sys.executable, os.path.abspath(__file__), "--worker", "--rows", str(args.rows),
          "--density", str(args.density), "--syncs", str(args.syncs)]
    procs = []
    for r in range(args.gpus):
        cmd = me if r else ["ncu", "--metrics", METRICS, "-k", KERNELS, "--cache-control", "none",
                            "--clock-control", "none", "--csv", "--log-file",
                            args.out + f"_n{args.gpus}.csv"] + me
        procs.append(subprocess.Popen(cmd, env=dict(env, RANK=str(r)), cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=900)[0] for p in procs]
    rcs = [p.returncode for p in procs]
    open(args.out + f"_n{args.gpus}.log", "w").write(
        "\n".join(f"== rank {r} rc={rc}\n{o[-4000:]}" for r, (rc, o) in enumerate(zip(rcs, outs))))
    print("rcs", rcs)
    return max(rcs)


if __name__ == "__main__":
    sys.exit(main())
