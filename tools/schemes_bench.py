#!/usr/bin/env python3
"""Balanced Parallelism vs Hierarchical Centralization on the bench workload
(SURVEY.md §8f row f3), one process per GPU:

  torchrun --nproc-per-node N tools/schemes_bench.py [--rows 1000000 --width 64 --density 0.01]

Per rank: the same dense gradient bench.py syncs (shared-core Zipf rows,
omega = 0.5).  Times are CUDA events on the launching stream, median over
steps, max over ranks.  Also reports:
  * profile_sparsity over the ranks' tensors and select_scheme's choice;
  * the device merge_sum throughput (zen_merge_sum, two 640K-entry tensors).
HC at N = 1 has no exchange; run it with N >= 2 (power of two).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--omega", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import numpy as np
    import torch
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_stream(torch.cuda.Stream())
    import bench
    import paper_2309_13254_b200 as zen
    from paper_2309_13254_b200 import schemes
    rows, width = args.rows, args.width
    per = int(np.ceil(args.density * rows))
    m = rows * width
    n = max(world, 2)
    live = bench.live_rows(rows, per, n, args.omega, 1.05, 3)
    mine = torch.from_numpy(bench.dense_gradient(rows, width, live[rank], 3 + rank)).cuda()
    stream = torch.cuda.current_stream()
    out = {"config": f"{rows}x{width}, {args.density:.1%} rows, omega {args.omega}", "n_gpus": world}

    def timed(fn, after=None):
        """device time of fn's enqueue (events on the stream), then `after`
        (the host-side wait / error check) outside the timed region"""
        for _ in range(3):
            fn()
            if after:
                after()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            if after:
                after()
            ts.append(a.elapsed_time(b))
        t = float(np.median(ts))
        if world > 1:
            x = torch.tensor([t], device="cuda", dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            t = float(x.item())
        return round(t, 4)

    if world > 1:
        bp = zen.BPSynchronizer(world, m, max_nnz=per * width + 4096, rank=rank)
        bp.connect_process_group()

        out["bp_ms"] = timed(lambda: bp.sync_dense([mine]), bp.wait)
        if world & (world - 1) == 0:
            hc = zen.HCSynchronizer(world, m, rank, max_nnz=per * width + 4096)
            hc.connect_process_group()

            out["hc_ms"] = timed(lambda: hc.sync_dense(mine), hc.wait)
            hi, hv = hc.result()
            bi, bv = bp.result()
            out["hc_equals_bp"] = bool(torch.equal(hi, bi) and torch.equal(hv.view(torch.int32),
                                                                           bv.view(torch.int32)))
            out["hc_sent_bits_rank0"] = [ib + vb for ib, vb in hc.stage_bits()]
        for scheme in ["ring", "agsparse", "omnireduce"]:
            if scheme == "ring" and world & (world - 1):
                continue
            sy = zen.HCSynchronizer(world, m, rank, max_nnz=per * width + 4096, scheme=scheme)
            sy.connect_process_group()
            out[f"{scheme}_ms"] = timed(lambda: sy.sync_dense(mine), sy.wait)
            si, sv = sy.result()
            bi, bv = bp.result()
            out[f"{scheme}_equals_bp_indices"] = bool(torch.equal(si, bi))
            del sy
    # merge throughput + profile on rank 0's device
    sp = [zen.to_sparse(torch.from_numpy(bench.dense_gradient(rows, width, live[w], 3 + w)).cuda())
          for w in range(n)]
    if rank == 0:
        a, b = (schemes._to_dev(t) for t in sp[:2])
        ms = timed(lambda: schemes._merge_dev(*a, *b, m)) if world == 1 else None
        if ms is None:
            for _ in range(3):
                schemes._merge_dev(*a, *b, m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                schemes._merge_dev(*a, *b, m)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
        u = schemes._merge_dev(*a, *b, m)[0].numel()
        nbytes = 12 * (a[0].numel() + b[0].numel() + u)
        out["merge_sum"] = {"entries_in": a[0].numel() + b[0].numel(), "entries_out": u,
                            "ms_per_call_incl_host_sync": round(ms, 4),
                            "algorithmic_GBps": round(nbytes / ms / 1e6, 1)}
        prof = zen.profile_sparsity([sp])
        out["profile"] = prof.to_json()
        out["select_scheme"] = zen.select_scheme(prof, n)
        out["t_bp_coefficient"] = zen.t_bp_coefficient(n, prof.gamma[n])
        out["t_hc_coefficient"] = zen.t_hc_coefficient(n, prof.gamma)
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
