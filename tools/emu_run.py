#!/usr/bin/env python3
"""Run K local-mode (emulated) BP syncs of the bench workload -- a clean
process for ncu captures of the n-worker kernels.  Diagnostic only."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--syncs", type=int, default=3)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import paper_2309_13254_b200 as zen
    torch.cuda.set_stream(torch.cuda.Stream())
    n = args.workers
    per = int(np.ceil(args.density * args.rows))
    rows = bench.live_rows(args.rows, per, n, 0.5, 1.05, 1)
    dd = [torch.from_numpy(bench.dense_gradient(args.rows, args.width, rows[w], 1 + w)).cuda()
          for w in range(n)]
    z = per * args.width
    bp = zen.BPSynchronizer(n, args.rows * args.width, max_nnz=int(z * 1.25) + 4096,
                            params=zen.HashParams(seed=1))
    for _ in range(args.syncs):
        bp.sync_dense(dd)
    bp.wait()
    print("ok", bp.result_count())


if __name__ == "__main__":
    main()
