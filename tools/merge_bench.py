#!/usr/bin/env python3
"""zen_merge_sum (the merge-path kernel of k_merge.cu) on two tensors shaped
like an HC stage of the bench workload: --z entries each, --overlap shared.
Prints per-call wall time (host syncs included) and, with --profile, the
kernel's own duration from CUPTI (diagnostic only).

  python tools/merge_bench.py [--z 640000] [--overlap 0.5] [--profile]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--z", type=int, default=640_000)
    ap.add_argument("--overlap", type=float, default=0.5)
    ap.add_argument("--m", type=int, default=64_000_000)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2309_13254_b200 import schemes
    g = torch.Generator(device="cuda").manual_seed(1)
    z, m = args.z, args.m
    perm = torch.randperm(m, device="cuda", generator=g)
    shared = int(args.overlap * z)
    a = torch.sort(perm[:z]).values
    b = torch.sort(torch.cat([perm[:shared], perm[z:2 * z - shared]])).values
    av = torch.randn(z, device="cuda", generator=g)
    bv = torch.randn(z, device="cuda", generator=g)
    for _ in range(5):
        schemes._merge_dev(a, av, b, bv, m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.iters):
        schemes._merge_dev(a, av, b, bv, m)
    wall = (time.perf_counter() - t0) / args.iters * 1e3
    out = {"z": z, "overlap": args.overlap, "wall_ms_per_call": round(wall, 4)}
    if args.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(10):
                schemes._merge_dev(a, av, b, bv, m)
            torch.cuda.synchronize()
        import re
        ks = {}
        for e in prof.events():
            if e.device_type.name == "CUDA":
                mm = re.search(r"(k_\w+)", e.name)
                nm = mm.group(1) if mm else e.name.split("(")[0].strip()
                ks.setdefault(nm, []).append(e.device_time_total)
        out["kernel_us"] = {k: round(sum(v) / len(v), 2) for k, v in ks.items()}
        u = schemes._merge_dev(a, av, b, bv, m)[0].numel()
        us = next((v for k, v in out["kernel_us"].items() if k.startswith("k_hc_merge")),
                  max(out["kernel_us"].values()))
        out["merge_algorithmic_GBps"] = round(12 * (2 * z + u) / us / 1e3, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
