#!/usr/bin/env python3
"""Time zen_sparsify_topk (CUDA events, synchronous C-ABI calls) on a sparse
embedding gradient (1M x 64, 1% rows) and on a dense Gaussian layer block
(16 x 1600^2), keep 1%.  Prints one JSON line."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2309_13254_b200 as zen
    lib, ctx = zen.load(), zen.context()
    g = torch.Generator(device="cuda").manual_seed(1)
    emb = torch.zeros(1_000_000, 64, device="cuda")
    live = torch.randperm(1_000_000, device="cuda", generator=g)[:10_000]
    emb[live] = torch.randn(10_000, 64, device="cuda", generator=g)
    lay = torch.randn(16 * 1600 * 1600, device="cuda", generator=g)
    out = {}
    for name, d in [("sparse_64M", emb.view(-1)), ("gauss_41M", lay)]:
        m = d.numel()
        keep = int(np.ceil(0.01 * m))
        oi = torch.empty(keep, dtype=torch.int64, device="cuda")
        ov = torch.empty(keep, dtype=torch.float32, device="cuda")
        got = C.c_uint64()

        def call():
            assert lib.zen_sparsify_topk(ctx.h, C.c_void_p(d.data_ptr()), m, 0.01,
                                         C.c_void_p(oi.data_ptr()), C.c_void_p(ov.data_ptr()),
                                         keep, C.byref(got)) == 0
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) / 20, 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
