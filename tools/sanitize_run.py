#!/usr/bin/env python3
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): every kernel family of the library on small
inputs, each result checked against the C oracle so a sanitizer run also
proves the outputs did not change.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers: the dense BP sync (local mode, n = 4: begin, extraction with the h0
counts, persistent push scatter, claims from the staging, table-scan depth
pass, fallback replay with a tight r2, aggregate/encode, per-chunk bases,
decode; eager and CUDA-graph replays), the sparse-input BP sync, the
standalone hierarchical hash with its layout dump (k_place / k_depth / serial
/ fallback), HashBitmap encode/decode, the wire formats, top-k and merge_sum.
Rank mode (CUDA-IPC peers) is not covered: one process per GPU, and the
peer-flag waits would hit their watchdog under the sanitizer's slowdown.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import torch
    import paper_2309_13254_b200 as zen
    from oracle import COracle
    co = COracle()
    torch.cuda.set_device(0)
    torch.cuda.set_stream(torch.cuda.Stream())
    rng = np.random.default_rng(7)
    rows, d, n = 3000, 64, 4
    m = rows * d
    dense, pairs = [], []
    core = rng.choice(rows, 20, replace=False)
    for _ in range(n):
        live = np.unique(np.concatenate([core, rng.choice(rows, 25, replace=False)]))
        g = np.zeros((rows, d), np.float32)
        g[live] = rng.integers(1, 17, (live.size, d)).astype(np.float32)
        dense.append(torch.from_numpy(g.ravel()).cuda())
        pairs.append(co.to_sparse(g.ravel()))
    for r2r in (0.1, 0.005):  # default sizes, then a fallback-replay r2
        want = co.bp_sync(m, pairs, r2_ratio=r2r)
        bp = zen.BPSynchronizer(n, m, max_nnz=m // 8, params=zen.HashParams(r2_ratio=r2r))
        for _ in range(3):  # eager capture, then graph replays
            bp.sync_dense(dense)
            bp.wait()
            oi, ov = bp.result()
            assert np.array_equal(oi.cpu().numpy().view(np.uint64), want.idx)
            assert np.array_equal(ov.cpu().numpy(), want.val)
        bp.sync_sparse([torch.from_numpy(i.view(np.int64)).cuda() for i, _ in pairs],
                       [torch.from_numpy(v).cuda() for _, v in pairs])
        bp.wait()
        oi, _ = bp.result()
        assert np.array_equal(oi.cpu().numpy().view(np.uint64), want.idx)
        for w in range(n):
            bp.collision_stats(w)
        del bp
    # standalone hash with the layout dump, tight sizes (serial + fallback)
    idx, val = pairs[0]
    fam = zen.HashFamily.make_worker(3, 1, 4, 3)
    r1 = max(1, idx.size // 3)  # loads ~z/4 < r1: no overflow, a tight r2 -> fallback
    got = zen.hash_memory_layout(zen.SparseTensor(m, idx, val), 4, fam, r1, max(1, r1 // 50))
    ref = co.hierarchical_hash(m, idx, val, co.family(3, 4, 3, worker=1), r1, max(1, r1 // 50),
                               layout=True)
    assert np.array_equal(got[2].slots, ref.slots)
    # codec, wire formats, top-k, merge
    t = zen.SparseTensor(m, idx, val)
    table = zen.bp_universe_table(m, n, 1)
    for s in range(n):
        mine = idx[co.partition_of(idx, co.derive_seed(1, 0), n) == s]
        ts = zen.SparseTensor(m, mine, np.ones(mine.size, np.float32))
        assert zen.decode(zen.encode(ts, zen.WireFormat.hash_bitmap(), table.universe(s)),
                          table.universe(s)) == ts
    for f in (zen.WireFormat.coo(), zen.WireFormat.coo(32), zen.WireFormat.bitmap(),
              zen.WireFormat.tensor_block(256)):
        assert zen.decode(zen.encode(t, f)) == t
    zen.sparsify_topk(dense[0], 0.01)
    zen.merge_sum(t, zen.SparseTensor(m, pairs[1][0], pairs[1][1]))
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
