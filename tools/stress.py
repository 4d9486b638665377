"""Repeat BP syncs and verify each result (union size + exact sums) -- race hunting."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2309_13254_b200 as zen
torch.cuda.set_stream(torch.cuda.Stream())
rows, d = 1_000_000, 64
per = 10000; z = per * d; m = rows * d
bad = 0
for ne in [8, 1, 4]:
    rows_e = bench.live_rows(rows, per, ne, 0.5, 1.05, 7)
    dd = [torch.from_numpy(bench.dense_gradient(rows, d, rows_e[w], 7 + w)).cuda() for w in range(ne)]
    acc = sum(x.double() for x in dd)
    want_idx = torch.nonzero(acc != 0).view(-1)
    be = zen.BPSynchronizer(ne, m, max_nnz=int(z * 1.25) + 4096)
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
        be.enable_timing(it % 2 == 0)
        be.sync_dense(dd)
        if it % 10 == 9 or it < 3:
            be.wait()
            oi, ov = be.result()
            ok = oi.numel() == want_idx.numel() and torch.equal(oi, want_idx) and torch.equal(ov.double(), acc[oi])
            if not ok:
                bad += 1
                print("MISMATCH n", ne, "it", it, oi.numel(), want_idx.numel(), flush=True)
            be.stage_times()
    be.wait()
    print("n", ne, "done", flush=True)
    del be
print("bad", bad)
