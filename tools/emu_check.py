import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2309_13254_b200 as zen
torch.cuda.set_stream(torch.cuda.Stream())
rows, d, ne = 1_000_000, 64, 8
per = 10000; z = per * d; m = rows * d
# main n=1 synchronizer first (as in bench)
live1 = bench.live_rows(rows, per, 1, 0.5, 1.05, 1)
d1 = torch.from_numpy(bench.dense_gradient(rows, d, live1[0], 1)).cuda()
bp = zen.BPSynchronizer(1, m, max_nnz=int(z * 1.25) + 4096)
for _ in range(5): bp.sync_dense([d1])
bp.wait(); print("n1 union", bp.result_count())
rows_e = bench.live_rows(rows, per, ne, 0.5, 1.05, 1)
dd = [torch.from_numpy(bench.dense_gradient(rows, d, rows_e[w], 1 + w)).cuda() for w in range(ne)]
nzr = np.zeros(rows, bool)
for w in range(ne): nzr[rows_e[w]] = True
want = int(nzr.sum()) * d
be = zen.BPSynchronizer(ne, m, max_nnz=int(z * 1.25) + 4096)
for it in range(3):
    be.sync_dense(dd); be.wait(); print("warm", it, be.result_count(), want)
be.enable_timing(True)
for it in range(10):
    be.sync_dense(dd)
torch.cuda.synchronize(); be.wait()
print("timed", be.result_count(), want, be.stage_times())
be.enable_timing(False)
for it in range(3):
    be.sync_dense(dd); be.wait(); print("after", it, be.result_count(), want)
