"""Replicates bench.py's flow (n=1 timed + e2e, then 8 emulated) with checks."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2309_13254_b200 as zen
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
rows, d, per = 1_000_000, 64, 10000
m, z = rows * d, per * d
live = bench.live_rows(rows, per, 1, 0.5, 1.05, 1)
host = bench.dense_gradient(rows, d, live[0], 1)
d1 = torch.from_numpy(host).cuda()
bp = zen.BPSynchronizer(1, m, max_nnz=int(z * 1.25) + 4096)
for _ in range(5): bp.sync_dense([d1])
bp.wait(); bp.stage_times(); bp.enable_timing(True)
for _ in range(20): bp.sync_dense([d1])
torch.cuda.synchronize(); bp.wait(); print("n1", bp.result_count(), bp.stage_times())
bp.enable_timing(False)
pin = torch.from_numpy(host).pin_memory()
oi = torch.empty(z + 16, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
ov = torch.empty(z + 16, dtype=torch.float32).pin_memory().numpy()
if "noe2e" not in sys.argv:
    for _ in range(11): c = bp.sync_host([pin.numpy()], oi, ov)
    print("e2e", c)
if "freebp" in sys.argv:
    del bp
    torch.cuda.synchronize()
def check(be, dd, tag):
    acc = sum(x.double() for x in dd)
    want = torch.nonzero(acc != 0).view(-1)
    be.wait()
    i, v = be.result()
    ok = i.numel() == want.numel() and torch.equal(i, want) and torch.equal(v.double(), acc[i])
    led, counts, agg = be.ledger()
    print(tag, "ok" if ok else "MISMATCH", i.numel(), want.numel(), "agg", agg.tolist(), "rowsums", counts.sum(1).tolist(), flush=True)
    return ok
for rep in range(3):
    ne = 8
    rows_e = bench.live_rows(rows, per, ne, 0.5, 1.05, 1)
    dd = [torch.from_numpy(bench.dense_gradient(rows, d, rows_e[w], 1 + w)).cuda() for w in range(ne)]
    be = zen.BPSynchronizer(ne, m, max_nnz=int(z * 1.25) + 4096)
    be.sync_dense(dd)
    if not check(be, dd, f"rep{rep} first"):
        import ctypes
        owner = zen.partition_of(np.arange(m, dtype=np.uint64), zen.derive_seed(1, 0), ne)
        nwm = (m + 63) // 64
        for s_ in range(2):
            buf = np.empty(nwm * 2, np.uint64)
            c = ctypes.c_uint64()
            zen.load().zen_bp_debug_part(be.h, 3, s_, 0, buf.ctypes.data, buf.ctypes.data, nwm, ctypes.byref(c))
            prefix = (buf[1::2] & 0xFFFFFFFF).astype(np.int64)
            cnt = (owner == s_).reshape(-1, 64).sum(1)
            exp_prefix = np.concatenate([[0], np.cumsum(cnt)[:-1]])
            bad_p = np.nonzero(prefix != exp_prefix)[0]
            popm = np.array([bin(int(x)).count('1') for x in buf[0::2][:4000]])
            print("  server", s_, "prefix bad words", bad_p.size, bad_p[:5], prefix[bad_p[:3]] if bad_p.size else "", exp_prefix[bad_p[:3]] if bad_p.size else "", "popc ok", bool((popm == cnt[:4000]).all()), flush=True)
            bits = np.empty(nwm // 4, np.uint64)
            zen.load().zen_bp_debug_part(be.h, 2, s_, 0, bits.ctypes.data, bits.ctypes.data, bits.size, ctypes.byref(c))
            print("  server", s_, "bitmap popcount", sum(bin(int(x)).count('1') for x in bits[:c.value]), flush=True)
    for _ in range(2): be.sync_dense(dd)
    check(be, dd, f"rep{rep} warm")
    be.enable_timing(True)
    for _ in range(10): be.sync_dense(dd)
    torch.cuda.synchronize()
    check(be, dd, f"rep{rep} timed")
    print(be.stage_times())
    del be, dd
