"""Create several n=8 local synchronisers at 1M x 64 and check each; dump diagnostics on failure."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import bench, paper_2309_13254_b200 as zen
from oracle import COracle
torch.cuda.set_stream(torch.cuda.Stream())
rows, d, per, ne = 1_000_000, 64, 10000, 8
m, z = rows * d, per * d
rows_e = bench.live_rows(rows, per, ne, 0.5, 1.05, 1)
dd = [torch.from_numpy(bench.dense_gradient(rows, d, rows_e[w], 1 + w)).cuda() for w in range(ne)]
acc = sum(x.double() for x in dd); want = torch.nonzero(acc != 0).view(-1)
pseed = zen.derive_seed(1, 0)
owner = None
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    be = zen.BPSynchronizer(ne, m, max_nnz=int(z * 1.25) + 4096)
    be.sync_dense(dd); be.wait()
    i, v = be.result()
    ok = i.numel() == want.numel() and torch.equal(i, want)
    led, counts, agg = be.ledger()
    print("rep", rep, "ok" if ok else "MISMATCH", i.numel(), agg.tolist(), flush=True)
    if not ok:
        if owner is None:
            owner = zen.partition_of(np.arange(m, dtype=np.uint64), pseed, ne)
        for s in range(2):
            own = np.empty(2 * ((m + 63) // 64), np.uint64)
            oi = np.empty(4 * ((m + 63) // 64), np.uint32)
            r = be.debug_part(3, s, 0, 4 * ((m + 63) // 64))
            raw = r[0].view(np.uint64).reshape(-1, 2) if False else None
            import ctypes
            buf = np.empty(((m + 63) // 64) * 2, np.uint64)
            c = ctypes.c_uint64()
            zen.load().zen_bp_debug_part(be.h, 3, s, 0, buf.ctypes.data, buf.ctypes.data, (m + 63) // 64, ctypes.byref(c))
            mask = buf[0::2]; prefix = (buf[1::2] & 0xFFFFFFFF).astype(np.int64)
            o = (owner == s).reshape(-1, 64)
            wm = (o * (1 << np.arange(64, dtype=np.uint64))).sum(1, dtype=np.uint64) if False else None
            cnt = o.sum(1)
            exp_prefix = np.concatenate([[0], np.cumsum(cnt)[:-1]])
            bad_p = np.nonzero(prefix != exp_prefix)[0]
            popm = np.array([bin(int(x)).count('1') for x in mask[:2000]])
            print("  server", s, "prefix bad words", bad_p.size, bad_p[:5], "popc ok(first2000)", bool((popm == cnt[:2000]).all()), flush=True)
            bits = np.empty((m // 64) // 8 + 64, np.uint64)
            zen.load().zen_bp_debug_part(be.h, 2, s, 0, bits.ctypes.data, bits.ctypes.data, bits.size, ctypes.byref(c))
            nw = c.value
            ones = sum(bin(int(x)).count('1') for x in bits[:nw])
            print("  server", s, "bitmap words", nw, "popcount", ones, flush=True)
    del be
