"""Full-size parity at every BASELINE config against the reference itself.

Each case runs the product path (dense fp32 gradients on the device ->
extraction -> hierarchical hash -> push -> aggregate/encode -> pull -> decode,
n workers emulated on one GPU in local mode, the same kernels as rank mode)
and the UNMODIFIED reference compiled in place (`oracle/_ref`,
`zen::run_balanced_parallelism`, zen/schemes.hpp:341-417) on identical inputs,
and compares bit for bit:

* the synchronised result (indices and fp32 value bits),
* the SimNet ledger (sent / received / index / value bits per node and stage),
* the n x n push count matrix (vs the reference's `partition_of`,
  zen/hashing.hpp:85-88) and every server's aggregate size,
* push/pull imbalance (zen/hashing.hpp:296-320),
* every worker's CollisionStats (zen/hashing.hpp:259-262 with the worker's
  own r1/r2, zen/schemes.hpp:363-367).

Configs (SURVEY.md §8d / BASELINE.json):
  C4  1M x 64 at 0.1 %, 1 %, 10 % density, n = 8, row-structured (omega=0.5, Zipf rows)
  C2  1M x 16 at 0.5 %, n = 8, Zipf rows
  C3  800K x 1024 at 1 %, n = 8 (819.2M elements per worker, 26 GB of dense input)
  C4g 1M x 64 at 1 %, n = 8, the reference's own element-granular generator
      (`zen::generate`, zen/workload.hpp:123-154)
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rows_inputs(rows, d, density, n, seed=1, omega=0.5, zipf=1.05):
    import bench
    per = int(np.ceil(density * rows))
    live = bench.live_rows(rows, per, n, omega, zipf, seed)
    pairs = []
    for w in range(n):
        r = np.sort(live[w]).astype(np.uint64)
        idx = (r[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)).ravel()
        val = np.random.default_rng(seed * 7919 + w).integers(1, 17, idx.size).astype(np.float32)
        pairs.append((idx, val))
    return pairs


def _dense_on_device(m, idx, val):
    g = torch.zeros(m, dtype=torch.float32, device="cuda")
    if idx.size:
        g[torch.from_numpy(idx.view(np.int64)).cuda()] = torch.from_numpy(val).cuda()
    return g


def _check_full(zen, co, ro, m, pairs, seed=1, check_stats=True, r2_ratio=0.1):
    n = len(pairs)
    lanes = os.cpu_count() or 1
    zmax = max(i.size for i, _ in pairs)
    bp = zen.BPSynchronizer(n, m, max_nnz=zmax + 4096,
                            params=zen.HashParams(seed=seed, r2_ratio=r2_ratio))
    dense = [_dense_on_device(m, i, v) for i, v in pairs]
    side = torch.cuda.Stream()
    for it in range(2):  # eager capture, then CUDA-graph replay
        with torch.cuda.stream(side):
            bp.sync_dense(dense)
        bp.wait()
    oi, ov = bp.result()
    got_i = oi.cpu().numpy().view(np.uint64)
    got_v = ov.cpu().numpy()
    led, counts, agg = bp.ledger()
    bal = bp.balance()
    stats = [bp.collision_stats(w) for w in range(n)] if check_stats else None
    del dense, oi, ov, bp
    torch.cuda.empty_cache()

    want = ro.bp_sync(m, pairs, seed=seed, lanes=lanes, r2_ratio=r2_ratio)
    np.testing.assert_array_equal(got_i, want.idx)
    np.testing.assert_array_equal(got_v.view(np.uint32), want.val.view(np.uint32))
    np.testing.assert_array_equal(led, want.ledger)
    assert bal is not None and want.balance is not None
    assert bal.push_imbalance == want.balance[0]
    assert bal.pull_imbalance == want.balance[1]
    pseed = ro.derive_seed(seed, 0)
    want_counts = np.stack([np.bincount(ro.partition_of(i, pseed, n), minlength=n)
                            for i, _ in pairs]).astype(counts.dtype)
    np.testing.assert_array_equal(counts, want_counts)
    assert int(agg.sum()) == want.idx.size
    if check_stats:
        for w, (i, v) in enumerate(pairs):
            r1, r2 = co.bp_sizes(2.0, r2_ratio, i.size, n)
            ws = ro.hierarchical_hash(m, i, v, seed, n, 3, r1, r2, worker=w, lanes=lanes)
            assert stats[w].serial_writes == ws.serial_writes, f"worker {w}"
            assert stats[w].placed_at_depth == ws.placed_at_depth, f"worker {w}"
    return want.idx.size


@pytest.mark.parametrize("density", [0.001, 0.01, 0.1])
def test_c4_rows_n8(zen, co, ro, density):
    rows, d = 1_000_000, 64
    u = _check_full(zen, co, ro, rows * d, _rows_inputs(rows, d, density, 8))
    assert u > 0


def test_c2_zipf_n8(zen, co, ro):
    rows, d = 1_000_000, 16
    _check_full(zen, co, ro, rows * d, _rows_inputs(rows, d, 0.005, 8, seed=2, zipf=1.05),
                seed=2)


def test_c4_reference_generator_n8(zen, co, ro):
    """Element-granular inputs from the reference's own generator at M = 64M."""
    m, n = 64_000_000, 8
    pairs = ro.generate(m, n, 0.01, 0.5, 20230923)
    _check_full(zen, co, ro, m, pairs, seed=5)


def test_c3_rows_n8(zen, co, ro):
    """800K x 1024 fp32 at 1 %: 819.2M elements, hash memory far larger than L2."""
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * 2**30:
        pytest.skip("C3 with 8 emulated workers needs ~110 GB of device memory")
    rows, d = 800_000, 1024
    _check_full(zen, co, ro, rows * d, _rows_inputs(rows, d, 0.01, 8, seed=3), seed=3)


def test_c4_tight_r2_fallback_n8(zen, co, ro):
    """r2 = 1 % of r1: every partition has more serial keys than serial slots,
    so the reference's order-dependent fallback scan (zen/hashing.hpp:170-175)
    places the rest -- the exact replay path -- at the headline size."""
    import time
    rows, d = 1_000_000, 64
    t = time.time()
    _check_full(zen, co, ro, rows * d, _rows_inputs(rows, d, 0.01, 8), r2_ratio=0.01)
    print(f"tight-r2 sync + reference check: {time.time() - t:.1f} s")
