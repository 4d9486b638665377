"""GPU parity: the sm_100a path through the C-ABI against the oracle.

Bit-exact for partition assignment, slot placement (lanes=1 layout), serial
region contents, CollisionStats, overflow partition, part contents, hash
bitmap payload bytes and output index sets; values are bit-exact too because
the aggregation folds workers in the reference's order (the north-star
tolerance, 1e-6 relative, is asserted where float inputs are used).
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import OracleError

pytestmark = pytest.mark.gpu
U64MAX = 2**64 - 1
RTOL = 1e-6  # north_star: fp32 aggregated values within 1e-6 relative


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


# ---------------------------------------------------------------- hashing ----

def test_partition_of_known_answers(zen):
    g = load_golden("hash_kat")
    idx = g["part_idx"]
    for pseed, n in g["part_cases"]:
        got = zen.partition_of(idx, int(pseed), int(n))
        np.testing.assert_array_equal(got, g[f"part_{pseed}_{n}"])


def test_hierarchical_hash_golden_layout(zen):
    g = load_golden("hhash")
    for i in range(int(g["ncases"][0])):
        p = f"c{i}_"
        m, seed, worker, n, k, r1, r2 = (int(v) for v in g[p + "meta"])
        fam = (zen.HashFamily.make(seed, n, k) if worker < 0 else
               zen.HashFamily.make_worker(seed, worker, n, k))
        t = zen.SparseTensor(m, g[p + "idx"], g[p + "val"])
        ovf = int(g[p + "overflow"][0])
        if ovf >= 0:
            with pytest.raises(zen.SerialOverflow) as e:
                zen.hierarchical_hash(t, n, fam, r1, r2)
            assert e.value.partition() == ovf, f"case {i}"
            continue
        parts, stats, lay = zen.hash_memory_layout(t, n, fam, r1, r2)
        np.testing.assert_array_equal(lay.slots, g[p + "slots"], err_msg=f"case {i}")
        np.testing.assert_array_equal(bits(lay.slot_values), bits(g[p + "slot_vals"]))
        np.testing.assert_array_equal(lay.depth, g[p + "depth"], err_msg=f"case {i}")
        got_idx = np.concatenate([q.indices() for q in parts.parts])
        got_val = np.concatenate([q.values() for q in parts.parts])
        np.testing.assert_array_equal(got_idx, g[p + "parts_idx"])
        np.testing.assert_array_equal(bits(got_val), bits(g[p + "parts_val"]))
        assert [q.nnz() for q in parts.parts] == list(g[p + "part_count"])
        assert [stats.serial_writes] + stats.placed_at_depth == list(g[p + "stats"])


def test_hierarchical_hash_random_vs_oracle(zen, co):
    rng = np.random.default_rng(5)
    for trial in range(40):
        m = int(rng.integers(100, 3_000_000))
        z = int(rng.integers(0, min(m // 2, 60_000) + 1))
        idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
        val = rng.standard_normal(z).astype(np.float32)
        n = int(rng.choice([1, 2, 3, 4, 5, 8, 16, 31, 64]))
        k = int(rng.integers(1, 6))
        mult = float(rng.choice([0.5, 1.0, 2.0, 4.0]))
        r1 = max(1, int(np.ceil(mult * z / n)))
        r2 = max(1, int(np.ceil(float(rng.choice([0.05, 0.1, 0.5])) * r1)))
        seed, w = int(rng.integers(0, 2**62)), int(rng.integers(0, 16))
        fam = zen.HashFamily.make_worker(seed, w, n, k)
        cfam = co.family(seed, n, k, worker=w)
        t = zen.SparseTensor(m, idx, val)
        try:
            want = co.hierarchical_hash(m, idx, val, cfam, r1, r2, layout=True)
        except OracleError as e:
            with pytest.raises(zen.SerialOverflow) as ge:
                zen.hierarchical_hash(t, n, fam, r1, r2)
            assert ge.value.partition() == e.partition
            continue
        parts, stats, lay = zen.hash_memory_layout(t, n, fam, r1, r2)
        np.testing.assert_array_equal(lay.slots, want.slots, err_msg=f"trial {trial}")
        np.testing.assert_array_equal(lay.depth, want.depth_of)
        np.testing.assert_array_equal(bits(lay.slot_values), bits(want.slot_vals))
        assert stats.serial_writes == want.serial_writes
        assert stats.placed_at_depth == want.placed_at_depth
        for q, wi, wv in zip(parts.parts, want.parts_idx, want.parts_val):
            np.testing.assert_array_equal(q.indices(), wi)
            np.testing.assert_array_equal(bits(q.values()), bits(wv))


def test_hierarchical_hash_c2_no_loss_and_invariance(zen, co):
    """acceptance C2 (acceptance.cpp:201-250) shape: M=1e6, d=1%, n=16; union == input."""
    rng = np.random.default_rng(777)
    m, nnz, n = 1_000_000, 10_000, 16
    r1, r2 = 2 * nnz // n, (2 * nnz // n) // 10
    for trial in range(25):
        idx = np.sort(rng.choice(m, nnz, replace=False)).astype(np.uint64)
        val = (1 + idx % 13).astype(np.float32)
        fam = zen.HashFamily.make_worker(trial, trial % 7, n, 3)
        t = zen.SparseTensor(m, idx, val)
        parts = zen.hierarchical_hash(t, n, fam, r1, r2)
        np.testing.assert_array_equal(np.sort(np.concatenate([p.indices() for p in parts.parts])), idx)
        # lane-count invariance: lanes is accepted; the layout is the lanes=1 one on every call
        again = zen.hierarchical_hash(t, n, fam, r1, r2, lanes=8)
        assert all(a == b for a, b in zip(parts.parts, again.parts))


def test_priority_claim_is_schedule_invariant(zen, co):
    """The lock-free priority claim has ONE outcome (deferred
    acceptance with a common priority order = serial dictatorship in ascending
    key order = the reference's lanes=1 greedy, zen/hashing.hpp:155-179), for
    any thread schedule: vary the claim kernel's grid and block size and the
    order in which keys claim (a permutation), and compare every slot with
    the oracle's sequential layout."""
    import ctypes as C
    from paper_2309_13254_b200 import _lib as L
    lib = L.load()
    rng = np.random.default_rng(11)
    m, z, n, k = 200_000, 20_000, 4, 3
    idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
    val = rng.standard_normal(idx.size).astype(np.float32)
    fam = zen.HashFamily.make(9, n, k)
    r1, r2 = 6_000, 600  # tight: many displacements, serial keys and a fallback-free run
    want = co.hierarchical_hash(m, idx, val, co.family(9, n, k), r1, r2, layout=True)
    schedules = [(0, 0, 0, 0), (1, 32, 0, 0), (3, 64, 7919, 13), (148, 256, 0, 0),
                 (37, 96, 104729, 5), (2000, 256, 1_000_003, 17), (5, 160, z - 1, 0)]
    try:
        for g, t, mul, add in schedules:
            assert lib.zen_debug_hash_schedule(g, t, mul, add) == 0
            parts, stats, lay = zen.hash_memory_layout(zen.SparseTensor(m, idx, val), n, fam, r1, r2)
            np.testing.assert_array_equal(lay.slots, want.slots, err_msg=f"schedule {g, t, mul, add}")
            np.testing.assert_array_equal(lay.depth, want.depth_of)
            assert stats.serial_writes == want.serial_writes
            assert stats.placed_at_depth == want.placed_at_depth
    finally:
        lib.zen_debug_hash_schedule(0, 0, 0, 0)


def test_to_sparse_golden(zen):
    g = load_golden("to_sparse")
    for name in ["mixed", "rows", "one", "allnz"]:
        t = zen.to_sparse(g[name + "_dense"])
        np.testing.assert_array_equal(t.indices(), g[name + "_idx"])
        np.testing.assert_array_equal(bits(t.values()), bits(g[name + "_val"]))


@pytest.mark.parametrize("m", [1, 7, 8191, 8192, 8193, 1_000_003, 6_400_000])
def test_to_sparse_sizes_and_alignment(zen, co, m):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(m)
    d = rng.standard_normal(m).astype(np.float32)
    d[rng.random(m) < 0.9] = 0.0
    d[rng.random(m) < 0.01] = -0.0
    want_i, want_v = co.to_sparse(d)
    t = zen.to_sparse(d)
    np.testing.assert_array_equal(t.indices(), want_i)
    np.testing.assert_array_equal(bits(t.values()), bits(want_v))
    if m > 8:  # misaligned base pointer: scalar path
        dd = torch.from_numpy(np.concatenate([[0.0], d]).astype(np.float32)).cuda()[1:]
        t2 = zen.to_sparse(dd)
        np.testing.assert_array_equal(t2.indices(), want_i)


# ------------------------------------------------------------------ codec ----

def test_universe_sizes_and_lists(zen, co):
    g = load_golden("codec")
    for row in g["universe_sizes"]:
        m, n, pseed = (int(v) for v in row[:3])
        tab = zen.HashUniverseTable(m, n, pseed)
        assert [tab.size(s) for s in range(n)] == [int(v) for v in row[3:3 + n]]
    for (m, n, pseed) in [(15, 3, 4), (1000, 7, 12345), (100_003, 16, 99), (64, 1, 5)]:
        tab = zen.HashUniverseTable(m, n, pseed)
        u = co.universe(m, n, pseed)
        for s in range(n):
            np.testing.assert_array_equal(tab.universe(s).indices, u.indices(s))
        assert sum(tab.size(s) for s in range(n)) == m


def test_hash_bitmap_fig7_worked_example(zen):
    g = load_golden("codec")
    seed, nbits = (int(v) for v in g["fig7"])
    tab = zen.HashUniverseTable(15, 3, seed)
    t = zen.SparseTensor(15, [5, 7], [0.3, 0.9])
    msg = zen.encode(t, zen.WireFormat.hash_bitmap(), tab.universe(0))
    assert msg.index_bits == nbits and msg.payload[0] & 0b111 == 0b110
    np.testing.assert_array_equal(msg.payload, g["fig7_payload"])
    assert zen.decode(msg, tab.universe(0)) == t


def test_hash_bitmap_golden_payloads(zen):
    g = load_golden("codec")
    for i in range(int(g["ncases"][0])):
        p = f"e{i}_"
        m, n, pseed, s, nbits = (int(v) for v in g[p + "meta"])
        tab = zen.HashUniverseTable(m, n, pseed)
        t = zen.SparseTensor(m, g[p + "idx"], g[p + "val"])
        msg = zen.encode(t, zen.WireFormat.hash_bitmap(), tab.universe(s))
        assert msg.index_bits == nbits
        np.testing.assert_array_equal(msg.payload, g[p + "payload"])
        back = zen.decode(msg, tab.universe(s))
        assert back == t


def test_hash_bitmap_errors(zen):
    tab = zen.HashUniverseTable(100, 4, 9)
    own0 = set(tab.universe(0).indices.tolist())
    foreign = next(i for i in range(100) if i not in own0)
    with pytest.raises(zen.IndexOutsideUniverse):
        zen.encode(zen.SparseTensor(100, [foreign], [1.0]), zen.WireFormat.hash_bitmap(),
                   tab.universe(0))
    t = zen.SparseTensor(100, sorted(own0)[:2], [1.0, 2.0])
    msg = zen.encode(t, zen.WireFormat.hash_bitmap(), tab.universe(0))
    msg.payload = msg.payload[:-1]
    with pytest.raises(zen.MalformedPayload):
        zen.decode(msg, tab.universe(0))
    msg = zen.encode(t, zen.WireFormat.hash_bitmap(), tab.universe(0))
    msg.count = 3
    msg.payload = np.concatenate([msg.payload, np.zeros(4, np.uint8)])
    with pytest.raises(zen.MalformedPayload):
        zen.decode(msg, tab.universe(0))


# --------------------------------------------------- balanced parallelism ----

def _inputs(zen, m, pairs):
    return [zen.SparseTensor(m, i, v) for i, v in pairs]


def test_bp_golden(zen):
    g = load_golden("bp")
    for i in range(int(g["ncases"][0])):
        p = f"b{i}_"
        n, m, gseed, seed, k = (int(v) for v in g[p + "meta"])
        r1m, r2r, _, _ = (float(v) for v in g[p + "params"])
        ins = _inputs(zen, m, [(g[p + f"in{w}_idx"], g[p + f"in{w}_val"]) for w in range(n)])
        params = zen.HashParams(k, r1m, r2r, 1, seed)
        code, part = (int(v) for v in g[p + "error"])
        net = zen.SimNet(n, 1.0)
        if code:
            with pytest.raises(zen.SerialOverflow) as e:
                zen.run_balanced_parallelism(ins, net, params)
            assert e.value.partition() == part
            continue
        out = zen.run_balanced_parallelism(ins, net, params)
        for r in out.results:
            np.testing.assert_array_equal(r.indices(), g[p + "idx"], err_msg=f"case {i}")
            np.testing.assert_array_equal(bits(r.values()), bits(g[p + "val"]))
        led = g[p + "ledger"]
        for st in range(2):
            assert out.traffic.stages[st].sent_bits == list(led[st, 0])
            assert out.traffic.stages[st].recv_bits == list(led[st, 1])
            assert out.traffic.stages[st].recv_index_bits == list(led[st, 2])
            assert out.traffic.stages[st].recv_value_bits == list(led[st, 3])
        want_bal = g[p + "balance"]
        if np.isnan(want_bal[0]):
            assert out.balance is None
        else:
            assert out.balance.push_imbalance == want_bal[0]
            assert out.balance.pull_imbalance == want_bal[1]


@pytest.mark.parametrize("n", [2, 3, 4, 8, 16])
def test_bp_random_vs_reference(zen, co, ro, n):
    """schemes_test OracleEqualAcrossNodeCounts (schemes_test.cpp:264-276), scaled up."""
    rng = np.random.default_rng(47 + n)
    for trial in range(3):
        m = int(rng.choice([20_000, 250_000, 1_000_000]))
        ins_np = ro.generate(m, n, 0.005 * (1 + trial), 0.5, int(rng.integers(0, 2**62)))
        seed = int(rng.integers(0, 2**62))
        want = ro.bp_sync(m, ins_np, seed=seed)
        out = zen.run_balanced_parallelism(_inputs(zen, m, ins_np), zen.SimNet(n, 1.0),
                                           zen.HashParams(seed=seed))
        np.testing.assert_array_equal(out.results[0].indices(), want.idx)
        np.testing.assert_array_equal(bits(out.results[0].values()), bits(want.val))
        for st in range(2):
            assert out.traffic.stages[st].recv_bits == list(want.ledger[st, 1])


def test_bp_float_values_within_tolerance(zen, co):
    rng = np.random.default_rng(3)
    m, n = 500_000, 8
    pairs = []
    core = rng.choice(m, 2000, replace=False)
    for w in range(n):
        extra = rng.choice(m, 3000, replace=False)
        idx = np.unique(np.concatenate([core, extra])).astype(np.uint64)
        pairs.append((idx, rng.uniform(-1, 1, idx.size).astype(np.float32)))
    want = co.bp_sync(m, pairs, seed=2)
    out = zen.run_balanced_parallelism(_inputs(zen, m, pairs), zen.SimNet(n, 1.0),
                                       zen.HashParams(seed=2))
    np.testing.assert_array_equal(out.results[0].indices(), want.idx)
    np.testing.assert_allclose(out.results[0].values(), want.val, rtol=RTOL, atol=0)


def test_bp_edge_cases(zen, co):
    # empty inputs synchronise to empty, balance unset (schemes_test.cpp:376-384)
    ins = [zen.SparseTensor(1000, [], []) for _ in range(4)]
    out = zen.run_balanced_parallelism(ins, zen.SimNet(4, 1.0))
    assert all(r.nnz() == 0 for r in out.results) and out.balance is None
    # one empty worker among loaded ones
    ins = [zen.SparseTensor(5000, [1, 2, 3], [1, 2, 3]), zen.SparseTensor(5000, [], [])]
    out = zen.run_balanced_parallelism(ins, zen.SimNet(2, 1.0))
    assert out.results[0].indices().tolist() == [1, 2, 3] and out.balance is None
    # zero sums are kept (merge_sum never filters, tensor.hpp:151-156)
    ins = [zen.SparseTensor(100, [7, 9], [1.5, 2.0]), zen.SparseTensor(100, [7], [-1.5])]
    out = zen.run_balanced_parallelism(ins, zen.SimNet(2, 1.0))
    assert out.results[0].indices().tolist() == [7, 9]
    assert out.results[0].values().tolist() == [0.0, 2.0]
    # n < 2 and universe mismatch are rejected like the reference (schemes.hpp:65-70)
    with pytest.raises(zen.Error):
        zen.run_balanced_parallelism([zen.SparseTensor(10, [1], [1])], zen.SimNet(1, 1.0))
    with pytest.raises(zen.UniverseMismatch):
        zen.run_balanced_parallelism([zen.SparseTensor(10, [1], [1]),
                                      zen.SparseTensor(11, [1], [1])], zen.SimNet(2, 1.0))


def test_bp_identical_tensors_pull_index_bits(zen, ro):
    """schemes_test.cpp:249-262: total pull index bits = (n-1) * M."""
    m, n = 4096, 4
    ins = ro.generate(m, n, 0.02, 1.0, 43)
    out = zen.run_balanced_parallelism(_inputs(zen, m, ins), zen.SimNet(n, 1.0))
    assert sum(out.traffic.stages[1].recv_index_bits) == 3 * m


def test_bp_retry_policy(zen, ro):
    """run_bp_with_retry doubles r2_ratio after SerialOverflow (experiment.hpp:128-140)."""
    m, n = 1000, 2
    ins = ro.generate(m, n, 0.1, 0.0, 53)
    p = zen.HashParams(r1_multiplier=0.5, r2_ratio=0.1)
    with pytest.raises(OracleError):  # needs the retries
        ro.bp_sync(m, ins, r1_multiplier=0.5, r2_ratio=0.1)
    with pytest.raises(zen.SerialOverflow):
        zen.run_balanced_parallelism(_inputs(zen, m, ins), zen.SimNet(n, 1.0), p)
    want = ro.bp_sync(m, ins, r1_multiplier=0.5, r2_ratio=0.1, retries=4)
    out = zen.run_bp_with_retry(_inputs(zen, m, ins), 1.0, p)
    np.testing.assert_array_equal(out.results[0].indices(), want.idx)
    np.testing.assert_array_equal(bits(out.results[0].values()), bits(want.val))


def test_bp_dense_pipeline_rows(zen, co):
    """Dense fp32 embedding gradients -> extraction -> full BP, vs the oracle."""
    torch = pytest.importorskip("torch")
    rows, d, n = 20_000, 64, 4
    m = rows * d
    rng = np.random.default_rng(9)
    dense, pairs = [], []
    core = rng.choice(rows, 100, replace=False)
    for w in range(n):
        live = np.unique(np.concatenate([core, rng.choice(rows, 100, replace=False)]))
        g = np.zeros((rows, d), np.float32)
        g[live] = rng.integers(1, 17, (live.size, d)).astype(np.float32)
        dense.append(torch.from_numpy(g.ravel()).cuda())
        pairs.append(co.to_sparse(g.ravel()))
    want = co.bp_sync(m, pairs, seed=1)
    bp = zen.BPSynchronizer(n, m, max_nnz=rows * d // 10)
    side = torch.cuda.Stream()
    for it in range(4):  # repeated syncs reuse epochs; it >= 2 replays the CUDA graph
        if it < 2:
            bp.sync_dense(dense)
        else:
            with torch.cuda.stream(side):
                bp.sync_dense(dense)
        bp.wait()
        oi, ov = bp.result()
        np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint64), want.idx)
        np.testing.assert_array_equal(bits(ov.cpu().numpy()), bits(want.val))
        led, counts, agg = bp.ledger()
        np.testing.assert_array_equal(led, want.ledger)
        np.testing.assert_array_equal(counts, want.counts)
        np.testing.assert_array_equal(agg, want.agg_counts)
    # end to end from host buffers
    hi, hv = np.empty(m, np.uint64), np.empty(m, np.float32)
    c = bp.sync_host([x.cpu().numpy() for x in dense], hi, hv)
    np.testing.assert_array_equal(hi[:c], want.idx)
    np.testing.assert_array_equal(bits(hv[:c]), bits(want.val))


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("n", [1, 2, 5])
def test_bp_dense_aggregate_paths(zen, co, monkeypatch, fused, n):
    """Both aggregates of the dense path -- the fused one-block-per-8-tiles kernel
    (k_agg_fused, group ranges from the push scatter + look-back) and the
    three-kernel mark/union/values -- against the oracle, on a universe whose
    size is not a multiple of the group, the word or the chunk (so the groups'
    words straddle and the last group is partial)."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("ZEN_AGG_FUSED", fused)
    rows, d = 30_011, 17
    m = rows * d
    rng = np.random.default_rng(40 + n)
    dense, pairs = [], []
    core = rng.choice(rows, 300, replace=False)
    for w in range(n):
        live = np.unique(np.concatenate([core, rng.choice(rows, 900, replace=False)]))
        g = np.zeros((rows, d), np.float32)
        g[live] = rng.integers(1, 17, (live.size, d)).astype(np.float32)
        g.ravel()[rng.choice(m, 2000, replace=False)] = 3.0  # scattered singletons
        dense.append(torch.from_numpy(g.ravel()).cuda())
        pairs.append(co.to_sparse(g.ravel()))
    # (the reference's BP needs n >= 2, zen/schemes.hpp:66; n = 1 is the input itself)
    want = co.bp_sync(m, pairs, seed=1) if n > 1 else None
    want_idx, want_val = (want.idx, want.val) if n > 1 else pairs[0]
    bp = zen.BPSynchronizer(n, m, max_nnz=m // 4)
    for _ in range(3):  # eager, then graph replays (look-back tags per sync)
        bp.sync_dense(dense)
        bp.wait()
        oi, ov = bp.result()
        np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint64), want_idx)
        np.testing.assert_array_equal(bits(ov.cpu().numpy()), bits(want_val))
        if n > 1:
            led, counts, agg = bp.ledger()
            np.testing.assert_array_equal(led, want.ledger)
            np.testing.assert_array_equal(agg, want.agg_counts)


@pytest.mark.parametrize("density", [0.01, 0.1, 0.5])
def test_bp_single_worker_full_rows(zen, co, density):
    """n = 1 with 64-wide rows (every non-empty bitmap word full: the decode's
    word-by-word path) mixed with a few partial rows (the generic path), vs the
    oracle; two syncs (graph replay)."""
    torch = pytest.importorskip("torch")
    rows, d = 200_000, 64
    m = rows * d
    rng = np.random.default_rng(int(density * 1000))
    g = np.zeros((rows, d), np.float32)
    live = rng.choice(rows, int(rows * density), replace=False)
    g[live] = rng.standard_normal((live.size, d)).astype(np.float32)
    part = rng.choice(rows, 50, replace=False)
    g[part, : d // 2] = 0.0  # some half rows
    dense = torch.from_numpy(g.ravel()).cuda()
    want_i, want_v = co.to_sparse(g.ravel())
    bp = zen.BPSynchronizer(1, m, max_nnz=want_i.size + 4096)
    for _ in range(2):
        bp.sync_dense([dense])
        bp.wait()
        oi, ov = bp.result()
        np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint64), want_i)
        np.testing.assert_array_equal(bits(ov.cpu().numpy()), bits(want_v))


def test_bp_single_worker_pipeline(zen, co):
    """n = 1 (the 1-GPU bench case): extraction + hash + self aggregate/encode/decode."""
    torch = pytest.importorskip("torch")
    m = 1_000_000
    rng = np.random.default_rng(1)
    g = np.zeros(m, np.float32)
    nz = rng.choice(m, 10_000, replace=False)
    g[nz] = rng.standard_normal(nz.size).astype(np.float32)
    bp = zen.BPSynchronizer(1, m, max_nnz=20_000)
    bp.sync_dense([torch.from_numpy(g).cuda()])
    bp.wait()
    oi, ov = bp.result()
    want_i, want_v = co.to_sparse(g)
    np.testing.assert_array_equal(oi.cpu().numpy().view(np.uint64), want_i)
    np.testing.assert_array_equal(bits(ov.cpu().numpy()), bits(want_v))
    st = bp.collision_stats(0)
    fam = co.family(1, 1, 3, worker=0)
    r1, r2 = co.bp_sizes(2.0, 0.1, want_i.size, 1)
    ref = co.hierarchical_hash(m, want_i, want_v, fam, r1, r2)
    assert st.serial_writes == ref.serial_writes and st.placed_at_depth == ref.placed_at_depth


@pytest.mark.parametrize("rehash", [None, "1"])
def test_bp_dense_collision_stats_probe_bits(zen, co, ro, monkeypatch, rehash):
    """Dense syncs, CollisionStats vs the reference's collision_stats with the
    claiming probe packed in the slot words (default) and with the readers
    re-hashing instead (ZEN_SLOT_REHASH=1, the path for M >= 2^30 - 1)."""
    torch = pytest.importorskip("torch")
    if rehash:
        monkeypatch.setenv("ZEN_SLOT_REHASH", rehash)
    rows, d, n = 40_000, 32, 3
    m = rows * d
    rng = np.random.default_rng(77)
    dense, pairs = [], []
    for w in range(n):
        live = rng.choice(rows, 2500, replace=False)
        g = np.zeros((rows, d), np.float32)
        g[live] = rng.integers(1, 17, (live.size, d)).astype(np.float32)
        dense.append(torch.from_numpy(g.ravel()).cuda())
        pairs.append(co.to_sparse(g.ravel()))
    # a tight r1 multiplier: long displacement chains, many serial keys
    params = zen.HashParams(seed=5, r1_multiplier=1.1)
    bp = zen.BPSynchronizer(n, m, max_nnz=m // 4, params=params)
    for _ in range(2):
        bp.sync_dense(dense)
        bp.wait()
    for w in range(n):
        r1, r2 = co.bp_sizes(1.1, 0.1, pairs[w][0].size, n)
        want = ro.hierarchical_hash(m, pairs[w][0], pairs[w][1], 5, n, 3, r1, r2, worker=w)
        st = bp.collision_stats(w)
        assert st.serial_writes == want.serial_writes
        assert st.placed_at_depth == want.placed_at_depth


def test_bp_collision_stats_match_reference(zen, co, ro):
    m, n = 200_000, 4
    ins = ro.generate(m, n, 0.01, 0.5, 5)
    bp = zen.BPSynchronizer(n, m, max_nnz=4000, params=zen.HashParams(seed=3))
    import torch
    bp.sync_sparse([torch.from_numpy(i.view(np.int64)).cuda() for i, _ in ins],
                   [torch.from_numpy(v).cuda() for _, v in ins])
    bp.wait()
    for w in range(n):
        r1, r2 = co.bp_sizes(2.0, 0.1, ins[w][0].size, n)
        want = ro.hierarchical_hash(m, ins[w][0], ins[w][1], 3, n, 3, r1, r2, worker=w)
        st = bp.collision_stats(w)
        assert st.serial_writes == want.serial_writes
        assert st.placed_at_depth == want.placed_at_depth


@pytest.mark.parametrize("n,rows", [(8, 1_000_000), (3, 400_000)])
def test_bp_full_size_properties(zen, n, rows):
    """BASELINE-size local sync (1M x 64 fp32, 1%/worker, n=8 emulated on one GPU)
    checked through size-independent properties: the result index set is the
    union of the inputs and every value is the exact integer sum."""
    torch = pytest.importorskip("torch")
    import bench
    d = 64
    per = int(np.ceil(0.01 * rows))
    live = bench.live_rows(rows, per, n, 0.5, 1.05, 1)
    dense = [torch.from_numpy(bench.dense_gradient(rows, d, live[w], 1 + w)).cuda() for w in range(n)]
    bp = zen.BPSynchronizer(n, rows * d, max_nnz=per * d + 4096)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        bp.sync_dense(dense)
        bp.sync_dense(dense)  # graph replay
    bp.wait()
    oi, ov = bp.result()
    acc = torch.zeros(rows * d, dtype=torch.float64, device="cuda")
    for x in dense:
        acc += x.double()
    nzr = torch.zeros(rows, dtype=torch.bool, device="cuda")
    for w in range(n):
        nzr[torch.from_numpy(live[w]).cuda()] = True
    want_idx = (torch.nonzero(nzr).view(-1, 1) * d + torch.arange(d, device="cuda")).view(-1)
    assert oi.numel() == want_idx.numel()
    assert torch.equal(oi, want_idx)
    assert torch.equal(ov.double(), acc[oi])
    led, counts, agg = bp.ledger()
    assert int(agg.sum()) == oi.numel()
    assert int(counts.sum()) == sum(int(torch.count_nonzero(x)) for x in dense)


def test_cpp_compat_dropin(zen):
    """The reference's own hashing/codec/schemes test cases through the C++
    drop-in header (tests/cpp/compat_test.cpp, built by `make compat_test`)."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "build", "compat_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "compat_test"], check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:]


@pytest.mark.parametrize("suite", ["hashing", "tensor", "codec", "simnet", "workload",
                                   "costmodel", "schemes"])
def test_reference_unit_suite_unmodified(zen, suite):
    """The reference's OWN GTest suite (proj/tests/<suite>_test.cpp), compiled
    unmodified against the drop-in by `make ref_tests` (zen/*.hpp -> compat.hpp
    with `namespace zen = zen_b200;`, a GTest shim) in the build container and
    run here on the B200."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "build", f"ref_{suite}_test")
    if not os.path.exists(exe):
        pytest.skip("built only where /root/reference exists (make ref_tests)")
    # schemes_test's OracleEqualAcrossNodeCounts asserts no SerialOverflow on
    # n = 16 workers of 100 entries (r1 = 13, r2 = 2 per partition): with
    # random inputs a 16-slot partition overflows in ~1e-3 of the draws, so it
    # passes for the reference generator's particular bits only.  The drop-in's
    # generator draws the same distribution, not the same bits
    # (DESIGN.md §6); that overflow is the reference's own behaviour on those
    # inputs, checked in test_bp_small_partitions_overflow_like_reference.
    skip = {"schemes": "BalancedParallelism.OracleEqualAcrossNodeCounts"}.get(suite)
    r = subprocess.run([exe] + ([f"--gtest_filter=-{skip}"] if skip else []),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-6000:]
    assert "[  PASSED  ]" in r.stdout


@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_reference_acceptance_unmodified(zen, criterion):
    """The reference's acceptance driver (proj/tests/acceptance.cpp), compiled
    unmodified against the drop-in, one criterion per run: C1 every scheme vs
    the dense-sum oracle (:120-199), C2 no loss / lane invariance (:201-250),
    C3 load balance (:255-330), C4 hash-bitmap size and Fig. 7 (:332-372), C5
    codec round trips (:376-431), C6 cost-model extremes (:433-496), C7
    simulator vs cost model (:498-547), C8 scheme orderings (:549-602), C9 the
    hash-memory sweep (:604-645)."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "build", "ref_acceptance")
    if not os.path.exists(exe):
        pytest.skip("built only where /root/reference exists (make ref_tests)")
    r = subprocess.run([exe, str(criterion)], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert f"[PASS] C{criterion}" in r.stdout


def test_bp_small_partitions_overflow_like_reference(zen, ro):
    """The shape of schemes_test's OracleEqualAcrossNodeCounts (n = 16,
    M = 20000, d = 0.005, omega = 0.5): on the device generator's inputs the
    drop-in and the reference agree sync by sync -- equal results, or the same
    SerialOverflow partition (zen/hashing.hpp:221-222) -- over many seeds."""
    agree = overflows = 0
    for seed in range(40):
        spec = zen.WorkloadSpec(universe=20000, nodes=16, density=0.005, omega=0.5, seed=seed)
        ins = zen.generate(spec)
        pairs = [(t.indices(), t.values()) for t in ins]
        try:
            want = ro.bp_sync(20000, pairs, seed=1000 + seed)
        except OracleError as e:
            with pytest.raises(zen.SerialOverflow) as ge:
                zen.run_balanced_parallelism(ins, zen.SimNet(16, 1.0), zen.HashParams(seed=1000 + seed))
            assert ge.value.partition() == e.partition
            overflows += 1
            continue
        out = zen.run_balanced_parallelism(ins, zen.SimNet(16, 1.0), zen.HashParams(seed=1000 + seed))
        np.testing.assert_array_equal(out.results[0].indices(), want.idx)
        np.testing.assert_array_equal(bits(out.results[0].values()), bits(want.val))
        agree += 1
    assert agree + overflows == 40 and agree > 0
