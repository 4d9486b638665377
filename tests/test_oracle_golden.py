"""Pin the C restatement (oracle/zen_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by oracle/make_golden.py through
oracle/_ref/libzenref.so -- the unmodified reference headers compiled in
place.  These tests run on CPU; they are what makes the oracle trustworthy
before it is used to check the CUDA path.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import OracleError

U64MAX = 2**64 - 1


def test_hash_family_known_answers(co):
    g = load_golden("hash_kat")
    for x, y in zip(g["mix_in"], g["mix_out"]):
        assert co.mix64(int(x)) == int(y)
    for (a, b), y in zip(g["derive_in"], g["derive_out"]):
        assert co.derive_seed(int(a), int(b)) == int(y)
    for row in g["families"]:
        seed, n, k, worker = (int(v) for v in row[:4])
        seeds = co.family_seeds(seed, n, k, None if worker == U64MAX else worker)
        assert seeds == [int(v) for v in row[4:5 + k]]
    idx = g["part_idx"]
    for pseed, n in g["part_cases"]:
        np.testing.assert_array_equal(co.partition_of(idx, int(pseed), int(n)),
                                      g[f"part_{pseed}_{n}"])


def test_slot_hash_known_answers(co):
    g = load_golden("hash_kat")
    idx = g["part_idx"][:2048]
    for (seed, n, k, r1, w) in [(1, 8, 3, 160000, 0), (99, 2, 4, 7, 3), (5, 16, 3, 1, 1)]:
        fam = co.family(seed, n, k, worker=w)
        want = g[f"slot_{seed}_{n}_{k}_{r1}_{w}"]
        got = np.array([[co.slot_of(fam, int(x), r, r1) for r in range(1, k + 1)] for x in idx])
        np.testing.assert_array_equal(got, want)


def _hcases():
    g = load_golden("hhash")
    return g, int(g["ncases"][0])


def test_hierarchical_hash_layout_stats_parts(co):
    g, nc = _hcases()
    saw_fallback = saw_overflow = saw_serial = 0
    for i in range(nc):
        p = f"c{i}_"
        m, seed, worker, n, k, r1, r2 = (int(v) for v in g[p + "meta"])
        fam = co.family(seed, n, k, worker=None if worker < 0 else worker)
        idx, val = g[p + "idx"], g[p + "val"]
        ovf = int(g[p + "overflow"][0])
        if ovf >= 0:
            with pytest.raises(OracleError) as e:
                co.hierarchical_hash(m, idx, val, fam, r1, r2)
            assert e.value.partition == ovf
            saw_overflow += 1
            continue
        res = co.hierarchical_hash(m, idx, val, fam, r1, r2, layout=True)
        np.testing.assert_array_equal(res.slots, g[p + "slots"])
        np.testing.assert_array_equal(res.slot_vals, g[p + "slot_vals"])
        np.testing.assert_array_equal(res.depth_of, g[p + "depth"])
        np.testing.assert_array_equal(np.concatenate(res.parts_idx), g[p + "parts_idx"])
        np.testing.assert_array_equal(np.concatenate(res.parts_val), g[p + "parts_val"])
        np.testing.assert_array_equal([x.size for x in res.parts_idx], g[p + "part_count"])
        assert [res.serial_writes] + res.placed_at_depth == list(g[p + "stats"])
        # a partition used the fallback scan when its serial keys exceed r2
        part = co.partition_of(idx, fam.partition_seed, n)
        serial = np.bincount(part[res.depth_of == 0], minlength=n) if idx.size else np.zeros(n)
        saw_fallback += int((serial > r2).any())
        saw_serial += int(res.serial_writes > 0)
    assert saw_overflow >= 2 and saw_fallback >= 1 and saw_serial >= 3


def test_to_sparse_golden(co):
    g = load_golden("to_sparse")
    for name in ["mixed", "rows", "one", "allnz"]:
        idx, val = co.to_sparse(g[name + "_dense"])
        np.testing.assert_array_equal(idx, g[name + "_idx"])
        np.testing.assert_array_equal(val.view(np.uint32), g[name + "_val"].view(np.uint32))


def test_hash_bitmap_codec_golden(co):
    g = load_golden("codec")
    seed, bits = (int(v) for v in g["fig7"])
    u = co.universe(15, 3, seed)
    payload, b = u.encode(0, np.array([5, 7], np.uint64), np.array([0.3, 0.9], np.float32))
    assert b == bits and payload[0] & 0b111 == 0b110
    np.testing.assert_array_equal(payload, g["fig7_payload"])
    for row in g["universe_sizes"]:
        m, n, pseed = (int(v) for v in row[:3])
        if m > 1_000_000:
            continue
        u = co.universe(m, n, pseed)
        assert [u.size(s) for s in range(n)] == [int(v) for v in row[3:3 + n]]
        assert sum(u.size(s) for s in range(n)) == m  # Σ|I_s| = M (codec_test.cpp:189-203)
    for i in range(int(g["ncases"][0])):
        p = f"e{i}_"
        m, n, pseed, s, bits = (int(v) for v in g[p + "meta"])
        u = co.universe(m, n, pseed)
        payload, b = u.encode(s, g[p + "idx"], g[p + "val"])
        assert b == bits
        np.testing.assert_array_equal(payload, g[p + "payload"])
        idx, val = u.decode(s, g[p + "payload"], g[p + "idx"].size)
        np.testing.assert_array_equal(idx, g[p + "idx"])
        np.testing.assert_array_equal(val, g[p + "val"])


def test_hash_bitmap_rejects_foreign_index_and_bad_payload(co):
    u = co.universe(100, 4, 9)
    own0 = set(u.indices(0).tolist())
    foreign = next(i for i in range(100) if i not in own0)
    with pytest.raises(OracleError):
        u.encode(0, np.array([foreign], np.uint64), np.ones(1, np.float32))
    payload, _ = u.encode(0, u.indices(0)[:2], np.ones(2, np.float32))
    with pytest.raises(OracleError):
        u.decode(0, payload[:-1], 2)  # size mismatch (codec.hpp:336-337)
    with pytest.raises(OracleError):
        u.decode(0, np.concatenate([payload, np.zeros(4, np.uint8)]), 3)  # popcount mismatch


def test_bp_sync_golden(co):
    g = load_golden("bp")
    for i in range(int(g["ncases"][0])):
        p = f"b{i}_"
        n, m, gseed, seed, k = (int(v) for v in g[p + "meta"])
        r1m, r2r, _, _ = (float(v) for v in g[p + "params"])
        ins = [(g[p + f"in{w}_idx"], g[p + f"in{w}_val"]) for w in range(n)]
        code, part = (int(v) for v in g[p + "error"])
        if code:
            with pytest.raises(OracleError) as e:
                co.bp_sync(m, ins, k=k, r1_multiplier=r1m, r2_ratio=r2r, seed=seed)
            assert e.value.code == code and e.value.partition == part
            continue
        res = co.bp_sync(m, ins, k=k, r1_multiplier=r1m, r2_ratio=r2r, seed=seed)
        np.testing.assert_array_equal(res.idx, g[p + "idx"])
        np.testing.assert_array_equal(res.val, g[p + "val"])
        np.testing.assert_array_equal(res.ledger, g[p + "ledger"])
        np.testing.assert_allclose(res.balance, g[p + "balance"], rtol=0, atol=0)


def test_oracle_matches_live_reference_random(co, ro):
    """Where the reference is compiled here, cross-check on fresh random inputs too."""
    rng = np.random.default_rng(99)
    for trial in range(60):
        m = int(rng.integers(10, 20000))
        z = int(rng.integers(0, m // 2 + 1))
        idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
        val = rng.standard_normal(z).astype(np.float32)
        n, k = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        seed, w = int(rng.integers(0, 2**62)), int(rng.integers(0, 8))
        r1 = int(rng.integers(1, 2 * z // n + 3))
        r2 = int(rng.integers(1, r1 + 3))
        fam = co.family(seed, n, k, worker=w)
        slots, svals, depth, ovf = ro.slot_layout(m, idx, val, seed, n, k, r1, r2, worker=w)
        if ovf >= 0:
            with pytest.raises(OracleError) as e:
                co.hierarchical_hash(m, idx, val, fam, r1, r2)
            assert e.value.partition == ovf
            continue
        res = co.hierarchical_hash(m, idx, val, fam, r1, r2, layout=True)
        np.testing.assert_array_equal(res.slots, slots)
        np.testing.assert_array_equal(res.depth_of, depth)
    for n in [2, 5, 8]:
        ins = ro.generate(30000, n, 0.01, 0.3, 1000 + n)
        a, b = co.bp_sync(30000, ins, seed=n), ro.bp_sync(30000, ins, seed=n)
        np.testing.assert_array_equal(a.idx, b.idx)
        np.testing.assert_array_equal(a.val, b.val)
        np.testing.assert_array_equal(a.ledger, b.ledger)


def _wire_kw(meta_row):
    kind, bs, cb, m, n, pseed, srv = (int(x) for x in meta_row[:7])
    return kind, m, {"block_size": bs, "coo_bits": cb}, n, pseed, srv


def test_wire_formats_golden(co):
    """Every WireKind's payload bytes, bit accounting, framing and decode
    (zen/codec.hpp:182-410) equal the reference's."""
    g = load_golden("wire")
    for c, row in enumerate(g["meta"]):
        kind, m, kw, n, pseed, srv = _wire_kw(row)
        u = co.universe(m, n, pseed) if kind == 4 else None
        idx, val = g[f"c{c}_idx"], g[f"c{c}_val"]
        payload, info = co.wire_encode(kind, m, idx, val, universe=u, server=srv, **kw)
        assert np.array_equal(payload, g[f"c{c}_payload"]), c
        assert [info["count"], info["index_bits"], info["value_bits"]] == [int(x) for x in row[7:]]
        framed = co.frame(kind, m, payload, info, **kw)
        assert np.array_equal(framed, g[f"c{c}_framed"]), c
        hdr, body = co.unframe(framed)
        assert np.array_equal(body, payload) and hdr["count"] == info["count"]
        di, dv = co.wire_decode(kind, m, info["count"], payload, universe=u, server=srv, **kw)
        assert np.array_equal(di, g[f"c{c}_didx"]) and np.array_equal(dv, g[f"c{c}_dval"]), c
    di, dv = co.wire_decode(1, 4000, 50, g["unsorted_payload"])
    assert np.array_equal(di, g["unsorted_idx"]) and np.array_equal(dv, g["unsorted_val"])


def test_wire_malformed_and_sparse_file(co):
    g = load_golden("wire")
    m = int(g["zspt_m"][0])
    raw = co.write_sparse(m, g["zspt_idx"], g["zspt_val"])
    assert np.array_equal(raw, g["zspt_bytes"])
    m2, i2, v2 = co.read_sparse(raw)
    assert m2 == m and np.array_equal(i2, g["zspt_idx"]) and np.array_equal(v2, g["zspt_val"])
    with pytest.raises(OracleError):
        co.read_sparse(np.frombuffer(b"ZSPX" + raw.tobytes()[4:], np.uint8))
    payload, info = co.wire_encode(1, 5000, g["c0_idx"], g["c0_val"])
    with pytest.raises(OracleError):  # size mismatch (codec.hpp:287)
        co.wire_decode(1, 5000, info["count"] + 1, payload)
    dup = np.concatenate([np.array([5, 5], np.uint64).view(np.uint8),
                          np.ones(2, np.float32).view(np.uint8)])
    with pytest.raises(OracleError):  # duplicate index (tensor.hpp:44)
        co.wire_decode(1, 5000, 2, dup)
    framed = co.frame(1, 5000, payload, info)
    with pytest.raises(OracleError):  # truncated frame
        co.unframe(framed[:-1])


def test_sparsify_topk_golden(co):
    g = load_golden("topk")
    for name in ["gauss", "ints"]:
        d = g[f"{name}_dense"]
        for f in g["fractions"]:
            key = f"{name}_{f}_idx"
            if key not in g:
                continue
            i, v = co.sparsify_topk(d, float(f))
            assert np.array_equal(i, g[key]) and np.array_equal(v, g[f"{name}_{f}_val"]), (name, f)


# ---- f3: Hierarchical Centralization, merge_sum, metrics, profile / selector ----

KIND_NAMES = {1: "coo", 2: "bitmap", 3: "tensor_block"}


def hc_case(g, c):
    m, n = (int(x) for x in g[f"c{c}_m"])
    ins = [(g[f"c{c}_in{w}_idx"], g[f"c{c}_in{w}_val"]) for w in range(n)]
    return m, n, ins


def test_hier_centralization_golden(co):
    """The restatement of run_hier_centralization + its SimNet ledger against
    the reference's outputs, every sized wire format."""
    g = load_golden("hc")
    for c in range(int(g["ncases"][0])):
        m, n, ins = hc_case(g, c)
        for f, (k, bs, cb) in enumerate(g["formats"]):
            i, v, led = co.hier_centralization(m, ins, KIND_NAMES[int(k)], int(bs), int(cb))
            np.testing.assert_array_equal(i, g[f"c{c}_f{f}_idx"], err_msg=f"case {c} fmt {f}")
            np.testing.assert_array_equal(v.view(np.uint32), g[f"c{c}_f{f}_val"].view(np.uint32))
            np.testing.assert_array_equal(led, g[f"c{c}_f{f}_ledger"])
        i, v = co.merge_sum(*ins[0], *ins[1])
        np.testing.assert_array_equal(i, g[f"c{c}_merge_idx"])
        np.testing.assert_array_equal(v.view(np.uint32), g[f"c{c}_merge_val"].view(np.uint32))


def test_profile_and_selector_golden(co):
    g = load_golden("hc")
    seen = 0
    for c in range(int(g["ncases"][0])):
        if f"c{c}_profile" not in g:
            continue
        m, n, ins = hc_case(g, c)
        d, gamma, skew, choice = co.profile(m, [ins, list(reversed(ins))])
        want = g[f"c{c}_profile"]
        assert (d, skew, choice) == (want[0], want[1], int(want[2]))
        for j in range(5):
            assert gamma.get(1 << j, np.nan) == want[3 + j] or np.isnan(want[3 + j])
        assert co.skewness(m, ins[0][0], n) == g[f"c{c}_metrics"][2]
        seen += 1
    assert seen >= 5


def test_hier_centralization_rejects_non_power_of_two(co):
    ins = [(np.array([w], np.uint64), np.ones(1, np.float32)) for w in range(6)]
    with pytest.raises(OracleError):
        co.hier_centralization(100, ins)


def test_hier_centralization_restatement_vs_reference(co, ro):
    rng = np.random.default_rng(17)
    for trial in range(12):
        n = 1 << int(rng.integers(1, 4))
        ins = ro.generate(2000, n, 0.01 + 0.01 * int(rng.integers(0, 5)),
                          0.25 * int(rng.integers(0, 4)), int(rng.integers(1, 1 << 30)))
        for kind in ["coo", "bitmap", "tensor_block"]:
            a = co.hier_centralization(2000, ins, kind, 32)
            b = ro.hier_centralization(2000, ins, kind, 32)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
            assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
        assert co.profile(2000, [ins]) == ro.profile(2000, [ins])


# ---- f4: the baseline schemes (run_scheme) ----

def test_baseline_schemes_golden(co):
    """The restatement of run_agsparse / run_ring_centralization /
    run_omnireduce_like / sparcml against the reference's outputs: every
    node's result, the ledger and the balance."""
    from make_golden import SCHEME_RUNS
    g = load_golden("schemes")
    for c in range(int(g["ncases"][0])):
        m, n = (int(x) for x in g[f"c{c}_m"])
        ins = [(g[f"c{c}_in{w}_idx"], g[f"c{c}_in{w}_val"]) for w in range(n)]
        for r, (name, comm, kind, bs) in enumerate(SCHEME_RUNS):
            k, cb = (("coo", 32) if kind == "coo32" else (kind, 64))
            res, led, bal = co.run_scheme(name, m, ins, comm, k, bs, cb)
            for w, (i, v) in enumerate(res):
                np.testing.assert_array_equal(i, g[f"c{c}_r{r}_w{w}_idx"], err_msg=f"{c} {name}")
                np.testing.assert_array_equal(v.view(np.uint32),
                                              g[f"c{c}_r{r}_w{w}_val"].view(np.uint32))
            np.testing.assert_array_equal(led, g[f"c{c}_r{r}_ledger"], err_msg=f"{c} {name}")
            key = f"c{c}_r{r}_balance"
            assert (bal is None) == (key not in g)
            if bal is not None:
                assert tuple(bal) == tuple(g[key])


def test_baseline_schemes_restatement_vs_reference(co, ro):
    """The f4 restatement against the compiled reference on fresh random cases
    (any n for AGsparse / OmniReduce; powers of two for the ring)."""
    rng = np.random.default_rng(41)
    for trial in range(8):
        n = int(rng.integers(2, 9))
        m = int(rng.integers(500, 5000))
        ins = ro.generate(m, n, 0.01 + 0.01 * int(rng.integers(0, 4)),
                          0.25 * int(rng.integers(0, 4)), int(rng.integers(1, 1 << 30)))
        runs = [("agsparse", None, None, 256), ("omnireduce", None, "tensor_block",
                                                  int(rng.integers(1, 100)))]
        if n & (n - 1) == 0:
            runs += [("ring-centralization", None, None, 256), ("agsparse", "hierarchy", None, 256)]
        for name, comm, kind, bs in runs:
            a = ro.run_scheme(name, m, ins, comm, kind, bs)
            b = co.run_scheme(name, m, ins, comm, kind, bs)
            for (ai, av), (bi, bv) in zip(a[0], b[0]):
                assert np.array_equal(ai, bi) and np.array_equal(av.view(np.uint32),
                                                                 bv.view(np.uint32))
            assert np.array_equal(a[1], b[1]) and a[2] == b[2], (trial, name)
