#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the REFERENCE ITSELF -- TEST INFRASTRUCTURE.

Every vector here comes from oracle/_ref/libzenref.so, i.e. the unmodified
reference headers (/root/reference/proj/include/zen) compiled in place by
oracle/Makefile.  The reference ships no golden vectors for this path (its
tests/data fixtures are absent), so these fixtures are what pin
both the C restatement (oracle/zen_oracle.c) and the CUDA path.

Run:  make -C oracle && python oracle/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from oracle import OracleError, RefOracle  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def random_tensor(rng, m, z):
    idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
    val = rng.integers(1, 17, z).astype(np.float32)
    return idx, val


def hash_kat(ro: RefOracle):
    rng = np.random.default_rng(2024)
    xs = np.concatenate([np.arange(64, dtype=np.uint64),
                         rng.integers(0, 2**63, 256, dtype=np.uint64) * 2 + 1,
                         np.array([2**64 - 1, 2**63, 2**40 - 1, 2**32 - 1, 2**32], np.uint64)])
    out = {"mix_in": xs, "mix_out": np.array([ro.mix64(int(x)) for x in xs], np.uint64)}
    pairs = rng.integers(0, 2**63, (64, 2), dtype=np.uint64)
    out["derive_in"] = pairs
    out["derive_out"] = np.array([ro.derive_seed(int(a), int(b)) for a, b in pairs], np.uint64)
    fams = []
    for seed in [0, 1, 7, 1234, 2**63 + 5]:
        for n in [1, 2, 3, 8, 16]:
            for k in [1, 3, 4]:
                for worker in [None, 0, 5]:
                    s = ro.family_seeds(seed, n, k, worker)
                    fams.append([seed, n, k, 2**64 - 1 if worker is None else worker] + s + [0] * (4 - k))
    out["families"] = np.array(fams, dtype=np.uint64)  # seed,n,k,worker,pseed,slot1..4
    idx = np.concatenate([np.arange(4096, dtype=np.uint64),
                          rng.integers(0, 819_200_000, 4096).astype(np.uint64)])
    out["part_idx"] = idx
    cases = []
    for pseed in [ro.derive_seed(1, 0), ro.derive_seed(2024, 0), 12345]:
        for n in [1, 2, 3, 4, 7, 8, 16, 64]:
            cases.append((pseed, n))
            out[f"part_{pseed}_{n}"] = ro.partition_of(idx, pseed, n)
    out["part_cases"] = np.array(cases, dtype=np.uint64)
    for (seed, n, k, r1, w) in [(1, 8, 3, 160000, 0), (99, 2, 4, 7, 3), (5, 16, 3, 1, 1)]:
        out[f"slot_{seed}_{n}_{k}_{r1}_{w}"] = ro.slot_of(seed, n, k, idx[:2048], r1, worker=w)
    return out


def find_colliding_pair(ro, seed, n, k, r1):
    """proj/tests/hashing_test.cpp:108-136: two indices colliding on h0 and all k slots."""
    idx = np.arange(3000, dtype=np.uint64)
    fam = ro.family_seeds(seed, n, k)
    parts = ro.partition_of(idx, fam[0], n)
    slots = ro.slot_of(seed, n, k, idx, r1)
    for x in range(3000):
        for y in range(x + 1, 3000):
            if parts[x] == parts[y] and np.array_equal(slots[x], slots[y]):
                return x, y
    raise RuntimeError("no colliding pair")


def hhash_cases(ro: RefOracle):
    rng = np.random.default_rng(7)
    cases = []
    # (m, z, seed, worker, n, k, r1, r2)
    for _ in range(24):
        m = int(rng.integers(100, 200_000))
        z = int(rng.integers(0, min(m // 2, 8000) + 1))
        n = int(rng.choice([1, 2, 3, 4, 8, 16]))
        k = int(rng.integers(1, 5))
        r1 = max(1, int(np.ceil(2.0 * z / n)))
        r2 = max(1, int(np.ceil(0.1 * r1)))
        cases.append((m, random_tensor(rng, m, z), int(rng.integers(0, 2**62)),
                      int(rng.integers(0, 8)), n, k, r1, r2))
    # C2-shaped (acceptance.cpp:201-250): M=1e6, d=1%, n=16, r1=2nnz/n, r2=r1/10
    cases.append((1_000_000, random_tensor(rng, 1_000_000, 10_000), 3, 3, 16, 3, 1250, 125))
    # tight regions: fallback scan and serial pressure (load <= r1 + r2)
    for _ in range(8):
        m = int(rng.integers(200, 3000))
        z = int(rng.integers(20, 120))
        n = int(rng.choice([1, 2, 4]))
        k = int(rng.integers(1, 4))
        t = random_tensor(rng, m, z)
        seed = int(rng.integers(0, 2**62))
        pseed = ro.family_seeds(seed, n, k)[0]
        load = np.bincount(ro.partition_of(t[0], pseed, n), minlength=n).max()
        r1 = max(1, int(load) // 3)
        r2 = max(1, int(load) - r1)  # capacity exactly the max load -> fallback scans
        cases.append((m, t, seed, None, n, k, r1, r2))
    # adversarial colliding pair goes serial (hashing_test.cpp:108-136)
    a, b = find_colliding_pair(ro, 4242, 4, 3, 2)
    cases.append((3000, (np.array([a, b], np.uint64), np.array([1.0, 2.0], np.float32)),
                  4242, None, 4, 3, 2, 4))
    # overflow: three indices of partition 0, capacity 2 (hashing_test.cpp:138-147)
    pseed = ro.family_seeds(7, 2, 2)[0]
    same = [x for x in range(100) if ro.partition_of(np.array([x], np.uint64), pseed, 2)[0] == 0][:3]
    cases.append((1000, (np.array(same, np.uint64), np.ones(3, np.float32)), 7, None, 2, 2, 1, 1))
    # overflow in several partitions: the first dropped key decides the partition
    t = random_tensor(rng, 5000, 600)
    cases.append((5000, t, 11, 2, 8, 3, 20, 10))
    # edge cases: empty tensor, single index (hashing_test.cpp:56-65), n = 1
    cases.append((1000, (np.zeros(0, np.uint64), np.zeros(0, np.float32)), 3, None, 8, 3, 4, 2))
    cases.append((1000, (np.array([123], np.uint64), np.array([2.5], np.float32)), 5, None, 8, 3,
                  4, 2))
    cases.append((50_000, random_tensor(rng, 50_000, 3000), 77, 0, 1, 3, 6000, 600))
    out = {}
    for i, (m, (idx, val), seed, worker, n, k, r1, r2) in enumerate(cases):
        p = f"c{i}_"
        out[p + "meta"] = np.array([m, seed, -1 if worker is None else worker, n, k, r1, r2],
                                   dtype=np.int64)
        out[p + "idx"], out[p + "val"] = idx, val
        slots, svals, depth, ovf = ro.slot_layout(m, idx, val, seed, n, k, r1, r2, worker=worker)
        out[p + "overflow"] = np.array([ovf], np.int64)
        out[p + "slots"], out[p + "slot_vals"], out[p + "depth"] = slots, svals, depth
        try:
            res = ro.hierarchical_hash(m, idx, val, seed, n, k, r1, r2, worker=worker)
            assert ovf < 0
            out[p + "parts_idx"] = np.concatenate(res.parts_idx) if idx.size else idx
            out[p + "parts_val"] = np.concatenate(res.parts_val) if idx.size else val
            out[p + "part_count"] = np.array([x.size for x in res.parts_idx], np.uint64)
            out[p + "stats"] = np.array([res.serial_writes] + res.placed_at_depth, np.uint64)
        except OracleError as e:
            assert e.code == 2 and e.partition == ovf, (e, ovf)
    out["ncases"] = np.array([len(cases)])
    return out


def to_sparse_cases(ro: RefOracle):
    rng = np.random.default_rng(3)
    out = {}
    d = rng.standard_normal(10_000).astype(np.float32)
    d[rng.random(10_000) < 0.97] = 0.0
    specials = np.array([0.0, -0.0, np.nan, np.inf, -np.inf, 1e-45, -1e-45, 1.17e-38, 3.4e38,
                         -0.0, 0.0, 1.0], np.float32)
    d[:specials.size] = specials
    d[5000:5000 + specials.size] = specials
    rows = np.zeros((500, 64), np.float32)  # row-structured embedding gradient
    live = rng.choice(500, 20, replace=False)
    rows[live] = rng.integers(1, 17, (20, 64)).astype(np.float32)
    rows[live[0], 5] = 0.0  # a hole inside a live row stays a hole
    for name, dense in [("mixed", d), ("rows", rows.ravel()), ("one", np.array([0.0], np.float32)),
                        ("allnz", np.arange(1, 130, dtype=np.float32))]:
        out[name + "_dense"] = dense
        out[name + "_idx"], out[name + "_val"] = ro.to_sparse(dense)
    return out


def codec_cases(ro: RefOracle):
    out = {}
    rng = np.random.default_rng(11)
    # Fig. 7 worked example (codec_test.cpp:107-133)
    fifteen = np.arange(15, dtype=np.uint64)
    for seed in range(200_000):
        # universe 0 of (15, 3, seed) must hold 5 at position 1 and 7 at position 2
        u0 = list(np.nonzero(ro.partition_of(fifteen, seed, 3) == 0)[0])
        if len(u0) >= 3 and 5 in u0 and 7 in u0 and u0.index(5) == 1 and u0.index(7) == 2:
            payload, bits = ro.hash_bitmap_encode(15, 3, seed, 0, np.array([5, 7], np.uint64),
                                                  np.array([0.3, 0.9], np.float32))
            out["fig7"] = np.array([seed, bits], np.uint64)
            out["fig7_payload"] = payload
            break
    sizes = []
    for (m, n, pseed) in [(15, 2, 4), (1000, 7, 12345), (1000, 16, 99), (6_400_000, 2, 1),
                          (100_000, 8, ro.derive_seed(1, 0))]:
        row = [m, n, pseed] + [ro.universe_size(m, n, pseed, s) for s in range(n)]
        sizes.append(row + [0] * (19 - len(row)))
    out["universe_sizes"] = np.array(sizes, np.uint64)
    cases = []
    for i in range(12):
        m = int(rng.integers(10, 60_000))
        n = int(rng.integers(1, 9))
        pseed = int(rng.integers(0, 2**62))
        s = int(rng.integers(0, n))
        all_idx = np.arange(m, dtype=np.uint64)
        own = all_idx[ro.partition_of(all_idx, pseed, n) == s]
        z = int(rng.integers(0, own.size + 1)) if i % 3 else min(own.size, 5)
        idx = np.sort(rng.choice(own, z, replace=False)).astype(np.uint64)
        val = rng.standard_normal(z).astype(np.float32)
        payload, bits = ro.hash_bitmap_encode(m, n, pseed, s, idx, val)
        back = ro.hash_bitmap_decode(m, n, pseed, s, payload, z)
        assert np.array_equal(back[0], idx)
        p = f"e{i}_"
        out[p + "meta"] = np.array([m, n, pseed, s, bits], np.uint64)
        out[p + "idx"], out[p + "val"], out[p + "payload"] = idx, val, payload
        cases.append(i)
    out["ncases"] = np.array([len(cases)])
    return out


def bp_cases(ro: RefOracle):
    out = {}
    rng = np.random.default_rng(47)
    cases = []
    for n in [2, 4, 8, 16]:
        for trial in range(2):
            cases.append((n, 20_000, 0.005, 0.5, int(rng.integers(0, 2**62)),
                          int(rng.integers(0, 2**62)), 3, 2.0, 0.1))
    cases.append((2, 6_400, 0.01, 0.5, 3, 1, 3, 2.0, 0.1))
    cases.append((4, 4096, 0.02, 1.0, 43, 1, 3, 2.0, 0.1))  # identical tensors, schemes_test:249
    cases.append((3, 10_000, 0.02, 0.0, 9, 77, 4, 1.0, 0.5))  # n not a power of two
    cases.append((2, 1000, 0.1, 0.0, 53, 1, 3, 0.02, 0.01))  # SerialOverflow (schemes_test:288)
    for i, (n, m, d, omega, gseed, seed, k, r1m, r2r) in enumerate(cases):
        ins = ro.generate(m, n, d, omega, gseed)
        p = f"b{i}_"
        out[p + "meta"] = np.array([n, m, gseed, seed, k], np.uint64)
        out[p + "params"] = np.array([r1m, r2r, d, omega], np.float64)
        for w, (ii, vv) in enumerate(ins):
            out[p + f"in{w}_idx"], out[p + f"in{w}_val"] = ii, vv
        try:
            res = ro.bp_sync(m, ins, k=k, r1_multiplier=r1m, r2_ratio=r2r, seed=seed)
            out[p + "idx"], out[p + "val"], out[p + "ledger"] = res.idx, res.val, res.ledger
            out[p + "balance"] = np.array(res.balance if res.balance else [np.nan, np.nan])
            out[p + "error"] = np.array([0, -1], np.int64)
        except OracleError as e:
            out[p + "error"] = np.array([e.code, e.partition], np.int64)
    out["ncases"] = np.array([len(cases)])
    return out


def wire_cases(ro: RefOracle):
    """Every WireKind (zen/codec.hpp:19-34) through the reference's encode,
    write_framed and decode; .zspt bytes (zen/tensor.hpp:257-264)."""
    rng = np.random.default_rng(1129)
    out, meta = {}, []
    # (kind, block_size, coo_bits, m, z, n, pseed, server)
    specs = [(1, 256, 64, 5000, 60, 1, 0, 0), (1, 256, 32, 5000, 60, 1, 0, 0),
             (1, 256, 64, 2**40, 33, 1, 0, 0), (1, 256, 64, 100, 0, 1, 0, 0),
             (2, 256, 64, 5000, 60, 1, 0, 0), (2, 256, 64, 77, 13, 1, 0, 0),
             (2, 256, 64, 64, 64, 1, 0, 0),
             (3, 256, 64, 5000, 60, 1, 0, 0), (3, 7, 64, 5000, 300, 1, 0, 0),
             (3, 1, 64, 999, 50, 1, 0, 0), (3, 100, 64, 1001, 1001, 1, 0, 0),
             (4, 256, 64, 20000, 0, 4, 777, 1), (4, 256, 64, 20000, 0, 3, 12345, 2),
             (4, 256, 64, 6400, 0, 1, 5, 0)]
    for c, (kind, bs, cb, m, z, n, pseed, srv) in enumerate(specs):
        if kind == 4:
            cand = np.arange(m, dtype=np.uint64)
            own = cand[ro.partition_of(cand, pseed, n) == srv]
            idx = np.sort(rng.choice(own, min(own.size, 97), replace=False)).astype(np.uint64)
        elif m > 2**32:
            idx = np.sort(rng.choice(2**20, z, replace=False).astype(np.uint64) * 1000003 + 2**33)
        else:
            idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
        val = rng.integers(-16, 17, idx.size).astype(np.float32)
        val[val == 0] = 0.5
        if kind == 3 and idx.size > 3:
            val[1] = 0.0  # explicit zeros are encoded but dropped by the decode
        payload, info = ro.wire_encode(kind, m, idx, val, bs, cb, n, pseed, srv)
        framed = ro.write_framed(kind, m, idx, val, bs, cb, n, pseed, srv)
        di, dv = ro.wire_decode(kind, m, info["count"], payload, bs, cb, n, pseed, srv)
        out[f"c{c}_idx"], out[f"c{c}_val"] = idx, val
        out[f"c{c}_payload"], out[f"c{c}_framed"] = payload, framed
        out[f"c{c}_didx"], out[f"c{c}_dval"] = di, dv
        meta.append([kind, bs, cb, m, n, pseed, srv, info["count"], info["index_bits"],
                     info["value_bits"]])
    out["meta"] = np.array(meta, np.uint64)
    # COO payload in arbitrary order: decode canonicalises (tensor.hpp:41, :72-84)
    idx = rng.choice(4000, 50, replace=False).astype(np.uint64)
    val = rng.integers(1, 9, 50).astype(np.float32)
    out["unsorted_payload"] = np.concatenate([idx.view(np.uint8), val.view(np.uint8)])
    out["unsorted_idx"], out["unsorted_val"] = ro.wire_decode(1, 4000, 50, out["unsorted_payload"])
    m = 123456
    idx = np.sort(rng.choice(m, 40, replace=False)).astype(np.uint64)
    val = rng.standard_normal(40).astype(np.float32)
    out["zspt_m"] = np.array([m], np.uint64)
    out["zspt_idx"], out["zspt_val"] = idx, val
    out["zspt_bytes"] = ro.write_sparse(m, idx, val)
    return out


def topk_cases(ro: RefOracle):
    """zen::sparsify_topk (zen/workload.hpp:157-178): ties, zeros, signs."""
    rng = np.random.default_rng(178)
    out, cases = {}, []
    dense = rng.standard_normal(20000).astype(np.float32)
    dense[rng.choice(20000, 4000, replace=False)] = 0.0
    dense[100:140] = 3.0          # a run of equal magnitudes: ties to the lower index
    dense[200:220] = -3.0
    dense[300] = -0.0
    ints = rng.integers(-4, 5, 5000).astype(np.float32)  # many ties
    for name, d in [("gauss", dense), ("ints", ints)]:
        out[f"{name}_dense"] = d
        for f in [1e-4, 0.001, 0.0021, 0.01, 0.05, 0.3, 0.9, 1.0]:
            i, v = ro.sparsify_topk(d, f)
            out[f"{name}_{f}_idx"], out[f"{name}_{f}_val"] = i, v
            cases.append(f)
    out["fractions"] = np.array(sorted(set(cases)), np.float64)
    return out


def hc_cases(ro: RefOracle):
    """zen::run_hier_centralization (zen/schemes.hpp:173-193) in every sized
    format, zen::merge_sum (tensor.hpp:133-167), the tensor metrics
    (tensor.hpp:111-213) and profile_sparsity + select_scheme
    (costmodel.hpp:139-195), on the shapes schemes_test.cpp uses."""
    out = {}
    cases = [(2, 50, None), (4, 1000, (0.05, 1.0, 13)), (8, 100000, (0.002, 0.0, 23)),
             (8, 100000, (0.002, 0.5, 23)), (8, 100000, (0.002, 1.0, 23)), (2, 2000, (0.03, 0.25, 5)),
             (4, 2000, (0.01, 0.75, 6)), (16, 20000, (0.01, 0.4, 7))]
    fmts = [("coo", 256, 64), ("coo", 256, 32), ("bitmap", 256, 64), ("tensor_block", 64, 64)]
    for c, (n, m, spec) in enumerate(cases):
        if spec is None:
            ins = [(np.array([1], np.uint64), np.array([2], np.float32)),
                   (np.array([2], np.uint64), np.array([3], np.float32))]
        else:
            ins = ro.generate(m, n, *spec)
        out[f"c{c}_m"] = np.array([m, n], np.uint64)
        for w, (i, v) in enumerate(ins):
            out[f"c{c}_in{w}_idx"], out[f"c{c}_in{w}_val"] = i, v
        for f, (kind, bs, cb) in enumerate(fmts):
            i, v, led = ro.hier_centralization(m, ins, kind, bs, cb)
            out[f"c{c}_f{f}_idx"], out[f"c{c}_f{f}_val"], out[f"c{c}_f{f}_ledger"] = i, v, led
        i, v = ro.merge_sum(m, *ins[0], *ins[1])
        out[f"c{c}_merge_idx"], out[f"c{c}_merge_val"] = i, v
        if all(len(i) for i, _ in ins):
            out[f"c{c}_metrics"] = np.array([ro.metric(0, m, ins[:2]), ro.metric(1, m, ins),
                                             ro.metric(2, m, ins[:1], n)], np.float64)
            d, g, sk, ch = ro.profile(m, [ins, list(reversed(ins))])
            out[f"c{c}_profile"] = np.array([d, sk, ch] + [g.get(1 << j, np.nan)
                                                           for j in range(5)], np.float64)
    out["formats"] = np.array([[{"coo": 1, "bitmap": 2, "tensor_block": 3}[k], bs, cb]
                               for k, bs, cb in fmts], np.uint32)
    out["ncases"] = np.array([len(cases)], np.uint32)
    return out


SCHEME_RUNS = [  # name, communication override, wire kind override, block size
    ("agsparse", None, None, 256), ("agsparse", "ring", None, 256),
    ("agsparse", "hierarchy", "tensor_block", 64), ("sparcml", None, None, 256),
    ("sparcml", None, "coo32", 256), ("ring-centralization", None, None, 256),
    ("ring-centralization", None, "bitmap", 256), ("omnireduce", None, None, 256),
    ("omnireduce", None, "tensor_block", 64), ("omnireduce", None, "tensor_block", 1000)]


def scheme_cases(ro: RefOracle):
    """zen::run_scheme over the baseline schemes (zen/schemes.hpp:119-328,
    420-465): every node's result, the SimNet ledger and the balance, on
    shapes from schemes_test.cpp (overlaps 0..1, n = 2..16, a value that
    cancels to exact zero for the OmniReduce block decode)."""
    out = {}
    cases = [(4, 2000, 0.03, 0.5, 3), (8, 5000, 0.01, 0.0, 4), (2, 777, 0.05, 1.0, 5),
             (4, 100000, 0.002, 0.25, 6), (16, 20000, 0.005, 0.4, 7)]
    for c, (n, m, d, om, seed) in enumerate(cases):
        ins = ro.generate(m, n, d, om, seed)
        if c == 0:  # a shared index whose values cancel: dropped by the block decode
            i0, v0 = ins[0]
            i1, v1 = ins[1]
            common = np.intersect1d(i0, i1)[:1]
            if common.size:
                v1 = v1.copy()
                v1[np.searchsorted(i1, common)] = -v0[np.searchsorted(i0, common)]
                ins[1] = (i1, v1)
        out[f"c{c}_m"] = np.array([m, n], np.uint64)
        for w, (i, v) in enumerate(ins):
            out[f"c{c}_in{w}_idx"], out[f"c{c}_in{w}_val"] = i, v
        for r, (name, comm, kind, bs) in enumerate(SCHEME_RUNS):
            k, cb = (("coo", 32) if kind == "coo32" else (kind, 64))
            res, led, bal = ro.run_scheme(name, m, ins, comm, k, bs, cb)
            for w, (i, v) in enumerate(res):
                out[f"c{c}_r{r}_w{w}_idx"], out[f"c{c}_r{r}_w{w}_val"] = i, v
            out[f"c{c}_r{r}_ledger"] = led
            if bal is not None:
                out[f"c{c}_r{r}_balance"] = np.array(bal, np.float64)
    out["ncases"] = np.array([len(cases)], np.uint32)
    return out


def main():
    ro = RefOracle()
    os.makedirs(OUT, exist_ok=True)
    for name, fn in [("hash_kat", hash_kat), ("hhash", hhash_cases), ("to_sparse", to_sparse_cases),
                     ("codec", codec_cases), ("bp", bp_cases), ("wire", wire_cases),
                     ("topk", topk_cases), ("hc", hc_cases),
                     ("schemes", scheme_cases)]:
        data = fn(ro)
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
