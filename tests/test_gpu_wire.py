"""GPU parity of the wire and file formats: every
WireKind's payload bytes, bit accounting, framing and decode through the
C-ABI (zen_encode / zen_decode / zen_frame_*) against the reference's own
bytes (tests/golden/wire.npz, made by oracle/make_golden.py from oracle/_ref),
plus the oracle on random cases and full-size round trips."""
import io

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
KINDS = {1: "coo", 2: "bitmap", 3: "tensor_block", 4: "hash_bitmap"}


def fmt_of(zen, row):
    kind, bs, cb = int(row[0]), int(row[1]), int(row[2])
    return zen.WireFormat(KINDS[kind], bs, cb)


def test_wire_golden_bytes_frames_and_decodes(zen):
    g = load_golden("wire")
    for c, row in enumerate(g["meta"]):
        kind, m, n, pseed, srv = int(row[0]), int(row[3]), int(row[4]), int(row[5]), int(row[6])
        fmt = fmt_of(zen, row)
        uni = zen.HashUniverseTable(m, n, pseed).universe(srv) if kind == 4 else None
        t = zen.SparseTensor(m, g[f"c{c}_idx"], g[f"c{c}_val"])
        msg = zen.encode(t, fmt, uni)
        np.testing.assert_array_equal(msg.payload, g[f"c{c}_payload"], err_msg=f"case {c}")
        assert [msg.count, msg.index_bits, msg.value_bits] == [int(x) for x in row[7:]]
        buf = io.BytesIO()
        zen.write_framed(buf, msg)
        np.testing.assert_array_equal(np.frombuffer(buf.getvalue(), np.uint8), g[f"c{c}_framed"])
        buf.seek(0)
        back = zen.read_framed(buf)
        assert back.format == fmt and back.count == msg.count
        d = zen.decode(back, uni)
        np.testing.assert_array_equal(d.indices(), g[f"c{c}_didx"])
        np.testing.assert_array_equal(d.values().view(np.uint32),
                                      g[f"c{c}_dval"].view(np.uint32))


def test_coo_decode_canonicalises_unsorted_payload(zen):
    g = load_golden("wire")
    msg = zen.EncodedMessage(zen.WireFormat.coo(), 4000, 50, 64 * 50, 32 * 50,
                             g["unsorted_payload"])
    d = zen.decode(msg)
    np.testing.assert_array_equal(d.indices(), g["unsorted_idx"])
    np.testing.assert_array_equal(d.values(), g["unsorted_val"])


def test_wire_errors(zen):
    t = zen.SparseTensor(2**40, [5, 2**33], [1.0, 2.0])
    with pytest.raises(zen.Error):  # codec.hpp:225 index does not fit
        zen.encode(t, zen.WireFormat.coo(32))
    ok = zen.encode(zen.SparseTensor(100, [1, 2], [1.0, 2.0]), zen.WireFormat.coo())
    bad = zen.EncodedMessage(ok.format, 100, 3, ok.index_bits, ok.value_bits, ok.payload)
    with pytest.raises(zen.MalformedPayload):  # size mismatch, codec.hpp:287
        zen.decode(bad)
    dup = np.concatenate([np.array([7, 7], "<u8").view(np.uint8),
                          np.ones(2, "<f4").view(np.uint8)])
    with pytest.raises(zen.Error):  # duplicate index, tensor.hpp:44
        zen.decode(zen.EncodedMessage(zen.WireFormat.coo(), 100, 2, 128, 64, dup))
    rng = np.concatenate([np.array([1, 100], "<u8").view(np.uint8),
                          np.ones(2, "<f4").view(np.uint8)])
    with pytest.raises(zen.Error):  # index outside [0, M)
        zen.decode(zen.EncodedMessage(zen.WireFormat.coo(), 100, 2, 128, 64, rng))
    tb = zen.encode(zen.SparseTensor(1000, [3, 700], [1.0, 2.0]), zen.WireFormat.tensor_block(100))
    p = tb.payload.copy()
    p[:8] = np.frombuffer(np.array([10], "<u8").tobytes(), np.uint8)  # block 10 -> begin 1000
    with pytest.raises(zen.MalformedPayload):  # codec.hpp:318 block id outside universe
        zen.decode(zen.EncodedMessage(tb.format, 1000, tb.count, tb.index_bits, tb.value_bits, p))
    with pytest.raises(zen.MalformedPayload):  # truncated / trailing bytes
        zen.decode(zen.EncodedMessage(tb.format, 1000, tb.count, tb.index_bits, tb.value_bits,
                                      tb.payload[:-4]))
    table = zen.HashUniverseTable(1000, 4, 7)
    own = table.universe(0).indices
    foreign = int(next(i for i in range(1000) if i not in set(own.tolist())))
    with pytest.raises(zen.IndexOutsideUniverse):
        zen.encode(zen.SparseTensor(1000, [foreign], [1.0]), zen.WireFormat.hash_bitmap(),
                   table.universe(0))
    buf = io.BytesIO()
    zen.write_framed(buf, ok)
    raw = buf.getvalue()
    with pytest.raises(zen.MalformedPayload):
        zen.read_framed(io.BytesIO(raw[:-1]))
    with pytest.raises(zen.MalformedPayload):  # unknown tag
        zen.read_framed(io.BytesIO(b"\x09" + raw[1:]))


@pytest.mark.parametrize("seed", range(4))
def test_wire_random_vs_oracle(zen, co, seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(10, 200_000))
    z = int(rng.integers(0, min(m, 3000)))
    idx = np.sort(rng.choice(m, z, replace=False)).astype(np.uint64)
    val = rng.standard_normal(z).astype(np.float32)
    t = zen.SparseTensor(m, idx, val)
    for kind, kw in [("coo", {"coo_bits": 64}), ("coo", {"coo_bits": 32}), ("bitmap", {}),
                     ("tensor_block", {"block_size": int(rng.integers(1, 300))})]:
        fmt = zen.WireFormat(kind, kw.get("block_size", 256), kw.get("coo_bits", 64))
        msg = zen.encode(t, fmt)
        want, info = co.wire_encode(kind, m, idx, val, **kw)
        np.testing.assert_array_equal(msg.payload, want)
        assert (msg.count, msg.index_bits, msg.value_bits) == \
            (info["count"], info["index_bits"], info["value_bits"])
        d = zen.decode(msg)
        wi, wv = co.wire_decode(kind, m, info["count"], want, **kw)
        np.testing.assert_array_equal(d.indices(), wi)
        np.testing.assert_array_equal(d.values(), wv)


def test_wire_full_size_round_trips(zen):
    """1M x 64 universe, 640K entries: every format round-trips exactly."""
    rng = np.random.default_rng(64)
    m = 64_000_000
    rows = np.sort(rng.choice(1_000_000, 10_000, replace=False)).astype(np.uint64)
    idx = (rows[:, None] * 64 + np.arange(64, dtype=np.uint64)).ravel()
    val = rng.integers(1, 17, idx.size).astype(np.float32)
    t = zen.SparseTensor(m, idx, val)
    for fmt in [zen.WireFormat.coo(), zen.WireFormat.coo(32), zen.WireFormat.bitmap(),
                zen.WireFormat.tensor_block(64), zen.WireFormat.tensor_block(256)]:
        msg = zen.encode(t, fmt)
        d = zen.decode(msg)
        assert d == t, fmt
    assert zen.encode(t, zen.WireFormat.tensor_block(64)).count == 10_000


def test_sparse_file_golden(zen, tmp_path):
    g = load_golden("wire")
    t = zen.SparseTensor(int(g["zspt_m"][0]), g["zspt_idx"], g["zspt_val"])
    p = tmp_path / "t.zspt"
    zen.write_sparse_file(str(p), t)
    np.testing.assert_array_equal(np.frombuffer(p.read_bytes(), np.uint8), g["zspt_bytes"])
    assert zen.read_sparse_file(str(p)) == t
