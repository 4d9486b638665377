"""ctypes front-end for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/:

* ``C``   -- oracle/liboracle.so, the plain-C restatement of the reference
  hot path (oracle/zen_oracle.c, every function cites zen/*.hpp lines).
* ``Ref`` -- oracle/_ref/libzenref.so, the reference's own headers compiled in
  place from /root/reference by oracle/Makefile (a thin extern "C" shim).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module.  The product (paper_2309_13254_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libzenref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

OK, INVALID, SERIAL_OVERFLOW, OUTSIDE, MALFORMED, EMPTY, MISMATCH = 0, 1, 2, 3, 4, 5, 6
NON_POWER_OF_TWO, MISSING_PROFILE_ENTRY = 7, 8


class OracleError(RuntimeError):
    def __init__(self, code, msg="", partition=-1):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code
        self.partition = partition


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _ZoFamily(C.Structure):
    _fields_ = [("partition_seed", C.c_uint64), ("slot_seeds", C.c_uint64 * 16),
                ("partitions", C.c_uint32), ("k", C.c_uint32)]


class _ZoParams(C.Structure):
    _fields_ = [("rehash_depth", C.c_uint32), ("r1_multiplier", C.c_double),
                ("r2_ratio", C.c_double), ("lanes", C.c_uint32), ("seed", C.c_uint64)]


class _ZoWire(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("block_size", C.c_uint32), ("coo_index_bits", C.c_uint32)]


class _ZoMsg(C.Structure):
    _fields_ = [("universe_size", C.c_uint64), ("count", C.c_uint64), ("index_bits", C.c_uint64),
                ("value_bits", C.c_uint64), ("payload_len", C.c_uint64)]


WIRE_KINDS = {"coo": 1, "bitmap": 2, "tensor_block": 3, "hash_bitmap": 4}


@dataclass
class HashResult:
    parts_idx: list
    parts_val: list
    serial_writes: int = 0
    placed_at_depth: list | None = None
    slots: np.ndarray | None = None
    slot_vals: np.ndarray | None = None
    depth_of: np.ndarray | None = None


@dataclass
class BPResult:
    idx: np.ndarray
    val: np.ndarray
    ledger: np.ndarray  # [2 stages][4 fields][n]
    balance: tuple | None
    counts: np.ndarray | None = None
    agg_counts: np.ndarray | None = None


class COracle:
    """The C restatement (oracle/zen_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        L = self.lib = C.CDLL(path)
        L.zo_mix64.restype = C.c_uint64
        L.zo_mix64.argtypes = [C.c_uint64]
        L.zo_derive_seed.restype = C.c_uint64
        L.zo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.zo_family_make.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(_ZoFamily)]
        L.zo_family_make_worker.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.POINTER(_ZoFamily)]
        L.zo_partition_of_many.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, u32p]
        L.zo_family_slot_of.restype = C.c_uint64
        L.zo_family_slot_of.argtypes = [C.POINTER(_ZoFamily), C.c_uint64, C.c_uint32, C.c_uint64]
        L.zo_hierarchical_hash.argtypes = [
            u64p, f32p, C.c_uint64, C.c_uint64, C.POINTER(_ZoFamily), C.c_uint64, C.c_uint64,
            u64p, f32p, u64p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
            u64p, C.POINTER(C.c_int64)]
        L.zo_to_sparse.restype = C.c_uint64
        L.zo_to_sparse.argtypes = [f32p, C.c_uint64, u64p, f32p]
        L.zo_merge_sum.restype = C.c_uint64
        L.zo_merge_sum.argtypes = [u64p, f32p, C.c_uint64, u64p, f32p, C.c_uint64, u64p, f32p]
        L.zo_universe_create.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p)]
        L.zo_universe_destroy.argtypes = [C.c_void_p]
        L.zo_universe_size.restype = C.c_uint64
        L.zo_universe_size.argtypes = [C.c_void_p, C.c_uint32]
        L.zo_universe_list.restype = C.POINTER(C.c_uint64)
        L.zo_universe_list.argtypes = [C.c_void_p, C.c_uint32]
        L.zo_hash_bitmap_encode.argtypes = [C.c_void_p, C.c_uint32, u64p, f32p, C.c_uint64, u8p,
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.zo_hash_bitmap_decode.argtypes = [C.c_void_p, C.c_uint32, u8p, C.c_uint64, C.c_uint64,
                                            u64p, f32p]
        L.zo_bp_sync.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), u64p,
            C.POINTER(_ZoParams), C.c_void_p, u64p, f32p, C.POINTER(C.c_uint64), u64p, u64p, u64p,
            f64p, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_uint32)]
        L.zo_bp_sizes.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint32,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.zo_wire_encode.argtypes = [C.POINTER(_ZoWire), C.c_void_p, C.c_uint32, C.c_uint64, u64p,
                                     f32p, C.c_uint64, u8p, C.c_uint64, C.POINTER(_ZoMsg)]
        L.zo_wire_decode.argtypes = [C.POINTER(_ZoWire), C.c_void_p, C.c_uint32,
                                     C.POINTER(_ZoMsg), u8p, u64p, f32p, C.c_uint64,
                                     C.POINTER(C.c_uint64)]
        L.zo_frame_header.argtypes = [C.POINTER(_ZoWire), C.POINTER(_ZoMsg), u8p]
        L.zo_frame_parse.argtypes = [u8p, C.c_uint64, C.POINTER(_ZoWire), C.POINTER(_ZoMsg)]
        L.zo_sparse_file_size.restype = C.c_uint64
        L.zo_sparse_file_size.argtypes = [C.c_uint64]
        L.zo_write_sparse.argtypes = [C.c_uint64, u64p, f32p, C.c_uint64, u8p]
        L.zo_read_sparse.argtypes = [u8p, C.c_uint64, C.POINTER(C.c_uint64), u64p, f32p,
                                     C.c_uint64, C.POINTER(C.c_uint64)]
        L.zo_sparsify_topk.restype = C.c_uint64
        L.zo_sparsify_topk.argtypes = [f32p, C.c_uint64, C.c_double, u64p, f32p]

    # -- hash family -------------------------------------------------------
    def mix64(self, x):
        return self.lib.zo_mix64(x)

    def derive_seed(self, m, s):
        return self.lib.zo_derive_seed(m, s)

    def family(self, seed, n, k, worker=None):
        f = _ZoFamily()
        rc = (self.lib.zo_family_make(seed, n, k, C.byref(f)) if worker is None else
              self.lib.zo_family_make_worker(seed, worker, n, k, C.byref(f)))
        if rc:
            raise OracleError(rc, "family")
        return f

    def family_seeds(self, seed, n, k, worker=None):
        f = self.family(seed, n, k, worker)
        return [f.partition_seed] + [f.slot_seeds[i] for i in range(k)]

    def partition_of(self, idx, pseed, n):
        idx = _u64(idx)
        out = np.empty(idx.size, np.uint32)
        self.lib.zo_partition_of_many(idx, idx.size, pseed, n, out)
        return out

    def slot_of(self, fam, index, rnd, r1):
        return self.lib.zo_family_slot_of(C.byref(fam), index, rnd, r1)

    # -- hierarchical hash ------------------------------------------------
    def hierarchical_hash(self, m, idx, val, fam, r1, r2, layout=False):
        idx, val = _u64(idx), _f32(val)
        n, k = fam.partitions, fam.k
        oi = np.empty(max(idx.size, 1), np.uint64)
        ov = np.empty(max(idx.size, 1), np.float32)
        pc = np.zeros(n, np.uint64)
        cells = n * (r1 + r2)
        slots = np.zeros(max(cells, 1), np.uint64) if layout else None
        svals = np.zeros(max(cells, 1), np.float32) if layout else None
        depth = np.zeros(max(idx.size, 1), np.uint32) if layout else None
        serial = C.c_uint64(0)
        pad = np.zeros(k, np.uint64)
        ovf = C.c_int64(-1)
        rc = self.lib.zo_hierarchical_hash(
            idx, val, idx.size, m, C.byref(fam), r1, r2, oi, ov, pc,
            slots.ctypes.data if layout else None, svals.ctypes.data if layout else None,
            depth.ctypes.data if layout else None, C.byref(serial), pad, C.byref(ovf))
        if rc == SERIAL_OVERFLOW:
            raise OracleError(rc, "serial overflow", ovf.value)
        if rc:
            raise OracleError(rc, "hierarchical_hash")
        offs = np.concatenate([[0], np.cumsum(pc)]).astype(np.int64)
        res = HashResult([oi[offs[p]:offs[p + 1]].copy() for p in range(n)],
                         [ov[offs[p]:offs[p + 1]].copy() for p in range(n)],
                         int(serial.value), [int(x) for x in pad])
        if layout:
            res.slots, res.slot_vals, res.depth_of = slots[:cells], svals[:cells], depth[:idx.size]
        return res

    def to_sparse(self, dense):
        dense = _f32(dense)
        idx = np.empty(max(dense.size, 1), np.uint64)
        val = np.empty(max(dense.size, 1), np.float32)
        c = self.lib.zo_to_sparse(dense, dense.size, idx, val)
        return idx[:c].copy(), val[:c].copy()

    def merge_sum(self, ia, va, ib, vb):
        ia, va, ib, vb = _u64(ia), _f32(va), _u64(ib), _f32(vb)
        io = np.empty(max(ia.size + ib.size, 1), np.uint64)
        vo = np.empty(max(ia.size + ib.size, 1), np.float32)
        c = self.lib.zo_merge_sum(ia, va, ia.size, ib, vb, ib.size, io, vo)
        return io[:c].copy(), vo[:c].copy()

    def aggregate(self, tensors):
        ai, av = _u64(tensors[0][0]), _f32(tensors[0][1])
        for ti, tv in tensors[1:]:
            ai, av = self.merge_sum(ai, av, ti, tv)
        return ai, av

    # -- universe / codec -------------------------------------------------
    def universe(self, m, n, pseed):
        return _Universe(self, m, n, pseed)

    # -- BP ----------------------------------------------------------------
    def bp_sizes(self, r1m, r2r, nnz, n):
        a, b = C.c_uint64(), C.c_uint64()
        self.lib.zo_bp_sizes(r1m, r2r, nnz, n, C.byref(a), C.byref(b))
        return a.value, b.value

    def bp_sync(self, m, inputs, k=3, r1_multiplier=2.0, r2_ratio=0.1, seed=1, universe=None):
        n = len(inputs)
        ins = [(_u64(i), _f32(v)) for i, v in inputs]
        nnz = np.array([i.size for i, _ in ins], np.uint64)
        ip = (C.c_void_p * n)(*[i.ctypes.data for i, _ in ins])
        vp = (C.c_void_p * n)(*[v.ctypes.data for _, v in ins])
        p = _ZoParams(k, r1_multiplier, r2_ratio, 1, seed)
        u = universe or self.universe(m, n, self.derive_seed(seed, 0))
        tot = int(nnz.sum())
        oi = np.empty(max(tot, 1), np.uint64)
        ov = np.empty(max(tot, 1), np.float32)
        oc = C.c_uint64(0)
        ledger = np.zeros(8 * n, np.uint64)
        counts = np.zeros(n * n, np.uint64)
        agg = np.zeros(n, np.uint64)
        bal = np.zeros(2, np.float64)
        bv = C.c_int(0)
        op, ow = C.c_int64(-1), C.c_uint32(0)
        rc = self.lib.zo_bp_sync(n, m, ip, vp, nnz, C.byref(p), u.h, oi, ov, C.byref(oc), ledger,
                                 counts, agg, bal, C.byref(bv), C.byref(op), C.byref(ow))
        if rc == SERIAL_OVERFLOW:
            e = OracleError(rc, "serial overflow", op.value)
            e.worker = ow.value
            raise e
        if rc:
            raise OracleError(rc, "bp_sync")
        c = oc.value
        return BPResult(oi[:c].copy(), ov[:c].copy(), ledger.reshape(2, 4, n),
                        (bal[0], bal[1]) if bv.value else None, counts.reshape(n, n), agg)


def _wire_cap(kind, m, z, block_size):
    k = WIRE_KINDS[kind] if isinstance(kind, str) else kind
    if k == 1:
        return 64 + 12 * z
    if k == 3:
        return 64 + (8 + 4 * block_size) * z
    return 64 + (m + 7) // 8 + 4 * z


def _wire(kind, block_size=256, coo_bits=64):
    return _ZoWire(WIRE_KINDS[kind] if isinstance(kind, str) else kind, block_size, coo_bits)


def _co_wire_encode(self, kind, m, idx, val, block_size=256, coo_bits=64, universe=None,
                    server=0):
    """zen::encode (zen/codec.hpp:213-278) -> (payload bytes, info dict)."""
    idx, val = _u64(idx), _f32(val)
    cap = _wire_cap(kind, m, idx.size, block_size)
    buf = np.zeros(cap, np.uint8)
    msg = _ZoMsg()
    rc = self.lib.zo_wire_encode(C.byref(_wire(kind, block_size, coo_bits)),
                                 universe.h if universe else None, server, m, idx, val, idx.size,
                                 buf, cap, C.byref(msg))
    if rc:
        raise OracleError(rc, "wire encode")
    return buf[:msg.payload_len].copy(), {"count": msg.count, "index_bits": msg.index_bits,
                                          "value_bits": msg.value_bits}


def _co_wire_decode(self, kind, m, count, payload, block_size=256, coo_bits=64, universe=None,
                    server=0):
    payload = np.ascontiguousarray(payload, np.uint8)
    msg = _ZoMsg(m, count, 0, 0, payload.size)
    cap = max(count, 1) * (block_size if WIRE_KINDS.get(kind, kind) == 3 else 1) + 1
    idx = np.empty(cap, np.uint64)
    val = np.empty(cap, np.float32)
    oc = C.c_uint64()
    rc = self.lib.zo_wire_decode(C.byref(_wire(kind, block_size, coo_bits)),
                                 universe.h if universe else None, server, C.byref(msg), payload,
                                 idx, val, cap, C.byref(oc))
    if rc:
        raise OracleError(rc, "wire decode")
    return idx[:oc.value].copy(), val[:oc.value].copy()


def _co_frame(self, kind, m, payload, info, block_size=256, coo_bits=64):
    """write_framed (zen/codec.hpp:356-366): 33-byte header + payload."""
    hdr = np.zeros(33, np.uint8)
    msg = _ZoMsg(m, info["count"], info["index_bits"], info["value_bits"], len(payload))
    self.lib.zo_frame_header(C.byref(_wire(kind, block_size, coo_bits)), C.byref(msg), hdr)
    return np.concatenate([hdr, np.asarray(payload, np.uint8)])


def _co_unframe(self, framed):
    framed = np.ascontiguousarray(framed, np.uint8)
    f, msg = _ZoWire(), _ZoMsg()
    rc = self.lib.zo_frame_parse(framed, framed.size, C.byref(f), C.byref(msg))
    if rc:
        raise OracleError(rc, "frame")
    return ({"kind": f.kind, "block_size": f.block_size, "coo_index_bits": f.coo_index_bits,
             "universe_size": msg.universe_size, "count": msg.count,
             "index_bits": msg.index_bits, "value_bits": msg.value_bits},
            framed[33:33 + msg.payload_len].copy())


def _co_write_sparse(self, m, idx, val):
    idx, val = _u64(idx), _f32(val)
    out = np.zeros(int(self.lib.zo_sparse_file_size(idx.size)), np.uint8)
    self.lib.zo_write_sparse(m, idx, val, idx.size, out)
    return out


def _co_read_sparse(self, data):
    data = np.ascontiguousarray(data, np.uint8)
    cap = max(data.size // 12, 1)
    idx = np.empty(cap, np.uint64)
    val = np.empty(cap, np.float32)
    m, c = C.c_uint64(), C.c_uint64()
    rc = self.lib.zo_read_sparse(data, data.size, C.byref(m), idx, val, cap, C.byref(c))
    if rc:
        raise OracleError(rc, "read_sparse")
    return m.value, idx[:c.value].copy(), val[:c.value].copy()


def _co_sparsify_topk(self, dense, fraction):
    dense = _f32(dense)
    keep = min(dense.size, int(np.ceil(fraction * dense.size))) if 0 < fraction <= 1 else 1
    idx = np.empty(max(keep, 1), np.uint64)
    val = np.empty(max(keep, 1), np.float32)
    c = self.lib.zo_sparsify_topk(dense, dense.size, fraction, idx, val)
    if c == 2**64 - 1:
        raise OracleError(1, "top-k fraction must be in (0,1]")
    return idx[:c].copy(), val[:c].copy()


COracle.wire_encode = _co_wire_encode
COracle.wire_decode = _co_wire_decode
COracle.frame = _co_frame
COracle.unframe = _co_unframe
COracle.write_sparse = _co_write_sparse
COracle.read_sparse = _co_read_sparse
COracle.sparsify_topk = _co_sparsify_topk


class _Universe:
    def __init__(self, co, m, n, pseed):
        self.co, self.m, self.n, self.pseed = co, m, n, pseed
        h = C.c_void_p()
        rc = co.lib.zo_universe_create(m, n, pseed, C.byref(h))
        if rc:
            raise OracleError(rc, "universe")
        self.h = h

    def __del__(self):
        try:
            self.co.lib.zo_universe_destroy(self.h)
        except Exception:
            pass

    def size(self, s):
        return int(self.co.lib.zo_universe_size(self.h, s))

    def indices(self, s):
        sz = self.size(s)
        p = self.co.lib.zo_universe_list(self.h, s)
        return np.ctypeslib.as_array(p, shape=(max(sz, 1),))[:sz].copy()

    def encode(self, s, idx, val):
        idx, val = _u64(idx), _f32(val)
        nbytes = (self.size(s) + 7) // 8 + 4 * idx.size
        payload = np.zeros(max(nbytes, 1), np.uint8)
        bits, bad = C.c_uint64(), C.c_uint64()
        rc = self.co.lib.zo_hash_bitmap_encode(self.h, s, idx, val, idx.size, payload,
                                               C.byref(bits), C.byref(bad))
        if rc:
            raise OracleError(rc, f"encode (index {bad.value})")
        return payload[:nbytes], bits.value

    def decode(self, s, payload, count):
        payload = np.ascontiguousarray(payload, np.uint8)
        idx = np.empty(max(count, 1), np.uint64)
        val = np.empty(max(count, 1), np.float32)
        rc = self.co.lib.zo_hash_bitmap_decode(self.h, s, payload, payload.size, count, idx, val)
        if rc:
            raise OracleError(rc, "decode")
        return idx[:count].copy(), val[:count].copy()


class RefOracle:
    """The reference itself (oracle/_ref/libzenref.so, compiled from /root/reference)."""

    def __init__(self, path=REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_partition.restype = C.c_int64
        L.ref_last_message.restype = C.c_char_p
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_family.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, u64p]
        L.ref_partition_of_many.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint32, u32p]
        L.ref_slot_of_many.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                       u64p, C.c_uint64, C.c_uint64, u64p]
        L.ref_hierarchical_hash.argtypes = [
            C.c_uint64, u64p, f32p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
            C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, u64p, f32p, u64p, u64p]
        L.ref_slot_layout.argtypes = [
            C.c_uint64, u64p, f32p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_uint32,
            C.c_uint32, C.c_uint64, C.c_uint64, u64p, f32p, u32p, C.POINTER(C.c_int64)]
        L.ref_to_sparse.restype = C.c_uint64
        L.ref_to_sparse.argtypes = [f32p, C.c_uint64, u64p, f32p]
        L.ref_generate.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, u64p, f32p, C.POINTER(C.c_uint64)]
        L.ref_universe_size.restype = C.c_uint64
        L.ref_universe_size.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
        L.ref_hash_bitmap_encode.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, u64p,
                                             f32p, C.c_uint64, u8p, C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64)]
        L.ref_hash_bitmap_decode.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, u8p,
                                             C.c_uint64, C.c_uint64, u64p, f32p,
                                             C.POINTER(C.c_uint64)]
        L.ref_bp_sync.argtypes = [
            C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), u64p, C.c_uint32,
            C.c_double, C.c_double, C.c_uint32, C.c_uint64, C.c_int, u64p, f32p,
            C.POINTER(C.c_uint64), u64p, f64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_aggregate.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_void_p), u64p, u64p, f32p, C.POINTER(C.c_uint64)]
        L.ref_wire_encode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                      C.c_uint64, C.c_uint32, u64p, f32p, C.c_uint64, u8p,
                                      C.c_uint64, u64p]
        L.ref_wire_decode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                      C.c_uint64, C.c_uint32, C.c_uint64, u8p, C.c_uint64, u64p,
                                      f32p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_write_framed.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                       C.c_uint64, C.c_uint32, u64p, f32p, C.c_uint64, u8p,
                                       C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_write_sparse.argtypes = [C.c_uint64, u64p, f32p, C.c_uint64, u8p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
        L.ref_sparsify_topk.argtypes = [f32p, C.c_uint64, C.c_double, u64p, f32p,
                                        C.POINTER(C.c_uint64)]
        vpp = C.POINTER(C.c_void_p)
        L.ref_merge_sum.argtypes = [C.c_uint64, u64p, f32p, C.c_uint64, u64p, f32p, C.c_uint64,
                                    u64p, f32p, C.POINTER(C.c_uint64)]
        L.ref_tensor_metric.argtypes = [C.c_int, C.c_uint32, C.c_uint64, vpp, vpp, u64p,
                                        C.c_uint32, C.POINTER(C.c_double)]
        L.ref_profile.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, vpp, vpp, u64p,
                                  C.POINTER(C.c_double), f64p, C.c_uint32, C.POINTER(C.c_double),
                                  C.POINTER(C.c_int)]
        L.ref_hier_centralization.argtypes = [
            C.c_uint32, C.c_uint64, vpp, vpp, u64p, C.c_uint32, C.c_uint32, C.c_uint32, u64p,
            f32p, C.POINTER(C.c_uint64), u64p, C.c_uint32, C.POINTER(C.c_uint32),
            C.POINTER(C.c_int)]
        L.ref_run_scheme.argtypes = [
            C.c_char_p, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, vpp,
            vpp, u64p, C.c_uint64, u64p, f32p, u64p, u64p, C.c_uint32, C.POINTER(C.c_uint32),
            f64p, C.POINTER(C.c_int)]
        L.ref_bench_step.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), C.c_uint32,
                                     C.c_double, C.c_double, C.c_uint32, C.c_uint64, C.c_int, f64p,
                                     C.POINTER(C.c_uint64)]

    def _check(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self.lib.ref_last_message().decode()}",
                              self.lib.ref_last_partition())

    def mix64(self, x):
        return self.lib.ref_mix64(x)

    def derive_seed(self, m, s):
        return self.lib.ref_derive_seed(m, s)

    def family_seeds(self, seed, n, k, worker=None):
        out = np.zeros(k + 1, np.uint64)
        self._check(self.lib.ref_family(seed, worker or 0, n, k, int(worker is not None), out),
                    "family")
        return [int(x) for x in out]

    def partition_of(self, idx, pseed, n):
        idx = _u64(idx)
        out = np.empty(idx.size, np.uint32)
        self.lib.ref_partition_of_many(idx, idx.size, pseed, n, out)
        return out

    def slot_of(self, seed, n, k, idx, r1, worker=None):
        idx = _u64(idx)
        out = np.empty(idx.size * k, np.uint64)
        self.lib.ref_slot_of_many(seed, worker or 0, n, k, int(worker is not None), idx, idx.size,
                                  r1, out)
        return out.reshape(idx.size, k)

    def hierarchical_hash(self, m, idx, val, seed, n, k, r1, r2, worker=None, lanes=1,
                          stats=True):
        idx, val = _u64(idx), _f32(val)
        oi = np.empty(max(idx.size, 1), np.uint64)
        ov = np.empty(max(idx.size, 1), np.float32)
        pc = np.zeros(n, np.uint64)
        st = np.zeros(k + 1, np.uint64)
        self._check(self.lib.ref_hierarchical_hash(m, idx, val, idx.size, seed, worker or 0,
                                                   int(worker is not None), n, k, r1, r2, lanes,
                                                   oi, ov, pc, st), "hierarchical_hash")
        offs = np.concatenate([[0], np.cumsum(pc)]).astype(np.int64)
        return HashResult([oi[offs[p]:offs[p + 1]].copy() for p in range(n)],
                          [ov[offs[p]:offs[p + 1]].copy() for p in range(n)],
                          int(st[0]), [int(x) for x in st[1:]])

    def slot_layout(self, m, idx, val, seed, n, k, r1, r2, worker=None):
        idx, val = _u64(idx), _f32(val)
        cells = n * (r1 + r2)
        slots = np.zeros(max(cells, 1), np.uint64)
        svals = np.zeros(max(cells, 1), np.float32)
        depth = np.zeros(max(idx.size, 1), np.uint32)
        ovf = C.c_int64(-1)
        self._check(self.lib.ref_slot_layout(m, idx, val, idx.size, seed, worker or 0,
                                             int(worker is not None), n, k, r1, r2, slots, svals,
                                             depth, C.byref(ovf)), "slot_layout")
        return slots[:cells], svals[:cells], depth[:idx.size], ovf.value

    def to_sparse(self, dense):
        dense = _f32(dense)
        idx = np.empty(max(dense.size, 1), np.uint64)
        val = np.empty(max(dense.size, 1), np.float32)
        c = self.lib.ref_to_sparse(dense, dense.size, idx, val)
        return idx[:c].copy(), val[:c].copy()

    def generate(self, m, nodes, density, omega, seed, hot_fraction=0.125, hot_mass=0.125):
        z = int(np.ceil(density * m))
        idx = np.zeros(max(z * nodes, 1), np.uint64)
        val = np.zeros(max(z * nodes, 1), np.float32)
        zz = C.c_uint64()
        self._check(self.lib.ref_generate(m, nodes, density, omega, hot_fraction, hot_mass, seed,
                                          idx, val, C.byref(zz)), "generate")
        z = zz.value
        return [(idx[w * z:(w + 1) * z].copy(), val[w * z:(w + 1) * z].copy())
                for w in range(nodes)]

    def universe_size(self, m, n, pseed, s):
        return int(self.lib.ref_universe_size(m, n, pseed, s))

    def hash_bitmap_encode(self, m, n, pseed, s, idx, val):
        idx, val = _u64(idx), _f32(val)
        size = self.universe_size(m, n, pseed, s)
        payload = np.zeros((size + 7) // 8 + 4 * idx.size + 1, np.uint8)
        bits, plen = C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_hash_bitmap_encode(m, n, pseed, s, idx, val, idx.size, payload,
                                                    C.byref(bits), C.byref(plen)), "encode")
        return payload[:plen.value].copy(), bits.value

    def hash_bitmap_decode(self, m, n, pseed, s, payload, count):
        payload = np.ascontiguousarray(payload, np.uint8)
        idx = np.empty(max(count, 1), np.uint64)
        val = np.empty(max(count, 1), np.float32)
        oc = C.c_uint64()
        self._check(self.lib.ref_hash_bitmap_decode(m, n, pseed, s, payload, payload.size, count,
                                                    idx, val, C.byref(oc)), "decode")
        return idx[:oc.value].copy(), val[:oc.value].copy()

    def _ptrs(self, inputs):
        n = len(inputs)
        ins = [(_u64(i), _f32(v)) for i, v in inputs]
        nnz = np.array([i.size for i, _ in ins], np.uint64)
        ip = (C.c_void_p * n)(*[i.ctypes.data for i, _ in ins])
        vp = (C.c_void_p * n)(*[v.ctypes.data for _, v in ins])
        return ins, nnz, ip, vp

    def bp_sync(self, m, inputs, k=3, r1_multiplier=2.0, r2_ratio=0.1, seed=1, lanes=1,
                retries=0):
        n = len(inputs)
        ins, nnz, ip, vp = self._ptrs(inputs)
        tot = int(nnz.sum())
        oi = np.empty(max(tot, 1), np.uint64)
        ov = np.empty(max(tot, 1), np.float32)
        oc = C.c_uint64()
        ledger = np.zeros(8 * n, np.uint64)
        bal = np.zeros(2, np.float64)
        bv, eq = C.c_int(0), C.c_int(0)
        self._check(self.lib.ref_bp_sync(n, m, ip, vp, nnz, k, r1_multiplier, r2_ratio, lanes,
                                         seed, retries, oi, ov, C.byref(oc), ledger, bal,
                                         C.byref(bv), C.byref(eq)), "bp_sync")
        assert eq.value == 1
        c = oc.value
        return BPResult(oi[:c].copy(), ov[:c].copy(), ledger.reshape(2, 4, n),
                        (bal[0], bal[1]) if bv.value else None)

    def aggregate(self, m, inputs):
        ins, nnz, ip, vp = self._ptrs(inputs)
        tot = int(nnz.sum())
        oi = np.empty(max(tot, 1), np.uint64)
        ov = np.empty(max(tot, 1), np.float32)
        oc = C.c_uint64()
        self._check(self.lib.ref_aggregate(len(inputs), m, ip, vp, nnz, oi, ov, C.byref(oc)),
                    "aggregate")
        return oi[:oc.value].copy(), ov[:oc.value].copy()

    def bench_step(self, m, dense_list, k=3, r1_multiplier=2.0, r2_ratio=0.1, lanes=1, seed=1,
                   reps=1):
        n = len(dense_list)
        ds = [_f32(d) for d in dense_list]
        dp = (C.c_void_p * n)(*[d.ctypes.data for d in ds])
        t = np.zeros(3, np.float64)
        rn = C.c_uint64()
        self._check(self.lib.ref_bench_step(n, m, dp, k, r1_multiplier, r2_ratio, lanes, seed,
                                            reps, t, C.byref(rn)), "bench_step")
        return {"to_sparse_ms": t[0], "sync_ms": t[1], "table_ms": t[2], "result_nnz": rn.value}


def _ref_wire_encode(self, kind, m, idx, val, block_size=256, coo_bits=64, n=1, pseed=0,
                     server=0):
    idx, val = _u64(idx), _f32(val)
    k = WIRE_KINDS[kind] if isinstance(kind, str) else kind
    cap = _wire_cap(k, m, idx.size, block_size)
    buf = np.zeros(cap, np.uint8)
    info = np.zeros(4, np.uint64)
    self._check(self.lib.ref_wire_encode(k, block_size, coo_bits, m, n, pseed, server, idx, val,
                                         idx.size, buf, cap, info), "wire encode")
    return buf[:int(info[3])].copy(), {"count": int(info[0]), "index_bits": int(info[1]),
                                       "value_bits": int(info[2])}


def _ref_wire_decode(self, kind, m, count, payload, block_size=256, coo_bits=64, n=1, pseed=0,
                     server=0):
    payload = np.ascontiguousarray(payload, np.uint8)
    k = WIRE_KINDS[kind] if isinstance(kind, str) else kind
    cap = max(count, 1) * (block_size if k == 3 else 1) + 1
    idx = np.empty(cap, np.uint64)
    val = np.empty(cap, np.float32)
    oc = C.c_uint64()
    self._check(self.lib.ref_wire_decode(k, block_size, coo_bits, m, n, pseed, server, count,
                                         payload, payload.size, idx, val, cap, C.byref(oc)),
                "wire decode")
    return idx[:oc.value].copy(), val[:oc.value].copy()


def _ref_write_framed(self, kind, m, idx, val, block_size=256, coo_bits=64, n=1, pseed=0,
                      server=0):
    idx, val = _u64(idx), _f32(val)
    k = WIRE_KINDS[kind] if isinstance(kind, str) else kind
    cap = 64 + _wire_cap(k, m, idx.size, block_size)
    buf = np.zeros(cap, np.uint8)
    ol = C.c_uint64()
    self._check(self.lib.ref_write_framed(k, block_size, coo_bits, m, n, pseed, server, idx, val,
                                          idx.size, buf, cap, C.byref(ol)), "write_framed")
    return buf[:ol.value].copy()


def _ref_write_sparse(self, m, idx, val):
    idx, val = _u64(idx), _f32(val)
    buf = np.zeros(24 + 12 * idx.size, np.uint8)
    ol = C.c_uint64()
    self._check(self.lib.ref_write_sparse(m, idx, val, idx.size, buf, buf.size, C.byref(ol)),
                "write_sparse")
    return buf[:ol.value].copy()


def _ref_sparsify_topk(self, dense, fraction):
    dense = _f32(dense)
    idx = np.empty(max(dense.size, 1), np.uint64)
    val = np.empty(max(dense.size, 1), np.float32)
    oc = C.c_uint64()
    self._check(self.lib.ref_sparsify_topk(dense, dense.size, fraction, idx, val, C.byref(oc)),
                "sparsify_topk")
    return idx[:oc.value].copy(), val[:oc.value].copy()


# ---- f3: merge_sum, metrics, profile / selector, Hierarchical Centralization ----

def _ref_merge_sum(self, m, ia, va, ib, vb):
    ia, va, ib, vb = _u64(ia), _f32(va), _u64(ib), _f32(vb)
    oi = np.empty(max(ia.size + ib.size, 1), np.uint64)
    ov = np.empty(max(ia.size + ib.size, 1), np.float32)
    oc = C.c_uint64()
    self._check(self.lib.ref_merge_sum(m, ia, va, ia.size, ib, vb, ib.size, oi, ov, C.byref(oc)),
                "merge_sum")
    return oi[:oc.value].copy(), ov[:oc.value].copy()


def _ref_metric(self, what, m, inputs, partitions=1):
    ins, nnz, ip, vp = self._ptrs(inputs)
    out = C.c_double()
    self._check(self.lib.ref_tensor_metric(what, len(inputs), m, ip, vp, nnz, partitions,
                                           C.byref(out)), "metric")
    return out.value


def _ref_profile(self, m, rounds):
    """profile_sparsity + select_scheme -> (d, {k: gamma}, skew, choice)."""
    r, n = len(rounds), len(rounds[0])
    flat = [t for rnd in rounds for t in rnd]
    ins, nnz, ip, vp = self._ptrs(flat)
    glen = max(n.bit_length(), 1)
    gamma = np.zeros(glen, np.float64)
    d, skew, ch = C.c_double(), C.c_double(), C.c_int()
    self._check(self.lib.ref_profile(r, n, m, ip, vp, nnz, C.byref(d), gamma, glen,
                                     C.byref(skew), C.byref(ch)), "profile")
    g = {1 << j: float(gamma[j]) for j in range(glen) if not np.isnan(gamma[j])}
    return d.value, g, skew.value, ch.value


def _ref_hier_centralization(self, m, inputs, kind="coo", block_size=256, coo_bits=64):
    """run_hier_centralization -> (idx, val, ledger[stages][4][n])."""
    n = len(inputs)
    ins, nnz, ip, vp = self._ptrs(inputs)
    tot = int(nnz.sum())
    oi = np.empty(max(tot, 1), np.uint64)
    ov = np.empty(max(tot, 1), np.float32)
    oc, ns, eq = C.c_uint64(), C.c_uint32(), C.c_int()
    ledger = np.zeros(8 * 4 * n, np.uint64)
    k = WIRE_KINDS[kind] if isinstance(kind, str) else kind
    self._check(self.lib.ref_hier_centralization(n, m, ip, vp, nnz, k, block_size, coo_bits, oi,
                                                 ov, C.byref(oc), ledger, 8, C.byref(ns),
                                                 C.byref(eq)), "hier_centralization")
    assert eq.value == 1
    return (oi[:oc.value].copy(), ov[:oc.value].copy(),
            ledger[:ns.value * 4 * n].reshape(ns.value, 4, n))


COMM = {"ring": 0, "hierarchy": 1, "point-to-point": 2}


def _ref_run_scheme(self, name, m, inputs, comm=None, kind=None, block_size=256, coo_bits=64):
    """run_scheme(scheme_config_from_name(name)) -> (results [(idx, val)] per
    node, ledger [stages][4][n], balance (push, pull) or None)."""
    n = len(inputs)
    ins, nnz, ip, vp = self._ptrs(inputs)
    cap = max(int(nnz.sum()), 1)
    oi = np.zeros(n * cap, np.uint64)
    ov = np.zeros(n * cap, np.float32)
    oc = np.zeros(n, np.uint64)
    ledger = np.zeros(16 * 4 * n, np.uint64)
    ns, bv = C.c_uint32(), C.c_int()
    bal = np.zeros(2, np.float64)
    k = 0 if kind is None else (WIRE_KINDS[kind] if isinstance(kind, str) else kind)
    self._check(self.lib.ref_run_scheme(name.encode(), -1 if comm is None else COMM[comm], k,
                                        block_size, coo_bits, n, m, ip, vp, nnz, cap, oi, ov, oc,
                                        ledger, 16, C.byref(ns), bal, C.byref(bv)), "run_scheme")
    res = [(oi[w * cap:w * cap + int(oc[w])].copy(), ov[w * cap:w * cap + int(oc[w])].copy())
           for w in range(n)]
    return res, ledger[:ns.value * 4 * n].reshape(ns.value, 4, n), \
        ((bal[0], bal[1]) if bv.value else None)


RefOracle.run_scheme = _ref_run_scheme
RefOracle.merge_sum = _ref_merge_sum
RefOracle.metric = _ref_metric
RefOracle.profile = _ref_profile
RefOracle.hier_centralization = _ref_hier_centralization


def _pow2(v):
    return v != 0 and (v & (v - 1)) == 0


def _co_sizes(self, kind, m, idx, val, block_size=256, coo_bits=64):
    """message_sizes (zen/codec.hpp:182-211) -> (index_bits, value_bits)."""
    z = len(idx)
    if kind == "coo":
        return coo_bits * z, 32 * z
    if kind == "bitmap":
        return m, 32 * z
    _, info = self.wire_encode(kind, m, idx, val, block_size, coo_bits)
    return info["index_bits"], info["value_bits"]


def _co_hier_centralization(self, m, inputs, kind="coo", block_size=256, coo_bits=64):
    """Restatement of zen::run_hier_centralization (zen/schemes.hpp:173-193):
    stage log2(bit) sends states[w] to w ^ bit, then every state becomes
    merge_sum(states[w], states[w ^ bit]) (zo_merge_sum, tensor.hpp:133-167).
    Returns (idx, val, ledger[stages][4][n]) like RefOracle."""
    n = len(inputs)
    if not _pow2(n):
        raise OracleError(NON_POWER_OF_TWO, "node count must be a power of two")
    states = [(_u64(i), _f32(v)) for i, v in inputs]
    stages = []
    bit = 1
    while bit < n:
        led = np.zeros((4, n), np.uint64)
        for w in range(n):
            ib, vb = _co_sizes(self, kind, m, *states[w], block_size, coo_bits)
            to = w ^ bit
            led[0, w] += ib + vb
            led[1, to] += ib + vb
            led[2, to] += ib
            led[3, to] += vb
        stages.append(led)
        states = [self.merge_sum(*states[w], *states[w ^ bit]) for w in range(n)]
        bit <<= 1
    for i, v in states[1:]:
        assert np.array_equal(i, states[0][0]) and np.array_equal(v.view(np.uint32),
                                                                   states[0][1].view(np.uint32))
    led = np.stack(stages) if stages else np.zeros((0, 4, n), np.uint64)
    return states[0][0], states[0][1], led


def _co_skewness(m, idx, partitions):
    """zen::skewness_ratio (zen/tensor.hpp:192-213)."""
    idx = _u64(idx)
    rng = (m + partitions - 1) // partitions
    best = 0.0
    for p in range(partitions):
        lo = p * rng
        if lo >= m:
            break
        hi = min(m, lo + rng)
        c = int(np.searchsorted(idx, np.uint64(hi)) - np.searchsorted(idx, np.uint64(lo)))
        best = max(best, float(c) / float(hi - lo))
    return best / (float(idx.size) / float(m))


def _co_profile(self, m, rounds):
    """Restatement of zen::profile_sparsity (zen/costmodel.hpp:151-195) and
    select_scheme (:139-149) -> (d, {k: gamma}, skew, choice 0 BP / 1 HC)."""
    n = len(rounds[0])
    gsum, skew_sum, dsum, dcount = {}, 0.0, 0.0, 0
    for rnd in rounds:
        pds = 0.0
        pi = pv = None
        for i, (ti, tv) in enumerate(rnd):
            d = float(len(ti)) / float(m)
            dsum += d
            dcount += 1
            pi, pv = (_u64(ti), _f32(tv)) if i == 0 else self.merge_sum(pi, pv, ti, tv)
            pds += d
            k = i + 1
            if _pow2(k):
                gsum[k] = gsum.get(k, 0.0) + (float(pi.size) / float(m)) / (pds / float(k))
            skew_sum += _co_skewness(m, ti, n)
    gamma = {k: gsum[k] / float(len(rounds)) for k in sorted(gsum)}
    gamma[1] = 1.0
    choice = -1
    if n in gamma:
        bp = (float(n) - 1.0) / float(n) * (gamma[n] + 1.0) if n > 1 else 0.0
        hc, k = 0.0, 1
        while k < n:
            hc += 1.0 if k == 1 else gamma[k]
            k *= 2
        choice = 0 if bp <= hc else 1
    return dsum / float(dcount), gamma, skew_sum / float(len(rounds) * n), choice


def _co_fold(self, parts):
    i, v = _u64(parts[0][0]), _f32(parts[0][1])
    for pi, pv in parts[1:]:
        i, v = self.merge_sum(i, v, pi, pv)
    return i, v


def _co_run_scheme(self, name, m, inputs, comm=None, kind=None, block_size=256, coo_bits=64):
    """Restatement of run_scheme (zen/schemes.hpp:420-442) for the centralized
    schemes and the OmniReduce-like one (BP has its own oracle): same return
    shape as RefOracle.run_scheme."""
    n = len(inputs)
    ins = [(_u64(i), _f32(v)) for i, v in inputs]
    kind = kind or ("tensor_block" if name == "omnireduce" else "coo")
    if name == "omnireduce":
        block_size = block_size if kind == "tensor_block" else 256
    stages = {}

    def send(stage, frm, to, ib, vb):
        led = stages.setdefault(stage, np.zeros((4, n), np.uint64))
        led[0, frm] += ib + vb
        led[1, to] += ib + vb
        led[2, to] += ib
        led[3, to] += vb

    def sz(t):
        return _co_sizes(self, kind, m, t[0], t[1], block_size, coo_bits)

    balance = None
    if name == "agsparse":  # schemes.hpp:119-168
        comm = comm or "point-to-point"
        if comm == "point-to-point":
            for w in range(n):
                for to in range(n):
                    if to != w:
                        send(0, w, to, *sz(ins[w]))
        elif comm == "ring":
            if not _pow2(n):
                raise OracleError(NON_POWER_OF_TWO)
            for st in range(n - 1):
                for w in range(n):
                    send(st, w, (w + 1) % n, *sz(ins[(w + n - st) % n]))
        else:
            if not _pow2(n):
                raise OracleError(NON_POWER_OF_TWO)
            hold = [[w] for w in range(n)]
            bit = 1
            while bit < n:
                prev = [list(h) for h in hold]
                for w in range(n):
                    for o in prev[w]:
                        send(bit.bit_length() - 1, w, w ^ bit, *sz(ins[o]))
                    hold[w] += prev[w ^ bit]
                bit <<= 1
        r = _co_fold(self, ins)
        results = [r] * n
    elif name == "sparcml":
        i, v, led = _co_hier_centralization(self, m, ins, kind, block_size, coo_bits)
        return [(i, v)] * n, led, None
    elif name == "ring-centralization":  # schemes.hpp:194-215
        if not _pow2(n):
            raise OracleError(NON_POWER_OF_TWO)
        tok = list(ins)
        for st in range(n - 1):
            for w in range(n):
                send(st, w, (w + 1) % n, *sz(tok[w]))
            tok = [self.merge_sum(*tok[(w + n - 1) % n], *ins[w]) for w in range(n)]
        results = tok
    elif name == "omnireduce":  # schemes.hpp:219-328
        rng = (m + n - 1) // n
        sl = [[(i[(i // rng) == p], v[(i // rng) == p]) for p in range(n)] for i, v in ins]

        def blocks(t, p):
            lo, hi = p * rng, min(m, p * rng + rng)
            b = np.unique((t[0] - np.uint64(lo)) // np.uint64(block_size)) if len(t[0]) else []
            vb = sum(32 * min(block_size, hi - (lo + int(x) * block_size)) for x in b)
            return 64 * len(b), vb
        for w in range(n):
            for p in range(n):
                if p != w and len(sl[w][p][0]):
                    send(0, w, p, *blocks(sl[w][p], p))
        agg = [_co_fold(self, [sl[w][p] for w in range(n)]) for p in range(n)]
        for p in range(n):
            if len(agg[p][0]):
                ib, vb = blocks(agg[p], p)
                for w in range(n):
                    if w != p:
                        send(1, p, w, ib, vb)
        ai = np.concatenate([a[0] for a in agg])
        av = np.concatenate([a[1] for a in agg])
        keep = av != 0.0
        results = [(ai[keep], av[keep])] * n
        if all(len(i) for i, _ in ins):
            push = max(float(n) * float(len(sl[w][p][0])) / float(len(ins[w][0]))
                       for w in range(n) for p in range(n))
            loads = [len(a[0]) for a in agg]
            pull = max(float(n) * float(x) / float(sum(loads)) for x in loads)
            balance = (push, pull)
    else:
        raise OracleError(INVALID, "scheme not restated: " + name)
    ns = max(stages) + 1 if stages else 0
    led = np.stack([stages.get(s, np.zeros((4, n), np.uint64)) for s in range(ns)]) \
        if ns else np.zeros((0, 4, n), np.uint64)
    return results, led, balance


COracle.run_scheme = _co_run_scheme
COracle.sizes = _co_sizes
COracle.hier_centralization = _co_hier_centralization
COracle.profile = _co_profile
COracle.skewness = staticmethod(_co_skewness)

RefOracle.wire_encode = _ref_wire_encode
RefOracle.wire_decode = _ref_wire_decode
RefOracle.write_framed = _ref_write_framed
RefOracle.write_sparse = _ref_write_sparse
RefOracle.sparsify_topk = _ref_sparsify_topk


def c_oracle():
    return COracle()


def ref_oracle():
    """The compiled reference, or None when oracle/_ref was never built."""
    return RefOracle() if os.path.exists(REF_SO) else None
