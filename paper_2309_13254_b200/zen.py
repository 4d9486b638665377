"""Python mirror of the reference's Balanced-Parallelism operator API.

Names, argument meaning and error behaviour follow the reference header-only
C++ library (/root/reference/proj/include/zen/*.hpp) so parity tests read like
its own tests; every heavy step runs in the sm_100a kernels behind the C-ABI
(include/zen_b200.h).  PyTorch is used only to own device memory and streams.

Reference interface -> here:
  zen::SparseTensor / DenseTensor        (tensor.hpp:19-91)   SparseTensor / DenseTensor
  zen::to_sparse                          (tensor.hpp:94-104)  to_sparse
  zen::HashFamily::make / make_worker     (hashing.hpp:46-82)  HashFamily.make / make_worker
  zen::partition_of                       (hashing.hpp:85-88)  partition_of
  zen::hierarchical_hash / collision_stats(hashing.hpp:251-262) hierarchical_hash / collision_stats
  zen::imbalance_push / imbalance_pull    (hashing.hpp:296-320) imbalance_push / imbalance_pull
  zen::HashUniverseTable / HashUniverse   (codec.hpp:39-72)    HashUniverseTable
  zen::encode / decode (HashBitmap)       (codec.hpp:213-350)  encode / decode
  zen::SimNet / TrafficReport             (simnet.hpp:15-120)  SimNet / TrafficReport
  zen::HashParams / SyncOutcome           (schemes.hpp:42-61)  HashParams / SyncOutcome
  zen::run_balanced_parallelism           (schemes.hpp:341-417) run_balanced_parallelism
  zen::bp_universe_table                  (schemes.hpp:332-335) bp_universe_table
  zen::run_bp_with_retry                  (experiment.hpp:128-140) run_bp_with_retry
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------- errors ----
# zen/errors.hpp:10-84


class Error(RuntimeError):
    """zen::Error"""


class EmptyTensor(Error):
    pass


class UniverseMismatch(Error):
    pass


class SerialOverflow(Error):
    def __init__(self, partition: int, msg: str = ""):
        super().__init__(msg or f"hash partition {partition} exceeded its slot capacity "
                         "(r2 too small for this workload)")
        self._partition = int(partition)

    def partition(self) -> int:
        return self._partition


class IndexOutsideUniverse(Error):
    pass


class MalformedPayload(Error):
    pass


class UnbalancedLedger(Error):
    pass


class SelfSend(Error):
    pass


class CudaError(Error):
    """Device failure.  There is no CPU fallback."""


class CapacityError(Error):
    pass


class PeerTimeout(Error):
    pass


class InfeasibleSpec(Error):
    """zen::InfeasibleSpec (errors.hpp:81-84)."""


def _lib():
    return L.load()


def _check(rc: int):
    if rc == L.OK:
        return
    lib = _lib()
    msg = lib.zen_last_error_message().decode(errors="replace")
    if rc == L.E_SERIAL_OVERFLOW:
        raise SerialOverflow(lib.zen_last_error_partition(), msg)
    if rc == L.E_OUTSIDE:
        raise IndexOutsideUniverse(msg)
    if rc == L.E_MALFORMED:
        raise MalformedPayload(msg)
    if rc == L.E_EMPTY:
        raise EmptyTensor(msg)
    if rc == L.E_MISMATCH:
        raise UniverseMismatch(msg)
    if rc == L.E_CAPACITY:
        raise CapacityError(msg)
    if rc == L.E_TIMEOUT:
        raise PeerTimeout(msg)
    if rc == L.E_INFEASIBLE:
        raise InfeasibleSpec(msg)
    if rc in (L.E_CUDA, L.E_OOM, L.E_PEER):
        raise CudaError(msg)
    raise Error(msg)


# -------------------------------------------------------------- devices ----

_CTX: dict = {}


def _torch():
    import torch
    return torch


class Context:
    """One zen_ctx per CUDA device, bound to torch's current stream."""

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        _check(_lib().zen_ctx_create(device, C.byref(h)))
        self.h = h

    def bind_stream(self):
        torch = _torch()
        s = torch.cuda.current_stream(self.device).cuda_stream
        _check(_lib().zen_ctx_set_stream(self.h, C.c_void_p(s)))
        return self

    def __del__(self):
        try:
            _lib().zen_ctx_destroy(self.h)
        except Exception:
            pass


def context(device: int | None = None) -> Context:
    torch = _torch()
    if device is None:
        device = torch.cuda.current_device()
    if device not in _CTX:
        _CTX[device] = Context(device)
    return _CTX[device].bind_stream()


def _dev(a, dtype):
    torch = _torch()
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=dtype)
    return t.cuda()


def _ptr(t):
    return C.c_void_p(t.data_ptr() if t.numel() else 0)


def _check_device_tensor(t, dtype_name: str, numel: int | None, device: int | None, what: str):
    """Refuse a CUDA tensor the kernels would misread: the C-ABI takes raw
    pointers, so a bf16 gradient (half the bytes), a strided view or a tensor
    on another GPU would otherwise be read out of bounds or silently wrong."""
    torch = _torch()
    want = getattr(torch, dtype_name)
    if not (hasattr(t, "is_cuda") and t.is_cuda):
        raise Error(f"{what}: expected a CUDA tensor")
    if t.dtype != want:
        raise Error(f"{what}: expected dtype {dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise Error(f"{what}: tensor must be contiguous")
    if numel is not None and t.numel() != numel:
        raise Error(f"{what}: expected {numel} elements, got {t.numel()}")
    if device is not None and t.device.index != device:
        raise Error(f"{what}: tensor is on cuda:{t.device.index}, the synchroniser on cuda:{device}")


# ------------------------------------------------------------ data model ----

class DenseTensor:
    """zen::DenseTensor (tensor.hpp:19-27)."""

    def __init__(self, values):
        self.values = np.ascontiguousarray(values, dtype=np.float32)
        if self.values.size == 0:
            raise Error("dense tensor must have at least one element")

    def size(self) -> int:
        return int(self.values.size)


class SparseTensor:
    """zen::SparseTensor (tensor.hpp:32-91): sorted unique u64 indices < M + f32 values."""

    def __init__(self, universe: int = 1, indices=(), values=(), _trusted: bool = False):
        if universe == 0:
            raise Error("sparse tensor universe must be at least 1")
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).ravel())
        val = np.ascontiguousarray(np.asarray(values, dtype=np.float32).ravel())
        if idx.size != val.size:
            raise Error("sparse tensor index/value lengths differ")
        if not _trusted and idx.size:
            if np.any(idx[1:] < idx[:-1]):
                order = np.argsort(idx, kind="stable")
                idx, val = idx[order], val[order]
            if idx[-1] >= universe:
                raise Error("sparse tensor index outside [0, M)")
            if np.any(idx[1:] == idx[:-1]):
                raise Error("duplicate index in sparse tensor")
        self._m = int(universe)
        self._idx = idx
        self._val = val

    @staticmethod
    def from_pairs(universe, pairs):
        pairs = sorted(pairs, key=lambda p: p[0])
        return SparseTensor(universe, [p[0] for p in pairs], [p[1] for p in pairs])

    def universe(self) -> int:
        return self._m

    def nnz(self) -> int:
        return int(self._idx.size)

    def empty(self) -> bool:
        return self._idx.size == 0

    def indices(self) -> np.ndarray:
        return self._idx

    def values(self) -> np.ndarray:
        return self._val

    def __eq__(self, o):  # tensor.hpp:67-69 (exact comparison)
        return (isinstance(o, SparseTensor) and self._m == o._m
                and np.array_equal(self._idx, o._idx)
                and np.array_equal(self._val.view(np.uint32), o._val.view(np.uint32)))

    def __repr__(self):
        return f"SparseTensor(M={self._m}, nnz={self.nnz()})"


@dataclass
class PartitionedSparseTensor:
    """zen::PartitionedSparseTensor (hashing.hpp:92-100)."""
    parts: list

    def total_nnz(self) -> int:
        return sum(p.nnz() for p in self.parts)


@dataclass
class CollisionStats:
    """zen::CollisionStats (hashing.hpp:104-113)."""
    serial_writes: int = 0
    placed_at_depth: list = field(default_factory=list)

    def total(self) -> int:
        return self.serial_writes + sum(self.placed_at_depth)


def _stats(c: L.CollisionStatsC) -> CollisionStats:
    return CollisionStats(int(c.serial_writes), [int(c.placed_at_depth[i]) for i in range(c.k)])


# ----------------------------------------------------------- hash family ----

def derive_seed(master: int, stream: int) -> int:
    return int(_lib().zen_derive_seed(master, stream))


class HashFamily:
    """zen::HashFamily (hashing.hpp:46-82); seeds derived by the library."""

    def __init__(self, c: L.HashFamilyC):
        self._c = c
        self.partition_seed = int(c.partition_seed)
        self.slot_seeds = [int(c.slot_seeds[i]) for i in range(c.k)]
        self.partitions = int(c.partitions)

    @staticmethod
    def make(seed: int, n: int, k: int) -> "HashFamily":
        c = L.HashFamilyC()
        _check(_lib().zen_hash_family_make(seed, n, k, C.byref(c)))
        return HashFamily(c)

    @staticmethod
    def make_worker(shared_seed: int, worker: int, n: int, k: int) -> "HashFamily":
        c = L.HashFamilyC()
        _check(_lib().zen_hash_family_make_worker(shared_seed, worker, n, k, C.byref(c)))
        return HashFamily(c)

    def depth(self) -> int:
        return len(self.slot_seeds)

    def partition_of(self, index):
        return partition_of(index, self.partition_seed, self.partitions)


def partition_of(index, partition_seed: int, n: int):
    """zen::partition_of (hashing.hpp:85-88), computed on the GPU; scalar or array."""
    torch = _torch()
    scalar = np.isscalar(index)
    idx = np.atleast_1d(np.asarray(index, dtype=np.uint64))
    ctx = context()
    d_idx = _dev(idx.view(np.int64), torch.int64)
    out = torch.empty(idx.size, dtype=torch.int32, device=d_idx.device)
    _check(_lib().zen_partition_of(ctx.h, _ptr(d_idx), idx.size, partition_seed, n, _ptr(out)))
    res = out.cpu().numpy().view(np.uint32)
    return int(res[0]) if scalar else res


# ------------------------------------------------------------ operators ----

def to_sparse(dense) -> SparseTensor:
    """zen::to_sparse (tensor.hpp:94-104) on the GPU (warp-ballot compaction)."""
    torch = _torch()
    if isinstance(dense, DenseTensor):
        dense = dense.values
    if isinstance(dense, np.ndarray) or not hasattr(dense, "is_cuda"):
        arr = np.ascontiguousarray(dense, dtype=np.float32).ravel()
        if arr.size == 0:
            raise Error("dense tensor must have at least one element")
        d = _dev(arr, torch.float32)
    else:
        d = dense.contiguous().view(-1)
    m = d.numel()
    ctx = context(d.device.index)
    cap = m
    oi = torch.empty(cap, dtype=torch.int64, device=d.device)
    ov = torch.empty(cap, dtype=torch.float32, device=d.device)
    nnz = C.c_uint64()
    _check(_lib().zen_to_sparse(ctx.h, _ptr(d), m, _ptr(oi), _ptr(ov), cap, C.byref(nnz)))
    c = nnz.value
    return SparseTensor(m, oi[:c].cpu().numpy().view(np.uint64), ov[:c].cpu().numpy(),
                        _trusted=True)


@dataclass
class HashLayout:
    """The detail::HashMemory after a run (hashing.hpp:121-146): slot words
    (0 = empty else index+1), slot values, and per-key placement depth."""
    slots: np.ndarray
    slot_values: np.ndarray
    depth: np.ndarray


def _run_hash(t: SparseTensor, n: int, family: HashFamily, r1: int, r2: int, layout: bool):
    torch = _torch()
    if family.partitions != n:
        raise Error("hash family partition count mismatch")
    ctx = context()
    z = t.nnz()
    d_idx = _dev(t.indices().view(np.int64), torch.int64)
    d_val = _dev(t.values(), torch.float32)
    dev = d_idx.device
    oi = torch.empty(max(z, 1), dtype=torch.int64, device=dev)
    ov = torch.empty(max(z, 1), dtype=torch.float32, device=dev)
    pc = (C.c_uint64 * n)()
    cells = n * (r1 + r2)
    ds = torch.empty(max(cells, 1), dtype=torch.int64, device=dev) if layout else None
    dv = torch.empty(max(cells, 1), dtype=torch.float32, device=dev) if layout else None
    dd = torch.empty(max(z, 1), dtype=torch.int32, device=dev) if layout else None
    st = L.CollisionStatsC()
    _check(_lib().zen_hierarchical_hash(
        ctx.h, _ptr(d_idx), _ptr(d_val), z, t.universe(), C.byref(family._c), r1, r2, _ptr(oi),
        _ptr(ov), pc, _ptr(ds) if layout else None, _ptr(dv) if layout else None,
        _ptr(dd) if layout else None, C.byref(st)))
    counts = [int(pc[p]) for p in range(n)]
    hi = oi.cpu().numpy().view(np.uint64)
    hv = ov.cpu().numpy()
    parts, off = [], 0
    for p in range(n):
        parts.append(SparseTensor(t.universe(), hi[off:off + counts[p]].copy(),
                                  hv[off:off + counts[p]].copy(), _trusted=True))
        off += counts[p]
    lay = None
    if layout:
        lay = HashLayout(ds[:cells].cpu().numpy().view(np.uint64), dv[:cells].cpu().numpy(),
                         dd[:z].cpu().numpy().view(np.uint32))
    return PartitionedSparseTensor(parts), _stats(st), lay


def hierarchical_hash(t: SparseTensor, n: int, family: HashFamily, r1: int, r2: int,
                      lanes: int = 1) -> PartitionedSparseTensor:
    """zen::hierarchical_hash (hashing.hpp:251-255).  `lanes` is accepted for
    signature parity; the device placement is always the lanes=1 layout."""
    if lanes < 1:
        raise Error("lane count must be at least 1")
    return _run_hash(t, n, family, r1, r2, False)[0]


def collision_stats(t: SparseTensor, n: int, family: HashFamily, r1: int, r2: int) -> CollisionStats:
    """zen::collision_stats (hashing.hpp:259-262)."""
    return _run_hash(t, n, family, r1, r2, False)[1]


def hash_memory_layout(t: SparseTensor, n: int, family: HashFamily, r1: int, r2: int):
    """(parts, stats, HashLayout) of one device run -- for bit-exact layout parity."""
    return _run_hash(t, n, family, r1, r2, True)


def imbalance_push(per_worker) -> float:
    """zen::imbalance_push (hashing.hpp:296-308)."""
    if not per_worker:
        raise Error("imbalance requires at least one worker")
    worst = 0.0
    for w in per_worker:
        total = w.total_nnz()
        if total == 0:
            raise EmptyTensor("imbalance undefined for a worker with no gradients")
        n = float(len(w.parts))
        for p in w.parts:
            worst = max(worst, n * p.nnz() / total)
    return worst


def imbalance_pull(server_loads, union_size: int) -> float:
    """zen::imbalance_pull (hashing.hpp:311-320)."""
    if len(server_loads) == 0:
        raise Error("imbalance requires at least one server")
    if union_size == 0:
        raise EmptyTensor("imbalance undefined for an empty union")
    n = float(len(server_loads))
    return max(n * float(x) / float(union_size) for x in server_loads)


# ------------------------------------------------- universe + hash bitmap ----

_WIRE_KINDS = {"coo": 1, "bitmap": 2, "tensor_block": 3, "hash_bitmap": 4}


@dataclass
class WireFormat:
    """zen::WireFormat (codec.hpp:20-35)."""
    kind: str = "coo"
    block_size: int = 256        # TensorBlock only
    coo_index_bits: int = 64     # COO only: 64 (default) or 32

    @staticmethod
    def coo(index_bits: int = 64):
        if index_bits not in (32, 64):
            raise Error("COO index width must be 32 or 64")
        return WireFormat("coo", 256, index_bits)

    @staticmethod
    def bitmap():
        return WireFormat("bitmap")

    @staticmethod
    def tensor_block(block_size: int = 256):
        if block_size < 1:
            raise Error("tensor block size must be at least 1")
        return WireFormat("tensor_block", block_size)

    @staticmethod
    def hash_bitmap():
        return WireFormat("hash_bitmap")

    def _c(self):
        return L.WireFormatC(_WIRE_KINDS[self.kind], self.block_size, self.coo_index_bits)


@dataclass
class HashUniverse:
    server_id: int
    universe_size: int
    _table: "HashUniverseTable"

    @property
    def indices(self) -> np.ndarray:
        return self._table._indices(self.server_id)


@dataclass
class EncodedMessage:
    """zen::EncodedMessage (codec.hpp:101-111)."""
    format: WireFormat
    universe_size: int
    count: int
    index_bits: int
    value_bits: int
    payload: np.ndarray

    def payload_bits(self) -> int:
        return self.index_bits + self.value_bits


class HashUniverseTable:
    """zen::HashUniverseTable (codec.hpp:47-72) built on the GPU as owner bit planes."""

    def __init__(self, universe_size: int, servers: int, partition_seed: int):
        if servers == 0:
            raise Error("hash universe table needs at least one server")
        self.ctx = context()
        h = C.c_void_p()
        _check(_lib().zen_universe_create(self.ctx.h, universe_size, servers, partition_seed,
                                          C.byref(h)))
        self.h = h
        self._m, self._n, self._pseed = universe_size, servers, partition_seed
        self._cache = {}

    def __del__(self):
        try:
            _lib().zen_universe_destroy(self.h)
        except Exception:
            pass

    def universe_size(self):
        return self._m

    def servers(self):
        return self._n

    def partition_seed(self):
        return self._pseed

    def size(self, s: int) -> int:
        return int(_lib().zen_universe_size(self.h, s))

    def universe(self, s: int) -> HashUniverse:
        if s >= self._n:
            raise IndexError("server out of range")
        return HashUniverse(s, self._m, self)

    def _indices(self, s):
        if s not in self._cache:
            torch = _torch()
            sz = self.size(s)
            out = torch.empty(max(sz, 1), dtype=torch.int64, device=f"cuda:{self.ctx.device}")
            _check(_lib().zen_universe_indices(self.h, s, _ptr(out)))
            self._cache[s] = out[:sz].cpu().numpy().view(np.uint64)
        return self._cache[s]


def bp_universe_table(universe_size: int, servers: int, seed: int) -> HashUniverseTable:
    """zen::bp_universe_table (schemes.hpp:332-335)."""
    return HashUniverseTable(universe_size, servers, derive_seed(seed, 0))


def encode(t: SparseTensor, fmt: WireFormat, universe: HashUniverse | None = None) -> EncodedMessage:
    """zen::encode (codec.hpp:213-278) on the GPU, every WireKind; payload bytes
    identical to the reference's."""
    torch = _torch()
    ctx = context()
    z = t.nnz()
    d_idx = _dev(t.indices().view(np.int64), torch.int64)
    d_val = _dev(t.values(), torch.float32)
    uh, s = None, 0
    if fmt.kind == "hash_bitmap":
        if universe is None:
            raise Error("hash bitmap requires a hash universe")
        uh, s = universe._table.h, universe.server_id
    info = L.MessageInfoC()
    f = fmt._c()
    rc = _lib().zen_encode(ctx.h, C.byref(f), uh, s, _ptr(d_idx), _ptr(d_val), z, t.universe(),
                           None, 0, C.byref(info))
    if rc not in (L.OK, L.E_CAPACITY):
        _check(rc)
    out = torch.empty(max(int(info.payload_bytes), 1), dtype=torch.uint8, device=d_idx.device)
    _check(_lib().zen_encode(ctx.h, C.byref(f), uh, s, _ptr(d_idx), _ptr(d_val), z, t.universe(),
                             _ptr(out), int(info.payload_bytes), C.byref(info)))
    return EncodedMessage(fmt, t.universe(), int(info.count), int(info.index_bits),
                          int(info.value_bits), out[:info.payload_bytes].cpu().numpy())


def decode(msg: EncodedMessage, universe: HashUniverse | None = None) -> SparseTensor:
    """zen::decode (codec.hpp:282-347) on the GPU, every WireKind."""
    torch = _torch()
    ctx = context()
    payload = np.ascontiguousarray(msg.payload, dtype=np.uint8)
    d_p = _dev(payload, torch.uint8)
    uh, s = None, 0
    if msg.format.kind == "hash_bitmap":
        if universe is None:
            raise Error("hash bitmap requires the encoding universe")
        uh, s = universe._table.h, universe.server_id
    cap = int(msg.count) * (msg.format.block_size if msg.format.kind == "tensor_block" else 1)
    oi = torch.empty(max(cap, 1), dtype=torch.int64, device=d_p.device)
    ov = torch.empty(max(cap, 1), dtype=torch.float32, device=d_p.device)
    info = L.MessageInfoC(msg.universe_size, msg.count, msg.index_bits, msg.value_bits,
                          payload.size)
    got = C.c_uint64()
    _check(_lib().zen_decode(ctx.h, C.byref(msg.format._c()), uh, s, C.byref(info), _ptr(d_p),
                             _ptr(oi), _ptr(ov), cap, C.byref(got)))
    z = got.value
    return SparseTensor(msg.universe_size, oi[:z].cpu().numpy().view(np.uint64),
                        ov[:z].cpu().numpy(), _trusted=True)


@dataclass
class WorkloadSpec:
    """zen::WorkloadSpec (workload.hpp:22-51)."""
    universe: int = 0
    nodes: int = 1
    density: float = 0.0
    omega: float = 0.0
    hot_fraction: float = 0.125
    hot_mass: float = 0.125
    seed: int = 0

    def nnz_per_node(self) -> int:
        return int(math.ceil(self.density * self.universe))

    def c(self) -> L.WorkloadSpecC:
        return L.WorkloadSpecC(self.universe, self.nodes, self.density, self.omega,
                               self.hot_fraction, self.hot_mass, self.seed)


def generate_device(spec: WorkloadSpec, node: int, device: int | None = None):
    """Node `node`'s tensor of zen::generate drawn on the GPU (zen_generate):
    (int64 indices, fp32 values) CUDA tensors, ascending."""
    torch = _torch()
    ctx = context(device)
    z = max(spec.nnz_per_node(), 1)
    dev = f"cuda:{ctx.device}"
    oi = torch.empty(z, dtype=torch.int64, device=dev)
    ov = torch.empty(z, dtype=torch.float32, device=dev)
    got = C.c_uint64()
    sc = spec.c()
    _check(_lib().zen_generate(ctx.h, C.byref(sc), node, _ptr(oi), _ptr(ov), z, C.byref(got)))
    return oi[:got.value], ov[:got.value]


def generate(spec: WorkloadSpec) -> list:
    """zen::generate (workload.hpp:119-154) on the device: spec.nodes tensors,
    the shared core + two-tier draws without replacement, integer values.
    Same spec as the reference, not the same bits (counter-based hashes
    instead of std::mt19937_64); deterministic for a seed."""
    out = []
    for node in range(spec.nodes):
        oi, ov = generate_device(spec, node)
        out.append(SparseTensor(spec.universe, oi.cpu().numpy().view(np.uint64), ov.cpu().numpy(),
                                _trusted=True))
    return out


def sparsify_topk(dense, fraction: float) -> SparseTensor:
    """zen::sparsify_topk (workload.hpp:157-178) on the GPU: the
    ceil(fraction*M) largest |v| (ties to the lower index), zeros dropped.
    `dense`: DenseTensor, numpy array or CUDA tensor (fp32)."""
    torch = _torch()
    if isinstance(dense, DenseTensor):
        dense = dense.values
    d = dense if (hasattr(dense, "is_cuda") and dense.is_cuda) else _dev(np.asarray(dense,
                                                                               np.float32),
                                                                    torch.float32)
    d = d.reshape(-1).contiguous()
    _check_device_tensor(d, "float32", None, None, "sparsify_topk")
    ctx = context(d.device.index)
    m = d.numel()
    keep = min(m, math.ceil(fraction * m)) if 0 < fraction <= 1 else 1
    oi = torch.empty(max(keep, 1), dtype=torch.int64, device=d.device)
    ov = torch.empty(max(keep, 1), dtype=torch.float32, device=d.device)
    got = C.c_uint64()
    _check(_lib().zen_sparsify_topk(ctx.h, _ptr(d), m, float(fraction), _ptr(oi), _ptr(ov), keep,
                                    C.byref(got)))
    z = got.value
    return SparseTensor(m, oi[:z].cpu().numpy().view(np.uint64), ov[:z].cpu().numpy(),
                        _trusted=True)


def message_sizes(t: SparseTensor, fmt: WireFormat, universe: HashUniverse | None = None):
    """zen::message_sizes (codec.hpp:182-211): (index_bits, value_bits)."""
    m = encode(t, fmt, universe)
    return m.index_bits, m.value_bits


def write_framed(stream, msg: EncodedMessage):
    """zen::write_framed (codec.hpp:356-366)."""
    if msg.payload is None or (len(msg.payload) == 0 and msg.payload_bits() != 0):
        raise Error("cannot frame a message without payload")
    hdr = np.zeros(L.FRAME_HEADER_BYTES, np.uint8)
    info = L.MessageInfoC(msg.universe_size, msg.count, msg.index_bits, msg.value_bits,
                          len(msg.payload))
    _check(_lib().zen_frame_header(C.byref(msg.format._c()), C.byref(info),
                                   hdr.ctypes.data_as(C.c_void_p)))
    stream.write(hdr.tobytes())
    stream.write(np.ascontiguousarray(msg.payload, np.uint8).tobytes())


def read_framed(stream) -> EncodedMessage:
    """zen::read_framed (codec.hpp:368-410)."""
    hdr = np.frombuffer(stream.read(L.FRAME_HEADER_BYTES), np.uint8).copy()
    if hdr.size < L.FRAME_HEADER_BYTES:
        raise MalformedPayload("unexpected end of stream")
    f, info = L.WireFormatC(), L.MessageInfoC()
    # header only (no payload bytes are read by the parse): available = max
    _check(_lib().zen_frame_parse(hdr.ctypes.data_as(C.c_void_p), 2**64 - 1, C.byref(f),
                                  C.byref(info)))
    payload = np.frombuffer(stream.read(int(info.payload_bytes)), np.uint8).copy()
    if payload.size < info.payload_bytes:
        raise MalformedPayload("frame payload truncated")
    kind = {v: k for k, v in _WIRE_KINDS.items()}[f.kind]
    return EncodedMessage(WireFormat(kind, f.block_size, f.coo_index_bits), info.universe_size,
                          info.count, info.index_bits, info.value_bits, payload)


# .zspt (zen/tensor.hpp:239-303): "ZSPT", u32 version 1, u64 M, u64 count, u64
# indices, f32 values -- host byte layout
_SPARSE_MAGIC = b"ZSPT"


def write_sparse(stream, t: SparseTensor):
    """zen::write_sparse (tensor.hpp:257-264)."""
    stream.write(_SPARSE_MAGIC)
    stream.write(np.array([1], "<u4").tobytes())
    stream.write(np.array([t.universe(), t.nnz()], "<u8").tobytes())
    stream.write(t.indices().astype("<u8").tobytes())
    stream.write(t.values().astype("<f4").tobytes())


def read_sparse(stream) -> SparseTensor:
    """zen::read_sparse (tensor.hpp:266-279)."""
    if stream.read(4) != _SPARSE_MAGIC:
        raise MalformedPayload("bad sparse tensor magic")
    raw = stream.read(4)
    if len(raw) < 4:
        raise MalformedPayload("unexpected end of stream")
    if np.frombuffer(raw, "<u4")[0] != 1:
        raise MalformedPayload("unsupported sparse tensor version")
    raw = stream.read(16)
    if len(raw) < 16:
        raise MalformedPayload("unexpected end of stream")
    m, c = (int(x) for x in np.frombuffer(raw, "<u8"))
    ib, vb = stream.read(8 * c), stream.read(4 * c)
    if len(ib) < 8 * c or len(vb) < 4 * c:
        raise MalformedPayload("unexpected end of stream")
    return SparseTensor(m, np.frombuffer(ib, "<u8").astype(np.uint64),
                        np.frombuffer(vb, "<f4").astype(np.float32))


def write_sparse_file(path: str, t: SparseTensor):
    with open(path, "wb") as f:
        write_sparse(f, t)


def read_sparse_file(path: str) -> SparseTensor:
    with open(path, "rb") as f:
        return read_sparse(f)


# ------------------------------------------------------------- transport ----

@dataclass
class StageRecord:
    """zen::StageRecord (simnet.hpp:15-25)."""
    sent_bits: list
    recv_bits: list
    recv_index_bits: list
    recv_value_bits: list
    stage_time: float = 0.0


@dataclass
class TrafficReport:
    """zen::TrafficReport (simnet.hpp:27-56)."""
    nodes: int = 0
    bandwidth: float = 0.0
    stages: list = field(default_factory=list)
    total_sent_bits: int = 0
    total_recv_bits: int = 0
    total_index_bits: int = 0
    total_value_bits: int = 0
    simulated_time: float = 0.0

    def to_json(self) -> dict:
        return {"n": self.nodes, "b": self.bandwidth,
                "stages": [{"time": s.stage_time, "sent_bits": s.sent_bits,
                            "recv_bits": s.recv_bits, "recv_index_bits": s.recv_index_bits,
                            "recv_value_bits": s.recv_value_bits} for s in self.stages],
                "totals": {"sent_bits": self.total_sent_bits, "recv_bits": self.total_recv_bits,
                           "index_bits": self.total_index_bits,
                           "value_bits": self.total_value_bits},
                "simulated_time": self.simulated_time}


class SimNet:
    """zen::SimNet (simnet.hpp:58-120).  On B200 the bytes really move over
    NVLink; this object keeps the reference's deterministic bit ledger."""

    def __init__(self, nodes: int, bandwidth: float, per_message_latency: float = 0.0):
        if nodes == 0:
            raise Error("network needs at least one node")
        if bandwidth <= 0.0:
            raise Error("bandwidth must be positive")
        self._n, self._b, self._lat = nodes, bandwidth, per_message_latency
        self._stages = []
        self._lat_charges = 0.0
        self._final = False

    def nodes(self):
        return self._n

    def bandwidth(self):
        return self._b

    def send(self, stage, frm, to, msg: EncodedMessage):
        if self._final:
            raise Error("cannot send after finalize")
        if frm == to:
            raise SelfSend("a node cannot send a message to itself")
        if frm >= self._n or to >= self._n:
            raise Error("node id out of range")
        if self._stages and stage + 1 < len(self._stages):
            raise Error("stage numbers must be non-decreasing")
        while len(self._stages) <= stage:
            z = [0] * self._n
            self._stages.append(StageRecord(list(z), list(z), list(z), list(z)))
        r = self._stages[stage]
        bits = msg.payload_bits()
        r.sent_bits[frm] += bits
        r.recv_bits[to] += bits
        r.recv_index_bits[to] += msg.index_bits
        r.recv_value_bits[to] += msg.value_bits
        self._lat_charges += self._lat

    def _record_ledger(self, ledger: np.ndarray, messages: int):
        """Install a [2][4][n] ledger measured by the device run."""
        if self._final:
            raise Error("cannot send after finalize")
        for st in range(ledger.shape[0]):
            while len(self._stages) <= st:
                z = [0] * self._n
                self._stages.append(StageRecord(list(z), list(z), list(z), list(z)))
            r = self._stages[st]
            for node in range(self._n):
                r.sent_bits[node] += int(ledger[st, 0, node])
                r.recv_bits[node] += int(ledger[st, 1, node])
                r.recv_index_bits[node] += int(ledger[st, 2, node])
                r.recv_value_bits[node] += int(ledger[st, 3, node])
        self._lat_charges += self._lat * messages

    def finalize(self) -> TrafficReport:
        if self._final:
            raise Error("network already finalized")
        self._final = True
        rep = TrafficReport(nodes=self._n, bandwidth=self._b, stages=self._stages)
        for s in rep.stages:
            sent, recv = sum(s.sent_bits), sum(s.recv_bits)
            rep.total_index_bits += sum(s.recv_index_bits)
            rep.total_value_bits += sum(s.recv_value_bits)
            if sent != recv:
                raise UnbalancedLedger("sent and received byte totals disagree")
            s.stage_time = float(max(s.recv_bits)) / self._b
            rep.total_sent_bits += sent
            rep.total_recv_bits += recv
            rep.simulated_time += s.stage_time
        rep.simulated_time += self._lat_charges
        return rep


# --------------------------------------------------- Balanced Parallelism ----

@dataclass
class HashParams:
    """zen::HashParams (schemes.hpp:55-61)."""
    rehash_depth: int = 3
    r1_multiplier: float = 2.0
    r2_ratio: float = 0.1
    lanes: int = 1
    seed: int = 1

    def c(self) -> L.HashParamsC:
        return L.HashParamsC(self.rehash_depth, self.r1_multiplier, self.r2_ratio, self.lanes,
                             self.seed)


@dataclass
class BalanceDetails:
    push_imbalance: float = 1.0
    pull_imbalance: float = 1.0


@dataclass
class SyncOutcome:
    """zen::SyncOutcome (schemes.hpp:49-53)."""
    results: list
    traffic: TrafficReport
    balance: BalanceDetails | None = None


def exchange_ipc_handles(handle: bytes, n: int, group=None) -> list:
    """All-gather one receive-arena handle per rank over torch.distributed
    (gloo or NCCL: plumbing only, the data path never uses it), rank-major,
    checked against the job size the synchroniser was created with."""
    import torch.distributed as dist
    if len(handle) != L.ZEN_IPC_HANDLE_BYTES:
        raise Error(f"IPC handle must be {L.ZEN_IPC_HANDLE_BYTES} bytes, got {len(handle)}")
    world = dist.get_world_size(group)
    if world != n:
        raise Error(f"process group has {world} ranks, the synchroniser {n} workers")
    handles = [None] * n
    dist.all_gather_object(handles, bytes(handle), group=group)
    return handles


class BPSynchronizer:
    """A device-resident BP synchroniser (zen_bp).  rank=None hosts all n
    workers on this GPU (exchange = local stores); rank=r is worker+server r of
    an n-process job whose push/pull are NVLink stores into peer inboxes."""

    def __init__(self, n: int, universe: int, max_nnz: int, params: HashParams | None = None,
                 rank: int | None = None, device: int | None = None):
        self.params = params or HashParams()
        self.n, self.universe, self.max_nnz = n, universe, max_nnz
        self.rank = rank
        self.ctx = context(device)
        h = C.c_void_p()
        pc = self.params.c()
        _check(_lib().zen_bp_create(self.ctx.h, n, L.ZEN_BP_LOCAL if rank is None else rank,
                                    universe, max_nnz, C.byref(pc), C.byref(h)))
        self.h = h
        self.local_workers = n if rank is None else 1

    def __del__(self):
        try:
            _lib().zen_bp_destroy(self.h)
        except Exception:
            pass

    def set_params(self, params: HashParams):
        pc = params.c()
        _check(_lib().zen_bp_set_params(self.h, C.byref(pc)))
        self.params = params

    # -- rank mode plumbing ---------------------------------------------------
    def ipc_handle(self) -> bytes:
        buf = (C.c_ubyte * L.ZEN_IPC_HANDLE_BYTES)()
        _check(_lib().zen_bp_ipc_handle(self.h, buf))
        return bytes(buf)

    def connect(self, handles: list):
        blob = b"".join(handles)
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(_lib().zen_bp_connect(self.h, buf))

    def connect_process_group(self, group=None):
        """Exchange CUDA IPC handles over torch.distributed (plumbing only)."""
        self.connect(exchange_ipc_handles(self.ipc_handle(), self.n, group))

    # -- synchronisation ------------------------------------------------------
    def sync_dense(self, dense):
        """dense: list of local_workers CUDA fp32 tensors of M elements."""
        if len(dense) != self.local_workers:
            raise Error(f"expected {self.local_workers} dense gradients, got {len(dense)}")
        for d in dense:
            _check_device_tensor(d, "float32", self.universe, self.ctx.device, "sync_dense")
        self.ctx.bind_stream()
        ptrs = (C.c_void_p * self.local_workers)(*[d.data_ptr() for d in dense])
        self._keep = dense
        _check(_lib().zen_bp_sync_dense(self.h, ptrs))

    def sync_sparse(self, idx_list, val_list):
        """idx_list/val_list: CUDA int64/fp32 tensors (sorted unique indices)."""
        k = self.local_workers
        if len(idx_list) != k or len(val_list) != k:
            raise Error(f"expected {k} index and value tensors")
        for i, v in zip(idx_list, val_list):
            if i.numel():
                _check_device_tensor(i, "int64", None, self.ctx.device, "sync_sparse indices")
                _check_device_tensor(v, "float32", i.numel(), self.ctx.device, "sync_sparse values")
        self.ctx.bind_stream()
        ip = (C.c_void_p * k)(*[t.data_ptr() if t.numel() else 0 for t in idx_list])
        vp = (C.c_void_p * k)(*[t.data_ptr() if t.numel() else 0 for t in val_list])
        nz = (C.c_uint64 * k)(*[t.numel() for t in idx_list])
        self._keep = (idx_list, val_list)
        _check(_lib().zen_bp_sync_sparse(self.h, ip, vp, nz))

    def apply_sgd(self, param, lr: float):
        """The step after the sync: param.view(-1)[idx] -= lr * val with the
        synced gradient, on the device (zen_axpy_sparse)."""
        self.wait()
        pi, pv, cnt = C.c_void_p(), C.c_void_p(), C.c_uint64()
        _check(_lib().zen_bp_result(self.h, C.byref(pi), C.byref(pv), C.byref(cnt)))
        flat = param.view(-1)
        self.ctx.bind_stream()
        _check(_lib().zen_axpy_sparse(self.ctx.h, _ptr(flat), flat.numel(), pi, pv, cnt.value,
                                      -float(lr)))

    def wait(self):
        _check(_lib().zen_bp_wait(self.h))

    def result_count(self) -> int:
        c = C.c_uint64()
        _check(_lib().zen_bp_result(self.h, None, None, C.byref(c)))
        return c.value

    def result(self):
        """(int64 CUDA tensor of indices, fp32 CUDA tensor of values), ascending."""
        torch = _torch()
        n = self.result_count()
        dev = f"cuda:{self.ctx.device}"
        oi = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        ov = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        c = C.c_uint64()
        _check(_lib().zen_bp_copy_result(self.h, _ptr(oi), _ptr(ov), max(n, 1), C.byref(c)))
        return oi[:n], ov[:n]

    def result_tensor(self) -> SparseTensor:
        oi, ov = self.result()
        return SparseTensor(self.universe, oi.cpu().numpy().view(np.uint64), ov.cpu().numpy(),
                            _trusted=True)

    def ledger(self):
        n = self.n
        led = np.zeros(8 * n, np.uint64)
        counts = np.zeros(n * n, np.uint64)
        agg = np.zeros(n, np.uint64)
        _check(_lib().zen_bp_traffic(self.h, led.ctypes.data, counts.ctypes.data,
                                     agg.ctypes.data))
        return led.reshape(2, 4, n), counts.reshape(n, n), agg

    def balance(self) -> BalanceDetails | None:
        a, b, v = C.c_double(), C.c_double(), C.c_int()
        _check(_lib().zen_bp_balance(self.h, C.byref(a), C.byref(b), C.byref(v)))
        return BalanceDetails(a.value, b.value) if v.value else None

    def collision_stats(self, worker: int) -> CollisionStats:
        st = L.CollisionStatsC()
        _check(_lib().zen_bp_collision_stats(self.h, worker, C.byref(st)))
        return _stats(st)

    def enable_timing(self, on=True):
        _check(_lib().zen_bp_enable_timing(self.h, int(on)))

    def stage_times(self):
        ms = np.zeros(L.ZEN_STAGES, np.float64)
        k = C.c_uint64()
        _check(_lib().zen_bp_stage_times(self.h, ms.ctypes.data, C.byref(k)))
        return ms, k.value

    def debug_part(self, what: int, server: int, worker: int, cap: int):
        """Diagnostics: (u32 idx, f32 val) of a local worker's keys (what=0) or
        of the part `worker` pushed to local `server` (what=1)."""
        oi = np.empty(max(cap, 1), np.uint32)
        ov = np.empty(max(cap, 1), np.float32)
        c = C.c_uint64()
        _check(_lib().zen_bp_debug_part(self.h, what, server, worker, oi.ctypes.data,
                                        ov.ctypes.data, cap, C.byref(c)))
        k = min(c.value, cap)
        return oi[:k], ov[:k], c.value

    def use_graph(self, on=True):
        """Replay dense syncs from a captured CUDA graph (needs a non-default stream)."""
        _check(_lib().zen_bp_use_graph(self.h, int(on)))

    def time_extract(self, dense, iters: int = 50) -> float:
        """Average ms of the extraction kernel alone (back-to-back launches on
        the current stream) -- the roofline kernel's live launch duration."""
        self.ctx.bind_stream()
        ms = C.c_double()
        _check(_lib().zen_bp_time_extract(self.h, C.c_void_p(dense.data_ptr()), iters,
                                           C.byref(ms)))
        return ms.value

    def kernels_per_sync(self) -> int:
        return int(_lib().zen_bp_kernels_per_sync(self.h))

    def sync_host(self, host_dense, out_idx: np.ndarray, out_val: np.ndarray) -> int:
        """End to end from HOST buffers (pinned recommended): H2D of the dense
        gradients, the sync, D2H of the result into out_idx (u64) / out_val
        (f32).  Returns the result count."""
        k = self.local_workers
        arrs = [np.ascontiguousarray(h, dtype=np.float32) for h in host_dense]
        dp = (C.c_void_p * k)(*[a.ctypes.data for a in arrs])
        assert out_idx.dtype == np.uint64 and out_val.dtype == np.float32
        c = C.c_uint64()
        _check(_lib().zen_bp_sync_host(self.h, dp, out_idx.ctypes.data, out_val.ctypes.data,
                                       min(out_idx.size, out_val.size), C.byref(c)))
        return c.value


_SYNC_CACHE: dict = {}


def _check_inputs(inputs, net):  # schemes.hpp:65-70
    if len(inputs) < 2:
        raise Error("synchronization needs at least two nodes")
    if len(inputs) != net.nodes():
        raise Error("input count must match the network size")
    for t in inputs:
        if t.universe() != inputs[0].universe():
            raise UniverseMismatch("tensors have different universe sizes")


def run_balanced_parallelism(inputs, net: SimNet, params: HashParams | None = None,
                             table: HashUniverseTable | None = None) -> SyncOutcome:
    """zen::run_balanced_parallelism (schemes.hpp:341-417) on the GPU.

    All n workers/servers run on the current device (zen_bp local mode): h0
    partitioning + priority-claim placement, stable multi-split push, fused
    aggregate + HashBitmap encode, HashBitmap decode.  The reference's SimNet
    ledger is filled with the traffic the run produced."""
    params = params or HashParams()
    _check_inputs(inputs, net)
    n = len(inputs)
    m = inputs[0].universe()
    pseed = derive_seed(params.seed, 0)
    if table is not None and (table.universe_size() != m or table.servers() != n
                              or table.partition_seed() != pseed):
        raise Error("hash universe table does not match this run")
    torch = _torch()
    cap = max(max(t.nnz() for t in inputs), 1)
    key = (torch.cuda.current_device(), n, m, params.seed)
    bp = _SYNC_CACHE.get(key)
    if bp is None or bp.max_nnz < cap:
        bp = BPSynchronizer(n, m, max(cap, bp.max_nnz if bp else 0), params)
        _SYNC_CACHE.clear()
        _SYNC_CACHE[key] = bp
    bp.set_params(params)
    idx = [_dev(t.indices().view(np.int64), torch.int64) for t in inputs]
    val = [_dev(t.values(), torch.float32) for t in inputs]
    bp.sync_sparse(idx, val)
    bp.wait()
    result = bp.result_tensor()
    ledger, counts, agg = bp.ledger()
    msgs = int(np.count_nonzero(counts) - np.count_nonzero(np.diag(counts))) + n * (n - 1)
    net._record_ledger(ledger, msgs)
    bal = bp.balance()
    return SyncOutcome([result] * n, net.finalize(), bal)


def run_bp_with_retry(inputs, bandwidth: float, params: HashParams,
                      table: HashUniverseTable | None = None, max_retries: int = 4) -> SyncOutcome:
    """zen::run_bp_with_retry (experiment.hpp:128-140): on SerialOverflow the
    run is retried with a doubled serial region."""
    params = HashParams(**params.__dict__)
    attempt = 0
    while True:
        net = SimNet(len(inputs), bandwidth)
        try:
            return run_balanced_parallelism(inputs, net, params, table)
        except SerialOverflow:
            if attempt >= max_retries:
                raise
            params.r2_ratio *= 2.0
            attempt += 1


def aggregate(tensors) -> SparseTensor:
    """zen::aggregate (tensor.hpp:171-176) -- host helper for tests/compat."""
    if not tensors:
        raise Error("aggregate requires at least one tensor")
    acc_i, acc_v = tensors[0].indices(), tensors[0].values()
    for t in tensors[1:]:
        if t.universe() != tensors[0].universe():
            raise UniverseMismatch("tensors have different universe sizes")
        ui = np.union1d(acc_i, t.indices())
        out = np.zeros(ui.size, np.float32)
        ia = np.searchsorted(ui, acc_i)
        ib = np.searchsorted(ui, t.indices())
        out[ia] = acc_v
        present = np.zeros(ui.size, bool)
        present[ia] = True
        both = present[ib]
        out[ib[both]] = out[ib[both]] + t.values()[both]
        out[ib[~both]] = t.values()[~both]
        acc_i, acc_v = ui.astype(np.uint64), out
    return SparseTensor(tensors[0].universe(), acc_i, acc_v, _trusted=True)
