"""Hierarchical Centralization, the sparsity profile and the scheme selector
 on the GPU.

Theorem 1 of the paper has two optima: Balanced Parallelism (zen.py, the hot
path) and Hierarchical Centralization, recursive doubling that merges at every
stage.  The selector picks between them from a measured sparsity profile.

Reference interface -> here:
  zen::merge_sum                      (tensor.hpp:133-167)  merge_sum (zen_merge_sum: the merge-path
                                                            kernel of k_merge.cu, fold in place)
  zen::density / overlap_ratio        (tensor.hpp:106-130)  density / overlap_ratio
  zen::densification_ratio            (tensor.hpp:178-189)  densification_ratio
  zen::skewness_ratio                 (tensor.hpp:193-213)  skewness_ratio (zen_range_counts)
  zen::SparsityProfile                (tensor.hpp:216-240)  SparsityProfile
  zen::profile_sparsity               (costmodel.hpp:153-195) profile_sparsity
  zen::CostInputs, t_* formulas       (costmodel.hpp:15-135) CostInputs, t_bp, t_hc, ...
  zen::select_scheme                  (costmodel.hpp:139-150) select_scheme
  zen::run_hier_centralization        (schemes.hpp:173-193) run_hier_centralization (one GPU)
  -- one process per GPU --                                  HCSynchronizer (NVLink stores into the
                                                            partners' CUDA-IPC arenas + zen_merge_sum;
                                                            NCCL/gloo only for the handle exchange)

Every fold is zen_merge_sum.  Its merge may put a shared index's two entries
in either order.  fp32 addition of two operands is commutative, so each value
equals the reference's a + b bit for bit.  The same argument makes all n HC
results identical, exactly as in the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .zen import (Error, EmptyTensor, SimNet, SparseTensor, SyncOutcome, UniverseMismatch,
                  WireFormat, _check, _check_device_tensor, _check_inputs, _lib, _ptr, _torch,
                  context)


class NonPowerOfTwo(Error):
    """zen::NonPowerOfTwo (errors.hpp:42-46)."""

    def __init__(self, msg: str = "node count must be a power of two"):
        super().__init__(msg)


class MissingProfileEntry(Error):
    """zen::MissingProfileEntry (errors.hpp)."""


def _pow2(v: int) -> bool:
    return v != 0 and (v & (v - 1)) == 0


# ------------------------------------------------------------- merge_sum ----

def _merge_dev(ai, av, bi, bv, m: int):
    """Device merge_sum of two canonical (int64 idx, f32 val) tensor pairs."""
    torch = _torch()
    dev = ai.device if ai.numel() else bi.device
    cap = ai.numel() + bi.numel()
    oi = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    ov = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    got = C.c_uint64()
    ctx = context(dev.index)
    _check(_lib().zen_merge_sum(ctx.h, _ptr(ai), _ptr(av), ai.numel(), _ptr(bi), _ptr(bv),
                                bi.numel(), m, _ptr(oi), _ptr(ov), cap, C.byref(got)))
    return oi[:got.value], ov[:got.value]


def _to_dev(t: SparseTensor):
    torch = _torch()
    return (torch.from_numpy(t.indices().view(np.int64)).cuda(),
            torch.from_numpy(t.values()).cuda())


def _to_host(m: int, i, v) -> SparseTensor:
    return SparseTensor(m, i.cpu().numpy().view(np.uint64), v.cpu().numpy(), _trusted=True)


def merge_sum(a: SparseTensor, b: SparseTensor) -> SparseTensor:
    """zen::merge_sum (tensor.hpp:133-167): union, shared indices summed."""
    if a.universe() != b.universe():
        raise UniverseMismatch("tensors have different universe sizes")
    i, v = _merge_dev(*_to_dev(a), *_to_dev(b), a.universe())
    return _to_host(a.universe(), i, v)


# --------------------------------------------------------------- metrics ----

def density(t: SparseTensor) -> float:
    """zen::density (tensor.hpp:106-108)."""
    return float(t.nnz()) / float(t.universe())


def overlap_ratio(a: SparseTensor, b: SparseTensor) -> float:
    """zen::overlap_ratio (tensor.hpp:111-130): |I_a ∩ I_b| / min(|I_a|, |I_b|);
    the intersection is na + nb - |union| from the device merge."""
    if a.universe() != b.universe():
        raise UniverseMismatch("tensors have different universe sizes")
    if a.empty() or b.empty():
        raise EmptyTensor("overlap ratio undefined for empty tensors")
    u, _ = _merge_dev(*_to_dev(a), *_to_dev(b), a.universe())
    common = a.nnz() + b.nnz() - u.numel()
    return float(common) / float(min(a.nnz(), b.nnz()))


def _union_count(tensors) -> int:
    i, v = _to_dev(tensors[0])
    for t in tensors[1:]:
        if t.universe() != tensors[0].universe():
            raise UniverseMismatch("tensors have different universe sizes")
        i, v = _merge_dev(i, v, *_to_dev(t), t.universe())
    return i.numel()


def densification_ratio(tensors) -> float:
    """zen::densification_ratio (tensor.hpp:178-189): density(aggregate) / mean density."""
    if not tensors:
        raise Error("densification ratio requires at least one tensor")
    mean_d = 0.0
    for t in tensors:
        if t.empty():
            raise EmptyTensor("densification ratio undefined with an empty tensor")
        mean_d += density(t)
    mean_d /= float(len(tensors))
    return (float(_union_count(tensors)) / float(tensors[0].universe())) / mean_d


def _range_counts_dev(i, m: int, partitions: int) -> np.ndarray:
    out = (C.c_uint64 * partitions)()
    ctx = context(i.device.index)
    _check(_lib().zen_range_counts(ctx.h, _ptr(i), i.numel(), m, partitions, out))
    return np.frombuffer(out, dtype=np.uint64).copy()


def skewness_ratio(t: SparseTensor, partitions: int) -> float:
    """zen::skewness_ratio (tensor.hpp:193-213): max density over ceil(M/n)
    ranges / whole density; range counts from zen_range_counts."""
    if partitions == 0:
        raise Error("skewness ratio requires at least one partition")
    if t.empty():
        raise EmptyTensor("skewness ratio undefined for an empty tensor")
    i, _ = _to_dev(t)
    return _skew_from_counts(_range_counts_dev(i, t.universe(), partitions), t.universe(),
                             partitions, t.nnz())


def _skew_from_counts(counts, m: int, partitions: int, nnz: int) -> float:
    rng = (m + partitions - 1) // partitions
    best = 0.0
    for p in range(partitions):
        lo = p * rng
        if lo >= m:
            break
        hi = min(m, lo + rng)
        best = max(best, float(int(counts[p])) / float(hi - lo))
    return best / (float(nnz) / float(m))


@dataclass
class SparsityProfile:
    """zen::SparsityProfile (tensor.hpp:216-240)."""
    d: float = 0.0
    gamma: dict = field(default_factory=dict)
    skew: dict = field(default_factory=dict)

    def validate(self):
        if not (0.0 < self.d <= 1.0):
            raise Error("profile density must be in (0,1]")
        if self.gamma.get(1) != 1.0:
            raise Error("profile gamma[1] must equal 1")
        prev = 0.0
        for k in sorted(self.gamma):
            g = self.gamma[k]
            if g < prev - 1e-9:
                raise Error("profile gamma must be non-decreasing in k")
            if g > float(k) + 1e-9:
                raise Error("profile gamma[k] must not exceed k")
            if self.d * g > 1.0 + 1e-9:
                raise Error("profile d*gamma[k] must not exceed 1")
            prev = g
        for s in self.skew.values():
            if s < 1.0 - 1e-9:
                raise Error("profile skew must be at least 1")

    def to_json(self) -> dict:  # costmodel.hpp profile_to_json
        return {"d": self.d, "gamma": {str(k): v for k, v in sorted(self.gamma.items())},
                "skew": {str(k): v for k, v in sorted(self.skew.items())}}


def profile_sparsity(rounds) -> SparsityProfile:
    """zen::profile_sparsity (costmodel.hpp:153-195): mean density, the
    densification ladder gamma[k] for power-of-two k, and the skew at n
    partitions, averaged over rounds.  The prefix unions are device merges; the
    double arithmetic follows the reference's order term for term."""
    if not rounds:
        raise Error("profiling requires at least one round")
    n = len(rounds[0])
    if n == 0:
        raise Error("profiling requires at least one tensor per round")
    gamma_sums: dict = {}
    skew_sum = density_sum = 0.0
    density_count = 0
    for rnd in rounds:
        if len(rnd) != n:
            raise Error("profiling rounds must have matching node counts")
        prefix_density_sum = 0.0
        pi = pv = None
        for i, t in enumerate(rnd):
            if t.empty():
                raise EmptyTensor("profiling requires non-empty tensors")
            density_sum += density(t)
            density_count += 1
            ti, tv = _to_dev(t)
            if i == 0:
                pi, pv = ti, tv
            else:
                if t.universe() != rnd[0].universe():
                    raise UniverseMismatch("tensors have different universe sizes")
                pi, pv = _merge_dev(pi, pv, ti, tv, t.universe())
            prefix_density_sum += density(t)
            k = i + 1
            if _pow2(k):
                dp = float(pi.numel()) / float(t.universe())
                gamma_sums[k] = gamma_sums.get(k, 0.0) + dp / (prefix_density_sum / float(k))
            skew_sum += _skew_from_counts(_range_counts_dev(ti, t.universe(), n), t.universe(),
                                          n, t.nnz())
    prof = SparsityProfile()
    prof.d = density_sum / float(density_count)
    for k in sorted(gamma_sums):
        prof.gamma[k] = gamma_sums[k] / float(len(rounds))
    prof.gamma[1] = 1.0
    prof.skew[n] = skew_sum / float(len(rounds) * n)
    return prof


# ------------------------------------------------------------ cost model ----

@dataclass
class CostInputs:
    """zen::CostInputs (costmodel.hpp:15-27); element units (one fp32 = 1)."""
    n: int = 1
    universe: float = 0.0
    d: float = 0.0
    b: float = 1.0
    gamma: dict = field(default_factory=dict)
    skew: float = 1.0
    broadcast_rounds: float = 1.0


def _gamma_at(c: CostInputs, k: int) -> float:
    if k == 1:
        return 1.0
    if k not in c.gamma:
        raise MissingProfileEntry(f"densification ratio for k={k} missing from profile")
    return c.gamma[k]


def t_bp_coefficient(n: int, gamma_n: float) -> float:
    """(n-1)/n * (gamma_n + 1), costmodel.hpp:53-58."""
    if n <= 1:
        return 0.0
    return (float(n) - 1.0) / float(n) * (gamma_n + 1.0)


def t_hc_coefficient(n: int, gamma: dict) -> float:
    """sum over log n stages of gamma at 2^(i-1), costmodel.hpp:62-77."""
    if not _pow2(n):
        raise NonPowerOfTwo("hierarchy requires a power-of-two n")
    s, k = 0.0, 1
    while k < n:
        if k == 1:
            s += 1.0
        else:
            if k not in gamma:
                raise MissingProfileEntry(f"densification ratio for k={k} missing from profile")
            s += gamma[k]
        k *= 2
    return s


def t_bp(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    return t_bp_coefficient(c.n, _gamma_at(c, c.n)) * 2.0 * c.universe * c.d / c.b


def t_hc(c: CostInputs) -> float:
    return t_hc_coefficient(c.n, c.gamma) * 2.0 * c.universe * c.d / c.b


def t_sparse_ps(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    g = _gamma_at(c, c.n)
    return 2.0 * (float(c.n) - 1.0) * (1.0 + g) * c.skew * c.d * c.universe / float(c.n) / c.b


def t_sparse_ps_broadcast(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    g = _gamma_at(c, c.n)
    push = 2.0 * (float(c.n) - 1.0) * c.skew * c.d * c.universe / float(c.n) / c.b
    return push + 2.0 * c.broadcast_rounds * g * c.d * c.universe / c.b


def t_ring_incremental(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    s = sum(_gamma_at(c, k) for k in range(1, c.n))
    return 2.0 * s * c.d * c.universe / float(c.n) / c.b


def t_hierarchy_incremental_lb(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    return 2.0 * (float(c.n) - 1.0) * c.d * c.universe / float(c.n) / c.b


def t_allreduce_dense(c: CostInputs) -> float:
    if c.n <= 1:
        return 0.0
    return 2.0 * (float(c.n) - 1.0) / float(c.n) * c.universe / c.b


BALANCED_PARALLELISM = "balanced-parallelism"
HIERARCHICAL_CENTRALIZATION = "hierarchical-centralization"


def select_scheme(profile: SparsityProfile, n: int) -> str:
    """zen::select_scheme (costmodel.hpp:139-150): the cheaper optimum by
    coefficient; ties go to Balanced Parallelism."""
    if n not in profile.gamma:
        raise MissingProfileEntry(f"densification ratio for k={n} missing from profile")
    bp = t_bp_coefficient(n, profile.gamma[n])
    hc = t_hc_coefficient(n, profile.gamma)
    return BALANCED_PARALLELISM if bp <= hc else HIERARCHICAL_CENTRALIZATION


# ------------------------------------------- Hierarchical Centralization ----

def _sizes_dev(i, v, m: int, fmt: WireFormat):
    """message_sizes (codec.hpp:182-211) of a device tensor: closed forms for
    COO / Bitmap, the device encoder's size pass for TensorBlock."""
    z = i.numel()
    if fmt.kind == "coo":
        return fmt.coo_index_bits * z, 32 * z
    if fmt.kind == "bitmap":
        return m, 32 * z
    if fmt.kind == "hash_bitmap":
        raise Error("hash bitmap requires a hash universe")
    info = L.MessageInfoC()
    f = fmt._c()
    rc = _lib().zen_encode(context(i.device.index).h, C.byref(f), None, 0, _ptr(i), _ptr(v), z, m,
                           None, 0, C.byref(info))
    if rc not in (L.OK, L.E_CAPACITY):
        _check(rc)
    return int(info.index_bits), int(info.value_bits)


class _Sized:
    """An accounting-only EncodedMessage (schemes.hpp:78-88, sized_message)."""

    def __init__(self, index_bits: int, value_bits: int):
        self.index_bits, self.value_bits = index_bits, value_bits

    def payload_bits(self) -> int:
        return self.index_bits + self.value_bits


def run_hier_centralization(inputs, net: SimNet, fmt: WireFormat | None = None) -> SyncOutcome:
    """zen::run_hier_centralization (schemes.hpp:173-193) with all n nodes on
    the current GPU.  Stage log2(bit): every node sends its state to w ^ bit
    (ledger from the exact wire sizes), then states[w] = merge_sum(states[w],
    states[w ^ bit]) on the device."""
    fmt = fmt or WireFormat.coo()
    _check_inputs(inputs, net)
    n = len(inputs)
    if not _pow2(n):
        raise NonPowerOfTwo()
    m = inputs[0].universe()
    states = [_to_dev(t) for t in inputs]
    bit = 1
    while bit < n:
        stage = bit.bit_length() - 1
        for w in range(n):
            net.send(stage, w, w ^ bit, _Sized(*_sizes_dev(*states[w], m, fmt)))
        states = [_merge_dev(*states[w], *states[w ^ bit], m) for w in range(n)]
        bit <<= 1
    results = [_to_host(m, i, v) for i, v in states]
    return SyncOutcome(results, net.finalize(), None)


class HCSynchronizer:
    """Hierarchical Centralization with one process per GPU (zen_hc_*): stage s
    pushes this rank's running aggregate into rank ^ 2^s's CUDA-IPC arena as
    NVLink stores and folds the received one with the merge-path merge_sum.
    Counts stay on the device; sync_dense replays one CUDA graph.  Every rank
    ends with aggregate(inputs), bit for bit."""

    SCHEMES = {"hc": 0, "ring": 1, "agsparse": 2, "omnireduce": 3, "agsparse-ring": 4,
               "agsparse-hierarchy": 5}

    def __init__(self, n: int, universe: int, rank: int, max_nnz: int,
                 fmt: WireFormat | None = None, device: int | None = None,
                 scheme: str = "hc"):
        """scheme: "hc" (run_hier_centralization), "ring"
        (run_ring_centralization), "agsparse" (run_agsparse point-to-point,
        any n), "agsparse-ring" / "agsparse-hierarchy" (run_agsparse with the
        ring / hierarchy forwarding patterns) or "omnireduce"
        (run_omnireduce_like, any n >= 2) -- the same NVLink push + device
        fold machinery."""
        if scheme not in self.SCHEMES:
            raise Error(f"unknown scheme {scheme}")
        if scheme in ("hc", "ring", "agsparse-ring", "agsparse-hierarchy") and not _pow2(n):
            raise NonPowerOfTwo()
        if fmt is not None and fmt.kind not in ("coo", "bitmap"):
            raise Error("rank-mode ledger supports COO and bitmap formats")
        self.n, self.m, self.rank, self.max_nnz = n, universe, rank, max_nnz
        self.scheme = scheme
        self.fmt = fmt or WireFormat.coo()
        self.ctx = context(device)
        self.h = C.c_void_p()
        _check(_lib().zen_hc_create_scheme(self.ctx.h, self.SCHEMES[scheme], n, rank, universe,
                                           max_nnz, C.byref(self.h)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                _lib().zen_hc_destroy(h)
            except Exception:
                pass
            self.h = None

    def ipc_handle(self) -> bytes:
        buf = (C.c_ubyte * L.ZEN_IPC_HANDLE_BYTES)()
        _check(_lib().zen_hc_ipc_handle(self.h, buf))
        return bytes(buf)

    def connect(self, handles: list):
        blob = b"".join(handles)
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(_lib().zen_hc_connect(self.h, buf))

    def connect_process_group(self, group=None):
        """Exchange CUDA IPC handles over torch.distributed (plumbing only)."""
        import torch.distributed as dist
        handles = [None] * self.n
        dist.all_gather_object(handles, self.ipc_handle(), group=group)
        self.connect(handles)

    def sync_dense(self, dense):
        """Asynchronous on the current stream: to_sparse + log2(n) stages."""
        d = dense.contiguous().view(-1)
        _check_device_tensor(d, "float32", self.m, self.ctx.device, "sync_dense")
        self.ctx.bind_stream()
        _check(_lib().zen_hc_sync_dense(self.h, _ptr(d)))

    def sync_sparse(self, idx, val):
        """idx (int64, sorted unique < M) / val (f32) on this rank's GPU."""
        i, v = idx.contiguous(), val.contiguous()
        if i.numel():
            _check_device_tensor(i, "int64", None, self.ctx.device, "sync_sparse indices")
            _check_device_tensor(v, "float32", i.numel(), self.ctx.device, "sync_sparse values")
        self.ctx.bind_stream()
        _check(_lib().zen_hc_sync_sparse(self.h, _ptr(i), _ptr(v), i.numel()))

    def wait(self):
        _check(_lib().zen_hc_wait(self.h))

    def result(self):
        """(int64 indices, f32 values) CUDA tensors of the aggregate, ascending."""
        torch = _torch()
        c = C.c_uint64()
        _check(_lib().zen_hc_result(self.h, None, None, C.byref(c)))
        z = c.value
        dev = torch.device("cuda", self.ctx.device)
        oi = torch.empty(max(z, 1), dtype=torch.int64, device=dev)
        ov = torch.empty(max(z, 1), dtype=torch.float32, device=dev)
        _check(_lib().zen_hc_copy_result(self.h, _ptr(oi), _ptr(ov), max(z, 1), C.byref(c)))
        return oi[:z], ov[:z]

    def sent_counts(self):
        """Entries this rank sent per push, in plan order (OmniReduce: the n-1
        range slices, then its range aggregate to each of the n-1 peers)."""
        ns = _lib().zen_hc_pushes(self.h)
        out = (C.c_uint64 * max(ns, 1))()
        _check(_lib().zen_hc_stage_counts(self.h, out))
        return [int(out[i]) for i in range(ns)]

    def balance(self, group=None):
        """OmniReduce-like only: BalanceDetails(push, pull) of the last sync as
        run_omnireduce_like reports them (schemes.hpp:297-313): push = max over
        workers w and ranges p of n*|slice_wp|/|I_w|, pull = max over owners
        of n*|range aggregate|/union; None when some input is empty.  Collective
        over the ranks (all-gathers the counts)."""
        import torch
        import torch.distributed as dist
        from .zen import BalanceDetails
        if self.scheme != "omnireduce":
            raise Error("balance is reported by the OmniReduce-like scheme")
        n, r = self.n, self.rank
        inp, res = C.c_uint64(), C.c_uint64()
        _check(_lib().zen_hc_counts(self.h, C.byref(inp), C.byref(res)))
        sc = self.sent_counts()
        slices = sc[:n - 1]
        own = inp.value - sum(slices)
        row = slices[:r] + [own] + slices[r:]  # slice p of this rank's input, p = 0..n-1
        agg = sc[n - 1] if n > 1 else own  # |aggregate of this rank's range|
        dev = "cpu" if dist.get_backend(group) == "gloo" else "cuda"
        t = torch.tensor([float(inp.value), float(agg)] + [float(x) for x in row],
                         dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(n)]
        dist.all_gather(allt, t, group=group)
        rows = [x.cpu().numpy() for x in allt]
        if any(x[0] == 0 for x in rows):
            return None
        push = max(float(n) * float(x[2 + p]) / float(x[0]) for x in rows for p in range(n))
        loads = [float(x[1]) for x in rows]
        pull = max(float(n) * ld / float(sum(loads)) for ld in loads)
        return BalanceDetails(push, pull)

    def stage_bits(self):
        """[(index_bits, value_bits)] this rank sent per push, in plan order
        (HC / ring: one per stage; AGsparse: one per peer) -- its row of the
        scheme's SimNet ledger."""
        ns = _lib().zen_hc_pushes(self.h)
        out = (C.c_uint64 * max(ns, 1))()
        _check(_lib().zen_hc_stage_counts(self.h, out))
        res = []
        for s in range(ns):
            z = int(out[s])
            res.append((self.fmt.coo_index_bits * z, 32 * z) if self.fmt.kind == "coo"
                       else (self.m, 32 * z))
        return res



# ----------------------------------------------- the design space (f4) ----
# zen/schemes.hpp:21-41, 119-168, 194-328, 418-470: the baseline schemes the
# paper compares against, with all n nodes on the current GPU.  Each keeps the
# reference's SimNet ledger message for message and its results bit for bit;
# every fold is the device merge_sum.

class UnsupportedCombination(Error):
    """zen::UnsupportedCombination (errors.hpp:48-52)."""


class CommPattern:
    Ring, Hierarchy, PointToPoint = "ring", "hierarchy", "point-to-point"


class Aggregation:
    Incremental, OneShot = "incremental", "one-shot"


class PartitionPattern:
    Centralization, Parallelism = "centralization", "parallelism"


class BalancePattern:
    Balanced, Imbalanced, NotApplicable = "balanced", "imbalanced", "not-applicable"


@dataclass
class SchemeConfig:
    """zen::SchemeConfig (schemes.hpp:27-41)."""
    communication: str = CommPattern.PointToPoint
    aggregation: str = Aggregation.OneShot
    partition: str = PartitionPattern.Centralization
    balance: str = BalancePattern.NotApplicable
    format: WireFormat = field(default_factory=WireFormat.coo)

    def validate(self):
        centralized = self.partition == PartitionPattern.Centralization
        if centralized != (self.balance == BalancePattern.NotApplicable):
            raise UnsupportedCombination(
                "the balance dimension applies exactly when the partition pattern is Parallelism")


def _fold_dev(states, m):
    """aggregate (tensor.hpp:171-176): left fold in the given order."""
    i, v = states[0]
    for t in states[1:]:
        i, v = _merge_dev(i, v, *t, m)
    return i, v


def run_agsparse(inputs, net: SimNet, pattern: str = CommPattern.PointToPoint,
                 fmt: WireFormat | None = None) -> SyncOutcome:
    """zen::run_agsparse (schemes.hpp:119-168): all-gather of whole tensors
    (point-to-point, ring or hierarchy ledger), then one aggregate."""
    fmt = fmt or WireFormat.coo()
    _check_inputs(inputs, net)
    n, m = len(inputs), inputs[0].universe()
    states = [_to_dev(t) for t in inputs]
    sizes = [_Sized(*_sizes_dev(*s, m, fmt)) for s in states]
    if pattern == CommPattern.PointToPoint:
        for w in range(n):
            for to in range(n):
                if to != w:
                    net.send(0, w, to, sizes[w])
    elif pattern == CommPattern.Ring:
        if not _pow2(n):
            raise NonPowerOfTwo()
        for s in range(n - 1):
            for w in range(n):
                net.send(s, w, (w + 1) % n, sizes[(w + n - s) % n])
    elif pattern == CommPattern.Hierarchy:
        if not _pow2(n):
            raise NonPowerOfTwo()
        holdings = [[w] for w in range(n)]
        bit = 1
        while bit < n:
            stage = bit.bit_length() - 1
            prev = [list(h) for h in holdings]
            for w in range(n):
                for origin in prev[w]:
                    net.send(stage, w, w ^ bit, sizes[origin])
                holdings[w] += prev[w ^ bit]
            bit <<= 1
    else:
        raise Error(f"unknown communication pattern {pattern}")
    result = _to_host(m, *_fold_dev(states, m))
    return SyncOutcome([result] * n, net.finalize(), None)


def run_ring_centralization(inputs, net: SimNet, fmt: WireFormat | None = None) -> SyncOutcome:
    """zen::run_ring_centralization (schemes.hpp:194-215): n-1 stages, each node
    forwards its running token to the next; token'[w] = merge_sum(token[w-1],
    input[w])."""
    fmt = fmt or WireFormat.coo()
    _check_inputs(inputs, net)
    n, m = len(inputs), inputs[0].universe()
    if not _pow2(n):
        raise NonPowerOfTwo()
    ins = [_to_dev(t) for t in inputs]
    tokens = list(ins)
    for s in range(n - 1):
        for w in range(n):
            net.send(s, w, (w + 1) % n, _Sized(*_sizes_dev(*tokens[w], m, fmt)))
        tokens = [_merge_dev(*tokens[(w + n - 1) % n], *ins[w], m) for w in range(n)]
    return SyncOutcome([_to_host(m, i, v) for i, v in tokens], net.finalize(), None)


def _range_slices(i, v, m, n):
    """Slices of a sorted device tensor by the contiguous ranges ceil(M/n)
    (schemes.hpp:240-252): zen_range_counts gives the boundaries."""
    counts = _range_counts_dev(i, m, n)
    out, at = [], 0
    for p in range(n):
        c = int(counts[p])
        out.append((i[at:at + c], v[at:at + c]))
        at += c
    return out


def _block_sizes(i, m, n, p, block_size):
    """block_sizes (schemes.hpp:255-270): 64 index bits per non-zero block,
    32 value bits per position of each (the range's last block may be short)."""
    rng = (m + n - 1) // n
    lo = p * rng
    hi = min(m, lo + rng)
    z = i.numel()
    if z == 0:
        return 0, 0
    nb = C.c_uint64()
    _check(_lib().zen_count_blocks(context(i.device.index).h, _ptr(i), z, lo, block_size,
                                   C.byref(nb)))
    blocks = nb.value
    value = 32 * block_size * blocks
    last = (int(i[-1].item()) - lo) // block_size  # only the block holding hi-1 can be short
    if lo + last * block_size + block_size > hi:
        value -= 32 * (lo + last * block_size + block_size - hi)
    return 64 * blocks, value


def run_omnireduce_like(inputs, net: SimNet, block_size: int = 256) -> SyncOutcome:
    """zen::run_omnireduce_like (schemes.hpp:219-328): contiguous ranges, block
    transport to the range owner, per-range aggregate in worker order, block
    broadcast back, exact zeros dropped by the block decode."""
    from .zen import BalanceDetails, PartitionedSparseTensor, imbalance_pull, imbalance_push
    _check_inputs(inputs, net)
    if block_size < 1:
        raise Error("block size must be at least 1")
    torch = _torch()
    n, m = len(inputs), inputs[0].universe()
    slices = [_range_slices(*_to_dev(t), m, n) for t in inputs]
    for w in range(n):
        for p in range(n):
            if p == w or slices[w][p][0].numel() == 0:
                continue
            net.send(0, w, p, _Sized(*_block_sizes(slices[w][p][0], m, n, p, block_size)))
    aggregated = [_fold_dev([slices[w][p] for w in range(n)], m) for p in range(n)]
    for p in range(n):
        if aggregated[p][0].numel() == 0:
            continue
        sz = _Sized(*_block_sizes(aggregated[p][0], m, n, p, block_size))
        for w in range(n):
            if w != p:
                net.send(1, p, w, sz)
    ai = torch.cat([a[0] for a in aggregated])
    av = torch.cat([a[1] for a in aggregated])
    oi = torch.empty(max(ai.numel(), 1), dtype=torch.int64, device=ai.device)
    ov = torch.empty(max(ai.numel(), 1), dtype=torch.float32, device=ai.device)
    got = C.c_uint64()
    _check(_lib().zen_compact_nonzero(context(ai.device.index).h, _ptr(ai), _ptr(av), ai.numel(),
                                      _ptr(oi), _ptr(ov), C.byref(got)))
    result = _to_host(m, oi[:got.value], ov[:got.value])
    balance = None
    if all(not t.empty() for t in inputs):
        parted = [PartitionedSparseTensor([_SizeOnly(s[0].numel()) for s in slices[w]])
                  for w in range(n)]
        loads = [a[0].numel() for a in aggregated]
        balance = BalanceDetails(imbalance_push(parted), imbalance_pull(loads, sum(loads)))
    return SyncOutcome([result] * n, net.finalize(), balance)


class _SizeOnly:
    def __init__(self, z):
        self._z = z

    def nnz(self):
        return self._z


def run_scheme(cfg: SchemeConfig, inputs, net: SimNet, params=None) -> SyncOutcome:
    """zen::run_scheme (schemes.hpp:420-442)."""
    from .zen import run_balanced_parallelism
    cfg.validate()
    if cfg.partition == PartitionPattern.Centralization:
        if cfg.aggregation == Aggregation.OneShot:
            return run_agsparse(inputs, net, cfg.communication, cfg.format)
        if cfg.communication == CommPattern.Hierarchy:
            return run_hier_centralization(inputs, net, cfg.format)
        if cfg.communication == CommPattern.Ring:
            return run_ring_centralization(inputs, net, cfg.format)
        raise UnsupportedCombination("point-to-point incremental centralization is not implemented")
    if cfg.communication == CommPattern.PointToPoint:
        if (cfg.aggregation == Aggregation.OneShot and cfg.balance == BalancePattern.Imbalanced
                and cfg.format.kind == "tensor_block"):
            return run_omnireduce_like(inputs, net, cfg.format.block_size)
        if cfg.aggregation == Aggregation.Incremental and cfg.balance == BalancePattern.Balanced:
            return run_balanced_parallelism(inputs, net, params)
    raise UnsupportedCombination("no implemented scheme matches this configuration")


KNOWN_SCHEME_NAMES = ["agsparse", "sparcml", "ring-centralization", "omnireduce",
                      "balanced-parallelism"]


def scheme_config_from_name(name: str) -> SchemeConfig:
    """zen::scheme_config_from_name (schemes.hpp:445-465)."""
    C_, P_ = PartitionPattern.Centralization, PartitionPattern.Parallelism
    if name == "agsparse":
        return SchemeConfig(CommPattern.PointToPoint, Aggregation.OneShot, C_,
                            BalancePattern.NotApplicable, WireFormat.coo())
    if name == "sparcml":
        return SchemeConfig(CommPattern.Hierarchy, Aggregation.Incremental, C_,
                            BalancePattern.NotApplicable, WireFormat.coo())
    if name == "ring-centralization":
        return SchemeConfig(CommPattern.Ring, Aggregation.Incremental, C_,
                            BalancePattern.NotApplicable, WireFormat.coo())
    if name == "omnireduce":
        return SchemeConfig(CommPattern.PointToPoint, Aggregation.OneShot, P_,
                            BalancePattern.Imbalanced, WireFormat.tensor_block())
    if name == "balanced-parallelism":
        return SchemeConfig(CommPattern.PointToPoint, Aggregation.Incremental, P_,
                            BalancePattern.Balanced, WireFormat.hash_bitmap())
    raise UnsupportedCombination("unknown scheme name: " + name)


# ------------------------------------------------- runtime scheme choice ----

class AutoSynchronizer:
    """select_scheme (costmodel.hpp:139-150) at run time, one process per GPU.

    The first `profile_rounds` syncs run Hierarchical Centralization.  Rank 0's
    HC state before stage s is the union of ranks [0, 2^s), so its stage counts
    are exactly profile_sparsity's prefix unions (costmodel.hpp:151-195) for
    k = 1, 2, 4, .., n; with the ranks' input counts (all-gathered) they give
    the densification ladder gamma[k].  After profiling, the cheaper optimum by
    the cost model serves every later sync: BP or HC.  Both return the same
    aggregate (bit-identical at every rank)."""

    def __init__(self, n: int, universe: int, rank: int, max_nnz: int, params=None,
                 profile_rounds: int = 1, group=None, policy: str = "cost-model"):
        """policy "cost-model": select_scheme on the profiled ladder (the
        reference's rule).  policy "measured": after profiling, time a few
        syncs of each scheme on the device (CUDA events, max over ranks) and
        keep the faster -- the traffic model ignores per-stage latency, which
        on NVLink can decide (at N=4 the model ties BP and HC)."""
        from .zen import BPSynchronizer
        if policy not in ("cost-model", "measured"):
            raise Error(f"unknown policy {policy}")
        self.policy = policy
        self.measured_ms = None
        self.n, self.m, self.rank, self.group = n, universe, rank, group
        self.profile_rounds = profile_rounds
        self.bp = BPSynchronizer(n, universe, max_nnz, params, rank=rank)
        self.hc = HCSynchronizer(n, universe, rank, max_nnz) if _pow2(n) else None
        self.choice = None if self.hc is not None else BALANCED_PARALLELISM
        self.profile = None
        self._gamma_sums, self._d_sum, self._rounds = {}, 0.0, 0
        self._active = self.hc if self.hc is not None else self.bp
        self._last = self._active

    def connect_process_group(self):
        self.bp.connect_process_group(self.group)
        if self.hc is not None:
            self.hc.connect_process_group(self.group)

    def _observe(self):
        import torch
        import torch.distributed as dist
        sent = [vb // 32 for _, vb in self.hc.stage_bits()]  # |U_1|, |U_2|, .., |U_{n/2}|
        i, _ = self.hc.result()
        unions = sent + [i.numel()]
        dev = "cpu" if dist.get_backend(self.group) == "gloo" else "cuda"
        own = torch.tensor([float(sent[0]) if sent else float(i.numel())], device=dev,
                           dtype=torch.float64)
        alln = [torch.zeros_like(own) for _ in range(self.n)]
        dist.all_gather(alln, own, group=self.group)
        d = [float(x[0]) / float(self.m) for x in alln]
        g = torch.tensor([float(u) for u in unions], device=dev, dtype=torch.float64)
        dist.broadcast(g, 0, group=self.group)
        unions = [float(x) for x in g.cpu().numpy()]
        self._d_sum += sum(d) / self.n
        k = 2
        for u in unions[1:]:
            mean_d = sum(d[:k]) / float(k)
            if mean_d > 0:
                self._gamma_sums[k] = self._gamma_sums.get(k, 0.0) + (u / float(self.m)) / mean_d
            k *= 2
        self._rounds += 1
        if self._rounds >= self.profile_rounds:
            gamma = {k: v / self._rounds for k, v in self._gamma_sums.items()}
            gamma[1] = 1.0
            self.profile = SparsityProfile(self._d_sum / self._rounds, gamma, {})
            self.choice = select_scheme(self.profile, self.n) if self.n in gamma \
                else BALANCED_PARALLELISM
            self._active = self.bp if self.choice == BALANCED_PARALLELISM else self.hc

    def _measure(self, dense, reps: int = 5):
        import torch
        import torch.distributed as dist
        stream = torch.cuda.current_stream()
        t = {}
        for name, run in [(BALANCED_PARALLELISM, lambda: self.bp.sync_dense([dense])),
                          (HIERARCHICAL_CENTRALIZATION, lambda: self.hc.sync_dense(dense))]:
            run()
            (self.bp if name == BALANCED_PARALLELISM else self.hc).wait()
            dist.barrier(group=self.group)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                run()
            e1.record(stream)
            (self.bp if name == BALANCED_PARALLELISM else self.hc).wait()
            x = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64,
                             device="cpu" if dist.get_backend(self.group) == "gloo" else "cuda")
            dist.all_reduce(x, op=dist.ReduceOp.MAX, group=self.group)
            t[name] = float(x.item())
        self.measured_ms = t
        self.choice = min(t, key=t.get)
        self._active = self.bp if self.choice == BALANCED_PARALLELISM else self.hc

    def sync_dense(self, dense):
        if self.choice is None:
            self._last = self.hc
            self.hc.sync_dense(dense)
            self.hc.wait()
            self._observe()
            if self.choice is not None and self.policy == "measured":
                self._measure(dense)  # both ran this input: either holds its result
                self._last = self._active
            return
        self._last = self._active
        if self._active is self.bp:
            self.bp.sync_dense([dense])
        else:
            self._active.sync_dense(dense)

    def wait(self):
        self._last.wait()

    def result(self):
        """(int64 indices, f32 values) of the last sync, whichever scheme ran it."""
        return self._last.result()
