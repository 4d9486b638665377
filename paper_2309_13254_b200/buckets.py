"""Mixed sparse / top-k / dense gradient buckets around the BP sync (SURVEY.md
§8f row f2: the step either side of the path).

The paper's end-to-end setting syncs a model's gradients
in buckets of three kinds:

  * ``"sparse"``: an embedding gradient that is sparse by construction (rows
    of the batch's tokens) -- the BP dense sync straight from the fp32
    gradient (extract -> hash -> push -> aggregate -> pull -> decode);
  * ``"topk"``: a dense layer's gradient sparsified on the device first
    (``zen_sparsify_topk``: the ceil(fraction*M) largest |v|, ties to the lower
    index, zeros dropped -- zen::sparsify_topk, zen/workload.hpp:158-178), then
    synced through BP's sparse input;
  * ``"dense"``: everything else, a plain NCCL all-reduce (sum) -- the
    reference's normalisation baseline ``t_allreduce_dense`` /
    ``allreduce_dense_time_bits`` (zen/costmodel.hpp:123-127,
    zen/experiment.hpp:161-169) made real.

After the sync, ``apply_sgd`` applies ``param -= lr * grad`` with the synced
sparse gradients on the device (``zen_axpy_sparse``) and the all-reduced (summed) dense
ones with torch.

One process per GPU (rank mode, CUDA-IPC peers) or one process with n = 1.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import _lib as L
from .schemes import CostInputs, t_allreduce_dense
from .zen import BPSynchronizer, Error, HashParams, _check, _check_device_tensor, _ptr, _torch, \
    context


def allreduce_dense_time_bits(n: int, universe: int, bandwidth: float) -> float:
    """zen::allreduce_dense_time_bits (experiment.hpp:161-169): the dense ring
    all-reduce time in the simulator's bit units (element bandwidth = b/32)."""
    return t_allreduce_dense(CostInputs(n=n, universe=float(universe), d=1.0,
                                        b=bandwidth / 32.0, gamma={1: 1.0}))


@dataclass
class Bucket:
    """kind: "sparse" | "topk" | "dense"; numel: fp32 elements; fraction: top-k."""
    kind: str
    numel: int
    fraction: float = 0.01
    max_nnz: int | None = None  # sparse buckets: capacity (default: numel // 8)


class MixedBucketSync:
    """Synchronise a list of gradient buckets of mixed kinds each step.

    ``step(grads)`` takes one contiguous fp32 CUDA tensor per bucket (this
    rank's gradient) and leaves, per bucket, the synced gradient: for sparse
    and top-k buckets the global sparse sum (``result(i)`` -> int64 indices,
    fp32 values, identical on every rank), for dense buckets the all-reduced
    sum in place.  Everything is asynchronous on the current stream except
    the capacity bookkeeping of ``result``.
    """

    def __init__(self, buckets, n: int = 1, rank: int | None = None,
                 params: HashParams | None = None, group=None):
        self.buckets = [b if isinstance(b, Bucket) else Bucket(*b) for b in buckets]
        self.n, self.rank, self.group = n, rank, group
        if n > 1 and rank is None:
            raise Error("rank mode needs this process's rank")
        self.ctx = context()
        self._bp, self._topk = [], []
        torch = _torch()
        for b in self.buckets:
            if b.kind not in ("sparse", "topk", "dense"):
                raise Error(f"unknown bucket kind {b.kind!r}")
            if b.kind == "dense":
                self._bp.append(None)
                self._topk.append(None)
                continue
            if b.kind == "topk":
                if not 0.0 < b.fraction <= 1.0:
                    raise Error("top-k fraction must be in (0,1]")
                keep = min(b.numel, math.ceil(b.fraction * b.numel))
                cap = keep
                dev = f"cuda:{self.ctx.device}"
                self._topk.append((keep, torch.empty(max(keep, 1), dtype=torch.int64, device=dev),
                                   torch.empty(max(keep, 1), dtype=torch.float32, device=dev)))
            else:
                cap = b.max_nnz or max(1, b.numel // 8)
                self._topk.append(None)
            bp = BPSynchronizer(n, b.numel, max_nnz=cap + 4096, params=params,
                                rank=None if n == 1 else rank)
            if n > 1:
                bp.connect_process_group(group)
            self._bp.append(bp)

    def step(self, grads):
        if len(grads) != len(self.buckets):
            raise Error(f"expected {len(self.buckets)} gradients, got {len(grads)}")
        lib = L.load()
        for b, g, bp, tk in zip(self.buckets, grads, self._bp, self._topk):
            _check_device_tensor(g, "float32", b.numel, self.ctx.device, f"{b.kind} bucket")
            if b.kind == "sparse":
                bp.sync_dense([g])
            elif b.kind == "topk":
                keep, ti, tv = tk
                got = C.c_uint64()
                self.ctx.bind_stream()
                _check(lib.zen_sparsify_topk(self.ctx.h, _ptr(g), b.numel, float(b.fraction),
                                             _ptr(ti), _ptr(tv), keep, C.byref(got)))
                k = got.value
                bp.sync_sparse([ti[:k]], [tv[:k]])
            elif self.n > 1:
                import torch.distributed as dist
                dist.all_reduce(g, group=self.group)

    def result(self, i: int):
        """Synced sparse gradient of bucket i (sparse / top-k): ascending int64
        indices and fp32 values on this rank's GPU."""
        bp = self._bp[i]
        if bp is None:
            raise Error("dense buckets are all-reduced in place")
        bp.wait()
        return bp.result()

    def apply_sgd(self, params, grads, lr: float):
        """params[i] -= lr * synced gradient i (sparse buckets on the device via
        zen_axpy_sparse; dense buckets: the all-reduced sum)."""
        for b, p, g, bp in zip(self.buckets, params, grads, self._bp):
            if bp is not None:
                bp.apply_sgd(p, lr)
            else:
                p.view(-1).sub_(g, alpha=lr)

    def normalized_to_allreduce(self, simulated_time: float, bandwidth: float = 1.0) -> float:
        """A SimNet time (TrafficReport.simulated_time at `bandwidth`) over the
        dense ring all-reduce of every bucket -- the paper's "normalized to
        AllReduce" axis (ExperimentRow, experiment.hpp:142-169)."""
        total = sum(b.numel for b in self.buckets)
        base = allreduce_dense_time_bits(self.n, total, bandwidth)
        return simulated_time / base if base else float("nan")
