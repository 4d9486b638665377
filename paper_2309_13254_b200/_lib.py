"""ctypes binding of the C-ABI in include/zen_b200.h.

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build``)
into ``paper_2309_13254_b200/lib/libzen_b200.so``.  There is no fallback: if
the library is missing or no sm_100a device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libzen_b200.so")

ZEN_MAX_K = 16
ZEN_MAX_PARTITIONS = 512
ZEN_MAX_WORKERS = 16
ZEN_IPC_HANDLE_BYTES = 64
ZEN_BP_LOCAL = 0xFFFFFFFF
ZEN_STAGES = 4
STAGE_NAMES = ("extract", "hash_push", "aggregate_encode_pull", "decode")

# zen_status
OK, E_INVALID, E_SERIAL_OVERFLOW, E_OUTSIDE, E_MALFORMED, E_EMPTY, E_MISMATCH, E_CUDA, \
    E_PEER, E_OOM, E_TIMEOUT, E_CAPACITY, E_INFEASIBLE = range(13)


class HashParamsC(C.Structure):
    _fields_ = [("rehash_depth", C.c_uint32), ("r1_multiplier", C.c_double),
                ("r2_ratio", C.c_double), ("lanes", C.c_uint32), ("seed", C.c_uint64)]


class HashFamilyC(C.Structure):
    _fields_ = [("partition_seed", C.c_uint64), ("slot_seeds", C.c_uint64 * ZEN_MAX_K),
                ("partitions", C.c_uint32), ("k", C.c_uint32)]


class CollisionStatsC(C.Structure):
    _fields_ = [("serial_writes", C.c_uint64), ("placed_at_depth", C.c_uint64 * ZEN_MAX_K),
                ("k", C.c_uint32)]


class WorkloadSpecC(C.Structure):
    _fields_ = [("universe", C.c_uint64), ("nodes", C.c_uint32), ("density", C.c_double),
                ("omega", C.c_double), ("hot_fraction", C.c_double), ("hot_mass", C.c_double),
                ("seed", C.c_uint64)]


class WireFormatC(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("block_size", C.c_uint32), ("coo_index_bits", C.c_uint32)]


class MessageInfoC(C.Structure):
    _fields_ = [("universe_size", C.c_uint64), ("count", C.c_uint64), ("index_bits", C.c_uint64),
                ("value_bits", C.c_uint64), ("payload_bytes", C.c_uint64)]


FRAME_HEADER_BYTES = 33  # ZEN_FRAME_HEADER_BYTES

vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
P = C.POINTER

_SIGS = {
    "zen_encode": (C.c_int, [vp, P(WireFormatC), vp, u32, vp, vp, u64, u64, vp, u64,
                             P(MessageInfoC)]),
    "zen_decode": (C.c_int, [vp, P(WireFormatC), vp, u32, P(MessageInfoC), vp, vp, vp, u64,
                             P(u64)]),
    "zen_frame_header": (C.c_int, [P(WireFormatC), P(MessageInfoC), vp]),
    "zen_frame_parse": (C.c_int, [vp, u64, P(WireFormatC), P(MessageInfoC)]),
    "zen_sparsify_topk": (C.c_int, [vp, vp, u64, C.c_double, vp, vp, u64, P(u64)]),
    "zen_axpy_sparse": (C.c_int, [vp, vp, u64, vp, vp, u64, C.c_float]),
    "zen_generate": (C.c_int, [vp, P(WorkloadSpecC), u32, vp, vp, u64, P(u64)]),
    "zen_merge_sum": (C.c_int, [vp, vp, vp, u64, vp, vp, u64, u64, vp, vp, u64, P(u64)]),
    "zen_range_counts": (C.c_int, [vp, vp, u64, u64, u32, P(u64)]),
    "zen_count_blocks": (C.c_int, [vp, vp, u64, u64, u64, P(u64)]),
    "zen_compact_nonzero": (C.c_int, [vp, vp, vp, u64, vp, vp, P(u64)]),
    "zen_hc_create": (C.c_int, [vp, u32, u32, u64, u64, P(vp)]),
    "zen_hc_create_scheme": (C.c_int, [vp, u32, u32, u32, u64, u64, P(vp)]),
    "zen_hc_pushes": (u32, [vp]),
    "zen_hc_counts": (C.c_int, [vp, P(u64), P(u64)]),
    "zen_hc_destroy": (None, [vp]),
    "zen_hc_ipc_handle": (C.c_int, [vp, vp]),
    "zen_hc_connect": (C.c_int, [vp, vp]),
    "zen_hc_sync_dense": (C.c_int, [vp, vp]),
    "zen_hc_sync_sparse": (C.c_int, [vp, vp, vp, u64]),
    "zen_hc_wait": (C.c_int, [vp]),
    "zen_hc_result": (C.c_int, [vp, P(vp), P(vp), P(u64)]),
    "zen_hc_copy_result": (C.c_int, [vp, vp, vp, u64, P(u64)]),
    "zen_hc_stage_counts": (C.c_int, [vp, P(u64)]),
    "zen_abi_version": (u32, []),
    "zen_status_string": (C.c_char_p, [C.c_int]),
    "zen_last_error_message": (C.c_char_p, []),
    "zen_last_error_partition": (C.c_int64, []),
    "zen_last_error_index": (u64, []),
    "zen_kernel_launches": (u64, []),
    "zen_derive_seed": (u64, [u64, u64]),
    "zen_debug_hash_schedule": (C.c_int, [u32, u32, u64, u64]),
    "zen_mix64": (u64, [u64]),
    "zen_seeded_hash": (u64, [u64, u64]),
    "zen_map_to_range": (u64, [u64, u64]),
    "zen_hash_family_make": (C.c_int, [u64, u32, u32, P(HashFamilyC)]),
    "zen_hash_family_make_worker": (C.c_int, [u64, u32, u32, u32, P(HashFamilyC)]),
    "zen_ctx_create": (C.c_int, [C.c_int, P(vp)]),
    "zen_ctx_destroy": (None, [vp]),
    "zen_ctx_set_stream": (C.c_int, [vp, vp]),
    "zen_ctx_stream": (vp, [vp]),
    "zen_ctx_own_stream": (vp, [vp]),
    "zen_ctx_synchronize": (C.c_int, [vp]),
    "zen_partition_of": (C.c_int, [vp, vp, u64, u64, u32, vp]),
    "zen_to_sparse": (C.c_int, [vp, vp, u64, vp, vp, u64, P(u64)]),
    "zen_hierarchical_hash": (C.c_int, [vp, vp, vp, u64, u64, P(HashFamilyC), u64, u64, vp, vp,
                                        P(u64), vp, vp, vp, P(CollisionStatsC)]),
    "zen_universe_create": (C.c_int, [vp, u64, u32, u64, P(vp)]),
    "zen_universe_destroy": (None, [vp]),
    "zen_universe_size": (u64, [vp, u32]),
    "zen_universe_indices": (C.c_int, [vp, u32, vp]),
    "zen_hash_bitmap_encode": (C.c_int, [vp, u32, vp, vp, u64, vp, P(u64), P(u64)]),
    "zen_hash_bitmap_decode": (C.c_int, [vp, u32, vp, u64, u64, vp, vp]),
    "zen_bp_create": (C.c_int, [vp, u32, u32, u64, u64, P(HashParamsC), P(vp)]),
    "zen_bp_destroy": (None, [vp]),
    "zen_bp_set_params": (C.c_int, [vp, P(HashParamsC)]),
    "zen_bp_ipc_handle": (C.c_int, [vp, vp]),
    "zen_bp_connect": (C.c_int, [vp, vp]),
    "zen_bp_sync_dense": (C.c_int, [vp, P(vp)]),
    "zen_bp_sync_sparse": (C.c_int, [vp, P(vp), P(vp), P(u64)]),
    "zen_bp_wait": (C.c_int, [vp]),
    "zen_bp_result": (C.c_int, [vp, P(vp), P(vp), P(u64)]),
    "zen_bp_copy_result": (C.c_int, [vp, vp, vp, u64, P(u64)]),
    "zen_bp_traffic": (C.c_int, [vp, vp, vp, vp]),
    "zen_bp_balance": (C.c_int, [vp, P(C.c_double), P(C.c_double), P(C.c_int)]),
    "zen_bp_collision_stats": (C.c_int, [vp, u32, P(CollisionStatsC)]),
    "zen_bp_enable_timing": (C.c_int, [vp, C.c_int]),
    "zen_bp_stage_times": (C.c_int, [vp, vp, P(u64)]),
    "zen_bp_kernels_per_sync": (u32, [vp]),
    "zen_bp_use_graph": (C.c_int, [vp, C.c_int]),
    "zen_bp_time_extract": (C.c_int, [vp, vp, u32, P(C.c_double)]),
    "zen_bp_sync_host": (C.c_int, [vp, P(vp), vp, vp, u64, P(u64)]),
    "zen_bp_debug_part": (C.c_int, [vp, C.c_int, u32, u32, vp, vp, u64, P(u64)]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load(path: str | None = None):
    """Load libzen_b200.so (raises if it was never built -- no fallback).
    ZEN_B200_LIB selects another build of the same library (A/B timing)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("ZEN_B200_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: build it with `make lib` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
