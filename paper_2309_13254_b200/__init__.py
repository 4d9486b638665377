"""B200-native Balanced-Parallelism sparse gradient synchronisation (Zen, arXiv 2309.13254).

The product is paper_2309_13254_b200/lib/libzen_b200.so (sm_100a kernels + C++
host) behind the C-ABI in include/zen_b200.h; this package is its Python
mirror of the reference operator API.
"""
from ._lib import EXPORTED, LIB_PATH, STAGE_NAMES, load  # noqa: F401
from .zen import (  # noqa: F401
    BalanceDetails, BPSynchronizer, CapacityError, CollisionStats, CudaError, DenseTensor,
    EmptyTensor, EncodedMessage, Error, HashFamily, HashLayout, HashParams, HashUniverse,
    HashUniverseTable, IndexOutsideUniverse, MalformedPayload, PartitionedSparseTensor,
    PeerTimeout, SerialOverflow, SimNet, SparseTensor, SyncOutcome, TrafficReport,
    UniverseMismatch, WireFormat, aggregate, bp_universe_table, collision_stats, context, decode,
    derive_seed, encode, exchange_ipc_handles, generate, generate_device, InfeasibleSpec,
    WorkloadSpec, hash_memory_layout, hierarchical_hash,
    imbalance_pull, imbalance_push,
    message_sizes, partition_of, read_framed, read_sparse, read_sparse_file,
    run_balanced_parallelism, run_bp_with_retry, sparsify_topk, to_sparse, write_framed,
    write_sparse,
    write_sparse_file)
from .schemes import (  # noqa: F401
    BALANCED_PARALLELISM, HIERARCHICAL_CENTRALIZATION, AutoSynchronizer, CostInputs, HCSynchronizer,
    MissingProfileEntry, NonPowerOfTwo, SparsityProfile, densification_ratio, density,
    merge_sum, overlap_ratio, profile_sparsity, run_hier_centralization, select_scheme,
    skewness_ratio, t_allreduce_dense, KNOWN_SCHEME_NAMES, Aggregation, BalancePattern,
    CommPattern, PartitionPattern, SchemeConfig, UnsupportedCombination, run_agsparse,
    run_omnireduce_like, run_ring_centralization, run_scheme, scheme_config_from_name, t_bp, t_bp_coefficient, t_hc, t_hc_coefficient,
    t_hierarchy_incremental_lb, t_ring_incremental, t_sparse_ps, t_sparse_ps_broadcast)
from .buckets import Bucket, MixedBucketSync, allreduce_dense_time_bits  # noqa: F401,E402
