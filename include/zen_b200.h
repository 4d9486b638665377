/*
 * zen_b200.h -- C-ABI of the B200-native Balanced-Parallelism sparse gradient
 * synchronisation path (Zen, arXiv 2309.13254).
 *
 * Library: paper_2309_13254_b200/lib/libzen_b200.so (sm_100a kernels + C++
 * host orchestrator).  Plain pointers and sizes only; "d_" arguments are CUDA
 * device pointers on the context's device, "h_" arguments host memory.
 *
 * Each entry point replaces one operator of the reference's header-only C++
 * API (/root/reference/proj/include/zen/ headers); the replaced interface is cited
 * on every declaration.  The C++ drop-in with the reference's own signatures
 * and exception types sits on top of this ABI in include/zen_b200/compat.hpp.
 *
 * Conventions (mirroring the reference, zen/errors.hpp:10-84):
 *  - every call returns a zen_status; ZEN_OK == 0.  On error a thread-local
 *    message (zen_last_error_message) and, for ZEN_E_SERIAL_OVERFLOW, the
 *    overflowing partition (zen_last_error_partition) are set, exactly the data
 *    zen::SerialOverflow carries.
 *  - standalone operators are synchronous on return, like the reference.
 *    The BP pipeline (zen_bp_*) is asynchronous on the context stream and
 *    CUDA-graph capturable; zen_bp_wait is the synchronisation point.
 *  - there is no CPU fallback: without a usable sm_100a device every call
 *    returns ZEN_E_CUDA.
 */
#ifndef ZEN_B200_H
#define ZEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZEN_B200_ABI_VERSION 1u
#define ZEN_MAX_K 16u            /* rehash depth k supported on device */
#define ZEN_MAX_PARTITIONS 512u  /* n for the standalone hierarchical hash */
#define ZEN_MAX_WORKERS 16u      /* n for the fused BP pipeline and the codec */
#define ZEN_IPC_HANDLE_BYTES 64u /* cudaIpcMemHandle_t */
#define ZEN_BP_LOCAL 0xFFFFFFFFu /* zen_bp_create rank: emulate all n workers on one GPU */
#define ZEN_STAGES 4u /* extract kernel | hash+push | aggregate+encode+pull | decode (incl. pull wait) */

/* zen/errors.hpp:10-84 plus the device-side failure classes */
typedef enum zen_status {
  ZEN_OK = 0,
  ZEN_E_INVALID = 1,              /* zen::Error (argument checks) */
  ZEN_E_SERIAL_OVERFLOW = 2,      /* zen::SerialOverflow(partition) */
  ZEN_E_INDEX_OUTSIDE_UNIVERSE = 3, /* zen::IndexOutsideUniverse */
  ZEN_E_MALFORMED = 4,            /* zen::MalformedPayload */
  ZEN_E_EMPTY = 5,                /* zen::EmptyTensor */
  ZEN_E_UNIVERSE_MISMATCH = 6,    /* zen::UniverseMismatch */
  ZEN_E_CUDA = 7,                 /* CUDA runtime / no sm_100a device */
  ZEN_E_PEER = 8,                 /* CUDA IPC / NVLink peer setup */
  ZEN_E_OOM = 9,
  ZEN_E_TIMEOUT = 10,             /* a peer never signalled (device-side watchdog) */
  ZEN_E_CAPACITY = 11,            /* nnz above the capacity the context was sized for */
  ZEN_E_INFEASIBLE = 12           /* zen::InfeasibleSpec (workload generator) */
} zen_status;

/* zen::HashParams, zen/schemes.hpp:55-61 (lanes is accepted and ignored: the
 * device placement always reproduces the deterministic lanes=1 layout) */
typedef struct zen_hash_params {
  uint32_t rehash_depth;
  double r1_multiplier;
  double r2_ratio;
  uint32_t lanes;
  uint64_t seed;
} zen_hash_params;

/* zen::HashFamily, zen/hashing.hpp:46-82 */
typedef struct zen_hash_family {
  uint64_t partition_seed;
  uint64_t slot_seeds[ZEN_MAX_K];
  uint32_t partitions;
  uint32_t k;
} zen_hash_family;

/* zen::CollisionStats, zen/hashing.hpp:104-113 */
typedef struct zen_collision_stats {
  uint64_t serial_writes;
  uint64_t placed_at_depth[ZEN_MAX_K];
  uint32_t k;
} zen_collision_stats;

typedef struct zen_ctx zen_ctx;           /* one device + stream + scratch */
typedef struct zen_universe zen_universe; /* zen::HashUniverseTable on device */
typedef struct zen_bp zen_bp;             /* one BP synchroniser (rank or local) */
typedef struct zen_hc zen_hc;             /* one Hierarchical Centralization rank */

/* ---- library --------------------------------------------------------- */
uint32_t zen_abi_version(void);
const char* zen_status_string(zen_status s);
const char* zen_last_error_message(void);
int64_t zen_last_error_partition(void); /* zen::SerialOverflow::partition(), errors.hpp:36 */
uint64_t zen_last_error_index(void);    /* offending index of ZEN_E_INDEX_OUTSIDE_UNIVERSE */
uint64_t zen_kernel_launches(void);     /* kernels this process launched through the library */

/* ---- hash family (host math) ------------------------------------------ */
/* detail::derive_seed, zen/hashing.hpp:37-39 */
uint64_t zen_derive_seed(uint64_t master, uint64_t stream);
/* detail::mix64 / seeded_hash / map_to_range, zen/hashing.hpp:18-34: the
 * scalar functions behind HashFamily::partition_of / slot_of and the
 * standalone partition_of (:73-88).  One hash per call: host arithmetic (the
 * batched device path is zen_partition_of below). */
uint64_t zen_mix64(uint64_t x);
uint64_t zen_seeded_hash(uint64_t x, uint64_t seed);
uint64_t zen_map_to_range(uint64_t h, uint64_t range);
/* HashFamily::make, zen/hashing.hpp:51-60 */
zen_status zen_hash_family_make(uint64_t seed, uint32_t n, uint32_t k, zen_hash_family* out);
/* HashFamily::make_worker, zen/hashing.hpp:64-69 */
zen_status zen_hash_family_make_worker(uint64_t shared_seed, uint32_t worker, uint32_t n,
                                       uint32_t k, zen_hash_family* out);

/* Test knob for the lock-free priority claim (the hash-memory placement of
 * zen_hierarchical_hash on this thread): grid / block size of the claim kernel
 * and a permutation i -> (i * perm_mul + perm_add) mod count of the order in
 * which keys claim (used only when gcd(perm_mul, count) = 1; threads: a
 * multiple of 32, at most 256).  The layout must
 * not change (the outcome is schedule invariant).  Zeros
 * restore the defaults. */
zen_status zen_debug_hash_schedule(uint32_t grid, uint32_t threads, uint64_t perm_mul,
                                   uint64_t perm_add);

/* ---- device context ---------------------------------------------------- */
zen_status zen_ctx_create(int device, zen_ctx** out);
void zen_ctx_destroy(zen_ctx* ctx);
/* use an external cudaStream_t (e.g. the framework's current stream; NULL is
 * the legacy default stream).  zen_ctx_own_stream returns the context's own
 * non-blocking stream (the initial one). */
zen_status zen_ctx_set_stream(zen_ctx* ctx, void* cuda_stream);
void* zen_ctx_own_stream(zen_ctx* ctx);
void* zen_ctx_stream(zen_ctx* ctx);
zen_status zen_ctx_synchronize(zen_ctx* ctx);

/* ---- standalone operators (synchronous) -------------------------------- */
/* zen::partition_of, zen/hashing.hpp:85-88 (and HashFamily::partition_of :73-76) */
zen_status zen_partition_of(zen_ctx* ctx, const uint64_t* d_idx, uint64_t count,
                            uint64_t partition_seed, uint32_t n, uint32_t* d_out);

/* zen::to_sparse, zen/tensor.hpp:94-104: d_idx/d_val need `capacity` slots;
 * returns ZEN_E_CAPACITY (with *nnz = true count) when they are too small. */
zen_status zen_to_sparse(zen_ctx* ctx, const float* d_dense, uint64_t m, uint64_t* d_idx,
                         float* d_val, uint64_t capacity, uint64_t* nnz);

/* zen::hierarchical_hash + zen::collision_stats + the detail::HashMemory
 * layout, zen/hashing.hpp:181-262.  Input: sorted unique indices < universe.
 * Output parts are concatenated in partition order, each ascending
 * (d_out_idx/d_out_val: count slots; part_count: host [n]).  Optional dumps:
 * d_slots [n*(r1+r2)] (0 = empty else index+1, as HashMemory.slots),
 * d_slot_vals [n*(r1+r2)], d_depth [count] (0 = serial/fallback, else round).
 * Placement is the reference's lanes=1 layout, bit-exact. */
zen_status zen_hierarchical_hash(zen_ctx* ctx, const uint64_t* d_idx, const float* d_val,
                                 uint64_t count, uint64_t universe, const zen_hash_family* family,
                                 uint64_t r1, uint64_t r2, uint64_t* d_out_idx, float* d_out_val,
                                 uint64_t* part_count, uint64_t* d_slots, float* d_slot_vals,
                                 uint32_t* d_depth, zen_collision_stats* stats);

/* ---- hash universe + HashBitmap codec ---------------------------------- */
/* HashUniverseTable(M, n, partition_seed), zen/codec.hpp:47-72 (M < 2^32) */
zen_status zen_universe_create(zen_ctx* ctx, uint64_t m, uint32_t n, uint64_t partition_seed,
                               zen_universe** out);
void zen_universe_destroy(zen_universe* u);
/* |I_s| = HashUniverseTable::universe(s).indices.size() */
uint64_t zen_universe_size(const zen_universe* u, uint32_t server);
/* materialise I_s (ascending) into d_out[zen_universe_size] */
zen_status zen_universe_indices(zen_universe* u, uint32_t server, uint64_t* d_out);
/* encode(t, WireFormat::hash_bitmap(), &universe(s)), zen/codec.hpp:266-277.
 * d_payload receives ceil(|I_s|/8) bitmap bytes then 4*count value bytes. */
zen_status zen_hash_bitmap_encode(zen_universe* u, uint32_t server, const uint64_t* d_idx,
                                  const float* d_val, uint64_t count, uint8_t* d_payload,
                                  uint64_t* index_bits, uint64_t* payload_bytes);
/* decode(msg, &universe(s)), zen/codec.hpp:333-347 (n <= ZEN_MAX_WORKERS) */
zen_status zen_hash_bitmap_decode(zen_universe* u, uint32_t server, const uint8_t* d_payload,
                                  uint64_t payload_bytes, uint64_t count, uint64_t* d_idx,
                                  float* d_val);

/* ---- wire formats: zen/codec.hpp:19-410 -------------------------------- */
/* zen::WireKind (codec.hpp:19) */
#define ZEN_WIRE_COO 1u
#define ZEN_WIRE_BITMAP 2u
#define ZEN_WIRE_TENSOR_BLOCK 3u
#define ZEN_WIRE_HASH_BITMAP 4u
#define ZEN_FRAME_HEADER_BYTES 33u /* write_framed header, codec.hpp:352-366 */
/* zen::WireFormat (codec.hpp:21-35): block_size for TensorBlock, index width
 * (32 or 64) for COO */
typedef struct zen_wire_format {
  uint32_t kind;
  uint32_t block_size;
  uint32_t coo_index_bits;
} zen_wire_format;
/* the header fields of zen::EncodedMessage (codec.hpp:101-111) */
typedef struct zen_message_info {
  uint64_t universe_size;
  uint64_t count;        /* entries (Coo/Bitmap/HashBitmap) or non-zero blocks (TensorBlock) */
  uint64_t index_bits;
  uint64_t value_bits;
  uint64_t payload_bytes;
} zen_message_info;
/* encode(t, fmt, universe), codec.hpp:213-278: device tensor (sorted unique
 * u64 indices < universe) -> device payload bytes, byte-identical to the
 * reference.  u/server only for ZEN_WIRE_HASH_BITMAP.  *out always carries the
 * sizes; ZEN_E_CAPACITY when capacity < out->payload_bytes.  The plain Bitmap
 * needs universe < 2^32. */
zen_status zen_encode(zen_ctx* ctx, const zen_wire_format* fmt, zen_universe* u, uint32_t server,
                      const uint64_t* d_idx, const float* d_val, uint64_t count, uint64_t universe,
                      uint8_t* d_payload, uint64_t capacity, zen_message_info* out);
/* decode(msg, universe), codec.hpp:282-347, plus the SparseTensor
 * canonicalisation (sorted on return; duplicate / out-of-range indices ->
 * ZEN_E_INVALID, tensor.hpp:36-46).  msg: universe_size, count, payload_bytes. */
zen_status zen_decode(zen_ctx* ctx, const zen_wire_format* fmt, zen_universe* u, uint32_t server,
                      const zen_message_info* msg, const uint8_t* d_payload, uint64_t* d_idx,
                      float* d_val, uint64_t capacity, uint64_t* count);
/* write_framed header (codec.hpp:356-366): out[ZEN_FRAME_HEADER_BYTES], host */
zen_status zen_frame_header(const zen_wire_format* fmt, const zen_message_info* msg, uint8_t* out);
/* read_framed header (codec.hpp:368-410): rebuilds the bit accounting and
 * checks it; ZEN_E_MALFORMED on a bad tag / mismatch / fewer than header +
 * payload bytes available */
zen_status zen_frame_parse(const uint8_t* in, uint64_t available, zen_wire_format* fmt,
                           zen_message_info* msg);

/* ---- merge_sum: zen/tensor.hpp:133-167 ---------------------------------- */
/* union of two sorted unique-index tensors over `universe`, shared indices
 * summed (fp32); the fold of every scheme (Hierarchical Centralization:
 * zen/schemes.hpp:173-193).  *count is set even on ZEN_E_CAPACITY. */
zen_status zen_merge_sum(zen_ctx* ctx, const uint64_t* a_idx, const float* a_val, uint64_t na,
                         const uint64_t* b_idx, const float* b_val, uint64_t nb,
                         uint64_t universe, uint64_t* d_idx, float* d_val, uint64_t capacity,
                         uint64_t* count);
/* per-range entry counts behind zen::skewness_ratio (zen/tensor.hpp:193-213):
 * h_counts[p] = entries of the sorted tensor in [p*ceil(M/n), (p+1)*ceil(M/n)) */
zen_status zen_range_counts(zen_ctx* ctx, const uint64_t* d_idx, uint64_t count,
                            uint64_t universe, uint32_t partitions, uint64_t* h_counts);

/* ---- OmniReduce-like block framing: zen/schemes.hpp:227-295 ------------ */
/* non-zero blocks of block_size positions counted from `origin` (sorted input) */
zen_status zen_count_blocks(zen_ctx* ctx, const uint64_t* d_idx, uint64_t count, uint64_t origin,
                            uint64_t block_size, uint64_t* blocks);
/* drop entries whose value is exactly zero, order kept (the block decode) */
zen_status zen_compact_nonzero(zen_ctx* ctx, const uint64_t* d_idx, const float* d_val,
                               uint64_t count, uint64_t* d_out_idx, float* d_out_val,
                               uint64_t* out_count);

/* ---- Hierarchical Centralization: zen/schemes.hpp:173-193 -------------- */
/* One process per GPU, n a power of two (zen::NonPowerOfTwo otherwise:
 * ZEN_E_INVALID).  Stage s (s < log2 n) sends this rank's running aggregate to
 * rank ^ 2^s as NVLink stores into that rank's CUDA-IPC arena and folds the
 * partner's with merge_sum (zen/tensor.hpp:133-167).  Every rank ends with
 * aggregate(inputs), bit-identical across ranks.  The ledger's sent bits at
 * stage s are message_sizes(state_s, fmt) with |state_s| from
 * zen_hc_stage_counts.  max_nnz bounds each rank's input. */
zen_status zen_hc_create(zen_ctx* ctx, uint32_t n, uint32_t rank, uint64_t universe,
                         uint64_t max_nnz, zen_hc** out);
/* the same machinery for the centralized baselines (§8f row f4):
 *   ZEN_SCHEME_HC        run_hier_centralization, zen/schemes.hpp:173-193
 *   ZEN_SCHEME_RING      run_ring_centralization, zen/schemes.hpp:194-215
 *                        (stage s: token -> rank+1; token' = merge(recv, input))
 *   ZEN_SCHEME_AGSPARSE  run_agsparse point-to-point, zen/schemes.hpp:119-168
 *                        (input -> every peer; aggregate in worker order; any n) */
#define ZEN_SCHEME_HC 0u
#define ZEN_SCHEME_RING 1u
#define ZEN_SCHEME_AGSPARSE 2u
#define ZEN_SCHEME_OMNIREDUCE 3u /* run_omnireduce_like, zen/schemes.hpp:219-328 (n >= 2):
                                    ranges -> owners, fold, owners' ranges -> all,
                                    concat with exact zeros dropped */
#define ZEN_SCHEME_AGSPARSE_RING 4u /* run_agsparse, CommPattern::Ring (zen/schemes.hpp:132-142):
                                       stage s forwards the input of rank - s to rank + 1 */
#define ZEN_SCHEME_AGSPARSE_HIER 5u /* run_agsparse, CommPattern::Hierarchy (:143-160):
                                       stage s sends every held input to rank ^ 2^s */
zen_status zen_hc_create_scheme(zen_ctx* ctx, uint32_t scheme, uint32_t n, uint32_t rank,
                                uint64_t universe, uint64_t max_nnz, zen_hc** out);
uint32_t zen_hc_pushes(const zen_hc* hc); /* pushes per sync (entries of zen_hc_stage_counts) */
/* this rank's input entries and result entries of the last sync (the
 * OmniReduce balance, zen/schemes.hpp:297-313, is built from these + the pushes) */
zen_status zen_hc_counts(zen_hc* hc, uint64_t* input_count, uint64_t* result_count);
void zen_hc_destroy(zen_hc* hc);
zen_status zen_hc_ipc_handle(zen_hc* hc, void* out); /* ZEN_IPC_HANDLE_BYTES */
zen_status zen_hc_connect(zen_hc* hc, const void* handles); /* n handles, rank-major */
/* asynchronous on the context stream; the dense form is graph-replayed */
zen_status zen_hc_sync_dense(zen_hc* hc, const float* d_dense);
zen_status zen_hc_sync_sparse(zen_hc* hc, const uint64_t* d_idx, const float* d_val,
                              uint64_t count);
zen_status zen_hc_wait(zen_hc* hc);
zen_status zen_hc_result(zen_hc* hc, const uint64_t** d_idx, const float** d_val,
                         uint64_t* count);
zen_status zen_hc_copy_result(zen_hc* hc, uint64_t* d_idx, float* d_val, uint64_t capacity,
                              uint64_t* count);
/* entries this rank sent per push, in plan order (HC / ring: one per stage;
 * AGsparse: one per peer) -- the SimNet ledger's sent side */
zen_status zen_hc_stage_counts(zen_hc* hc, uint64_t* counts);

/* ---- workload generator (zen::generate, zen/workload.hpp:22-154) ------- */
/* zen::WorkloadSpec */
typedef struct zen_workload_spec {
  uint64_t universe;   /* M */
  uint32_t nodes;      /* n */
  double density;      /* d, per node */
  double omega;        /* target pairwise overlap: shared core of ceil(omega*d*M) */
  double hot_fraction; /* hot tier = the first llround(hot_fraction*M) indices */
  double hot_mass;     /* share of the draws that land in the hot tier */
  uint64_t seed;
} zen_workload_spec;
/* Node `node`'s tensor of zen::generate on the device: ceil(d*M) distinct
 * ascending indices (the shared core + draws from the two-tier distribution
 * without replacement), integer values in [1, 16].  Same spec as the
 * reference, drawn from counter-based hashes (not libstdc++'s mt19937_64
 * streams), so the same seed gives the same tensors on every call and rank.
 * ZEN_E_INFEASIBLE where WorkloadSpec::validate throws InfeasibleSpec
 * (workload.hpp:34-50); ZEN_E_CAPACITY (with *count = the size) when
 * capacity < ceil(d*M).  Synchronous. */
zen_status zen_generate(zen_ctx* ctx, const zen_workload_spec* spec, uint32_t node,
                        uint64_t* d_idx, float* d_val, uint64_t capacity, uint64_t* count);

/* ---- apply: the step after the sync ------------------------------------ */
/* d_dense[idx[i]] += alpha * val[i] for a sorted unique sparse tensor (an SGD
 * step on a synced gradient: alpha = -lr; zen_bp_result gives the synced
 * tensor on the device).  The indices are validated first (ascending, unique,
 * < m, as a SparseTensor guarantees); an invalid tensor -> ZEN_E_INVALID with
 * d_dense untouched.  Synchronous. */
zen_status zen_axpy_sparse(zen_ctx* ctx, float* d_dense, uint64_t m, const uint64_t* d_idx,
                           const float* d_val, uint64_t count, float alpha);

/* ---- top-k sparsification: zen::sparsify_topk ------------------------- */
/* zen/workload.hpp:157-178: the ceil(fraction*m) largest-magnitude entries of
 * a dense fp32 gradient (ties to the lower index), exact zeros dropped,
 * ascending -- bit-exact with the reference.  m < 2^32; NaN magnitudes rank
 * above +inf (the reference's order is undefined for NaN).  *count is set even
 * when ZEN_E_CAPACITY is returned.  Workspace is cached in the context. */
zen_status zen_sparsify_topk(zen_ctx* ctx, const float* d_dense, uint64_t m, double fraction,
                             uint64_t* d_idx, float* d_val, uint64_t capacity, uint64_t* count);

/* ---- Balanced Parallelism: zen::run_balanced_parallelism -------------- */
/* zen/schemes.hpp:341-417.  rank = ZEN_BP_LOCAL hosts all n workers/servers on
 * this context's GPU (exchange = local stores); otherwise this process is
 * worker+server `rank` of n (one process per GPU), and the push/pull are
 * fused into the hash scatter / encode kernels as NVLink stores into peer
 * inboxes mapped by zen_bp_connect.  max_nnz sizes every buffer.  M < 2^32.
 * n == 1 is accepted (the reference requires n >= 2, zen/schemes.hpp:66; the
 * compat layer keeps that check). */
zen_status zen_bp_create(zen_ctx* ctx, uint32_t n, uint32_t rank, uint64_t universe,
                         uint64_t max_nnz, const zen_hash_params* params, zen_bp** out);
void zen_bp_destroy(zen_bp* bp);
/* change k/r1_multiplier/r2_ratio/seed (run_bp_with_retry doubles r2_ratio,
 * zen/experiment.hpp:128-140) */
zen_status zen_bp_set_params(zen_bp* bp, const zen_hash_params* params);
/* rank mode: this rank's CUDA IPC handle (ZEN_IPC_HANDLE_BYTES) and the
 * connection to all n handles (rank-major, n * ZEN_IPC_HANDLE_BYTES) */
zen_status zen_bp_ipc_handle(zen_bp* bp, void* out);
zen_status zen_bp_connect(zen_bp* bp, const void* handles);
/* one synchronisation from dense fp32 gradients [local workers][M] (device) */
zen_status zen_bp_sync_dense(zen_bp* bp, const float* const* d_dense);
/* one synchronisation from sparse inputs (sorted unique u64 indices < M) --
 * the reference's own input (vector<SparseTensor>) */
zen_status zen_bp_sync_sparse(zen_bp* bp, const uint64_t* const* d_idx,
                              const float* const* d_val, const uint64_t* nnz);
/* wait for the last sync and surface its errors in the reference's order
 * (SerialOverflow of the lowest worker first) */
zen_status zen_bp_wait(zen_bp* bp);
/* the synchronised result (identical on every node, SyncOutcome::results),
 * ascending, device-resident until the next sync */
zen_status zen_bp_result(zen_bp* bp, const uint64_t** d_idx, const float** d_val,
                         uint64_t* count);
/* D2D copy of the result into caller buffers (capacity entries) */
zen_status zen_bp_copy_result(zen_bp* bp, uint64_t* d_idx, float* d_val, uint64_t capacity,
                              uint64_t* count);
/* TrafficReport bits (zen/simnet.hpp:15-56) as the reference ledger would
 * record them: ledger [2 stages][4: sent, recv, recv_index, recv_value][n];
 * counts [n*n] |I_w^s| (worker-major); agg_counts [n] U_s.  Any may be NULL. */
zen_status zen_bp_traffic(zen_bp* bp, uint64_t* ledger, uint64_t* counts, uint64_t* agg_counts);
/* BalanceDetails (zen/schemes.hpp:42-45, :397-410); *valid = 0 when some
 * input was empty (the reference leaves balance unset) */
zen_status zen_bp_balance(zen_bp* bp, double* push, double* pull, int* valid);
/* CollisionStats of a local worker's hierarchical hash in the last sync */
zen_status zen_bp_collision_stats(zen_bp* bp, uint32_t worker, zen_collision_stats* out);
/* per-stage CUDA-event timing of every sync while enabled */
zen_status zen_bp_enable_timing(zen_bp* bp, int on);
/* sums over timed syncs since the last call (ms, [ZEN_STAGES]); resets */
zen_status zen_bp_stage_times(zen_bp* bp, double* ms, uint64_t* syncs);
/* kernels launched per sync (this rank) */
uint32_t zen_bp_kernels_per_sync(const zen_bp* bp);
/* replay dense syncs from a captured CUDA graph (default on; needs a
 * non-legacy stream, see zen_ctx_set_stream) */
zen_status zen_bp_use_graph(zen_bp* bp, int on);
/* average duration (ms) of the extraction kernel alone over `iters`
 * back-to-back launches on the context stream (roofline measurement; uses the
 * synchroniser's workspace, so not concurrently with a sync) */
zen_status zen_bp_time_extract(zen_bp* bp, const float* d_dense, uint32_t iters, double* ms);
/* end to end from HOST buffers: H2D of the dense gradients (pinned host
 * memory recommended), the sync, D2H of the result. */
zen_status zen_bp_sync_host(zen_bp* bp, const float* const* h_dense, uint64_t* h_idx,
                            float* h_val, uint64_t capacity, uint64_t* count);

/* diagnostics (tests only): what = 0 -> a local worker's compacted keys (u32
 * indices); what = 1 -> the part `worker` pushed into local `server`'s inbox */
zen_status zen_bp_debug_part(zen_bp* bp, int what, uint32_t server, uint32_t worker,
                             uint32_t* h_idx, float* h_val, uint64_t capacity, uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* ZEN_B200_H */
