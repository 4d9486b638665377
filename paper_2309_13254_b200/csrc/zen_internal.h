// zen_internal.h -- structures shared by the host orchestrator and the
// sm_100a kernels, plus the kernel launcher declarations.  Not part of the
// public C-ABI (include/zen_b200.h).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace zen {

constexpr uint32_t kMaxK = 16;          // rehash depth supported on device
constexpr uint32_t kMaxPartitions = 512;   // n for the standalone hash
constexpr uint32_t kMaxWorkers = 16;    // n for the fused BP pipeline
constexpr uint32_t kHashTile = 256;     // keys per hash tile (one per thread)
constexpr uint32_t kExtractTile = 8192; // floats per extraction tile
constexpr uint32_t kDecodeTileWords = 128;  // 64-index words per decode tile (= block size)
constexpr uint32_t kPrefixBlockWords = 2048;  // bitmap words per popcount-prefix block (512 threads x 4)
                                              // (256 threads x 8 consecutive words)
constexpr uint64_t kKeyBits = 40;       // slot word: [63:40] epoch, [39:0] index+1
constexpr uint64_t kKeyMask = (1ull << kKeyBits) - 1ull;
constexpr uint64_t kPeerTimeoutNs = 30ull * 1000ull * 1000ull * 1000ull;

// HashFamily folded for the device: pc = G*(partition_seed+1), sc[i] =
// G*(slot_seed_i+1) with G = 0x9e3779b97f4a7c15 (zen/hashing.hpp:27-29).
struct DevFamily {
  uint64_t pc;
  uint64_t sc[kMaxK];
  uint32_t n;
  uint32_t k;
  uint32_t db;  // u32 slot words: low bits holding the claiming probe (0 = none)
};

// probe bits packed under the key in the BP pipeline's u32 slot words:
// word = (index + 1) << db | probe.  Needs 2^db >= k and (m + 1) << db < 2^32;
// otherwise 0 and the readers recompute the probe from the hashes.
inline uint32_t slot_probe_bits(uint32_t k, uint64_t m) {
  for (uint32_t db = 1; db <= 4; ++db)
    if ((1u << db) >= k) return ((m + 1) << db) < 0xFFFFFFFFull ? db : 0u;
  return 0u;
}

struct LookbackCtl {
  uint32_t ticket;
  uint32_t done;
  uint32_t tag;
  uint32_t pad;
};

// Per-run hash-stage header in device memory.  r1/r2 may be derived on device
// from the extracted nnz (zen/schemes.hpp:363-367) so a whole BP iteration is
// free of host round trips.
struct HashHdr {
  uint64_t count;        // z (input keys)
  uint64_t r1, r2, stride;
  uint64_t ovf_word;     // min over dropped keys of (key << 16 | p); ~0 = none
  uint32_t epoch;        // hash-memory epoch (1 .. 0xFFFFFE)
  uint32_t ntiles;
  uint32_t derive;       // 1: compute r1/r2 from count with r1_mult/r2_ratio
  uint32_t done;         // scatter blocks finished
  uint32_t iter;         // BP iteration counter (peer flag value)
  uint32_t fallback_any;
  uint32_t status;       // device-side error bits (kErr*), sticky until read
  uint32_t fb_done;      // fallback blocks finished
  double r1_mult, r2_ratio;
  uint64_t bad_index;    // IndexOutsideUniverse witness (min), ~0 = none
  uint32_t work[3];      // push-scatter groups, claim groups, push-scatter blocks done (per sync)
  uint32_t go[2];        // rank mode: push / pull arrival, released by the one polling block
};

constexpr uint32_t kErrTimeout = 1u, kErrOutside = 2u, kErrCapacity = 4u;

// Header a worker writes into every server's inbox (peer memory) after its
// scatter: its whole count row so every rank can rebuild the n x n matrix
// (TrafficReport / imbalance) without another exchange.
struct PushHdr {
  unsigned long long flag;  // = iteration when the data below is valid
  uint64_t nnz;             // worker's z
  uint64_t ovf_word;        // worker's overflow witness
  uint32_t counts[kMaxWorkers];  // |I_w^s| for s = 0..n-1
  uint32_t status;
  uint32_t pad;
};

// Header a server writes into every receiver's pull inbox after encoding.
struct PullHdr {
  unsigned long long flag;
  uint64_t agg_count;  // U_s
  uint64_t bad_index;
  uint32_t status;
  uint32_t pad;
};

// Per-64-index word record of the server's own universe: which of the 64
// indices it owns and how many of its indices precede the word (the rank base
// for HashBitmap positions, zen/codec.hpp:146-158).
struct OwnWord {
  uint64_t mask;
  uint32_t prefix;
  uint32_t pad;
};

// Dense BP data path counters (k_extract.cu PART tiles -> k_push.cu): the
// per-(partition, extraction tile) counts and their sums over 32-tile chunks
// and 1024-tile super chunks.  A tile's partition base is then a sum of at
// most 31 + 31 + ceil(tiles/1024) L2-resident words -- no scan kernel.
struct PushCounts {
  uint32_t* tcnt;   // [n][ntiles] plain stores (every tile, every sync)
  uint32_t* ccnt;   // [n][nchunk] atomics, zeroed by the per-sync begin kernel
  uint32_t* scnt;   // [n][nsup]   atomics, zeroed by the per-sync begin kernel
  uint32_t ntiles, nchunk, nsup, n;
  uint64_t pc;      // G * (partition_seed + 1)
  const void* st_idx;  // the extraction staging (K keys): the side path reads it in place
  uint32_t scatter_grid, place_grid;  // persistent grids (resident blocks)
  uint32_t reorder;       // push scatter regroups each round into per-part runs (peer stores)
  uint32_t fused_signal;  // the push scatter's last block publishes the push (rank mode)
  // local mode (every server on this GPU): the scatter also marks each entry
  // in its server's presence bitmap (k_agg_mark's work), per server p:
  uint32_t mark;
  const OwnWord* const* mk_own;        // [n] server p's {mask, prefix} per 64-index word
  unsigned long long* const* mk_pw;    // [n] server p's presence rows (row w: + w * nws_p)
  uint32_t* const* mk_pre;             // [n] server p's value-base rows (atomicMin, ~0 = none)
  const uint64_t* mk_nws;              // [n] server p's row stride in words
  // the side chain forks right after the extraction and takes z, the loads
  // and r1 / r2 from these counts itself (nothing the push scatter writes)
  uint32_t early;
  // the claims keep the depth histogram themselves (+1 when a key takes a
  // slot, -1 when a key is displaced from one): no table scan, the memory is
  // vacated by a plain clear kernel
  uint32_t inline_hist;
};

// ---- kernel launchers (implemented in k_*.cu) ------------------------------
// All are asynchronous on `stream`; counts live in device memory.

// extraction: dense fp32 -> sorted COO (K = uint32_t or uint64_t).
// Workspace: tile-local staging of the non-zeros (ntiles * kExtractTile
// entries), per-tile counts and exclusive bases.
template <typename K>
struct ExtractWs {
  K* st_idx;
  float* st_val;
  uint32_t* tile_cnt;
  uint64_t* tile_base;
  uint32_t* blk_tile;  // [ceil(cap/256)+1]: tile holding output position 256*b
  uint64_t nblk;       // compaction blocks the workspace was sized for
};
template <typename K>
void launch_extract(const float* dense, uint64_t m, const ExtractWs<K>& ws, K* out_idx,
                    float* out_val, uint64_t* d_count, uint64_t capacity, uint32_t* d_status_bits,
                    cudaStream_t stream);
// pipeline split: tiles + scan fused with the hash begin, then the
// compaction fused with the priority-claim placement
template <typename K>
struct HashArgs;
template <typename K>
void launch_extract_tiles(const float* dense, uint64_t m, const ExtractWs<K>& ws,
                          cudaStream_t stream);
template <typename K>
void launch_extract_scan_begin(uint64_t m, const ExtractWs<K>& ws, const HashArgs<K>& ha,
                               uint64_t capacity, cudaStream_t stream);
// compaction fused with the data path's partition pass (replaces k_part)
template <typename K>
void launch_extract_compact_part(uint64_t m, const ExtractWs<K>& ws, const HashArgs<K>& a,
                                 uint32_t n, cudaStream_t stream);

void launch_partition_of(const uint64_t* idx, uint64_t count, uint64_t pc, uint32_t n,
                         uint32_t* out, cudaStream_t stream);

// hash-memory slot word per key width (zen_hash_dev.cuh Slot<>): u64 with an
// epoch field for the standalone hash, u32 (vacant = ~0) for the BP pipeline
template <typename K>
using SlotOf = typename std::conditional<sizeof(K) == 4, unsigned int, unsigned long long>::type;

template <typename K>
struct HashArgs {
  const K* idx;
  const float* val;
  DevFamily fam;
  HashHdr* hdr;
  SlotOf<K>* slots;           // n * stride_cap words
  float* slot_vals;           // optional (layout dump)
  uint32_t* meta;             // [cap] side path: packed p | depth | serial rank (zen_hash_dev.cuh)
  uint32_t* pmeta;            // [cap] data path: p | (rank in tile among same-p keys) << 16
  uint32_t* tile_cnt;         // [n][tiles_cap] per-tile counts -> exclusive offsets
  uint32_t* tile_scnt;        // [n][tiles_cap] serial counts -> offsets
  uint64_t tiles_cap;         // ceil(cap / kHashTile)
  uint32_t* load;             // [n]
  uint32_t* sload;            // [n] serial keys per partition
  uint64_t* part_off;         // [n] exclusive offsets (contiguous output mode)
  uint32_t* fallback;         // [n]
  uint32_t* stats;            // [n * (k+1)] depth histogram per partition
  uint32_t* fb_stats;         // [n * (k+1)]
  uint64_t* stats_out;        // [k+1] final: serial, depth1..k
  // scatter destinations
  int dst_table;              // 0: contiguous out (out_idx + part_off[p]); 1: pointer tables
  K* out_idx;
  float* out_val;
  K* const* dst_idx;          // [n] device pointer table
  float* const* dst_val;      // [n]
  uint64_t dst_cap;           // capacity per destination part
  uint64_t cap;               // key capacity (grid sizing)
  uint64_t stride_cap;        // r1 + r2 capacity of the hash memory
  // push signalling (pipeline): headers in each server's inbox
  PushHdr* const* push_hdr;   // [n] or nullptr
  uint32_t* const* dst_gbase; // [n] owner p's row for this worker: entries before each
                              // 8-tile group (the fused aggregate's ranges) or nullptr
  uint32_t me;
  int peer;                   // destinations include other GPUs (system-scope release)
  PushCounts xc;              // dense data path (zero-initialised otherwise)
  // claim schedule of k_place (test knob, zen_debug_hash_schedule): grid,
  // block size and a permutation i -> (i * perm_mul + perm_add) mod z of the
  // order in which keys claim; 0 = defaults / identity
  uint32_t place_grid, place_threads;
  uint64_t perm_mul, perm_add;
};

// The hash run = begin (r1/r2, epoch, counters) + a DATA path (partition
// ranks, scan, scatter = the push, push signal) + a SIDE path (placement,
// depths, serial slots, fallback, CollisionStats) that the BP pipeline runs on
// a forked stream, concurrently with the exchange.  launch_hash = all, serial.
template <typename K>
void launch_hash(const HashArgs<K>& a, uint32_t n, uint32_t k, cudaStream_t stream);
template <typename K>
void launch_hash_begin(const HashArgs<K>& a, cudaStream_t stream);
template <typename K>
void launch_hash_part(const HashArgs<K>& a, uint32_t n, cudaStream_t stream);
// part: run k_part first (else the partition pass already ran: compaction or
// launch_hash_part).  The side path reads k_part's partitions (pmeta).
template <typename K>
void launch_hash_critical(const HashArgs<K>& a, uint32_t n, bool part, cudaStream_t stream);
template <typename K>
void launch_hash_side(const HashArgs<K>& a, uint32_t n, bool place, cudaStream_t stream,
                      unsigned ctas_per_sm);
template <typename K>
void launch_push_signal(const HashArgs<K>& a, cudaStream_t stream);

// Dense BP data path (k_push.cu): per-sync begin (header + counter reset),
// extraction tiles with the h0 counts (k_extract.cu), and the push scatter
// straight from the extraction staging into the owners' inboxes (which also
// writes the ascending key list the side path's placement reads).
template <typename K>
void launch_bp_begin(const HashArgs<K>& a, cudaStream_t stream);
template <typename K>
void launch_extract_tiles_part(const float* dense, uint64_t m, const ExtractWs<K>& ws,
                               const HashArgs<K>& a, cudaStream_t stream);
template <typename K>
void launch_push_scatter(const HashArgs<K>& a, const ExtractWs<K>& ws, cudaStream_t stream);
// BP side path after the push scatter: the priority claims, the table-scan
// depth pass (CollisionStats + fallback detection), then the (data-dependent)
// fallback replay
template <typename K>
void launch_hash_side_bp(const HashArgs<K>& a, cudaStream_t stream, unsigned ctas_per_sm,
                         bool place);
// the claims of a dense sync, straight from the extraction staging (k_push.cu)
template <typename K>
void launch_place_tiles(const HashArgs<K>& a, cudaStream_t stream, unsigned ctas_per_sm);
template <typename K>
void launch_vacate(const HashArgs<K>& a, cudaStream_t stream);
// resident blocks of the persistent push scatter
template <typename K>
unsigned push_scatter_grid(bool peer, uint32_t ntiles);


// universe tables (HashUniverseTable, zen/codec.hpp:47-72) as bit planes
void launch_tables_planes(uint64_t m, uint32_t n, uint64_t pc, uint32_t nplanes,
                          unsigned long long* planes, uint32_t* chunk_cnt, cudaStream_t stream);
void launch_tables_scan(uint32_t* chunk_cnt_to_prefix, uint64_t nchunks, uint32_t n,
                        uint64_t* totals, cudaStream_t stream);
void launch_tables_own(uint64_t m, uint32_t n, uint32_t s, uint32_t nplanes,
                       const unsigned long long* planes, const uint32_t* cprefix, OwnWord* own,
                       uint32_t* sel, uint64_t nsel, cudaStream_t stream);

// aggregate + HashBitmap encode of one server, look-back free and
// proportional to (bitmap words + entries):
//  mark   : every received entry sets its rank bit in its worker's presence
//           bitmap P_w (a part is sorted by rank, so entry i of part w is the
//           i-th set bit of P_w);
//  union  : U = OR_w P_w, written straight into every destination's pull
//           inbox (the HashBitmap, NVLink stores in rank mode), plus popcount
//           prefixes of U and of every P_w;
//  values : per set bit of U, fold the contributors' values in worker order
//           (the reference's left fold) and store the value at its rank in U.
struct AggArgs {
  uint32_t n, s;
  uint64_t m;
  const uint32_t* const* in_idx;  // [n] parts w -> s, worker order
  const float* const* in_val;
  const PushHdr* const* in_hdr;   // [n] headers (counts) or nullptr
  const uint64_t* in_count;       // [n] counts when in_hdr == nullptr (standalone encode)
  const uint32_t* const* in_load; // [n] local mode: worker w's partition loads (count = [s])
  const OwnWord* own;
  uint64_t bs;                    // |I_s|
  uint64_t nw;                    // ceil(bs / 64) (>= 1)
  uint64_t nws;                   // row stride of pw / pre: nw rounded up to 8 words
  uint32_t nblk;                  // ceil(nw / kPrefixBlockWords)
  unsigned long long* pw;         // [n * nws] per-worker presence, zeroed per sync
  uint32_t* pre;                  // [(n + 1) * nws] block-local exclusive popcounts (U = n)
  uint32_t* blk;                  // [(n + 1) * nblk] block totals -> exclusive prefixes
  uint32_t* done;                 // [2] blocks-finished counters (self-resetting)
  uint32_t ndst;
  unsigned long long* const* dst_bits;  // [ndst]
  float* const* dst_vals;               // [ndst]
  PullHdr* const* dst_hdr;              // [ndst] or nullptr
  uint64_t val_cap;
  uint64_t* agg_count;            // U_s (device)
  HashHdr* hdr;                   // iteration / error bits / bad index
  int wait_push;                  // wait for in_hdr[w]->flag >= hdr->iter
  int gate;                       // 1: the wait is gated inside k_agg_mark (no k_wait_push)
  int peer;                       // destinations include other GPUs (system-scope release)
  // BP pull: per 32-word chunk of the GLOBAL index space, the number of U_s
  // bits before the chunk's first position in I_s -- the receivers' decode
  // reads its value bases here instead of re-scanning every pulled bitmap
  const uint32_t* cprefix;        // universe chunk prefixes [nchunks * n] (null: off)
  uint64_t nchunks;               // ceil(M / 2048)
  const unsigned long long* own_bits;  // this server's local copy of U (a dst_bits entry)
  uint32_t* const* dst_cbase;     // [ndst] -> (nchunks + 1) u32 per receiver
  int whole;                      // the universe has one server: rank in I_0 = index (no own table)
  const uint32_t* solo_gbase;     // one worker, dense sync: its entries before each 8-tile
                                  // group (push scatter) -> the union builds U from the
                                  // entries and k_agg_mark is skipped; else nullptr
  int pre_min;                    // value bases come from the scatter's atomicMin marks:
                                  // reset each word read to ~0 (ZEN_SCATTER_MARK=1)
  // Fused aggregate (local mode, dense syncs; k_agg_fused): one block per 8
  // extraction tiles (65536 indices) does mark + union + prefix + fold.
  const uint32_t* const* in_gbase; // [n] worker w's entries before each group (its push scatter)
  uint32_t ntiles;                 // extraction tiles
  uint32_t ngroups;                // ceil(ntiles / 8): the fused grid
  const uint4* gtab;               // [ngroups + 1] {R0, jA, first chunk, 0} (k_agg_groups)
  uint32_t span;                   // max bitmap words of one group (shared-memory rows)
  unsigned long long* lbf;         // [ngroups] look-back words (iteration-tagged)
};
// static group table of the fused aggregate (setup): gtab, and *span
void launch_agg_groups(const AggArgs& a, uint32_t* span, cudaStream_t stream);
inline size_t agg_fused_smem(uint32_t n, uint32_t span) { return size_t(12) * (n + 1) * span + 16; }
// marked: the presence bitmaps and value bases were already written by the
// push scatter (local mode, dense syncs), so k_agg_mark is skipped
void launch_aggregate(const AggArgs& a, cudaStream_t stream, bool marked = false,
                      bool fused = false);

// decode of all servers' HashBitmap messages into the global sorted result
struct DecodeArgs {
  uint32_t n;
  uint64_t m;
  uint32_t nplanes;
  const unsigned long long* planes;
  const uint32_t* cprefix;                 // [nchunks32 * n]
  const unsigned long long* const* bits;   // [n] (nullptr: server absent)
  const float* const* vals;                // [n]
  const uint64_t* bs;                      // [n] |I_s| (device)
  const uint64_t* nwords_s;                // [n] bitmap words per server (device)
  const uint32_t* blk_start;               // [n + 1] first prefix block of each server
  uint32_t total_blocks;
  const PullHdr* const* pull_hdr;          // [n] or nullptr
  uint32_t* bpre;                          // [n * words_stride] block-local word popcount prefix
  uint32_t* bpre_blk;                      // [n * blk_stride] block totals -> exclusive prefix
  uint64_t words_stride;                   // per-server stride in bpre
  uint64_t blk_stride;
  uint32_t* done;                          // blocks-finished counter (self-resetting)
  uint64_t* out_idx;
  float* out_val;
  uint64_t* out_count;
  uint64_t out_cap;
  HashHdr* hdr;
  int wait_pull;
  int gate;                                // 1: the wait is gated inside k_decode (no k_wait_pull)
  uint32_t* popc_total;                    // [n] per-server popcount (malformed check)
  const uint32_t* const* cbase;            // [n] pulled per-chunk value bases (BP), or null:
                                           // the prefixes come from k_bpre
};
void launch_decode_parts(const DecodeArgs& a, cudaStream_t stream);

// device workload generator (k_gen.cu)
void launch_gen_tier(uint64_t base, uint64_t range, uint64_t key_seed,
                     const unsigned long long* core, uint64_t core_in_tier, uint64_t want,
                     unsigned long long* bits, uint32_t* blk, cudaStream_t s);
void launch_gen_collect(const unsigned long long* bits, const unsigned long long* core,
                        uint64_t nw, uint32_t* blk, uint64_t* total, uint64_t vseed,
                        uint64_t* out_idx, float* out_val, uint64_t cap, cudaStream_t s);

// small helpers
void launch_u64_to_u32(const uint64_t* in, uint32_t* out, uint64_t n, cudaStream_t stream);
void launch_fill_u64(unsigned long long* p, uint64_t n, uint64_t v, cudaStream_t stream);

// wire formats (k_wire.cu)
constexpr uint32_t kWireIdxOverflow = 1u, kWireUnsorted = 2u, kWireDup = 4u, kWireRange = 8u,
                   kWireMalformed = 16u;
void launch_coo_encode(const uint64_t* idx, const float* val, uint64_t count, int ib,
                       uint8_t* payload, uint32_t* status, cudaStream_t s);
void launch_coo_decode(const uint8_t* payload, uint64_t count, int ib, uint64_t m, uint64_t* idx,
                       float* val, uint32_t* status, cudaStream_t s);
void launch_check_canonical(const uint64_t* idx, uint64_t count, uint64_t m, uint32_t* status,
                            cudaStream_t s);
size_t wire_scan_bytes(uint64_t n);
size_t wire_sort_bytes(uint64_t n);
size_t wire_select_bytes(uint64_t n);
void launch_tb_blocks(const uint64_t* idx, uint64_t count, uint64_t block, uint32_t* first,
                      uint32_t* bpos, void* tmp, size_t tmp_bytes, cudaStream_t s);
void launch_tb_write(const uint64_t* idx, const float* val, uint64_t count, uint64_t block,
                     const uint32_t* first, const uint32_t* bpos, uint8_t* payload, cudaStream_t s);
void launch_tb_walk(const uint8_t* payload, uint64_t len, uint64_t count, uint64_t block,
                    uint64_t m, uint64_t* off, uint64_t* begin, uint32_t* blen, uint32_t* status,
                    cudaStream_t s);
constexpr uint32_t kWireIrregularLayout = 32u;  // k_tb_offsets: fall back to the walk
void launch_tb_offsets(const uint8_t* payload, uint64_t len, uint64_t count, uint64_t block,
                       uint64_t m, uint64_t* off, uint64_t* begin, uint32_t* blen,
                       uint32_t* status, cudaStream_t s);
void launch_tb_expand_select(const uint8_t* payload, uint64_t nb, uint64_t block,
                             const uint64_t* off, const uint64_t* begin, const uint32_t* blen,
                             uint64_t* sidx, float* sval, uint8_t* flag, uint64_t* out_idx,
                             float* out_val, uint64_t* d_count, void* tmp, size_t tmp_bytes,
                             cudaStream_t s);
void launch_sort_pairs(const uint64_t* ki, uint64_t* ko, const float* vi, float* vo,
                       uint64_t count, void* tmp, size_t tmp_bytes, cudaStream_t s);

// top-k sparsification (k_topk.cu + the tile pass of k_extract.cu)
size_t topk_state_bytes();
size_t topk_threshold_offset();
void launch_topk_select(const float* dense, uint64_t m, uint64_t keep, void* state,
                        uint32_t* hist, cudaStream_t s);
void launch_select_tiles(const float* dense, uint64_t m, const ExtractWs<uint32_t>& ws,
                         const uint32_t* key, cudaStream_t stream);
void launch_topk_finish(const ExtractWs<uint32_t>& ws, uint32_t ntiles, void* state,
                        uint32_t* hist, uint32_t* tile_ties, uint64_t* tie_base, uint64_t* out_base,
                        uint64_t* out_count, uint64_t* out_idx, float* out_val, uint64_t cap,
                        cudaStream_t s);

// Hierarchical Centralization + merge_sum (k_merge.cu)
struct HcMergeArgs {
  const uint64_t* a_idx;  // first input (this rank's state), sorted unique
  const float* a_val;
  const uint64_t* a_cnt;
  uint64_t a_cap;
  const uint64_t* b_idx;  // second input (the partner's state, received locally)
  const float* b_val;
  const uint64_t* b_cnt;
  uint64_t b_cap;
  uint64_t* o_idx;  // merge_sum(a, b); *o_cnt = the true size, writes clamp at o_cap
  float* o_val;
  uint64_t* o_cnt;
  uint64_t o_cap;
  unsigned long long* lb_status;  // look-back words, one per tile
  LookbackCtl* ctl;
  uint32_t* err;                        // kErr* bits (kErrOutside: unsorted input)
  const unsigned long long* wait_flag;   // local ready flags to acquire (nullptr: none)
  const unsigned long long* wait_flag2;
  unsigned long long* done_flag;         // senders' done flags to release (nullptr: none)
  unsigned long long* done_flag2;
  const unsigned long long* epoch;       // local sync counter (nullptr: 0)
  uint64_t* stage_cnt;                   // receives |a| (the ledger), may be null
  const uint64_t* a_bnd;                 // optional [begin, end) of a / b inside their
  const uint64_t* b_bnd;                 // buffers (device words; count = end - begin)
  uint64_t* splits;                      // optional [tiles + 1]: the tiles' merge-path splits,
                                         // computed by a one-wave pre-pass (k_hc_splits)
};
struct HcPushArgs {
  const uint64_t* src_idx;
  const float* src_val;
  const uint64_t* src_cnt;
  uint64_t* dst_idx;  // the partner's receive buffer (peer memory)
  float* dst_val;
  uint64_t* dst_cnt;
  uint64_t cap;
  unsigned long long* ready_flag;       // the partner's ready flag
  const unsigned long long* done_flag;  // local: the partner consumed the last push
  const unsigned long long* epoch;
  LookbackCtl* ctl;
  uint32_t* err;
  uint64_t* sent_cnt;  // receives the pushed count (the ledger)
  const uint64_t* src_bnd;  // optional [begin, end) of the source (device words)
  const unsigned long long* src_wait;  // optional local ready flag of the source (forwarding)
};
// n sorted, index-disjoint, ascending segments -> one tensor, exact zeros
// dropped (the block decode of run_omnireduce_like, zen/schemes.hpp:289-295)
struct HcConcatArgs {
  const uint64_t* const* seg_idx;  // [n] device pointer tables
  const float* const* seg_val;
  const uint64_t* const* seg_cnt;
  const unsigned long long* const* wait;  // [n] ready flags to acquire (null entries: none)
  unsigned long long* const* done;        // [n] senders' done flags to release (null: none)
  uint32_t n;
  uint64_t seg_cap;
  uint64_t* o_idx;
  float* o_val;
  uint64_t* o_cnt;
  uint64_t o_cap;
  unsigned long long* lb_status;
  LookbackCtl* ctl;
  uint32_t* err;
  const unsigned long long* epoch;
};
void launch_hc_concat(const HcConcatArgs& a, uint32_t tiles, cudaStream_t stream);
// bnd[p] = lower_bound(idx[0, *count), min(M, p*ceil(M/parts))), p in [0, parts]
void launch_hc_bounds(const uint64_t* idx, const uint64_t* count, uint64_t m, uint32_t parts,
                      uint64_t* bnd, cudaStream_t stream);
uint32_t hc_merge_tiles(uint64_t max_entries);
void launch_hc_merge(const HcMergeArgs& a, uint32_t tiles, cudaStream_t stream);
void launch_hc_push(const HcPushArgs& a, cudaStream_t stream);
void launch_hc_begin(unsigned long long* epoch, cudaStream_t stream);
void launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t stream);

// OmniReduce-like helpers (k_wire.cu)
void launch_count_blocks(const uint64_t* idx, uint64_t count, uint64_t origin, uint64_t block,
                         unsigned long long* out, cudaStream_t s);
void launch_compact_nonzero(const uint64_t* idx, const float* val, uint64_t count, uint8_t* flag,
                            uint64_t* out_idx, float* out_val, uint64_t* d_count, void* tmp,
                            size_t tmp_bytes, cudaStream_t s);

// bnd[p] = lower_bound(idx, min(M, p*ceil(M/parts))), p in [0, parts] (k_util.cu)
void launch_range_bounds(const uint64_t* idx, uint64_t count, uint64_t m, uint32_t parts,
                         uint64_t* bnd, cudaStream_t stream);

// RAII launch policy for the calling thread (see zen_common.cuh launch_k)
struct LaunchScope {
  LaunchScope(bool pdl, bool low_priority);
  ~LaunchScope();
  bool prev_pdl;
  int prev_prio;
};

}  // namespace zen
