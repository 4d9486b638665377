/*
 * zen_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference (arXiv 2309.13254 "zensim",
 * /root/reference/proj/include/zen/ headers) Balanced-Parallelism hot path.
 * It is the parity checker for the sm_100a kernels: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product library (paper_2309_13254_b200/lib/libzen_b200.so)
 * never links or calls it.
 *
 * Pinning: every function is checked against vectors produced by the
 * reference itself (oracle/_ref, built from the reference headers by
 * oracle/Makefile; fixtures in tests/golden/, generator oracle/make_golden.cpp).
 * Semantics follow the reference's lanes=1 (single-lane, ascending-key) run,
 * which is the only deterministic slot layout the reference defines
 * (zen/hashing.hpp:212-213, :259-262).
 */
#ifndef ZEN_ORACLE_H
#define ZEN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZO_MAX_K 16

enum { ZO_OK = 0, ZO_E_INVALID = 1, ZO_E_SERIAL_OVERFLOW = 2, ZO_E_INDEX_OUTSIDE_UNIVERSE = 3,
       ZO_E_MALFORMED = 4, ZO_E_EMPTY = 5, ZO_E_UNIVERSE_MISMATCH = 6 };

/* zen/hashing.hpp:18-39 */
uint64_t zo_mix64(uint64_t x);
uint64_t zo_seeded_hash(uint64_t x, uint64_t seed);
uint64_t zo_map_to_range(uint64_t h, uint64_t range);
uint64_t zo_derive_seed(uint64_t master, uint64_t stream);

/* zen/hashing.hpp:46-82 (HashFamily) */
typedef struct zo_family {
  uint64_t partition_seed;
  uint64_t slot_seeds[ZO_MAX_K];
  uint32_t partitions;
  uint32_t k;
} zo_family;

int zo_family_make(uint64_t seed, uint32_t n, uint32_t k, zo_family *out);
int zo_family_make_worker(uint64_t shared_seed, uint32_t worker, uint32_t n, uint32_t k,
                          zo_family *out);
uint32_t zo_family_partition_of(const zo_family *f, uint64_t index);
uint64_t zo_family_slot_of(const zo_family *f, uint64_t index, uint32_t round, uint64_t r1);
/* zen/hashing.hpp:85-88 */
uint32_t zo_partition_of(uint64_t index, uint64_t partition_seed, uint32_t n);
void zo_partition_of_many(const uint64_t *idx, uint64_t count, uint64_t partition_seed, uint32_t n,
                          uint32_t *out);

/* zen/hashing.hpp:155-262, lanes == 1.
 * parts: concatenated in partition order, each part sorted ascending
 *        (out_idx/out_val have room for `count`; part_count[n]).
 * slots/slot_vals: optional dump of the n*(r1+r2) hash memory (0 = empty,
 *        else index+1; slot values), exactly HashMemory after the run.
 * depth_of: optional per-input-key depth (0 = serial/fallback, else round).
 * Returns ZO_OK, ZO_E_SERIAL_OVERFLOW (*overflow_partition set) or ZO_E_INVALID. */
int zo_hierarchical_hash(const uint64_t *idx, const float *val, uint64_t count, uint64_t universe,
                         const zo_family *f, uint64_t r1, uint64_t r2, uint64_t *out_idx,
                         float *out_val, uint64_t *part_count, uint64_t *slots, float *slot_vals,
                         uint32_t *depth_of, uint64_t *serial_writes, uint64_t *placed_at_depth,
                         int64_t *overflow_partition);

/* zen/tensor.hpp:94-104 */
uint64_t zo_to_sparse(const float *dense, uint64_t m, uint64_t *idx, float *val);

/* zen/tensor.hpp:133-167; returns output count (out arrays sized na+nb). */
uint64_t zo_merge_sum(const uint64_t *ia, const float *va, uint64_t na, const uint64_t *ib,
                      const float *vb, uint64_t nb, uint64_t *io, float *vo);

/* HashUniverseTable (zen/codec.hpp:47-72) as owner/rank arrays over [0, M). */
typedef struct zo_universe {
  uint64_t m;
  uint32_t n;
  uint64_t partition_seed;
  uint32_t *owner; /* [m] */
  uint64_t *rank;  /* [m] position of idx inside its server's sorted list */
  uint64_t *sizes; /* [n] |I_s| */
  uint64_t **lists;/* [n][sizes[s]] sorted I_s */
} zo_universe;

int zo_universe_create(uint64_t m, uint32_t n, uint64_t partition_seed, zo_universe **out);
void zo_universe_destroy(zo_universe *u);
uint64_t zo_universe_size(const zo_universe *u, uint32_t s);
const uint64_t *zo_universe_list(const zo_universe *u, uint32_t s);

/* HashBitmap encode (zen/codec.hpp:266-277): payload = ceil(|I_s|/8) bitmap
 * bytes (LSB-first) then 4*count value bytes.  *bad_index set on
 * ZO_E_INDEX_OUTSIDE_UNIVERSE. */
int zo_hash_bitmap_encode(const zo_universe *u, uint32_t server, const uint64_t *idx,
                          const float *val, uint64_t count, uint8_t *payload,
                          uint64_t *index_bits, uint64_t *bad_index);
/* HashBitmap decode (zen/codec.hpp:333-347). */
int zo_hash_bitmap_decode(const zo_universe *u, uint32_t server, const uint8_t *payload,
                          uint64_t payload_len, uint64_t count, uint64_t *idx, float *val);

/* zen/schemes.hpp:55-61 */
typedef struct zo_hash_params {
  uint32_t rehash_depth;
  double r1_multiplier;
  double r2_ratio;
  uint32_t lanes;
  uint64_t seed;
} zo_hash_params;

/* run_balanced_parallelism (zen/schemes.hpp:341-417).
 * ledger: [2 stages][4 fields: sent, recv, recv_index, recv_value][n] bits.
 * counts: optional [n*n] push part sizes (worker-major), agg_counts: optional [n] U_s.
 * balance[2] = {push, pull}; *balance_valid = 1 iff every input non-empty.
 * out_idx/out_val sized >= sum(nnz). */
int zo_bp_sync(uint32_t n, uint64_t m, const uint64_t *const *idx, const float *const *val,
               const uint64_t *nnz, const zo_hash_params *params, const zo_universe *u,
               uint64_t *out_idx, float *out_val, uint64_t *out_count, uint64_t *ledger,
               uint64_t *counts, uint64_t *agg_counts, double *balance, int *balance_valid,
               int64_t *overflow_partition, uint32_t *overflow_worker);

/* r1/r2 sizing of run_balanced_parallelism (zen/schemes.hpp:363-367). */
void zo_bp_sizes(double r1_multiplier, double r2_ratio, uint64_t nnz, uint32_t n, uint64_t *r1,
                 uint64_t *r2);

/* zen/hashing.hpp:296-320 */
double zo_imbalance_pull(const uint64_t *loads, uint32_t n, uint64_t union_size);

/* ---- wire and file formats: zen/codec.hpp:19-34, 182-347, 352-410;
 *      zen/tensor.hpp:239-303 ------------------------------------------- */
enum { ZO_WIRE_COO = 1, ZO_WIRE_BITMAP = 2, ZO_WIRE_TENSOR_BLOCK = 3, ZO_WIRE_HASH_BITMAP = 4 };
typedef struct zo_wire_format {
  uint32_t kind, block_size, coo_index_bits;
} zo_wire_format;
typedef struct zo_message {
  uint64_t universe_size, count, index_bits, value_bits, payload_len;
} zo_message;

/* encode (codec.hpp:213-278); u/server only for ZO_WIRE_HASH_BITMAP.  Input
 * sorted unique < m.  Returns ZO_E_INVALID when cap is too small or a 32-bit
 * COO index overflows, ZO_E_INDEX_OUTSIDE_UNIVERSE for foreign indices. */
int zo_wire_encode(const zo_wire_format *f, const zo_universe *u, uint32_t server, uint64_t m,
                   const uint64_t *idx, const float *val, uint64_t count, uint8_t *payload,
                   uint64_t cap, zo_message *out);
/* decode (codec.hpp:282-347) + the SparseTensor canonicalisation (sort when
 * unsorted; duplicate / out-of-range -> ZO_E_INVALID, tensor.hpp:36-46). */
int zo_wire_decode(const zo_wire_format *f, const zo_universe *u, uint32_t server,
                   const zo_message *msg, const uint8_t *payload, uint64_t *idx, float *val,
                   uint64_t cap, uint64_t *out_count);
/* write_framed / read_framed header (codec.hpp:356-410): 33 bytes, LE. */
enum { ZO_FRAME_HEADER = 33 };
void zo_frame_header(const zo_wire_format *f, const zo_message *msg, uint8_t out[33]);
int zo_frame_parse(const uint8_t *hdr, uint64_t len, zo_wire_format *f, zo_message *msg);
/* .zspt (tensor.hpp:257-285): "ZSPT", u32 version 1, u64 M, u64 count, idx, val */
uint64_t zo_sparse_file_size(uint64_t count);
void zo_write_sparse(uint64_t m, const uint64_t *idx, const float *val, uint64_t count,
                     uint8_t *out);
int zo_read_sparse(const uint8_t *in, uint64_t len, uint64_t *m, uint64_t *idx, float *val,
                   uint64_t cap, uint64_t *count);
/* sparsify_topk (workload.hpp:157-178): the ceil(fraction*m) largest |v|, ties
 * to the lower index, exact zeros dropped, ascending.  Returns the count or
 * UINT64_MAX for a fraction outside (0, 1]. */
uint64_t zo_sparsify_topk(const float *dense, uint64_t m, double fraction, uint64_t *idx,
                          float *val);

#ifdef __cplusplus
}
#endif
#endif
