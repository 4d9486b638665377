/*
 * zen_oracle.c -- TEST INFRASTRUCTURE ONLY (see zen_oracle.h).
 *
 * Plain-C restatement of the reference Balanced-Parallelism path
 * (/root/reference/proj/include/zen/ headers).  Every function cites the
 * reference lines it follows.  It is pinned against the reference itself
 * (tests/golden/ fixtures, produced by oracle/make_golden.py from oracle/_ref, the
 * reference headers) by tests/test_oracle_golden.py.
 */
#include "zen_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- hash family: zen/hashing.hpp:18-39 ------------------------------- */

uint64_t zo_mix64(uint64_t x) { /* hashing.hpp:18-25 (splitmix64 finalizer) */
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

uint64_t zo_seeded_hash(uint64_t x, uint64_t seed) { /* hashing.hpp:27-29 */
  return zo_mix64(x + 0x9e3779b97f4a7c15ULL * (seed + 1));
}

uint64_t zo_map_to_range(uint64_t h, uint64_t range) { /* hashing.hpp:32-34 */
  return (uint64_t)(((unsigned __int128)h * range) >> 64);
}

uint64_t zo_derive_seed(uint64_t master, uint64_t stream) { /* hashing.hpp:37-39 */
  return zo_mix64(master ^ zo_mix64(stream + 0x5851f42d4c957f2dULL));
}

int zo_family_make(uint64_t seed, uint32_t n, uint32_t k, zo_family *out) { /* hashing.hpp:51-60 */
  if (n == 0 || k == 0 || k > ZO_MAX_K) return ZO_E_INVALID;
  memset(out, 0, sizeof(*out));
  out->partitions = n;
  out->k = k;
  out->partition_seed = zo_derive_seed(seed, 0);
  for (uint32_t i = 0; i < k; ++i) out->slot_seeds[i] = zo_derive_seed(seed, 1 + i);
  return ZO_OK;
}

int zo_family_make_worker(uint64_t shared, uint32_t worker, uint32_t n, uint32_t k,
                          zo_family *out) { /* hashing.hpp:64-69 */
  int rc = zo_family_make(shared, n, k, out);
  if (rc) return rc;
  for (uint32_t i = 0; i < k; ++i)
    out->slot_seeds[i] = zo_derive_seed(shared, ((uint64_t)worker + 2) * 1024 + i);
  return ZO_OK;
}

uint32_t zo_family_partition_of(const zo_family *f, uint64_t index) { /* hashing.hpp:73-76 */
  return (uint32_t)zo_map_to_range(zo_seeded_hash(index + 1, f->partition_seed), f->partitions);
}

uint64_t zo_family_slot_of(const zo_family *f, uint64_t index, uint32_t round,
                           uint64_t r1) { /* hashing.hpp:79-81, round is 1-based */
  return zo_map_to_range(zo_seeded_hash(index + 1, f->slot_seeds[round - 1]), r1);
}

uint32_t zo_partition_of(uint64_t index, uint64_t pseed, uint32_t n) { /* hashing.hpp:85-88 */
  return (uint32_t)zo_map_to_range(zo_seeded_hash(index + 1, pseed), n);
}

void zo_partition_of_many(const uint64_t *idx, uint64_t count, uint64_t pseed, uint32_t n,
                          uint32_t *out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = zo_partition_of(idx[i], pseed, n);
}

/* ---- hierarchical hash, lanes = 1: zen/hashing.hpp:121-243 ------------- */

typedef struct {
  uint64_t idx;
  float val;
} zo_pair;

static int cmp_pair(const void *a, const void *b) {
  const zo_pair *x = (const zo_pair *)a, *y = (const zo_pair *)b;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int zo_hierarchical_hash(const uint64_t *idx, const float *val, uint64_t count, uint64_t universe,
                         const zo_family *f, uint64_t r1, uint64_t r2, uint64_t *out_idx,
                         float *out_val, uint64_t *part_count, uint64_t *slots_out,
                         float *slot_vals_out, uint32_t *depth_of, uint64_t *serial_writes,
                         uint64_t *placed_at_depth, int64_t *overflow_partition) {
  /* validation: hashing.hpp:184-187 */
  const uint32_t n = f->partitions;
  if (n == 0 || r1 < 1) return ZO_E_INVALID;
  const uint32_t k = f->k;
  const uint64_t stride = r1 + r2;
  const uint64_t cells = (uint64_t)n * stride;
  /* HashMemory: hashing.hpp:128-136 (slots 0 = empty, cursors start at r1) */
  uint64_t *slots = (uint64_t *)calloc(cells ? cells : 1, sizeof(uint64_t));
  float *values = (float *)calloc(cells ? cells : 1, sizeof(float));
  uint64_t *cursors = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  for (uint32_t p = 0; p < n; ++p) cursors[p] = r1;
  int64_t overflow = -1;
  uint64_t serial = 0;
  uint64_t at_depth[ZO_MAX_K] = {0};

  /* lanes == 1: keys in input (ascending) order, hashing.hpp:199-213 */
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t index = idx[i];
    const uint64_t shifted = index + 1;
    const uint32_t p = zo_family_partition_of(f, index);
    const uint64_t base = (uint64_t)p * stride;
    uint32_t depth = 0;
    int placed = 0;
    /* place_index: hashing.hpp:155-179 */
    for (uint32_t round = 1; round <= k && !placed; ++round) {
      const uint64_t q = zo_family_slot_of(f, index, round, r1);
      if (slots[base + q] == 0) { /* try_claim :138-145 */
        slots[base + q] = shifted;
        values[base + q] = val[i];
        depth = round;
        placed = 1;
      }
    }
    if (!placed) {
      const uint64_t q = cursors[p]++; /* serial cursor :164 */
      if (q < stride) {
        slots[base + q] = shifted;
        values[base + q] = val[i];
        placed = 1;
      } else {
        for (uint64_t s = 0; s < r1 && !placed; ++s) { /* fallback scan :173-175 */
          if (slots[base + s] == 0) {
            slots[base + s] = shifted;
            values[base + s] = val[i];
            placed = 1;
          }
        }
        if (!placed && overflow < 0) overflow = (int64_t)p; /* :176-177 */
      }
    }
    if (depth == 0)
      ++serial;
    else
      ++at_depth[depth - 1];
    if (depth_of) depth_of[i] = depth;
  }

  int rc = ZO_OK;
  if (overflow >= 0) { /* :221-222 */
    if (overflow_partition) *overflow_partition = overflow;
    rc = ZO_E_SERIAL_OVERFLOW;
  } else {
    if (serial_writes) *serial_writes = serial;
    if (placed_at_depth)
      for (uint32_t d = 0; d < k; ++d) placed_at_depth[d] = at_depth[d];
    /* extraction + per-partition sort: :231-241 (from_pairs, tensor.hpp:48-59) */
    uint64_t off = 0;
    zo_pair *pairs = (zo_pair *)malloc((size_t)(stride ? stride : 1) * sizeof(zo_pair));
    for (uint32_t p = 0; p < n; ++p) {
      const uint64_t base = (uint64_t)p * stride;
      uint64_t c = 0;
      for (uint64_t s = 0; s < stride; ++s) {
        if (slots[base + s] != 0) {
          pairs[c].idx = slots[base + s] - 1;
          pairs[c].val = values[base + s];
          ++c;
        }
      }
      qsort(pairs, c, sizeof(zo_pair), cmp_pair);
      for (uint64_t j = 0; j < c; ++j) {
        if (pairs[j].idx >= universe) rc = ZO_E_INVALID;
        out_idx[off + j] = pairs[j].idx;
        out_val[off + j] = pairs[j].val;
      }
      part_count[p] = c;
      off += c;
    }
    free(pairs);
  }
  if (slots_out) memcpy(slots_out, slots, cells * sizeof(uint64_t));
  if (slot_vals_out) memcpy(slot_vals_out, values, cells * sizeof(float));
  free(slots);
  free(values);
  free(cursors);
  return rc;
}

/* ---- extraction: zen/tensor.hpp:94-104 --------------------------------- */

uint64_t zo_to_sparse(const float *dense, uint64_t m, uint64_t *idx, float *val) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < m; ++i) {
    if (dense[i] != 0.0f) { /* tensor.hpp:98: -0.0 dropped, NaN kept */
      idx[c] = i;
      val[c] = dense[i];
      ++c;
    }
  }
  return c;
}

/* ---- aggregation: zen/tensor.hpp:133-167 -------------------------------- */

uint64_t zo_merge_sum(const uint64_t *ia, const float *va, uint64_t na, const uint64_t *ib,
                      const float *vb, uint64_t nb, uint64_t *io, float *vo) {
  uint64_t i = 0, j = 0, o = 0;
  while (i < na && j < nb) {
    if (ia[i] < ib[j]) {
      io[o] = ia[i];
      vo[o++] = va[i++];
    } else if (ia[i] > ib[j]) {
      io[o] = ib[j];
      vo[o++] = vb[j++];
    } else {
      io[o] = ia[i];
      vo[o++] = va[i] + vb[j]; /* left fold: acc + next worker (tensor.hpp:153) */
      ++i;
      ++j;
    }
  }
  for (; i < na; ++i) {
    io[o] = ia[i];
    vo[o++] = va[i];
  }
  for (; j < nb; ++j) {
    io[o] = ib[j];
    vo[o++] = vb[j];
  }
  return o;
}

/* ---- hash universe: zen/codec.hpp:47-72 --------------------------------- */

int zo_universe_create(uint64_t m, uint32_t n, uint64_t pseed, zo_universe **out) {
  if (n == 0) return ZO_E_INVALID;
  zo_universe *u = (zo_universe *)calloc(1, sizeof(zo_universe));
  u->m = m;
  u->n = n;
  u->partition_seed = pseed;
  u->owner = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
  u->rank = (uint64_t *)malloc((size_t)(m ? m : 1) * sizeof(uint64_t));
  u->sizes = (uint64_t *)calloc(n, sizeof(uint64_t));
  u->lists = (uint64_t **)calloc(n, sizeof(uint64_t *));
  for (uint64_t i = 0; i < m; ++i) { /* single O(M) scan, codec.hpp:57-59 */
    const uint32_t s = zo_partition_of(i, pseed, n);
    u->owner[i] = s;
    u->rank[i] = u->sizes[s]++;
  }
  for (uint32_t s = 0; s < n; ++s)
    u->lists[s] = (uint64_t *)malloc((size_t)(u->sizes[s] ? u->sizes[s] : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) u->lists[u->owner[i]][u->rank[i]] = i;
  *out = u;
  return ZO_OK;
}

void zo_universe_destroy(zo_universe *u) {
  if (!u) return;
  for (uint32_t s = 0; s < u->n; ++s) free(u->lists[s]);
  free(u->lists);
  free(u->sizes);
  free(u->rank);
  free(u->owner);
  free(u);
}

uint64_t zo_universe_size(const zo_universe *u, uint32_t s) { return u->sizes[s]; }
const uint64_t *zo_universe_list(const zo_universe *u, uint32_t s) { return u->lists[s]; }

/* ---- hash bitmap codec: zen/codec.hpp:136-158, 266-277, 333-347 -------- */

int zo_hash_bitmap_encode(const zo_universe *u, uint32_t server, const uint64_t *idx,
                          const float *val, uint64_t count, uint8_t *payload,
                          uint64_t *index_bits, uint64_t *bad_index) {
  const uint64_t bits = u->sizes[server];
  const uint64_t bytes = (bits + 7) / 8;
  for (uint64_t i = 0; i < count; ++i) { /* universe_positions: codec.hpp:146-158 */
    if (idx[i] >= u->m || u->owner[idx[i]] != server) {
      if (bad_index) *bad_index = idx[i];
      return ZO_E_INDEX_OUTSIDE_UNIVERSE;
    }
  }
  memset(payload, 0, (size_t)bytes);
  for (uint64_t i = 0; i < count; ++i) { /* set_bit: codec.hpp:136-138 (LSB first) */
    const uint64_t p = u->rank[idx[i]];
    payload[p >> 3] |= (uint8_t)(1u << (p & 7));
  }
  memcpy(payload + bytes, val, (size_t)count * 4); /* values, ascending index (LE) */
  if (index_bits) *index_bits = bits;
  return ZO_OK;
}

int zo_hash_bitmap_decode(const zo_universe *u, uint32_t server, const uint8_t *payload,
                          uint64_t payload_len, uint64_t count, uint64_t *idx, float *val) {
  const uint64_t bits = u->sizes[server];
  const uint64_t bytes = (bits + 7) / 8;
  if (payload_len != bytes + 4 * count) return ZO_E_MALFORMED; /* codec.hpp:336-337 */
  uint64_t c = 0;
  for (uint64_t p = 0; p < bits; ++p) { /* codec.hpp:340-341 */
    if ((payload[p >> 3] >> (p & 7)) & 1u) {
      if (c >= count) return ZO_E_MALFORMED;
      idx[c++] = u->lists[server][p];
    }
  }
  if (c != count) return ZO_E_MALFORMED; /* codec.hpp:342 */
  memcpy(val, payload + bytes, (size_t)count * 4);
  return ZO_OK;
}

/* ---- balanced parallelism: zen/schemes.hpp:341-417 ---------------------- */

void zo_bp_sizes(double r1_mult, double r2_ratio, uint64_t nnz, uint32_t n, uint64_t *r1,
                 uint64_t *r2) { /* schemes.hpp:363-367 */
  uint64_t a = (uint64_t)ceil(r1_mult * (double)nnz / (double)n);
  if (a < 1) a = 1;
  uint64_t b = (uint64_t)ceil(r2_ratio * (double)a);
  if (b < 1) b = 1;
  *r1 = a;
  *r2 = b;
}

double zo_imbalance_pull(const uint64_t *loads, uint32_t n, uint64_t union_size) {
  double worst = 0.0; /* hashing.hpp:311-320 */
  for (uint32_t s = 0; s < n; ++s) {
    double r = (double)n * (double)loads[s] / (double)union_size;
    if (r > worst) worst = r;
  }
  return worst;
}

#define LEDGER(st, field, node) ledger[((st)*4 + (field)) * n + (node)]

int zo_bp_sync(uint32_t n, uint64_t m, const uint64_t *const *idx, const float *const *val,
               const uint64_t *nnz, const zo_hash_params *params, const zo_universe *u,
               uint64_t *out_idx, float *out_val, uint64_t *out_count, uint64_t *ledger,
               uint64_t *counts, uint64_t *agg_counts, double *balance, int *balance_valid,
               int64_t *overflow_partition, uint32_t *overflow_worker) {
  if (n < 2) return ZO_E_INVALID; /* check_inputs: schemes.hpp:66 */
  const uint64_t pseed = zo_derive_seed(params->seed, 0); /* schemes.hpp:349 */
  if (u->m != m || u->n != n || u->partition_seed != pseed) return ZO_E_INVALID; /* :354-356 */
  if (ledger) memset(ledger, 0, sizeof(uint64_t) * 2 * 4 * n);
  uint64_t total = 0;
  for (uint32_t w = 0; w < n; ++w) total += nnz[w];
  /* parted[w] parts concatenated: parts_idx[w] + offsets */
  uint64_t **pidx = (uint64_t **)calloc(n, sizeof(uint64_t *));
  float **pval = (float **)calloc(n, sizeof(float *));
  uint64_t *pcnt = (uint64_t *)calloc((size_t)n * n, sizeof(uint64_t));
  int rc = ZO_OK;
  for (uint32_t w = 0; w < n && rc == ZO_OK; ++w) { /* push: schemes.hpp:360-373 */
    zo_family f;
    rc = zo_family_make_worker(params->seed, w, n, params->rehash_depth, &f);
    if (rc) break;
    uint64_t r1, r2;
    zo_bp_sizes(params->r1_multiplier, params->r2_ratio, nnz[w], n, &r1, &r2);
    pidx[w] = (uint64_t *)malloc((size_t)(nnz[w] ? nnz[w] : 1) * sizeof(uint64_t));
    pval[w] = (float *)malloc((size_t)(nnz[w] ? nnz[w] : 1) * sizeof(float));
    int64_t ovf = -1;
    rc = zo_hierarchical_hash(idx[w], val[w], nnz[w], m, &f, r1, r2, pidx[w], pval[w],
                              pcnt + (size_t)w * n, NULL, NULL, NULL, NULL, NULL, &ovf);
    if (rc == ZO_E_SERIAL_OVERFLOW) {
      if (overflow_partition) *overflow_partition = ovf;
      if (overflow_worker) *overflow_worker = w;
      break;
    }
    if (ledger)
      for (uint32_t s = 0; s < n; ++s) {
        const uint64_t c = pcnt[(size_t)w * n + s];
        if (s == w || c == 0) continue; /* :370 skip self and empty parts */
        LEDGER(0, 0, w) += 96 * c;      /* COO 64-bit index + 32-bit value (codec.hpp:186-189) */
        LEDGER(0, 1, s) += 96 * c;
        LEDGER(0, 2, s) += 64 * c;
        LEDGER(0, 3, s) += 32 * c;
      }
  }
  if (rc == ZO_OK) {
    if (counts) memcpy(counts, pcnt, sizeof(uint64_t) * n * n);
    /* aggregate per server in worker order: schemes.hpp:375-380 */
    uint64_t *acc_i = (uint64_t *)malloc((size_t)(total ? total : 1) * sizeof(uint64_t));
    float *acc_v = (float *)malloc((size_t)(total ? total : 1) * sizeof(float));
    uint64_t *tmp_i = (uint64_t *)malloc((size_t)(total ? total : 1) * sizeof(uint64_t));
    float *tmp_v = (float *)malloc((size_t)(total ? total : 1) * sizeof(float));
    uint64_t out_off = 0;
    uint64_t *loads = (uint64_t *)calloc(n, sizeof(uint64_t));
    /* per-server results land in server order; merge_disjoint afterwards */
    uint64_t **sidx = (uint64_t **)calloc(n, sizeof(uint64_t *));
    float **sval = (float **)calloc(n, sizeof(float *));
    for (uint32_t s = 0; s < n && rc == ZO_OK; ++s) {
      uint64_t na = 0;
      for (uint32_t w = 0; w < n; ++w) {
        uint64_t off = 0;
        for (uint32_t q = 0; q < s; ++q) off += pcnt[(size_t)w * n + q];
        const uint64_t c = pcnt[(size_t)w * n + s];
        const uint64_t no = zo_merge_sum(acc_i, acc_v, na, pidx[w] + off, pval[w] + off, c, tmp_i,
                                         tmp_v);
        memcpy(acc_i, tmp_i, no * sizeof(uint64_t));
        memcpy(acc_v, tmp_v, no * sizeof(float));
        na = no;
      }
      loads[s] = na;
      /* pull: encode + decode through the codec, schemes.hpp:383-390 */
      const uint64_t bytes = (u->sizes[s] + 7) / 8;
      uint8_t *payload = (uint8_t *)malloc((size_t)(bytes + 4 * na + 1));
      uint64_t ib = 0, bad = 0;
      rc = zo_hash_bitmap_encode(u, s, acc_i, acc_v, na, payload, &ib, &bad);
      if (rc) {
        free(payload);
        break;
      }
      if (ledger)
        for (uint32_t w = 0; w < n; ++w) {
          if (w == s) continue; /* pull always sent, even when empty (:387-388) */
          LEDGER(1, 0, s) += ib + 32 * na;
          LEDGER(1, 1, w) += ib + 32 * na;
          LEDGER(1, 2, w) += ib;
          LEDGER(1, 3, w) += 32 * na;
        }
      sidx[s] = (uint64_t *)malloc((size_t)(na ? na : 1) * sizeof(uint64_t));
      sval[s] = (float *)malloc((size_t)(na ? na : 1) * sizeof(float));
      rc = zo_hash_bitmap_decode(u, s, payload, bytes + 4 * na, na, sidx[s], sval[s]);
      free(payload);
    }
    if (rc == ZO_OK) {
      /* merge_disjoint (schemes.hpp:91-113): n-way merge of disjoint sorted parts */
      uint64_t *cur = (uint64_t *)calloc(n, sizeof(uint64_t));
      for (;;) {
        int best = -1;
        for (uint32_t s = 0; s < n; ++s)
          if (cur[s] < loads[s] && (best < 0 || sidx[s][cur[s]] < sidx[best][cur[best]]))
            best = (int)s;
        if (best < 0) break;
        out_idx[out_off] = sidx[best][cur[best]];
        out_val[out_off] = sval[best][cur[best]];
        ++out_off;
        ++cur[best];
      }
      free(cur);
      *out_count = out_off;
      if (agg_counts) memcpy(agg_counts, loads, sizeof(uint64_t) * n);
      /* balance: schemes.hpp:397-410 */
      int all_loaded = 1;
      for (uint32_t w = 0; w < n; ++w) all_loaded = all_loaded && nnz[w] > 0;
      if (balance_valid) *balance_valid = all_loaded;
      if (all_loaded && balance) {
        double worst = 0.0; /* imbalance_push: hashing.hpp:296-308 */
        for (uint32_t w = 0; w < n; ++w)
          for (uint32_t s = 0; s < n; ++s) {
            double r = (double)n * (double)pcnt[(size_t)w * n + s] / (double)nnz[w];
            if (r > worst) worst = r;
          }
        balance[0] = worst;
        uint64_t uni = 0;
        for (uint32_t s = 0; s < n; ++s) uni += loads[s];
        balance[1] = zo_imbalance_pull(loads, n, uni);
      }
    }
    for (uint32_t s = 0; s < n; ++s) {
      free(sidx[s]);
      free(sval[s]);
    }
    free(sidx);
    free(sval);
    free(loads);
    free(acc_i);
    free(acc_v);
    free(tmp_i);
    free(tmp_v);
  }
  for (uint32_t w = 0; w < n; ++w) {
    free(pidx[w]);
    free(pval[w]);
  }
  free(pidx);
  free(pval);
  free(pcnt);
  return rc;
}

/* ---- wire formats: zen/codec.hpp ---------------------------------------- */

static void put_le(uint8_t *p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t *p, int bytes) {
  uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

int zo_wire_encode(const zo_wire_format *f, const zo_universe *u, uint32_t server, uint64_t m,
                   const uint64_t *idx, const float *val, uint64_t count, uint8_t *payload,
                   uint64_t cap, zo_message *out) {
  zo_message msg = {m, count, 0, 32 * count, 0};
  switch (f->kind) {
    case ZO_WIRE_COO: { /* codec.hpp:218-234: all indices, then all values */
      const uint32_t ib = f->coo_index_bits;
      if (ib != 32 && ib != 64) return ZO_E_INVALID;
      msg.index_bits = (uint64_t)ib * count;
      msg.payload_len = (ib / 8 + 4) * count;
      if (msg.payload_len > cap) return ZO_E_INVALID;
      for (uint64_t i = 0; i < count; ++i) {
        if (ib == 32 && idx[i] > 0xffffffffULL) return ZO_E_INVALID;
        put_le(payload + i * (ib / 8), idx[i], (int)(ib / 8));
      }
      memcpy(payload + (uint64_t)(ib / 8) * count, val, (size_t)count * 4);
      break;
    }
    case ZO_WIRE_BITMAP: { /* codec.hpp:236-243: bitmap over [0, M), then values */
      const uint64_t bytes = (m + 7) / 8;
      msg.index_bits = m;
      msg.payload_len = bytes + 4 * count;
      if (msg.payload_len > cap) return ZO_E_INVALID;
      memset(payload, 0, (size_t)bytes);
      for (uint64_t i = 0; i < count; ++i) payload[idx[i] >> 3] |= (uint8_t)(1u << (idx[i] & 7));
      memcpy(payload + bytes, val, (size_t)count * 4);
      break;
    }
    case ZO_WIRE_TENSOR_BLOCK: { /* codec.hpp:244-262 + nonzero_blocks :167-178 */
      const uint64_t b = f->block_size;
      if (b < 1) return ZO_E_INVALID;
      uint64_t nb = 0, values = 0, pos = 0, i = 0;
      while (i < count) { /* sizes first */
        const uint64_t id = idx[i] / b, begin = id * b;
        const uint64_t len = (m - begin < b) ? m - begin : b;
        while (i < count && idx[i] < begin + len) ++i;
        ++nb;
        values += len;
      }
      msg.count = nb;
      msg.index_bits = 64 * nb;
      msg.value_bits = 32 * values;
      msg.payload_len = 8 * nb + 4 * values;
      if (msg.payload_len > cap) return ZO_E_INVALID;
      i = 0;
      while (i < count) {
        const uint64_t id = idx[i] / b, begin = id * b;
        const uint64_t len = (m - begin < b) ? m - begin : b;
        put_le(payload + pos, id, 8);
        pos += 8;
        for (uint64_t e = begin; e < begin + len; ++e) {
          float v = 0.0f;
          if (i < count && idx[i] == e) v = val[i++];
          memcpy(payload + pos, &v, 4);
          pos += 4;
        }
      }
      break;
    }
    case ZO_WIRE_HASH_BITMAP: {
      if (!u) return ZO_E_INVALID;
      const uint64_t bytes = (u->sizes[server] + 7) / 8;
      msg.payload_len = bytes + 4 * count;
      if (msg.payload_len > cap) return ZO_E_INVALID;
      const int rc = zo_hash_bitmap_encode(u, server, idx, val, count, payload, &msg.index_bits, NULL);
      if (rc) return rc;
      break;
    }
    default:
      return ZO_E_INVALID;
  }
  if (out) *out = msg;
  return ZO_OK;
}

/* SparseTensor(M, idx, val): sort when unsorted, then range/duplicate checks
 * (tensor.hpp:36-46, canonicalize :72-84) */
static int canonical(uint64_t m, uint64_t *idx, float *val, uint64_t n) {
  int sorted = 1;
  for (uint64_t i = 1; i < n && sorted; ++i) sorted = idx[i - 1] <= idx[i];
  if (!sorted) {
    zo_pair *p = (zo_pair *)malloc((size_t)(n ? n : 1) * sizeof(zo_pair));
    for (uint64_t i = 0; i < n; ++i) p[i] = (zo_pair){idx[i], val[i]};
    qsort(p, (size_t)n, sizeof(zo_pair), cmp_pair);
    for (uint64_t i = 0; i < n; ++i) {
      idx[i] = p[i].idx;
      val[i] = p[i].val;
    }
    free(p);
  }
  for (uint64_t i = 0; i < n; ++i) {
    if (idx[i] >= m) return ZO_E_INVALID;
    if (i > 0 && idx[i] == idx[i - 1]) return ZO_E_INVALID;
  }
  return ZO_OK;
}

int zo_wire_decode(const zo_wire_format *f, const zo_universe *u, uint32_t server,
                   const zo_message *msg, const uint8_t *payload, uint64_t *idx, float *val,
                   uint64_t cap, uint64_t *out_count) {
  const uint64_t m = msg->universe_size, count = msg->count, len = msg->payload_len;
  uint64_t n = 0;
  switch (f->kind) {
    case ZO_WIRE_COO: { /* codec.hpp:285-296 */
      const uint64_t ib = f->coo_index_bits / 8;
      if (len != (ib + 4) * count) return ZO_E_MALFORMED;
      if (count > cap) return ZO_E_INVALID;
      for (uint64_t i = 0; i < count; ++i) idx[i] = get_le(payload + i * ib, (int)ib);
      memcpy(val, payload + ib * count, (size_t)count * 4);
      n = count;
      break;
    }
    case ZO_WIRE_BITMAP: { /* codec.hpp:297-310 */
      const uint64_t bytes = (m + 7) / 8;
      if (len != bytes + 4 * count) return ZO_E_MALFORMED;
      for (uint64_t b = 0; b < m; ++b)
        if ((payload[b >> 3] >> (b & 7)) & 1u) {
          if (n >= count || n >= cap) return ZO_E_MALFORMED;
          idx[n++] = b;
        }
      if (n != count) return ZO_E_MALFORMED;
      memcpy(val, payload + bytes, (size_t)count * 4);
      break;
    }
    case ZO_WIRE_TENSOR_BLOCK: { /* codec.hpp:311-331 */
      const uint64_t b = f->block_size;
      uint64_t pos = 0;
      for (uint64_t k = 0; k < count; ++k) {
        if (pos + 8 > len) return ZO_E_MALFORMED; /* take_value: payload truncated */
        const uint64_t id = get_le(payload + pos, 8);
        pos += 8;
        const uint64_t begin = id * b;
        if (begin >= m) return ZO_E_MALFORMED;
        const uint64_t blen = (m - begin < b) ? m - begin : b;
        for (uint64_t e = 0; e < blen; ++e) {
          if (pos + 4 > len) return ZO_E_MALFORMED;
          float v;
          memcpy(&v, payload + pos, 4);
          pos += 4;
          if (v != 0.0f) {
            if (n >= cap) return ZO_E_INVALID;
            idx[n] = begin + e;
            val[n++] = v;
          }
        }
      }
      if (pos != len) return ZO_E_MALFORMED;
      break;
    }
    case ZO_WIRE_HASH_BITMAP: {
      if (!u) return ZO_E_INVALID;
      if (count > cap) return ZO_E_INVALID;
      const int rc = zo_hash_bitmap_decode(u, server, payload, len, count, idx, val);
      if (rc) return rc;
      n = count;
      break;
    }
    default:
      return ZO_E_MALFORMED;
  }
  const int rc = canonical(m, idx, val, n);
  if (rc) return rc;
  *out_count = n;
  return ZO_OK;
}

void zo_frame_header(const zo_wire_format *f, const zo_message *msg, uint8_t out[33]) {
  out[0] = (uint8_t)f->kind; /* codec.hpp:358-363 */
  put_le(out + 1, f->block_size, 4);
  put_le(out + 5, f->coo_index_bits, 4);
  put_le(out + 9, msg->universe_size, 8);
  put_le(out + 17, msg->count, 8);
  put_le(out + 25, msg->index_bits + msg->value_bits, 8);
}

int zo_frame_parse(const uint8_t *h, uint64_t len, zo_wire_format *f, zo_message *msg) {
  if (len < 33) return ZO_E_MALFORMED;
  const uint8_t tag = h[0]; /* codec.hpp:368-410 */
  if (tag < 1 || tag > 4) return ZO_E_MALFORMED;
  f->kind = tag;
  f->block_size = (uint32_t)get_le(h + 1, 4);
  f->coo_index_bits = (uint32_t)get_le(h + 5, 4);
  msg->universe_size = get_le(h + 9, 8);
  msg->count = get_le(h + 17, 8);
  const uint64_t bits = get_le(h + 25, 8), c = msg->count;
  switch (tag) {
    case ZO_WIRE_COO:
      msg->index_bits = (uint64_t)f->coo_index_bits * c;
      msg->value_bits = 32 * c;
      msg->payload_len = (f->coo_index_bits / 8 + 4) * c;
      break;
    case ZO_WIRE_BITMAP:
      msg->index_bits = msg->universe_size;
      msg->value_bits = 32 * c;
      msg->payload_len = (msg->universe_size + 7) / 8 + 4 * c;
      break;
    case ZO_WIRE_TENSOR_BLOCK:
      msg->index_bits = 64 * c;
      msg->value_bits = bits >= msg->index_bits ? bits - msg->index_bits : 0;
      if (msg->value_bits % 32) return ZO_E_MALFORMED;
      msg->payload_len = 8 * c + msg->value_bits / 8;
      break;
    default: /* hash bitmap */
      msg->index_bits = bits >= 32 * c ? bits - 32 * c : 0;
      msg->value_bits = 32 * c;
      msg->payload_len = (msg->index_bits + 7) / 8 + 4 * c;
      break;
  }
  if (msg->index_bits + msg->value_bits != bits) return ZO_E_MALFORMED;
  if (len < 33 + msg->payload_len) return ZO_E_MALFORMED; /* payload truncated */
  return ZO_OK;
}

/* ---- .zspt: zen/tensor.hpp:239-285 -------------------------------------- */

uint64_t zo_sparse_file_size(uint64_t count) { return 24 + 12 * count; }

void zo_write_sparse(uint64_t m, const uint64_t *idx, const float *val, uint64_t count,
                     uint8_t *out) {
  memcpy(out, "ZSPT", 4);
  put_le(out + 4, 1, 4);
  put_le(out + 8, m, 8);
  put_le(out + 16, count, 8);
  for (uint64_t i = 0; i < count; ++i) put_le(out + 24 + 8 * i, idx[i], 8);
  memcpy(out + 24 + 8 * count, val, (size_t)count * 4);
}

int zo_read_sparse(const uint8_t *in, uint64_t len, uint64_t *m, uint64_t *idx, float *val,
                   uint64_t cap, uint64_t *count) {
  if (len < 8 || memcmp(in, "ZSPT", 4) != 0) return ZO_E_MALFORMED;
  if (get_le(in + 4, 4) != 1) return ZO_E_MALFORMED;
  if (len < 24) return ZO_E_MALFORMED;
  *m = get_le(in + 8, 8);
  const uint64_t c = get_le(in + 16, 8);
  if (len < 24 + 12 * c) return ZO_E_MALFORMED;
  if (c > cap) return ZO_E_INVALID;
  for (uint64_t i = 0; i < c; ++i) idx[i] = get_le(in + 24 + 8 * i, 8);
  memcpy(val, in + 24 + 8 * c, (size_t)c * 4);
  *count = c;
  if (*m == 0) return ZO_E_INVALID;
  return canonical(*m, idx, val, c);
}

/* ---- sparsify_topk: zen/workload.hpp:157-178 ---------------------------- */

static const float *g_topk_dense;
static int cmp_topk(const void *a, const void *b) { /* |v| descending, index ascending */
  const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  const float mx = fabsf(g_topk_dense[x]), my = fabsf(g_topk_dense[y]);
  if (mx != my) return mx > my ? -1 : 1;
  return x < y ? -1 : x > y;
}

uint64_t zo_sparsify_topk(const float *dense, uint64_t m, double fraction, uint64_t *idx,
                          float *val) {
  if (!(fraction > 0.0 && fraction <= 1.0)) return UINT64_MAX;
  uint64_t keep = (uint64_t)ceil(fraction * (double)m);
  if (keep > m) keep = m;
  uint64_t *order = (uint64_t *)malloc((size_t)(m ? m : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) order[i] = i;
  g_topk_dense = dense;
  qsort(order, (size_t)m, sizeof(uint64_t), cmp_topk);
  zo_pair *p = (zo_pair *)malloc((size_t)(keep ? keep : 1) * sizeof(zo_pair));
  uint64_t n = 0;
  for (uint64_t i = 0; i < keep; ++i)
    if (dense[order[i]] != 0.0f) p[n++] = (zo_pair){order[i], dense[order[i]]};
  qsort(p, (size_t)n, sizeof(zo_pair), cmp_pair);
  for (uint64_t i = 0; i < n; ++i) {
    idx[i] = p[i].idx;
    val[i] = p[i].val;
  }
  free(p);
  free(order);
  return n;
}
