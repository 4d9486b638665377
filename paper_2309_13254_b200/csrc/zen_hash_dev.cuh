// zen_hash_dev.cuh -- device pieces of the hierarchical hash shared by the
// hash kernels and the extraction compaction (which fuses the placement).
#pragma once

#include "zen_common.cuh"

namespace zen_dev {

// slot word epoch field: newer runs carry smaller words (see k_hash.cu)
__device__ __forceinline__ uint64_t epoch_word(uint32_t epoch) {
  return (uint64_t)(0xFFFFFFu - (epoch & 0xFFFFFFu)) << zen::kKeyBits;
}

// Slot word codecs (zen::SlotOf<K>).  u64 (standalone hash, indices < 2^40):
// [63:40] = 0xFFFFFF - epoch, [39:0] = index+1, so stale epochs lose every
// atomicMin and the memory is never cleared.  u32 (the BP pipeline, M < 2^32
// - 1): the word is index+1, 0xFFFFFFFF = vacant -- half the bytes, so the
// hash memory stays L2-resident twice as long; the depth pass clears the
// words it read, which keeps the memory vacant between syncs.
template <typename W>
struct Slot;
// The u32 words also carry the claiming probe t below the key when
// DevFamily.db > 0: (index+1) << db | t.  The min-claim order is unchanged
// (a key meets itself at no slot), and the probe a key holds a slot by is
// always its FIRST probe onto that slot (a key displaced from slot c by a
// smaller key can never win c back), so readers take the depth from the word
// instead of re-hashing.
template <>
struct Slot<unsigned long long> {
  static constexpr unsigned long long kVacant = ~0ull;
  __device__ __forceinline__ static unsigned long long make(uint64_t ew, uint64_t key, uint32_t = 0,
                                                            uint32_t = 0) {
    return ew | key;
  }
  __device__ __forceinline__ static bool vacant(unsigned long long w, uint64_t ew) {
    return w > (ew | zen::kKeyMask);  // empty or an older epoch
  }
  __device__ __forceinline__ static uint64_t key(unsigned long long w, uint32_t = 0) {
    return w & zen::kKeyMask;
  }
  __device__ __forceinline__ static uint32_t probe(unsigned long long, uint32_t) { return 0; }
};
template <>
struct Slot<unsigned int> {
  static constexpr unsigned int kVacant = 0xFFFFFFFFu;
  __device__ __forceinline__ static unsigned int make(uint64_t, uint64_t key, uint32_t t = 0,
                                                      uint32_t db = 0) {
    return ((unsigned int)key << db) | (db ? t : 0u);
  }
  __device__ __forceinline__ static bool vacant(unsigned int w, uint64_t) { return w == kVacant; }
  __device__ __forceinline__ static uint64_t key(unsigned int w, uint32_t db = 0) { return w >> db; }
  __device__ __forceinline__ static uint32_t probe(unsigned int w, uint32_t db) {
    return w & ((1u << db) - 1u);
  }
};

// Priority claim of one key (deferred acceptance, smallest key wins):
// reproduces place_index's parallel-region layout of the lanes=1 run
// (zen/hashing.hpp:155-163) for any thread schedule.
template <typename W>
__device__ __forceinline__ void place_key(const zen::DevFamily& fam, W* slots, uint64_t key,
                                          uint64_t r1, uint64_t stride, uint64_t ew) {
  using S = Slot<W>;
  const uint32_t p = part_of(fam, key);
  W* base = slots + (uint64_t)p * stride;
  uint64_t cur = key;
  uint32_t t = 0;
  const uint32_t k = fam.k;
  const uint32_t db = sizeof(W) == 4 ? fam.db : 0u;
  while (true) {
    const uint64_t c = slot_of(fam, cur, t, r1);
    const W old = atomicMin(base + c, S::make(ew, cur, t, db));
    if (S::vacant(old, ew)) break;  // empty or stale epoch: cur now holds c
    const uint64_t ok = S::key(old, db);
    if (ok > cur) {  // cur displaced a larger key: it resumes after its first c
      cur = ok;
      uint32_t f = 0;
      if (db)
        f = S::probe(old, db);
      else
        while (f < k && slot_of(fam, cur, f, r1) != c) ++f;
      t = f + 1;
    } else {
      ++t;  // rejected by a smaller key
    }
    if (t >= k) break;  // cur ends serial
  }
}

// KPT independent claims per thread, interleaved: every round issues the
// pending atomicMin of each unfinished key before consuming any result, so a
// thread keeps KPT L2 atomics in flight instead of one (same protocol and
// outcome as place_key: the stable matching does not depend on the schedule).
template <int KPT, typename W>
__device__ __forceinline__ void place_keys(const zen::DevFamily& fam, W* slots,
                                           const uint64_t (&key)[KPT], const uint32_t (&part)[KPT],
                                           uint32_t nvalid, uint64_t r1, uint64_t stride,
                                           uint64_t ew) {
  using S = Slot<W>;
  W* base[KPT];
  uint64_t cur[KPT];
  uint32_t t[KPT];
  bool act[KPT];
  const uint32_t k = fam.k;
  const uint32_t db = sizeof(W) == 4 ? fam.db : 0u;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    act[j] = (uint32_t)j < nvalid;
    cur[j] = key[j];
    t[j] = 0;
    base[j] = slots + (act[j] ? (uint64_t)part[j] * stride : 0ull);
  }
  bool any = nvalid > 0;
  while (any) {
    uint64_t c[KPT];
    W old[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (act[j]) {
        c[j] = slot_of(fam, cur[j], t[j], r1);
        old[j] = atomicMin(base[j] + c[j], S::make(ew, cur[j], t[j], db));
      }
    }
    any = false;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (!act[j]) continue;
      if (S::vacant(old[j], ew)) {  // empty or stale epoch: cur holds c
        act[j] = false;
        continue;
      }
      const uint64_t ok = S::key(old[j], db);
      if (ok > cur[j]) {  // displaced a larger key: it resumes after its first c
        cur[j] = ok;
        uint32_t f = 0;
        if (db)
          f = S::probe(old[j], db);
        else
          while (f < k && slot_of(fam, ok, f, r1) != c[j]) ++f;
        t[j] = f + 1;
      } else {
        ++t[j];
      }
      if (t[j] >= k) act[j] = false;  // ends serial
      any |= act[j];
    }
  }
}

// Continuation of claims already under way: item j is key cur[j] of
// partition part[j] about to try probe t[j] (same protocol as place_keys).
// hist (optional, shared memory, [part][depth] with depth = probe + 1): the
// final occupants' depth histogram kept incrementally -- +1 when a key takes
// a slot, -1 at the displaced key's depth when it loses one.
template <int KPT, typename W>
__device__ __forceinline__ void place_from(const zen::DevFamily& fam, W* slots, uint64_t (&cur)[KPT],
                                           uint32_t (&t)[KPT], const uint32_t (&part)[KPT],
                                           uint32_t nvalid, uint64_t r1, uint64_t stride,
                                           uint64_t ew, int* hist = nullptr) {
  using S = Slot<W>;
  W* base[KPT];
  bool act[KPT];
  const uint32_t k = fam.k;
  const uint32_t db = sizeof(W) == 4 ? fam.db : 0u;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    act[j] = (uint32_t)j < nvalid && t[j] < k;
    base[j] = slots + (act[j] ? (uint64_t)part[j] * stride : 0ull);
  }
  bool any = true;
  while (any) {
    uint64_t c[KPT];
    W old[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j)
      if (act[j]) {
        c[j] = slot_of(fam, cur[j], t[j], r1);
        old[j] = atomicMin(base[j] + c[j], S::make(ew, cur[j], t[j], db));
      }
    any = false;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      if (!act[j]) continue;
      if (S::vacant(old[j], ew)) {
        if (hist) atomicAdd(&hist[part[j] * (k + 1) + t[j] + 1], 1);
        act[j] = false;
        continue;
      }
      const uint64_t ok = S::key(old[j], db);
      if (ok > cur[j]) {
        cur[j] = ok;
        uint32_t f = 0;
        if (db)
          f = S::probe(old[j], db);
        else
          while (f < k && slot_of(fam, ok, f, r1) != c[j]) ++f;
        if (hist) {
          atomicAdd(&hist[part[j] * (k + 1) + t[j] + 1], 1);  // the displacer holds c
          atomicAdd(&hist[part[j] * (k + 1) + f + 1], -1);    // the displaced lost it
        }
        t[j] = f + 1;
      } else {
        ++t[j];
      }
      if (t[j] >= k) act[j] = false;
      any |= act[j];
    }
  }
}

// Hash-memory sizes of this sync from the extraction's h0 counts: the same
// arithmetic as the push scatter's first block (zen/schemes.hpp:363-367), so
// a side chain forked right after the extraction depends on nothing the
// scatter writes.  Every thread computes it (the super-chunk sums are a few
// L2-resident words per partition).
struct SideSizes {
  uint64_t z, r1, r2, stride;
  bool bad;
};
template <typename K>
__device__ __forceinline__ SideSizes side_sizes(const zen::HashArgs<K>& a) {
  const zen::PushCounts& x = a.xc;
  const zen::HashHdr* h = a.hdr;
  SideSizes q{};
  if (!x.early) {
    q.z = h->count;
    q.r1 = h->r1;
    q.r2 = h->r2;
    q.stride = h->stride;
    q.bad = (h->status & zen::kErrCapacity) != 0;
    return q;
  }
  const uint32_t n = a.fam.n;
  for (uint64_t i = 0; i < (uint64_t)n * x.nsup; ++i) q.z += x.scnt[i];
  q.r1 = (uint64_t)ceil(h->r1_mult * (double)q.z / (double)n);
  if (q.r1 < 1) q.r1 = 1;
  q.r2 = (uint64_t)ceil(h->r2_ratio * (double)q.r1);
  if (q.r2 < 1) q.r2 = 1;
  q.stride = q.r1 + q.r2;
  q.bad = q.z > a.cap || q.stride > a.stride_cap;
  return q;
}
// partition p's load (early side chain) or the scatter's count
template <typename K>
__device__ __forceinline__ uint32_t side_load(const zen::HashArgs<K>& a, uint32_t p) {
  const zen::PushCounts& x = a.xc;
  if (!x.early) return a.load[p];
  uint32_t l = 0;
  for (uint32_t i = 0; i < x.nsup; ++i) l += x.scnt[(uint64_t)p * x.nsup + i];
  return l;
}

// meta word of a key after the post pass: partition (9 bits), depth (5),
// stable rank in its 256-key tile among same-partition keys (8) and among
// same-partition serial keys (8).
__device__ __forceinline__ uint32_t pack_meta(uint32_t p, uint32_t depth, uint32_t rank,
                                              uint32_t srank) {
  return p | (depth << 9) | (rank << 14) | (srank << 22);
}
__device__ __forceinline__ uint32_t meta_part(uint32_t m) { return m & 0x1FFu; }
__device__ __forceinline__ uint32_t meta_depth(uint32_t m) { return (m >> 9) & 0x1Fu; }
__device__ __forceinline__ uint32_t meta_rank(uint32_t m) { return (m >> 14) & 0xFFu; }
__device__ __forceinline__ uint32_t meta_srank(uint32_t m) { return (m >> 22) & 0xFFu; }

// per-run header reset + r1/r2 from the (device-resident) key count,
// zen/schemes.hpp:363-367.  Called by one block.
template <typename K>
__device__ __forceinline__ void hash_begin_body(const zen::HashArgs<K>& a) {
  zen::HashHdr* h = a.hdr;
  const uint32_t n = a.fam.n, k = a.fam.k;
  if (threadIdx.x == 0) {
    // all header loads issue together, then the stores (one round trip each)
    const uint64_t z = h->count;
    const uint32_t derive = h->derive, epoch = h->epoch, iter = h->iter;
    const double r1m = h->r1_mult, r2r = h->r2_ratio;
    uint64_t r1 = h->r1, r2 = h->r2;
    if (derive) {
      r1 = (uint64_t)ceil(r1m * (double)z / (double)n);
      if (r1 < 1) r1 = 1;
      r2 = (uint64_t)ceil(r2r * (double)r1);
      if (r2 < 1) r2 = 1;
      h->r1 = r1;
      h->r2 = r2;
    }
    h->stride = r1 + r2;
    h->epoch = epoch + 1u;
    h->ovf_word = ~0ull;
    h->done = 0;
    h->fb_done = 0;
    h->fallback_any = 0;
    h->ntiles = (uint32_t)((z + zen::kHashTile - 1) / zen::kHashTile);
    h->iter = iter + 1u;
    h->bad_index = ~0ull;
    if (z > a.cap || r1 + r2 > a.stride_cap) atomicOr(&h->status, zen::kErrCapacity);
  }
  for (uint32_t i = threadIdx.x; i < n * (k + 1); i += blockDim.x) {
    a.stats[i] = 0;
    a.fb_stats[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) a.fallback[i] = 0;
}

}  // namespace zen_dev
