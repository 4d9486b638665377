// k_hash.cu -- hierarchical hashing (Algorithm 1; zen/hashing.hpp:121-262) on sm_100a.
//
// Bit-exact with the reference's single-lane run (the only layout the
// reference defines deterministically, zen/hashing.hpp:212-213 and :259-262).
// Split into two independent paths so that the hash memory placement -- which
// the parts do not depend on -- runs off the critical path of a BP sync:
//
// DATA PATH (feeds the push):
//  part    : one key per thread, 256-key tiles: h0 partition and the key's
//            stable rank inside its tile among same-partition keys
//            (match_any + per-warp counts); per-(partition, tile) counts.
//  scan    : one block per partition scans its tile counts -> loads.
//  scatter : position = tile offset + rank, i.e. a stable multi-split by h0 ->
//            the parts, ascending as from_pairs sorts (zen/tensor.hpp:48-59).
//            In the BP pipeline the destinations are the owners' inboxes, so
//            the push (NVLink stores in rank mode) is fused here.  Overflow
//            (load > r1+r2) depends on the loads only: its witness is the
//            (r1+r2+1)-th key of an overfull partition, the globally smallest
//            of which is the reference's first drop (zen/hashing.hpp:176-177).
//
// SIDE PATH (hash memory layout + CollisionStats, concurrent with the push):
//  place   : lock-free PRIORITY CLAIM.  Slots are u64 words
//            [63:40] = 0xFFFFFF - epoch, [39:0] = index+1; a key proposes with
//            atomicMin, so the smallest key wins every slot it ever asks for
//            and a displaced key resumes after the first occurrence of that
//            slot in its own probe list.  Deferred acceptance with one common
//            priority order has a unique stable outcome = serial dictatorship
//            in ascending key order = the reference's lanes=1 greedy, for ANY
//            thread schedule.  Older epochs carry larger words, so stale slots
//            lose automatically: no memset of the hash memory per run.
//  depth   : the first probe whose slot holds the key gives its depth, else it
//            is serial; stable serial ranks per tile; depth histogram.
//  serial  : per-partition scan of serial counts; serial keys take slot
//            r1 + (ascending serial rank).
//  fallback: partitions whose serial keys exceed r2 hit the order-dependent
//            fallback scan (zen/hashing.hpp:170-175) and are replayed
//            sequentially (rare: ~3% serial vs r2 = 10% of r1).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "zen_common.cuh"
#include "zen_hash_dev.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kInvalid = 0xFFFFFFFFu;
static_assert(kHashTile == kThreads, "one key per thread");

template <typename K>
__global__ void k_hash_begin(HashArgs<K> a) {
  zen_dev::pdl_entry();
  hash_begin_body(a);
}

// ------------------------------------------------------------- data path ----

template <typename K>
__global__ void __launch_bounds__(kThreads) k_part(HashArgs<K> a) {
  zen_dev::pdl_entry();
  extern __shared__ uint32_t sm[];
  const uint32_t n = a.fam.n;
  uint32_t* wc = sm;  // [kWarps][n] key counts -> cross-warp prefixes
  const HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint32_t tile = blockIdx.x;
  if (tile >= h->ntiles) return;
  const uint64_t z = h->count;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t q = threadIdx.x; q < kWarps * n; q += kThreads) wc[q] = 0;
  const uint64_t i = (uint64_t)tile * kHashTile + threadIdx.x;
  const bool valid = i < z;
  const uint32_t p = valid ? part_of(a.fam, (uint64_t)a.idx[i] + 1) : kInvalid;
  __syncthreads();
  const uint32_t g = __match_any_sync(0xffffffffu, p);
  const uint32_t wr = __popc(g & lanemask_lt());
  if (valid && lane == (uint32_t)(__ffs(g) - 1)) wc[warp * n + p] = __popc(g);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < n; q += kThreads) {
    uint32_t acc = 0;
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t t = wc[w * n + q];
      wc[w * n + q] = acc;
      acc += t;
    }
    a.tile_cnt[(uint64_t)q * a.tiles_cap + tile] = acc;
  }
  __syncthreads();
  if (valid) a.pmeta[i] = p | ((wc[warp * n + p] + wr) << 16);
}

// exclusive scan of `ntiles` per-tile counts, in place (one block)
__device__ __forceinline__ uint32_t block_scan_tiles(uint32_t* arr, uint32_t ntiles,
                                                     uint32_t* sscan) {
  constexpr int E = 4;
  uint32_t carry = 0;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x * E) {
    const uint32_t t0 = b + threadIdx.x * E;
    uint32_t v[E], local = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      v[e] = (t0 + e < ntiles) ? arr[t0 + e] : 0u;
      local += v[e];
    }
    uint32_t tot;
    uint32_t ex = carry + block_exclusive_sum(local, sscan, &tot);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (t0 + e < ntiles) arr[t0 + e] = ex;
      ex += v[e];
    }
    carry += tot;
  }
  return carry;
}

template <typename K>
__global__ void __launch_bounds__(1024) k_part_scan(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sscan[33];
  HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint32_t p = blockIdx.x;
  const uint32_t total =
      block_scan_tiles(a.tile_cnt + (uint64_t)p * a.tiles_cap, h->ntiles, sscan);
  if (threadIdx.x == 0) a.load[p] = total;
}

// one key per thread per tile, kScatterTiles tiles per block, every load of
// the block's tiles issued before the stores
constexpr int kScatterTiles = 4;

template <typename K>
__global__ void __launch_bounds__(kThreads) k_scatter(HashArgs<K> a) {
  zen_dev::pdl_entry();
  extern __shared__ uint64_t soff[];  // [n] part offsets (contiguous mode)
  const uint32_t n = a.fam.n;
  HashHdr* h = a.hdr;
  const bool ok = !(h->status & kErrCapacity);
  const uint64_t z = h->count, r1 = h->r1, r2 = h->r2;
  const uint32_t ntiles = h->ntiles, tile0 = blockIdx.x * kScatterTiles;
  if (!a.dst_table) {
    if (threadIdx.x == 0) {
      uint64_t off = 0;
      for (uint32_t q = 0; q < n; ++q) {
        soff[q] = off;
        off += a.load[q];
      }
    }
    __syncthreads();
  }
  if (!ok || tile0 >= ntiles) return;
  uint32_t pm[kScatterTiles], p[kScatterTiles];
  K x[kScatterTiles];
  float v[kScatterTiles];
  uint64_t pos[kScatterTiles];
#pragma unroll
  for (int j = 0; j < kScatterTiles; ++j) {
    const uint64_t i = (uint64_t)(tile0 + j) * kHashTile + threadIdx.x;
    pm[j] = 0;
    if (tile0 + j < ntiles && i < z) {
      pm[j] = a.pmeta[i] | 0x80000000u;  // bit 31: valid (ranks are < 2^15)
      x[j] = a.idx[i];
      v[j] = a.val[i];
    }
  }
#pragma unroll
  for (int j = 0; j < kScatterTiles; ++j) {
    p[j] = pm[j] & 0xFFFFu;
    pos[j] = (pm[j] >> 31) ? (uint64_t)a.tile_cnt[(uint64_t)p[j] * a.tiles_cap + tile0 + j] +
                                 ((pm[j] >> 16) & 0x7FFFu)
                           : 0;
  }
#pragma unroll
  for (int j = 0; j < kScatterTiles; ++j) {
    if (!(pm[j] >> 31)) continue;
    if (a.dst_table) {
      if (pos[j] < a.dst_cap) {
        a.dst_idx[p[j]][pos[j]] = x[j];
        a.dst_val[p[j]][pos[j]] = v[j];
      } else {
        atomicOr(&h->status, kErrCapacity);
      }
    } else {
      a.out_idx[soff[p[j]] + pos[j]] = x[j];
      a.out_val[soff[p[j]] + pos[j]] = v[j];
    }
    if (pos[j] == r1 + r2)
      atomicMin((unsigned long long*)&h->ovf_word, (((uint64_t)x[j] + 1) << 16) | p[j]);
  }
}

// Pipeline scatter (pointer-table destinations): the tile's keys are first
// reordered in shared memory into their partitions' runs (block offset of p +
// stable rank), so consecutive threads store consecutive positions of one
// destination part -- full-line (NVLink) stores instead of ~n short segments
// per warp.
template <typename K>
__global__ void __launch_bounds__(kThreads) k_scatter_runs(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ K s_x[kHashTile];
  __shared__ float s_v[kHashTile];
  __shared__ uint16_t s_p[kHashTile];
  __shared__ uint32_t s_boff[kMaxWorkers], s_base[kMaxWorkers];
  const uint32_t n = a.fam.n;
  HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint32_t tile = blockIdx.x, ntiles = h->ntiles;
  if (tile >= ntiles) return;
  const uint64_t z = h->count, r1 = h->r1, r2 = h->r2;
  const uint64_t left = z - (uint64_t)tile * kHashTile;
  const uint32_t keys = left < kHashTile ? (uint32_t)left : kHashTile;
  if (threadIdx.x < 32) {  // per-partition counts of this tile -> block offsets
    const uint32_t q = threadIdx.x;
    uint32_t base = 0, cnt = 0;
    if (q < n) {
      base = a.tile_cnt[(uint64_t)q * a.tiles_cap + tile];
      const uint32_t next =
          tile + 1 < ntiles ? a.tile_cnt[(uint64_t)q * a.tiles_cap + tile + 1] : a.load[q];
      cnt = next - base;
    }
    const uint32_t inc = warp_inclusive_sum(cnt);
    if (q < n) {
      s_boff[q] = inc - cnt;
      s_base[q] = base;
    }
  }
  __syncthreads();
  const uint64_t i = (uint64_t)tile * kHashTile + threadIdx.x;
  if (threadIdx.x < keys) {
    const uint32_t pm = a.pmeta[i];
    const uint32_t p = pm & 0xFFFFu;
    const uint32_t slot = s_boff[p] + (pm >> 16);
    s_x[slot] = a.idx[i];
    s_v[slot] = a.val[i];
    s_p[slot] = (uint16_t)p;
  }
  __syncthreads();
  if (threadIdx.x >= keys) return;
  const uint32_t t = threadIdx.x, p = s_p[t];
  const uint64_t pos = (uint64_t)s_base[p] + (t - s_boff[p]);
  const K x = s_x[t];
  if (pos < a.dst_cap) {
    a.dst_idx[p][pos] = x;
    a.dst_val[p][pos] = s_v[t];
  } else {
    atomicOr(&h->status, kErrCapacity);
  }
  if (pos == r1 + r2)
    atomicMin((unsigned long long*)&h->ovf_word, (((uint64_t)x + 1) << 16) | p);
}

// Push signalling: one block after the scatter (the kernel boundary completes
// every part store, NVLink stores in rank mode): this worker's count row into
// every server's inbox header, then the flag (release, system scope).
template <typename K>
__global__ void k_push_signal(HashArgs<K> a) {
  zen_dev::pdl_entry();
  HashHdr* h = a.hdr;
  const uint32_t n = a.fam.n;
  fence_for(a.peer);
  const bool cap_ok = !(h->status & kErrCapacity);
  const uint64_t ovf = *(volatile uint64_t*)&h->ovf_word;
  const uint32_t st = *(volatile uint32_t*)&h->status;
  const uint64_t z = h->count;
  const uint32_t iter = h->iter;
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
    PushHdr* ph = a.push_hdr[s];
    ph->nnz = z;
    ph->ovf_word = ovf;
    ph->status = st;
    for (uint32_t q = 0; q < n; ++q) ph->counts[q] = cap_ok ? a.load[q] : 0u;
    // the release orders this thread's header stores before the flag (no
    // second fence: the same thread wrote them)
    st_release_sys(&ph->flag, (unsigned long long)iter);
  }
}

// ------------------------------------------------------------- side path ----

template <typename K>
__global__ void __launch_bounds__(kThreads) k_place(HashArgs<K> a) {
  zen_dev::pdl_entry();
  const HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint64_t z = h->count, r1 = h->r1, stride = h->stride;
  const uint64_t ew = epoch_word(h->epoch);
  constexpr int KPT = 4;  // claims in flight per thread
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < z; i0 += nthr * KPT) {
    uint64_t key[KPT];
    uint32_t part[KPT];
    uint32_t nv = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
      uint64_t i = i0 + (uint64_t)j * nthr;
      if (a.perm_mul && i < z)  // test knob: another claim order, same outcome
        i = (uint64_t)(((unsigned __int128)i * a.perm_mul + a.perm_add) % z);
      key[j] = i < z ? (uint64_t)a.idx[i] + 1 : 0ull;
      part[j] = i < z ? (a.pmeta[i] & 0xFFFFu) : 0u;  // h0 from the data path's pass
      nv += i < z ? 1u : 0u;
    }
    place_keys<KPT>(a.fam, a.slots, key, part, nv, r1, stride, ew);
  }
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_depth(HashArgs<K> a) {
  zen_dev::pdl_entry();
  extern __shared__ uint32_t sm[];
  const uint32_t n = a.fam.n, k = a.fam.k;
  uint32_t* ws = sm;  // [kWarps][n] serial counts -> cross-warp prefixes
  const HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint64_t z = h->count, r1 = h->r1, stride = h->stride;
  const uint64_t ew = epoch_word(h->epoch);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t ntiles = h->ntiles;
  // grid-stride over tiles: the side path keeps to a fraction of the SMs
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < kWarps * n; q += kThreads) ws[q] = 0;
    const uint64_t i = (uint64_t)tile * kHashTile + threadIdx.x;
    const bool valid = i < z;
    uint32_t p = kInvalid, depth = 0;
    if (valid) {
      const uint64_t key = (uint64_t)a.idx[i] + 1;
      p = a.pmeta[i] & 0xFFFFu;  // h0 from the data path's partition pass
      const uint64_t base = (uint64_t)p * stride;
      // the first four candidates are loaded together (k = 3 by default)
      uint64_t c4[4];
      SlotOf<K> s4[4];
#pragma unroll
      for (uint32_t t = 0; t < 4; ++t)
        if (t < k) {
          c4[t] = slot_of(a.fam, key, t, r1);
          s4[t] = a.slots[base + c4[t]];
        }
      uint64_t hit = ~0ull;
#pragma unroll
      for (uint32_t t = 0; t < 4; ++t)
        if (t < k && depth == 0 && s4[t] == Slot<SlotOf<K>>::make(ew, key)) {
          depth = t + 1;
          hit = c4[t];
        }
      for (uint32_t t = 4; depth == 0 && t < k; ++t) {
        const uint64_t c = slot_of(a.fam, key, t, r1);
        if (a.slots[base + c] == Slot<SlotOf<K>>::make(ew, key)) {
          depth = t + 1;
          hit = c;
        }
      }
      if (depth && a.slot_vals) a.slot_vals[base + hit] = a.val[i];
    }
    __syncthreads();
    const uint32_t ks = (valid && depth == 0) ? p : kInvalid;
    const uint32_t gs = __match_any_sync(0xffffffffu, ks);
    const uint32_t wsr = __popc(gs & lanemask_lt());
    if (ks != kInvalid && lane == (uint32_t)(__ffs(gs) - 1)) ws[warp * n + p] = __popc(gs);
    const uint32_t kd = valid ? (p * 32u + depth) : kInvalid;
    const uint32_t gd = __match_any_sync(0xffffffffu, kd);
    if (valid && lane == (uint32_t)(__ffs(gd) - 1))
      atomicAdd(&a.stats[p * (k + 1) + depth], (uint32_t)__popc(gd));
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < n; q += kThreads) {
      uint32_t acc = 0;
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = ws[w * n + q];
        ws[w * n + q] = acc;
        acc += t;
      }
      a.tile_scnt[(uint64_t)q * a.tiles_cap + tile] = acc;
    }
    __syncthreads();
    if (valid) a.meta[i] = pack_meta(p, depth, 0, depth == 0 ? ws[warp * n + p] + wsr : 0u);
  }
}

template <typename K>
__global__ void __launch_bounds__(1024) k_serial_scan(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sscan[33];
  HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint32_t p = blockIdx.x;
  const uint32_t total =
      block_scan_tiles(a.tile_scnt + (uint64_t)p * a.tiles_cap, h->ntiles, sscan);
  if (threadIdx.x == 0) {
    a.sload[p] = total;
    const uint32_t fb = (total > h->r2 && (uint64_t)a.load[p] <= h->r1 + h->r2) ? 1u : 0u;
    a.fallback[p] = fb;
    if (fb) atomicOr(&h->fallback_any, 1u);
  }
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_serial_scatter(HashArgs<K> a) {
  zen_dev::pdl_entry();
  HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint64_t z = h->count;
  for (uint64_t i = (uint64_t)blockIdx.x * kHashTile + threadIdx.x; i < z;
       i += (uint64_t)gridDim.x * kHashTile) {
    const uint32_t tile = (uint32_t)(i / kHashTile);
    const uint32_t m = a.meta[i];
    if (meta_depth(m) != 0) continue;
    const uint32_t p = meta_part(m);
    const uint64_t spos = (uint64_t)a.tile_scnt[(uint64_t)p * a.tiles_cap + tile] + meta_srank(m);
    if (spos < h->r2) {
      const uint64_t s = (uint64_t)p * h->stride + h->r1 + spos;
      a.slots[s] = Slot<SlotOf<K>>::make(epoch_word(h->epoch), (uint64_t)a.idx[i] + 1);
      if (a.slot_vals) a.slot_vals[s] = a.val[i];
    }
  }
}

// Sequential replay of partitions that reached the fallback scan, exactly as
// place_index (zen/hashing.hpp:155-179) in ascending key order; the last block
// folds the per-partition histograms into CollisionStats.  One block per
// flagged partition: the block scans the keys in ascending order 256 at a
// time (a ballot collects the partition's keys) and one thread places them in
// order.  Slots only ever fill during the replay, so the smallest vacant
// parallel slot (the fallback scan's answer) never moves backwards: the scan
// resumes from the previous answer instead of from slot 0, and the whole
// replay costs O(keys + r1) instead of O(keys * r1).  The keys come from the
// ascending list (standalone / sparse syncs) or straight from the extraction
// staging, tile by tile (dense syncs).
template <typename K>
__device__ __forceinline__ void fallback_place(const HashArgs<K>& a, SlotOf<K>* base, uint64_t key,
                                               uint64_t r1, uint64_t stride, uint64_t ew,
                                               uint64_t& cursor, uint64_t& fbp, uint32_t& depth,
                                               int64_t& slot) {
  using S = Slot<SlotOf<K>>;
  const uint32_t k = a.fam.k;
  depth = 0;
  slot = -1;
  for (uint32_t t0 = 0; t0 < k && slot < 0; t0 += 4) {  // four probes in flight
    uint64_t c[4];
    SlotOf<K> w[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if (t0 + q < k) {
        c[q] = slot_of(a.fam, key, t0 + q, r1);
        w[q] = base[c[q]];
      }
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if (slot < 0 && t0 + q < k && S::vacant(w[q], ew)) {
        slot = (int64_t)c[q];
        depth = t0 + q + 1;
      }
  }
  if (slot < 0) {
    const uint64_t q = cursor++;
    if (q < stride) {
      slot = (int64_t)q;
    } else {
      while (fbp < r1 && !S::vacant(base[fbp], ew)) ++fbp;
      if (fbp < r1) slot = (int64_t)fbp;
    }
  }
  if (slot >= 0) base[slot] = S::make(ew, key, depth ? depth - 1 : 0u, sizeof(SlotOf<K>) == 4 ? a.fam.db : 0u);
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_fallback(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ K list[kThreads];
  __shared__ uint32_t lpos[kThreads];
  __shared__ uint32_t wcount[kWarps];
  __shared__ uint32_t s_last, s_T;
  __shared__ uint32_t fstat[kMaxK + 1];
  HashHdr* h = a.hdr;
  const uint32_t n = a.fam.n, k = a.fam.k, lane = lane_id(), warp = threadIdx.x >> 5;
  // (early side chain: the scatter's overflow witness may still be pending;
  // an overflowing partition is never flagged -- its load exceeds r1 + r2 --
  // and the overflow fails the whole sync on the host)
  const SideSizes sz = side_sizes(a);
  const bool ok = !sz.bad && (a.xc.early || h->ovf_word == ~0ull) && h->fallback_any;
  const K* st = static_cast<const K*>(a.xc.st_idx);
  for (uint32_t p = blockIdx.x; ok && p < n; p += gridDim.x) {
    if (!a.fallback[p]) continue;
    const uint64_t z = sz.z, r1 = sz.r1, stride = sz.stride;
    const uint64_t ew = epoch_word(h->epoch);
    using S = Slot<SlotOf<K>>;
    SlotOf<K>* base = a.slots + (uint64_t)p * stride;
    for (uint64_t q = threadIdx.x; q < stride; q += kThreads) base[q] = S::kVacant;
    if (threadIdx.x <= k) fstat[threadIdx.x] = 0;
    __syncthreads();
    uint64_t cursor = r1, fbp = 0;
    // one chunk of up to 256 ascending keys: collect partition p's, place in order
    auto chunk = [&](bool valid, K key, uint64_t pos) {
      const bool mine = valid && part_of(a.fam, (uint64_t)key + 1) == p;
      const uint32_t bal = __ballot_sync(0xffffffffu, mine);
      if (lane == 0) wcount[warp] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, total = 0;
      for (int w = 0; w < kWarps; ++w) {
        if (w < (int)warp) before += wcount[w];
        total += wcount[w];
      }
      if (mine) {
        list[before + __popc(bal & lanemask_lt())] = key;
        lpos[before + __popc(bal & lanemask_lt())] = (uint32_t)pos;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (uint32_t e = 0; e < total; ++e) {
          uint32_t depth;
          int64_t slot;
          fallback_place(a, base, (uint64_t)list[e] + 1, r1, stride, ew, cursor, fbp, depth, slot);
          if (!st) {  // the layout dump's depths and slot values
            a.meta[lpos[e]] = pack_meta(p, depth, 0, 0);
            if (slot >= 0 && a.slot_vals) a.slot_vals[(uint64_t)p * stride + slot] = a.val[lpos[e]];
          }
          fstat[depth] += 1;
        }
      }
      __syncthreads();
    };
    if (st) {  // dense sync: the staging, tile by tile in ascending order
      const PushCounts& x = a.xc;
      for (uint32_t t = 0; t < x.ntiles; ++t) {
        if (threadIdx.x < 32) {
          uint32_t c = lane < n ? x.tcnt[(uint64_t)lane * x.ntiles + t] : 0u;
          c = __reduce_add_sync(0xffffffffu, c);
          if (lane == 0) s_T = c;
        }
        __syncthreads();
        const uint32_t T = s_T;
        for (uint32_t c0 = 0; c0 < T; c0 += kThreads) {
          const uint32_t j = c0 + threadIdx.x;
          chunk(j < T, j < T ? st[(uint64_t)t * kExtractTile + j] : (K)0, 0);
        }
        __syncthreads();  // s_T reuse
      }
    } else {
      for (uint64_t c0 = 0; c0 < z; c0 += kThreads) {
        const uint64_t i = c0 + threadIdx.x;
        chunk(i < z, i < z ? a.idx[i] : (K)0, i);
      }
    }
    if (threadIdx.x <= k) a.fb_stats[p * (k + 1) + threadIdx.x] = fstat[threadIdx.x];
    __syncthreads();
    if (sizeof(SlotOf<K>) == 4)  // epoch-free words (BP): leave the partition vacant
      for (uint64_t q = threadIdx.x; q < stride; q += kThreads) base[q] = S::kVacant;
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(&h->fb_done, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x <= k) {  // CollisionStats: serial, depth 1..k
    uint64_t s = 0;
    for (uint32_t p = 0; p < n; ++p)
      s += (a.fallback[p] ? ((volatile uint32_t*)a.fb_stats)[p * (k + 1) + threadIdx.x]
                          : ((volatile uint32_t*)a.stats)[p * (k + 1) + threadIdx.x]);
    a.stats_out[threadIdx.x] = s;
  }
}

// BP side path, after the claims (k_place): the depth histogram from the
// TABLE instead of the keys.  Every parallel slot held in this epoch holds
// exactly one key, whose depth is the first probe t with slot_of(key, t) ==
// the slot -- a hash recomputation, not a random load -- and a key holding no
// slot is serial, so serial_p = load_p - (slots held in p).  One coalesced
// pass over the n*r1 parallel slots replaces k probes per key.  A BP sync
// exposes only CollisionStats (zen/hashing.hpp:259-262), so no serial slot is
// written; when a partition has more serial keys than its r2 serial slots,
// the reference's order-dependent fallback scan (zen/hashing.hpp:170-175)
// changes later placements and the last block flags the partition for the
// exact replay (k_fallback).  Otherwise the last block folds CollisionStats.
template <typename K>
__global__ void __launch_bounds__(kThreads) k_depth_scan(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s_hist[kMaxWorkers * (kMaxK + 1)];
  __shared__ uint32_t s_last;
  HashHdr* h = a.hdr;
  const uint32_t n = a.fam.n, k = a.fam.k, lane = lane_id();
  const SideSizes sz = side_sizes(a);
  const bool ok = !sz.bad;
  const uint64_t r1 = sz.r1, r2 = sz.r2, stride = sz.stride;
  const uint64_t ew = epoch_word(h->epoch);
  for (uint32_t i = threadIdx.x; i < n * (k + 1); i += kThreads) s_hist[i] = 0;
  __syncthreads();
  // grid.y = partition: the parallel region [p*stride, p*stride + r1)
  const uint32_t p = blockIdx.y;
  using W = SlotOf<K>;
  using S = Slot<W>;
  W* region = a.slots + (uint64_t)p * stride;
  const uint32_t db = sizeof(W) == 4 ? a.fam.db : 0u;
  const uint64_t nthr = (uint64_t)gridDim.x * kThreads;
  constexpr int R = 4;  // slots per thread per round, loads issued together
  for (uint64_t c0 = (uint64_t)blockIdx.x * kThreads + (threadIdx.x & ~31u); ok && c0 < r1;
       c0 += nthr * R) {  // warp-uniform trip count (full-mask match_any below)
    W w[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint64_t c = c0 + (uint64_t)j * nthr + lane;
      w[j] = c < r1 ? region[c] : S::kVacant;
    }
    if (sizeof(W) == 4) {  // epoch-free words: vacate what was read for the next sync
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint64_t c = c0 + (uint64_t)j * nthr + lane;
        if (!S::vacant(w[j], ew)) region[c] = S::kVacant;
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint64_t c = c0 + (uint64_t)j * nthr + lane;
      uint32_t d = 0;
      if (!S::vacant(w[j], ew)) {  // held in this sync (c < r1 implied)
        if (db) {  // the claiming probe is in the word
          d = S::probe(w[j], db) + 1;
        } else {
          const uint64_t key = S::key(w[j]);
          uint32_t t = 0;
          while (t + 1 < k && slot_of(a.fam, key, t, r1) != c) ++t;
          d = t + 1;
        }
      }
      const uint32_t g = __match_any_sync(0xffffffffu, d);
      if (d && lane == (uint32_t)(__ffs(g) - 1)) atomicAdd(&s_hist[p * (k + 1) + d], (uint32_t)__popc(g));
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n * (k + 1); i += kThreads)
    if (s_hist[i]) atomicAdd(&a.stats[i], s_hist[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(&h->done, 1u) == gridDim.x * gridDim.y - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < n) {  // serial = keys of p holding no slot
    const uint32_t q = threadIdx.x;
    volatile uint32_t* st = a.stats + q * (k + 1);
    uint32_t held = 0;
    for (uint32_t d = 1; d <= k; ++d) held += st[d];
    const uint32_t load = side_load(a, q);
    const uint32_t serial = load - held;
    st[0] = serial;
    const uint32_t fb = (ok && serial > r2 && (uint64_t)load <= stride) ? 1u : 0u;
    a.fallback[q] = fb;
    if (fb) atomicOr(&h->fallback_any, 1u);
  }
  __syncthreads();
  if (threadIdx.x <= k && !((volatile uint32_t*)&h->fallback_any)[0]) {
    uint64_t sum = 0;
    for (uint32_t q = 0; q < n; ++q) sum += ((volatile uint32_t*)a.stats)[q * (k + 1) + threadIdx.x];
    a.stats_out[threadIdx.x] = sum;
  }
  if (threadIdx.x == 0) h->done = 0;
}

// ----------------------------------------------------------------- utils ----

__global__ void k_partition_of(const uint64_t* __restrict__ idx, uint64_t count, uint64_t pc,
                               uint32_t n, uint32_t* __restrict__ out) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = part_of_seed(pc, n, idx[i] + 1);
}

__global__ void k_u64_to_u32(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                             uint64_t n) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)in[i];
}

__global__ void k_fill_u64(unsigned long long* p, uint64_t n, uint64_t v) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (unsigned)(g < cap ? g : cap);
}

}  // namespace

template <typename K>
void launch_hash_begin(const HashArgs<K>& a, cudaStream_t stream) {
  launch_k(k_hash_begin<K>, 1, 256, 0, stream, a);
  count_launch();
}

template <typename K>
void launch_hash_part(const HashArgs<K>& a, uint32_t n, cudaStream_t stream) {
  const unsigned tiles = (unsigned)std::max<uint64_t>(a.tiles_cap, 1);
  launch_k(k_part<K>, tiles, kThreads, kWarps * n * sizeof(uint32_t), stream, a);
  count_launch();
}

template <typename K>
void launch_hash_critical(const HashArgs<K>& a, uint32_t n, bool part, cudaStream_t stream) {
  const unsigned tiles = (unsigned)std::max<uint64_t>(a.tiles_cap, 1);
  if (part) {  // else fused into the compaction (k_extract_compact_part)
    launch_k(k_part<K>, tiles, kThreads, kWarps * n * sizeof(uint32_t), stream, a);
    count_launch();
  }
  launch_k(k_part_scan<K>, n, 1024, 0, stream, a);
  if (a.dst_table && a.peer)  // NVLink destinations: full-line stores (measured -3 us at n=4;
                             // local stores gain nothing from the reorder)
    launch_k(k_scatter_runs<K>, tiles, kThreads, 0, stream, a);
  else
    launch_k(k_scatter<K>, (tiles + kScatterTiles - 1) / kScatterTiles, kThreads,
             a.dst_table ? 0 : n * sizeof(uint64_t), stream, a);
  for (int i = 0; i < 2; ++i) count_launch();
  if (a.push_hdr) {
    launch_k(k_push_signal<K>, 1, 32, 0, stream, a);
    count_launch();
  }
}

template <typename K>
void launch_hash_side(const HashArgs<K>& a, uint32_t n, bool place, cudaStream_t stream,
                      unsigned ctas_per_sm) {
  const unsigned tiles = (unsigned)std::max<uint64_t>(a.tiles_cap, 1);
  // concurrent with the critical path the grids are capped (2 CTAs per SM) so
  // the side path does not crowd out the critical path's kernels
  const unsigned side = std::min<unsigned>(tiles, 148 * ctas_per_sm);
  if (place) {
    const unsigned bt = a.place_threads ? a.place_threads : kThreads;
    const unsigned g = a.place_grid ? a.place_grid : grid_for(a.cap, kThreads, 148 * ctas_per_sm);
    launch_k(k_place<K>, g, bt, 0, stream, a);
    count_launch();
  }
  launch_k(k_depth<K>, side, kThreads, kWarps * n * sizeof(uint32_t), stream, a);
  launch_k(k_serial_scan<K>, n, 1024, 0, stream, a);
  launch_k(k_serial_scatter<K>, side, kThreads, 0, stream, a);
  launch_k(k_fallback<K>, grid_for(n, 1, 148), kThreads, 0, stream, a);
  for (int i = 0; i < 4; ++i) count_launch();
}

template <typename K>
void launch_hash_side_bp(const HashArgs<K>& a, cudaStream_t stream, unsigned ctas_per_sm,
                         bool place) {
  if (place) {  // sparse syncs: claims over the ascending key list (dense: k_place_tiles)
    launch_k(k_place<K>, grid_for(a.cap, kThreads * 4, 148 * ctas_per_sm), kThreads, 0, stream, a);
    count_launch();
  }
  if (a.xc.inline_hist) {  // the claims kept the histogram: only vacate the memory
    launch_vacate<K>(a, stream);
    launch_k(k_fallback<K>, grid_for(a.fam.n, 1, 148), kThreads, 0, stream, a);
    count_launch();
    return;
  }
  const unsigned gx = std::max(1u, grid_for(a.stride_cap, kThreads * 4, 148 * ctas_per_sm) / a.fam.n);
  launch_k(k_depth_scan<K>, dim3(gx, a.fam.n), kThreads, 0, stream, a);
  // the replay is data dependent: it returns at once unless a partition was flagged
  launch_k(k_fallback<K>, grid_for(a.fam.n, 1, 148), kThreads, 0, stream, a);
  for (int i = 0; i < 2; ++i) count_launch();
}

template <typename K>
void launch_hash(const HashArgs<K>& a, uint32_t n, uint32_t k, cudaStream_t stream) {
  launch_hash_begin<K>(a, stream);
  launch_hash_critical<K>(a, n, true, stream);
  launch_hash_side<K>(a, n, true, stream, 16);
  (void)k;
}

template <typename K>
void launch_push_signal(const HashArgs<K>& a, cudaStream_t stream) {
  launch_k(k_push_signal<K>, 1, 32, 0, stream, a);
  count_launch();
}

#define ZEN_INST(K)                                                                         \
  template void launch_push_signal<K>(const HashArgs<K>&, cudaStream_t);                   \
  template void launch_hash<K>(const HashArgs<K>&, uint32_t, uint32_t, cudaStream_t);       \
  template void launch_hash_begin<K>(const HashArgs<K>&, cudaStream_t);                     \
  template void launch_hash_part<K>(const HashArgs<K>&, uint32_t, cudaStream_t);            \
  template void launch_hash_critical<K>(const HashArgs<K>&, uint32_t, bool, cudaStream_t);        \
  template void launch_hash_side<K>(const HashArgs<K>&, uint32_t, bool, cudaStream_t, unsigned); \
  template void launch_hash_side_bp<K>(const HashArgs<K>&, cudaStream_t, unsigned, bool);
ZEN_INST(uint32_t)
ZEN_INST(uint64_t)
#undef ZEN_INST

void launch_partition_of(const uint64_t* idx, uint64_t count, uint64_t pc, uint32_t n,
                         uint32_t* out, cudaStream_t stream) {
  launch_k(k_partition_of, grid_for(count, 256, 148 * 8), 256, 0, stream, idx, count, pc, n, out);
  count_launch();
}

void launch_u64_to_u32(const uint64_t* in, uint32_t* out, uint64_t n, cudaStream_t stream) {
  launch_k(k_u64_to_u32, grid_for(n, 256, 148 * 8), 256, 0, stream, in, out, n);
  count_launch();
}

void launch_fill_u64(unsigned long long* p, uint64_t n, uint64_t v, cudaStream_t stream) {
  launch_k(k_fill_u64, grid_for(n, 256, 148 * 8), 256, 0, stream, p, n, v);
  count_launch();
}

}  // namespace zen
