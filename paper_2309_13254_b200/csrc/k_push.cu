// k_push.cu -- the dense Balanced-Parallelism data path after extraction:
// hierarchical hash parts + push (zen/hashing.hpp:181-243, zen/schemes.hpp:360-372).
//
// The extraction tiles (k_extract.cu, PART) already stage every non-zero in
// ascending order inside its 8192-element tile window and publish, per h0
// partition, the tile's count plus 32-tile and 1024-tile sums.  One kernel then
// does the rest of the critical path:
//
//  k_push_scatter : one block per 8 extraction tiles.  Its base in partition
//                   p is sum(1024-tile sums before it) + sum(32-tile sums
//                   before it inside its super chunk) + sum(tile counts before
//                   it inside its chunk): three lane-parallel L2 reads and a
//                   warp sum.  The block's entries (its tiles' staging windows
//                   back to back) are then split by h0 in ascending order
//                   (match_any ranks + per-partition warp scans), reordered in
//                   shared memory into per-partition runs and stored straight
//                   into the owners' inboxes (NVLink stores in rank mode), so
//                   each part is ascending exactly as from_pairs sorts it
//                   (zen/tensor.hpp:48-59).  Overflow depends on the loads
//                   only: position r1+r2 of a part is its first dropped key
//                   (zen/hashing.hpp:176-177), the global minimum of which is
//                   the reference's SerialOverflow witness.
//
// The same kernel writes the ascending key list with each key's partition, from
// which the hash-memory placement (the lock-free priority claim + the depth
// pass, k_hash.cu) runs on the side stream, off the critical path.  Before it:
// k_bp_begin (first kernel of a sync: header + counter reset, its latency
// hidden under the extraction's first loads).
#include <cstdlib>

#include "zen_common.cuh"
#include "zen_hash_dev.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kPushThreads = 256;
constexpr int kPushWarps = kPushThreads / 32;
constexpr int kPushPer = 4;                          // entries per thread per round
constexpr int kPushRound = kPushThreads * kPushPer;  // 1024 entries per round
constexpr int kPushTiles = 8;  // extraction tiles per block (divides 32: chunk-aligned)

template <typename K>
__global__ void __launch_bounds__(256) k_bp_begin(HashArgs<K> a) {
  zen_dev::pdl_entry();
  const PushCounts x = a.xc;
  if (blockIdx.x == 0) {
    HashHdr* h = a.hdr;
    const uint32_t n = a.fam.n, k = a.fam.k;
    if (threadIdx.x == 0) {
      const uint32_t epoch = h->epoch, iter = h->iter;
      h->epoch = epoch + 1u;
      h->iter = iter + 1u;
      h->ovf_word = ~0ull;
      h->done = 0;
      h->fb_done = 0;
      h->fallback_any = 0;
      h->bad_index = ~0ull;
      h->work[0] = 0;
      h->work[1] = 0;
      h->work[2] = 0;
    }
    for (uint32_t i = threadIdx.x; i < n * (k + 1); i += blockDim.x) {
      a.stats[i] = 0;
      a.fb_stats[i] = 0;
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      a.fallback[i] = 0;
      a.load[i] = 0;
    }
  }
  // ccnt and scnt are one allocation (host: bp_alloc_worker)
  const uint64_t words = (uint64_t)x.n * (x.nchunk + x.nsup);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (uint64_t)gridDim.x * blockDim.x)
    x.ccnt[i] = 0;
}

// Tile-group prologue shared by the scatter and the claims: the entries of
// the group's kPushTiles extraction tiles (their staging windows back to
// back) and the exclusive prefix over the tiles.
__device__ __forceinline__ uint32_t group_prefix(const PushCounts& x, uint32_t n, uint32_t t0,
                                                 uint32_t* s_tpre) {
  const uint32_t lane = lane_id();
  uint32_t c = 0;
  const uint32_t t = t0 + lane;
  if (lane < (uint32_t)kPushTiles && t < x.ntiles)
    for (uint32_t p = 0; p < n; ++p) c += x.tcnt[(uint64_t)p * x.ntiles + t];
  const uint32_t inc = warp_inclusive_sum(c);
  if (lane < (uint32_t)kPushTiles) s_tpre[lane + 1] = inc;
  if (lane == 0) s_tpre[0] = 0;
  return __shfl_sync(0xffffffffu, inc, kPushTiles - 1);
}

// staging address of group entry e (its tile: s_tpre[i] <= e < s_tpre[i + 1])
__device__ __forceinline__ uint64_t group_src(const uint32_t* s_tpre, uint32_t t0, uint32_t e) {
  uint32_t i = 0;
#pragma unroll
  for (int q = 1; q < kPushTiles; ++q) i += (s_tpre[q] <= e) ? 1u : 0u;
  return (uint64_t)(t0 + i) * kExtractTile + (e - s_tpre[i]);
}

// Persistent blocks take tile groups from a counter (balanced however skewed
// the rows are).  REORDER (peer destinations): each round's entries are
// regrouped in shared memory into per-partition runs, so consecutive threads
// store consecutive positions of one part -- full-line NVLink stores.  Local
// destinations skip the regrouping: a warp's entries of one partition land on
// consecutive positions and L2 merges the partial sectors, so a round needs a
// single block barrier, and the next round's staging loads are issued before
// the current round's stores.
template <typename K, bool REORDER>
__global__ void __launch_bounds__(kPushThreads)
    k_push_scatter(HashArgs<K> a, const K* __restrict__ st_idx, const float* __restrict__ st_val) {
  zen_dev::pdl_entry();
  __shared__ uint64_t s_base[kMaxWorkers];
  __shared__ uint32_t s_run[kMaxWorkers], s_tot[kMaxWorkers];
  __shared__ uint32_t s_off[kMaxWorkers];
  __shared__ uint32_t s_tpre[kPushTiles + 1];
  __shared__ uint32_t s_pre[kPushPer * kPushWarps][kMaxWorkers];  // [sub-round j, warp][p]
  __shared__ uint32_t s_wh[2][kPushWarps][kMaxWorkers];  // per-warp partition counts (2 rounds)
  __shared__ K s_x[REORDER ? kPushRound : 1];
  __shared__ float s_v[REORDER ? kPushRound : 1];
  __shared__ uint8_t s_p[REORDER ? kPushRound : 1];
  __shared__ uint64_t s_z;
  __shared__ uint32_t s_group;
  const PushCounts& x = a.xc;
  const uint32_t n = a.fam.n, lane = lane_id(), warp = threadIdx.x >> 5;
  HashHdr* h = a.hdr;
  if (warp == 0) {  // z = sum of the super-chunk counts (block 0 also publishes the loads)
    uint64_t z = 0;
    for (uint32_t p = 0; p < n; ++p) {
      uint64_t l = 0;
      for (uint32_t i = lane; i < x.nsup; i += 32) l += x.scnt[(uint64_t)p * x.nsup + i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      if (blockIdx.x == 0 && lane == 0) a.load[p] = (uint32_t)l;
      z += l;
    }
    if (lane == 0) s_z = z;
  }
  __syncthreads();
  // z and the worker's sizes r1, r2 (zen/schemes.hpp:363-367), the same in every block
  const uint64_t z = s_z;
  uint64_t r1 = (uint64_t)ceil(h->r1_mult * (double)z / (double)n);
  if (r1 < 1) r1 = 1;
  uint64_t r2 = (uint64_t)ceil(h->r2_ratio * (double)r1);
  if (r2 < 1) r2 = 1;
  const bool bad = z > a.cap || r1 + r2 > a.stride_cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    h->count = z;
    h->r1 = r1;
    h->r2 = r2;
    h->stride = r1 + r2;
    h->ntiles = (uint32_t)((z + kHashTile - 1) / kHashTile);
    if (bad) atomicOr(&h->status, kErrCapacity);
  }
  const uint64_t lim = r1 + r2;
  const uint32_t ngroups = (x.ntiles + kPushTiles - 1) / kPushTiles;
  for (; !bad;) {
    if (threadIdx.x == 0) s_group = atomicAdd(&h->work[0], 1u);
    if (warp == 0 && lane < n) s_run[lane] = 0;
    __syncthreads();
    const uint32_t g = s_group;
    if (g >= ngroups) break;
    const uint32_t t0 = g * kPushTiles;
    uint32_t T = 0;
    if (warp == 1) T = group_prefix(x, n, t0, s_tpre);
    // partition bases of the group's first tile: three levels of counts, lane-parallel
    {
      const uint32_t sup = t0 >> 10, c_lo = sup << 5, c_hi = t0 >> 5, t_lo = c_hi << 5;
      for (uint32_t p = warp; p < n; p += kPushWarps) {
        const uint32_t* sc = x.scnt + (uint64_t)p * x.nsup;
        uint64_t acc = 0;
        if (c_lo + lane < c_hi) acc += x.ccnt[(uint64_t)p * x.nchunk + c_lo + lane];
        if (t_lo + lane < t0) acc += x.tcnt[(uint64_t)p * x.ntiles + t_lo + lane];
        for (uint32_t i = lane; i < sup; i += 32) acc += sc[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          s_base[p] = acc;
          if (a.dst_gbase) a.dst_gbase[p][g] = (uint32_t)acc;  // owner p's range of this group
        }
      }
    }
    __syncthreads();
    T = s_tpre[kPushTiles];
    if (!REORDER && n == 1 && !x.mark) {
      // one partition: the stable split is the identity, entry e of the group
      // goes to base + e -- a plain gather-copy, no ranks, no barriers
      const uint64_t b0 = s_base[0];
      for (uint32_t e0 = threadIdx.x; e0 < T; e0 += kPushRound) {
        K xv[kPushPer];
        float vv[kPushPer];
#pragma unroll
        for (int j = 0; j < kPushPer; ++j) {
          const uint32_t e = e0 + j * kPushThreads;
          if (e < T) {
            const uint64_t src = group_src(s_tpre, t0, e);
            xv[j] = st_idx[src];
            vv[j] = st_val[src];
          }
        }
#pragma unroll
        for (int j = 0; j < kPushPer; ++j) {
          const uint32_t e = e0 + j * kPushThreads;
          const uint64_t pos = b0 + e;
          if (e < T) {
            if (pos < a.dst_cap) {
              a.dst_idx[0][pos] = xv[j];
              a.dst_val[0][pos] = vv[j];
            } else {
              atomicOr(&h->status, kErrCapacity);
            }
            if (pos == lim) atomicMin((unsigned long long*)&h->ovf_word, ((uint64_t)xv[j] + 1) << 16);
          }
        }
      }
      continue;  // the loop head's barrier orders the next group's shared writes
    }
    if (!REORDER) {
      // lane p < n keeps partition p's running offset; rounds are pipelined
      uint32_t run = 0;
      const uint64_t mybase = lane < n ? s_base[lane] : 0ull;
      uint32_t parity = 0;
      K xn[kPushPer];
      float vn[kPushPer];
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const uint32_t e = warp * (32 * kPushPer) + j * 32 + lane;
        if (e < T) {
          const uint64_t src = group_src(s_tpre, t0, e);
          xn[j] = st_idx[src];
          vn[j] = st_val[src];
        }
      }
      for (uint32_t r0 = 0; r0 < T; r0 += kPushRound, parity ^= 1u) {
        K xv[kPushPer];
        float vv[kPushPer];
        uint32_t pv[kPushPer], rk[kPushPer];
#pragma unroll
        for (int j = 0; j < kPushPer; ++j) {
          xv[j] = xn[j];
          vv[j] = vn[j];
          const uint32_t e = r0 + warp * (32 * kPushPer) + j * 32 + lane;
          pv[j] = e < T ? part_of(a.fam, (uint64_t)xv[j] + 1) : 0xFFFFFFFFu;
          const uint32_t en = e + kPushRound;  // next round's entry
          if (en < T) {
            const uint64_t src = group_src(s_tpre, t0, en);
            xn[j] = st_idx[src];
            vn[j] = st_val[src];
          }
        }
        // per-warp stable ranks: a warp's entries are (j, lane)-ascending; the
        // leader of each partition group keeps the warp's running count
        uint32_t* wh = s_wh[parity][warp];
        if (lane < kMaxWorkers) wh[lane] = 0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kPushPer; ++j) {
          const uint32_t gm = __match_any_sync(0xffffffffu, pv[j]);
          const uint32_t leader = __ffs(gm) - 1;
          uint32_t before = 0;
          if (pv[j] != 0xFFFFFFFFu && lane == leader) {
            before = wh[pv[j]];
            wh[pv[j]] = before + __popc(gm);
          }
          rk[j] = __shfl_sync(0xffffffffu, before, leader) + __popc(gm & lanemask_lt());
          __syncwarp();
        }
        __syncthreads();
        // lane p < n: this warp's offset in partition p and the round's total
        uint32_t woff = 0, tot = 0;
        if (lane < n) {
#pragma unroll
          for (int w = 0; w < kPushWarps; ++w) {
            const uint32_t c = s_wh[parity][w][lane];
            woff += (w < (int)warp) ? c : 0u;
            tot += c;
          }
        }
#pragma unroll
        for (int j = 0; j < kPushPer; ++j) {
          const uint32_t p = pv[j];
          const uint64_t b = __shfl_sync(0xffffffffu, mybase + run + woff, p < kMaxWorkers ? p : 0u);
          const uint64_t pos = b + rk[j];
          const bool st = p != 0xFFFFFFFFu && pos < a.dst_cap;
          if (p != 0xFFFFFFFFu) {
            if (st) {
              a.dst_idx[p][pos] = xv[j];
              a.dst_val[p][pos] = vv[j];
            } else {
              atomicOr(&h->status, kErrCapacity);
            }
            if (pos == lim)
              atomicMin((unsigned long long*)&h->ovf_word, (((uint64_t)xv[j] + 1) << 16) | p);
          }
          if (x.mark) {
            // k_agg_mark's work, for servers on this GPU: the entry's rank in
            // I_p (zen/codec.hpp:146-158) sets its bit in this worker's
            // presence row of server p, one atomicOr per (server, word) per
            // warp; the word's first part index (the value base the fold
            // needs) by atomicMin -- the group leader holds the smallest
            uint64_t word = ~0ull;
            uint64_t bit = 0;
            if (st) {
              const uint64_t key = xv[j];
              const OwnWord ow = x.mk_own[p][key >> 6];
              const uint32_t r = ow.prefix + (uint32_t)__popcll(ow.mask & lowmask64(key & 63u));
              word = ((uint64_t)p << 40) | (r >> 6);
              bit = 1ull << (r & 63u);
            }
            const uint32_t g = __match_any_sync(0xffffffffu, word);
            const uint32_t lo = __reduce_or_sync(g, (uint32_t)bit);
            const uint32_t hi = __reduce_or_sync(g, (uint32_t)(bit >> 32));
            if (st && lane == (uint32_t)(__ffs(g) - 1)) {
              const uint64_t row = (uint64_t)a.me * x.mk_nws[p] + (word & ((1ull << 40) - 1));
              atomicOr(x.mk_pw[p] + row, ((unsigned long long)hi << 32) | lo);
              atomicMin(x.mk_pre[p] + row, (uint32_t)pos);
            }
          }
        }
        run += tot;
      }
      continue;  // the loop head's barrier orders the next group's shared writes
    }
    for (uint32_t r0 = 0; r0 < T; r0 += kPushRound) {
      K xv[kPushPer];
      float vv[kPushPer];
      uint32_t pv[kPushPer], rk[kPushPer];
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const uint32_t e = r0 + j * kPushThreads + threadIdx.x;
        pv[j] = 0xFFFFFFFFu;
        if (e < T) {
          const uint64_t src = group_src(s_tpre, t0, e);
          xv[j] = st_idx[src];
          vv[j] = st_val[src];
          pv[j] = part_of(a.fam, (uint64_t)xv[j] + 1);
        }
      }
      for (uint32_t i = threadIdx.x; i < kPushPer * kPushWarps * kMaxWorkers; i += kPushThreads)
        (&s_pre[0][0])[i] = 0;
      __syncthreads();  // s_pre cleared
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const uint32_t e = r0 + j * kPushThreads + threadIdx.x;
        const uint32_t gm = __match_any_sync(0xffffffffu, pv[j]);
        rk[j] = __popc(gm & lanemask_lt());
        if (e < T && lane == (uint32_t)(__ffs(gm) - 1)) s_pre[j * kPushWarps + warp][pv[j]] = __popc(gm);
      }
      __syncthreads();
      // per partition: exclusive scan over the round's (sub-round, warp) rows, in
      // ascending entry order
      for (uint32_t p = warp; p < n; p += kPushWarps) {
        const uint32_t v = s_pre[lane][p];
        const uint32_t inc = warp_inclusive_sum(v);
        s_pre[lane][p] = inc - v;
        if (lane == 31) s_tot[p] = inc;
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t v = lane < n ? s_tot[lane] : 0u;
        const uint32_t inc = warp_inclusive_sum(v);
        if (lane < n) s_off[lane] = inc - v;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const uint32_t e = r0 + j * kPushThreads + threadIdx.x;
        if (e < T) {
          const uint32_t p = pv[j];
          const uint32_t slot = s_off[p] + s_pre[j * kPushWarps + warp][p] + rk[j];
          s_x[slot] = xv[j];
          s_v[slot] = vv[j];
          s_p[slot] = (uint8_t)p;
        }
      }
      __syncthreads();
      const uint32_t cnt = min(T - r0, (uint32_t)kPushRound);
      for (uint32_t sl = threadIdx.x; sl < cnt; sl += kPushThreads) {
        const uint32_t p = s_p[sl];
        const uint64_t pos = s_base[p] + s_run[p] + (sl - s_off[p]);
        const K key = s_x[sl];
        if (pos < a.dst_cap) {
          a.dst_idx[p][pos] = key;
          a.dst_val[p][pos] = s_v[sl];
        } else {
          atomicOr(&h->status, kErrCapacity);
        }
        if (pos == lim)
          atomicMin((unsigned long long*)&h->ovf_word, (((uint64_t)key + 1) << 16) | p);
      }
      __syncthreads();
      if (threadIdx.x < n) s_run[threadIdx.x] += s_tot[threadIdx.x];
    }
  }
  // rank mode: the push signal (k_hash.cu k_push_signal) from the last block
  // to finish -- every block fences its NVLink stores (system scope) before it
  // counts itself done, so the count row and the release of the flag follow
  // every part store of this worker
  if (a.push_hdr && x.fused_signal) {
    __shared__ uint32_t s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_for(a.peer);
      s_last = (atomicAdd(&h->work[2], 1u) == gridDim.x - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {
      fence_for(a.peer);
      const bool cap_ok = !(*(volatile uint32_t*)&h->status & kErrCapacity);
      const uint64_t ovf = *(volatile uint64_t*)&h->ovf_word;
      const uint32_t st = *(volatile uint32_t*)&h->status;
      for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
        PushHdr* ph = a.push_hdr[s];
        ph->nnz = z;
        ph->ovf_word = ovf;
        ph->status = st;
        for (uint32_t q = 0; q < n; ++q) ph->counts[q] = cap_ok ? a.load[q] : 0u;
      }
      __syncthreads();
      fence_for(a.peer);
      for (uint32_t s = threadIdx.x; s < n; s += blockDim.x)
        st_release_sys(&a.push_hdr[s]->flag, (unsigned long long)h->iter);
    }
  }
}

// Side path, the hash-memory placement of the dense data path: the lock-free
// priority claim (zen_hash_dev.cuh place_keys) of every
// staged key, read straight from the extraction staging -- the claims' outcome
// does not depend on the order keys claim in, so no ascending key list is
// built.  Persistent blocks take tile groups from a counter.
template <typename K>
__global__ void __launch_bounds__(kPushThreads) k_place_tiles(HashArgs<K> a) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s_tpre[kPushTiles + 1];
  __shared__ uint32_t s_group;
  const PushCounts& x = a.xc;
  HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const K* st = static_cast<const K*>(x.st_idx);
  const uint32_t n = a.fam.n, warp = threadIdx.x >> 5;
  const uint64_t r1 = h->r1, stride = h->stride;
  const uint64_t ew = epoch_word(h->epoch);
  const uint32_t ngroups = (x.ntiles + kPushTiles - 1) / kPushTiles;
  constexpr int KPT = 4;
  for (;;) {
    if (threadIdx.x == 0) s_group = atomicAdd(&h->work[1], 1u);
    __syncthreads();
    const uint32_t g = s_group;
    if (g >= ngroups) break;
    const uint32_t t0 = g * kPushTiles;
    if (warp == 0) group_prefix(x, n, t0, s_tpre);
    __syncthreads();
    const uint32_t T = s_tpre[kPushTiles];
    for (uint32_t e0 = threadIdx.x; e0 < T; e0 += kPushThreads * KPT) {
      uint64_t key[KPT];
      uint32_t part[KPT], nv = 0;
#pragma unroll
      for (int j = 0; j < KPT; ++j) {
        const uint32_t e = e0 + j * kPushThreads;  // valid entries form a prefix in j
        key[j] = e < T ? (uint64_t)st[group_src(s_tpre, t0, e)] + 1 : 0ull;
        part[j] = e < T ? part_of(a.fam, key[j]) : 0u;
        nv += e < T ? 1u : 0u;
      }
      place_keys<KPT>(a.fam, a.slots, key, part, nv, r1, stride, ew);
    }
    __syncthreads();  // s_tpre / s_group reuse
  }
}

// Two-phase claims (default): every entry of a 1024-entry round makes its
// FIRST claim (four atomics in flight per thread); only the entries that were
// rejected or displaced a key -- a minority at the reference's load factor --
// are compacted into a shared-memory list and continue (place_from), so a
// warp no longer runs until the longest chain among its 128 keys ends with
// most lanes idle.  Same protocol, same matching (schedule-independent).
template <typename K, bool HIST>
__global__ void __launch_bounds__(kPushThreads) k_place_tiles2(HashArgs<K> a) {
  zen_dev::pdl_entry();
  using W = SlotOf<K>;
  using S = Slot<W>;
  __shared__ uint32_t s_tpre[kPushTiles + 1];
  __shared__ uint32_t s_group, s_np[2];  // pending counts, alternating rounds
  __shared__ uint32_t s_key[kPushRound];  // pending: key (index + 1)
  __shared__ uint16_t s_pt[kPushRound];   // pending: partition << 5 | next probe
  __shared__ int s_hist[kMaxWorkers * (kMaxK + 1)];  // inline depth histogram (this block)
  __shared__ uint32_t s_last;
  const PushCounts& x = a.xc;
  HashHdr* h = a.hdr;
  const SideSizes sz = side_sizes(a);
  if (sz.bad) return;
  // HIST: the variant with the counter code (the counters themselves are on
  // only with x.inline_hist); !HIST: the lean variant (48 vs 59 registers)
  int* hist = (HIST && x.inline_hist) ? s_hist : nullptr;
  if (hist)
    for (uint32_t i = threadIdx.x; i < kMaxWorkers * (kMaxK + 1); i += kPushThreads) s_hist[i] = 0;
  const K* st = static_cast<const K*>(x.st_idx);
  const uint32_t n = a.fam.n, k = a.fam.k, warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t db = sizeof(W) == 4 ? a.fam.db : 0u;
  const uint64_t r1 = sz.r1, stride = sz.stride;
  const uint64_t ew = epoch_word(h->epoch);
  const uint32_t ngroups = (x.ntiles + kPushTiles - 1) / kPushTiles;
  if (threadIdx.x == 0) s_np[0] = s_np[1] = 0;
  uint32_t par = 0;
  for (;;) {
    if (threadIdx.x == 0) s_group = atomicAdd(&h->work[1], 1u);
    __syncthreads();
    const uint32_t g = s_group;
    if (g >= ngroups) break;
    const uint32_t t0 = g * kPushTiles;
    if (warp == 0) group_prefix(x, n, t0, s_tpre);
    __syncthreads();
    const uint32_t T = s_tpre[kPushTiles];
    for (uint32_t e0 = 0; e0 < T; e0 += kPushRound) {
      uint64_t key[kPushPer];
      uint32_t part[kPushPer], c[kPushPer];
      W old[kPushPer];
      bool v[kPushPer];
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const uint32_t e = e0 + j * kPushThreads + threadIdx.x;
        v[j] = e < T;
        key[j] = v[j] ? (uint64_t)st[group_src(s_tpre, t0, e)] + 1 : 0ull;
      }
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        part[j] = (v[j] && n > 1) ? part_of(a.fam, key[j]) : 0u;
        if (v[j]) {
          c[j] = (uint32_t)slot_of(a.fam, key[j], 0, r1);
          old[j] = atomicMin(a.slots + (uint64_t)part[j] * stride + c[j], S::make(ew, key[j], 0, db));
        }
      }
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        uint64_t nk = key[j];
        uint32_t nt = 1;
        bool go = v[j] && !S::vacant(old[j], ew);
        if (hist && v[j] && !go) atomicAdd(&hist[part[j] * (k + 1) + 1], 1);  // took c at probe 0
        if (go) {
          const uint64_t ok = S::key(old[j], db);
          if (ok > key[j]) {  // displaced a larger key: it resumes after its first c
            nk = ok;
            uint32_t f = 0;
            if (db)
              f = S::probe(old[j], db);
            else
              while (f < k && slot_of(a.fam, ok, f, r1) != c[j]) ++f;
            nt = f + 1;
            if (hist) {
              atomicAdd(&hist[part[j] * (k + 1) + 1], 1);
              atomicAdd(&hist[part[j] * (k + 1) + f + 1], -1);
            }
          }
          go = nt < k;  // else: ends serial
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, go);
        uint32_t b = 0;
        if (bal && lane == 0) b = atomicAdd(&s_np[par], (uint32_t)__popc(bal));
        b = __shfl_sync(0xffffffffu, b, 0) + __popc(bal & lanemask_lt());
        if (go) {
          s_key[b] = (uint32_t)nk;
          s_pt[b] = (uint16_t)((part[j] << 5) | nt);
        }
      }
      __syncthreads();
      const uint32_t np = s_np[par];
      if (threadIdx.x == 0) s_np[par ^ 1] = 0;  // the next round's (its pushes follow a barrier)
      for (uint32_t i0 = 0; i0 < np; i0 += 2 * kPushThreads) {
        uint64_t cur[2];
        uint32_t t[2], pp[2], nv = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t i = i0 + j * kPushThreads + threadIdx.x;  // valid items: a prefix in j
          cur[j] = i < np ? s_key[i] : 0ull;
          const uint32_t q = i < np ? s_pt[i] : 0u;
          pp[j] = q >> 5;
          t[j] = q & 31u;
          nv += i < np ? 1u : 0u;
        }
        place_from<2>(a.fam, a.slots, cur, t, pp, nv, r1, stride, ew, hist);
      }
      __syncthreads();  // the list is consumed
      par ^= 1;
    }
    __syncthreads();  // s_tpre / s_group / s_np reuse
  }
  if (!hist) return;
  // inline histogram: this block's net counts, then the last block turns the
  // totals into CollisionStats and the fallback flags (k_depth_scan's job)
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n * (k + 1); i += kPushThreads)
    if (s_hist[i]) atomicAdd(&a.stats[i], (uint32_t)s_hist[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(&h->done, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < n) {  // serial = keys of p holding no slot
    const uint32_t q = threadIdx.x;
    volatile uint32_t* stq = a.stats + q * (k + 1);
    uint32_t held = 0;
    for (uint32_t d = 1; d <= k; ++d) held += stq[d];
    const uint32_t load = side_load(a, q);
    const uint32_t serial = load - held;
    stq[0] = serial;
    const uint32_t fb = (serial > sz.r2 && (uint64_t)load <= sz.stride) ? 1u : 0u;
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

// inline-histogram side chain: vacate the parallel regions the claims used
template <typename K>
__global__ void __launch_bounds__(256) k_vacate(HashArgs<K> a) {
  zen_dev::pdl_entry();
  using W = SlotOf<K>;
  const SideSizes sz = side_sizes(a);
  if (sz.bad) return;
  // per partition, no division per word; 16-byte stores over the aligned middle
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr uint32_t kPer = 16 / sizeof(W);  // words per 16-byte store
  for (uint32_t p = 0; p < a.fam.n; ++p) {
    W* base = a.slots + (uint64_t)p * sz.stride;
    const uint64_t mis = ((16 - (reinterpret_cast<uintptr_t>(base) & 15)) & 15) / sizeof(W);
    const uint64_t head = mis < sz.r1 ? mis : sz.r1;
    const uint64_t nvec = (sz.r1 - head) / kPer;
    for (uint64_t c = t; c < head; c += nth) base[c] = Slot<W>::kVacant;
    uint4* v = reinterpret_cast<uint4*>(base + head);
    for (uint64_t c = t; c < nvec; c += nth) v[c] = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (uint64_t c = head + nvec * kPer + t; c < sz.r1; c += nth) base[c] = Slot<W>::kVacant;
  }
}

}  // namespace

template <typename K>
void launch_bp_begin(const HashArgs<K>& a, cudaStream_t stream) {
  const uint64_t words = (uint64_t)a.xc.n * (a.xc.nchunk + a.xc.nsup);
  const unsigned g = (unsigned)std::min<uint64_t>(std::max<uint64_t>((words + 1023) / 1024, 1), 148);
  launch_k(k_bp_begin<K>, g, 256, 0, stream, a);
  count_launch();
}

template <typename K>
void launch_push_scatter(const HashArgs<K>& a, const ExtractWs<K>& ws, cudaStream_t stream) {
  launch_k(a.xc.reorder ? k_push_scatter<K, true> : k_push_scatter<K, false>,
           a.xc.scatter_grid,
           kPushThreads, 0, stream, a, (const K*)ws.st_idx, (const float*)ws.st_val);
  count_launch();
}

template <typename K>
void launch_vacate(const HashArgs<K>& a, cudaStream_t stream) {
  const uint64_t cells = (uint64_t)a.fam.n * a.stride_cap;
  launch_k(k_vacate<K>, (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((cells + 1023) / 1024, 148 * 8)),
           256, 0, stream, a);
  count_launch();
}

template <typename K>
void launch_place_tiles(const HashArgs<K>& a, cudaStream_t stream, unsigned ctas_per_sm) {
  const unsigned groups = (a.xc.ntiles + kPushTiles - 1) / kPushTiles;
  static const bool v1 = std::getenv("ZEN_PLACE_V1") != nullptr;  // (A/B: one-phase claims)
  // Rank mode takes the lean variant; local mode the counter-carrying one even
  // with the counters off: measured (profiles/r07/place_variant_ab.txt), the
  // lean one is faster with peers (N=2 0.1427 -> 0.1388 ms, N=4 0.1715 ->
  // 0.1682) but slower beside the one-worker aggregate (N=1 0.0938 -> 0.0965
  // ms: more claim blocks fit next to the union and crowd it)
  launch_k(v1 ? k_place_tiles<K>
              : (a.xc.inline_hist || !a.peer) ? k_place_tiles2<K, true> : k_place_tiles2<K, false>,
           std::max(1u, std::min(groups, 148u * ctas_per_sm)), kPushThreads, 0, stream, a);
  count_launch();
}

// resident blocks of the persistent scatter (the whole grid in one wave)
template <typename K>
unsigned push_scatter_grid(bool peer, uint32_t ntiles) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, peer ? k_push_scatter<K, true> : k_push_scatter<K, false>, kPushThreads, 0);
  // (the REORDER variant needs more shared memory: its occupancy bounds both)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned groups = (ntiles + kPushTiles - 1) / kPushTiles;
  return std::max(1u, std::min(groups, (unsigned)(std::max(per_sm, 1) * sms)));
}

#define ZEN_INST(K)                                                                          \
  template void launch_bp_begin<K>(const HashArgs<K>&, cudaStream_t);                        \
  template void launch_push_scatter<K>(const HashArgs<K>&, const ExtractWs<K>&, cudaStream_t); \
  template void launch_place_tiles<K>(const HashArgs<K>&, cudaStream_t, unsigned);            \
  template void launch_vacate<K>(const HashArgs<K>&, cudaStream_t);                            \
  template unsigned push_scatter_grid<K>(bool, uint32_t);
ZEN_INST(uint32_t)
#undef ZEN_INST
template void launch_vacate<uint64_t>(const HashArgs<uint64_t>&, cudaStream_t);

}  // namespace zen
