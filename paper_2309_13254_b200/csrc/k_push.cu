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
// The same kernel writes the ascending key list with each key's partition and
// runs the hash-memory placement (the lock-free priority claim, k_hash.cu) of
// the keys it holds in registers, so only the depth pass (k_depth_bp:
// CollisionStats, fallback detection) is left for the side stream.  Before it:
// k_bp_begin (first kernel of a sync: header + counter reset, its latency
// hidden under the extraction's first loads).
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

template <typename K>
__global__ void __launch_bounds__(kPushThreads)
    k_push_scatter(HashArgs<K> a, const K* __restrict__ st_idx, const float* __restrict__ st_val) {
  zen_dev::pdl_entry();
  __shared__ uint64_t s_base[kMaxWorkers];
  __shared__ uint32_t s_run[kMaxWorkers], s_tot[kMaxWorkers];
  __shared__ uint32_t s_off[kMaxWorkers];
  __shared__ uint32_t s_tpre[kPushTiles + 1];  // entry prefix over the block's tiles
  __shared__ uint32_t s_pre[kPushPer * kPushWarps][kMaxWorkers];  // [sub-round j, warp][p]
  __shared__ K s_x[kPushRound];
  __shared__ float s_v[kPushRound];
  __shared__ uint8_t s_p[kPushRound];
  __shared__ uint64_t s_z;
  const PushCounts& x = a.xc;
  const uint32_t n = a.fam.n, lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t t0 = blockIdx.x * kPushTiles;
  HashHdr* h = a.hdr;
  if (warp == 0) {
    const uint64_t l = lane < n ? (uint64_t)a.load[lane] : 0ull;
    uint64_t z = l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) s_z = z;
    if (lane < n) s_run[lane] = 0;
  } else if (warp == 1) {  // entries per tile of this block
    uint32_t c = 0;
    const uint32_t t = t0 + lane;
    if (lane < (uint32_t)kPushTiles && t < x.ntiles)
      for (uint32_t p = 0; p < n; ++p) c += x.tcnt[(uint64_t)p * x.ntiles + t];
    const uint32_t inc = warp_inclusive_sum(c);
    if (lane < (uint32_t)kPushTiles) s_tpre[lane + 1] = inc;
    if (lane == 0) s_tpre[0] = 0;
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
  const uint32_t T = s_tpre[kPushTiles];
  if (bad || T == 0) return;
  // partition bases of the block's first tile: three levels of counts, lane-parallel
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
      if (lane == 0) s_base[p] = acc;
    }
  }
  __syncthreads();
  if (threadIdx.x < (uint32_t)kPushTiles && t0 + threadIdx.x < x.ntiles) {
    uint64_t b = 0;
    for (uint32_t p = 0; p < n; ++p) b += s_base[p];
    x.tbase[t0 + threadIdx.x] = b + s_tpre[threadIdx.x];  // the side path's compaction offsets
  }
  const uint64_t lim = r1 + r2;
  uint64_t bstart = 0;  // the block's first ascending position (its first tile's tbase)
  for (uint32_t p = 0; p < n; ++p) bstart += s_base[p];
  const uint64_t ew = epoch_word(h->epoch);
  K* keys = const_cast<K*>(a.idx);
  for (uint32_t r0 = 0; r0 < T; r0 += kPushRound) {
    for (uint32_t i = threadIdx.x; i < kPushPer * kPushWarps * kMaxWorkers; i += kPushThreads)
      (&s_pre[0][0])[i] = 0;
    K xv[kPushPer];
    float vv[kPushPer];
    uint32_t pv[kPushPer], rk[kPushPer];
#pragma unroll
    for (int j = 0; j < kPushPer; ++j) {
      const uint32_t e = r0 + j * kPushThreads + threadIdx.x;
      if (e < T) {
        uint32_t i = 0;  // the entry's tile: s_tpre[i] <= e < s_tpre[i + 1]
#pragma unroll
        for (int q = 1; q < kPushTiles; ++q) i += (s_tpre[q] <= e) ? 1u : 0u;
        const uint64_t src = (uint64_t)(t0 + i) * kExtractTile + (e - s_tpre[i]);
        xv[j] = st_idx[src];
        vv[j] = st_val[src];
      }
    }
    __syncthreads();  // s_pre cleared
#pragma unroll
    for (int j = 0; j < kPushPer; ++j) {
      const uint32_t e = r0 + j * kPushThreads + threadIdx.x;
      pv[j] = e < T ? part_of(a.fam, (uint64_t)xv[j] + 1) : 0xFFFFFFFFu;
      if (e < T) {  // the ascending key list + partitions the side path's depth pass reads
        keys[bstart + e] = xv[j];
        a.pmeta[bstart + e] = pv[j];
      }
      const uint32_t g = __match_any_sync(0xffffffffu, pv[j]);
      rk[j] = __popc(g & lanemask_lt());
      if (e < T && lane == (uint32_t)(__ffs(g) - 1)) s_pre[j * kPushWarps + warp][pv[j]] = __popc(g);
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
    // hierarchical hash placement of this round's keys: the lock-free priority
    // claim (k_hash.cu, zen_hash_dev.cuh place_keys) -- every key of the sync
    // has claimed once this kernel ends, which the depth pass needs
    if (a.slots) {
      uint64_t kk[kPushPer];
      uint32_t nv = 0;
#pragma unroll
      for (int j = 0; j < kPushPer; ++j) {
        const bool v = r0 + j * kPushThreads + threadIdx.x < T;  // valid j form a prefix
        kk[j] = v ? (uint64_t)xv[j] + 1 : 0ull;
        nv += v ? 1u : 0u;
      }
      place_keys<kPushPer>(a.fam, a.slots, kk, pv, nv, r1, lim, ew);
    }
    __syncthreads();
    if (threadIdx.x < n) s_run[threadIdx.x] += s_tot[threadIdx.x];
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
  launch_k(k_push_scatter<K>, (a.xc.ntiles + kPushTiles - 1) / kPushTiles, kPushThreads, 0, stream,
           a, (const K*)ws.st_idx,
           (const float*)ws.st_val);
  count_launch();
}

#define ZEN_INST(K)                                                                          \
  template void launch_bp_begin<K>(const HashArgs<K>&, cudaStream_t);                        \
  template void launch_push_scatter<K>(const HashArgs<K>&, const ExtractWs<K>&, cudaStream_t);
ZEN_INST(uint32_t)
#undef ZEN_INST

}  // namespace zen
