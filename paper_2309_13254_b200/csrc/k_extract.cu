// k_extract.cu -- non-zero extraction (zen::to_sparse, zen/tensor.hpp:94-104)
//
// Dense fp32 gradient -> COO (ascending index, v != 0.0f: -0.0 dropped, NaN
// kept).  HBM-bound: 4 B read per element.
//
// Three look-back-free phases (a decoupled look-back serialises ~G/32 L2
// round trips per wave of G resident tiles, which capped the one-pass version
// at ~26% of HBM bandwidth):
//  1. k_extract_tiles: a tile is 8192 floats; warp w owns 1 KiB-contiguous
//     units and walks them in 4 iterations of 256-bit streaming loads (ld.v8,
//     L1 no-allocate, L2 evict-first); a warp ballot skips all-zero units (zero
//     embedding rows cost only their read); per-iteration warp scans give each
//     lane its in-order offset, and the tile's non-zeros land tile-locally in a
//     staging area.  Fully parallel: every block is independent.
//  2. k_extract_scan: one block scans the per-tile counts (in the BP pipeline
//     the same block then starts the hash run: r1/r2 from the count).
//  3. k_extract_compact: one thread per output position finds its tile by a
//     binary search over the tile bases (balanced however skewed the tiles
//     are) and moves the entry to its final ascending position.  In the BP
//     pipeline the same thread runs the hierarchical hash's priority claim for
//     the key it moves (fused place).
#include "zen_common.cuh"
#include "zen_hash_dev.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kThreads = 256;
constexpr int kIters = 4;  // 8-float units per lane
constexpr int kUnit = 8;

// element predicates of the tile pass: to_sparse keeps v != 0.0f
// (-0.0 dropped, NaN kept; zen/tensor.hpp:94-104); the top-k selection keeps
// non-zero magnitudes at or above a threshold key (k_topk.cu)
struct NonZero {
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ bool operator()(float v) const { return v != 0.0f; }
};
struct MagnitudeAtLeast {
  const uint32_t* key_ptr;  // threshold computed on the device (k_topk.cu)
  uint32_t key;             // |v| as IEEE bits (sign cleared): monotone in |v|
  __device__ __forceinline__ void init() { key = *key_ptr; }
  __device__ __forceinline__ bool operator()(float v) const {
    const uint32_t k = __float_as_uint(v) & 0x7fffffffu;
    return k >= key && k != 0u;
  }
};

// PART (the dense BP data path): each tile also computes the h0 partition of
// its non-zeros (partition_of, zen/hashing.hpp:85-88) and publishes its
// per-partition counts at three levels (tile, 32-tile chunk, 1024-tile super
// chunk; k_push.cu), so the push scatter finds every tile's partition bases
// without a scan kernel.  The dense loads are issued before the PDL wait: the
// gradient does not come from the predecessor (the per-sync begin kernel).
template <typename K, typename Pred = NonZero, bool PART = false>
__global__ void __launch_bounds__(kThreads, 4)
    k_extract_tiles(const float* __restrict__ dense, uint64_t m, K* __restrict__ st_idx,
                    float* __restrict__ st_val, uint32_t* __restrict__ tile_cnt,
                    Pred pred = Pred(), PushCounts pc = PushCounts{},
                    uint32_t* __restrict__ load = nullptr) {
  if (!PART) zen_dev::pdl_entry();
  pred.init();
  __shared__ uint32_t s_warp_tot[kThreads / 32];
  __shared__ uint32_t s_wpc[PART ? kThreads / 32 : 1][PART ? kMaxWorkers : 1];
  const uint32_t tile = blockIdx.x;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t unit0 = (uint64_t)tile * (kExtractTile / kUnit) + (uint64_t)warp * 128 + lane;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(dense) & 31u) == 0) &&
                      ((uint64_t)(tile + 1) * kExtractTile <= m);
  f8 v[kIters];
  if (vec_ok) {
#pragma unroll
    for (int j = 0; j < kIters; ++j) v[j] = ld_stream_f8(dense + (unit0 + (uint64_t)j * 32) * kUnit);
  } else {
#pragma unroll
    for (int j = 0; j < kIters; ++j) {
      const uint64_t e = (unit0 + (uint64_t)j * 32) * kUnit;
#pragma unroll
      for (int c = 0; c < kUnit; ++c) v[j].v[c] = e + c < m ? dense[e + c] : 0.0f;
    }
  }
  if (PART) zen_dev::pdl_entry();
  uint32_t nzbits = 0;  // 8 bits per iteration
#pragma unroll
  for (int j = 0; j < kIters; ++j)
#pragma unroll
    for (int c = 0; c < kUnit; ++c) nzbits |= (uint32_t)pred(v[j].v[c]) << (kUnit * j + c);
  // in-warp offsets in ascending element order (iteration, lane, component)
  uint32_t off[kIters];
  uint32_t wrun = 0;
  if (__ballot_sync(0xffffffffu, nzbits != 0)) {
#pragma unroll
    for (int j = 0; j < kIters; ++j) {
      const uint32_t c = __popc((nzbits >> (kUnit * j)) & 0xFFu);
      const uint32_t inc = warp_inclusive_sum(c);
      off[j] = wrun + inc - c;
      wrun += __shfl_sync(0xffffffffu, inc, 31);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kIters; ++j) off[j] = 0;
  }
  if (lane == 0) s_warp_tot[warp] = wrun;
  if (PART) {
    // the h0 partition counts: 8-bit per-partition counters per lane
    // (<= 32 non-zeros per lane), one warp reduction per partition, summed
    // across warps after the block's one barrier
    uint64_t c0 = 0, c1 = 0;
    const bool any = __ballot_sync(0xffffffffu, nzbits != 0) != 0;
    if (any && pc.n == 1) {
      c0 = __popc(nzbits);  // map_to_range(h, 1) == 0: one partition, no hash
    } else if (any) {
      for (uint32_t b = nzbits; b; b &= b - 1) {
        const uint32_t q = __ffs(b) - 1;
        const uint64_t e = (unit0 + (uint64_t)(q >> 3) * 32) * kUnit + (q & 7u);
        const uint32_t p = part_of_seed(pc.pc, pc.n, e + 1);
        if (p < 8) c0 += 1ull << (8 * p); else c1 += 1ull << (8 * (p - 8));
      }
    }
    for (uint32_t p = 0; p < pc.n; ++p) {
      const uint32_t f = (uint32_t)(((p < 8 ? c0 : c1) >> (8 * (p & 7))) & 0xFFu);
      const uint32_t t = any ? __reduce_add_sync(0xffffffffu, f) : 0u;
      if (lane == 0) s_wpc[warp][p] = t;
    }
  }
  __syncthreads();
  if (PART) {
    if (threadIdx.x < pc.n) {
      const uint32_t p = threadIdx.x;
      uint32_t c = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) c += s_wpc[w][p];
      pc.tcnt[(uint64_t)p * pc.ntiles + tile] = c;
      if (c) {  // (no per-partition total here: thousands of tiles on one word
                // would serialise at its L2 slice; the scatter sums the super chunks)
        atomicAdd(pc.ccnt + (uint64_t)p * pc.nchunk + (tile >> 5), c);
        atomicAdd(pc.scnt + (uint64_t)p * pc.nsup + (tile >> 10), c);
      }
    }
  }
  uint32_t wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const uint32_t t = s_warp_tot[w];
    wbase += (w < (int)warp) ? t : 0u;
    total += t;
  }
  if (threadIdx.x == 0) tile_cnt[tile] = total;
  if (nzbits) {
    const uint64_t base = (uint64_t)tile * kExtractTile + wbase;
#pragma unroll
    for (int j = 0; j < kIters; ++j) {
      const uint32_t b = (nzbits >> (kUnit * j)) & 0xFFu;
      if (!b) continue;
      uint64_t pos = base + off[j];
      const uint64_t e = (unit0 + (uint64_t)j * 32) * kUnit;
#pragma unroll
      for (int c = 0; c < kUnit; ++c) {
        if ((b >> c) & 1u) {
          st_idx[pos] = (K)(e + c);
          st_val[pos] = v[j].v[c];
          ++pos;
        }
      }
    }
  }
}

// Exclusive scan of the tile counts -> tile_base; and for every compaction
// block b (output positions [256b, 256b+256)) the tile holding position 256b
// (blk_tile[b]), so the compaction needs no binary search over all tiles.
template <typename K, bool BEGIN>
__global__ void __launch_bounds__(1024) k_extract_scan(uint32_t* __restrict__ tile_cnt,
                                                       uint32_t ntiles, uint64_t* d_count,
                                                       uint64_t capacity, uint32_t* err,
                                                       uint64_t* tile_base,
                                                       uint32_t* __restrict__ blk_tile,
                                                       uint64_t nblk, HashArgs<K> ha) {
  zen_dev::pdl_entry();
  __shared__ uint64_t sscan[33];
  constexpr int E = 8;
  uint64_t carry = 0;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x * E) {
    const uint32_t t0 = b + threadIdx.x * E;
    uint32_t v[E];
    if (t0 + E <= ntiles) {  // tile_cnt is 256-B aligned, t0 % 8 == 0
      const uint4 a0 = reinterpret_cast<const uint4*>(tile_cnt + t0)[0];
      const uint4 a1 = reinterpret_cast<const uint4*>(tile_cnt + t0)[1];
      v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w;
      v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = (t0 + e < ntiles) ? tile_cnt[t0 + e] : 0u;
    }
    uint64_t local = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) local += v[e];
    uint64_t tot;
    uint64_t ex = carry + block_exclusive_sum(local, sscan, &tot);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (t0 + e < ntiles) {
        tile_base[t0 + e] = ex;
        // blocks whose first position falls in this tile
        const uint64_t end = ex + v[e];
        for (uint64_t b = (ex + 255) / 256; b * 256 < end && b < nblk; ++b)
          blk_tile[b] = t0 + e;
      }
      ex += v[e];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *d_count = carry;
    if (carry > capacity) atomicOr(err, kErrCapacity);
  }
  if (BEGIN) {
    __syncthreads();
    hash_begin_body(ha);
  }
}

// one thread per output position (balanced)
template <typename K>
__global__ void __launch_bounds__(256)
    k_extract_compact(const K* __restrict__ st_idx, const float* __restrict__ st_val,
                      const uint64_t* __restrict__ tile_base, uint32_t ntiles,
                      const uint64_t* d_count, K* __restrict__ out_idx,
                      float* __restrict__ out_val, uint64_t capacity,
                      const uint32_t* __restrict__ blk_tile) {
  zen_dev::pdl_entry();
  const uint64_t z = *d_count;
  const uint64_t b0 = (uint64_t)blockIdx.x * blockDim.x;
  const uint64_t i = b0 + threadIdx.x;
  const uint64_t zc = min(z, capacity);
  if (i >= zc) return;
  // tiles of the block's positions: [blk_tile[b], blk_tile[b+1]]
  uint32_t lo = blk_tile[blockIdx.x];
  uint32_t hi = (b0 + blockDim.x < zc) ? blk_tile[blockIdx.x + 1] + 1 : ntiles;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (tile_base[mid] <= i) lo = mid; else hi = mid;
  }
  const uint64_t src = (uint64_t)lo * kExtractTile + (i - tile_base[lo]);
  out_idx[i] = st_idx[src];
  out_val[i] = st_val[src];
}

// BP pipeline: compaction fused with the data path's partition pass
// (k_hash.cu k_part): each block handles kCompactTiles consecutive 256-key
// hash tiles, one key per thread per tile, with every tile's loads issued
// before any is used (the per-key work is a chain of dependent loads:
// block->tile map, tile base, staged entry), then per tile: h0 partition,
// the key's stable rank among the tile's same-partition keys and the
// per-(partition, tile) counts.
constexpr int kCompactTiles = 4;

template <typename K>
__global__ void __launch_bounds__(256, 4)
    k_extract_compact_part(const K* __restrict__ st_idx, const float* __restrict__ st_val,
                           const uint64_t* __restrict__ tile_base, uint32_t ntiles,
                           const uint32_t* __restrict__ blk_tile, HashArgs<K> a) {
  zen_dev::pdl_entry();
  extern __shared__ uint32_t wc[];  // [kCompactTiles][8 warps][n] counts -> prefixes
  const HashHdr* h = a.hdr;
  if (h->status & kErrCapacity) return;
  const uint64_t z = h->count;
  const uint32_t tile0 = blockIdx.x * kCompactTiles;
  if ((uint64_t)tile0 * kHashTile >= z) return;
  const uint32_t n = a.fam.n, lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t q = threadIdx.x; q < kCompactTiles * 8 * n; q += blockDim.x) wc[q] = 0;
  uint32_t p[kCompactTiles];
  K x[kCompactTiles];
  float v[kCompactTiles];
  bool valid[kCompactTiles];
#pragma unroll
  for (int j = 0; j < kCompactTiles; ++j) {
    const uint32_t tile = tile0 + j;
    const uint64_t b0 = (uint64_t)tile * kHashTile;
    const uint64_t i = b0 + threadIdx.x;
    valid[j] = i < z;
    p[j] = 0xFFFFFFFFu;
    if (valid[j]) {
      uint32_t lo = blk_tile[tile];
      uint32_t hi = (b0 + kHashTile < z) ? blk_tile[tile + 1] + 1 : ntiles;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tile_base[mid] <= i) lo = mid; else hi = mid;
      }
      const uint64_t src = (uint64_t)lo * kExtractTile + (i - tile_base[lo]);
      x[j] = st_idx[src];
      v[j] = st_val[src];
    }
  }
#pragma unroll
  for (int j = 0; j < kCompactTiles; ++j) {
    const uint64_t i = (uint64_t)(tile0 + j) * kHashTile + threadIdx.x;
    if (valid[j]) {
      const_cast<K*>(a.idx)[i] = x[j];  // the worker's compacted keys (HashArgs input)
      const_cast<float*>(a.val)[i] = v[j];
      p[j] = part_of(a.fam, (uint64_t)x[j] + 1);
    }
  }
  __syncthreads();  // wc cleared
  uint32_t wr[kCompactTiles];
#pragma unroll
  for (int j = 0; j < kCompactTiles; ++j) {
    const uint32_t g = __match_any_sync(0xffffffffu, p[j]);
    wr[j] = __popc(g & lanemask_lt());
    if (valid[j] && lane == (uint32_t)(__ffs(g) - 1)) wc[(j * 8 + warp) * n + p[j]] = __popc(g);
  }
  __syncthreads();
  for (uint32_t jq = threadIdx.x; jq < kCompactTiles * n; jq += blockDim.x) {
    const uint32_t j = jq / n, q = jq - j * n, tile = tile0 + j;
    uint32_t acc = 0;
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = wc[(j * 8 + w) * n + q];
      wc[(j * 8 + w) * n + q] = acc;
      acc += t;
    }
    if (tile < a.tiles_cap) a.tile_cnt[(uint64_t)q * a.tiles_cap + tile] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kCompactTiles; ++j) {
    const uint64_t i = (uint64_t)(tile0 + j) * kHashTile + threadIdx.x;
    if (valid[j]) a.pmeta[i] = p[j] | ((wc[(j * 8 + warp) * n + p[j]] + wr[j]) << 16);
  }
}

}  // namespace

inline unsigned blocks_for(uint64_t n) { return (unsigned)std::max<uint64_t>((n + 255) / 256, 1); }

template <typename K>
void launch_extract(const float* dense, uint64_t m, const ExtractWs<K>& ws, K* out_idx,
                    float* out_val, uint64_t* d_count, uint64_t capacity, uint32_t* d_status_bits,
                    cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  launch_k(k_extract_tiles<K, NonZero>, ntiles, kThreads, 0, stream, dense, m, ws.st_idx,
           ws.st_val, ws.tile_cnt, NonZero(), PushCounts{}, (uint32_t*)nullptr);
  launch_k(k_extract_scan<K, false>, 1, 1024, 0, stream, ws.tile_cnt, ntiles, d_count, capacity,
           d_status_bits, ws.tile_base, ws.blk_tile, ws.nblk, HashArgs<K>{});
  launch_k(k_extract_compact<K>, blocks_for(std::min<uint64_t>(capacity, m)), 256, 0, stream,
           ws.st_idx, ws.st_val, ws.tile_base, ntiles, d_count, out_idx, out_val, capacity,
           ws.blk_tile);
  for (int i = 0; i < 3; ++i) count_launch();
}

template <typename K>
void launch_extract_tiles(const float* dense, uint64_t m, const ExtractWs<K>& ws,
                          cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  launch_k(k_extract_tiles<K, NonZero>, ntiles, kThreads, 0, stream, dense, m, ws.st_idx,
           ws.st_val, ws.tile_cnt, NonZero(), PushCounts{}, (uint32_t*)nullptr);
  count_launch();
}

template <typename K>
void launch_extract_scan_begin(uint64_t m, const ExtractWs<K>& ws, const HashArgs<K>& ha,
                               uint64_t capacity, cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  launch_k(k_extract_scan<K, true>, 1, 1024, 0, stream, ws.tile_cnt, ntiles, &ha.hdr->count,
           capacity, &ha.hdr->status, ws.tile_base, ws.blk_tile, ws.nblk, ha);
  count_launch();
}

template <typename K>
void launch_extract_compact_part(uint64_t m, const ExtractWs<K>& ws, const HashArgs<K>& a,
                                 uint32_t n, cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  const uint64_t blocks = (std::max<uint64_t>(a.tiles_cap, 1) + kCompactTiles - 1) / kCompactTiles;
  launch_k(k_extract_compact_part<K>, (unsigned)blocks, 256,
           kCompactTiles * 8 * n * sizeof(uint32_t), stream, ws.st_idx, ws.st_val, ws.tile_base,
           ntiles, ws.blk_tile, a);
  count_launch();
}

// dense BP data path: staging + h0 partition counts (k_push.cu consumes them)
template <typename K>
void launch_extract_tiles_part(const float* dense, uint64_t m, const ExtractWs<K>& ws,
                               const HashArgs<K>& a, cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  launch_k(k_extract_tiles<K, NonZero, true>, ntiles, kThreads, 0, stream, dense, m, ws.st_idx,
           ws.st_val, ws.tile_cnt, NonZero(), a.xc, a.load);
  count_launch();
}

// top-k: stage the non-zero elements with |v| at or above the threshold key
void launch_select_tiles(const float* dense, uint64_t m, const ExtractWs<uint32_t>& ws,
                         const uint32_t* key, cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  launch_k(k_extract_tiles<uint32_t, MagnitudeAtLeast>, ntiles, kThreads, 0, stream, dense, m,
           ws.st_idx, ws.st_val, ws.tile_cnt, MagnitudeAtLeast{key, 0u}, PushCounts{},
           (uint32_t*)nullptr);
  count_launch();
}

#define ZEN_INST(K)                                                                              \
  template void launch_extract<K>(const float*, uint64_t, const ExtractWs<K>&, K*, float*,      \
                                  uint64_t*, uint64_t, uint32_t*, cudaStream_t);                 \
  template void launch_extract_tiles<K>(const float*, uint64_t, const ExtractWs<K>&,           \
                                        cudaStream_t);                                           \
  template void launch_extract_tiles_part<K>(const float*, uint64_t, const ExtractWs<K>&,      \
                                             const HashArgs<K>&, cudaStream_t);                  \
  template void launch_extract_scan_begin<K>(uint64_t, const ExtractWs<K>&, const HashArgs<K>&, \
                                             uint64_t, cudaStream_t);                            \
  template void launch_extract_compact_part<K>(uint64_t, const ExtractWs<K>&, const HashArgs<K>&, \
                                               uint32_t, cudaStream_t);
ZEN_INST(uint32_t)
ZEN_INST(uint64_t)
#undef ZEN_INST

}  // namespace zen
