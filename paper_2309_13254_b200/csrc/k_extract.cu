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
//  2. k_extract_scan: one block scans the per-tile counts.
//  3. k_extract_compact: one warp per tile moves its staged entries to the
//     final ascending position.  In the BP pipeline the same pass runs the
//     hierarchical hash's priority claim for every key it moves (fused place).
#include "zen_common.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kThreads = 256;
constexpr int kIters = 4;  // 8-float units per lane
constexpr int kUnit = 8;

template <typename K>
__global__ void __launch_bounds__(kThreads, 4)
    k_extract_tiles(const float* __restrict__ dense, uint64_t m, K* __restrict__ st_idx,
                    float* __restrict__ st_val, uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t s_warp_tot[kThreads / 32];
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
  uint32_t nzbits = 0;  // 8 bits per iteration
#pragma unroll
  for (int j = 0; j < kIters; ++j)
#pragma unroll
    for (int c = 0; c < kUnit; ++c) nzbits |= (uint32_t)(v[j].v[c] != 0.0f) << (kUnit * j + c);
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
  __syncthreads();
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

__global__ void __launch_bounds__(1024) k_extract_scan(uint32_t* __restrict__ tile_cnt,
                                                       uint32_t ntiles, uint64_t* d_count,
                                                       uint64_t capacity, uint32_t* err,
                                                       uint64_t* tile_base) {
  __shared__ uint64_t sscan[33];
  uint64_t carry = 0;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x) {
    const uint32_t t = b + threadIdx.x;
    const uint64_t v = t < ntiles ? tile_cnt[t] : 0u;
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum(v, sscan, &tot);
    if (t < ntiles) tile_base[t] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *d_count = carry;
    if (carry > capacity) atomicOr(err, kErrCapacity);
  }
}

__device__ __forceinline__ uint64_t epoch_word(uint32_t epoch) {
  return (uint64_t)(0xFFFFFFu - (epoch & 0xFFFFFFu)) << kKeyBits;
}

// Priority claim of one key (see k_hash.cu): smallest key wins every slot.
__device__ __forceinline__ void place_key(const DevFamily& fam, unsigned long long* slots,
                                          uint64_t key, uint64_t r1, uint64_t stride, uint64_t ew) {
  const uint32_t p = part_of(fam, key);
  unsigned long long* base = slots + (uint64_t)p * stride;
  uint64_t cur = key;
  uint32_t t = 0;
  const uint32_t k = fam.k;
  while (true) {
    const uint64_t c = slot_of(fam, cur, t, r1);
    const unsigned long long old = atomicMin(base + c, (unsigned long long)(ew | cur));
    if (old > (ew | kKeyMask)) break;
    const uint64_t ok = old & kKeyMask;
    if (ok > cur) {
      cur = ok;
      uint32_t f = 0;
      while (f < k && slot_of(fam, cur, f, r1) != c) ++f;
      t = f + 1;
    } else {
      ++t;
    }
    if (t >= k) break;
  }
}

// one warp per extraction tile; optionally fuses the hash placement
template <typename K, bool PLACE>
__global__ void __launch_bounds__(256)
    k_extract_compact(const K* __restrict__ st_idx, const float* __restrict__ st_val,
                      const uint32_t* __restrict__ tile_cnt, const uint64_t* __restrict__ tile_base,
                      uint32_t ntiles, K* __restrict__ out_idx, float* __restrict__ out_val,
                      uint64_t capacity, DevFamily fam, HashHdr* hdr,
                      unsigned long long* slots) {
  const uint32_t tile = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tile >= ntiles) return;
  uint64_t r1 = 0, stride = 0, ew = 0;
  bool place = PLACE;
  if (PLACE) {
    place = !(hdr->status & kErrCapacity);
    r1 = hdr->r1;
    stride = hdr->stride;
    ew = epoch_word(hdr->epoch);
  }
  const uint32_t cnt = tile_cnt[tile];
  const uint64_t base = tile_base[tile];
  const uint64_t src = (uint64_t)tile * kExtractTile;
  for (uint32_t j = lane_id(); j < cnt; j += 32) {
    const K x = st_idx[src + j];
    const float v = st_val[src + j];
    if (base + j < capacity) {
      out_idx[base + j] = x;
      out_val[base + j] = v;
      if (PLACE && place) place_key(fam, slots, (uint64_t)x + 1, r1, stride, ew);
    }
  }
}

}  // namespace

template <typename K>
void launch_extract(const float* dense, uint64_t m, const ExtractWs<K>& ws, K* out_idx,
                    float* out_val, uint64_t* d_count, uint64_t capacity, uint32_t* d_status_bits,
                    cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  k_extract_tiles<K><<<ntiles, kThreads, 0, stream>>>(dense, m, ws.st_idx, ws.st_val, ws.tile_cnt);
  k_extract_scan<<<1, 1024, 0, stream>>>(ws.tile_cnt, ntiles, d_count, capacity, d_status_bits,
                                         ws.tile_base);
  k_extract_compact<K, false><<<(ntiles + 7) / 8, 256, 0, stream>>>(
      ws.st_idx, ws.st_val, ws.tile_cnt, ws.tile_base, ntiles, out_idx, out_val, capacity,
      DevFamily{}, nullptr, nullptr);
  for (int i = 0; i < 3; ++i) count_launch();
}

template <typename K>
void launch_extract_tiles(const float* dense, uint64_t m, const ExtractWs<K>& ws,
                          uint64_t* d_count, uint64_t capacity, uint32_t* d_status_bits,
                          cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  k_extract_tiles<K><<<ntiles, kThreads, 0, stream>>>(dense, m, ws.st_idx, ws.st_val, ws.tile_cnt);
  k_extract_scan<<<1, 1024, 0, stream>>>(ws.tile_cnt, ntiles, d_count, capacity, d_status_bits,
                                         ws.tile_base);
  count_launch();
  count_launch();
}

template <typename K>
void launch_extract_compact_place(uint64_t m, const ExtractWs<K>& ws, K* out_idx, float* out_val,
                                  uint64_t capacity, const DevFamily& fam, HashHdr* hdr,
                                  unsigned long long* slots, cudaStream_t stream) {
  const uint32_t ntiles = (uint32_t)((m + kExtractTile - 1) / kExtractTile);
  k_extract_compact<K, true><<<(ntiles + 7) / 8, 256, 0, stream>>>(
      ws.st_idx, ws.st_val, ws.tile_cnt, ws.tile_base, ntiles, out_idx, out_val, capacity, fam,
      hdr, slots);
  count_launch();
}

#define ZEN_INST(K)                                                                              \
  template void launch_extract<K>(const float*, uint64_t, const ExtractWs<K>&, K*, float*,      \
                                  uint64_t*, uint64_t, uint32_t*, cudaStream_t);                 \
  template void launch_extract_tiles<K>(const float*, uint64_t, const ExtractWs<K>&, uint64_t*, \
                                        uint64_t, uint32_t*, cudaStream_t);                      \
  template void launch_extract_compact_place<K>(uint64_t, const ExtractWs<K>&, K*, float*,      \
                                                uint64_t, const DevFamily&, HashHdr*,           \
                                                unsigned long long*, cudaStream_t);
ZEN_INST(uint32_t)
ZEN_INST(uint64_t)
#undef ZEN_INST

}  // namespace zen
