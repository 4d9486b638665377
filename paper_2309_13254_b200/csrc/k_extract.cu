// k_extract.cu -- non-zero extraction (zen::to_sparse, zen/tensor.hpp:94-104)
//
// Dense fp32 gradient -> COO (ascending index, v != 0.0f: -0.0 dropped, NaN
// kept) in ONE pass over HBM.  HBM-bound: 4 B read per element, 4+sizeof(K)
// B written per non-zero.
//
// Layout: a tile is 8192 floats = 1024 eight-float units; warp w of the
// 256-thread block owns the contiguous units [w*128, w*128+128) and walks them
// in 4 coalesced 1 KiB iterations of 256-bit loads (ld.v8, L1 no-allocate, L2
// evict-first).  Each lane keeps its 32 floats in registers, a warp ballot
// skips all-zero iterations (zero embedding rows cost nothing beyond the
// read), per-iteration warp scans give each lane its in-order offset, and the
// tile's global offset comes from a decoupled look-back, so the output is
// written once, in order, without a second pass.
#include "zen_common.cuh"

namespace zen {
namespace {

using namespace zen_dev;

constexpr int kThreads = 256;
constexpr int kIters = 4;  // 8-float units per lane
constexpr int kUnit = 8;

template <typename K>
__global__ void __launch_bounds__(kThreads) k_extract(const float* __restrict__ dense, uint64_t m,
                                                      K* __restrict__ out_idx,
                                                      float* __restrict__ out_val,
                                                      uint64_t* d_count, uint64_t capacity,
                                                      unsigned long long* lb_status,
                                                      LookbackCtl* ctl, uint32_t* err,
                                                      uint32_t ntiles) {
  __shared__ uint32_t s_ticket;
  __shared__ uint32_t s_warp_tot[kThreads / 32];
  __shared__ uint64_t s_warp_base[kThreads / 32];
  __shared__ uint64_t s_tile_base;
  const uint32_t tag = *(volatile uint32_t*)&ctl->tag;
  const uint32_t tile = take_ticket(ctl, &s_ticket);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t unit0 = (uint64_t)tile * (kExtractTile / kUnit) + (uint64_t)warp * 128 + lane;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(dense) & 31u) == 0);

  f8 v[kIters];
#pragma unroll
  for (int j = 0; j < kIters; ++j) {
    const uint64_t e = (unit0 + (uint64_t)j * 32) * kUnit;
    if (vec_ok && e + kUnit <= m) {
      v[j] = ld_stream_f8(dense + e);
    } else {
#pragma unroll
      for (int c = 0; c < kUnit; ++c) v[j].v[c] = e + c < m ? dense[e + c] : 0.0f;
    }
  }
  uint32_t nzbits = 0;  // 8 bits per iteration
#pragma unroll
  for (int j = 0; j < kIters; ++j)
#pragma unroll
    for (int c = 0; c < kUnit; ++c) nzbits |= (uint32_t)(v[j].v[c] != 0.0f) << (kUnit * j + c);
  // per-iteration in-warp offsets (ascending element order: iteration, lane, component)
  uint32_t off[kIters];
  uint32_t wrun = 0;
  if (__ballot_sync(0xffffffffu, nzbits != 0)) {
#pragma unroll
    for (int j = 0; j < kIters; ++j) {
      const uint32_t c = __popc((nzbits >> (kUnit * j)) & 0xFFu);
      if (__ballot_sync(0xffffffffu, c != 0)) {
        const uint32_t inc = warp_inclusive_sum(c);
        off[j] = wrun + inc - c;
        wrun += __shfl_sync(0xffffffffu, inc, 31);
      } else {
        off[j] = wrun;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kIters; ++j) off[j] = 0;
  }
  if (lane == 0) s_warp_tot[warp] = wrun;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < kThreads / 32 ? s_warp_tot[lane] : 0u;
    const uint32_t inc = warp_inclusive_sum(t);
    const uint64_t total = __shfl_sync(0xffffffffu, inc, 31);
    if (lane < kThreads / 32) s_warp_base[lane] = inc - t;
    const uint64_t base = lookback_warp(lb_status, tile, tag, total);
    if (lane == 0) {
      s_tile_base = base;
      if (tile == ntiles - 1) {
        *d_count = base + total;
        if (base + total > capacity) atomicOr(err, kErrCapacity);
      }
    }
  }
  __syncthreads();
  if (nzbits) {
    uint64_t pos0 = s_tile_base + s_warp_base[warp];
#pragma unroll
    for (int j = 0; j < kIters; ++j) {
      uint32_t b = (nzbits >> (kUnit * j)) & 0xFFu;
      uint64_t pos = pos0 + off[j];
      const uint64_t e = (unit0 + (uint64_t)j * 32) * kUnit;
#pragma unroll
      for (int c = 0; c < kUnit; ++c) {
        if ((b >> c) & 1u) {
          if (pos < capacity) {
            out_idx[pos] = (K)(e + c);
            out_val[pos] = v[j].v[c];
          }
          ++pos;
        }
      }
    }
  }
  finish_tile(ctl, ntiles);
}

}  // namespace

extern void count_launch();

template <typename K>
void launch_extract(const float* dense, uint64_t m, K* out_idx, float* out_val, uint64_t* d_count,
                    uint64_t capacity, unsigned long long* status, LookbackCtl* ctl,
                    uint32_t* d_status_bits, cudaStream_t stream) {
  const uint64_t ntiles = (m + kExtractTile - 1) / kExtractTile;
  k_extract<K><<<(unsigned)ntiles, kThreads, 0, stream>>>(dense, m, out_idx, out_val, d_count,
                                                          capacity, status, ctl, d_status_bits,
                                                          (uint32_t)ntiles);
  count_launch();
}

template void launch_extract<uint32_t>(const float*, uint64_t, uint32_t*, float*, uint64_t*,
                                       uint64_t, unsigned long long*, LookbackCtl*, uint32_t*,
                                       cudaStream_t);
template void launch_extract<uint64_t>(const float*, uint64_t, uint64_t*, float*, uint64_t*,
                                       uint64_t, unsigned long long*, LookbackCtl*, uint32_t*,
                                       cudaStream_t);

}  // namespace zen
