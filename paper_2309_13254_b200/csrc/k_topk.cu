// k_topk.cu -- zen::sparsify_topk (zen/workload.hpp:157-178) on sm_100a:
// keep the ceil(fraction * M) largest-magnitude entries of a dense fp32
// gradient, ties broken toward the lower index, exact zeros dropped, output
// ascending.  Bit-exact with the reference's partial_sort order.
//
// The magnitude key is the IEEE bit pattern with the sign cleared, which is
// monotone in |v| for every non-NaN value.  (The reference's comparator is not
// a strict weak order on NaN; here NaN magnitudes rank above +inf.)
//
// Radix select in three digit levels, [31:21] [20:10] [9:0]:
//   hist1   full pass over the dense input, 2048-bin histogram of the top digit
//   select  one block: the digit of the k-th largest key; the bucket's lower
//           bound becomes the staging threshold
//   tiles   full pass (the extraction tile kernel with predicate
//           |v| >= bucket floor, non-zero): every kept entry plus the rest of
//           the threshold bucket staged tile-locally in index order
//   hist2/3 over the staged entries only (a warp per tile), each followed by a
//           select -> threshold key T and the number r of T-ties to keep (the
//           r lowest-indexed ones)
//   ties    a warp per tile: the tile's T-ties and entries above T
//   scan    one block: per tile, ties before it -> entries it keeps -> base
//   compact a warp per tile: > T entries, plus ties while the global tie
//           rank is below r, written in ascending index order.
// Two HBM passes over the dense input in all (an earlier version collected
// the bucket with a second full pass before the tile pass: three); everything
// else touches the staged entries only.
#include "zen_common.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kBins = 2048;
constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7fffffffu; }

// Level-1 histogram: 32-byte streaming loads, warp-aggregated shared atomics
__global__ void __launch_bounds__(kThreads, 4) k_topk_hist1(const float* __restrict__ dense,
                                                         uint64_t m, uint32_t* __restrict__ hist) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sh[kBins];
  for (int i = threadIdx.x; i < kBins; i += kThreads) sh[i] = 0;
  __syncthreads();
  const uint64_t nvec = m / 8;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(dense) & 31u) == 0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  // kU independent 32-byte loads in flight per thread before any binning
  // (one load per iteration left the pass at ~55% of HBM bandwidth)
  constexpr int kU = 4;
  uint32_t run_bin = 0, run_cnt = 0;  // warp-uniform
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kU; base < (vec_ok ? nvec : 0);
       base += stride * kU) {  // warp-uniform trip count
    f8 v[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const uint64_t u = base + (uint64_t)j * kThreads + threadIdx.x;
      if (u < nvec) v[j] = ld_stream_f8(dense + u * 8);
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const uint64_t u = base + (uint64_t)j * kThreads + threadIdx.x;
      // fast path: all 8 x 32 keys of this warp-wide load in one bin (a run of
      // zeros) -- one vote instead of eight
      const uint32_t f0 = mag_key(v[j].v[0]) >> 21;
      bool same = u < nvec;
#pragma unroll
      for (int c = 1; c < 8; ++c) same &= (mag_key(v[j].v[c]) >> 21) == f0;
      const uint32_t w0 = __shfl_sync(0xffffffffu, f0, 0);
      if (__all_sync(0xffffffffu, same && f0 == w0)) {
        if (w0 == run_bin) {
          run_cnt += 256;
        } else {
          if (lane_id() == 0 && run_cnt) atomicAdd(&sh[run_bin], run_cnt);
          run_bin = w0;
          run_cnt = 256;
        }
        continue;
      }
      // otherwise straight to the shared histogram: a per-element warp vote
      // here left a dense layer's pass instruction-bound (67% issue-active)
      if (same) {  // this lane's 8 keys share a bin (e.g. zeros next to a live row)
        atomicAdd(&sh[f0], 8u);
      } else if (u < nvec) {
#pragma unroll
        for (int c = 0; c < 8; ++c) atomicAdd(&sh[mag_key(v[j].v[c]) >> 21], 1u);
      }
    }
  }
  if (lane_id() == 0 && run_cnt) atomicAdd(&sh[run_bin], run_cnt);
  const uint64_t tail0 = vec_ok ? nvec * 8 : 0;
  for (uint64_t i = tail0 + (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < m; i += stride)
    atomicAdd(&sh[mag_key(dense[i]) >> 21], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kThreads)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

struct TopkState {
  uint32_t prefix;  // key bits fixed so far
  uint32_t k;       // rank (1-based) still to find among keys matching the prefix
  uint64_t above;   // keys strictly above the current bucket
  uint32_t T;       // final threshold key
  uint32_t r;       // ties of T to keep
  uint32_t ncand;   // unused (the level-2 candidate list of the three-pass version)
  uint32_t nsel;    // |output| before zero dropping is accounted (set by the scan)
};

// per-call state + histogram reset as a kernel (graph-capturable, keeps the
// programmatic-launch chain; no host buffer outlives the call)
__global__ void __launch_bounds__(256) k_topk_init(TopkState* st, uint32_t keep,
                                                   uint32_t* __restrict__ hist) {
  zen_dev::pdl_entry();
  if (threadIdx.x == 0) *st = TopkState{0u, keep, 0ull, 0u, 0u, 0u, 0u};
  for (uint32_t i = threadIdx.x; i < (uint32_t)kBins; i += blockDim.x) hist[i] = 0;
}

// one block: the bucket of the k-th largest key among hist[0..kBins); the
// histogram is cleared for the next level
__global__ void __launch_bounds__(1024) k_topk_select(uint32_t* __restrict__ hist, int shift,
                                                      int digit_bits, TopkState* st, int last) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sscan[33];
  __shared__ uint32_t s_bin, s_above;
  constexpr int E = kBins / 1024;
  const uint32_t k = st->k;
  if (threadIdx.x == 0) s_bin = 0xFFFFFFFFu;  // ordered by the scan's barriers
  // suffix sums from the top bin down: thread t owns bins [kBins-1-E*t-E+1 .. kBins-1-E*t]
  uint32_t c[E], local = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    c[e] = hist[kBins - 1 - (threadIdx.x * E + e)];
    local += c[e];
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum(local, sscan, &tot);
  uint32_t run = ex;  // keys in bins above this thread's first bin
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t bin = kBins - 1 - (threadIdx.x * E + e);
    if (run < k && run + c[e] >= k) {
      s_bin = bin;
      s_above = run;
    }
    run += c[e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    // levels 2 and 3 count staged (non-zero) keys only: a rank beyond them
    // lies among the zeros of bucket 0, so the digit is 0 and T ends at 0
    // (every non-zero kept)
    const bool found = s_bin != 0xFFFFFFFFu;
    const uint32_t bin = found ? s_bin : 0u, above = found ? s_above : tot;
    st->prefix |= bin << shift;
    st->above += above;
    st->k = k - above;
    st->T = st->prefix;  // level 1: the staging floor; last level: the threshold
    if (last) st->r = st->k;  // ties of T that rank inside the top `keep`
  }
  (void)digit_bits;
}

// Levels 2 and 3 over the tile-staged entries (a warp per tile): keys whose
// higher digits equal the prefix so far feed the next digit's histogram
__global__ void __launch_bounds__(kThreads) k_topk_hist_staged(
    const float* __restrict__ st_val, const uint32_t* __restrict__ tile_cnt, uint32_t ntiles,
    const TopkState* st, uint32_t* __restrict__ hist, int shift) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sh[kBins];
  for (int i = threadIdx.x; i < kBins; i += kThreads) sh[i] = 0;
  __syncthreads();
  const int hi = shift == 0 ? 10 : 21;  // bits above the digit: [31:21] or [31:10]
  const uint32_t want = st->prefix >> hi, lane = lane_id(), mask = (1u << (hi - shift)) - 1;
  const uint32_t nwarps = gridDim.x * (kThreads / 32);
  for (uint32_t tile = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); tile < ntiles;
       tile += nwarps) {
    const uint32_t n = tile_cnt[tile];
    const float* v = st_val + (uint64_t)tile * kExtractTile;
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t key = mag_key(v[i]);
      if ((key >> hi) == want) atomicAdd(&sh[(key >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kThreads)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// per tile: ties (key == T) and entries above T among the staged candidates
// (the staged set also holds the threshold bucket's entries below T);
// tile_ties[0, ntiles) = ties, tile_ties[ntiles, 2 ntiles) = above
__global__ void __launch_bounds__(kThreads) k_topk_ties(const float* __restrict__ st_val,
                                                        const uint32_t* __restrict__ tile_cnt,
                                                        uint32_t ntiles, const TopkState* st,
                                                        uint32_t* __restrict__ tile_ties) {
  zen_dev::pdl_entry();
  // a warp per tile: a tile stages ~1-2% of its 8192 elements
  const uint32_t tile = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (tile >= ntiles) return;
  const uint32_t n = tile_cnt[tile], T = st->T;
  uint32_t c = 0, g = 0;
  for (uint32_t i = lane_id(); i < n; i += 32) {
    const uint32_t key = mag_key(st_val[(uint64_t)tile * kExtractTile + i]);
    c += key == T ? 1u : 0u;
    g += key > T ? 1u : 0u;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  g = __reduce_add_sync(0xffffffffu, g);
  if (lane_id() == 0) {
    tile_ties[tile] = c;
    tile_ties[ntiles + tile] = g;
  }
}

// one block over the tiles: ties before each tile -> the tile's kept entries
// (all > T plus the ties whose global rank is below r) -> output base
__global__ void __launch_bounds__(1024) k_topk_scan(const uint32_t* __restrict__ tile_cnt,
                                                    const uint32_t* __restrict__ tile_ties,
                                                    uint32_t ntiles, TopkState* st,
                                                    uint64_t* __restrict__ tie_base,
                                                    uint64_t* __restrict__ out_base,
                                                    uint64_t* out_count) {
  zen_dev::pdl_entry();
  __shared__ uint64_t sscan[33];
  const uint64_t r = st->T ? st->r : 0;  // T = 0: the ties are zeros, dropped
  // one scan of packed (ties << 32 | above-T) counts (both totals stay below
  // m < 2^32): the first r ties in index order are kept, so a tile's output
  // base is above_before + min(r, ties_before)
  uint64_t carry = 0;
  constexpr int E = 8;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x * E) {
    const uint32_t t0 = b + threadIdx.x * E;
    uint64_t pk[E], lsum = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool in = t0 + e < ntiles;
      pk[e] = in ? ((uint64_t)tile_ties[t0 + e] << 32 | tile_ties[ntiles + t0 + e]) : 0;
      lsum += pk[e];
    }
    uint64_t tot;
    uint64_t ex = carry + block_exclusive_sum(lsum, sscan, &tot);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (t0 + e < ntiles) {
        const uint64_t tb = ex >> 32;
        tie_base[t0 + e] = tb;
        out_base[t0 + e] = (ex & 0xffffffffull) + (tb < r ? tb : r);
      }
      ex += pk[e];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const uint64_t tb = carry >> 32;
    *out_count = (carry & 0xffffffffull) + (tb < r ? tb : r);
  }
}

// a warp per tile: stable selection of the staged candidates (a tile stages
// ~1-2% of its 8192 elements, so a block per tile idled most of its lanes)
__global__ void __launch_bounds__(kThreads) k_topk_compact(
    const uint32_t* __restrict__ st_idx, const float* __restrict__ st_val,
    const uint32_t* __restrict__ tile_cnt, uint32_t ntiles, const uint64_t* __restrict__ tie_base,
    const uint64_t* __restrict__ out_base, const TopkState* st, uint64_t* __restrict__ out_idx,
    float* __restrict__ out_val, uint64_t cap) {
  zen_dev::pdl_entry();
  const uint32_t tile = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (tile >= ntiles) return;
  const uint32_t n = tile_cnt[tile], T = st->T;
  const uint64_t r = T ? st->r : 0;
  uint64_t tb = tie_base[tile], ob = out_base[tile];
  const uint32_t lt = lanemask_lt();
  for (uint32_t c0 = 0; c0 < n; c0 += 32) {  // warp-uniform trip count
    const uint32_t i = c0 + lane_id();
    const bool in = i < n;
    const uint64_t src = (uint64_t)tile * kExtractTile + i;
    const float v = in ? st_val[src] : 0.0f;
    const uint32_t key = mag_key(v);
    const bool tie = in && key == T;
    const uint32_t tbal = __ballot_sync(0xffffffffu, tie);
    const bool keep = in && (key > T || (tie && tb + __popc(tbal & lt) < r));
    const uint32_t kbal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const uint64_t pos = ob + __popc(kbal & lt);
      if (pos < cap) {
        out_idx[pos] = st_idx[src];
        out_val[pos] = v;
      }
    }
    tb += __popc(tbal);
    ob += __popc(kbal);
  }
}

inline unsigned pass_grid(uint64_t m) {  // hist1: 4 resident CTAs per SM (55 registers)
  const uint64_t g = (m / 8 + kThreads - 1) / kThreads;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148 * 4));
}

}  // namespace

size_t topk_state_bytes() { return sizeof(TopkState); }
size_t topk_threshold_offset() { return offsetof(TopkState, T); }

// level 1 of the radix select: state, histogram, staging floor on `s`
void launch_topk_select(const float* dense, uint64_t m, uint64_t keep, void* state_v,
                        uint32_t* hist, cudaStream_t s) {
  TopkState* st = static_cast<TopkState*>(state_v);
  launch_k(k_topk_init, 1, 256, 0, s, st, (uint32_t)keep, hist);
  launch_k(k_topk_hist1, pass_grid(m), kThreads, 0, s, dense, m, hist);
  launch_k(k_topk_select, 1, 1024, 0, s, hist, 21, 11, st, 0);
  for (int i = 0; i < 3; ++i) count_launch();
}

// after the tile pass staged the >= T candidates (launch_select_tiles)
void launch_topk_finish(const ExtractWs<uint32_t>& ws, uint32_t ntiles, void* state_v,
                        uint32_t* hist, uint32_t* tile_ties, uint64_t* tie_base, uint64_t* out_base,
                        uint64_t* out_count, uint64_t* out_idx, float* out_val, uint64_t cap,
                        cudaStream_t s) {
  TopkState* st = static_cast<TopkState*>(state_v);
  const unsigned hgrid = std::max(1u, std::min(148u * 8, (ntiles + 7) / 8));
  launch_k(k_topk_hist_staged, hgrid, kThreads, 0, s, ws.st_val, ws.tile_cnt, ntiles, st, hist,
           10);
  launch_k(k_topk_select, 1, 1024, 0, s, hist, 10, 11, st, 0);
  launch_k(k_topk_hist_staged, hgrid, kThreads, 0, s, ws.st_val, ws.tile_cnt, ntiles, st, hist,
           0);
  launch_k(k_topk_select, 1, 1024, 0, s, hist, 0, 10, st, 1);
  launch_k(k_topk_ties, (ntiles + 7) / 8, kThreads, 0, s, ws.st_val, ws.tile_cnt, ntiles, st, tile_ties);
  launch_k(k_topk_scan, 1, 1024, 0, s, ws.tile_cnt, tile_ties, ntiles, st, tie_base, out_base,
           out_count);
  launch_k(k_topk_compact, (ntiles + 7) / 8, kThreads, 0, s, ws.st_idx, ws.st_val, ws.tile_cnt,
           ntiles, tie_base, out_base, st, out_idx, out_val, cap);
  for (int i = 0; i < 7; ++i) count_launch();
}

}  // namespace zen
