// Hierarchical Centralization on B200: recursive
// doubling (zen/schemes.hpp:173-193), one process per GPU.
//
// Stage s of rank r with partner q = r ^ 2^s:
//   k_hc_push   my state -> q's receive buffer for stage s, as NVLink stores
//               into q's CUDA-IPC arena.  The last block releases q.ready[s].
//   k_hc_merge  merge_sum(my state, received state) -> my next state
//               (zen/tensor.hpp:133-167).  Every block first acquires
//               my.ready[s].  The last block releases q.done[s]: "your stage-s
//               push was consumed", which q waits on before its next push into
//               my receive buffer (one sync later).
// Counts stay in device memory, so a whole sync is one CUDA graph with no host
// round trip.
//
// The merge is a merge-path merge.  Each 2048-entry tile of the merged
// sequence finds its split of the two sorted inputs by binary search, merges in
// shared memory and folds each shared index into one entry.  A decoupled
// look-back places the tile's unique entries.  On a tie the first input's entry
// comes first, so a shared index sums to a + b, the reference's operand order.
#include <cstdint>
#include <cstdlib>

#include "zen_common.cuh"
#include "zen_internal.h"

namespace zen {

extern void count_launch();

namespace {

using namespace zen_dev;

constexpr uint32_t kMergeThreads = 256;
constexpr uint32_t kMergeItems = 8;
constexpr uint32_t kMergeTile = kMergeThreads * kMergeItems;  // merged positions per tile

// number of A entries among the first d merged positions (A first on ties)
template <typename KA, typename KB>
__device__ __forceinline__ uint64_t merge_split(const KA& A, uint64_t na, const KB& B, uint64_t nb,
                                                uint64_t d) {
  uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// the same split found by one warp: 32 probes per round trip (a 33-ary
// search) instead of one, so a split over millions of entries costs ~5
// dependent loads.  All lanes call; all get the result.  Always returns a
// value in the search range, even for unsorted input.
template <typename KA, typename KB>
__device__ __forceinline__ uint64_t merge_split_warp(const KA& A, uint64_t na, const KB& B,
                                                     uint64_t nb, uint64_t d) {
  const uint32_t lane = lane_id();
  uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (hi > lo) {
    const uint64_t span = hi - lo;
    if (span <= 32) {
      bool p = false;
      if (lane < span) {
        const uint64_t i = lo + lane;
        p = A[i] <= B[d - 1 - i];
      }
      return lo + __popc(__ballot_sync(0xffffffffu, p));
    }
    const uint64_t i = lo + span * (lane + 1) / 33;  // strictly increasing in [lo, hi)
    const uint32_t k = __popc(__ballot_sync(0xffffffffu, A[i] <= B[d - 1 - i]));
    const uint64_t nlo = k ? lo + span * k / 33 + 1 : lo;
    hi = k < 32 ? lo + span * (k + 1) / 33 : hi;
    lo = nlo;
  }
  return lo;
}

struct SmemArr {  // indexable view of a shared-memory slice
  const uint64_t* p;
  __device__ __forceinline__ uint64_t operator[](uint64_t i) const { return p[i]; }
};

// the merge inputs' counts (sub-ranges applied, clamped to capacity)
__device__ __forceinline__ void merge_inputs(HcMergeArgs& a, uint64_t& na, uint64_t& nb,
                                             bool report) {
  na = *(volatile const uint64_t*)a.a_cnt;
  nb = *(volatile const uint64_t*)a.b_cnt;
  if (a.a_bnd) {  // a sub-range of the buffer (an OmniReduce range slice)
    const uint64_t b0 = a.a_bnd[0], b1 = a.a_bnd[1];
    a.a_idx += b0;
    a.a_val += b0;
    na = b1 > b0 ? b1 - b0 : 0;
  }
  if (a.b_bnd) {
    const uint64_t b0 = a.b_bnd[0], b1 = a.b_bnd[1];
    a.b_idx += b0;
    a.b_val += b0;
    nb = b1 > b0 ? b1 - b0 : 0;
  }
  if (na > a.a_cap || nb > a.b_cap) {
    if (report) atomicOr(a.err, kErrCapacity);
    na = na > a.a_cap ? a.a_cap : na;
    nb = nb > a.b_cap ? a.b_cap : nb;
  }
}

// One-wave pre-pass: one warp per tile boundary computes its merge-path split
// (33-ary search), so the merge's tiles -- possibly several waves of them --
// start from a single load instead of ~5 dependent rounds each.
__global__ void __launch_bounds__(256) k_hc_splits(HcMergeArgs a, uint32_t tiles) {
  pdl_entry();
  const uint32_t tid = threadIdx.x;
  const uint64_t ep = a.epoch ? *(volatile const unsigned long long*)a.epoch : 0;
  if (tid == 0) {
    if (a.wait_flag && !wait_flag(a.wait_flag, ep, kPeerTimeoutNs)) atomicOr(a.err, kErrTimeout);
    if (a.wait_flag2 && !wait_flag(a.wait_flag2, ep, kPeerTimeoutNs)) atomicOr(a.err, kErrTimeout);
  }
  __syncthreads();
  uint64_t na, nb;
  merge_inputs(a, na, nb, false);
  const uint64_t tot = na + nb;
  const uint32_t t = blockIdx.x * 8 + (tid >> 5);
  if (t > tiles) return;  // warp-uniform
  uint64_t d = uint64_t(t) * kMergeTile;
  d = d < tot ? d : tot;
  const uint64_t sp = merge_split_warp(a.a_idx, na, a.b_idx, nb, d);
  if ((tid & 31) == 0) a.splits[t] = sp;
}

__global__ void __launch_bounds__(kMergeThreads) k_hc_merge(HcMergeArgs a) {
  pdl_entry();
  __shared__ uint64_t sk[kMergeTile];
  __shared__ float sv[kMergeTile];
  __shared__ uint64_t s_split[2];
  __shared__ uint32_t s_warp[kMergeThreads / 32];
  __shared__ unsigned long long s_red[32];
  const uint32_t tid = threadIdx.x;
  const uint64_t ep = a.epoch ? *(volatile const unsigned long long*)a.epoch : 0;
  if (tid == 0) {
    if (a.wait_flag && !wait_flag(a.wait_flag, ep, kPeerTimeoutNs)) atomicOr(a.err, kErrTimeout);
    if (a.wait_flag2 && !wait_flag(a.wait_flag2, ep, kPeerTimeoutNs)) atomicOr(a.err, kErrTimeout);
  }
  // tiles in launch order (single-pass scans rely on in-order block dispatch);
  // the barrier orders the flag acquire above before any input read
  __syncthreads();
  const uint32_t tile = blockIdx.x;
  const uint32_t tag = *(volatile uint32_t*)&a.ctl->tag;
  uint64_t na, nb;
  merge_inputs(a, na, nb, tid == 0);
  const uint64_t tot = na + nb;
  const uint64_t lo = uint64_t(tile) * kMergeTile;
  const bool live = lo < tot;
  const uint64_t hi = live ? (tot - lo < kMergeTile ? tot : lo + kMergeTile) : lo;
  if (tile == 0 && tid == 0 && a.stage_cnt) *a.stage_cnt = na;

  // ---- tile split + staging ----
  if (a.splits) {  // computed by the pre-pass
    if (live && tid < 2) s_split[tid] = a.splits[tile + tid];
  } else if (live && tid < 64) {
    const uint64_t sp = merge_split_warp(a.a_idx, na, a.b_idx, nb, tid < 32 ? lo : hi);
    if ((tid & 31) == 0) s_split[tid >> 5] = sp;
  }
  __syncthreads();
  uint64_t a0 = live ? s_split[0] : 0, a1 = live ? s_split[1] : 0;
  uint64_t b0 = lo - a0, b1 = hi - a1;
  if (a1 < a0 || b1 < b0) {  // only unsorted input: skip the tile, report it
    if (tid == 0) atomicOr(a.err, kErrOutside);
    a1 = a0;
    b1 = b0;
  }
  const uint32_t la = (uint32_t)(a1 - a0), lb = (uint32_t)(b1 - b0);
  const uint32_t len = la + lb;
  for (uint32_t x = tid; x < len; x += kMergeThreads) {
    if (x < la) {
      sk[x] = a.a_idx[a0 + x];
      sv[x] = a.a_val[a0 + x];
    } else {
      sk[x] = a.b_idx[b0 + x - la];
      sv[x] = a.b_val[b0 + x - la];
    }
  }
  __syncthreads();

  // ---- per-thread merge of up to 8 positions ----
  uint64_t key[kMergeItems];
  float val[kMergeItems];
  bool keep[kMergeItems];
  uint32_t u = 0;
  const uint32_t d = tid * kMergeItems;
  if (d < len) {
    const SmemArr A{sk}, B{sk + la};
    uint32_t i = (uint32_t)merge_split(A, la, B, lb, d), j = d - i;
    // merged predecessor of local position d (the larger of the two last consumed)
    bool has_prev;
    uint64_t prev = 0;
    if (d == 0) {
      const bool pa = a0 > 0, pb = b0 > 0;
      has_prev = pa || pb;
      const uint64_t ka = pa ? a.a_idx[a0 - 1] : 0, kb = pb ? a.b_idx[b0 - 1] : 0;
      prev = pa && pb ? (ka > kb ? ka : kb) : (pa ? ka : kb);
    } else {
      has_prev = true;
      const uint64_t ka = i > 0 ? A[i - 1] : 0, kb = j > 0 ? B[j - 1] : 0;
      prev = i > 0 && j > 0 ? (ka > kb ? ka : kb) : (i > 0 ? ka : kb);
    }
    const uint32_t cnt = len - d < kMergeItems ? len - d : kMergeItems;
#pragma unroll
    for (uint32_t k = 0; k < kMergeItems; ++k) {
      if (k < cnt) {
        const bool ta = i < la && (j >= lb || A[i] <= B[j]);
        key[k] = ta ? A[i] : B[j];
        val[k] = ta ? sv[i] : sv[la + j];
        if (ta) ++i; else ++j;
      }
    }
    // the merged entry after this thread's last one (next thread's or next tile's)
    bool has_next = false;
    uint64_t nkey = 0;
    float nval = 0.f;
    if (d + cnt < len) {
      has_next = true;
      const bool ta = i < la && (j >= lb || A[i] <= B[j]);
      nkey = ta ? A[i] : B[j];
      nval = ta ? sv[i] : sv[la + j];
    } else if (hi < tot) {
      has_next = true;
      const bool ta = a1 < na && (b1 >= nb || a.a_idx[a1] <= a.b_idx[b1]);
      nkey = ta ? a.a_idx[a1] : a.b_idx[b1];
      nval = ta ? a.a_val[a1] : a.b_val[b1];
    }
#pragma unroll
    for (uint32_t k = 0; k < kMergeItems; ++k) {
      keep[k] = false;
      if (k < cnt) {
        const bool dup = k == 0 ? (has_prev && prev == key[0]) : key[k - 1] == key[k];
        keep[k] = !dup;
        if (!dup) {
          // a shared index is (A entry, B entry), adjacent: fold b into a
          if (k + 1 < cnt) {
            if (key[k + 1] == key[k]) val[k] = val[k] + val[k + 1];
          } else if (has_next && nkey == key[k]) {
            val[k] = val[k] + nval;
          }
          ++u;
        }
      }
    }
  }

  // ---- block scan of the unique counts ----
  const uint32_t lane = tid & 31, warp = tid >> 5;
  uint32_t incl = u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();  // also: every thread is done reading sk/sv
  uint32_t wbase = 0, agg = 0;
#pragma unroll
  for (uint32_t w = 0; w < kMergeThreads / 32; ++w) {
    const uint32_t t = s_warp[w];
    if (w < warp) wbase += t;
    agg += t;
  }
  uint32_t pos = wbase + incl - u;
  if (d < len) {
#pragma unroll
    for (uint32_t k = 0; k < kMergeItems; ++k)
      if (keep[k]) {
        sk[pos] = key[k];
        sv[pos] = val[k];
        ++pos;
      }
  }
  // block-wide look-back: the grid is one wave, so a warp-wide walk would go
  // back window by window through every tile in flight
  const uint64_t excl = lookback_block(a.lb_status, tile, tag, agg, s_red);
  __syncthreads();  // the staged entries in sk/sv (tile 0 returns without a barrier)
  for (uint32_t x = tid; x < agg; x += kMergeThreads) {
    const uint64_t o = excl + x;
    if (o < a.o_cap) {
      a.o_idx[o] = sk[x];
      a.o_val[o] = sv[x];
    }
  }
  if (tid == 0) {
    const uint64_t total = excl + agg;
    if ((live && hi == tot) || (tot == 0 && tile == 0)) {
      if (total > a.o_cap) atomicOr(a.err, kErrCapacity);
      *a.o_cnt = total;  // the true size; readers clamp to their capacity
    }
  }
  // the last tile's prefix needed every tile's aggregate, which each tile
  // publishes after its last read of the inputs and of the tag: the tag can
  // advance and the senders can reuse their buffers
  const bool last = blockIdx.x == gridDim.x - 1;
  if (last && tid == 0) {
    const uint32_t t = (tag + 1u) & 0xFFFFFFu;
    a.ctl->tag = t ? t : 1u;
  }
  if (last && tid == 0) {
    if (a.done_flag || a.done_flag2) __threadfence_system();
    if (a.done_flag) st_release_sys(a.done_flag, ep);
    if (a.done_flag2) st_release_sys(a.done_flag2, ep);
  }
}

// my state -> the partner's receive buffer (peer stores); the last block
// publishes the count and releases the partner's ready flag.
__global__ void __launch_bounds__(256) k_hc_push(HcPushArgs a) {
  pdl_entry();
  const uint32_t tid = threadIdx.x;
  const uint64_t ep = *(volatile const unsigned long long*)a.epoch;
  // the partner consumed what this rank pushed into the same buffer last sync
  if (tid == 0 && ep > 1 && !wait_flag(a.done_flag, ep - 1, kPeerTimeoutNs))
    atomicOr(a.err, kErrTimeout);
  // a forwarded tensor: it must have arrived in this rank's slot
  if (tid == 0 && a.src_wait && !wait_flag(a.src_wait, ep, kPeerTimeoutNs))
    atomicOr(a.err, kErrTimeout);
  __syncthreads();
  uint64_t n = *(volatile const uint64_t*)a.src_cnt;
  uint64_t off = 0;
  if (a.src_bnd) {  // a sub-range of the source buffer
    off = a.src_bnd[0];
    n = a.src_bnd[1] > off ? a.src_bnd[1] - off : 0;
    a.src_idx += off;
    a.src_val += off;
  }
  if (n > a.cap) {
    if (tid == 0 && blockIdx.x == 0) atomicOr(a.err, kErrCapacity);
    n = a.cap;
  }
  const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + tid, stride = uint64_t(gridDim.x) * blockDim.x;
  if (off & 3) {  // a misaligned slice: element copies (still coalesced)
    for (uint64_t x = g; x < n; x += stride) {
      a.dst_idx[x] = a.src_idx[x];
      a.dst_val[x] = a.src_val[x];
    }
    if (blockIdx.x == 0 && tid == 0) {
      *a.dst_cnt = n;
      if (a.sent_cnt) *a.sent_cnt = n;
    }
    if (finish_tile(a.ctl, gridDim.x, /*sys=*/true) && tid == 0) {
      __threadfence_system();
      st_release_sys(a.ready_flag, ep);
    }
    return;
  }
  // buffers are 256-byte aligned: 16-byte vectors, then the tails
  // four independent 16-byte loads in flight per thread, then their stores
  const uint64_t n2 = n >> 1, n4 = n >> 2;
  const ulonglong2* si = reinterpret_cast<const ulonglong2*>(a.src_idx);
  ulonglong2* di = reinterpret_cast<ulonglong2*>(a.dst_idx);
  for (uint64_t x = g; x < n2; x += 4 * stride) {
    ulonglong2 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x + u * stride < n2) t[u] = si[x + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x + u * stride < n2) di[x + u * stride] = t[u];
  }
  const float4* sv = reinterpret_cast<const float4*>(a.src_val);
  float4* dv = reinterpret_cast<float4*>(a.dst_val);
  for (uint64_t x = g; x < n4; x += 4 * stride) {
    float4 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x + u * stride < n4) t[u] = sv[x + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x + u * stride < n4) dv[x + u * stride] = t[u];
  }
  if (blockIdx.x == 0) {
    if (tid == 0 && (n & 1)) a.dst_idx[n - 1] = a.src_idx[n - 1];
    if (tid < (n & 3)) a.dst_val[(n4 << 2) + tid] = a.src_val[(n4 << 2) + tid];
    if (tid == 0) {
      *a.dst_cnt = n;
      if (a.sent_cnt) *a.sent_cnt = n;
    }
  }
  if (finish_tile(a.ctl, gridDim.x, /*sys=*/true) && tid == 0) {
    __threadfence_system();
    st_release_sys(a.ready_flag, ep);
  }
}

// n disjoint ascending segments -> one tensor with exact zeros dropped; tiles
// of the concatenated position space, a block scan of the kept entries and a
// decoupled look-back for their output positions.
constexpr uint32_t kConcatMaxSeg = 256;

__global__ void __launch_bounds__(kMergeThreads) k_hc_concat(HcConcatArgs a) {
  pdl_entry();
  __shared__ uint64_t s_pre[kConcatMaxSeg + 1];
  __shared__ uint32_t s_warp[kMergeThreads / 32];
  __shared__ unsigned long long s_red[32];
  const uint32_t tid = threadIdx.x, n = a.n;
  const uint64_t ep = *(volatile const unsigned long long*)a.epoch;
  if (tid < n && a.wait[tid] && !wait_flag(a.wait[tid], ep, kPeerTimeoutNs))
    atomicOr(a.err, kErrTimeout);
  __syncthreads();  // orders the flag acquires above before any segment read
  const uint32_t tile = blockIdx.x;
  const uint32_t tag = *(volatile uint32_t*)&a.ctl->tag;
  if (tid == 0) {
    uint64_t run = 0;
    for (uint32_t p = 0; p < n; ++p) {
      s_pre[p] = run;
      uint64_t c = *(volatile const uint64_t*)a.seg_cnt[p];
      if (c > a.seg_cap) {
        atomicOr(a.err, kErrCapacity);
        c = a.seg_cap;
      }
      run += c;
    }
    s_pre[n] = run;
  }
  __syncthreads();
  const uint64_t tot = s_pre[n];
  uint32_t keep = 0;
  uint64_t key[kMergeItems];
  float val[kMergeItems];
  const uint64_t base = uint64_t(tile) * kMergeTile + uint64_t(tid) * kMergeItems;
#pragma unroll
  for (uint32_t k = 0; k < kMergeItems; ++k) {
    const uint64_t x = base + k;
    val[k] = 0.f;
    if (x < tot) {
      uint32_t lo = 0, hi = n;  // segment: last p with s_pre[p] <= x
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_pre[mid] <= x) lo = mid; else hi = mid;
      }
      key[k] = a.seg_idx[lo][x - s_pre[lo]];
      val[k] = a.seg_val[lo][x - s_pre[lo]];
      if (val[k] != 0.0f) keep |= 1u << k;
    }
  }
  const uint32_t u = __popc(keep), lane = tid & 31, warp = tid >> 5;
  uint32_t incl = u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t wbase = 0, agg = 0;
#pragma unroll
  for (uint32_t w = 0; w < kMergeThreads / 32; ++w) {
    const uint32_t t = s_warp[w];
    if (w < warp) wbase += t;
    agg += t;
  }
  const uint64_t excl = lookback_block(a.lb_status, tile, tag, agg, s_red);
  uint64_t pos = excl + wbase + incl - u;
#pragma unroll
  for (uint32_t k = 0; k < kMergeItems; ++k)
    if ((keep >> k) & 1u) {
      if (pos < a.o_cap) {
        a.o_idx[pos] = key[k];
        a.o_val[pos] = val[k];
      }
      ++pos;
    }
  if (tid == 0 && (base < tot || tile == 0) &&
      (uint64_t(tile + 1) * kMergeTile >= tot)) {  // the tile holding the last position
    const uint64_t total = excl + agg;
    if (total > a.o_cap) atomicOr(a.err, kErrCapacity);
    *a.o_cnt = total;
  }
  // the last tile: every tile has read its segments and the tag (as k_hc_merge)
  if (blockIdx.x == gridDim.x - 1) {
    if (tid == 0) {
      const uint32_t t = (tag + 1u) & 0xFFFFFFu;
      a.ctl->tag = t ? t : 1u;
      __threadfence_system();
    }
    __syncthreads();
    if (tid < n && a.done[tid]) st_release_sys(a.done[tid], ep);
  }
}

__global__ void k_hc_bounds(const uint64_t* __restrict__ idx, const uint64_t* count, uint64_t m,
                            uint32_t parts, uint64_t* __restrict__ bnd) {
  pdl_entry();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  const uint64_t c = *(volatile const uint64_t*)count;
  const uint64_t range = (m + parts - 1) / parts;
  const uint64_t key = p == parts ? m : (uint64_t(p) * range < m ? uint64_t(p) * range : m);
  uint64_t lo = 0, hi = c;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < key) lo = mid + 1; else hi = mid;
  }
  bnd[p] = lo;
}

__global__ void k_hc_begin(unsigned long long* epoch) {
  pdl_entry();
  if (threadIdx.x == 0) *epoch = *epoch + 1;
}

__global__ void k_set_u64(uint64_t* p, uint64_t v) {
  pdl_entry();
  if (threadIdx.x == 0) *p = v;
}

}  // namespace

uint32_t hc_merge_tiles(uint64_t max_entries) {
  return (uint32_t)((max_entries + kMergeTile - 1) / kMergeTile) + 1;
}

void launch_hc_merge(const HcMergeArgs& a, uint32_t tiles, cudaStream_t stream) {
  // the split pre-pass is on unless ZEN_MERGE_PREPASS=0 (A/B: HC at N=4
  // 0.1975 vs 0.2005 ms; the merge kernel itself 25.3 -> 20.5 us at 640K+640K)
  static const bool pre = [] {
    const char* e = std::getenv("ZEN_MERGE_PREPASS");
    return !(e && e[0] == '0');
  }();
  HcMergeArgs m = a;
  if (!pre) m.splits = nullptr;
  if (m.splits) {
    launch_k(k_hc_splits, (tiles + 1 + 7) / 8, 256, 0, stream, m, tiles);
    count_launch();
  }
  launch_k(k_hc_merge, tiles, kMergeThreads, 0, stream, m);
  count_launch();
}

void launch_hc_push(const HcPushArgs& a, cudaStream_t stream) {
  launch_k(k_hc_push, 148 * 2, 256, 0, stream, a);
  count_launch();
}

void launch_hc_concat(const HcConcatArgs& a, uint32_t tiles, cudaStream_t stream) {
  launch_k(k_hc_concat, tiles, kMergeThreads, 0, stream, a);
  count_launch();
}

void launch_hc_bounds(const uint64_t* idx, const uint64_t* count, uint64_t m, uint32_t parts,
                      uint64_t* bnd, cudaStream_t stream) {
  launch_k(k_hc_bounds, (parts + 256) / 256, 256, 0, stream, idx, count, m, parts, bnd);
  count_launch();
}

void launch_hc_begin(unsigned long long* epoch, cudaStream_t stream) {
  launch_k(k_hc_begin, 1, 32, 0, stream, epoch);
  count_launch();
}

void launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t stream) {
  launch_k(k_set_u64, 1, 32, 0, stream, p, v);
  count_launch();
}

}  // namespace zen
