// k_codec.cu -- the owner side of Balanced Parallelism on sm_100a.
//
//  tables    : HashUniverseTable (zen/codec.hpp:47-72) without materialising
//              the M x 8 B sorted lists: per 64-index word, ceil(log2 n) owner
//              bit planes (the information minimum), per-32-word chunk prefix
//              counts per server, and for each local server a {mask, rank
//              base} record per word.
//  aggregate : per-owner sum (merge_sum left fold in worker order,
//              zen/schemes.hpp:375-380; zen/tensor.hpp:133-167) FUSED with the
//              HashBitmap encode (zen/codec.hpp:266-277): each worker's part
//              becomes a presence bitmap over I_s; their OR is the HashBitmap,
//              written straight into every receiver's pull inbox (NVLink
//              stores in rank mode); popcount prefixes locate every value, and
//              the values of a union bit are folded in worker order (bit-exact,
//              zero sums kept).  Work ~ bitmap words + entries, no look-back.
//  decode    : all servers' (bitmap, values) -> the global ascending result
//              (decode zen/codec.hpp:333-347 + merge_disjoint
//              zen/schemes.hpp:91-113).  Per global word, each server's owned
//              positions are a contiguous bit range of its bitmap; a software
//              pdep deposits them into the owner mask; a tile's first output
//              position is sum_s popcount_s(below the tile), so tiles are
//              independent; warps expand set bits cooperatively (coalesced
//              stores).  Output order falls out of the global word order.
#include "zen_common.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

// ---------------------------------------------------------------- tables ----

__device__ __forceinline__ uint64_t valid_mask(uint64_t m, uint64_t w) {
  const uint64_t lo = w * 64;
  return (lo + 64 <= m) ? ~0ull : lowmask64((uint32_t)(m - lo));
}

__device__ __forceinline__ uint64_t owner_mask(const unsigned long long* pl, uint32_t nplanes,
                                               uint32_t s, uint64_t vmask) {
  uint64_t ms = vmask;
  for (uint32_t j = 0; j < nplanes; ++j) ms &= ((s >> j) & 1u) ? pl[j] : ~pl[j];
  return ms;
}

// register-resident variant for the decode (n <= 16 -> at most 4 planes)
__device__ __forceinline__ uint64_t owner_mask4(const unsigned long long (&pl)[4],
                                                uint32_t nplanes, uint32_t s, uint64_t vmask) {
  uint64_t ms = vmask;
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j)
    if (j < nplanes) ms &= ((s >> j) & 1u) ? pl[j] : ~pl[j];
  return ms;
}

// one thread per 64-index word; warps cover 32 consecutive words (a chunk)
__global__ void __launch_bounds__(256) k_tables_planes(uint64_t m, uint32_t n, uint64_t pc,
                                                       uint32_t nplanes,
                                                       unsigned long long* planes,
                                                       uint32_t* chunk_cnt, uint64_t nwords) {
  zen_dev::pdl_entry();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;  // multiple of 32
  for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x; w0 < nwords; w0 += stride) {
    const uint64_t w = w0 + threadIdx.x;
    unsigned long long pl[16] = {0};
    uint64_t vmask = 0;
    if (w < nwords) {
      vmask = valid_mask(m, w);
      for (uint32_t b = 0; b < 64; ++b) {
        if (!((vmask >> b) & 1ull)) break;
        const uint32_t o = part_of_seed(pc, n, w * 64 + b + 1);
        for (uint32_t j = 0; j < nplanes; ++j) pl[j] |= (unsigned long long)((o >> j) & 1u) << b;
      }
      for (uint32_t j = 0; j < nplanes; ++j) planes[w * nplanes + j] = pl[j];
    }
    const uint64_t chunk = w0 / 32 + (threadIdx.x >> 5);
    for (uint32_t s = 0; s < n; ++s) {
      const uint32_t c = w < nwords ? __popcll(owner_mask(pl, nplanes, s, vmask)) : 0u;
      const uint32_t tot = __reduce_add_sync(0xffffffffu, c);
      if (lane_id() == 0 && chunk * 32 < nwords) chunk_cnt[chunk * n + s] = tot;
    }
  }
}

// in-place exclusive scan over chunks, per server; totals[s] = |I_s|
__global__ void __launch_bounds__(1024) k_tables_scan(uint32_t* cc, uint64_t nchunks, uint32_t n,
                                                      uint64_t* totals) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sscan[33];
  for (uint32_t s = 0; s < n; ++s) {
    uint64_t carry = 0;
    for (uint64_t b = 0; b < nchunks; b += blockDim.x) {
      const uint64_t c = b + threadIdx.x;
      const uint32_t v = c < nchunks ? cc[c * n + s] : 0u;
      uint32_t tot;
      const uint32_t ex = block_exclusive_sum(v, sscan, &tot);
      if (c < nchunks) cc[c * n + s] = (uint32_t)(carry + ex);
      carry += tot;
    }
    if (threadIdx.x == 0) totals[s] = carry;
  }
}

__global__ void __launch_bounds__(256) k_tables_own(uint64_t m, uint32_t n, uint32_t s,
                                                    uint32_t nplanes,
                                                    const unsigned long long* planes,
                                                    const uint32_t* cprefix, OwnWord* own,
                                                    uint32_t* sel, uint64_t nsel, uint64_t nwords) {
  zen_dev::pdl_entry();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x; w0 < nwords; w0 += stride) {
    const uint64_t w = w0 + threadIdx.x;
    uint64_t ms = 0;
    if (w < nwords) ms = owner_mask(planes + w * nplanes, nplanes, s, valid_mask(m, w));
    const uint32_t c = __popcll(ms);
    const uint32_t inc = warp_inclusive_sum(c);
    const uint64_t chunk = w0 / 32 + (threadIdx.x >> 5);
    if (w < nwords) {
      const uint32_t prefix = cprefix[chunk * n + s] + inc - c;
      own[w] = OwnWord{ms, prefix, 0u};
    }
  }
}

// ------------------------------------------------------------- aggregate ----

constexpr int kAggThreads = 256;
constexpr int kPrefixThreads = 512;  // union / bpre blocks (256-thread blocks measured no faster)
constexpr int kWPT = kPrefixBlockWords / kPrefixThreads;  // consecutive words per thread (4)

__device__ __forceinline__ uint32_t part_count(const AggArgs& a, uint32_t w) {
  if (a.in_hdr) return *(volatile const uint32_t*)&a.in_hdr[w]->counts[a.s];  // peers (rank mode)
  if (a.in_load) return a.in_load[w][a.s];  // local mode: the workers' own counters
  return (uint32_t)a.in_count[w];
}

// one worker, one-server universe, no scatter marks: U is the worker's row
__device__ __forceinline__ bool solo_part(const AggArgs& a) {
  return a.whole && a.n == 1 && !a.pre_min;
}

// Phase 1: every received entry sets its HashBitmap position (its rank in I_s,
// zen/codec.hpp:146-158) in its worker's presence bitmap.
__global__ void __launch_bounds__(kAggThreads) k_agg_mark(AggArgs a) {
  zen_dev::pdl_entry();
  __shared__ uint64_t pre[kMaxWorkers + 1];
  const uint32_t n = a.n;
  if (a.wait_push && a.gate)  // rank mode: the n pushes have arrived (no k_wait_push)
    arrival_gate(n, [&](uint32_t w) { return (const unsigned long long*)&a.in_hdr[w]->flag; },
                 &a.hdr->go[0], *(volatile uint32_t*)&a.hdr->iter, &a.hdr->status);
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (uint32_t w = 0; w < n; ++w) {
      pre[w] = acc;
      acc += part_count(a, w);
    }
    pre[n] = acc;
  }
  __syncthreads();
  const uint64_t total = pre[n];
  const uint32_t lane = lane_id();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int R = 4;  // entries per thread per round, loads issued together
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); base < total;
       base += R * stride) {  // warp-uniform trip count: full-mask shuffles below
    uint32_t w[R], key[R];
    uint64_t e[R];
    bool in[R];
    OwnWord ow[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint64_t i = base + q * stride + lane;
      in[q] = i < total;
      w[q] = 0;
      if (in[q])
        while (i >= pre[w[q] + 1]) ++w[q];
      e[q] = in[q] ? i - pre[w[q]] : 0;  // index inside worker w's part
      key[q] = in[q] ? a.in_idx[w[q]][e[q]] : 0u;
    }
#pragma unroll
    for (int q = 0; q < R; ++q)  // (a one-server universe: I_0 is every index, rank = index)
      ow[q] = a.whole ? OwnWord{~0ull, key[q] & ~63u, 0u} : a.own[in[q] ? key[q] >> 6 : 0];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (base + q * stride >= total) break;  // warp-uniform
      const bool owned = in[q] && ((ow[q].mask >> (key[q] & 63u)) & 1ull);
      if (in[q] && !owned) {
        atomicMin((unsigned long long*)&a.hdr->bad_index, (unsigned long long)key[q]);
        atomicOr(&a.hdr->status, kErrOutside);
      }
      const uint32_t r = ow[q].prefix + (uint32_t)__popcll(ow[q].mask & lowmask64(key[q] & 63u));
      // consecutive keys share bitmap words: one atomic per distinct word per warp
      unsigned long long* word = owned ? a.pw + (uint64_t)w[q] * a.nws + (r >> 6) : nullptr;
      const uint64_t bit = owned ? 1ull << (r & 63u) : 0ull;
      const uint32_t grp = __match_any_sync(0xffffffffu, (unsigned long long)word);
      const uint32_t lo = __reduce_or_sync(grp, (uint32_t)bit);
      const uint32_t hi = __reduce_or_sync(grp, (uint32_t)(bit >> 32));
      if (owned && lane == (uint32_t)(__ffs(grp) - 1))
        atomicOr(word, ((unsigned long long)hi << 32) | lo);
      // The part is ascending, so its entries in bitmap word j are consecutive:
      // the first of them is at part index = worker w's popcount prefix at j,
      // which the fold needs -- written here instead of scanned later.
      if (solo_part(a)) continue;  // (no value bases: the union copies the values)
      const uint32_t jw = owned ? (r >> 6) : 0xFFFFFFFFu;
      uint32_t prev_w = __shfl_up_sync(0xffffffffu, w[q], 1);
      uint32_t prev_j = __shfl_up_sync(0xffffffffu, jw, 1);
      if (in[q] && owned && (lane == 0 || prev_w != w[q]) && e[q] > 0) {
        const uint32_t pk = a.in_idx[w[q]][e[q] - 1];  // previous entry of the same part
        const OwnWord po = a.whole ? OwnWord{~0ull, pk & ~63u, 0u} : a.own[pk >> 6];
        prev_w = w[q];
        prev_j = (po.prefix + (uint32_t)__popcll(po.mask & lowmask64(pk & 63u))) >> 6;
      }
      if (owned && (e[q] == 0 || prev_w != w[q] || prev_j != jw))
        a.pre[(uint64_t)w[q] * a.nws + jw] = (uint32_t)e[q];
    }
  }
}

// Phase 2: U = OR_w P_w -> every destination; block-local popcount prefixes of
// U and each P_w; the last block turns the block totals into exclusive
// prefixes and records U_s.
__device__ __forceinline__ void load8(const unsigned long long* p, unsigned long long (&v)[kWPT]) {
  const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p);  // 64 B, 64 B aligned
#pragma unroll
  for (int i = 0; i < kWPT / 2; ++i) {
    const ulonglong2 t = q[i];
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(unsigned long long* p, const unsigned long long (&v)[kWPT]) {
  ulonglong2* q = reinterpret_cast<ulonglong2*>(p);
#pragma unroll
  for (int i = 0; i < kWPT / 2; ++i) q[i] = make_ulonglong2(v[2 * i], v[2 * i + 1]);
}
__device__ __forceinline__ void store8u(uint32_t* p, const uint32_t (&v)[kWPT]) {
  static_assert(kWPT % 2 == 0, "pairs of words per thread");
  uint2* q = reinterpret_cast<uint2*>(p);  // 8 B aligned (kWPT even)
#pragma unroll
  for (int i = 0; i < kWPT / 2; ++i) q[i] = make_uint2(v[2 * i], v[2 * i + 1]);
}

// Phase 2: U = OR_w P_w -> every destination, and the popcount prefix of U
// (block-local per word + block totals; the last block turns the totals into
// exclusive prefixes and records U_s).  Workers' own prefixes come from
// k_agg_mark, so only U is scanned.
__global__ void __launch_bounds__(kPrefixThreads) k_agg_union(AggArgs a) {
  zen_dev::pdl_entry();
  constexpr int kW = kPrefixThreads / 32;
  __shared__ uint32_t wsum[kW];
  __shared__ uint32_t s_last;
  const uint32_t n = a.n, lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t j0 = (uint64_t)blockIdx.x * kPrefixBlockWords + (uint64_t)threadIdx.x * kWPT;
  const bool live = j0 < a.nw;
  unsigned long long U[kWPT];
#pragma unroll
  for (int i = 0; i < kWPT; ++i) U[i] = 0;
  const bool from_entries = solo_part(a) && a.solo_gbase != nullptr;
  if (from_entries) {
    // One worker, dense sync: U is its part, so the block builds its 2048
    // words from the part's entries of its two 8-tile groups (their range
    // from the push scatter's group bases) in shared memory -- the mark
    // kernel and the presence row are not needed.
    __shared__ unsigned long long sU[kPrefixBlockWords];
    for (uint32_t i = threadIdx.x; i < kPrefixBlockWords; i += kPrefixThreads) sU[i] = 0ull;
    __syncthreads();
    static_assert(kPrefixBlockWords * 64 == 2 * 8 * kExtractTile, "two push groups per block");
    const uint32_t g0 = 2 * blockIdx.x;
    const uint32_t cnt = part_count(a, 0);
    const uint32_t lo = g0 < a.ngroups ? a.solo_gbase[g0] : cnt;
    const uint32_t hi = g0 + 2 < a.ngroups ? a.solo_gbase[g0 + 2] : cnt;
    const uint64_t kbase = (uint64_t)blockIdx.x * kPrefixBlockWords * 64;
    const uint32_t* keys = a.in_idx[0];
    constexpr int R = 4;  // rounds of keys in flight per warp (loads first)
    for (uint32_t e0 = lo + warp * 32; e0 < hi; e0 += R * kPrefixThreads) {  // warp-uniform
      uint32_t key[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const uint32_t e = e0 + q * kPrefixThreads + lane;
        key[q] = e < hi ? keys[e] : 0u;
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (e0 + q * kPrefixThreads >= hi) break;  // warp-uniform
        const bool v = e0 + q * kPrefixThreads + lane < hi;
        const uint32_t jw = v ? (uint32_t)(((uint64_t)key[q] - kbase) >> 6) : 0xFFFFFFFFu;
        const uint64_t bit = v ? 1ull << (key[q] & 63u) : 0ull;
        const uint32_t grp = __match_any_sync(0xffffffffu, jw);
        const uint32_t blo = __reduce_or_sync(grp, (uint32_t)bit);
        const uint32_t bhi = __reduce_or_sync(grp, (uint32_t)(bit >> 32));
        if (v && lane == (uint32_t)(__ffs(grp) - 1))
          atomicOr(&sU[jw], ((unsigned long long)bhi << 32) | blo);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kWPT; ++i) U[i] = sU[threadIdx.x * kWPT + i];
  } else if (live) {
#pragma unroll 4
    for (uint32_t x = 0; x < n; ++x) {  // (unrolled: several rows' loads in flight)
      unsigned long long v[kWPT];
      load8(a.pw + (uint64_t)x * a.nws + j0, v);
#pragma unroll
      for (int i = 0; i < kWPT; ++i) U[i] |= v[i];
    }
  }
  if (live) {
    // the union bitmap (the HashBitmap: LSB-first = little-endian words)
    for (uint32_t d = 0; d < a.ndst; ++d) store8(a.dst_bits[d] + j0, U);
    if (solo_part(a) && !from_entries) {  // the last reader of the presence row: clean it
      bool any = false;
#pragma unroll
      for (int i = 0; i < kWPT; ++i) any |= U[i] != 0ull;
      if (any) {
        unsigned long long z[kWPT];
#pragma unroll
        for (int i = 0; i < kWPT; ++i) z[i] = 0ull;
        store8(a.pw + j0, z);
      }
    }
  }
  if (solo_part(a)) {
    // One worker of a one-server universe: U = its presence row, so the U rank
    // of entry e's bit is e itself and the folded values are the part's values
    // in order -- the fold is a copy, done here (no dependence on the prefix).
    const uint64_t cnt = min((uint64_t)part_count(a, 0), a.val_cap);
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const float* src = a.in_val[0];
    for (uint32_t d = 0; d < a.ndst; ++d) {
      float* dst = a.dst_vals[d];
      const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0;
      const uint64_t nv = vec ? cnt / 4 : 0;
      for (uint64_t i = t; i < nv; i += nth)
        reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
      for (uint64_t i = nv * 4 + t; i < cnt; i += nth) dst[i] = src[i];
    }
  }
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < kWPT; ++i) t += __popcll(U[i]);
  const uint32_t inc = warp_inclusive_sum(t);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {  // exclusive prefix over the block's warps
    const uint32_t v = lane < (uint32_t)kW ? wsum[lane] : 0u;
    const uint32_t wi = warp_inclusive_sum(v);
    if (lane < (uint32_t)kW) wsum[lane] = wi - v;
    if (lane == 31) a.blk[(uint64_t)n * a.nblk + blockIdx.x] = wi;
  }
  __syncthreads();
  if (live) {
    uint32_t pre[kWPT];
    uint32_t run = wsum[warp] + inc - t;
#pragma unroll
    for (int i = 0; i < kWPT; ++i) {
      pre[i] = run;
      run += __popcll(U[i]);
    }
    store8u(a.pre + (uint64_t)n * a.nws + j0, pre);
  }
  // last block: exclusive prefix of the block totals, |U_s|
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (atomicAdd(&a.done[0], 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (warp == 0) {
    const uint32_t total = warp_exscan_l2(a.blk + (uint64_t)n * a.nblk, a.nblk);
    if (lane == 0) {
      *a.agg_count = total;
      a.done[0] = 0;
    }
  }
}

// Phase 3: one thread per bitmap word stages its words in shared memory; the
// warp then expands the union bits cooperatively (one output value per lane,
// consecutive lanes -> consecutive positions).  Value of a union bit = fold
// of its contributors' values in ascending worker order (zen/tensor.hpp:151-153).
constexpr int kValThreads = 128;

template <int NMAX>
__global__ void __launch_bounds__(kValThreads) k_agg_values(AggArgs a) {
  zen_dev::pdl_entry();
  __shared__ unsigned long long spw[kValThreads][NMAX];
  __shared__ uint32_t sbase[kValThreads][NMAX];
  const uint32_t n = a.n, lane = lane_id();
  const uint64_t j = (uint64_t)blockIdx.x * kValThreads + threadIdx.x;
  if (a.dst_cbase) {
    // the receivers' value bases per global chunk: U's popcount below the
    // chunk's first position P in I_s = block prefix + word prefix + the
    // word's low bits (this server's prefixes of U, final since k_agg_union)
    const uint64_t nth = (uint64_t)gridDim.x * kValThreads;
    for (uint64_t c = j; c <= a.nchunks; c += nth) {
      const uint64_t P = c < a.nchunks ? (uint64_t)a.cprefix[c * n + a.s] : a.bs;
      const uint64_t w = P >> 6;
      uint32_t b;
      if (w >= a.nw) {
        b = (uint32_t)*a.agg_count;
      } else {
        b = a.blk[(uint64_t)n * a.nblk + w / kPrefixBlockWords] + a.pre[(uint64_t)n * a.nws + w] +
            (uint32_t)__popcll(a.own_bits[w] & lowmask64((uint32_t)(P & 63)));
      }
      for (uint32_t d = 0; d < a.ndst; ++d) a.dst_cbase[d][c] = b;
    }
  }
  if (solo_part(a)) return;  // the union copied the values (and cleaned the row)
  const bool valid = j < a.nw;
  const uint32_t pb = (uint32_t)(j / kPrefixBlockWords);
  // every worker's presence word first, then the value bases, then the
  // clean-up stores: stores between the loads would serialise them (the rows
  // share one array, so the compiler cannot move a load above a store)
  unsigned long long U = 0, v[NMAX];
  uint32_t b[NMAX];
#pragma unroll
  for (int w = 0; w < NMAX; ++w) v[w] = (w < (int)n && valid) ? a.pw[(uint64_t)w * a.nws + j] : 0ull;
#pragma unroll
  for (int w = 0; w < NMAX; ++w)  // part index of the word's first entry (k_agg_mark)
    b[w] = v[w] ? a.pre[(uint64_t)w * a.nws + j] : 0u;
#pragma unroll
  for (int w = 0; w < NMAX; ++w) {
    if (v[w]) {
      a.pw[(uint64_t)w * a.nws + j] = 0ull;  // last reader: clean for the next sync
      if (a.pre_min) a.pre[(uint64_t)w * a.nws + j] = ~0u;  // scatter marks: atomicMin
    }
    spw[threadIdx.x][w] = v[w];
    sbase[threadIdx.x][w] = b[w];
    U |= v[w];
  }
  const uint64_t ubase = (valid && U) ? (uint64_t)a.blk[(uint64_t)n * a.nblk + pb] +
                                            a.pre[(uint64_t)n * a.nws + j] : 0ull;
  const uint32_t c = __popcll(U);
  const uint32_t inc = warp_inclusive_sum(c);
  const uint32_t x = inc - c;
  const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
  // output position of the warp's first value = ubase of its first non-empty lane
  const uint32_t first = __ffs(__ballot_sync(0xffffffffu, c != 0));
  const uint64_t wbase = first ? __shfl_sync(0xffffffffu, ubase, first - 1) : 0ull;
  const uint32_t row0 = threadIdx.x & ~31u;
  __syncwarp();
  // (unrolling this loop 4x with every value load of the pass issued first
  // measured no faster: 0.1085 ms either way, aggregate 44.3 vs 43.2 us)
  for (uint32_t k0 = 0; k0 < T; k0 += 32) {
    const uint32_t k = k0 + lane;
    uint32_t L = 0;
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1) {
      const uint32_t xc = __shfl_sync(0xffffffffu, x, L + step);
      if (xc <= k) L += step;
    }
    const unsigned long long UL = __shfl_sync(0xffffffffu, U, L);
    const uint32_t xL = __shfl_sync(0xffffffffu, x, L);
    if (k < T) {
      const uint32_t bit = (UL == ~0ull) ? k - xL : select64(UL, k - xL);
      const uint64_t lm = lowmask64(bit);
      float v = 0.0f;
      bool seen = false;
#pragma unroll
      for (int w = 0; w < NMAX; ++w) {
        if (w < (int)n) {
          const unsigned long long pwv = spw[row0 + L][w];
          if ((pwv >> bit) & 1ull) {
            const float t = a.in_val[w][sbase[row0 + L][w] + __popcll(pwv & lm)];
            v = seen ? v + t : t;
            seen = true;
          }
        }
      }
      const uint64_t pos = wbase + k;
      if (pos < a.val_cap)
        for (uint32_t d = 0; d < a.ndst; ++d) a.dst_vals[d][pos] = v;
    }
  }
}

// ------------------------------------------------------- fused aggregate ----
// Dense syncs: mark + union + prefix + fold + pull in ONE kernel.  Block
// g owns the 8 extraction tiles [8g, 8g + 8) -- indices [65536 g, 65536 (g+1))
// -- whose I_s positions are [R0(g), R0(g+1)) (static: the universe chunk
// prefixes).  It takes the bitmap words [jA, jB) with jA = ceil(R0 / 64), so
// every word has one owner; the owner of a word that straddles two groups
// also reads up to 63 entries past its own (the next group's first ones) and
// skips its leading entries below 64 jA (the previous owner took them).
//  * each worker's entries of the group are a contiguous run of its part,
//    from the base its push scatter wrote for the group (no search);
//  * presence rows in shared memory (warp-aggregated atomicOr), no global
//    presence bitmaps, no clean-up stores;
//  * one block scan gives every worker's and U's word prefixes; a decoupled
//    look-back over the groups gives the block's first output position;
//  * then the HashBitmap words, the folded values (worker order,
//    zen/tensor.hpp:151-153) and the receivers' per-chunk value bases.
constexpr int kFusedThreads = 256;
constexpr uint32_t kFusedTiles = 8;  // tiles per group (65536 indices = 32 chunks)

// setup: per group g in [0, ngroups]: R0, jA = ceil(R0 / 64) (nw at the end),
// the first universe chunk c with cprefix >= 64 jA (nchunks at the end), and
// the largest span jA(g + 1) - jA(g)
__global__ void k_agg_groups(AggArgs a, uint32_t* span) {
  zen_dev::pdl_entry();
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > a.ngroups) return;
  auto jA_of = [&](uint32_t q, uint64_t* R0) {
    const uint64_t r = q < a.ngroups ? (uint64_t)a.cprefix[(uint64_t)q * 32 * a.n + a.s] : a.bs;
    if (R0) *R0 = r;
    return q < a.ngroups ? (r + 63) / 64 : a.nw;
  };
  uint64_t R0;
  const uint64_t jA = jA_of(g, &R0);
  uint64_t cs = a.nchunks;
  if (g < a.ngroups) {  // lower bound over the (nondecreasing) chunk prefixes
    uint64_t lo = 0, hi = a.nchunks;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if ((uint64_t)a.cprefix[mid * a.n + a.s] >= 64 * jA)
        hi = mid;
      else
        lo = mid + 1;
    }
    cs = lo;
    atomicMax(span, (uint32_t)(jA_of(g + 1, nullptr) - jA));
  }
  const_cast<uint4*>(a.gtab)[g] = make_uint4((uint32_t)R0, (uint32_t)jA, (uint32_t)cs, 0u);
}

template <int NMAX>
__global__ void __launch_bounds__(kFusedThreads, 7) k_agg_fused(AggArgs a) {  // 7/SM: one wave at 64M
  zen_dev::pdl_entry();
  extern __shared__ unsigned long long fsm[];
  __shared__ uint32_t s_lo[kMaxWorkers], s_skip[kMaxWorkers], s_off[kMaxWorkers + 1];
  __shared__ uint32_t s_stop[kFusedThreads / 32], s_sum[kFusedThreads / 32];
  __shared__ uint32_t s_wsum[33];
  const uint32_t n = a.n, s = a.s, lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t WB = a.span;
  unsigned long long* spw = fsm;                  // [n][WB] presence rows
  unsigned long long* sU = fsm + (size_t)n * WB;  // [WB] union
  uint32_t* spre = reinterpret_cast<uint32_t*>(sU + WB);  // [(n + 1) * WB] flat exclusive scan
  for (uint32_t i = threadIdx.x; i < n * WB; i += kFusedThreads) spw[i] = 0ull;
  if (threadIdx.x < n) s_skip[threadIdx.x] = 0;
  __syncthreads();
  // groups in block order: a block only waits on lower blocks, which were
  // dispatched before it (the single-pass scan's usual assumption)
  const uint32_t g = blockIdx.x;
  const uint4 G0 = a.gtab[g], G1 = a.gtab[g + 1];
  const uint32_t jA = G0.y, nwb = G1.y - G0.y;
  const uint64_t rA = 64ull * jA, rB = 64ull * G1.y;
  const bool ext = rB > (uint64_t)G1.x;  // the last word reaches into the next group
  if (threadIdx.x < n) {  // worker w's entries of the group: [gbase[g], gbase[g + 1])
    const uint32_t w = threadIdx.x;
    const uint32_t cnt = part_count(a, w);
    const uint32_t lo = a.in_gbase[w][g];
    const uint32_t hi = g + 1 < a.ngroups ? a.in_gbase[w][g + 1] : cnt;
    s_lo[w] = lo;
    s_off[w + 1] = (hi - lo) + (ext ? min(64u, cnt - hi) : 0u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < n; ++w) {
      const uint32_t l = s_off[w + 1];
      s_off[w] = acc;
      acc += l;
    }
    s_off[n] = acc;
  }
  __syncthreads();
  // phase 1: entries -> presence bits (4 per thread per round, loads first)
  const uint32_t E = s_off[n];
  constexpr int R = 4;
  for (uint32_t base = warp * 32; base < E; base += R * kFusedThreads) {  // warp-uniform
    uint32_t w[R], key[R];
    bool in[R];
    OwnWord ow[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint32_t i = base + q * kFusedThreads + lane;
      in[q] = i < E;
      w[q] = 0;
      if (in[q])
        while (i >= s_off[w[q] + 1]) ++w[q];
      key[q] = in[q] ? a.in_idx[w[q]][s_lo[w[q]] + (i - s_off[w[q]])] : 0u;
    }
#pragma unroll
    for (int q = 0; q < R; ++q)  // (a one-server universe: I_0 is every index, rank = index)
      ow[q] = a.whole ? OwnWord{~0ull, key[q] & ~63u, 0u} : a.own[in[q] ? key[q] >> 6 : 0];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (base + q * kFusedThreads >= E) break;  // warp-uniform
      bool live = in[q] && ((ow[q].mask >> (key[q] & 63u)) & 1ull);
      if (in[q] && !live) {
        atomicMin((unsigned long long*)&a.hdr->bad_index, (unsigned long long)key[q]);
        atomicOr(&a.hdr->status, kErrOutside);
      }
      const uint64_t r = ow[q].prefix + (uint64_t)__popcll(ow[q].mask & lowmask64(key[q] & 63u));
      if (live && r < rA) {
        atomicAdd(&s_skip[w[q]], 1u);  // the previous group's last word
        live = false;
      }
      live = live && r < rB;
      unsigned long long* word = live ? spw + (size_t)w[q] * WB + (uint32_t)((r >> 6) - jA) : nullptr;
      const uint64_t bit = live ? 1ull << (r & 63u) : 0ull;
      const uint32_t grp = __match_any_sync(0xffffffffu, (unsigned long long)word);
      const uint32_t lo = __reduce_or_sync(grp, (uint32_t)bit);
      const uint32_t hi = __reduce_or_sync(grp, (uint32_t)(bit >> 32));
      if (live && lane == (uint32_t)(__ffs(grp) - 1)) atomicOr(word, ((unsigned long long)hi << 32) | lo);
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nwb; j += kFusedThreads) {
    unsigned long long u = 0;
    for (uint32_t w = 0; w < n; ++w) u |= spw[(size_t)w * WB + j];
    sU[j] = u;
  }
  __syncthreads();
  // phase 2: one exclusive scan over the rows [w0 .. w(n-1), U] of nwb words
  const uint32_t L = (n + 1) * nwb;
  const uint32_t per = (L + kFusedThreads - 1) / kFusedThreads;
  const uint32_t f0 = min(threadIdx.x * per, L), f1 = min(f0 + per, L);
  uint32_t sum = 0;
  if (f0 < f1) {
    uint32_t row = f0 / nwb, j = f0 - row * nwb;
    for (uint32_t f = f0; f < f1; ++f) {
      sum += __popcll(row < n ? spw[(size_t)row * WB + j] : sU[j]);
      if (++j == nwb) { j = 0; ++row; }
    }
  }
  uint32_t tot;
  uint32_t run = block_exclusive_sum(sum, s_wsum, &tot);
  if (f0 < f1) {
    uint32_t row = f0 / nwb, j = f0 - row * nwb;
    for (uint32_t f = f0; f < f1; ++f) {
      spre[(size_t)row * WB + j] = run;
      run += __popcll(row < n ? spw[(size_t)row * WB + j] : sU[j]);
      if (++j == nwb) { j = 0; ++row; }
    }
  }
  __syncthreads();
  const uint32_t urow = n * WB;
  const uint32_t ub0 = nwb ? spre[urow] : tot;  // flat prefix where the U row starts
  // phase 3: decoupled look-back over the groups -> the block's first position.
  // The whole block reads 256 predecessors per round (nearest first) and stops
  // at the nearest one that already holds its inclusive prefix.
  const uint32_t utot = tot - ub0;
  const unsigned long long tag =
      (unsigned long long)(*(volatile uint32_t*)&a.hdr->iter & 0x3FFFFFFFu) << 34;
  // (relaxed: the look-back consumes nothing but these words themselves)
  if (threadIdx.x == 0) st_relaxed_gpu(&a.lbf[g], tag | ((g == 0 ? 2ull : 1ull) << 32) | utot);
  uint32_t excl = 0;
  // One worker: U is its own part, so the groups before g hold exactly the
  // part's entries before g -- the push scatter's base -- and no look-back.
  if (n == 1) excl = s_lo[0];
  for (int64_t k = n == 1 ? 0 : g; k > 0; k -= kFusedThreads) {  // block-uniform
    const int64_t idx = k - 1 - (int64_t)threadIdx.x;
    unsigned long long v = tag | (2ull << 32);  // before group 0: inclusive 0
    if (idx >= 0) {
      do {
        v = ld_relaxed_gpu(&a.lbf[idx]);
      } while ((v >> 34) != (tag >> 34) || ((v >> 32) & 3ull) == 0);
    }
    const uint32_t incl = __ballot_sync(0xffffffffu, ((v >> 32) & 3ull) == 2);
    if (lane == 0) s_stop[warp] = incl ? warp * 32 + (uint32_t)(__ffs(incl) - 1) : 0xFFFFFFFFu;
    __syncthreads();
    uint32_t stop = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < kFusedThreads / 32; ++q) stop = min(stop, s_stop[q]);
    const uint32_t part = __reduce_add_sync(0xffffffffu, threadIdx.x <= stop ? (uint32_t)v : 0u);
    if (lane == 0) s_sum[warp] = part;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kFusedThreads / 32; ++q) excl += s_sum[q];
    __syncthreads();  // s_stop / s_sum reuse
    if (stop != 0xFFFFFFFFu) break;
  }
  if (threadIdx.x == 0 && g != 0) st_relaxed_gpu(&a.lbf[g], tag | (2ull << 32) | (excl + utot));
  // phase 4a: the HashBitmap words
  for (uint32_t j = threadIdx.x; j < nwb; j += kFusedThreads)
    for (uint32_t d = 0; d < a.ndst; ++d) a.dst_bits[d][jA + j] = sU[j];
  // phase 4b: the receivers' value base per universe chunk
  for (uint32_t c = G0.z + threadIdx.x; c < G1.z; c += kFusedThreads) {
    const uint64_t P = a.cprefix[(uint64_t)c * n + s];
    uint32_t b = excl + utot;
    if (P < rB) {
      const uint32_t lj = (uint32_t)((P >> 6) - jA);
      b = excl + (spre[urow + lj] - ub0) + (uint32_t)__popcll(sU[lj] & lowmask64((uint32_t)(P & 63)));
    }
    for (uint32_t d = 0; d < a.ndst; ++d) a.dst_cbase[d][c] = b;
  }
  if (g == a.ngroups - 1 && threadIdx.x == 0) {
    for (uint32_t d = 0; d < a.ndst; ++d) a.dst_cbase[d][a.nchunks] = excl + utot;
    *a.agg_count = excl + utot;
  }
  // phase 4c: values, warps over 32-word spans; lanes expand set bits together
  for (uint32_t j0 = warp * 32; j0 < nwb; j0 += kFusedThreads) {
    const uint32_t j = j0 + lane;
    const unsigned long long U = j < nwb ? sU[j] : 0ull;
    const uint32_t c = __popcll(U);
    const uint32_t inc = warp_inclusive_sum(c);
    const uint32_t x = inc - c;
    const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
    const uint64_t wbase = (uint64_t)excl + (spre[urow + j0] - ub0);
    constexpr int B = NMAX <= 2 ? 4 : (NMAX <= 4 ? 2 : 1);  // expansions in flight per lane
    for (uint32_t k0 = 0; k0 < T; k0 += 32 * B) {  // warp-uniform
      float t[B][NMAX];
      uint32_t pres[B];
      uint64_t pos[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const uint32_t k = k0 + b * 32 + lane;
        uint32_t Lw = 0;
#pragma unroll
        for (uint32_t step = 16; step >= 1; step >>= 1) {
          const uint32_t xc = __shfl_sync(0xffffffffu, x, Lw + step);
          if (xc <= k) Lw += step;
        }
        const unsigned long long UL = __shfl_sync(0xffffffffu, U, Lw);
        const uint32_t xL = __shfl_sync(0xffffffffu, x, Lw);
        pres[b] = 0;
        pos[b] = wbase + k;
        if (k < T) {
          const uint32_t bit = (UL == ~0ull) ? k - xL : select64(UL, k - xL);
          const uint64_t lm = lowmask64(bit);
          const uint32_t jj = j0 + Lw;
#pragma unroll
          for (int w = 0; w < NMAX; ++w) {
            if (w >= (int)n) break;
            const unsigned long long pwv = spw[(size_t)w * WB + jj];
            if ((pwv >> bit) & 1ull) {  // every present worker's value load issued first
              const uint32_t e = s_lo[w] + s_skip[w] +
                                 (spre[(size_t)w * WB + jj] - spre[(size_t)w * WB]) +
                                 (uint32_t)__popcll(pwv & lm);
              t[b][w] = a.in_val[w][e];
              pres[b] |= 1u << w;
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (!pres[b]) continue;
        float v = 0.0f;
        bool seen = false;
#pragma unroll
        for (int w = 0; w < NMAX; ++w)
          if ((pres[b] >> w) & 1u) {  // worker order (zen/tensor.hpp:151-153)
            v = seen ? v + t[b][w] : t[b][w];
            seen = true;
          }
        if (pos[b] < a.val_cap)
          for (uint32_t d = 0; d < a.ndst; ++d) a.dst_vals[d][pos[b]] = v;
      }
    }
  }
}

// Pull signalling (rank mode): one block after the values kernel -- the kernel
// boundary completes every NVLink store of the encode -- publishes U_s and
// then the flag with release semantics at system scope.
__global__ void k_agg_signal(AggArgs a) {
  zen_dev::pdl_entry();
  __threadfence_system();
  const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
  const uint64_t u = *(volatile uint64_t*)a.agg_count;
  const uint32_t st = *(volatile uint32_t*)&a.hdr->status;
  const uint64_t bad = *(volatile uint64_t*)&a.hdr->bad_index;
  for (uint32_t d = threadIdx.x; d < a.ndst; d += blockDim.x) {
    a.dst_hdr[d]->agg_count = u;
    a.dst_hdr[d]->status = st;
    a.dst_hdr[d]->bad_index = bad;
    st_release_sys(&a.dst_hdr[d]->flag, (unsigned long long)iter);  // orders the three above
  }
}

// Rank mode: ONE warp waits for the n peers' flags (lane w polls flag w), so
// the heavy kernels behind it (launched early by PDL) never poll: a grid of
// CTAs spinning on the same lines with system-scope acquires slows the NVLink
// stores they wait for.
__global__ void k_wait_push(AggArgs a) {
  zen_dev::pdl_entry();
  const uint32_t w = threadIdx.x;
  if (w >= a.n) return;
  const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
  if (!wait_flag(&a.in_hdr[w]->flag, iter, kPeerTimeoutNs)) atomicOr(&a.hdr->status, kErrTimeout);
}

// ---------------------------------------------------------------- decode ----

// Word popcount prefix of each server's bitmap: block-local (2048 words per
// block, 8 consecutive words per thread) + block totals; the last block turns
// the totals into exclusive prefixes, per-server popcounts and |result|.
__global__ void __launch_bounds__(kPrefixThreads) k_bpre(DecodeArgs a) {
  zen_dev::pdl_entry();
  __shared__ uint32_t sscan[33];
  __shared__ uint32_t s_last;
  const uint32_t n = a.n;
  uint32_t s = 0;
  while (s + 1 < n && blockIdx.x >= a.blk_start[s + 1]) ++s;
  const uint32_t blk = blockIdx.x - a.blk_start[s];
  const unsigned long long* bits = a.bits[s];
  const uint64_t nw = a.nwords_s[s];
  const uint64_t w0 = (uint64_t)blk * kPrefixBlockWords + threadIdx.x * (uint64_t)kWPT;
  unsigned long long v[kWPT];
  const bool live = bits && w0 < nw;
  if (live) load8(bits + w0, v);  // rows are padded to 8 words
  uint32_t c[kWPT];
  uint32_t local = 0;
#pragma unroll
  for (int i = 0; i < kWPT; ++i) {
    c[i] = local;
    local += live ? (uint32_t)__popcll(v[i]) : 0u;
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum(local, sscan, &tot);
  if (live) {
#pragma unroll
    for (int i = 0; i < kWPT; ++i) c[i] += ex;
    store8u(a.bpre + s * a.words_stride + w0, c);
  }
  if (threadIdx.x == 0) {
    a.bpre_blk[s * a.blk_stride + blk] = tot;
    __threadfence();
    s_last = (atomicAdd(a.done, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  __shared__ uint64_t totals[kMaxWorkers];
  for (uint32_t x = warp; x < n; x += kPrefixThreads / 32) {
    const uint32_t nb = a.blk_start[x + 1] - a.blk_start[x];
    const uint32_t total = warp_exscan_l2(a.bpre_blk + x * a.blk_stride, nb);
    if (lane == 0) {
      a.popc_total[x] = total;
      totals[x] = total;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t u = 0;
    for (uint32_t x = 0; x < n; ++x) u += totals[x];
    *a.out_count = u;
    *a.done = 0;
  }
}

__global__ void k_wait_pull(DecodeArgs a) {
  zen_dev::pdl_entry();
  const uint32_t s = threadIdx.x;
  if (s >= a.n || !a.bits[s]) return;
  const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
  if (!wait_flag(&a.pull_hdr[s]->flag, iter, kPeerTimeoutNs)) atomicOr(&a.hdr->status, kErrTimeout);
}

// popcount of server s's bitmap bits [0, P)
__device__ __forceinline__ uint64_t bitmap_prefix(const DecodeArgs& a, uint32_t s, uint64_t P) {
  const uint64_t j = P >> 6;
  const uint32_t o = (uint32_t)(P & 63);
  if (j >= a.nwords_s[s]) return a.popc_total[s];
  return (uint64_t)a.bpre_blk[s * a.blk_stride + j / kPrefixBlockWords] +
         a.bpre[s * a.words_stride + j] + (uint64_t)__popcll(a.bits[s][j] & lowmask64(o));
}

// One warp per 32-word chunk of the global index space (one word per lane),
// warps fully independent.  Lane s first takes server s's slice of the chunk:
// bits [cp_s, cpn_s) of its bitmap and the number of its set bits below them
// (base_s, from the k_bpre prefixes).  A chunk whose slices are all empty
// ends there (most chunks at embedding sparsity).  Otherwise, per word, each
// server's owned positions are a contiguous bit range of its bitmap,
// deposited into the owner mask; the value index of a word's first bit of
// server s is base_s + (s's set bits in the chunk's earlier words), and its
// first output position is sum_s base_s + (set bits of all servers in the
// earlier words): both are warp scans, so no per-word prefix is read and no
// block-wide scan is needed.  Servers go in groups of four, all loads of a
// group issued before use, four counts packed per 64-bit scan.  Warps then
// expand their set bits cooperatively (coalesced stores).
constexpr int kDecThreads = 128;

__device__ __forceinline__ uint32_t field16(uint64_t v, int g) {
  return (uint32_t)(v >> (16 * g)) & 0xFFFFu;
}

template <int NMAX>
__global__ void __launch_bounds__(kDecThreads) k_decode(DecodeArgs a, uint64_t nwords) {
  zen_dev::pdl_entry();
  if (a.wait_pull && a.gate)  // rank mode: the n pulls have arrived (no k_wait_pull)
    arrival_gate(a.n,
                 [&](uint32_t s) {
                   return a.bits[s] ? (const unsigned long long*)&a.pull_hdr[s]->flag : nullptr;
                 },
                 &a.hdr->go[1], *(volatile uint32_t*)&a.hdr->iter, &a.hdr->status);
  constexpr int kDecGroup = NMAX < 4 ? NMAX : 4;  // servers per packed scan
  __shared__ unsigned long long spres[kDecThreads][NMAX];
  __shared__ uint32_t svb[kDecThreads][NMAX];
  __shared__ unsigned long long spl[kDecThreads][4];
  const uint32_t n = a.n, lane = lane_id(), np = a.nplanes;
  const uint64_t w = (uint64_t)blockIdx.x * kDecThreads + threadIdx.x;
  const uint64_t chunk = w >> 5;
  const uint64_t nchunks = (nwords + 31) / 32;
  if (chunk >= nchunks) return;  // warp-uniform
  const bool valid = w < nwords;
  // server `lane`'s slice of the chunk and its value base
  uint64_t cp = 0, base = 0, end = 0;
  if (lane < n && a.bits[lane]) {
    cp = a.cprefix[chunk * n + lane];
    if (a.cbase) {  // BP: the server sent its value base for every global chunk
      base = a.cbase[lane][chunk];
      end = a.cbase[lane][chunk + 1];
    } else {
      const uint64_t cpn =
          (chunk + 1 < nchunks) ? (uint64_t)a.cprefix[(chunk + 1) * n + lane] : a.bs[lane];
      base = bitmap_prefix(a, lane, cp);
      end = (cpn > cp) ? bitmap_prefix(a, lane, cpn) : base;
    }
  }
  if (a.cbase && w == 0 && lane == 0) {  // |result| = sum_s U_s (k_bpre's job otherwise)
    uint64_t u = 0;
    for (uint32_t s = 0; s < n; ++s) u += a.bits[s] ? a.cbase[s][nchunks] : 0u;
    *a.out_count = u;
  }
  if (!__any_sync(0xffffffffu, end > base)) return;
  uint64_t ob = base;  // chunk's first output position = sum_s base_s
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ob += __shfl_xor_sync(0xffffffffu, ob, o);
  unsigned long long pl[4] = {0, 0, 0, 0};
  const uint64_t vmask = valid ? valid_mask(a.m, w) : 0ull;
  if (valid) {
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j)
      if (j < np) pl[j] = a.planes[w * np + j];
  }
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) spl[threadIdx.x][j] = pl[j];
  uint64_t G = 0;
#pragma unroll
  for (int s0 = 0; s0 < NMAX; s0 += kDecGroup) {
    uint64_t ms[kDecGroup];
    uint32_t c[kDecGroup];
    uint64_t packed = 0;
#pragma unroll
    for (int g = 0; g < kDecGroup; ++g) {
      const uint32_t s = s0 + g;
      ms[g] = (s < n) ? owner_mask4(pl, np, s, vmask) : 0ull;
      c[g] = __popcll(ms[g]);
      packed |= (uint64_t)c[g] << (16 * g);
    }
    const uint64_t incp = warp_inclusive_sum(packed);  // four 16-bit fields, no carries
    uint64_t P[kDecGroup];
    unsigned long long lo[kDecGroup], hi[kDecGroup];
#pragma unroll
    for (int g = 0; g < kDecGroup; ++g) {
      const uint32_t s = s0 + g;
      P[g] = __shfl_sync(0xffffffffu, cp, s & 31) + field16(incp, g) - c[g];
      lo[g] = hi[g] = 0ull;
      const unsigned long long* bits = (s < n) ? a.bits[s] : nullptr;
      if (bits && c[g]) {
        const uint64_t j = P[g] >> 6;
        lo[g] = bits[j];
        if ((P[g] & 63) + c[g] > 64) hi[g] = bits[j + 1];
      }
    }
    uint64_t xb[kDecGroup];
    uint64_t pk = 0;
#pragma unroll
    for (int g = 0; g < kDecGroup; ++g) {
      const uint32_t o = (uint32_t)(P[g] & 63);
      uint64_t x = lo[g] >> o;
      if (o + c[g] > 64) x |= (uint64_t)hi[g] << (64 - o);
      xb[g] = c[g] ? (x & lowmask64(c[g])) : 0ull;
      pk |= (uint64_t)__popcll(xb[g]) << (16 * g);
    }
    const uint64_t incv = warp_inclusive_sum(pk);
#pragma unroll
    for (int g = 0; g < kDecGroup; ++g) {
      const uint32_t s = s0 + g;
      if (s >= NMAX) break;
      const uint64_t bs_ = __shfl_sync(0xffffffffu, base, s & 31);
      unsigned long long pres = 0;
      if (xb[g]) {
        pres = (c[g] == 64) ? xb[g] : deposit64(xb[g], ms[g]);
        G |= pres;
      }
      spres[threadIdx.x][s] = pres;
      svb[threadIdx.x][s] = (uint32_t)(bs_ + field16(incv, g) - field16(pk, g));
    }
  }
  __syncwarp();
  const uint32_t cnt = __popcll(G);
  const uint32_t inc = warp_inclusive_sum(cnt);
  const uint32_t x = inc - cnt;
  const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
  const uint32_t row0 = threadIdx.x & ~31u;
  const uint64_t wrow = (w & ~31ull);
  if (n == 1) {
    // One server and every non-empty word of the chunk full (dense rows):
    // the warp expands word by word, lane l taking bits l and 32 + l --
    // consecutive outputs and consecutive values, no per-bit search.
    const uint32_t nz = __ballot_sync(0xffffffffu, G != 0ull);
    if (__ballot_sync(0xffffffffu, G == ~0ull) == nz) {
      for (uint32_t m = nz; m; m &= m - 1) {
        const uint32_t L = (uint32_t)(__ffs(m) - 1);
        const uint64_t o = ob + __shfl_sync(0xffffffffu, x, L);
        const uint32_t vb = svb[row0 + L][0];
        const uint64_t idx0 = (wrow + L) * 64;
        const float v0 = a.vals[0][vb + lane], v1 = a.vals[0][vb + 32 + lane];
        if (o + lane < a.out_cap) {
          a.out_idx[o + lane] = idx0 + lane;
          a.out_val[o + lane] = v0;
        }
        if (o + 32 + lane < a.out_cap) {
          a.out_idx[o + 32 + lane] = idx0 + 32 + lane;
          a.out_val[o + 32 + lane] = v1;
        }
      }
      return;
    }
  }
  constexpr int UNR = 4;  // outputs per lane per pass, loads issued first
  for (uint32_t k0 = 0; k0 < T; k0 += 32 * UNR) {
    float v[UNR];
    uint64_t oidx[UNR];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const uint32_t k = k0 + q * 32 + lane;
      uint32_t L = 0;
#pragma unroll
      for (uint32_t step = 16; step >= 1; step >>= 1) {
        const uint32_t xc = __shfl_sync(0xffffffffu, x, L + step);
        if (xc <= k) L += step;
      }
      const unsigned long long GL = __shfl_sync(0xffffffffu, G, L);
      const uint32_t xL = __shfl_sync(0xffffffffu, x, L);
      if (k < T) {
        const uint32_t bit = (GL == ~0ull) ? k - xL : select64(GL, k - xL);  // full rows: direct
        uint32_t s = 0;  // owner of the bit, from the word's owner planes
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j)
          if (j < np) s |= (uint32_t)((spl[row0 + L][j] >> bit) & 1ull) << j;
        const unsigned long long p = spres[row0 + L][s];
        v[q] = a.vals[s][svb[row0 + L][s] + __popcll(p & lowmask64(bit))];
        oidx[q] = (wrow + L) * 64 + bit;
      }
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const uint32_t k = k0 + q * 32 + lane;
      const uint64_t pos = ob + k;
      if (k < T && pos < a.out_cap) {
        a.out_idx[pos] = oidx[q];
        a.out_val[pos] = v[q];
      }
    }
  }
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (unsigned)(g < cap ? g : cap);
}

}  // namespace

void launch_tables_planes(uint64_t m, uint32_t n, uint64_t pc, uint32_t nplanes,
                          unsigned long long* planes, uint32_t* chunk_cnt, cudaStream_t stream) {
  const uint64_t nwords = (m + 63) / 64;
  launch_k(k_tables_planes, grid_for(nwords, 256, 148 * 16), 256, 0, stream, m, n, pc, nplanes, planes,
                                                                        chunk_cnt, nwords);
  count_launch();
}

void launch_tables_scan(uint32_t* cc, uint64_t nchunks, uint32_t n, uint64_t* totals,
                        cudaStream_t stream) {
  launch_k(k_tables_scan, 1, 1024, 0, stream, cc, nchunks, n, totals);
  count_launch();
}

void launch_tables_own(uint64_t m, uint32_t n, uint32_t s, uint32_t nplanes,
                       const unsigned long long* planes, const uint32_t* cprefix, OwnWord* own,
                       uint32_t* sel, uint64_t nsel, cudaStream_t stream) {
  const uint64_t nwords = (m + 63) / 64;
  launch_k(k_tables_own, grid_for(nwords, 256, 148 * 16), 256, 0, stream, m, n, s, nplanes, planes,
                                                                     cprefix, own, sel, nsel,
                                                                     nwords);
  count_launch();
}

void launch_agg_groups(const AggArgs& a, uint32_t* span, cudaStream_t stream) {
  launch_k(k_agg_groups, (a.ngroups + 1 + 255) / 256, 256, 0, stream, a, span);
  count_launch();
}

void launch_aggregate(const AggArgs& a, cudaStream_t stream, bool marked, bool fused) {
  if (fused) {
    if (a.wait_push) {
      launch_k(k_wait_push, 1, 32, 0, stream, a);
      count_launch();
    }
    const size_t sm = agg_fused_smem(a.n, a.span);
    auto kern = a.n <= 1 ? k_agg_fused<1>
              : a.n <= 2 ? k_agg_fused<2>
              : a.n <= 4 ? k_agg_fused<4>
              : a.n <= 8 ? k_agg_fused<8> : k_agg_fused<16>;
    if (sm > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_k(kern, a.ngroups, kFusedThreads, sm, stream, a);
    count_launch();
    if (a.dst_hdr) {
      launch_k(k_agg_signal, 1, 32, 0, stream, a);
      count_launch();
    }
    return;
  }
  // a.pw is all-zero here: zeroed at allocation, re-zeroed by k_agg_values
  if (a.wait_push && !a.gate) {
    launch_k(k_wait_push, 1, 32, 0, stream, a);
    count_launch();
  }
  // (one worker, dense sync: the union builds U from the entries, no marks)
  const bool from_entries = a.whole && a.n == 1 && !a.pre_min && a.solo_gbase;
  if (!marked && !from_entries) {
    launch_k(k_agg_mark, 148 * 8, kAggThreads, 0, stream, a);
    count_launch();
  }
  launch_k(k_agg_union, a.nblk, kPrefixThreads, 0, stream, a);
  // (one worker of a one-server universe: the values kernel only writes the chunk bases)
  const bool solo = a.whole && a.n == 1 && !a.pre_min;
  const unsigned g = (unsigned)(((solo ? a.nchunks + 1 : a.nw) + kValThreads - 1) / kValThreads);
  if (a.n <= 2)
    launch_k(k_agg_values<2>, g, kValThreads, 0, stream, a);
  else if (a.n <= 4)
    launch_k(k_agg_values<4>, g, kValThreads, 0, stream, a);
  else if (a.n <= 8)
    launch_k(k_agg_values<8>, g, kValThreads, 0, stream, a);
  else
    launch_k(k_agg_values<16>, g, kValThreads, 0, stream, a);
  for (int i = 0; i < 2; ++i) count_launch();
  if (a.dst_hdr) {
    launch_k(k_agg_signal, 1, 32, 0, stream, a);
    count_launch();
  }
}

void launch_decode_parts(const DecodeArgs& a, cudaStream_t stream) {
  const uint64_t nwords = (a.m + 63) / 64;
  const uint32_t ntiles = (uint32_t)((nwords + kDecThreads - 1) / kDecThreads);
  if (a.wait_pull && !a.gate) {
    launch_k(k_wait_pull, 1, 32, 0, stream, a);
    count_launch();
  }
  if (!a.cbase) {
    launch_k(k_bpre, a.total_blocks ? a.total_blocks : 1, kPrefixThreads, 0, stream, a);
    count_launch();
  }
  constexpr unsigned T = kDecThreads;
  if (a.n <= 2)
    launch_k(k_decode<2>, ntiles, T, 0, stream, a, nwords);
  else if (a.n <= 4)
    launch_k(k_decode<4>, ntiles, T, 0, stream, a, nwords);
  else if (a.n <= 8)
    launch_k(k_decode<8>, ntiles, T, 0, stream, a, nwords);
  else
    launch_k(k_decode<16>, ntiles, T, 0, stream, a, nwords);
  count_launch();
}

}  // namespace zen
