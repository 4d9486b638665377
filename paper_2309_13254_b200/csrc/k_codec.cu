// k_codec.cu -- the owner side of Balanced Parallelism on sm_100a.
//
//  tables    : HashUniverseTable (zen/codec.hpp:47-72) without materialising
//              the M x 8 B sorted lists: per 64-index word, ceil(log2 n) owner
//              bit planes (the information minimum), per-32-word chunk prefix
//              counts per server, and for each local server a {mask, rank
//              base} record per word plus select samples every 4096 ranks.
//  aggregate : per-owner sum (merge_sum left fold in worker order,
//              zen/schemes.hpp:375-380; zen/tensor.hpp:133-167) FUSED with the
//              HashBitmap encode (zen/codec.hpp:266-277).  A block owns 4096
//              consecutive ranks of I_s: it binary-searches each worker's
//              sorted part for the chunk, accumulates in shared memory worker
//              by worker (bit-exact fold order, zero sums kept), and emits the
//              64 bitmap words + the compacted values -- optionally straight
//              into every receiver's pull inbox over NVLink (the pull fused
//              with the encode).  Value offsets come from a decoupled look-back.
//  decode    : all servers' (bitmap, values) -> the global ascending result
//              (decode zen/codec.hpp:333-347 + merge_disjoint
//              zen/schemes.hpp:91-113).  Per global word, each server's owned
//              positions are a contiguous bit range of its bitmap; a software
//              pdep deposits them into the owner mask, and a popcount prefix of
//              each bitmap locates the values.  Output order falls out of the
//              global word order: no k-way merge.
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
      // select sample: the word holding rank q*kAggChunk
      const uint64_t q = ((uint64_t)prefix + kAggChunk - 1) / kAggChunk;
      const uint64_t r = q * kAggChunk;
      if (c && r < (uint64_t)prefix + c && q < nsel)
        sel[q] = (uint32_t)(w * 64 + select64(ms, (uint32_t)(r - prefix)));
    }
  }
}

// ------------------------------------------------------------- aggregate ----

constexpr int kAggThreads = 256;

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kAggThreads) k_aggregate(AggArgs a, uint32_t nq) {
  __shared__ float acc[kAggChunk];
  __shared__ uint32_t pres[kAggChunk / 32];
  __shared__ uint32_t rng[2 * kMaxWorkers];
  __shared__ uint32_t sscan[33];
  __shared__ uint32_t s_ticket;
  __shared__ uint64_t s_base;
  const uint32_t n = a.n, s = a.s;
  const uint32_t tag = *(volatile uint32_t*)&a.lb_ctl->tag;
  const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
  if (a.wait_push && threadIdx.x < n) {
    if (!wait_flag(&a.in_hdr[threadIdx.x]->flag, iter, kPeerTimeoutNs))
      atomicOr(&a.hdr->status, kErrTimeout);
  }
  __syncthreads();
  const uint32_t q = take_ticket(a.lb_ctl, &s_ticket);
  const uint32_t lo = a.sel[q], hi = a.sel[q + 1];
  if (threadIdx.x < 2 * n) {
    const uint32_t w = threadIdx.x >> 1;
    const uint32_t cnt = a.in_hdr ? *(volatile uint32_t*)&a.in_hdr[w]->counts[s]
                                  : (uint32_t)a.in_count[w];
    rng[threadIdx.x] = lower_bound_u32(a.in_idx[w], cnt, (threadIdx.x & 1) ? hi : lo);
  }
  if (threadIdx.x < kAggChunk / 32) pres[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t r0 = (uint64_t)q * kAggChunk;
  for (uint32_t w = 0; w < n; ++w) {  // worker order = the reference's left fold
    const uint32_t* __restrict__ ix = a.in_idx[w];
    const float* __restrict__ vx = a.in_val[w];
    for (uint32_t e = rng[2 * w] + threadIdx.x; e < rng[2 * w + 1]; e += kAggThreads) {
      const uint32_t key = ix[e];
      const float v = vx[e];
      const OwnWord ow = a.own[key >> 6];
      const uint32_t bit = key & 63u;
      if (!((ow.mask >> bit) & 1ull)) {
        atomicMin((unsigned long long*)&a.hdr->bad_index, (unsigned long long)key);
        atomicOr(&a.hdr->status, kErrOutside);
        continue;
      }
      const uint32_t r = (uint32_t)(ow.prefix + __popcll(ow.mask & lowmask64(bit)) - r0);
      const uint32_t m = 1u << (r & 31);
      if (pres[r >> 5] & m) {
        acc[r] += v;
      } else {
        acc[r] = v;
        atomicOr(&pres[r >> 5], m);
      }
    }
    __syncthreads();
  }
  // 16 ranks per thread, in rank order
  const uint32_t bits16 = (pres[threadIdx.x >> 1] >> ((threadIdx.x & 1) * 16)) & 0xFFFFu;
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum((uint32_t)__popc(bits16), sscan, &tot);
  if (threadIdx.x < 32) {
    const uint64_t base = lookback_warp(a.lb_status, q, tag, tot);
    if (threadIdx.x == 0) {
      s_base = base;
      if (q == nq - 1) *a.agg_count = base + tot;
    }
  }
  __syncthreads();
  const uint64_t nwords = (a.bs + 63) / 64;
  if (threadIdx.x < kAggChunk / 64) {
    const uint64_t j = (uint64_t)q * (kAggChunk / 64) + threadIdx.x;
    if (j < nwords) {
      const unsigned long long word =
          (unsigned long long)pres[2 * threadIdx.x] | ((unsigned long long)pres[2 * threadIdx.x + 1] << 32);
      for (uint32_t d = 0; d < a.ndst; ++d) a.dst_bits[d][j] = word;
    }
  }
  if (bits16) {
    uint64_t pos = s_base + ex;
    uint32_t b = bits16;
    while (b) {
      const uint32_t i = __ffs(b) - 1;
      b &= b - 1;
      const float v = acc[threadIdx.x * 16 + i];
      if (pos < a.val_cap)
        for (uint32_t d = 0; d < a.ndst; ++d) a.dst_vals[d][pos] = v;
      ++pos;
    }
  }
  const bool last = finish_tile(a.lb_ctl, nq, a.dst_hdr != nullptr);
  if (last && a.dst_hdr) {  // pull signalling: publish U_s, then the flag
    __threadfence_system();
    const uint64_t u = *(volatile uint64_t*)a.agg_count;
    const uint32_t st = *(volatile uint32_t*)&a.hdr->status;
    const uint64_t bad = *(volatile uint64_t*)&a.hdr->bad_index;
    for (uint32_t d = threadIdx.x; d < a.ndst; d += kAggThreads) {
      a.dst_hdr[d]->agg_count = u;
      a.dst_hdr[d]->status = st;
      a.dst_hdr[d]->bad_index = bad;
    }
    __syncthreads();
    __threadfence_system();
    for (uint32_t d = threadIdx.x; d < a.ndst; d += kAggThreads)
      st_release_sys(&a.dst_hdr[d]->flag, (unsigned long long)iter);
  }
}

// ---------------------------------------------------------------- decode ----

// word popcount prefix of each server's bitmap, block-local (8192 words per
// block; 256 threads x 32 contiguous words)
__global__ void __launch_bounds__(256) k_bpre(DecodeArgs a, const uint32_t* blk_start,
                                             const uint64_t* nwords_s) {
  __shared__ uint32_t sscan[33];
  const uint32_t n = a.n;
  const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
  if (a.wait_pull && threadIdx.x < n) {
    if (a.bits[threadIdx.x] &&
        !wait_flag(&a.pull_hdr[threadIdx.x]->flag, iter, kPeerTimeoutNs))
      atomicOr(&a.hdr->status, kErrTimeout);
  }
  __syncthreads();
  uint32_t s = 0;
  while (s + 1 < n && blockIdx.x >= blk_start[s + 1]) ++s;
  const uint32_t blk = blockIdx.x - blk_start[s];
  const unsigned long long* bits = a.bits[s];
  const uint64_t nw = nwords_s[s];
  const uint64_t w0 = (uint64_t)blk * kPrefixBlockWords + threadIdx.x * 32ull;
  uint32_t c[32];
  uint32_t local = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    c[i] = local;
    const uint64_t w = w0 + i;
    local += (bits && w < nw) ? (uint32_t)__popcll(bits[w]) : 0u;
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum(local, sscan, &tot);
  uint32_t* out = a.bpre + s * a.words_stride;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint64_t w = w0 + i;
    if (w < nw) out[w] = ex + c[i];
  }
  if (threadIdx.x == 0) a.bpre_blk[s * a.blk_stride + blk] = tot;
}

__global__ void k_bpre_scan(DecodeArgs a, const uint32_t* blk_start) {
  // one warp per server
  const uint32_t s = threadIdx.x >> 5;
  if (s >= a.n) return;
  const uint32_t nb = blk_start[s + 1] - blk_start[s];
  uint32_t* b = a.bpre_blk + s * a.blk_stride;
  uint32_t carry = 0;
  for (uint32_t i0 = 0; i0 < nb; i0 += 32) {
    const uint32_t i = i0 + lane_id();
    const uint32_t v = i < nb ? b[i] : 0u;
    const uint32_t inc = warp_inclusive_sum(v);
    if (i < nb) b[i] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane_id() == 0) a.popc_total[s] = carry;
}

template <int NMAX>
__global__ void __launch_bounds__(256) k_decode(DecodeArgs a, uint64_t nwords, uint32_t ntiles) {
  __shared__ uint32_t sscan[33];
  __shared__ uint32_t s_ticket;
  __shared__ uint64_t s_base;
  const uint32_t n = a.n;
  const uint32_t tag = *(volatile uint32_t*)&a.lb_ctl->tag;
  const uint32_t tile = take_ticket(a.lb_ctl, &s_ticket);
  const uint64_t w = (uint64_t)tile * kDecodeTileWords + threadIdx.x;
  const bool valid = w < nwords;
  unsigned long long pl[4] = {0, 0, 0, 0};
  const uint64_t vmask = valid ? valid_mask(a.m, w) : 0ull;
  if (valid) {
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j)
      if (j < a.nplanes) pl[j] = a.planes[w * a.nplanes + j];
  }
  const uint64_t chunk = w >> 5;
  uint64_t pres[NMAX];
  uint32_t vbase[NMAX];
  uint64_t G = 0;
#pragma unroll
  for (int s = 0; s < NMAX; ++s) {
    pres[s] = 0;
    vbase[s] = 0;
    if (s < (int)n) {
      const uint64_t ms = owner_mask4(pl, a.nplanes, (uint32_t)s, vmask);
      const uint32_t c = __popcll(ms);
      const uint32_t inc = warp_inclusive_sum(c);
      const unsigned long long* bits = a.bits[s];
      if (bits && c) {
        const uint64_t P = (uint64_t)a.cprefix[chunk * n + s] + inc - c;
        const uint64_t j = P >> 6;
        const uint32_t o = (uint32_t)(P & 63);
        const unsigned long long w0 = bits[j];
        uint64_t x = w0 >> o;
        if (o + c > 64) x |= (uint64_t)bits[j + 1] << (64 - o);
        x &= lowmask64(c);
        if (x) {
          pres[s] = deposit64(x, ms);
          vbase[s] = a.bpre_blk[s * a.blk_stride + j / kPrefixBlockWords] +
                     a.bpre[s * a.words_stride + j] + (uint32_t)__popcll(w0 & lowmask64(o));
          G |= pres[s];
        }
      }
    }
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum((uint32_t)__popcll(G), sscan, &tot);
  if (threadIdx.x < 32) {
    const uint64_t base = lookback_warp(a.lb_status, tile, tag, tot);
    if (threadIdx.x == 0) {
      s_base = base;
      if (tile == ntiles - 1) *a.out_count = base + tot;
    }
  }
  __syncthreads();
  uint64_t pos = s_base + ex;
  while (G) {
    const uint32_t i = __ffsll((long long)G) - 1;
    G &= G - 1;
    float v = 0.0f;
#pragma unroll
    for (int s = 0; s < NMAX; ++s) {
      if ((pres[s] >> i) & 1ull) {
        v = a.vals[s][vbase[s] + __popcll(pres[s] & lowmask64(i))];
      }
    }
    if (pos < a.out_cap) {
      a.out_idx[pos] = w * 64 + i;
      a.out_val[pos] = v;
    }
    ++pos;
  }
  finish_tile(a.lb_ctl, ntiles);
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
  k_tables_planes<<<grid_for(nwords, 256, 148 * 16), 256, 0, stream>>>(m, n, pc, nplanes, planes,
                                                                        chunk_cnt, nwords);
  count_launch();
}

void launch_tables_scan(uint32_t* cc, uint64_t nchunks, uint32_t n, uint64_t* totals,
                        cudaStream_t stream) {
  k_tables_scan<<<1, 1024, 0, stream>>>(cc, nchunks, n, totals);
  count_launch();
}

void launch_tables_own(uint64_t m, uint32_t n, uint32_t s, uint32_t nplanes,
                       const unsigned long long* planes, const uint32_t* cprefix, OwnWord* own,
                       uint32_t* sel, uint64_t nsel, cudaStream_t stream) {
  const uint64_t nwords = (m + 63) / 64;
  k_tables_own<<<grid_for(nwords, 256, 148 * 16), 256, 0, stream>>>(m, n, s, nplanes, planes,
                                                                     cprefix, own, sel, nsel,
                                                                     nwords);
  count_launch();
}

void launch_aggregate(const AggArgs& a, cudaStream_t stream) {
  const uint32_t nq = (uint32_t)((a.bs + kAggChunk - 1) / kAggChunk);
  k_aggregate<<<nq ? nq : 1, kAggThreads, 0, stream>>>(a, nq ? nq : 1);
  count_launch();
}

// blk_start / nwords_s live in device memory right after the DecodeArgs
// scratch (passed by the orchestrator through bpre_blk's tail); see engine.
void launch_decode_parts(const DecodeArgs& a, const uint32_t* d_blk_start,
                         const uint64_t* d_nwords_s, uint32_t total_blocks, cudaStream_t stream) {
  k_bpre<<<total_blocks ? total_blocks : 1, 256, 0, stream>>>(a, d_blk_start, d_nwords_s);
  k_bpre_scan<<<1, 32 * kMaxWorkers, 0, stream>>>(a, d_blk_start);
  const uint64_t nwords = (a.m + 63) / 64;
  const uint32_t ntiles = (uint32_t)((nwords + kDecodeTileWords - 1) / kDecodeTileWords);
  if (a.n <= 2)
    k_decode<2><<<ntiles, 256, 0, stream>>>(a, nwords, ntiles);
  else if (a.n <= 4)
    k_decode<4><<<ntiles, 256, 0, stream>>>(a, nwords, ntiles);
  else if (a.n <= 8)
    k_decode<8><<<ntiles, 256, 0, stream>>>(a, nwords, ntiles);
  else
    k_decode<16><<<ntiles, 256, 0, stream>>>(a, nwords, ntiles);
  for (int i = 0; i < 3; ++i) count_launch();
}

}  // namespace zen
