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

__device__ __forceinline__ uint32_t part_count(const AggArgs& a, uint32_t w) {
  return a.in_hdr ? *(volatile const uint32_t*)&a.in_hdr[w]->counts[a.s] : (uint32_t)a.in_count[w];
}

__device__ __forceinline__ void wait_push(const AggArgs& a) {
  if (a.wait_push && threadIdx.x < a.n) {
    const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
    if (!wait_flag(&a.in_hdr[threadIdx.x]->flag, iter, kPeerTimeoutNs))
      atomicOr(&a.hdr->status, kErrTimeout);
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t rank_of(const OwnWord* own, uint32_t key) {
  const OwnWord ow = own[key >> 6];
  return ow.prefix + (uint32_t)__popcll(ow.mask & lowmask64(key & 63u));
}

// Phase 1: rank of every received entry in I_s (HashBitmap position,
// zen/codec.hpp:146-158) and, per worker, the first entry of every chunk.
// Thread per (w, e) with e in [0, cnt_w] (e = cnt_w is the end sentinel).
__global__ void __launch_bounds__(kAggThreads) k_agg_rank(AggArgs a) {
  __shared__ uint64_t pre[kMaxWorkers + 1];
  wait_push(a);
  const uint32_t n = a.n;
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (uint32_t w = 0; w < n; ++w) {
      pre[w] = acc;
      acc += (uint64_t)part_count(a, w) + 1;
    }
    pre[n] = acc;
  }
  __syncthreads();
  const uint64_t total = pre[n];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t w = 0;
    while (i >= pre[w + 1]) ++w;
    const uint32_t e = (uint32_t)(i - pre[w]);
    const uint32_t cnt = (uint32_t)(pre[w + 1] - pre[w] - 1);
    const uint32_t* ix = a.in_idx[w];
    int64_t c_e;
    if (e < cnt) {
      const uint32_t key = ix[e];
      const OwnWord ow = a.own[key >> 6];
      if (!((ow.mask >> (key & 63u)) & 1ull)) {
        atomicMin((unsigned long long*)&a.hdr->bad_index, (unsigned long long)key);
        atomicOr(&a.hdr->status, kErrOutside);
      }
      const uint32_t r = ow.prefix + (uint32_t)__popcll(ow.mask & lowmask64(key & 63u));
      a.rank[(uint64_t)w * a.cap + e] = r;
      c_e = r / kAggChunk;
    } else {
      c_e = a.nq;
    }
    const int64_t c_prev = e == 0 ? -1 : (int64_t)(rank_of(a.own, ix[e - 1]) / kAggChunk);
    uint32_t* st = a.start + (uint64_t)w * (a.nq + 1);
    for (int64_t c = c_prev + 1; c <= c_e; ++c) st[c] = e;
  }
}

// Phase 2: one block per chunk of kAggChunk ranks.  Workers are folded in
// order 0..n-1 (the reference's left fold, zen/schemes.hpp:377-378), in shared
// memory; zero sums stay present.  The chunk's 64 bitmap words go straight to
// every destination; its values are compacted into a chunk-local staging slot.
__global__ void __launch_bounds__(kAggThreads) k_agg_chunk(AggArgs a) {
  __shared__ float acc[kAggChunk];
  __shared__ uint32_t pres[kAggChunk / 32];
  __shared__ uint32_t sscan[33];
  const uint32_t n = a.n, q = blockIdx.x;
  if (threadIdx.x < kAggChunk / 32) pres[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t r0 = q * kAggChunk;
  for (uint32_t w = 0; w < n; ++w) {
    const uint32_t* st = a.start + (uint64_t)w * (a.nq + 1);
    const uint32_t b = st[q], e = st[q + 1];
    const uint32_t* __restrict__ rk = a.rank + (uint64_t)w * a.cap;
    const float* __restrict__ vx = a.in_val[w];
    for (uint32_t i = b + threadIdx.x; i < e; i += kAggThreads) {
      const uint32_t r = rk[i] - r0;
      const float v = vx[i];
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
  const uint64_t nwords = (a.bs + 63) / 64;
  if (threadIdx.x < kAggChunk / 64) {
    const uint64_t j = (uint64_t)q * (kAggChunk / 64) + threadIdx.x;
    if (j < nwords) {
      const unsigned long long word = (unsigned long long)pres[2 * threadIdx.x] |
                                      ((unsigned long long)pres[2 * threadIdx.x + 1] << 32);
      for (uint32_t d = 0; d < a.ndst; ++d) a.dst_bits[d][j] = word;
      if (a.dst_hdr) __threadfence_system();
    }
  }
  // 16 ranks per thread, in rank order
  const uint32_t bits16 = (pres[threadIdx.x >> 1] >> ((threadIdx.x & 1) * 16)) & 0xFFFFu;
  uint32_t tot;
  uint32_t pos = block_exclusive_sum((uint32_t)__popc(bits16), sscan, &tot);
  float* stg = a.staging + (uint64_t)q * kAggChunk;
  uint32_t b = bits16;
  while (b) {
    const uint32_t i = __ffs(b) - 1;
    b &= b - 1;
    stg[pos++] = acc[threadIdx.x * 16 + i];
  }
  if (threadIdx.x == 0) a.chunk_cnt[q] = tot;
}

__global__ void __launch_bounds__(1024) k_agg_scan(AggArgs a) {
  __shared__ uint64_t sscan[33];
  uint64_t carry = 0;
  for (uint32_t b = 0; b < a.nq; b += blockDim.x) {
    const uint32_t t = b + threadIdx.x;
    const uint64_t v = t < a.nq ? a.chunk_cnt[t] : 0u;
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum(v, sscan, &tot);
    if (t < a.nq) a.chunk_base[t] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *a.agg_count = carry;
}

// Phase 4: one warp per chunk moves the staged values to their final position
// in every destination (NVLink stores into peer pull inboxes in rank mode);
// the last block publishes U_s and the pull flag with release semantics.
__global__ void __launch_bounds__(256) k_agg_values(AggArgs a) {
  __shared__ uint32_t s_last;
  const uint32_t q = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (q < a.nq) {
    const uint32_t cnt = a.chunk_cnt[q];
    const uint64_t base = a.chunk_base[q];
    const float* stg = a.staging + (uint64_t)q * kAggChunk;
    for (uint32_t j = lane_id(); j < cnt; j += 32) {
      const float v = stg[j];
      if (base + j < a.val_cap)
        for (uint32_t d = 0; d < a.ndst; ++d) a.dst_vals[d][base + j] = v;
    }
  }
  if (!a.dst_hdr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t d = atomicAdd(a.done, 1u);
    s_last = (d == gridDim.x - 1) ? 1u : 0u;
    if (s_last) *a.done = 0;
  }
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
    const uint64_t u = *(volatile uint64_t*)a.agg_count;
    const uint32_t st = *(volatile uint32_t*)&a.hdr->status;
    const uint64_t bad = *(volatile uint64_t*)&a.hdr->bad_index;
    for (uint32_t d = threadIdx.x; d < a.ndst; d += blockDim.x) {
      a.dst_hdr[d]->agg_count = u;
      a.dst_hdr[d]->status = st;
      a.dst_hdr[d]->bad_index = bad;
    }
    __syncthreads();
    __threadfence_system();
    for (uint32_t d = threadIdx.x; d < a.ndst; d += blockDim.x)
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
  if (a.wait_pull && threadIdx.x < n) {
    const uint32_t iter = *(volatile uint32_t*)&a.hdr->iter;
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

// popcount of server s's bitmap bits [0, P)
__device__ __forceinline__ uint64_t bitmap_prefix(const DecodeArgs& a, uint32_t s, uint64_t P,
                                                  uint64_t nw) {
  const uint64_t j = P >> 6;
  const uint32_t o = (uint32_t)(P & 63);
  if (j >= nw) return a.popc_total[s];
  const unsigned long long* bits = a.bits[s];
  return (uint64_t)a.bpre_blk[s * a.blk_stride + j / kPrefixBlockWords] +
         a.bpre[s * a.words_stride + j] + (uint64_t)__popcll(bits[j] & lowmask64(o));
}

// One block: finish the bitmap prefixes (scan of block sums per server), then
// the output size of every decode tile straight from the tables -- for server
// s a tile covers the bit range [P_s(t), P_s(t+1)) of its bitmap -- and their
// exclusive scan.  No data pass, no look-back.
__global__ void __launch_bounds__(1024) k_dec_plan(DecodeArgs a, const uint32_t* blk_start,
                                                   const uint64_t* nwords_s, uint32_t ntiles,
                                                   uint64_t nchunks) {
  __shared__ uint64_t sscan[33];
  const uint32_t n = a.n;
  {
    const uint32_t s = threadIdx.x >> 5;
    if (s < n) {
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
  }
  __syncthreads();
  uint64_t carry = 0;
  constexpr uint32_t kChunksPerTile = kDecodeTileWords / 32;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x) {
    const uint32_t t = b + threadIdx.x;
    uint64_t v = 0;
    if (t < ntiles) {
      const uint64_t c0 = (uint64_t)t * kChunksPerTile, c1 = c0 + kChunksPerTile;
      for (uint32_t s = 0; s < n; ++s) {
        if (!a.bits[s]) continue;
        const uint64_t nw = nwords_s[s];
        const uint64_t P0 = a.cprefix[c0 * n + s];
        const uint64_t P1 = c1 < nchunks ? (uint64_t)a.cprefix[c1 * n + s] : a.bs[s];
        v += bitmap_prefix(a, s, P1, nw) - bitmap_prefix(a, s, P0, nw);
      }
    }
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum(v, sscan, &tot);
    if (t < ntiles) a.tile_base[t] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *a.out_count = carry;
}

template <int NMAX>
__global__ void __launch_bounds__(256) k_decode(DecodeArgs a, uint64_t nwords) {
  __shared__ uint32_t sscan[33];
  const uint32_t n = a.n;
  const uint32_t tile = blockIdx.x;
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
          pres[s] = (c == 64) ? x : deposit64(x, ms);
          vbase[s] = a.bpre_blk[s * a.blk_stride + j / kPrefixBlockWords] +
                     a.bpre[s * a.words_stride + j] + (uint32_t)__popcll(w0 & lowmask64(o));
          G |= pres[s];
        }
      }
    }
  }
  uint32_t tot;
  const uint32_t ex = block_exclusive_sum((uint32_t)__popcll(G), sscan, &tot);
  uint64_t pos = a.tile_base[tile] + ex;
  while (G) {
    const uint32_t i = __ffsll((long long)G) - 1;
    G &= G - 1;
    float v = 0.0f;
#pragma unroll
    for (int s = 0; s < NMAX; ++s) {
      if ((pres[s] >> i) & 1ull) v = a.vals[s][vbase[s] + __popcll(pres[s] & lowmask64(i))];
    }
    if (pos < a.out_cap) {
      a.out_idx[pos] = w * 64 + i;
      a.out_val[pos] = v;
    }
    ++pos;
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
  uint64_t tot_cap = (uint64_t)a.n * (a.cap + 1);
  k_agg_rank<<<grid_for(tot_cap, kAggThreads, 148 * 8), kAggThreads, 0, stream>>>(a);
  k_agg_chunk<<<a.nq, kAggThreads, 0, stream>>>(a);
  k_agg_scan<<<1, 1024, 0, stream>>>(a);
  k_agg_values<<<(a.nq + 7) / 8, 256, 0, stream>>>(a);
  for (int i = 0; i < 4; ++i) count_launch();
}

void launch_decode_parts(const DecodeArgs& a, const uint32_t* d_blk_start,
                         const uint64_t* d_nwords_s, uint32_t total_blocks, cudaStream_t stream) {
  const uint64_t nwords = (a.m + 63) / 64;
  const uint32_t ntiles = (uint32_t)((nwords + kDecodeTileWords - 1) / kDecodeTileWords);
  const uint64_t nchunks = (nwords + 31) / 32;
  k_bpre<<<total_blocks ? total_blocks : 1, 256, 0, stream>>>(a, d_blk_start, d_nwords_s);
  k_dec_plan<<<1, 1024, 0, stream>>>(a, d_blk_start, d_nwords_s, ntiles, nchunks);
  if (a.n <= 2)
    k_decode<2><<<ntiles, 256, 0, stream>>>(a, nwords);
  else if (a.n <= 4)
    k_decode<4><<<ntiles, 256, 0, stream>>>(a, nwords);
  else if (a.n <= 8)
    k_decode<8><<<ntiles, 256, 0, stream>>>(a, nwords);
  else
    k_decode<16><<<ntiles, 256, 0, stream>>>(a, nwords);
  for (int i = 0; i < 3; ++i) count_launch();
}

}  // namespace zen
