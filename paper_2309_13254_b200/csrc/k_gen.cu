// k_gen.cu -- the reference's synthetic workload (zen::generate,
// zen/workload.hpp:22-154) on the device: per node, ceil(d*M) distinct
// indices = a shared core of ceil(omega*d*M) plus the rest drawn from the
// two-tier distribution (hot_mass of the draws uniform in the first
// hot_fraction*M indices, the others uniform in the cold remainder), without
// replacement and avoiding the core, ascending, integer values in [1, 16].
//
// Same spec, not the same bits: the reference draws from std::mt19937_64
// through libstdc++'s distributions one index at a time (a rejection loop over
// an unordered_set).  Here a draw of K distinct indices from a tier is the
// first K positions of a keyed pseudo-random PERMUTATION of the tier (a
// 4-round Feistel network on the next power of four, cycle-walked into the
// range): distinct by construction, uniform, and every position is computed
// independently, so the draw is parallel and deterministic for a seed on any
// schedule.  Avoiding the core = taking the first K positions whose index is
// not in the core bitmap (a flag pass, a scan of the block counts, a take
// pass).  The host splits the node's draws between the tiers with a binomial
// draw (the reference flips hot_mass per accepted draw) capped at each tier's
// free capacity (TwoTierSampler's spill, workload.hpp:79-100).
//
//  k_gen_flag / k_gen_scan / k_gen_take : one tier's draw
//  k_gen_count / k_gen_scan / k_gen_write : bitmap (node | core) -> ascending
//                 indices, values from a hash of (seed, node, index)
#include "zen_common.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

constexpr int kGenThreads = 256;
constexpr int kGenWordsPerBlock = 1024;  // 4 words per thread (collect passes)
constexpr int kGenPosPerBlock = 1024;    // 4 positions per thread (draw passes)

struct Perm {  // keyed bijection of [0, range)
  uint64_t range;
  uint32_t hb;    // half width in bits: 4^hb >= range
  uint64_t key[4];
};

__device__ __forceinline__ uint64_t feistel(uint64_t x, const Perm& P) {
  const uint64_t mask = (1ull << P.hb) - 1ull;
  uint64_t L = x >> P.hb, R = x & mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t f = mix64(R + P.key[r]) & mask;
    const uint64_t nl = R;
    R = L ^ f;
    L = nl;
  }
  return (L << P.hb) | R;
}

__device__ __forceinline__ uint64_t permute(uint64_t i, const Perm& P) {
  uint64_t x = feistel(i, P);
  while (x >= P.range) x = feistel(x, P);  // cycle walking stays a bijection of [0, range)
  return x;
}

__device__ __forceinline__ bool in_core(const unsigned long long* core, uint64_t idx) {
  return core && ((core[idx >> 6] >> (idx & 63)) & 1ull);
}

// per block of 1024 positions: how many of them land outside the core
__global__ void __launch_bounds__(kGenThreads)
    k_gen_flag(Perm P, uint64_t base, const unsigned long long* __restrict__ core, uint64_t npos,
               uint32_t* __restrict__ blk) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s[33];
  const uint64_t p0 = (uint64_t)blockIdx.x * kGenPosPerBlock + threadIdx.x * 4;
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (p0 + q < npos) c += in_core(core, base + permute(p0 + q, P)) ? 0u : 1u;
  uint32_t tot;
  block_exclusive_sum(c, s, &tot);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

// the first `want` non-core positions set their index in the node bitmap
__global__ void __launch_bounds__(kGenThreads)
    k_gen_take(Perm P, uint64_t base, const unsigned long long* __restrict__ core, uint64_t npos,
               const uint32_t* __restrict__ blk, uint64_t want, unsigned long long* __restrict__ bits) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s[33];
  const uint64_t p0 = (uint64_t)blockIdx.x * kGenPosPerBlock + threadIdx.x * 4;
  uint64_t x[4];
  bool ok[4];
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    ok[q] = false;
    if (p0 + q < npos) {
      x[q] = base + permute(p0 + q, P);
      ok[q] = !in_core(core, x[q]);
    }
    c += ok[q] ? 1u : 0u;
  }
  uint32_t tot;
  uint64_t rank = (uint64_t)blk[blockIdx.x] + block_exclusive_sum(c, s, &tot);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (ok[q]) {
      if (rank < want) atomicOr(bits + (x[q] >> 6), 1ull << (x[q] & 63));
      ++rank;
    }
}

// per block of 1024 words: popcount of (bits | core)
__global__ void __launch_bounds__(kGenThreads)
    k_gen_count(const unsigned long long* __restrict__ bits, const unsigned long long* __restrict__ core,
                uint64_t nw, uint32_t* __restrict__ blk) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s[33];
  const uint64_t w0 = (uint64_t)blockIdx.x * kGenWordsPerBlock + threadIdx.x * 4;
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (w0 + q < nw) c += __popcll(bits[w0 + q] | (core ? core[w0 + q] : 0ull));
  uint32_t tot;
  block_exclusive_sum(c, s, &tot);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

// one block: exclusive scan of the block totals, total count
__global__ void __launch_bounds__(1024) k_gen_scan(uint32_t* __restrict__ blk, uint32_t nblk,
                                                   uint64_t* __restrict__ total) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s[33];
  uint32_t carry = 0;
  for (uint32_t b = 0; b < nblk; b += blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < nblk ? blk[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_sum(v, s, &tot);
    if (i < nblk) blk[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kGenThreads)
    k_gen_write(const unsigned long long* __restrict__ bits,
                const unsigned long long* __restrict__ core, uint64_t nw,
                const uint32_t* __restrict__ blk, uint64_t vseed, uint64_t* __restrict__ out_idx,
                float* __restrict__ out_val, uint64_t cap) {
  zen_dev::pdl_entry();
  __shared__ uint32_t s[33];
  const uint64_t w0 = (uint64_t)blockIdx.x * kGenWordsPerBlock + threadIdx.x * 4;
  unsigned long long v[4];
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = (w0 + q < nw) ? (bits[w0 + q] | (core ? core[w0 + q] : 0ull)) : 0ull;
    c += __popcll(v[q]);
  }
  uint32_t tot;
  uint64_t pos = (uint64_t)blk[blockIdx.x] + block_exclusive_sum(c, s, &tot);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    for (unsigned long long y = v[q]; y; y &= y - 1, ++pos) {
      const uint64_t idx = (w0 + q) * 64 + (uint64_t)(__ffsll((long long)y) - 1);
      if (pos < cap) {
        out_idx[pos] = idx;
        out_val[pos] = (float)(1u + (uint32_t)(mix64(vseed ^ mix64(idx)) % 16u));
      }
    }
}

}  // namespace

// K distinct indices of [base, base + range) not in `core`, into `bits`
void launch_gen_tier(uint64_t base, uint64_t range, uint64_t key_seed, const unsigned long long* core,
                     uint64_t core_in_tier, uint64_t want, unsigned long long* bits, uint32_t* blk,
                     cudaStream_t s) {
  if (!want) return;
  Perm P{};
  P.range = range;
  P.hb = 1;
  while ((1ull << (2 * P.hb)) < range) ++P.hb;
  uint64_t k = key_seed;
  for (int r = 0; r < 4; ++r) {
    k = k * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL;
    P.key[r] = k ^ (k >> 29);
  }
  const uint64_t npos = std::min<uint64_t>(range, want + core_in_tier);
  const uint32_t nblk = (uint32_t)((npos + kGenPosPerBlock - 1) / kGenPosPerBlock);
  launch_k(k_gen_flag, nblk, kGenThreads, 0, s, P, base, core, npos, blk);
  launch_k(k_gen_scan, 1, 1024, 0, s, blk, nblk, (uint64_t*)nullptr);
  launch_k(k_gen_take, nblk, kGenThreads, 0, s, P, base, core, npos, (const uint32_t*)blk, want,
           bits);
  for (int i = 0; i < 3; ++i) count_launch();
}

void launch_gen_collect(const unsigned long long* bits, const unsigned long long* core,
                        uint64_t nw, uint32_t* blk, uint64_t* total, uint64_t vseed,
                        uint64_t* out_idx, float* out_val, uint64_t cap, cudaStream_t s) {
  const uint32_t nblk = (uint32_t)((nw + kGenWordsPerBlock - 1) / kGenWordsPerBlock);
  launch_k(k_gen_count, std::max(nblk, 1u), kGenThreads, 0, s, bits, core, nw, blk);
  launch_k(k_gen_scan, 1, 1024, 0, s, blk, nblk, total);
  if (out_idx)
    launch_k(k_gen_write, std::max(nblk, 1u), kGenThreads, 0, s, bits, core, nw,
             (const uint32_t*)blk, vseed, out_idx, out_val, cap);
  for (int i = 0; i < (out_idx ? 3 : 2); ++i) count_launch();
}

}  // namespace zen
