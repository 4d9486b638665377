// k_util.cu -- small device helpers behind the standalone C-ABI operators:
// HashMemory dumps (reference 0 = empty sentinel), CollisionStats depths, and
// the materialised universe list I_s.
#include "zen_common.cuh"
#include "zen_hash_dev.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

__global__ void k_dump_slots(const unsigned long long* __restrict__ slots, uint64_t cells,
                             uint64_t ew, const float* __restrict__ vals,
                             uint64_t* __restrict__ out_slots, float* __restrict__ out_vals) {
  zen_dev::pdl_entry();
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cells;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long w = slots[c];
    const bool live = (w & ~kKeyMask) == ew;
    if (out_slots) out_slots[c] = live ? (w & kKeyMask) : 0ull;  // index+1, 0 = empty
    if (out_vals) out_vals[c] = live ? vals[c] : 0.0f;
  }
}

__global__ void k_meta_depth(const uint32_t* __restrict__ meta, uint64_t count,
                             uint32_t* __restrict__ out) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = meta_depth(meta[i]);
}

__global__ void k_universe_indices(const OwnWord* __restrict__ own, uint64_t nwords,
                                   uint64_t* __restrict__ out) {
  zen_dev::pdl_entry();
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
       w += (uint64_t)gridDim.x * blockDim.x) {
    const OwnWord o = own[w];
    uint64_t m = o.mask;
    uint64_t pos = o.prefix;
    while (m) {
      const uint32_t b = __ffsll((long long)m) - 1;
      m &= m - 1;
      out[pos++] = w * 64 + b;
    }
  }
}

// the apply step after a sync: dense[idx[i]] += alpha * val[i] (indices
// unique, so no atomics); an SGD step on the synced gradient is alpha = -lr
__global__ void k_axpy_sparse(float* __restrict__ dense, uint64_t m,
                              const uint64_t* __restrict__ idx, const float* __restrict__ val,
                              uint64_t count, float alpha, uint32_t* status) {
  zen_dev::pdl_entry();
  // R entries per thread per round with every load issued before the
  // read-modify-writes: one index -> parameter latency chain per round, not
  // per entry
  constexpr int R = 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < count;
       base += R * stride) {
    uint64_t x[R];
    float v[R], d[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint64_t i = base + q * stride;
      x[q] = i < count ? idx[i] : ~0ull;
      v[q] = i < count ? val[i] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) d[q] = x[q] < m ? dense[x[q]] : 0.0f;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (base + q * stride >= count) break;
      if (x[q] < m)
        dense[x[q]] = fmaf(alpha, v[q], d[q]);
      else
        atomicOr(status, 1u);
    }
  }
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint64_t n) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// universe_positions' ownership check (zen/codec.hpp:146-158): every index
// must be < M and owned by the server; the smallest offender is reported.
__global__ void k_check_owned(const uint64_t* __restrict__ idx, uint64_t count, uint64_t m,
                              const OwnWord* __restrict__ own, HashHdr* hdr) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = idx[i];
    const bool ok = x < m && ((own[x >> 6].mask >> (x & 63)) & 1ull);
    if (!ok) {
      atomicMin((unsigned long long*)&hdr->bad_index, (unsigned long long)x);
      atomicOr(&hdr->status, kErrOutside);
    }
  }
}

inline unsigned grid_for(uint64_t work) {
  uint64_t g = (work + 255) / 256;
  if (g < 1) g = 1;
  return (unsigned)(g < 148 * 8 ? g : 148 * 8);
}

}  // namespace

void launch_dump_slots(const unsigned long long* slots, uint64_t cells, uint32_t epoch,
                       const float* vals, uint64_t* out_slots, float* out_vals,
                       cudaStream_t stream) {
  const uint64_t ew = (uint64_t)(0xFFFFFFu - (epoch & 0xFFFFFFu)) << kKeyBits;
  launch_k(k_dump_slots, grid_for(cells), 256, 0, stream, slots, cells, ew, vals, out_slots, out_vals);
  count_launch();
}

void launch_meta_depth(const uint32_t* meta, uint64_t count, uint32_t* out, cudaStream_t stream) {
  launch_k(k_meta_depth, grid_for(count), 256, 0, stream, meta, count, out);
  count_launch();
}

void launch_universe_indices(const OwnWord* own, uint64_t nwords, uint64_t* out,
                             cudaStream_t stream) {
  launch_k(k_universe_indices, grid_for(nwords), 256, 0, stream, own, nwords, out);
  count_launch();
}

void launch_check_owned(const uint64_t* idx, uint64_t count, uint64_t m, const OwnWord* own,
                        HashHdr* hdr, cudaStream_t stream) {
  launch_k(k_check_owned, grid_for(count), 256, 0, stream, idx, count, m, own, hdr);
  count_launch();
}

void launch_axpy_sparse(float* dense, uint64_t m, const uint64_t* idx, const float* val,
                        uint64_t count, float alpha, uint32_t* status, cudaStream_t stream) {
  if (!count) return;
  launch_k(k_axpy_sparse, grid_for(count), 256, 0, stream, dense, m, idx, val, count, alpha, status);
  count_launch();
}

__global__ void k_range_bounds(const uint64_t* __restrict__ idx, uint64_t count, uint64_t m,
                               uint32_t parts, uint64_t* __restrict__ bnd) {
  pdl_entry();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  const uint64_t range = (m + parts - 1) / parts;
  const uint64_t key = p == parts ? m : (uint64_t(p) * range < m ? uint64_t(p) * range : m);
  uint64_t lo = 0, hi = count;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (idx[mid] < key) lo = mid + 1; else hi = mid;
  }
  bnd[p] = lo;
}

void launch_range_bounds(const uint64_t* idx, uint64_t count, uint64_t m, uint32_t parts,
                         uint64_t* bnd, cudaStream_t stream) {
  launch_k(k_range_bounds, (parts + 256) / 256, 256, 0, stream, idx, count, m, parts, bnd);
  count_launch();
}

void launch_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t stream) {
  launch_k(k_u32_to_u64, grid_for(n), 256, 0, stream, in, out, n);
  count_launch();
}

}  // namespace zen
