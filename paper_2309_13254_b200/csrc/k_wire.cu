// k_wire.cu -- the reference's wire formats on device (zen/codec.hpp:19-347):
// COO (all indices, then all values; 64- or 32-bit indices), TensorBlock
// (u64 block id + the block's dense values, per non-zero block) and the
// payload side of the plain Bitmap (which is the HashBitmap over the identity
// universe, k_codec.cu).  Payload bytes are little-endian and byte-identical
// to zen::encode; decodes apply the SparseTensor canonicalisation (sort when
// unsorted, duplicate / out-of-range rejection, zen/tensor.hpp:36-46).
//
// Payload pointers carry no alignment promise (a framed message puts the
// payload at byte 33), so payload accesses go through byte-exact helpers that
// use a vector access only when the address allows it.
#include <cub/cub.cuh>

#include "zen_common.cuh"

namespace zen {
extern void count_launch();
namespace {

using namespace zen_dev;

__device__ __forceinline__ void put_bytes(uint8_t* p, uint64_t v, int nbytes) {
  if (nbytes == 8 && !(reinterpret_cast<uintptr_t>(p) & 7)) {
    *reinterpret_cast<uint64_t*>(p) = v;
  } else if (nbytes == 4 && !(reinterpret_cast<uintptr_t>(p) & 3)) {
    *reinterpret_cast<uint32_t*>(p) = (uint32_t)v;
  } else {
    for (int b = 0; b < nbytes; ++b) p[b] = (uint8_t)(v >> (8 * b));
  }
}
__device__ __forceinline__ uint64_t get_bytes(const uint8_t* p, int nbytes) {
  if (nbytes == 8 && !(reinterpret_cast<uintptr_t>(p) & 7)) return *reinterpret_cast<const uint64_t*>(p);
  if (nbytes == 4 && !(reinterpret_cast<uintptr_t>(p) & 3)) return *reinterpret_cast<const uint32_t*>(p);
  uint64_t v = 0;
  for (int b = 0; b < nbytes; ++b) v |= (uint64_t)p[b] << (8 * b);
  return v;
}
__device__ __forceinline__ void put_f32(uint8_t* p, float v) { put_bytes(p, __float_as_uint(v), 4); }
__device__ __forceinline__ float get_f32(const uint8_t* p) { return __uint_as_float((uint32_t)get_bytes(p, 4)); }


// COO encode (codec.hpp:218-234): one entry per thread
__global__ void k_coo_encode(const uint64_t* __restrict__ idx, const float* __restrict__ val,
                             uint64_t count, int ib, uint8_t* payload, uint32_t* status) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = idx[i];
    if (ib == 4 && x > 0xffffffffull) atomicOr(status, kWireIdxOverflow);
    put_bytes(payload + i * ib, x, ib);
    put_f32(payload + count * ib + 4 * i, val[i]);
  }
}

// COO decode (codec.hpp:285-296) + canonical checks against the neighbour
__global__ void k_coo_decode(const uint8_t* __restrict__ payload, uint64_t count, int ib,
                             uint64_t m, uint64_t* __restrict__ idx, float* __restrict__ val,
                             uint32_t* status) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = get_bytes(payload + i * ib, ib);
    idx[i] = x;
    val[i] = get_f32(payload + count * ib + 4 * i);
    if (x >= m) atomicOr(status, kWireRange);
    if (i > 0) {
      const uint64_t p = get_bytes(payload + (i - 1) * ib, ib);
      if (p > x) atomicOr(status, kWireUnsorted);
      if (p == x) atomicOr(status, kWireDup);
    }
  }
}

// sorted-array checks (after a sort): duplicates and range
__global__ void k_check_canonical(const uint64_t* __restrict__ idx, uint64_t count, uint64_t m,
                                  uint32_t* status) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (idx[i] >= m) atomicOr(status, kWireRange);
    if (i > 0 && idx[i - 1] == idx[i]) atomicOr(status, kWireDup);
    if (i > 0 && idx[i - 1] > idx[i]) atomicOr(status, kWireUnsorted);
  }
}

// TensorBlock encode (codec.hpp:244-262, nonzero_blocks :167-178): flag the
// first entry of every non-zero block
__global__ void k_tb_flags(const uint64_t* __restrict__ idx, uint64_t count, uint64_t block,
                           uint32_t* __restrict__ first) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    first[i] = (i == 0 || idx[i] / block != idx[i - 1] / block) ? 1u : 0u;
}

// block b starts at byte b * (8 + 4 * block) (only the universe's last block
// can be shorter, and it is the last in the payload); the payload is zeroed
__global__ void k_tb_write(const uint64_t* __restrict__ idx, const float* __restrict__ val,
                           uint64_t count, uint64_t block, const uint32_t* __restrict__ first,
                           const uint32_t* __restrict__ bpos, uint8_t* payload) {
  zen_dev::pdl_entry();
  const uint64_t stride = 8 + 4 * block;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = bpos[i] - 1;  // inclusive count of first-flags - 1 = this entry's block
    const uint64_t id = idx[i] / block;
    uint8_t* base = payload + b * stride;
    if (first[i]) put_bytes(base, id, 8);
    put_f32(base + 8 + 4 * (idx[i] - id * block), val[i]);
  }
}

// TensorBlock decode, pass 1 (one thread): block offsets follow from the
// sequence of block lengths (min(block, M - begin)), exactly as the
// reference's sequential read (codec.hpp:311-331)
__global__ void k_tb_walk(const uint8_t* __restrict__ payload, uint64_t len, uint64_t count,
                          uint64_t block, uint64_t m, uint64_t* __restrict__ off,
                          uint64_t* __restrict__ begin, uint32_t* __restrict__ blen,
                          uint32_t* status) {
  zen_dev::pdl_entry();
  if (threadIdx.x || blockIdx.x) return;
  uint64_t pos = 0;
  for (uint64_t b = 0; b < count; ++b) {
    if (pos + 8 > len) {
      atomicOr(status, kWireMalformed);
      return;
    }
    const uint64_t id = get_bytes(payload + pos, 8);
    const uint64_t bg = id * block;  // wrapping u64 product, as the reference computes it
    if (bg >= m) {
      atomicOr(status, kWireMalformed);
      return;
    }
    const uint64_t l = (m - bg < block) ? m - bg : block;
    if (pos + 8 + 4 * l > len) {
      atomicOr(status, kWireMalformed);
      return;
    }
    off[b] = pos + 8;
    begin[b] = bg;
    blen[b] = (uint32_t)l;
    pos += 8 + 4 * l;
  }
  if (pos != len) atomicOr(status, kWireMalformed);
}

// TensorBlock decode, fast pass 1: every block of a well-formed, ascending
// payload sits at b * (8 + 4 * block) -- only the universe's last block can
// be shorter, and it is then the last one.  Anything else (including every
// malformed payload) sets kWireIrregular and the host reruns the sequential
// walk above, which reproduces the reference's reading exactly.
constexpr uint32_t kWireIrregular = 32u;
__global__ void k_tb_offsets(const uint8_t* __restrict__ payload, uint64_t len, uint64_t count,
                             uint64_t block, uint64_t m, uint64_t* __restrict__ off,
                             uint64_t* __restrict__ begin, uint32_t* __restrict__ blen,
                             uint32_t* status) {
  zen_dev::pdl_entry();
  const uint64_t stride = 8 + 4 * block;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < count;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = b * stride;
    if (pos + 8 > len) {
      atomicOr(status, kWireIrregular);
      continue;
    }
    const uint64_t bg = get_bytes(payload + pos, 8) * block;
    if (bg >= m) {
      atomicOr(status, kWireIrregular);
      continue;
    }
    const uint64_t l = (m - bg < block) ? m - bg : block;
    const uint64_t end = pos + 8 + 4 * l;
    if ((l != block && b + 1 != count) || end > len || (b + 1 == count && end != len))
      atomicOr(status, kWireIrregular);
    off[b] = pos + 8;
    begin[b] = bg;
    blen[b] = (uint32_t)l;
  }
}

// pass 2: every value slot -> (index, value, non-zero flag)
__global__ void k_tb_expand(const uint8_t* __restrict__ payload, uint64_t nb, uint64_t block,
                            const uint64_t* __restrict__ off, const uint64_t* __restrict__ begin,
                            const uint32_t* __restrict__ blen, uint64_t* __restrict__ sidx,
                            float* __restrict__ sval, uint8_t* __restrict__ flag) {
  zen_dev::pdl_entry();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb * block;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = t / block, e = t - b * block;
    bool nz = false;
    if (e < blen[b]) {
      const float v = get_f32(payload + off[b] + 4 * e);
      nz = v != 0.0f;
      sval[t] = v;
      sidx[t] = begin[b] + e;
    }
    flag[t] = nz ? 1 : 0;
  }
}

inline unsigned grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148 * 16));
}

}  // namespace

void launch_coo_encode(const uint64_t* idx, const float* val, uint64_t count, int ib,
                       uint8_t* payload, uint32_t* status, cudaStream_t s) {
  if (!count) return;
  launch_k(k_coo_encode, grid_for(count), 256, 0, s, idx, val, count, ib, payload, status);
  count_launch();
}

void launch_coo_decode(const uint8_t* payload, uint64_t count, int ib, uint64_t m, uint64_t* idx,
                       float* val, uint32_t* status, cudaStream_t s) {
  if (!count) return;
  launch_k(k_coo_decode, grid_for(count), 256, 0, s, payload, count, ib, m, idx, val, status);
  count_launch();
}

void launch_check_canonical(const uint64_t* idx, uint64_t count, uint64_t m, uint32_t* status,
                            cudaStream_t s) {
  if (!count) return;
  launch_k(k_check_canonical, grid_for(count), 256, 0, s, idx, count, m, status);
  count_launch();
}

// cub scratch sizing + runs, shared by the host side (capi.cpp owns the memory)
size_t wire_scan_bytes(uint64_t n) {
  size_t b = 0;
  cub::DeviceScan::InclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return b;
}
size_t wire_sort_bytes(uint64_t n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const float*)nullptr, (float*)nullptr, (int)n);
  return b;
}
size_t wire_select_bytes(uint64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, (const uint64_t*)nullptr, (const uint8_t*)nullptr,
                             (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)n);
  cub::DeviceSelect::Flagged(nullptr, b, (const float*)nullptr, (const uint8_t*)nullptr,
                             (float*)nullptr, (uint64_t*)nullptr, (int64_t)n);
  return std::max(a, b);
}

void launch_tb_blocks(const uint64_t* idx, uint64_t count, uint64_t block, uint32_t* first,
                      uint32_t* bpos, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  if (!count) return;
  launch_k(k_tb_flags, grid_for(count), 256, 0, s, idx, count, block, first);
  count_launch();
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, first, bpos, (int)count, s);
  count_launch();
}

void launch_tb_write(const uint64_t* idx, const float* val, uint64_t count, uint64_t block,
                     const uint32_t* first, const uint32_t* bpos, uint8_t* payload, cudaStream_t s) {
  if (!count) return;
  launch_k(k_tb_write, grid_for(count), 256, 0, s, idx, val, count, block, first, bpos, payload);
  count_launch();
}

void launch_tb_walk(const uint8_t* payload, uint64_t len, uint64_t count, uint64_t block,
                    uint64_t m, uint64_t* off, uint64_t* begin, uint32_t* blen, uint32_t* status,
                    cudaStream_t s) {
  launch_k(k_tb_walk, 1, 32, 0, s, payload, len, count, block, m, off, begin, blen, status);
  count_launch();
}

void launch_tb_offsets(const uint8_t* payload, uint64_t len, uint64_t count, uint64_t block,
                       uint64_t m, uint64_t* off, uint64_t* begin, uint32_t* blen,
                       uint32_t* status, cudaStream_t s) {
  if (!count) return;
  launch_k(k_tb_offsets, grid_for(count), 256, 0, s, payload, len, count, block, m, off, begin,
           blen, status);
  count_launch();
}

void launch_tb_expand_select(const uint8_t* payload, uint64_t nb, uint64_t block,
                             const uint64_t* off, const uint64_t* begin, const uint32_t* blen,
                             uint64_t* sidx, float* sval, uint8_t* flag, uint64_t* out_idx,
                             float* out_val, uint64_t* d_count, void* tmp, size_t tmp_bytes,
                             cudaStream_t s) {
  const uint64_t slots = nb * block;
  if (!slots) return;
  launch_k(k_tb_expand, grid_for(slots), 256, 0, s, payload, nb, block, off, begin, blen, sidx,
           sval, flag);
  count_launch();
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, sidx, flag, out_idx, d_count, (int64_t)slots, s);
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, sval, flag, out_val, d_count, (int64_t)slots, s);
  count_launch();
  count_launch();
}

void launch_sort_pairs(const uint64_t* ki, uint64_t* ko, const float* vi, float* vo,
                       uint64_t count, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  if (!count) return;
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ki, ko, vi, vo, (int)count, 0, 64, s);
  count_launch();
}

}  // namespace zen

// ---- OmniReduce-like range blocks (zen/schemes.hpp:227-244) -----------------
namespace zen {
namespace {
// 1 where a sorted entry opens a new block of `block` positions counted from
// `origin`; a single counter gathers them (tiny key sets)
__global__ void k_count_blocks(const uint64_t* __restrict__ idx, uint64_t count, uint64_t origin,
                               uint64_t block, unsigned long long* out) {
  zen_dev::pdl_entry();
  uint32_t c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    c += (i == 0 || (idx[i] - origin) / block != (idx[i - 1] - origin) / block) ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void k_nonzero_flags(const float* __restrict__ val, uint64_t count, uint8_t* flag) {
  zen_dev::pdl_entry();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    flag[i] = val[i] != 0.0f ? 1 : 0;
}
}  // namespace

void launch_count_blocks(const uint64_t* idx, uint64_t count, uint64_t origin, uint64_t block,
                         unsigned long long* out, cudaStream_t s) {
  if (!count) return;
  launch_k(k_count_blocks, (unsigned)std::min<uint64_t>(grid_for(count), 148 * 8), 256, 0, s, idx,
           count, origin, block, out);
  count_launch();
}

void launch_compact_nonzero(const uint64_t* idx, const float* val, uint64_t count, uint8_t* flag,
                            uint64_t* out_idx, float* out_val, uint64_t* d_count, void* tmp,
                            size_t tmp_bytes, cudaStream_t s) {
  if (!count) return;
  launch_k(k_nonzero_flags, grid_for(count), 256, 0, s, val, count, flag);
  count_launch();
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, idx, flag, out_idx, d_count, (int64_t)count, s);
  cub::DeviceSelect::Flagged(tmp, tmp_bytes, val, flag, out_val, d_count, (int64_t)count, s);
  count_launch();
  count_launch();
}
}  // namespace zen
