// zen_common.cuh -- device building blocks shared by the sm_100a kernels.
//
// * the reference hash family (zen/hashing.hpp:18-88), bit-exact on device;
// * warp/block scans and the decoupled look-back used by every stream
//   compaction on the path (extraction, aggregate+encode, decode);
// * system-scope acquire/release helpers for the NVLink peer flags.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "zen_internal.h"

namespace zen_dev {

// ---- programmatic dependent launch (sm_90+) --------------------------------
// Every kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization
// (launch_k below), so a kernel's CTAs become resident while its predecessor
// drains and the launch latency between the ~20 dependent kernels of a sync
// overlaps.  Correctness: pdl_entry() is the first statement of every kernel;
// griddepcontrol.wait returns only once all prerequisite grids have completed
// and their memory is visible, so no kernel touches global memory before its
// predecessor is done.  launch_dependents lets the next grid start launching
// as soon as every CTA of this grid is running.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


// ---- hash family: zen/hashing.hpp:18-39 -----------------------------------
// mix64 is the splitmix64 finalizer; seeded_hash(x, s) = mix64(x + G*(s+1))
// with wrapping u64 arithmetic, so the per-seed constant G*(s+1) is folded on
// the host (DevFamily.pc / .sc) and the device does one add + mix per hash.
// map_to_range(h, r) = (u128(h) * r) >> 64 is exactly __umul64hi(h, r).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// map_to_range for r < 2^32: (h * r) >> 64 = (h_hi * r + ((h_lo * r) >> 32)) >> 32
// exactly -- two 32x32->64 multiplies instead of a full 64-bit mul-hi.
__device__ __forceinline__ uint64_t map_to_range32(uint64_t h, uint32_t r) {
  const uint64_t lo = (uint64_t)(uint32_t)h * r;
  const uint64_t hi = (h >> 32) * (uint64_t)r;
  return (hi + (lo >> 32)) >> 32;
}
__device__ __forceinline__ uint64_t map_to_range(uint64_t h, uint64_t r) {
  return (r >> 32) ? __umul64hi(h, r) : map_to_range32(h, (uint32_t)r);
}

// key = index + 1 (zen/hashing.hpp:44-45, :73-76, :79-81)
__device__ __forceinline__ uint32_t part_of(const zen::DevFamily& f, uint64_t key) {
  return (uint32_t)map_to_range32(mix64(key + f.pc), f.n);
}
__device__ __forceinline__ uint64_t slot_of(const zen::DevFamily& f, uint64_t key, uint32_t t,
                                            uint64_t r1) {  // t is 0-based (round t+1)
  return map_to_range(mix64(key + f.sc[t]), r1);
}
__device__ __forceinline__ uint32_t part_of_seed(uint64_t pc, uint32_t n, uint64_t key) {
  return (uint32_t)map_to_range32(mix64(key + pc), n);
}

// ---- bit helpers ------------------------------------------------------------
__device__ __forceinline__ uint64_t lowmask64(uint32_t b) {  // b in [0, 64]
  return b >= 64 ? ~0ull : ((1ull << b) - 1ull);
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// position of the (q+1)-th set bit of a 64-bit mask (q < popc(mask))
// position of the q-th (0-based) set bit of mask (q < popc(mask)); branch-light
// binary descent on popcounts (sm_100 has no native FNS; __fns is emulated)
__device__ __forceinline__ uint32_t select64(uint64_t mask, uint32_t q) {
  uint32_t pos = 0;
  uint32_t c = __popc((uint32_t)mask);
  uint32_t w = (uint32_t)mask;
  if (q >= c) {
    q -= c;
    w = (uint32_t)(mask >> 32);
    pos = 32;
  }
  c = __popc(w & 0xFFFFu);
  if (q >= c) { q -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xFFu);
  if (q >= c) { q -= c; w >>= 8; pos += 8; }
  c = __popc(w & 0xFu);
  if (q >= c) { q -= c; w >>= 4; pos += 4; }
  c = __popc(w & 0x3u);
  if (q >= c) { q -= c; w >>= 2; pos += 2; }
  if (q >= (w & 1u)) pos += 1;
  return pos;
}
// pdep: deposit the low popc(mask) bits of src into mask's set bits.  Full
// slices (every owned bit present, e.g. whole embedding rows) take the fast
// path; otherwise the uniform-cost "expand" of Hacker's Delight (7-5): six
// parallel-suffix steps build the shift masks, six shifts move the bits.
__device__ __forceinline__ uint64_t deposit64(uint64_t src, uint64_t mask) {
  const uint32_t c = __popcll(mask);
  if (src == (c == 64 ? ~0ull : ((1ull << c) - 1ull))) return mask;
  uint64_t m = mask, mk = ~mask << 1, sh[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    uint64_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    mp ^= mp << 32;
    const uint64_t mv = mp & m;
    sh[i] = mv;
    m = (m ^ mv) | (mv >> (1 << i));
    mk &= ~mp;
  }
  uint64_t x = src;
#pragma unroll
  for (int i = 5; i >= 0; --i) x = (x & ~sh[i]) | ((x << (1 << i)) & sh[i]);
  return x & mask;
}

// ---- scans ------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= (uint32_t)o) v += u;
  }
  return v;
}

// Block-wide exclusive scan (blockDim multiple of 32, <= 1024). `smem` needs
// 33 slots. Returns the exclusive prefix; *total receives the block sum.
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* smem, T* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_inclusive_sum(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nw ? smem[lane] : T(0);
    T si = warp_inclusive_sum(s);
    if (lane < nw) smem[lane] = si - s;
    if (lane == nw - 1) smem[32] = si;
  }
  __syncthreads();
  T r = smem[warp] + inc - v;
  *total = smem[32];
  __syncthreads();
  return r;
}

// In-place exclusive scan of cnt u32 values by ONE warp, for "last block"
// finishing passes: each lane owns a contiguous chunk; loads go through L2
// (ld.cg, the values were written by other blocks) and are batched, so the
// cost is ~2 L2 round trips rather than cnt/32 serial ones.  Returns the total.
__device__ __forceinline__ uint32_t warp_exscan_l2(uint32_t* b, uint32_t cnt) {
  const uint32_t lane = lane_id(), per = (cnt + 31) / 32;
  const uint32_t lo = min(lane * per, cnt), hi = min(lo + per, cnt);
  uint32_t sum = 0;
#pragma unroll 8
  for (uint32_t i = lo; i < hi; ++i) sum += __ldcg(b + i);
  const uint32_t inc = warp_inclusive_sum(sum);
  uint32_t run = inc - sum;
#pragma unroll 8
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t v = __ldcg(b + i);
    __stcg(b + i, run);
    run += v;
  }
  return __shfl_sync(0xffffffffu, inc, 31);
}

// ---- decoupled look-back ----------------------------------------------------
// Status word per tile: [63:40] launch tag (24 bits), [39:38] flag, [37:0] value.
// Tags come from a per-kernel control block {ticket, done, tag} that the last
// block of every launch advances, so no memset is needed between launches and
// the whole sequence stays CUDA-graph replayable.
constexpr uint64_t LB_FLAG_AGG = 1ull, LB_FLAG_PRE = 2ull;
constexpr uint64_t LB_VAL_MASK = (1ull << 38) - 1ull;

__device__ __forceinline__ uint64_t lb_pack(uint32_t tag, uint64_t flag, uint64_t v) {
  return ((uint64_t)(tag & 0xFFFFFFu) << 40) | (flag << 38) | (v & LB_VAL_MASK);
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Called by every thread of warp 0 of the tile's block after the block knows
// its aggregate; returns the exclusive prefix of the tile (same on all lanes).
// The flag and the value share one 64-bit word and nothing else is published
// with them, so the stores need no fence (a fence.sc here costs microseconds
// per tile).
__device__ __forceinline__ uint64_t lookback_warp(unsigned long long* status, uint32_t tile,
                                                  uint32_t tag, uint64_t aggregate) {
  const uint32_t lane = lane_id();
  if (tile == 0) {
    if (lane == 0) {
      st_relaxed_gpu(status, lb_pack(tag, LB_FLAG_PRE, aggregate));
    }
    return 0;
  }
  if (lane == 0) {
    st_relaxed_gpu(status + tile, lb_pack(tag, LB_FLAG_AGG, aggregate));
  }
  uint64_t exclusive = 0;
  int64_t base = (int64_t)tile - 1;
  const uint64_t tagbits = (uint64_t)(tag & 0xFFFFFFu);
  while (true) {
    const int64_t t = base - (int64_t)lane;
    uint64_t w = 0, flag = 0, val = 0;
    if (t >= 0) {
      while (true) {
        w = ld_relaxed_gpu(status + t);
        flag = ((w >> 40) == tagbits) ? ((w >> 38) & 3ull) : 0ull;
        if (flag) break;
        __nanosleep(32);
      }
      val = w & LB_VAL_MASK;
    } else {
      flag = LB_FLAG_PRE;  // virtual predecessor of tile 0
      val = 0;
    }
    const uint32_t pre_mask = __ballot_sync(0xffffffffu, flag == LB_FLAG_PRE);
    // first lane (closest predecessor) holding an inclusive prefix
    const uint32_t stop = __ffs(pre_mask) - 1;  // pre_mask != 0 only if some lane saw PRE
    uint64_t contrib = (pre_mask && lane > stop) ? 0 : val;
    if (pre_mask == 0) contrib = val;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
    exclusive += contrib;
    if (pre_mask) break;
    base -= 32;
  }
  if (lane == 0) {
    st_relaxed_gpu(status + tile, lb_pack(tag, LB_FLAG_PRE, exclusive + aggregate));
  }
  return exclusive;
}

// Block-wide decoupled look-back: the block's threads inspect blockDim.x
// predecessors per round trip (the warp form: 32), for grids whose tiles are
// all in flight at once, where a tile deep in the wave would otherwise walk
// back window by window.  Every thread calls it after the block knows its
// aggregate; returns the exclusive prefix on every thread.  s_red: >= 32 words.
__device__ __forceinline__ uint64_t lookback_block(unsigned long long* status, uint32_t tile,
                                                   uint32_t tag, uint64_t aggregate,
                                                   unsigned long long* s_red) {
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5, nw = blockDim.x >> 5;
  if (tile == 0) {
    if (tid == 0) st_relaxed_gpu(status, lb_pack(tag, LB_FLAG_PRE, aggregate));
    return 0;
  }
  if (tid == 0) st_relaxed_gpu(status + tile, lb_pack(tag, LB_FLAG_AGG, aggregate));
  const uint64_t tagbits = (uint64_t)(tag & 0xFFFFFFu);
  uint64_t exclusive = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t t = base - (int64_t)tid;  // thread i looks i tiles further back
    uint64_t flag = LB_FLAG_PRE, val = 0;   // t < 0: the virtual predecessor of tile 0
    if (t >= 0) {
      while (true) {
        const uint64_t w = ld_relaxed_gpu(status + t);
        flag = ((w >> 40) == tagbits) ? ((w >> 38) & 3ull) : 0ull;
        if (flag) {
          val = w & LB_VAL_MASK;
          break;
        }
        __nanosleep(32);
      }
    }
    const uint32_t pm = __ballot_sync(0xffffffffu, flag == LB_FLAG_PRE);
    if (lane == 0) s_red[warp] = pm ? (uint64_t)(warp * 32 + __ffs(pm) - 1) : ~0ull;
    __syncthreads();
    uint64_t stop = ~0ull;
    for (uint32_t w = 0; w < nw; ++w) stop = s_red[w] < stop ? s_red[w] : stop;
    uint64_t c = (stop != ~0ull && tid > stop) ? 0 : val;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __syncthreads();
    if (lane == 0) s_red[warp] = c;
    __syncthreads();
    for (uint32_t w = 0; w < nw; ++w) exclusive += s_red[w];
    __syncthreads();
    if (stop != ~0ull) break;
    base -= (int64_t)blockDim.x;
  }
  if (tid == 0) st_relaxed_gpu(status + tile, lb_pack(tag, LB_FLAG_PRE, exclusive + aggregate));
  return exclusive;
}

// Dynamic tile ticket; ensures tiles start in order so look-back progresses.
__device__ __forceinline__ uint32_t take_ticket(zen::LookbackCtl* ctl, uint32_t* smem_slot) {
  if (threadIdx.x == 0) *smem_slot = atomicAdd(&ctl->ticket, 1u);
  __syncthreads();
  const uint32_t t = *smem_slot;
  __syncthreads();
  return t;
}
// Last block to finish resets the ticket and advances the tag.  Returns true
// (on every thread of the block) for that last block; must be called by all
// threads.  `sys` upgrades the fence to system scope (peer-visible stores).
__device__ __forceinline__ bool finish_tile(zen::LookbackCtl* ctl, uint32_t ntiles,
                                            bool sys = false) {
  __shared__ uint32_t s_is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sys) __threadfence_system(); else __threadfence();
    const uint32_t d = atomicAdd(&ctl->done, 1u);
    s_is_last = (d == ntiles - 1) ? 1u : 0u;
    if (s_is_last) {
      ctl->ticket = 0;
      ctl->done = 0;
      uint32_t t = (ctl->tag + 1u) & 0xFFFFFFu;
      ctl->tag = t ? t : 1u;  // 0 is reserved for "never written"
      __threadfence();
    }
  }
  __syncthreads();
  return s_is_last != 0;
}

// ---- system-scope flags (NVLink peers) -------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// release fence: system scope when peers (other GPUs) read what we wrote
__device__ __forceinline__ void fence_for(bool peer) {
  if (peer)
    __threadfence_system();
  else
    __threadfence();
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *flag >= want (acquire, system scope). Returns false on timeout.
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool wait_flag(const unsigned long long* flag, uint64_t want,
                                          uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_sys(flag) < want) {
    if (globaltimer_ns() - t0 > timeout_ns) return false;
    __nanosleep(64);
  }
  return true;
}

// Rank mode arrival gate inside a consumer kernel: warp 0 of block 0 polls
// the n peers' system-scope flags (lane s: flag s, with the watchdog) and then
// releases a LOCAL word; every block's thread 0 acquires that word at gpu
// scope.  Acquire (sys) -> release (gpu) -> acquire (gpu) is a causality
// chain, so every block sees the peers' data; and no grid of CTAs spins on
// NVLink lines (which slows the stores being waited for).
template <typename FlagOf>
__device__ __forceinline__ void arrival_gate(uint32_t n, FlagOf flag_of, uint32_t* go,
                                             uint32_t iter, uint32_t* status) {
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const unsigned long long* f = threadIdx.x < n ? flag_of(threadIdx.x) : nullptr;
    if (f && !wait_flag(f, iter, zen::kPeerTimeoutNs)) atomicOr(status, zen::kErrTimeout);
    __syncwarp();
    if (threadIdx.x == 0) st_release_gpu(go, iter);
  }
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_gpu(go) != iter) {
      if (globaltimer_ns() - t0 > zen::kPeerTimeoutNs) break;  // the poller reports it
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// 256-bit streaming load (sm_100 ld.v8): read once, no L1 allocation, evict
// first from L2 (keeps the resident tables/hash memory in the 126 MB L2 while
// the dense gradient streams through).  p must be 32-byte aligned.
struct f8 {
  float v[8];
};
__device__ __forceinline__ f8 ld_stream_f8(const void* p) {
  uint32_t r[8];
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
  f8 o;
#pragma unroll
  for (int i = 0; i < 8; ++i) o.v[i] = __uint_as_float(r[i]);
  return o;
}

}  // namespace zen_dev

namespace zen {
// Launch policy of the calling host thread (capi.cpp): programmatic dependent
// launch on/off and the CTA scheduling priority.  The BP side path (hash-memory
// layout) launches with PDL off and the least priority so that it fills the
// SMs the latency-bound critical path leaves idle instead of delaying it.
bool launch_pdl();
int launch_priority();

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = launch_pdl() ? 1 : 0;
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = launch_priority();
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace zen
