// capi.cpp -- C++ host side of the C-ABI (include/zen_b200.h).
//
// Owns devices, streams, workspaces and the cross-GPU plumbing; every byte of
// gradient data is touched only by the sm_100a kernels in k_*.cu.  There is no
// CPU fallback: a missing or non-sm_100 device is an error.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "zen_b200.h"
#include "zen_internal.h"

namespace zen {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static bool pdl_env() {
  static const bool on = [] {
    const char* e = std::getenv("ZEN_PDL");  // ZEN_PDL=0: A/B measurement
    return !(e && e[0] == '0');
  }();
  return on;
}
static int prio_range(bool least) {
  static int lo = 0, hi = 0;
  static const bool init = [] {
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least, hi = greatest
    return true;
  }();
  (void)init;
  return least ? lo : hi;
}
static thread_local bool t_pdl = true;
static thread_local int t_prio = 1 << 30;  // "unset": greatest priority
bool launch_pdl() { return t_pdl && pdl_env(); }
int launch_priority() { return t_prio == (1 << 30) ? prio_range(false) : t_prio; }
LaunchScope::LaunchScope(bool pdl, bool low_priority) : prev_pdl(t_pdl), prev_prio(t_prio) {
  t_pdl = pdl;
  t_prio = prio_range(low_priority);
}
LaunchScope::~LaunchScope() {
  t_pdl = prev_pdl;
  t_prio = prev_prio;
}

// extra small kernels (k_util.cu)
void launch_axpy_sparse(float* dense, uint64_t m, const uint64_t* idx, const float* val,
                        uint64_t count, float alpha, uint32_t* status, cudaStream_t stream);
void launch_dump_slots(const unsigned long long* slots, uint64_t cells, uint32_t epoch,
                       const float* vals, uint64_t* out_slots, float* out_vals,
                       cudaStream_t stream);
void launch_meta_depth(const uint32_t* meta, uint64_t count, uint32_t* out, cudaStream_t stream);
void launch_universe_indices(const OwnWord* own, uint64_t nwords, uint64_t* out,
                             cudaStream_t stream);
void launch_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t stream);
void launch_check_owned(const uint64_t* idx, uint64_t count, uint64_t m, const OwnWord* own,
                        HashHdr* hdr, cudaStream_t stream);
}  // namespace zen

using namespace zen;

namespace {

thread_local std::string t_msg;
thread_local int64_t t_part = -1;
thread_local uint64_t t_index = 0;

zen_status fail(zen_status s, const std::string& msg, int64_t part = -1) {
  t_msg = msg;
  t_part = part;
  return s;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      cudaGetLastError();                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? ZEN_E_OOM : ZEN_E_CUDA,             \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    }                                                                                   \
  } while (0)

#define CKR(expr)                       \
  do {                                  \
    zen_status s_ = (expr);             \
    if (s_ != ZEN_OK) return s_;        \
  } while (0)

constexpr uint64_t kG = 0x9e3779b97f4a7c15ULL;

uint64_t h_mix64(uint64_t x) {  // zen/hashing.hpp:18-25
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}
uint64_t h_derive(uint64_t m, uint64_t s) {  // zen/hashing.hpp:37-39
  return h_mix64(m ^ h_mix64(s + 0x5851f42d4c957f2dULL));
}

DevFamily fold(const zen_hash_family& f) {
  DevFamily d{};
  d.pc = kG * (f.partition_seed + 1);
  for (uint32_t i = 0; i < f.k; ++i) d.sc[i] = kG * (f.slot_seeds[i] + 1);
  d.n = f.partitions;
  d.k = f.k;
  return d;
}

uint32_t planes_for(uint32_t n) {
  if (n <= 1) return 0;
  uint32_t b = 0;
  while ((1u << b) < n) ++b;
  return b;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// Stream that orders setup-time zeroing and uploads.  PyTorch streams are
// cudaStreamNonBlocking, so legacy-stream cudaMemset/cudaMemcpy would NOT be
// ordered before kernels on the framework's stream: every API entry point
// scopes this to its context stream.
thread_local cudaStream_t t_setup = nullptr;
struct SetupStream {
  cudaStream_t prev;
  explicit SetupStream(cudaStream_t s) : prev(t_setup) { t_setup = s; }
  ~SetupStream() { t_setup = prev; }
};

// RAII list of device allocations
struct DevMem {
  std::vector<void*> ptrs;
  ~DevMem() { release(); }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  template <typename T>
  zen_status alloc(T** out, size_t count, bool zero = true) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    CK(cudaMalloc(&p, bytes));
    ptrs.push_back(p);
    if (zero) CK(cudaMemsetAsync(p, 0, bytes, t_setup));
    *out = static_cast<T*>(p);
    return ZEN_OK;
  }
};

template <typename T>
zen_status upload(T* d, const T* h, size_t count) {
  CK(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, t_setup));
  CK(cudaStreamSynchronize(t_setup));  // h may be a temporary
  return ZEN_OK;
}

}  // namespace

// ------------------------------------------------------------------ ctx ----

// top-k sparsification workspace, kept per context and grown on demand (the
// staging of the tile pass is 8 B per dense element)
struct TopkWs {
  DevMem mem;
  uint64_t m = 0;
  void* state = nullptr;
  uint32_t* hist = nullptr;
  ExtractWs<uint32_t> ex{};
  uint32_t* tile_ties = nullptr;
  uint64_t *tie_base = nullptr, *out_base = nullptr, *out_count = nullptr;
};

// grow-only device scratch of a context, carved up by one synchronous call at
// a time (the API is externally synchronous per context, like the reference)
struct Scratch {
  char* base = nullptr;
  size_t cap = 0;
  ~Scratch() {
    if (base) cudaFree(base);
  }
};
struct Bump {
  char* p = nullptr;
  size_t used = 0;
  template <typename T>
  T* get(size_t n) {
    T* r = reinterpret_cast<T*>(p + used);
    used += align256(std::max<size_t>(n, 1) * sizeof(T));
    return r;
  }
};
inline size_t bump_bytes(std::initializer_list<size_t> sizes) {
  size_t t = 0;
  for (size_t b : sizes) t += align256(std::max<size_t>(b, 1));
  return t;
}

struct zen_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  zen_universe* ident = nullptr;  // identity universe of the plain Bitmap format (lazy)
  std::unique_ptr<TopkWs> topk;
  Scratch scratch;
};

namespace {
zen_status ctx_scratch(zen_ctx* c, size_t bytes, Bump* out) {
  if (c->scratch.cap < bytes) {
    CK(cudaStreamSynchronize(c->stream));
    const size_t want = std::max(bytes, c->scratch.cap * 2);
    if (c->scratch.base) cudaFree(c->scratch.base);
    c->scratch.base = nullptr;
    c->scratch.cap = 0;
    if (cudaMalloc(&c->scratch.base, want) != cudaSuccess) {
      cudaGetLastError();
      return fail(ZEN_E_OOM, "cudaMalloc (scratch) failed");
    }
    c->scratch.cap = want;
  }
  out->p = c->scratch.base;
  out->used = 0;
  return ZEN_OK;
}
}  // namespace

extern "C" {

uint32_t zen_abi_version(void) { return ZEN_B200_ABI_VERSION; }

const char* zen_status_string(zen_status s) {
  switch (s) {
    case ZEN_OK: return "ok";
    case ZEN_E_INVALID: return "invalid argument";
    case ZEN_E_SERIAL_OVERFLOW: return "serial overflow";
    case ZEN_E_INDEX_OUTSIDE_UNIVERSE: return "index outside universe";
    case ZEN_E_MALFORMED: return "malformed payload";
    case ZEN_E_EMPTY: return "empty tensor";
    case ZEN_E_UNIVERSE_MISMATCH: return "universe mismatch";
    case ZEN_E_CUDA: return "cuda error";
    case ZEN_E_PEER: return "peer setup error";
    case ZEN_E_OOM: return "out of device memory";
    case ZEN_E_TIMEOUT: return "peer timeout";
    case ZEN_E_CAPACITY: return "capacity exceeded";
    case ZEN_E_INFEASIBLE: return "infeasible workload spec";
  }
  return "unknown";
}
const char* zen_last_error_message(void) { return t_msg.c_str(); }
int64_t zen_last_error_partition(void) { return t_part; }
uint64_t zen_last_error_index(void) { return t_index; }
uint64_t zen_kernel_launches(void) { return g_launches.load(); }

uint64_t zen_derive_seed(uint64_t master, uint64_t stream) { return h_derive(master, stream); }
uint64_t zen_mix64(uint64_t x) { return h_mix64(x); }
uint64_t zen_seeded_hash(uint64_t x, uint64_t seed) { return h_mix64(x + kG * (seed + 1)); }
uint64_t zen_map_to_range(uint64_t h, uint64_t range) {
  return uint64_t((static_cast<unsigned __int128>(h) * range) >> 64);
}

zen_status zen_hash_family_make(uint64_t seed, uint32_t n, uint32_t k, zen_hash_family* out) {
  // HashFamily::make, zen/hashing.hpp:51-60
  if (!out) return fail(ZEN_E_INVALID, "null output");
  if (n == 0) return fail(ZEN_E_INVALID, "hash family needs at least one partition");
  if (k == 0) return fail(ZEN_E_INVALID, "hash family needs at least one slot hash");
  if (k > ZEN_MAX_K) return fail(ZEN_E_INVALID, "rehash depth above ZEN_MAX_K");
  std::memset(out, 0, sizeof(*out));
  out->partitions = n;
  out->k = k;
  out->partition_seed = h_derive(seed, 0);
  for (uint32_t i = 0; i < k; ++i) out->slot_seeds[i] = h_derive(seed, 1 + i);
  return ZEN_OK;
}

zen_status zen_hash_family_make_worker(uint64_t shared, uint32_t worker, uint32_t n, uint32_t k,
                                       zen_hash_family* out) {
  // HashFamily::make_worker, zen/hashing.hpp:64-69
  CKR(zen_hash_family_make(shared, n, k, out));
  for (uint32_t i = 0; i < k; ++i) out->slot_seeds[i] = h_derive(shared, (uint64_t(worker) + 2) * 1024 + i);
  return ZEN_OK;
}

zen_status zen_ctx_create(int device, zen_ctx** out) {
  if (!out) return fail(ZEN_E_INVALID, "null output");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(ZEN_E_CUDA, "no CUDA device: the zen_b200 path has no CPU fallback");
  }
  if (device < 0 || device >= count) return fail(ZEN_E_INVALID, "device ordinal out of range");
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(ZEN_E_CUDA, std::string("zen_b200 kernels are built for sm_100a; device is ") +
                                prop.name);
  auto* c = new zen_ctx();
  c->device = device;
  DevGuard g(device);
  e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(ZEN_E_CUDA, cudaGetErrorString(e));
  }
  c->stream = c->own;
  *out = c;
  return ZEN_OK;
}

void zen_ctx_destroy(zen_ctx* c) {
  if (!c) return;
  DevGuard g(c->device);
  if (c->ident) zen_universe_destroy(c->ident);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

zen_status zen_ctx_set_stream(zen_ctx* c, void* s) {
  if (!c) return fail(ZEN_E_INVALID, "null ctx");
  c->stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
  return ZEN_OK;
}
void* zen_ctx_own_stream(zen_ctx* c) { return c ? (void*)c->own : nullptr; }
void* zen_ctx_stream(zen_ctx* c) { return c ? (void*)c->stream : nullptr; }
zen_status zen_ctx_synchronize(zen_ctx* c) {
  if (!c) return fail(ZEN_E_INVALID, "null ctx");
  DevGuard g(c->device);
  CK(cudaStreamSynchronize(c->stream));
  return ZEN_OK;
}

// ------------------------------------------------------------ standalone ----

zen_status zen_partition_of(zen_ctx* c, const uint64_t* d_idx, uint64_t count, uint64_t pseed,
                            uint32_t n, uint32_t* d_out) {
  if (!c || (!d_idx && count) || (!d_out && count)) return fail(ZEN_E_INVALID, "null argument");
  if (n == 0) return fail(ZEN_E_INVALID, "partition count must be at least 1");
  if (!count) return ZEN_OK;
  DevGuard g(c->device);
  launch_partition_of(d_idx, count, kG * (pseed + 1), n, d_out, c->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return ZEN_OK;
}

zen_status zen_to_sparse(zen_ctx* c, const float* d_dense, uint64_t m, uint64_t* d_idx,
                         float* d_val, uint64_t capacity, uint64_t* nnz) {
  if (!c || !d_dense || !nnz) return fail(ZEN_E_INVALID, "null argument");
  if (m == 0) return fail(ZEN_E_INVALID, "dense tensor must have at least one element");  // tensor.hpp:24
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  DevMem mem;
  const uint64_t ntiles = (m + kExtractTile - 1) / kExtractTile;
  ExtractWs<uint64_t> ws{};
  uint64_t* d_count;
  uint32_t* err;
  CKR(mem.alloc(&ws.st_idx, ntiles * kExtractTile, false));
  CKR(mem.alloc(&ws.st_val, ntiles * kExtractTile, false));
  CKR(mem.alloc(&ws.tile_cnt, ntiles));
  CKR(mem.alloc(&ws.tile_base, ntiles));
  ws.nblk = (std::min<uint64_t>(capacity, m) + 255) / 256;
  CKR(mem.alloc(&ws.blk_tile, ws.nblk + 1));
  CKR(mem.alloc(&d_count, 1));
  CKR(mem.alloc(&err, 1));
  launch_extract<uint64_t>(d_dense, m, ws, d_idx, d_val, d_count, capacity, err, c->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(nnz, d_count, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (*nnz > capacity) return fail(ZEN_E_CAPACITY, "output capacity below the non-zero count");
  return ZEN_OK;
}

namespace {
struct HashSchedule {
  uint32_t grid = 0, threads = 0;
  uint64_t mul = 0, add = 0;
};
thread_local HashSchedule t_sched;
}  // namespace

zen_status zen_debug_hash_schedule(uint32_t grid, uint32_t threads, uint64_t perm_mul,
                                   uint64_t perm_add) {
  if (threads && (threads % 32 || threads > 256))
    return fail(ZEN_E_INVALID, "threads must be a multiple of 32, <= 256");
  t_sched = HashSchedule{grid, threads, perm_mul, perm_add};
  return ZEN_OK;
}

zen_status zen_hierarchical_hash(zen_ctx* c, const uint64_t* d_idx, const float* d_val,
                                 uint64_t count, uint64_t universe, const zen_hash_family* fam,
                                 uint64_t r1, uint64_t r2, uint64_t* d_out_idx, float* d_out_val,
                                 uint64_t* part_count, uint64_t* d_slots, float* d_slot_vals,
                                 uint32_t* d_depth, zen_collision_stats* stats) {
  // validation: zen/hashing.hpp:184-187
  if (!c || !fam || !part_count) return fail(ZEN_E_INVALID, "null argument");
  const uint32_t n = fam->partitions, k = fam->k;
  if (n == 0) return fail(ZEN_E_INVALID, "hierarchical hash needs at least one partition");
  if (n > ZEN_MAX_PARTITIONS) return fail(ZEN_E_INVALID, "partition count above ZEN_MAX_PARTITIONS");
  if (k == 0 || k > ZEN_MAX_K) return fail(ZEN_E_INVALID, "rehash depth out of range");
  if (r1 < 1) return fail(ZEN_E_INVALID, "parallel region must have at least one slot");
  if (universe > kKeyMask) return fail(ZEN_E_INVALID, "universe above 2^40 - 1");
  if (count && (!d_idx || !d_val || !d_out_idx || !d_out_val))
    return fail(ZEN_E_INVALID, "null tensor pointer");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const uint64_t stride = r1 + r2;
  const uint64_t cells = uint64_t(n) * stride;
  const uint64_t cap = std::max<uint64_t>(count, 1);
  const uint64_t ntiles = (cap + kHashTile - 1) / kHashTile;
  DevMem mem;
  HashArgs<uint64_t> a{};
  a.idx = d_idx;
  a.val = d_val;
  a.fam = fold(*fam);
  CKR(mem.alloc(&a.hdr, 1));
  CKR(mem.alloc(&a.slots, cells, false));
  CK(cudaMemsetAsync(a.slots, 0xFF, std::max<size_t>(cells * 8, 16), t_setup));
  const bool dump = d_slots || d_slot_vals;
  if (dump) CKR(mem.alloc(&a.slot_vals, cells));
  CKR(mem.alloc(&a.meta, cap));
  CKR(mem.alloc(&a.pmeta, cap));
  CKR(mem.alloc(&a.tile_cnt, ntiles * n));
  CKR(mem.alloc(&a.tile_scnt, ntiles * n));
  CKR(mem.alloc(&a.load, n));
  CKR(mem.alloc(&a.sload, n));
  CKR(mem.alloc(&a.part_off, n));
  CKR(mem.alloc(&a.fallback, n));
  CKR(mem.alloc(&a.stats, n * (k + 1)));
  CKR(mem.alloc(&a.fb_stats, n * (k + 1)));
  CKR(mem.alloc(&a.stats_out, k + 1));
  a.dst_table = 0;
  a.out_idx = d_out_idx;
  a.out_val = d_out_val;
  a.cap = cap;
  a.tiles_cap = ntiles;
  a.stride_cap = stride;
  a.place_grid = t_sched.grid;
  a.place_threads = t_sched.threads;
  if (t_sched.mul && count && std::gcd(t_sched.mul % count, count) == 1) {
    a.perm_mul = t_sched.mul % count;  // a bijection of [0, count)
    a.perm_add = t_sched.add % count;
  }
  HashHdr h{};
  h.count = count;
  h.r1 = r1;
  h.r2 = r2;
  h.derive = 0;
  h.epoch = 0;
  h.bad_index = ~0ull;
  CKR(upload(a.hdr, &h, 1));
  launch_hash<uint64_t>(a, n, k, c->stream);
  CK(cudaGetLastError());
  HashHdr hr{};
  std::vector<uint32_t> load(n);
  std::vector<uint64_t> st(k + 1);
  CK(cudaMemcpyAsync(&hr, a.hdr, sizeof(hr), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(load.data(), a.load, n * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(st.data(), a.stats_out, (k + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
  if (dump) {
    launch_dump_slots(a.slots, cells, 1, a.slot_vals, d_slots, d_slot_vals, c->stream);
  }
  if (d_depth && count) launch_meta_depth(a.meta, count, d_depth, c->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  if (hr.status & kErrCapacity) return fail(ZEN_E_CAPACITY, "hash workspace capacity");
  if (hr.ovf_word != ~0ull) {  // zen/hashing.hpp:221-222
    const uint32_t p = uint32_t(hr.ovf_word & 0xFFFF);
    return fail(ZEN_E_SERIAL_OVERFLOW,
                "hash partition " + std::to_string(p) +
                    " exceeded its slot capacity (r2 too small for this workload)",
                p);
  }
  for (uint32_t p = 0; p < n; ++p) part_count[p] = load[p];
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->k = k;
    stats->serial_writes = st[0];
    for (uint32_t d = 0; d < k; ++d) stats->placed_at_depth[d] = st[1 + d];
  }
  return ZEN_OK;
}

}  // extern "C"

// --------------------------------------------------------------- universe ----

struct zen_universe {
  zen_ctx* ctx = nullptr;
  uint64_t m = 0;
  uint32_t n = 0;
  uint64_t pseed = 0;
  uint32_t nplanes = 0;
  uint64_t nwords = 0, nchunks = 0;
  std::vector<uint64_t> bs;
  DevMem mem;
  unsigned long long* planes = nullptr;
  uint32_t* cprefix = nullptr;
  uint64_t* d_bs = nullptr;
  std::vector<OwnWord*> own;

  zen_status build() {
    nplanes = planes_for(n);
    nwords = (m + 63) / 64;
    nchunks = (nwords + 31) / 32;
    CKR(mem.alloc(&planes, std::max<uint64_t>(nwords * nplanes, 1)));
    CKR(mem.alloc(&cprefix, nchunks * n));
    CKR(mem.alloc(&d_bs, n));
    launch_tables_planes(m, n, kG * (pseed + 1), nplanes, planes, cprefix, ctx->stream);
    launch_tables_scan(cprefix, nchunks, n, d_bs, ctx->stream);
    CK(cudaGetLastError());
    bs.resize(n);
    CK(cudaMemcpyAsync(bs.data(), d_bs, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    own.assign(n, nullptr);
    return ZEN_OK;
  }
  // {mask, rank base} per word and select samples for server s (lazy)
  zen_status ensure_own(uint32_t s) {
    if (own[s]) return ZEN_OK;
    CKR(mem.alloc(&own[s], nwords));
    launch_tables_own(m, n, s, nplanes, planes, cprefix, own[s], nullptr, 0, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return ZEN_OK;
  }
};

namespace {

// Decoder scratch for a set of present servers; shared by the standalone codec
// and the BP receiver.
struct Decoder {
  DevMem mem;
  uint32_t* bpre = nullptr;
  uint32_t* bpre_blk = nullptr;
  uint32_t* blk_start = nullptr;
  uint64_t* nwords_s = nullptr;
  uint32_t* popc_total = nullptr;
  uint32_t* done = nullptr;
  uint64_t words_stride = 0, blk_stride = 0;
  uint32_t total_blocks = 0;

  zen_status init(const zen_universe* u, const std::vector<bool>& present) {
    const uint32_t n = u->n;
    std::vector<uint32_t> bstart(n + 1, 0);
    std::vector<uint64_t> nws(n, 0);
    for (uint32_t s = 0; s < n; ++s) {
      nws[s] = (u->bs[s] + 63) / 64;
      words_stride = std::max(words_stride, nws[s]);
      const uint32_t nb = present[s] ? uint32_t((nws[s] + kPrefixBlockWords - 1) / kPrefixBlockWords) : 0u;
      blk_stride = std::max<uint64_t>(blk_stride, nb);
      bstart[s + 1] = bstart[s] + nb;
    }
    total_blocks = bstart[n];
    words_stride = (std::max<uint64_t>(words_stride, 1) + 7) & ~uint64_t(7);
    blk_stride = std::max<uint64_t>(blk_stride, 1);
    CKR(mem.alloc(&bpre, words_stride * n));
    CKR(mem.alloc(&bpre_blk, blk_stride * n));
    CKR(mem.alloc(&blk_start, n + 1));
    CKR(mem.alloc(&nwords_s, n));
    CKR(mem.alloc(&popc_total, n));
    CKR(mem.alloc(&done, 1));
    CKR(upload(blk_start, bstart.data(), n + 1));
    CKR(upload(nwords_s, nws.data(), n));
    return ZEN_OK;
  }
  void fill(DecodeArgs& a, const zen_universe* u) const {
    a.n = u->n;
    a.m = u->m;
    a.nplanes = u->nplanes;
    a.planes = u->planes;
    a.cprefix = u->cprefix;
    a.bs = u->d_bs;
    a.nwords_s = nwords_s;
    a.blk_start = blk_start;
    a.total_blocks = total_blocks;
    a.bpre = bpre;
    a.bpre_blk = bpre_blk;
    a.words_stride = words_stride;
    a.blk_stride = blk_stride;
    a.done = done;
    a.popc_total = popc_total;
  }
  void launch(const DecodeArgs& a, cudaStream_t st) const { launch_decode_parts(a, st); }
};

// scratch of the aggregate + encode (see k_codec.cu)
zen_status alloc_agg_ws(DevMem& mem, AggArgs& a, uint32_t nparts, uint64_t bs) {
  a.nw = std::max<uint64_t>((bs + 63) / 64, 1);
  a.nws = (a.nw + 7) & ~uint64_t(7);
  a.nblk = uint32_t((a.nw + kPrefixBlockWords - 1) / kPrefixBlockWords);
  CKR(mem.alloc(&a.pw, size_t(nparts) * a.nws));
  CKR(mem.alloc(&a.pre, size_t(nparts + 1) * a.nws, false));
  // worker rows start at ~0: the push scatter's marks take atomicMin (local
  // mode) and k_agg_values resets every row word it reads
  CK(cudaMemsetAsync(a.pre, 0xFF, size_t(nparts) * a.nws * sizeof(uint32_t), t_setup));
  CKR(mem.alloc(&a.blk, size_t(nparts + 1) * a.nblk));
  CKR(mem.alloc(&a.done, 2));
  return ZEN_OK;
}

}  // namespace

extern "C" {

zen_status zen_universe_create(zen_ctx* c, uint64_t m, uint32_t n, uint64_t pseed,
                               zen_universe** out) {
  if (!c || !out) return fail(ZEN_E_INVALID, "null argument");
  if (n == 0) return fail(ZEN_E_INVALID, "hash universe table needs at least one server");
  if (n > ZEN_MAX_PARTITIONS) return fail(ZEN_E_INVALID, "server count above ZEN_MAX_PARTITIONS");
  if (m == 0 || m >= 0xFFFFFFFFull) return fail(ZEN_E_INVALID, "universe must be in [1, 2^32-1)");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  auto u = std::make_unique<zen_universe>();
  u->ctx = c;
  u->m = m;
  u->n = n;
  u->pseed = pseed;
  CKR(u->build());
  *out = u.release();
  return ZEN_OK;
}

void zen_universe_destroy(zen_universe* u) {
  if (!u) return;
  DevGuard g(u->ctx->device);
  delete u;
}

uint64_t zen_universe_size(const zen_universe* u, uint32_t s) {
  return (u && s < u->n) ? u->bs[s] : 0;
}

zen_status zen_universe_indices(zen_universe* u, uint32_t s, uint64_t* d_out) {
  if (!u || s >= u->n) return fail(ZEN_E_INVALID, "bad universe/server");
  DevGuard g(u->ctx->device);
  SetupStream setup_(u->ctx->stream);
  CKR(u->ensure_own(s));
  launch_universe_indices(u->own[s], u->nwords, d_out, u->ctx->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(u->ctx->stream));
  return ZEN_OK;
}

zen_status zen_hash_bitmap_encode(zen_universe* u, uint32_t s, const uint64_t* d_idx,
                                  const float* d_val, uint64_t count, uint8_t* d_payload,
                                  uint64_t* index_bits, uint64_t* payload_bytes) {
  if (!u || s >= u->n) return fail(ZEN_E_INVALID, "bad universe/server");
  if (count && (!d_idx || !d_val)) return fail(ZEN_E_INVALID, "null tensor");
  zen_ctx* c = u->ctx;
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  CKR(u->ensure_own(s));
  const uint64_t bs = u->bs[s];
  const uint64_t nw = (bs + 63) / 64;
  const uint64_t bitmap_bytes = (bs + 7) / 8;
  DevMem mem;
  uint32_t* keys;
  unsigned long long* bits;
  float* vals;
  HashHdr* hdr;
  uint64_t* aggc;
  uint64_t* d_cnt;
  const uint32_t** in_idx;
  const float** in_val;
  unsigned long long** dst_bits;
  float** dst_vals;
  CKR(mem.alloc(&keys, std::max<uint64_t>(count, 1)));
  CKR(mem.alloc(&bits, (std::max<uint64_t>(nw, 1) + 7) & ~uint64_t(7)));
  CKR(mem.alloc(&vals, std::max<uint64_t>(count, 1)));
  CKR(mem.alloc(&hdr, 1));
  CKR(mem.alloc(&aggc, 1));
  CKR(mem.alloc(&d_cnt, 1));
  CKR(mem.alloc(&in_idx, 1));
  CKR(mem.alloc(&in_val, 1));
  CKR(mem.alloc(&dst_bits, 1));
  CKR(mem.alloc(&dst_vals, 1));
  HashHdr h{};
  h.bad_index = ~0ull;
  CKR(upload(hdr, &h, 1));
  CKR(upload(d_cnt, &count, 1));
  const uint32_t* ki = keys;
  const float* vi = d_val;
  CKR(upload(in_idx, &ki, 1));
  CKR(upload(in_val, &vi, 1));
  CKR(upload(dst_bits, &bits, 1));
  CKR(upload(dst_vals, &vals, 1));
  if (count) {
    launch_check_owned(d_idx, count, u->m, u->own[s], hdr, c->stream);
    HashHdr hc{};
    CK(cudaMemcpyAsync(&hc, hdr, sizeof(hc), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hc.status & kErrOutside) {  // universe_positions, zen/codec.hpp:152-154
      t_index = hc.bad_index;
      return fail(ZEN_E_INDEX_OUTSIDE_UNIVERSE, "index " + std::to_string(hc.bad_index) +
                                                    " is not owned by server " + std::to_string(s));
    }
    launch_u64_to_u32(d_idx, keys, count, c->stream);
  }
  AggArgs a{};
  a.n = 1;
  a.s = s;
  a.m = u->m;
  a.in_idx = in_idx;
  a.in_val = in_val;
  a.in_hdr = nullptr;
  a.in_count = d_cnt;
  a.own = u->own[s];
  a.bs = bs;
  CKR(alloc_agg_ws(mem, a, 1, bs));
  a.ndst = 1;
  a.dst_bits = dst_bits;
  a.dst_vals = dst_vals;
  a.dst_hdr = nullptr;
  a.val_cap = count;
  a.agg_count = aggc;
  a.hdr = hdr;
  a.wait_push = 0;
  launch_aggregate(a, c->stream);
  CK(cudaGetLastError());
  HashHdr hr{};
  uint64_t u_count = 0;
  CK(cudaMemcpyAsync(&hr, hdr, sizeof(hr), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&u_count, aggc, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (hr.status & kErrOutside) {  // universe_positions, zen/codec.hpp:152-154
    t_index = hr.bad_index;
    return fail(ZEN_E_INDEX_OUTSIDE_UNIVERSE, "index " + std::to_string(hr.bad_index) +
                                                  " is not owned by server " + std::to_string(s));
  }
  if (u_count != count) return fail(ZEN_E_INVALID, "tensor indices not sorted/unique or >= M");
  if (bitmap_bytes)
    CK(cudaMemcpyAsync(d_payload, bits, bitmap_bytes, cudaMemcpyDeviceToDevice, c->stream));
  if (count)
    CK(cudaMemcpyAsync(d_payload + bitmap_bytes, vals, count * 4, cudaMemcpyDeviceToDevice,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (index_bits) *index_bits = bs;
  if (payload_bytes) *payload_bytes = bitmap_bytes + 4 * count;
  return ZEN_OK;
}

zen_status zen_hash_bitmap_decode(zen_universe* u, uint32_t s, const uint8_t* d_payload,
                                  uint64_t payload_bytes, uint64_t count, uint64_t* d_idx,
                                  float* d_val) {
  if (!u || s >= u->n) return fail(ZEN_E_INVALID, "bad universe/server");
  if (u->n > ZEN_MAX_WORKERS) return fail(ZEN_E_INVALID, "decode supports n <= ZEN_MAX_WORKERS");
  zen_ctx* c = u->ctx;
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const uint64_t bs = u->bs[s];
  const uint64_t nw = (bs + 63) / 64;
  const uint64_t bitmap_bytes = (bs + 7) / 8;
  if (payload_bytes != bitmap_bytes + 4 * count)  // zen/codec.hpp:336-337
    return fail(ZEN_E_MALFORMED, "hash bitmap payload size mismatch");
  DevMem mem;
  unsigned long long* bits;
  float* vals;
  HashHdr* hdr;
  uint64_t* out_count;
  const unsigned long long** bits_t;
  const float** vals_t;
  CKR(mem.alloc(&bits, (std::max<uint64_t>(nw, 1) + 7) & ~uint64_t(7)));
  CKR(mem.alloc(&vals, std::max<uint64_t>(count, 1)));
  CKR(mem.alloc(&hdr, 1));
  CKR(mem.alloc(&out_count, 1));
  CKR(mem.alloc(&bits_t, u->n));
  CKR(mem.alloc(&vals_t, u->n));
  if (bitmap_bytes)
    CK(cudaMemcpyAsync(bits, d_payload, bitmap_bytes, cudaMemcpyDeviceToDevice, c->stream));
  if (count)
    CK(cudaMemcpyAsync(vals, d_payload + bitmap_bytes, count * 4, cudaMemcpyDeviceToDevice,
                       c->stream));
  std::vector<const unsigned long long*> hb(u->n, nullptr);
  std::vector<const float*> hv(u->n, nullptr);
  hb[s] = bits;
  hv[s] = vals;
  CKR(upload(bits_t, hb.data(), u->n));
  CKR(upload(vals_t, hv.data(), u->n));
  std::vector<bool> present(u->n, false);
  present[s] = true;
  Decoder dec;
  CKR(dec.init(u, present));
  uint64_t* tmp_idx;
  float* tmp_val;
  CKR(mem.alloc(&tmp_idx, std::max<uint64_t>(count, 1)));
  CKR(mem.alloc(&tmp_val, std::max<uint64_t>(count, 1)));
  DecodeArgs a{};
  dec.fill(a, u);
  a.bits = bits_t;
  a.vals = vals_t;
  a.pull_hdr = nullptr;
  a.out_idx = tmp_idx;
  a.out_val = tmp_val;
  a.out_count = out_count;
  a.out_cap = count;
  a.hdr = hdr;
  a.wait_pull = 0;
  dec.launch(a, c->stream);
  CK(cudaGetLastError());
  std::vector<uint32_t> popc(u->n);
  uint64_t oc = 0;
  CK(cudaMemcpyAsync(popc.data(), dec.popc_total, u->n * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&oc, out_count, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (popc[s] != count || oc != count)  // zen/codec.hpp:342
    return fail(ZEN_E_MALFORMED, "hash bitmap population mismatch");
  if (count) {
    CK(cudaMemcpyAsync(d_idx, tmp_idx, count * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(d_val, tmp_val, count * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return ZEN_OK;
}

}  // extern "C"

// ------------------------------------------------------------ wire formats ----
// zen::encode / zen::decode for every WireKind and the frame header
// (zen/codec.hpp:19-410).  Synchronous, like the reference's calls.

namespace {

zen_status wire_check_format(const zen_wire_format* f) {
  if (!f) return fail(ZEN_E_INVALID, "null wire format");
  if (f->kind < ZEN_WIRE_COO || f->kind > ZEN_WIRE_HASH_BITMAP)
    return fail(ZEN_E_MALFORMED, "unknown wire format tag");
  if (f->kind == ZEN_WIRE_COO && f->coo_index_bits != 32 && f->coo_index_bits != 64)
    return fail(ZEN_E_INVALID, "COO index width must be 32 or 64");
  if (f->kind == ZEN_WIRE_TENSOR_BLOCK && f->block_size < 1)
    return fail(ZEN_E_INVALID, "tensor block size must be at least 1");
  return ZEN_OK;
}

// the plain Bitmap is the HashBitmap over the one-server (identity) universe
zen_status identity_universe(zen_ctx* c, uint64_t m, zen_universe** out) {
  if (m >= 0xFFFFFFFFull) return fail(ZEN_E_INVALID, "bitmap universe must be below 2^32");
  if (!c->ident || zen_universe_size(c->ident, 0) != m) {
    if (c->ident) zen_universe_destroy(c->ident);
    c->ident = nullptr;
    CKR(zen_universe_create(c, m, 1, 0, &c->ident));
  }
  *out = c->ident;
  return ZEN_OK;
}

zen_status wire_status(uint32_t st) {
  if (st & kWireIdxOverflow) return fail(ZEN_E_INVALID, "index does not fit a 32-bit COO entry");
  if (st & kWireMalformed) return fail(ZEN_E_MALFORMED, "tensor block payload malformed");
  if (st & kWireRange) return fail(ZEN_E_INVALID, "sparse tensor index outside [0, M)");
  if (st & kWireDup) return fail(ZEN_E_INVALID, "duplicate index in sparse tensor");
  return ZEN_OK;
}

// input of an encode: a valid SparseTensor (sorted, unique, < M)
zen_status wire_check_input(zen_ctx* c, const uint64_t* d_idx, uint64_t count, uint64_t m,
                            uint32_t* st) {
  if (!count) return ZEN_OK;
  launch_check_canonical(d_idx, count, m, st, c->stream);
  uint32_t h = 0;
  CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (h) return fail(ZEN_E_INVALID, "tensor indices not sorted/unique or >= M");
  return ZEN_OK;
}

}  // namespace

extern "C" {

zen_status zen_encode(zen_ctx* c, const zen_wire_format* f, zen_universe* u, uint32_t server,
                      const uint64_t* d_idx, const float* d_val, uint64_t count, uint64_t m,
                      uint8_t* d_payload, uint64_t capacity, zen_message_info* out) {
  if (!c || !out) return fail(ZEN_E_INVALID, "null argument");
  CKR(wire_check_format(f));
  if (m == 0) return fail(ZEN_E_INVALID, "sparse tensor universe must be at least 1");
  if (count && (!d_idx || !d_val)) return fail(ZEN_E_INVALID, "null tensor");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const bool tb = f->kind == ZEN_WIRE_TENSOR_BLOCK;
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({4, tb ? 4 * count : 0, tb ? 4 * count : 0,
                                 tb ? wire_scan_bytes(count) : 0}), &sc));
  uint32_t* st = sc.get<uint32_t>(1);
  CK(cudaMemsetAsync(st, 0, 4, c->stream));
  CKR(wire_check_input(c, d_idx, count, m, st));
  zen_message_info info{m, count, 0, 32 * count, 0};
  switch (f->kind) {
    case ZEN_WIRE_COO: {
      const int ib = int(f->coo_index_bits / 8);
      info.index_bits = uint64_t(f->coo_index_bits) * count;
      info.payload_bytes = uint64_t(ib + 4) * count;
      *out = info;
      if (info.payload_bytes > capacity) return fail(ZEN_E_CAPACITY, "payload capacity");
      if (count && !d_payload) return fail(ZEN_E_INVALID, "null payload");
      launch_coo_encode(d_idx, d_val, count, ib, d_payload, st, c->stream);
      uint32_t h = 0;
      CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      return wire_status(h);
    }
    case ZEN_WIRE_BITMAP:
    case ZEN_WIRE_HASH_BITMAP: {
      zen_universe* uu = u;
      uint32_t s = server;
      if (f->kind == ZEN_WIRE_BITMAP) {
        CKR(identity_universe(c, m, &uu));
        s = 0;
      } else {
        if (!uu) return fail(ZEN_E_INVALID, "hash bitmap requires a hash universe");
        if (s >= uu->n) return fail(ZEN_E_INVALID, "bad universe/server");
        if (uu->m != m) return fail(ZEN_E_UNIVERSE_MISMATCH, "tensor and universe sizes differ");
      }
      const uint64_t bs = uu->bs[s];
      info.index_bits = bs;
      info.payload_bytes = (bs + 7) / 8 + 4 * count;
      *out = info;
      if (info.payload_bytes > capacity) return fail(ZEN_E_CAPACITY, "payload capacity");
      uint64_t ib = 0, pb = 0;
      return zen_hash_bitmap_encode(uu, s, d_idx, d_val, count, d_payload, &ib, &pb);
    }
    default: {  // ZEN_WIRE_TENSOR_BLOCK
      const uint64_t B = f->block_size;
      uint64_t nb = 0, last = 0;
      uint32_t *first = nullptr, *bpos = nullptr;
      if (count) {
        const size_t tmp_bytes = wire_scan_bytes(count);
        first = sc.get<uint32_t>(count);
        bpos = sc.get<uint32_t>(count);
        void* tmp = sc.get<uint8_t>(tmp_bytes);
        launch_tb_blocks(d_idx, count, B, first, bpos, tmp, tmp_bytes, c->stream);
        uint32_t hb = 0;
        CK(cudaMemcpyAsync(&hb, bpos + count - 1, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&last, d_idx + count - 1, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        nb = hb;
      }
      const uint64_t begin_last = (last / B) * B;
      const uint64_t len_last = nb ? std::min<uint64_t>(B, m - begin_last) : 0;
      const uint64_t values = nb ? (nb - 1) * B + len_last : 0;
      info.count = nb;
      info.index_bits = 64 * nb;
      info.value_bits = 32 * values;
      info.payload_bytes = 8 * nb + 4 * values;
      *out = info;
      if (info.payload_bytes > capacity) return fail(ZEN_E_CAPACITY, "payload capacity");
      if (!count) return ZEN_OK;
      CK(cudaMemsetAsync(d_payload, 0, info.payload_bytes, c->stream));
      launch_tb_write(d_idx, d_val, count, B, first, bpos, d_payload, c->stream);
      CK(cudaStreamSynchronize(c->stream));
      return ZEN_OK;
    }
  }
}

zen_status zen_decode(zen_ctx* c, const zen_wire_format* f, zen_universe* u, uint32_t server,
                      const zen_message_info* msg, const uint8_t* d_payload, uint64_t* d_idx,
                      float* d_val, uint64_t capacity, uint64_t* count) {
  if (!c || !msg || !count) return fail(ZEN_E_INVALID, "null argument");
  CKR(wire_check_format(f));
  const uint64_t m = msg->universe_size, n = msg->count, len = msg->payload_bytes;
  if (m == 0) return fail(ZEN_E_INVALID, "sparse tensor universe must be at least 1");
  if (len && !d_payload) return fail(ZEN_E_INVALID, "null payload");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const uint64_t slots = f->kind == ZEN_WIRE_TENSOR_BLOCK ? n * f->block_size : 0;
  const uint64_t maxout = f->kind == ZEN_WIRE_TENSOR_BLOCK ? slots : n;
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({4, 8, 8 * n, 8 * n, 4 * n, 8 * slots, 4 * slots, slots,
                                 8 * slots, 4 * slots, wire_select_bytes(slots), 8 * maxout,
                                 4 * maxout, wire_sort_bytes(maxout)}),
                  &sc));
  uint32_t* st = sc.get<uint32_t>(1);
  CK(cudaMemsetAsync(st, 0, 4, c->stream));
  uint64_t got = 0;
  switch (f->kind) {
    case ZEN_WIRE_COO: {
      const int ib = int(f->coo_index_bits / 8);
      if (len != uint64_t(ib + 4) * n) return fail(ZEN_E_MALFORMED, "COO payload size mismatch");
      *count = n;
      if (n > capacity) return fail(ZEN_E_CAPACITY, "output capacity");
      launch_coo_decode(d_payload, n, ib, m, d_idx, d_val, st, c->stream);
      got = n;
      break;
    }
    case ZEN_WIRE_BITMAP:
    case ZEN_WIRE_HASH_BITMAP: {
      zen_universe* uu = u;
      uint32_t s = server;
      if (f->kind == ZEN_WIRE_BITMAP) {
        CKR(identity_universe(c, m, &uu));
        s = 0;
      } else if (!uu) {
        return fail(ZEN_E_INVALID, "hash bitmap requires the encoding universe");
      }
      *count = n;
      if (n > capacity) return fail(ZEN_E_CAPACITY, "output capacity");
      return zen_hash_bitmap_decode(uu, s, d_payload, len, n, d_idx, d_val);
    }
    default: {  // ZEN_WIRE_TENSOR_BLOCK
      const uint64_t B = f->block_size;
      uint64_t* dcount = sc.get<uint64_t>(1);
      uint64_t* off = sc.get<uint64_t>(n);
      uint64_t* begin = sc.get<uint64_t>(n);
      uint32_t* blen = sc.get<uint32_t>(n);
      // parallel offsets for a regular payload; the sequential walk otherwise
      launch_tb_offsets(d_payload, len, n, B, m, off, begin, blen, st, c->stream);
      uint32_t h = 0;
      CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if ((h & kWireIrregularLayout) || (n == 0 && len != 0)) {
        CK(cudaMemsetAsync(st, 0, 4, c->stream));
        launch_tb_walk(d_payload, len, n, B, m, off, begin, blen, st, c->stream);
        CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (h) return wire_status(h);
      }
      if (slots) {
        uint64_t* sidx = sc.get<uint64_t>(slots);
        float* sval = sc.get<float>(slots);
        uint8_t* flag = sc.get<uint8_t>(slots);
        uint64_t* oi = sc.get<uint64_t>(slots);
        float* ov = sc.get<float>(slots);
        const size_t tb = wire_select_bytes(slots);
        void* tmp = sc.get<uint8_t>(tb);
        launch_tb_expand_select(d_payload, n, B, off, begin, blen, sidx, sval, flag, oi, ov,
                                dcount, tmp, tb, c->stream);
        CK(cudaMemcpyAsync(&got, dcount, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *count = got;
        if (got > capacity) return fail(ZEN_E_CAPACITY, "output capacity");
        if (got) {
          CK(cudaMemcpyAsync(d_idx, oi, got * 8, cudaMemcpyDeviceToDevice, c->stream));
          CK(cudaMemcpyAsync(d_val, ov, got * 4, cudaMemcpyDeviceToDevice, c->stream));
        }
      }
      *count = got;
      break;
    }
  }
  // SparseTensor(M, idx, val): sort when unsorted, then range / duplicate checks
  launch_check_canonical(d_idx, got, m, st, c->stream);
  uint32_t h = 0;
  CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (h & kWireUnsorted) {
    const size_t tb = wire_sort_bytes(got);
    uint64_t* ki = sc.get<uint64_t>(got);
    float* vi = sc.get<float>(got);
    void* tmp = sc.get<uint8_t>(tb);
    CK(cudaMemcpyAsync(ki, d_idx, got * 8, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(vi, d_val, got * 4, cudaMemcpyDeviceToDevice, c->stream));
    launch_sort_pairs(ki, d_idx, vi, d_val, got, tmp, tb, c->stream);
    CK(cudaMemsetAsync(st, 0, 4, c->stream));
    launch_check_canonical(d_idx, got, m, st, c->stream);
    CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return wire_status(h & ~kWireUnsorted);
}

zen_status zen_frame_header(const zen_wire_format* f, const zen_message_info* msg, uint8_t* out) {
  if (!f || !msg || !out) return fail(ZEN_E_INVALID, "null argument");
  auto put = [&](size_t at, uint64_t v, int nb) {
    for (int b = 0; b < nb; ++b) out[at + b] = uint8_t(v >> (8 * b));
  };
  put(0, f->kind, 1);
  put(1, f->block_size, 4);
  put(5, f->coo_index_bits, 4);
  put(9, msg->universe_size, 8);
  put(17, msg->count, 8);
  put(25, msg->index_bits + msg->value_bits, 8);
  return ZEN_OK;
}

zen_status zen_frame_parse(const uint8_t* in, uint64_t available, zen_wire_format* f,
                           zen_message_info* msg) {
  if (!in || !f || !msg) return fail(ZEN_E_INVALID, "null argument");
  if (available < ZEN_FRAME_HEADER_BYTES) return fail(ZEN_E_MALFORMED, "unexpected end of stream");
  auto get = [&](size_t at, int nb) {
    uint64_t v = 0;
    for (int b = 0; b < nb; ++b) v |= uint64_t(in[at + b]) << (8 * b);
    return v;
  };
  const uint64_t tag = get(0, 1);
  if (tag < 1 || tag > 4) return fail(ZEN_E_MALFORMED, "unknown wire format tag");
  f->kind = uint32_t(tag);
  f->block_size = uint32_t(get(1, 4));
  f->coo_index_bits = uint32_t(get(5, 4));
  msg->universe_size = get(9, 8);
  msg->count = get(17, 8);
  const uint64_t bits = get(25, 8), c = msg->count;
  switch (tag) {  // codec.hpp:380-405: accounting rebuilt from the format, then checked
    case ZEN_WIRE_COO:
      msg->index_bits = uint64_t(f->coo_index_bits) * c;
      msg->value_bits = 32 * c;
      msg->payload_bytes = (f->coo_index_bits / 8 + 4) * c;
      break;
    case ZEN_WIRE_BITMAP:
      msg->index_bits = msg->universe_size;
      msg->value_bits = 32 * c;
      msg->payload_bytes = (msg->universe_size + 7) / 8 + 4 * c;
      break;
    case ZEN_WIRE_TENSOR_BLOCK:
      msg->index_bits = 64 * c;
      msg->value_bits = bits >= msg->index_bits ? bits - msg->index_bits : 0;
      if (msg->value_bits % 32)
        return fail(ZEN_E_MALFORMED, "tensor block value bits not 32-aligned");
      msg->payload_bytes = 8 * c + msg->value_bits / 8;
      break;
    default:
      msg->index_bits = bits >= 32 * c ? bits - 32 * c : 0;
      msg->value_bits = 32 * c;
      msg->payload_bytes = (msg->index_bits + 7) / 8 + 4 * c;
      break;
  }
  if (msg->index_bits + msg->value_bits != bits)
    return fail(ZEN_E_MALFORMED, "frame bit accounting mismatch");
  if (available < ZEN_FRAME_HEADER_BYTES + msg->payload_bytes)
    return fail(ZEN_E_MALFORMED, "frame payload truncated");
  return ZEN_OK;
}

}  // extern "C"

// ------------------------------------------------------------- merge_sum ----
// zen::merge_sum (zen/tensor.hpp:133-167): the fold step of every scheme;
// Hierarchical Centralization (zen/schemes.hpp:173-193) is one per stage.

extern "C" zen_status zen_merge_sum(zen_ctx* c, const uint64_t* a_idx, const float* a_val,
                                    uint64_t na, const uint64_t* b_idx, const float* b_val,
                                    uint64_t nb, uint64_t universe, uint64_t* d_idx,
                                    float* d_val, uint64_t capacity, uint64_t* count) {
  if (!c || !count) return fail(ZEN_E_INVALID, "null argument");
  if ((na && (!a_idx || !a_val)) || (nb && (!b_idx || !b_val)))
    return fail(ZEN_E_INVALID, "null tensor");
  if (na + nb >= (1ull << 31)) return fail(ZEN_E_INVALID, "merge above 2^31 entries");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  // one merge-path kernel (k_merge.cu); counts in device memory
  const uint32_t tiles = hc_merge_tiles(na + nb);
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({32, sizeof(LookbackCtl), 8ull * tiles, 8ull * (tiles + 2)}), &sc));
  uint64_t* st = sc.get<uint64_t>(4);  // [na, nb, out count, status]
  LookbackCtl* ctl = sc.get<LookbackCtl>(1);
  unsigned long long* lb = sc.get<unsigned long long>(tiles);
  uint64_t* splits = sc.get<uint64_t>(tiles + 2);
  const uint64_t h_in[4] = {na, nb, 0, 0};
  CK(cudaMemcpyAsync(st, h_in, 32, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(ctl, 0, sizeof(LookbackCtl), c->stream));
  CK(cudaMemsetAsync(lb, 0, 8ull * tiles, c->stream));
  // both inputs must be SparseTensors of the same universe (tensor.hpp:133-135)
  uint32_t* err = (uint32_t*)(st + 3);
  launch_check_canonical(a_idx, na, universe, err, c->stream);
  launch_check_canonical(b_idx, nb, universe, err, c->stream);
  HcMergeArgs m{};
  m.a_idx = a_idx;
  m.a_val = a_val;
  m.a_cnt = st;
  m.a_cap = na;
  m.b_idx = b_idx;
  m.b_val = b_val;
  m.b_cnt = st + 1;
  m.b_cap = nb;
  m.o_idx = d_idx;
  m.o_val = d_val;
  m.o_cnt = st + 2;
  m.o_cap = capacity;
  m.lb_status = lb;
  m.ctl = ctl;
  m.err = err + 1;  // merge bits apart from the input check's
  m.splits = splits;
  launch_hc_merge(m, tiles, c->stream);
  uint64_t h[4];
  CK(cudaMemcpyAsync(h, st, 32, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const uint32_t in_bits = uint32_t(h[3]), merge_bits = uint32_t(h[3] >> 32);
  if (in_bits || (merge_bits & kErrOutside))
    return fail(ZEN_E_INVALID, "tensor indices not sorted/unique or >= M");
  *count = h[2];
  if (h[2] > capacity) return fail(ZEN_E_CAPACITY, "output capacity");
  return ZEN_OK;
}

// Non-zero blocks of `block_size` positions counted from `origin` in a sorted
// tensor: the block framing of run_omnireduce_like (zen/schemes.hpp:227-244).
extern "C" zen_status zen_count_blocks(zen_ctx* c, const uint64_t* d_idx, uint64_t count,
                                       uint64_t origin, uint64_t block_size, uint64_t* blocks) {
  if (!c || !blocks || (count && !d_idx)) return fail(ZEN_E_INVALID, "null argument");
  if (block_size == 0) return fail(ZEN_E_INVALID, "block size must be at least 1");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({8}), &sc));
  unsigned long long* d = sc.get<unsigned long long>(1);
  CK(cudaMemsetAsync(d, 0, 8, c->stream));
  launch_count_blocks(d_idx, count, origin, block_size, d, c->stream);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *blocks = h;
  return ZEN_OK;
}

// Drops the entries whose value is exactly zero (+0.0 or -0.0), keeping order:
// the block decoding of run_omnireduce_like (zen/schemes.hpp:289-295).
extern "C" zen_status zen_compact_nonzero(zen_ctx* c, const uint64_t* d_idx, const float* d_val,
                                          uint64_t count, uint64_t* d_out_idx, float* d_out_val,
                                          uint64_t* out_count) {
  if (!c || !out_count || (count && (!d_idx || !d_val || !d_out_idx || !d_out_val)))
    return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const size_t tb = wire_select_bytes(count);
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({8, count, tb}), &sc));
  uint64_t* d = sc.get<uint64_t>(1);
  uint8_t* flag = sc.get<uint8_t>(count);
  void* tmp = sc.get<uint8_t>(tb);
  CK(cudaMemsetAsync(d, 0, 8, c->stream));
  launch_compact_nonzero(d_idx, d_val, count, flag, d_out_idx, d_out_val, d, tmp, tb, c->stream);
  CK(cudaMemcpyAsync(out_count, d, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ZEN_OK;
}

// zen::skewness_ratio's per-range counts (zen/tensor.hpp:193-213): entries of
// the sorted tensor in each of `partitions` contiguous ranges of ceil(M/n).
extern "C" zen_status zen_range_counts(zen_ctx* c, const uint64_t* d_idx, uint64_t count,
                                       uint64_t universe, uint32_t partitions,
                                       uint64_t* h_counts) {
  if (!c || !h_counts || (count && !d_idx)) return fail(ZEN_E_INVALID, "null argument");
  if (!partitions || !universe) return fail(ZEN_E_INVALID, "partitions and universe must be >= 1");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({8ull * (partitions + 1)}), &sc));
  uint64_t* bnd = sc.get<uint64_t>(partitions + 1);
  launch_range_bounds(d_idx, count, universe, partitions, bnd, c->stream);
  std::vector<uint64_t> h(partitions + 1);
  CK(cudaMemcpyAsync(h.data(), bnd, 8ull * (partitions + 1), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (uint32_t p = 0; p < partitions; ++p) h_counts[p] = h[p + 1] - h[p];
  return ZEN_OK;
}

// ----------------------------------------------------------------- apply ----

namespace {
// Split `draws` between the hot tier [0, hot) and the cold tier [hot, m): the
// reference flips hot_mass for every accepted draw (a binomial count) and
// spills into the other tier once one is full (workload.hpp:79-100).
void gen_split(uint64_t draws, double hot_mass, uint64_t hot_free, uint64_t cold_free,
               uint64_t stream, uint64_t* hot_n, uint64_t* cold_n) {
  std::mt19937_64 rng(stream);
  uint64_t h = draws;
  if (hot_mass < 1.0) {
    std::binomial_distribution<uint64_t> b(draws, std::max(0.0, hot_mass));
    h = b(rng);
  }
  h = std::min(h, hot_free);
  uint64_t c = draws - h;
  if (c > cold_free) {
    c = cold_free;
    h = draws - c;
  }
  *hot_n = h;
  *cold_n = c;
}
}  // namespace

extern "C" zen_status zen_generate(zen_ctx* c, const zen_workload_spec* sp, uint32_t node,
                                   uint64_t* d_idx, float* d_val, uint64_t capacity,
                                   uint64_t* count) {
  if (!c || !sp || !count) return fail(ZEN_E_INVALID, "null argument");
  // WorkloadSpec::validate (workload.hpp:34-50)
  const double m_d = double(sp->universe);
  if (sp->universe < 1) return fail(ZEN_E_INFEASIBLE, "universe must be at least 1");
  if (sp->nodes < 1) return fail(ZEN_E_INFEASIBLE, "node count must be at least 1");
  if (!(sp->density > 0.0 && sp->density <= 1.0)) return fail(ZEN_E_INFEASIBLE, "density must be in (0,1]");
  if (sp->density * m_d < 1.0) return fail(ZEN_E_INFEASIBLE, "density*universe must be at least 1");
  if (sp->omega < 0.0 || sp->omega > 1.0) return fail(ZEN_E_INFEASIBLE, "omega must be in [0,1]");
  if (!(sp->hot_fraction > 0.0 && sp->hot_fraction <= 1.0))
    return fail(ZEN_E_INFEASIBLE, "hot_fraction must be in (0,1]");
  if (sp->hot_mass < 0.0 || sp->hot_mass > 1.0) return fail(ZEN_E_INFEASIBLE, "hot_mass must be in [0,1]");
  if (sp->density * m_d * (1.0 + double(sp->nodes) * (1.0 - sp->omega)) > m_d)
    return fail(ZEN_E_INFEASIBLE, "cannot fit disjoint remainders: d*M*(1+n*(1-omega)) > M");
  if (node >= sp->nodes) return fail(ZEN_E_INVALID, "node out of range");
  if (sp->universe >= (1ull << 40)) return fail(ZEN_E_INVALID, "universe above 2^40");
  const uint64_t m = sp->universe;
  const uint64_t nnz = uint64_t(std::ceil(sp->density * m_d));
  const uint64_t core_n = std::min<uint64_t>(nnz, uint64_t(std::ceil(sp->omega * sp->density * m_d)));
  const uint64_t hot = std::min<uint64_t>(m, std::max<uint64_t>(1, uint64_t(std::llround(sp->hot_fraction * m_d))));
  const double hot_mass = (m - hot) == 0 ? 1.0 : sp->hot_mass;
  *count = nnz;
  if (nnz > 0xFFFFFFFFull) return fail(ZEN_E_INVALID, "more than 2^32 - 1 indices per node");
  if (capacity < nnz) return fail(ZEN_E_CAPACITY, "output capacity below ceil(density * universe)");
  if (!d_idx || !d_val) return fail(ZEN_E_INVALID, "null output");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const uint64_t nw = (m + 63) / 64;
  const uint64_t nblk = (nw + 1023) / 1024;
  const uint64_t npos_max = nnz + core_n;
  const uint64_t nblk_draw = (npos_max + 1023) / 1024 + 1;
  Bump sc;
  CKR(ctx_scratch(c, bump_bytes({8 * nw, 8 * nw, 4 * std::max(nblk, nblk_draw), 8}), &sc));
  unsigned long long* core = sc.get<unsigned long long>(nw);
  unsigned long long* bits = sc.get<unsigned long long>(nw);
  uint32_t* blk = sc.get<uint32_t>(std::max(nblk, nblk_draw));
  uint64_t* total = sc.get<uint64_t>(1);
  CK(cudaMemsetAsync(core, 0, 8 * nw, c->stream));
  CK(cudaMemsetAsync(bits, 0, 8 * nw, c->stream));
  const uint64_t cold = m - hot;
  // the shared core: the same draw on every node (workload.hpp:130-139)
  const uint64_t cs = h_derive(sp->seed, 0xc07e);
  uint64_t core_h, core_c;
  gen_split(core_n, hot_mass, hot, cold, cs, &core_h, &core_c);
  launch_gen_tier(0, hot, cs ^ 1, nullptr, 0, core_h, core, blk, c->stream);
  launch_gen_tier(hot, cold, cs ^ 2, nullptr, 0, core_c, core, blk, c->stream);
  // this node's remainder, avoiding the core (workload.hpp:141-151)
  const uint64_t ns = h_derive(sp->seed, 0x10000 + node);
  uint64_t node_h, node_c;
  gen_split(nnz - core_n, hot_mass, hot - core_h, cold - core_c, ns, &node_h, &node_c);
  if (node_h + node_c != nnz - core_n) return fail(ZEN_E_INFEASIBLE, "index universe exhausted");
  launch_gen_tier(0, hot, ns ^ 1, core, core_h, node_h, bits, blk, c->stream);
  launch_gen_tier(hot, cold, ns ^ 2, core, core_c, node_c, bits, blk, c->stream);
  launch_gen_collect(bits, core, nw, blk, total, h_derive(sp->seed, 0x20000 + node), d_idx, d_val,
                     capacity, c->stream);
  uint64_t got = 0;
  CK(cudaMemcpyAsync(&got, total, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (got != nnz) return fail(ZEN_E_CUDA, "generator count mismatch");
  return ZEN_OK;
}

extern "C" zen_status zen_axpy_sparse(zen_ctx* c, float* d_dense, uint64_t m,
                                      const uint64_t* d_idx, const float* d_val, uint64_t count,
                                      float alpha) {
  if (!c) return fail(ZEN_E_INVALID, "null ctx");
  if (count && (!d_dense || !d_idx || !d_val)) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  Bump sc;
  CKR(ctx_scratch(c, 256, &sc));
  uint32_t* st = sc.get<uint32_t>(1);
  CK(cudaMemsetAsync(st, 0, 4, c->stream));
  // validate first (ascending, unique, < M: the SparseTensor invariant), so an
  // invalid tensor leaves the parameters untouched and no update is lost to a
  // duplicate index
  CKR(wire_check_input(c, d_idx, count, m, st));
  launch_axpy_sparse(d_dense, m, d_idx, d_val, count, alpha, st, c->stream);
  uint32_t h = 0;
  CK(cudaMemcpyAsync(&h, st, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (h) return fail(ZEN_E_INVALID, "sparse tensor index outside [0, M)");
  return ZEN_OK;
}

// ----------------------------------------------------------------- top-k ----
// zen::sparsify_topk (zen/workload.hpp:157-178), k_topk.cu

extern "C" zen_status zen_sparsify_topk(zen_ctx* c, const float* d_dense, uint64_t m,
                                        double fraction, uint64_t* d_idx, float* d_val,
                                        uint64_t capacity, uint64_t* count) {
  if (!c || !count) return fail(ZEN_E_INVALID, "null argument");
  if (!(fraction > 0.0 && fraction <= 1.0)) return fail(ZEN_E_INVALID, "top-k fraction must be in (0,1]");
  if (m == 0) return fail(ZEN_E_INVALID, "dense tensor must have at least one element");
  if (m >= 0xFFFFFFFFull) return fail(ZEN_E_INVALID, "top-k universe must be below 2^32");
  if (!d_dense) return fail(ZEN_E_INVALID, "null dense tensor");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  const uint64_t keep = std::min<uint64_t>(m, (uint64_t)std::ceil(fraction * double(m)));
  const uint32_t ntiles = uint32_t((m + kExtractTile - 1) / kExtractTile);
  if (!c->topk || c->topk->m < m) {
    c->topk.reset(new TopkWs);
    TopkWs& w = *c->topk;
    w.m = m;
    CKR(w.mem.alloc((uint8_t**)&w.state, topk_state_bytes()));
    CKR(w.mem.alloc(&w.hist, 2048));
    CKR(w.mem.alloc(&w.ex.st_idx, uint64_t(ntiles) * kExtractTile, false));
    CKR(w.mem.alloc(&w.ex.st_val, uint64_t(ntiles) * kExtractTile, false));
    CKR(w.mem.alloc(&w.ex.tile_cnt, ntiles));
    CKR(w.mem.alloc(&w.tile_ties, 2ull * ntiles));  // ties, then entries above T
    CKR(w.mem.alloc(&w.tie_base, ntiles));
    CKR(w.mem.alloc(&w.out_base, ntiles));
    CKR(w.mem.alloc(&w.out_count, 1));
  }
  TopkWs& w = *c->topk;
  cudaStream_t st = c->stream;
  launch_topk_select(d_dense, m, keep, w.state, w.hist, st);
  launch_select_tiles(d_dense, m, w.ex,
                      reinterpret_cast<const uint32_t*>(static_cast<char*>(w.state) +
                                                        topk_threshold_offset()),
                      st);
  launch_topk_finish(w.ex, ntiles, w.state, w.hist, w.tile_ties, w.tie_base, w.out_base, w.out_count,
                     d_idx, d_val, capacity, st);
  CK(cudaGetLastError());
  uint64_t n = 0;
  CK(cudaMemcpyAsync(&n, w.out_count, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *count = n;
  if (n > capacity) return fail(ZEN_E_CAPACITY, "output capacity below the kept entries");
  return ZEN_OK;
}

// --------------------------------------------------------------------- BP ----

namespace {

// Byte layout of one node's receive arena (identical on every rank, so peers
// can compute each other's sub-pointers from the base alone).
struct ArenaLayout {
  size_t inbox_idx = 0, inbox_val = 0, push_hdr = 0, pull_hdr = 0, inbox_gbase = 0;
  std::vector<size_t> pull_bits, pull_vals, pull_cbase;
  size_t bytes = 0;
};

ArenaLayout make_layout(uint32_t n, uint64_t cap, const std::vector<uint64_t>& nw,
                        const std::vector<uint64_t>& valcap, bool with_pull,
                        uint64_t nchunks, uint64_t ngroups) {
  ArenaLayout L;
  size_t off = 0;
  L.inbox_gbase = off;  // [n workers][ngroups] entries before each 8-tile group
  off += align256(size_t(n) * ngroups * 4);
  L.inbox_idx = off;
  off += align256(size_t(n) * cap * 4);
  L.inbox_val = off;
  off += align256(size_t(n) * cap * 4);
  L.push_hdr = off;
  off += align256(n * sizeof(PushHdr));
  L.pull_hdr = off;
  off += align256(n * sizeof(PullHdr));
  L.pull_bits.assign(n, 0);
  L.pull_vals.assign(n, 0);
  L.pull_cbase.assign(n, 0);
  if (with_pull) {
    for (uint32_t s = 0; s < n; ++s) {  // per-chunk value bases (k_agg_values -> k_decode)
      L.pull_cbase[s] = off;
      off += align256((nchunks + 1) * 4);
    }
    for (uint32_t s = 0; s < n; ++s) {
      L.pull_bits[s] = off;
      off += align256(std::max<uint64_t>(nw[s], 1) * 8);
    }
    for (uint32_t s = 0; s < n; ++s) {
      L.pull_vals[s] = off;
      off += align256(std::max<uint64_t>(valcap[s], 1) * 4);
    }
  }
  L.bytes = off;
  return L;
}

struct Arena {
  char* base = nullptr;
  bool owned = false;
  uint32_t* inbox_idx(const ArenaLayout& L) const { return (uint32_t*)(base + L.inbox_idx); }
  uint32_t* inbox_gbase(const ArenaLayout& L) const { return (uint32_t*)(base + L.inbox_gbase); }
  float* inbox_val(const ArenaLayout& L) const { return (float*)(base + L.inbox_val); }
  PushHdr* push_hdr(const ArenaLayout& L) const { return (PushHdr*)(base + L.push_hdr); }
  PullHdr* pull_hdr(const ArenaLayout& L) const { return (PullHdr*)(base + L.pull_hdr); }
  unsigned long long* bits(const ArenaLayout& L, uint32_t s) const {
    return (unsigned long long*)(base + L.pull_bits[s]);
  }
  float* vals(const ArenaLayout& L, uint32_t s) const { return (float*)(base + L.pull_vals[s]); }
  uint32_t* cbase(const ArenaLayout& L, uint32_t s) const {
    return (uint32_t*)(base + L.pull_cbase[s]);
  }
};

struct Worker {
  uint32_t id = 0;
  uint32_t* keys = nullptr;
  float* vals = nullptr;
  HashArgs<uint32_t> a{};
  ExtractWs<uint32_t> ex{};
  uint64_t h_count = 0;  // staging for sparse inputs (stable address)
};

struct Server {
  uint32_t id = 0;
  AggArgs a{};
  uint64_t* agg_count = nullptr;
  bool fused = false;  // dense syncs take k_agg_fused (local mode)
};

constexpr int kRing = 1024;

}  // namespace

struct zen_bp {
  zen_ctx* ctx = nullptr;
  uint32_t n = 0, rank = 0;
  bool local = true;
  uint64_t m = 0, cap = 0, stride_cap = 0;
  uint32_t ngroups = 0;  // 8-tile groups of the dense path (fused aggregate blocks)
  zen_hash_params params{};
  std::unique_ptr<zen_universe> uni;
  DevMem mem;
  std::vector<Worker> workers;
  std::vector<Server> servers;
  ArenaLayout L, L0;  // L: with pull (rank / arena 0), L0: inbox only (local arenas 1..n-1)
  std::vector<Arena> arenas;  // local: n; rank: n (own + mapped peers)
  bool connected = false;
  Decoder dec;
  DecodeArgs da{};
  uint64_t* out_idx = nullptr;
  float* out_val = nullptr;
  uint64_t* out_count = nullptr;
  uint64_t out_cap = 0;
  std::vector<uint64_t> nw, valcap;
  // host view after zen_bp_wait
  bool collected = false;
  uint64_t h_result = 0;
  std::vector<uint64_t> h_counts, h_nnz, h_agg;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // kRing * (ZEN_STAGES + 1)
  uint64_t ev_head = 0, ev_tail = 0;
  double stage_ms[ZEN_STAGES] = {0, 0, 0, 0};
  uint64_t timed = 0;
  uint32_t kernels_per_sync = 0;
  // e2e staging
  std::vector<float*> dense_dev;
  uint32_t* chk = nullptr;  // status word of the sparse-input validation
  // hash-memory side path stream + fork/join events
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // CUDA graph of the dense sync
  bool use_graph = true;
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t gdef = nullptr;
  std::vector<const void*> gkey;
  std::vector<cudaEvent_t> gev;
  std::vector<cudaGraphNode_t> gev_nodes;
  uint32_t graph_kernels = 0;

  Arena& arena_of(uint32_t r) { return arenas[r]; }
  const ArenaLayout& layout_of(uint32_t r) const { return (local && r != 0) ? L0 : L; }
};

namespace {

zen_status bp_alloc_worker(zen_bp* bp, Worker& w) {
  const uint32_t n = bp->n, k = bp->params.rehash_depth;
  const uint64_t cap = bp->cap;
  const uint64_t ntiles = (cap + kHashTile - 1) / kHashTile;
  DevMem& mem = bp->mem;
  CKR(mem.alloc(&w.keys, cap));
  CKR(mem.alloc(&w.vals, cap));
  HashArgs<uint32_t>& a = w.a;
  a.idx = w.keys;
  a.val = w.vals;
  CKR(mem.alloc(&a.hdr, 1));
  // u32 slot words (vacant = ~0), kept vacant between syncs by the depth pass
  CKR(mem.alloc(&a.slots, size_t(n) * bp->stride_cap, false));
  CK(cudaMemsetAsync(a.slots, 0xFF, size_t(n) * bp->stride_cap * sizeof(*a.slots), t_setup));
  a.slot_vals = nullptr;
  CKR(mem.alloc(&a.meta, cap));
  CKR(mem.alloc(&a.pmeta, cap));
  CKR(mem.alloc(&a.tile_cnt, ntiles * n));
  CKR(mem.alloc(&a.tile_scnt, ntiles * n));
  CKR(mem.alloc(&a.load, n));
  CKR(mem.alloc(&a.sload, n));
  CKR(mem.alloc(&a.part_off, n));
  CKR(mem.alloc(&a.fallback, n));
  CKR(mem.alloc(&a.stats, n * (ZEN_MAX_K + 1)));
  CKR(mem.alloc(&a.fb_stats, n * (ZEN_MAX_K + 1)));
  CKR(mem.alloc(&a.stats_out, ZEN_MAX_K + 1));
  a.dst_table = 1;
  a.cap = cap;
  a.tiles_cap = ntiles;
  a.dst_cap = cap;
  a.stride_cap = bp->stride_cap;
  a.me = w.id;
  a.peer = bp->local ? 0 : 1;
  uint32_t** dst_idx;
  float** dst_val;
  PushHdr** push_hdr;
  CKR(mem.alloc(&dst_idx, n));
  CKR(mem.alloc(&dst_val, n));
  CKR(mem.alloc(&push_hdr, n));
  a.dst_idx = dst_idx;
  a.dst_val = dst_val;
  a.push_hdr = push_hdr;
  uint32_t** dst_gbase;
  CKR(mem.alloc(&dst_gbase, n));
  a.dst_gbase = dst_gbase;
  HashHdr h{};
  h.derive = 1;
  h.r1_mult = bp->params.r1_multiplier;
  h.r2_ratio = bp->params.r2_ratio;
  h.bad_index = ~0ull;
  CKR(upload(a.hdr, &h, 1));
  const uint64_t ext_tiles = (bp->m + kExtractTile - 1) / kExtractTile;
  CKR(mem.alloc(&w.ex.st_idx, ext_tiles * kExtractTile, false));
  CKR(mem.alloc(&w.ex.st_val, ext_tiles * kExtractTile, false));
  CKR(mem.alloc(&w.ex.tile_cnt, ext_tiles));
  CKR(mem.alloc(&w.ex.tile_base, ext_tiles));
  w.ex.nblk = (std::min<uint64_t>(bp->cap, bp->m) + 255) / 256;
  CKR(mem.alloc(&w.ex.blk_tile, w.ex.nblk + 1));
  // dense data path: per-(partition, tile) counts + chunk / super-chunk sums
  PushCounts& x = a.xc;
  x.ntiles = (uint32_t)ext_tiles;
  x.nchunk = (uint32_t)((ext_tiles + 31) / 32);
  x.nsup = (uint32_t)((ext_tiles + 1023) / 1024);
  x.n = n;
  CKR(mem.alloc(&x.tcnt, size_t(n) * x.ntiles));
  CKR(mem.alloc(&x.ccnt, size_t(n) * (x.nchunk + x.nsup)));
  x.scnt = x.ccnt + size_t(n) * x.nchunk;
  x.st_idx = w.ex.st_idx;
  // peer destinations: regroup each round into per-part runs (full-line NVLink
  // stores; measured N=4 0.177 vs 0.188 ms, N=2 equal) unless ZEN_PUSH_REORDER=0.
  // The push is published by a one-block kernel after the scatter; the
  // alternative, the scatter's last block (ZEN_PUSH_SIGNAL_FUSED=1), measured
  // slower (N=2 0.146 vs 0.139 ms, N=4 0.181 vs 0.177 ms: every block's
  // system-scope fence + counter, then one late block, costs more than a
  // programmatic launch)
  const char* ro = std::getenv("ZEN_PUSH_REORDER");
  x.reorder = (!bp->local && !(ro && ro[0] == '0')) ? 1u : 0u;
  const char* sf = std::getenv("ZEN_PUSH_SIGNAL_FUSED");
  x.fused_signal = (sf && sf[0] == '1') ? 1u : 0u;
  x.scatter_grid = push_scatter_grid<uint32_t>(x.reorder != 0, x.ntiles);
  zen_hash_family f;
  CKR(zen_hash_family_make_worker(bp->params.seed, w.id, n, k, &f));
  a.fam = fold(f);
  a.fam.db = std::getenv("ZEN_SLOT_REHASH") ? 0u : slot_probe_bits(k, bp->m);  // (env: A/B only)
  x.pc = a.fam.pc;
  return ZEN_OK;
}

// rank mode: the peers' arrival is awaited by a one-warp kernel before the
// consumer.  Gating it inside the consumer instead (one polling block releases
// a local word, ZEN_WAIT_GATE=1) measured slower: N=2 0.149 vs 0.141 ms, N=4
// 0.185 vs 0.180 ms (every block of the consumer holds an SM slot while it
// waits, where the one-warp kernel lets the consumer's blocks launch at once)
bool gate_waits() {
  const char* e = std::getenv("ZEN_WAIT_GATE");
  return e && e[0] == '1';
}

zen_status bp_alloc_server(zen_bp* bp, Server& s) {
  const uint32_t n = bp->n;
  DevMem& mem = bp->mem;
  CKR(bp->uni->ensure_own(s.id));
  CKR(mem.alloc(&s.agg_count, 1));
  AggArgs& a = s.a;
  a.n = n;
  a.s = s.id;
  a.m = bp->m;
  const uint32_t** in_idx;
  const float** in_val;
  const PushHdr** in_hdr;
  CKR(mem.alloc(&in_idx, n));
  CKR(mem.alloc(&in_val, n));
  CKR(mem.alloc(&in_hdr, n));
  a.in_idx = in_idx;
  a.in_val = in_val;
  a.in_hdr = in_hdr;
  const uint32_t** in_load;
  CKR(mem.alloc(&in_load, n));
  a.in_load = in_load;
  a.in_count = nullptr;
  a.own = bp->uni->own[s.id];
  a.whole = n == 1 ? 1 : 0;
  a.bs = bp->uni->bs[s.id];
  CKR(alloc_agg_ws(mem, a, n, a.bs));
  a.ndst = bp->local ? 1 : n;
  unsigned long long** db;
  float** dv;
  PullHdr** dh;
  CKR(mem.alloc(&db, a.ndst));
  CKR(mem.alloc(&dv, a.ndst));
  CKR(mem.alloc(&dh, a.ndst));
  uint32_t** dc;
  CKR(mem.alloc(&dc, a.ndst));
  a.dst_bits = db;
  a.dst_vals = dv;
  a.dst_cbase = dc;
  a.cprefix = bp->uni->cprefix;
  a.nchunks = bp->uni->nchunks;
  a.dst_hdr = bp->local ? nullptr : dh;
  a.val_cap = bp->valcap[s.id];
  a.agg_count = s.agg_count;
  a.wait_push = bp->local ? 0 : 1;
  a.peer = bp->local ? 0 : 1;
  a.gate = gate_waits() ? 1 : 0;
  return ZEN_OK;
}

// fused aggregate: the static group table of every server and its
// shared-memory span (the group entry bases are wired with the arenas)
zen_status bp_setup_fused(zen_bp* bp) {
  uint32_t* d_span;
  CKR(bp->mem.alloc(&d_span, 1));
  const uint32_t ntiles = bp->workers[0].a.xc.ntiles;
  for (auto& s : bp->servers) {
    AggArgs& a = s.a;
    a.ntiles = ntiles;
    a.ngroups = bp->ngroups;
    uint4* gtab;
    CKR(bp->mem.alloc(&gtab, size_t(a.ngroups) + 1));
    a.gtab = gtab;
    CKR(bp->mem.alloc(&a.lbf, a.ngroups));  // zeroed: no iteration tag matches
    const uint32_t** ig;
    CKR(bp->mem.alloc(&ig, bp->n));
    a.in_gbase = ig;
    CK(cudaMemsetAsync(d_span, 0, sizeof(uint32_t), bp->ctx->stream));
    launch_agg_groups(a, d_span, bp->ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(bp->ctx->stream));
    CK(cudaMemcpy(&a.span, d_span, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    a.span = std::max(a.span, 1u);
    s.fused = agg_fused_smem(bp->n, a.span) <= 227 * 1024;  // (always at n <= 16)
  }
  return ZEN_OK;
}

// fill the device pointer tables once all arenas are known
zen_status bp_wire(zen_bp* bp) {
  const uint32_t n = bp->n;
  for (auto& w : bp->workers) {
    std::vector<uint32_t*> di(n);
    std::vector<float*> dv(n);
    std::vector<PushHdr*> ph(n);
    for (uint32_t p = 0; p < n; ++p) {
      const Arena& A = bp->arena_of(p);
      const ArenaLayout& L = bp->layout_of(p);
      di[p] = A.inbox_idx(L) + size_t(w.id) * bp->cap;
      dv[p] = A.inbox_val(L) + size_t(w.id) * bp->cap;
      ph[p] = A.push_hdr(L) + w.id;
    }
    CKR(upload(const_cast<uint32_t**>(w.a.dst_idx), di.data(), n));
    CKR(upload(const_cast<float**>(w.a.dst_val), dv.data(), n));
    CKR(upload(const_cast<PushHdr**>(w.a.push_hdr), ph.data(), n));
    std::vector<uint32_t*> dg(n);
    for (uint32_t p = 0; p < n; ++p)
      dg[p] = bp->arena_of(p).inbox_gbase(bp->layout_of(p)) + size_t(w.id) * bp->ngroups;
    CKR(upload(const_cast<uint32_t**>(w.a.dst_gbase), dg.data(), n));
    // local mode: the servers read the workers' counters directly, so there
    // is no push header / signal kernel
    if (bp->local) w.a.push_hdr = nullptr;
  }
  std::vector<const uint32_t*> loads;
  for (auto& w : bp->workers) loads.push_back(w.a.load);
  for (auto& s : bp->servers) {
    const Arena& A = bp->arena_of(s.id);
    const ArenaLayout& L = bp->layout_of(s.id);
    std::vector<const uint32_t*> ii(n);
    std::vector<const float*> iv(n);
    std::vector<const PushHdr*> ih(n);
    for (uint32_t w = 0; w < n; ++w) {
      ii[w] = A.inbox_idx(L) + size_t(w) * bp->cap;
      iv[w] = A.inbox_val(L) + size_t(w) * bp->cap;
      ih[w] = A.push_hdr(L) + w;
    }
    CKR(upload(const_cast<const uint32_t**>(s.a.in_idx), ii.data(), n));
    CKR(upload(const_cast<const float**>(s.a.in_val), iv.data(), n));
    CKR(upload(const_cast<const PushHdr**>(s.a.in_hdr), ih.data(), n));
    // one local worker: the union builds U from its entries (dense syncs)
    const char* ue = std::getenv("ZEN_UNION_ENTRIES");  // (=0: mark + union, A/B)
    if (bp->local && n == 1 && !(ue && ue[0] == '0')) {
      s.a.solo_gbase = A.inbox_gbase(L);
      s.a.ngroups = bp->ngroups;
    }
    if (s.a.in_gbase) {
      std::vector<const uint32_t*> ig(n);
      for (uint32_t w = 0; w < n; ++w) ig[w] = A.inbox_gbase(L) + size_t(w) * bp->ngroups;
      CKR(upload(const_cast<const uint32_t**>(s.a.in_gbase), ig.data(), n));
    }
    if (bp->local) {
      CKR(upload(const_cast<const uint32_t**>(s.a.in_load), loads.data(), n));
      s.a.in_hdr = nullptr;
    }
    std::vector<unsigned long long*> db(s.a.ndst);
    std::vector<float*> dvv(s.a.ndst);
    std::vector<PullHdr*> dh(s.a.ndst);
    std::vector<uint32_t*> dcb(s.a.ndst);
    for (uint32_t d = 0; d < s.a.ndst; ++d) {
      const uint32_t r = bp->local ? 0 : d;  // local: one shared pull inbox (arena 0)
      const Arena& R = bp->arena_of(r);
      db[d] = R.bits(bp->L, s.id);
      dvv[d] = R.vals(bp->L, s.id);
      dh[d] = R.pull_hdr(bp->L) + s.id;
      dcb[d] = R.cbase(bp->L, s.id);
    }
    // this server's own (local) copy of U, read back for the chunk bases
    s.a.own_bits = db[bp->local ? 0 : s.id];
    CKR(upload(const_cast<unsigned long long**>(s.a.dst_bits), db.data(), s.a.ndst));
    CKR(upload(const_cast<float**>(s.a.dst_vals), dvv.data(), s.a.ndst));
    CKR(upload(const_cast<uint32_t**>(s.a.dst_cbase), dcb.data(), s.a.ndst));
    if (s.a.dst_hdr) CKR(upload(const_cast<PullHdr**>(s.a.dst_hdr), dh.data(), s.a.ndst));
  }
  // receiver: this node's pull inbox (local: arena 0)
  const Arena& R = bp->arena_of(bp->local ? 0 : bp->rank);
  std::vector<const unsigned long long*> hb(n);
  std::vector<const float*> hv(n);
  std::vector<const PullHdr*> hh(n);
  std::vector<const uint32_t*> hc(n);
  for (uint32_t s = 0; s < n; ++s) {
    hb[s] = R.bits(bp->L, s);
    hv[s] = R.vals(bp->L, s);
    hh[s] = R.pull_hdr(bp->L) + s;
    hc[s] = R.cbase(bp->L, s);
  }
  CKR(upload(const_cast<const uint32_t**>(bp->da.cbase), hc.data(), n));
  CKR(upload(const_cast<const unsigned long long**>(bp->da.bits), hb.data(), n));
  CKR(upload(const_cast<const float**>(bp->da.vals), hv.data(), n));
  CKR(upload(const_cast<const PullHdr**>(bp->da.pull_hdr), hh.data(), n));
  bp->connected = true;
  return ZEN_OK;
}

uint64_t stride_cap_for(const zen_hash_params& p, uint64_t cap, uint32_t n) {
  uint64_t r1 = (uint64_t)std::ceil(p.r1_multiplier * double(cap) / double(n));
  r1 = std::max<uint64_t>(r1, 1);
  uint64_t r2 = (uint64_t)std::ceil(p.r2_ratio * double(r1));
  r2 = std::max<uint64_t>(r2, 1);
  return r1 + r2;
}

}  // namespace

extern "C" {

zen_status zen_bp_create(zen_ctx* c, uint32_t n, uint32_t rank, uint64_t universe,
                         uint64_t max_nnz, const zen_hash_params* params, zen_bp** out) {
  if (!c || !params || !out) return fail(ZEN_E_INVALID, "null argument");
  if (n == 0 || n > ZEN_MAX_WORKERS) return fail(ZEN_E_INVALID, "worker count must be 1..16");
  if (rank != ZEN_BP_LOCAL && rank >= n) return fail(ZEN_E_INVALID, "rank out of range");
  if (universe == 0 || universe >= 0xFFFFFFFFull)
    return fail(ZEN_E_INVALID, "universe must be in [1, 2^32-1)");
  if (params->rehash_depth == 0 || params->rehash_depth > ZEN_MAX_K)
    return fail(ZEN_E_INVALID, "rehash depth out of range");
  if (!(params->r1_multiplier > 0) || !(params->r2_ratio > 0))
    return fail(ZEN_E_INVALID, "r1_multiplier and r2_ratio must be positive");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  auto bp = std::make_unique<zen_bp>();
  bp->ctx = c;
  bp->n = n;
  bp->local = rank == ZEN_BP_LOCAL;
  bp->rank = bp->local ? 0 : rank;
  bp->m = universe;
  bp->cap = std::max<uint64_t>(std::min<uint64_t>(max_nnz, universe), 1);
  bp->params = *params;
  bp->stride_cap = stride_cap_for(*params, bp->cap, n);
  // universe tables for (M, n, derive_seed(seed, 0)) -- bp_universe_table, zen/schemes.hpp:332-335
  bp->uni = std::make_unique<zen_universe>();
  bp->uni->ctx = c;
  bp->uni->m = universe;
  bp->uni->n = n;
  bp->uni->pseed = h_derive(params->seed, 0);
  CKR(bp->uni->build());
  bp->nw.resize(n);
  bp->valcap.resize(n);
  for (uint32_t s = 0; s < n; ++s) {
    bp->nw[s] = (bp->uni->bs[s] + 63) / 64;
    bp->valcap[s] = std::min<uint64_t>(bp->uni->bs[s], uint64_t(n) * bp->cap);
  }
  bp->ngroups = uint32_t(((bp->m + kExtractTile - 1) / kExtractTile + 7) / 8);
  bp->L = make_layout(n, bp->cap, bp->nw, bp->valcap, true, bp->uni->nchunks, bp->ngroups);
  bp->L0 = make_layout(n, bp->cap, bp->nw, bp->valcap, false, bp->uni->nchunks, bp->ngroups);
  CK(cudaStreamCreateWithFlags(&bp->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&bp->fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&bp->join, cudaEventDisableTiming));
  const uint32_t nlocal = bp->local ? n : 1;
  for (uint32_t i = 0; i < nlocal; ++i) {
    Worker w;
    w.id = bp->local ? i : bp->rank;
    bp->workers.push_back(w);
    Server s;
    s.id = w.id;
    bp->servers.push_back(s);
  }
  for (auto& w : bp->workers) CKR(bp_alloc_worker(bp.get(), w));
  for (auto& s : bp->servers) CKR(bp_alloc_server(bp.get(), s));
  if (bp->local) {  // every server on this GPU: the push scatter marks for k_agg_mark
    std::vector<const OwnWord*> own(n);
    std::vector<unsigned long long*> pw(n);
    std::vector<uint32_t*> pre(n);
    std::vector<uint64_t> nws(n);
    for (auto& s : bp->servers) {
      own[s.id] = s.a.own;
      pw[s.id] = s.a.pw;
      pre[s.id] = s.a.pre;
      nws[s.id] = s.a.nws;
    }
    const OwnWord** d_own;
    unsigned long long** d_pw;
    uint32_t** d_pre;
    uint64_t* d_nws;
    CKR(bp->mem.alloc(&d_own, n));
    CKR(bp->mem.alloc(&d_pw, n));
    CKR(bp->mem.alloc(&d_pre, n));
    CKR(bp->mem.alloc(&d_nws, n));
    CKR(upload(d_own, own.data(), n));
    CKR(upload(d_pw, pw.data(), n));
    CKR(upload(d_pre, pre.data(), n));
    CKR(upload(d_nws, nws.data(), n));
    // opt-in (ZEN_SCATTER_MARK=1): measured slower -- N=1 0.124 vs 0.109 ms,
    // 8 emulated workers 1.55 vs 1.19 ms: the rank lookups and atomics lengthen
    // the scatter on the critical path by more than the mark kernel they save
    const char* mk = std::getenv("ZEN_SCATTER_MARK");
    for (auto& s : bp->servers) s.a.pre_min = (mk && mk[0] == '1') ? 1 : 0;
    for (auto& w : bp->workers) {
      w.a.xc.mark = (mk && mk[0] == '1') ? 1u : 0u;
      w.a.xc.mk_own = d_own;
      w.a.xc.mk_pw = d_pw;
      w.a.xc.mk_pre = d_pre;
      w.a.xc.mk_nws = d_nws;
    }
  }
  // The fused aggregate (dense syncs) replaces mark + union + values by one
  // kernel per server.  Measured (profiles/r07/fused_aggregate_ab.txt), it
  // wins from 4 workers up -- 8 emulated on one GPU: aggregate 0.342 vs 0.408
  // ms; rank mode N=4: 0.180 vs 0.184 ms -- and loses below (N=1: 0.121 vs
  // 0.109 ms, N=2: 0.152 vs 0.143 ms: each block runs its phases back to back
  // where the three kernels overlap them).  ZEN_AGG_FUSED=1 / =0 forces it.
  const char* fz = std::getenv("ZEN_AGG_FUSED");
  const bool fused = fz ? fz[0] == '1' : n >= 4;
  if (fused) CKR(bp_setup_fused(bp.get()));
  // arenas
  bp->arenas.assign(n, Arena{});
  for (uint32_t r = 0; r < n; ++r) {
    if (!bp->local && r != bp->rank) continue;
    const ArenaLayout& L = bp->layout_of(r);
    void* p = nullptr;
    CK(cudaMalloc(&p, L.bytes));
    CK(cudaMemsetAsync(p, 0, L.bytes, t_setup));
    bp->arenas[r].base = (char*)p;
    bp->arenas[r].owned = true;
  }
  // receiver
  std::vector<bool> present(n, true);
  CKR(bp->dec.init(bp->uni.get(), present));
  bp->out_cap = std::min<uint64_t>(universe, uint64_t(n) * bp->cap);
  CKR(bp->mem.alloc(&bp->out_idx, bp->out_cap));
  CKR(bp->mem.alloc(&bp->out_val, bp->out_cap));
  CKR(bp->mem.alloc(&bp->out_count, 1));
  CKR(bp->mem.alloc(&bp->chk, 1));
  DecodeArgs& da = bp->da;
  bp->dec.fill(da, bp->uni.get());
  const unsigned long long** bits_t;
  const float** vals_t;
  const PullHdr** ph_t;
  const uint32_t** cb_t;
  CKR(bp->mem.alloc(&bits_t, n));
  CKR(bp->mem.alloc(&vals_t, n));
  CKR(bp->mem.alloc(&ph_t, n));
  CKR(bp->mem.alloc(&cb_t, n));
  da.cbase = cb_t;
  da.bits = bits_t;
  da.vals = vals_t;
  da.pull_hdr = ph_t;
  da.out_idx = bp->out_idx;
  da.out_val = bp->out_val;
  da.out_count = bp->out_count;
  da.out_cap = bp->out_cap;
  da.hdr = bp->workers[0].a.hdr;
  da.wait_pull = bp->local ? 0 : 1;
  da.gate = gate_waits() ? 1 : 0;
  for (auto& s : bp->servers) {
    const Worker* w = nullptr;
    for (auto& ww : bp->workers)
      if (ww.id == s.id) w = &ww;
    s.a.hdr = w->a.hdr;
  }
  if (bp->local || n == 1) CKR(bp_wire(bp.get()));
  CK(cudaDeviceSynchronize());
  *out = bp.release();
  return ZEN_OK;
}

void zen_bp_destroy(zen_bp* bp) {
  if (!bp) return;
  DevGuard g(bp->ctx->device);
  cudaDeviceSynchronize();
  for (uint32_t r = 0; r < bp->arenas.size(); ++r) {
    if (!bp->arenas[r].base) continue;
    if (bp->arenas[r].owned)
      cudaFree(bp->arenas[r].base);
    else
      cudaIpcCloseMemHandle(bp->arenas[r].base);
  }
  for (auto e : bp->ev) cudaEventDestroy(e);
  for (auto e : bp->gev) cudaEventDestroy(e);
  if (bp->fork) cudaEventDestroy(bp->fork);
  if (bp->join) cudaEventDestroy(bp->join);
  if (bp->side) cudaStreamDestroy(bp->side);
  if (bp->gexec) cudaGraphExecDestroy(bp->gexec);
  if (bp->gdef) cudaGraphDestroy(bp->gdef);
  for (auto p : bp->dense_dev) cudaFree(p);
  delete bp;
}

zen_status zen_bp_set_params(zen_bp* bp, const zen_hash_params* p) {
  if (!bp || !p) return fail(ZEN_E_INVALID, "null argument");
  if (p->rehash_depth == 0 || p->rehash_depth > ZEN_MAX_K)
    return fail(ZEN_E_INVALID, "rehash depth out of range");
  if (p->seed != bp->params.seed) return fail(ZEN_E_INVALID, "changing the seed needs a new zen_bp");
  DevGuard g(bp->ctx->device);
  SetupStream setup_(bp->ctx->stream);
  CK(cudaStreamSynchronize(bp->ctx->stream));
  bp->params = *p;
  const uint64_t sc = stride_cap_for(*p, bp->cap, bp->n);
  for (auto& w : bp->workers) {
    if (sc > bp->stride_cap) {
      SlotOf<uint32_t>* slots;
      CKR(bp->mem.alloc(&slots, size_t(bp->n) * sc, false));
      CK(cudaMemsetAsync(slots, 0xFF, size_t(bp->n) * sc * sizeof(*slots), t_setup));
      w.a.slots = slots;
      w.a.stride_cap = sc;
    }
    CKR(upload(&w.a.hdr->r1_mult, &p->r1_multiplier, 1));
    CKR(upload(&w.a.hdr->r2_ratio, &p->r2_ratio, 1));
    zen_hash_family f;
    CKR(zen_hash_family_make_worker(p->seed, w.id, bp->n, p->rehash_depth, &f));
    w.a.fam = fold(f);
    w.a.fam.db = std::getenv("ZEN_SLOT_REHASH") ? 0u : slot_probe_bits(p->rehash_depth, bp->m);
  }
  bp->stride_cap = std::max(bp->stride_cap, sc);
  if (bp->gexec) cudaGraphExecDestroy(bp->gexec);
  if (bp->gdef) cudaGraphDestroy(bp->gdef);
  bp->gexec = nullptr;
  bp->gdef = nullptr;
  bp->gkey.clear();
  return ZEN_OK;
}

zen_status zen_bp_ipc_handle(zen_bp* bp, void* out) {
  if (!bp || !out) return fail(ZEN_E_INVALID, "null argument");
  if (bp->local) return fail(ZEN_E_INVALID, "local-mode synchroniser has no IPC handle");
  DevGuard g(bp->ctx->device);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, bp->arenas[bp->rank].base));
  std::memcpy(out, &h, sizeof(h));
  return ZEN_OK;
}

zen_status zen_bp_connect(zen_bp* bp, const void* handles) {
  if (!bp || !handles) return fail(ZEN_E_INVALID, "null argument");
  if (bp->local) return ZEN_OK;
  DevGuard g(bp->ctx->device);
  SetupStream setup_(bp->ctx->stream);
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (uint32_t r = 0; r < bp->n; ++r) {
    if (r == bp->rank || bp->arenas[r].base) continue;
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ZEN_E_PEER, std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(r) +
                                  "): " + cudaGetErrorString(e));
    }
    bp->arenas[r].base = (char*)p;
    bp->arenas[r].owned = false;
  }
  CKR(bp_wire(bp));
  CK(cudaDeviceSynchronize());
  return ZEN_OK;
}

}  // extern "C"

namespace {

// Enqueue one synchronisation.  `ev` (ZEN_STAGES + 1 events) brackets the
// stages when non-null.
zen_status bp_enqueue(zen_bp* bp, bool from_dense, const float* const* dense, cudaEvent_t* ev) {
  cudaStream_t st = bp->ctx->stream;
  if (ev) CK(cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal));
  // the side path's width follows the key capacity: at embedding-scale
  // sparsity it stays narrow (the latency-bound critical path keeps the SMs),
  // at millions of keys it needs the whole GPU not to become the tail (rank
  // mode keeps it narrower: its aggregate waits on the peers, and measured at
  // n=4 one more CTA per SM costs the critical path 10 us)
  static const char* side_env = std::getenv("ZEN_SIDE_CTAS");  // tuning override
  const unsigned side_ctas = side_env ? (unsigned)std::max(1, std::atoi(side_env))
                                      : (unsigned)std::min<uint64_t>(
                                            6, std::max<uint64_t>(2, bp->cap >> (bp->local ? 18 : 20)));
  // diagnostic only (timeline studies): no hash-memory side path at all, so
  // no CollisionStats -- never set for a result that is checked or reported
  static const bool diag_no_side = std::getenv("ZEN_DIAG_NO_SIDE") != nullptr;
  // The claims can keep the depth histogram themselves (+1 / -1 per slot
  // change, shared-memory counters) instead of the table-scan depth pass;
  // measured (profiles/r07/hist_inline_ab.txt) faster with several local
  // workers or many keys (8 emulated 1.026 -> 1.008 ms, 10 % 0.334 -> 0.331)
  // and slower at 1 % N=1 (0.0958 -> 0.102: the counters lengthen the claims,
  // which run beside the aggregate).  ZEN_HIST_INLINE=0/1 forces it.
  static const char* ih = std::getenv("ZEN_HIST_INLINE");
  const bool inline_hist =
      (ih ? ih[0] == '1' : (bp->local && (bp->n > 1 || bp->cap >= (4u << 20)))) &&
      !std::getenv("ZEN_PLACE_V1");  // (the one-phase claims keep no histogram)
  static const char* fe = std::getenv("ZEN_FORK_EARLY");
  const bool fork_early =
      fe ? fe[0] == '1'
         : (bp->cap < (4u << 20) && (bp->local ? bp->n == 1 : bp->n >= 4));
  auto fork_side = [&](Worker& w, bool dense_path) -> zen_status {
    if (diag_no_side) return ZEN_OK;
    CK(cudaEventRecord(bp->fork, st));
    CK(cudaStreamWaitEvent(bp->side, bp->fork, 0));
    // Programmatic launch inside the side chain (claims -> depth -> replay)
    // measured faster with several local workers or many keys (8 emulated
    // 1.057 -> 1.007 ms, 10 % N=1 0.361 -> 0.352) and slower otherwise (1 % N=1 0.1060 ->
    // 0.1073, rank N=2 0.138 -> 0.149, N=4 0.178 -> 0.186: the early-launched
    // blocks hold SM slots the critical path needs); profiles/r07/side_pdl_ab.txt
    static const char* spdl = std::getenv("ZEN_SIDE_PDL");  // (=0/1 forces it)
    static const char* sprio = std::getenv("ZEN_SIDE_PRIO");
    // (one worker: taken at large key capacities, where the claims run long)
    const bool side_pdl = spdl ? spdl[0] == '1' : (bp->local && (bp->n > 1 || bp->cap >= (4u << 20)));
    LaunchScope low(side_pdl, /*low_priority=*/!(sprio && sprio[0] == '0'));
    // claims (dense: straight from the extraction staging) + table-scan depth
    // pass (CollisionStats) + the data-dependent fallback replay
    HashArgs<uint32_t> sa = w.a;
    if (dense_path) {
      sa.xc.early = fork_early ? 1u : 0u;  // sizes from the extraction's counts
      sa.xc.inline_hist = inline_hist ? 1u : 0u;
      launch_place_tiles<uint32_t>(sa, bp->side, side_ctas);
    } else {
      sa.xc.st_idx = nullptr;  // the ascending key list, not the staging
    }
    launch_hash_side_bp<uint32_t>(sa, bp->side, side_ctas, /*place=*/!dense_path);
    return ZEN_OK;
  };
  if (from_dense) {
    // stage 0: per-sync reset, then the HBM-bound extraction (which also
    // computes every non-zero's h0 partition and the per-tile partition counts)
    for (auto& w : bp->workers) launch_bp_begin<uint32_t>(w.a, st);
    for (size_t i = 0; i < bp->workers.size(); ++i)
      launch_extract_tiles_part<uint32_t>(dense[i], bp->m, bp->workers[i].ex, bp->workers[i].a, st);
    if (ev) CK(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    // stage 1: the push -- one kernel from the staging into the owners'
    // inboxes; the hash-memory side path of each worker forks onto bp->side
    // and joins at the end of the sync
    // The side chain (claims + depth + replay) reads only the extraction's
    // staging and counts, so it can fork right after the extraction and run
    // beside the push; measured (profiles/r07/fork_early_ab.txt) that wins
    // when the claims are short -- N=1 1 % 0.1011 -> 0.0968 ms, rank N=4
    // 0.179 -> 0.168 ms -- and loses with many keys (10 % N=1 0.341 ->
    // 0.366: the claims take the SMs the push needs), several local workers
    // (8 emulated 1.024 -> 1.034) or two ranks (N=2 0.1395 -> 0.1416).
    // ZEN_FORK_EARLY=0/1 forces it.
    if (fork_early)
      for (auto& w : bp->workers) CKR(fork_side(w, true));
    for (auto& w : bp->workers) {
      launch_push_scatter<uint32_t>(w.a, w.ex, st);  // + the push signal (rank mode)
      if (!fork_early) CKR(fork_side(w, true));
      if (w.a.push_hdr && !w.a.xc.fused_signal) launch_push_signal<uint32_t>(w.a, st);
    }
  } else {
    if (ev) CK(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    for (auto& w : bp->workers) {
      launch_hash_begin<uint32_t>(w.a, st);
      launch_hash_part<uint32_t>(w.a, bp->n, st);  // the side path reads its partitions
      launch_hash_critical<uint32_t>(w.a, bp->n, /*part=*/false, st);
      CKR(fork_side(w, false));  // after the loads (k_part_scan) the depth pass reads
    }
  }
  if (ev) CK(cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal));
  // dense syncs in local mode: the push scatter already marked every entry
  const bool marked = from_dense && bp->local && !bp->workers.empty() &&
                      bp->workers[0].a.xc.mark;
  for (auto& s : bp->servers) {
    AggArgs aa = s.a;
    if (!from_dense) aa.solo_gbase = nullptr;  // (sparse inputs: no push-group bases)
    launch_aggregate(aa, st, marked, from_dense && s.fused);
  }
  if (ev) CK(cudaEventRecordWithFlags(ev[3], st, cudaEventRecordExternal));
  bp->dec.launch(bp->da, st);
  if (ev) CK(cudaEventRecordWithFlags(ev[4], st, cudaEventRecordExternal));
  if (!diag_no_side) {
    CK(cudaEventRecord(bp->join, bp->side));
    CK(cudaStreamWaitEvent(st, bp->join, 0));
  }
  CK(cudaGetLastError());
  return ZEN_OK;
}

void bp_drop_graph(zen_bp* bp) {
  if (bp->gexec) cudaGraphExecDestroy(bp->gexec);
  if (bp->gdef) cudaGraphDestroy(bp->gdef);
  bp->gexec = nullptr;
  bp->gdef = nullptr;
  bp->gkey.clear();
}

zen_status bp_run(zen_bp* bp, bool from_dense, const float* const* dense) {
  if (!bp->connected) return fail(ZEN_E_PEER, "zen_bp_connect has not been called");
  DevGuard g(bp->ctx->device);
  cudaStream_t st = bp->ctx->stream;
  bp->collected = false;
  if (bp->timing && bp->ev_head - bp->ev_tail >= (uint64_t)kRing)
    return fail(ZEN_E_INVALID, "timing ring full: call zen_bp_stage_times");
  // (the BP hash memory is epoch-free: the depth pass leaves it vacant)
  cudaEvent_t* ring = bp->timing ? &bp->ev[(bp->ev_head % kRing) * (ZEN_STAGES + 1)] : nullptr;
  // CUDA-graph replay of the whole dense sync (not capturable on the legacy stream)
  const bool graph = bp->use_graph && from_dense && st != nullptr;
  if (!graph) {
    const uint64_t before = g_launches.load();
    CKR(bp_enqueue(bp, from_dense, dense, ring));
    bp->kernels_per_sync = uint32_t(g_launches.load() - before);
  } else {
    // stage-event nodes only in the timing variant: an event node between two
    // kernels breaks their programmatic edge (~6 us each on B200)
    std::vector<const void*> key(dense, dense + bp->workers.size());
    key.push_back((const void*)st);
    key.push_back(bp->timing ? (const void*)1 : nullptr);
    if (!bp->gexec || key != bp->gkey) {
      bp_drop_graph(bp);
      if (bp->gev.empty()) {
        bp->gev.resize(ZEN_STAGES + 1);
        for (auto& e : bp->gev) CK(cudaEventCreate(&e));
      }
      const uint64_t before = g_launches.load();
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      zen_status rc = bp_enqueue(bp, true, dense, bp->timing ? bp->gev.data() : nullptr);
      cudaGraph_t graph_def = nullptr;
      cudaError_t e = cudaStreamEndCapture(st, &graph_def);
      if (rc != ZEN_OK) {
        if (graph_def) cudaGraphDestroy(graph_def);
        return rc;
      }
      CK(e);
      bp->graph_kernels = uint32_t(g_launches.load() - before);
      g_launches.fetch_sub(bp->graph_kernels);  // counted again at each launch below
      CK(cudaGraphInstantiate(&bp->gexec, graph_def, 0));
      size_t nn = 0;
      CK(cudaGraphGetNodes(graph_def, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CK(cudaGraphGetNodes(graph_def, nodes.data(), &nn));
      bp->gev_nodes.assign(ZEN_STAGES + 1, nullptr);
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev;
        CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
        for (uint32_t i = 0; i <= ZEN_STAGES; ++i)
          if (ev == bp->gev[i]) bp->gev_nodes[i] = nd;
      }
      bp->gdef = graph_def;
      bp->gkey = key;
    }
    if (ring)
      for (uint32_t i = 0; i <= ZEN_STAGES; ++i)  // retarget the stage events
        CK(cudaGraphExecEventRecordNodeSetEvent(bp->gexec, bp->gev_nodes[i], ring[i]));
    CK(cudaGraphLaunch(bp->gexec, st));
    g_launches.fetch_add(bp->graph_kernels);
    bp->kernels_per_sync = bp->graph_kernels;
  }
  if (bp->timing) ++bp->ev_head;
  return ZEN_OK;
}

zen_status bp_collect(zen_bp* bp) {
  if (bp->collected) return ZEN_OK;
  const uint32_t n = bp->n;
  cudaStream_t st = bp->ctx->stream;
  const uint32_t me = bp->local ? 0 : bp->rank;
  const Arena& A = bp->arena_of(me);
  std::vector<PushHdr> ph(n);
  std::vector<PullHdr> pl(n);
  CK(cudaMemcpyAsync(ph.data(), A.push_hdr(bp->L), n * sizeof(PushHdr), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(pl.data(), A.pull_hdr(bp->L), n * sizeof(PullHdr), cudaMemcpyDeviceToHost, st));
  std::vector<HashHdr> hh(bp->workers.size());
  for (size_t i = 0; i < bp->workers.size(); ++i)
    CK(cudaMemcpyAsync(&hh[i], bp->workers[i].a.hdr, sizeof(HashHdr), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&bp->h_result, bp->out_count, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  uint32_t status = 0;
  for (auto& h : hh) status |= h.status;
  for (uint32_t w = 0; w < n; ++w) status |= ph[w].status | pl[w].status;
  if (status) {  // sticky device errors are reported once, then cleared
    for (auto& w : bp->workers) CK(cudaMemsetAsync(&w.a.hdr->status, 0, 4, st));
    CK(cudaStreamSynchronize(st));
  }
  if (status & kErrTimeout) return fail(ZEN_E_TIMEOUT, "a peer never signalled (check that every rank calls sync)");
  if (status & kErrCapacity) return fail(ZEN_E_CAPACITY, "nnz above the max_nnz the synchroniser was created with");
  bp->h_counts.assign(size_t(n) * n, 0);
  bp->h_nnz.assign(n, 0);
  bp->h_agg.assign(n, 0);
  for (uint32_t w = 0; w < n; ++w) {
    for (uint32_t s = 0; s < n; ++s) bp->h_counts[size_t(w) * n + s] = ph[w].counts[s];
    bp->h_nnz[w] = ph[w].nnz;
    bp->h_agg[w] = pl[w].agg_count;
  }
  if (bp->local) {  // no push headers in local mode: the workers' own counters
    std::vector<uint32_t> ld(n);
    for (size_t i = 0; i < bp->workers.size(); ++i) {
      const uint32_t w = bp->workers[i].id;
      CK(cudaMemcpy(ld.data(), bp->workers[i].a.load, n * 4, cudaMemcpyDeviceToHost));
      const bool cap_ok = !(hh[i].status & kErrCapacity);
      for (uint32_t s = 0; s < n; ++s) bp->h_counts[size_t(w) * n + s] = cap_ok ? ld[s] : 0;
      bp->h_nnz[w] = hh[i].count;
      ph[w].ovf_word = hh[i].ovf_word;
    }
  }
  if (bp->local)  // no pull headers in local mode: U_s from each server's counter
    for (auto& s : bp->servers) {
      CK(cudaMemcpy(&bp->h_agg[s.id], s.agg_count, 8, cudaMemcpyDeviceToHost));
    }
  for (uint32_t w = 0; w < n; ++w) {  // run_balanced_parallelism throws at the first worker
    if (ph[w].ovf_word != ~0ull) {
      const uint32_t p = uint32_t(ph[w].ovf_word & 0xFFFF);
      return fail(ZEN_E_SERIAL_OVERFLOW,
                  "hash partition " + std::to_string(p) +
                      " exceeded its slot capacity (r2 too small for this workload)",
                  p);
    }
  }
  if (status & kErrOutside) return fail(ZEN_E_INDEX_OUTSIDE_UNIVERSE, "index outside universe");
  if (bp->h_result > bp->out_cap) return fail(ZEN_E_CAPACITY, "result above capacity");
  bp->collected = true;
  return ZEN_OK;
}

}  // namespace

extern "C" {

zen_status zen_bp_sync_dense(zen_bp* bp, const float* const* d_dense) {
  if (!bp || !d_dense) return fail(ZEN_E_INVALID, "null argument");
  for (size_t i = 0; i < bp->workers.size(); ++i)
    if (!d_dense[i]) return fail(ZEN_E_INVALID, "null dense gradient");
  return bp_run(bp, true, d_dense);
}

zen_status zen_bp_sync_sparse(zen_bp* bp, const uint64_t* const* d_idx, const float* const* d_val,
                              const uint64_t* nnz) {
  if (!bp || !d_idx || !d_val || !nnz) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  cudaStream_t st = bp->ctx->stream;
  for (size_t i = 0; i < bp->workers.size(); ++i) {
    Worker& w = bp->workers[i];
    if (nnz[i] > bp->cap) return fail(ZEN_E_CAPACITY, "nnz above max_nnz");
    if (nnz[i] && (!d_idx[i] || !d_val[i])) return fail(ZEN_E_INVALID, "null tensor");
    // a SparseTensor's invariant (zen/tensor.hpp:36-45: ascending, unique,
    // < M) is checked before the u32 narrowing below can wrap an index
    if (nnz[i]) {
      CK(cudaMemsetAsync(bp->chk, 0, 4, st));
      CKR(wire_check_input(bp->ctx, d_idx[i], nnz[i], bp->m, bp->chk));
    }
    w.h_count = nnz[i];
    if (nnz[i]) {
      launch_u64_to_u32(d_idx[i], w.keys, nnz[i], st);
      CK(cudaMemcpyAsync(w.vals, d_val[i], nnz[i] * 4, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemcpyAsync(&w.a.hdr->count, &w.h_count, 8, cudaMemcpyHostToDevice, st));
  }
  return bp_run(bp, false, nullptr);
}

zen_status zen_bp_wait(zen_bp* bp) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  return bp_collect(bp);
}

zen_status zen_bp_result(zen_bp* bp, const uint64_t** d_idx, const float** d_val,
                         uint64_t* count) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CKR(bp_collect(bp));
  if (d_idx) *d_idx = bp->out_idx;
  if (d_val) *d_val = bp->out_val;
  if (count) *count = bp->h_result;
  return ZEN_OK;
}

zen_status zen_bp_copy_result(zen_bp* bp, uint64_t* d_idx, float* d_val, uint64_t capacity,
                              uint64_t* count) {
  if (!bp || !count) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CKR(bp_collect(bp));
  *count = bp->h_result;
  if (bp->h_result > capacity) return fail(ZEN_E_CAPACITY, "result buffer too small");
  cudaStream_t st = bp->ctx->stream;
  if (bp->h_result) {
    CK(cudaMemcpyAsync(d_idx, bp->out_idx, bp->h_result * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d_val, bp->out_val, bp->h_result * 4, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  return ZEN_OK;
}

zen_status zen_bp_traffic(zen_bp* bp, uint64_t* ledger, uint64_t* counts, uint64_t* agg) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CKR(bp_collect(bp));
  const uint32_t n = bp->n;
  if (counts) std::memcpy(counts, bp->h_counts.data(), size_t(n) * n * 8);
  if (agg) std::memcpy(agg, bp->h_agg.data(), n * 8);
  if (ledger) {  // the SimNet ledger of run_balanced_parallelism, zen/schemes.hpp:369-372, :386-388
    std::memset(ledger, 0, sizeof(uint64_t) * 8 * n);
    auto at = [&](int st, int f, uint32_t node) -> uint64_t& { return ledger[(st * 4 + f) * n + node]; };
    for (uint32_t w = 0; w < n; ++w)
      for (uint32_t s = 0; s < n; ++s) {
        const uint64_t c = bp->h_counts[size_t(w) * n + s];
        if (s == w || c == 0) continue;
        at(0, 0, w) += 96 * c;  // COO: 64-bit index + 32-bit value (zen/codec.hpp:186-189)
        at(0, 1, s) += 96 * c;
        at(0, 2, s) += 64 * c;
        at(0, 3, s) += 32 * c;
      }
    for (uint32_t s = 0; s < n; ++s) {
      const uint64_t ib = bp->uni->bs[s], vb = 32 * bp->h_agg[s];  // codec.hpp:202-207
      for (uint32_t w = 0; w < n; ++w) {
        if (w == s) continue;
        at(1, 0, s) += ib + vb;
        at(1, 1, w) += ib + vb;
        at(1, 2, w) += ib;
        at(1, 3, w) += vb;
      }
    }
  }
  return ZEN_OK;
}

zen_status zen_bp_balance(zen_bp* bp, double* push, double* pull, int* valid) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CKR(bp_collect(bp));
  const uint32_t n = bp->n;
  bool all = true;
  for (uint32_t w = 0; w < n; ++w) all = all && bp->h_nnz[w] > 0;
  if (valid) *valid = all ? 1 : 0;
  if (!all) return ZEN_OK;
  double worst = 0.0;  // imbalance_push, zen/hashing.hpp:296-308
  for (uint32_t w = 0; w < n; ++w)
    for (uint32_t s = 0; s < n; ++s)
      worst = std::max(worst, double(n) * double(bp->h_counts[size_t(w) * n + s]) / double(bp->h_nnz[w]));
  if (push) *push = worst;
  uint64_t uni = 0;  // imbalance_pull, zen/hashing.hpp:311-320
  for (uint32_t s = 0; s < n; ++s) uni += bp->h_agg[s];
  double wp = 0.0;
  for (uint32_t s = 0; s < n; ++s) wp = std::max(wp, double(n) * double(bp->h_agg[s]) / double(uni));
  if (pull) *pull = wp;
  return ZEN_OK;
}

zen_status zen_bp_collision_stats(zen_bp* bp, uint32_t worker, zen_collision_stats* out) {
  if (!bp || !out) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  SetupStream setup_(bp->ctx->stream);
  CKR(bp_collect(bp));
  for (auto& w : bp->workers) {
    if (w.id != worker) continue;
    const uint32_t k = bp->params.rehash_depth;
    std::vector<uint64_t> st(k + 1);
    CK(cudaMemcpy(st.data(), w.a.stats_out, (k + 1) * 8, cudaMemcpyDeviceToHost));
    std::memset(out, 0, sizeof(*out));
    out->k = k;
    out->serial_writes = st[0];
    for (uint32_t d = 0; d < k; ++d) out->placed_at_depth[d] = st[1 + d];
    return ZEN_OK;
  }
  return fail(ZEN_E_INVALID, "worker not hosted by this synchroniser");
}

zen_status zen_bp_enable_timing(zen_bp* bp, int on) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  if (on && bp->ev.empty()) {
    bp->ev.resize(size_t(kRing) * (ZEN_STAGES + 1));
    for (auto& e : bp->ev) CK(cudaEventCreate(&e));
  }
  bp->timing = on != 0;
  return ZEN_OK;
}

zen_status zen_bp_stage_times(zen_bp* bp, double* ms, uint64_t* syncs) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CK(cudaStreamSynchronize(bp->ctx->stream));
  for (; bp->ev_tail < bp->ev_head; ++bp->ev_tail) {
    const uint64_t slot = bp->ev_tail % kRing;
    for (uint32_t s = 0; s < ZEN_STAGES; ++s) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, bp->ev[slot * (ZEN_STAGES + 1) + s],
                              bp->ev[slot * (ZEN_STAGES + 1) + s + 1]));
      bp->stage_ms[s] += t;
    }
    ++bp->timed;
  }
  for (uint32_t s = 0; s < ZEN_STAGES; ++s) {
    if (ms) ms[s] = bp->stage_ms[s];
    bp->stage_ms[s] = 0;
  }
  if (syncs) *syncs = bp->timed;
  bp->timed = 0;
  return ZEN_OK;
}

uint32_t zen_bp_kernels_per_sync(const zen_bp* bp) { return bp ? bp->kernels_per_sync : 0; }

zen_status zen_bp_use_graph(zen_bp* bp, int on) {
  if (!bp) return fail(ZEN_E_INVALID, "null argument");
  bp->use_graph = on != 0;
  return ZEN_OK;
}

zen_status zen_bp_time_extract(zen_bp* bp, const float* d_dense, uint32_t iters, double* ms) {
  if (!bp || !d_dense || !ms || !iters) return fail(ZEN_E_INVALID, "null argument");
  if (bp->workers.empty()) return fail(ZEN_E_INVALID, "no local worker");
  DevGuard g(bp->ctx->device);
  cudaStream_t st = bp->ctx->stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // the sync's own extraction kernel (staging + h0 partition counts); its
  // counters only accumulate here and are reset by the next sync's begin
  Worker& w0 = bp->workers[0];
  // ZEN_DIAG_EXTRACT_PLAIN=1: the tile pass without the h0 counts (diagnosis)
  static const bool plain = std::getenv("ZEN_DIAG_EXTRACT_PLAIN") != nullptr;
  auto one = [&] {
    if (plain)
      launch_extract_tiles<uint32_t>(d_dense, bp->m, w0.ex, st);
    else
      launch_extract_tiles_part<uint32_t>(d_dense, bp->m, w0.ex, w0.a, st);
  };
  one();  // warm-up
  CK(cudaEventRecord(e0, st));
  for (uint32_t i = 0; i < iters; ++i) one();
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = double(t) / iters;
  return ZEN_OK;
}

zen_status zen_bp_sync_host(zen_bp* bp, const float* const* h_dense, uint64_t* h_idx,
                            float* h_val, uint64_t capacity, uint64_t* count) {
  if (!bp || !h_dense || !count) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  SetupStream setup_(bp->ctx->stream);
  cudaStream_t st = bp->ctx->stream;
  if (bp->dense_dev.empty()) {
    for (size_t i = 0; i < bp->workers.size(); ++i) {
      void* p = nullptr;
      CK(cudaMalloc(&p, bp->m * 4));
      bp->dense_dev.push_back((float*)p);
    }
  }
  for (size_t i = 0; i < bp->workers.size(); ++i)
    CK(cudaMemcpyAsync(bp->dense_dev[i], h_dense[i], bp->m * 4, cudaMemcpyHostToDevice, st));
  CKR(bp_run(bp, true, bp->dense_dev.data()));
  CKR(bp_collect(bp));
  *count = bp->h_result;
  if (bp->h_result > capacity) return fail(ZEN_E_CAPACITY, "host result buffer too small");
  if (bp->h_result) {
    CK(cudaMemcpyAsync(h_idx, bp->out_idx, bp->h_result * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_val, bp->out_val, bp->h_result * 4, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return ZEN_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- debug ----
// Test/diagnostic access to a local worker's compacted keys and a local
// server's inbox part (what worker `w` pushed to it).  Not on the hot path.
extern "C" zen_status zen_bp_debug_part(zen_bp* bp, int what, uint32_t server, uint32_t worker,
                                        uint32_t* h_idx, float* h_val, uint64_t cap,
                                        uint64_t* count) {
  if (!bp || !count) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(bp->ctx->device);
  CK(cudaStreamSynchronize(bp->ctx->stream));
  if (what == 0) {  // compacted keys of a local worker (values: sparse-input syncs only)
    for (auto& w : bp->workers) {
      if (w.id != worker) continue;
      HashHdr h{};
      CK(cudaMemcpy(&h, w.a.hdr, sizeof(h), cudaMemcpyDeviceToHost));
      *count = h.count;
      const uint64_t c = std::min(cap, h.count);
      CK(cudaMemcpy(h_idx, w.keys, c * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h_val, w.vals, c * 4, cudaMemcpyDeviceToHost));
      return ZEN_OK;
    }
    return fail(ZEN_E_INVALID, "worker not local");
  }
  if (what == 2 || what == 3) {  // 2: server's pull bitmap words; 3: own table (mask, prefix)
    if (server >= bp->n) return fail(ZEN_E_INVALID, "bad server");
    if (what == 2) {
      const Arena& R = bp->arena_of(bp->local ? 0 : bp->rank);
      const uint64_t nw = bp->nw[server];
      *count = nw;
      CK(cudaMemcpy(h_idx, R.bits(bp->L, server), std::min(cap, nw) * 8, cudaMemcpyDeviceToHost));
      return ZEN_OK;
    }
    CKR(bp->uni->ensure_own(server));
    *count = bp->uni->nwords;
    CK(cudaMemcpy(h_idx, bp->uni->own[server], std::min(cap, bp->uni->nwords) * 16,
                  cudaMemcpyDeviceToHost));
    return ZEN_OK;
  }
  // inbox part worker -> server (server must be local)
  const Arena& A = bp->arena_of(server);
  if (!A.base || (!bp->local && server != bp->rank)) return fail(ZEN_E_INVALID, "server not local");
  const ArenaLayout& L = bp->layout_of(server);
  PushHdr ph{};
  if (bp->local) {
    if (worker >= bp->workers.size()) return fail(ZEN_E_INVALID, "bad worker");
    CK(cudaMemcpy(&ph.counts[server], bp->workers[worker].a.load + server, 4,
                  cudaMemcpyDeviceToHost));
  } else {
    CK(cudaMemcpy(&ph, A.push_hdr(L) + worker, sizeof(ph), cudaMemcpyDeviceToHost));
  }
  *count = ph.counts[server];
  const uint64_t c = std::min<uint64_t>(cap, ph.counts[server]);
  CK(cudaMemcpy(h_idx, A.inbox_idx(L) + size_t(worker) * bp->cap, c * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_val, A.inbox_val(L) + size_t(worker) * bp->cap, c * 4, cudaMemcpyDeviceToHost));
  return ZEN_OK;
}

// ======================================== centralized schemes, rank mode ==
// One process per GPU, NVLink stores into the peers' CUDA-IPC arenas, every
// fold the merge-path merge_sum (k_merge.cu); counts never leave the device,
// so a dense sync is one CUDA graph.
//   ZEN_SCHEME_HC       run_hier_centralization (zen/schemes.hpp:173-193):
//                       stage s: state -> rank^2^s, state' = merge(state, recv)
//   ZEN_SCHEME_RING     run_ring_centralization (zen/schemes.hpp:194-215):
//                       stage s: token -> rank+1, token' = merge(recv, input)
//   ZEN_SCHEME_AGSPARSE run_agsparse, point-to-point (zen/schemes.hpp:119-168):
//                       input -> every peer, then aggregate in worker order

namespace {
constexpr uint32_t kHcMaxRanks = 256;

struct HcHdr {
  unsigned long long epoch;
  unsigned long long ready[2 * kHcMaxRanks];  // receive slot j was filled (epoch)
  unsigned long long done[2 * kHcMaxRanks];  // this rank's push i was consumed
  uint64_t cnt[3];                        // [input, state 0, state 1] counts
  uint64_t rcnt[2 * kHcMaxRanks];         // receive slot counts
  uint64_t sent[2 * kHcMaxRanks];         // entries of this rank's i-th push (ledger)
  uint64_t bnd[kHcMaxRanks + 1];          // OmniReduce: range bounds of the input
  uint32_t err;                           // kErr* bits
  uint32_t in_err;                        // kWire* bits of the input check
};

constexpr int kBufIn = 0, kBufSt0 = 1, kBufSt1 = 2, kBufRecv = 3;  // + slot

struct HcPush {
  int src;
  uint32_t dst, slot;
  uint64_t cap;
  int src_bnd = -1;   // OmniReduce: the source is input range [bnd[i], bnd[i+1])
  int src_wait = -1;  // AGsparse forwarding: the source slot's ready flag to acquire
};
struct HcMerge {
  int a, b, out;
  int wait[2];       // receive slots to acquire (-1: none)
  int done_rank[2];  // senders whose pushes this merge consumes (-1: none) ...
  int done_idx[2];   // ... and the index of that push in the sender's plan
  uint64_t a_cap, b_cap;
  int a_bnd = -1, b_bnd = -1;  // OmniReduce: an operand is input range i
};
struct HcStage {
  bool bounds = false;  // OmniReduce: range bounds of the input first
  std::vector<HcPush> push;
  std::vector<HcMerge> merge;
  int concat_out = -1;  // OmniReduce: concat (zeros dropped) of the ranges into this buffer
};
}  // namespace

struct zen_hc {
  zen_ctx* ctx = nullptr;
  uint32_t scheme = ZEN_SCHEME_HC;
  uint32_t n = 0, rank = 0;
  uint64_t m = 0, max_nnz = 0, cap = 0;
  std::vector<HcStage> plan;
  int result_buf = kBufSt0;
  uint32_t nslots = 0;
  std::vector<size_t> off_idx, off_val;  // per buffer id
  std::vector<uint64_t> buf_cap;
  size_t bytes = 0;
  char* base = nullptr;
  std::vector<char*> peer;  // arena base per rank (own at `rank`)
  bool connected = false;
  DevMem mem;
  ExtractWs<uint64_t> ex{};
  unsigned long long* lb = nullptr;
  uint64_t* splits = nullptr;
  LookbackCtl* ctl_merge = nullptr;
  LookbackCtl* ctl_push = nullptr;
  cudaGraph_t gdef = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const float* gdense = nullptr;
  cudaStream_t gstream = nullptr;
  uint32_t graph_kernels = 0;
  uint32_t npush = 0;
  uint64_t h_result = 0;
  int omni_acc = -1;  // OmniReduce: the buffer holding this rank's range aggregate
  // OmniReduce concat tables (device), built at connect
  const uint64_t** c_idx = nullptr;
  const float** c_val = nullptr;
  const uint64_t** c_cnt = nullptr;
  const unsigned long long** c_wait = nullptr;
  unsigned long long** c_done = nullptr;
  HcHdr* hdr(uint32_t r) const { return reinterpret_cast<HcHdr*>(peer[r]); }
  uint32_t nslots_used() const { return uint32_t(buf_cap.size()) - kBufRecv; }
  uint64_t* idx(uint32_t r, int b) const { return reinterpret_cast<uint64_t*>(peer[r] + off_idx[b]); }
  float* val(uint32_t r, int b) const { return reinterpret_cast<float*>(peer[r] + off_val[b]); }
  uint64_t* cntp(uint32_t r, int b) const {
    return b < kBufRecv ? &hdr(r)->cnt[b] : &hdr(r)->rcnt[b - kBufRecv];
  }
};

namespace {

// The per-rank plan of a scheme: pushes and folds per stage, and the buffers.
// A sender's push i waits until the receiver released done[i] for the
// previous sync; the receiver releases it after the fold that consumed it.
void hc_plan(zen_hc* h) {
  const uint32_t n = h->n, r = h->rank;
  const uint64_t z = h->max_nnz, M = h->m;
  auto capk = [&](uint64_t k) { return std::min<uint64_t>(M, k * z); };
  h->buf_cap = {capk(1), h->cap, h->cap};
  auto merge = [](int a, int b, int out, uint64_t ac, uint64_t bc) {
    return HcMerge{a, b, out, {-1, -1}, {-1, -1}, {0, 0}, ac, bc, -1, -1};
  };
  if (h->scheme == ZEN_SCHEME_HC) {
    uint32_t L = 0;
    while ((1u << L) < n) ++L;
    int cur = kBufIn;
    for (uint32_t s = 0; s < L; ++s) {
      const uint32_t q = r ^ (1u << s);
      const int out = (s & 1) ? kBufSt1 : kBufSt0;
      HcStage st;
      st.push.push_back({cur, q, s, capk(1ull << s)});
      HcMerge mg = merge(cur, kBufRecv + int(s), out, capk(1ull << s), capk(1ull << s));
      mg.wait[0] = int(s);
      mg.done_rank[0] = int(q);
      mg.done_idx[0] = int(s);  // q's s-th push
      st.merge.push_back(mg);
      h->plan.push_back(st);
      h->buf_cap.push_back(capk(1ull << s));
      cur = out;
    }
    h->result_buf = cur;
  } else if (h->scheme == ZEN_SCHEME_RING) {
    int tok = kBufIn;
    for (uint32_t s = 0; s + 1 < n; ++s) {
      const uint32_t next = (r + 1) % n, prev = (r + n - 1) % n;
      const int out = (s & 1) ? kBufSt1 : kBufSt0;
      HcStage st;
      st.push.push_back({tok, next, s, capk(s + 1)});
      // token'[w] = merge_sum(token[w-1], input[w]): the received token first
      HcMerge mg = merge(kBufRecv + int(s), kBufIn, out, capk(s + 1), capk(1));
      mg.wait[0] = int(s);
      mg.done_rank[0] = int(prev);
      mg.done_idx[0] = int(s);
      st.merge.push_back(mg);
      h->plan.push_back(st);
      h->buf_cap.push_back(capk(s + 1));
      tok = out;
    }
    h->result_buf = tok;
  } else if (h->scheme == ZEN_SCHEME_OMNIREDUCE) {
    // run_omnireduce_like (zen/schemes.hpp:219-328): range p = [p*R, (p+1)*R),
    // R = ceil(M/n).  Stage 0: slice p of the input -> owner p (slot = sender);
    // the owner folds the n slices in worker order.  Stage 1: the owner's
    // aggregate -> every peer (slot n + owner); every rank concatenates the
    // n ranges and drops exact zeros (the block decode).
    const uint64_t R = (M + n - 1) / n;
    auto rcap = [&](uint32_t p) {
      const uint64_t lo = uint64_t(p) * R, hi = std::min(M, lo + R);
      return std::min<uint64_t>(hi > lo ? hi - lo : 0, uint64_t(n) * z);
    };
    auto idx0 = [&](uint32_t sender) { return int(r < sender ? r : r - 1); };  // stage-0 push index
    HcStage s0;
    s0.bounds = true;
    for (uint32_t q = 0; q < n; ++q)
      if (q != r) {
        HcPush p{kBufIn, q, r, capk(1)};
        p.src_bnd = int(q);
        s0.push.push_back(p);
      }
    auto slice = [&](uint32_t w, int* buf, int* bnd) {
      *buf = w == r ? kBufIn : kBufRecv + int(w);
      *bnd = w == r ? int(r) : -1;
    };
    int acc, acc_bnd;
    slice(0, &acc, &acc_bnd);
    for (uint32_t w = 1; w < n; ++w) {
      const int out = (w & 1) ? kBufSt0 : kBufSt1;
      int b, b_bnd;
      slice(w, &b, &b_bnd);
      HcMerge mg = merge(acc, b, out, capk(w), capk(1));
      mg.a_bnd = acc_bnd;
      mg.b_bnd = b_bnd;
      int k = 0;
      if (w == 1 && r != 0) {
        mg.wait[k] = 0;
        mg.done_rank[k] = 0;
        mg.done_idx[k++] = idx0(0);
      }
      if (w != r) {
        mg.wait[k] = int(w);
        mg.done_rank[k] = int(w);
        mg.done_idx[k++] = idx0(w);
      }
      s0.merge.push_back(mg);
      acc = out;
      acc_bnd = -1;
    }
    h->plan.push_back(s0);
    HcStage s1;
    for (uint32_t q = 0; q < n; ++q)
      if (q != r) s1.push.push_back({acc, q, n + r, rcap(r)});
    s1.concat_out = acc == kBufSt0 ? kBufSt1 : kBufSt0;
    h->plan.push_back(s1);
    for (uint32_t j = 0; j < n; ++j) h->buf_cap.push_back(capk(1));  // slices
    for (uint32_t p = 0; p < n; ++p) h->buf_cap.push_back(rcap(p));  // owners' ranges
    h->omni_acc = acc;
    h->result_buf = s1.concat_out;
  } else {  // AGsparse (zen/schemes.hpp:119-168): slot j holds worker j's input
    // pushes of one rank, in order: (stage, destination, origin), per pattern
    const uint32_t pattern = h->scheme;
    auto pushes_of = [&](uint32_t q) {
      std::vector<std::array<uint32_t, 3>> v;
      if (pattern == ZEN_SCHEME_AGSPARSE) {  // point-to-point: one stage
        for (uint32_t d = 0; d < n; ++d)
          if (d != q) v.push_back({0u, d, q});
      } else if (pattern == ZEN_SCHEME_AGSPARSE_RING) {  // stage s forwards origin q - s
        for (uint32_t st = 0; st + 1 < n; ++st) v.push_back({st, (q + 1) % n, (q + n - st) % n});
      } else {  // hierarchy: stage s sends every held origin to q ^ 2^s
        std::vector<uint32_t> hold{q};
        for (uint32_t bit = 1, st = 0; bit < n; bit <<= 1, ++st) {
          for (uint32_t o : hold) v.push_back({st, q ^ bit, o});
          // the partner held the same-size aligned group: origins of its group
          const uint32_t base = (q ^ bit) & ~(bit - 1);
          for (uint32_t o = base; o < base + bit; ++o) hold.push_back(o);
        }
      }
      return v;
    };
    // who delivered origin o to this rank, and as which of its pushes
    std::vector<int> from(n, -1), from_idx(n, -1);
    for (uint32_t q = 0; q < n; ++q) {
      if (q == r) continue;
      const auto v = pushes_of(q);
      for (size_t i = 0; i < v.size(); ++i)
        if (v[i][1] == r) {
          from[v[i][2]] = int(q);
          from_idx[v[i][2]] = int(i);
        }
    }
    auto in_of = [&](uint32_t w) { return w == r ? kBufIn : kBufRecv + int(w); };
    const auto mine = pushes_of(r);
    uint32_t nst = 0;
    for (const auto& e : mine) nst = std::max(nst, e[0] + 1);
    h->plan.assign(std::max(nst, 1u), HcStage{});
    for (const auto& e : mine) {
      HcPush p{in_of(e[2]), e[1], e[2], capk(1)};
      p.src_wait = e[2] == r ? -1 : int(e[2]);  // a forwarded origin must have arrived
      h->plan[e[0]].push.push_back(p);
    }
    HcStage& last = h->plan.back();
    int acc = in_of(0);
    for (uint32_t w = 1; w < n; ++w) {
      const int out = (w & 1) ? kBufSt0 : kBufSt1;
      HcMerge mg = merge(acc, in_of(w), out, capk(w), capk(1));
      int k = 0;
      if (w == 1 && r != 0) {  // worker 0's input arrives too
        mg.wait[k] = 0;
        mg.done_rank[k] = from[0];
        mg.done_idx[k++] = from_idx[0];
      }
      if (w != r) {
        mg.wait[k] = int(w);
        mg.done_rank[k] = from[w];
        mg.done_idx[k++] = from_idx[w];
      }
      last.merge.push_back(mg);
      acc = out;
    }
    // every rank's arena must have the same layout: peers address it with
    // their own offsets (this rank's own slot stays unused)
    for (uint32_t j = 0; j < n; ++j) h->buf_cap.push_back(capk(1));
    h->result_buf = acc;
  }
}

zen_status hc_enqueue(zen_hc* h, const float* dense, const uint64_t* in_idx, const float* in_val,
                      uint64_t in_count) {
  cudaStream_t st = h->ctx->stream;
  const uint32_t r = h->rank;
  HcHdr* me = h->hdr(r);
  launch_hc_begin(&me->epoch, st);
  if (dense) {
    launch_extract<uint64_t>(dense, h->m, h->ex, h->idx(r, kBufIn), h->val(r, kBufIn),
                             &me->cnt[kBufIn], h->max_nnz, &me->err, st);
  } else {
    if (in_count) {
      CK(cudaMemcpyAsync(h->idx(r, kBufIn), in_idx, in_count * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(h->val(r, kBufIn), in_val, in_count * 4, cudaMemcpyDeviceToDevice, st));
    }
    launch_check_canonical(in_idx, in_count, h->m, &me->in_err, st);
    launch_set_u64(&me->cnt[kBufIn], in_count, st);
  }
  uint32_t pi = 0;
  for (const HcStage& stg : h->plan) {
    if (stg.bounds) launch_hc_bounds(h->idx(r, kBufIn), &me->cnt[kBufIn], h->m, h->n, me->bnd, st);
    for (const HcPush& p : stg.push) {
      HcPushArgs a{};
      a.src_idx = h->idx(r, p.src);
      a.src_val = h->val(r, p.src);
      a.src_cnt = h->cntp(r, p.src);
      a.dst_idx = h->idx(p.dst, kBufRecv + int(p.slot));
      a.dst_val = h->val(p.dst, kBufRecv + int(p.slot));
      a.dst_cnt = &h->hdr(p.dst)->rcnt[p.slot];
      a.cap = p.cap;
      a.ready_flag = &h->hdr(p.dst)->ready[p.slot];
      a.done_flag = &me->done[pi];
      a.epoch = &me->epoch;
      a.ctl = h->ctl_push;
      a.err = &me->err;
      a.sent_cnt = &me->sent[pi++];
      a.src_bnd = p.src_bnd >= 0 ? &me->bnd[p.src_bnd] : nullptr;
      a.src_wait = p.src_wait >= 0 ? &me->ready[p.src_wait] : nullptr;
      launch_hc_push(a, st);
    }
    for (const HcMerge& mg : stg.merge) {
      HcMergeArgs a{};
      a.a_idx = h->idx(r, mg.a);
      a.a_val = h->val(r, mg.a);
      a.a_cnt = h->cntp(r, mg.a);
      a.a_cap = mg.a_cap;
      a.b_idx = h->idx(r, mg.b);
      a.b_val = h->val(r, mg.b);
      a.b_cnt = h->cntp(r, mg.b);
      a.b_cap = mg.b_cap;
      a.o_idx = h->idx(r, mg.out);
      a.o_val = h->val(r, mg.out);
      a.o_cnt = h->cntp(r, mg.out);
      a.o_cap = h->cap;
      a.lb_status = h->lb;
      a.ctl = h->ctl_merge;
      a.err = &me->err;
      a.wait_flag = mg.wait[0] >= 0 ? &me->ready[mg.wait[0]] : nullptr;
      a.wait_flag2 = mg.wait[1] >= 0 ? &me->ready[mg.wait[1]] : nullptr;
      a.done_flag = mg.done_rank[0] >= 0
                        ? &h->hdr(uint32_t(mg.done_rank[0]))->done[mg.done_idx[0]] : nullptr;
      a.done_flag2 = mg.done_rank[1] >= 0
                         ? &h->hdr(uint32_t(mg.done_rank[1]))->done[mg.done_idx[1]] : nullptr;
      a.epoch = &me->epoch;
      a.a_bnd = mg.a_bnd >= 0 ? &me->bnd[mg.a_bnd] : nullptr;
      a.b_bnd = mg.b_bnd >= 0 ? &me->bnd[mg.b_bnd] : nullptr;
      a.splits = h->splits;
      launch_hc_merge(a, hc_merge_tiles(mg.a_cap + mg.b_cap), st);
    }
    if (stg.concat_out >= 0) {
      HcConcatArgs c{};
      c.seg_idx = h->c_idx;
      c.seg_val = h->c_val;
      c.seg_cnt = h->c_cnt;
      c.wait = h->c_wait;
      c.done = h->c_done;
      c.n = h->n;
      c.seg_cap = h->cap;
      c.o_idx = h->idx(r, stg.concat_out);
      c.o_val = h->val(r, stg.concat_out);
      c.o_cnt = h->cntp(r, stg.concat_out);
      c.o_cap = h->cap;
      c.lb_status = h->lb;
      c.ctl = h->ctl_merge;
      c.err = &me->err;
      c.epoch = &me->epoch;
      launch_hc_concat(c, hc_merge_tiles(h->cap), st);
    }
  }
  h->npush = pi;
  return ZEN_OK;
}

void hc_drop_graph(zen_hc* h) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gdef) cudaGraphDestroy(h->gdef);
  h->gexec = nullptr;
  h->gdef = nullptr;
  h->gdense = nullptr;
  h->gstream = nullptr;
}

}  // namespace

extern "C" {

zen_status zen_hc_create_scheme(zen_ctx* c, uint32_t scheme, uint32_t n, uint32_t rank,
                                uint64_t universe, uint64_t max_nnz, zen_hc** out) {
  if (!c || !out) return fail(ZEN_E_INVALID, "null argument");
  if (scheme > ZEN_SCHEME_AGSPARSE_HIER) return fail(ZEN_E_INVALID, "unknown scheme");
  const bool pow2 = n != 0 && (n & (n - 1)) == 0;
  if (scheme == ZEN_SCHEME_OMNIREDUCE && n < 2)
    return fail(ZEN_E_INVALID, "synchronization needs at least two nodes");
  if (n == 0 || ((scheme == ZEN_SCHEME_HC || scheme == ZEN_SCHEME_RING ||
                  scheme == ZEN_SCHEME_AGSPARSE_RING || scheme == ZEN_SCHEME_AGSPARSE_HIER) &&
                 !pow2))
    return fail(ZEN_E_INVALID, "node count must be a power of two");
  if (n > kHcMaxRanks) return fail(ZEN_E_INVALID, "node count above 256");
  if (rank >= n) return fail(ZEN_E_INVALID, "rank out of range");
  if (universe == 0) return fail(ZEN_E_INVALID, "universe must be at least 1");
  if (max_nnz == 0) return fail(ZEN_E_INVALID, "max_nnz must be at least 1");
  DevGuard g(c->device);
  SetupStream setup_(c->stream);
  std::unique_ptr<zen_hc> h(new zen_hc);
  h->ctx = c;
  h->scheme = scheme;
  h->n = n;
  h->rank = rank;
  h->m = universe;
  h->max_nnz = std::min(max_nnz, universe);
  h->cap = std::min<uint64_t>(universe, uint64_t(n) * h->max_nnz);
  hc_plan(h.get());
  size_t off = align256(sizeof(HcHdr));
  h->off_idx.resize(h->buf_cap.size());
  h->off_val.resize(h->buf_cap.size());
  for (size_t b = 0; b < h->buf_cap.size(); ++b) {
    h->off_idx[b] = off;
    off += align256(h->buf_cap[b] * 8);
    h->off_val[b] = off;
    off += align256(h->buf_cap[b] * 4);
  }
  h->bytes = off;
  CK(cudaMalloc(&h->base, h->bytes));
  CK(cudaMemsetAsync(h->base, 0, sizeof(HcHdr), c->stream));
  h->peer.assign(n, nullptr);
  h->peer[rank] = h->base;
  h->connected = n == 1;
  const uint64_t ntiles = (universe + kExtractTile - 1) / kExtractTile;
  CKR(h->mem.alloc(&h->ex.st_idx, ntiles * kExtractTile, false));
  CKR(h->mem.alloc(&h->ex.st_val, ntiles * kExtractTile, false));
  CKR(h->mem.alloc(&h->ex.tile_cnt, ntiles));
  CKR(h->mem.alloc(&h->ex.tile_base, ntiles));
  h->ex.nblk = (h->max_nnz + 255) / 256;
  CKR(h->mem.alloc(&h->ex.blk_tile, h->ex.nblk + 1));
  uint64_t max_tiles = hc_merge_tiles(h->cap);  // (the OmniReduce concat)
  for (const auto& stg : h->plan)
    for (const auto& mg : stg.merge)
      max_tiles = std::max<uint64_t>(max_tiles, hc_merge_tiles(mg.a_cap + mg.b_cap));
  CKR(h->mem.alloc(&h->lb, max_tiles));
  CKR(h->mem.alloc(&h->splits, max_tiles + 2));
  CKR(h->mem.alloc(&h->ctl_merge, 1));
  CKR(h->mem.alloc(&h->ctl_push, 1));
  CK(cudaStreamSynchronize(c->stream));
  *out = h.release();
  return ZEN_OK;
}

zen_status zen_hc_create(zen_ctx* c, uint32_t n, uint32_t rank, uint64_t universe,
                         uint64_t max_nnz, zen_hc** out) {
  return zen_hc_create_scheme(c, ZEN_SCHEME_HC, n, rank, universe, max_nnz, out);
}

void zen_hc_destroy(zen_hc* h) {
  if (!h) return;
  DevGuard g(h->ctx->device);
  cudaDeviceSynchronize();
  hc_drop_graph(h);
  for (uint32_t r = 0; r < h->n; ++r)
    if (r != h->rank && h->peer[r]) cudaIpcCloseMemHandle(h->peer[r]);
  if (h->base) cudaFree(h->base);
  delete h;
}

zen_status zen_hc_ipc_handle(zen_hc* h, void* out) {
  if (!h || !out) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(h->ctx->device);
  cudaIpcMemHandle_t ih;
  CK(cudaIpcGetMemHandle(&ih, h->base));
  std::memcpy(out, &ih, sizeof(ih));
  return ZEN_OK;
}

zen_status zen_hc_connect(zen_hc* h, const void* handles) {
  if (!h || !handles) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(h->ctx->device);
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  std::vector<uint32_t> need;  // only the ranks the plan touches
  for (const auto& stg : h->plan) {
    for (const auto& p : stg.push) need.push_back(p.dst);
    for (const auto& mg : stg.merge)
      for (int k = 0; k < 2; ++k)
        if (mg.done_rank[k] >= 0) need.push_back(uint32_t(mg.done_rank[k]));
  }
  for (uint32_t r : need) {
    if (h->peer[r]) continue;
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ZEN_E_PEER, std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(r) +
                                  "): " + cudaGetErrorString(e));
    }
    h->peer[r] = static_cast<char*>(p);
  }
  if (h->scheme == ZEN_SCHEME_OMNIREDUCE) {  // the concat's segment and flag tables
    const uint32_t n = h->n, r = h->rank;
    std::vector<const uint64_t*> ci(n), cc(n);
    std::vector<const float*> cv(n);
    std::vector<const unsigned long long*> cw(n);
    std::vector<unsigned long long*> cd(n);
    for (uint32_t p = 0; p < n; ++p) {
      if (!h->peer[p]) {
        void* q = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&q, hs[p], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(ZEN_E_PEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
        h->peer[p] = static_cast<char*>(q);
      }
      const int b = p == r ? h->omni_acc : kBufRecv + int(n + p);
      ci[p] = h->idx(r, b);
      cv[p] = h->val(r, b);
      cc[p] = h->cntp(r, b);
      cw[p] = p == r ? nullptr : &h->hdr(r)->ready[n + p];
      // owner p's stage-1 push to this rank: index (n-1) + position of r among p's peers
      cd[p] = p == r ? nullptr : &h->hdr(p)->done[(n - 1) + (r < p ? r : r - 1)];
    }
    if (!h->c_idx) {
      CKR(h->mem.alloc(&h->c_idx, n));
      CKR(h->mem.alloc(&h->c_val, n));
      CKR(h->mem.alloc(&h->c_cnt, n));
      CKR(h->mem.alloc(&h->c_wait, n));
      CKR(h->mem.alloc(&h->c_done, n));
    }
    SetupStream setup_(h->ctx->stream);
    CKR(upload(h->c_idx, ci.data(), n));
    CKR(upload(h->c_val, cv.data(), n));
    CKR(upload(h->c_cnt, cc.data(), n));
    CKR(upload(h->c_wait, cw.data(), n));
    CKR(upload(h->c_done, cd.data(), n));
  }
  h->connected = true;
  hc_drop_graph(h);
  return ZEN_OK;
}

zen_status zen_hc_sync_dense(zen_hc* h, const float* d_dense) {
  if (!h || !d_dense) return fail(ZEN_E_INVALID, "null argument");
  if (!h->connected) return fail(ZEN_E_INVALID, "zen_hc_connect has not been called");
  DevGuard g(h->ctx->device);
  cudaStream_t st = h->ctx->stream;
  if (st == nullptr) {  // the legacy stream cannot be captured
    CKR(hc_enqueue(h, d_dense, nullptr, nullptr, 0));
    return ZEN_OK;
  }
  if (!h->gexec || h->gdense != d_dense || h->gstream != st) {
    hc_drop_graph(h);
    const uint64_t before = g_launches.load();
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    zen_status rc = hc_enqueue(h, d_dense, nullptr, nullptr, 0);
    cudaGraph_t gd = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &gd);
    if (rc != ZEN_OK) {
      if (gd) cudaGraphDestroy(gd);
      return rc;
    }
    CK(e);
    h->graph_kernels = uint32_t(g_launches.load() - before);
    g_launches.fetch_sub(h->graph_kernels);
    CK(cudaGraphInstantiate(&h->gexec, gd, 0));
    h->gdef = gd;
    h->gdense = d_dense;
    h->gstream = st;
  }
  CK(cudaGraphLaunch(h->gexec, st));
  g_launches.fetch_add(h->graph_kernels);
  return ZEN_OK;
}

zen_status zen_hc_sync_sparse(zen_hc* h, const uint64_t* d_idx, const float* d_val,
                              uint64_t count) {
  if (!h) return fail(ZEN_E_INVALID, "null argument");
  if (count && (!d_idx || !d_val)) return fail(ZEN_E_INVALID, "null tensor");
  if (count > h->max_nnz) return fail(ZEN_E_CAPACITY, "input above max_nnz");
  if (!h->connected) return fail(ZEN_E_INVALID, "zen_hc_connect has not been called");
  DevGuard g(h->ctx->device);
  return hc_enqueue(h, nullptr, d_idx, d_val, count);
}

zen_status zen_hc_wait(zen_hc* h) {
  if (!h) return fail(ZEN_E_INVALID, "null argument");
  DevGuard g(h->ctx->device);
  HcHdr hh;
  CK(cudaMemcpyAsync(&hh, h->base, sizeof(HcHdr), cudaMemcpyDeviceToHost, h->ctx->stream));
  CK(cudaStreamSynchronize(h->ctx->stream));
  if (hh.err || hh.in_err) {
    const uint32_t e = hh.err, ie = hh.in_err;
    uint32_t zero[2] = {0, 0};
    CK(cudaMemcpy(&h->hdr(h->rank)->err, zero, 8, cudaMemcpyHostToDevice));
    if (e & kErrTimeout) return fail(ZEN_E_TIMEOUT, "a scheme partner never signalled");
    if (ie) return fail(ZEN_E_INVALID, "tensor indices not sorted/unique or >= M");
    if (e & kErrOutside) return fail(ZEN_E_INVALID, "a fold saw unsorted input (err bits " + std::to_string(e) + ")");
    std::string c = "non-zeros above capacity (counts: input " + std::to_string(hh.cnt[0]) +
                    ", states " + std::to_string(hh.cnt[1]) + "/" + std::to_string(hh.cnt[2]) +
                    ", received";
    for (uint32_t j = 0; j < h->nslots_used(); ++j) c += " " + std::to_string(hh.rcnt[j]);
    return fail(ZEN_E_CAPACITY, c + "; max_nnz " + std::to_string(h->max_nnz) + ")");
  }
  h->h_result = h->result_buf < kBufRecv ? hh.cnt[h->result_buf] : 0;
  return ZEN_OK;
}

zen_status zen_hc_result(zen_hc* h, const uint64_t** d_idx, const float** d_val,
                         uint64_t* count) {
  if (!h) return fail(ZEN_E_INVALID, "null argument");
  CKR(zen_hc_wait(h));
  if (d_idx) *d_idx = h->idx(h->rank, h->result_buf);
  if (d_val) *d_val = h->val(h->rank, h->result_buf);
  if (count) *count = h->h_result;
  return ZEN_OK;
}

zen_status zen_hc_copy_result(zen_hc* h, uint64_t* d_idx, float* d_val, uint64_t capacity,
                              uint64_t* count) {
  if (!h || !count) return fail(ZEN_E_INVALID, "null argument");
  const uint64_t* si;
  const float* sv;
  CKR(zen_hc_result(h, &si, &sv, count));
  if (*count > capacity) return fail(ZEN_E_CAPACITY, "result buffer too small");
  cudaStream_t st = h->ctx->stream;
  if (*count) {
    CK(cudaMemcpyAsync(d_idx, si, *count * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d_val, sv, *count * 4, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  return ZEN_OK;
}

zen_status zen_hc_stage_counts(zen_hc* h, uint64_t* counts) {
  if (!h || !counts) return fail(ZEN_E_INVALID, "null argument");
  CKR(zen_hc_wait(h));
  HcHdr hh;
  CK(cudaMemcpy(&hh, h->base, sizeof(HcHdr), cudaMemcpyDeviceToHost));
  uint32_t i = 0;
  for (const auto& stg : h->plan)
    for (size_t k = 0; k < stg.push.size(); ++k, ++i) counts[i] = hh.sent[i];
  return ZEN_OK;
}

zen_status zen_hc_counts(zen_hc* h, uint64_t* input_count, uint64_t* result_count) {
  if (!h) return fail(ZEN_E_INVALID, "null argument");
  CKR(zen_hc_wait(h));
  HcHdr hh;
  CK(cudaMemcpy(&hh, h->base, sizeof(HcHdr), cudaMemcpyDeviceToHost));
  if (input_count) *input_count = hh.cnt[kBufIn];
  if (result_count) *result_count = h->h_result;
  return ZEN_OK;
}

uint32_t zen_hc_pushes(const zen_hc* h) {
  uint32_t c = 0;
  if (h)
    for (const auto& stg : h->plan) c += uint32_t(stg.push.size());
  return c;
}

}  // extern "C"
