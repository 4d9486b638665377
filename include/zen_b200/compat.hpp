// zen_b200/compat.hpp -- header-only C++ drop-in for the reference's
// Balanced-Parallelism operator API (/root/reference/proj/include/zen/*.hpp),
// backed by the sm_100a kernels behind the C-ABI (include/zen_b200.h).
//
// Same names, argument meaning and exception types as the reference, in
// namespace zen_b200 (a reference user switches with `namespace zen = zen_b200;`
// for the operators below):
//
//   reference                                   here
//   zen::Error & subclasses (errors.hpp)        zen_b200::Error & subclasses
//   zen::SparseTensor / DenseTensor (tensor.hpp) zen_b200::SparseTensor / DenseTensor
//   zen::to_sparse (tensor.hpp:94)              zen_b200::to_sparse
//   zen::HashFamily (hashing.hpp:46)            zen_b200::HashFamily
//   zen::partition_of (hashing.hpp:85)          zen_b200::partition_of
//   zen::hierarchical_hash (hashing.hpp:251)    zen_b200::hierarchical_hash
//   zen::collision_stats (hashing.hpp:259)      zen_b200::collision_stats
//   zen::imbalance_push/pull (hashing.hpp:296)  zen_b200::imbalance_push/pull
//   zen::HashUniverseTable (codec.hpp:47)       zen_b200::HashUniverseTable
//   zen::encode/decode, every WireKind,          zen_b200::encode/decode,
//   message_sizes, write/read_framed (codec.hpp) message_sizes, write/read_framed
//   zen::write/read_sparse[_file] (tensor.hpp)  zen_b200::write/read_sparse[_file]
//   zen::SimNet / TrafficReport (simnet.hpp)    zen_b200::SimNet / TrafficReport
//   zen::HashParams / SyncOutcome (schemes.hpp) zen_b200::HashParams / SyncOutcome
//   zen::run_balanced_parallelism (schemes.hpp:341)  zen_b200::run_balanced_parallelism
//   zen::bp_universe_table (schemes.hpp:332)    zen_b200::bp_universe_table
//   zen::run_bp_with_retry (experiment.hpp:128) zen_b200::run_bp_with_retry
//   zen::merge_sum / aggregate (tensor.hpp:133) zen_b200::merge_sum / aggregate
//   zen::density, overlap/densification/skewness_ratio (tensor.hpp:106-213)
//                                               zen_b200::(same names)
//   zen::SparsityProfile, profile_sparsity,     zen_b200::(same names)
//   select_scheme, t_bp/t_hc[_coefficient] (costmodel.hpp)
//   zen::run_hier_centralization (schemes.hpp:173) zen_b200::run_hier_centralization
//   zen::run_agsparse / run_ring_centralization / run_omnireduce_like,
//   SchemeConfig, run_scheme, scheme_config_from_name (schemes.hpp:21-470)
//                                               zen_b200::(same names)
//
// Host containers stay std::vector (value semantics, as in the reference); the
// device copies are made per call.  For a device-resident, allocation-free
// sync use the zen_bp_* C-ABI directly (bench.py does).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <istream>
#include <ostream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "zen_b200.h"

namespace zen_b200 {

// ---- errors: zen/errors.hpp:10-84 ------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
class EmptyTensor : public Error {
 public:
  explicit EmptyTensor(const std::string& w = "operation requires a non-empty tensor") : Error(w) {}
};
class UniverseMismatch : public Error {
 public:
  explicit UniverseMismatch(const std::string& w = "tensors have different universe sizes")
      : Error(w) {}
};
class SerialOverflow : public Error {
 public:
  explicit SerialOverflow(uint32_t partition, const std::string& w = "")
      : Error(w.empty() ? "hash partition " + std::to_string(partition) +
                              " exceeded its slot capacity (r2 too small for this workload)"
                        : w),
        partition_(partition) {}
  uint32_t partition() const { return partition_; }

 private:
  uint32_t partition_;
};
class IndexOutsideUniverse : public Error {
 public:
  explicit IndexOutsideUniverse(const std::string& w) : Error(w) {}
};
class MalformedPayload : public Error {
 public:
  explicit MalformedPayload(const std::string& w) : Error(w) {}
};
class SelfSend : public Error {
 public:
  explicit SelfSend(const std::string& w = "a node cannot send a message to itself") : Error(w) {}
};
class UnbalancedLedger : public Error {
 public:
  explicit UnbalancedLedger(const std::string& w = "sent and received byte totals disagree")
      : Error(w) {}
};
class NonPowerOfTwo : public Error {  // errors.hpp:42-46
 public:
  explicit NonPowerOfTwo(const std::string& what = "node count must be a power of two")
      : Error(what) {}
};

class UnsupportedCombination : public Error {  // errors.hpp:48-52
 public:
  explicit UnsupportedCombination(const std::string& what = "unsupported scheme configuration")
      : Error(what) {}
};

class MissingProfileEntry : public Error {  // errors.hpp:54-57
 public:
  explicit MissingProfileEntry(const std::string& what) : Error(what) {}
};

class InfeasibleSpec : public Error {  // errors.hpp:81-84
 public:
  explicit InfeasibleSpec(const std::string& what) : Error(what) {}
};

class DeviceError : public Error {  // no CPU fallback exists
 public:
  explicit DeviceError(const std::string& w) : Error(w) {}
};

namespace detail {
// zen/hashing.hpp:18-39
inline uint64_t mix64(uint64_t x) { return zen_mix64(x); }
inline uint64_t seeded_hash(uint64_t x, uint64_t seed) { return zen_seeded_hash(x, seed); }
inline uint64_t map_to_range(uint64_t h, uint64_t range) { return zen_map_to_range(h, range); }
inline uint64_t derive_seed(uint64_t master, uint64_t stream) {
  return zen_derive_seed(master, stream);
}

inline void check(zen_status s) {
  if (s == ZEN_OK) return;
  const std::string msg = zen_last_error_message();
  switch (s) {
    case ZEN_E_SERIAL_OVERFLOW: throw SerialOverflow(uint32_t(zen_last_error_partition()), msg);
    case ZEN_E_INDEX_OUTSIDE_UNIVERSE: throw IndexOutsideUniverse(msg);
    case ZEN_E_MALFORMED: throw MalformedPayload(msg);
    case ZEN_E_EMPTY: throw EmptyTensor(msg);
    case ZEN_E_UNIVERSE_MISMATCH: throw UniverseMismatch(msg);
    case ZEN_E_INFEASIBLE: throw InfeasibleSpec(msg);
    case ZEN_E_CUDA:
    case ZEN_E_PEER:
    case ZEN_E_OOM:
    case ZEN_E_TIMEOUT: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

// device buffer
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count) : n(count) {
    if (cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess)
      throw DeviceError("cudaMalloc failed");
  }
  DBuf(const std::vector<T>& h) : DBuf(h.size()) {
    if (!h.empty()) cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  }
  ~DBuf() { cudaFree(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  std::vector<T> host(size_t count) const {
    std::vector<T> h(count);
    if (count) cudaMemcpy(h.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost);
    return h;
  }
};

// one context per process (device 0 unless ZEN_B200_DEVICE says otherwise)
// One context per host thread: the reference's operators are pure functions
// that callers run from many threads at once (acceptance.cpp's parallel_for),
// and a context's scratch and stream serve one caller at a time.
inline zen_ctx* ctx() {
  thread_local std::unique_ptr<zen_ctx, void (*)(zen_ctx*)> c = [] {
    int dev = 0;
    if (const char* e = std::getenv("ZEN_B200_DEVICE")) dev = std::atoi(e);
    cudaSetDevice(dev);
    zen_ctx* h = nullptr;
    check(zen_ctx_create(dev, &h));
    // the legacy default stream: ordered with the blocking cudaMemcpy calls
    // this header uses for its per-call host<->device copies
    check(zen_ctx_set_stream(h, nullptr));
    return std::unique_ptr<zen_ctx, void (*)(zen_ctx*)>(h, zen_ctx_destroy);
  }();
  return c.get();
}
}  // namespace detail

// ---- data model: zen/tensor.hpp:19-91 ---------------------------------------
struct DenseTensor {
  std::vector<float> values;
  DenseTensor() = default;
  explicit DenseTensor(std::vector<float> v) : values(std::move(v)) {
    if (values.empty()) throw Error("dense tensor must have at least one element");
  }
  uint64_t size() const { return values.size(); }
};

class SparseTensor {
 public:
  SparseTensor() : universe_(1) {}
  SparseTensor(uint64_t universe, std::vector<uint64_t> indices, std::vector<float> values)
      : universe_(universe), indices_(std::move(indices)), values_(std::move(values)) {
    if (universe_ == 0) throw Error("sparse tensor universe must be at least 1");
    if (indices_.size() != values_.size()) throw Error("sparse tensor index/value lengths differ");
    if (!std::is_sorted(indices_.begin(), indices_.end())) {
      std::vector<size_t> o(indices_.size());
      for (size_t i = 0; i < o.size(); ++i) o[i] = i;
      std::sort(o.begin(), o.end(), [this](size_t a, size_t b) { return indices_[a] < indices_[b]; });
      std::vector<uint64_t> ii(o.size());
      std::vector<float> vv(o.size());
      for (size_t i = 0; i < o.size(); ++i) {
        ii[i] = indices_[o[i]];
        vv[i] = values_[o[i]];
      }
      indices_.swap(ii);
      values_.swap(vv);
    }
    for (size_t i = 0; i < indices_.size(); ++i) {
      if (indices_[i] >= universe_) throw Error("sparse tensor index outside [0, M)");
      if (i > 0 && indices_[i] == indices_[i - 1]) throw Error("duplicate index in sparse tensor");
    }
  }
  static SparseTensor from_pairs(uint64_t universe, std::vector<std::pair<uint64_t, float>> pairs) {
    std::sort(pairs.begin(), pairs.end(), [](auto& a, auto& b) { return a.first < b.first; });
    std::vector<uint64_t> i(pairs.size());
    std::vector<float> v(pairs.size());
    for (size_t k = 0; k < pairs.size(); ++k) {
      i[k] = pairs[k].first;
      v[k] = pairs[k].second;
    }
    return SparseTensor(universe, std::move(i), std::move(v));
  }
  uint64_t universe() const { return universe_; }
  uint64_t nnz() const { return indices_.size(); }
  bool empty() const { return indices_.empty(); }
  const std::vector<uint64_t>& indices() const { return indices_; }
  const std::vector<float>& values() const { return values_; }
  friend bool operator==(const SparseTensor& a, const SparseTensor& b) {
    return a.universe_ == b.universe_ && a.indices_ == b.indices_ &&
           a.values_.size() == b.values_.size() &&
           std::memcmp(a.values_.data(), b.values_.data(), a.values_.size() * 4) == 0;
  }
  friend bool operator!=(const SparseTensor& a, const SparseTensor& b) { return !(a == b); }

 private:
  uint64_t universe_;
  std::vector<uint64_t> indices_;
  std::vector<float> values_;
};

// zen::to_sparse (tensor.hpp:94-104), on the GPU
inline SparseTensor to_sparse(const DenseTensor& dense) {
  const uint64_t m = dense.size();
  if (m == 0) throw Error("dense tensor must have at least one element");
  detail::DBuf<float> d(dense.values);
  detail::DBuf<uint64_t> oi(m);
  detail::DBuf<float> ov(m);
  uint64_t nnz = 0;
  detail::check(zen_to_sparse(detail::ctx(), d.p, m, oi.p, ov.p, m, &nnz));
  return SparseTensor(m, oi.host(nnz), ov.host(nnz));
}

// zen::sparsify_topk (workload.hpp:157-178) on the device: the ceil(f*M)
// largest |v| (ties to the lower index), exact zeros dropped
inline SparseTensor sparsify_topk(const DenseTensor& dense, double fraction) {
  if (!(fraction > 0.0 && fraction <= 1.0)) throw Error("top-k fraction must be in (0,1]");
  const uint64_t m = dense.size();
  const uint64_t keep = std::min<uint64_t>(m, uint64_t(std::ceil(fraction * double(m))));
  detail::DBuf<float> d(dense.values);
  detail::DBuf<uint64_t> oi(std::max<uint64_t>(keep, 1));
  detail::DBuf<float> ov(std::max<uint64_t>(keep, 1));
  uint64_t got = 0;
  detail::check(zen_sparsify_topk(detail::ctx(), d.p, m, fraction, oi.p, ov.p, keep, &got));
  return SparseTensor(m, oi.host(got), ov.host(got));
}

// ---- hashing: zen/hashing.hpp -----------------------------------------------
struct PartitionedSparseTensor {
  std::vector<SparseTensor> parts;
  uint64_t total_nnz() const {
    uint64_t s = 0;
    for (auto& p : parts) s += p.nnz();
    return s;
  }
};

struct CollisionStats {
  uint64_t serial_writes = 0;
  std::vector<uint64_t> placed_at_depth;
  uint64_t total() const {
    uint64_t s = serial_writes;
    for (auto c : placed_at_depth) s += c;
    return s;
  }
};

struct HashFamily {
  uint64_t partition_seed = 0;
  std::vector<uint64_t> slot_seeds;
  uint32_t partitions = 1;

  static HashFamily make(uint64_t seed, uint32_t n, uint32_t k) {
    zen_hash_family f;
    detail::check(zen_hash_family_make(seed, n, k, &f));
    return from(f);
  }
  static HashFamily make_worker(uint64_t shared, uint32_t worker, uint32_t n, uint32_t k) {
    zen_hash_family f;
    detail::check(zen_hash_family_make_worker(shared, worker, n, k, &f));
    return from(f);
  }
  uint32_t depth() const { return uint32_t(slot_seeds.size()); }
  // zen/hashing.hpp:73-81 (round is 1-based)
  uint32_t partition_of(uint64_t index) const {
    return uint32_t(zen_map_to_range(zen_seeded_hash(index + 1, partition_seed), partitions));
  }
  uint64_t slot_of(uint64_t index, uint32_t round, uint64_t r1) const {
    return zen_map_to_range(zen_seeded_hash(index + 1, slot_seeds.at(round - 1)), r1);
  }
  zen_hash_family c() const {
    zen_hash_family f{};
    f.partition_seed = partition_seed;
    for (size_t i = 0; i < slot_seeds.size(); ++i) f.slot_seeds[i] = slot_seeds[i];
    f.partitions = partitions;
    f.k = depth();
    return f;
  }

 private:
  static HashFamily from(const zen_hash_family& f) {
    HashFamily h;
    h.partition_seed = f.partition_seed;
    h.slot_seeds.assign(f.slot_seeds, f.slot_seeds + f.k);
    h.partitions = f.partitions;
    return h;
  }
};

// zen::partition_of (hashing.hpp:85-88): one index (host math) ...
inline uint32_t partition_of(uint64_t index, uint64_t partition_seed, uint32_t n) {
  return uint32_t(zen_map_to_range(zen_seeded_hash(index + 1, partition_seed), n));
}
// ... or a batch, on the GPU
inline std::vector<uint32_t> partition_of(const std::vector<uint64_t>& idx, uint64_t pseed,
                                          uint32_t n) {
  detail::DBuf<uint64_t> d(idx);
  detail::DBuf<uint32_t> o(idx.size());
  detail::check(zen_partition_of(detail::ctx(), d.p, idx.size(), pseed, n, o.p));
  return o.host(idx.size());
}

namespace detail {
inline std::pair<PartitionedSparseTensor, CollisionStats> run_hierarchical_hash(
    const SparseTensor& t, uint32_t n, const HashFamily& family, uint64_t r1, uint64_t r2,
    uint32_t lanes) {
  if (family.partitions != n) throw Error("hash family partition count mismatch");
  if (lanes < 1) throw Error("lane count must be at least 1");
  const uint64_t z = t.nnz();
  DBuf<uint64_t> di(t.indices());
  DBuf<float> dv(t.values());
  DBuf<uint64_t> oi(z);
  DBuf<float> ov(z);
  std::vector<uint64_t> pc(n);
  zen_collision_stats st;
  const zen_hash_family f = family.c();
  check(zen_hierarchical_hash(ctx(), di.p, dv.p, z, t.universe(), &f, r1, r2, oi.p, ov.p,
                              pc.data(), nullptr, nullptr, nullptr, &st));
  auto hi = oi.host(z);
  auto hv = ov.host(z);
  PartitionedSparseTensor out;
  uint64_t off = 0;
  for (uint32_t p = 0; p < n; ++p) {
    out.parts.emplace_back(t.universe(),
                           std::vector<uint64_t>(hi.begin() + off, hi.begin() + off + pc[p]),
                           std::vector<float>(hv.begin() + off, hv.begin() + off + pc[p]));
    off += pc[p];
  }
  CollisionStats cs;
  cs.serial_writes = st.serial_writes;
  cs.placed_at_depth.assign(st.placed_at_depth, st.placed_at_depth + st.k);
  return {std::move(out), std::move(cs)};
}
}  // namespace detail

inline PartitionedSparseTensor hierarchical_hash(const SparseTensor& t, uint32_t n,
                                                 const HashFamily& family, uint64_t r1,
                                                 uint64_t r2, uint32_t lanes = 1) {
  return detail::run_hierarchical_hash(t, n, family, r1, r2, lanes).first;
}

inline CollisionStats collision_stats(const SparseTensor& t, uint32_t n, const HashFamily& family,
                                      uint64_t r1, uint64_t r2) {
  return detail::run_hierarchical_hash(t, n, family, r1, r2, 1).second;
}

// zen::strawman_hash (hashing.hpp:266-291): the paper's single-hash,
// last-writer-wins strawman, kept as a baseline only (it loses data by
// design).  Host arithmetic: the winner of a cell is the largest index that
// maps to it, because the reference writes the cells in ascending index order.
inline std::pair<PartitionedSparseTensor, uint64_t> strawman_hash(const SparseTensor& t,
                                                                  uint32_t n, uint64_t r,
                                                                  uint64_t seed) {
  if (n == 0 || r == 0) throw Error("strawman hash needs n >= 1 and r >= 1");
  const uint64_t cells = uint64_t(n) * r;
  const uint64_t hs = zen_derive_seed(seed, 77);
  std::vector<int64_t> owner(cells, -1);
  const auto& idx = t.indices();
  for (size_t i = 0; i < idx.size(); ++i)
    owner[zen_map_to_range(zen_seeded_hash(idx[i] + 1, hs), cells)] = int64_t(i);
  PartitionedSparseTensor out;
  uint64_t kept = 0;
  for (uint32_t p = 0; p < n; ++p) {
    std::vector<std::pair<uint64_t, float>> cell;
    for (uint64_t c = uint64_t(p) * r; c < uint64_t(p + 1) * r; ++c)
      if (owner[c] >= 0) cell.emplace_back(idx[size_t(owner[c])], t.values()[size_t(owner[c])]);
    kept += cell.size();
    out.parts.push_back(SparseTensor::from_pairs(t.universe(), std::move(cell)));
  }
  return {std::move(out), t.nnz() - kept};
}

inline double imbalance_push(const std::vector<PartitionedSparseTensor>& per_worker) {
  if (per_worker.empty()) throw Error("imbalance requires at least one worker");
  double worst = 0.0;
  for (const auto& w : per_worker) {
    const uint64_t total = w.total_nnz();
    if (total == 0) throw EmptyTensor("imbalance undefined for a worker with no gradients");
    const double n = double(w.parts.size());
    for (const auto& p : w.parts) worst = std::max(worst, n * double(p.nnz()) / double(total));
  }
  return worst;
}

inline double imbalance_pull(const std::vector<uint64_t>& loads, uint64_t union_size) {
  if (loads.empty()) throw Error("imbalance requires at least one server");
  if (union_size == 0) throw EmptyTensor("imbalance undefined for an empty union");
  const double n = double(loads.size());
  double worst = 0.0;
  for (auto l : loads) worst = std::max(worst, n * double(l) / double(union_size));
  return worst;
}

// ---- codec: zen/codec.hpp ---------------------------------------------------
enum class WireKind : uint8_t { Coo = 1, Bitmap = 2, TensorBlock = 3, HashBitmap = 4 };
struct WireFormat {  // codec.hpp:21-35
  WireKind kind = WireKind::Coo;
  uint32_t block_size = 256;
  uint32_t coo_index_bits = 64;
  static WireFormat coo(uint32_t index_bits = 64) {
    if (index_bits != 32 && index_bits != 64) throw Error("COO index width must be 32 or 64");
    return {WireKind::Coo, 256, index_bits};
  }
  static WireFormat bitmap() { return {WireKind::Bitmap, 256, 64}; }
  static WireFormat tensor_block(uint32_t block_size = 256) {
    if (block_size < 1) throw Error("tensor block size must be at least 1");
    return {WireKind::TensorBlock, block_size, 64};
  }
  static WireFormat hash_bitmap() { return {WireKind::HashBitmap, 256, 64}; }
};

struct EncodedMessage {
  WireFormat format;
  uint64_t universe_size = 0;
  uint64_t count = 0;
  uint64_t index_bits = 0;
  uint64_t value_bits = 0;
  std::vector<uint8_t> payload;
  uint64_t payload_bits() const { return index_bits + value_bits; }
};

class HashUniverseTable;
// Reads like the reference's `std::vector<uint64_t> indices` member
// (codec.hpp:38-42): the server's sorted universe, materialised from the
// device tables on first use (they never build the M x 8 B lists).
struct HashUniverseIndices {
  const HashUniverseTable* table = nullptr;
  uint32_t server = 0;
  mutable std::shared_ptr<std::vector<uint64_t>> cache{};
  const std::vector<uint64_t>& get() const;
  operator const std::vector<uint64_t>&() const { return get(); }
  size_t size() const { return get().size(); }
  bool empty() const { return get().empty(); }
  uint64_t operator[](size_t i) const { return get()[i]; }
  uint64_t front() const { return get().front(); }
  uint64_t back() const { return get().back(); }
  std::vector<uint64_t>::const_iterator begin() const { return get().begin(); }
  std::vector<uint64_t>::const_iterator end() const { return get().end(); }
};

struct HashUniverse {
  uint32_t server_id = 0;
  uint64_t universe_size = 0;
  const HashUniverseTable* table = nullptr;
  HashUniverseIndices indices{};
  std::vector<uint64_t> indices_copy() const;
};

class HashUniverseTable {
 public:
  HashUniverseTable(uint64_t universe_size, uint32_t servers, uint64_t partition_seed)
      : m_(universe_size), n_(servers), pseed_(partition_seed) {
    if (servers == 0) throw Error("hash universe table needs at least one server");
    zen_universe* u = nullptr;
    detail::check(zen_universe_create(detail::ctx(), m_, n_, pseed_, &u));
    u_.reset(u);
    for (uint32_t s = 0; s < n_; ++s)
      us_.push_back(HashUniverse{s, m_, this, HashUniverseIndices{this, s}});
  }
  uint64_t universe_size() const { return m_; }
  uint32_t servers() const { return n_; }
  uint64_t partition_seed() const { return pseed_; }
  const HashUniverse& universe(uint32_t s) const { return us_.at(s); }
  uint64_t size(uint32_t s) const { return zen_universe_size(u_.get(), s); }
  zen_universe* handle() const { return u_.get(); }

 private:
  struct Del {
    void operator()(zen_universe* u) const { zen_universe_destroy(u); }
  };
  uint64_t m_;
  uint32_t n_;
  uint64_t pseed_;
  std::unique_ptr<zen_universe, Del> u_;
  std::vector<HashUniverse> us_;
};

inline const std::vector<uint64_t>& HashUniverseIndices::get() const {
  if (!cache) cache = std::make_shared<std::vector<uint64_t>>(table->universe(server).indices_copy());
  return *cache;
}

inline std::vector<uint64_t> HashUniverse::indices_copy() const {
  const uint64_t sz = table->size(server_id);
  detail::DBuf<uint64_t> d(sz);
  detail::check(zen_universe_indices(table->handle(), server_id, d.p));
  return d.host(sz);
}

inline HashUniverseTable bp_universe_table(uint64_t universe_size, uint32_t servers,
                                           uint64_t seed) {
  return HashUniverseTable(universe_size, servers, zen_derive_seed(seed, 0));
}

namespace detail {
inline zen_wire_format wire_c(const WireFormat& f) {
  return zen_wire_format{uint32_t(f.kind), f.block_size, f.coo_index_bits};
}
inline zen_universe* universe_handle(const WireFormat& f, const HashUniverse* u,
                                     uint32_t* server) {
  if (f.kind != WireKind::HashBitmap) return nullptr;
  *server = u->server_id;
  return u->table->handle();
}
}  // namespace detail

// encode(t, fmt, universe) -- codec.hpp:213-278, every WireKind, on the GPU
inline EncodedMessage encode(const SparseTensor& t, const WireFormat& fmt,
                             const HashUniverse* universe = nullptr) {
  if (fmt.kind == WireKind::HashBitmap && universe == nullptr)
    throw Error("hash bitmap requires a hash universe");
  uint32_t s = 0;
  zen_universe* u = detail::universe_handle(fmt, universe, &s);
  const zen_wire_format f = detail::wire_c(fmt);
  detail::DBuf<uint64_t> di(t.indices());
  detail::DBuf<float> dv(t.values());
  zen_message_info info{};
  const zen_status rc = zen_encode(detail::ctx(), &f, u, s, di.p, dv.p, t.nnz(), t.universe(),
                                   nullptr, 0, &info);
  if (rc != ZEN_OK && rc != ZEN_E_CAPACITY) detail::check(rc);
  detail::DBuf<uint8_t> dp(info.payload_bytes);
  detail::check(zen_encode(detail::ctx(), &f, u, s, di.p, dv.p, t.nnz(), t.universe(), dp.p,
                           info.payload_bytes, &info));
  EncodedMessage msg;
  msg.format = fmt;
  msg.universe_size = t.universe();
  msg.count = info.count;
  msg.index_bits = info.index_bits;
  msg.value_bits = info.value_bits;
  msg.payload = dp.host(info.payload_bytes);
  return msg;
}

// message_sizes(t, fmt, universe) -- codec.hpp:92-96, 182-211
struct MessageSizes {
  uint64_t index_bits = 0;
  uint64_t value_bits = 0;
  uint64_t payload_bits() const { return index_bits + value_bits; }
};
inline MessageSizes message_sizes(const SparseTensor& t, const WireFormat& fmt,
                                  const HashUniverse* universe = nullptr) {
  const auto m = encode(t, fmt, universe);
  return {m.index_bits, m.value_bits};
}

// decode(msg, universe) -- codec.hpp:282-347, every WireKind, on the GPU
inline SparseTensor decode(const EncodedMessage& msg, const HashUniverse* universe = nullptr) {
  if (msg.format.kind == WireKind::HashBitmap && universe == nullptr)
    throw Error("hash bitmap requires the encoding universe");
  uint32_t s = 0;
  zen_universe* u = detail::universe_handle(msg.format, universe, &s);
  const zen_wire_format f = detail::wire_c(msg.format);
  const uint64_t cap =
      msg.count * (msg.format.kind == WireKind::TensorBlock ? msg.format.block_size : 1);
  detail::DBuf<uint8_t> dp(msg.payload);
  detail::DBuf<uint64_t> oi(cap);
  detail::DBuf<float> ov(cap);
  zen_message_info info{msg.universe_size, msg.count, msg.index_bits, msg.value_bits,
                        msg.payload.size()};
  uint64_t got = 0;
  detail::check(zen_decode(detail::ctx(), &f, u, s, &info, dp.p, oi.p, ov.p, cap, &got));
  return SparseTensor(msg.universe_size, oi.host(got), ov.host(got));
}

// write_framed / read_framed -- codec.hpp:352-410
inline void write_framed(std::ostream& os, const EncodedMessage& msg) {
  if (msg.payload.empty() && msg.payload_bits() != 0)
    throw Error("cannot frame a message without payload");
  const zen_wire_format f = detail::wire_c(msg.format);
  zen_message_info info{msg.universe_size, msg.count, msg.index_bits, msg.value_bits,
                        msg.payload.size()};
  uint8_t hdr[ZEN_FRAME_HEADER_BYTES];
  detail::check(zen_frame_header(&f, &info, hdr));
  os.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  os.write(reinterpret_cast<const char*>(msg.payload.data()),
           static_cast<std::streamsize>(msg.payload.size()));
}

inline EncodedMessage read_framed(std::istream& is) {
  uint8_t hdr[ZEN_FRAME_HEADER_BYTES];
  is.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  if (!is) throw MalformedPayload("unexpected end of stream");
  zen_wire_format f{};
  zen_message_info info{};
  detail::check(zen_frame_parse(hdr, ~uint64_t(0), &f, &info));  // header only
  EncodedMessage msg;
  msg.format = WireFormat{WireKind(f.kind), f.block_size, f.coo_index_bits};
  msg.universe_size = info.universe_size;
  msg.count = info.count;
  msg.index_bits = info.index_bits;
  msg.value_bits = info.value_bits;
  msg.payload.resize(info.payload_bytes);
  is.read(reinterpret_cast<char*>(msg.payload.data()),
          static_cast<std::streamsize>(msg.payload.size()));
  if (!is) throw MalformedPayload("frame payload truncated");
  return msg;
}

// .zspt -- tensor.hpp:239-303 (host byte layout, little-endian)
namespace detail {
template <typename T>
inline void write_le(std::ostream& os, T v) {
  unsigned char b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  os.write(reinterpret_cast<const char*>(b), sizeof(T));
}
template <typename T>
inline T read_le(std::istream& is) {
  unsigned char b[sizeof(T)];
  is.read(reinterpret_cast<char*>(b), sizeof(T));
  if (!is) throw MalformedPayload("unexpected end of stream");
  T v;
  std::memcpy(&v, b, sizeof(T));
  return v;
}
}  // namespace detail

inline void write_sparse(std::ostream& os, const SparseTensor& t) {
  os.write("ZSPT", 4);
  detail::write_le<uint32_t>(os, 1);
  detail::write_le<uint64_t>(os, t.universe());
  detail::write_le<uint64_t>(os, t.nnz());
  for (uint64_t i : t.indices()) detail::write_le<uint64_t>(os, i);
  for (float v : t.values()) detail::write_le<float>(os, v);
}

inline SparseTensor read_sparse(std::istream& is) {
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "ZSPT", 4) != 0) throw MalformedPayload("bad sparse tensor magic");
  if (detail::read_le<uint32_t>(is) != 1) throw MalformedPayload("unsupported sparse tensor version");
  const uint64_t m = detail::read_le<uint64_t>(is);
  const uint64_t count = detail::read_le<uint64_t>(is);
  std::vector<uint64_t> idx(count);
  for (auto& i : idx) i = detail::read_le<uint64_t>(is);
  std::vector<float> val(count);
  for (auto& v : val) v = detail::read_le<float>(is);
  return SparseTensor(m, std::move(idx), std::move(val));
}

inline void write_sparse_file(const std::string& path, const SparseTensor& t) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw Error("cannot open " + path + " for writing");
  write_sparse(os, t);
}

inline SparseTensor read_sparse_file(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw Error("cannot open " + path);
  return read_sparse(is);
}

// ---- merge_sum and the sparsity metrics: zen/tensor.hpp:106-213 ------------
namespace detail {
struct DevTensor {  // a device copy of a SparseTensor (or of a merge result)
  uint64_t m = 1, n = 0;
  std::unique_ptr<DBuf<uint64_t>> idx;
  std::unique_ptr<DBuf<float>> val;
  DevTensor() = default;
  explicit DevTensor(const SparseTensor& t)
      : m(t.universe()), n(t.nnz()), idx(new DBuf<uint64_t>(t.indices())),
        val(new DBuf<float>(t.values())) {}
  SparseTensor host() const { return SparseTensor(m, idx->host(n), val->host(n)); }
};
inline DevTensor merge_dev(const DevTensor& a, const DevTensor& b) {
  if (a.m != b.m) throw UniverseMismatch();
  DevTensor o;
  o.m = a.m;
  o.idx.reset(new DBuf<uint64_t>(a.n + b.n));
  o.val.reset(new DBuf<float>(a.n + b.n));
  check(zen_merge_sum(ctx(), a.idx->p, a.val->p, a.n, b.idx->p, b.val->p, b.n, a.m, o.idx->p,
                      o.val->p, a.n + b.n, &o.n));
  return o;
}
inline bool is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }
}  // namespace detail

// zen::merge_sum (tensor.hpp:133-167), the merge-path kernel on the GPU
inline SparseTensor merge_sum(const SparseTensor& a, const SparseTensor& b) {
  if (a.universe() != b.universe()) throw UniverseMismatch();
  return detail::merge_dev(detail::DevTensor(a), detail::DevTensor(b)).host();
}

// zen::aggregate (tensor.hpp:171-176)
inline SparseTensor aggregate(const std::vector<SparseTensor>& tensors) {
  if (tensors.empty()) throw Error("aggregate requires at least one tensor");
  detail::DevTensor acc(tensors.front());
  for (size_t i = 1; i < tensors.size(); ++i) acc = detail::merge_dev(acc, detail::DevTensor(tensors[i]));
  return acc.host();
}

inline double density(const SparseTensor& t) { return double(t.nnz()) / double(t.universe()); }

inline double overlap_ratio(const SparseTensor& a, const SparseTensor& b) {  // tensor.hpp:111-130
  if (a.universe() != b.universe()) throw UniverseMismatch();
  if (a.empty() || b.empty()) throw EmptyTensor("overlap ratio undefined for empty tensors");
  const auto u = detail::merge_dev(detail::DevTensor(a), detail::DevTensor(b));
  return double(a.nnz() + b.nnz() - u.n) / double(std::min(a.nnz(), b.nnz()));
}

inline double densification_ratio(const std::vector<SparseTensor>& tensors) {  // :178-189
  if (tensors.empty()) throw Error("densification ratio requires at least one tensor");
  double mean_d = 0.0;
  for (const auto& t : tensors) {
    if (t.empty()) throw EmptyTensor("densification ratio undefined with an empty tensor");
    mean_d += density(t);
  }
  mean_d /= double(tensors.size());
  detail::DevTensor acc(tensors.front());
  for (size_t i = 1; i < tensors.size(); ++i) acc = detail::merge_dev(acc, detail::DevTensor(tensors[i]));
  return (double(acc.n) / double(tensors.front().universe())) / mean_d;
}

namespace detail {
inline double skew_from_counts(const std::vector<uint64_t>& counts, uint64_t m, uint32_t parts,
                               uint64_t nnz) {
  const uint64_t range = (m + parts - 1) / parts;
  double best = 0.0;
  for (uint64_t p = 0; p < parts; ++p) {
    const uint64_t lo = p * range;
    if (lo >= m) break;
    const uint64_t hi = std::min(m, lo + range);
    best = std::max(best, double(counts[p]) / double(hi - lo));
  }
  return best / (double(nnz) / double(m));
}
inline std::vector<uint64_t> range_counts(const DevTensor& t, uint32_t parts) {
  std::vector<uint64_t> c(parts);
  check(zen_range_counts(ctx(), t.idx->p, t.n, t.m, parts, c.data()));
  return c;
}
}  // namespace detail

inline double skewness_ratio(const SparseTensor& t, uint32_t partitions) {  // :192-213
  if (partitions == 0) throw Error("skewness ratio requires at least one partition");
  if (t.empty()) throw EmptyTensor("skewness ratio undefined for an empty tensor");
  return detail::skew_from_counts(detail::range_counts(detail::DevTensor(t), partitions),
                                  t.universe(), partitions, t.nnz());
}

// ---- synthetic workloads: zen/workload.hpp ----------------------------------
struct WorkloadSpec {  // workload.hpp:22-51
  uint64_t universe = 0;
  uint32_t nodes = 1;
  double density = 0.0;
  double omega = 0.0;
  double hot_fraction = 0.125;
  double hot_mass = 0.125;
  uint64_t seed = 0;
  uint64_t nnz_per_node() const { return uint64_t(std::ceil(density * double(universe))); }
  zen_workload_spec c() const {
    return zen_workload_spec{universe, nodes, density, omega, hot_fraction, hot_mass, seed};
  }
  void validate() const {  // the device generator applies the same checks
    if (universe < 1) throw InfeasibleSpec("universe must be at least 1");
    if (nodes < 1) throw InfeasibleSpec("node count must be at least 1");
    if (!(density > 0.0 && density <= 1.0)) throw InfeasibleSpec("density must be in (0,1]");
    if (density * double(universe) < 1.0) throw InfeasibleSpec("density*universe must be at least 1");
    if (omega < 0.0 || omega > 1.0) throw InfeasibleSpec("omega must be in [0,1]");
    if (!(hot_fraction > 0.0 && hot_fraction <= 1.0)) throw InfeasibleSpec("hot_fraction must be in (0,1]");
    if (hot_mass < 0.0 || hot_mass > 1.0) throw InfeasibleSpec("hot_mass must be in [0,1]");
    if (density * double(universe) * (1.0 + double(nodes) * (1.0 - omega)) > double(universe))
      throw InfeasibleSpec("cannot fit disjoint remainders: d*M*(1+n*(1-omega)) > M");
  }
};

// zen::generate (workload.hpp:119-154) drawn on the device (zen_generate):
// the shared core + two-tier draws without replacement, integer values.
// Same spec as the reference, not the same bits (counter-based hashes instead
// of std::mt19937_64); deterministic for a seed.
inline std::vector<SparseTensor> generate(const WorkloadSpec& spec) {
  spec.validate();
  const uint64_t z = spec.nnz_per_node();
  detail::DBuf<uint64_t> di(std::max<uint64_t>(z, 1));
  detail::DBuf<float> dv(std::max<uint64_t>(z, 1));
  const zen_workload_spec c = spec.c();
  std::vector<SparseTensor> out;
  for (uint32_t node = 0; node < spec.nodes; ++node) {
    uint64_t got = 0;
    detail::check(zen_generate(detail::ctx(), &c, node, di.p, dv.p, z, &got));
    out.push_back(SparseTensor(spec.universe, di.host(got), dv.host(got)));
  }
  return out;
}

struct WorkloadMeasurement {  // workload.hpp:180-184
  double mean_pairwise_overlap = 0.0;
  std::map<uint64_t, double> gamma;
  std::map<uint32_t, double> skew;
};

// workload.hpp:189-221: mean pairwise overlap, densification over prefixes,
// mean skewness at power-of-two partition counts (each a device operator)
inline WorkloadMeasurement measure(const std::vector<SparseTensor>& tensors) {
  if (tensors.size() < 2) throw Error("measurement requires at least two tensors");
  for (const auto& t : tensors)
    if (t.empty()) throw EmptyTensor("measurement undefined with empty tensors");
  WorkloadMeasurement out;
  double pairs = 0.0;
  uint64_t np = 0;
  for (size_t i = 0; i < tensors.size(); ++i)
    for (size_t j = i + 1; j < tensors.size(); ++j, ++np) pairs += overlap_ratio(tensors[i], tensors[j]);
  out.mean_pairwise_overlap = pairs / double(np);
  SparseTensor acc = tensors.front();
  double dsum = density(acc);
  out.gamma[1] = 1.0;
  for (size_t k = 2; k <= tensors.size(); ++k) {
    acc = merge_sum(acc, tensors[k - 1]);
    dsum += density(tensors[k - 1]);
    out.gamma[k] = density(acc) / (dsum / double(k));
  }
  for (uint32_t parts = 1; parts <= tensors.size(); parts *= 2) {
    double sk = 0.0;
    for (const auto& t : tensors) sk += skewness_ratio(t, parts);
    out.skew[parts] = sk / double(tensors.size());
  }
  return out;
}

// ---- sparsity profile and scheme selection: zen/costmodel.hpp ---------------
struct SparsityProfile {  // tensor.hpp:216-240
  double d = 0.0;
  std::map<uint64_t, double> gamma;
  std::map<uint32_t, double> skew;
  // the profile's invariants (tensor.hpp:221-238): d in (0,1], gamma[1] = 1,
  // gamma non-decreasing with gamma[k] <= k and d*gamma[k] <= 1, skew >= 1
  void validate() const {
    if (!(d > 0.0 && d <= 1.0)) throw Error("profile density must be in (0,1]");
    auto one = gamma.find(1);
    if (one == gamma.end() || one->second != 1.0) throw Error("profile gamma[1] must equal 1");
    double last = 0.0;
    for (const auto& kv : gamma) {
      if (kv.second < last - 1e-9) throw Error("profile gamma must be non-decreasing in k");
      if (kv.second > double(kv.first) + 1e-9) throw Error("profile gamma[k] must not exceed k");
      if (d * kv.second > 1.0 + 1e-9) throw Error("profile d*gamma[k] must not exceed 1");
      last = kv.second;
    }
    for (const auto& kv : skew)
      if (kv.second < 1.0 - 1e-9) throw Error("profile skewness must be at least 1");
  }
};

// (n-1)/n * (gamma_n + 1), costmodel.hpp:53-58
inline double t_bp_coefficient(uint32_t n, double gamma_n) {
  return n <= 1 ? 0.0 : (double(n) - 1.0) / double(n) * (gamma_n + 1.0);
}
// sum over log n stages of gamma at 2^(i-1), costmodel.hpp:62-77
inline double t_hc_coefficient(uint32_t n, const std::map<uint64_t, double>& gamma) {
  if (!detail::is_pow2(n)) throw NonPowerOfTwo("hierarchy requires a power-of-two n");
  double sum = 0.0;
  for (uint64_t k = 1; k < n; k *= 2) {
    if (k == 1) {
      sum += 1.0;
      continue;
    }
    auto it = gamma.find(k);
    if (it == gamma.end())
      throw MissingProfileEntry("densification ratio for k=" + std::to_string(k) +
                                " missing from profile");
    sum += it->second;
  }
  return sum;
}

// ---- closed-form communication times (costmodel.hpp:14-128), element units --
struct CostInputs {
  uint32_t n = 1;
  double universe = 0.0;  // M
  double d = 0.0;
  double b = 1.0;  // elements per time unit
  std::map<uint64_t, double> gamma;
  double skew = 1.0;
  double broadcast_rounds = 1.0;
};
namespace detail {
inline double gamma_of(const CostInputs& c, uint64_t k) {
  if (k == 1) return 1.0;
  auto it = c.gamma.find(k);
  if (it == c.gamma.end())
    throw MissingProfileEntry("densification ratio for k=" + std::to_string(k) + " missing from profile");
  return it->second;
}
}  // namespace detail
inline double t_bp(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  return t_bp_coefficient(c.n, detail::gamma_of(c, c.n)) * 2.0 * c.universe * c.d / c.b;
}
inline double t_hc(const CostInputs& c) {
  return t_hc_coefficient(c.n, c.gamma) * 2.0 * c.universe * c.d / c.b;
}
inline double t_sparse_ps(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  const double g = detail::gamma_of(c, c.n);
  return 2.0 * (double(c.n) - 1.0) * (1.0 + g) * c.skew * c.d * c.universe / double(c.n) / c.b;
}
inline double t_sparse_ps_broadcast(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  const double g = detail::gamma_of(c, c.n);
  return 2.0 * (double(c.n) - 1.0) * c.skew * c.d * c.universe / double(c.n) / c.b +
         2.0 * c.broadcast_rounds * g * c.d * c.universe / c.b;
}
inline double t_ring_incremental(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  double sum = 0.0;
  for (uint64_t k = 1; k < c.n; ++k) sum += detail::gamma_of(c, k);
  return 2.0 * sum * c.d * c.universe / double(c.n) / c.b;
}
inline double t_hierarchy_incremental_lb(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  return 2.0 * (double(c.n) - 1.0) * c.d * c.universe / double(c.n) / c.b;
}
inline double t_allreduce_dense(const CostInputs& c) {
  if (c.n <= 1) return 0.0;
  return 2.0 * (double(c.n) - 1.0) / double(c.n) * c.universe / c.b;
}
// experiment.hpp:161-169: the dense all-reduce baseline in bit units
inline double allreduce_dense_time_bits(uint32_t n, uint64_t universe, double bandwidth) {
  CostInputs c;
  c.n = n;
  c.universe = double(universe);
  c.d = 1.0;
  c.b = bandwidth / 32.0;
  c.gamma[1] = 1.0;
  return t_allreduce_dense(c);
}

enum class SchemeChoice { BalancedParallelism, HierarchicalCentralization };
inline const char* to_string(SchemeChoice s) {
  return s == SchemeChoice::BalancedParallelism ? "balanced-parallelism"
                                                : "hierarchical-centralization";
}

// zen::select_scheme (costmodel.hpp:139-149): ties go to Balanced Parallelism
inline SchemeChoice select_scheme(const SparsityProfile& p, uint32_t n) {
  auto it = p.gamma.find(n);
  if (it == p.gamma.end())
    throw MissingProfileEntry("densification ratio for k=" + std::to_string(n) +
                              " missing from profile");
  return t_bp_coefficient(n, it->second) <= t_hc_coefficient(n, p.gamma)
             ? SchemeChoice::BalancedParallelism
             : SchemeChoice::HierarchicalCentralization;
}

// zen::profile_sparsity (costmodel.hpp:151-195); prefix unions by device merges
inline SparsityProfile profile_sparsity(const std::vector<std::vector<SparseTensor>>& rounds) {
  if (rounds.empty()) throw Error("profiling requires at least one round");
  const size_t n = rounds.front().size();
  if (n == 0) throw Error("profiling requires at least one tensor per round");
  SparsityProfile prof;
  std::map<uint64_t, double> gamma_sums;
  double skew_sum = 0.0, density_sum = 0.0;
  uint64_t density_count = 0;
  for (const auto& round : rounds) {
    if (round.size() != n) throw Error("profiling rounds must have matching node counts");
    double prefix_density_sum = 0.0;
    detail::DevTensor prefix;
    for (size_t i = 0; i < n; ++i) {
      const SparseTensor& t = round[i];
      if (t.empty()) throw EmptyTensor("profiling requires non-empty tensors");
      density_sum += density(t);
      ++density_count;
      detail::DevTensor dt(t);
      skew_sum += detail::skew_from_counts(detail::range_counts(dt, uint32_t(n)), t.universe(),
                                           uint32_t(n), t.nnz());
      prefix = i == 0 ? std::move(dt) : detail::merge_dev(prefix, dt);
      prefix_density_sum += density(t);
      const uint64_t k = i + 1;
      if (detail::is_pow2(k))
        gamma_sums[k] += (double(prefix.n) / double(t.universe())) /
                         (prefix_density_sum / double(k));
    }
  }
  prof.d = density_sum / double(density_count);
  for (const auto& [k, sum] : gamma_sums) prof.gamma[k] = sum / double(rounds.size());
  prof.gamma[1] = 1.0;
  prof.skew[uint32_t(n)] = skew_sum / double(rounds.size() * n);
  return prof;
}

#ifdef NLOHMANN_JSON_VERSION_MAJOR
// the profile document (costmodel.hpp:191-219), when nlohmann/json is included
inline nlohmann::json profile_to_json(const SparsityProfile& p) {
  nlohmann::json j;
  j["d"] = p.d;
  j["gamma"] = nlohmann::json::object();
  for (const auto& kv : p.gamma) j["gamma"][std::to_string(kv.first)] = kv.second;
  j["skew"] = nlohmann::json::object();
  for (const auto& kv : p.skew) j["skew"][std::to_string(kv.first)] = kv.second;
  return j;
}
inline SparsityProfile profile_from_json(const nlohmann::json& j) {
  SparsityProfile p;
  if (!j.contains("d") || !j["d"].is_number()) throw MissingProfileEntry("profile json lacks a numeric 'd'");
  p.d = j["d"].get<double>();
  if (!j.contains("gamma") || !j["gamma"].is_object())
    throw MissingProfileEntry("profile json lacks a 'gamma' object");
  for (const auto& it : j["gamma"].items()) {
    if (!it.value().is_number()) throw MissingProfileEntry("gamma entries must be numeric");
    p.gamma[std::stoull(it.key())] = it.value().get<double>();
  }
  if (j.contains("skew"))
    for (const auto& it : j["skew"].items()) p.skew[uint32_t(std::stoul(it.key()))] = it.value().get<double>();
  return p;
}
#endif

// ---- transport ledger: zen/simnet.hpp ---------------------------------------
struct StageRecord {
  std::vector<uint64_t> sent_bits, recv_bits, recv_index_bits, recv_value_bits;
  double stage_time = 0.0;
  explicit StageRecord(uint32_t n)
      : sent_bits(n, 0), recv_bits(n, 0), recv_index_bits(n, 0), recv_value_bits(n, 0) {}
};

struct TrafficReport {
  uint32_t nodes = 0;
  double bandwidth = 0.0;
  std::vector<StageRecord> stages;
  uint64_t total_sent_bits = 0, total_recv_bits = 0, total_index_bits = 0, total_value_bits = 0;
  double simulated_time = 0.0;
#ifdef NLOHMANN_JSON_VERSION_MAJOR
  // the reference's report document (simnet.hpp:37-55), when nlohmann/json is
  // included before this header (as the reference's own headers do)
  nlohmann::json to_json() const {
    nlohmann::json j;
    j["n"] = nodes;
    j["b"] = bandwidth;
    j["stages"] = nlohmann::json::array();
    for (const auto& st : stages)
      j["stages"].push_back({{"time", st.stage_time}, {"sent_bits", st.sent_bits},
                             {"recv_bits", st.recv_bits}, {"recv_index_bits", st.recv_index_bits},
                             {"recv_value_bits", st.recv_value_bits}});
    j["totals"] = {{"sent_bits", total_sent_bits}, {"recv_bits", total_recv_bits},
                   {"index_bits", total_index_bits}, {"value_bits", total_value_bits}};
    j["simulated_time"] = simulated_time;
    return j;
  }
#endif
};

// value-payload time in COO-equivalent fp32 element units (simnet.hpp:125-134):
// per stage the largest received value payload, two elements per value
inline double value_payload_time_coo_equivalent(const TrafficReport& r) {
  double elems = 0.0;
  for (const auto& st : r.stages) {
    uint64_t mx = 0;
    for (uint64_t v : st.recv_value_bits) mx = std::max(mx, v);
    elems += double(mx) / 32.0 * 2.0;
  }
  return elems / (r.bandwidth / 32.0);
}

// The reference's accounting network.  On B200 the bytes really move over
// NVLink; this keeps the deterministic bit ledger (stage time = max recv / b).
class SimNet {
 public:
  SimNet(uint32_t nodes, double bandwidth, double latency = 0.0)
      : n_(nodes), b_(bandwidth), lat_(latency) {
    if (nodes == 0) throw Error("network needs at least one node");
    if (bandwidth <= 0.0) throw Error("bandwidth must be positive");
  }
  uint32_t nodes() const { return n_; }
  double bandwidth() const { return b_; }
  // simnet.hpp:71-85
  void send(uint32_t stage, uint32_t from, uint32_t to, const EncodedMessage& msg) {
    if (final_) throw Error("cannot send after finalize");
    if (from == to) throw SelfSend();
    if (from >= n_ || to >= n_) throw Error("node id out of range");
    if (!stages_.empty() && stage + 1 < stages_.size())
      throw Error("stage numbers must be non-decreasing");
    while (stages_.size() <= stage) stages_.emplace_back(n_);
    StageRecord& r = stages_[stage];
    r.sent_bits[from] += msg.payload_bits();
    r.recv_bits[to] += msg.payload_bits();
    r.recv_index_bits[to] += msg.index_bits;
    r.recv_value_bits[to] += msg.value_bits;
    lat_charges_ += lat_;
  }
  // ledger[2][4][n] as produced by zen_bp_traffic
  void record(const std::vector<uint64_t>& ledger, uint64_t messages) {
    if (final_) throw Error("cannot send after finalize");
    for (uint32_t st = 0; st < 2; ++st) {
      while (stages_.size() <= st) stages_.emplace_back(n_);
      for (uint32_t v = 0; v < n_; ++v) {
        stages_[st].sent_bits[v] += ledger[(st * 4 + 0) * n_ + v];
        stages_[st].recv_bits[v] += ledger[(st * 4 + 1) * n_ + v];
        stages_[st].recv_index_bits[v] += ledger[(st * 4 + 2) * n_ + v];
        stages_[st].recv_value_bits[v] += ledger[(st * 4 + 3) * n_ + v];
      }
    }
    lat_charges_ += lat_ * double(messages);
  }
  TrafficReport finalize() {  // simnet.hpp:87-111
    if (final_) throw Error("network already finalized");
    final_ = true;
    TrafficReport r;
    r.nodes = n_;
    r.bandwidth = b_;
    r.stages = std::move(stages_);
    for (auto& s : r.stages) {
      uint64_t sent = 0, recv = 0, mx = 0;
      for (uint32_t v = 0; v < n_; ++v) {
        sent += s.sent_bits[v];
        recv += s.recv_bits[v];
        mx = std::max(mx, s.recv_bits[v]);
        r.total_index_bits += s.recv_index_bits[v];
        r.total_value_bits += s.recv_value_bits[v];
      }
      if (sent != recv) throw UnbalancedLedger();
      s.stage_time = double(mx) / b_;
      r.total_sent_bits += sent;
      r.total_recv_bits += recv;
      r.simulated_time += s.stage_time;
    }
    r.simulated_time += lat_charges_;
    return r;
  }

 private:
  uint32_t n_;
  double b_, lat_, lat_charges_ = 0.0;
  bool final_ = false;
  std::vector<StageRecord> stages_;
};

// ---- Balanced Parallelism: zen/schemes.hpp:330-417 --------------------------
struct HashParams {
  uint32_t rehash_depth = 3;
  double r1_multiplier = 2.0;
  double r2_ratio = 0.1;
  uint32_t lanes = 1;
  uint64_t seed = 1;
};

struct BalanceDetails {
  double push_imbalance = 1.0;
  double pull_imbalance = 1.0;
};

struct SyncOutcome {
  std::vector<SparseTensor> results;
  TrafficReport traffic;
  std::optional<BalanceDetails> balance;
};

inline SyncOutcome run_balanced_parallelism(const std::vector<SparseTensor>& inputs, SimNet& net,
                                            const HashParams& params = {},
                                            const HashUniverseTable* table = nullptr) {
  if (inputs.size() < 2) throw Error("synchronization needs at least two nodes");
  if (inputs.size() != net.nodes()) throw Error("input count must match the network size");
  for (const auto& t : inputs)
    if (t.universe() != inputs.front().universe()) throw UniverseMismatch();
  const uint32_t n = uint32_t(inputs.size());
  const uint64_t m = inputs.front().universe();
  if (table && (table->universe_size() != m || table->servers() != n ||
                table->partition_seed() != zen_derive_seed(params.seed, 0)))
    throw Error("hash universe table does not match this run");
  uint64_t cap = 1;
  for (const auto& t : inputs) cap = std::max<uint64_t>(cap, t.nnz());
  zen_hash_params hp{params.rehash_depth, params.r1_multiplier, params.r2_ratio, params.lanes,
                     params.seed};
  zen_bp* bp = nullptr;
  detail::check(zen_bp_create(detail::ctx(), n, ZEN_BP_LOCAL, m, cap, &hp, &bp));
  std::unique_ptr<zen_bp, void (*)(zen_bp*)> guard(bp, zen_bp_destroy);
  std::vector<std::unique_ptr<detail::DBuf<uint64_t>>> di;
  std::vector<std::unique_ptr<detail::DBuf<float>>> dv;
  std::vector<const uint64_t*> ip;
  std::vector<const float*> vp;
  std::vector<uint64_t> nnz;
  for (const auto& t : inputs) {
    di.emplace_back(new detail::DBuf<uint64_t>(t.indices()));
    dv.emplace_back(new detail::DBuf<float>(t.values()));
    ip.push_back(di.back()->p);
    vp.push_back(dv.back()->p);
    nnz.push_back(t.nnz());
  }
  detail::check(zen_bp_sync_sparse(bp, ip.data(), vp.data(), nnz.data()));
  detail::check(zen_bp_wait(bp));
  uint64_t count = 0;
  detail::check(zen_bp_result(bp, nullptr, nullptr, &count));
  detail::DBuf<uint64_t> oi(count);
  detail::DBuf<float> ov(count);
  detail::check(zen_bp_copy_result(bp, oi.p, ov.p, count, &count));
  SparseTensor result(m, oi.host(count), ov.host(count));
  std::vector<uint64_t> ledger(8 * n), counts(size_t(n) * n), agg(n);
  detail::check(zen_bp_traffic(bp, ledger.data(), counts.data(), agg.data()));
  uint64_t msgs = uint64_t(n) * (n - 1);  // pull: always sent (schemes.hpp:387-388)
  for (uint32_t w = 0; w < n; ++w)
    for (uint32_t s = 0; s < n; ++s) msgs += (s != w && counts[size_t(w) * n + s]) ? 1 : 0;
  net.record(ledger, msgs);
  SyncOutcome out;
  out.results.assign(n, result);
  out.traffic = net.finalize();
  double push = 0, pull = 0;
  int valid = 0;
  detail::check(zen_bp_balance(bp, &push, &pull, &valid));
  if (valid) out.balance = BalanceDetails{push, pull};
  return out;
}

// zen::run_bp_with_retry (experiment.hpp:128-140)
inline SyncOutcome run_bp_with_retry(const std::vector<SparseTensor>& inputs, double bandwidth,
                                     HashParams params, const HashUniverseTable* table = nullptr,
                                     int max_retries = 4) {
  for (int attempt = 0;; ++attempt) {
    SimNet net(uint32_t(inputs.size()), bandwidth);
    try {
      return run_balanced_parallelism(inputs, net, params, table);
    } catch (const SerialOverflow&) {
      if (attempt >= max_retries) throw;
      params.r2_ratio *= 2.0;
    }
  }
}

// zen::run_hier_centralization (zen/schemes.hpp:173-193): recursive doubling
// with a device merge_sum per node and stage; all n nodes on this GPU (the
// multi-GPU form is the zen_hc_* C-ABI, one process per GPU)
inline SyncOutcome run_hier_centralization(const std::vector<SparseTensor>& inputs, SimNet& net,
                                           WireFormat fmt = WireFormat::coo()) {
  if (inputs.size() < 2) throw Error("synchronization needs at least two nodes");
  if (inputs.size() != net.nodes()) throw Error("input count must match the network size");
  for (const auto& t : inputs)
    if (t.universe() != inputs.front().universe()) throw UniverseMismatch();
  if (!detail::is_pow2(inputs.size())) throw NonPowerOfTwo();
  const uint32_t n = uint32_t(inputs.size());
  std::vector<detail::DevTensor> states;
  for (const auto& t : inputs) states.emplace_back(t);
  for (uint32_t bit = 1; bit < n; bit <<= 1) {
    uint32_t stage = 0;
    while ((1u << stage) != bit) ++stage;
    for (uint32_t w = 0; w < n; ++w) {  // sized_message (schemes.hpp:78-88)
      const detail::DevTensor& st = states[w];
      EncodedMessage msg;
      msg.format = fmt;
      msg.universe_size = st.m;
      msg.count = st.n;
      msg.value_bits = 32 * st.n;  // message_sizes, codec.hpp:182-211
      if (fmt.kind == WireKind::Coo) {
        msg.index_bits = uint64_t(fmt.coo_index_bits) * st.n;
      } else if (fmt.kind == WireKind::Bitmap) {
        msg.index_bits = st.m;
      } else if (fmt.kind == WireKind::HashBitmap) {
        throw Error("hash bitmap requires a hash universe");
      } else {  // tensor blocks: the device encoder's size pass
        zen_wire_format f = detail::wire_c(fmt);
        zen_message_info info{};
        const zen_status rc = zen_encode(detail::ctx(), &f, nullptr, 0, st.idx->p, st.val->p,
                                         st.n, st.m, nullptr, 0, &info);
        if (rc != ZEN_OK && rc != ZEN_E_CAPACITY) detail::check(rc);
        msg.index_bits = info.index_bits;
        msg.value_bits = info.value_bits;
      }
      net.send(stage, w, w ^ bit, msg);
    }
    std::vector<detail::DevTensor> next;
    for (uint32_t w = 0; w < n; ++w) next.push_back(detail::merge_dev(states[w], states[w ^ bit]));
    states = std::move(next);
  }
  SyncOutcome out;
  for (const auto& st : states) out.results.push_back(st.host());
  out.traffic = net.finalize();
  return out;
}

// ---- the design space: zen/schemes.hpp:21-41, 119-168, 194-328, 418-470 -----
enum class CommPattern { Ring, Hierarchy, PointToPoint };
enum class Aggregation { Incremental, OneShot };
enum class PartitionPattern { Centralization, Parallelism };
enum class BalancePattern { Balanced, Imbalanced, NotApplicable };

struct SchemeConfig {
  CommPattern communication = CommPattern::PointToPoint;
  Aggregation aggregation = Aggregation::OneShot;
  PartitionPattern partition = PartitionPattern::Centralization;
  BalancePattern balance = BalancePattern::NotApplicable;
  WireFormat format = WireFormat::coo();
  void validate() const {
    const bool centralized = partition == PartitionPattern::Centralization;
    if (centralized != (balance == BalancePattern::NotApplicable))
      throw UnsupportedCombination(
          "the balance dimension applies exactly when the partition pattern is Parallelism");
  }
};

struct RunParams {
  HashParams hash;
};

namespace detail {
inline void check_scheme_inputs(const std::vector<SparseTensor>& inputs, const SimNet& net) {
  if (inputs.size() < 2) throw Error("synchronization needs at least two nodes");
  if (inputs.size() != net.nodes()) throw Error("input count must match the network size");
  for (const auto& t : inputs)
    if (t.universe() != inputs.front().universe()) throw UniverseMismatch();
}
// message_sizes of a device tensor (codec.hpp:182-211)
inline EncodedMessage sized(const DevTensor& t, const WireFormat& fmt) {
  EncodedMessage msg;
  msg.format = fmt;
  msg.universe_size = t.m;
  msg.count = t.n;
  msg.value_bits = 32 * t.n;
  if (fmt.kind == WireKind::Coo) {
    msg.index_bits = uint64_t(fmt.coo_index_bits) * t.n;
  } else if (fmt.kind == WireKind::Bitmap) {
    msg.index_bits = t.m;
  } else if (fmt.kind == WireKind::HashBitmap) {
    throw Error("hash bitmap requires a hash universe");
  } else {
    zen_wire_format f = wire_c(fmt);
    zen_message_info info{};
    const zen_status rc =
        zen_encode(ctx(), &f, nullptr, 0, t.idx->p, t.val->p, t.n, t.m, nullptr, 0, &info);
    if (rc != ZEN_OK && rc != ZEN_E_CAPACITY) check(rc);
    msg.count = info.count;
    msg.index_bits = info.index_bits;
    msg.value_bits = info.value_bits;
  }
  return msg;
}
inline DevTensor fold(const std::vector<const DevTensor*>& parts) {
  DevTensor acc = merge_dev(*parts[0], DevTensor(SparseTensor(parts[0]->m, {}, {})));
  for (size_t i = 1; i < parts.size(); ++i) acc = merge_dev(acc, *parts[i]);
  return acc;
}
inline DevTensor slice(const DevTensor& t, uint64_t at, uint64_t count) {
  DevTensor s;
  s.m = t.m;
  s.n = count;
  s.idx.reset(new DBuf<uint64_t>(count));
  s.val.reset(new DBuf<float>(count));
  if (count) {
    cudaMemcpy(s.idx->p, t.idx->p + at, count * 8, cudaMemcpyDeviceToDevice);
    cudaMemcpy(s.val->p, t.val->p + at, count * 4, cudaMemcpyDeviceToDevice);
  }
  return s;
}
}  // namespace detail

// zen::run_agsparse (schemes.hpp:119-168)
inline SyncOutcome run_agsparse(const std::vector<SparseTensor>& inputs, SimNet& net,
                                CommPattern pattern = CommPattern::PointToPoint,
                                WireFormat fmt = WireFormat::coo()) {
  detail::check_scheme_inputs(inputs, net);
  const uint32_t n = uint32_t(inputs.size());
  std::vector<detail::DevTensor> ins;
  for (const auto& t : inputs) ins.emplace_back(t);
  std::vector<EncodedMessage> msg;
  for (const auto& t : ins) msg.push_back(detail::sized(t, fmt));
  if (pattern == CommPattern::PointToPoint) {
    for (uint32_t w = 0; w < n; ++w)
      for (uint32_t to = 0; to < n; ++to)
        if (to != w) net.send(0, w, to, msg[w]);
  } else if (pattern == CommPattern::Ring) {
    if (!detail::is_pow2(n)) throw NonPowerOfTwo();
    for (uint32_t s = 0; s + 1 < n; ++s)
      for (uint32_t w = 0; w < n; ++w) net.send(s, w, (w + 1) % n, msg[(w + n - s) % n]);
  } else {
    if (!detail::is_pow2(n)) throw NonPowerOfTwo();
    std::vector<std::vector<uint32_t>> hold(n);
    for (uint32_t w = 0; w < n; ++w) hold[w] = {w};
    for (uint32_t bit = 1, stage = 0; bit < n; bit <<= 1, ++stage) {
      auto prev = hold;
      for (uint32_t w = 0; w < n; ++w) {
        for (uint32_t id : prev[w]) net.send(stage, w, w ^ bit, msg[id]);
        hold[w].insert(hold[w].end(), prev[w ^ bit].begin(), prev[w ^ bit].end());
      }
    }
  }
  std::vector<const detail::DevTensor*> ps;
  for (const auto& t : ins) ps.push_back(&t);
  SyncOutcome out;
  out.results.assign(n, detail::fold(ps).host());
  out.traffic = net.finalize();
  return out;
}

// zen::run_ring_centralization (schemes.hpp:194-215)
inline SyncOutcome run_ring_centralization(const std::vector<SparseTensor>& inputs, SimNet& net,
                                           WireFormat fmt = WireFormat::coo()) {
  detail::check_scheme_inputs(inputs, net);
  if (!detail::is_pow2(inputs.size())) throw NonPowerOfTwo();
  const uint32_t n = uint32_t(inputs.size());
  std::vector<detail::DevTensor> ins, tok;
  for (const auto& t : inputs) ins.emplace_back(t);
  for (const auto& t : inputs) tok.emplace_back(t);
  for (uint32_t s = 0; s + 1 < n; ++s) {
    for (uint32_t w = 0; w < n; ++w) net.send(s, w, (w + 1) % n, detail::sized(tok[w], fmt));
    std::vector<detail::DevTensor> next;
    for (uint32_t w = 0; w < n; ++w) next.push_back(detail::merge_dev(tok[(w + n - 1) % n], ins[w]));
    tok = std::move(next);
  }
  SyncOutcome out;
  for (const auto& t : tok) out.results.push_back(t.host());
  out.traffic = net.finalize();
  return out;
}

// zen::run_omnireduce_like (schemes.hpp:219-328)
inline SyncOutcome run_omnireduce_like(const std::vector<SparseTensor>& inputs, SimNet& net,
                                       uint32_t block_size = 256) {
  detail::check_scheme_inputs(inputs, net);
  if (block_size < 1) throw Error("block size must be at least 1");
  const uint32_t n = uint32_t(inputs.size());
  const uint64_t m = inputs.front().universe(), range = (m + n - 1) / n;
  std::vector<std::vector<detail::DevTensor>> sl(n);
  for (uint32_t w = 0; w < n; ++w) {
    detail::DevTensor t(inputs[w]);
    const auto cnt = detail::range_counts(t, n);
    uint64_t at = 0;
    for (uint32_t p = 0; p < n; ++p) {
      sl[w].push_back(detail::slice(t, at, cnt[p]));
      at += cnt[p];
    }
  }
  auto blocks = [&](const detail::DevTensor& t, uint32_t p) {
    EncodedMessage msg;
    msg.format = WireFormat::tensor_block(block_size);
    msg.universe_size = m;
    if (!t.n) return msg;
    const uint64_t lo = uint64_t(p) * range, hi = std::min(m, lo + range);
    uint64_t nb = 0, last = 0;
    detail::check(zen_count_blocks(detail::ctx(), t.idx->p, t.n, lo, block_size, &nb));
    cudaMemcpy(&last, t.idx->p + t.n - 1, 8, cudaMemcpyDeviceToHost);
    const uint64_t lb = (last - lo) / block_size, end = lo + (lb + 1) * block_size;
    msg.count = nb;
    msg.index_bits = 64 * nb;
    msg.value_bits = 32 * block_size * nb - (end > hi ? 32 * (end - hi) : 0);
    return msg;
  };
  for (uint32_t w = 0; w < n; ++w)
    for (uint32_t p = 0; p < n; ++p)
      if (p != w && sl[w][p].n) net.send(0, w, p, blocks(sl[w][p], p));
  std::vector<detail::DevTensor> agg;
  for (uint32_t p = 0; p < n; ++p) {
    std::vector<const detail::DevTensor*> ps;
    for (uint32_t w = 0; w < n; ++w) ps.push_back(&sl[w][p]);
    agg.push_back(detail::fold(ps));
  }
  for (uint32_t p = 0; p < n; ++p) {
    if (!agg[p].n) continue;
    const EncodedMessage msg = blocks(agg[p], p);
    for (uint32_t w = 0; w < n; ++w)
      if (w != p) net.send(1, p, w, msg);
  }
  uint64_t total = 0;
  for (const auto& a : agg) total += a.n;
  detail::DBuf<uint64_t> ci(total);
  detail::DBuf<float> cv(total);
  uint64_t at = 0;
  for (const auto& a : agg) {
    if (a.n) {
      cudaMemcpy(ci.p + at, a.idx->p, a.n * 8, cudaMemcpyDeviceToDevice);
      cudaMemcpy(cv.p + at, a.val->p, a.n * 4, cudaMemcpyDeviceToDevice);
    }
    at += a.n;
  }
  detail::DBuf<uint64_t> oi(total);
  detail::DBuf<float> ov(total);
  uint64_t kept = 0;
  detail::check(zen_compact_nonzero(detail::ctx(), ci.p, cv.p, total, oi.p, ov.p, &kept));
  SyncOutcome out;
  out.results.assign(n, SparseTensor(m, oi.host(kept), ov.host(kept)));
  bool loaded = true;
  for (const auto& t : inputs) loaded = loaded && !t.empty();
  if (loaded) {  // imbalance_push / imbalance_pull (hashing.hpp:296-320)
    BalanceDetails b;
    double worst = 0.0;
    for (uint32_t w = 0; w < n; ++w)
      for (uint32_t p = 0; p < n; ++p)
        worst = std::max(worst, double(n) * double(sl[w][p].n) / double(inputs[w].nnz()));
    b.push_imbalance = worst;
    worst = 0.0;
    for (const auto& a : agg) worst = std::max(worst, double(n) * double(a.n) / double(total));
    b.pull_imbalance = worst;
    out.balance = b;
  }
  out.traffic = net.finalize();
  return out;
}

// zen::run_scheme (schemes.hpp:420-442)
inline SyncOutcome run_scheme(const SchemeConfig& cfg, const std::vector<SparseTensor>& inputs,
                              SimNet& net, const RunParams& params = {}) {
  cfg.validate();
  if (cfg.partition == PartitionPattern::Centralization) {
    if (cfg.aggregation == Aggregation::OneShot)
      return run_agsparse(inputs, net, cfg.communication, cfg.format);
    if (cfg.communication == CommPattern::Hierarchy)
      return run_hier_centralization(inputs, net, cfg.format);
    if (cfg.communication == CommPattern::Ring)
      return run_ring_centralization(inputs, net, cfg.format);
    throw UnsupportedCombination("point-to-point incremental centralization is not implemented");
  }
  if (cfg.communication == CommPattern::PointToPoint) {
    if (cfg.aggregation == Aggregation::OneShot && cfg.balance == BalancePattern::Imbalanced &&
        cfg.format.kind == WireKind::TensorBlock)
      return run_omnireduce_like(inputs, net, cfg.format.block_size);
    if (cfg.aggregation == Aggregation::Incremental && cfg.balance == BalancePattern::Balanced)
      return run_balanced_parallelism(inputs, net, params.hash);
  }
  throw UnsupportedCombination("no implemented scheme matches this configuration");
}

// zen::scheme_config_from_name / known_scheme_names (schemes.hpp:445-470)
inline SchemeConfig scheme_config_from_name(const std::string& name) {
  using C = CommPattern;
  using A = Aggregation;
  using P = PartitionPattern;
  using B = BalancePattern;
  if (name == "agsparse") return {C::PointToPoint, A::OneShot, P::Centralization, B::NotApplicable, WireFormat::coo()};
  if (name == "sparcml") return {C::Hierarchy, A::Incremental, P::Centralization, B::NotApplicable, WireFormat::coo()};
  if (name == "ring-centralization") return {C::Ring, A::Incremental, P::Centralization, B::NotApplicable, WireFormat::coo()};
  if (name == "omnireduce") return {C::PointToPoint, A::OneShot, P::Parallelism, B::Imbalanced, WireFormat::tensor_block()};
  if (name == "balanced-parallelism") return {C::PointToPoint, A::Incremental, P::Parallelism, B::Balanced, WireFormat::hash_bitmap()};
  throw UnsupportedCombination("unknown scheme name: " + name);
}
inline const std::vector<std::string>& known_scheme_names() {
  static const std::vector<std::string> names = {"agsparse", "sparcml", "ring-centralization",
                                                 "omnireduce", "balanced-parallelism"};
  return names;
}

// ---- experiment driver pieces: zen/experiment.hpp ---------------------------
struct ExperimentConfig {  // experiment.hpp:24-38 (the key=value parser is CLI, out of scope)
  WorkloadSpec workload;
  std::vector<std::string> schemes = known_scheme_names();
  std::vector<uint32_t> n_list = {4, 8, 16};
  double bandwidth = 1e9;
  uint32_t trials = 1;
  uint32_t hash_depth = 3;
  double r1_multiplier = 2.0;
  double r2_ratio = 0.1;
  uint32_t lanes = 1;
  uint32_t block_size = 256;
  std::string out_dir = "out";
  std::string tensors_dir;
};

struct HashSweepCell {  // experiment.hpp:356-364
  double r1_multiplier = 0.0;
  uint32_t rehash_depth = 0;
  double serial_fraction = 0.0;
  std::vector<uint64_t> placed_at_depth;
  uint64_t loss = 0;
  double wall_ms = 0.0;
  bool overflow = false;
};

// The hash-memory geometry sweep of the paper's §4.3 study (zensim
// bench-hash, experiment.hpp:366-401): one generated tensor through the
// device hierarchical hash for r1 multiplier x rehash depth, the serial
// region opened wide (r2 = r1) so the serial fraction is measured.
inline std::vector<HashSweepCell> bench_hash(const ExperimentConfig& cfg) {
  WorkloadSpec spec = cfg.workload;
  spec.nodes = 1;
  const SparseTensor t = generate(spec)[0];
  const uint64_t nnz = t.nnz();
  const uint32_t n = cfg.workload.nodes;
  std::vector<HashSweepCell> cells;
  for (double mult : {1.0, 2.0, 4.0})
    for (uint32_t k : {1u, 2u, 3u, 4u}) {
      HashSweepCell cell;
      cell.r1_multiplier = mult;
      cell.rehash_depth = k;
      const HashFamily fam = HashFamily::make_worker(cfg.workload.seed, 0, n, k);
      const uint64_t r1 = std::max<uint64_t>(1, uint64_t(mult * double(nnz) / double(n)));
      try {
        const auto t0 = std::chrono::steady_clock::now();
        auto res = detail::run_hierarchical_hash(t, n, fam, r1, r1, cfg.lanes);
        cell.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        cell.serial_fraction = double(res.second.serial_writes) / double(nnz);
        cell.placed_at_depth = res.second.placed_at_depth;
        cell.loss = nnz - res.first.total_nnz();
      } catch (const SerialOverflow&) {
        cell.overflow = true;
      }
      cells.push_back(cell);
    }
  return cells;
}

// codec.hpp:76-90: total index bits of a hash-bitmap pull (sum of |I_s| over
// the servers, from the device universe tables) and of a plain-bitmap pull
inline uint64_t pull_hash_bitmap_total_bits(uint64_t universe_size, uint32_t servers,
                                            uint64_t partition_seed) {
  HashUniverseTable t(universe_size, servers, partition_seed);
  uint64_t total = 0;
  for (uint32_t s = 0; s < servers; ++s) total += t.size(s);
  return total;
}
inline uint64_t pull_plain_bitmap_total_bits(uint64_t universe_size, uint32_t servers) {
  return uint64_t(servers) * universe_size;
}

}  // namespace zen_b200
