// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/zen/*.hpp, compiled in place by
// oracle/Makefile into oracle/_ref/libzenref.so; nothing from the reference is
// copied into this repo).  It lets the Python tests and bench.py's reference
// arm call the reference's own code: the golden fixtures, the pinning of the C
// restatement (oracle/zen_oracle.c) and the CPU baseline all come through here.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "zen/codec.hpp"
#include "zen/costmodel.hpp"
#include "zen/errors.hpp"
#include "zen/experiment.hpp"
#include "zen/hashing.hpp"
#include "zen/schemes.hpp"
#include "zen/simnet.hpp"
#include "zen/tensor.hpp"
#include "zen/workload.hpp"

namespace {
enum { ZR_OK = 0, ZR_INVALID = 1, ZR_OVERFLOW = 2, ZR_OUTSIDE = 3, ZR_MALFORMED = 4, ZR_EMPTY = 5,
       ZR_MISMATCH = 6, ZR_NONPOW2 = 7, ZR_MISSING = 8, ZR_OTHER = 9, ZR_UNSUPPORTED = 10 };

thread_local int64_t g_last_partition = -1;
thread_local char g_last_msg[512];

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ZR_OK;
  } catch (const zen::SerialOverflow& e) {
    g_last_partition = e.partition();
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_OVERFLOW;
  } catch (const zen::IndexOutsideUniverse& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_OUTSIDE;
  } catch (const zen::MalformedPayload& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_MALFORMED;
  } catch (const zen::EmptyTensor& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_EMPTY;
  } catch (const zen::NonPowerOfTwo& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_NONPOW2;
  } catch (const zen::UnsupportedCombination& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_UNSUPPORTED;
  } catch (const zen::MissingProfileEntry& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_MISSING;
  } catch (const zen::UniverseMismatch& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_MISMATCH;
  } catch (const zen::Error& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_INVALID;
  } catch (const std::exception& e) {
    std::snprintf(g_last_msg, sizeof g_last_msg, "%s", e.what());
    return ZR_OTHER;
  }
}

zen::SparseTensor make_tensor(uint64_t m, const uint64_t* idx, const float* val, uint64_t n) {
  return zen::SparseTensor(m, std::vector<uint64_t>(idx, idx + n), std::vector<float>(val, val + n));
}

zen::HashFamily make_family(uint64_t seed, uint32_t worker, uint32_t n, uint32_t k, int as_worker) {
  return as_worker ? zen::HashFamily::make_worker(seed, worker, n, k)
                   : zen::HashFamily::make(seed, n, k);
}
}  // namespace

extern "C" {

int64_t ref_last_partition() { return g_last_partition; }
const char* ref_last_message() { return g_last_msg; }

uint64_t ref_mix64(uint64_t x) { return zen::detail::mix64(x); }
uint64_t ref_derive_seed(uint64_t m, uint64_t s) { return zen::detail::derive_seed(m, s); }

// HashFamily seeds: out[0] = partition seed, out[1..k] = slot seeds.
int ref_family(uint64_t seed, uint32_t worker, uint32_t n, uint32_t k, int as_worker,
               uint64_t* out) {
  return guarded([&] {
    auto f = make_family(seed, worker, n, k, as_worker);
    out[0] = f.partition_seed;
    for (uint32_t i = 0; i < k; ++i) out[1 + i] = f.slot_seeds[i];
  });
}

void ref_partition_of_many(const uint64_t* idx, uint64_t count, uint64_t pseed, uint32_t n,
                           uint32_t* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = zen::partition_of(idx[i], pseed, n);
}

void ref_slot_of_many(uint64_t seed, uint32_t worker, uint32_t n, uint32_t k, int as_worker,
                      const uint64_t* idx, uint64_t count, uint64_t r1, uint64_t* out /*[count*k]*/) {
  auto f = make_family(seed, worker, n, k, as_worker);
  for (uint64_t i = 0; i < count; ++i)
    for (uint32_t r = 1; r <= k; ++r) out[i * k + (r - 1)] = f.slot_of(idx[i], r, r1);
}

// zen::hierarchical_hash + zen::collision_stats. Parts are concatenated in
// partition order. stats[0] = serial_writes, stats[1..k] = placed_at_depth.
int ref_hierarchical_hash(uint64_t m, const uint64_t* idx, const float* val, uint64_t count,
                          uint64_t seed, uint32_t worker, int as_worker, uint32_t n, uint32_t k,
                          uint64_t r1, uint64_t r2, uint32_t lanes, uint64_t* out_idx,
                          float* out_val, uint64_t* part_count, uint64_t* stats) {
  return guarded([&] {
    auto t = make_tensor(m, idx, val, count);
    auto f = make_family(seed, worker, n, k, as_worker);
    auto parts = zen::hierarchical_hash(t, n, f, r1, r2, lanes);
    uint64_t off = 0;
    for (uint32_t p = 0; p < n; ++p) {
      const auto& pt = parts.parts[p];
      std::copy(pt.indices().begin(), pt.indices().end(), out_idx + off);
      std::copy(pt.values().begin(), pt.values().end(), out_val + off);
      part_count[p] = pt.nnz();
      off += pt.nnz();
    }
    if (stats) {
      auto cs = zen::collision_stats(t, n, f, r1, r2);
      stats[0] = cs.serial_writes;
      for (uint32_t d = 0; d < k; ++d) stats[1 + d] = cs.placed_at_depth[d];
    }
  });
}

// The lanes=1 hash memory after placement, driven through the reference's own
// detail::HashMemory and detail::place_index in the exact order
// detail::run_hierarchical_hash uses for one lane (zen/hashing.hpp:189-213).
int ref_slot_layout(uint64_t m, const uint64_t* idx, const float* val, uint64_t count,
                    uint64_t seed, uint32_t worker, int as_worker, uint32_t n, uint32_t k,
                    uint64_t r1, uint64_t r2, uint64_t* slots, float* slot_vals, uint32_t* depth_of,
                    int64_t* overflow) {
  return guarded([&] {
    auto t = make_tensor(m, idx, val, count);
    auto f = make_family(seed, worker, n, k, as_worker);
    zen::detail::HashMemory mem(n, r1, r2);
    std::atomic<int64_t> ovf{-1};
    for (uint64_t i = 0; i < count; ++i) {
      const uint32_t d = zen::detail::place_index(mem, f, t.indices()[i], t.values()[i], ovf);
      if (depth_of) depth_of[i] = d;
    }
    const uint64_t cells = uint64_t(n) * (r1 + r2);
    for (uint64_t c = 0; c < cells; ++c) {
      slots[c] = mem.slots[c].load();
      slot_vals[c] = slots[c] ? mem.values[c] : 0.0f;
    }
    *overflow = ovf.load();
  });
}

uint64_t ref_to_sparse(const float* dense, uint64_t m, uint64_t* idx, float* val) {
  zen::DenseTensor d(std::vector<float>(dense, dense + m));
  auto t = zen::to_sparse(d);
  std::copy(t.indices().begin(), t.indices().end(), idx);
  std::copy(t.values().begin(), t.values().end(), val);
  return t.nnz();
}

// zen::generate: every node gets exactly nnz_per_node entries.
int ref_generate(uint64_t m, uint32_t nodes, double density, double omega, double hot_fraction,
                 double hot_mass, uint64_t seed, uint64_t* idx, float* val, uint64_t* nnz_out) {
  return guarded([&] {
    zen::WorkloadSpec spec;
    spec.universe = m;
    spec.nodes = nodes;
    spec.density = density;
    spec.omega = omega;
    spec.hot_fraction = hot_fraction;
    spec.hot_mass = hot_mass;
    spec.seed = seed;
    auto ts = zen::generate(spec);
    const uint64_t z = spec.nnz_per_node();
    for (uint32_t w = 0; w < nodes; ++w) {
      std::copy(ts[w].indices().begin(), ts[w].indices().end(), idx + w * z);
      std::copy(ts[w].values().begin(), ts[w].values().end(), val + w * z);
    }
    *nnz_out = z;
  });
}

uint64_t ref_universe_size(uint64_t m, uint32_t n, uint64_t pseed, uint32_t s) {
  zen::HashUniverseTable t(m, n, pseed);
  return t.universe(s).indices.size();
}

// HashBitmap encode of a tensor owned by server s. payload sized by caller
// (ceil(|I_s|/8) + 4*count). Returns index_bits through *bits.
int ref_hash_bitmap_encode(uint64_t m, uint32_t n, uint64_t pseed, uint32_t s, const uint64_t* idx,
                           const float* val, uint64_t count, uint8_t* payload, uint64_t* bits,
                           uint64_t* payload_len) {
  return guarded([&] {
    zen::HashUniverseTable table(m, n, pseed);
    auto msg = zen::encode(make_tensor(m, idx, val, count), zen::WireFormat::hash_bitmap(),
                           &table.universe(s));
    std::memcpy(payload, msg.payload.data(), msg.payload.size());
    *bits = msg.index_bits;
    *payload_len = msg.payload.size();
  });
}

int ref_hash_bitmap_decode(uint64_t m, uint32_t n, uint64_t pseed, uint32_t s,
                           const uint8_t* payload, uint64_t payload_len, uint64_t count,
                           uint64_t* idx, float* val, uint64_t* out_count) {
  return guarded([&] {
    zen::HashUniverseTable table(m, n, pseed);
    zen::EncodedMessage msg;
    msg.format = zen::WireFormat::hash_bitmap();
    msg.universe_size = m;
    msg.count = count;
    msg.index_bits = table.universe(s).indices.size();
    msg.value_bits = 32 * count;
    msg.payload.assign(payload, payload + payload_len);
    auto t = zen::decode(msg, &table.universe(s));
    std::copy(t.indices().begin(), t.indices().end(), idx);
    std::copy(t.values().begin(), t.values().end(), val);
    *out_count = t.nnz();
  });
}

// zen::run_balanced_parallelism (retry=0) or zen::run_bp_with_retry (retry>0).
// ledger: [2][4][n] = stage x {sent, recv, recv_index, recv_value} x node.
// counts: [n*n] parts |I_w^s| are not exposed by the reference API; pass NULL.
int ref_bp_sync(uint32_t n, uint64_t m, const uint64_t* const* idx, const float* const* val,
                const uint64_t* nnz, uint32_t k, double r1_mult, double r2_ratio, uint32_t lanes,
                uint64_t seed, int retries, uint64_t* out_idx, float* out_val, uint64_t* out_count,
                uint64_t* ledger, double* balance, int* balance_valid, int* all_equal) {
  return guarded([&] {
    std::vector<zen::SparseTensor> inputs;
    for (uint32_t w = 0; w < n; ++w) inputs.push_back(make_tensor(m, idx[w], val[w], nnz[w]));
    zen::HashParams hp;
    hp.rehash_depth = k;
    hp.r1_multiplier = r1_mult;
    hp.r2_ratio = r2_ratio;
    hp.lanes = lanes;
    hp.seed = seed;
    zen::SyncOutcome out;
    if (retries > 0) {
      out = zen::run_bp_with_retry(inputs, 1.0, hp, nullptr, retries);
    } else {
      zen::SimNet net(n, 1.0);
      out = zen::run_balanced_parallelism(inputs, net, hp);
    }
    const auto& r = out.results[0];
    std::copy(r.indices().begin(), r.indices().end(), out_idx);
    std::copy(r.values().begin(), r.values().end(), out_val);
    *out_count = r.nnz();
    int eq = 1;
    for (const auto& x : out.results) eq = eq && (x == r);
    if (all_equal) *all_equal = eq;
    if (ledger) {
      std::memset(ledger, 0, sizeof(uint64_t) * 8 * n);
      for (size_t st = 0; st < out.traffic.stages.size() && st < 2; ++st) {
        const auto& s = out.traffic.stages[st];
        for (uint32_t node = 0; node < n; ++node) {
          ledger[(st * 4 + 0) * n + node] = s.sent_bits[node];
          ledger[(st * 4 + 1) * n + node] = s.recv_bits[node];
          ledger[(st * 4 + 2) * n + node] = s.recv_index_bits[node];
          ledger[(st * 4 + 3) * n + node] = s.recv_value_bits[node];
        }
      }
    }
    if (balance_valid) *balance_valid = out.balance.has_value();
    if (balance && out.balance) {
      balance[0] = out.balance->push_imbalance;
      balance[1] = out.balance->pull_imbalance;
    }
  });
}

// zen::aggregate over n tensors (the scheme-independent oracle, tensor.hpp:171-176).
int ref_aggregate(uint32_t n, uint64_t m, const uint64_t* const* idx, const float* const* val,
                  const uint64_t* nnz, uint64_t* out_idx, float* out_val, uint64_t* out_count) {
  return guarded([&] {
    std::vector<zen::SparseTensor> inputs;
    for (uint32_t w = 0; w < n; ++w) inputs.push_back(make_tensor(m, idx[w], val[w], nnz[w]));
    auto r = zen::aggregate(inputs);
    std::copy(r.indices().begin(), r.indices().end(), out_idx);
    std::copy(r.values().begin(), r.values().end(), out_val);
    *out_count = r.nnz();
  });
}

// CPU baseline probe: to_sparse of every worker's dense gradient, then
// run_balanced_parallelism with a prebuilt universe table and `lanes` lane
// threads (n >= 2), or hierarchical_hash(n=1) when n == 1 (the reference rejects
// n < 2, zen/schemes.hpp:66). Times in ms: t[0] = to_sparse total, t[1] = sync,
// t[2] = table build (one-time, excluded from the step).
int ref_bench_step(uint32_t n, uint64_t m, const float* const* dense, uint32_t k, double r1_mult,
                   double r2_ratio, uint32_t lanes, uint64_t seed, int reps, double* t,
                   uint64_t* result_nnz) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::unique_ptr<zen::HashUniverseTable> table;
    auto t0 = clk::now();
    if (n >= 2) table = std::make_unique<zen::HashUniverseTable>(zen::bp_universe_table(m, n, seed));
    t[2] = ms(t0, clk::now());
    t[0] = t[1] = 0.0;
    // the reference's DenseTensor holds its own copy: built once, outside the
    // timed region (a training loop hands to_sparse an existing DenseTensor)
    std::vector<zen::DenseTensor> dts;
    for (uint32_t w = 0; w < n; ++w)
      dts.push_back(zen::DenseTensor(std::vector<float>(dense[w], dense[w] + m)));
    for (int r = 0; r < reps; ++r) {
      auto a = clk::now();
      std::vector<zen::SparseTensor> inputs;
      for (uint32_t w = 0; w < n; ++w) inputs.push_back(zen::to_sparse(dts[w]));
      auto b = clk::now();
      zen::HashParams hp;
      hp.rehash_depth = k;
      hp.r1_multiplier = r1_mult;
      hp.r2_ratio = r2_ratio;
      hp.lanes = lanes;
      hp.seed = seed;
      if (n >= 2) {
        zen::SimNet net(n, 1.0);
        auto out = zen::run_balanced_parallelism(inputs, net, hp, table.get());
        *result_nnz = out.results[0].nnz();
      } else {
        auto f = zen::HashFamily::make_worker(seed, 0, 1, k);
        const uint64_t z = inputs[0].nnz();
        const uint64_t r1 = std::max<uint64_t>(1, uint64_t(std::ceil(r1_mult * double(z))));
        const uint64_t r2 = std::max<uint64_t>(1, uint64_t(std::ceil(r2_ratio * double(r1))));
        auto parts = zen::hierarchical_hash(inputs[0], 1, f, r1, r2, lanes);
        *result_nnz = parts.total_nnz();
      }
      auto c = clk::now();
      t[0] += ms(a, b);
      t[1] += ms(b, c);
    }
    t[0] /= reps;
    t[1] /= reps;
  });
}

// zen::encode for every WireKind (zen/codec.hpp:213-278).  kind: 1 coo,
// 2 bitmap, 3 tensor block, 4 hash bitmap (n/pseed/s used for 4 only).
// info: [count, index_bits, value_bits, payload_len]
int ref_wire_encode(uint32_t kind, uint32_t block_size, uint32_t coo_bits, uint64_t m,
                    uint32_t n, uint64_t pseed, uint32_t s, const uint64_t* idx, const float* val,
                    uint64_t count, uint8_t* payload, uint64_t capacity, uint64_t* info) {
  return guarded([&] {
    zen::WireFormat fmt = kind == 1 ? zen::WireFormat::coo(coo_bits)
                          : kind == 2 ? zen::WireFormat::bitmap()
                          : kind == 3 ? zen::WireFormat::tensor_block(block_size)
                                      : zen::WireFormat::hash_bitmap();
    std::unique_ptr<zen::HashUniverseTable> table;
    if (kind == 4) table.reset(new zen::HashUniverseTable(m, n, pseed));
    auto msg = zen::encode(make_tensor(m, idx, val, count), fmt,
                           table ? &table->universe(s) : nullptr);
    if (msg.payload.size() > capacity) throw zen::Error("payload capacity");
    std::memcpy(payload, msg.payload.data(), msg.payload.size());
    info[0] = msg.count;
    info[1] = msg.index_bits;
    info[2] = msg.value_bits;
    info[3] = msg.payload.size();
  });
}

// zen::decode (zen/codec.hpp:282-347) of a payload with the given header fields
int ref_wire_decode(uint32_t kind, uint32_t block_size, uint32_t coo_bits, uint64_t m,
                    uint32_t n, uint64_t pseed, uint32_t s, uint64_t count, const uint8_t* payload,
                    uint64_t payload_len, uint64_t* idx, float* val, uint64_t capacity,
                    uint64_t* out_count) {
  return guarded([&] {
    zen::EncodedMessage msg;
    msg.format = kind == 1 ? zen::WireFormat::coo(coo_bits)
                 : kind == 2 ? zen::WireFormat::bitmap()
                 : kind == 3 ? zen::WireFormat::tensor_block(block_size)
                             : zen::WireFormat::hash_bitmap();
    msg.universe_size = m;
    msg.count = count;
    msg.payload.assign(payload, payload + payload_len);
    std::unique_ptr<zen::HashUniverseTable> table;
    if (kind == 4) table.reset(new zen::HashUniverseTable(m, n, pseed));
    auto t = zen::decode(msg, table ? &table->universe(s) : nullptr);
    if (t.nnz() > capacity) throw zen::Error("output capacity");
    std::copy(t.indices().begin(), t.indices().end(), idx);
    std::copy(t.values().begin(), t.values().end(), val);
    *out_count = t.nnz();
  });
}

// zen::write_framed (zen/codec.hpp:356-366) of zen::encode's message -> bytes
int ref_write_framed(uint32_t kind, uint32_t block_size, uint32_t coo_bits, uint64_t m,
                     uint32_t n, uint64_t pseed, uint32_t s, const uint64_t* idx, const float* val,
                     uint64_t count, uint8_t* out, uint64_t capacity, uint64_t* out_len) {
  return guarded([&] {
    zen::WireFormat fmt = kind == 1 ? zen::WireFormat::coo(coo_bits)
                          : kind == 2 ? zen::WireFormat::bitmap()
                          : kind == 3 ? zen::WireFormat::tensor_block(block_size)
                                      : zen::WireFormat::hash_bitmap();
    std::unique_ptr<zen::HashUniverseTable> table;
    if (kind == 4) table.reset(new zen::HashUniverseTable(m, n, pseed));
    auto msg = zen::encode(make_tensor(m, idx, val, count), fmt,
                           table ? &table->universe(s) : nullptr);
    std::ostringstream os;
    zen::write_framed(os, msg);
    const std::string b = os.str();
    if (b.size() > capacity) throw zen::Error("frame capacity");
    std::memcpy(out, b.data(), b.size());
    *out_len = b.size();
  });
}

// zen::write_sparse (zen/tensor.hpp:257-264) -> .zspt bytes
int ref_write_sparse(uint64_t m, const uint64_t* idx, const float* val, uint64_t count,
                     uint8_t* out, uint64_t capacity, uint64_t* out_len) {
  return guarded([&] {
    std::ostringstream os;
    zen::write_sparse(os, make_tensor(m, idx, val, count));
    const std::string b = os.str();
    if (b.size() > capacity) throw zen::Error("capacity");
    std::memcpy(out, b.data(), b.size());
    *out_len = b.size();
  });
}

// zen::sparsify_topk (zen/workload.hpp:157-178)
int ref_sparsify_topk(const float* dense, uint64_t m, double fraction, uint64_t* idx, float* val,
                      uint64_t* out_count) {
  return guarded([&] {
    zen::DenseTensor d(std::vector<float>(dense, dense + m));
    auto t = zen::sparsify_topk(d, fraction);
    std::copy(t.indices().begin(), t.indices().end(), idx);
    std::copy(t.values().begin(), t.values().end(), val);
    *out_count = t.nnz();
  });
}

// zen::merge_sum (zen/tensor.hpp:133-167)
int ref_merge_sum(uint64_t m, const uint64_t* ai, const float* av, uint64_t na, const uint64_t* bi,
                  const float* bv, uint64_t nb, uint64_t* out_idx, float* out_val,
                  uint64_t* out_count) {
  return guarded([&] {
    auto r = zen::merge_sum(make_tensor(m, ai, av, na), make_tensor(m, bi, bv, nb));
    std::copy(r.indices().begin(), r.indices().end(), out_idx);
    std::copy(r.values().begin(), r.values().end(), out_val);
    *out_count = r.nnz();
  });
}

// zen::overlap_ratio / densification_ratio / skewness_ratio (zen/tensor.hpp:111-213).
// what: 0 overlap(t0, t1), 1 densification(all), 2 skewness(t0, partitions)
int ref_tensor_metric(int what, uint32_t n, uint64_t m, const uint64_t* const* idx,
                      const float* const* val, const uint64_t* nnz, uint32_t partitions,
                      double* out) {
  return guarded([&] {
    std::vector<zen::SparseTensor> ts;
    for (uint32_t w = 0; w < n; ++w) ts.push_back(make_tensor(m, idx[w], val[w], nnz[w]));
    if (what == 0) *out = zen::overlap_ratio(ts.at(0), ts.at(1));
    else if (what == 1) *out = zen::densification_ratio(ts);
    else *out = zen::skewness_ratio(ts.at(0), partitions);
  });
}

// zen::profile_sparsity over R rounds of n tensors (zen/costmodel.hpp:151-195)
// and zen::select_scheme(profile, n) (:139-149).  gamma[j] = gamma at k = 2^j,
// j <= log2(n) (NaN where absent); *choice: 0 BP, 1 HC, -1 when select throws.
int ref_profile(uint32_t rounds, uint32_t n, uint64_t m, const uint64_t* const* idx,
                const float* const* val, const uint64_t* nnz, double* d, double* gamma,
                uint32_t gamma_len, double* skew, int* choice) {
  return guarded([&] {
    std::vector<std::vector<zen::SparseTensor>> rs(rounds);
    for (uint32_t r = 0; r < rounds; ++r)
      for (uint32_t w = 0; w < n; ++w)
        rs[r].push_back(make_tensor(m, idx[r * n + w], val[r * n + w], nnz[r * n + w]));
    auto p = zen::profile_sparsity(rs);
    *d = p.d;
    for (uint32_t j = 0; j < gamma_len; ++j) {
      auto it = p.gamma.find(1ull << j);
      gamma[j] = it == p.gamma.end() ? std::numeric_limits<double>::quiet_NaN() : it->second;
    }
    *skew = p.skew.at(n);
    try {
      *choice = zen::select_scheme(p, n) == zen::SchemeChoice::BalancedParallelism ? 0 : 1;
    } catch (const zen::MissingProfileEntry&) {
      *choice = -1;
    }
  });
}

// zen::run_hier_centralization (zen/schemes.hpp:173-193); wire kind as in
// ref_wire_encode (1 coo, 2 bitmap, 3 tensor block).  ledger: [stages][4][n];
// *stages = recorded stage count (<= max_stages).
int ref_hier_centralization(uint32_t n, uint64_t m, const uint64_t* const* idx,
                            const float* const* val, const uint64_t* nnz, uint32_t kind,
                            uint32_t block_size, uint32_t coo_bits, uint64_t* out_idx,
                            float* out_val, uint64_t* out_count, uint64_t* ledger,
                            uint32_t max_stages, uint32_t* stages, int* all_equal) {
  return guarded([&] {
    std::vector<zen::SparseTensor> inputs;
    for (uint32_t w = 0; w < n; ++w) inputs.push_back(make_tensor(m, idx[w], val[w], nnz[w]));
    zen::WireFormat fmt = kind == 2   ? zen::WireFormat::bitmap()
                          : kind == 3 ? zen::WireFormat::tensor_block(block_size)
                                      : zen::WireFormat::coo(coo_bits);
    zen::SimNet net(n, 1.0);
    auto out = zen::run_hier_centralization(inputs, net, fmt);
    const auto& r = out.results[0];
    std::copy(r.indices().begin(), r.indices().end(), out_idx);
    std::copy(r.values().begin(), r.values().end(), out_val);
    *out_count = r.nnz();
    int eq = 1;
    for (const auto& x : out.results) eq = eq && (x == r);
    *all_equal = eq;
    const uint32_t ns = uint32_t(std::min<size_t>(max_stages, out.traffic.stages.size()));
    *stages = ns;
    for (uint32_t st = 0; st < ns; ++st) {
      const auto& s = out.traffic.stages[st];
      for (uint32_t node = 0; node < n; ++node) {
        ledger[(st * 4 + 0) * n + node] = s.sent_bits[node];
        ledger[(st * 4 + 1) * n + node] = s.recv_bits[node];
        ledger[(st * 4 + 2) * n + node] = s.recv_index_bits[node];
        ledger[(st * 4 + 3) * n + node] = s.recv_value_bits[node];
      }
    }
  });
}

// zen::run_scheme (zen/schemes.hpp:420-442) on scheme_config_from_name(name),
// optionally overriding the communication pattern (0 ring, 1 hierarchy, 2
// point-to-point; -1 keep) and the wire format (kind 0 keeps it).  Every
// node's result goes out (n * cap entries), with the ledger [stages][4][n]
// and the balance when the scheme measures one.
int ref_run_scheme(const char* name, int comm, uint32_t kind, uint32_t block_size,
                   uint32_t coo_bits, uint32_t n, uint64_t m, const uint64_t* const* idx,
                   const float* const* val, const uint64_t* nnz, uint64_t cap, uint64_t* out_idx,
                   float* out_val, uint64_t* out_counts, uint64_t* ledger, uint32_t max_stages,
                   uint32_t* stages, double* balance, int* balance_valid) {
  return guarded([&] {
    std::vector<zen::SparseTensor> inputs;
    for (uint32_t w = 0; w < n; ++w) inputs.push_back(make_tensor(m, idx[w], val[w], nnz[w]));
    zen::SchemeConfig cfg = zen::scheme_config_from_name(name);
    if (comm == 0) cfg.communication = zen::CommPattern::Ring;
    if (comm == 1) cfg.communication = zen::CommPattern::Hierarchy;
    if (comm == 2) cfg.communication = zen::CommPattern::PointToPoint;
    if (kind == 1) cfg.format = zen::WireFormat::coo(coo_bits);
    if (kind == 2) cfg.format = zen::WireFormat::bitmap();
    if (kind == 3) cfg.format = zen::WireFormat::tensor_block(block_size);
    zen::SimNet net(n, 1.0);
    auto out = zen::run_scheme(cfg, inputs, net);
    for (uint32_t w = 0; w < n; ++w) {
      const auto& r = out.results[w];
      if (r.nnz() > cap) throw zen::Error("result capacity");
      std::copy(r.indices().begin(), r.indices().end(), out_idx + size_t(w) * cap);
      std::copy(r.values().begin(), r.values().end(), out_val + size_t(w) * cap);
      out_counts[w] = r.nnz();
    }
    const uint32_t ns = uint32_t(std::min<size_t>(max_stages, out.traffic.stages.size()));
    *stages = ns;
    for (uint32_t st = 0; st < ns; ++st) {
      const auto& s = out.traffic.stages[st];
      for (uint32_t node = 0; node < n; ++node) {
        ledger[(st * 4 + 0) * n + node] = s.sent_bits[node];
        ledger[(st * 4 + 1) * n + node] = s.recv_bits[node];
        ledger[(st * 4 + 2) * n + node] = s.recv_index_bits[node];
        ledger[(st * 4 + 3) * n + node] = s.recv_value_bits[node];
      }
    }
    *balance_valid = out.balance.has_value();
    if (out.balance) {
      balance[0] = out.balance->push_imbalance;
      balance[1] = out.balance->pull_imbalance;
    }
  });
}

}  // extern "C"
