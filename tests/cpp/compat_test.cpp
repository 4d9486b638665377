// compat_test.cpp -- the reference's own unit-test cases for the hot path
// (proj/tests/hashing_test.cpp, codec_test.cpp, schemes_test.cpp), re-expressed
// against the C++ drop-in (include/zen_b200/compat.hpp) on the GPU.  A tiny
// assertion runner stands in for GTest (absent in this image).
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>

#include "zen_b200/compat.hpp"

namespace z = zen_b200;

static int g_fail = 0, g_checks = 0;
#define EXPECT(c)                                                               \
  do {                                                                          \
    ++g_checks;                                                                 \
    if (!(c)) {                                                                 \
      ++g_fail;                                                                 \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);                \
    }                                                                           \
  } while (0)
#define EXPECT_THROW(stmt, T)            \
  do {                                   \
    bool thrown_ = false;                \
    try {                                \
      stmt;                              \
    } catch (const T&) {                 \
      thrown_ = true;                    \
    }                                    \
    EXPECT(thrown_);                     \
  } while (0)

static z::SparseTensor random_tensor(uint64_t m, uint64_t nnz, std::mt19937_64& rng) {
  std::unordered_set<uint64_t> seen;
  std::vector<std::pair<uint64_t, float>> pairs;
  std::uniform_int_distribution<uint64_t> pick(0, m - 1);
  std::uniform_int_distribution<int> value(1, 16);
  while (pairs.size() < nnz) {
    const uint64_t idx = pick(rng);
    if (seen.insert(idx).second) pairs.emplace_back(idx, float(value(rng)));
  }
  return z::SparseTensor::from_pairs(m, std::move(pairs));
}

static std::set<uint64_t> union_of(const z::PartitionedSparseTensor& p) {
  std::set<uint64_t> out;
  for (auto& t : p.parts) out.insert(t.indices().begin(), t.indices().end());
  return out;
}

// independent dense-array oracle (tensor_test.cpp:30-49)
static z::SparseTensor dense_sum(const std::vector<z::SparseTensor>& ts) {
  const uint64_t m = ts[0].universe();
  std::vector<double> acc(m, 0.0);
  std::vector<char> hit(m, 0);
  for (auto& t : ts)
    for (size_t i = 0; i < t.nnz(); ++i) {
      acc[t.indices()[i]] += t.values()[i];
      hit[t.indices()[i]] = 1;
    }
  std::vector<uint64_t> idx;
  std::vector<float> val;
  for (uint64_t i = 0; i < m; ++i)
    if (hit[i]) {
      idx.push_back(i);
      val.push_back(float(acc[i]));
    }
  return z::SparseTensor(m, idx, val);
}

static std::vector<z::SparseTensor> workload(uint32_t n, uint64_t m, double d, double omega,
                                             uint64_t seed) {
  std::mt19937_64 rng(seed);
  const uint64_t nnz = uint64_t(std::ceil(d * double(m)));
  const uint64_t core = uint64_t(std::ceil(omega * double(nnz)));
  auto c = random_tensor(m, core, rng);
  std::vector<z::SparseTensor> out;
  for (uint32_t w = 0; w < n; ++w) {
    std::set<uint64_t> s(c.indices().begin(), c.indices().end());
    std::uniform_int_distribution<uint64_t> pick(0, m - 1);
    while (s.size() < nnz) s.insert(pick(rng));
    std::vector<uint64_t> idx(s.begin(), s.end());
    std::vector<float> val(idx.size());
    std::uniform_int_distribution<int> value(1, 16);
    for (auto& v : val) v = float(value(rng));
    out.emplace_back(m, idx, val);
  }
  return out;
}

static std::map<std::string, std::function<void()>>& tests() {
  static std::map<std::string, std::function<void()>> t;
  return t;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { tests()[n] = std::move(f); }
};
#define TEST(name) \
  static void name(); \
  static Reg reg_##name(#name, name); \
  static void name()

// ---- hashing_test.cpp ------------------------------------------------------
TEST(HashFamily_DeterministicAcrossInstances) {
  auto a = z::HashFamily::make(1234, 16, 3), b = z::HashFamily::make(1234, 16, 3);
  EXPECT(a.partition_seed == b.partition_seed && a.slot_seeds == b.slot_seeds);
  auto pa = z::partition_of(std::vector<uint64_t>{0, 1, 17, 123456789}, a.partition_seed, 16);
  auto pb = z::partition_of(std::vector<uint64_t>{0, 1, 17, 123456789}, b.partition_seed, 16);
  EXPECT(pa == pb);
}

TEST(HashFamily_PartitionHashIsRoughlyUniform) {
  auto f = z::HashFamily::make(99, 16, 1);
  std::vector<uint64_t> idx(160000);
  for (uint64_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::vector<uint64_t> counts(16, 0);
  for (auto p : z::partition_of(idx, f.partition_seed, 16)) ++counts[p];
  for (auto c : counts) EXPECT(std::fabs(double(c) - 10000.0) <= 6.0 * std::sqrt(10000.0));
}

TEST(HierarchicalHash_SingleIndexLandsInItsPartition) {
  auto f = z::HashFamily::make(5, 8, 3);
  z::SparseTensor t(1000, {123}, {2.5f});
  auto parts = z::hierarchical_hash(t, 8, f, 4, 2);
  const uint32_t p = f.partition_of(123);  // the member form, zen/hashing.hpp:73-76
  for (uint32_t i = 0; i < 8; ++i) EXPECT(parts.parts[i].nnz() == (i == p ? 1u : 0u));
  EXPECT(parts.parts[p].values()[0] == 2.5f);
}

TEST(HierarchicalHash_NoLossOnRandomWorkloads) {
  std::mt19937_64 rng(17);
  for (int trial = 0; trial < 50; ++trial) {
    auto t = random_tensor(100000, 1000, rng);
    auto f = z::HashFamily::make(trial, 16, 3);
    const uint64_t r1 = 2 * 1000 / 16;
    auto parts = z::hierarchical_hash(t, 16, f, r1, r1 / 10 + 1);
    std::set<uint64_t> in(t.indices().begin(), t.indices().end());
    EXPECT(union_of(parts) == in);
    EXPECT(parts.total_nnz() == t.nnz());
  }
}

TEST(HierarchicalHash_ResultIsLaneCountInvariant) {
  std::mt19937_64 rng(29);
  for (int trial = 0; trial < 10; ++trial) {
    auto t = random_tensor(50000, 2000, rng);
    auto f = z::HashFamily::make(1000 + trial, 8, 3);
    auto ref = z::hierarchical_hash(t, 8, f, 500, 50, 1);
    for (uint32_t lanes : {2u, 4u, 8u}) {
      auto parts = z::hierarchical_hash(t, 8, f, 500, 50, lanes);
      for (uint32_t p = 0; p < 8; ++p) EXPECT(parts.parts[p] == ref.parts[p]);
    }
  }
}

TEST(HierarchicalHash_PartitionAssignmentConsistentAcrossWorkers) {
  std::mt19937_64 rng(31);
  auto t = random_tensor(10000, 500, rng);
  auto w0 = z::HashFamily::make_worker(777, 0, 8, 3), w1 = z::HashFamily::make_worker(777, 1, 8, 3);
  EXPECT(w0.slot_seeds != w1.slot_seeds);
  auto p0 = z::hierarchical_hash(t, 8, w0, 256, 32), p1 = z::hierarchical_hash(t, 8, w1, 256, 32);
  for (uint32_t p = 0; p < 8; ++p) EXPECT(p0.parts[p].indices() == p1.parts[p].indices());
}

TEST(HierarchicalHash_SerialOverflowWhenCapacityInsufficient) {
  auto f = z::HashFamily::make(7, 2, 2);
  std::vector<uint64_t> cand(200);
  for (uint64_t i = 0; i < cand.size(); ++i) cand[i] = i;
  auto part = z::partition_of(cand, f.partition_seed, 2);
  std::vector<uint64_t> same;
  for (uint64_t i = 0; i < cand.size() && same.size() < 3; ++i)
    if (part[i] == 0) same.push_back(i);
  z::SparseTensor t(1000, same, {1, 1, 1});
  EXPECT_THROW(z::hierarchical_hash(t, 2, f, 1, 1), z::SerialOverflow);
}

TEST(HierarchicalHash_NoOverflowWhenCapacityIsSufficient) {
  std::mt19937_64 rng(37);
  for (int trial = 0; trial < 20; ++trial) {
    auto t = random_tensor(2000, 200, rng);
    auto f = z::HashFamily::make(trial, 4, 2);
    std::vector<uint64_t> load(4, 0);
    for (auto p : z::partition_of(t.indices(), f.partition_seed, 4)) ++load[p];
    const uint64_t mx = *std::max_element(load.begin(), load.end());
    auto parts = z::hierarchical_hash(t, 4, f, 2, mx, 4);
    EXPECT(parts.total_nnz() == t.nnz());
  }
}

TEST(CollisionStats_CountsSumToInputSize) {
  std::mt19937_64 rng(43);
  auto t = random_tensor(100000, 5000, rng);
  auto f = z::HashFamily::make(61, 16, 4);
  auto st = z::collision_stats(t, 16, f, 2 * 5000 / 16, 5000);
  EXPECT(st.total() == t.nnz());
}

TEST(CollisionStats_SerialFractionSmallWithDefaults) {
  std::mt19937_64 rng(47);
  int ok = 0;
  for (int trial = 0; trial < 100; ++trial) {
    auto t = random_tensor(200000, 2000, rng);
    auto f = z::HashFamily::make(trial * 3 + 1, 8, 4);
    auto st = z::collision_stats(t, 8, f, 2 * 2000 / 8, 2000);
    if (double(st.serial_writes) / double(t.nnz()) < 0.02) ++ok;
  }
  EXPECT(ok >= 95);
}

TEST(Imbalance_KnownAnswers) {
  EXPECT(z::imbalance_pull({30, 70}, 100) == 1.4);
  EXPECT(z::imbalance_pull({50, 50}, 100) == 1.0);
  EXPECT_THROW(z::imbalance_pull({0, 0}, 0), z::EmptyTensor);
}

// ---- codec_test.cpp (HashBitmap rows) ---------------------------------------
TEST(HashUniverseTable_PartitionsTheFullRange) {
  z::HashUniverseTable table(1000, 7, 12345);
  uint64_t total = 0;
  std::set<uint64_t> seen;
  for (uint32_t s = 0; s < 7; ++s) {
    auto idx = table.universe(s).indices_copy();
    EXPECT(std::is_sorted(idx.begin(), idx.end()));
    for (auto i : idx) EXPECT(seen.insert(i).second);
    total += idx.size();
  }
  EXPECT(total == 1000u);
}

TEST(HashBitmap_WorkedExampleWithFifteenElements) {
  for (uint64_t seed = 0; seed < 200000; ++seed) {
    z::HashUniverseTable table(15, 3, seed);
    const auto& u = table.universe(0);
    auto idx = u.indices_copy();
    if (idx.size() < 3) continue;
    auto pos = [&](uint64_t x) {
      auto it = std::find(idx.begin(), idx.end(), x);
      return it == idx.end() ? size_t(-1) : size_t(it - idx.begin());
    };
    if (pos(5) != 1 || pos(7) != 2) continue;
    z::SparseTensor t(15, {5, 7}, {0.3f, 0.9f});
    auto msg = z::encode(t, z::WireFormat::hash_bitmap(), &u);
    EXPECT(msg.index_bits == idx.size());
    EXPECT(!msg.payload.empty() && (msg.payload[0] & 0b111) == 0b110);
    auto back = z::decode(msg, &u);
    EXPECT(back == t);
    return;
  }
  EXPECT(false);
}

TEST(HashBitmap_RejectsIndicesOutsideTheUniverse) {
  z::HashUniverseTable table(100, 4, 9);
  const auto& u = table.universe(0);
  auto idx = u.indices_copy();
  uint64_t foreign = 0;
  while (std::binary_search(idx.begin(), idx.end(), foreign)) ++foreign;
  z::SparseTensor t(100, {foreign}, {1.0f});
  EXPECT_THROW(z::encode(t, z::WireFormat::hash_bitmap(), &u), z::IndexOutsideUniverse);
}

TEST(RoundTrip_HashBitmapSlices) {
  std::mt19937_64 rng(77);
  for (int trial = 0; trial < 40; ++trial) {
    const uint64_t m = 1 + rng() % 2000;
    auto t = random_tensor(m, rng() % (m / 2 + 1), rng);
    z::HashUniverseTable table(m, 1 + uint32_t(rng() % 5), rng());
    for (uint32_t s = 0; s < table.servers(); ++s) {
      auto uidx = table.universe(s).indices_copy();
      std::vector<std::pair<uint64_t, float>> pairs;
      for (size_t i = 0; i < t.nnz(); ++i)
        if (std::binary_search(uidx.begin(), uidx.end(), t.indices()[i]))
          pairs.emplace_back(t.indices()[i], t.values()[i]);
      auto slice = z::SparseTensor::from_pairs(m, std::move(pairs));
      auto msg = z::encode(slice, z::WireFormat::hash_bitmap(), &table.universe(s));
      EXPECT(z::decode(msg, &table.universe(s)) == slice);
    }
  }
}

// ---- schemes_test.cpp (BP rows) ----------------------------------------------
TEST(BalancedParallelism_IdenticalTensorsPullTotalIndexBitsEqualM) {
  const uint64_t m = 4096;
  auto inputs = workload(4, m, 0.02, 1.0, 43);
  z::SimNet net(4, 1.0);
  auto out = z::run_balanced_parallelism(inputs, net);
  EXPECT(out.results[0] == dense_sum(inputs));
  uint64_t sum = 0;
  for (uint32_t w = 0; w < 4; ++w) sum += out.traffic.stages[1].recv_index_bits[w];
  EXPECT(sum == 3 * m);
}

TEST(BalancedParallelism_OracleEqualAcrossNodeCounts) {
  std::mt19937_64 rng(47);
  for (uint32_t n : {2u, 4u, 8u, 16u}) {
    for (int trial = 0; trial < 6; ++trial) {
      auto inputs = workload(n, 20000, 0.005, 0.5, rng());
      z::HashParams params;
      params.seed = rng();
      params.lanes = 1 + trial % 4;
      // small partitions (r2 = 2 at n = 16) can overflow for some seeds; the
      // reference's experiment harness retries with a doubled r2 ratio
      auto out = z::run_bp_with_retry(inputs, 1.0, params);
      const auto want = dense_sum(inputs);
      for (auto& r : out.results) EXPECT(r == want);
    }
  }
}

TEST(BalancedParallelism_BalancedAtScale) {
  auto inputs = workload(16, 1000000, 0.01, 0.5, 51);
  z::SimNet net(16, 1.0);
  auto out = z::run_balanced_parallelism(inputs, net);
  EXPECT(out.balance.has_value());
  EXPECT(out.balance && out.balance->push_imbalance < 1.1);
  EXPECT(out.balance && out.balance->pull_imbalance < 1.1);
}

TEST(BalancedParallelism_SerialOverflowPropagates) {
  auto inputs = workload(2, 1000, 0.1, 0.0, 53);
  z::SimNet net(2, 1.0);
  z::HashParams params;
  params.r1_multiplier = 0.02;
  params.r2_ratio = 0.01;
  EXPECT_THROW(z::run_balanced_parallelism(inputs, net, params), z::SerialOverflow);
  auto out = z::run_bp_with_retry(inputs, 1.0, z::HashParams{3, 0.5, 0.1, 1, 1});
  EXPECT(out.results[0] == dense_sum(inputs));
}

TEST(EdgeCases_EmptyInputsSynchronizeToEmpty) {
  std::vector<z::SparseTensor> inputs(4, z::SparseTensor(1000, {}, {}));
  z::SimNet net(4, 1.0);
  auto out = z::run_balanced_parallelism(inputs, net);
  for (auto& r : out.results) EXPECT(r.nnz() == 0u);
  EXPECT(!out.balance.has_value());
}

TEST(Tensor_ToSparseDropsSignedZeroKeepsNaN) {
  z::DenseTensor d({0.0f, -0.0f, 1.5f, NAN, 0.0f, -2.0f});
  auto t = z::to_sparse(d);
  EXPECT((t.indices() == std::vector<uint64_t>{2, 3, 5}));
}

// ---- codec_test.cpp / tensor_test.cpp: every wire format, framing, .zspt ----
TEST(CooEncoding_SizesFollowTheWidth) {
  std::mt19937_64 rng(1);
  auto t = random_tensor(1000, 25, rng);
  auto msg64 = z::encode(t, z::WireFormat::coo(64));
  EXPECT(msg64.index_bits == 64u * 25 && msg64.value_bits == 32u * 25);
  auto msg32 = z::encode(t, z::WireFormat::coo(32));
  EXPECT(msg32.index_bits == 32u * 25);
  EXPECT(z::decode(msg64) == t);
  EXPECT(z::decode(msg32) == t);
}

TEST(BitmapEncoding_IndexCostIsTheUniverse) {
  std::mt19937_64 rng(2);
  auto t = random_tensor(500, 100, rng);
  auto msg = z::encode(t, z::WireFormat::bitmap());
  EXPECT(msg.index_bits == 500u && msg.value_bits == 3200u);
  EXPECT(z::decode(msg) == t);
}

TEST(EmptyTensor_AllFormatsCarryZeroValueBits) {
  z::SparseTensor t(64, {}, {});
  for (auto fmt : {z::WireFormat::coo(), z::WireFormat::bitmap(), z::WireFormat::tensor_block(16)}) {
    auto msg = z::encode(t, fmt);
    EXPECT(msg.value_bits == 0u);
    EXPECT(z::decode(msg) == t);
  }
}

TEST(TensorBlockEncoding_ReconstructsShortLastAndCost) {
  z::SparseTensor t(32, {3, 4, 17}, {1.0f, 2.0f, 3.0f});
  auto msg = z::encode(t, z::WireFormat::tensor_block(8));
  EXPECT(msg.index_bits == 2u * 64 && msg.value_bits == 2u * 8 * 32);
  EXPECT(z::decode(msg) == t);
  z::SparseTensor s(20, {19}, {5.0f});
  auto m2 = z::encode(s, z::WireFormat::tensor_block(8));
  EXPECT(m2.value_bits == 4u * 32);
  EXPECT(z::decode(m2) == s);
  std::vector<uint64_t> idx;
  std::vector<float> val;
  for (uint64_t b = 0; b < 8; ++b) {
    idx.push_back(b * 256 + 7);
    val.push_back(1.0f);
  }
  z::SparseTensor u(8 * 256, idx, val);
  EXPECT(z::encode(u, z::WireFormat::tensor_block(256)).payload_bits() >
         z::encode(u, z::WireFormat::coo()).payload_bits());
}

TEST(RoundTrip_RandomTensorsAcrossAllFormats) {
  std::mt19937_64 rng(77);
  for (int trial = 0; trial < 30; ++trial) {
    const uint64_t m = 1 + rng() % 2000;
    auto t = random_tensor(m, rng() % (m / 2 + 1), rng);
    for (auto fmt : {z::WireFormat::coo(64), z::WireFormat::coo(32), z::WireFormat::bitmap(),
                     z::WireFormat::tensor_block(1 + uint32_t(rng() % 300))}) {
      auto msg = z::encode(t, fmt);
      EXPECT(msg.payload_bits() == msg.index_bits + msg.value_bits);
      EXPECT(z::decode(msg) == t);
      auto sizes = z::message_sizes(t, fmt);
      EXPECT(sizes.index_bits == msg.index_bits && sizes.value_bits == msg.value_bits);
    }
  }
}

TEST(Framing_RoundTripsAndRejectsTruncation) {
  std::mt19937_64 rng(111);
  for (int trial = 0; trial < 10; ++trial) {
    const uint64_t m = 1 + rng() % 500;
    auto t = random_tensor(m, rng() % (m / 2 + 1), rng);
    for (auto fmt : {z::WireFormat::coo(64), z::WireFormat::coo(32), z::WireFormat::bitmap(),
                     z::WireFormat::tensor_block(7)}) {
      auto msg = z::encode(t, fmt);
      std::stringstream ss;
      z::write_framed(ss, msg);
      auto back = z::read_framed(ss);
      EXPECT(back.index_bits == msg.index_bits && back.value_bits == msg.value_bits);
      EXPECT(back.payload == msg.payload);
      EXPECT(z::decode(back) == t);
    }
  }
  auto msg = z::encode(random_tensor(100, 10, rng), z::WireFormat::coo());
  std::stringstream ss;
  z::write_framed(ss, msg);
  std::string bytes = ss.str();
  bytes.resize(bytes.size() - 3);
  std::stringstream truncated(bytes);
  EXPECT_THROW(z::read_framed(truncated), z::MalformedPayload);
}

TEST(Decode_RejectsCorruptCounts) {
  std::mt19937_64 rng(131);
  auto msg = z::encode(random_tensor(64, 6, rng), z::WireFormat::bitmap());
  msg.count += 1;
  EXPECT_THROW(z::decode(msg), z::MalformedPayload);
}

TEST(Serialization_RoundTripsAndRejectsBadMagic) {
  std::mt19937_64 rng(141);
  auto t = random_tensor(5000, 40, rng);
  std::stringstream ss;
  z::write_sparse(ss, t);
  EXPECT(z::read_sparse(ss) == t);
  std::stringstream bad(std::string("ZSPX") + std::string(20, '\0'));
  EXPECT_THROW(z::read_sparse(bad), z::MalformedPayload);
}

// ---- schemes_test.cpp: HierCentralization; costmodel_test.cpp: SelectScheme ----
static void expect_oracle_equal(const z::SyncOutcome& out, const std::vector<z::SparseTensor>& in) {
  const auto want = z::aggregate(in);
  // the reference oracle folds left in worker order; HC sums pairwise in a
  // tree, so values are compared within fp32 rounding, indices exactly
  for (const auto& r : out.results) {
    EXPECT(r.indices() == want.indices());
    bool close = r.values().size() == want.values().size();
    for (size_t i = 0; close && i < r.values().size(); ++i)
      close = std::fabs(r.values()[i] - want.values()[i]) <=
              1e-5f * std::max(1.0f, std::fabs(want.values()[i]));
    EXPECT(close);
    EXPECT(r == out.results.front());
  }
}

TEST(HierCentralization_TwoNodesExchangeOnce) {
  z::SparseTensor a(50, {1}, {2}), b(50, {2}, {3});
  z::SimNet net(2, 1.0);
  auto out = z::run_hier_centralization({a, b}, net);
  expect_oracle_equal(out, {a, b});
  EXPECT(out.traffic.stages.size() == 1u);
}

TEST(HierCentralization_FullOverlapReceivesCommonSetLogNTimes) {
  auto inputs = workload(4, 1000, 0.05, 1.0, 13);
  const uint64_t zz = inputs[0].nnz();
  z::SimNet net(4, 1.0);
  auto out = z::run_hier_centralization(inputs, net);
  expect_oracle_equal(out, inputs);
  EXPECT(out.traffic.stages.size() == 2u);
  for (uint32_t node = 0; node < 4; ++node) {
    uint64_t total = 0;
    for (const auto& s : out.traffic.stages) total += s.recv_bits[node];
    EXPECT(total == 2 * zz * 96);
  }
}

TEST(HierCentralization_OracleEqualOnRandomCases) {
  std::mt19937_64 rng(17);
  for (int trial = 0; trial < 25; ++trial) {
    const uint32_t n = 1u << (1 + rng() % 3);
    auto inputs = workload(n, 2000, 0.01 + 0.01 * double(rng() % 5), 0.25 * double(rng() % 4), rng());
    z::SimNet net(n, 1.0);
    expect_oracle_equal(z::run_hier_centralization(inputs, net), inputs);
  }
}

TEST(HierCentralization_RejectsNonPowerOfTwo) {
  auto inputs = workload(6, 1000, 0.01, 0.0, 3);
  z::SimNet net(6, 1.0);
  EXPECT_THROW(z::run_hier_centralization(inputs, net), z::NonPowerOfTwo);
}

TEST(HierCentralization_ReceivedBitsShrinkAsOverlapGrows) {
  std::vector<uint64_t> totals;
  for (double omega : {0.0, 0.5, 1.0}) {
    auto inputs = workload(8, 100000, 0.002, omega, 23);
    z::SimNet net(8, 1.0);
    totals.push_back(z::run_hier_centralization(inputs, net).traffic.total_recv_bits);
  }
  EXPECT(totals[0] > totals[1] && totals[1] > totals[2]);
}

TEST(SelectScheme_FullOverlapAndNoOverlap) {
  z::SparsityProfile p;
  p.d = 0.01;
  for (uint64_t k = 1; k <= 16; k *= 2) p.gamma[k] = 1.0;
  EXPECT(z::select_scheme(p, 16) == z::SchemeChoice::BalancedParallelism);
  z::SparsityProfile q;
  q.d = 0.001;
  for (uint64_t k = 1; k <= 16; k *= 2) q.gamma[k] = double(k);
  EXPECT(z::select_scheme(q, 8) == z::SchemeChoice::HierarchicalCentralization);
  EXPECT(z::select_scheme(q, 16) == z::SchemeChoice::HierarchicalCentralization);
  z::SparsityProfile t;
  t.gamma = {{1, 1.0}, {2, 1.0}};
  EXPECT(z::select_scheme(t, 2) == z::SchemeChoice::BalancedParallelism);  // tie -> BP
  EXPECT_THROW(z::t_hc_coefficient(6, q.gamma), z::NonPowerOfTwo);
  z::SparsityProfile u;
  u.gamma = {{1, 1.0}, {4, 2.0}};
  EXPECT_THROW(z::select_scheme(u, 4), z::MissingProfileEntry);
}

TEST(ProfileSparsity_MatchesItsDefinition) {
  auto inputs = workload(4, 20000, 0.02, 0.5, 77);
  auto p = z::profile_sparsity({inputs});
  EXPECT(p.gamma.at(1) == 1.0);
  EXPECT(std::fabs(p.gamma.at(4) - z::densification_ratio(inputs)) < 1e-12);
  EXPECT(std::fabs(p.d - z::density(inputs[0])) < 1e-12);
  EXPECT(p.skew.at(4) >= 1.0);
  EXPECT(std::fabs(z::overlap_ratio(inputs[0], inputs[0]) - 1.0) < 1e-12);
  auto m = z::merge_sum(inputs[0], inputs[1]);
  const double common = z::overlap_ratio(inputs[0], inputs[1]) * double(inputs[0].nnz());
  EXPECT(m.nnz() == inputs[0].nnz() + inputs[1].nnz() - uint64_t(std::llround(common)));
}

// ---- schemes_test.cpp: AgSparse, RingCentralization, OmniReduce, RunScheme ----
static void expect_exact(const z::SyncOutcome& out, const std::vector<z::SparseTensor>& in) {
  const auto want = z::aggregate(in);  // integer-valued workloads: every order sums exactly
  EXPECT(out.results.size() == in.size());
  for (const auto& r : out.results) EXPECT(r == want);
}

TEST(AgSparse_TwoDisjointNodesReceiveEachOthersPayload) {
  z::SparseTensor a(100, {1, 2, 3}, {1, 1, 1}), b(100, {10, 11}, {2, 2});
  z::SimNet net(2, 1.0);
  auto out = z::run_agsparse({a, b}, net);
  expect_exact(out, {a, b});
  EXPECT(out.traffic.stages[0].recv_bits[0] == 2u * 96);
  EXPECT(out.traffic.stages[0].recv_bits[1] == 3u * 96);
}

TEST(AgSparse_AllPatternsMoveTheSameBitsAndAgree) {
  auto inputs = workload(8, 5000, 0.01, 0.3, 7);
  std::vector<uint64_t> totals;
  for (auto pat : {z::CommPattern::PointToPoint, z::CommPattern::Ring, z::CommPattern::Hierarchy}) {
    z::SimNet net(8, 1.0);
    auto out = z::run_agsparse(inputs, net, pat);
    expect_exact(out, inputs);
    totals.push_back(out.traffic.total_recv_bits);
  }
  EXPECT(totals[0] == totals[1] && totals[0] == totals[2]);
}

TEST(AgSparse_ReceivedBitsGrowLinearlyInN) {
  std::vector<double> per_node;
  for (uint32_t n : {4u, 8u, 16u}) {
    auto inputs = workload(n, 100000, 0.005, 0.5, 11);
    z::SimNet net(n, 1.0);
    per_node.push_back(double(z::run_agsparse(inputs, net).traffic.total_recv_bits) / n);
  }
  EXPECT(std::fabs(per_node[1] / per_node[0] - 7.0 / 3.0) < 0.01);
  EXPECT(std::fabs(per_node[2] / per_node[1] - 15.0 / 7.0) < 0.01);
}

TEST(RingCentralization_FullOverlapReceivesCommonSetNMinusOneTimes) {
  auto inputs = workload(4, 1000, 0.05, 1.0, 29);
  const uint64_t zz = inputs[0].nnz();
  z::SimNet net(4, 1.0);
  auto out = z::run_ring_centralization(inputs, net);
  expect_exact(out, inputs);
  EXPECT(out.traffic.stages.size() == 3u);
  for (uint32_t node = 0; node < 4; ++node) {
    uint64_t total = 0;
    for (const auto& st : out.traffic.stages) total += st.recv_bits[node];
    EXPECT(total == 3 * zz * 96);
  }
}

TEST(RingCentralization_StageDensityFollowsTheWindow) {
  std::vector<z::SparseTensor> inputs;
  for (uint64_t i = 0; i < 4; ++i) inputs.push_back(z::SparseTensor(100, {i * 10, i * 10 + 1}, {1, 1}));
  z::SimNet net(4, 1.0);
  auto out = z::run_ring_centralization(inputs, net);
  expect_exact(out, inputs);
  for (uint32_t st = 0; st < 3; ++st) EXPECT(out.traffic.stages[st].recv_bits[0] == (st + 1) * 2 * 96);
}

TEST(OmniReduce_UniformInputsStayBalanced) {
  auto inputs = workload(8, 100000, 0.01, 0.0, 31);
  z::SimNet net(8, 1.0);
  auto out = z::run_omnireduce_like(inputs, net, 64);
  expect_exact(out, inputs);
  EXPECT(out.balance.has_value() && out.balance->push_imbalance < 1.3);
}

TEST(OmniReduce_OracleEqualOnRandomCases) {
  std::mt19937_64 rng(41);
  for (int trial = 0; trial < 25; ++trial) {
    const uint32_t n = 2 + rng() % 7;
    auto inputs = workload(n, 3000, 0.02, 0.25 * double(rng() % 4), rng());
    z::SimNet net(n, 1.0);
    expect_exact(z::run_omnireduce_like(inputs, net, uint32_t(1 + rng() % 100)), inputs);
  }
}

TEST(RunScheme_DispatchAndRejections) {
  auto inputs = workload(4, 2000, 0.02, 0.5, 59);
  for (const auto& name : z::known_scheme_names()) {
    z::SimNet net(4, 1.0);
    expect_exact(z::run_scheme(z::scheme_config_from_name(name), inputs, net), inputs);
  }
  z::SimNet na(4, 1.0), nb(4, 1.0);
  auto direct = z::run_agsparse(inputs, na);
  auto via = z::run_scheme(z::scheme_config_from_name("agsparse"), inputs, nb);
  EXPECT(direct.traffic.total_recv_bits == via.traffic.total_recv_bits);
  EXPECT(direct.results[0] == via.results[0]);
  z::SchemeConfig cfg;
  cfg.balance = z::BalancePattern::Balanced;
  z::SimNet n1(4, 1.0);
  EXPECT_THROW(z::run_scheme(cfg, inputs, n1), z::UnsupportedCombination);
  z::SchemeConfig c2;
  c2.communication = z::CommPattern::Ring;
  c2.aggregation = z::Aggregation::Incremental;
  c2.partition = z::PartitionPattern::Parallelism;
  c2.balance = z::BalancePattern::Imbalanced;
  z::SimNet n2(4, 1.0);
  EXPECT_THROW(z::run_scheme(c2, inputs, n2), z::UnsupportedCombination);
  EXPECT_THROW(z::scheme_config_from_name("nope"), z::UnsupportedCombination);
}

TEST(EdgeCases_EmptyInputsSynchronizeToEmptyEveryScheme) {
  std::vector<z::SparseTensor> inputs(4, z::SparseTensor(1000, {}, {}));
  for (const auto& name : z::known_scheme_names()) {
    z::SimNet net(4, 1.0);
    auto out = z::run_scheme(z::scheme_config_from_name(name), inputs, net);
    for (const auto& r : out.results) EXPECT(r.nnz() == 0u);
    EXPECT(!out.balance.has_value());
  }
}

TEST(Uniformity_AllNodesAgreeForEveryScheme) {
  auto inputs = workload(8, 20000, 0.01, 0.3, 79);
  for (const auto& name : z::known_scheme_names()) {
    z::SimNet net(8, 1.0);
    auto out = z::run_scheme(z::scheme_config_from_name(name), inputs, net);
    for (size_t i = 1; i < out.results.size(); ++i) EXPECT(out.results[i] == out.results[0]);
  }
}

int main() {
  for (auto& [name, fn] : tests()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
