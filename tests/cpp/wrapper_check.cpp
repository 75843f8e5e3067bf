// C++ caller of include/bht_b200.hpp, written the way a caller of the reference's table.hpp is written
// (proj/tests/test_table.cpp shapes): build, bulk find, per-key find_key, error behaviour.  Exit code 0 = all checks pass.
// With the argument "nogpu" only the host-side checks run (used by the CPU test tier).
#include <cstdio>
#include <cstring>
#include <random>
#include <unordered_set>
#include <vector>

#include "bht_b200.hpp"

using namespace bht::gpu;

#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                          \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool nogpu = argc > 1 && std::strcmp(argv[1], "nogpu") == 0;
  // test_core.cpp:28-65
  table_config c = make_config(table_kind::bp2ht, 1000, 0.8, 32);
  CHECK(c.num_buckets == 40 && c.capacity == 1280 && c.n_hashes == 2);
  CHECK(make_config(table_kind::iht, 1000, 0.8, 16).threshold == 12);
  CHECK(make_config(table_kind::bcht, 1000000, 0.9, 16).max_chain == 140);
  CHECK(make_config(table_kind::bcht, 100000, 0.9, 16, std::nullopt, 0, 512).max_chain == 512);
  CHECK(throws<std::invalid_argument>([] { make_config(table_kind::bcht, 0, 0.5, 16); }));
  CHECK(throws<std::invalid_argument>([] { make_config(table_kind::bcht, 10, 0.5, 12); }));
  CHECK(throws<std::invalid_argument>([] { make_config(table_kind::one_cht, 10, 0.5, 2); }));
  CHECK(throws<std::invalid_argument>([] { make_config(table_kind::iht, 10, 0.5, 16, 17u); }));
  CHECK(hash_count(table_kind::one_cht) == 4 && hash_count(table_kind::bcht) == 3);
  CHECK(value_for_key(0xA5A5A5A5u) == 0x7FFFFFFFu);
  // test_hash.cpp:14-28
  CHECK(bht_bucket_index_host(1, 0, 10, 7) == 7 && bht_bucket_index_host(3, 4, 3, 7) == 1 && bht_bucket_index_host(2, 0, 5, 4294967290u) == 4);
  if (nogpu) {
    std::puts("wrapper host checks ok");
    return 0;
  }

  const std::uint64_t n = 200000;
  std::mt19937_64 gen(5);
  std::unordered_set<key_type> seen;
  std::vector<key_type> keys, absent;
  while (keys.size() < n || absent.size() < n) {
    key_type k = static_cast<key_type>(gen() >> 32);
    if (k == empty_key || !seen.insert(k).second) continue;
    (keys.size() < n ? keys : absent).push_back(k);
  }
  for (table_kind kind : {table_kind::bcht, table_kind::bp2ht, table_kind::iht, table_kind::one_cht}) {
    const std::uint32_t b = kind == table_kind::one_cht ? 1 : 16;
    const double lf = kind == table_kind::bcht ? 0.9 : 0.75;
    table_config cfg = make_config(kind, n, lf, b, std::nullopt, 77);
    auto [table, outcome] = build(keys.data(), n, cfg);
    CHECK(outcome.success && outcome.inserted == n && !outcome.failed_key);
    CHECK(table.inserted() == n && table.occupied_slots() == n && table.count_inadmissible() == 0);
    std::vector<value_type> out(n);
    find_stats st;
    table.find(keys.data(), out.data(), n, mem_space::host, nullptr, &st);
    CHECK(st.hits == n);
    for (std::uint64_t i = 0; i < n; ++i) CHECK(out[i] == value_for_key(keys[i]));
    table.find(absent.data(), out.data(), n);
    for (std::uint64_t i = 0; i < n; ++i) CHECK(out[i] == empty_value);
    CHECK(table.find_key(keys[3]) == value_for_key(keys[3]));
    CHECK(!table.find_key(absent[3]));
    // kind mismatch -> std::logic_error (table.cpp:15-17)
    const table_kind other = kind == table_kind::bp2ht ? table_kind::iht : table_kind::bp2ht;
    CHECK(throws<std::logic_error>([&] { table.find_as(other, keys.data(), out.data(), 1); }));
    // store round trip (dump_store layout: bucket-major LE u64)
    auto store = table.download_store();
    hash_table copy(cfg);
    copy.upload_store(store);
    CHECK(copy.inserted() == n);
    copy.find(keys.data(), out.data(), n);
    for (std::uint64_t i = 0; i < n; ++i) CHECK(out[i] == value_for_key(keys[i]));
  }
  // capacity overflow -> std::invalid_argument (table.cpp:225); wrong hash count (table.cpp:22-23)
  table_config small = make_config(table_kind::bcht, 16, 1.0, 16);
  CHECK(throws<std::invalid_argument>([&] { build(keys.data(), 17, small); }));
  table_config bad = small;
  bad.n_hashes = 2;
  CHECK(throws<std::invalid_argument>([&] { hash_table t(bad); }));
  std::puts("wrapper checks ok");
  return 0;
}
