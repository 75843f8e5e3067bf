// C++ caller of include/bht_b200.hpp, written the way a caller of the reference's table.hpp is written
// (proj/tests/test_table.cpp shapes): build, bulk find, per-key find_key, error behaviour.  Exit code 0 = all checks pass.
// With the argument "nogpu" only the host-side checks run (used by the CPU test tier).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <unordered_set>
#include <sstream>
#include <algorithm>
#include <vector>

#include <cuda_runtime_api.h>  // device buffers for the chunked build (the library links its own static runtime)

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
  // workload generators: the same stream as std::mt19937_64 + first-occurrence rejection (keygen.cpp:50-64)
  {
    const std::size_t m = 50000;
    key_set ks = generate_keys(7, m);
    std::mt19937_64 eng(7);
    std::unordered_set<key_type> dedupe;
    std::vector<key_type> want;
    while (want.size() < m) {
      key_type k = static_cast<key_type>(eng() >> 32);
      if (k == empty_key || !dedupe.insert(k).second) continue;
      want.push_back(k);
    }
    CHECK(ks.keys == want && ks.seed == 7);
    auto qs = generate_queries(ks, 0.5, 1000, 5);
    std::size_t positives = 0;
    for (const query& q : qs) {
      positives += q.expected_present;
      CHECK(q.expected_present == (dedupe.count(q.key) != 0));
      if (q.expected_present) CHECK(q.expected_value == value_for_key(q.key));
    }
    CHECK(qs.size() == 1000 && positives == 500);  // test_keygen.cpp:64-69
    CHECK(throws<std::invalid_argument>([&] { generate_queries(ks, 1.1, 10, 1); }));
    CHECK(throws<std::invalid_argument>([&] { generate_queries(ks, 1.0, m + 1, 1); }));
    save_keys("keys_roundtrip.bin", ks);  // test_keygen.cpp:78-86
    CHECK(load_keys("keys_roundtrip.bin", ks.seed).keys == ks.keys);
    std::remove("keys_roundtrip.bin");
    CHECK(throws<std::runtime_error>([] { load_keys("/nonexistent/dir/keys.bin", 0); }));
  }
  // trial protocol (test_experiments.cpp:113-138)
  {
    trial_cell cell;
    cell.params = {table_kind::bcht, 16, 80};
    cell.n = 10000;
    cell.lf = 0.1;
    cell.trials = 3;
    cell.seed = 7;
    cell.positive_ratios = {1.0, 0.0};
    trial_outcome o = run_trial(cell);
    CHECK(o.successes == 3 && o.failures == 0 && !o.budget_exhausted);
    CHECK(o.insert_mean_probes == 1.0 && o.find_mean_probes[0] == 1.0 && o.find_mean_probes[1] == 1.0);
    trial_cell hard;
    hard.params = {table_kind::bp2ht, 8, 80};
    hard.n = 10000;
    hard.lf = 1.0;
    hard.trials = 1;
    hard.max_failures = 5;
    hard.seed = 7;
    trial_outcome h = run_trial(hard);
    CHECK(h.budget_exhausted && h.successes == 0 && h.failures == 5);
  }
  // success rate far below / above a variant's threshold (test_experiments.cpp:192-198) and the CSV line format
  {
    auto r = run_success_rate({table_kind::bcht, 16, 80}, 5000, {0.01, 0.5}, 20, 7);
    CHECK(r.points.size() == 2 && r.points[0].fraction() == 1.0 && r.points[1].fraction() == 1.0);
    CHECK(r.max_load_factor && *r.max_load_factor == 0.5);
    auto hard = run_success_rate({table_kind::bp2ht, 16, 80}, 5000, {0.5, 1.0}, 5, 7);
    CHECK(hard.points[0].successes == 5 && hard.points[1].successes == 0 && *hard.max_load_factor == 0.5);
    result_record rec;
    rec.kind = table_kind::iht; rec.b = 16; rec.threshold_pct = 75; rec.n = 3000; rec.realized_lf = 0.797872; rec.op = "find";
    rec.positive_ratio = 0.0; rec.mean_probes = 3.0; rec.ops_per_sec = 1.5e7; rec.successes = 2; rec.failures = 0; rec.seed = 42;
    CHECK(csv_line(rec) == "iht,16,75,3000,0.797872,find,0,3,1.5e+07,2,0,42");
    rec.kind = table_kind::bcht; rec.threshold_pct.reset(); rec.op = "insert"; rec.positive_ratio.reset(); rec.mean_probes = 1.10823;
    CHECK(csv_line(rec) == "bcht,16,,3000,0.797872,insert,,1.10823,1.5e+07,2,0,42");
    CHECK(std::string(result_csv_header) == "kind,b,threshold_pct,n,realized_lf,op,positive_ratio,mean_probes,ops_per_sec,successes,failures,seed");
  }
  // run_experiment / write_csv (test_experiments.cpp:140-190): record order, cell seeds, CSV shape
  {
    experiment_spec spec;
    spec.kinds = {{table_kind::bcht, 16, 80}, {table_kind::iht, 16, 75}};
    spec.n_grid = {4000};
    spec.lf_grid = {0.1, 0.5};
    spec.positive_ratios = {1.0, 0.0};
    spec.trials = 2;
    spec.seed = 42;
    experiment_result res = run_experiment(spec);
    CHECK(res.records.size() == 12 && !res.any_budget_exhausted() && res.wall_seconds > 0.0);
    for (std::size_t i = 0; i < res.records.size(); ++i) {
      const result_record& r = res.records[i];
      const bool iht = i >= 6;
      CHECK(r.kind == (iht ? table_kind::iht : table_kind::bcht) && r.b == 16 && r.n == 4000 && r.seed == 42);
      CHECK(r.threshold_pct.has_value() == iht && (!iht || *r.threshold_pct == 75));
      CHECK(r.successes == 2 && r.failures == 0 && r.ops_per_sec > 0.0);
      CHECK(r.op == (i % 3 == 0 ? "insert" : "find"));
      CHECK(r.positive_ratio.has_value() == (i % 3 != 0));
      if (i % 3 == 1) CHECK(*r.positive_ratio == 1.0);
      if (i % 3 == 2) CHECK(*r.positive_ratio == 0.0);
      if (!iht && i < 3) CHECK(r.mean_probes == 1.0);           // bcht at load factor 0.1: one probe, whatever the op
      if (iht && i % 3 == 2) CHECK(r.mean_probes == 3.0);       // iht negative queries read all three buckets
      if (iht && i % 3 == 1) CHECK(r.mean_probes >= 1.0 && r.mean_probes < 1.5);
    }
    CHECK(res.records[0].realized_lf < res.records[3].realized_lf);  // lf grid order inside a kind
    // the same cell through run_trial directly: same seed derivation -> same table geometry, same probe means (up to the
    // order in which concurrent claims land)
    trial_cell cell;
    cell.params = spec.kinds[1]; cell.n = 4000; cell.lf = 0.5; cell.positive_ratios = spec.positive_ratios; cell.trials = 2;
    cell.seed = cell_seed(42, 3);
    trial_outcome o = run_trial(cell);
    CHECK(std::fabs(o.find_mean_probes[0] - res.records[10].mean_probes) < 0.02 && o.realized_lf == res.records[9].realized_lf);
    std::ostringstream csv;
    write_csv(csv, res);
    const std::string text = csv.str();
    CHECK(text.rfind(std::string(result_csv_header) + "\n", 0) == 0);
    CHECK(static_cast<std::size_t>(std::count(text.begin(), text.end(), '\n')) == 13);
    CHECK(text.find("\niht,16,75,4000,") != std::string::npos && text.find("\nbcht,16,,4000,") != std::string::npos);
    spec.scen = scenario::success_rate;
    spec.lf_grid = {0.01, 0.5};
    spec.success_trials = 5;
    experiment_result sr = run_experiment(spec);
    CHECK(sr.records.size() == 4);
    for (const result_record& r : sr.records) CHECK(r.op == "build" && r.successes == 5 && r.failures == 0 && !r.positive_ratio);
    experiment_spec bad;
    CHECK(throws<std::invalid_argument>([&] { run_experiment(bad); }));
  }
  // set_blocked_insert is part of the handle API (host batches are always staged in caller order; the device-resident
  // schedules are covered by tests/test_gpu_parity.py::test_build_parity_routed)
  {
    table_config cfg = make_config(table_kind::bcht, n, 0.9, 16, std::nullopt, 9);
    for (int mode : {0, 2, 3}) {
      hash_table t(cfg);
      t.set_blocked_insert(mode);
      std::vector<value_type> vals(n), out(n);
      for (std::uint64_t i = 0; i < n; ++i) vals[i] = value_for_key(keys[i]);
      build_outcome o = t.insert(keys.data(), vals.data(), n);
      CHECK(o.success && t.count_inadmissible() == 0);
      t.find(keys.data(), out.data(), n);
      CHECK(out == vals);
    }
  }
  // the chunked build through the C++ layer: host keys copied to the device in three pieces, fed, ended
  {
    table_config cfg = make_config(table_kind::bcht, n, 0.9, 16, std::nullopt, 10);
    hash_table t(cfg);
    t.set_blocked_insert(3);
    t.set_repair(true);
    std::vector<value_type> vals(n), out(n);
    for (std::uint64_t i = 0; i < n; ++i) vals[i] = value_for_key(keys[i]);
    key_type* dk = nullptr;
    CHECK(cudaMalloc(reinterpret_cast<void**>(&dk), n * sizeof(key_type)) == cudaSuccess);
    CHECK(cudaMemcpy(dk, keys.data(), n * sizeof(key_type), cudaMemcpyHostToDevice) == cudaSuccess);
    t.build_begin(n);
    CHECK(throws<std::invalid_argument>([&] { t.insert(keys.data(), vals.data(), 4); }));  // a chunked build is open
    const std::uint64_t cut1 = n / 3, cut2 = n / 2 + 1;
    t.build_feed(dk, nullptr, cut1);
    t.build_feed(dk + cut1, nullptr, cut2 - cut1);
    t.build_feed(dk + cut2, nullptr, n - cut2);
    build_outcome o = t.build_end();
    CHECK(o.success && o.inserted == n && t.last_build_schedule() == 3 && t.count_inadmissible() == 0);
    t.find(keys.data(), out.data(), n);
    CHECK(out == vals);
    cudaFree(dk);
  }
  std::puts("wrapper checks ok");
  return 0;
}
