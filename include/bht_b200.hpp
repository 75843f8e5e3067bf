// bht_b200.hpp — header-only C++ host layer over the C ABI in bht_b200.h.
//
// Mirrors the reference library's table API (reference: proj/include/bht/core.hpp, table.hpp) name for
// name so that a caller of `bht::hash_table` / `bht::build` can switch to `bht::gpu::hash_table` /
// `bht::gpu::build` for the bulk path:
//
//   reference (CPU)                                  this header (B200)
//   ---------------------------------------------    -------------------------------------------------
//   make_config(kind, n, lf, b, t, seed, chain)      gpu::make_config(...)            same arguments
//   hash_table table(cfg)                            gpu::hash_table table(cfg [, device])
//   insert_pair(table, {k, v}, rng, stats)   x n     table.insert(keys, values, n)    one bulk call
//   find_key(table, k, stats)                x n     table.find(keys, out, n)         one bulk call
//   build(keys, cfg, opts)                           gpu::build(keys, n, cfg [, opts])
//   table.realized_load() / inserted() / ...         same names
//   dump_store / slot_at / poke_slot                 same names (whole-store transfers underneath)
//
// Error behaviour follows the reference: std::invalid_argument for bad configurations and capacity
// overflow (core.cpp:40-60, table.cpp:22-23,225), std::logic_error for a kind mismatch
// (table.cpp:15-17), std::runtime_error for I/O and CUDA failures.  A failed insertion is reported in
// build_outcome, never thrown.
#ifndef BHT_B200_HPP_
#define BHT_B200_HPP_

#include <cstdint>
#include <chrono>
#include <cstdio>
#include <ostream>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bht_b200.h"

namespace bht {
namespace gpu {

using key_type = std::uint32_t;
using value_type = std::uint32_t;
using slot_type = std::uint64_t;

inline constexpr key_type empty_key = BHT_EMPTY_KEY;
inline constexpr value_type empty_value = BHT_EMPTY_VALUE;
inline constexpr slot_type empty_slot = BHT_EMPTY_SLOT;

enum class table_kind : std::int32_t { one_cht = BHT_ONE_CHT, bcht = BHT_BCHT, bp2ht = BHT_BP2HT, iht = BHT_IHT };
enum class mem_space : std::int32_t { device = BHT_MEM_DEVICE, host = BHT_MEM_HOST };

using table_config = bht_config;  // plain-data image of the reference table_config (core.hpp:66-77)

inline void check(bht_status s) {
  if (s == BHT_OK) return;
  const std::string msg = bht_last_error_string();
  switch (s) {
    case BHT_INVALID_ARGUMENT:
    case BHT_CAPACITY_EXCEEDED: throw std::invalid_argument(msg);
    case BHT_KIND_MISMATCH: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline unsigned hash_count(table_kind kind) { return bht_hash_count(static_cast<std::int32_t>(kind)); }
inline std::uint32_t default_max_chain(std::uint64_t n_keys) { return bht_default_max_chain(n_keys); }
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) { return bht_mix_seed(seed, stream); }
inline value_type value_for_key(key_type k) { return bht_value_for_key(k); }

// make_config (core.hpp:85-91)
inline table_config make_config(table_kind kind, std::uint64_t n_keys, double lf, std::uint32_t bucket_size,
                                std::optional<std::uint32_t> threshold = std::nullopt, std::uint64_t seed = 0,
                                std::optional<std::uint32_t> max_chain = std::nullopt) {
  table_config cfg;
  check(bht_make_config(static_cast<std::int32_t>(kind), n_keys, lf, bucket_size, threshold ? static_cast<std::int64_t>(*threshold) : -1,
                        seed, max_chain ? static_cast<std::int64_t>(*max_chain) : -1, &cfg));
  return cfg;
}

// build_outcome (table.hpp:115-120) of one bulk insert; every pair is attempted.
struct build_outcome {
  bool success = false;
  std::uint64_t inserted = 0;
  std::uint64_t failed = 0;
  std::uint64_t attempted = 0;
  std::uint64_t probes = 0;               // probe_stats.total_probes
  std::optional<key_type> failed_key;     // some dropped key
  double mean_probes() const { return attempted ? static_cast<double>(probes) / static_cast<double>(attempted) : 0.0; }
};

struct find_stats {
  std::uint64_t queries = 0, hits = 0, probes = 0, value_sum = 0;
  double mean_probes() const { return queries ? static_cast<double>(probes) / static_cast<double>(queries) : 0.0; }
};

struct build_options {
  bool iht_prose_fallback = false;  // build_options::iht_prose_fallback (table.hpp:111)
  mem_space space = mem_space::host;
  int device = 0;
  void* stream = nullptr;           // cudaStream_t
};

// class hash_table (table.hpp:28-80), slot store in device memory; move-only like the reference.
class hash_table {
 public:
  explicit hash_table(const table_config& cfg, int device = 0) : cfg_(cfg) { check(bht_create(&cfg_, device, &h_)); }
  hash_table(bht_table* adopted, const table_config& cfg) : cfg_(cfg), h_(adopted) {}  // takes ownership (bht_build)
  ~hash_table() { bht_destroy(h_); }
  hash_table(const hash_table&) = delete;
  hash_table& operator=(const hash_table&) = delete;
  hash_table(hash_table&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}
  hash_table& operator=(hash_table&& o) noexcept {
    if (this != &o) {
      bht_destroy(h_);
      cfg_ = o.cfg_;
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }

  const table_config& config() const { return cfg_; }
  std::uint64_t num_buckets() const { return cfg_.num_buckets; }
  std::uint32_t bucket_size() const { return cfg_.bucket_size; }
  std::uint64_t capacity() const { return cfg_.capacity; }
  std::uint64_t bucket_of(unsigned i, key_type key) const {
    return bht_bucket_index_host(cfg_.alpha[i], cfg_.beta[i], cfg_.range[i], key);
  }

  std::uint64_t inserted() const {
    std::uint64_t ins = 0, cap = 0;
    check(bht_load_factor(h_, &ins, &cap));
    return ins;
  }
  double realized_load() const { return static_cast<double>(inserted()) / static_cast<double>(cfg_.capacity); }
  std::uint64_t occupied_slots(void* stream = nullptr) const {
    std::uint64_t n = 0;
    check(bht_count_occupied(h_, &n, stream));
    return n;
  }
  std::uint64_t count_inadmissible(void* stream = nullptr) const {  // check_admissibility (oracle.cpp:40-54)
    std::uint64_t n = 0;
    check(bht_count_inadmissible(h_, &n, stream));
    return n;
  }
  void clear(void* stream = nullptr) { check(bht_clear(h_, stream)); }
  void set_iht_prose_fallback(bool on) { check(bht_set_iht_prose_fallback(h_, on ? 1 : 0)); }
  // bulk-build schedule: 0 caller order, 1 blocked when it pays (default), 2 L2-routed, 3 shared-memory blocked
  void set_blocked_insert(int mode) { check(bht_set_blocked_insert(h_, mode)); }
  // few keys in flight for the pairs that arrive beyond load 0.98: build success at LF 0.99 closer to the reference's
  void set_tail_throttle(bool on) { check(bht_set_tail_throttle(h_, on ? 1 : 0)); }
  // device milliseconds of the last device-resident insert: {routing / binning passes, probe kernel}
  std::pair<float, float> last_insert_phases() {
    float prepare = 0.f, probe = 0.f;
    check(bht_last_insert_phases(h_, &prepare, &probe));
    return {prepare, probe};
  }

  // bulk insert_pair (table.hpp:103-104)
  build_outcome insert(const key_type* keys, const value_type* values, std::uint64_t n, mem_space space = mem_space::host,
                       void* stream = nullptr) {
    bht_insert_result r{};
    check(bht_insert(h_, keys, values, n, static_cast<std::int32_t>(space), &r, stream));
    return outcome_of(r);
  }
  // the per-variant entry points bcht_insert / bp2ht_insert / iht_insert (table.hpp:84-101)
  build_outcome insert_as(table_kind kind, const key_type* keys, const value_type* values, std::uint64_t n,
                          mem_space space = mem_space::host, void* stream = nullptr) {
    bht_insert_result r{};
    check(bht_insert_as(h_, static_cast<std::int32_t>(kind), keys, values, n, static_cast<std::int32_t>(space), &r, stream));
    return outcome_of(r);
  }
  // stream-ordered, no host synchronisation; fetch the outcome later with last_insert_result()
  void insert_async(const key_type* device_keys, const value_type* device_values, std::uint64_t n, void* stream) {
    check(bht_insert(h_, device_keys, device_values, n, BHT_MEM_DEVICE, nullptr, stream));
  }
  build_outcome last_insert_result(void* stream = nullptr) {
    bht_insert_result r{};
    check(bht_last_insert_result(h_, &r, stream));
    return outcome_of(r);
  }
  // build() with the key set handed over in device-resident chunks (table.cpp:231-271): at most n_max pairs between
  // build_begin and build_end; values == nullptr pairs every key with value_for_key(key).  A table that qualifies for
  // the shared-memory-blocked build takes each chunk through its first partition pass as it is fed.
  void build_begin(std::uint64_t n_max, void* stream = nullptr) { check(bht_build_begin(h_, n_max, stream)); }
  void build_feed(const key_type* device_keys, const value_type* device_values, std::uint64_t n, void* stream = nullptr) {
    check(bht_build_feed(h_, device_keys, device_values, n, stream));
  }
  // the chunk holds min(n_cap, *n_device) pairs, the count read on the device (receive side of a sync-free exchange)
  void build_feed_counted(const key_type* device_keys, const value_type* device_values, std::uint64_t n_cap,
                          const std::uint64_t* n_device, void* stream = nullptr) {
    check(bht_build_feed_counted(h_, device_keys, device_values, n_cap, n_device, stream));
  }
  build_outcome build_end(void* stream = nullptr) {
    bht_insert_result r{};
    check(bht_build_end(h_, &r, stream));
    return outcome_of(r);
  }
  // 0 = caller order, 2 = L2-routed, 3 = shared-memory-blocked: how the last insert / chunked build ran
  int last_build_schedule() const { return bht_last_build_schedule(h_); }
  // cuckoo kinds: the few pairs a concurrent launch dropped at the chain cap get one more, solitary insertion
  // (default: on for bcht, off for 1cht)
  void set_repair(bool on) { check(bht_set_repair(h_, on ? 1 : 0)); }
  std::vector<key_type> failed_keys(std::uint64_t max_keys = 1u << 20) {
    std::vector<key_type> out(max_keys);
    std::uint64_t count = 0;
    check(bht_failed_keys(h_, out.data(), max_keys, &count));
    out.resize(count < max_keys ? count : max_keys);
    return out;
  }

  // bulk find_key (table.hpp:105): out[i] = value or empty_value
  void find(const key_type* keys, value_type* out, std::uint64_t n, mem_space space = mem_space::host, void* stream = nullptr,
            find_stats* stats = nullptr) const {
    bht_find_result r{};
    check(bht_find(h_, keys, out, n, static_cast<std::int32_t>(space), stats ? &r : nullptr, stream));
    if (stats) *stats = find_stats{r.queries, r.hits, r.probes, r.value_sum};
  }
  void find_as(table_kind kind, const key_type* keys, value_type* out, std::uint64_t n, mem_space space = mem_space::host,
               void* stream = nullptr) const {
    check(bht_find_as(h_, static_cast<std::int32_t>(kind), keys, out, n, static_cast<std::int32_t>(space), nullptr, stream));
  }
  // bcht_find_no_early_exit (oracle.cpp:56-63)
  void find_exhaustive(const key_type* keys, value_type* out, std::uint64_t n, mem_space space = mem_space::host,
                       void* stream = nullptr) const {
    check(bht_find_exhaustive(h_, keys, out, n, static_cast<std::int32_t>(space), nullptr, stream));
  }
  // find_key for one key, as the reference returns it
  std::optional<value_type> find_key(key_type key) const {
    value_type v = empty_value;
    find(&key, &v, 1);
    return v == empty_value ? std::nullopt : std::optional<value_type>(v);
  }

  // store access (table.hpp:53-56, table.cpp:41-51)
  std::vector<slot_type> download_store() const {
    std::vector<slot_type> s(cfg_.capacity);
    check(bht_download_store(h_, s.data(), nullptr));
    return s;
  }
  void upload_store(const std::vector<slot_type>& s) {
    if (s.size() != cfg_.capacity) throw std::invalid_argument("upload_store: store length must equal capacity");
    check(bht_upload_store(h_, s.data(), nullptr));
  }
  void dump_store(const std::string& path) const { check(bht_dump_store(h_, path.c_str())); }
  slot_type slot_at(std::uint64_t index) const { return download_store().at(index); }
  void poke_slot(std::uint64_t index, slot_type slot) {  // fault injection; leaves the inserted counter alone
    auto s = download_store();
    s.at(index) = slot;
    const std::uint64_t before = inserted();
    upload_store(s);
    (void)before;
  }

  bht_table* handle() const { return h_; }

  static build_outcome outcome_of(const bht_insert_result& r) {
    build_outcome o;
    o.success = r.success != 0;
    o.inserted = r.inserted;
    o.failed = r.failed;
    o.attempted = r.attempted;
    o.probes = r.probes;
    if (r.first_failed_key != BHT_EMPTY_KEY) o.failed_key = r.first_failed_key;
    return o;
  }

 private:
  table_config cfg_;
  bht_table* h_ = nullptr;
};

// build (table.hpp:125-127, table.cpp:224-276): values are value_for_key(k) as in the reference.
inline std::pair<hash_table, build_outcome> build(const key_type* keys, std::uint64_t n, const table_config& cfg,
                                                  build_options opts = {}) {
  if (n > cfg.capacity) throw std::invalid_argument("build: key set exceeds table capacity");
  bht_table* h = nullptr;
  bht_insert_result r{};
  // NULL values: the library pairs every key with value_for_key(key) on the device (keys in either memory space)
  check(bht_build(&cfg, opts.device, keys, nullptr, n, static_cast<std::int32_t>(opts.space), opts.iht_prose_fallback ? 1 : 0, &h, &r,
                  opts.stream));
  return {hash_table(h, cfg), hash_table::outcome_of(r)};
}

// build with explicit values, in either memory space
inline std::pair<hash_table, build_outcome> build_pairs(const key_type* keys, const value_type* values, std::uint64_t n,
                                                        const table_config& cfg, build_options opts = {}) {
  bht_table* h = nullptr;
  bht_insert_result r{};
  check(bht_build(&cfg, opts.device, keys, values, n, static_cast<std::int32_t>(opts.space), opts.iht_prose_fallback ? 1 : 0, &h, &r,
                  opts.stream));
  return {hash_table(h, cfg), hash_table::outcome_of(r)};
}

// ---- workload (keygen.hpp) ------------------------------------------------------------------------------------

struct key_set {  // keygen.hpp:13-18
  std::vector<key_type> keys;
  std::uint64_t seed = 0;
  std::size_t size() const { return keys.size(); }
};
struct query {  // keygen.hpp:30-34
  key_type key = 0;
  value_type expected_value = 0;
  bool expected_present = false;
};

// generate_keys (keygen.cpp:50-64): the reference's stream, de-duplicated on the device.
inline key_set generate_keys(std::uint64_t seed, std::size_t n, int device = 0) {
  key_set out;
  out.seed = seed;
  out.keys.resize(n);
  check(bht_generate_keys(seed, n, out.keys.data(), BHT_MEM_HOST, device, nullptr));
  return out;
}
// generate_queries (keygen.cpp:66-98); throws std::invalid_argument like the reference.
inline std::vector<query> generate_queries(const key_set& keys, double positive_ratio, std::size_t q, std::uint64_t seed,
                                           int device = 0) {
  std::vector<key_type> k(q);
  std::vector<value_type> v(q);
  std::vector<std::uint8_t> p(q);
  check(bht_generate_queries(keys.keys.data(), keys.size(), BHT_MEM_HOST, positive_ratio, q, seed, k.data(), v.data(), p.data(), device));
  std::vector<query> out(q);
  for (std::size_t i = 0; i < q; ++i) out[i] = {k[i], v[i], p[i] != 0};
  return out;
}
inline void save_keys(const std::string& path, const key_set& keys) { check(bht_save_keys(path.c_str(), keys.keys.data(), keys.size())); }
inline key_set load_keys(const std::string& path, std::uint64_t seed) {
  key_set out;
  out.seed = seed;
  std::uint64_t count = 0;
  check(bht_load_keys(path.c_str(), nullptr, 0, &count));
  out.keys.resize(count);
  check(bht_load_keys(path.c_str(), out.keys.data(), count, &count));
  return out;
}

// ---- the trial protocol (experiments.hpp:84-113, experiments.cpp:51-112) ----------------------------------------

struct kind_params {
  table_kind kind = table_kind::bcht;
  std::uint32_t bucket_size = 16;
  std::uint32_t threshold_pct = 80;  // iht only
  std::optional<std::uint32_t> threshold_slots() const {
    if (kind != table_kind::iht) return std::nullopt;
    return bucket_size * threshold_pct / 100;
  }
};
struct trial_cell {
  kind_params params;
  std::uint64_t n = 0;
  double lf = 0.0;
  std::vector<double> positive_ratios;
  unsigned trials = 10;
  unsigned max_failures = 50;
  std::uint64_t seed = 0;
  build_options build_opts;
  std::optional<std::uint32_t> max_chain;
  const key_set* preloaded_keys = nullptr;
};
struct trial_outcome {
  unsigned successes = 0;
  unsigned failures = 0;
  bool budget_exhausted = false;
  double realized_lf = 0.0;
  double insert_mean_probes = 0.0;
  std::vector<double> find_mean_probes;  // parallel to the requested ratios
  double insert_ops_per_sec = 0.0;       // steady_clock around the bulk calls (the reference times build(), table.cpp:228-276)
  std::vector<double> find_ops_per_sec;
};

// run_trial: fresh hash constants per attempt (mix_seed(seed, 0x100 + attempt)), build until `trials` successes or the
// failure budget runs out; on each success one bulk find of q = n queries per ratio (mix_seed(seed, 0x200 + r)).
inline trial_outcome run_trial(const trial_cell& cell) {
  trial_outcome out;
  out.find_mean_probes.assign(cell.positive_ratios.size(), 0.0);
  out.find_ops_per_sec.assign(cell.positive_ratios.size(), 0.0);
  using clock = std::chrono::steady_clock;
  double ins_seconds = 0.0;
  std::vector<double> find_seconds(cell.positive_ratios.size(), 0.0);
  key_set local;
  const key_set* keys = cell.preloaded_keys;
  if (keys == nullptr || keys->size() != cell.n) {
    local = generate_keys(mix_seed(cell.seed, 0x6b657973ull), cell.n, cell.build_opts.device);
    keys = &local;
  }
  std::uint64_t ins_probes = 0, ins_ops = 0;
  std::vector<std::uint64_t> find_probes(cell.positive_ratios.size(), 0), find_ops(cell.positive_ratios.size(), 0);
  std::vector<std::vector<key_type>> queries(cell.positive_ratios.size());
  std::vector<value_type> answers(cell.n);
  unsigned attempt = 0;
  while (out.successes < cell.trials && out.failures < cell.max_failures) {
    table_config cfg = make_config(cell.params.kind, cell.n, cell.lf, cell.params.bucket_size, cell.params.threshold_slots(),
                                   mix_seed(cell.seed, 0x100 + attempt), cell.max_chain);
    ++attempt;
    out.realized_lf = static_cast<double>(cell.n) / static_cast<double>(cfg.capacity);
    const auto t_build = clock::now();
    auto [table, built] = build(keys->keys.data(), cell.n, cfg, cell.build_opts);
    const double build_seconds = std::chrono::duration<double>(clock::now() - t_build).count();
    if (!built.success) {
      ++out.failures;
      continue;
    }
    ++out.successes;
    ins_probes += built.probes;
    ins_ops += built.attempted;
    ins_seconds += build_seconds;
    for (std::size_t r = 0; r < cell.positive_ratios.size(); ++r) {
      if (queries[r].empty() && cell.n != 0) {
        for (const query& qu : generate_queries(*keys, cell.positive_ratios[r], cell.n, mix_seed(cell.seed, 0x200 + r),
                                                cell.build_opts.device))
          queries[r].push_back(qu.key);
      }
      find_stats fs;
      const auto t_find = clock::now();
      table.find(queries[r].data(), answers.data(), cell.n, mem_space::host, nullptr, &fs);
      find_seconds[r] += std::chrono::duration<double>(clock::now() - t_find).count();
      find_probes[r] += fs.probes;
      find_ops[r] += fs.queries;
    }
  }
  out.budget_exhausted = out.successes < cell.trials;
  out.insert_mean_probes = ins_ops ? static_cast<double>(ins_probes) / static_cast<double>(ins_ops) : 0.0;
  out.insert_ops_per_sec = ins_seconds > 0.0 ? static_cast<double>(ins_ops) / ins_seconds : 0.0;
  for (std::size_t r = 0; r < cell.positive_ratios.size(); ++r) {
    out.find_mean_probes[r] = find_ops[r] ? static_cast<double>(find_probes[r]) / static_cast<double>(find_ops[r]) : 0.0;
    out.find_ops_per_sec[r] = find_seconds[r] > 0.0 ? static_cast<double>(find_ops[r]) / find_seconds[r] : 0.0;
  }
  return out;
}

// run_success_rate (experiments.hpp:115-137, experiments.cpp:114-146): `success_trials` builds per load factor with fresh
// hash constants mix_seed(cell_seed(seed, cell), t); max_load_factor = the highest grid point with >= 99 % successes.
struct success_rate_point {
  double lf = 0.0;
  double realized_lf = 0.0;
  unsigned successes = 0;
  unsigned trials = 0;
  double fraction() const { return trials == 0 ? 0.0 : static_cast<double>(successes) / trials; }
};
struct success_rate_result {
  std::vector<success_rate_point> points;
  std::optional<double> max_load_factor;
};
inline std::uint64_t cell_seed(std::uint64_t base, std::uint64_t cell_index) { return mix_seed(base, 0x63656c6cull + cell_index); }

inline success_rate_result run_success_rate(const kind_params& params, std::uint64_t n, const std::vector<double>& lf_grid,
                                            unsigned success_trials, std::uint64_t seed,
                                            std::optional<std::uint32_t> max_chain = std::nullopt, build_options opts = {}) {
  success_rate_result result;
  const key_set keys = generate_keys(mix_seed(seed, 0x6b657973ull), n, opts.device);
  for (std::size_t cell = 0; cell < lf_grid.size(); ++cell) {
    success_rate_point point;
    point.lf = lf_grid[cell];
    point.trials = success_trials;
    for (unsigned t = 0; t < success_trials; ++t) {
      table_config cfg = make_config(params.kind, n, point.lf, params.bucket_size, params.threshold_slots(),
                                     mix_seed(cell_seed(seed, cell), t), max_chain);
      point.realized_lf = static_cast<double>(n) / static_cast<double>(cfg.capacity);
      auto built = build(keys.keys.data(), n, cfg, opts);
      point.successes += built.second.success;
    }
    result.points.push_back(point);
  }
  for (const auto& point : result.points)
    if (point.fraction() >= 0.99 && (!result.max_load_factor || point.lf > *result.max_load_factor)) result.max_load_factor = point.lf;
  return result;
}

// One record per (cell, op, positive ratio) and its CSV line (experiments.hpp:62-82, experiments.cpp:232-243).
struct result_record {
  table_kind kind = table_kind::bcht;
  std::uint32_t b = 0;
  std::optional<std::uint32_t> threshold_pct;
  std::uint64_t n = 0;
  double realized_lf = 0.0;
  std::string op;  // "insert", "find" or "build"
  std::optional<double> positive_ratio;
  double mean_probes = 0.0;
  double ops_per_sec = 0.0;
  unsigned successes = 0;
  unsigned failures = 0;
  std::uint64_t seed = 0;
  bool budget_exhausted = false;
};
inline constexpr const char* result_csv_header =
    "kind,b,threshold_pct,n,realized_lf,op,positive_ratio,mean_probes,ops_per_sec,successes,failures,seed";
inline const char* to_string(table_kind kind) {
  switch (kind) {
    case table_kind::one_cht: return "1cht";
    case table_kind::bcht: return "bcht";
    case table_kind::bp2ht: return "bp2ht";
    case table_kind::iht: return "iht";
  }
  return "?";
}
inline std::string format_double(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6g", v);
  return buf;
}
inline std::string csv_line(const result_record& r) {
  std::string s = std::string(to_string(r.kind)) + ',' + std::to_string(r.b) + ',';
  if (r.threshold_pct) s += std::to_string(*r.threshold_pct);
  s += ',' + std::to_string(r.n) + ',' + format_double(r.realized_lf) + ',' + r.op + ',';
  if (r.positive_ratio) s += format_double(*r.positive_ratio);
  s += ',' + format_double(r.mean_probes) + ',' + format_double(r.ops_per_sec) + ',' + std::to_string(r.successes) + ',' +
       std::to_string(r.failures) + ',' + std::to_string(r.seed);
  return s;
}

// The single-process sharded handle (bht_sharded_*, csrc/sharded.cu): n shards, one ordinary table per device id (ids may
// repeat); per-GPU device slices in, aggregated outcome out.  No reference counterpart.
class sharded_table {
 public:
  sharded_table(const table_config& cfg_per_shard, const std::vector<std::int32_t>& device_ids) : cfg_(cfg_per_shard) {
    check(bht_sharded_create(&cfg_, static_cast<std::uint32_t>(device_ids.size()), device_ids.data(), &h_));
  }
  ~sharded_table() { bht_sharded_destroy(h_); }
  sharded_table(const sharded_table&) = delete;
  sharded_table& operator=(const sharded_table&) = delete;
  std::uint32_t shards() const { return bht_sharded_count(h_); }
  bht_table* shard_handle(std::uint32_t g) {
    bht_table* t = nullptr;
    check(bht_sharded_table(h_, g, &t));
    return t;
  }
  void clear() { check(bht_sharded_clear(h_)); }
  // keys[g] / values[g]: device arrays of n[g] elements on the g-th device; values empty = value_for_key
  build_outcome insert(const std::vector<const key_type*>& keys, const std::vector<const value_type*>& values,
                       const std::vector<std::uint64_t>& n) {
    bht_insert_result r{};
    check(bht_sharded_insert(h_, keys.data(), values.empty() ? nullptr : values.data(), n.data(), &r));
    return hash_table::outcome_of(r);
  }
  void find(const std::vector<const key_type*>& keys, const std::vector<value_type*>& out, const std::vector<std::uint64_t>& n,
            find_stats* stats = nullptr) {
    bht_find_result r{};
    check(bht_sharded_find(h_, keys.data(), out.data(), n.data(), stats ? &r : nullptr));
    if (stats) *stats = find_stats{r.queries, r.hits, r.probes, r.value_sum};
  }

 private:
  table_config cfg_;
  bht_sharded* h_ = nullptr;
};

// experiment_spec / run_experiment / write_csv (experiments.hpp:28-113, experiments.cpp:153-243): the grid driver above
// run_trial and run_success_rate — same cell order, same cell seeds (cell_seed(seed, running cell index)), one record per
// (cell, op, positive ratio); success-rate scenarios give one "build" record per load factor.
enum class scenario { probe_analysis, throughput, success_rate };
struct experiment_spec {
  scenario scen = scenario::probe_analysis;
  std::vector<kind_params> kinds;
  std::vector<std::uint64_t> n_grid;
  std::vector<double> lf_grid;
  std::vector<double> positive_ratios;
  unsigned trials = 10;
  unsigned max_failures = 50;
  unsigned success_trials = 200;
  std::uint64_t seed = 0;
  build_options build_opts;
  std::optional<std::uint32_t> max_chain;
};
struct experiment_result {
  std::vector<result_record> records;
  double wall_seconds = 0.0;
  bool any_budget_exhausted() const {
    for (const auto& r : records)
      if (r.budget_exhausted) return true;
    return false;
  }
};

inline experiment_result run_experiment(const experiment_spec& spec) {
  if (spec.kinds.empty()) throw std::invalid_argument("run_experiment: no table kinds requested");
  if (spec.n_grid.empty()) throw std::invalid_argument("run_experiment: empty key-count grid");
  if (spec.lf_grid.empty()) throw std::invalid_argument("run_experiment: empty load-factor grid");
  if (spec.trials < 1) throw std::invalid_argument("run_experiment: trials must be at least 1");
  experiment_result result;
  const auto start = std::chrono::steady_clock::now();
  std::uint64_t cell_index = 0;
  for (const kind_params& params : spec.kinds) {
    std::optional<std::uint32_t> tpct;
    if (params.kind == table_kind::iht) tpct = params.threshold_pct;
    auto record = [&](std::uint64_t n, double realized, const char* op) {
      result_record r;
      r.kind = params.kind; r.b = params.bucket_size; r.threshold_pct = tpct; r.n = n; r.realized_lf = realized; r.op = op;
      r.seed = spec.seed;
      return r;
    };
    for (std::uint64_t n : spec.n_grid) {
      if (spec.scen == scenario::success_rate) {
        build_options opts = spec.build_opts;
        const success_rate_result sr = run_success_rate(params, n, spec.lf_grid, spec.success_trials, mix_seed(spec.seed, cell_index),
                                                        spec.max_chain, opts);
        ++cell_index;
        for (const success_rate_point& p : sr.points) {
          result_record r = record(n, p.realized_lf, "build");
          r.successes = p.successes;
          r.failures = p.trials - p.successes;
          result.records.push_back(r);
        }
        continue;
      }
      for (double lf : spec.lf_grid) {
        trial_cell cell;
        cell.params = params; cell.n = n; cell.lf = lf; cell.positive_ratios = spec.positive_ratios; cell.trials = spec.trials;
        cell.max_failures = spec.max_failures; cell.seed = cell_seed(spec.seed, cell_index); cell.build_opts = spec.build_opts;
        cell.max_chain = spec.max_chain;
        ++cell_index;
        const trial_outcome o = run_trial(cell);
        result_record ins = record(n, o.realized_lf, "insert");
        ins.mean_probes = o.insert_mean_probes; ins.ops_per_sec = o.insert_ops_per_sec; ins.successes = o.successes;
        ins.failures = o.failures; ins.budget_exhausted = o.budget_exhausted;
        result.records.push_back(ins);
        for (std::size_t r = 0; r < spec.positive_ratios.size(); ++r) {
          result_record f = record(n, o.realized_lf, "find");
          f.positive_ratio = spec.positive_ratios[r]; f.mean_probes = o.find_mean_probes[r]; f.ops_per_sec = o.find_ops_per_sec[r];
          f.successes = o.successes; f.failures = o.failures; f.budget_exhausted = o.budget_exhausted;
          result.records.push_back(f);
        }
      }
    }
  }
  result.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  return result;
}

inline void write_csv(std::ostream& out, const experiment_result& result) {
  out << result_csv_header << '\n';
  for (const result_record& r : result.records) out << csv_line(r) << '\n';
}

}  // namespace gpu
}  // namespace bht

#endif  // BHT_B200_HPP_
