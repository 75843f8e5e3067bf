// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the UNMODIFIED reference library.  It is compiled, together with the
// reference's own src/table.cpp, src/keygen.cpp, src/oracle.cpp (and src/core.cpp when
// nlohmann/json.hpp can be found, else oracle/ref_core_min.cpp) taken where they lie under
// /root/reference/proj, into oracle/_ref/libbht_ref.so by oracle/Makefile.  No reference source
// is copied into this repository; this file only calls the reference's public API
// (proj/include/bht/*.hpp).  Used to (1) validate the plain-C restatement in bht_oracle.c,
// (2) generate tests/golden fixtures, (3) act as the CPU baseline (`cpu_baseline.kind = "reference"`).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <thread>
#include <vector>

#include "bht/core.hpp"
#include "bht/hash.hpp"
#include "bht/keygen.hpp"
#include "bht/oracle.hpp"
#include "bht/sector_model.hpp"
#include "bht/table.hpp"
#ifdef REF_HAS_EXPERIMENTS  // src/experiments.cpp + src/core.cpp need nlohmann/json.hpp (oracle/Makefile)
#include <sstream>

#include "bht/experiments.hpp"
#endif

namespace {

struct pod_config {  // == bht_config (include/bht_b200.h) == or_config (oracle/bht_oracle.h)
  std::int32_t kind;
  std::uint32_t bucket_size;
  std::uint64_t num_buckets;
  std::uint64_t capacity;
  std::uint32_t n_hashes;
  std::uint32_t threshold;
  std::uint32_t max_chain;
  std::uint32_t reserved;
  std::uint64_t seed;
  std::uint64_t alpha[4];
  std::uint64_t beta[4];
  std::uint64_t range[4];
};

bht::table_config to_ref(const pod_config& p) {
  bht::table_config c;
  c.kind = static_cast<bht::table_kind>(p.kind);
  c.bucket_size = p.bucket_size;
  c.num_buckets = p.num_buckets;
  c.capacity = p.capacity;
  c.threshold = p.threshold;
  c.max_chain = p.max_chain;
  c.seed = p.seed;
  for (std::uint32_t i = 0; i < p.n_hashes && i < 4; ++i)
    c.hashes.push_back(bht::hash_params{p.alpha[i], p.beta[i], p.range[i]});
  return c;
}

void from_ref(const bht::table_config& c, pod_config* p) {
  std::memset(p, 0, sizeof *p);
  p->kind = static_cast<std::int32_t>(c.kind);
  p->bucket_size = c.bucket_size;
  p->num_buckets = c.num_buckets;
  p->capacity = c.capacity;
  p->n_hashes = static_cast<std::uint32_t>(c.hashes.size());
  p->threshold = c.threshold;
  p->max_chain = c.max_chain;
  p->seed = c.seed;
  for (std::size_t i = 0; i < c.hashes.size() && i < 4; ++i) {
    p->alpha[i] = c.hashes[i].alpha;
    p->beta[i] = c.hashes[i].beta;
    p->range[i] = c.hashes[i].range;
  }
}

struct ref_table {
  bht::hash_table table;
  explicit ref_table(bht::hash_table&& t) : table(std::move(t)) {}
};

}  // namespace

// The library is compiled with -fvisibility=hidden so that the reference's (and nlohmann's) inline functions bind
// inside this .so — a process that also loads torch carries another nlohmann::json with the same symbol names.
#pragma GCC visibility push(default)
extern "C" {

std::size_t ref_sizeof_config() { return sizeof(pod_config); }

std::uint64_t ref_bucket_index(std::uint64_t alpha, std::uint64_t beta, std::uint64_t range, std::uint32_t key) {
  return bht::bucket_index(bht::hash_params{alpha, beta, range}, key);
}
std::uint64_t ref_splitmix64(std::uint64_t x) { return bht::splitmix64(x); }
std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t stream) { return bht::mix_seed(seed, stream); }
void ref_xorshift_stream(std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
  bht::xorshift_rng rng(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.next();
}
void ref_next_below_stream(std::uint64_t seed, std::uint32_t bound, std::uint64_t n, std::uint32_t* out) {
  bht::xorshift_rng rng(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.next_below(bound);
}
std::uint32_t ref_hash_count(std::int32_t kind) { return bht::hash_count(static_cast<bht::table_kind>(kind)); }
std::uint32_t ref_default_max_chain(std::uint64_t n) { return bht::default_max_chain(n); }
std::uint64_t ref_pack_pair(std::uint32_t k, std::uint32_t v) { return bht::pack_pair({k, v}); }
std::uint32_t ref_value_for_key(std::uint32_t k) { return bht::value_for_key(k); }
double ref_predict_sectors(std::int32_t kind, std::uint32_t b, double probes, std::int32_t op) {
  return bht::predict_sectors(static_cast<bht::table_kind>(kind), b, probes,
                              op == 0 ? bht::op_kind::insert : bht::op_kind::find);
}
std::uint32_t ref_bucket_sectors(std::uint32_t b) { return bht::sector_model::bucket_sectors(b); }

// 0 ok, 1 std::invalid_argument
int ref_make_config(std::int32_t kind, std::uint64_t n, double lf, std::uint32_t b, std::int64_t threshold,
                    std::uint64_t seed, std::int64_t max_chain, pod_config* out) {
  try {
    std::optional<std::uint32_t> t = threshold >= 0 ? std::optional<std::uint32_t>(static_cast<std::uint32_t>(threshold)) : std::nullopt;
    std::optional<std::uint32_t> mc = max_chain >= 0 ? std::optional<std::uint32_t>(static_cast<std::uint32_t>(max_chain)) : std::nullopt;
    from_ref(bht::make_config(static_cast<bht::table_kind>(kind), n, lf, b, t, seed, mc), out);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

void ref_generate_keys(std::uint64_t seed, std::uint64_t n, std::uint32_t* out) {
  bht::key_set ks = bht::generate_keys(seed, n);
  std::memcpy(out, ks.keys.data(), n * sizeof(std::uint32_t));
}

// generate_queries (keygen.cpp:66-98). Returns 0, or 1 on invalid_argument.
int ref_generate_queries(const std::uint32_t* keys, std::uint64_t n, double ratio, std::uint64_t q, std::uint64_t seed,
                         std::uint32_t* out_keys, std::uint32_t* out_expected, std::uint8_t* out_present) {
  try {
    bht::key_set ks;
    ks.keys.assign(keys, keys + n);
    auto qs = bht::generate_queries(ks, ratio, q, seed);
    for (std::uint64_t i = 0; i < q; ++i) {
      out_keys[i] = qs[i].key;
      if (out_expected) out_expected[i] = qs[i].expected_present ? qs[i].expected_value : bht::empty_value;
      if (out_present) out_present[i] = qs[i].expected_present;
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

ref_table* ref_table_create(const pod_config* cfg) {
  try {
    return new ref_table(bht::hash_table(to_ref(*cfg)));
  } catch (const std::exception&) {
    return nullptr;
  }
}
void ref_table_destroy(ref_table* t) { delete t; }
std::uint64_t ref_table_inserted(const ref_table* t) { return t->table.inserted(); }
std::uint64_t ref_occupied_slots(const ref_table* t) { return t->table.occupied_slots(); }
std::uint64_t ref_slot_at(const ref_table* t, std::uint64_t i) { return t->table.slot_at(i); }
void ref_poke_slot(ref_table* t, std::uint64_t i, std::uint64_t s) { t->table.poke_slot(i, s); }
void ref_download_store(const ref_table* t, std::uint64_t* dst) {
  for (std::uint64_t i = 0; i < t->table.capacity(); ++i) dst[i] = t->table.slot_at(i);
}
// poke_slot over the whole store. `inserted` is not adjusted (the reference has no setter).
void ref_upload_store(ref_table* t, const std::uint64_t* src) {
  for (std::uint64_t i = 0; i < t->table.capacity(); ++i) t->table.poke_slot(i, src[i]);
}

std::uint64_t ref_rng_init(std::uint64_t) { return 0; }  // rng state is held inside ref_rng below

struct ref_rng {
  bht::xorshift_rng rng;
  explicit ref_rng(std::uint64_t seed) : rng(seed) {}
};
ref_rng* ref_rng_create(std::uint64_t seed) { return new ref_rng(seed); }
void ref_rng_destroy(ref_rng* r) { delete r; }

// insert_pair (table.cpp:203-212): 1 inserted, 0 failed, -1 logic_error
int ref_insert_pair(ref_table* t, std::uint32_t key, std::uint32_t value, ref_rng* rng, int prose, std::uint64_t* probes) {
  try {
    bht::probe_stats st{bht::op_kind::insert};
    bool ok = bht::insert_pair(t->table, {key, value}, rng->rng, st, prose != 0);
    if (probes) *probes += st.total_probes;
    return ok ? 1 : 0;
  } catch (const std::logic_error&) {
    return -1;
  }
}

// Explicit per-variant entry points so kind-mismatch behaviour (table.cpp:15-17) can be pinned.
int ref_variant_insert(ref_table* t, int variant, std::uint32_t key, std::uint32_t value, ref_rng* rng, int prose,
                       std::uint64_t* probes) {
  try {
    bht::probe_stats st{bht::op_kind::insert};
    bool ok = false;
    if (variant == 2) ok = bht::bp2ht_insert(t->table, {key, value}, st);
    else if (variant == 3) ok = bht::iht_insert(t->table, {key, value}, st, prose != 0);
    else ok = bht::bcht_insert(t->table, {key, value}, rng->rng, st);
    if (probes) *probes += st.total_probes;
    return ok ? 1 : 0;
  } catch (const std::logic_error&) {
    return -1;
  }
}

int ref_find_key(const ref_table* t, std::uint32_t key, std::uint32_t* value, std::uint64_t* probes) {
  bht::probe_stats st{bht::op_kind::find};
  auto v = bht::find_key(t->table, key, st);
  if (probes) *probes += st.total_probes;
  if (value) *value = v ? *v : bht::empty_value;
  return v ? 1 : 0;
}

int ref_find_key_no_early_exit(const ref_table* t, std::uint32_t key, std::uint32_t* value) {
  auto v = bht::bcht_find_no_early_exit(t->table, key);
  if (value) *value = v ? *v : bht::empty_value;
  return v ? 1 : 0;
}

// Sequential insert_pair loop with explicit values, one rng stream seeded like build()
// (table.cpp:232): stops at the first failure when stop_on_failure != 0.
std::int64_t ref_insert_pairs(ref_table* t, const std::uint32_t* keys, const std::uint32_t* values, std::uint64_t n,
                              int prose, int stop_on_failure, std::uint64_t* probes, std::uint8_t* failed_flags) {
  bht::xorshift_rng rng(bht::mix_seed(t->table.config().seed, 0x65766963ull));
  bht::probe_stats st{bht::op_kind::insert};
  std::int64_t ok = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    std::uint32_t v = values ? values[i] : bht::value_for_key(keys[i]);
    bool r = bht::insert_pair(t->table, {keys[i], v}, rng, st, prose != 0);
    ok += r;
    if (failed_flags) failed_flags[i] = !r;
    if (!r && stop_on_failure) break;
  }
  if (probes) *probes = st.total_probes;
  return ok;
}

// build() itself (table.cpp:224-276). mode 0 sequential, 1 parallel. Returns a new table handle
// (nullptr if build throws). out[0]=success out[1]=inserted out[2]=failed_key or ~0 out[3]=probes
// out[4]=elapsed nanoseconds of the build() call.
ref_table* ref_build(const std::uint32_t* keys, std::uint64_t n, const pod_config* cfg, int mode, unsigned workers,
                     int prose, std::uint64_t* out) {
  try {
    bht::key_set ks;
    ks.keys.assign(keys, keys + n);
    bht::build_options opts;
    opts.mode = mode ? bht::build_mode::parallel : bht::build_mode::sequential;
    opts.workers = workers;
    opts.iht_prose_fallback = prose != 0;
    bht::table_config c = to_ref(*cfg);
    auto t0 = std::chrono::steady_clock::now();
    auto built = bht::build(ks, c, opts);
    auto t1 = std::chrono::steady_clock::now();
    if (out) {
      out[0] = built.second.success;
      out[1] = built.second.inserted;
      out[2] = built.second.failed_key ? *built.second.failed_key : ~0ull;
      out[3] = built.second.probes.total_probes;
      out[4] = static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    }
    return new ref_table(std::move(built.first));
  } catch (const std::exception&) {
    return nullptr;
  }
}

// The caller-side find loop (experiments.cpp:92), optionally chunked over `threads` host threads
// (harness-side threading; the reference itself has no parallel find). Returns hits.
std::uint64_t ref_find_bulk(const ref_table* t, const std::uint32_t* keys, std::uint64_t n, std::uint32_t* out,
                            unsigned threads, std::uint64_t* probes, std::uint64_t* elapsed_ns) {
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = static_cast<unsigned>(std::min<std::uint64_t>(threads, std::max<std::uint64_t>(n, 1)));
  std::vector<std::uint64_t> hits(threads, 0), pr(threads, 0);
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&](unsigned w) {
    const std::uint64_t chunk = (n + threads - 1) / threads;
    const std::uint64_t lo = std::min<std::uint64_t>(w * chunk, n), hi = std::min<std::uint64_t>(lo + chunk, n);
    bht::probe_stats st{bht::op_kind::find};
    std::uint64_t h = 0;
    for (std::uint64_t i = lo; i < hi; ++i) {
      auto v = bht::find_key(t->table, keys[i], st);
      h += v.has_value();
      if (out) out[i] = v ? *v : bht::empty_value;
    }
    hits[w] = h;
    pr[w] = st.total_probes;
  };
  if (threads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < threads; ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  auto t1 = std::chrono::steady_clock::now();
  std::uint64_t h = 0, p = 0;
  for (unsigned w = 0; w < threads; ++w) {
    h += hits[w];
    p += pr[w];
  }
  if (probes) *probes = p;
  if (elapsed_ns) *elapsed_ns = static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
  return h;
}

// check_membership (oracle.cpp:13-38): out = {false_negatives, wrong_values, false_positives}.
// Values must be value_for_key(k), as the reference's reference_map assumes.
void ref_check_membership(const ref_table* t, const std::uint32_t* keys, std::uint64_t n, std::uint64_t n_negative,
                          std::uint64_t seed, std::uint64_t* out) {
  bht::key_set ks;
  ks.keys.assign(keys, keys + n);
  auto rep = bht::check_membership(t->table, ks, n_negative, seed);
  out[0] = rep.false_negatives;
  out[1] = rep.wrong_values;
  out[2] = rep.false_positives;
}

std::uint64_t ref_check_admissibility(const ref_table* t) { return bht::check_admissibility(t->table); }

unsigned ref_hardware_concurrency() { return std::max(1u, std::thread::hardware_concurrency()); }


// ---- experiment protocol and wire formats (experiments.cpp, core.cpp:70-109); 0 when compiled without them ----
int ref_has_experiments() {
#ifdef REF_HAS_EXPERIMENTS
  return 1;
#else
  return 0;
#endif
}

#ifdef REF_HAS_EXPERIMENTS
static std::size_t copy_out(const std::string& text, char* buf, std::size_t cap) {
  if (buf != nullptr && cap != 0) {
    const std::size_t k = std::min(cap - 1, text.size());
    std::memcpy(buf, text.data(), k);
    buf[k] = 0;
  }
  return text.size();
}

// config_to_json; returns the text length (call with a large enough buffer).
std::size_t ref_config_to_json(const pod_config* cfg, char* buf, std::size_t cap) {
  return copy_out(bht::config_to_json(to_ref(*cfg)), buf, cap);
}
int ref_config_from_json(const char* text, pod_config* out) {
  try {
    from_ref(bht::config_from_json(text), out);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
// spec_to_json(spec_from_json(text)): the canonical form of an experiment spec.
std::size_t ref_spec_roundtrip(const char* text, char* buf, std::size_t cap) {
  try {
    return copy_out(bht::spec_to_json(bht::spec_from_json(text)), buf, cap);
  } catch (const std::exception&) {
    return 0;
  }
}
// run_experiment(spec_from_json(text)) on the CPU, written with write_csv (format 0) or write_json (format 1).
std::size_t ref_run_experiment(const char* spec_json, int format, char* buf, std::size_t cap) {
  try {
    bht::experiment_result r = bht::run_experiment(bht::spec_from_json(spec_json));
    std::ostringstream out;
    if (format == 0) bht::write_csv(out, r); else bht::write_json(out, r);
    return copy_out(out.str(), buf, cap);
  } catch (const std::exception&) {
    return 0;
  }
}
// run_trial: out = {successes, failures, budget_exhausted, realized_lf, insert_mean_probes, find_mean_probes[n_ratios]}
int ref_run_trial(std::int32_t kind, std::uint32_t b, std::uint32_t threshold_pct, std::uint64_t n, double lf,
                  const double* ratios, std::uint32_t n_ratios, unsigned trials, unsigned max_failures, std::uint64_t seed,
                  double* out) {
  try {
    bht::trial_cell cell;
    cell.params = {static_cast<bht::table_kind>(kind), b, threshold_pct};
    cell.n = n;
    cell.lf = lf;
    cell.positive_ratios.assign(ratios, ratios + n_ratios);
    cell.trials = trials;
    cell.max_failures = max_failures;
    cell.seed = seed;
    bht::trial_outcome o = bht::run_trial(cell);
    out[0] = o.successes, out[1] = o.failures, out[2] = o.budget_exhausted, out[3] = o.realized_lf, out[4] = o.insert_mean_probes;
    for (std::uint32_t r = 0; r < n_ratios; ++r) out[5 + r] = o.find_mean_probes[r];
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
// run_success_rate: successes per grid point.
int ref_run_success_rate(std::int32_t kind, std::uint32_t b, std::uint32_t threshold_pct, std::uint64_t n, const double* lf_grid,
                         std::uint32_t n_lf, unsigned success_trials, std::uint64_t seed, std::uint32_t* successes) {
  try {
    auto r = bht::run_success_rate({static_cast<bht::table_kind>(kind), b, threshold_pct}, n,
                                   std::vector<double>(lf_grid, lf_grid + n_lf), success_trials, seed);
    for (std::uint32_t i = 0; i < n_lf; ++i) successes[i] = r.points[i].successes;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
#endif
}
#pragma GCC visibility pop
