// ref_core_min.cpp — TEST INFRASTRUCTURE ONLY; FALLBACK translation unit.
//
// The reference's src/core.cpp needs <nlohmann/json.hpp> for its config-JSON helpers.  When that
// header cannot be found, oracle/Makefile links this file instead of core.cpp.  It supplies only
// the four core.cpp symbols the hot path links against (to_string, parse_table_kind,
// default_max_chain, make_config; core.cpp:10-68) by forwarding to the plain-C restatement in
// bht_oracle.c, and reports through ref_core_is_reference() that make_config is then NOT the
// reference's own code (tests skip the make_config cross-check in that case).
#include <stdexcept>

#include "bht/core.hpp"
#include "bht_oracle.h"

namespace bht {

const char* to_string(table_kind kind) {
  static const char* names[] = {"1cht", "bcht", "bp2ht", "iht"};
  auto i = static_cast<unsigned>(kind);
  return i < 4 ? names[i] : "?";
}

std::optional<table_kind> parse_table_kind(const std::string& name) {
  for (int i = 0; i < 4; ++i)
    if (name == to_string(static_cast<table_kind>(i))) return static_cast<table_kind>(i);
  return std::nullopt;
}

std::uint32_t default_max_chain(std::uint64_t n_keys) { return or_default_max_chain(n_keys); }

table_config make_config(table_kind kind, std::uint64_t n_keys, double lf, std::uint32_t bucket_size,
                         std::optional<std::uint32_t> threshold, std::uint64_t seed,
                         std::optional<std::uint32_t> max_chain) {
  or_config c;
  if (or_make_config(static_cast<int>(kind), n_keys, lf, bucket_size, threshold ? static_cast<std::int64_t>(*threshold) : -1,
                     seed, max_chain ? static_cast<std::int64_t>(*max_chain) : -1, &c))
    throw std::invalid_argument("make_config: invalid argument");
  table_config out;
  out.kind = kind;
  out.num_buckets = c.num_buckets;
  out.bucket_size = c.bucket_size;
  out.capacity = c.capacity;
  out.threshold = c.threshold;
  out.max_chain = c.max_chain;
  out.seed = c.seed;
  for (std::uint32_t i = 0; i < c.n_hashes; ++i) out.hashes.push_back(hash_params{c.alpha[i], c.beta[i], c.range[i]});
  return out;
}

}  // namespace bht

extern "C" __attribute__((visibility("default"))) int ref_core_is_reference() { return 0; }
