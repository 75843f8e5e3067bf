// hash_stage.cuh — the hash stage: h(k; a, b) = ((a*k + b) mod 4294967291) mod L
//
// Replaces bucket_index (reference: proj/include/bht/hash.hpp:21-23), which evaluates the formula
// with two 64-bit `%`.  Here it is division-free and bit-identical:
//
//   mod p   p = 2^32 - 5, so 2^32 = 5 (mod p).  x = a*k + b < 2^64 is folded twice,
//           x -> 5*hi(x) + lo(x) < 6*2^32 -> 5*hi + lo < 2^32 + 25, followed by ONE conditional
//           subtraction of p (z - p = z + 5 - 2^32, and z < 2p).
//   mod L   Lemire/Kaser/Kurz "fastmod": with M = ceil(2^64 / L), r mod L = mulhi64(M*r mod 2^64, L)
//           exactly for every 32-bit r and L.  M is precomputed on the host per hash function.
//
// The same code compiles for the host (bht_bucket_index_host) so the CPU tests can check the
// arithmetic against the oracle without a GPU.
#pragma once
#include <cstdint>

namespace bht_b200 {

constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint64_t kEmptySlot = 0xFFFFFFFFFFFFFFFFull;
constexpr uint64_t kPrime = 4294967291ull;

struct HashFn {
  uint32_t alpha;  // < 2^32 (the reference draws alpha in [1, p-1], keygen.cpp:20)
  uint32_t beta;   // < 2^32 (beta in [0, p-1], keygen.cpp:21)
  uint32_t range;  // L, 1 <= L < 2^32
  uint32_t pad;
  uint64_t magic;  // ceil(2^64 / L) mod 2^64  (0 when L == 1)
};

inline HashFn make_hash_fn(uint64_t alpha, uint64_t beta, uint64_t range) {
  HashFn h;
  h.alpha = static_cast<uint32_t>(alpha);
  h.beta = static_cast<uint32_t>(beta);
  h.range = static_cast<uint32_t>(range);
  h.pad = 0;
  h.magic = 0xFFFFFFFFFFFFFFFFull / range + 1ull;  // wraps to 0 for range == 1, which yields 0
  return h;
}

// (alpha*key + beta) mod p, result in [0, p).
__host__ __device__ __forceinline__ uint32_t linear_mod_prime(uint32_t alpha, uint32_t beta, uint32_t key) {
  const uint64_t x = static_cast<uint64_t>(alpha) * key + beta;                    // IMAD.WIDE
  const uint64_t y = (x >> 32) * 5ull + static_cast<uint32_t>(x);                  // < 6 * 2^32
  const uint64_t z = (y >> 32) * 5ull + static_cast<uint32_t>(y);                  // < 2^32 + 25
  uint32_t r = static_cast<uint32_t>(z);
  if (z >= kPrime) r += 5u;                                                        // z - p (mod 2^32)
  return r;
}

// r mod range via the precomputed 64-bit reciprocal; r, range < 2^32.
__host__ __device__ __forceinline__ uint32_t mod_range(uint32_t r, uint32_t range, uint64_t magic) {
  const uint64_t low = magic * r;  // mod 2^64
  const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(low)) * range;
  const uint64_t u = (low >> 32) * range + (t >> 32);  // no overflow: (2^32-1)^2 + 2^32 - 1 < 2^64
  return static_cast<uint32_t>(u >> 32);
}

__host__ __device__ __forceinline__ uint32_t bucket_index(const HashFn& h, uint32_t key) {
  return mod_range(linear_mod_prime(h.alpha, h.beta, key), h.range, h.magic);
}

// Shard routing of the multi-GPU table: owner = (g(k) * n_shards) >> 32, g = (a*k+b) mod p.
__host__ __device__ __forceinline__ uint32_t shard_of(uint32_t alpha, uint32_t beta, uint32_t n_shards, uint32_t key) {
  return static_cast<uint32_t>((static_cast<uint64_t>(linear_mod_prime(alpha, beta, key)) * n_shards) >> 32);
}

// splitmix64 / mix_seed / xorshift64 as in hash.hpp:25-62 (eviction victim choice).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream + 0x9E3779B97F4A7C15ull));
}
__host__ __device__ __forceinline__ uint64_t xorshift_init(uint64_t seed) {
  const uint64_t s = splitmix64(seed);
  return s ? s : 0xD1B54A32D192ED03ull;
}
__host__ __device__ __forceinline__ uint32_t xorshift_next_below(uint64_t& state, uint32_t bound) {
  uint64_t x = state;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  state = x;
  return static_cast<uint32_t>(((x >> 32) * bound) >> 32);
}

// next_below for the lanes that draw (`draw`); the others keep their state and get 0.
__host__ __device__ __forceinline__ uint32_t xorshift_next_below_if(uint64_t& state, uint32_t bound, bool draw) {
  uint64_t x = state;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  state = draw ? x : state;
  return draw ? static_cast<uint32_t>(((x >> 32) * bound) >> 32) : 0u;
}

// Synthetic workload (bht_generate_unique_keys): a keyed bijection of the 32-bit counter, every step
// invertible mod 2^32, cycle-walked once past the sentinel so that counters [0, 2^32-2] map one-to-one
// onto user keys [0, 2^32-2] (the key universe of core.hpp:23-24) without keygen.cpp's rejection set.
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t k0, uint32_t k1, uint32_t x) {
  x ^= k0;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x += k1;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}
__host__ __device__ __forceinline__ uint32_t unique_key(uint32_t k0, uint32_t k1, uint32_t counter) {
  uint32_t y = mix32(k0, k1, counter);
  if (y == kEmptyKey) y = mix32(k0, k1, y);  // the sentinel is no fixed point unless nothing maps to it
  return y;
}
// value_for_key (reference: proj/include/bht/keygen.hpp:23-26): the value build() pairs with a key (table.cpp:234).
__host__ __device__ __forceinline__ uint32_t value_for_key(uint32_t key) {
  const uint32_t v = key ^ 0x5A5A5A5Au;
  return v == kEmptyKey ? (v & 0x7FFFFFFFu) : v;
}
// A value stream independent of the key bijection, never the sentinel.
__host__ __device__ __forceinline__ uint32_t synthetic_value(uint32_t k1, uint32_t key) {
  const uint32_t v = mix32(k1 ^ 0x9E3779B9u, 0x7F4A7C15u, key);
  return v == kEmptyKey ? 0x5A5A5A5Au : v;
}

}  // namespace bht_b200
