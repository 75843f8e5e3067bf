// hash_stage.cuh — the hash stage: h(k; a, b) = ((a*k + b) mod 4294967291) mod L
//
// Replaces bucket_index (reference: proj/include/bht/hash.hpp:21-23), which evaluates the formula
// with two 64-bit `%`.  Here it is division-free and bit-identical:
//
//   mod p   p = 2^32 - 5, so 2^32 = 5 (mod p).  x = a*k + b < 2^64 is folded twice,
//           x -> 5*hi(x) + lo(x) < 6*2^32 -> 5*hi + lo < 2^32 + 25, followed by ONE conditional
//           subtraction of p (z - p = z + 5 - 2^32, and z < 2p).  On the device the three multiply-adds are
//           written with carry chains (mad.lo.cc / madc.hi), 10 integer instructions.
//   mod L   q' = mulhi32(r, floor(2^32 / L)) is floor(r / L) or one less (the reciprocal is short by less than
//           2^-32 per unit of r, and r < 2^32), so r - q'*L is in [0, 2L) and one unsigned min with itself
//           minus L finishes: 4 instructions (IMAD.HI, IMAD, VIADDMNMX), against 6 64-bit ones for Lemire's
//           exact 64-bit reciprocal.  The reciprocal is precomputed on the host per hash function.
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
  uint32_t recip;  // floor(2^32 / L), saturated to 2^32 - 1 for L == 1
  uint64_t pad;
};

inline HashFn make_hash_fn(uint64_t alpha, uint64_t beta, uint64_t range) {
  HashFn h;
  h.alpha = static_cast<uint32_t>(alpha);
  h.beta = static_cast<uint32_t>(beta);
  h.range = static_cast<uint32_t>(range);
  const uint64_t q = (1ull << 32) / range;
  h.recip = q > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(q);  // L == 1: r - (r - 1) = 1, then min(1, 0) = 0
  h.pad = 0;
  return h;
}

// (alpha*key + beta) mod p, result in [0, p).
__host__ __device__ __forceinline__ uint32_t linear_mod_prime(uint32_t alpha, uint32_t beta, uint32_t key) {
#ifdef __CUDA_ARCH__
  uint32_t lo, hi, ylo, yhi, zlo, carry;
  asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.u32 %1, %2, %3, 0;" : "=r"(lo), "=r"(hi) : "r"(alpha), "r"(key), "r"(beta));  // x
  asm("mad.lo.cc.u32 %0, %2, 5, %3;\n\tmadc.hi.u32 %1, %2, 5, 0;" : "=r"(ylo), "=r"(yhi) : "r"(hi), "r"(lo));  // y = 5*hi(x) + lo(x)
  asm("mad.lo.cc.u32 %0, %2, 5, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(zlo), "=r"(carry) : "r"(yhi), "r"(ylo));      // z = 5*hi(y) + lo(y)
  return (carry != 0u || zlo >= static_cast<uint32_t>(kPrime)) ? zlo + 5u : zlo;                                  // z - p (mod 2^32)
#else
  const uint64_t x = static_cast<uint64_t>(alpha) * key + beta;
  const uint64_t y = (x >> 32) * 5ull + static_cast<uint32_t>(x);                  // < 6 * 2^32
  const uint64_t z = (y >> 32) * 5ull + static_cast<uint32_t>(y);                  // < 2^32 + 25
  uint32_t r = static_cast<uint32_t>(z);
  if (z >= kPrime) r += 5u;                                                        // z - p (mod 2^32)
  return r;
#endif
}

// r mod range via the precomputed 32-bit reciprocal; r, range < 2^32.
__host__ __device__ __forceinline__ uint32_t mod_range(uint32_t r, uint32_t range, uint32_t recip) {
#ifdef __CUDA_ARCH__
  const uint32_t q = __umulhi(r, recip);
#else
  const uint32_t q = static_cast<uint32_t>((static_cast<uint64_t>(r) * recip) >> 32);
#endif
  const uint32_t rem = r - q * range;         // in [0, 2 * range)
  const uint32_t less = rem - range;          // wraps to a huge value when rem < range
  return rem < less ? rem : less;
}

__host__ __device__ __forceinline__ uint32_t bucket_index(const HashFn& h, uint32_t key) {
  return mod_range(linear_mod_prime(h.alpha, h.beta, key), h.range, h.recip);
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
