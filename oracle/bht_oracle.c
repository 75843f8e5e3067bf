/*
 * bht_oracle.c — TEST INFRASTRUCTURE ONLY (see bht_oracle.h).
 *
 * CPU restatement, in plain C, of the reference algorithm for the bulk insert / bulk find path.
 * Each function cites the reference lines it follows (paths relative to /root/reference/proj).
 * Single-threaded and deliberately simple: one pass over memory per probe, real 64-bit `%`.
 * Parity pinned against the reference's golden vectors and oracle/_ref (tests/test_oracle_*.py).
 */
#include "bht_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { K_ONE_CHT = 0, K_BCHT = 1, K_BP2HT = 2, K_IHT = 3 };

struct or_table {
  or_config cfg;
  uint64_t* store; /* capacity slots, bucket-major */
  uint64_t inserted;
};

/* ------------------------------------------------------------------ hash.hpp */

/* include/bht/hash.hpp:21-23 — ((alpha*key + beta) mod p) mod range in 64-bit arithmetic. */
uint64_t or_bucket_index(uint64_t alpha, uint64_t beta, uint64_t range, uint32_t key) {
  uint64_t lin = alpha * (uint64_t)key + beta;
  return (lin % OR_PRIME) % range;
}

/* include/bht/hash.hpp:25-30 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* include/bht/hash.hpp:33-35 */
uint64_t or_mix_seed(uint64_t seed, uint64_t stream) {
  return or_splitmix64(seed ^ or_splitmix64(stream + 0x9E3779B97F4A7C15ull));
}

/* include/bht/hash.hpp:41-43 — xorshift_rng constructor */
uint64_t or_rng_init(uint64_t seed) {
  uint64_t s = or_splitmix64(seed);
  return s ? s : 0xD1B54A32D192ED03ull;
}

/* include/bht/hash.hpp:45-52 — Marsaglia 13/7/17 */
static uint64_t rng_next(uint64_t* state) {
  uint64_t x = *state;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  *state = x;
  return x;
}

/* include/bht/hash.hpp:56-58 */
static uint32_t rng_next_below(uint64_t* state, uint32_t bound) {
  return (uint32_t)(((rng_next(state) >> 32) * (uint64_t)bound) >> 32);
}

void or_xorshift_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  uint64_t st = or_rng_init(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&st);
}

void or_next_below_stream(uint64_t seed, uint32_t bound, uint64_t n, uint32_t* out) {
  uint64_t st = or_rng_init(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng_next_below(&st, bound);
}

/* ------------------------------------------------------------------ core.hpp / core.cpp */

/* include/bht/core.hpp:49-57 */
uint32_t or_hash_count(int32_t kind) {
  switch (kind) {
    case K_ONE_CHT: return 4;
    case K_BCHT: return 3;
    case K_BP2HT: return 2;
    case K_IHT: return 3;
    default: return 0;
  }
}

/* src/core.cpp:28-31 — max(7 * ceil(log2 n), 128), ceil(log2 n) = bit_width(n-1), 1 for n <= 1 */
uint32_t or_default_max_chain(uint64_t n_keys) {
  uint32_t log2n = 1;
  if (n_keys > 1) {
    uint64_t v = n_keys - 1;
    log2n = 0;
    while (v) {
      ++log2n;
      v >>= 1;
    }
  }
  uint32_t c = 7u * log2n;
  return c > 128u ? c : 128u;
}

/* include/bht/core.hpp:35-37 */
uint64_t or_pack_pair(uint32_t key, uint32_t value) { return ((uint64_t)value << 32) | key; }

size_t or_sizeof_config(void) { return sizeof(or_config); }

static int is_pow2(uint32_t v) { return v != 0 && (v & (v - 1)) == 0; }

/* src/core.cpp:33-68 (make_config) with the hash-constant draw of src/keygen.cpp:14-26. */
int or_make_config(int32_t kind, uint64_t n_keys, double lf, uint32_t bucket_size, int64_t threshold,
                   uint64_t seed, int64_t max_chain, or_config* out) {
  if (kind < K_ONE_CHT || kind > K_IHT) return 1;
  if (n_keys == 0) return 1;                                          /* core.cpp:40 */
  if (!(lf > 0.0) || lf > 1.0) return 1;                              /* core.cpp:41 */
  if (bucket_size == 0 || bucket_size > 64 || !is_pow2(bucket_size)) return 1; /* core.cpp:42-43 */
  if (kind == K_ONE_CHT && bucket_size != 1) return 1;                /* core.cpp:44-45 */

  or_config c;
  memset(&c, 0, sizeof c);
  c.kind = kind;
  c.bucket_size = bucket_size;
  c.num_buckets = (uint64_t)ceil((double)n_keys / (lf * (double)bucket_size)); /* core.cpp:50-51 */
  c.capacity = c.num_buckets * bucket_size;
  c.seed = seed;
  if (kind == K_IHT) { /* core.cpp:55-61 */
    c.threshold = threshold >= 0 ? (uint32_t)threshold : bucket_size * 80u / 100u;
    if (c.threshold > bucket_size) return 1;
    if (c.threshold == 0) return 1;
  }
  if (kind == K_ONE_CHT || kind == K_BCHT) /* core.cpp:62-63 */
    c.max_chain = max_chain >= 0 ? (uint32_t)max_chain : or_default_max_chain(n_keys);

  /* core.cpp:65-66 + keygen.cpp:14-26: alpha = 1 + next_below(p-1), beta = next_below(p) */
  uint64_t st = or_rng_init(or_mix_seed(seed, 0x68617368ull));
  const uint32_t p32 = (uint32_t)OR_PRIME;
  c.n_hashes = or_hash_count(kind);
  for (uint32_t i = 0; i < c.n_hashes; ++i) {
    c.alpha[i] = 1u + (uint64_t)rng_next_below(&st, p32 - 1u);
    c.beta[i] = rng_next_below(&st, p32);
    c.range[i] = c.num_buckets;
  }
  *out = c;
  return 0;
}

/* ------------------------------------------------------------------ keygen */

/* include/bht/keygen.hpp:23-26 */
uint32_t or_value_for_key(uint32_t key) {
  uint32_t v = key ^ 0x5A5A5A5Au;
  return v == 0xFFFFFFFFu ? (v & 0x7FFFFFFFu) : v;
}

/* std::mt19937_64 (Matsumoto & Nishimura 2004, the engine keygen.cpp:54 instantiates). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

void or_mt19937_64_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

/* src/keygen.cpp:50-64 — top 32 bits of each draw, sentinel and repeats rejected, first
 * occurrence order kept.  The std::unordered_set is replaced by an open-addressing set. */
void or_generate_keys(uint64_t seed, uint64_t n, uint32_t* out) {
  if (n == 0) return;
  uint64_t cap = 16;
  while (cap < n * 2) cap <<= 1;
  uint32_t* set = (uint32_t*)malloc(cap * sizeof(uint32_t));
  memset(set, 0xFF, cap * sizeof(uint32_t));
  mt64 g;
  mt64_seed(&g, seed);
  uint64_t have = 0;
  while (have < n) {
    uint32_t k = (uint32_t)(mt64_next(&g) >> 32);
    if (k == OR_EMPTY_KEY) continue;
    uint64_t pos = (k * 0x9E3779B97F4A7C15ull) >> 11 & (cap - 1);
    int dup = 0;
    while (set[pos] != OR_EMPTY_KEY) {
      if (set[pos] == k) {
        dup = 1;
        break;
      }
      pos = (pos + 1) & (cap - 1);
    }
    if (dup) continue;
    set[pos] = k;
    out[have++] = k;
  }
  free(set);
}

/* ------------------------------------------------------------------ sector model */

/* include/bht/sector_model.hpp:18-20 */
uint32_t or_bucket_sectors(uint32_t bucket_size) { return (bucket_size * 8u + 31u) / 32u; }

/* include/bht/sector_model.hpp:26-31 */
double or_predict_sectors(int32_t kind, uint32_t bucket_size, double mean_probes, int32_t op) {
  double read_cost = kind == K_ONE_CHT ? 2.0 : (double)or_bucket_sectors(bucket_size);
  double sectors = mean_probes * read_cost;
  if (op == 0) sectors += 1.0;
  return sectors;
}

/* ------------------------------------------------------------------ table store */

/* src/table.cpp:21-32 — wrong hash count rejected, store filled with empty_slot. */
or_table* or_table_create(const or_config* cfg) {
  if (cfg->kind < K_ONE_CHT || cfg->kind > K_IHT) return NULL;
  if (cfg->n_hashes != or_hash_count(cfg->kind)) return NULL;
  or_table* t = (or_table*)malloc(sizeof(or_table));
  if (!t) return NULL;
  t->cfg = *cfg;
  t->inserted = 0;
  size_t bytes = (size_t)cfg->capacity * sizeof(uint64_t);
  t->store = (uint64_t*)malloc(bytes ? bytes : 8);
  if (!t->store) {
    free(t);
    return NULL;
  }
  memset(t->store, 0xFF, bytes);
  return t;
}

void or_table_destroy(or_table* t) {
  if (!t) return;
  free(t->store);
  free(t);
}

uint64_t or_table_inserted(const or_table* t) { return t->inserted; }

/* src/table.cpp:34-39 */
uint64_t or_occupied_slots(const or_table* t) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < t->cfg.capacity; ++i) c += (uint32_t)t->store[i] != OR_EMPTY_KEY;
  return c;
}

uint64_t or_slot_at(const or_table* t, uint64_t index) { return t->store[index]; }
void or_poke_slot(or_table* t, uint64_t index, uint64_t slot) { t->store[index] = slot; }
void or_download_store(const or_table* t, uint64_t* dst) {
  memcpy(dst, t->store, (size_t)t->cfg.capacity * 8);
}
void or_upload_store(or_table* t, const uint64_t* src) {
  memcpy(t->store, src, (size_t)t->cfg.capacity * 8);
  t->inserted = or_occupied_slots(t);
}

/* ------------------------------------------------------------------ bucket primitive */

static uint64_t* bucket_ptr(const or_table* t, uint64_t bucket_id) {
  return t->store + bucket_id * t->cfg.bucket_size;
}

static uint64_t hash_of(const or_table* t, unsigned i, uint32_t key) {
  return or_bucket_index(t->cfg.alpha[i], t->cfg.beta[i], t->cfg.range[i], key);
}

/* include/bht/bucket.hpp:26-31 over a bucket read (bucket.hpp:18-21 = one probe) */
static uint32_t bucket_load(const uint64_t* b, uint32_t size) {
  uint32_t load = 0;
  for (uint32_t i = 0; i < size; ++i) load += (uint32_t)b[i] != OR_EMPTY_KEY;
  return load;
}

/* include/bht/bucket.hpp:36-41 — lowest matching slot */
static int bucket_find(const uint64_t* b, uint32_t size, uint32_t key, uint32_t* value) {
  for (uint32_t i = 0; i < size; ++i)
    if ((uint32_t)b[i] == key) {
      *value = (uint32_t)(b[i] >> 32);
      return 1;
    }
  return 0;
}

/* include/bht/bucket.hpp:45-50 — single-threaded CAS(empty -> pair), returns prior contents */
static uint64_t bucket_cas(uint64_t* b, uint64_t pair, uint32_t slot) {
  uint64_t prior = b[slot];
  if (prior == OR_EMPTY_SLOT) b[slot] = pair;
  return prior;
}

/* include/bht/bucket.hpp:53-55 */
static uint64_t bucket_exch(uint64_t* b, uint64_t pair, uint32_t slot) {
  uint64_t prior = b[slot];
  b[slot] = pair;
  return prior;
}

/* ------------------------------------------------------------------ the four variants */

/* src/table.cpp:53-92 (bcht and one_cht) */
static int cuckoo_insert(or_table* t, uint32_t key, uint32_t value, uint64_t* rng, uint64_t* probes) {
  const unsigned h = t->cfg.n_hashes;
  const uint32_t b = t->cfg.bucket_size;
  uint64_t pair = or_pack_pair(key, value);
  uint64_t bucket_id = hash_of(t, 0, key);
  uint32_t chain = 0;
  for (;;) {
    uint64_t* bk = bucket_ptr(t, bucket_id);
    ++*probes;
    uint32_t load = bucket_load(bk, b);
    if (load == b) {
      if (chain == t->cfg.max_chain) return 0; /* table.cpp:67: cap checked before the exchange */
      uint64_t victim = bucket_exch(bk, pair, rng_next_below(rng, b)); /* table.cpp:71 */
      uint32_t vkey = (uint32_t)victim;
      uint64_t cand[4] = {0, 0, 0, 0};
      for (unsigned i = 0; i < h; ++i) cand[i] = hash_of(t, i, vkey);
      uint64_t next = cand[0];
      for (unsigned i = 0; i < h; ++i) /* table.cpp:74-80: lowest index that maps here */
        if (cand[i] == bucket_id) {
          next = cand[(i + 1) % h];
          break;
        }
      pair = victim;
      bucket_id = next;
      ++chain;
    } else if (bucket_cas(bk, pair, load) == OR_EMPTY_SLOT) { /* table.cpp:85 */
      ++t->inserted;
      return 1;
    }
  }
}

/* src/table.cpp:94-107 — early exit on any probed bucket that is not full */
static int cuckoo_find(const or_table* t, uint32_t key, uint32_t* value, uint64_t* probes, int early_exit) {
  for (unsigned i = 0; i < t->cfg.n_hashes; ++i) {
    const uint64_t* bk = bucket_ptr(t, hash_of(t, i, key));
    ++*probes;
    if (bucket_find(bk, t->cfg.bucket_size, key, value)) return 1;
    if (early_exit && bucket_load(bk, t->cfg.bucket_size) != t->cfg.bucket_size) return 0;
  }
  return 0;
}

/* src/table.cpp:109-130 */
static int p2_insert(or_table* t, uint32_t key, uint32_t value, uint64_t* probes) {
  const uint32_t b = t->cfg.bucket_size;
  uint64_t* b0 = bucket_ptr(t, hash_of(t, 0, key));
  uint64_t* b1 = bucket_ptr(t, hash_of(t, 1, key));
  for (;;) {
    *probes += 2;
    uint32_t l0 = bucket_load(b0, b), l1 = bucket_load(b1, b);
    if (l0 == b && l1 == b) return 0;
    uint64_t* choice = l0 <= l1 ? b0 : b1; /* tie -> first hash (table.cpp:124) */
    if (bucket_cas(choice, or_pack_pair(key, value), l0 < l1 ? l0 : l1) == OR_EMPTY_SLOT) {
      ++t->inserted;
      return 1;
    }
  }
}

/* src/table.cpp:132-142 — no early exit */
static int p2_find(const or_table* t, uint32_t key, uint32_t* value, uint64_t* probes) {
  ++*probes;
  if (bucket_find(bucket_ptr(t, hash_of(t, 0, key)), t->cfg.bucket_size, key, value)) return 1;
  ++*probes;
  return bucket_find(bucket_ptr(t, hash_of(t, 1, key)), t->cfg.bucket_size, key, value);
}

/* src/table.cpp:144-186 */
static int iceberg_insert(or_table* t, uint32_t key, uint32_t value, int prose, uint64_t* probes) {
  const uint32_t b = t->cfg.bucket_size;
  uint64_t* primary = bucket_ptr(t, hash_of(t, 0, key));
  for (;;) {
    ++*probes;
    uint32_t pl = bucket_load(primary, b);
    uint64_t* choice = primary;
    uint32_t cl = pl;
    if (pl >= t->cfg.threshold) { /* table.cpp:159: at or past the threshold */
      uint64_t* s0 = bucket_ptr(t, hash_of(t, 1, key));
      uint64_t* s1 = bucket_ptr(t, hash_of(t, 2, key));
      *probes += 2;
      uint32_t l0 = bucket_load(s0, b), l1 = bucket_load(s1, b);
      if (prose || l0 != b || l1 != b) { /* table.cpp:169 */
        if (l0 <= l1) {
          choice = s0;
          cl = l0;
        } else {
          choice = s1;
          cl = l1;
        }
      }
    }
    if (cl == b) return 0; /* table.cpp:180 */
    if (bucket_cas(choice, or_pack_pair(key, value), cl) == OR_EMPTY_SLOT) {
      ++t->inserted;
      return 1;
    }
  }
}

/* src/table.cpp:188-201 */
static int iceberg_find(const or_table* t, uint32_t key, uint32_t* value, uint64_t* probes) {
  for (unsigned i = 0; i < 3; ++i) {
    ++*probes;
    if (bucket_find(bucket_ptr(t, hash_of(t, i, key)), t->cfg.bucket_size, key, value)) return 1;
  }
  return 0;
}

/* src/table.cpp:203-212 */
int or_insert_pair(or_table* t, uint32_t key, uint32_t value, uint64_t* rng_state, int prose,
                   uint64_t* probes) {
  uint64_t scratch = 0;
  if (!probes) probes = &scratch;
  switch (t->cfg.kind) {
    case K_ONE_CHT:
    case K_BCHT: return cuckoo_insert(t, key, value, rng_state, probes);
    case K_BP2HT: return p2_insert(t, key, value, probes);
    case K_IHT: return iceberg_insert(t, key, value, prose, probes);
  }
  return -1;
}

/* src/table.cpp:214-222 */
int or_find_key(const or_table* t, uint32_t key, uint32_t* value, uint64_t* probes) {
  uint64_t scratch = 0;
  uint32_t v = OR_EMPTY_KEY;
  if (!probes) probes = &scratch;
  int r = -1;
  switch (t->cfg.kind) {
    case K_ONE_CHT:
    case K_BCHT: r = cuckoo_find(t, key, &v, probes, 1); break;
    case K_BP2HT: r = p2_find(t, key, &v, probes); break;
    case K_IHT: r = iceberg_find(t, key, &v, probes); break;
  }
  if (value) *value = r == 1 ? v : OR_EMPTY_KEY;
  return r;
}

/* src/oracle.cpp:56-63 */
int or_find_key_no_early_exit(const or_table* t, uint32_t key, uint32_t* value) {
  uint64_t scratch = 0;
  uint32_t v = OR_EMPTY_KEY;
  int r = cuckoo_find(t, key, &v, &scratch, 0);
  if (value) *value = r ? v : OR_EMPTY_KEY;
  return r;
}

/* src/table.cpp:224-238 — sequential build, one rng stream, stop at the first failure */
int64_t or_build(or_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, int prose,
                 uint64_t* probes, uint64_t* failed_index) {
  if (n > t->cfg.capacity) return -1; /* table.cpp:225 */
  uint64_t rng = or_rng_init(or_mix_seed(t->cfg.seed, 0x65766963ull));
  uint64_t p = 0;
  uint64_t i = 0;
  for (; i < n; ++i) {
    uint32_t v = values ? values[i] : or_value_for_key(keys[i]);
    if (or_insert_pair(t, keys[i], v, &rng, prose, &p) != 1) break;
  }
  if (probes) *probes = p;
  if (failed_index) *failed_index = i;
  return (int64_t)t->inserted;
}

int64_t or_insert_all(or_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                      int prose, uint64_t* probes, uint8_t* failed_flags) {
  uint64_t rng = or_rng_init(or_mix_seed(t->cfg.seed, 0x65766963ull));
  uint64_t p = 0;
  int64_t ok = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t v = values ? values[i] : or_value_for_key(keys[i]);
    int r = or_insert_pair(t, keys[i], v, &rng, prose, &p);
    ok += r == 1;
    if (failed_flags) failed_flags[i] = r != 1;
  }
  if (probes) *probes = p;
  return ok;
}

/* src/experiments.cpp:92 / src/oracle.cpp:21-27 — the caller-side find loop */
uint64_t or_find_bulk(const or_table* t, const uint32_t* keys, uint64_t n, uint32_t* out,
                      uint64_t* probes) {
  uint64_t p = 0, hits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t v;
    hits += or_find_key(t, keys[i], &v, &p) == 1;
    if (out) out[i] = v;
  }
  if (probes) *probes = p;
  return hits;
}

/* src/oracle.cpp:40-54 */
uint64_t or_check_admissibility(const or_table* t) {
  uint64_t bad = 0;
  for (uint64_t s = 0; s < t->cfg.capacity; ++s) {
    uint32_t key = (uint32_t)t->store[s];
    if (key == OR_EMPTY_KEY) continue;
    uint64_t bucket_id = s / t->cfg.bucket_size;
    int ok = 0;
    for (unsigned i = 0; i < t->cfg.n_hashes && !ok; ++i) ok = hash_of(t, i, key) == bucket_id;
    bad += !ok;
  }
  return bad;
}

/* Multi-GPU routing: owner = (((alpha*k+beta) mod p) * G) >> 32. */
uint32_t or_shard_of(uint64_t alpha, uint64_t beta, uint32_t n_shards, uint32_t key) {
  uint64_t r = (alpha * (uint64_t)key + beta) % OR_PRIME;
  return (uint32_t)((r * (uint64_t)n_shards) >> 32);
}
