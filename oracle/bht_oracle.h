/*
 * bht_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded CPU restatement of the reference's bulk hash-table path
 * (reference tree: /root/reference/proj).  It exists to check the CUDA product; nothing under
 * paper_2108_07232_b200/ or include/ may call, link or import it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks this restatement against the golden
 * vectors of the reference's own tests (proj/tests/test_hash.cpp, test_core.cpp, test_bucket.cpp,
 * test_table.cpp, test_metrics.cpp) and against outputs of the unmodified reference compiled into
 * oracle/_ref/libbht_ref.so (fixtures committed under tests/golden/).
 */
#ifndef BHT_ORACLE_H_
#define BHT_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_EMPTY_KEY 0xFFFFFFFFu
#define OR_EMPTY_SLOT 0xFFFFFFFFFFFFFFFFull
#define OR_PRIME 4294967291ull

/* Same layout as bht_config in include/bht_b200.h (asserted by tests via or_sizeof_config). */
typedef struct or_config {
  int32_t kind; /* 0 one_cht, 1 bcht, 2 bp2ht, 3 iht (core.hpp:43) */
  uint32_t bucket_size;
  uint64_t num_buckets;
  uint64_t capacity;
  uint32_t n_hashes;
  uint32_t threshold;
  uint32_t max_chain;
  uint32_t reserved;
  uint64_t seed;
  uint64_t alpha[4];
  uint64_t beta[4];
  uint64_t range[4];
} or_config;

typedef struct or_table or_table;

/* hash.hpp */
uint64_t or_bucket_index(uint64_t alpha, uint64_t beta, uint64_t range, uint32_t key);
uint64_t or_splitmix64(uint64_t x);
uint64_t or_mix_seed(uint64_t seed, uint64_t stream);
void or_xorshift_stream(uint64_t seed, uint64_t n, uint64_t* out);
void or_next_below_stream(uint64_t seed, uint32_t bound, uint64_t n, uint32_t* out);

/* core.hpp / core.cpp */
uint32_t or_hash_count(int32_t kind);
uint32_t or_default_max_chain(uint64_t n_keys);
/* returns 0, or 1 where the reference throws std::invalid_argument */
int or_make_config(int32_t kind, uint64_t n_keys, double lf, uint32_t bucket_size, int64_t threshold,
                   uint64_t seed, int64_t max_chain, or_config* out);
uint64_t or_pack_pair(uint32_t key, uint32_t value);
size_t or_sizeof_config(void);

/* keygen.hpp / keygen.cpp */
uint32_t or_value_for_key(uint32_t key);
void or_mt19937_64_stream(uint64_t seed, uint64_t n, uint64_t* out);
void or_generate_keys(uint64_t seed, uint64_t n, uint32_t* out);

/* sector_model.hpp; op 0 = insert, 1 = find */
uint32_t or_bucket_sectors(uint32_t bucket_size);
double or_predict_sectors(int32_t kind, uint32_t bucket_size, double mean_probes, int32_t op);

/* table.hpp / table.cpp */
or_table* or_table_create(const or_config* cfg); /* NULL where the reference throws */
void or_table_destroy(or_table* t);
uint64_t or_table_inserted(const or_table* t);
uint64_t or_occupied_slots(const or_table* t);
uint64_t or_slot_at(const or_table* t, uint64_t index);
void or_poke_slot(or_table* t, uint64_t index, uint64_t slot);
void or_download_store(const or_table* t, uint64_t* dst);
void or_upload_store(or_table* t, const uint64_t* src);

/* Evaluates insert_pair / find_key for one key. rng_state is the xorshift state (in/out).
 * Return: 1 inserted / found, 0 failed / absent, -1 kind mismatch (std::logic_error). */
int or_insert_pair(or_table* t, uint32_t key, uint32_t value, uint64_t* rng_state, int prose,
                   uint64_t* probes);
int or_find_key(const or_table* t, uint32_t key, uint32_t* value, uint64_t* probes);
int or_find_key_no_early_exit(const or_table* t, uint32_t key, uint32_t* value);
uint64_t or_rng_init(uint64_t seed); /* xorshift_rng ctor: splitmix64 + zero remap */

/* build(), sequential mode: rng = xorshift_rng(mix_seed(cfg.seed, 0x65766963)); stops at the
 * first failure. values == NULL selects value_for_key. Returns #inserted; *failed_index = index
 * of the failing key or n. -1 if n > capacity (std::invalid_argument). */
int64_t or_build(or_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, int prose,
                 uint64_t* probes, uint64_t* failed_index);
/* Bulk variant that keeps going after failures (what a bulk GPU insert does); failed keys are
 * flagged in failed_flags (may be NULL). */
int64_t or_insert_all(or_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                      int prose, uint64_t* probes, uint8_t* failed_flags);
/* caller-side find loop (experiments.cpp:92): out[i] = value or 0xFFFFFFFF. Returns #hits. */
uint64_t or_find_bulk(const or_table* t, const uint32_t* keys, uint64_t n, uint32_t* out,
                      uint64_t* probes);

/* oracle.cpp:40-54 */
uint64_t or_check_admissibility(const or_table* t);

/* shard routing of the multi-GPU table (no reference counterpart; restated from DESIGN.md) */
uint32_t or_shard_of(uint64_t alpha, uint64_t beta, uint32_t n_shards, uint32_t key);

#ifdef __cplusplus
}
#endif
#endif
