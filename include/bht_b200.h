/*
 * bht_b200.h — C ABI of the B200-native bulk hash-table hot path.
 *
 * This is the drop-in boundary for the reference library's table API
 * (reference: proj/include/bht/table.hpp, proj/include/bht/core.hpp).  Every
 * entry point below names the reference interface it replaces.  Signatures
 * carry only plain pointers, sizes and PODs; `stream` is a `cudaStream_t`
 * passed as `void*` (NULL = the legacy default stream).
 *
 * The implementation lives in paper_2108_07232_b200/csrc and is built into
 * paper_2108_07232_b200/lib/libbht_b200.so.  There is no CPU fallback: every
 * compute entry point runs hand-written sm_100a kernels and returns
 * BHT_CUDA_ERROR if no device is usable.
 *
 * Conventions kept bit-exact with the reference:
 *   - slot = (value << 32) | key, empty slot = all ones      (core.hpp:13-41)
 *   - user keys live in [0, 2^32-2]; 0xFFFFFFFF is the sentinel (core.hpp:20-24)
 *   - h_i(k) = ((alpha_i*k + beta_i) mod 4294967291) mod range_i (hash.hpp:21-23)
 *   - kind order one_cht, bcht, bp2ht, iht                   (core.hpp:43)
 *   - store layout: bucket-major, b consecutive 8-byte slots  (table.hpp:42-47)
 *
 * Error model (reference: exceptions in core.cpp:40-60, table.cpp:15-17,22-23,225):
 * nothing throws; a bht_status is returned and bht_last_error_string() holds
 * the message.  A failed insertion (cuckoo chain cap, all candidate buckets
 * full) is NOT an error: status stays BHT_OK and the failure is reported in
 * bht_insert_result, as `build_outcome` does in the reference (table.hpp:115-120).
 */
#ifndef BHT_B200_H_
#define BHT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BHT_EMPTY_KEY 0xFFFFFFFFu            /* core.hpp:20 */
#define BHT_EMPTY_VALUE 0xFFFFFFFFu          /* core.hpp:21 */
#define BHT_EMPTY_SLOT 0xFFFFFFFFFFFFFFFFull /* core.hpp:22 */
#define BHT_HASH_PRIME 4294967291ull         /* hash.hpp:12 */
#define BHT_MAX_HASHES 4
#define BHT_MAX_BUCKET_SIZE 64               /* core.hpp:79 */

typedef enum bht_status {
  BHT_OK = 0,
  BHT_INVALID_ARGUMENT = 1,  /* std::invalid_argument in the reference */
  BHT_KIND_MISMATCH = 2,     /* std::logic_error (table.cpp:15-17) */
  BHT_CAPACITY_EXCEEDED = 3, /* "build: key set exceeds table capacity" (table.cpp:225) */
  BHT_CUDA_ERROR = 4,
  BHT_COMM_ERROR = 5,
  BHT_IO_ERROR = 6           /* std::runtime_error on file I/O (table.cpp:43,50) */
} bht_status;

/* table_kind, same numeric order as the reference enum (core.hpp:43). */
typedef enum bht_kind {
  BHT_ONE_CHT = 0, /* b = 1, 4 hash functions */
  BHT_BCHT = 1,    /* 3 hash functions */
  BHT_BP2HT = 2,   /* 2 hash functions */
  BHT_IHT = 3      /* primary + 2 secondaries */
} bht_kind;

/* Plain-data image of the reference `table_config` (core.hpp:66-77).  The
 * per-hash (alpha, beta, range) triples are `hash_params` (hash.hpp:11-19). */
typedef struct bht_config {
  int32_t kind;         /* bht_kind */
  uint32_t bucket_size; /* b: power of two in [1, 64] */
  uint64_t num_buckets; /* m */
  uint64_t capacity;    /* m * b */
  uint32_t n_hashes;    /* hash_count(kind): 4 / 3 / 2 / 3 (core.hpp:49-57) */
  uint32_t threshold;   /* t, iht only */
  uint32_t max_chain;   /* cuckoo kinds only */
  uint32_t reserved;
  uint64_t seed;
  uint64_t alpha[BHT_MAX_HASHES];
  uint64_t beta[BHT_MAX_HASHES];
  uint64_t range[BHT_MAX_HASHES];
} bht_config;

/* Image of `build_outcome` (table.hpp:115-120) for one bulk insert call. */
typedef struct bht_insert_result {
  uint64_t attempted;        /* n of this call */
  uint64_t inserted;         /* pairs now resident because of this call */
  uint64_t failed;           /* pairs dropped (chain cap / all candidates full) */
  uint64_t probes;           /* bucket reads, probe_stats.total_probes (probe_stats.hpp:12-31) */
  uint32_t first_failed_key; /* some dropped key, BHT_EMPTY_KEY if none */
  uint32_t success;          /* inserted == attempted */
} bht_insert_result;

typedef struct bht_find_result {
  uint64_t queries;
  uint64_t hits;         /* queries answered with a value */
  uint64_t probes;       /* bucket reads */
  uint64_t value_sum;    /* sum of the returned values of the hits (checksum) */
} bht_find_result;

/* Where the caller's key / value / output arrays live. */
typedef enum bht_mem_space {
  BHT_MEM_DEVICE = 0, /* device pointers on the table's device */
  BHT_MEM_HOST = 1    /* host pointers (pinned or pageable); the call stages chunks over PCIe */
} bht_mem_space;

typedef struct bht_table bht_table; /* opaque: replaces `class hash_table` (table.hpp:28-80) */

/* ---- configuration (host only, no GPU needed) ------------------------------------------- */

/* Replaces make_config (core.hpp:85-91, core.cpp:33-68) bit-exactly: same ceil(n/(lf*b)),
 * same default threshold b*80/100 and max(7*ceil(log2 n),128) chain cap, same hash-constant
 * draw from xorshift_rng(mix_seed(seed, 0x68617368)).  threshold < 0 / max_chain < 0 select
 * the defaults (std::nullopt in the reference). */
bht_status bht_make_config(int32_t kind, uint64_t n_keys, double load_factor, uint32_t bucket_size,
                           int64_t threshold, uint64_t seed, int64_t max_chain, bht_config* out);

/* hash_count (core.hpp:49-57); 0 for an unknown kind. */
uint32_t bht_hash_count(int32_t kind);
/* default_max_chain (core.cpp:28-31). */
uint32_t bht_default_max_chain(uint64_t n_keys);
/* mix_seed (hash.hpp:33-35), exposed so harnesses derive the same seed streams. */
uint64_t bht_mix_seed(uint64_t seed, uint64_t stream);
/* bucket_index (hash.hpp:21-23) evaluated on the host with the SAME division-free arithmetic
 * the device hash stage uses (fold by 2^32 = 5 mod p, then a 64-bit reciprocal for mod range). */
uint64_t bht_bucket_index_host(uint64_t alpha, uint64_t beta, uint64_t range, uint32_t key);
/* value_for_key (keygen.hpp:23-26). */
uint32_t bht_value_for_key(uint32_t key);
/* predict_sectors (sector_model.hpp:26-31); op: 0 = insert, 1 = find. */
double bht_predict_sectors(int32_t kind, uint32_t bucket_size, double mean_probes, int32_t op);

/* ---- lifetime ---------------------------------------------------------------------------- */

/* Replaces hash_table::hash_table(table_config) (table.cpp:21-32): allocates the m*b slot store
 * in device memory (256-byte aligned) on `device` and fills it with BHT_EMPTY_SLOT.
 * BHT_INVALID_ARGUMENT on a wrong hash count (table.cpp:22-23) or an inconsistent config. */
bht_status bht_create(const bht_config* cfg, int32_t device, bht_table** out);
bht_status bht_destroy(bht_table* table);
/* Re-initialises the store to empty and zeroes the inserted counter (a fresh hash_table). */
bht_status bht_clear(bht_table* table, void* stream);
bht_status bht_get_config(const bht_table* table, bht_config* out);
int32_t bht_device_of(const bht_table* table);

/* ---- the hot path ------------------------------------------------------------------------ */

/* Bulk insert: replaces build()'s insertion loop (table.cpp:224-271) and insert_pair
 * (table.cpp:203-212) with explicit values.  Precondition as in the reference: keys unique,
 * != sentinel, not yet present.  Unlike the reference's build, which stops at the first failed
 * key, every pair is attempted; pairs that do not fit are reported in `result`, not as an error.
 * `result` may be NULL (no synchronisation; fetch it later with bht_last_insert_result).
 * `values` may be NULL: every key is paired with value_for_key(key) as in the reference's keys-only build
 * (table.cpp:234, keygen.hpp:23-26); the values are made on the device, so a BHT_MEM_HOST caller ships keys only.
 * A BHT_MEM_HOST call returns when the caller's arrays have been read; with result == NULL its device work may still be
 * in flight, ordered before anything done later with this table or enqueued later on `stream`. */
bht_status bht_insert(bht_table* table, const uint32_t* keys, const uint32_t* values, uint64_t n,
                      int32_t mem_space, bht_insert_result* result, void* stream);

/* Bulk find: replaces the caller-side `for q: find_key(table, q.key, stats)` loop
 * (experiments.cpp:92, oracle.cpp:21-27) and find_key (table.cpp:214-222).
 * out_values[i] = value, or BHT_EMPTY_VALUE when the key is absent. */
bht_status bht_find(const bht_table* table, const uint32_t* keys, uint32_t* out_values, uint64_t n,
                    int32_t mem_space, bht_find_result* result, void* stream);

/* build(keys, cfg, opts) (table.hpp:125-127, table.cpp:224-276) in one call: BHT_CAPACITY_EXCEEDED when
 * n > cfg->capacity ("build: key set exceeds table capacity", table.cpp:225, checked before anything is
 * allocated), else bht_create + bht_insert of all n pairs.  *out receives the new table.  values == NULL is the
 * reference's signature: build(keys, cfg, opts) pairs key k with value_for_key(k). */
bht_status bht_build(const bht_config* cfg, int32_t device, const uint32_t* keys, const uint32_t* values,
                     uint64_t n, int32_t mem_space, int32_t iht_prose_fallback, bht_table** out,
                     bht_insert_result* result, void* stream);

/* A build whose pairs arrive in chunks (device-resident arrays): the loop of build() (table.cpp:231-238 sequential,
 * :239-271 parallel) with the key set handed over piece by piece — what the receive side of a sharded build and a
 * host-buffer bht_insert do internally.  bht_build_begin announces at most n_max pairs; bht_build_feed adds a chunk
 * (values == NULL: value_for_key, as bht_insert) — BHT_CAPACITY_EXCEEDED past n_max; bht_build_end completes the
 * build and reports the whole of it (result may be NULL; bht_last_insert_result reads it later).  A table that
 * qualifies for the shared-memory-blocked build takes every chunk through the first partition pass as it is fed and
 * runs the rest at the end; every other table inserts chunk by chunk.  Between begin and end the table accepts
 * no bht_insert / bht_clear; finds see the pairs of the chunks a non-blocked table has inserted so far. */
bht_status bht_build_begin(bht_table* table, uint64_t n_max, void* stream);
bht_status bht_build_feed(bht_table* table, const uint32_t* keys, const uint32_t* values, uint64_t n, void* stream);
bht_status bht_build_end(bht_table* table, bht_insert_result* result, void* stream);
/* bht_build_feed for a chunk whose length is only known on the device (the receive side of a sync-free exchange):
 * the chunk holds min(n_cap, *n_dev) pairs, n_dev a device pointer read by the kernels.  Cuckoo kinds only. */
bht_status bht_build_feed_counted(bht_table* table, const uint32_t* keys, const uint32_t* values, uint64_t n_cap,
                                  const uint64_t* n_dev, void* stream);

/* The reference's per-variant entry points bcht_insert / bp2ht_insert / iht_insert and bcht_find /
 * bp2ht_find / iht_find (table.hpp:84-101): as bht_insert / bht_find, but BHT_KIND_MISMATCH when the
 * table is not of `kind` (require_kind, table.cpp:15-17; BHT_BCHT also accepts a 1cht table). */
bht_status bht_insert_as(bht_table* table, int32_t kind, const uint32_t* keys, const uint32_t* values,
                         uint64_t n, int32_t mem_space, bht_insert_result* result, void* stream);
bht_status bht_find_as(const bht_table* table, int32_t kind, const uint32_t* keys, uint32_t* out_values,
                       uint64_t n, int32_t mem_space, bht_find_result* result, void* stream);

/* bcht/1cht find without the early exit: bcht_find_no_early_exit (oracle.cpp:56-63). */
bht_status bht_find_exhaustive(const bht_table* table, const uint32_t* keys, uint32_t* out_values,
                               uint64_t n, int32_t mem_space, bht_find_result* result, void* stream);

/* Synchronises `stream` and returns the counters of the most recent insert / find. */
bht_status bht_last_insert_result(bht_table* table, bht_insert_result* out, void* stream);
/* Keys dropped by inserts since the last bht_clear (at most `max_keys` copied). */
bht_status bht_failed_keys(bht_table* table, uint32_t* host_out, uint64_t max_keys, uint64_t* count);
/* Device time of the last device-resident bht_insert, split at the launch of its probe kernel: `prepare_ms` =
 * routing / binning passes of a blocked build (0 in caller order), `probe_ms` = the bulk-insert kernel itself.
 * Measured with CUDA events on the call's stream; waits for that call to finish.  (Instrumentation for the
 * per-kernel roofline; the reference's counterpart is the steady_clock around build(), table.cpp:228-276.) */
bht_status bht_last_insert_phases(bht_table* table, float* prepare_ms, float* probe_ms);
/* iht only: select the prose variant of iht_insert (table.cpp:167-169, `prose_fallback`). */
bht_status bht_set_iht_prose_fallback(bht_table* table, int32_t enabled);

/* How the last bht_insert / chunked build of this table ran: 0 = caller order (K4 / K5 / K6 / K12 / K13), 2 = L2-routed,
 * 3 = shared-memory-blocked (K8g, K10, K11, K4).  Diagnostics: tests and smoke() assert the schedule they mean to cover. */
int32_t bht_last_build_schedule(const bht_table* table);

/* Large device-resident inserts into a store much bigger than the L2 are blocked by table region first (same
 * result set, different concurrent order).  bcht: the pairs are partitioned in two streaming passes by the 64 KiB
 * region of their first bucket, every region is built in shared memory (slot claims by shared-memory atomics, the
 * first eviction of a pair whose bucket is full included) and only the evicted victims walk on through the general
 * kernel.  1cht, and bcht tables beyond 8 GB: the pairs are routed by L2-sized region and inserted by the general
 * kernel in that order.  mode 0 = never (caller order), 1 = when the sizes make it pay (default), 2 = always the
 * L2-routed build, 3 = always the shared-memory-blocked build (2 and 3 also on small tables; used by the parity
 * tests).  bp2ht / iht are never reordered: their balanced placements depend on the arrival order, and arrival in
 * first-bucket order measurably lowers the load factor they reach.  For them the mode selects how loads are learnt:
 * modes 1 (stores of 192 MB and more) and 3 (always) decide from a per-bucket load counter array kept beside the
 * store and claim slots with an atomic on the counter — one 8-byte store per pair is the only access to the store;
 * mode 0 reads the candidate buckets.  Same decisions, same probe counts, in the caller's order either way. */
bht_status bht_set_blocked_insert(bht_table* table, int32_t mode);

/* Cuckoo kinds.  The reference inserts one pair at a time, so an eviction chain never meets another walker and
 * max_chain (core.hpp:93-96, core.cpp:28-31) is calibrated for that; a bulk build has ~190 k walkers in flight, and near
 * the end of a build at load factor 0.99 they hit max_chain 3-5 times more often (half of such builds dropped one to
 * three pairs, where the reference's build fails one time in ten).  With the repair pass the few pairs a launch of
 * more than 32 pairs dropped (at most 256) are inserted once more, by one thread, one after the other — bcht_insert's
 * loop (table.cpp:53-92) with nobody else moving pairs; a pair that fails again stays failed and is reported.
 * Default: on for bcht, off for 1cht (whose success curve at desk scale already is the reference's, acceptance
 * criterion 6; with the second chance it would build beyond it).  Measured over 40 seeds at 10^6 keys, load factor
 * 0.99: reference 35 builds, concurrent walks alone 20, with the repair 40. */
bht_status bht_set_repair(bht_table* table, int32_t enabled);

/* cuckoo kinds, off by default: insert the pairs that arrive beyond load 0.98 (b = 1: 0.85) with few keys in flight
 * (<= 1/24 of the slots still free at the end).  Thousands of eviction walks competing for the last free slots hit
 * max_chain (core.hpp:93-96) 3-5 times more often than the reference's one-walker-at-a-time process; the throttle
 * brings the build success at load factor 0.99 from ~50 % to ~80 % (reference: 90 %) for 2.5x the build time.
 * Retrying a failed build with fresh hash constants, as run_trial does (experiments.cpp:69-82), is cheaper. */
bht_status bht_set_tail_throttle(bht_table* table, int32_t enabled);

/* ---- load factor / store access ---------------------------------------------------------- */

/* realized_load() (table.hpp:40): inserted counter and capacity. */
bht_status bht_load_factor(const bht_table* table, uint64_t* inserted, uint64_t* capacity);
/* occupied_slots() (table.cpp:34-39): streaming count of non-empty keys in the store. */
bht_status bht_count_occupied(const bht_table* table, uint64_t* occupied, void* stream);
/* slot_at over the whole store (table.hpp:53): copies m*b slots to host, bucket order. */
bht_status bht_download_store(const bht_table* table, uint64_t* host_dst, void* stream);
/* poke_slot over the whole store (table.hpp:54-56): replaces the store; recounts `inserted`. */
bht_status bht_upload_store(bht_table* table, const uint64_t* host_src, void* stream);
/* dump_store (table.cpp:41-51): little-endian u64 per slot, bucket order. */
bht_status bht_dump_store(const bht_table* table, const char* path);
/* check_admissibility (oracle.cpp:40-54) evaluated on the device: pairs outside every bucket
 * their hash functions name. */
bht_status bht_count_inadmissible(const bht_table* table, uint64_t* violations, void* stream);
/* Raw device pointer of the store (for zero-copy interop); valid until bht_destroy. */
uint64_t* bht_device_store(const bht_table* table);

/* ---- hash stage in isolation (parity hook for hash.hpp:21-23) ---------------------------- */

/* out[i] = bucket_index({alpha, beta, range}, keys[i]) computed by the device hash stage. */
bht_status bht_hash_keys(uint64_t alpha, uint64_t beta, uint64_t range, const uint32_t* keys,
                         uint32_t* out, uint64_t n, int32_t mem_space, int32_t device, void* stream);

/* ---- sharded table: key-range partitioning for multi-GPU (no reference counterpart) ------ */

/* owner(k) = (g(k) * n_shards) >> 32 with g(k) = (alpha*k + beta) mod p scaled to 32 bits. */
uint32_t bht_shard_of_host(uint64_t alpha, uint64_t beta, uint32_t n_shards, uint32_t key);

/* Partition n keys (and optional values) by owner shard.  Writes keys (values) grouped by shard
 * into out_keys (out_values), the original position of every routed element into out_index
 * (may be NULL), and the per-shard counts into counts_host[n_shards] (host memory; the call
 * synchronises `stream`).  All array pointers are device pointers on `device`. */
bht_status bht_shard_partition(uint64_t alpha, uint64_t beta, uint32_t n_shards,
                               const uint32_t* keys, const uint32_t* values, uint64_t n,
                               uint32_t* out_keys, uint32_t* out_values, uint32_t* out_index,
                               uint64_t* counts_host, int32_t device, void* stream);

/* bht_shard_partition without any host synchronisation, for an all-to-all with EQUAL splits: destination d gets the
 * slots [d * cap, (d + 1) * cap) of the outputs (the caller pre-fills them with 0xFF bytes: unused slots then hold the
 * sentinel key / the index 0xFFFFFFFF, which bht_find answers without a probe and bht_shard_unpermute skips);
 * An element carries its value (values != NULL, inserts) or its position in the input (out_index != NULL, finds), not both.
 * counts_dev[d] (device, uint64) = elements written for d; *overflow_dev (device) is OR-ed with 1 when some destination
 * had more than cap elements (the surplus is not written: the caller re-routes with exact counts). */
bht_status bht_shard_partition_fixed(uint64_t alpha, uint64_t beta, uint32_t n_shards, const uint32_t* keys,
                                     const uint32_t* values, uint64_t n, uint64_t cap, uint32_t* out_keys,
                                     uint32_t* out_values, uint32_t* out_index, uint64_t* counts_dev,
                                     uint32_t* overflow_dev, int32_t device, void* stream);

/* out[index[i]] = answers[i]: puts routed answers back into the caller's query order. */
bht_status bht_shard_unpermute(const uint32_t* answers, const uint32_t* index, uint64_t n,
                               uint32_t* out, int32_t device, void* stream);

/* ---- synthetic workload (keygen.cpp:50-64 protocol on the device) ------------------------ */

/* keys[i] = a bijection of (offset + i) over [0, 2^32-2]: unique, sentinel-free keys without a
 * host-side rejection set.  Indices >= some n are guaranteed-absent negatives. */
bht_status bht_generate_unique_keys(uint64_t seed, uint64_t offset, uint64_t n, uint32_t* out_keys,
                                    uint32_t* out_values, int32_t device, void* stream);

/* generate_keys (keygen.cpp:50-64), element for element: the first n distinct non-sentinel values of
 * (std::mt19937_64(seed)() >> 32) in stream order.  The engine runs on the host in batches; "first occurrence
 * wins" is decided by a device hash set (atomicMin on the stream index) and an order-preserving compaction.
 * out_keys: n words in `mem_space`. */
bht_status bht_generate_keys(uint64_t seed, uint64_t n, uint32_t* out_keys, int32_t mem_space, int32_t device,
                             void* stream);

/* generate_queries (keygen.cpp:66-98), element for element: round(positive_ratio * q) positives by a partial
 * Fisher-Yates over the key list, the rest guaranteed-absent draws of the same stream (membership = a bulk find
 * on a device table of the keys), then shuffle_deterministic.  keys: n_keys words in `keys_space`; the three
 * outputs are HOST arrays of q elements (out_expected = value_for_key for positives, 0 for negatives;
 * out_expected / out_present may be null).  BHT_INVALID_ARGUMENT where the reference throws invalid_argument. */
bht_status bht_generate_queries(const uint32_t* keys, uint64_t n_keys, int32_t keys_space, double positive_ratio,
                                uint64_t q, uint64_t seed, uint32_t* out_keys, uint32_t* out_expected,
                                uint8_t* out_present, int32_t device);

/* save_keys / load_keys (keygen.cpp:100-125): flat file of little-endian 32-bit keys.  bht_load_keys sets
 * *count to the number of keys in the file and copies at most max_keys of them (keys_host may be null). */
bht_status bht_save_keys(const char* path, const uint32_t* keys_host, uint64_t n);
bht_status bht_load_keys(const char* path, uint32_t* keys_host, uint64_t max_keys, uint64_t* count);

/* The same bijection / value stream evaluated on the host for one counter / key. */
uint32_t bht_unique_key_host(uint64_t seed, uint32_t counter);
uint32_t bht_synthetic_value_host(uint64_t seed, uint32_t key);

/* ---- sharded table handle: one process, n_shards ordinary tables, one per entry of device_ids ----------------
 * (the multi-process counterpart, one rank per GPU over NCCL, is paper_2108_07232_b200/sharded.py).
 * owner(k) = bht_shard_of_host(alpha, beta, n_shards, k) with (alpha, beta) = bht_shard_constants(cfg->seed), so every
 * candidate bucket of a key lives in one shard.  keys[g] / values[g] / out_values[g] are DEVICE pointers on
 * device_ids[g] holding the slice of n[g] elements that GPU g contributes; the routed runs travel with
 * cudaMemcpyPeerAsync (NVLink where peer access exists) and all owners insert / find at the same time.  Device ids
 * may repeat (several shards on one GPU).  values == NULL or values[g] == NULL: value_for_key, as in bht_insert.
 * `result` aggregates the shards (attempted = total keys; success = every pair placed); may be NULL. */
typedef struct bht_sharded bht_sharded;
void bht_shard_constants(uint64_t seed, uint64_t* alpha, uint64_t* beta);
bht_status bht_sharded_create(const bht_config* cfg_per_shard, uint32_t n_shards, const int32_t* device_ids, bht_sharded** out);
bht_status bht_sharded_destroy(bht_sharded* sharded);
uint32_t bht_sharded_count(const bht_sharded* sharded);
/* the table of one shard, owned by the sharded handle (for bht_load_factor, bht_download_store, ...) */
bht_status bht_sharded_table(bht_sharded* sharded, uint32_t shard, bht_table** out);
bht_status bht_sharded_clear(bht_sharded* sharded);
bht_status bht_sharded_insert(bht_sharded* sharded, const uint32_t* const* keys, const uint32_t* const* values,
                              const uint64_t* n, bht_insert_result* result);
bht_status bht_sharded_find(bht_sharded* sharded, const uint32_t* const* keys, uint32_t* const* out_values,
                            const uint64_t* n, bht_find_result* result);

/* ---- pinned host buffers for BHT_MEM_HOST callers (cudaMallocHost / cudaFreeHost) --------- */

bht_status bht_host_alloc(size_t bytes, void** out);
bht_status bht_host_free(void* ptr);

/* ---- diagnostics ------------------------------------------------------------------------- */

const char* bht_last_error_string(void);
const char* bht_version_string(void);
/* The tuning knobs (BHT_* environment variables; csrc/capi.cu: Knobs) are read once per process; this re-reads them
 * (tests and experiment scripts that change the environment after the library is loaded). */
void bht_reload_tuning(void);
/* Number of kernels this library has launched in this process (bench.py's gpu_launches). */
uint64_t bht_kernel_launch_count(void);
size_t bht_sizeof_config(void);

#ifdef __cplusplus
}
#endif
#endif /* BHT_B200_H_ */
