// kernels.h — host-side launch interface between the C ABI (capi.cu) and the kernel TUs.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "probe_engine.cuh"

namespace bht_b200 {

// find.cu — K3 bulk_find<kind, b>.  early_exit selects bcht_find's non-full early exit
// (table.cpp:104); without it the same kernel is bp2ht_find / iht_find / bcht_find_no_early_exit.
cudaError_t launch_find(const TableView& t, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                        DevCounters* ctr, uint32_t* work_cursor, int sm_count, cudaStream_t stream);

// Input of the bulk inserts: two arrays (the caller's keys / values) or one array of packed pairs
// {key, value} (what the region router writes for an L2-blocked build).  Read once: streaming loads.
struct PairSource {
  const uint32_t* keys;
  const uint32_t* values;  // null: `keys` holds packed pairs
  // cuckoo kernel only, optional: where the walk of pair i starts — bits 0..30 the bucket, bit 31 the chain length
  // so far (0 or 1) — for pairs whose first eviction already happened (build_blocked.cu); kStartAtH0 = a fresh pair
  const uint32_t* start = nullptr;
};
constexpr uint32_t kStartAtH0 = 0xFFFFFFFFu;
constexpr uint32_t kStartTombstone = 0xFFFFFFFEu;  // a reserved list entry that holds no pair (the blocked build filled a hole)

struct InsertLaunch {
  PairSource src;
  uint64_t n;
  DevCounters* ctr;
  uint32_t* failed_keys;  // dropped-pair log (failed_cap keys, then failed_cap values) and its capacity
  uint64_t failed_cap;
  uint32_t max_repair = 0;  // cuckoo: after the launch, up to this many dropped pairs are inserted once more, one at a time
  uint32_t* work_cursor;  // one zeroed device word per launch (Stream)
  int sm_count;
  int max_ctas_per_sm;    // 0 = whatever fits; a routed (L2-blocked) build keeps fewer keys in flight
  int max_grid = 0;       // cuckoo: cap on the CTAs of the launch (experiments on the number of keys in flight)
  bool direct;            // cuckoo, 4 <= b <= 16: register-resident probe (direct_load) instead of the staged one
  bool routed = false;    // cuckoo: the pairs arrive grouped by table region in table order (L2-blocked build)
  const unsigned long long* n_dev = nullptr;  // cuckoo: when set, the pair count is read on the device (<= n)
  cudaStream_t stream;
};

// insert_cuckoo.cu — K4 (bcht, 1cht); insert_p2.cu — K5 (bp2ht); insert_iht.cu — K6 (iht).
cudaError_t launch_insert_cuckoo(const TableView& t, const InsertLaunch& a);
cudaError_t launch_insert_p2(const TableView& t, const InsertLaunch& a);
cudaError_t launch_insert_iht(const TableView& t, const InsertLaunch& a);

// insert_claim.cu — K12 (bp2ht) / K13 (iht): counter-claimed insert.  `loads`: one 32-bit load counter per bucket
// (claim_loads_bytes), exact for the store (zero for an empty one, else rebuilt by launch_load_count).
size_t claim_loads_bytes(uint64_t num_buckets);
cudaError_t launch_load_count(const TableView& t, uint32_t* loads, int sm_count, cudaStream_t stream);
cudaError_t launch_claim_insert(const TableView& t, uint32_t* loads, const InsertLaunch& a, bool iht);

// build_blocked.cu — K8g group_scatter + K10 bin_split + K11 region_build: the shared-memory-blocked first pass of a
// cuckoo build.
struct BlockedPlan {
  uint32_t n_regions;    // fine regions (one CTA of K11 each); 0: the blocked build does not apply
  uint32_t region_log2;  // buckets per fine region (64 KiB of slots)
  uint32_t b_log2;
  uint32_t cap;          // pairs per bin (one bin per fine region)
  uint32_t per;          // fine regions per group of the first partition level
  uint32_t n_groups;     // groups (<= kMaxShards)
  uint32_t group_cap;    // pairs per group segment
};
// The counter block and the dropped-key log of the table (what the bulk-insert kernels report failures to).
struct FailLog {
  DevCounters* ctr;
  uint32_t* failed_keys;
  uint64_t failed_cap;
};
BlockedPlan plan_blocked_build(const TableView& t, uint64_t n);
size_t blocked_scratch_bytes(const BlockedPlan& p, uint64_t n);
// Places every pair whose H0 bucket has room; for the others the first eviction is done in place and the victim is
// left in *spill_out (packed pairs + where their walk goes on, *spill_count_out of them, device pointers into
// `scratch`) for launch_insert_cuckoo.
cudaError_t launch_blocked_build(const TableView& t, const BlockedPlan& p, const uint32_t* keys, const uint32_t* values,
                                 uint64_t n, bool fresh, void* scratch, const FailLog& log, int sm_count, cudaStream_t stream,
                                 PairSource* spill_out, const unsigned long long** spill_count_out);
// The same build in steps, for a batch that arrives in chunks (n = the most pairs the chunks may add up to, the value
// the plan and the scratch were sized for): begin, then scatter once per chunk (K8g), then finish (K10 + K11).
cudaError_t blocked_build_begin(const BlockedPlan& p, uint64_t n, void* scratch, cudaStream_t stream);
cudaError_t blocked_build_scatter(const TableView& t, const BlockedPlan& p, uint64_t n, void* scratch, const uint32_t* keys,
                                  const uint32_t* values, uint64_t len, const FailLog& log, int sm_count, cudaStream_t stream,
                                  const unsigned long long* len_dev = nullptr);  // when set: min(len, *len_dev) pairs, read on the device
cudaError_t blocked_build_finish(const TableView& t, const BlockedPlan& p, uint64_t n, void* scratch, bool fresh,
                                 const FailLog& log, int sm_count, cudaStream_t stream, PairSource* spill_out,
                                 const unsigned long long** spill_count_out);

// util.cu — K0 fill, K7 count, admissibility, hash hook, K8/K9 shard routing, synthetic keys.
cudaError_t launch_fill_empty(uint64_t* store, uint64_t n_slots, int sm_count, cudaStream_t stream);
cudaError_t launch_count_occupied(const uint64_t* store, uint64_t n_slots, unsigned long long* out, int sm_count,
                                  cudaStream_t stream);
cudaError_t launch_count_inadmissible(const TableView& t, unsigned long long* out, int sm_count, cudaStream_t stream);
cudaError_t launch_hash_keys(const HashFn& h, const uint32_t* keys, uint32_t* out, uint64_t n, int sm_count,
                             cudaStream_t stream);
// values[i] = value_for_key(keys[i]): the pairing of a keys-only build (table.cpp:234)
cudaError_t launch_derive_values(const uint32_t* keys, uint32_t* values, uint64_t n, int sm_count, cudaStream_t stream);
constexpr int kMaxShards = 256;
// counts / cursors: n_dest device words each; scratch8: n bytes (4-byte aligned) for the per-key destinations.
// out_* receive the elements grouped by destination.
cudaError_t launch_shard_route(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys, const uint32_t* values,
                               uint64_t n, uint8_t* scratch8, unsigned long long* counts, unsigned long long* cursors,
                               uint32_t* out_keys, uint32_t* out_values, uint32_t* out_index, int sm_count, cudaStream_t stream);
// K8s (build_blocked.cu): routing into fixed segments of `cap` elements per destination (what a sync-free all-to-all with
// equal splits sends) in ONE pass with the partition machinery of the blocked build (no classify pass, no destination
// bytes).  counts (device) are clamped to cap, *overflow is set when a destination had more; nothing is copied to the
// host.  insert side: values != null; find side: out_index receives the elements' positions.
cudaError_t launch_shard_split_fixed(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys, const uint32_t* values,
                                     uint64_t n, uint64_t cap, uint32_t* cursor32, unsigned long long* counts, uint32_t* overflow,
                                     uint32_t* out_keys, uint32_t* out_values, uint32_t* out_index, int sm_count, cudaStream_t stream);
// Groups pairs by the table region (n_regions contiguous ranges of buckets) of their first bucket; out_pairs
// receives n packed {key, value} pairs (8 bytes each).
cudaError_t launch_region_route(const HashFn& h0, uint32_t n_regions, const uint32_t* keys, const uint32_t* values, uint64_t n,
                                uint8_t* scratch8, unsigned long long* counts, unsigned long long* cursors, uint32_t* out_pairs,
                                int sm_count, cudaStream_t stream);
cudaError_t launch_unpermute(const uint32_t* answers, const uint32_t* index, uint64_t n, uint32_t* out, int sm_count,
                             cudaStream_t stream);
cudaError_t launch_generate_keys(uint64_t seed, uint64_t offset, uint64_t n, uint32_t* keys, uint32_t* values,
                                 int sm_count, cudaStream_t stream);

// Bumped by every launch_* above (bht_kernel_launch_count).
void note_launch();
uint64_t launch_count();

// Persistent grid: enough CTAs of `block` threads (+ `smem` dynamic bytes) to fill the device, never
// more than the work.
template <typename Kernel>
inline int persistent_grid(Kernel kernel, int block, int smem, int sm_count, uint64_t work_items,
                           uint64_t items_per_block, int max_per_sm = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
  if (max_per_sm > 0 && per_sm > max_per_sm) per_sm = max_per_sm;
  uint64_t need = (work_items + items_per_block - 1) / items_per_block;
  if (need < 1) need = 1;
  const uint64_t fill = static_cast<uint64_t>(per_sm) * static_cast<uint64_t>(sm_count);
  return static_cast<int>(need < fill ? need : fill);
}

}  // namespace bht_b200
