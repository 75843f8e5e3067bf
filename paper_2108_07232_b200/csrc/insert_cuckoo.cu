// insert_cuckoo.cu — K4: bulk insert for the cuckoo tables (bcht: b >= 1, 3 hashes; 1cht: b = 1, 4 hashes).
//
// Replaces bcht_insert (reference: proj/src/table.cpp:53-92) as driven by build()'s loop
// (table.cpp:224-271):
//   probe the current bucket (first H0);
//   full  -> fail if `chain == max_chain` (cap checked BEFORE the exchange, table.cpp:67), else
//            atomicExch the pair into slot rng.next_below(b) (table.cpp:71), continue with the
//            victim in the bucket named by the hash function AFTER the lowest-index one that maps
//            the victim to this bucket (table.cpp:72-80), ++chain;
//   else  -> atomicCAS(empty -> pair) at slot index = load (table.cpp:85); on a lost race re-probe
//            the same bucket.
// Slot layout may differ from a sequential CPU build (concurrent order); the stored multiset, the
// admissibility of every pair and every query answer do not.
//
// Every lane runs exactly that loop as a state machine over (pair in hand, bucket, chain): one
// loop iteration = one probe round of the warp.  The 32 buckets of a round are fetched together by
// the probe engine, each lane scans its own bucket and issues its own 64-bit atomicCAS / atomicExch,
// and a lane that placed its pair takes the next pair of the warp's slice — eviction chains of one
// lane never idle the other 31.
// The eviction RNG is the reference's xorshift64 (hash.hpp:39-62), one stream per lane seeded
// mix_seed(seed, 0x65766963 + lane id) like the per-worker streams of table.cpp:13,251.
#include "insert_common.cuh"

namespace bht_b200 {

// DIRECT selects the register-resident probe (direct_load) instead of the shared-memory staged one.
template <int B, int H, bool DIRECT>
__global__ void __launch_bounds__(block_threads<B>(1), DIRECT ? 5 : 6)
bulk_insert_cuckoo_kernel(const __grid_constant__ TableView t, const PairSource src, uint64_t n,
                          const unsigned long long* __restrict__ n_dev, const bool routed,
                          DevCounters* __restrict__ ctr, uint32_t* __restrict__ failed_keys, uint64_t failed_cap,
                          uint32_t* __restrict__ work_cursor) {
  using G = Geo<B>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  if (n_dev != nullptr) n = min(n, static_cast<uint64_t>(*n_dev));  // spill list of a blocked build: counted on the device
  const uint32_t stage = DIRECT ? 0u : smem_u32(smem) + (threadIdx.x >> 5) * G::WARP_BYTES;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);

  uint64_t rng = xorshift_init(mix_seed(t.seed, 0x65766963ull + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x));
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;

  PairFeed feed;
  feed.init(src, n, t.chunk_log2, work_cursor, lane);
  bool have = false;
  uint32_t key = 0, val = 0, bid = 0, chain = 0, retries = 0;
  // A lost CAS at slot L proves that slot L is taken now, and occupied slots form a prefix (probe_engine.cuh):
  // the re-snapshot of the reference loop (table.cpp:89) can only report a load > L, so the lane goes straight
  // for slot L + 1 next round without reading the bucket again (`hint`; B = "the bucket is full").
  constexpr uint32_t kNoHint = 0xFFFFFFFFu;
  constexpr uint32_t kSitOut = 0xFFFFFFFEu;  // routed builds: the lane's next bucket is being prefetched into L2
  uint32_t hint = kNoHint;

  // Routed (L2-blocked) build: the pairs arrive grouped by table region in table order, so input position and
  // table position advance together.  (1) A sequential sweep runs `kSweepAhead` of the table ahead of the
  // window: whenever the warp starts a chunk it prefetches the matching slice of the store into L2, so first
  // touches of a bucket are L2 hits.  (2) A bucket outside the region (the next bucket of an evicted pair) is
  // prefetched as soon as it is known and the lane sits one round out; it reads the line when it has arrived.
  // Every round of a warp then waits for L2, not for the slowest HBM access among its 32 lanes.
  const uint32_t lines_per_bucket = (B * 8 + 127) / 128;
  const uint64_t n_lines = (t.num_buckets * B * 8 + 127) / 128;
  uint32_t swept_chunk = 0xFFFFFFFFu;
  if (routed) {  // cold start: the first `sweep_ahead_bytes` of the store
    const uint64_t ahead = min(static_cast<uint64_t>(t.sweep_ahead_bytes) >> 7, n_lines);
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    for (uint64_t l = warp * 32 + lane; l < ahead; l += static_cast<uint64_t>(Stream::grid_warps()) * 32)
      prefetch_l2(reinterpret_cast<const char*>(t.store) + (l << 7));
  }

  for (;;) {
    uint32_t start = kStartAtH0;
    if (feed.refill(src, t.chunk_log2, work_cursor, have, lane, key, val, &start)) {
      have = true;
      // a fresh pair starts at H0 with an empty chain; a victim of the blocked build's in-place first eviction goes
      // on where build_blocked.cu left it
      bid = start == kStartAtH0 ? bucket_index(t.h[0], key) : (start & 0x7FFFFFFFu);
      chain = start == kStartAtH0 ? 0u : (start >> 31);
      if (start == kStartTombstone) have = false;  // the blocked build filled a hole: the list entry holds no pair
      retries = 0;
      hint = kNoHint;
    }
    if (!__any_sync(kFullMask, have)) break;
    if (routed && feed.st.cur != swept_chunk && feed.st.cur < feed.st.n_chunks) {  // warp-uniform
      swept_chunk = feed.st.cur;
      // the slice of this chunk: lines [c * L / n_chunks, (c + 1) * L / n_chunks), shifted ahead
      const uint64_t first = static_cast<uint64_t>(swept_chunk) * n_lines / feed.st.n_chunks;
      const uint64_t last = (static_cast<uint64_t>(swept_chunk) + 1) * n_lines / feed.st.n_chunks;
      const uint64_t ahead = (static_cast<uint64_t>(t.sweep_ahead_bytes) >> 7);
      for (uint64_t l = first + lane; l < last; l += 32)
        if (l + ahead < n_lines) prefetch_l2(reinterpret_cast<const char*>(t.store) + ((l + ahead) << 7));
    }

    const bool sitting = have && hint == kSitOut;
    const bool snapshot = have && hint == kNoHint;
    uint32_t load = hint;
    if constexpr (DIRECT) {
      const uint32_t l = direct_load<B>(t.store, snapshot ? bid : kNoBucket, lane);
      if (snapshot) load = l;
    } else {
      fetch_issue<B>(stage, t.store, snapshot ? bid : kNoBucket, lane);
      if (G::STAGED) fetch_wait();
      if (snapshot) load = scan_bucket<B, false>(stage, t.store, bid, key, lane).load;
    }
    n_probe += snapshot;
    hint = kNoHint;
    // Decide first, then issue the lane's one atomic, then look at the results: the claims (CAS) and the
    // evictions (EXCH) of a round are all in flight together instead of one divergent path after the other.
    const bool claim = have && !sitting && load < B;
    const bool dropped = have && !sitting && !claim && chain >= t.max_chain;  // cap checked BEFORE the exchange (table.cpp:67)
    const bool evict = have && !sitting && !claim && !dropped;
    const uint32_t slot = claim ? load : xorshift_next_below_if(rng, B, evict);
    unsigned long long* target = store + static_cast<uint64_t>(bid) * B + slot;
    const unsigned long long pair = pack_pair(key, val);
    unsigned long long got_c = 0, got_e = 0;  // separate registers: no write-after-write wait between the two
    if (claim) got_c = atomicCAS(target, kEmptySlot, pair);
    if (evict) got_e = atomicExch(target, pair);
    __syncwarp();  // every row is scanned (the next round may overwrite it) and both kinds of atomics are issued
    if (have) {
      if (claim) {
        if (got_c == kEmptySlot) {
          ++n_ins;
          have = false;
        } else if (++retries > t.retry_cap) {
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, key, val);
          have = false;
        } else {
          hint = load + 1;  // lost the slot
        }
      } else if (dropped) {
        ++n_fail;
        record_failed(ctr, failed_keys, failed_cap, key, val);  // the pair in hand is the one dropped
        have = false;
      } else if (evict) {
        const uint32_t vk = static_cast<uint32_t>(got_e);
        if (vk == kEmptyKey) {  // exchanged into a hole: only possible on an uploaded store
          ++n_ins;
          have = false;
        } else {
          uint32_t cand[H];
#pragma unroll
          for (int i = 0; i < H; ++i) cand[i] = bucket_index(t.h[i], vk);
          uint32_t next = cand[0];
#pragma unroll
          for (int i = H - 1; i >= 0; --i)  // lowest matching index wins (table.cpp:74-80)
            if (cand[i] == bid) next = cand[(i + 1) % H];
          key = vk;
          val = static_cast<uint32_t>(got_e >> 32);
          bid = next;
          ++chain;
          if (routed) {  // most likely outside the region: fetch it into L2 now, read it the round after next
#pragma unroll
            for (uint32_t l = 0; l < lines_per_bucket; ++l)
              prefetch_l2(reinterpret_cast<const char*>(t.store + static_cast<uint64_t>(bid) * B) + l * 128);
            hint = kSitOut;
          }
        }
      }
    }
  }

  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

// ---- repair pass ------------------------------------------------------------------------------------------------
// The reference inserts one pair at a time: an eviction chain never meets another walker, and max_chain
// (core.cpp:28-31) is calibrated for that.  A bulk build has ~190 k walkers in flight; near the end of a build at load
// factor 0.99 they are as many as the free slots that remain, take the slots each other was heading for, and hit
// max_chain 3-5 times more often — 50 % of such builds dropped one to three pairs where the reference's build fails
// 10 % of the time (profiles/r01j_*).  So the (few) pairs a launch dropped are inserted ONCE MORE here, by a single
// thread, one after the other, with nobody else moving pairs: the insertion loop of table.cpp:53-92 verbatim, a fresh
// chain of at most max_chain evictions, cap tested before the exchange, lowest-index rotation.  A pair that fails
// again stays failed.  More than `max_repair` dropped pairs means the table is simply over-full: nothing is repaired.
template <int B, int H>
__global__ void repair_dropped_kernel(const __grid_constant__ TableView t, DevCounters* __restrict__ ctr,
                                      uint32_t* __restrict__ failed_keys, uint64_t failed_cap, uint32_t max_repair) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long n_fail = ctr->failed;  // this call's drops: the last n_fail entries of the log
  const unsigned long long end = ctr->failed_recorded;
  if (n_fail == 0 || n_fail > max_repair || end > failed_cap || n_fail > end) return;
  const unsigned long long first = end - n_fail;
  volatile unsigned long long* store = reinterpret_cast<volatile unsigned long long*>(t.store);
  uint64_t rng = xorshift_init(mix_seed(t.seed, 0x72657072ull));
  unsigned long long kept = 0, probes = 0;
  uint32_t tag = 0;
  for (unsigned long long i = first; i < end; ++i) {
    uint32_t key = failed_keys[i], val = failed_keys[failed_cap + i];
    uint32_t bid = bucket_index(t.h[0], key), chain = 0;
    bool placed = false;
    for (;;) {
      ++probes;
      volatile unsigned long long* bucket = store + static_cast<uint64_t>(bid) * B;
      uint32_t load = 0;
      while (load < B && static_cast<uint32_t>(bucket[load]) != kEmptyKey) ++load;  // first empty slot = the load (occupied slots form a prefix)
      if (load < B) {
        bucket[load] = pack_pair(key, val);
        placed = true;
        break;
      }
      if (chain >= t.max_chain) break;  // cap checked BEFORE the exchange (table.cpp:67)
      const uint32_t slot = xorshift_next_below(rng, B);
      const unsigned long long old = bucket[slot];
      bucket[slot] = pack_pair(key, val);
      key = static_cast<uint32_t>(old);
      val = static_cast<uint32_t>(old >> 32);
      uint32_t cand[H];
#pragma unroll
      for (int h = 0; h < H; ++h) cand[h] = bucket_index(t.h[h], key);
      uint32_t next = cand[0];
#pragma unroll
      for (int h = H - 1; h >= 0; --h)  // lowest matching index wins (table.cpp:74-80)
        if (cand[h] == bid) next = cand[(h + 1) % H];
      bid = next;
      ++chain;
    }
    if (!placed) {  // the pair in hand now is the one dropped
      failed_keys[first + kept] = key;
      failed_keys[failed_cap + first + kept] = val;
      ++kept;
      tag = max(tag, key + 1u);
    }
  }
  const unsigned long long repaired = n_fail - kept;
  ctr->failed = kept;
  ctr->failed_recorded = first + kept;
  ctr->failed_key_tag = tag;
  ctr->inserted += repaired;
  ctr->inserted_total += repaired;
  ctr->insert_probes += probes;
}

template <int B, int H>
static cudaError_t launch_repair(const TableView& t, const InsertLaunch& a) {
  if (a.max_repair == 0) return cudaSuccess;
  repair_dropped_kernel<B, H><<<1, 32, 0, a.stream>>>(t, a.ctr, a.failed_keys, a.failed_cap, a.max_repair);
  note_launch();
  return cudaGetLastError();
}

template <int B, int H>
static cudaError_t launch_one(const TableView& t, const InsertLaunch& a) {
  if constexpr (B >= 4 && B <= 16) {
    if (a.direct) {
      auto kernel = bulk_insert_cuckoo_kernel<B, H, true>;
      constexpr int block = block_threads<B>(1);
      int grid = persistent_grid(kernel, block, 0, a.sm_count, a.n, block, a.max_ctas_per_sm);
      if (a.max_grid > 0 && grid > a.max_grid) grid = a.max_grid;
      kernel<<<grid, block, 0, a.stream>>>(t, a.src, a.n, a.n_dev, a.routed, a.ctr, a.failed_keys, a.failed_cap, a.work_cursor);
      note_launch();
      const cudaError_t e = cudaGetLastError();
      return e != cudaSuccess ? e : launch_repair<B, H>(t, a);
    }
  }
  auto kernel = bulk_insert_cuckoo_kernel<B, H, false>;
  constexpr int block = block_threads<B>(1);
  constexpr int smem = (block / 32) * Geo<B>::WARP_BYTES;
  int grid = persistent_grid(kernel, block, smem, a.sm_count, a.n, block, a.max_ctas_per_sm);
  if (a.max_grid > 0 && grid > a.max_grid) grid = a.max_grid;
  kernel<<<grid, block, smem, a.stream>>>(t, a.src, a.n, a.n_dev, a.routed, a.ctr, a.failed_keys, a.failed_cap, a.work_cursor);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? e : launch_repair<B, H>(t, a);
}

cudaError_t launch_insert_cuckoo(const TableView& t, const InsertLaunch& a) {
  if (a.n == 0) return cudaSuccess;
  if (t.n_hashes == 4) {
    if (t.bucket_size != 1) return cudaErrorInvalidValue;
    return launch_one<1, 4>(t, a);
  }
  if (t.n_hashes != 3) return cudaErrorInvalidValue;
#define CALL(BB) launch_one<BB, 3>(t, a)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
