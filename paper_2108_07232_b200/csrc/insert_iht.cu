// insert_iht.cu — K6: bulk insert for the iceberg table (iht).
//
// Replaces iht_insert (reference: proj/src/table.cpp:144-186): probe the primary bucket; when its
// load is AT OR PAST the threshold t (`load >= t`, table.cpp:159, pinned by
// proj/tests/test_table.cpp:125-137) probe both secondaries and take the less loaded one (tie s0)
// unless both are full, in which case the primary stays the choice — except under `prose_fallback`,
// where the secondary is taken regardless (table.cpp:167-169).  A full choice fails the insert
// (table.cpp:180); otherwise atomicCAS(empty -> pair) at slot = load of the choice; on a lost race
// decide again.  1 or 3 probes per pair.
//
// Lane state machine: phase 0 fetches the primary; a lane whose primary is at or past the threshold
// keeps that load and, in phase 1, fetches both secondaries (two staging rows per lane); phase 2
// decides from the loads it holds.  Lanes in different phases share the same probe rounds.
// A lost CAS at slot L proves slot L of that bucket is taken and occupied slots form a prefix
// (probe_engine.cuh): the reference's restart from the primary (table.cpp:183-185) could only see
// that bucket at load > L and every other load at least as high as before, so the lane raises its
// copy of the one load to L + 1 and decides again without re-reading anything it already holds (the
// secondaries are still fetched the first time the primary reaches the threshold).
#include "insert_common.cuh"

namespace bht_b200 {

template <int B>
__global__ void __launch_bounds__(block_threads<B>(2))
bulk_insert_iht_kernel(const __grid_constant__ TableView t, const PairSource src, uint64_t n,
                       DevCounters* __restrict__ ctr, uint32_t* __restrict__ failed_keys, uint64_t failed_cap,
                       uint32_t* __restrict__ work_cursor) {
  using G = Geo<B>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const uint32_t stage0 = smem_u32(smem) + (threadIdx.x >> 5) * (2 * G::WARP_BYTES);
  const uint32_t stage1 = stage0 + G::WARP_BYTES;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;

  PairFeed feed;
  feed.init(src, n, t.chunk_log2, work_cursor, lane);
  bool have = false, sec_known = false;  // sec_known: l0 / l1 hold the loads of the secondaries
  uint32_t phase = 0;                    // 0: fetch the primary, 1: fetch the secondaries, 2: decide from what is held
  uint32_t key = 0, val = 0, pb = 0, pl = 0, s0 = 0, s1 = 0, l0 = 0, l1 = 0, retries = 0;

  for (;;) {
    if (feed.refill(src, t.chunk_log2, work_cursor, have, lane, key, val)) {
      have = true;
      phase = 0;
      sec_known = false;
      pb = bucket_index(t.h[0], key);
      retries = 0;
    }
    if (!__any_sync(kFullMask, have)) break;

    fetch_issue<B>(stage0, t.store, have && phase != 2 ? (phase == 1 ? s0 : pb) : kNoBucket, lane);
    fetch_issue<B>(stage1, t.store, have && phase == 1 ? s1 : kNoBucket, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      if (phase == 0) {
        pl = scan_bucket<B, false>(stage0, t.store, pb, key, lane).load;
        n_probe += 1;
      } else if (phase == 1) {
        l0 = scan_bucket<B, false>(stage0, t.store, s0, key, lane).load;
        l1 = scan_bucket<B, false>(stage1, t.store, s1, key, lane).load;
        n_probe += 2;
        sec_known = true;
      }
      phase = 2;
      bool claim = false;
      uint32_t cb = pb, cl = pl, which = 0;  // which: 0 primary, 1 s0, 2 s1
      if (pl < t.threshold) {
        claim = true;
      } else if (!sec_known) {
        phase = 1;  // secondaries next round
        s0 = bucket_index(t.h[1], key);
        s1 = bucket_index(t.h[2], key);
      } else {
        claim = true;
        if (t.prose || l0 != B || l1 != B) {
          if (l0 <= l1) {
            cb = s0, cl = l0, which = 1;
          } else {
            cb = s1, cl = l1, which = 2;
          }
        }
      }
      if (claim) {
        if (cl == B || retries > t.retry_cap) {
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, key);
          have = false;
        } else if (atomicCAS(store + static_cast<uint64_t>(cb) * B + cl, kEmptySlot, pack_pair(key, val)) == kEmptySlot) {
          ++n_ins;
          have = false;
        } else {
          ++retries;  // lost the slot: that bucket holds at least cl + 1 pairs
          if (which == 0) pl = cl + 1;
          else if (which == 1) l0 = cl + 1;
          else l1 = cl + 1;
        }
      }
    }
    if (G::STAGED) __syncwarp();
  }
  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

template <int B>
static cudaError_t launch_one(const TableView& t, const InsertLaunch& a) {
  auto kernel = bulk_insert_iht_kernel<B>;
  constexpr int block = block_threads<B>(2);
  constexpr int smem = (block / 32) * 2 * Geo<B>::WARP_BYTES;
  int grid = persistent_grid(kernel, block, smem, a.sm_count, a.n, block, a.max_ctas_per_sm);
  // Balanced placements are decided on snapshots: with more keys in flight than a fraction of the buckets, every
  // key would choose against an (almost) empty table and the load balance — and with it the find probe means and
  // the reachable load factor — would drift from the sequential process the reference analyses.  Keep the window
  // at or below one key in flight per four buckets (a table of >= 900 k buckets still fills the whole device).
  const uint64_t window_ctas = (t.num_buckets / 4 + block - 1) / block;
  if (static_cast<uint64_t>(grid) > window_ctas) grid = static_cast<int>(window_ctas < 1 ? 1 : window_ctas);
  kernel<<<grid, block, smem, a.stream>>>(t, a.src, a.n, a.ctr, a.failed_keys, a.failed_cap, a.work_cursor);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_insert_iht(const TableView& t, const InsertLaunch& a) {
  if (a.n == 0) return cudaSuccess;
  if (t.n_hashes != 3) return cudaErrorInvalidValue;
#define CALL(BB) launch_one<BB>(t, a)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
