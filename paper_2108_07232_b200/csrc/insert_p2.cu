// insert_p2.cu — K5: bulk insert for the bucketed power-of-two-choices table (bp2ht).
//
// Replaces bp2ht_insert (reference: proj/src/table.cpp:109-130): read BOTH candidate buckets
// (2 probes, always), fail only if both are full, otherwise atomicCAS(empty -> pair) at slot
// min(load0, load1) of the less loaded bucket, ties to H0 (table.cpp:124); on a lost race decide
// again.  Placed pairs never move.
//
// One round of a warp fetches 2 x 32 buckets (two staging rows per lane); each lane compares its two
// loads and issues its own claim; lanes that lost their CAS repeat, the others take new pairs.
// A lost CAS at slot L proves that slot L of that bucket is taken and occupied slots form a prefix
// (probe_engine.cuh), so the reference's re-snapshot (table.cpp:127-129) could only report load > L
// there: the lane raises its copy of that load to L + 1 and decides again WITHOUT reading the buckets
// a second time.  Probe counts therefore stay at exactly 2 per pair however many keys of a small
// table are in flight together (bp2ht b = 16, 200 k keys, all in flight: 3.6 probes per pair with the
// re-read, 2.0 without).
#include "insert_common.cuh"

namespace bht_b200 {

template <int B>
__global__ void __launch_bounds__(block_threads<B>(2))
bulk_insert_p2_kernel(const __grid_constant__ TableView t, const PairSource src, uint64_t n,
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
  bool have = false;
  uint32_t key = 0, val = 0, b0 = 0, b1 = 0, l0 = 0, l1 = 0, retries = 0;
  bool known = false;  // l0 / l1 hold the loads of b0 / b1 (snapshot, raised by lost claims)

  for (;;) {
    if (feed.refill(src, t.chunk_log2, work_cursor, have, lane, key, val)) {
      have = true;
      b0 = bucket_index(t.h[0], key);
      b1 = bucket_index(t.h[1], key);
      retries = 0;
      known = false;
    }
    if (!__any_sync(kFullMask, have)) break;

    const bool snapshot = have && !known;
    fetch_issue<B>(stage0, t.store, snapshot ? b0 : kNoBucket, lane);
    fetch_issue<B>(stage1, t.store, snapshot ? b1 : kNoBucket, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      if (snapshot) {
        l0 = scan_bucket<B, false>(stage0, t.store, b0, key, lane).load;
        l1 = scan_bucket<B, false>(stage1, t.store, b1, key, lane).load;
        n_probe += 2;
        known = true;
      }
      if ((l0 == B && l1 == B) || retries > t.retry_cap) {
        ++n_fail;
        record_failed(ctr, failed_keys, failed_cap, key);
        have = false;
      } else {
        const uint32_t cb = l0 <= l1 ? b0 : b1;  // tie -> first hash function
        const uint32_t cl = l0 <= l1 ? l0 : l1;
        if (atomicCAS(store + static_cast<uint64_t>(cb) * B + cl, kEmptySlot, pack_pair(key, val)) == kEmptySlot) {
          ++n_ins;
          have = false;
        } else {
          ++retries;
          if (l0 <= l1) l0 = cl + 1; else l1 = cl + 1;  // lost the slot: that bucket holds at least cl + 1 pairs
        }
      }
    }
    if (G::STAGED) __syncwarp();
  }
  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

template <int B>
static cudaError_t launch_one(const TableView& t, const InsertLaunch& a) {
  auto kernel = bulk_insert_p2_kernel<B>;
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

cudaError_t launch_insert_p2(const TableView& t, const InsertLaunch& a) {
  if (a.n == 0) return cudaSuccess;
  if (t.n_hashes != 2) return cudaErrorInvalidValue;
#define CALL(BB) launch_one<BB>(t, a)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
