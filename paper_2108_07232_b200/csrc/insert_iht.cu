// insert_iht.cu — K6: bulk insert for the iceberg table (iht).
//
// Replaces iht_insert (reference: proj/src/table.cpp:144-186): probe the primary bucket; when its
// load is AT OR PAST the threshold t (`load >= t`, table.cpp:159, pinned by
// proj/tests/test_table.cpp:125-137) probe both secondaries and take the less loaded one (tie s0)
// unless both are full, in which case the primary stays the choice — except under `prose_fallback`,
// where the secondary is taken regardless (table.cpp:167-169).  A full choice fails the insert
// (table.cpp:180); otherwise atomicCAS(empty -> pair) at slot = load of the choice; on a lost race
// start over from the primary.  1 or 3 probes per attempt.
//
// Lane state machine with two phases: phase 0 fetches the primary; a lane whose primary is at or past
// the threshold keeps that load and, in phase 1, fetches both secondaries (two staging rows per lane)
// before choosing.  Lanes in different phases share the same probe rounds.
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
  bool have = false, overflow = false;  // overflow: phase 1 (primary already read, at or past t)
  uint32_t key = 0, val = 0, pb = 0, pl = 0, s0 = 0, s1 = 0, retries = 0;

  for (;;) {
    if (feed.refill(src, t.chunk_log2, work_cursor, have, lane, key, val)) {
      have = true;
      overflow = false;
      pb = bucket_index(t.h[0], key);
      retries = 0;
    }
    if (!__any_sync(kFullMask, have)) break;

    fetch_issue<B>(stage0, t.store, have ? (overflow ? s0 : pb) : kNoBucket, lane);
    fetch_issue<B>(stage1, t.store, have && overflow ? s1 : kNoBucket, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      bool claim = false;
      uint32_t cb = pb, cl = 0;
      if (!overflow) {
        pl = scan_bucket<B, false>(stage0, t.store, pb, key, lane).load;
        n_probe += 1;
        if (pl >= t.threshold) {
          overflow = true;  // secondaries next round
          s0 = bucket_index(t.h[1], key);
          s1 = bucket_index(t.h[2], key);
        } else {
          claim = true;
          cl = pl;
        }
      } else {
        const uint32_t l0 = scan_bucket<B, false>(stage0, t.store, s0, key, lane).load;
        const uint32_t l1 = scan_bucket<B, false>(stage1, t.store, s1, key, lane).load;
        n_probe += 2;
        claim = true;
        cl = pl;
        if (t.prose || l0 != B || l1 != B) {
          if (l0 <= l1) {
            cb = s0;
            cl = l0;
          } else {
            cb = s1;
            cl = l1;
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
          ++retries;
          overflow = false;  // lost the slot: start over from the primary
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
  const int grid = persistent_grid(kernel, block, smem, a.sm_count, a.n, block, a.max_ctas_per_sm);
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
