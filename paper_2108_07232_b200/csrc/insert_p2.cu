// insert_p2.cu — K5: bulk insert for the bucketed power-of-two-choices table (bp2ht).
//
// Replaces bp2ht_insert (reference: proj/src/table.cpp:109-130): read BOTH candidate buckets
// (2 probes, always), fail only if both are full, otherwise atomicCAS(empty -> pair) at slot
// min(load0, load1) of the less loaded bucket, ties to H0 (table.cpp:124); on a lost race read both
// again.  Placed pairs never move.
//
// One round of a warp fetches 2 x 32 buckets (two staging rows per lane); each lane compares its two
// loads and issues its own claim; lanes that lost their CAS repeat, the others take new pairs.
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
  uint32_t key = 0, val = 0, b0 = 0, b1 = 0, retries = 0;

  for (;;) {
    if (feed.refill(src, t.chunk_log2, work_cursor, have, lane, key, val)) {
      have = true;
      b0 = bucket_index(t.h[0], key);
      b1 = bucket_index(t.h[1], key);
      retries = 0;
    }
    if (!__any_sync(kFullMask, have)) break;

    fetch_issue<B>(stage0, t.store, have ? b0 : kNoBucket, lane);
    fetch_issue<B>(stage1, t.store, have ? b1 : kNoBucket, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      const uint32_t l0 = scan_bucket<B, false>(stage0, t.store, b0, key, lane).load;
      const uint32_t l1 = scan_bucket<B, false>(stage1, t.store, b1, key, lane).load;
      n_probe += 2;
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
  const int grid = persistent_grid(kernel, block, smem, a.sm_count, a.n, block, a.max_ctas_per_sm);
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
