// insert_p2.cu — K5: bulk insert for the bucketed power-of-two-choices table (bp2ht).
//
// Replaces bp2ht_insert (reference: proj/src/table.cpp:109-130): read BOTH candidate buckets
// (2 probes, always), fail only if both are full, otherwise atomicCAS(empty -> pair) at slot
// min(load0, load1) of the less loaded bucket, ties to H0 (table.cpp:124); on a lost race read both
// again.  Placed pairs never move.
//
// The 2 x 32 bucket reads of a warp batch go through the paired probe engine (8 lines in flight per
// tile step group), and the 32 claims are one warp-wide 64-bit atomicCAS.  Lanes that lost their CAS
// repeat the round; rounds with few pending lanes skip the idle probe steps.
#include "insert_common.cuh"

namespace bht_b200 {

template <int B>
__global__ void __launch_bounds__(kInsertBlock)
bulk_insert_p2_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys,
                      const uint32_t* __restrict__ values, uint64_t n, DevCounters* __restrict__ ctr,
                      uint32_t* __restrict__ failed_keys, uint64_t failed_cap) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t n_batches = (n + 31) >> 5;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;

  for (uint64_t batch = warp; batch < n_batches; batch += n_warps) {
    const uint64_t idx = (batch << 5) + lane;
    const bool valid = idx < n;
    const uint32_t key = valid ? __ldcs(keys + idx) : kEmptyKey;
    const uint32_t val = valid ? __ldcs(values + idx) : kEmptyKey;
    bool pending = valid;
    const uint32_t b0 = bucket_index(t.h[0], key);
    const uint32_t b1 = bucket_index(t.h[1], key);
    uint32_t retries = 0;

    while (__any_sync(kFullMask, pending)) {
      uint32_t l0, l1;
      probe_load_pair<B>(t.store, b0, b1, pending, lane, l0, l1);
      if (pending) {
        n_probe += 2;
        if ((l0 == B && l1 == B) || retries > t.retry_cap) {
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, key);
          pending = false;
        } else {
          const uint32_t cb = l0 <= l1 ? b0 : b1;  // tie -> first hash function
          const uint32_t cl = l0 <= l1 ? l0 : l1;
          const unsigned long long old =
              atomicCAS(store + static_cast<uint64_t>(cb) * B + cl, kEmptySlot, pack_pair(key, val));
          if (old == kEmptySlot) {
            ++n_ins;
            pending = false;
          } else {
            ++retries;
          }
        }
      }
    }
  }
  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

template <int B>
static cudaError_t launch_one(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                              DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                              cudaStream_t stream) {
  auto kernel = bulk_insert_p2_kernel<B>;
  const int grid = persistent_grid(kernel, kInsertBlock, sm_count, n, kInsertBlock);
  kernel<<<grid, kInsertBlock, 0, stream>>>(t, keys, values, n, ctr, failed_keys, failed_cap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_insert_p2(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                             DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (t.n_hashes != 2) return cudaErrorInvalidValue;
#define CALL(BB) launch_one<BB>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
