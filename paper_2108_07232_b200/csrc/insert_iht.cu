// insert_iht.cu — K6: bulk insert for the iceberg table (iht).
//
// Replaces iht_insert (reference: proj/src/table.cpp:144-186): probe the primary bucket; when its
// load is AT OR PAST the threshold t (`load >= t`, table.cpp:159, pinned by
// proj/tests/test_table.cpp:125-137) probe both secondaries and take the less loaded one (tie s0)
// unless both are full, in which case the primary stays the choice — except under `prose_fallback`,
// where the secondary is taken regardless (table.cpp:167-169).  A full choice fails the insert
// (table.cpp:180); otherwise atomicCAS(empty -> pair) at slot = load of the choice; on a lost race
// start over from the primary.  1 or 3 probes per attempt.
#include "insert_common.cuh"

namespace bht_b200 {

template <int B>
__global__ void __launch_bounds__(kInsertBlock)
bulk_insert_iht_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys,
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
    const uint32_t pb = bucket_index(t.h[0], key);
    uint32_t retries = 0;

    while (__any_sync(kFullMask, pending)) {
      uint32_t pl;
      probe_load<B>(t.store, pb, pending, lane, pl);
      const bool overflow = pending && pl >= t.threshold;
      uint32_t s0 = 0, s1 = 0, l0 = 0, l1 = 0;
      if (__any_sync(kFullMask, overflow)) {
        s0 = bucket_index(t.h[1], key);
        s1 = bucket_index(t.h[2], key);
        probe_load_pair<B>(t.store, s0, s1, overflow, lane, l0, l1);
      }
      if (pending) {
        n_probe += overflow ? 3 : 1;
        uint32_t cb = pb, cl = pl;
        if (overflow && (t.prose || l0 != B || l1 != B)) {
          if (l0 <= l1) {
            cb = s0;
            cl = l0;
          } else {
            cb = s1;
            cl = l1;
          }
        }
        if (cl == B || retries > t.retry_cap) {
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, key);
          pending = false;
        } else {
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
  auto kernel = bulk_insert_iht_kernel<B>;
  const int grid = persistent_grid(kernel, kInsertBlock, sm_count, n, kInsertBlock);
  kernel<<<grid, kInsertBlock, 0, stream>>>(t, keys, values, n, ctr, failed_keys, failed_cap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_insert_iht(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                              DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                              cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (t.n_hashes != 3) return cudaErrorInvalidValue;
#define CALL(BB) launch_one<BB>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
