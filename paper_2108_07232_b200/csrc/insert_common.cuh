// insert_common.cuh — pieces shared by the three bulk-insert kernels.
#pragma once
#include "kernels.h"

namespace bht_b200 {

// Appends a dropped key to the table's failed-key log (the GPU image of build_outcome::failed_key,
// reference: proj/include/bht/table.hpp:115-120; a bulk insert can drop more than one).
__device__ __forceinline__ void record_failed(DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, uint32_t key) {
  const unsigned long long pos = atomicAdd(&ctr->failed_recorded, 1ull);
  if (pos < failed_cap) failed_keys[pos] = key;
  atomicMax(&ctr->failed_key_tag, key + 1u);
}

__device__ __forceinline__ void flush_insert_counters(DevCounters* ctr, int lane, uint32_t n_ins, uint32_t n_fail,
                                                      uint32_t n_probe) {
  const unsigned long long a = warp_sum(n_ins), f = warp_sum(n_fail), p = warp_sum(n_probe);
  if (lane == 0) {
    if (a) {
      atomicAdd(&ctr->inserted, a);
      atomicAdd(&ctr->inserted_total, a);
    }
    if (f) atomicAdd(&ctr->failed, f);
    if (p) atomicAdd(&ctr->insert_probes, p);
  }
}

// The (key, value) stream of one warp: the next 32 pairs of the warp's slice are prefetched one
// round ahead; idle lanes take them in order.
struct PairFeed {
  Stream st;
  const uint32_t* keys;
  const uint32_t* values;
  uint32_t ahead_k, ahead_v;

  __device__ __forceinline__ void init(const uint32_t* __restrict__ k, const uint32_t* __restrict__ v, uint64_t n, int lane) {
    st = warp_stream(n);
    keys = k;
    values = v;
    prefetch(lane);
  }
  __device__ __forceinline__ void prefetch(int lane) {
    const uint32_t p = st.cursor + lane;
    const bool in = p < st.len;
    const uint64_t g = st.at(p);
    ahead_k = in ? __ldg(keys + g) : 0u;
    ahead_v = in ? __ldg(values + g) : 0u;
  }
  // Returns true for lanes that received a fresh pair.
  __device__ __forceinline__ bool refill(bool have, int lane, uint32_t& key, uint32_t& val) {
    const uint32_t idle = __ballot_sync(kFullMask, !have);
    if (idle == 0 || st.cursor >= st.len) return false;
    const uint32_t rank = __popc(idle & ((1u << lane) - 1u));
    const uint32_t fk = __shfl_sync(kFullMask, ahead_k, rank);
    const uint32_t fv = __shfl_sync(kFullMask, ahead_v, rank);
    const bool got = !have && st.cursor + rank < st.len;
    if (got) {
      key = fk;
      val = fv;
    }
    st.cursor = min(st.cursor + __popc(idle), st.len);
    prefetch(lane);
    return got;
  }
};

#define BHT_DISPATCH_BUCKET_SIZE(b, CALL)  \
  switch (b) {                             \
    case 1: return CALL(1);                \
    case 2: return CALL(2);                \
    case 4: return CALL(4);                \
    case 8: return CALL(8);                \
    case 16: return CALL(16);              \
    case 32: return CALL(32);              \
    case 64: return CALL(64);              \
    default: return cudaErrorInvalidValue; \
  }

}  // namespace bht_b200
