// insert_common.cuh — pieces shared by the three bulk-insert kernels.
#pragma once
#include "kernels.h"

namespace bht_b200 {

// Appends a dropped key to the table's failed-key log (the GPU image of build_outcome::failed_key,
// reference: proj/include/bht/table.hpp:115-120; a bulk insert can drop more than one).
// The log holds failed_cap keys followed by failed_cap values (the value of a dropped pair lets the cuckoo repair pass,
// insert_cuckoo.cu, insert it once more).
__device__ __forceinline__ void record_failed(DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, uint32_t key,
                                              uint32_t value = 0u) {
  const unsigned long long pos = atomicAdd(&ctr->failed_recorded, 1ull);
  if (pos < failed_cap) {
    failed_keys[pos] = key;
    failed_keys[failed_cap + pos] = value;
  }
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

// The (key, value) stream of one warp: the next 32 pairs of the warp's stream are prefetched one
// round ahead; idle lanes take them in order.
struct PairFeed {
  Stream st;
  uint32_t ahead_k, ahead_v, ahead_s;
  uint32_t ahead_n;  // how many of the 32 prefetched pairs exist (warp-uniform)

  // src / shift / cursor are kernel parameters: passed at every call rather than kept in registers
  __device__ __forceinline__ void init(const PairSource& src, uint64_t n, uint32_t shift, uint32_t* cursor, int lane) {
    st.init(n, shift, cursor, lane);
    prefetch(src, shift, lane);
  }
  __device__ __forceinline__ void prefetch(const PairSource& src, uint32_t shift, int lane) {
    uint64_t g;
    const bool in = st.index(lane, shift, g);
    ahead_k = ahead_v = 0u;
    ahead_s = kStartAtH0;
    if (in && src.start != nullptr) ahead_s = __ldcs(src.start + g);  // kernel-uniform pointer test
    if (in) {
      if (src.values == nullptr) {  // kernel-uniform
        const uint2 kv = __ldcs(reinterpret_cast<const uint2*>(src.keys) + g);
        ahead_k = kv.x;
        ahead_v = kv.y;
      } else {
        ahead_k = __ldcs(src.keys + g);
        ahead_v = __ldcs(src.values + g);
      }
    }
    ahead_n = __popc(__ballot_sync(kFullMask, in));
  }
  // Returns true for lanes that received a fresh pair.
  __device__ __forceinline__ bool refill(const PairSource& src, uint32_t shift, uint32_t* cursor, bool have, int lane,
                                         uint32_t& key, uint32_t& val, uint32_t* start = nullptr) {
    const uint32_t idle = __ballot_sync(kFullMask, !have);
    if (idle == 0 || ahead_n == 0) return false;
    const uint32_t rank = __popc(idle & ((1u << lane) - 1u));
    const uint32_t fk = __shfl_sync(kFullMask, ahead_k, rank);
    const uint32_t fv = __shfl_sync(kFullMask, ahead_v, rank);
    uint32_t fs = kStartAtH0;
    if (start != nullptr && src.start != nullptr) fs = __shfl_sync(kFullMask, ahead_s, rank);  // warp-uniform branch
    const bool got = !have && rank < ahead_n;
    if (got) {
      key = fk;
      val = fv;
      if (start != nullptr) *start = fs;
    }
    st.advance(min(static_cast<uint32_t>(__popc(idle)), ahead_n), shift, cursor, lane);
    prefetch(src, shift, lane);
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
