// probe_engine.cuh — the bucket probe engine.
//
// Replaces bucket_ref (reference: proj/include/bht/bucket.hpp:16-63): the snapshot read of a whole
// bucket (= one probe, bucket.hpp:18-21), compute_load (:26-31), full (:33) and find_key_value
// (:36-41).  cas_at_slot / exch_at_slot (:45-55) are single 64-bit atomics issued by the callers.
//
// Geometry.  A bucket of B 8-byte slots is read by a tile of LPB = B/2 lanes, each issuing ONE
// 16-byte vector load (two slots), so a b=16 bucket is one fully-used 128-byte line fetched by 8
// lanes and a warp-wide load instruction covers 4 buckets (B=1 is one 8-byte load per lane).
// Match / load results come from __ballot_sync + __ffs / __popc over the tile's slice of the warp
// ballot.
//
// Batching.  Every lane owns one key.  The LPB lanes of a tile serve their own LPB keys in LPB
// steps (step u serves the key of tile lane u), and up to BATCH = 8 steps have their loads issued
// back to back before any is consumed, so one warp keeps up to 8 x 4 = 32 independent 128-byte
// lines in flight.  Steps in which no tile of the warp has a pending key are skipped (warp-uniform
// branch), which keeps later probe rounds cheap.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hash_stage.cuh"

namespace bht_b200 {

constexpr unsigned kFullMask = 0xFFFFFFFFu;

template <int B>
struct Geo {
  static_assert(B == 1 || B == 2 || B == 4 || B == 8 || B == 16 || B == 32 || B == 64, "bucket size");
  static constexpr int SPL = B >= 2 ? 2 : 1;      // slots per lane
  static constexpr int LPB = B / SPL;             // lanes per bucket (tile width)
  static constexpr int BATCH = LPB < 8 ? LPB : 8; // probe steps whose loads are batched
  static constexpr int PAIR_BATCH = LPB < 4 ? LPB : 4;
  static constexpr uint32_t GMASK = LPB == 32 ? 0xFFFFFFFFu : ((1u << LPB) - 1u);
};

// Two adjacent slots as loaded by one lane: (k0, v0) = slot 2*sub, (k1, v1) = slot 2*sub+1.
struct Slot2 {
  uint32_t k0, v0, k1, v1;
};

__device__ __forceinline__ Slot2 empty_slot2() { return Slot2{kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey}; }

// Read-only table (find): non-coherent path, no L1 allocation — every line is used exactly once.
__device__ __forceinline__ uint4 ld_table_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_table_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
// Table under construction (insert): L2-coherent loads; L1 may hold stale lines across SMs.
__device__ __forceinline__ uint4 ld_table_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ uint2 ld_table_cg_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}

// One lane's share of bucket `bid`: slots [SPL*sub, SPL*sub + SPL).
template <int B, bool COHERENT>
__device__ __forceinline__ Slot2 load_lane(const uint64_t* __restrict__ store, uint32_t bid, int sub) {
  const uint64_t* p = store + static_cast<uint64_t>(bid) * B + sub * Geo<B>::SPL;
  if constexpr (B >= 2) {
    const uint4 v = COHERENT ? ld_table_cg_v4(p) : ld_table_nc_v4(p);
    return Slot2{v.x, v.y, v.z, v.w};
  } else {
    const uint2 v = COHERENT ? ld_table_cg_v2(p) : ld_table_nc_v2(p);
    return Slot2{v.x, v.y, kEmptyKey, kEmptyKey};
  }
}

// OR of the per-tile activity masks: bit u set <=> some tile of the warp has a pending key at tile
// lane u.  Warp-uniform.
template <int LPB>
__device__ __forceinline__ uint32_t union_over_tiles(uint32_t act) {
#pragma unroll
  for (int s = LPB; s < 32; s <<= 1) act |= act >> s;
  return act;
}

// ---- find probe -----------------------------------------------------------------------------
// For every lane with my_active: one probe of bucket my_bid looking for my_key.
//   found   <=> some slot holds my_key (lowest slot wins, bucket.hpp:36-41)
//   value   value of that slot
//   notfull <=> the bucket has an empty slot (!full(), bucket.hpp:33)
template <int B>
__device__ __forceinline__ void probe_find(const uint64_t* __restrict__ store, uint32_t my_bid, bool my_active,
                                           uint32_t my_key, int lane, bool& found, uint32_t& value, bool& notfull) {
  using G = Geo<B>;
  found = false;
  notfull = false;
  value = kEmptyKey;
  if constexpr (G::LPB == 1) {
    if (my_active) {
      const Slot2 s = load_lane<B, false>(store, my_bid, 0);
      const bool m0 = s.k0 == my_key;
      const bool m1 = B == 2 && s.k1 == my_key;
      found = m0 || m1;
      value = m0 ? s.v0 : (m1 ? s.v1 : kEmptyKey);
      notfull = s.k0 == kEmptyKey || (B == 2 && s.k1 == kEmptyKey);
    }
  } else {
    const int sub = lane & (G::LPB - 1);
    const int gbase = lane & ~(G::LPB - 1);
    const uint32_t act = __ballot_sync(kFullMask, my_active);
    const uint32_t any = union_over_tiles<G::LPB>(act);
    const uint32_t mine = (act >> gbase) & G::GMASK;
#pragma unroll
    for (int base = 0; base < G::LPB; base += G::BATCH) {
      Slot2 s[G::BATCH];
#pragma unroll
      for (int u = 0; u < G::BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;  // warp-uniform
        const uint32_t bid = __shfl_sync(kFullMask, my_bid, base + u, G::LPB);
        s[u] = ((mine >> (base + u)) & 1u) ? load_lane<B, false>(store, bid, sub) : empty_slot2();
      }
#pragma unroll
      for (int u = 0; u < G::BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;
        const uint32_t qk = __shfl_sync(kFullMask, my_key, base + u, G::LPB);
        const bool a = (mine >> (base + u)) & 1u;
        const bool m0 = a && s[u].k0 == qk;
        const bool m1 = a && s[u].k1 == qk;
        const uint32_t bm = __ballot_sync(kFullMask, m0 || m1);
        const uint32_t be = __ballot_sync(kFullMask, s[u].k0 == kEmptyKey || s[u].k1 == kEmptyKey);
        const uint32_t gm = (bm >> gbase) & G::GMASK;
        const uint32_t myval = m0 ? s[u].v0 : s[u].v1;
        const int src = gm ? (__ffs(gm) - 1) : 0;
        const uint32_t val = __shfl_sync(kFullMask, myval, src, G::LPB);
        if (sub == base + u) {
          found = gm != 0;
          value = gm ? val : kEmptyKey;
          notfull = ((be >> gbase) & G::GMASK) != 0;
        }
      }
    }
  }
}

// ---- load probe (insert side) ---------------------------------------------------------------
// For every lane with my_active: load = number of occupied slots of bucket my_bid
// (compute_load, bucket.hpp:26-31), read through L2 so concurrent inserts are visible.
template <int B>
__device__ __forceinline__ void probe_load(const uint64_t* __restrict__ store, uint32_t my_bid, bool my_active,
                                           int lane, uint32_t& load) {
  using G = Geo<B>;
  load = 0;
  if constexpr (G::LPB == 1) {
    if (my_active) {
      const Slot2 s = load_lane<B, true>(store, my_bid, 0);
      load = (s.k0 != kEmptyKey) + (B == 2 && s.k1 != kEmptyKey);
    }
  } else {
    const int sub = lane & (G::LPB - 1);
    const int gbase = lane & ~(G::LPB - 1);
    const uint32_t act = __ballot_sync(kFullMask, my_active);
    const uint32_t any = union_over_tiles<G::LPB>(act);
    const uint32_t mine = (act >> gbase) & G::GMASK;
#pragma unroll
    for (int base = 0; base < G::LPB; base += G::BATCH) {
      Slot2 s[G::BATCH];
#pragma unroll
      for (int u = 0; u < G::BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;
        const uint32_t bid = __shfl_sync(kFullMask, my_bid, base + u, G::LPB);
        s[u] = ((mine >> (base + u)) & 1u) ? load_lane<B, true>(store, bid, sub) : empty_slot2();
      }
#pragma unroll
      for (int u = 0; u < G::BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;
        const uint32_t n0 = __ballot_sync(kFullMask, s[u].k0 != kEmptyKey);
        const uint32_t n1 = __ballot_sync(kFullMask, s[u].k1 != kEmptyKey);
        if (sub == base + u) load = __popc((n0 >> gbase) & G::GMASK) + __popc((n1 >> gbase) & G::GMASK);
      }
    }
  }
}

// Two buckets per key (bp2ht both choices, iht both secondaries): loads of bid_a and bid_b.
template <int B>
__device__ __forceinline__ void probe_load_pair(const uint64_t* __restrict__ store, uint32_t bid_a, uint32_t bid_b,
                                                bool my_active, int lane, uint32_t& load_a, uint32_t& load_b) {
  using G = Geo<B>;
  load_a = 0;
  load_b = 0;
  if constexpr (G::LPB == 1) {
    if (my_active) {
      const Slot2 a = load_lane<B, true>(store, bid_a, 0);
      const Slot2 b = load_lane<B, true>(store, bid_b, 0);
      load_a = (a.k0 != kEmptyKey) + (B == 2 && a.k1 != kEmptyKey);
      load_b = (b.k0 != kEmptyKey) + (B == 2 && b.k1 != kEmptyKey);
    }
  } else {
    const int sub = lane & (G::LPB - 1);
    const int gbase = lane & ~(G::LPB - 1);
    const uint32_t act = __ballot_sync(kFullMask, my_active);
    const uint32_t any = union_over_tiles<G::LPB>(act);
    const uint32_t mine = (act >> gbase) & G::GMASK;
#pragma unroll
    for (int base = 0; base < G::LPB; base += G::PAIR_BATCH) {
      Slot2 sa[G::PAIR_BATCH], sb[G::PAIR_BATCH];
#pragma unroll
      for (int u = 0; u < G::PAIR_BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;
        const uint32_t ba = __shfl_sync(kFullMask, bid_a, base + u, G::LPB);
        const uint32_t bb = __shfl_sync(kFullMask, bid_b, base + u, G::LPB);
        const bool a = (mine >> (base + u)) & 1u;
        sa[u] = a ? load_lane<B, true>(store, ba, sub) : empty_slot2();
        sb[u] = a ? load_lane<B, true>(store, bb, sub) : empty_slot2();
      }
#pragma unroll
      for (int u = 0; u < G::PAIR_BATCH; ++u) {
        if (!((any >> (base + u)) & 1u)) continue;
        const uint32_t a0 = __ballot_sync(kFullMask, sa[u].k0 != kEmptyKey);
        const uint32_t a1 = __ballot_sync(kFullMask, sa[u].k1 != kEmptyKey);
        const uint32_t b0 = __ballot_sync(kFullMask, sb[u].k0 != kEmptyKey);
        const uint32_t b1 = __ballot_sync(kFullMask, sb[u].k1 != kEmptyKey);
        if (sub == base + u) {
          load_a = __popc((a0 >> gbase) & G::GMASK) + __popc((a1 >> gbase) & G::GMASK);
          load_b = __popc((b0 >> gbase) & G::GMASK) + __popc((b1 >> gbase) & G::GMASK);
        }
      }
    }
  }
}

// Tile-synchronous probe: all LPB lanes of a tile pass the same bid / have; returns the load of
// that one bucket to every lane of the tile (used by the eviction state machine).
template <int B>
__device__ __forceinline__ uint32_t tile_probe_load(const uint64_t* __restrict__ store, uint32_t bid, bool have, int lane) {
  using G = Geo<B>;
  const int sub = lane & (G::LPB - 1);
  const Slot2 s = have ? load_lane<B, true>(store, bid, sub) : empty_slot2();
  if constexpr (G::LPB == 1) {
    return (s.k0 != kEmptyKey) + (B == 2 && s.k1 != kEmptyKey);
  } else {
    const int gbase = lane & ~(G::LPB - 1);
    const uint32_t n0 = __ballot_sync(kFullMask, s.k0 != kEmptyKey);
    const uint32_t n1 = __ballot_sync(kFullMask, s.k1 != kEmptyKey);
    return __popc((n0 >> gbase) & G::GMASK) + __popc((n1 >> gbase) & G::GMASK);
  }
}

// ---- shared kernel plumbing -----------------------------------------------------------------

struct TableView {
  uint64_t* store;
  HashFn h[4];
  uint64_t num_buckets;
  uint64_t seed;
  uint32_t n_hashes;
  uint32_t bucket_size;
  uint32_t threshold;
  uint32_t max_chain;
  uint32_t prose;
  uint32_t retry_cap;  // bound on CAS-loss retries per key (a legit table needs <= 3*b)
};

struct DevCounters {
  // ---- per call: zeroed at the start of every bht_insert / bht_find ----
  unsigned long long inserted;
  unsigned long long failed;
  unsigned long long insert_probes;
  unsigned long long find_hits;
  unsigned long long find_probes;
  unsigned long long find_value_sum;
  unsigned int failed_key_tag;  // max over dropped keys of key + 1; 0 = none dropped
  unsigned int pad;
  // ---- since bht_clear / bht_upload_store ----
  unsigned long long scratch;          // count_occupied / count_inadmissible result
  unsigned long long failed_recorded;  // entries appended to the failed-key log
  unsigned long long inserted_total;
};
constexpr size_t kPerCallCounterBytes = 7 * sizeof(unsigned long long);

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

__device__ __forceinline__ uint64_t pack_pair(uint32_t key, uint32_t value) {
  return (static_cast<uint64_t>(value) << 32) | key;
}

}  // namespace bht_b200
