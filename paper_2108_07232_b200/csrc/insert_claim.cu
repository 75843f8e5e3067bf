// insert_claim.cu — K12 / K13: counter-claimed bulk insert for the balanced tables (bp2ht, iht) when the store lives in HBM.
//
// bp2ht_insert / iht_insert (reference: proj/src/table.cpp:109-130, 144-186) read their candidate buckets only to learn
// their LOADS (bucket.hpp:26-31); the claim itself is one CAS at slot = load (table.cpp:126,181).  On a 444 MB store
// that is 2 (bp2ht) or 1-3 (iht) random 128-byte line reads per pair plus the write-back of the claimed sector, and the
// kernels of insert_p2.cu / insert_iht.cu run at HBM's random-access ceiling (44-48 G accesses/s).  Here the loads live
// in a side array — one 32-bit counter per bucket, 14 MB for 3.5 M buckets, L2-resident — kept exact by the inserts
// themselves:
//   read the counters of the candidates (L2 hits), decide exactly as the reference does (less loaded, ties to the first
//   hash function; iht: primary while its load is below t), claim slot = old counter with one atomic on the counter, and
//   write the pair with one 8-byte store.  The store is the only HBM access of an insertion.
// The order of the decisions is the caller's order (a sliding window of keys in flight, as in the other kernels), so the
// placement statistics are those of the reference's process; nothing is grouped by bucket.
// Claim rules:  bp2ht — CAS on the counter from the load that was read to load + 1; a bucket that moved is decided again
//   with fresh loads (the lost-race case of table.cpp:127-129), no probe is counted twice.
//   iht secondaries — atomicAdd on the counter; a returned value >= b means the bucket filled up since it was read: the
//   lane marks it full and decides again.  A counter can therefore overshoot b by the number of such late claimers (at most the keys in flight,
//   far below 2^32, even when every key of a batch is the same); every reader clamps it.
//   iht primary — the rule "stay while load < t" (table.cpp:159) is enforced exactly with a CAS on the counter word.
// The counters are rebuilt from the store (load_count_kernel) whenever something else may have written slots
// (bht_upload_store, the per-bucket CAS kernels of small batches, bht_device_store).
// Measured on B200 (tools/microbench/random_store.cu): 2 counter reads + atomicAdd + 8-byte store = 24.7 G keys/s over a
// 444 MB table, against 14.9 G keys/s for the bucket-reading bp2ht kernel.
#include <algorithm>

#include "insert_common.cuh"

namespace bht_b200 {

namespace {

constexpr int kClaimBlock = 256;

__device__ __forceinline__ uint32_t read_load(const uint32_t* __restrict__ loads, uint32_t bucket, uint32_t b) {
  return min(__ldcg(loads + bucket), b);
}
// Claims the next slot of `bucket`: returns the slot index, or b when the bucket is (now) full.
__device__ __forceinline__ uint32_t claim_slot(uint32_t* __restrict__ loads, uint32_t bucket, uint32_t b) {
  return min(atomicAdd(loads + bucket, 1u), b);
}
// Claims slot = load of `bucket` only while load < limit (iht primary): returns the slot, or the load that stopped it.
__device__ __forceinline__ uint32_t claim_slot_below(uint32_t* __restrict__ loads, uint32_t bucket, uint32_t limit, uint32_t b,
                                                      bool& claimed) {
  uint32_t old = __ldcg(loads + bucket);
  for (;;) {
    if (old >= limit) {
      claimed = false;
      return min(old, b);
    }
    const uint32_t seen = atomicCAS(loads + bucket, old, old + 1u);
    if (seen == old) {
      claimed = true;
      return old;
    }
    old = seen;
  }
}

__device__ __forceinline__ uint4 load4(const uint32_t* __restrict__ p, uint64_t i, uint64_t n, bool aligned) {
  if (aligned && i + 4 <= n) return __ldcs(reinterpret_cast<const uint4*>(p + i));
  uint4 r = make_uint4(0, 0, 0, 0);
  if (i < n) r.x = p[i];
  if (i + 1 < n) r.y = p[i + 1];
  if (i + 2 < n) r.z = p[i + 2];
  if (i + 3 < n) r.w = p[i + 3];
  return r;
}

// load of every bucket = 1 + index of its last occupied slot (compute_load whenever the occupied slots form a prefix)
__global__ void __launch_bounds__(kClaimBlock)
load_count_kernel(const uint64_t* __restrict__ store, uint64_t num_buckets, uint32_t b, uint32_t* __restrict__ loads) {
  for (uint64_t bucket = static_cast<uint64_t>(blockIdx.x) * kClaimBlock + threadIdx.x; bucket < num_buckets;
       bucket += static_cast<uint64_t>(gridDim.x) * kClaimBlock) {
    uint32_t load = 0;
    for (uint32_t s = 0; s < b; ++s)
      if (static_cast<uint32_t>(store[bucket * b + s]) != kEmptyKey) load = s + 1;
    loads[bucket] = load;
  }
}

// ---- K12: bp2ht -----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kClaimBlock)
claim_insert_p2_kernel(const __grid_constant__ TableView t, uint32_t* __restrict__ loads, const PairSource src, uint64_t n, bool aligned,
                       DevCounters* __restrict__ ctr, uint32_t* __restrict__ failed_keys, uint64_t failed_cap) {
  const uint32_t B = t.bucket_size;
  const int lane = threadIdx.x & 31;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kClaimBlock * 4;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * kClaimBlock + threadIdx.x) * 4; i < n; i += stride) {
    uint32_t k[4], v[4];
    if (src.values == nullptr) {  // packed pairs
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint2 kv = i + e < n ? __ldcs(reinterpret_cast<const uint2*>(src.keys) + i + e) : make_uint2(0u, 0u);
        k[e] = kv.x, v[e] = kv.y;
      }
    } else {
      const uint4 k4 = load4(src.keys, i, n, aligned), v4 = load4(src.values, i, n, aligned);
      k[0] = k4.x, k[1] = k4.y, k[2] = k4.z, k[3] = k4.w;
      v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
    }
    uint32_t b0[4], b1[4], l0[4], l1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      b0[e] = bucket_index(t.h[0], k[e]);
      b1[e] = bucket_index(t.h[1], k[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // the two probes of table.cpp:113-116: the loads of both candidates
      l0[e] = read_load(loads, b0[e], B);
      l1[e] = read_load(loads, b1[e], B);
    }
    // The claim is a CAS from the load that was read to load + 1: a bucket that changed in between is decided again with
    // its fresh load, exactly the lost-race path of table.cpp:127-129.  (A blind atomicAdd would let hundreds of thousands
    // of keys in flight act on the same stale loads; measured, that costs bp2ht 0.03-0.05 of achievable load factor.)
    // First one attempt for each of the four keys, all in flight together; then the retries.
    uint32_t cb[4], cl[4], seen[4];
    bool tried[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool first = l0[e] <= l1[e];  // tie -> first hash function (table.cpp:124)
      cb[e] = first ? b0[e] : b1[e];
      cl[e] = first ? l0[e] : l1[e];
      tried[e] = i + e < n && cl[e] < B;
      seen[e] = cl[e];
      if (tried[e]) seen[e] = atomicCAS(loads + cb[e], cl[e], cl[e] + 1u);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (i + e >= n) continue;
      n_probe += 2;
      bool placed = tried[e] && seen[e] == cl[e];
      while (!placed) {
        if (tried[e]) {  // the chosen bucket moved: take its fresh load, look at the other one again, decide again
          const uint32_t fresh = min(seen[e], B);
          if (cb[e] == b0[e]) l0[e] = fresh, l1[e] = b0[e] == b1[e] ? fresh : read_load(loads, b1[e], B);
          else l1[e] = fresh, l0[e] = read_load(loads, b0[e], B);
        }
        if (l0[e] == B && l1[e] == B) break;  // both full: the insertion fails (table.cpp:118-119)
        const bool first = l0[e] <= l1[e];
        cb[e] = first ? b0[e] : b1[e];
        cl[e] = first ? l0[e] : l1[e];
        tried[e] = true;
        seen[e] = atomicCAS(loads + cb[e], cl[e], cl[e] + 1u);
        placed = seen[e] == cl[e];
      }
      if (placed) {
        store[static_cast<uint64_t>(cb[e]) * B + cl[e]] = pack_pair(k[e], v[e]);
        ++n_ins;
      } else {
        ++n_fail;
        record_failed(ctr, failed_keys, failed_cap, k[e]);
      }
    }
  }
  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

// ---- K13: iht --------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kClaimBlock)
claim_insert_iht_kernel(const __grid_constant__ TableView t, uint32_t* __restrict__ loads, const PairSource src, uint64_t n, bool aligned,
                        DevCounters* __restrict__ ctr, uint32_t* __restrict__ failed_keys, uint64_t failed_cap) {
  const uint32_t B = t.bucket_size;
  const int lane = threadIdx.x & 31;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kClaimBlock * 4;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * kClaimBlock + threadIdx.x) * 4; i < n; i += stride) {
    uint32_t k[4], v[4];
    if (src.values == nullptr) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint2 kv = i + e < n ? __ldcs(reinterpret_cast<const uint2*>(src.keys) + i + e) : make_uint2(0u, 0u);
        k[e] = kv.x, v[e] = kv.y;
      }
    } else {
      const uint4 k4 = load4(src.keys, i, n, aligned), v4 = load4(src.values, i, n, aligned);
      k[0] = k4.x, k[1] = k4.y, k[2] = k4.z, k[3] = k4.w;
      v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
    }
    // The four keys of a thread go through the steps together, so that their counter reads and atomics are in flight
    // at the same time: (1) read the primaries' counters, (2) one CAS attempt each where the load is below t, (3) the
    // rare retries, (4) the secondaries' counters of the keys that leave the primary, (5) their claims.
    uint32_t pb[4], pw[4], pl[4], seen[4];
    bool live[4], tried[4], done[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      live[e] = i + e < n;
      pb[e] = bucket_index(t.h[0], k[e]);
      pw[e] = live[e] ? __ldcg(loads + pb[e]) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pl[e] = min(pw[e], B);
      tried[e] = live[e] && pl[e] < t.threshold;  // stays while load < t (table.cpp:159)
      seen[e] = pw[e];
      if (tried[e]) seen[e] = atomicCAS(loads + pb[e], pw[e], pw[e] + 1u);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      done[e] = !live[e];
      if (!live[e]) continue;
      n_probe += 1;  // the primary (table.cpp:153-156)
      bool claimed = tried[e] && seen[e] == pw[e];
      if (tried[e] && !claimed) pl[e] = claim_slot_below(loads, pb[e], t.threshold, B, claimed);  // the word moved: retry
      if (claimed) {
        store[static_cast<uint64_t>(pb[e]) * B + pl[e]] = pack_pair(k[e], v[e]);
        ++n_ins;
        done[e] = true;
      }
    }
    uint32_t s0[4], s1[4], l0[4], l1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s0[e] = s1[e] = l0[e] = l1[e] = 0;
      if (!done[e]) {
        s0[e] = bucket_index(t.h[1], k[e]);
        s1[e] = bucket_index(t.h[2], k[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!done[e]) {
        l0[e] = read_load(loads, s0[e], B);
        l1[e] = read_load(loads, s1[e], B);
        n_probe += 2;  // both secondaries (table.cpp:160-163)
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (done[e]) continue;
      for (;;) {
        uint32_t cb = pb[e], cl = pl[e];
        int which = 0;
        if (t.prose || l0[e] != B || l1[e] != B) {  // unless both are full (and not prose), the less loaded secondary, tie s0
          if (l0[e] <= l1[e]) cb = s0[e], cl = l0[e], which = 1;
          else cb = s1[e], cl = l1[e], which = 2;
        }
        if (cl == B) {  // a full choice fails the insert (table.cpp:180)
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, k[e]);
          break;
        }
        const uint32_t slot = claim_slot(loads, cb, B);
        if (slot < B) {
          store[static_cast<uint64_t>(cb) * B + slot] = pack_pair(k[e], v[e]);
          ++n_ins;
          break;
        }
        if (which == 0) pl[e] = B;
        else if (which == 1) l0[e] = B;
        else l1[e] = B;
        if (s0[e] == s1[e] && which != 0) l0[e] = l1[e] = B;
      }
    }
  }
  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

}  // namespace

size_t claim_loads_bytes(uint64_t num_buckets) { return num_buckets * sizeof(uint32_t); }

cudaError_t launch_load_count(const TableView& t, uint32_t* loads, int sm_count, cudaStream_t stream) {
  const int grid = static_cast<int>(std::min<uint64_t>((t.num_buckets + kClaimBlock - 1) / kClaimBlock, static_cast<uint64_t>(sm_count) * 8));
  load_count_kernel<<<grid, kClaimBlock, 0, stream>>>(t.store, t.num_buckets, t.bucket_size, loads);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_claim_insert(const TableView& t, uint32_t* loads, const InsertLaunch& a, bool iht) {
  if (a.n == 0) return cudaSuccess;
  const bool aligned = a.src.values != nullptr &&
                       ((reinterpret_cast<uintptr_t>(a.src.keys) | reinterpret_cast<uintptr_t>(a.src.values)) & 15) == 0;
  uint64_t blocks = (a.n + kClaimBlock * 4 - 1) / (kClaimBlock * 4);
  // the same window as the bucket-reading kernels: at most one key in flight per four buckets (insert_p2.cu)
  const uint64_t window = std::max<uint64_t>(1, (t.num_buckets / 4 + kClaimBlock * 4 - 1) / (kClaimBlock * 4));
  blocks = std::min(blocks, std::min<uint64_t>(window, static_cast<uint64_t>(a.sm_count) * 8));
  if (iht)
    claim_insert_iht_kernel<<<static_cast<int>(blocks), kClaimBlock, 0, a.stream>>>(t, loads, a.src, a.n, aligned, a.ctr, a.failed_keys,
                                                                                  a.failed_cap);
  else
    claim_insert_p2_kernel<<<static_cast<int>(blocks), kClaimBlock, 0, a.stream>>>(t, loads, a.src, a.n, aligned, a.ctr, a.failed_keys,
                                                                                 a.failed_cap);
  note_launch();
  return cudaGetLastError();
}

}  // namespace bht_b200
