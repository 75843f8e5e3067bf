// probe_engine.cuh — the bucket probe engine.
//
// Replaces bucket_ref (reference: proj/include/bht/bucket.hpp:16-63): the snapshot read of a whole
// bucket (= one probe, bucket.hpp:18-21), compute_load (:26-31), full (:33) and find_key_value
// (:36-41).  cas_at_slot / exch_at_slot (:45-55) are single 64-bit atomics issued by the callers.
//
// Shape of one probe round of a warp (32 keys, one per lane):
//
//   fetch   A bucket of B 8-byte slots is B/2 16-byte chunks.  A tile of C = B/2 lanes copies one
//           bucket with ONE 16-byte cp.async (LDGSTS, L2-only) per lane straight into shared
//           memory, so a warp-wide copy instruction moves 32/C whole buckets, every 32-byte sector
//           it touches is fully used (128-byte aligned buckets at b = 16), and no register is tied
//           up while the line is in flight: a warp keeps 32 buckets outstanding for the cost of
//           C instructions, and the SM keeps (resident warps x 32) lines in flight.
//   scan    After cp.async.wait_group + __syncwarp every lane scans ITS OWN key's bucket from
//           shared memory with 16-byte LDS: 32 keys are matched in parallel by plain per-lane
//           compares — no ballots, no shuffles, no serialisation over the tile.
//
// Shared-memory layout: one row of 16*C bytes per lane; chunk c of row r is stored at position
// c ^ g(r), an XOR swizzle that makes both the tile-wise writes and the lane-wise reads
// bank-conflict free (see swizzle()).  Buckets of 1 or 2 slots are a single 8/16-byte load per
// lane and skip the staging.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "hash_stage.cuh"

namespace bht_b200 {

constexpr unsigned kFullMask = 0xFFFFFFFFu;
constexpr uint32_t kNoBucket = 0xFFFFFFFFu;  // "this lane has no probe this round" (bucket ids are < 2^32 - 1)

template <int B>
struct Geo {
  static_assert(B == 1 || B == 2 || B == 4 || B == 8 || B == 16 || B == 32 || B == 64, "bucket size");
  static constexpr bool STAGED = B >= 4;            // fetched through shared memory
  static constexpr int C = B >= 2 ? B / 2 : 1;      // 16-byte chunks per bucket = lanes per fetch tile
  static constexpr int T = 32 / C;                  // buckets fetched by one warp-wide copy instruction
  static constexpr int ROW_BYTES = B * 8;
  static constexpr int WARP_BYTES = STAGED ? 32 * ROW_BYTES : 0;  // staging bytes per warp per probed bucket
  // g(r): rows whose chunks share a bank group under a 16-byte access get different rotations
  __device__ static __forceinline__ uint32_t swizzle(uint32_t row) {
    if constexpr (C >= 8) return row & (C - 1);
    else if constexpr (C == 4) return (row >> 1) & 3;
    else return (row >> 2) & 1;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// 16-byte global -> shared copy that bypasses L1 (coherent at L2: sees other SMs' atomics).
// src_bytes = 16 copies, src_bytes = 0 zero-fills the destination without touching global memory, so
// lanes without a probe stay on the same branch-free instruction stream.
__device__ __forceinline__ void cp_async_16(uint32_t smem_dst, uint64_t gmem_src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gmem_src), "r"(src_bytes) : "memory");
}
// a * b + c with a 32-bit a, b and a 64-bit c: one IMAD.WIDE
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint4 ldg_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
// 16-byte load that ptxas may not narrow into the components actually consumed (two 4-byte loads would ask L2 for
// every sector of the bucket twice): volatile = relaxed, system scope, served by L2 like .cg.
__device__ __forceinline__ uint4 ldg_whole_v4(const void* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ uint2 ldg_cg_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}

// Result of scanning one bucket for one key.
struct Scan {
  uint32_t load;   // occupied slots (compute_load, bucket.hpp:26-31); with WANT_KEY only B (full) or 0 (not full)
  uint32_t value;  // value of the lowest slot holding the key (find_key_value, bucket.hpp:36-41)
  bool found;
};

// ---- fetch ------------------------------------------------------------------------------------
// Every lane names the bucket it wants (my_bid, or kNoBucket).  Staged sizes: the warp copies all
// named buckets into `stage` (shared address of this warp's 32 rows).  Call fetch_wait() before
// scanning, and __syncwarp() after scanning before the rows are fetched into again.
template <int B>
__device__ __forceinline__ void fetch_issue(uint32_t stage, const uint64_t* __restrict__ store, uint32_t my_bid, int lane) {
  using G = Geo<B>;
  if constexpr (G::STAGED) {
    const uint32_t sub = lane & (G::C - 1);
    const uint32_t t = lane / G::C;
    if (!__any_sync(kFullMask, my_bid != kNoBucket)) return;  // warp-uniform: nobody probes (iht second row)
    const uint64_t lane_src = reinterpret_cast<uint64_t>(store) + sub * 16;
#pragma unroll
    for (int u = 0; u < G::C; ++u) {
      const uint32_t row = u * G::T + t;
      const uint32_t bid = __shfl_sync(kFullMask, my_bid, row);
      const bool on = bid != kNoBucket;
      const uint32_t dst = stage + row * G::ROW_BYTES + ((sub ^ G::swizzle(row)) << 4);
      cp_async_16(dst, mad_wide(on ? bid : 0u, G::ROW_BYTES, lane_src), on ? 16u : 0u);
    }
  }
}

__device__ __forceinline__ void fetch_wait() {
  cp_async_wait_all();
  __syncwarp();
}

// ---- load of a staged bucket (insert side) ------------------------------------------------------
// Slots are only ever claimed at index = load (table.cpp:85) and full buckets never drain, so the
// occupied slots of a bucket are a prefix and compute_load's popcount (bucket.hpp:26-31) equals the
// index of the first empty slot.  That index is found with a 4-ary search: 4 independent 4-byte
// reads per level instead of B reads in total (b = 16: 4 + 3 reads, two dependent levels).
__device__ __forceinline__ uint32_t staged_key(uint32_t base, uint32_t slot) {
  return lds_u32((base ^ ((slot >> 1) << 4)) + ((slot & 1u) << 3));
}
// occupied slots among [lo, lo + L - 1), given that slot lo + L - 1 is empty
template <int L>
__device__ __forceinline__ uint32_t prefix_below(uint32_t base, uint32_t lo) {
  if constexpr (L == 1) {
    return 0;
  } else if constexpr (L == 2) {
    return staged_key(base, lo) != kEmptyKey;
  } else {
    constexpr int Q = L / 4;
    const uint32_t a = staged_key(base, lo + Q - 1), b = staged_key(base, lo + 2 * Q - 1), c = staged_key(base, lo + 3 * Q - 1);
    const uint32_t q = (a != kEmptyKey) + (b != kEmptyKey) + (c != kEmptyKey);
    return q * Q + prefix_below<Q>(base, lo + q * Q);
  }
}
template <int B>
__device__ __forceinline__ uint32_t staged_prefix_load(uint32_t base) {
  constexpr int S = B / 4;
  const uint32_t a = staged_key(base, S - 1), b = staged_key(base, 2 * S - 1), c = staged_key(base, 3 * S - 1),
                 d = staged_key(base, 4 * S - 1);
  const uint32_t q = (a != kEmptyKey) + (b != kEmptyKey) + (c != kEmptyKey) + (d != kEmptyKey);
  if (q == 4) return B;
  return q * S + prefix_below<S>(base, q * S);
}

// ---- direct load (insert side, register-resident) ------------------------------------------------
// The bucket never touches shared memory: the C = B/2 lanes of a tile read one bucket with one 16-byte
// LDG each (iteration u of a tile serves the key of the tile's u-th lane), count their occupied slots and
// add the counts up inside the tile (packed bytes + shuffle butterfly).  load = occupied slots (they form a
// prefix, see staged_prefix_load).  No LDGSTS shared-memory write, no LDS: less work for the SM's load/store
// pipe than the staged engine, at the price of B/2 x 4 registers held while the lines are in flight —
// the trade that pays when the probes are L2-resident and few keys in flight suffice (routed builds).
template <int B>
__device__ __forceinline__ uint32_t direct_load(const uint64_t* __restrict__ store, uint32_t my_bid, int lane) {
  static_assert(B >= 4 && B <= 16, "direct engine: 4 <= b <= 16");
  constexpr int C = B / 2;
  const int sub = lane & (C - 1);
  const int tile_base = lane & ~(C - 1);
  uint4 v[C];
#pragma unroll
  for (int u = 0; u < C; ++u) {
    const uint32_t bid = __shfl_sync(kFullMask, my_bid, tile_base + u);
    v[u] = make_uint4(0u, 0u, 0u, 0u);
    if (bid != kNoBucket) v[u] = ldg_whole_v4(store + static_cast<uint64_t>(bid) * B + sub * 2);
  }
  // Occupied slots seen by this lane in iteration u go to byte u % 4 of acc[u / 4]; a butterfly over the C lanes of
  // the tile then adds the bytes up for all C keys at once (a byte never exceeds B <= 16, so nothing carries):
  // log2(C) shuffles per accumulator instead of two ballots + two popcounts per key.
  uint32_t acc[(C + 3) / 4] = {};
#pragma unroll
  for (int u = 0; u < C; ++u) {
    const uint32_t occ = (v[u].x != kEmptyKey) + (v[u].z != kEmptyKey);
    acc[u / 4] += occ << (8 * (u % 4));
  }
#pragma unroll
  for (int a = 0; a < (C + 3) / 4; ++a) {
#pragma unroll
    for (int o = 1; o < C; o <<= 1) acc[a] += __shfl_xor_sync(kFullMask, acc[a], o);
  }
  uint32_t mine = acc[0];
  if constexpr (C > 4) mine = sub < 4 ? acc[0] : acc[1];
  return (mine >> (8 * (sub & 3))) & 0xFFu;
}

// ---- scan -------------------------------------------------------------------------------------
// The lane's own bucket: staged sizes read row `lane` of `stage`; b <= 2 loads straight from
// global memory through L2.  WANT_KEY = false skips the key match (insert needs the load only).
template <int B, bool WANT_KEY>
__device__ __forceinline__ Scan scan_bucket(uint32_t stage, const uint64_t* __restrict__ store, uint32_t bid, uint32_t key,
                                            int lane) {
  using G = Geo<B>;
  Scan r;
  r.load = 0;
  r.value = kEmptyKey;
  r.found = false;
  if constexpr (!G::STAGED) {
    if constexpr (B == 1) {
      const uint2 s = ldg_cg_v2(store + bid);
      r.load = s.x != kEmptyKey;
      if (WANT_KEY && s.x == key) {
        r.found = true;
        r.value = s.y;
      }
    } else {
      const uint4 s = ldg_cg_v4(store + static_cast<uint64_t>(bid) * 2);
      r.load = (s.x != kEmptyKey) + (s.z != kEmptyKey);
      if (WANT_KEY) {
        if (s.z == key) { r.found = true; r.value = s.w; }
        if (s.x == key) { r.found = true; r.value = s.y; }  // lowest slot wins
      }
    }
  } else {
    const uint32_t row = stage + lane * G::ROW_BYTES;
    const uint32_t base = row + (G::swizzle(lane) << 4);  // row is ROW_BYTES-aligned: XOR below stays inside it
    if constexpr (WANT_KEY) {
      // find: value of the lowest matching slot + "has an empty slot" (0xFFFFFFFF is the largest key)
      uint32_t top = 0, value = kEmptyKey;
#pragma unroll
      for (int c = G::C - 1; c >= 0; --c) {  // descending, so the lowest matching slot is the one kept
        const uint4 s = lds_v4(base ^ (c << 4));
        top = max(top, max(s.x, s.z));
        value = s.z == key ? s.w : value;
        value = s.x == key ? s.y : value;
      }
      // stored values never equal the sentinel (core.hpp:20-24), so it doubles as "no match"
      r.value = value;
      r.found = value != kEmptyKey;
      r.load = top == kEmptyKey ? 0u : static_cast<uint32_t>(B);  // only full / not full is reported
    } else {
      r.load = staged_prefix_load<B>(base);
    }
  }
  return r;
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
  uint32_t chunk_log2;  // log2 of the work-stream chunk (see Stream)
  uint32_t sweep_ahead_bytes;  // routed builds: how far ahead of the insert window the store is prefetched into L2
};

// h_i(key) with a per-lane i: the constants are picked with selects (a divergent constant-bank
// index would serialise).
template <int H>
__device__ __forceinline__ uint32_t bucket_index_sel(const TableView& t, uint32_t i, uint32_t key) {
  HashFn h = t.h[0];
#pragma unroll
  for (int j = 1; j < H; ++j) {
    if (i == static_cast<uint32_t>(j)) h = t.h[j];
  }
  return bucket_index(h, key);
}

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

// ---- work distribution ------------------------------------------------------------------------
// The input is cut into chunks of 2^chunk_log2 elements.  Chunk w goes to warp w of the grid; every further
// chunk is claimed from a global cursor (one atomicAdd per chunk, issued one chunk ahead so its latency is
// never waited for) by whichever warp runs dry first.  So the keys in flight always form one narrow window
// that slides over the input in order — input that is grouped by table region therefore probes one L2-sized
// region at a time — and no warp is left with a tail of work when the others are done.
// Every warp streams through its chunks as a lane-level state machine: a lane that has finished its key
// takes the next unread key of the warp's stream, so every probe round is dense (32 probes per warp) no
// matter how many rounds individual keys need.  The next 32 keys of the stream are prefetched one round
// ahead and handed out with a shuffle.
constexpr uint32_t kDefaultChunkLog2 = 8;

struct Stream {
  uint32_t n_chunks, last_len;  // the last chunk may be partial
  uint32_t cur, nxt;            // chunk held / chunk claimed ahead (warp-uniform); >= n_chunks = none
  uint32_t cur_len;             // elements of `cur` (0 when none)
  uint32_t pos;                 // next unread element of `cur`

  __device__ __forceinline__ static uint32_t grid_warps() {
    return static_cast<uint32_t>((static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5);
  }
  __device__ __forceinline__ uint32_t len_of(uint32_t chunk, uint32_t shift) const {
    return chunk + 1 < n_chunks ? (1u << shift) : (chunk + 1 == n_chunks ? last_len : 0u);
  }
  // `cursor`: one global word per launch, zero at launch.  Nothing is claimed when the grid covers the input.
  __device__ __forceinline__ uint32_t claim(uint32_t* cursor, int lane) const {
    const uint32_t n_warps = grid_warps();
    if (n_chunks <= n_warps) return n_chunks;
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(cursor, 1u);
    return n_warps + __shfl_sync(kFullMask, c, 0);
  }
  __device__ __forceinline__ void init(uint64_t n, uint32_t shift, uint32_t* cursor, int lane) {
    n_chunks = static_cast<uint32_t>((n + (1ull << shift) - 1) >> shift);
    last_len = static_cast<uint32_t>(n - (static_cast<uint64_t>(n_chunks - (n != 0)) << shift));
    cur = static_cast<uint32_t>((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    cur_len = len_of(cur, shift);
    pos = 0;
    nxt = claim(cursor, lane);
  }
  // Global index of stream element pos + off (off < 32); false when the stream ends before it.
  __device__ __forceinline__ bool index(uint32_t off, uint32_t shift, uint64_t& idx) const {
    const uint32_t p = pos + off;
    idx = (static_cast<uint64_t>(cur) << shift) + p;
    if (pos + 32 <= cur_len) return true;  // warp-uniform: `nxt` (maybe still in flight) is not touched
    if (p < cur_len) return true;
    const uint32_t q = p - cur_len;  // spills into the chunk claimed ahead (chunks hold >= 32 elements)
    idx = (static_cast<uint64_t>(nxt) << shift) + q;
    return cur_len != 0 && q < len_of(nxt, shift);
  }
  // k (<= 32) elements were handed out.
  __device__ __forceinline__ void advance(uint32_t k, uint32_t shift, uint32_t* cursor, int lane) {
    pos += k;
    if (pos >= cur_len && cur_len != 0) {
      pos -= cur_len;
      cur = nxt;
      cur_len = len_of(cur, shift);
      if (cur_len != 0) nxt = claim(cursor, lane);
    }
  }
};

// Threads per block for a kernel that stages `rows_per_lane` buckets of B slots per lane: keeps the
// staging area of a block at or below 32 KiB so that several blocks share an SM.
template <int B>
constexpr int block_threads(int rows_per_lane) {
  int t = 256;
  while (t > 32 && (t / 32) * Geo<B>::WARP_BYTES * rows_per_lane > 32 * 1024) t /= 2;
  return t;
}

}  // namespace bht_b200
