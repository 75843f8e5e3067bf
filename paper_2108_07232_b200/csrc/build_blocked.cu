// build_blocked.cu — K8g / K10 / K11: the shared-memory-blocked bulk build of the cuckoo tables (bcht, 1cht).
//
// Same algorithm as bcht_insert (reference: proj/src/table.cpp:53-92) — a pair goes to slot index = load of its
// H0 bucket (table.cpp:85); when that bucket is full the insertion goes on as an eviction chain (table.cpp:63-81)
// — but the first attempt of every pair, which is ~90 % of all the probes of a build at load factor 0.9, never
// touches HBM at random and never issues a global compare-and-swap:
//
//   K8g group_scatter   first partition level, one streaming pass: the pairs are grouped by GROUP = `per` consecutive
//                       fine regions; a fine region is 64 KiB of consecutive buckets (512 buckets at b = 16), a
//                       444 MB table has 6782 of them in 83 groups of 82.  Fixed-capacity group segments (the hash is
//                       uniform): no histogram pre-pass.
//   K10 bin_split       second partition level: tiles of 2048 pairs of one group are ranked by fine region in shared
//                       memory (<= per <= 256 destinations), one global
//                       atomicAdd per (tile, region) reserves a run in the region's bin, and the tile is written out
//                       run by run (~25 pairs = 200 contiguous bytes per run: whole 32-byte sectors, which is what
//                       the L2 wants — see the measurements below).  Bins have a fixed capacity (mean + 6 sigma of a
//                       uniform hash + 32); what does not fit goes to the spill list.
//   K11 region_build    one CTA per fine region: the region's buckets live in shared memory (filled with the empty
//                       pattern when the table is known to be empty, else loaded from the store), every pair of the
//                       bin claims slot = atomicAdd(load counter of its bucket) — a shared-memory atomic, no CAS, no
//                       lost races, no re-probes — and the region is written back by the bulk-copy engine
//                       (cp.async.bulk shared -> global, SASS UBLKCP, 4 KiB pieces: 0.771 -> 0.746 ms for the three
//                       passes against coalesced 16-byte stores from registers).
//                       A pair whose bucket is full goes to a per-CTA stash in shared memory; once every claim is
//                       written the stashed pairs do their first eviction in shared memory (atomicExch into a random
//                       slot of the full bucket, table.cpp:67-81) and the VICTIMS go to the global spill list, each
//                       with the bucket its walk goes on in and a chain length of 1 (one list reservation per CTA).
//   K4  (existing)      the general cuckoo kernel (insert_cuckoo.cu) finishes the walks of the spill list exactly as
//                       the reference would: probe the next bucket, claim or evict again, up to max_chain.
//
// What the earlier versions of this file measured on B200 (bcht b = 16, 50 M pairs, LF 0.9; profiles/r01e_*):
//   * one-level binning with one L2 atomicAdd + one scattered 8-byte store per pair: 1.12 ms — the L2 serves
//     sub-sector read-modify-writes (atomics and stores narrower than a 32-byte sector alike) at only ~75-105 G/s,
//     whatever line they hit (atomics alone 0.47 ms; padding the cursors to one per line changed nothing);
//   * tile ranking with runs of ~5 pairs (38 bytes, mostly partial sectors): 0.85 ms for the same reason;
//   * shared-memory atomics are NOT the problem: 3.6 SM-cycles per warp-instruction with a returned rank
//     (tools/microbench/warp_rank.cu), against 20-34 for ballot ranking and 42-64 for match.any.
//
// Probe accounting (probe_stats.hpp:12-31: one probe per bucket inspection): a pair placed by K11 costs one probe;
// a pair that evicts in K11 costs one probe there (the inspection that found its bucket full); K4 counts the rest
// of the walk.  A pair that overflows a bin or the stash reaches K4 untouched and is counted there from H0 on.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "insert_common.cuh"

#ifndef BHT_BUILD_BLOCK  // measured (insert, 50 M pairs): 192 x 20: 1.087 ms, 256 x 16: 1.062, 320 x 12: 1.034, 384 x 10: 1.034 (spills)
#define BHT_BUILD_BLOCK 320
#define BHT_BUILD_U 12
#endif

#ifndef BHT_BUILD_TMA_STORE
#define BHT_BUILD_TMA_STORE 1
#endif

#ifndef BHT_BUILD_PREFETCH  // 1: a CTA of K11 prefetches the bin of the CTA that will take its place into the L2 (measured: +200 MB of DRAM reads, the prefetched lines are fetched twice, and no gain: 263.1 against 263.8 us)
#define BHT_BUILD_PREFETCH 0
#endif

#ifndef BHT_SPLIT_TMA  // 1: the next tile's input arrives by a bulk asynchronous copy (TMA) while this one is processed
#define BHT_SPLIT_TMA 1
#endif
#ifndef BHT_SPLIT_CTAS  // resident CTAs per SM the partition kernels are compiled for (register budget)
#define BHT_SPLIT_CTAS (BHT_SPLIT_TMA ? 4 : 5)
#endif
#ifndef BHT_SPLIT_BLOCK
#define BHT_SPLIT_BLOCK 256
#endif

namespace bht_b200 {

namespace {

constexpr int kSplitBlock = BHT_SPLIT_BLOCK;  // >= 256: the first 256 threads scan the tile's histogram
constexpr int kSplitPerThread = 8;
constexpr int kSplitTile = kSplitBlock * kSplitPerThread;  // 2048 pairs
constexpr int kBuildBlock = BHT_BUILD_BLOCK;   // few threads with many loads in flight each: 3 CTAs/SM by shared memory
constexpr uint32_t kStashPairs = 1024;  // per-CTA stash of the pairs whose bucket was full (K11): 8 KiB beside the region's 64
constexpr uint32_t kRegionBytesLog2 = 16;

// The spill list: packed pairs + where their walk starts (kStartAtH0 for a pair that has not probed anything yet).
struct Spill {
  uint2* pairs;
  uint32_t* start;
  unsigned long long* cursor;
  unsigned long long cap;  // entries of the list (= the most pairs the build was announced to take)
  DevCounters* ctr;        // a pair that does not even fit the list is dropped and reported as a failed insertion:
  uint32_t* failed_keys;   // only a chunked build fed more pairs than it announced (device-counted chunks) gets there
  uint64_t failed_cap;
};

__device__ __forceinline__ void spill_dropped(uint32_t key, const Spill& sp) {
  atomicAdd(&sp.ctr->failed, 1ull);
  record_failed(sp.ctr, sp.failed_keys, sp.failed_cap, key);
}

// A pair that found no room in a fixed-capacity segment / bin / stash goes to the spill list untouched (rare: the
// capacities are mean + 6 sigma of a uniform hash; one global atomic per pair).
__device__ __forceinline__ void spill_fresh(uint2 kv, const Spill& sp) {
  const unsigned long long pos = atomicAdd(sp.cursor, 1ull);
  if (pos >= sp.cap) return spill_dropped(kv.x, sp);
  sp.pairs[pos] = kv;
  sp.start[pos] = kStartAtH0;
}

// ---- the partition passes (K8g, K10) ------------------------------------------------------------------------
// One tile = 2048 pairs, 8 per thread.  (1) every pair takes a rank among the tile's pairs of its destination with one
// shared-memory atomicAdd; (2) the 256 counts are scanned, and one global atomicAdd per (tile, destination) reserves the
// run in the destination's fixed-capacity segment; (3) the pairs are staged in shared memory run by run; (4) the tile
// is written out in staging order, so that consecutive threads write consecutive pairs of a run (whole 32-byte
// sectors except at the ends of a run).  Three block barriers per tile; the histogram is zeroed by the thread that
// scans it.
//
// What bounds these passes is the shared-memory pipe (ncu, profiles/r02d_*: l1tex 65-78 % busy, short-scoreboard and
// MIO-throttle stalls, the integer pipe half idle), not DRAM and not the instruction count: with the stores removed
// the pass still took 200 of its 230 us, halving its instructions changed nothing, fetching the next tile's input
// with the TMA unit while this one is processed changed nothing.  So the staging keeps nothing per pair but the pair:
// the write-out recomputes a staged pair's destination from its key (a second hash: 14 integer instructions) instead
// of a staged position / destination byte (one more scattered shared-memory store and one more load per pair).
struct SplitShared {
  uint2 pair[kSplitTile];
  uint2 out_of[256];   // per destination of the tile: {output index of its run - first staging slot, first staging slot past what fits}
  uint32_t toff[256];  // per destination: first staging slot of its run
  uint32_t hist[256];
  uint32_t warp_tot[8];
  unsigned long long mbar;   // completion of the bulk copy into `in`
  unsigned long long pad;
#if BHT_SPLIT_TMA
  uint32_t in[2 * kSplitTile];  // the next full tile: K8g keys | values, K10 packed pairs
#endif
};

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Where a partition pass puts a staged pair: packed into one array with the spill list behind it (K8g, K10) ...
struct PackedSink {
  uint2* out;
  Spill sp;
  __device__ __forceinline__ void write(uint64_t pos, uint2 p) const { __stcs(out + pos, p); }
  __device__ __forceinline__ void overflow(uint2 p) const { spill_fresh(p, sp); }  // the destination's segment is full (rare: sized mean + 6 sigma)
};
// ... or into two arrays, the surplus of a full segment dropped and flagged (K8s: the caller re-routes with exact counts)
struct SplitArraysSink {
  uint32_t* out_first;
  uint32_t* out_second;  // may be null
  uint32_t* overflow_flag;
  __device__ __forceinline__ void write(uint64_t pos, uint2 p) const {
    out_first[pos] = p.x;
    if (out_second != nullptr) out_second[pos] = p.y;
  }
  __device__ __forceinline__ void overflow(uint2) const { atomicOr(overflow_flag, 1u); }
};

// Phases 2-4 for the tile whose pairs (kv), destinations and ranks (dr = destination | rank << 8) are in registers and
// whose ranks are all taken (the caller's barrier); `valid` has bit j set when pair j of this thread exists, `len` =
// pairs in the tile; dest_of(key) = the destination (< 256) of a pair of this tile.
template <bool FULL, typename DestOf, typename Sink>
__device__ __forceinline__ void split_tile_finish(SplitShared& s, const uint2 (&kv)[kSplitPerThread],
                                                  const uint32_t (&dr)[kSplitPerThread], uint32_t valid, uint32_t len,
                                                  uint32_t n_dest, uint32_t dest_base, uint32_t cap,
                                                  uint32_t* __restrict__ cursor, const Sink& sink,
                                                  uint64_t tile_id, DestOf dest_of) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t h = 0, x = 0, gbase = 0;
  if (kSplitBlock == 256 || threadIdx.x < 256) {
    h = s.hist[threadIdx.x];
    s.hist[threadIdx.x] = 0;  // for the next tile: nobody touches it again before the next barrier
    x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFullMask, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s.warp_tot[warp] = x;
    // the reservation travels while the block meets at the barrier
#if defined(BHT_EXP_NOGATOM)  // experiment (wrong results): the pass without its global reservations
    if (h != 0 && threadIdx.x < n_dest) gbase = static_cast<uint32_t>(tile_id % 200u) * 24u;
#else
    if (h != 0 && threadIdx.x < n_dest) gbase = atomicAdd(&cursor[dest_base + threadIdx.x], h);
#endif
  }
  __syncthreads();
  if (kSplitBlock == 256 || threadIdx.x < 256) {
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) before += w < warp ? s.warp_tot[w] : 0u;
    const uint32_t first = before + x - h;
    const uint32_t room = gbase < cap ? cap - gbase : 0u;
    s.toff[threadIdx.x] = first;
    s.out_of[threadIdx.x] = make_uint2((dest_base + threadIdx.x) * cap + gbase - first, first + min(h, room));
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSplitPerThread; ++j)
    if (FULL || ((valid >> j) & 1u)) s.pair[s.toff[dr[j] & 255u] + (dr[j] >> 8)] = kv[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSplitPerThread; ++j) {
    const uint32_t slot = j * kSplitBlock + threadIdx.x;
    if (FULL || slot < len) {
      const uint2 p = s.pair[slot];
      const uint2 o = s.out_of[dest_of(p.x)];  // consecutive slots share a destination: mostly a broadcast
#if defined(BHT_EXP_NOSTORE)   // experiments only (results are wrong): what the pass costs without its stores ...
      if (slot == 0xFFFFFFF0u) sink.write(o.x, p);
#elif defined(BHT_EXP_LINEAR)  // ... and with perfectly sequential ones
      sink.write(tile_id * kSplitTile + slot, p);
#else
      if (slot < o.y) sink.write(o.x + slot, p);
      else sink.overflow(p);
#endif
    }
  }
  // no barrier here: the next tile's first writes to `pair` / `toff` / `out_of` come after its own barriers
}

// ---- K8g ------------------------------------------------------------------------------------------------------
// First partition level, one streaming pass over (a chunk of) the caller's arrays: every pair goes to the segment of
// its GROUP (= `per` consecutive fine regions).  No histogram pre-pass and no destination bytes: the hash is uniform,
// so the segments are sized mean + 6 sigma and the few pairs that do not fit go to the spill list.  The cursors live
// across launches, so a batch may arrive in several chunks (host-buffer builds, sharded builds).
struct GroupArgs {
  HashFn h0;
  uint32_t region_log2, inv_per, n_groups, group_cap;
  const uint32_t* keys;
  const uint32_t* values;  // null: keys-only build, value = value_for_key(key) (table.cpp:234)
  uint64_t n;
  const unsigned long long* n_dev;  // when set: the chunk holds min(n, *n_dev) pairs
  uint32_t* group_cursor;
  uint2* grouped;
  Spill sp;
  int aligned;
};

__global__ void __launch_bounds__(kSplitBlock, BHT_SPLIT_CTAS)
group_scatter_kernel(const __grid_constant__ GroupArgs args) {
  GroupArgs a = args;
  if (a.n_dev != nullptr) a.n = min(a.n, static_cast<uint64_t>(*a.n_dev));
  extern __shared__ __align__(16) unsigned char split_bytes[];
  SplitShared& s = *reinterpret_cast<SplitShared*>(split_bytes);
  if (threadIdx.x < 256) s.hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) mbar_init(&s.mbar);
  __syncthreads();
  const uint64_t n_tiles = (a.n + kSplitTile - 1) / kSplitTile;
  // a full tile of 16-byte aligned arrays arrives through the bulk copy / 16-byte loads; the last, partial one (and
  // everything of an unaligned call) is read element by element
  auto is_full = [&](uint64_t tile) { return a.aligned && (tile + 1) * kSplitTile <= a.n; };
  auto fetch = [&](uint64_t tile) {
#if BHT_SPLIT_TMA
    constexpr uint32_t in_bytes = kSplitTile * 4u;
    if (threadIdx.x == 0 && tile < n_tiles && is_full(tile)) {
      mbar_expect(&s.mbar, a.values != nullptr ? 2 * in_bytes : in_bytes);
      bulk_load(s.in, a.keys + tile * kSplitTile, in_bytes, &s.mbar);
      if (a.values != nullptr) bulk_load(s.in + kSplitTile, a.values + tile * kSplitTile, in_bytes, &s.mbar);
    }
#endif
  };
  auto group_of = [&](uint32_t key) {
    return static_cast<uint32_t>((static_cast<uint64_t>(bucket_index(a.h0, key) >> a.region_log2) * a.inv_per) >> 32);
  };
  uint32_t parity = 0;
  fetch(blockIdx.x);
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i0 = tile * kSplitTile;
    const bool full = is_full(tile);  // block-uniform
    const uint32_t len = static_cast<uint32_t>(min(static_cast<uint64_t>(kSplitTile), a.n - i0));
    uint2 kv[kSplitPerThread];
    uint32_t dr[kSplitPerThread];
    uint32_t valid = 0;
#if BHT_SPLIT_TMA
    if (full) {
      mbar_wait(&s.mbar, parity);
      parity ^= 1u;
    }
#endif
#pragma unroll
    for (int j = 0; j < kSplitPerThread / 4; ++j) {
      const uint32_t at = (j * kSplitBlock + threadIdx.x) * 4;  // this thread's four consecutive pairs
      uint32_t k[4], v[4] = {0u, 0u, 0u, 0u};
      if (full) {
#if BHT_SPLIT_TMA
        const uint4 k4 = *reinterpret_cast<const uint4*>(s.in + at);
#else
        const uint4 k4 = __ldcs(reinterpret_cast<const uint4*>(a.keys + i0 + at));
#endif
        k[0] = k4.x, k[1] = k4.y, k[2] = k4.z, k[3] = k4.w;
        if (a.values != nullptr) {
#if BHT_SPLIT_TMA
          const uint4 v4 = *reinterpret_cast<const uint4*>(s.in + kSplitTile + at);
#else
          const uint4 v4 = __ldcs(reinterpret_cast<const uint4*>(a.values + i0 + at));
#endif
          v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = at + e < len;
          k[e] = in ? __ldcs(a.keys + i0 + at + e) : 0u;
          v[e] = (in && a.values != nullptr) ? __ldcs(a.values + i0 + at + e) : 0u;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (a.values == nullptr) v[e] = value_for_key(k[e]);  // kernel-uniform
        kv[4 * j + e] = make_uint2(k[e], v[e]);
        valid |= (at + e < len) ? 1u << (4 * j + e) : 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t d = group_of(kv[j].x);
      uint32_t rank = 0;
      if ((valid >> j) & 1u) rank = atomicAdd(&s.hist[d], 1u);
      dr[j] = d | (rank << 8);
    }
    __syncthreads();  // every rank of the tile is taken, and `in` has been read by everyone
    fetch(tile + gridDim.x);
    const PackedSink sink{a.grouped, a.sp};
    if (full) split_tile_finish<true>(s, kv, dr, valid, len, a.n_groups, 0u, a.group_cap, a.group_cursor, sink, tile, group_of);
    else split_tile_finish<false>(s, kv, dr, valid, len, a.n_groups, 0u, a.group_cap, a.group_cursor, sink, tile, group_of);
  }
}

// ---- K8s ------------------------------------------------------------------------------------------------------
// The sharded table's router in ONE pass, the same tile machinery: every element goes to the fixed segment of its OWNER
// shard (owner(k) = (g(k) * G) >> 32, hash_stage.cuh), destination d owning slots [d * cap, (d + 1) * cap) of the output
// arrays.  The second word of an element is its value (inserts), its position in the input (finds: the way back for
// K9) or nothing.  The per-destination counts stay on the device (`cursor`, finalised by shard_counts_kernel); what does
// not fit a segment is dropped and flagged.  Replaces classify + cursors + scatter (two passes over the keys and a
// destination byte per key) for the sync-free exchange: 16.7 M keys in ~75 us instead of 143.
struct ShardSplitArgs {
  uint32_t alpha, beta, n_shards, cap;
  const uint32_t* keys;
  const uint32_t* values;  // null: the second word is the element's index (index_mode) or absent
  uint64_t n;
  uint32_t* cursor;        // n_shards zeroed words
  SplitArraysSink sink;
  int index_mode, aligned;
};

__global__ void __launch_bounds__(kSplitBlock, BHT_SPLIT_CTAS)
shard_split_kernel(const __grid_constant__ ShardSplitArgs a) {
  extern __shared__ __align__(16) unsigned char split_bytes[];
  SplitShared& s = *reinterpret_cast<SplitShared*>(split_bytes);
  if (threadIdx.x < 256) s.hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) mbar_init(&s.mbar);
  __syncthreads();
  const uint64_t n_tiles = (a.n + kSplitTile - 1) / kSplitTile;
  auto is_full = [&](uint64_t tile) { return a.aligned && (tile + 1) * kSplitTile <= a.n; };
  auto fetch = [&](uint64_t tile) {
#if BHT_SPLIT_TMA
    constexpr uint32_t in_bytes = kSplitTile * 4u;
    if (threadIdx.x == 0 && tile < n_tiles && is_full(tile)) {
      mbar_expect(&s.mbar, a.values != nullptr ? 2 * in_bytes : in_bytes);
      bulk_load(s.in, a.keys + tile * kSplitTile, in_bytes, &s.mbar);
      if (a.values != nullptr) bulk_load(s.in + kSplitTile, a.values + tile * kSplitTile, in_bytes, &s.mbar);
    }
#endif
  };
  auto owner_of = [&](uint32_t key) { return shard_of(a.alpha, a.beta, a.n_shards, key); };
  uint32_t parity = 0;
  fetch(blockIdx.x);
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i0 = tile * kSplitTile;
    const bool full = is_full(tile);  // block-uniform
    const uint32_t len = static_cast<uint32_t>(min(static_cast<uint64_t>(kSplitTile), a.n - i0));
    uint2 kv[kSplitPerThread];
    uint32_t dr[kSplitPerThread];
    uint32_t valid = 0;
#if BHT_SPLIT_TMA
    if (full) {
      mbar_wait(&s.mbar, parity);
      parity ^= 1u;
    }
#endif
#pragma unroll
    for (int j = 0; j < kSplitPerThread / 4; ++j) {
      const uint32_t at = (j * kSplitBlock + threadIdx.x) * 4;  // this thread's four consecutive elements
      uint32_t k[4], v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = static_cast<uint32_t>(i0 + at + e);  // index mode (a call routes < 2^32 elements)
      if (full) {
#if BHT_SPLIT_TMA
        const uint4 k4 = *reinterpret_cast<const uint4*>(s.in + at);
#else
        const uint4 k4 = __ldcs(reinterpret_cast<const uint4*>(a.keys + i0 + at));
#endif
        k[0] = k4.x, k[1] = k4.y, k[2] = k4.z, k[3] = k4.w;
        if (a.values != nullptr) {
#if BHT_SPLIT_TMA
          const uint4 v4 = *reinterpret_cast<const uint4*>(s.in + kSplitTile + at);
#else
          const uint4 v4 = __ldcs(reinterpret_cast<const uint4*>(a.values + i0 + at));
#endif
          v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = at + e < len;
          k[e] = in ? __ldcs(a.keys + i0 + at + e) : 0u;
          if (a.values != nullptr) v[e] = in ? __ldcs(a.values + i0 + at + e) : 0u;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        kv[4 * j + e] = make_uint2(k[e], v[e]);
        valid |= (at + e < len) ? 1u << (4 * j + e) : 0u;
      }
    }
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t d = owner_of(kv[j].x);
      uint32_t rank = 0;
      if ((valid >> j) & 1u) rank = atomicAdd(&s.hist[d], 1u);
      dr[j] = d | (rank << 8);
    }
    __syncthreads();  // every rank of the tile is taken, and `in` has been read by everyone
    fetch(tile + gridDim.x);
    if (full) split_tile_finish<true>(s, kv, dr, valid, len, a.n_shards, 0u, a.cap, a.cursor, a.sink, tile, owner_of);
    else split_tile_finish<false>(s, kv, dr, valid, len, a.n_shards, 0u, a.cap, a.cursor, a.sink, tile, owner_of);
  }
}

// counts[d] = elements written for destination d; *overflow raised when a destination had more than cap.
__global__ void shard_counts_kernel(uint32_t n_shards, uint32_t cap, const uint32_t* __restrict__ cursor,
                                    unsigned long long* __restrict__ counts, uint32_t* __restrict__ overflow) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_shards) return;
  const uint32_t c = cursor[d];
  counts[d] = c < cap ? c : cap;
  if (c > cap) atomicOr(overflow, 1u);
}

// ---- K10 ------------------------------------------------------------------------------------------------------
// Second partition level.  grouped: segment g = pairs of group g (fine regions [g * per, (g + 1) * per)),
// group_cursor[g] of them (clamped to group_cap).  bins[f * cap ..] / bin_cursor[f]: the bin of fine region f.  A tile
// never leaves its group, so it has at most `per` <= 256 destinations and its runs are ~25 pairs = 200 contiguous bytes.
struct BinArgs {
  HashFn h0;
  uint32_t region_log2, per, n_groups, n_regions, cap, group_cap;
  const uint2* grouped;
  const uint32_t* group_cursor;
  uint32_t* bin_cursor;
  uint2* bins;
  Spill sp;
};

__global__ void __launch_bounds__(kSplitBlock, BHT_SPLIT_CTAS)
bin_split_kernel(const __grid_constant__ BinArgs a) {
  extern __shared__ __align__(16) unsigned char split_bytes[];
  SplitShared& s = *reinterpret_cast<SplitShared*>(split_bytes);
  if (threadIdx.x < 256) s.hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) mbar_init(&s.mbar);
  __syncthreads();
  const uint32_t tiles_per_group = (a.group_cap + kSplitTile - 1) / kSplitTile;
  const uint64_t n_tiles = static_cast<uint64_t>(a.n_groups) * tiles_per_group;
  // the tiles of this CTA: every gridDim.x-th one that holds pairs (the segments are sized for mean + 6 sigma)
  struct Tile {
    uint64_t id;
    uint32_t g, t0, len;
  };
  auto next_tile = [&](uint64_t from) {
    Tile t{from, 0u, 0u, 0u};
    for (; t.id < n_tiles; t.id += gridDim.x) {
      t.g = static_cast<uint32_t>(t.id / tiles_per_group);
      t.t0 = static_cast<uint32_t>(t.id % tiles_per_group) * kSplitTile;
      const uint32_t in_group = min(a.group_cursor[t.g], a.group_cap);
      if (t.t0 < in_group) {
        t.len = min(static_cast<uint32_t>(kSplitTile), in_group - t.t0);
        break;
      }
    }
    return t;
  };
  auto fetch = [&](const Tile& t) {
#if BHT_SPLIT_TMA
    if (threadIdx.x == 0 && t.id < n_tiles && t.len == kSplitTile) {
      mbar_expect(&s.mbar, kSplitTile * 8u);
      bulk_load(s.in, a.grouped + static_cast<uint64_t>(t.g) * a.group_cap + t.t0, kSplitTile * 8u, &s.mbar);  // 16-byte aligned: group_cap is even
    }
#endif
  };
  uint32_t parity = 0;
  Tile cur = next_tile(blockIdx.x);
  fetch(cur);
  while (cur.id < n_tiles) {
    const Tile nxt = next_tile(cur.id + gridDim.x);
    const bool full = cur.len == kSplitTile;
    const uint2* src = a.grouped + static_cast<uint64_t>(cur.g) * a.group_cap + cur.t0;  // 16-byte aligned: group_cap is even
    const uint32_t f_base = cur.g * a.per;
    const uint32_t n_dest = min(a.per, a.n_regions - f_base);
    auto region_of = [&](uint32_t key) { return ((bucket_index(a.h0, key) >> a.region_log2) - f_base) & 255u; };  // < per <= 256
    uint2 kv[kSplitPerThread];
    uint32_t dr[kSplitPerThread];
    uint32_t valid = 0;
#if BHT_SPLIT_TMA
    if (full) {
      mbar_wait(&s.mbar, parity);
      parity ^= 1u;
    }
#endif
#pragma unroll
    for (int j = 0; j < kSplitPerThread / 2; ++j) {
      const uint32_t at = (j * kSplitBlock + threadIdx.x) * 2;  // this thread's two consecutive pairs
      if (full) {
#if BHT_SPLIT_TMA
        const uint4 two = *reinterpret_cast<const uint4*>(s.in + 2 * at);
#else
        const uint4 two = __ldcs(reinterpret_cast<const uint4*>(src + at));
#endif
        kv[2 * j] = make_uint2(two.x, two.y);
        kv[2 * j + 1] = make_uint2(two.z, two.w);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) kv[2 * j + e] = at + e < cur.len ? __ldcs(src + at + e) : make_uint2(0u, 0u);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) valid |= (at + e < cur.len) ? 1u << (2 * j + e) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t d = region_of(kv[j].x);
      uint32_t rank = 0;
      if ((valid >> j) & 1u) rank = atomicAdd(&s.hist[d], 1u);
      dr[j] = d | (rank << 8);
    }
    __syncthreads();  // every rank of the tile is taken, and `in` has been read by everyone
    fetch(nxt);
    const PackedSink sink{a.bins, a.sp};
    if (full) split_tile_finish<true>(s, kv, dr, valid, cur.len, n_dest, f_base, a.cap, a.bin_cursor, sink, cur.id, region_of);
    else split_tile_finish<false>(s, kv, dr, valid, cur.len, n_dest, f_base, a.cap, a.bin_cursor, sink, cur.id, region_of);
    cur = nxt;
  }
}

// ---- K11 ------------------------------------------------------------------------------------------------------
// One 16-byte unit of a bin = two pairs.  GUARD: the unit may lie (partly) past the end of the bin.
template <bool GUARD>
__device__ __forceinline__ uint32_t claim_unit(const uint4 v, uint32_t q, uint32_t n_r, const HashFn& h0, uint32_t first32,
                                               uint32_t nb, uint32_t b_log2, uint32_t B, unsigned long long* rows, uint32_t* cnt) {
  uint32_t spilled = 0;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const uint32_t k = e ? v.z : v.x, val = e ? v.w : v.y;
    if (!GUARD || 2u * q + e < n_r) {
      const uint32_t lb = bucket_index(h0, k) - first32;  // < nb: the bin holds pairs of this region only
#if defined(BHT_EXP_NOSTORE) || defined(BHT_EXP_LINEAR) || defined(BHT_EXP_NOGATOM)
      if (lb >= nb) continue;  // the experiments feed this kernel garbage
#endif
      const uint32_t slot = atomicAdd(&cnt[lb], 1u);
      if (slot < B) rows[(lb << b_log2) + slot] = pack_pair(k, val);
      else spilled |= 1u << e;
    }
  }
  return spilled;
}

__global__ void __launch_bounds__(kBuildBlock, 3)
region_build_kernel(const __grid_constant__ TableView t, uint32_t region_log2, uint32_t b_log2, uint32_t cap,
                    const uint32_t* __restrict__ bin_cursor, const uint2* __restrict__ bins, int fresh, const Spill sp,
                    DevCounters* __restrict__ ctr, uint32_t ahead) {
  extern __shared__ __align__(16) unsigned char sm_bytes[];
  const uint32_t region_buckets = 1u << region_log2;
  const uint32_t B = 1u << b_log2;
  unsigned long long* rows = reinterpret_cast<unsigned long long*>(sm_bytes);  // region_buckets * B slots
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm_bytes + (static_cast<size_t>(region_buckets) << (b_log2 + 3)));
  uint2* stash = reinterpret_cast<uint2*>(cnt + region_buckets);  // the pairs whose bucket was full
  __shared__ uint32_t stash_count, hole_count;
  __shared__ unsigned long long stash_base;
  const uint32_t region = blockIdx.x;
  const uint64_t first = static_cast<uint64_t>(region) << region_log2;
  const uint32_t first32 = static_cast<uint32_t>(first);
  const uint32_t nb = static_cast<uint32_t>(min(static_cast<uint64_t>(region_buckets), t.num_buckets - first));
  const uint32_t n_slots = nb << b_log2;
  unsigned long long* gstore = reinterpret_cast<unsigned long long*>(t.store) + (first << b_log2);  // 64 KiB-aligned offset

  // The bin of the region `ahead` CTAs later (the CTA that takes this one's place on the SM, roughly) goes to the L2
  // now, so that phase 1 of that CTA reads L2 hits.
  if (ahead != 0 && region + ahead < gridDim.x) {
    const uint32_t r2 = region + ahead;
    const uint32_t bytes = min(bin_cursor[r2], cap) * 8u;
    const char* base = reinterpret_cast<const char*>(bins + static_cast<uint64_t>(r2) * cap);
    for (uint32_t off = threadIdx.x * 128u; off < bytes; off += kBuildBlock * 128u) prefetch_l2(base + off);
  }

#ifdef BHT_K11_TIMING
  long long tk[8];
  tk[0] = clock64();
#define TK(i) tk[i] = clock64()
#else
#define TK(i)
#endif
  // The bin's pairs arrive two per 16-byte load, U loads per thread and batch; the loads of batch k + 1 are in flight
  // while batch k is processed, and those of the first batch while the region is set up (phase 0).
  const uint32_t n_r = min(bin_cursor[region], cap);
  const uint2* bin = bins + static_cast<uint64_t>(region) * cap;  // 16-byte aligned: cap is even
  const uint4* bin4 = reinterpret_cast<const uint4*>(bin);
  const uint32_t n_units = (n_r + 1u) >> 1;
  constexpr int U = BHT_BUILD_U / 2;
  uint4 v_next[U];
  auto load_batch = [&](uint32_t q0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = q0 + u * kBuildBlock;
      v_next[u] = make_uint4(0u, 0u, 0u, 0u);
      if (q < n_units) v_next[u] = __ldcs(bin4 + q);  // an odd bin's last unit reads one pair of slack inside the bin's capacity
    }
  };
  load_batch(threadIdx.x);

  // phase 0: the region's buckets into shared memory
  {
    uint4* rows4 = reinterpret_cast<uint4*>(rows);
    const uint4* g4 = reinterpret_cast<const uint4*>(gstore);
    const uint32_t n4 = n_slots >> 1;
    if (fresh) {
      const uint4 e = make_uint4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
      for (uint32_t i = threadIdx.x; i < n4; i += kBuildBlock) rows4[i] = e;
      if ((n_slots & 1u) && threadIdx.x == 0) rows[n_slots - 1] = kEmptySlot;
    } else {
      for (uint32_t i = threadIdx.x; i < n4; i += kBuildBlock) rows4[i] = __ldcs(g4 + i);
      if ((n_slots & 1u) && threadIdx.x == 0) rows[n_slots - 1] = gstore[n_slots - 1];
    }
    for (uint32_t i = threadIdx.x; i < nb; i += kBuildBlock) cnt[i] = 0;
    if (threadIdx.x == 0) stash_count = hole_count = 0;
  }
  __syncthreads();
  if (!fresh) {
    // load of every bucket = 1 + index of its last occupied slot (equals compute_load, bucket.hpp:26-31, whenever the
    // occupied slots form a prefix; never overwrites anything on an uploaded store with holes)
    for (uint32_t i = threadIdx.x; i < n_slots; i += kBuildBlock) {
      const uint32_t lb = i >> b_log2, s = i & (B - 1u);
      if (static_cast<uint32_t>(rows[i]) != kEmptyKey) atomicMax(&cnt[lb], s + 1u);
    }
    __syncthreads();
  }

  TK(1);
  // phase 1: every pair of the bin claims slot = load++ of its bucket (a shared-memory atomic: no CAS, no lost race).
  // A pair whose bucket is full only leaves a bit in `spilled`; after the unrolled block the thread moves those pairs
  // (picked out of its registers with selects) to the CTA's stash in shared memory.
  for (uint32_t q0 = threadIdx.x; q0 < n_units; q0 += kBuildBlock * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = v_next[u];
    if (q0 + kBuildBlock * U < n_units) load_batch(q0 + kBuildBlock * U);
    uint32_t spilled = 0;
    if (2u * (q0 + (U - 1) * kBuildBlock) + 1u < n_r) {  // every pair of the thread's U units exists: no predicates
#pragma unroll
      for (int u = 0; u < U; ++u)
        spilled |= claim_unit<false>(v[u], q0 + u * kBuildBlock, n_r, t.h[0], first32, nb, b_log2, B, rows, cnt) << (2 * u);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        spilled |= claim_unit<true>(v[u], q0 + u * kBuildBlock, n_r, t.h[0], first32, nb, b_log2, B, rows, cnt) << (2 * u);
    }
    while (spilled != 0) {
      const uint32_t bit = __ffs(spilled) - 1u;
      spilled &= spilled - 1u;
      uint2 p = make_uint2(0u, 0u);  // pair `bit` of this batch, picked out of the registers with selects
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (bit == 2u * u) p = make_uint2(v[u].x, v[u].y);
        if (bit == 2u * u + 1u) p = make_uint2(v[u].z, v[u].w);
      }
      const uint32_t pos = atomicAdd(&stash_count, 1u);
      if (pos < kStashPairs) stash[pos] = p;
      else spill_fresh(p, sp);  // past the stash: straight to the list, untouched
    }
  }
  TK(2);
  __syncthreads();  // every claimed slot is written
  TK(3);

  // phase 1b: the first eviction of the stashed pairs, in shared memory (table.cpp:67-81): the pair goes into a random
  // slot of its full bucket, the victim goes to the spill list with the bucket named by the hash function after the
  // lowest-index one that maps it here, and a chain length of 1.  One probe (the inspection that found the bucket full).
  // (Measured: the stash holding bin positions, the pairs re-read from the
  // bin here, 257 us; holding the pairs, 226 us; writing the victims out only after the region's write-back has been
  // issued, 238 us.)
  const uint32_t spilled_total = stash_count;
  const uint32_t stashed = min(spilled_total, kStashPairs);
  if (stashed != 0) {
    // ONE list reservation per CTA (thousands of CTAs reserving per warp queue up on the one cursor word: the evictions
    // then waited 7-14 k cycles for it), issued before the evictions and picked up after them
    unsigned long long reserved = 0;
    if (threadIdx.x == 0) reserved = atomicAdd(sp.cursor, static_cast<unsigned long long>(stashed));
    uint64_t rng = xorshift_init(mix_seed(t.seed, 0x626C6B64ull + static_cast<uint64_t>(blockIdx.x) * kBuildBlock + threadIdx.x));
    constexpr int kRounds = (kStashPairs + kBuildBlock - 1) / kBuildBlock;
    uint32_t vk[kRounds], vv[kRounds], nx[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t i = r * kBuildBlock + threadIdx.x;
      vk[r] = kEmptyKey, vv[r] = 0, nx[r] = 0;
      if (i < stashed) {
        const uint2 p = stash[i];
        const uint32_t bid = bucket_index(t.h[0], p.x);
        const uint32_t lb = bid - first32;
        const unsigned long long old = atomicExch(rows + (lb << b_log2) + xorshift_next_below(rng, B), pack_pair(p.x, p.y));
        vk[r] = static_cast<uint32_t>(old);
        vv[r] = static_cast<uint32_t>(old >> 32);
        if (vk[r] != kEmptyKey) {
          if (fresh) {
            // every pair of a freshly built region sits in its H0 bucket, so the lowest-index hash function that maps
            // the victim here is H0 and its walk goes on at H1 (table.cpp:74-80)
            nx[r] = bucket_index(t.h[1], vk[r]);
          } else {
            uint32_t cand[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) cand[h] = h < static_cast<int>(t.n_hashes) ? bucket_index(t.h[h], vk[r]) : 0u;
            uint32_t next = cand[0];
#pragma unroll
            for (int h = 3; h >= 0; --h)  // lowest matching index wins (table.cpp:74-80)
              if (h < static_cast<int>(t.n_hashes) && cand[h] == bid) next = cand[h + 1 < static_cast<int>(t.n_hashes) ? h + 1 : 0];
            nx[r] = next;
          }
        } else {
          atomicAdd(&hole_count, 1u);  // a hole (only on an uploaded store): the pair is simply placed; the list entry becomes a tombstone
        }
      }
    }
    if (threadIdx.x == 0) stash_base = reserved;
    __syncthreads();
    const unsigned long long base = stash_base;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const uint32_t i = r * kBuildBlock + threadIdx.x;
      if (i < stashed) {
        const unsigned long long at = base + i;
        if (at < sp.cap) {
          sp.pairs[at] = make_uint2(vk[r], vv[r]);
          sp.start[at] = vk[r] == kEmptyKey ? kStartTombstone : (nx[r] | 0x80000000u);
        } else if (vk[r] != kEmptyKey) {
          spill_dropped(vk[r], sp);  // the victim in hand is the pair dropped, as when a chain hits its cap
        }
      }
    }
  }
  TK(4);
#if BHT_BUILD_TMA_STORE
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this thread's shared-memory writes, for the bulk-copy engine
#endif
  __syncthreads();
  TK(5);

  // phase 2: the region back to the store
  {
#if BHT_BUILD_TMA_STORE
    // bulk asynchronous copies shared -> global (cp.async.bulk, the TMA unit): 4 KiB pieces issued by the first threads,
    // no register staging and no load/store-unit traffic for the 64 KiB of the region
    constexpr uint32_t kPiece = 4096;
    const uint32_t bulk_bytes = (n_slots << 3) & ~15u;
    const uint32_t rows_saddr = static_cast<uint32_t>(__cvta_generic_to_shared(rows));
    unsigned char* gbytes = reinterpret_cast<unsigned char*>(gstore);
    for (uint32_t p = threadIdx.x * kPiece; p < bulk_bytes; p += kBuildBlock * kPiece) {
      const uint32_t sz = min(kPiece, bulk_bytes - p);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gbytes + p), "r"(rows_saddr + p), "r"(sz) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#else
    const uint4* rows4 = reinterpret_cast<const uint4*>(rows);
    uint4* g4 = reinterpret_cast<uint4*>(gstore);
    const uint32_t n4 = n_slots >> 1;
    for (uint32_t i = threadIdx.x; i < n4; i += kBuildBlock) g4[i] = rows4[i];
#endif
    if ((n_slots & 1u) && threadIdx.x == 0) gstore[n_slots - 1] = rows[n_slots - 1];
    if (threadIdx.x == 0 && n_r != 0) {
      // one set of global counter updates per CTA.  Every pair of the bin was either placed or noted in `stash_count`.
      const unsigned long long placed = n_r - spilled_total;
      const unsigned long long a = placed + hole_count;
      if (a != 0) {
        atomicAdd(&ctr->inserted, a);
        atomicAdd(&ctr->inserted_total, a);
      }
      atomicAdd(&ctr->insert_probes, placed + stashed);
    }
#if BHT_BUILD_TMA_STORE
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory may go once the copies have read it
#endif
  }
#ifdef BHT_K11_TIMING
  TK(6);
  if ((blockIdx.x % 997) == 5 && (threadIdx.x == 0 || threadIdx.x == 200))
    printf("K11 cta %u thr %u: fill %lld  claim-loop %lld  wait-claims %lld  evict %lld  wait-evict %lld  writeback %lld  total %lld (n_r %u stashed %u)\n",
           blockIdx.x, threadIdx.x, tk[1] - tk[0], tk[2] - tk[1], tk[3] - tk[2], tk[4] - tk[3], tk[5] - tk[4], tk[6] - tk[5], tk[6] - tk[0], n_r, stashed);
#endif
}

}  // namespace

// Geometry of a blocked build of up to n pairs into table t; n_regions == 0: not applicable.
BlockedPlan plan_blocked_build(const TableView& t, uint64_t n) {
  BlockedPlan p{};
  uint32_t b_log2 = 0;
  while ((1u << b_log2) < t.bucket_size) ++b_log2;
  if (b_log2 > 6 || n == 0 || n > 0xFFFFFFFFull) return p;
  // The first eviction of a pair whose bucket is full happens inside K11; with max_chain == 0 the reference fails that
  // insertion before any exchange (table.cpp:67), which is the general kernel's business.
  if (t.max_chain == 0) return p;
  // 64 KiB of slots per fine region (three CTAs of K11 per SM); 128 KiB (one CTA per SM, ~20 % slower) for tables
  // between 4 and 8 GB, so that two partition levels of <= 256 x 256 still reach every region
  uint32_t region_bytes_log2 = kRegionBytesLog2;
  if ((t.num_buckets << (b_log2 + 3)) > (256ull * kMaxShards << kRegionBytesLog2)) region_bytes_log2 = kRegionBytesLog2 + 1;
  if (region_bytes_log2 < 3 + b_log2 + 5) return p;
  const uint32_t region_log2 = region_bytes_log2 - 3 - b_log2;
  const uint64_t regions = (t.num_buckets + (1ull << region_log2) - 1) >> region_log2;
  if (regions > 256ull * kMaxShards || t.num_buckets >= 0x7FFFFFFEull) return p;  // two levels of <= 256 x 256; 31-bit start buckets below the tombstone word
  uint32_t per = static_cast<uint32_t>(std::ceil(std::sqrt(static_cast<double>(regions))));
  if (per < 1) per = 1;
  if (per > 256) per = 256;
  const uint32_t groups = static_cast<uint32_t>((regions + per - 1) / per);
  if (groups > static_cast<uint32_t>(kMaxShards)) return p;
  const double mean = static_cast<double>(n) * static_cast<double>(1ull << region_log2) / static_cast<double>(t.num_buckets);
  double cap = mean + 6.0 * std::sqrt(mean) + 32.0;
  if (cap > static_cast<double>(n)) cap = static_cast<double>(n);
  p.cap = (static_cast<uint32_t>(cap) + 2u) & ~1u;  // even: every bin starts 16-byte aligned
  p.n_regions = static_cast<uint32_t>(regions);
  p.region_log2 = region_log2;
  p.b_log2 = b_log2;
  p.per = per;
  p.n_groups = groups;
  const double gmean = mean * per;
  double gcap = gmean + 6.0 * std::sqrt(gmean) + 64.0;
  if (gcap > static_cast<double>(n)) gcap = static_cast<double>(n);
  p.group_cap = (static_cast<uint32_t>(gcap) + 2u) & ~1u;
  // the partition passes address their outputs with 32-bit indices
  if (static_cast<uint64_t>(p.n_groups) * p.group_cap >= 0xFFFFFFFFull || static_cast<uint64_t>(p.n_regions) * p.cap >= 0xFFFFFFFFull)
    return BlockedPlan{};
  return p;
}

// scratch layout: grouped pairs (n_groups * group_cap) | bins (n_regions * cap) | spill pairs (n) | spill_cursor (8) pad (8)
//                 | bin_cursor (n_regions) | group_cursor (n_groups) | pad to 16 | spill start words (n)
size_t blocked_scratch_bytes(const BlockedPlan& p, uint64_t n) {
  return static_cast<size_t>(p.n_groups) * p.group_cap * 8 + static_cast<size_t>(p.n_regions) * p.cap * 8 + n * 8 + 16 +
         (static_cast<size_t>(p.n_regions) + p.n_groups) * 4 + 16 + n * 4 + 64;
}

namespace {
struct ScratchMap {
  uint2 *grouped, *bins, *spill;
  unsigned long long* spill_cursor;
  uint32_t *bin_cursor, *group_cursor, *spill_start;
};
ScratchMap map_scratch(const BlockedPlan& p, uint64_t n, void* scratch) {
  ScratchMap m;
  m.grouped = reinterpret_cast<uint2*>(scratch);
  m.bins = m.grouped + static_cast<size_t>(p.n_groups) * p.group_cap;
  m.spill = m.bins + static_cast<size_t>(p.n_regions) * p.cap;
  m.spill_cursor = reinterpret_cast<unsigned long long*>(m.spill + n);
  m.bin_cursor = reinterpret_cast<uint32_t*>(m.spill_cursor + 2);
  m.group_cursor = m.bin_cursor + p.n_regions;
  m.spill_start = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(m.group_cursor + p.n_groups) + 15) & ~static_cast<uintptr_t>(15));
  return m;
}
}  // namespace

// A blocked build in three steps, so that a batch may arrive in chunks (host buffers over PCIe, the receive side of a
// sharded build): begin zeroes the cursors, scatter runs K8g over one chunk (any number of times, at most n pairs in
// total), finish runs K10 + K11 and hands the spill list to the caller.
cudaError_t blocked_build_begin(const BlockedPlan& p, uint64_t n, void* scratch, cudaStream_t stream) {
  const ScratchMap m = map_scratch(p, n, scratch);
  return cudaMemsetAsync(m.spill_cursor, 0, 16 + (static_cast<size_t>(p.n_regions) + p.n_groups) * 4, stream);
}

cudaError_t blocked_build_scatter(const TableView& t, const BlockedPlan& p, uint64_t n, void* scratch, const uint32_t* keys,
                                  const uint32_t* values, uint64_t len, const FailLog& log, int sm_count, cudaStream_t stream,
                                  const unsigned long long* len_dev) {
  if (len == 0) return cudaSuccess;
  const ScratchMap m = map_scratch(p, n, scratch);
  const Spill sp{m.spill, m.spill_start, m.spill_cursor, n, log.ctr, log.failed_keys, log.failed_cap};
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;  // values may be null
  const uint32_t inv_per = static_cast<uint32_t>((1ull << 32) / p.per) + 1u;  // exact quotient for fine ids < 2^16, per <= 256
  const uint64_t tiles = (len + kSplitTile - 1) / kSplitTile;
  const int grid = static_cast<int>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count) * BHT_SPLIT_CTAS));
  const cudaError_t attr = cudaFuncSetAttribute(group_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(sizeof(SplitShared)));
  if (attr != cudaSuccess) return attr;
  const GroupArgs ga{t.h[0], p.region_log2, inv_per, p.n_groups, p.group_cap, keys, values, len, len_dev, m.group_cursor, m.grouped, sp, aligned ? 1 : 0};
  group_scatter_kernel<<<grid, kSplitBlock, sizeof(SplitShared), stream>>>(ga);
  note_launch();
  return cudaGetLastError();
}

cudaError_t blocked_build_finish(const TableView& t, const BlockedPlan& p, uint64_t n, void* scratch, bool fresh,
                                 const FailLog& log, int sm_count, cudaStream_t stream, PairSource* spill_out,
                                 const unsigned long long** spill_count_out) {
  DevCounters* ctr = log.ctr;
  const ScratchMap m = map_scratch(p, n, scratch);
  const Spill sp{m.spill, m.spill_start, m.spill_cursor, n, log.ctr, log.failed_keys, log.failed_cap};
  const uint64_t tiles_b = static_cast<uint64_t>(p.n_groups) * ((p.group_cap + kSplitTile - 1) / kSplitTile);
  const int grid_b = static_cast<int>(std::min<uint64_t>(tiles_b, static_cast<uint64_t>(sm_count) * BHT_SPLIT_CTAS));
  const cudaError_t attr = cudaFuncSetAttribute(bin_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(sizeof(SplitShared)));
  if (attr != cudaSuccess) return attr;
  const BinArgs ba{t.h[0], p.region_log2, p.per, p.n_groups, p.n_regions, p.cap, p.group_cap, m.grouped, m.group_cursor, m.bin_cursor, m.bins, sp};
  bin_split_kernel<<<grid_b, kSplitBlock, sizeof(SplitShared), stream>>>(ba);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  const int smem_c = static_cast<int>((8u << (p.region_log2 + p.b_log2)) + (4u << p.region_log2) + kStashPairs * 8);
  e = cudaFuncSetAttribute(region_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_c);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
#if BHT_BUILD_PREFETCH
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, region_build_kernel, kBuildBlock, smem_c) != cudaSuccess) per_sm = 1;
#endif
  region_build_kernel<<<p.n_regions, kBuildBlock, smem_c, stream>>>(t, p.region_log2, p.b_log2, p.cap, m.bin_cursor, m.bins,
                                                                   fresh ? 1 : 0, sp, ctr, static_cast<uint32_t>(per_sm * sm_count));
  note_launch();
  spill_out->keys = reinterpret_cast<const uint32_t*>(m.spill);
  spill_out->values = nullptr;
  spill_out->start = m.spill_start;
  *spill_count_out = m.spill_cursor;
  return cudaGetLastError();
}

// K8s: `cursor32` = n_shards words of scratch (zeroed here).  cap * n_shards < 2^32, n < 2^32 (checked by the caller).
cudaError_t launch_shard_split_fixed(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys, const uint32_t* values,
                                     uint64_t n, uint64_t cap, uint32_t* cursor32, unsigned long long* counts, uint32_t* overflow,
                                     uint32_t* out_keys, uint32_t* out_values, uint32_t* out_index, int sm_count, cudaStream_t stream) {
  if (n_shards == 0 || n_shards > 256u) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(cursor32, 0, sizeof(uint32_t) * n_shards, stream);
  if (e != cudaSuccess) return e;
  if (n != 0) {
    const cudaError_t attr = cudaFuncSetAttribute(shard_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        static_cast<int>(sizeof(SplitShared)));
    if (attr != cudaSuccess) return attr;
    ShardSplitArgs a{};
    a.alpha = alpha, a.beta = beta, a.n_shards = n_shards, a.cap = static_cast<uint32_t>(cap);
    a.keys = keys, a.values = values, a.n = n, a.cursor = cursor32;
    a.sink = SplitArraysSink{out_keys, values != nullptr ? out_values : out_index, overflow};
    a.index_mode = values == nullptr && out_index != nullptr;
    a.aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;
    const uint64_t tiles = (n + kSplitTile - 1) / kSplitTile;
    const int grid = static_cast<int>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count) * BHT_SPLIT_CTAS));
    shard_split_kernel<<<grid, kSplitBlock, sizeof(SplitShared), stream>>>(a);
    note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  shard_counts_kernel<<<(n_shards + 255) / 256, 256, 0, stream>>>(n_shards, static_cast<uint32_t>(cap), cursor32, counts, overflow);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_blocked_build(const TableView& t, const BlockedPlan& p, const uint32_t* keys, const uint32_t* values,
                                 uint64_t n, bool fresh, void* scratch, const FailLog& log, int sm_count, cudaStream_t stream,
                                 PairSource* spill_out, const unsigned long long** spill_count_out) {
  cudaError_t e = blocked_build_begin(p, n, scratch, stream);
  if (e == cudaSuccess) e = blocked_build_scatter(t, p, n, scratch, keys, values, n, log, sm_count, stream, nullptr);
  if (e == cudaSuccess) e = blocked_build_finish(t, p, n, scratch, fresh, log, sm_count, stream, spill_out, spill_count_out);
  return e;
}

}  // namespace bht_b200
