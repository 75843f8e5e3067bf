// build_blocked.cu — K10 / K11: the shared-memory-blocked bulk build of the cuckoo tables (bcht, 1cht).
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
//                       A pair whose bucket is full goes to a per-CTA stash; once every claim is written the stashed
//                       pairs do their first eviction in shared memory (atomicExch into a random slot of the full
//                       bucket, table.cpp:67-81) and the VICTIMS go to the global spill list, each with the bucket
//                       its walk goes on in and a chain length of 1 (one list reservation per CTA).
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
#include <cstdlib>

#include "insert_common.cuh"

#ifndef BHT_BUILD_BLOCK  // measured (insert, 50 M pairs): 192 x 20: 1.087 ms, 256 x 16: 1.062, 320 x 12: 1.034, 384 x 10: 1.034 (spills)
#define BHT_BUILD_BLOCK 320
#define BHT_BUILD_U 12
#endif

#ifndef BHT_BUILD_TMA_STORE
#define BHT_BUILD_TMA_STORE 1
#endif

namespace bht_b200 {

namespace {

constexpr int kSplitBlock = 256;
#ifndef BHT_SPLIT_PER_THREAD
#define BHT_SPLIT_PER_THREAD 8
#endif
constexpr int kSplitPerThread = BHT_SPLIT_PER_THREAD;
constexpr int kSplitTile = kSplitBlock * kSplitPerThread;  // 2048 pairs
constexpr int kBuildBlock = BHT_BUILD_BLOCK;   // few threads with many loads in flight each: 3 CTAs/SM by shared memory
constexpr uint32_t kStashPairs = 1024;  // per-CTA stash of spilled pairs (K11)
constexpr uint32_t kRegionBytesLog2 = 16;

// The spill list: packed pairs + where their walk starts (kStartAtH0 for a pair that has not probed anything yet).
struct Spill {
  uint2* pairs;
  uint32_t* start;
  unsigned long long* cursor;
};

// Appends the pairs of the lanes with `spilled` to the spill list as fresh pairs: one global atomic per warp (rare paths).
__device__ __forceinline__ void spill_append(bool spilled, uint2 kv, const Spill& sp, int lane) {
  uint2* __restrict__ spill = sp.pairs;
  unsigned long long* __restrict__ spill_cursor = sp.cursor;
  const uint32_t m = __ballot_sync(kFullMask, spilled);
  if (m == 0) return;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(spill_cursor, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(kFullMask, base, leader);
  if (spilled) {
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    spill[pos] = kv;
    sp.start[pos] = kStartAtH0;
  }
}

// ---- K8g ------------------------------------------------------------------------------------------------------
// First partition level, one pass: every pair goes to the segment of its GROUP (= `per` consecutive fine regions).
// Tiles of 2048 pairs are ranked by group in shared memory, one global atomicAdd per (tile, group) reserves a run in
// the group's fixed-capacity segment, the tile is staged by group and written out run by run (~25 pairs per run).
// No histogram pre-pass and no destination bytes: the hash is uniform, so the segments are sized mean + 6 sigma and the
// few pairs that do not fit go to the spill list.
__device__ __forceinline__ uint4 load_group4(const uint32_t* __restrict__ p, uint64_t i, uint64_t n, bool aligned) {
  if (aligned && i + 4 <= n) return __ldcs(reinterpret_cast<const uint4*>(p + i));
  uint4 r = make_uint4(0, 0, 0, 0);
  if (i < n) r.x = p[i];
  if (i + 1 < n) r.y = p[i + 1];
  if (i + 2 < n) r.z = p[i + 2];
  if (i + 3 < n) r.w = p[i + 3];
  return r;
}

__global__ void __launch_bounds__(kSplitBlock)
group_scatter_kernel(const __grid_constant__ HashFn h0, uint32_t region_log2, uint32_t inv_per, uint32_t n_groups, uint32_t group_cap,
                     const uint32_t* __restrict__ keys, const uint32_t* __restrict__ values, uint64_t n, bool aligned,
                     uint32_t* __restrict__ group_cursor, uint2* __restrict__ grouped, const Spill sp) {
  __shared__ uint2 s_pair[kSplitTile];
  __shared__ uint8_t s_dest[kSplitTile];
  __shared__ uint32_t hist[256], tile_off[256], base_of[256], warp_tot[kSplitBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n_tiles = (n + kSplitTile - 1) / kSplitTile;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t i0 = tile * kSplitTile;
    hist[threadIdx.x] = 0;
    __syncthreads();
    constexpr int kGroups = kSplitPerThread / 4;  // groups of 4 consecutive pairs per thread
    uint32_t k[kGroups][4], v[kGroups][4], dst[kGroups][4], rank[kGroups][4];
#pragma unroll
    for (int j = 0; j < kGroups; ++j) {
      const uint64_t i = i0 + (static_cast<uint64_t>(j) * kSplitBlock + threadIdx.x) * 4;
      const uint4 k4 = load_group4(keys, i, n, aligned);
      k[j][0] = k4.x, k[j][1] = k4.y, k[j][2] = k4.z, k[j][3] = k4.w;
      if (values != nullptr) {
        const uint4 v4 = load_group4(values, i, n, aligned);
        v[j][0] = v4.x, v[j][1] = v4.y, v[j][2] = v4.z, v[j][3] = v4.w;
      } else {  // keys-only build: the value is value_for_key(key) (table.cpp:234)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[j][e] = value_for_key(k[j][e]);
      }
    }
#pragma unroll
    for (int j = 0; j < kGroups; ++j) {
      const uint64_t i = i0 + (static_cast<uint64_t>(j) * kSplitBlock + threadIdx.x) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        dst[j][e] = static_cast<uint32_t>((static_cast<uint64_t>(bucket_index(h0, k[j][e]) >> region_log2) * inv_per) >> 32);
        rank[j][e] = 0;
        if (i + e < n) rank[j][e] = atomicAdd(&hist[dst[j][e]], 1u);
      }
    }
    __syncthreads();
    {
      const uint32_t h = hist[threadIdx.x];
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) warp_tot[warp] = x;
      __syncthreads();
      uint32_t before = 0;
      for (int w = 0; w < warp; ++w) before += warp_tot[w];
      tile_off[threadIdx.x] = before + x - h;
      base_of[threadIdx.x] = (h != 0 && threadIdx.x < n_groups) ? atomicAdd(&group_cursor[threadIdx.x], h) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kGroups; ++j) {
      const uint64_t i = i0 + (static_cast<uint64_t>(j) * kSplitBlock + threadIdx.x) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (i + e < n) {
          const uint32_t slot = tile_off[dst[j][e]] + rank[j][e];
          s_pair[slot] = make_uint2(k[j][e], v[j][e]);
          s_dest[slot] = static_cast<uint8_t>(dst[j][e]);
        }
      }
    }
    __syncthreads();
    const uint32_t in_tile = static_cast<uint32_t>(n - i0 < kSplitTile ? n - i0 : kSplitTile);
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t slot = j * kSplitBlock + threadIdx.x;
      const bool in = slot < in_tile;
      uint2 out = make_uint2(0u, 0u);
      bool fits = false;
      if (in) {
        const uint32_t d = s_dest[slot];
        const uint32_t pos = base_of[d] + (slot - tile_off[d]);
        out = s_pair[slot];
        fits = pos < group_cap;
        if (fits) __stcs(grouped + static_cast<uint64_t>(d) * group_cap + pos, out);
      }
      spill_append(in && !fits, out, sp, lane);
    }
    __syncthreads();
  }
}

// ---- K10 ------------------------------------------------------------------------------------------------------
// grouped: segment g = pairs of group g (fine regions [g * per, (g + 1) * per)), group_cursor[g] of them (clamped to
// group_cap).  bins[f * cap ..] / bin_cursor[f]: the bin of fine region f.  A tile never leaves its group.
__global__ void __launch_bounds__(kSplitBlock)
bin_split_kernel(const __grid_constant__ HashFn h0, uint32_t region_log2, uint32_t per, uint32_t n_groups, uint32_t n_regions,
                 uint32_t cap, uint32_t group_cap, const uint2* __restrict__ grouped, const uint32_t* __restrict__ group_cursor,
                 uint32_t* __restrict__ bin_cursor, uint2* __restrict__ bins, const Spill sp) {
  __shared__ uint2 s_pair[kSplitTile];
  __shared__ uint8_t s_local[kSplitTile];
  __shared__ uint32_t hist[256], tile_off[256], base_of[256], warp_tot[kSplitBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tiles_per_group = (group_cap + kSplitTile - 1) / kSplitTile;
  const uint64_t n_tiles = static_cast<uint64_t>(n_groups) * tiles_per_group;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint32_t g = static_cast<uint32_t>(tile / tiles_per_group);
    const uint32_t t0 = static_cast<uint32_t>(tile % tiles_per_group) * kSplitTile;
    const uint32_t in_group = min(group_cursor[g], group_cap);
    if (t0 >= in_group) continue;  // block-uniform
    const uint32_t len = min(static_cast<uint32_t>(kSplitTile), in_group - t0);
    const uint2* src = grouped + static_cast<uint64_t>(g) * group_cap + t0;
    const uint32_t f_base = g * per;
    hist[threadIdx.x] = 0;
    __syncthreads();

    uint2 kv[kSplitPerThread];
    uint32_t local[kSplitPerThread], rank[kSplitPerThread];
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t i = j * kSplitBlock + threadIdx.x;
      kv[j] = i < len ? __ldcs(src + i) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t i = j * kSplitBlock + threadIdx.x;
      local[j] = (bucket_index(h0, kv[j].x) >> region_log2) - f_base;  // < per <= 256 for every pair of the group
      rank[j] = 0;
      if (i < len && local[j] < 256u) rank[j] = atomicAdd(&hist[local[j]], 1u);
    }
    __syncthreads();
    // exclusive scan of hist + one global reservation per destination of the tile
    {
      const uint32_t h = hist[threadIdx.x];
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) warp_tot[warp] = x;
      __syncthreads();
      uint32_t before = 0;
      for (int w = 0; w < warp; ++w) before += warp_tot[w];
      tile_off[threadIdx.x] = before + x - h;
      const uint32_t f = f_base + threadIdx.x;
      base_of[threadIdx.x] = (h != 0 && f < n_regions) ? atomicAdd(&bin_cursor[f], h) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t i = j * kSplitBlock + threadIdx.x;
      if (i < len && local[j] < 256u) {
        const uint32_t slot = tile_off[local[j]] + rank[j];
        s_pair[slot] = kv[j];
        s_local[slot] = static_cast<uint8_t>(local[j]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSplitPerThread; ++j) {
      const uint32_t slot = j * kSplitBlock + threadIdx.x;
      const bool in = slot < len;
      uint2 out = make_uint2(0u, 0u);
      bool fits = false;
      if (in) {
        const uint32_t l = s_local[slot];
        const uint32_t pos = base_of[l] + (slot - tile_off[l]);
        out = s_pair[slot];
        fits = pos < cap;
        if (fits) bins[static_cast<uint64_t>(f_base + l) * cap + pos] = out;
      }
      spill_append(in && !fits, out, sp, lane);
    }
    __syncthreads();
  }
}

// ---- K11 ------------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kBuildBlock)
region_build_kernel(const __grid_constant__ TableView t, uint32_t region_log2, uint32_t b_log2, uint32_t cap,
                    const uint32_t* __restrict__ bin_cursor, const uint2* __restrict__ bins, int fresh, const Spill sp,
                    DevCounters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char sm_bytes[];
  const uint32_t region_buckets = 1u << region_log2;
  const uint32_t B = 1u << b_log2;
  unsigned long long* rows = reinterpret_cast<unsigned long long*>(sm_bytes);  // region_buckets * B slots
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm_bytes + (static_cast<size_t>(region_buckets) << (b_log2 + 3)));
  uint2* stash = reinterpret_cast<uint2*>(cnt + region_buckets);
  __shared__ uint32_t stash_count, placed_count, hole_count;
  __shared__ unsigned long long stash_base;
  const int lane = threadIdx.x & 31;
  const uint32_t region = blockIdx.x;
  const uint64_t first = static_cast<uint64_t>(region) << region_log2;
  const uint32_t nb = static_cast<uint32_t>(min(static_cast<uint64_t>(region_buckets), t.num_buckets - first));
  const uint32_t n_slots = nb << b_log2;
  unsigned long long* gstore = reinterpret_cast<unsigned long long*>(t.store) + (first << b_log2);  // 64 KiB-aligned offset

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
    if (threadIdx.x == 0) stash_count = placed_count = hole_count = 0;
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

  // phase 1: every pair of the bin claims slot = load++ of its bucket
  const uint32_t n_r = min(bin_cursor[region], cap);
  const uint2* bin = bins + static_cast<uint64_t>(region) * cap;
  uint32_t n_ins = 0;
  constexpr int U = BHT_BUILD_U;  // pairs in flight per thread: a 64 KiB region holds ~29 pairs per thread at load factor 0.9
  for (uint32_t i0 = threadIdx.x; i0 - lane < n_r; i0 += kBuildBlock * U) {  // warp-uniform trip count
    uint2 kv[U];
    bool in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * kBuildBlock;
      in[u] = i < n_r;
      kv[u] = make_uint2(0u, 0u);
      if (in[u]) kv[u] = __ldcs(bin + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool spilled = false;
      if (in[u]) {
        const uint32_t lb = bucket_index(t.h[0], kv[u].x) - static_cast<uint32_t>(first);
        const uint32_t slot = lb < nb ? atomicAdd(&cnt[lb], 1u) : B;
        if (slot < B) {
          rows[(lb << b_log2) + slot] = pack_pair(kv[u].x, kv[u].y);
          ++n_ins;
        } else {
          spilled = true;
        }
      }
      // spilled pairs: into the CTA's stash (one shared-memory atomic per warp); past its end, straight to the list
      const uint32_t m = __ballot_sync(kFullMask, spilled);
      if (m != 0) {
        const int leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&stash_count, static_cast<uint32_t>(__popc(m)));
        base = __shfl_sync(kFullMask, base, leader);
        const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
        const bool stashed = spilled && pos < kStashPairs;
        if (stashed) stash[pos] = kv[u];
        spill_append(spilled && !stashed, kv[u], sp, lane);
      }
    }
  }
  {  // one set of global counter updates per CTA (not per warp: thousands of CTAs would hammer three addresses)
    uint32_t w = n_ins;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(kFullMask, w, o);
    if (lane == 0 && w != 0) atomicAdd(&placed_count, w);
  }
  __syncthreads();  // every claimed slot is written

  // phase 1b: the first eviction of the stashed pairs, in shared memory (table.cpp:67-81): the pair goes into a random
  // slot of its full bucket, the victim goes to the spill list with the bucket named by the hash function after the
  // lowest-index one that maps it here, and a chain length of 1.  One probe (the inspection that found the bucket full).
  const uint32_t stashed = min(stash_count, kStashPairs);
  if (threadIdx.x == 0 && stashed != 0) stash_base = atomicAdd(sp.cursor, static_cast<unsigned long long>(stashed));
  __syncthreads();
  if (stashed != 0) {
    uint64_t rng = xorshift_init(mix_seed(t.seed, 0x626C6B64ull + static_cast<uint64_t>(blockIdx.x) * kBuildBlock + threadIdx.x));
    for (uint32_t i = threadIdx.x; i < stashed; i += kBuildBlock) {
      const uint2 p = stash[i];
      const uint32_t bid = bucket_index(t.h[0], p.x);
      const uint32_t lb = bid - static_cast<uint32_t>(first);
      const unsigned long long old = atomicExch(rows + (lb << b_log2) + xorshift_next_below(rng, B), pack_pair(p.x, p.y));
      const uint32_t vk = static_cast<uint32_t>(old);
      uint32_t next = 0;
      if (vk != kEmptyKey) {
        uint32_t cand[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) cand[h] = h < static_cast<int>(t.n_hashes) ? bucket_index(t.h[h], vk) : 0u;
        next = cand[0];
#pragma unroll
        for (int h = 3; h >= 0; --h)  // lowest matching index wins (table.cpp:74-80)
          if (h < static_cast<int>(t.n_hashes) && cand[h] == bid) next = cand[h + 1 < static_cast<int>(t.n_hashes) ? h + 1 : 0];
      }
      // a hole (only on an uploaded store): the pair is simply placed; the reserved list entry becomes a tombstone
      if (vk == kEmptyKey) atomicAdd(&hole_count, 1u);
      sp.pairs[stash_base + i] = make_uint2(vk, static_cast<uint32_t>(old >> 32));
      sp.start[stash_base + i] = next | 0x80000000u;
    }
  }
#if BHT_BUILD_TMA_STORE
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this thread's shared-memory writes, for the bulk-copy engine
#endif
  __syncthreads();

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
    if (threadIdx.x == 0 && (placed_count != 0 || stashed != 0)) {
      const unsigned long long a = static_cast<unsigned long long>(placed_count) + hole_count;
      if (a != 0) {
        atomicAdd(&ctr->inserted, a);
        atomicAdd(&ctr->inserted_total, a);
      }
      atomicAdd(&ctr->insert_probes, static_cast<unsigned long long>(placed_count) + stashed);
    }
#if BHT_BUILD_TMA_STORE
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory may go once the copies have read it
#endif
  }
}

}  // namespace

// Geometry of a blocked build of n pairs into table t; n_regions == 0: not applicable.
BlockedPlan plan_blocked_build(const TableView& t, uint64_t n) {
  BlockedPlan p{};
  uint32_t b_log2 = 0;
  while ((1u << b_log2) < t.bucket_size) ++b_log2;
  if (b_log2 > 6 || n == 0 || n > 0xFFFFFFFFull) return p;
  // 64 KiB of slots per fine region (three CTAs of K11 per SM); 128 KiB (one CTA per SM, ~20 % slower) for tables
  // between 4 and 8 GB, so that two partition levels of <= 256 x 256 still reach every region
  uint32_t region_bytes_log2 = kRegionBytesLog2;
  if ((t.num_buckets << (b_log2 + 3)) > (256ull * kMaxShards << kRegionBytesLog2)) region_bytes_log2 = kRegionBytesLog2 + 1;
  if (const char* e = std::getenv("BHT_REGION_BYTES_LOG2")) region_bytes_log2 = static_cast<uint32_t>(std::atoi(e));  // tuning knob
  if (region_bytes_log2 < 12 || region_bytes_log2 > 17 || region_bytes_log2 < 3 + b_log2 + 5) return p;
  const uint32_t region_log2 = region_bytes_log2 - 3 - b_log2;
  const uint64_t regions = (t.num_buckets + (1ull << region_log2) - 1) >> region_log2;
  if (regions > 256ull * kMaxShards || t.num_buckets > 0x7FFFFFFFull) return p;  // two levels of <= 256 x 256; 31-bit start buckets
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
  return p;
}

// scratch layout: grouped pairs (n_groups * group_cap) | bins (n_regions * cap) | spill pairs (n) | spill_cursor (8) pad (8)
//                 | bin_cursor (n_regions) | group_cursor (n_groups) | pad to 16 | spill start words (n)
size_t blocked_scratch_bytes(const BlockedPlan& p, uint64_t n) {
  return static_cast<size_t>(p.n_groups) * p.group_cap * 8 + static_cast<size_t>(p.n_regions) * p.cap * 8 + n * 8 + 16 +
         (static_cast<size_t>(p.n_regions) + p.n_groups) * 4 + 16 + n * 4 + 64;
}

cudaError_t launch_blocked_build(const TableView& t, const BlockedPlan& p, const uint32_t* keys, const uint32_t* values,
                                 uint64_t n, bool fresh, void* scratch, DevCounters* ctr, int sm_count, cudaStream_t stream,
                                 PairSource* spill_out, const unsigned long long** spill_count_out) {
  unsigned char* s = static_cast<unsigned char*>(scratch);
  uint2* grouped = reinterpret_cast<uint2*>(s);
  uint2* bins = grouped + static_cast<size_t>(p.n_groups) * p.group_cap;
  uint2* spill = bins + static_cast<size_t>(p.n_regions) * p.cap;
  unsigned long long* spill_cursor = reinterpret_cast<unsigned long long*>(spill + n);
  uint32_t* bin_cursor = reinterpret_cast<uint32_t*>(spill_cursor + 2);
  uint32_t* group_cursor = bin_cursor + p.n_regions;
  uint32_t* spill_start = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(group_cursor + p.n_groups) + 15) & ~static_cast<uintptr_t>(15));
  const Spill sp{spill, spill_start, spill_cursor};
  cudaError_t e = cudaMemsetAsync(spill_cursor, 0, 16 + (static_cast<size_t>(p.n_regions) + p.n_groups) * 4, stream);
  if (e != cudaSuccess) return e;

  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;  // values may be null
  const uint32_t inv_per = static_cast<uint32_t>((1ull << 32) / p.per) + 1u;  // exact quotient for fine ids < 2^16, per <= 256
  const uint64_t tiles_a = (n + kSplitTile - 1) / kSplitTile;
  const int grid_a = static_cast<int>(std::min<uint64_t>(tiles_a, static_cast<uint64_t>(sm_count) * 8));
  group_scatter_kernel<<<grid_a, kSplitBlock, 0, stream>>>(t.h[0], p.region_log2, inv_per, p.n_groups, p.group_cap, keys, values, n,
                                                          aligned, group_cursor, grouped, sp);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  const uint64_t tiles_b = static_cast<uint64_t>(p.n_groups) * ((p.group_cap + kSplitTile - 1) / kSplitTile);
  const int grid_b = static_cast<int>(std::min<uint64_t>(tiles_b, static_cast<uint64_t>(sm_count) * 8));
  bin_split_kernel<<<grid_b, kSplitBlock, 0, stream>>>(t.h[0], p.region_log2, p.per, p.n_groups, p.n_regions, p.cap, p.group_cap,
                                                      grouped, group_cursor, bin_cursor, bins, sp);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  const int smem_c = static_cast<int>((8u << (p.region_log2 + p.b_log2)) + (4u << p.region_log2) + kStashPairs * 8);
  e = cudaFuncSetAttribute(region_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_c);
  if (e != cudaSuccess) return e;
  region_build_kernel<<<p.n_regions, kBuildBlock, smem_c, stream>>>(t, p.region_log2, p.b_log2, p.cap, bin_cursor, bins,
                                                                   fresh ? 1 : 0, sp, ctr);
  note_launch();
  spill_out->keys = reinterpret_cast<const uint32_t*>(spill);
  spill_out->values = nullptr;
  spill_out->start = spill_start;
  *spill_count_out = spill_cursor;
  return cudaGetLastError();
}

}  // namespace bht_b200
