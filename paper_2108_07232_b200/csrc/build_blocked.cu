// build_blocked.cu — K10 / K11: the shared-memory-blocked bulk build of the bucketed cuckoo table (bcht, 8 <= b <= 32).
//
// Same algorithm as bcht_insert (reference: proj/src/table.cpp:53-92) — a pair goes to slot index = load of its
// H0 bucket (table.cpp:85); when that bucket is full the insertion goes on as an eviction chain (table.cpp:63-81)
// — but the first attempt of every pair, which is ~90 % of all the probes of a build at load factor 0.9, never
// touches HBM at random and never issues a compare-and-swap:
//
//   K10 bin_scatter    one streaming pass: every pair is appended to the BIN of its first bucket.  A bin covers 32
//                      consecutive buckets (4 KiB of slots at b = 16; a 444 MB table has 108 k bins).  The position
//                      inside the bin is one global atomicAdd on the bin's cursor (L2 atomics on ~100 k distinct
//                      addresses: no hot spot, and cheaper per lane than a shared-memory atomic); the pair is
//                      written with one 8-byte store that the L2 merges with its neighbours into full sectors
//                      (the open ends of all bins together are a few MB).  Bins have a fixed capacity (mean +
//                      6 sigma of a uniform hash + 32); what does not fit goes to the spill list.
//   K11 bin_build      one WARP per bin, lane l owns bucket l of the bin: the 32 buckets live in shared memory
//                      (filled with the empty pattern when the table is known to be empty, else loaded from the
//                      store); the warp reads 32 pairs at a time, five ballots over the bits of the local bucket
//                      index give every pair its rank among the pairs of the same bucket and every owner lane
//                      the number of arrivals, so slot = load + rank needs no atomic at all (shared-memory atomics
//                      cost 2 cycles per lane on this part and were the bottleneck of the first version); the
//                      bin is written back with coalesced 16-byte stores.  No block-level barrier anywhere.
//                      A pair whose bucket is full goes to a small per-warp stash that is flushed to the global
//                      spill list 32+ pairs at a time (one global atomic per flush).
//   K4  (existing)     the general cuckoo kernel (insert_cuckoo.cu) inserts the spill list: it probes H0, finds
//                      the bucket full, exchanges a random victim and walks the chain exactly as the reference.
//
// STATUS (measured on B200, bcht b = 16, 50 M pairs, LF 0.9; profiles/r01e_blocked_build.txt): K10 1.12 ms, K11
// 0.33 ms, K4 on the 5.4 M spilled pairs 0.32 ms = 1.79 ms, the same as the L2-routed build (insert_cuckoo.cu,
// 1.80 ms), which therefore stays the default; this path is selected with bht_set_blocked_insert(table, 3).
// K11 is where it should be (pure streaming + ballots).  K10 is bound by the L2: 50 M atomics with a return take
// 0.47 ms alone (105 G/s) and 50 M scattered 8-byte stores another 0.65 ms — a store that covers part of a 32-byte
// sector costs the L2 a read-modify-write (~77 G/s), whatever line it hits.  An earlier version ranked the pairs
// of 32 K-pair tiles with shared-memory atomics instead: 2 cycles per lane (ATOMS), 0.85 ms.  The way forward is a
// two-level partition whose ranks come from ballots (as in K11) and whose runs are written as whole sectors.
//
// Probe accounting (probe_stats.hpp:12-31: one probe per bucket inspection): a pair placed by K11 costs one probe;
// a spilled pair is not counted here — its inspection of the full H0 bucket is the first probe K4 counts for it.
// HBM traffic of K10 + K11: read keys + values, write and read the bins, write (or read and write) the store once,
// all streaming — about 24 B per pair plus 8 B per slot, against 174 B per pair of random sectors.
#include <cmath>
#include <cstdlib>

#include "insert_common.cuh"

namespace bht_b200 {

namespace {

constexpr int kScatterBlock = 256;
constexpr int kBuildBlock = 256;
constexpr int kBuildWarps = kBuildBlock / 32;
constexpr uint32_t kBinLog2 = 5;      // buckets per bin = lanes per warp
constexpr uint32_t kStashPairs = 64;  // per-warp stash of spilled pairs

__device__ __forceinline__ uint4 load_group(const uint32_t* __restrict__ p, uint64_t i, uint64_t n, bool aligned) {
  if (aligned && i + 4 <= n) return __ldcs(reinterpret_cast<const uint4*>(p + i));
  uint4 r = make_uint4(0, 0, 0, 0);
  if (i < n) r.x = p[i];
  if (i + 1 < n) r.y = p[i + 1];
  if (i + 2 < n) r.z = p[i + 2];
  if (i + 3 < n) r.w = p[i + 3];
  return r;
}

// Appends the pairs of the lanes with `spilled` to the spill list: one global atomic per warp (rare path of K10).
__device__ __forceinline__ void spill_append(bool spilled, uint2 kv, uint2* __restrict__ spill,
                                             unsigned long long* __restrict__ spill_cursor, int lane) {
  const uint32_t m = __ballot_sync(kFullMask, spilled);
  if (m == 0) return;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(spill_cursor, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(kFullMask, base, leader);
  if (spilled) spill[base + __popc(m & ((1u << lane) - 1u))] = kv;
}

// ---- K10 ------------------------------------------------------------------------------------------------------
constexpr int kScatterGroups = 2;  // groups of 4 consecutive pairs per thread and iteration: 8 atomics in flight

__global__ void __launch_bounds__(kScatterBlock)
bin_scatter_kernel(const __grid_constant__ HashFn h0, uint32_t cap, uint32_t cursor_shift, const uint32_t* __restrict__ keys,
                   const uint32_t* __restrict__ values, uint64_t n, bool aligned, uint32_t* __restrict__ bin_cursor,
                   uint2* __restrict__ bins, uint2* __restrict__ spill, unsigned long long* __restrict__ spill_cursor) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kScatterBlock * 4;  // one group per thread
  const uint64_t first = (static_cast<uint64_t>(blockIdx.x) * kScatterBlock + threadIdx.x) * 4;
  // warp-uniform trip count: the warp's first element decides
  for (uint64_t i = first; i - lane * 4 < n; i += stride * kScatterGroups) {
    uint32_t k[kScatterGroups][4], v[kScatterGroups][4], pos[kScatterGroups][4], bin[kScatterGroups][4];
#pragma unroll
    for (int g = 0; g < kScatterGroups; ++g) {
      const uint4 k4 = load_group(keys, i + g * stride, n, aligned);
      const uint4 v4 = load_group(values, i + g * stride, n, aligned);
      k[g][0] = k4.x, k[g][1] = k4.y, k[g][2] = k4.z, k[g][3] = k4.w;
      v[g][0] = v4.x, v[g][1] = v4.y, v[g][2] = v4.z, v[g][3] = v4.w;
    }
#pragma unroll
    for (int g = 0; g < kScatterGroups; ++g) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bin[g][j] = bucket_index(h0, k[g][j]) >> kBinLog2;
        pos[g][j] = 0;
        if (i + g * stride + j < n) pos[g][j] = atomicAdd(&bin_cursor[static_cast<size_t>(bin[g][j]) << cursor_shift], 1u);
      }
    }
#pragma unroll
    for (int g = 0; g < kScatterGroups; ++g) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool in = i + g * stride + j < n;
        const bool fits = in && pos[g][j] < cap;
        const uint2 kv = make_uint2(k[g][j], v[g][j]);
        if (fits) bins[static_cast<uint64_t>(bin[g][j]) * cap + pos[g][j]] = kv;
        spill_append(in && !fits, kv, spill, spill_cursor, lane);
      }
    }
  }
}

// ---- K11 ------------------------------------------------------------------------------------------------------
// Per-warp shared memory: 32 * B slots of the bin, then the stash.
template <int B>
__global__ void __launch_bounds__(kBuildBlock)
bin_build_kernel(const __grid_constant__ TableView t, uint32_t n_bins, uint32_t cap, uint32_t cursor_shift,
                 const uint32_t* __restrict__ bin_cursor,
                 const uint2* __restrict__ bins, int fresh, uint2* __restrict__ spill,
                 unsigned long long* __restrict__ spill_cursor, DevCounters* __restrict__ ctr) {
  constexpr uint32_t kBinSlots = 32u * B;
  constexpr uint32_t kWarpSlots = kBinSlots + kStashPairs;
  extern __shared__ __align__(16) unsigned long long sm_slots[];
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  unsigned long long* rows = sm_slots + (threadIdx.x >> 5) * kWarpSlots;
  unsigned long long* stash = rows + kBinSlots;
  uint32_t stashed = 0;  // warp-uniform
  uint32_t n_ins = 0;
  const uint32_t n_warps = gridDim.x * kBuildWarps;

  for (uint32_t bin = blockIdx.x * kBuildWarps + (threadIdx.x >> 5); bin < n_bins; bin += n_warps) {
    const uint64_t first = static_cast<uint64_t>(bin) << kBinLog2;
    const uint32_t nb = static_cast<uint32_t>(min(static_cast<uint64_t>(32), t.num_buckets - first));
    const uint32_t n_slots = nb * B;  // even: B >= 8
    unsigned long long* gstore = reinterpret_cast<unsigned long long*>(t.store) + first * B;
    uint32_t load = 0;  // of the lane's own bucket

    // the bin's buckets into shared memory
    if (fresh) {
      const uint4 e = make_uint4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
      for (uint32_t i = lane; i < kBinSlots / 2; i += 32) reinterpret_cast<uint4*>(rows)[i] = e;
    } else {
      for (uint32_t i = lane; i < n_slots / 2; i += 32)
        reinterpret_cast<uint4*>(rows)[i] = __ldcs(reinterpret_cast<const uint4*>(gstore) + i);
      __syncwarp();
      // load = 1 + index of the last occupied slot (equals compute_load, bucket.hpp:26-31, whenever the occupied
      // slots form a prefix; never overwrites anything on an uploaded store with holes).  Slot i of the bin is
      // inspected by lane i % 32; a ballot hands the occupancy bits of each bucket to its owner lane.
#pragma unroll
      for (uint32_t base = 0; base < kBinSlots; base += 32) {
        const uint32_t i = base + lane;
        const bool occ = i < n_slots && static_cast<uint32_t>(rows[i]) != kEmptyKey;
        const uint32_t m = __ballot_sync(kFullMask, occ);
        if constexpr (B >= 32) {  // a bucket spans B / 32 ballots
          if (static_cast<uint32_t>(lane) == base / B && m != 0) load = (base % B) + 32u - __clz(m);
        } else {  // a ballot covers 32 / B buckets
          const uint32_t owner_first = base / B;
          const uint32_t sub = static_cast<uint32_t>(lane) - owner_first;
          if (sub < 32u / B) {
            const uint32_t bits = (m >> (sub * B)) & ((B >= 32) ? 0xFFFFFFFFu : ((1u << (B & 31)) - 1u));
            if (bits != 0) load = 32u - __clz(bits);
          }
        }
      }
    }
    __syncwarp();

    const uint32_t n_r = min(bin_cursor[static_cast<size_t>(bin) << cursor_shift], cap);
    const uint2* src = bins + static_cast<uint64_t>(bin) * cap;
    constexpr int U = 4;
    for (uint32_t i0 = 0; i0 < n_r; i0 += 32 * U) {
      uint2 kv[U];
      bool in[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        in[u] = i < n_r;
        kv[u] = make_uint2(0u, 0u);
        if (in[u]) kv[u] = __ldcs(src + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i0 + u * 32 >= n_r) break;  // warp-uniform
        const uint32_t lb = (bucket_index(t.h[0], kv[u].x) - static_cast<uint32_t>(first)) & 31u;
        // peers = lanes whose pair goes to the same bucket as mine; mine = lanes whose pair goes to MY bucket
        uint32_t peers = __ballot_sync(kFullMask, in[u]);
        uint32_t mine = peers;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const uint32_t mk = __ballot_sync(kFullMask, (lb >> k) & 1u);
          peers &= ((lb >> k) & 1u) ? mk : ~mk;
          mine &= ((lane >> k) & 1) ? mk : ~mk;
        }
        const uint32_t slot = __shfl_sync(kFullMask, load, lb) + __popc(peers & lt_mask);
        load += __popc(mine);
        const bool placed = in[u] && slot < B;
        if (placed) {
          rows[lb * B + slot] = pack_pair(kv[u].x, kv[u].y);
          ++n_ins;
        }
        // spilled pairs: into the stash, flushed 32+ at a time
        const uint32_t sm = __ballot_sync(kFullMask, in[u] && !placed);
        if (sm != 0) {
          if (in[u] && !placed) stash[stashed + __popc(sm & lt_mask)] = pack_pair(kv[u].x, kv[u].y);
          stashed += __popc(sm);
          if (stashed >= 32) {
            __syncwarp();
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(spill_cursor, static_cast<unsigned long long>(stashed));
            base = __shfl_sync(kFullMask, base, 0);
            unsigned long long* out = reinterpret_cast<unsigned long long*>(spill) + base;
            out[lane] = stash[lane];
            if (lane + 32u < stashed) out[lane + 32] = stash[lane + 32];
            stashed = 0;
            __syncwarp();
          }
        }
      }
    }
    __syncwarp();

    // the bin back to the store, coalesced
    for (uint32_t i = lane; i < n_slots / 2; i += 32)
      reinterpret_cast<uint4*>(gstore)[i] = reinterpret_cast<const uint4*>(rows)[i];
    __syncwarp();
  }

  if (stashed != 0) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(spill_cursor, static_cast<unsigned long long>(stashed));
    base = __shfl_sync(kFullMask, base, 0);
    unsigned long long* out = reinterpret_cast<unsigned long long*>(spill) + base;
    if (static_cast<uint32_t>(lane) < stashed) out[lane] = stash[lane];
    if (lane + 32u < stashed) out[lane + 32] = stash[lane + 32];
  }
  flush_insert_counters(ctr, lane, n_ins, 0u, n_ins);
}

template <int B>
cudaError_t launch_bin_build(const TableView& t, const BlockedPlan& p, const uint32_t* bin_cursor, const uint2* bins, bool fresh,
                             uint2* spill, unsigned long long* spill_cursor, DevCounters* ctr, int sm_count, cudaStream_t stream) {
  auto kernel = bin_build_kernel<B>;
  const int smem = kBuildWarps * (32 * B + kStashPairs) * 8;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = persistent_grid(kernel, kBuildBlock, smem, sm_count, p.n_regions, kBuildWarps);
  kernel<<<grid, kBuildBlock, smem, stream>>>(t, p.n_regions, p.cap, p.cursor_shift, bin_cursor, bins, fresh ? 1 : 0, spill, spill_cursor, ctr);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

// Geometry of a blocked build of n pairs into table t; n_regions == 0: not applicable.
BlockedPlan plan_blocked_build(const TableView& t, uint64_t n) {
  BlockedPlan p{};
  if (t.bucket_size != 8 && t.bucket_size != 16 && t.bucket_size != 32) return p;
  if (n == 0 || n > 0xFFFFFFFFull) return p;
  const uint64_t bins = (t.num_buckets + 31) >> kBinLog2;
  const double mean = static_cast<double>(n) * 32.0 / static_cast<double>(t.num_buckets);
  double cap = mean + 6.0 * std::sqrt(mean) + 32.0;
  if (cap > static_cast<double>(n)) cap = static_cast<double>(n);
  p.cap = (static_cast<uint32_t>(cap) + 2u) & ~1u;  // even: every bin starts 16-byte aligned
  p.n_regions = static_cast<uint32_t>(bins);
  p.region_log2 = kBinLog2;
  p.b_log2 = t.bucket_size == 8 ? 3 : (t.bucket_size == 16 ? 4 : 5);
  // Spacing of the bin cursors (4 << shift bytes).  Measured: no effect (1.12 ms for 50 M pairs at 4, 32 and 128
  // bytes) — the L2 is limited by the number of sub-sector read-modify-writes, not by which line they hit.
  p.cursor_shift = 0;
  if (const char* e = std::getenv("BHT_CURSOR_SHIFT")) p.cursor_shift = static_cast<uint32_t>(std::atoi(e)) & 7u;
  return p;
}

size_t blocked_scratch_bytes(const BlockedPlan& p, uint64_t n) {
  return static_cast<size_t>(p.n_regions) * p.cap * 8 + n * 8 + 16 + ((static_cast<size_t>(p.n_regions) * 4) << p.cursor_shift) + 16;
}

// scratch layout: bins | spill | spill_cursor (8) pad (8) | bin_cursor
cudaError_t launch_blocked_build(const TableView& t, const BlockedPlan& p, const uint32_t* keys, const uint32_t* values,
                                 uint64_t n, bool fresh, void* scratch, DevCounters* ctr, int sm_count, cudaStream_t stream,
                                 const uint2** spill_out, const unsigned long long** spill_count_out) {
  unsigned char* s = static_cast<unsigned char*>(scratch);
  uint2* bins = reinterpret_cast<uint2*>(s);
  uint2* spill = bins + static_cast<size_t>(p.n_regions) * p.cap;
  unsigned long long* spill_cursor = reinterpret_cast<unsigned long long*>(spill + n);
  uint32_t* bin_cursor = reinterpret_cast<uint32_t*>(spill_cursor + 2);
  cudaError_t e = cudaMemsetAsync(spill_cursor, 0, 16 + ((static_cast<size_t>(p.n_regions) * 4) << p.cursor_shift), stream);
  if (e != cudaSuccess) return e;

  const bool aligned = (reinterpret_cast<uintptr_t>(keys) % 16 == 0) && (reinterpret_cast<uintptr_t>(values) % 16 == 0);
  const int grid_a = persistent_grid(bin_scatter_kernel, kScatterBlock, 0, sm_count, n, kScatterBlock * 4 * kScatterGroups);
  bin_scatter_kernel<<<grid_a, kScatterBlock, 0, stream>>>(t.h[0], p.cap, p.cursor_shift, keys, values, n, aligned, bin_cursor, bins, spill,
                                                          spill_cursor);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  switch (t.bucket_size) {
    case 8: e = launch_bin_build<8>(t, p, bin_cursor, bins, fresh, spill, spill_cursor, ctr, sm_count, stream); break;
    case 16: e = launch_bin_build<16>(t, p, bin_cursor, bins, fresh, spill, spill_cursor, ctr, sm_count, stream); break;
    case 32: e = launch_bin_build<32>(t, p, bin_cursor, bins, fresh, spill, spill_cursor, ctr, sm_count, stream); break;
    default: return cudaErrorInvalidValue;
  }
  *spill_out = spill;
  *spill_count_out = spill_cursor;
  return e;
}

}  // namespace bht_b200
