// util.cu — the streaming kernels around the probe path.
//
//   K0  fill_empty          hash_table ctor fill (reference: proj/src/table.cpp:30-31)
//   K7  count_occupied      occupied_slots (table.cpp:34-39)
//       count_inadmissible  check_admissibility (proj/src/oracle.cpp:40-54)
//       hash_keys           bucket_index in isolation (proj/include/bht/hash.hpp:21-23)
//   K8  shard_histogram / shard_offsets / shard_scatter   owner-shard routing (no reference counterpart)
//   K9  unpermute           answers back into query order
//       generate_keys       unique sentinel-free keys from a counter (keygen.cpp:50-64 contract)
//
// All are HBM-streaming kernels: 16-byte accesses, grid = a multiple of the SM count, grid-stride.
#include "kernels.h"

#include <atomic>

namespace bht_b200 {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

constexpr int kStreamBlock = 256;

static inline int stream_grid(int sm_count, uint64_t items, uint64_t items_per_block, int ctas_per_sm = 8) {
  uint64_t need = (items + items_per_block - 1) / items_per_block;
  if (need < 1) need = 1;
  const uint64_t fill = static_cast<uint64_t>(sm_count) * ctas_per_sm;
  return static_cast<int>(need < fill ? need : fill);
}

// ---- K0 ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock) fill_empty_kernel(uint64_t* __restrict__ store, uint64_t n_slots) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n2 = n_slots >> 1;
  ulonglong2* v = reinterpret_cast<ulonglong2*>(store);  // the store is 256-byte aligned
  const ulonglong2 e = make_ulonglong2(kEmptySlot, kEmptySlot);
  for (uint64_t i = tid; i < n2; i += stride) v[i] = e;
  if (tid == 0 && (n_slots & 1)) store[n_slots - 1] = kEmptySlot;
}

cudaError_t launch_fill_empty(uint64_t* store, uint64_t n_slots, int sm_count, cudaStream_t stream) {
  if (n_slots == 0) return cudaSuccess;
  fill_empty_kernel<<<stream_grid(sm_count, n_slots, kStreamBlock * 8), kStreamBlock, 0, stream>>>(store, n_slots);
  note_launch();
  return cudaGetLastError();
}

// ---- K7 ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock)
count_occupied_kernel(const uint64_t* __restrict__ store, uint64_t n_slots, unsigned long long* __restrict__ out) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n2 = n_slots >> 1;
  const uint4* v = reinterpret_cast<const uint4*>(store);
  unsigned long long c = 0;
  for (uint64_t i = tid; i < n2; i += stride) {
    const uint4 s = __ldcs(v + i);
    c += (s.x != kEmptyKey) + (s.z != kEmptyKey);  // key = low half of each slot (core.hpp:35-41)
  }
  if (tid == 0 && (n_slots & 1)) c += static_cast<uint32_t>(store[n_slots - 1]) != kEmptyKey;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_occupied(const uint64_t* store, uint64_t n_slots, unsigned long long* out, int sm_count,
                                  cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess || n_slots == 0) return e;
  count_occupied_kernel<<<stream_grid(sm_count, n_slots, kStreamBlock * 8), kStreamBlock, 0, stream>>>(store, n_slots,
                                                                                                      out);
  note_launch();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kStreamBlock)
count_inadmissible_kernel(const __grid_constant__ TableView t, unsigned long long* __restrict__ out) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n_slots = t.num_buckets * t.bucket_size;
  const uint32_t shift = __ffs(t.bucket_size) - 1;  // b is a power of two (core.cpp:42-43)
  unsigned long long c = 0;
  for (uint64_t i = tid; i < n_slots; i += stride) {
    const uint64_t s = __ldcs(t.store + i);
    const uint32_t key = static_cast<uint32_t>(s);
    if (key == kEmptyKey) continue;
    const uint32_t bucket = static_cast<uint32_t>(i >> shift);
    bool ok = false;
    for (uint32_t j = 0; j < t.n_hashes; ++j) ok |= bucket_index(t.h[j], key) == bucket;
    c += !ok;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_count_inadmissible(const TableView& t, unsigned long long* out, int sm_count, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  const uint64_t n_slots = t.num_buckets * t.bucket_size;
  count_inadmissible_kernel<<<stream_grid(sm_count, n_slots, kStreamBlock * 4), kStreamBlock, 0, stream>>>(t, out);
  note_launch();
  return cudaGetLastError();
}

// ---- hash stage hook ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock)
hash_keys_kernel(const __grid_constant__ HashFn h, const uint32_t* __restrict__ keys, uint32_t* __restrict__ out,
                 uint64_t n) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = tid; i < n; i += stride) out[i] = bucket_index(h, keys[i]);
}

cudaError_t launch_hash_keys(const HashFn& h, const uint32_t* keys, uint32_t* out, uint64_t n, int sm_count,
                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  hash_keys_kernel<<<stream_grid(sm_count, n, kStreamBlock * 4), kStreamBlock, 0, stream>>>(h, keys, out, n);
  note_launch();
  return cudaGetLastError();
}

// ---- values of a keys-only build: values[i] = value_for_key(keys[i]) (table.cpp:234) ------------------------------
__global__ void __launch_bounds__(kStreamBlock)
derive_values_kernel(const uint32_t* __restrict__ keys, uint32_t* __restrict__ values, uint64_t n, bool aligned) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = tid * 4; i < n; i += stride * 4) {
    if (aligned && i + 4 <= n) {
      const uint4 k = *reinterpret_cast<const uint4*>(keys + i);
      *reinterpret_cast<uint4*>(values + i) = make_uint4(value_for_key(k.x), value_for_key(k.y), value_for_key(k.z), value_for_key(k.w));
    } else {
      for (uint64_t j = i; j < n && j < i + 4; ++j) values[j] = value_for_key(keys[j]);
    }
  }
}

cudaError_t launch_derive_values(const uint32_t* keys, uint32_t* values, uint64_t n, int sm_count, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;
  derive_values_kernel<<<stream_grid(sm_count, n, kStreamBlock * 4), kStreamBlock, 0, stream>>>(keys, values, n, aligned);
  note_launch();
  return cudaGetLastError();
}

// ---- K8: routing by owner shard (multi-GPU) or by table region (L2-blocked build) ------------------
// Pass 1 hashes every key once: it writes the destination of each key as one byte (dest8, n bytes of scratch)
// and builds the per-destination histogram in per-thread private shared-memory counters (no atomics, no bank
// conflicts).  A one-CTA scan turns the histogram into cursors.  Pass 2 handles tiles of kTile elements: every
// element is ranked inside its tile with a shared-memory atomic, the tile reserves one contiguous range per
// destination with a single global atomic, the elements are grouped by destination in shared memory and written
// out run by run, so consecutive threads write consecutive addresses (a direct scatter would touch about one
// sector per element).  Order inside a destination is arbitrary; out_index carries the way back.  Output:
// packed {key, value} pairs (the input format of the L2-blocked insert) or separate arrays.
// Keys / values / dest8 are read with 16-byte (4-byte for dest8) loads: the arrays must be 16-byte aligned
// (cudaMalloc'ed or torch tensors; the launchers fall back to element loads otherwise).
constexpr int kGroupsPerThread = 2;                   // groups of 4 consecutive elements
constexpr int kTile = kStreamBlock * kGroupsPerThread * 4;  // 2048

struct ShardRouter {  // owner(k) = (g(k) * G) >> 32
  uint32_t alpha, beta, n;
  __device__ __forceinline__ uint32_t operator()(uint32_t key) const { return shard_of(alpha, beta, n, key); }
};
struct RegionRouter {  // region of the key's FIRST bucket: floor(h0(k) * R / m), monotone in the bucket index
  HashFn h0;
  uint32_t mult;  // floor(R * 2^32 / m)
  __device__ __forceinline__ uint32_t operator()(uint32_t key) const {
    return static_cast<uint32_t>((static_cast<uint64_t>(bucket_index(h0, key)) * mult) >> 32);
  }
};

__device__ __forceinline__ uint4 load4(const uint32_t* p, uint64_t i, uint64_t n, bool aligned) {
  if (aligned && i + 4 <= n) return __ldcs(reinterpret_cast<const uint4*>(p + i));
  uint4 r = make_uint4(0, 0, 0, 0);
  if (i < n) r.x = __ldcs(p + i);
  if (i + 1 < n) r.y = __ldcs(p + i + 1);
  if (i + 2 < n) r.z = __ldcs(p + i + 2);
  if (i + 3 < n) r.w = __ldcs(p + i + 3);
  return r;
}

// PRIVATE: hist = n_dest rows of kStreamBlock counters, row-major: thread t owns column t (bank t % 32), plain
// read-modify-write.  Otherwise (many destinations): one shared row of n_dest counters, shared-memory atomics.
template <typename Router, bool PRIVATE>
__global__ void __launch_bounds__(kStreamBlock)
route_classify_kernel(const __grid_constant__ Router route, uint32_t n_dest, const uint32_t* __restrict__ keys, uint64_t n,
                      bool aligned, uint8_t* __restrict__ dest8, unsigned long long* __restrict__ counts) {
  extern __shared__ uint32_t hist_private[];
  constexpr uint32_t kRow = PRIVATE ? kStreamBlock : 1;
  for (uint32_t i = threadIdx.x; i < n_dest * kRow; i += kStreamBlock) hist_private[i] = 0;
  __syncthreads();
  uint32_t* mine = hist_private + (PRIVATE ? threadIdx.x : 0);
  auto bump = [&](uint32_t d) {
    if constexpr (PRIVATE) mine[d * kRow] += 1;
    else atomicAdd(&mine[d], 1u);
  };
  const uint64_t groups = (n + 3) >> 2;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < groups; g += stride) {
    const uint64_t i = g << 2;
    const uint4 k = load4(keys, i, n, aligned);
    const uint32_t d0 = route(k.x), d1 = route(k.y), d2 = route(k.z), d3 = route(k.w);
    if (i + 4 <= n) {
      *reinterpret_cast<uint32_t*>(dest8 + i) = d0 | (d1 << 8) | (d2 << 16) | (d3 << 24);  // dest8 is 4-byte aligned
      bump(d0);
      bump(d1);
      bump(d2);
      bump(d3);
    } else {
      const uint32_t d[4] = {d0, d1, d2, d3};
      for (uint32_t j = 0; i + j < n; ++j) {
        dest8[i + j] = static_cast<uint8_t>(d[j]);
        bump(d[j]);
      }
    }
  }
  __syncthreads();
  if constexpr (PRIVATE) {  // column sums: warp w reduces rows w, w + 8, ...
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t s = warp; s < n_dest; s += kStreamBlock / 32) {
      unsigned long long c = 0;
      for (int j = lane; j < kStreamBlock; j += 32) c += hist_private[s * kStreamBlock + j];
      c = warp_sum(c);
      if (lane == 0 && c) atomicAdd(&counts[s], c);
    }
  } else {
    for (uint32_t s = threadIdx.x; s < n_dest; s += kStreamBlock)
      if (hist_private[s]) atomicAdd(&counts[s], static_cast<unsigned long long>(hist_private[s]));
  }
}

__global__ void route_offsets_kernel(uint32_t n_dest, const unsigned long long* __restrict__ counts,
                                     unsigned long long* __restrict__ cursors) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long run = 0;
    for (uint32_t s = 0; s < n_dest; ++s) {
      cursors[s] = run;
      run += counts[s];
    }
  }
}

template <bool PACKED, bool INDEX>
__global__ void __launch_bounds__(kStreamBlock)
route_scatter_kernel(uint32_t n_dest, const uint32_t* __restrict__ keys, const uint32_t* __restrict__ values,
                     const uint8_t* __restrict__ dest8, uint64_t n, bool aligned, unsigned long long* __restrict__ cursors,
                     uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_values, uint32_t* __restrict__ out_index) {
  __shared__ uint2 s_pair[kTile];       // {key, value} grouped by destination
  __shared__ uint8_t s_dest[kTile];
  __shared__ uint32_t s_index[INDEX ? kTile : 1];
  __shared__ uint32_t hist[kMaxShards];       // elements of this tile per destination
  __shared__ uint32_t tile_off[kMaxShards];   // exclusive scan of hist
  __shared__ unsigned long long base_of[kMaxShards];
  __shared__ uint32_t warp_tot[kStreamBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n_tiles = (n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    for (uint32_t s = threadIdx.x; s < n_dest; s += blockDim.x) hist[s] = 0;
    __syncthreads();
    const uint64_t base = tile * kTile;
    uint4 key[kGroupsPerThread], val[kGroupsPerThread];
    uint32_t dst[kGroupsPerThread];
#pragma unroll
    for (int j = 0; j < kGroupsPerThread; ++j) {
      const uint64_t i = base + (static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x) * 4;
      key[j] = load4(keys, i, n, aligned);
      val[j] = values != nullptr ? load4(values, i, n, aligned) : make_uint4(0, 0, 0, 0);
      dst[j] = 0;
      if (i + 4 <= n) {
        dst[j] = __ldcs(reinterpret_cast<const uint32_t*>(dest8 + i));
      } else {
        for (uint32_t e = 0; i + e < n; ++e) dst[j] |= static_cast<uint32_t>(dest8[i + e]) << (8 * e);
      }
    }
    uint32_t rank[kGroupsPerThread][4];
#pragma unroll
    for (int j = 0; j < kGroupsPerThread; ++j) {
      const uint64_t i = base + (static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (i + e < n) rank[j][e] = atomicAdd(&hist[(dst[j] >> (8 * e)) & 0xFFu], 1u);
    }
    __syncthreads();
    // exclusive scan of hist (n_dest <= 256 = one element per thread) + one global reservation per destination
    {
      const uint32_t h = threadIdx.x < n_dest ? hist[threadIdx.x] : 0u;
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) warp_tot[warp] = x;
      __syncthreads();
      uint32_t before = 0;
#pragma unroll
      for (int w = 0; w < kStreamBlock / 32; ++w) before += w < warp ? warp_tot[w] : 0u;
      if (threadIdx.x < n_dest) {
        tile_off[threadIdx.x] = before + x - h;
        base_of[threadIdx.x] = h ? atomicAdd(&cursors[threadIdx.x], static_cast<unsigned long long>(h)) : 0ull;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kGroupsPerThread; ++j) {
      const uint64_t i = base + (static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x) * 4;
      const uint32_t k4[4] = {key[j].x, key[j].y, key[j].z, key[j].w};
      const uint32_t v4[4] = {val[j].x, val[j].y, val[j].z, val[j].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (i + e < n) {
          const uint32_t d = (dst[j] >> (8 * e)) & 0xFFu;
          const uint32_t slot = tile_off[d] + rank[j][e];
          s_pair[slot] = make_uint2(k4[e], v4[e]);
          s_dest[slot] = static_cast<uint8_t>(d);
          if constexpr (INDEX) s_index[slot] = static_cast<uint32_t>(i + e);
        }
      }
    }
    __syncthreads();
    const uint32_t in_tile = static_cast<uint32_t>(n - base < kTile ? n - base : kTile);
#pragma unroll
    for (int j = 0; j < kGroupsPerThread * 4; ++j) {
      const uint32_t slot = j * kStreamBlock + threadIdx.x;
      if (slot < in_tile) {
        const uint32_t d = s_dest[slot];
        const unsigned long long pos = base_of[d] + (slot - tile_off[d]);
        const uint2 kv = s_pair[slot];
        if constexpr (PACKED) {
          __stcs(reinterpret_cast<uint2*>(out_keys) + pos, kv);
        } else {
          out_keys[pos] = kv.x;
          if (out_values != nullptr) out_values[pos] = kv.y;
        }
        if constexpr (INDEX) out_index[pos] = s_index[slot];
      }
    }
    __syncthreads();
  }
}

// scratch8: n bytes (4-byte aligned) for the per-key destinations.
template <typename Router, bool PACKED, bool INDEX>
static cudaError_t route(const Router& r, uint32_t n_dest, const uint32_t* keys, const uint32_t* values, uint64_t n,
                         uint8_t* scratch8, unsigned long long* counts, unsigned long long* cursors, uint32_t* out_keys,
                         uint32_t* out_values, uint32_t* out_index, int sm_count, cudaStream_t stream) {
  if (n_dest == 0 || n_dest > static_cast<uint32_t>(kMaxShards)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * n_dest, stream);
  if (e != cudaSuccess) return e;
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(values)) & 15) == 0;
  if (n != 0) {
    const bool priv = n_dest <= 48;  // 1 KiB of private counters per destination: <= 48 KiB, >= 4 CTAs per SM
    auto kernel = priv ? route_classify_kernel<Router, true> : route_classify_kernel<Router, false>;
    const int smem = static_cast<int>(n_dest * (priv ? kStreamBlock : 1) * sizeof(uint32_t));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kStreamBlock, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
    kernel<<<stream_grid(sm_count, n, kStreamBlock * 16, per_sm), kStreamBlock, smem, stream>>>(r, n_dest, keys, n, aligned, scratch8,
                                                                                              counts);
    note_launch();
  }
  route_offsets_kernel<<<1, 32, 0, stream>>>(n_dest, counts, cursors);
  note_launch();
  if (n != 0) {
    route_scatter_kernel<PACKED, INDEX><<<stream_grid(sm_count, n, kTile, 8), kStreamBlock, 0, stream>>>(
        n_dest, keys, values, scratch8, n, aligned, cursors, out_keys, out_values, out_index);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_shard_route(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys, const uint32_t* values,
                               uint64_t n, uint8_t* scratch8, unsigned long long* counts, unsigned long long* cursors,
                               uint32_t* out_keys, uint32_t* out_values, uint32_t* out_index, int sm_count, cudaStream_t stream) {
  const ShardRouter r{alpha, beta, n_shards};
  if (out_index != nullptr)
    return route<ShardRouter, false, true>(r, n_shards, keys, values, n, scratch8, counts, cursors, out_keys, out_values,
                                           out_index, sm_count, stream);
  return route<ShardRouter, false, false>(r, n_shards, keys, values, n, scratch8, counts, cursors, out_keys, out_values, nullptr,
                                          sm_count, stream);
}

cudaError_t launch_region_route(const HashFn& h0, uint32_t n_regions, const uint32_t* keys, const uint32_t* values, uint64_t n,
                                uint8_t* scratch8, unsigned long long* counts, unsigned long long* cursors, uint32_t* out_pairs,
                                int sm_count, cudaStream_t stream) {
  RegionRouter r;
  r.h0 = h0;
  r.mult = static_cast<uint32_t>((static_cast<uint64_t>(n_regions) << 32) / h0.range);  // n_regions < range
  return route<RegionRouter, true, false>(r, n_regions, keys, values, n, scratch8, counts, cursors, out_pairs, nullptr, nullptr,
                                          sm_count, stream);
}

// ---- K9 ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock)
unpermute_kernel(const uint32_t* __restrict__ answers, const uint32_t* __restrict__ index, uint64_t n,
                 uint32_t* __restrict__ out) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = tid; i < n; i += stride) {
    const uint32_t at = __ldcs(index + i);
    if (at != 0xFFFFFFFFu) out[at] = __ldcs(answers + i);  // 0xFFFFFFFF: a padding slot of a fixed-segment exchange
  }
}

cudaError_t launch_unpermute(const uint32_t* answers, const uint32_t* index, uint64_t n, uint32_t* out, int sm_count,
                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  unpermute_kernel<<<stream_grid(sm_count, n, kStreamBlock * 4), kStreamBlock, 0, stream>>>(answers, index, n, out);
  note_launch();
  return cudaGetLastError();
}

// ---- synthetic keys ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock)
generate_keys_kernel(uint64_t seed, uint64_t offset, uint64_t n, uint32_t* __restrict__ keys,
                     uint32_t* __restrict__ values) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (uint64_t i = tid; i < n; i += stride) {
    const uint32_t key = unique_key(k0, k1, static_cast<uint32_t>(offset + i));
    keys[i] = key;
    if (values != nullptr) values[i] = synthetic_value(k1, key);
  }
}

cudaError_t launch_generate_keys(uint64_t seed, uint64_t offset, uint64_t n, uint32_t* keys, uint32_t* values,
                                 int sm_count, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  generate_keys_kernel<<<stream_grid(sm_count, n, kStreamBlock * 4), kStreamBlock, 0, stream>>>(seed, offset, n, keys,
                                                                                               values);
  note_launch();
  return cudaGetLastError();
}

}  // namespace bht_b200
