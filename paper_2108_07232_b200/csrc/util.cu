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

// ---- K8: owner-shard routing -------------------------------------------------------------------
// One CTA handles tiles of kTile keys.  Pass 1 builds the per-shard histogram; a one-CTA scan turns it
// into cursors; pass 2 ranks every key inside its CTA tile with shared-memory atomics, reserves one
// contiguous range per (tile, shard) with a single global atomic, and writes keys / values / origin
// index.  Order inside a shard is arbitrary; out_index carries the way back.
constexpr int kKeysPerThread = 8;
constexpr int kTile = kStreamBlock * kKeysPerThread;

__global__ void __launch_bounds__(kStreamBlock)
shard_histogram_kernel(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* __restrict__ keys, uint64_t n,
                       unsigned long long* __restrict__ counts) {
  __shared__ uint32_t hist[kMaxShards];
  for (uint32_t s = threadIdx.x; s < n_shards; s += blockDim.x) hist[s] = 0;
  __syncthreads();
  const uint64_t n_tiles = (n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t base = tile * kTile;
#pragma unroll
    for (int j = 0; j < kKeysPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x;
      if (i < n) atomicAdd(&hist[shard_of(alpha, beta, n_shards, __ldcs(keys + i))], 1u);
    }
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < n_shards; s += blockDim.x)
    if (hist[s]) atomicAdd(&counts[s], static_cast<unsigned long long>(hist[s]));
}

__global__ void shard_offsets_kernel(uint32_t n_shards, const unsigned long long* __restrict__ counts,
                                     unsigned long long* __restrict__ cursors) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long run = 0;
    for (uint32_t s = 0; s < n_shards; ++s) {
      cursors[s] = run;
      run += counts[s];
    }
  }
}

__global__ void __launch_bounds__(kStreamBlock)
shard_scatter_kernel(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* __restrict__ keys,
                     const uint32_t* __restrict__ values, uint64_t n, unsigned long long* __restrict__ cursors,
                     uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_values,
                     uint32_t* __restrict__ out_index) {
  __shared__ uint32_t hist[kMaxShards];
  __shared__ unsigned long long base_of[kMaxShards];
  const uint64_t n_tiles = (n + kTile - 1) / kTile;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    for (uint32_t s = threadIdx.x; s < n_shards; s += blockDim.x) hist[s] = 0;
    __syncthreads();
    const uint64_t base = tile * kTile;
    uint32_t key[kKeysPerThread], shard[kKeysPerThread], rank[kKeysPerThread];
#pragma unroll
    for (int j = 0; j < kKeysPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x;
      if (i < n) {
        key[j] = __ldcs(keys + i);
        shard[j] = shard_of(alpha, beta, n_shards, key[j]);
        rank[j] = atomicAdd(&hist[shard[j]], 1u);
      }
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < n_shards; s += blockDim.x)
      base_of[s] = hist[s] ? atomicAdd(&cursors[s], static_cast<unsigned long long>(hist[s])) : 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kKeysPerThread; ++j) {
      const uint64_t i = base + static_cast<uint64_t>(j) * kStreamBlock + threadIdx.x;
      if (i < n) {
        const unsigned long long pos = base_of[shard[j]] + rank[j];
        out_keys[pos] = key[j];
        if (values != nullptr) out_values[pos] = __ldcs(values + i);
        if (out_index != nullptr) out_index[pos] = static_cast<uint32_t>(i);
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_shard_histogram(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys, uint64_t n,
                                   unsigned long long* counts, int sm_count, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * n_shards, stream);
  if (e != cudaSuccess || n == 0) return e;
  shard_histogram_kernel<<<stream_grid(sm_count, n, kTile), kStreamBlock, 0, stream>>>(alpha, beta, n_shards, keys, n,
                                                                                       counts);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_scatter(uint32_t alpha, uint32_t beta, uint32_t n_shards, const uint32_t* keys,
                                 const uint32_t* values, uint64_t n, const unsigned long long* counts,
                                 unsigned long long* cursors, uint32_t* out_keys, uint32_t* out_values,
                                 uint32_t* out_index, int sm_count, cudaStream_t stream) {
  shard_offsets_kernel<<<1, 32, 0, stream>>>(n_shards, counts, cursors);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || n == 0) return e;
  shard_scatter_kernel<<<stream_grid(sm_count, n, kTile), kStreamBlock, 0, stream>>>(
      alpha, beta, n_shards, keys, values, n, cursors, out_keys, out_values, out_index);
  note_launch();
  return cudaGetLastError();
}

// ---- K9 ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kStreamBlock)
unpermute_kernel(const uint32_t* __restrict__ answers, const uint32_t* __restrict__ index, uint64_t n,
                 uint32_t* __restrict__ out) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = tid; i < n; i += stride) out[__ldcs(index + i)] = __ldcs(answers + i);
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
