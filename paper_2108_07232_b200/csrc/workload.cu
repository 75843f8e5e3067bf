// workload.cu — the reference's synthetic workload, bit-exact, with the set operations on the GPU.
//
// Replaces generate_keys / generate_queries / save_keys / load_keys (reference: proj/src/keygen.cpp:50-125).
// The reference draws from ONE std::mt19937_64 stream per call and keeps "seen" / "member" sets in
// std::unordered_set; the sets are what makes it slow (44 s for 50 M keys).  Here
//   * the engine stays on the host — it is a sequential generator by definition and 50 M draws take ~0.2 s —
//     and runs in batches whose state is rewound to the exact draw the reference would have stopped at;
//   * "first occurrence wins" de-duplication of generate_keys is a device hash set of (key, stream index) with
//     atomicMin on the index, followed by an order-preserving compaction (count / scan / scatter);
//   * the membership rejection of generate_queries' negatives is a bulk find on a device table built from the key
//     set with this library's own bulk build;
//   * the two Fisher-Yates passes (partial shuffle of the positives, final shuffle) are data-dependent sequential
//     swaps and stay on the host.
// Outputs equal the reference's element for element (tests/test_gpu_workload.py against oracle/_ref, and the
// golden fixtures of tests/golden on the CPU side for the host pieces).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "../../include/bht_b200.h"
#include "kernels.h"

using namespace bht_b200;

namespace bht_b200 {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

constexpr unsigned long long kNoEntry = ~0ull;
constexpr int kBlock = 256;
constexpr int kItems = 4;  // consecutive candidates per thread in the compaction kernels
constexpr int kTile = kBlock * kItems;

__device__ __forceinline__ uint32_t scramble(uint32_t k) {
  k ^= k >> 16;
  k *= 0x85EBCA6Bu;
  k ^= k >> 13;
  k *= 0xC2B2AE35u;
  k ^= k >> 16;
  return k;
}

// Device set of (key, smallest stream index at which the key was drawn): open addressing, linear probing, one
// 64-bit word per entry = key << 32 | index, so atomicMin on the word keeps the first occurrence of a key.
__global__ void __launch_bounds__(kBlock)
first_seen_insert_kernel(const uint32_t* __restrict__ cand, uint64_t m, uint32_t base_index,
                         unsigned long long* __restrict__ slots, uint32_t mask) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; i < m; i += stride) {
    const uint32_t k = cand[i];
    if (k == kEmptyKey) continue;  // the sentinel is skipped, never stored (keygen.cpp:58)
    const unsigned long long entry = (static_cast<unsigned long long>(k) << 32) | (base_index + static_cast<uint32_t>(i));
    uint32_t s = scramble(k) & mask;
    for (;;) {
      unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(slots + s);
      if (cur == kNoEntry) {
        cur = atomicCAS(slots + s, kNoEntry, entry);
        if (cur == kNoEntry) break;
      }
      if (static_cast<uint32_t>(cur >> 32) == k) {
        atomicMin(slots + s, entry);
        break;
      }
      s = (s + 1) & mask;
    }
  }
}

__global__ void __launch_bounds__(kBlock)
first_seen_flag_kernel(const uint32_t* __restrict__ cand, uint64_t m, uint32_t base_index,
                       const unsigned long long* __restrict__ slots, uint32_t mask, uint8_t* __restrict__ keep) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kBlock;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x; i < m; i += stride) {
    const uint32_t k = cand[i];
    uint8_t first = 0;
    if (k != kEmptyKey) {
      uint32_t s = scramble(k) & mask;
      for (;;) {
        const unsigned long long cur = slots[s];
        if (static_cast<uint32_t>(cur >> 32) == k || cur == kNoEntry) {
          first = static_cast<uint32_t>(cur) == base_index + static_cast<uint32_t>(i);
          break;
        }
        s = (s + 1) & mask;
      }
    }
    keep[i] = first;
  }
}

// Order-preserving compaction of the kept candidates: per-tile counts, one-CTA scan, scatter.
__device__ __forceinline__ uint32_t tile_flags(const uint8_t* __restrict__ keep, uint64_t m, uint64_t first) {
  uint32_t f = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (first + j < m && keep[first + j]) f |= 1u << j;
  return f;
}

__global__ void __launch_bounds__(kBlock)
compact_count_kernel(const uint8_t* __restrict__ keep, uint64_t m, unsigned long long* __restrict__ tile_counts) {
  __shared__ uint32_t warp_sums[kBlock / 32];
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kTile + threadIdx.x * kItems;
  uint32_t c = __popc(tile_flags(keep, m, first));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFullMask, c, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kBlock / 32; ++w) t += warp_sums[w];
    tile_counts[blockIdx.x] = t;
  }
}

// tile_counts -> exclusive offsets in place; tile_counts[n_tiles] = total.
__global__ void __launch_bounds__(1024) compact_scan_kernel(unsigned long long* __restrict__ tile_counts, uint64_t n_tiles) {
  __shared__ unsigned long long partial[1024];
  const uint64_t per = (n_tiles + 1023) / 1024;
  const uint64_t lo = min(n_tiles, threadIdx.x * per), hi = min(n_tiles, lo + per);
  unsigned long long sum = 0;
  for (uint64_t i = lo; i < hi; ++i) sum += tile_counts[i];
  partial[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int i = 0; i < 1024; ++i) {
      const unsigned long long v = partial[i];
      partial[i] = run;
      run += v;
    }
    tile_counts[n_tiles] = run;
  }
  __syncthreads();
  unsigned long long run = partial[threadIdx.x];
  for (uint64_t i = lo; i < hi; ++i) {
    const unsigned long long v = tile_counts[i];
    tile_counts[i] = run;
    run += v;
  }
}

// Kept candidate number r (0-based, in stream order) goes to out[r] for r < room.
__global__ void __launch_bounds__(kBlock)
compact_scatter_kernel(const uint32_t* __restrict__ cand, const uint8_t* __restrict__ keep, uint64_t m,
                       const unsigned long long* __restrict__ tile_offsets, uint64_t room, uint32_t* __restrict__ out) {
  __shared__ uint32_t warp_sums[kBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kTile + threadIdx.x * kItems;
  const uint32_t f = tile_flags(keep, m, first);
  const uint32_t c = __popc(f);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < warp; ++w) before += warp_sums[w];
  unsigned long long pos = tile_offsets[blockIdx.x] + before + (incl - c);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (f & (1u << j)) {
      if (pos < room) out[pos] = cand[first + j];
      ++pos;
    }
  }
}

int grid_for(uint64_t items, int per_block, int sm_count) {
  const uint64_t need = (items + per_block - 1) / per_block;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(need, static_cast<uint64_t>(sm_count) * 16)));
}

bht_status wl_fail(bht_status s, const std::string& msg) {
  set_last_error(msg);
  return s;
}
bht_status wl_cuda(cudaError_t e, const char* what) {
  set_last_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return BHT_CUDA_ERROR;
}
#define WL_CUDA(expr)                                   \
  do {                                                  \
    cudaError_t e__ = (expr);                           \
    if (e__ != cudaSuccess) {                           \
      cleanup();                                        \
      return wl_cuda(e__, #expr);                       \
    }                                                   \
  } while (0)

// Bounded uniform draw by rejection, exactly keygen.cpp:33-40.
uint64_t uniform_below(std::mt19937_64& eng, uint64_t bound) {
  const uint64_t limit = std::numeric_limits<uint64_t>::max() - std::numeric_limits<uint64_t>::max() % bound;
  uint64_t x;
  do {
    x = eng();
  } while (x >= limit);
  return x % bound;
}

}  // namespace

extern "C" {

// generate_keys (keygen.cpp:50-64): the first n distinct non-sentinel values of (eng() >> 32), in stream order.
bht_status bht_generate_keys(uint64_t seed, uint64_t n, uint32_t* out_keys, int32_t mem_space, int32_t device, void* stream_v) {
  if (n != 0 && out_keys == nullptr) return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_keys: null output");
  if (n > 0xFFFFFFFEull) return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_keys: more keys than the 32-bit universe holds");
  if (mem_space != BHT_MEM_DEVICE && mem_space != BHT_MEM_HOST) return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_keys: bad mem_space");
  if (n == 0) return BHT_OK;
  int prev_device = -1;
  cudaGetDevice(&prev_device);
  if (cudaSetDevice(device) != cudaSuccess) return wl_fail(BHT_CUDA_ERROR, "bht_generate_keys: cudaSetDevice failed");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_v);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int sms = prop.multiProcessorCount;

  // the set must hold every candidate ever drawn: duplicates are rare (n^2 / 2^33), leave slack for the top-ups
  uint64_t want_slots = 2 * (n + n / 16 + (1u << 16));
  uint64_t n_slots = 1;
  while (n_slots < want_slots) n_slots <<= 1;
  if (n_slots > (1ull << 32)) n_slots = 1ull << 32;
  const uint32_t mask = static_cast<uint32_t>(n_slots - 1);

  unsigned long long* slots = nullptr;
  uint32_t *d_cand = nullptr, *d_out = nullptr, *h_cand = nullptr;
  uint8_t* d_keep = nullptr;
  unsigned long long* d_tiles = nullptr;
  auto cleanup = [&]() {
    if (slots) cudaFree(slots);
    if (d_cand) cudaFree(d_cand);
    if (d_keep) cudaFree(d_keep);
    if (d_tiles) cudaFree(d_tiles);
    if (d_out && mem_space == BHT_MEM_HOST) cudaFree(d_out);
    if (h_cand) cudaFreeHost(h_cand);
    if (prev_device >= 0) cudaSetDevice(prev_device);
  };

  const uint64_t batch_cap = n + n / 64 + (1u << 16);
  WL_CUDA(cudaMalloc(&slots, n_slots * sizeof(unsigned long long)));
  WL_CUDA(cudaMemsetAsync(slots, 0xFF, n_slots * sizeof(unsigned long long), stream));
  WL_CUDA(cudaMalloc(&d_cand, batch_cap * sizeof(uint32_t)));
  WL_CUDA(cudaMalloc(&d_keep, batch_cap));
  WL_CUDA(cudaMalloc(&d_tiles, ((batch_cap + kTile - 1) / kTile + 1) * sizeof(unsigned long long)));
  WL_CUDA(cudaMallocHost(&h_cand, batch_cap * sizeof(uint32_t)));
  if (mem_space == BHT_MEM_HOST) {
    WL_CUDA(cudaMalloc(&d_out, n * sizeof(uint32_t)));
  } else {
    d_out = out_keys;
  }

  std::mt19937_64 eng(seed);
  uint64_t accepted = 0, drawn = 0, set_entries = 0;
  while (accepted < n) {
    const uint64_t missing = n - accepted;
    const uint64_t m = std::min(batch_cap, accepted == 0 ? batch_cap : std::max<uint64_t>(2 * missing, 1u << 16));
    if (drawn + m > 0xFFFFFFFFull || set_entries + m > n_slots - (n_slots >> 3)) {
      cleanup();
      return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_keys: candidate stream outgrew the de-duplication set");
    }
    for (uint64_t i = 0; i < m; ++i) h_cand[i] = static_cast<uint32_t>(eng() >> 32);
    WL_CUDA(cudaMemcpyAsync(d_cand, h_cand, m * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    first_seen_insert_kernel<<<grid_for(m, kBlock, sms), kBlock, 0, stream>>>(d_cand, m, static_cast<uint32_t>(drawn), slots, mask);
    note_launch();
    first_seen_flag_kernel<<<grid_for(m, kBlock, sms), kBlock, 0, stream>>>(d_cand, m, static_cast<uint32_t>(drawn), slots, mask, d_keep);
    note_launch();
    const uint64_t n_tiles = (m + kTile - 1) / kTile;
    compact_count_kernel<<<static_cast<unsigned>(n_tiles), kBlock, 0, stream>>>(d_keep, m, d_tiles);
    note_launch();
    compact_scan_kernel<<<1, 1024, 0, stream>>>(d_tiles, n_tiles);
    note_launch();
    compact_scatter_kernel<<<static_cast<unsigned>(n_tiles), kBlock, 0, stream>>>(d_cand, d_keep, m, d_tiles, missing, d_out + accepted);
    note_launch();
    WL_CUDA(cudaGetLastError());
    unsigned long long kept = 0;
    WL_CUDA(cudaMemcpyAsync(&kept, d_tiles + n_tiles, sizeof(kept), cudaMemcpyDeviceToHost, stream));
    WL_CUDA(cudaStreamSynchronize(stream));  // also: h_cand is free for the next batch
    accepted += std::min<uint64_t>(kept, missing);
    drawn += m;
    set_entries += m;
  }
  if (mem_space == BHT_MEM_HOST) {
    WL_CUDA(cudaMemcpyAsync(out_keys, d_out, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    WL_CUDA(cudaStreamSynchronize(stream));
  }
  cleanup();
  return BHT_OK;
}

// generate_queries (keygen.cpp:66-98).  Host outputs (the final shuffle is a host pass): q keys, their expected
// values (value_for_key for positives, 0 for negatives, as the reference's `query`), and the presence tags.
bht_status bht_generate_queries(const uint32_t* keys, uint64_t n_keys, int32_t keys_space, double positive_ratio, uint64_t q,
                                uint64_t seed, uint32_t* out_keys, uint32_t* out_expected, uint8_t* out_present, int32_t device) {
  if (!(positive_ratio >= 0.0 && positive_ratio <= 1.0))
    return wl_fail(BHT_INVALID_ARGUMENT, "generate_queries: positive_ratio must be in [0, 1]");
  const uint64_t n_pos = static_cast<uint64_t>(std::llround(positive_ratio * static_cast<double>(q)));
  if (n_pos > n_keys) return wl_fail(BHT_INVALID_ARGUMENT, "generate_queries: not enough keys for the requested positive ratio");
  if ((n_keys != 0 && keys == nullptr) || (q != 0 && out_keys == nullptr))
    return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_queries: null argument");
  if (keys_space != BHT_MEM_DEVICE && keys_space != BHT_MEM_HOST) return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_queries: bad keys_space");
  if (q == 0) return BHT_OK;
  int prev_device = -1;
  cudaGetDevice(&prev_device);
  if (cudaSetDevice(device) != cudaSuccess) return wl_fail(BHT_CUDA_ERROR, "bht_generate_queries: cudaSetDevice failed");

  bht_table* member = nullptr;
  uint32_t *d_keys = nullptr, *d_cand = nullptr, *d_ans = nullptr, *h_cand = nullptr, *h_ans = nullptr;
  auto cleanup = [&]() {
    if (member) bht_destroy(member);
    if (d_keys && keys_space == BHT_MEM_HOST) cudaFree(d_keys);
    if (d_cand) cudaFree(d_cand);
    if (d_ans) cudaFree(d_ans);
    if (h_cand) cudaFreeHost(h_cand);
    if (h_ans) cudaFreeHost(h_ans);
    if (prev_device >= 0) cudaSetDevice(prev_device);
  };

  struct Query { uint32_t key, expected; uint8_t present; };
  std::vector<Query> out;
  out.reserve(q);
  std::mt19937_64 eng(mix_seed(seed, 0x71756572ull));

  // positives: partial Fisher-Yates over a copy of the key list
  std::vector<uint32_t> pool(n_keys);
  if (n_keys != 0) {
    if (keys_space == BHT_MEM_HOST) std::copy(keys, keys + n_keys, pool.begin());
    else WL_CUDA(cudaMemcpy(pool.data(), keys, n_keys * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
  for (uint64_t i = 0; i < n_pos; ++i) {
    const uint64_t j = i + uniform_below(eng, pool.size() - i);
    std::swap(pool[i], pool[j]);
    out.push_back({pool[i], bht_value_for_key(pool[i]), 1});
  }

  // negatives: rejection against the inserted set = bulk find on a device table of the keys
  const uint64_t n_neg = q - n_pos;
  if (n_neg != 0) {
    if (n_keys != 0) {
      if (keys_space == BHT_MEM_HOST) {
        WL_CUDA(cudaMalloc(&d_keys, n_keys * sizeof(uint32_t)));
        WL_CUDA(cudaMemcpy(d_keys, keys, n_keys * sizeof(uint32_t), cudaMemcpyHostToDevice));
      } else {
        d_keys = const_cast<uint32_t*>(keys);
      }
      bool built = false;
      for (uint64_t attempt = 0; attempt < 16 && !built; ++attempt) {
        bht_config cfg;
        bht_status s = bht_make_config(BHT_BCHT, n_keys, 0.8, 16, -1, mix_seed(seed, 0x6d656d62ull + attempt), -1, &cfg);
        if (s != BHT_OK) { cleanup(); return s; }
        bht_insert_result r{};
        s = bht_create(&cfg, device, &member);
        if (s == BHT_OK) s = bht_insert(member, d_keys, d_keys, n_keys, BHT_MEM_DEVICE, &r, nullptr);  // values unused
        if (s != BHT_OK) { cleanup(); return s; }
        built = r.success != 0;
        if (!built) { bht_destroy(member); member = nullptr; }
      }
      if (!built) { cleanup(); return wl_fail(BHT_INVALID_ARGUMENT, "bht_generate_queries: membership table did not build (duplicate keys?)"); }
    }
    const uint64_t batch_cap = n_neg + n_neg / 32 + (1u << 16);
    WL_CUDA(cudaMallocHost(&h_cand, batch_cap * sizeof(uint32_t)));
    if (member != nullptr) {
      WL_CUDA(cudaMallocHost(&h_ans, batch_cap * sizeof(uint32_t)));
      WL_CUDA(cudaMalloc(&d_cand, batch_cap * sizeof(uint32_t)));
      WL_CUDA(cudaMalloc(&d_ans, batch_cap * sizeof(uint32_t)));
    }
    uint64_t have = 0;
    while (have < n_neg) {
      const uint64_t missing = n_neg - have;
      const uint64_t m = std::min(batch_cap, have == 0 ? batch_cap : std::max<uint64_t>(2 * missing, 1u << 16));
      const std::mt19937_64 before = eng;
      for (uint64_t i = 0; i < m; ++i) h_cand[i] = static_cast<uint32_t>(eng() >> 32);
      if (member != nullptr) {
        WL_CUDA(cudaMemcpy(d_cand, h_cand, m * sizeof(uint32_t), cudaMemcpyHostToDevice));
        bht_status s = bht_find(member, d_cand, d_ans, m, BHT_MEM_DEVICE, nullptr, nullptr);
        if (s != BHT_OK) { cleanup(); return s; }
        WL_CUDA(cudaMemcpy(h_ans, d_ans, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      }
      uint64_t used = m;
      for (uint64_t i = 0; i < m; ++i) {
        const uint32_t k = h_cand[i];
        if (k == BHT_EMPTY_KEY || (member != nullptr && h_ans[i] != BHT_EMPTY_KEY)) continue;
        out.push_back({k, 0u, 0});
        if (++have == n_neg) {
          used = i + 1;
          break;
        }
      }
      if (used != m) {  // rewind to the draw after the last one the reference would have consumed
        eng = before;
        eng.discard(used);
      }
    }
  }

  // shuffle_deterministic (keygen.cpp:42-46)
  for (uint64_t i = out.size(); i > 1; --i) std::swap(out[i - 1], out[uniform_below(eng, i)]);
  for (uint64_t i = 0; i < q; ++i) {
    out_keys[i] = out[i].key;
    if (out_expected) out_expected[i] = out[i].expected;
    if (out_present) out_present[i] = out[i].present;
  }
  cleanup();
  return BHT_OK;
}

// save_keys / load_keys (keygen.cpp:100-125): flat file of little-endian 32-bit keys.
bht_status bht_save_keys(const char* path, const uint32_t* keys_host, uint64_t n) {
  if (path == nullptr || (n != 0 && keys_host == nullptr)) return wl_fail(BHT_INVALID_ARGUMENT, "bht_save_keys: null argument");
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return wl_fail(BHT_IO_ERROR, std::string("save_keys: cannot open ") + path);
  std::vector<unsigned char> buf(1 << 16);
  uint64_t i = 0;
  bool ok = true;
  while (i < n && ok) {
    const uint64_t chunk = std::min<uint64_t>(n - i, buf.size() / 4);
    for (uint64_t j = 0; j < chunk; ++j) {
      const uint32_t k = keys_host[i + j];
      buf[4 * j] = k & 0xFF, buf[4 * j + 1] = (k >> 8) & 0xFF, buf[4 * j + 2] = (k >> 16) & 0xFF, buf[4 * j + 3] = (k >> 24) & 0xFF;
    }
    ok = std::fwrite(buf.data(), 4, chunk, f) == chunk;
    i += chunk;
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return wl_fail(BHT_IO_ERROR, std::string("save_keys: write failed for ") + path);
  return BHT_OK;
}

// *count = keys in the file; at most max_keys of them are copied to keys_host (which may be null to size a buffer).
bht_status bht_load_keys(const char* path, uint32_t* keys_host, uint64_t max_keys, uint64_t* count) {
  if (path == nullptr || count == nullptr) return wl_fail(BHT_INVALID_ARGUMENT, "bht_load_keys: null argument");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return wl_fail(BHT_IO_ERROR, std::string("load_keys: cannot open ") + path);
  unsigned char b[4];
  uint64_t i = 0;
  while (std::fread(b, 1, 4, f) == 4) {  // a trailing partial word is ignored, as the reference's read loop does
    if (keys_host != nullptr && i < max_keys)
      keys_host[i] = static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) | (static_cast<uint32_t>(b[2]) << 16) |
                     (static_cast<uint32_t>(b[3]) << 24);
    ++i;
  }
  std::fclose(f);
  *count = i;
  return BHT_OK;
}

}  // extern "C"
