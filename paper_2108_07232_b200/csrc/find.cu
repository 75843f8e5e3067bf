// find.cu — K3: bulk find for all four tables.
//
// Replaces the caller-side `for q: find_key(table, q.key, stats)` loop (reference:
// proj/src/experiments.cpp:92, proj/src/oracle.cpp:21-27) and the per-variant finds:
//   bcht_find  (table.cpp:94-107)  serial probes H0..H(h-1), stop on a hit or on a non-full bucket
//   bp2ht_find (table.cpp:132-142) H0 then H1, no early exit
//   iht_find   (table.cpp:188-201) primary, s0, s1, no early exit
//   bcht_find_no_early_exit (oracle.cpp:56-63)
// Probe counts are identical to the reference's (one per bucket read), so the algorithmic bytes of
// a launch are probes x ceil(8b/32) x 32 B (sector_model.hpp:18-31).
//
// Bound: HBM, random 128-byte lines.  Each warp owns 32 keys per batch; probe round i hashes the
// still-pending keys with H_i and reads their buckets through the batched probe engine.
#include "kernels.h"

namespace bht_b200 {

constexpr int kFindBlock = 256;

template <int B, int H, bool EARLY_EXIT>
__global__ void __launch_bounds__(kFindBlock)
bulk_find_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys, uint32_t* __restrict__ out,
                 uint64_t n, DevCounters* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t n_batches = (n + 31) >> 5;

  uint32_t probes = 0, hits = 0;
  unsigned long long vsum = 0;

  for (uint64_t batch = warp; batch < n_batches; batch += n_warps) {
    const uint64_t idx = (batch << 5) + lane;
    const bool valid = idx < n;
    const uint32_t key = valid ? __ldcs(keys + idx) : kEmptyKey;
    uint32_t result = kEmptyKey;
    bool pending = valid && key != kEmptyKey;  // the sentinel is never a stored key (core.hpp:23-24)

#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (i > 0 && !__any_sync(kFullMask, pending)) break;
      const uint32_t bid = bucket_index(t.h[i], key);
      bool found, notfull;
      uint32_t value;
      probe_find<B>(t.store, bid, pending, key, lane, found, value, notfull);
      if (pending) {
        ++probes;
        if (found) {
          result = value;
          pending = false;
          ++hits;
          vsum += value;
        } else if (EARLY_EXIT && notfull) {
          pending = false;  // a bucket that ever evicted stays full (table.cpp:104)
        }
      }
    }
    if (valid) __stcs(out + idx, result);
  }

  const unsigned long long p = warp_sum(probes), h = warp_sum(hits), s = warp_sum(vsum);
  if (lane == 0 && ctr != nullptr) {
    if (p) atomicAdd(&ctr->find_probes, p);
    if (h) atomicAdd(&ctr->find_hits, h);
    if (s) atomicAdd(&ctr->find_value_sum, s);
  }
}

template <int B, int H, bool EARLY_EXIT>
static cudaError_t launch_one(const TableView& t, const uint32_t* keys, uint32_t* out, uint64_t n, DevCounters* ctr,
                              int sm_count, cudaStream_t stream) {
  auto kernel = bulk_find_kernel<B, H, EARLY_EXIT>;
  const int grid = persistent_grid(kernel, kFindBlock, sm_count, n, kFindBlock);
  kernel<<<grid, kFindBlock, 0, stream>>>(t, keys, out, n, ctr);
  note_launch();
  return cudaGetLastError();
}

template <int B>
static cudaError_t launch_b(const TableView& t, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                            DevCounters* ctr, int sm_count, cudaStream_t stream) {
  switch (t.n_hashes) {
    case 2: return launch_one<B, 2, false>(t, keys, out, n, ctr, sm_count, stream);
    case 3:
      return early_exit ? launch_one<B, 3, true>(t, keys, out, n, ctr, sm_count, stream)
                        : launch_one<B, 3, false>(t, keys, out, n, ctr, sm_count, stream);
    case 4:
      if constexpr (B == 1)
        return early_exit ? launch_one<1, 4, true>(t, keys, out, n, ctr, sm_count, stream)
                          : launch_one<1, 4, false>(t, keys, out, n, ctr, sm_count, stream);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_find(const TableView& t, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                        DevCounters* ctr, int sm_count, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  switch (t.bucket_size) {
    case 1: return launch_b<1>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 2: return launch_b<2>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 4: return launch_b<4>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 8: return launch_b<8>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 16: return launch_b<16>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 32: return launch_b<32>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    case 64: return launch_b<64>(t, early_exit, keys, out, n, ctr, sm_count, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bht_b200
