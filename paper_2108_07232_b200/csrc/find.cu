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
// Bound: HBM, random 128-byte lines.  Each lane carries one query through its probe sequence
// (state: key, position, next hash index); a lane whose query is answered takes the next query of
// the warp's slice, so each round of a warp is 32 independent bucket fetches.
#include "kernels.h"

namespace bht_b200 {

template <int B, int H, bool EARLY_EXIT>
__global__ void __launch_bounds__(block_threads<B>(1))
bulk_find_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys, uint32_t* __restrict__ out,
                 uint64_t n, DevCounters* __restrict__ ctr, uint32_t* __restrict__ work_cursor) {
  using G = Geo<B>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const uint32_t stage = smem_u32(smem) + (threadIdx.x >> 5) * G::WARP_BYTES;
  const uint32_t lt_mask = (1u << lane) - 1u;

  Stream st;
  st.init(n, t.chunk_log2, work_cursor, lane);
  uint32_t probes = 0, hits = 0;
  unsigned long long vsum = 0;

  bool have = false;
  uint32_t key = 0, round = 0;
  uint64_t idx = 0;
  // the next 32 queries of the stream, one per lane, and how many of them exist
  uint32_t ahead, ahead_n;
  {
    uint64_t g;
    const bool in = st.index(lane, t.chunk_log2, g);
    ahead = in ? __ldcs(keys + g) : 0u;
    ahead_n = __popc(__ballot_sync(kFullMask, in));
  }

  for (;;) {
    // ---- refill: idle lanes take the next unread queries, in order
    const uint32_t idle = __ballot_sync(kFullMask, !have);
    if (idle != 0 && ahead_n != 0) {
      const uint32_t rank = __popc(idle & lt_mask);
      const uint32_t fresh = __shfl_sync(kFullMask, ahead, rank);
      if (!have && rank < ahead_n) {
        key = fresh;
        st.index(rank, t.chunk_log2, idx);
        round = 0;
        have = true;
      }
      st.advance(min(static_cast<uint32_t>(__popc(idle)), ahead_n), t.chunk_log2, work_cursor, lane);
      uint64_t g;
      const bool in = st.index(lane, t.chunk_log2, g);
      ahead = in ? __ldcs(keys + g) : 0u;
      ahead_n = __popc(__ballot_sync(kFullMask, in));
    }
    if (!__any_sync(kFullMask, have)) break;

    // ---- one probe per lane
    // the sentinel is never a stored key (core.hpp:23-24): it is answered "absent" without a probe
    const bool probing = have && key != kEmptyKey;
    const uint32_t bid = probing ? bucket_index_sel<H>(t, round, key) : kNoBucket;
    fetch_issue<B>(stage, t.store, bid, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      bool done = true;
      uint32_t answer = kEmptyKey;
      if (probing) {
        const Scan s = scan_bucket<B, true>(stage, t.store, bid, key, lane);
        ++probes;
        if (s.found) {
          answer = s.value;
          ++hits;
          vsum += s.value;
        } else if ((EARLY_EXIT && s.load < B) || round == H - 1) {
          // a bucket that ever evicted stays full (table.cpp:104); or every candidate was read
        } else {
          ++round;
          done = false;
        }
      }
      if (done) {
        __stcs(out + idx, answer);
        have = false;
      }
    }
    if (G::STAGED) __syncwarp();  // all rows scanned before the next round overwrites them
  }

  if (ctr != nullptr) {
    const unsigned long long p = warp_sum(probes), h = warp_sum(hits), s = warp_sum(vsum);
    if (lane == 0) {
      if (p) atomicAdd(&ctr->find_probes, p);
      if (h) atomicAdd(&ctr->find_hits, h);
      if (s) atomicAdd(&ctr->find_value_sum, s);
    }
  }
}

template <int B, int H, bool EARLY_EXIT>
static cudaError_t launch_one(const TableView& t, const uint32_t* keys, uint32_t* out, uint64_t n, DevCounters* ctr,
                              uint32_t* work_cursor, int sm_count, cudaStream_t stream) {
  auto kernel = bulk_find_kernel<B, H, EARLY_EXIT>;
  constexpr int block = block_threads<B>(1);
  constexpr int smem = (block / 32) * Geo<B>::WARP_BYTES;
  const int grid = persistent_grid(kernel, block, smem, sm_count, n, block);
  kernel<<<grid, block, smem, stream>>>(t, keys, out, n, ctr, work_cursor);
  note_launch();
  return cudaGetLastError();
}

template <int B>
static cudaError_t launch_b(const TableView& t, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                            DevCounters* ctr, uint32_t* work_cursor, int sm_count, cudaStream_t stream) {
  switch (t.n_hashes) {
    case 2: return launch_one<B, 2, false>(t, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 3:
      return early_exit ? launch_one<B, 3, true>(t, keys, out, n, ctr, work_cursor, sm_count, stream)
                        : launch_one<B, 3, false>(t, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 4:
      if constexpr (B == 1)
        return early_exit ? launch_one<1, 4, true>(t, keys, out, n, ctr, work_cursor, sm_count, stream)
                          : launch_one<1, 4, false>(t, keys, out, n, ctr, work_cursor, sm_count, stream);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_find(const TableView& t, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                        DevCounters* ctr, uint32_t* work_cursor, int sm_count, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  switch (t.bucket_size) {
    case 1: return launch_b<1>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 2: return launch_b<2>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 4: return launch_b<4>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 8: return launch_b<8>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 16: return launch_b<16>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 32: return launch_b<32>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    case 64: return launch_b<64>(t, early_exit, keys, out, n, ctr, work_cursor, sm_count, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bht_b200
