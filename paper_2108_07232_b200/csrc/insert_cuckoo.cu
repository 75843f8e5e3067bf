// insert_cuckoo.cu — K4: bulk insert for the cuckoo tables (bcht: b >= 1, 3 hashes; 1cht: b = 1, 4 hashes).
//
// Replaces bcht_insert (reference: proj/src/table.cpp:53-92) as driven by build()'s loop
// (table.cpp:224-271):
//   probe the current bucket (first H0);
//   full  -> fail if `chain == max_chain` (cap checked BEFORE the exchange, table.cpp:67), else
//            atomicExch the pair into slot rng.next_below(b) (table.cpp:71), continue with the
//            victim in the bucket named by the hash function AFTER the lowest-index one that maps
//            the victim to this bucket (table.cpp:72-80), ++chain;
//   else  -> atomicCAS(empty -> pair) at slot index = load (table.cpp:85); on a lost race re-probe
//            the same bucket.
// Slot layout may differ from a sequential CPU build (concurrent order); the stored multiset, the
// admissibility of every pair and every query answer do not.
//
// Two phases per warp batch of 32 pairs:
//   fast path  all first-bucket probes batched through the probe engine (up to 32 lines in flight
//              per warp), then ONE warp-wide 64-bit atomicCAS in which every lane claims slot
//              `load` of its own bucket;
//   slow path  pairs whose first bucket was full, or that lost the CAS, run the reference loop as
//              a per-tile state machine (tile = b/2 lanes): tile lane 0 issues the atomic and the
//              old pair is broadcast with a shuffle, as in the paper's Listing 2.
// The eviction RNG is the reference's xorshift64 (hash.hpp:39-62), one stream per tile seeded
// mix_seed(seed, 0x65766963 + tile) like the per-worker streams of table.cpp:13,251.
#include "insert_common.cuh"

namespace bht_b200 {

template <int B, int H>
__global__ void __launch_bounds__(kInsertBlock)
bulk_insert_cuckoo_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys,
                          const uint32_t* __restrict__ values, uint64_t n, DevCounters* __restrict__ ctr,
                          uint32_t* __restrict__ failed_keys, uint64_t failed_cap) {
  using G = Geo<B>;
  const int lane = threadIdx.x & 31;
  const int sub = lane & (G::LPB - 1);
  const int gbase = lane & ~(G::LPB - 1);
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t n_batches = (n + 31) >> 5;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);

  // one eviction stream per tile; all lanes of a tile keep identical copies of the state
  uint64_t rng = xorshift_init(mix_seed(t.seed, 0x65766963ull + warp * (32 / G::LPB) + (lane / G::LPB)));

  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;

  for (uint64_t batch = warp; batch < n_batches; batch += n_warps) {
    const uint64_t idx = (batch << 5) + lane;
    const bool valid = idx < n;
    const uint32_t key = valid ? __ldcs(keys + idx) : kEmptyKey;
    const uint32_t val = valid ? __ldcs(values + idx) : kEmptyKey;
    bool pending = valid;
    const uint32_t bid = bucket_index(t.h[0], key);

    // ---- fast path: batched first probes + one vector CAS ----
    uint32_t load;
    probe_load<B>(t.store, bid, pending, lane, load);
    if (pending) {
      ++n_probe;
      if (load < B) {
        const unsigned long long old =
            atomicCAS(store + static_cast<uint64_t>(bid) * B + load, kEmptySlot, pack_pair(key, val));
        if (old == kEmptySlot) {
          pending = false;
          ++n_ins;
        }
      }
    }

    // ---- slow path: per-tile cuckoo state machine ----
    const uint32_t slow = __ballot_sync(kFullMask, pending);
    if (slow == 0) continue;
    uint32_t gpend = (slow >> gbase) & G::GMASK;  // tile-uniform queue of this tile's pending lanes
    // a first probe that saw a full bucket is not repeated: full buckets never drain, so the
    // snapshot is still valid and the reference's single probe + exchange is reproduced exactly
    const uint32_t saw_full = (__ballot_sync(kFullMask, pending && load == B) >> gbase) & G::GMASK;
    bool have = false, known_full = false;
    uint32_t ck = 0, cv = 0, cb = 0, chain = 0, retries = 0;
    for (;;) {
      const bool fetch = !have && gpend != 0;
      const int src = fetch ? (__ffs(gpend) - 1) : 0;
      const uint32_t nk = __shfl_sync(kFullMask, key, src, G::LPB);
      const uint32_t nv = __shfl_sync(kFullMask, val, src, G::LPB);
      const uint32_t nb = __shfl_sync(kFullMask, bid, src, G::LPB);
      if (fetch) {
        ck = nk;
        cv = nv;
        cb = nb;
        chain = 0;
        retries = 0;
        have = true;
        known_full = (saw_full >> src) & 1u;
        gpend &= gpend - 1;
      }
      if (!__any_sync(kFullMask, have)) break;

      const bool reprobe = have && !known_full;
      uint32_t ld = tile_probe_load<B>(t.store, cb, reprobe, lane);
      if (known_full) ld = B;
      known_full = false;
      const bool full = ld == B;
      const bool do_fail = have && ((full && chain == t.max_chain) || retries > t.retry_cap);
      const bool do_exch = have && full && !do_fail;
      const bool do_cas = have && !full && !do_fail;
      uint32_t slot = ld;
      if (do_exch) slot = xorshift_next_below(rng, B);
      unsigned long long old = 0;
      if (sub == 0 && have) {
        n_probe += reprobe;
        unsigned long long* p = store + static_cast<uint64_t>(cb) * B + slot;
        if (do_exch) old = atomicExch(p, pack_pair(ck, cv));
        else if (do_cas) old = atomicCAS(p, kEmptySlot, pack_pair(ck, cv));
      }
      old = __shfl_sync(kFullMask, old, 0, G::LPB);

      if (do_fail) {
        if (sub == 0) {
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, ck);  // the pair in hand is the one dropped
        }
        have = false;
      } else if (do_cas) {
        if (old == kEmptySlot) {
          if (sub == 0) ++n_ins;
          have = false;
        } else {
          ++retries;  // lost the slot to a concurrent insert; re-snapshot the same bucket
        }
      } else if (do_exch) {
        const uint32_t vk = static_cast<uint32_t>(old);
        if (vk == kEmptyKey) {  // exchanged into a hole: only possible on an uploaded store
          if (sub == 0) ++n_ins;
          have = false;
        } else {
          uint32_t cand[H];
#pragma unroll
          for (int i = 0; i < H; ++i) cand[i] = bucket_index(t.h[i], vk);
          uint32_t next = cand[0];
#pragma unroll
          for (int i = H - 1; i >= 0; --i)  // lowest matching index wins (table.cpp:74-80)
            if (cand[i] == cb) next = cand[(i + 1) % H];
          ck = vk;
          cv = static_cast<uint32_t>(old >> 32);
          cb = next;
          ++chain;
        }
      }
    }
  }

  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

template <int B, int H>
static cudaError_t launch_one(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                              DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                              cudaStream_t stream) {
  auto kernel = bulk_insert_cuckoo_kernel<B, H>;
  const int grid = persistent_grid(kernel, kInsertBlock, sm_count, n, kInsertBlock);
  kernel<<<grid, kInsertBlock, 0, stream>>>(t, keys, values, n, ctr, failed_keys, failed_cap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_insert_cuckoo(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                                 DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                                 cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (t.n_hashes == 4) {
    if (t.bucket_size != 1) return cudaErrorInvalidValue;
    return launch_one<1, 4>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
  }
  if (t.n_hashes != 3) return cudaErrorInvalidValue;
  switch (t.bucket_size) {
    case 1: return launch_one<1, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 2: return launch_one<2, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 4: return launch_one<4, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 8: return launch_one<8, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 16: return launch_one<16, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 32: return launch_one<32, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    case 64: return launch_one<64, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bht_b200
