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
// Every lane runs exactly that loop as a state machine over (pair in hand, bucket, chain): one
// loop iteration = one probe round of the warp.  The 32 buckets of a round are fetched together by
// the probe engine, each lane scans its own bucket and issues its own 64-bit atomicCAS / atomicExch,
// and a lane that placed its pair takes the next pair of the warp's slice — eviction chains of one
// lane never idle the other 31.
// The eviction RNG is the reference's xorshift64 (hash.hpp:39-62), one stream per lane seeded
// mix_seed(seed, 0x65766963 + lane id) like the per-worker streams of table.cpp:13,251.
#include "insert_common.cuh"

namespace bht_b200 {

template <int B, int H>
__global__ void __launch_bounds__(block_threads<B>(1))
bulk_insert_cuckoo_kernel(const __grid_constant__ TableView t, const uint32_t* __restrict__ keys,
                          const uint32_t* __restrict__ values, uint64_t n, DevCounters* __restrict__ ctr,
                          uint32_t* __restrict__ failed_keys, uint64_t failed_cap) {
  using G = Geo<B>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const uint32_t stage = smem_u32(smem) + (threadIdx.x >> 5) * G::WARP_BYTES;
  unsigned long long* store = reinterpret_cast<unsigned long long*>(t.store);

  uint64_t rng = xorshift_init(mix_seed(t.seed, 0x65766963ull + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x));
  uint32_t n_ins = 0, n_fail = 0, n_probe = 0;

  PairFeed feed;
  feed.init(keys, values, n, lane);
  bool have = false;
  uint32_t key = 0, val = 0, bid = 0, chain = 0, retries = 0;

  for (;;) {
    if (feed.refill(have, lane, key, val)) {
      have = true;
      bid = bucket_index(t.h[0], key);
      chain = 0;
      retries = 0;
    }
    if (!__any_sync(kFullMask, have)) break;

    fetch_issue<B>(stage, t.store, have ? bid : kNoBucket, lane);
    if (G::STAGED) fetch_wait();
    if (have) {
      const Scan s = scan_bucket<B, false>(stage, t.store, bid, key, lane);
      ++n_probe;
      unsigned long long* bucket = store + static_cast<uint64_t>(bid) * B;
      if (s.load < B) {
        if (atomicCAS(bucket + s.load, kEmptySlot, pack_pair(key, val)) == kEmptySlot) {
          ++n_ins;
          have = false;
        } else if (++retries > t.retry_cap) {  // lost the slot; re-snapshot the same bucket next round
          ++n_fail;
          record_failed(ctr, failed_keys, failed_cap, key);
          have = false;
        }
      } else if (chain == t.max_chain) {
        ++n_fail;
        record_failed(ctr, failed_keys, failed_cap, key);  // the pair in hand is the one dropped
        have = false;
      } else {
        const unsigned long long old = atomicExch(bucket + xorshift_next_below(rng, B), pack_pair(key, val));
        const uint32_t vk = static_cast<uint32_t>(old);
        if (vk == kEmptyKey) {  // exchanged into a hole: only possible on an uploaded store
          ++n_ins;
          have = false;
        } else {
          uint32_t cand[H];
#pragma unroll
          for (int i = 0; i < H; ++i) cand[i] = bucket_index(t.h[i], vk);
          uint32_t next = cand[0];
#pragma unroll
          for (int i = H - 1; i >= 0; --i)  // lowest matching index wins (table.cpp:74-80)
            if (cand[i] == bid) next = cand[(i + 1) % H];
          key = vk;
          val = static_cast<uint32_t>(old >> 32);
          bid = next;
          ++chain;
        }
      }
    }
    if (G::STAGED) __syncwarp();
  }

  flush_insert_counters(ctr, lane, n_ins, n_fail, n_probe);
}

template <int B, int H>
static cudaError_t launch_one(const TableView& t, const uint32_t* keys, const uint32_t* values, uint64_t n,
                              DevCounters* ctr, uint32_t* failed_keys, uint64_t failed_cap, int sm_count,
                              cudaStream_t stream) {
  auto kernel = bulk_insert_cuckoo_kernel<B, H>;
  constexpr int block = block_threads<B>(1);
  constexpr int smem = (block / 32) * Geo<B>::WARP_BYTES;
  const int grid = persistent_grid(kernel, block, smem, sm_count, n, block);
  kernel<<<grid, block, smem, stream>>>(t, keys, values, n, ctr, failed_keys, failed_cap);
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
#define CALL(BB) launch_one<BB, 3>(t, keys, values, n, ctr, failed_keys, failed_cap, sm_count, stream)
  BHT_DISPATCH_BUCKET_SIZE(t.bucket_size, CALL)
#undef CALL
}

}  // namespace bht_b200
