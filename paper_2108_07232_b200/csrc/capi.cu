// capi.cu — the C ABI of include/bht_b200.h: C++ host code over the sm_100a kernels.
//
// Each entry point names the reference interface it replaces in include/bht_b200.h.  This file owns
// what `class hash_table` owns in the reference (proj/include/bht/table.hpp:28-80): the config, the
// slot store (device memory here) and the inserted counter; plus the staging pipeline that moves
// host-resident key / value / answer arrays over PCIe in chunks while the probe kernels run.
//
// There is no CPU fallback anywhere in this file: without a usable device every compute entry point
// returns BHT_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "../../include/bht_b200.h"
#include "kernels.h"

using namespace bht_b200;

namespace {

thread_local std::string g_error;

bht_status fail(bht_status s, const std::string& msg) {
  g_error = msg;
  return s;
}
bht_status cuda_fail(cudaError_t e, const char* what) {
  g_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return BHT_CUDA_ERROR;
}
#define BHT_CUDA(expr)                                        \
  do {                                                        \
    cudaError_t e__ = (expr);                                 \
    if (e__ != cudaSuccess) return cuda_fail(e__, #expr);     \
  } while (0)

struct DeviceScope {  // every call runs on the table's device and leaves the caller's device as it was
  int prev = -1;
  bool switched = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceScope(int device) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != device) {
      err = cudaSetDevice(device);
      switched = err == cudaSuccess;
    }
  }
  ~DeviceScope() {
    if (switched) cudaSetDevice(prev);
  }
};
#define BHT_ON_DEVICE(dev)       \
  DeviceScope scope__(dev);      \
  if (scope__.err != cudaSuccess) return cuda_fail(scope__.err, "cudaSetDevice")

// Tuning / experiment knobs from the environment, read ONCE per process (the first call that needs them), never on
// the call path.  -1 / negative = not set.
struct Knobs {
  long stage_chunk_log2, insert_ctas, insert_grid, direct, sweep_mb, claim_insert, region_mb, smem_build, blocked_ctas,
      tail_throttle, tail_div, chunk_log2;
  double tail_lf;
};
long env_long(const char* name, long unset) {
  const char* e = std::getenv(name);
  return e != nullptr ? std::atol(e) : unset;
}
Knobs load_knobs() {
  Knobs v;
  v.stage_chunk_log2 = env_long("BHT_STAGE_CHUNK_LOG2", 22);  // 18..22
  v.insert_ctas = env_long("BHT_INSERT_CTAS", -1);            // keys in flight (tools/exp_success_inflight.py)
  v.insert_grid = env_long("BHT_INSERT_GRID", -1);
  v.direct = env_long("BHT_DIRECT", 1);              // 0 = staged engine everywhere, 1 = direct engine (4 <= b <= 16), 2 = direct for routed builds only
  v.sweep_mb = env_long("BHT_SWEEP_MB", 16);         // L2 prefetch distance of a routed build, 0 = off
  v.claim_insert = env_long("BHT_CLAIM_INSERT", -1); // 0 = never, 1 = always the counter-claimed bp2ht / iht insert
  v.region_mb = env_long("BHT_REGION_MB", 48);       // region size of the L2-routed build, 0 = off
  v.smem_build = env_long("BHT_SMEM_BUILD", 1);      // 0: fall back to the L2-routed build
  v.blocked_ctas = env_long("BHT_BLOCKED_CTAS", 0);  // resident CTAs per SM of a routed build's insert kernel, 0 = whatever fits
  v.tail_throttle = env_long("BHT_TAIL_THROTTLE", -1);
  v.tail_div = env_long("BHT_TAIL_DIV", 24);
  v.chunk_log2 = env_long("BHT_CHUNK_LOG2", static_cast<long>(kDefaultChunkLog2));  // work-stream chunk (probe_engine.cuh, Stream)
  const char* lf = std::getenv("BHT_TAIL_LF");
  v.tail_lf = lf != nullptr ? std::atof(lf) : -1.0;
  return v;
}
Knobs& knobs_storage() {
  static Knobs k = load_knobs();
  return k;
}
const Knobs& knobs() { return knobs_storage(); }

// Stream-ordered scratch (routing / binning buffers, up to ~28 bytes per pair of a blocked build) comes from a pool the
// library owns, one per device, kept cached while any table lives on the device and handed back to the driver when
// the last one is destroyed — the process's default pool is left as the application configured it.
struct ScratchPools {
  std::mutex mu;
  cudaMemPool_t pool[64] = {};
  int users[64] = {};
} g_pools;
cudaMemPool_t scratch_pool(int device) { return device >= 0 && device < 64 ? g_pools.pool[device] : nullptr; }
void scratch_pool_acquire(int device) {
  if (device < 0 || device >= 64) return;
  std::lock_guard<std::mutex> lock(g_pools.mu);
  if (g_pools.pool[device] == nullptr) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      unsigned long long keep = ~0ull;  // cached across calls; trimmed when the last table of the device goes
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      g_pools.pool[device] = pool;
    } else {
      cudaGetLastError();  // fall back to the default pool (scratch_alloc)
    }
  }
  ++g_pools.users[device];
}
void scratch_pool_release(int device) {
  if (device < 0 || device >= 64) return;
  std::lock_guard<std::mutex> lock(g_pools.mu);
  if (--g_pools.users[device] == 0 && g_pools.pool[device] != nullptr) cudaMemPoolTrimTo(g_pools.pool[device], 0);
}

constexpr int kStageSlots = 3;
constexpr uint64_t kStageChunk = 1ull << 22;  // keys per staged chunk: 16 MiB per array over PCIe (measured: 2^19..2^24 — 2^22 is the fastest)
constexpr uint64_t kStageChunkMin = 1ull << 18;

// Length of the staged chunk that starts at `off`: chunks double from kStageChunkMin up to kStageChunk and halve
// again towards the end, so the pipeline fills and drains in ~1 MiB steps (the first copy-in and the last
// kernel / copy-out are the only parts of a host-buffer call that nothing overlaps).
uint64_t stage_chunk_len(uint64_t off, uint64_t n, bool ramp_up = true) {
  const long v = knobs().stage_chunk_log2;
  const uint64_t chunk_max = 1ull << (v < 18 ? 18 : (v > 22 ? 22 : v));
  // (no ramp-up when the device is still busy with an earlier call's work: nothing could start on a small first
  // chunk anyway, and full-size chunks put three slots' worth of copies under that work)
  const uint64_t up = ramp_up ? std::max(kStageChunkMin, off) : chunk_max;
  const uint64_t down = std::max(kStageChunkMin, (n - off) / 2);
  return std::min(std::min(chunk_max, n - off), std::min(up, down));
}
constexpr uint64_t kFailedLogCap = 1ull << 20;
constexpr uint32_t kMaxRepair = 256;  // dropped pairs of one launch that get a second, solitary insertion (insert_cuckoo.cu)
constexpr uint32_t kRetryCap = 1024;

// Host <-> device staging for BHT_MEM_HOST calls: kStageSlots chunks in flight, copy-in, probe kernel
// and copy-out on three streams chained by events.
struct Staging {
  bool ready = false;
  uint32_t* keys[kStageSlots] = {};
  uint32_t* vals[kStageSlots] = {};  // values (insert) or answers (find)
  cudaStream_t h2d = nullptr, d2h = nullptr, compute = nullptr;
  cudaEvent_t in_done[kStageSlots] = {}, kernel_done[kStageSlots] = {}, out_done[kStageSlots] = {};
};

}  // namespace

namespace bht_b200 {
void set_last_error(const std::string& msg) { g_error = msg; }  // for the other host TUs (workload.cu)
}  // namespace bht_b200

struct bht_table {
  bht_config cfg{};
  int device = 0;
  int sm_count = 148;
  TableView view{};
  DevCounters* ctr = nullptr;       // device
  DevCounters* ctr_host = nullptr;  // pinned mirror
  uint32_t* failed_keys = nullptr;  // device log of dropped keys
  // bht_set_blocked_insert: 0 = caller order, 1 = blocked when worth it (default), 2 = always the L2-routed
  // build, 3 = always the shared-memory-blocked build (bcht, 8 <= b <= 32; else as 2); bp2ht / iht are never blocked
  int blocked_insert = 1;
  int last_schedule = 0;  // how the last insert / chunked build ran: 0 = caller order, 2 = L2-routed, 3 = shared-memory-blocked
  bool known_empty = true;  // no slot has been written since create / clear: a blocked build need not read the store
  // The fill of create / clear is deferred until something reads or partially writes the store: a shared-memory-blocked
  // build into an empty table writes every region of the store exactly once, empty slots included (K11), so the fill
  // is fused into it; every other use of the store calls materialize_clear first.
  std::atomic<bool> clear_pending{false};
  // The deferred fill runs on the stream of whichever call pays the debt; calls on OTHER streams are ordered after it
  // through this event for as long as it has not completed.
  cudaEvent_t fill_done = nullptr;
  cudaStream_t fill_stream = nullptr;
  std::atomic<bool> fill_recorded{false};
  cudaEvent_t build_done = nullptr;  // end of the device work of a host-buffer insert (which returns once the copies are in)
  // bht_build_begin / _feed / _end: one build whose pairs arrive in chunks
  struct Session {
    bool active = false;
    bool blocked = false;  // shared-memory-blocked build: chunks go through K8g, the rest happens at the end
    BlockedPlan plan{};
    void* scratch = nullptr;
    uint64_t n_max = 0, fed = 0;
    bool fresh = false;
  } session;
  uint64_t host_inserted = 0;  // upper bound of the pairs in the store, kept on the host (tail_plan)
  bool tail_throttle = false;  // bht_set_tail_throttle
  bool repair_dropped = false;  // bht_set_repair (default: on for bcht, off for 1cht), see repair_dropped_kernel (insert_cuckoo.cu)
  // bp2ht / iht: one 32-bit load counter per bucket for the counter-claimed insert (insert_claim.cu); loads_valid =
  // the counters describe the store (false after anything else may have written slots: they are rebuilt on demand)
  uint32_t* loads = nullptr;
  bool loads_valid = false;
  // device-resident bht_insert: events around the preparation (routing / binning) and the probe kernel of the last
  // call, for bht_last_insert_phases (per-kernel roofline of bench.py)
  cudaEvent_t phase_ev[3] = {};
  bool phases_recorded = false;
  uint32_t* cursors = nullptr;        // device: ring of per-launch work cursors (Stream, probe_engine.cuh)
  std::atomic<uint32_t> cursor_seq{0};
  Staging stage;
  std::mutex mu;  // serialises calls that touch the counter block / staging buffers
};

namespace {

uint32_t hash_count_of(int32_t kind) {
  switch (kind) {
    case BHT_ONE_CHT: return 4;
    case BHT_BCHT: return 3;
    case BHT_BP2HT: return 2;
    case BHT_IHT: return 3;
    default: return 0;
  }
}

bool is_pow2(uint32_t x) { return x != 0 && (x & (x - 1)) == 0; }

bht_status validate_config(const bht_config& c) {
  const uint32_t h = hash_count_of(c.kind);
  if (h == 0) return fail(BHT_INVALID_ARGUMENT, "bht_create: unknown table kind");
  // hash_table::hash_table (table.cpp:22-23)
  if (c.n_hashes != h) return fail(BHT_INVALID_ARGUMENT, "hash_table: config has the wrong number of hash functions");
  if (!is_pow2(c.bucket_size) || c.bucket_size > BHT_MAX_BUCKET_SIZE)
    return fail(BHT_INVALID_ARGUMENT, "bht_create: bucket_size must be a power of two in [1, 64]");
  if (c.kind == BHT_ONE_CHT && c.bucket_size != 1) return fail(BHT_INVALID_ARGUMENT, "bht_create: 1cht requires bucket_size 1");
  if (c.num_buckets == 0 || c.capacity != c.num_buckets * c.bucket_size)
    return fail(BHT_INVALID_ARGUMENT, "bht_create: capacity must equal num_buckets * bucket_size > 0");
  if (c.num_buckets > 0xFFFFFFFFull) return fail(BHT_INVALID_ARGUMENT, "bht_create: num_buckets must fit 32 bits");
  if (c.kind == BHT_IHT && (c.threshold == 0 || c.threshold > c.bucket_size))
    return fail(BHT_INVALID_ARGUMENT, "bht_create: iht threshold must be in [1, bucket_size]");
  for (uint32_t i = 0; i < h; ++i) {
    if (c.alpha[i] > 0xFFFFFFFFull || c.beta[i] > 0xFFFFFFFFull)
      return fail(BHT_INVALID_ARGUMENT, "bht_create: hash constants must fit 32 bits (the reference draws them below p)");
    if (c.range[i] == 0 || c.range[i] > c.num_buckets)
      return fail(BHT_INVALID_ARGUMENT, "bht_create: hash range must be in [1, num_buckets]");
  }
  return BHT_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of a device, asked once (cudaGetDeviceProperties costs milliseconds per call: it was 8 ms of host time per
// chunk of a sharded find).
int device_sm_count(int device) {
  static std::atomic<int> cached[64];
  if (device < 0 || device >= 64) return 148;
  int v = cached[device].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    cached[device].store(v, std::memory_order_relaxed);
  }
  return v;
}

bht_status ensure_staging(bht_table* t) {
  Staging& s = t->stage;
  if (s.ready) return BHT_OK;
  for (int i = 0; i < kStageSlots; ++i) {
    BHT_CUDA(cudaMalloc(&s.keys[i], kStageChunk * sizeof(uint32_t)));
    BHT_CUDA(cudaMalloc(&s.vals[i], kStageChunk * sizeof(uint32_t)));
    BHT_CUDA(cudaEventCreateWithFlags(&s.in_done[i], cudaEventDisableTiming));
    BHT_CUDA(cudaEventCreateWithFlags(&s.kernel_done[i], cudaEventDisableTiming));
    BHT_CUDA(cudaEventCreateWithFlags(&s.out_done[i], cudaEventDisableTiming));
  }
  BHT_CUDA(cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking));
  BHT_CUDA(cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking));
  BHT_CUDA(cudaStreamCreateWithFlags(&s.compute, cudaStreamNonBlocking));
  s.ready = true;
  return BHT_OK;
}

void release_staging(Staging& s) {
  for (int i = 0; i < kStageSlots; ++i) {
    if (s.keys[i]) cudaFree(s.keys[i]);
    if (s.vals[i]) cudaFree(s.vals[i]);
    if (s.in_done[i]) cudaEventDestroy(s.in_done[i]);
    if (s.kernel_done[i]) cudaEventDestroy(s.kernel_done[i]);
    if (s.out_done[i]) cudaEventDestroy(s.out_done[i]);
  }
  if (s.h2d) cudaStreamDestroy(s.h2d);
  if (s.d2h) cudaStreamDestroy(s.d2h);
  if (s.compute) cudaStreamDestroy(s.compute);
  s = Staging{};
}

bht_status read_counters(bht_table* t, cudaStream_t stream) {
  BHT_CUDA(cudaMemcpyAsync(t->ctr_host, t->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, stream));
  BHT_CUDA(cudaStreamSynchronize(stream));
  return BHT_OK;
}

void fill_insert_result(const bht_table* t, uint64_t attempted, bht_insert_result* r) {
  const DevCounters& c = *t->ctr_host;
  r->attempted = attempted;
  r->inserted = c.inserted;
  r->failed = c.failed;
  r->probes = c.insert_probes;
  r->first_failed_key = c.failed_key_tag ? c.failed_key_tag - 1u : BHT_EMPTY_KEY;
  r->success = c.inserted == attempted ? 1u : 0u;
}

constexpr uint32_t kCursorSlots = 256;

// A zeroed work cursor for one probe-kernel launch on `stream`.  Launches that may overlap (finds on different
// streams) get different words of the ring.
cudaError_t next_cursor(bht_table* t, cudaStream_t stream, uint32_t** out) {
  *out = t->cursors + (t->cursor_seq.fetch_add(1, std::memory_order_relaxed) % kCursorSlots);
  return cudaMemsetAsync(*out, 0, sizeof(uint32_t), stream);
}

cudaError_t launch_insert_kind(bht_table* t, PairSource src, uint64_t n, int max_ctas_per_sm, cudaStream_t stream,
                               bool routed = false, const unsigned long long* n_dev = nullptr, int max_grid = 0) {
  InsertLaunch a;
  a.src = src;
  a.n = n;
  a.routed = routed;
  a.n_dev = n_dev;
  a.ctr = t->ctr;
  a.failed_keys = t->failed_keys;
  a.failed_cap = kFailedLogCap;
  // (a launch of at most one warp's worth of pairs has no concurrency to make up for: one pair per launch is the
  // reference's insert_pair exactly, failed insertions included)
  a.max_repair = (t->repair_dropped && n > 32) ? kMaxRepair : 0u;
  a.sm_count = t->sm_count;
  a.max_ctas_per_sm = max_ctas_per_sm;
  const Knobs& k = knobs();
  if (k.insert_ctas > 0) a.max_ctas_per_sm = static_cast<int>(k.insert_ctas);
  a.max_grid = k.insert_grid >= 0 ? static_cast<int>(k.insert_grid) : max_grid;
  // the direct engine is the default: measured faster for 4 <= b <= 16 in caller order and in routed builds
  a.direct = k.direct == 1 || (k.direct == 2 && routed);
  a.stream = stream;
  cudaError_t e = next_cursor(t, stream, &a.work_cursor);
  if (e != cudaSuccess) return e;
  t->view.sweep_ahead_bytes = static_cast<uint32_t>((k.sweep_mb < 0 ? 0 : (k.sweep_mb > 1024 ? 1024 : k.sweep_mb)) << 20);
  switch (t->cfg.kind) {
    case BHT_ONE_CHT:
    case BHT_BCHT:
      return launch_insert_cuckoo(t->view, a);
    case BHT_BP2HT:
    case BHT_IHT: {
      // Counter-claimed insert (insert_claim.cu) when the store lives in HBM (or when forced, mode 3): the candidates'
      // loads come from the L2-resident counter array and the only HBM access of an insertion is the 8-byte store.
      // Small tables keep the bucket-reading kernels (their probes are L2 hits anyway); whatever they write makes the
      // counters stale, and they are rebuilt from the store before the next counter-claimed launch.
      const bool big = t->cfg.capacity * sizeof(uint64_t) >= (192ull << 20);
      const bool claim = t->loads != nullptr && (k.claim_insert >= 0 ? k.claim_insert != 0 : (t->blocked_insert == 3 || (t->blocked_insert == 1 && big)));
      if (claim) {
        if (!t->loads_valid) {
          e = launch_load_count(t->view, t->loads, t->sm_count, stream);
          if (e != cudaSuccess) return e;
          t->loads_valid = true;
        }
        return launch_claim_insert(t->view, t->loads, a, t->cfg.kind == BHT_IHT);
      }
      t->loads_valid = false;
      return t->cfg.kind == BHT_BP2HT ? launch_insert_p2(t->view, a) : launch_insert_iht(t->view, a);
    }
    default: return cudaErrorInvalidValue;
  }
}

// Number of table regions for an L2-blocked insert of n device-resident pairs; 1 = insert in caller order.
// Worth it only when the store is well beyond the L2 and the batch is large enough to amortise the routing
// pass.  BHT_REGION_MB (environment) overrides the region size; 0 disables blocking.
uint32_t blocked_regions(const bht_table* t, uint64_t n) {
  const long region_mb = knobs().region_mb;
  if (region_mb <= 0 || t->blocked_insert == 0 || n > 0x7FFFFFFFull) return 1;
  const uint64_t store_bytes = t->cfg.capacity * sizeof(uint64_t);
  const bool forced = t->blocked_insert >= 2;  // bht_set_blocked_insert(table, 2): route whatever the sizes (tests)
  // Only the cuckoo tables are routed by default.  Processing the pairs in H0 order correlates arrival time with
  // the first candidate bucket; evictions make bcht / 1cht indifferent to that (same probe counts, same success),
  // but the balanced placements of bp2ht / iht are order-sensitive: early regions spill into everybody's second
  // choice and the last regions find both candidates full (bp2ht b=16 LF 0.8, 50 M keys: 9302 pairs dropped).
  const bool cuckoo = t->cfg.kind == BHT_BCHT || t->cfg.kind == BHT_ONE_CHT;
  if (!cuckoo) return 1;  // not even when forced: a routed bp2ht / iht build is a different (worse) table
  if (!forced && (n < (4ull << 20) || store_bytes < (192ull << 20))) return 1;
  uint64_t r = (store_bytes + (static_cast<uint64_t>(region_mb) << 20) - 1) / (static_cast<uint64_t>(region_mb) << 20);
  if (forced && r < 4) r = 4;
  if (r > static_cast<uint64_t>(kMaxShards)) r = kMaxShards;
  if (r >= t->cfg.num_buckets) r = t->cfg.num_buckets - 1;  // the router needs n_regions < hash range
  return static_cast<uint32_t>(r < 2 ? 1 : r);
}

// Plan of a shared-memory-blocked build (build_blocked.cu) of n device-resident pairs, n_regions == 0 when it is
// not used: the default for large bcht batches (1.06 ms against 1.81 ms for the L2-routed build, b = 16, 50 M pairs,
// LF 0.9); tables beyond 8 GB of slots (more than 256 x 256 fine regions of 128 KiB) take the L2-routed build.
BlockedPlan smem_blocked_plan(const bht_table* t, uint64_t n) {
  BlockedPlan none{};
  const bool cuckoo = t->cfg.kind == BHT_BCHT || t->cfg.kind == BHT_ONE_CHT;
  if (!cuckoo || n == 0 || t->blocked_insert == 0 || t->blocked_insert == 2) return none;
  const bool forced = t->blocked_insert == 3;
  if (!forced) {
    // 1cht takes the L2-routed build by default: the blocked build makes every first attempt before any eviction walk,
    // which at b = 1 shifts the probe means 1.6-3 % below the reference's interleaved process (2.0225 against 2.0554
    // probes per insert at LF 0.8) for a 4-9 % gain in time; at b = 16 the shift is 0.1 % and the gain 50 %.
    if (t->cfg.kind != BHT_BCHT) return none;
    if (knobs().smem_build == 0) return none;
    const uint64_t store_bytes = t->cfg.capacity * sizeof(uint64_t);
    // every region is read / written once whatever n: only for batches that are a sizeable part of the table
    if (n < (4ull << 20) || store_bytes < (192ull << 20) || n * 8 < t->cfg.capacity) return none;
  }
  return plan_blocked_build(t->view, n);
}

// Resident CTAs per SM of the insert kernel of a routed build: with the probes L2-resident a few hundred keys in
// flight per SM saturate the path, and fewer keys in flight mean fewer lost slot races inside the region.
// BHT_BLOCKED_CTAS (environment) overrides; 0 = whatever fits.
int blocked_ctas_per_sm() {
  return static_cast<int>(knobs().blocked_ctas);
}

// Optional (bht_set_tail_throttle): the last pairs of a cuckoo build that ends at a very high load are inserted with
// few keys in flight.  Measured (tools/exp_success_inflight.py, exp_success_tail.py, exp_success_tailcfg.py; bcht b = 16,
// LF 0.99, profiles/r01j_lf099_success_vs_concurrency.txt): with 190 k insertions in flight to the end, 50 % of 5 M-key
// builds succeed, with 4 k in flight 68 %, with 256 in flight 95 %; the CPU reference: 90 %.  Only the end matters — the
// last 2 % of the pairs at 256 in flight: 88 % — and it is not about the long chains themselves (finishing every chain
// past 24 evictions in a single CTA changes nothing): when the walkers in flight are as many as the free slots that
// remain, they take the slots each other was heading for, and max_chain, which the reference calibrates for one walker
// at a time, is hit 3-5 times more often.  With the throttle the pairs that arrive beyond load 0.98 go in a second
// launch whose grid keeps the keys in flight at or below 1/24 of the slots that will still be free at the end: 82 % of
// 5 M-key builds succeed, for 2.5x the build time.  It is OFF by default because retrying a failed build with fresh
// hash constants (what the reference's trial protocol does) is cheaper than throttling: 0.96 ms against 1.59 ms per
// successful 5 M-key build, 4.3 ms against 6.2 ms at 50 M keys.
struct TailPlan {
  uint64_t tail = 0;  // pairs at the end of the batch that get the throttled launch
  int grid = 0;       // its CTA cap
};
TailPlan tail_plan(const bht_table* t, uint64_t n) {
  TailPlan p;
  if (t->cfg.kind != BHT_BCHT && t->cfg.kind != BHT_ONE_CHT) return p;
  bool on = t->tail_throttle;
  if (knobs().tail_throttle >= 0) on = knobs().tail_throttle != 0;  // experiment override
  if (!on) return p;
  const double cap = static_cast<double>(t->cfg.capacity);
  const uint32_t b = t->cfg.bucket_size;
  double lf = b == 1 ? 0.85 : (b == 2 ? 0.90 : (b == 4 ? 0.95 : 0.98));
  if (knobs().tail_lf > 0.0) lf = knobs().tail_lf;
  const uint64_t before = std::min<uint64_t>(t->host_inserted, t->cfg.capacity);
  const uint64_t after = std::min<uint64_t>(before + n, t->cfg.capacity);
  const uint64_t threshold = static_cast<uint64_t>(lf * cap);
  if (after <= threshold) return p;
  p.tail = std::min<uint64_t>(n, after - std::max(before, threshold));
  const uint64_t free_at_end = t->cfg.capacity - after;
  const uint64_t divisor = static_cast<uint64_t>(std::max(1l, knobs().tail_div));
  const uint64_t lanes = std::max<uint64_t>(256, free_at_end / divisor);
  p.grid = static_cast<int>(std::min<uint64_t>((lanes + 255) / 256, 1u << 20));
  if (p.grid >= t->sm_count * 4) p = TailPlan{};  // no real throttle: one launch
  return p;
}

// Deferring the fill pays when the next build is likely to be the shared-memory-blocked one (which writes every slot
// itself): bcht tables beyond the L2 in the default mode, any cuckoo table when that build is forced.  Everything else
// is filled at once, so that no later call pays for it.
bool defer_fill_pays(const bht_table* t) {
  const bool cuckoo = t->cfg.kind == BHT_BCHT || t->cfg.kind == BHT_ONE_CHT;
  if (!cuckoo || t->blocked_insert == 0 || t->blocked_insert == 2) return false;
  if (t->blocked_insert == 3) return true;
  return t->cfg.kind == BHT_BCHT && t->cfg.capacity * sizeof(uint64_t) >= (192ull << 20);
}

// Orders `stream` after a deferred fill that another stream ran and that may still be in flight.
cudaError_t order_after_fill(bht_table* t, cudaStream_t stream) {
  if (!t->fill_recorded.load(std::memory_order_acquire)) return cudaSuccess;
  if (cudaEventQuery(t->fill_done) == cudaSuccess) {  // long done: nothing to order against any more
    t->fill_recorded.store(false, std::memory_order_release);
    return cudaSuccess;
  }
  cudaGetLastError();  // cudaErrorNotReady is not an error
  return stream == t->fill_stream ? cudaSuccess : cudaStreamWaitEvent(stream, t->fill_done, 0);
}

// Writes the empty pattern a deferred create / clear still owes (caller holds t->mu, or is the only user of t), and
// orders `stream` after the fill when an earlier call ran it on another stream.
cudaError_t materialize_clear(bht_table* t, cudaStream_t stream) {
  if (!t->clear_pending.load(std::memory_order_acquire)) return order_after_fill(t, stream);
  cudaError_t e = launch_fill_empty(t->view.store, t->cfg.capacity, t->sm_count, stream);
  if (e == cudaSuccess) e = cudaEventRecord(t->fill_done, stream);
  if (e == cudaSuccess) {
    t->fill_stream = stream;
    t->fill_recorded.store(true, std::memory_order_release);
    t->clear_pending.store(false, std::memory_order_release);
  }
  return e;
}

bool kind_matches(int32_t table_kind, int32_t as_kind) {
  // bcht_insert / bcht_find accept both cuckoo kinds (table.cpp:55,96)
  const bool cuckoo = table_kind == BHT_ONE_CHT || table_kind == BHT_BCHT;
  if (as_kind == BHT_BCHT || as_kind == BHT_ONE_CHT) return cuckoo;
  return table_kind == as_kind;
}

// Stream-ordered scratch from the library's own pool of the table's device (see scratch_pool).
cudaError_t scratch_alloc(const bht_table* t, void** p, size_t bytes, cudaStream_t stream) {
  cudaMemPool_t pool = scratch_pool(t->device);
  return pool != nullptr ? cudaMallocFromPoolAsync(p, bytes, pool, stream) : cudaMallocAsync(p, bytes, stream);
}

// Finishes a shared-memory-blocked build whose pairs are all in the group segments: K10 + K11, then the general kernel
// over the spill list (its length stays on the device).  The deferred fill is cancelled only once K11 is enqueued.
cudaError_t finish_blocked(bht_table* t, const BlockedPlan& plan, uint64_t n, void* scratch, bool fresh, bool fused_fill,
                           cudaStream_t stream) {
  PairSource spill{};
  const unsigned long long* spill_count = nullptr;
  cudaError_t e = blocked_build_finish(t->view, plan, n, scratch, fresh, FailLog{t->ctr, t->failed_keys, kFailedLogCap}, t->sm_count,
                                       stream, &spill, &spill_count);
  if (e != cudaSuccess) return e;
  if (fused_fill) t->clear_pending.store(false, std::memory_order_release);  // the region build writes every slot of the store
  e = cudaEventRecord(t->phase_ev[1], stream);
  if (e == cudaSuccess) e = launch_insert_kind(t, spill, n, 0, stream, false, spill_count);
  return e;
}

bht_status do_insert(bht_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, int32_t mem_space,
                     bht_insert_result* result, void* stream_v) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_insert: null table");
  if (n != 0 && keys == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_insert: null keys");
  if (mem_space != BHT_MEM_DEVICE && mem_space != BHT_MEM_HOST) return fail(BHT_INVALID_ARGUMENT, "bht_insert: bad mem_space");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->session.active) return fail(BHT_INVALID_ARGUMENT, "bht_insert: a chunked build (bht_build_begin) is open on this table");
  cudaStream_t stream = as_stream(stream_v);
  // values == NULL: the keys-only build of the reference, every key paired with value_for_key(key) (table.cpp:234).
  // Host callers then ship keys only; the values are made on the device.
  const bool derive = values == nullptr;
  struct AsyncBuffer {  // stream-ordered scratch, released on every exit path
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~AsyncBuffer() { if (p != nullptr) cudaFreeAsync(p, s); }
  } derived, scratch;
  derived.s = scratch.s = stream;

  BHT_CUDA(cudaMemsetAsync(t->ctr, 0, kPerCallCounterBytes, stream));
  const TailPlan tail = tail_plan(t, n);
  const uint64_t n_all = n;
  n -= tail.tail;  // the schedules below take the first part of the batch, the throttled launch the rest
  if (mem_space == BHT_MEM_DEVICE) {
    BHT_CUDA(cudaEventRecord(t->phase_ev[0], stream));
    const BlockedPlan plan = smem_blocked_plan(t, n);
    const uint32_t regions = plan.n_regions != 0 ? 1 : blocked_regions(t, n);
    // a blocked build into the known-empty table writes every slot itself: the fill it still owes is fused into it
    const bool fused_fill = plan.n_regions != 0 && t->known_empty && n != 0 && t->clear_pending.load(std::memory_order_acquire);
    if (!fused_fill) BHT_CUDA(materialize_clear(t, stream));
    if (derive && n_all != 0 && (plan.n_regions == 0 || tail.tail != 0)) {
      // the shared-memory-blocked build makes the values in its first pass; every other schedule reads an array
      BHT_CUDA(scratch_alloc(t, &derived.p, n_all * sizeof(uint32_t), stream));
      BHT_CUDA(launch_derive_values(keys, static_cast<uint32_t*>(derived.p), n_all, t->sm_count, stream));
      if (plan.n_regions == 0) values = static_cast<const uint32_t*>(derived.p);
    }
    const uint32_t* tail_values = derive ? static_cast<const uint32_t*>(derived.p) : values;
    if (plan.n_regions != 0) {
      // Shared-memory-blocked build (build_blocked.cu): bin the pairs by the shared-memory-sized table region of
      // their first bucket, build every region in shared memory, then run the general kernel over the pairs whose
      // first bucket was full (their count stays on the device).
      BHT_CUDA(scratch_alloc(t, &scratch.p, blocked_scratch_bytes(plan, n), stream));
      cudaError_t e = blocked_build_begin(plan, n, scratch.p, stream);
      if (e == cudaSuccess)
        e = blocked_build_scatter(t->view, plan, n, scratch.p, keys, values, n, FailLog{t->ctr, t->failed_keys, kFailedLogCap},
                                  t->sm_count, stream);
      if (e == cudaSuccess) e = finish_blocked(t, plan, n, scratch.p, t->known_empty, fused_fill, stream);
      if (e != cudaSuccess) return cuda_fail(e, "bht_insert (shared-memory blocked)");
      t->last_schedule = 3;
    } else if (regions > 1) {
      // L2-blocked build: group the pairs by the table region of their first bucket, then insert region by
      // region, so that bucket fetches, claims and the write-back of dirty sectors happen while the region
      // is L2-resident (the probe kernels deal their input out as one sliding window, probe_engine.cuh).
      // scratch: n packed {key, value} pairs | counts | cursors | n destination bytes
      BHT_CUDA(scratch_alloc(t, &scratch.p, 2 * n * sizeof(uint32_t) + 2 * regions * sizeof(unsigned long long) + n, stream));
      uint32_t* packed = static_cast<uint32_t*>(scratch.p);
      unsigned long long* counts = reinterpret_cast<unsigned long long*>(packed + 2 * n);
      uint8_t* dest8 = reinterpret_cast<uint8_t*>(counts + 2 * regions);
      cudaError_t e = launch_region_route(t->view.h[0], regions, keys, values, n, dest8, counts, counts + regions, packed,
                                          t->sm_count, stream);
      if (e == cudaSuccess) e = cudaEventRecord(t->phase_ev[1], stream);
      if (e == cudaSuccess) e = launch_insert_kind(t, PairSource{packed, nullptr}, n, blocked_ctas_per_sm(), stream, true);
      if (e != cudaSuccess) return cuda_fail(e, "bht_insert (blocked)");
      t->last_schedule = 2;
    } else {
      BHT_CUDA(cudaEventRecord(t->phase_ev[1], stream));
      BHT_CUDA(launch_insert_kind(t, PairSource{keys, values}, n, 0, stream));
      t->last_schedule = 0;
    }
    if (tail.tail != 0)
      BHT_CUDA(launch_insert_kind(t, PairSource{keys + n, tail_values + n}, tail.tail, 0, stream, false, nullptr, tail.grid));
    BHT_CUDA(cudaEventRecord(t->phase_ev[2], stream));
    t->phases_recorded = true;
  } else if (n_all != 0) {
    // Host-resident arrays: chunks cross PCIe through the staging slots while the device works on the chunks that have
    // arrived.  A batch that qualifies for the shared-memory-blocked build feeds every chunk to its first partition
    // pass (K8g) as it lands and runs the rest (K10, K11, the walks) once the last chunk is in; everything else goes
    // through the general kernel chunk by chunk.  The call returns when the caller's arrays have been read; the device
    // work still in flight is ordered before anything enqueued later on `stream` or done later with this table.
    n = n_all;
    const uint64_t n_main = n_all - tail.tail;
    bht_status s = ensure_staging(t);
    if (s != BHT_OK) return s;
    Staging& st = t->stage;
    const BlockedPlan plan = tail.tail == 0 ? smem_blocked_plan(t, n) : BlockedPlan{};
    const bool blocked = plan.n_regions != 0;
    t->last_schedule = blocked ? 3 : 0;
    const bool fused_fill = blocked && t->known_empty && t->clear_pending.load(std::memory_order_acquire);
    if (!fused_fill) BHT_CUDA(materialize_clear(t, stream));
    cudaEvent_t start = st.out_done[0];  // reuse as the "counters are zeroed" marker
    BHT_CUDA(cudaEventRecord(start, stream));
    BHT_CUDA(cudaStreamWaitEvent(st.compute, start, 0));
    scratch.s = st.compute;
    if (blocked) {
      BHT_CUDA(scratch_alloc(t, &scratch.p, blocked_scratch_bytes(plan, n), st.compute));
      BHT_CUDA(blocked_build_begin(plan, n, scratch.p, st.compute));
    }
    uint64_t chunks = 0;
    for (uint64_t c = 0, off = 0; off < n; ++c) {
      const int slot = static_cast<int>(c % kStageSlots);
      uint64_t len = stage_chunk_len(off, n);
      if (off < n_main) len = std::min(len, n_main - off);  // a chunk is either before or inside the throttled tail
      chunks = c + 1;
      // the slot's last consumer — of this call or of an earlier one whose device work is still in flight — is done
      BHT_CUDA(cudaStreamWaitEvent(st.h2d, st.kernel_done[slot], 0));
      BHT_CUDA(cudaMemcpyAsync(st.keys[slot], keys + off, len * sizeof(uint32_t), cudaMemcpyHostToDevice, st.h2d));
      if (!derive) BHT_CUDA(cudaMemcpyAsync(st.vals[slot], values + off, len * sizeof(uint32_t), cudaMemcpyHostToDevice, st.h2d));
      BHT_CUDA(cudaEventRecord(st.in_done[slot], st.h2d));
      BHT_CUDA(cudaStreamWaitEvent(st.compute, st.in_done[slot], 0));
      if (blocked) {
        BHT_CUDA(blocked_build_scatter(t->view, plan, n, scratch.p, st.keys[slot], derive ? nullptr : st.vals[slot], len,
                                       FailLog{t->ctr, t->failed_keys, kFailedLogCap}, t->sm_count, st.compute));
      } else {
        if (derive) BHT_CUDA(launch_derive_values(st.keys[slot], st.vals[slot], len, t->sm_count, st.compute));
        BHT_CUDA(launch_insert_kind(t, PairSource{st.keys[slot], st.vals[slot]}, len, 0, st.compute, false, nullptr,
                                    off >= n_main ? tail.grid : 0));
      }
      BHT_CUDA(cudaEventRecord(st.kernel_done[slot], st.compute));
      off += len;
    }
    if (blocked) {
      const cudaError_t e = finish_blocked(t, plan, n, scratch.p, t->known_empty, fused_fill, st.compute);
      if (e != cudaSuccess) return cuda_fail(e, "bht_insert (host buffers, shared-memory blocked)");
    }
    BHT_CUDA(cudaEventRecord(t->build_done, st.compute));
    BHT_CUDA(cudaStreamWaitEvent(stream, t->build_done, 0));
    BHT_CUDA(cudaEventSynchronize(st.in_done[(chunks - 1) % kStageSlots]));  // the caller's host arrays are free again on return
  }
  n = n_all;
  if (n != 0) t->known_empty = false;
  t->host_inserted = std::min<uint64_t>(t->host_inserted + n, t->cfg.capacity);
  if (result != nullptr) {
    bht_status s = read_counters(t, stream);
    if (s != BHT_OK) return s;
    fill_insert_result(t, n, result);
  }
  return BHT_OK;
}

// ---- a build whose pairs arrive in chunks (device-resident): bht_build_begin / _feed / _end ----------------------
bht_status session_begin(bht_table* t, uint64_t n_max, void* stream_v) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build_begin: null table");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->session.active) return fail(BHT_INVALID_ARGUMENT, "bht_build_begin: a chunked build is already open on this table");
  cudaStream_t stream = as_stream(stream_v);
  bht_table::Session ses;
  ses.n_max = n_max;
  ses.fresh = t->known_empty;
  BHT_CUDA(cudaMemsetAsync(t->ctr, 0, kPerCallCounterBytes, stream));
  BHT_CUDA(cudaEventRecord(t->phase_ev[0], stream));
  ses.plan = n_max != 0 ? smem_blocked_plan(t, n_max) : BlockedPlan{};
  ses.blocked = ses.plan.n_regions != 0;
  if (ses.blocked) {
    BHT_CUDA(scratch_alloc(t, &ses.scratch, blocked_scratch_bytes(ses.plan, n_max), stream));
    const cudaError_t e = blocked_build_begin(ses.plan, n_max, ses.scratch, stream);
    if (e != cudaSuccess) {
      cudaFreeAsync(ses.scratch, stream);
      return cuda_fail(e, "bht_build_begin");
    }
  }
  ses.active = true;
  t->session = ses;
  t->last_schedule = ses.blocked ? 3 : 0;
  return BHT_OK;
}

bht_status session_feed(bht_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, void* stream_v,
                        const unsigned long long* n_dev = nullptr) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build_feed: null table");
  if (n != 0 && keys == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build_feed: null keys");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  bht_table::Session& ses = t->session;
  if (!ses.active) return fail(BHT_INVALID_ARGUMENT, "bht_build_feed: no chunked build is open (bht_build_begin)");
  // a device-counted chunk only names an upper bound: what actually arrives beyond n_max is dropped and reported as
  // failed insertions by the kernels (build_blocked.cu, Spill::cap)
  if (n_dev == nullptr && ses.fed + n > ses.n_max)
    return fail(BHT_CAPACITY_EXCEEDED, "bht_build_feed: more pairs than bht_build_begin announced");
  cudaStream_t stream = as_stream(stream_v);
  if (n == 0) return BHT_OK;
  if (n_dev != nullptr && !ses.blocked && t->cfg.kind != BHT_BCHT && t->cfg.kind != BHT_ONE_CHT)
    return fail(BHT_INVALID_ARGUMENT, "bht_build_feed_counted: device-side counts are for the cuckoo kinds");
  if (ses.blocked) {
    BHT_CUDA(blocked_build_scatter(t->view, ses.plan, ses.n_max, ses.scratch, keys, values, n,
                                   FailLog{t->ctr, t->failed_keys, kFailedLogCap}, t->sm_count, stream, n_dev));
  } else {
    BHT_CUDA(materialize_clear(t, stream));
    void* derived = nullptr;
    if (values == nullptr) {
      BHT_CUDA(scratch_alloc(t, &derived, n * sizeof(uint32_t), stream));
      const cudaError_t e = launch_derive_values(keys, static_cast<uint32_t*>(derived), n, t->sm_count, stream);
      if (e != cudaSuccess) {
        cudaFreeAsync(derived, stream);
        return cuda_fail(e, "bht_build_feed");
      }
      values = static_cast<const uint32_t*>(derived);
    }
    const cudaError_t e = launch_insert_kind(t, PairSource{keys, values}, n, 0, stream, false, n_dev);
    if (derived != nullptr) cudaFreeAsync(derived, stream);
    if (e != cudaSuccess) return cuda_fail(e, "bht_build_feed");
    t->known_empty = false;
  }
  ses.fed += n;
  return BHT_OK;
}

bht_status session_end(bht_table* t, bht_insert_result* result, void* stream_v) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build_end: null table");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  bht_table::Session& ses = t->session;
  if (!ses.active) return fail(BHT_INVALID_ARGUMENT, "bht_build_end: no chunked build is open (bht_build_begin)");
  cudaStream_t stream = as_stream(stream_v);
  cudaError_t e = cudaSuccess;
  if (ses.blocked) {
    if (ses.fed != 0) {
      const bool fused_fill = ses.fresh && t->known_empty && t->clear_pending.load(std::memory_order_acquire);
      if (!fused_fill) e = materialize_clear(t, stream);
      if (e == cudaSuccess) e = finish_blocked(t, ses.plan, ses.n_max, ses.scratch, ses.fresh && t->known_empty, fused_fill, stream);
    }
    cudaFreeAsync(ses.scratch, stream);
  } else {
    e = cudaEventRecord(t->phase_ev[1], stream);
  }
  const uint64_t fed = ses.fed;
  ses = bht_table::Session{};
  if (e != cudaSuccess) return cuda_fail(e, "bht_build_end");
  BHT_CUDA(cudaEventRecord(t->phase_ev[2], stream));
  t->phases_recorded = true;
  if (fed != 0) t->known_empty = false;
  t->host_inserted = std::min<uint64_t>(t->host_inserted + fed, t->cfg.capacity);
  if (result != nullptr) {
    const bht_status s = read_counters(t, stream);
    if (s != BHT_OK) return s;
    // every fed pair ends up inserted or failed; with device-counted chunks `fed` is only an upper bound
    fill_insert_result(t, t->ctr_host->inserted + t->ctr_host->failed, result);
  }
  return BHT_OK;
}

bht_status do_find(const bht_table* ct, bool early_exit, const uint32_t* keys, uint32_t* out, uint64_t n,
                   int32_t mem_space, bht_find_result* result, void* stream_v) {
  if (ct == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_find: null table");
  if (n != 0 && (keys == nullptr || out == nullptr)) return fail(BHT_INVALID_ARGUMENT, "bht_find: null keys / out_values");
  if (mem_space != BHT_MEM_DEVICE && mem_space != BHT_MEM_HOST) return fail(BHT_INVALID_ARGUMENT, "bht_find: bad mem_space");
  bht_table* t = const_cast<bht_table*>(ct);  // the counter block and staging buffers are scratch state
  BHT_ON_DEVICE(t->device);
  cudaStream_t stream = as_stream(stream_v);

  if (t->clear_pending.load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(t->mu);
    BHT_CUDA(materialize_clear(t, stream));
  } else {
    BHT_CUDA(order_after_fill(t, stream));
  }
  if (mem_space == BHT_MEM_DEVICE && result == nullptr) {
    // lock-free: concurrent finds on different streams share nothing but the read-only store
    uint32_t* cursor = nullptr;
    BHT_CUDA(next_cursor(t, stream, &cursor));
    BHT_CUDA(launch_find(t->view, early_exit, keys, out, n, nullptr, cursor, t->sm_count, stream));
    return BHT_OK;
  }

  std::lock_guard<std::mutex> lock(t->mu);
  DevCounters* ctr = result != nullptr ? t->ctr : nullptr;
  if (ctr != nullptr) BHT_CUDA(cudaMemsetAsync(t->ctr, 0, kPerCallCounterBytes, stream));
  if (mem_space == BHT_MEM_DEVICE) {
    uint32_t* cursor = nullptr;
    BHT_CUDA(next_cursor(t, stream, &cursor));
    BHT_CUDA(launch_find(t->view, early_exit, keys, out, n, ctr, cursor, t->sm_count, stream));
  } else if (n != 0) {
    bht_status s = ensure_staging(t);
    if (s != BHT_OK) return s;
    Staging& st = t->stage;
    // everything already queued on the caller's stream (inserts, the counter reset) precedes the chunks
    cudaEvent_t start = st.in_done[0];
    BHT_CUDA(cudaEventRecord(start, stream));
    BHT_CUDA(cudaStreamWaitEvent(st.compute, start, 0));
    uint64_t chunks = 0;
    const bool device_idle = cudaEventQuery(t->build_done) == cudaSuccess;  // no host-buffer build still in flight
    if (!device_idle) cudaGetLastError();
    for (uint64_t c = 0, off = 0; off < n; ++c) {
      const int slot = static_cast<int>(c % kStageSlots);
      const uint64_t len = stage_chunk_len(off, n, device_idle);
      chunks = c + 1;
      // (also against the kernels of an earlier host-buffer insert, which returns before its device work is done)
      BHT_CUDA(cudaStreamWaitEvent(st.h2d, st.kernel_done[slot], 0));                       // keys[slot] consumed
      if (c >= kStageSlots) BHT_CUDA(cudaStreamWaitEvent(st.compute, st.out_done[slot], 0));  // vals[slot] drained
      BHT_CUDA(cudaMemcpyAsync(st.keys[slot], keys + off, len * sizeof(uint32_t), cudaMemcpyHostToDevice, st.h2d));
      BHT_CUDA(cudaEventRecord(st.in_done[slot], st.h2d));
      BHT_CUDA(cudaStreamWaitEvent(st.compute, st.in_done[slot], 0));
      uint32_t* cursor = nullptr;
      BHT_CUDA(next_cursor(t, st.compute, &cursor));
      BHT_CUDA(launch_find(t->view, early_exit, st.keys[slot], st.vals[slot], len, ctr, cursor, t->sm_count, st.compute));
      BHT_CUDA(cudaEventRecord(st.kernel_done[slot], st.compute));
      BHT_CUDA(cudaStreamWaitEvent(st.d2h, st.kernel_done[slot], 0));
      BHT_CUDA(cudaMemcpyAsync(out + off, st.vals[slot], len * sizeof(uint32_t), cudaMemcpyDeviceToHost, st.d2h));
      BHT_CUDA(cudaEventRecord(st.out_done[slot], st.d2h));
      off += len;
    }
    BHT_CUDA(cudaStreamWaitEvent(stream, st.kernel_done[(chunks - 1) % kStageSlots], 0));
    BHT_CUDA(cudaStreamSynchronize(st.d2h));  // answers are in the caller's host array on return
    BHT_CUDA(cudaStreamSynchronize(stream));
  }
  if (result != nullptr) {
    bht_status s = read_counters(t, stream);
    if (s != BHT_OK) return s;
    result->queries = n;
    result->hits = t->ctr_host->find_hits;
    result->probes = t->ctr_host->find_probes;
    result->value_sum = t->ctr_host->find_value_sum;
  }
  return BHT_OK;
}

}  // namespace

extern "C" {

// ---- configuration ------------------------------------------------------------------------------

uint32_t bht_hash_count(int32_t kind) { return hash_count_of(kind); }

uint32_t bht_default_max_chain(uint64_t n_keys) {
  // default_max_chain (core.cpp:28-31): max(7 * ceil(log2 n), 128), ceil(log2 n) = bit_width(n - 1)
  uint32_t log2n = 1;
  if (n_keys > 1) {
    log2n = 0;
    for (uint64_t v = n_keys - 1; v != 0; v >>= 1) ++log2n;
  }
  return std::max<uint32_t>(7u * log2n, 128u);
}

uint64_t bht_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

uint64_t bht_bucket_index_host(uint64_t alpha, uint64_t beta, uint64_t range, uint32_t key) {
  if (alpha > 0xFFFFFFFFull || beta > 0xFFFFFFFFull || range == 0 || range > 0xFFFFFFFFull) {
    g_error = "bht_bucket_index_host: alpha, beta and range must fit 32 bits, range > 0";
    return ~0ull;
  }
  return bucket_index(make_hash_fn(alpha, beta, range), key);
}

uint32_t bht_value_for_key(uint32_t key) {
  // value_for_key (keygen.hpp:23-26): k ^ 0x5A5A5A5A; the one image that hits the sentinel is masked
  const uint32_t v = key ^ 0x5A5A5A5Au;
  return v == BHT_EMPTY_VALUE ? (v & 0x7FFFFFFFu) : v;
}

double bht_predict_sectors(int32_t kind, uint32_t bucket_size, double mean_probes, int32_t op) {
  // sector_model.hpp:18-31: a bucket read costs ceil(8b/32) sectors, 2 for 1cht (DRAM-to-L2 granularity is
  // 64 bytes); an insert adds the one sector its atomic writes back.
  const double per_probe = kind == BHT_ONE_CHT ? 2.0 : static_cast<double>((bucket_size * 8u + 31u) / 32u);
  return mean_probes * per_probe + (op == 0 ? 1.0 : 0.0);
}

bht_status bht_make_config(int32_t kind, uint64_t n_keys, double lf, uint32_t bucket_size, int64_t threshold,
                           uint64_t seed, int64_t max_chain, bht_config* out) {
  if (out == nullptr) return fail(BHT_INVALID_ARGUMENT, "make_config: null output");
  if (hash_count_of(kind) == 0) return fail(BHT_INVALID_ARGUMENT, "make_config: unknown table kind");
  // core.cpp:40-46, same order and messages
  if (n_keys == 0) return fail(BHT_INVALID_ARGUMENT, "make_config: n_keys must be positive");
  if (!(lf > 0.0) || lf > 1.0) return fail(BHT_INVALID_ARGUMENT, "make_config: load factor must be in (0, 1]");
  if (!is_pow2(bucket_size) || bucket_size > BHT_MAX_BUCKET_SIZE)
    return fail(BHT_INVALID_ARGUMENT, "make_config: bucket_size must be a power of two in [1, 64]");
  if (kind == BHT_ONE_CHT && bucket_size != 1) return fail(BHT_INVALID_ARGUMENT, "make_config: 1cht requires bucket_size 1");

  bht_config c;
  std::memset(&c, 0, sizeof c);
  c.kind = kind;
  c.bucket_size = bucket_size;
  c.num_buckets = static_cast<uint64_t>(std::ceil(static_cast<double>(n_keys) / (lf * static_cast<double>(bucket_size))));
  c.capacity = c.num_buckets * bucket_size;
  c.seed = seed;
  c.n_hashes = hash_count_of(kind);
  if (kind == BHT_IHT) {
    c.threshold = threshold >= 0 ? static_cast<uint32_t>(threshold) : bucket_size * 80u / 100u;
    if (c.threshold > bucket_size) return fail(BHT_INVALID_ARGUMENT, "make_config: threshold exceeds bucket_size");
    if (c.threshold == 0) return fail(BHT_INVALID_ARGUMENT, "make_config: iht threshold must be positive");
  }
  if (kind == BHT_ONE_CHT || kind == BHT_BCHT)
    c.max_chain = max_chain >= 0 ? static_cast<uint32_t>(max_chain) : bht_default_max_chain(n_keys);

  // draw_hash_params (keygen.cpp:14-26) on xorshift_rng(mix_seed(seed, 0x68617368)) (core.cpp:65-66)
  uint64_t rng = xorshift_init(mix_seed(seed, 0x68617368ull));
  const uint32_t p = static_cast<uint32_t>(BHT_HASH_PRIME);
  for (uint32_t i = 0; i < c.n_hashes; ++i) {
    c.alpha[i] = 1ull + xorshift_next_below(rng, p - 1u);
    c.beta[i] = xorshift_next_below(rng, p);
    c.range[i] = c.num_buckets;
  }
  *out = c;
  return BHT_OK;
}

// ---- lifetime -----------------------------------------------------------------------------------

bht_status bht_create(const bht_config* cfg, int32_t device, bht_table** out) {
  if (cfg == nullptr || out == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_create: null argument");
  *out = nullptr;
  bht_status vs = validate_config(*cfg);
  if (vs != BHT_OK) return vs;
  int n_dev = 0;
  BHT_CUDA(cudaGetDeviceCount(&n_dev));
  if (device < 0 || device >= n_dev) return fail(BHT_CUDA_ERROR, "bht_create: no such CUDA device");
  BHT_ON_DEVICE(device);

  bht_table* t = new (std::nothrow) bht_table();
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_create: out of host memory");
  t->cfg = *cfg;
  t->device = device;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e == cudaSuccess && prop.major < 10) {
    delete t;
    return fail(BHT_CUDA_ERROR, "bht_create: kernels are built for sm_100a only; this device is older");
  }
  if (e == cudaSuccess) t->sm_count = prop.multiProcessorCount;
  scratch_pool_acquire(device);

  uint64_t* store = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&store, cfg->capacity * sizeof(uint64_t));  // cudaMalloc aligns to >= 256 B
  if (e == cudaSuccess) e = cudaMalloc(&t->ctr, sizeof(DevCounters));
  if (e == cudaSuccess) e = cudaMallocHost(&t->ctr_host, sizeof(DevCounters));
  if (e == cudaSuccess) e = cudaMalloc(&t->failed_keys, 2 * kFailedLogCap * sizeof(uint32_t));  // keys, then values
  if (e == cudaSuccess) e = cudaMalloc(&t->cursors, kCursorSlots * sizeof(uint32_t));
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) e = cudaEventCreate(&t->phase_ev[i]);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t->fill_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t->build_done, cudaEventDisableTiming);
  if (e == cudaSuccess && (cfg->kind == BHT_BP2HT || cfg->kind == BHT_IHT)) {
    e = cudaMalloc(&t->loads, claim_loads_bytes(cfg->num_buckets));
    if (e == cudaSuccess) e = cudaMemset(t->loads, 0, claim_loads_bytes(cfg->num_buckets));
    t->loads_valid = e == cudaSuccess;
  }
  if (e == cudaSuccess) e = cudaMemset(t->ctr, 0, sizeof(DevCounters));
  t->cfg = *cfg;
  t->repair_dropped = cfg->kind == BHT_BCHT;
  if (defer_fill_pays(t)) t->clear_pending.store(true);  // filled by its first user (materialize_clear) or by a blocked build
  else if (e == cudaSuccess) e = launch_fill_empty(store, cfg->capacity, t->sm_count, nullptr);
  if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  if (e != cudaSuccess) {
    if (store) cudaFree(store);
    if (t->ctr) cudaFree(t->ctr);
    if (t->ctr_host) cudaFreeHost(t->ctr_host);
    if (t->failed_keys) cudaFree(t->failed_keys);
    if (t->cursors) cudaFree(t->cursors);
    if (t->loads) cudaFree(t->loads);
    for (cudaEvent_t ev : t->phase_ev)
      if (ev) cudaEventDestroy(ev);
    if (t->fill_done) cudaEventDestroy(t->fill_done);
    if (t->build_done) cudaEventDestroy(t->build_done);
    scratch_pool_release(device);
    delete t;
    return cuda_fail(e, "bht_create");
  }

  TableView& v = t->view;
  v.store = store;
  for (uint32_t i = 0; i < cfg->n_hashes; ++i) v.h[i] = make_hash_fn(cfg->alpha[i], cfg->beta[i], cfg->range[i]);
  for (uint32_t i = cfg->n_hashes; i < 4; ++i) v.h[i] = make_hash_fn(1, 0, 1);
  v.num_buckets = cfg->num_buckets;
  v.seed = cfg->seed;
  v.n_hashes = cfg->n_hashes;
  v.bucket_size = cfg->bucket_size;
  v.threshold = cfg->threshold;
  v.max_chain = cfg->max_chain;
  v.prose = 0;
  v.retry_cap = kRetryCap;
  {
    const long c = knobs().chunk_log2;
    v.chunk_log2 = static_cast<uint32_t>(c < 5 ? 5 : (c > 16 ? 16 : c));
  }
  *out = t;
  return BHT_OK;
}

bht_status bht_destroy(bht_table* t) {
  if (t == nullptr) return BHT_OK;
  BHT_ON_DEVICE(t->device);
  cudaDeviceSynchronize();
  release_staging(t->stage);
  cudaFree(t->view.store);
  cudaFree(t->ctr);
  cudaFreeHost(t->ctr_host);
  cudaFree(t->failed_keys);
  cudaFree(t->cursors);
  if (t->loads) cudaFree(t->loads);
  for (cudaEvent_t ev : t->phase_ev)
    if (ev) cudaEventDestroy(ev);
  if (t->session.active && t->session.scratch != nullptr) cudaFree(t->session.scratch);
  if (t->fill_done) cudaEventDestroy(t->fill_done);
  if (t->build_done) cudaEventDestroy(t->build_done);
  scratch_pool_release(t->device);
  delete t;
  return BHT_OK;
}

bht_status bht_clear(bht_table* t, void* stream) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_clear: null table");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->session.active) return fail(BHT_INVALID_ARGUMENT, "bht_clear: a chunked build (bht_build_begin) is open on this table");
  if (defer_fill_pays(t)) {
    t->clear_pending.store(true, std::memory_order_release);  // deferred, see bht_table::clear_pending
  } else {
    BHT_CUDA(launch_fill_empty(t->view.store, t->cfg.capacity, t->sm_count, as_stream(stream)));
    t->clear_pending.store(false, std::memory_order_release);
  }
  BHT_CUDA(cudaMemsetAsync(t->ctr, 0, sizeof(DevCounters), as_stream(stream)));
  t->known_empty = true;
  t->host_inserted = 0;
  if (t->loads != nullptr) {
    BHT_CUDA(cudaMemsetAsync(t->loads, 0, claim_loads_bytes(t->cfg.num_buckets), as_stream(stream)));
    t->loads_valid = true;
  }
  return BHT_OK;
}

bht_status bht_get_config(const bht_table* t, bht_config* out) {
  if (t == nullptr || out == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_get_config: null argument");
  *out = t->cfg;
  return BHT_OK;
}

int32_t bht_device_of(const bht_table* t) { return t ? t->device : -1; }

// ---- the hot path -------------------------------------------------------------------------------

bht_status bht_insert(bht_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, int32_t mem_space,
                      bht_insert_result* result, void* stream) {
  return do_insert(t, keys, values, n, mem_space, result, stream);
}

bht_status bht_build(const bht_config* cfg, int32_t device, const uint32_t* keys, const uint32_t* values, uint64_t n,
                     int32_t mem_space, int32_t iht_prose_fallback, bht_table** out, bht_insert_result* result, void* stream) {
  if (cfg == nullptr || out == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build: null argument");
  *out = nullptr;
  // build(): the capacity check comes before the table exists (table.cpp:225)
  if (n > cfg->capacity) return fail(BHT_CAPACITY_EXCEEDED, "build: key set exceeds table capacity");
  bht_table* t = nullptr;
  bht_status s = bht_create(cfg, device, &t);
  if (s != BHT_OK) return s;
  if (iht_prose_fallback && cfg->kind == BHT_IHT) t->view.prose = 1u;
  s = do_insert(t, keys, values, n, mem_space, result, stream);
  if (s != BHT_OK) {
    bht_destroy(t);
    return s;
  }
  *out = t;
  return BHT_OK;
}

bht_status bht_build_begin(bht_table* t, uint64_t n_max, void* stream) { return session_begin(t, n_max, stream); }
bht_status bht_build_feed(bht_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n, void* stream) {
  return session_feed(t, keys, values, n, stream);
}
bht_status bht_build_feed_counted(bht_table* t, const uint32_t* keys, const uint32_t* values, uint64_t n_cap,
                                  const uint64_t* n_dev, void* stream) {
  if (n_dev == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_build_feed_counted: null device count");
  return session_feed(t, keys, values, n_cap, stream, reinterpret_cast<const unsigned long long*>(n_dev));
}
bht_status bht_build_end(bht_table* t, bht_insert_result* result, void* stream) { return session_end(t, result, stream); }

bht_status bht_insert_as(bht_table* t, int32_t kind, const uint32_t* keys, const uint32_t* values, uint64_t n,
                         int32_t mem_space, bht_insert_result* result, void* stream) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_insert_as: null table");
  if (!kind_matches(t->cfg.kind, kind)) return fail(BHT_KIND_MISMATCH, "insert: table kind does not match the variant");
  return do_insert(t, keys, values, n, mem_space, result, stream);
}

bht_status bht_find(const bht_table* t, const uint32_t* keys, uint32_t* out, uint64_t n, int32_t mem_space,
                    bht_find_result* result, void* stream) {
  const bool cuckoo = t != nullptr && (t->cfg.kind == BHT_ONE_CHT || t->cfg.kind == BHT_BCHT);
  return do_find(t, cuckoo, keys, out, n, mem_space, result, stream);
}

bht_status bht_find_as(const bht_table* t, int32_t kind, const uint32_t* keys, uint32_t* out, uint64_t n,
                       int32_t mem_space, bht_find_result* result, void* stream) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_find_as: null table");
  if (!kind_matches(t->cfg.kind, kind)) return fail(BHT_KIND_MISMATCH, "find: table kind does not match the variant");
  return bht_find(t, keys, out, n, mem_space, result, stream);
}

bht_status bht_find_exhaustive(const bht_table* t, const uint32_t* keys, uint32_t* out, uint64_t n, int32_t mem_space,
                               bht_find_result* result, void* stream) {
  return do_find(t, false, keys, out, n, mem_space, result, stream);
}

bht_status bht_last_insert_result(bht_table* t, bht_insert_result* out, void* stream) {
  if (t == nullptr || out == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_last_insert_result: null argument");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  bht_status s = read_counters(t, as_stream(stream));
  if (s != BHT_OK) return s;
  const DevCounters& c = *t->ctr_host;
  fill_insert_result(t, c.inserted + c.failed, out);
  return BHT_OK;
}

bht_status bht_failed_keys(bht_table* t, uint32_t* host_out, uint64_t max_keys, uint64_t* count) {
  if (t == nullptr || count == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_failed_keys: null argument");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  BHT_CUDA(cudaDeviceSynchronize());
  bht_status s = read_counters(t, nullptr);
  if (s != BHT_OK) return s;
  *count = t->ctr_host->failed_recorded;
  const uint64_t n = std::min<uint64_t>(std::min<uint64_t>(*count, kFailedLogCap), max_keys);
  if (n != 0 && host_out != nullptr)
    BHT_CUDA(cudaMemcpy(host_out, t->failed_keys, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return BHT_OK;
}

bht_status bht_last_insert_phases(bht_table* t, float* prepare_ms, float* probe_ms) {
  if (t == nullptr || prepare_ms == nullptr || probe_ms == nullptr)
    return fail(BHT_INVALID_ARGUMENT, "bht_last_insert_phases: null argument");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  if (!t->phases_recorded) return fail(BHT_INVALID_ARGUMENT, "bht_last_insert_phases: no device-resident insert yet");
  BHT_CUDA(cudaEventSynchronize(t->phase_ev[2]));
  BHT_CUDA(cudaEventElapsedTime(prepare_ms, t->phase_ev[0], t->phase_ev[1]));
  BHT_CUDA(cudaEventElapsedTime(probe_ms, t->phase_ev[1], t->phase_ev[2]));
  return BHT_OK;
}

bht_status bht_set_iht_prose_fallback(bht_table* t, int32_t enabled) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_set_iht_prose_fallback: null table");
  if (t->cfg.kind != BHT_IHT) return fail(BHT_KIND_MISMATCH, "iht_insert: table kind does not match the variant");
  t->view.prose = enabled ? 1u : 0u;
  return BHT_OK;
}

bht_status bht_set_repair(bht_table* t, int32_t enabled) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_set_repair: null table");
  t->repair_dropped = enabled != 0;
  return BHT_OK;
}

bht_status bht_set_tail_throttle(bht_table* t, int32_t enabled) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_set_tail_throttle: null table");
  t->tail_throttle = enabled != 0;
  return BHT_OK;
}

int32_t bht_last_build_schedule(const bht_table* t) { return t != nullptr ? t->last_schedule : -1; }

bht_status bht_set_blocked_insert(bht_table* t, int32_t enabled) {
  if (t == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_set_blocked_insert: null table");
  if (enabled < 0 || enabled > 3) return fail(BHT_INVALID_ARGUMENT, "bht_set_blocked_insert: mode must be 0, 1, 2 or 3");
  t->blocked_insert = enabled;
  return BHT_OK;
}

// ---- load factor / store access -----------------------------------------------------------------

bht_status bht_load_factor(const bht_table* ct, uint64_t* inserted, uint64_t* capacity) {
  if (ct == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_load_factor: null table");
  bht_table* t = const_cast<bht_table*>(ct);
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  BHT_CUDA(cudaDeviceSynchronize());
  bht_status s = read_counters(t, nullptr);
  if (s != BHT_OK) return s;
  if (inserted) *inserted = t->ctr_host->inserted_total;
  if (capacity) *capacity = t->cfg.capacity;
  return BHT_OK;
}

bht_status bht_count_occupied(const bht_table* ct, uint64_t* occupied, void* stream) {
  if (ct == nullptr || occupied == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_count_occupied: null argument");
  bht_table* t = const_cast<bht_table*>(ct);
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  BHT_CUDA(materialize_clear(t, as_stream(stream)));
  BHT_CUDA(launch_count_occupied(t->view.store, t->cfg.capacity, &t->ctr->scratch, t->sm_count, as_stream(stream)));
  bht_status s = read_counters(t, as_stream(stream));
  if (s != BHT_OK) return s;
  *occupied = t->ctr_host->scratch;
  return BHT_OK;
}

bht_status bht_count_inadmissible(const bht_table* ct, uint64_t* violations, void* stream) {
  if (ct == nullptr || violations == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_count_inadmissible: null argument");
  bht_table* t = const_cast<bht_table*>(ct);
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  BHT_CUDA(materialize_clear(t, as_stream(stream)));
  BHT_CUDA(launch_count_inadmissible(t->view, &t->ctr->scratch, t->sm_count, as_stream(stream)));
  bht_status s = read_counters(t, as_stream(stream));
  if (s != BHT_OK) return s;
  *violations = t->ctr_host->scratch;
  return BHT_OK;
}

bht_status bht_download_store(const bht_table* t, uint64_t* host_dst, void* stream) {
  if (t == nullptr || host_dst == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_download_store: null argument");
  BHT_ON_DEVICE(t->device);
  {
    bht_table* mt = const_cast<bht_table*>(t);
    std::lock_guard<std::mutex> lock(mt->mu);
    BHT_CUDA(materialize_clear(mt, as_stream(stream)));
  }
  BHT_CUDA(cudaMemcpyAsync(host_dst, t->view.store, t->cfg.capacity * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                           as_stream(stream)));
  BHT_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return BHT_OK;
}

bht_status bht_upload_store(bht_table* t, const uint64_t* host_src, void* stream) {
  if (t == nullptr || host_src == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_upload_store: null argument");
  BHT_ON_DEVICE(t->device);
  std::lock_guard<std::mutex> lock(t->mu);
  cudaStream_t s = as_stream(stream);
  t->known_empty = false;
  t->loads_valid = false;
  t->clear_pending.store(false, std::memory_order_release);  // every slot is overwritten
  BHT_CUDA(cudaMemcpyAsync(t->view.store, host_src, t->cfg.capacity * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  BHT_CUDA(cudaMemsetAsync(t->ctr, 0, sizeof(DevCounters), s));
  BHT_CUDA(launch_count_occupied(t->view.store, t->cfg.capacity, &t->ctr->inserted_total, t->sm_count, s));
  const bht_status rs = read_counters(t, s);
  if (rs == BHT_OK) t->host_inserted = t->ctr_host->inserted_total;
  return rs;
}

bht_status bht_dump_store(const bht_table* t, const char* path) {
  if (t == nullptr || path == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_dump_store: null argument");
  const uint64_t n = t->cfg.capacity;
  uint64_t* host = static_cast<uint64_t*>(std::malloc(n * sizeof(uint64_t)));
  if (host == nullptr) return fail(BHT_IO_ERROR, "dump_store: out of host memory");
  bht_status s = bht_download_store(t, host, nullptr);
  if (s != BHT_OK) {
    std::free(host);
    return s;
  }
  std::FILE* f = std::fopen(path, "wb");
  if (f == nullptr) {
    std::free(host);
    return fail(BHT_IO_ERROR, std::string("dump_store: cannot open ") + path);
  }
  // little-endian u64 per slot in bucket order (table.cpp:41-51); every supported host is little-endian
  const bool ok = std::fwrite(host, sizeof(uint64_t), n, f) == n;
  const bool closed = std::fclose(f) == 0;
  std::free(host);
  if (!ok || !closed) return fail(BHT_IO_ERROR, std::string("dump_store: write failed for ") + path);
  return BHT_OK;
}

uint64_t* bht_device_store(const bht_table* t) {
  if (t == nullptr) return nullptr;
  bht_table* mt = const_cast<bht_table*>(t);
  {
    std::lock_guard<std::mutex> lock(mt->mu);
    if (mt->clear_pending.load()) {  // the caller gets a store that is what the API said it was, whatever stream it uses next
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(mt->device);
      if (materialize_clear(mt, nullptr) == cudaSuccess) cudaStreamSynchronize(nullptr);
      cudaSetDevice(prev);
    }
  }
  mt->known_empty = false;  // the caller may write slots behind the library's back
  mt->loads_valid = false;
  return t->view.store;
}

// ---- hash stage in isolation ----------------------------------------------------------------------

bht_status bht_hash_keys(uint64_t alpha, uint64_t beta, uint64_t range, const uint32_t* keys, uint32_t* out, uint64_t n,
                         int32_t mem_space, int32_t device, void* stream) {
  if (alpha > 0xFFFFFFFFull || beta > 0xFFFFFFFFull || range == 0 || range > 0xFFFFFFFFull)
    return fail(BHT_INVALID_ARGUMENT, "bht_hash_keys: alpha, beta and range must fit 32 bits, range > 0");
  if (n != 0 && (keys == nullptr || out == nullptr)) return fail(BHT_INVALID_ARGUMENT, "bht_hash_keys: null argument");
  BHT_ON_DEVICE(device);
  const int sm_count_dev = device_sm_count(device);
  const HashFn h = make_hash_fn(alpha, beta, range);
  cudaStream_t s = as_stream(stream);
  if (mem_space == BHT_MEM_DEVICE) {
    BHT_CUDA(launch_hash_keys(h, keys, out, n, sm_count_dev, s));
    return BHT_OK;
  }
  if (n == 0) return BHT_OK;
  uint32_t *dk = nullptr, *dout = nullptr;
  BHT_CUDA(cudaMalloc(&dk, n * sizeof(uint32_t)));
  cudaError_t e = cudaMalloc(&dout, n * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dk, keys, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_hash_keys(h, dk, dout, n, sm_count_dev, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(dk);
  if (dout) cudaFree(dout);
  if (e != cudaSuccess) return cuda_fail(e, "bht_hash_keys");
  return BHT_OK;
}

// ---- sharded table: routing -------------------------------------------------------------------------

uint32_t bht_shard_of_host(uint64_t alpha, uint64_t beta, uint32_t n_shards, uint32_t key) {
  return shard_of(static_cast<uint32_t>(alpha), static_cast<uint32_t>(beta), n_shards, key);
}

bht_status bht_shard_partition(uint64_t alpha, uint64_t beta, uint32_t n_shards, const uint32_t* keys,
                               const uint32_t* values, uint64_t n, uint32_t* out_keys, uint32_t* out_values,
                               uint32_t* out_index, uint64_t* counts_host, int32_t device, void* stream) {
  if (alpha > 0xFFFFFFFFull || beta > 0xFFFFFFFFull) return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition: constants must fit 32 bits");
  if (n_shards == 0 || n_shards > static_cast<uint32_t>(kMaxShards))
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition: n_shards must be in [1, 256]");
  if (n > 0xFFFFFFFFull) return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition: at most 2^32 - 1 elements per call");
  if (counts_host == nullptr || (n != 0 && (keys == nullptr || out_keys == nullptr)) || (values != nullptr && out_values == nullptr))
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition: null argument");
  BHT_ON_DEVICE(device);
  const int sm_count_dev = device_sm_count(device);
  cudaStream_t s = as_stream(stream);
  unsigned long long* scratch = nullptr;  // counts | cursors | n destination bytes
  BHT_CUDA(cudaMallocAsync(&scratch, 2 * sizeof(unsigned long long) * n_shards + n, s));
  const uint32_t a = static_cast<uint32_t>(alpha), b = static_cast<uint32_t>(beta);
  cudaError_t e = launch_shard_route(a, b, n_shards, keys, values, n, reinterpret_cast<uint8_t*>(scratch + 2 * n_shards), scratch,
                                     scratch + n_shards, out_keys, out_values,
                                     out_index, sm_count_dev, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(counts_host, scratch, sizeof(uint64_t) * n_shards, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(scratch, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "bht_shard_partition");
  return BHT_OK;
}

bht_status bht_shard_partition_fixed(uint64_t alpha, uint64_t beta, uint32_t n_shards, const uint32_t* keys,
                                     const uint32_t* values, uint64_t n, uint64_t cap, uint32_t* out_keys, uint32_t* out_values,
                                     uint32_t* out_index, uint64_t* counts_dev, uint32_t* overflow_dev, int32_t device,
                                     void* stream) {
  if (alpha > 0xFFFFFFFFull || beta > 0xFFFFFFFFull) return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition_fixed: constants must fit 32 bits");
  if (n_shards == 0 || n_shards > static_cast<uint32_t>(kMaxShards))
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition_fixed: n_shards must be in [1, 256]");
  if (n > 0xFFFFFFFFull || cap == 0 || cap * n_shards > 0xFFFFFFFFull)
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition_fixed: at most 2^32 - 1 elements / output slots per call");
  if (counts_dev == nullptr || overflow_dev == nullptr || (n != 0 && (keys == nullptr || out_keys == nullptr)) ||
      (values != nullptr && out_values == nullptr))
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition_fixed: null argument");
  if (values != nullptr && out_index != nullptr)
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_partition_fixed: an element carries its value (inserts) or its position (finds), not both");
  BHT_ON_DEVICE(device);
  const int sm_count = device_sm_count(device);
  cudaStream_t s = as_stream(stream);
  uint32_t* scratch = nullptr;  // one cursor word per destination
  BHT_CUDA(cudaMallocAsync(&scratch, sizeof(uint32_t) * n_shards, s));
  // index mode without values: the second output array carries the positions; a keys-only call carries nothing
  const cudaError_t e = launch_shard_split_fixed(static_cast<uint32_t>(alpha), static_cast<uint32_t>(beta), n_shards, keys, values, n, cap,
                                                 scratch, reinterpret_cast<unsigned long long*>(counts_dev), overflow_dev, out_keys,
                                                 out_values, out_index, sm_count, s);
  cudaFreeAsync(scratch, s);
  if (e != cudaSuccess) return cuda_fail(e, "bht_shard_partition_fixed");
  return BHT_OK;
}

bht_status bht_shard_unpermute(const uint32_t* answers, const uint32_t* index, uint64_t n, uint32_t* out, int32_t device,
                               void* stream) {
  if (n != 0 && (answers == nullptr || index == nullptr || out == nullptr))
    return fail(BHT_INVALID_ARGUMENT, "bht_shard_unpermute: null argument");
  BHT_ON_DEVICE(device);
  const int sm_count_dev = device_sm_count(device);
  BHT_CUDA(launch_unpermute(answers, index, n, out, sm_count_dev, as_stream(stream)));
  return BHT_OK;
}

// ---- synthetic workload ------------------------------------------------------------------------------

bht_status bht_generate_unique_keys(uint64_t seed, uint64_t offset, uint64_t n, uint32_t* out_keys, uint32_t* out_values,
                                    int32_t device, void* stream) {
  if (n != 0 && out_keys == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_generate_unique_keys: null output");
  if (offset + n > 0xFFFFFFFFull || offset + n < offset)
    return fail(BHT_INVALID_ARGUMENT, "bht_generate_unique_keys: offset + n exceeds the 2^32 - 1 user keys");
  BHT_ON_DEVICE(device);
  const int sm_count_dev = device_sm_count(device);
  BHT_CUDA(launch_generate_keys(seed, offset, n, out_keys, out_values, sm_count_dev, as_stream(stream)));
  return BHT_OK;
}

uint32_t bht_unique_key_host(uint64_t seed, uint32_t counter) {
  return unique_key(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), counter);
}
uint32_t bht_synthetic_value_host(uint64_t seed, uint32_t key) { return synthetic_value(static_cast<uint32_t>(seed >> 32), key); }

// ---- pinned host buffers for BHT_MEM_HOST callers -----------------------------------------------------

bht_status bht_host_alloc(size_t bytes, void** out) {
  if (out == nullptr) return fail(BHT_INVALID_ARGUMENT, "bht_host_alloc: null output");
  BHT_CUDA(cudaMallocHost(out, bytes));
  return BHT_OK;
}
bht_status bht_host_free(void* p) {
  if (p != nullptr) BHT_CUDA(cudaFreeHost(p));
  return BHT_OK;
}

// ---- diagnostics -------------------------------------------------------------------------------------

void bht_reload_tuning(void) { knobs_storage() = load_knobs(); }
const char* bht_last_error_string(void) { return g_error.c_str(); }
const char* bht_version_string(void) { return "bht_b200 0.1 (sm_100a)"; }
uint64_t bht_kernel_launch_count(void) { return launch_count(); }
size_t bht_sizeof_config(void) { return sizeof(bht_config); }

}  // extern "C"
