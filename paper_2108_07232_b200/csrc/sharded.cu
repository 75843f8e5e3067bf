// sharded.cu — the sharded table handle of the C ABI: one process, G shards, every shard an ordinary single-GPU table
// on its own device (no reference counterpart: the reference is single-process).
//
// Ownership is a function of the key alone, owner(k) = (g(k) * G) >> 32 with g(k) = (a*k + b) mod p an independent
// member of the table's hash family (hash.hpp:21-23), so all candidate buckets of a key live in one shard.
//
//   insert:  per source device  K8 partition by owner (util.cu)  ->  counts to the host  ->  peer copies of the (key,
//            value) runs into the owners' receive buffers (cudaMemcpyPeerAsync: NVLink between devices with peer access,
//            a plain device copy inside one device)  ->  every owner's bulk insert, all devices at once
//   find:    partition with the original positions  ->  peer copies of the key runs  ->  every owner's bulk find  ->
//            peer copies of the answer runs back  ->  K9 un-permute into the caller's order on the source device
//
// The multi-process variant of the same scheme (one rank per GPU, NCCL all-to-all) is paper_2108_07232_b200/sharded.py;
// both route with the same constants (bht_shard_constants) and so build the same shards.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/bht_b200.h"
#include "kernels.h"

namespace bht_b200 {
void set_last_error(const std::string& msg);  // capi.cu
}

using namespace bht_b200;

namespace {

bht_status sh_fail(bht_status s, const std::string& msg) {
  set_last_error(msg);
  return s;
}
bht_status sh_cuda_fail(cudaError_t e, const char* what) {
  set_last_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return BHT_CUDA_ERROR;
}
#define SH_CUDA(expr)                                          \
  do {                                                         \
    cudaError_t e__ = (expr);                                  \
    if (e__ != cudaSuccess) return sh_cuda_fail(e__, #expr);   \
  } while (0)
#define SH_OK(expr)                       \
  do {                                    \
    bht_status s__ = (expr);              \
    if (s__ != BHT_OK) return s__;        \
  } while (0)

struct DeviceGuard {  // the caller's current device is restored on every exit path
  int prev = 0;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// A device buffer that only ever grows (the handle keeps its routing buffers between calls).
struct Grow {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p != nullptr) {
      cudaError_t e = cudaFree(p);
      if (e != cudaSuccess) return e;
      p = nullptr;
      bytes = 0;
    }
    want += want / 8 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p != nullptr) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct Shard {
  int device = 0;
  int sm_count = 0;
  bht_table* table = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t sent = nullptr, done = nullptr;
  // source side: the caller's slice grouped by owner; owner side: what the other shards sent
  Grow send_keys, send_vals, send_index, route_scratch, recv_keys, recv_vals, answers;
};

}  // namespace

struct bht_sharded {
  std::vector<Shard> shards;
  uint32_t alpha = 1, beta = 0;
  bht_config cfg{};
};

namespace {

uint64_t splitmix64_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void destroy_shards(bht_sharded* s) {
  for (Shard& sh : s->shards) {
    cudaSetDevice(sh.device);
    if (sh.table) bht_destroy(sh.table);
    for (Grow* g : {&sh.send_keys, &sh.send_vals, &sh.send_index, &sh.route_scratch, &sh.recv_keys, &sh.recv_vals, &sh.answers}) g->release();
    if (sh.sent) cudaEventDestroy(sh.sent);
    if (sh.done) cudaEventDestroy(sh.done);
    if (sh.stream) cudaStreamDestroy(sh.stream);
  }
  s->shards.clear();
}

// Partition every source slice by owner.  counts[g * G + d] = elements of source g owned by shard d.
bht_status route_all(bht_sharded* s, const uint32_t* const* keys, const uint32_t* const* values, const uint64_t* n, bool with_values,
                     bool with_index, std::vector<uint64_t>& counts) {
  const uint32_t G = static_cast<uint32_t>(s->shards.size());
  counts.assign(static_cast<size_t>(G) * G, 0);
  for (uint32_t g = 0; g < G; ++g) {
    Shard& sh = s->shards[g];
    if (n[g] == 0) continue;
    if (n[g] > 0xFFFFFFFFull) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded: at most 2^32 - 1 elements per slice");
    if (keys[g] == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded: null key slice");
    SH_CUDA(cudaSetDevice(sh.device));
    SH_CUDA(sh.send_keys.reserve(n[g] * sizeof(uint32_t)));
    if (with_values) SH_CUDA(sh.send_vals.reserve(n[g] * sizeof(uint32_t)));
    if (with_index) SH_CUDA(sh.send_index.reserve(n[g] * sizeof(uint32_t)));
    SH_CUDA(sh.route_scratch.reserve(2 * sizeof(unsigned long long) * G + n[g] + 16));
    unsigned long long* cnt = sh.route_scratch.as<unsigned long long>();
    const uint32_t* vals = with_values ? values[g] : nullptr;
    uint32_t* derived = nullptr;
    if (with_values && vals == nullptr) {  // keys-only build: value_for_key(key), made on the source device (table.cpp:234)
      SH_CUDA(sh.answers.reserve(n[g] * sizeof(uint32_t)));
      derived = sh.answers.as<uint32_t>();
      SH_CUDA(launch_derive_values(keys[g], derived, n[g], sh.sm_count, sh.stream));
      vals = derived;
    }
    SH_CUDA(launch_shard_route(s->alpha, s->beta, G, keys[g], vals, n[g], reinterpret_cast<uint8_t*>(cnt + 2 * G), cnt, cnt + G,
                               sh.send_keys.as<uint32_t>(), with_values ? sh.send_vals.as<uint32_t>() : nullptr,
                               with_index ? sh.send_index.as<uint32_t>() : nullptr, sh.sm_count, sh.stream));
    SH_CUDA(cudaMemcpyAsync(&counts[static_cast<size_t>(g) * G], cnt, sizeof(uint64_t) * G, cudaMemcpyDeviceToHost, sh.stream));
  }
  for (uint32_t g = 0; g < G; ++g) {
    SH_CUDA(cudaSetDevice(s->shards[g].device));
    SH_CUDA(cudaStreamSynchronize(s->shards[g].stream));
  }
  return BHT_OK;
}

}  // namespace

extern "C" {

void bht_shard_constants(uint64_t seed, uint64_t* alpha, uint64_t* beta) {
  // drawn as draw_hash_params does (keygen.cpp:14-26) from xorshift_rng(mix_seed(seed, 'shar')): independent of the
  // table's own constants, the same in every process
  uint64_t state = splitmix64_host(bht_mix_seed(seed, 0x73686172ull));
  if (state == 0) state = 0xD1B54A32D192ED03ull;
  auto next_below = [&state](uint64_t bound) {
    uint64_t x = state;
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    state = x;
    return ((x >> 32) * bound) >> 32;
  };
  const uint64_t a = 1 + next_below(4294967291ull - 1), b = next_below(4294967291ull);
  if (alpha) *alpha = a;
  if (beta) *beta = b;
}

bht_status bht_sharded_create(const bht_config* cfg_per_shard, uint32_t n_shards, const int32_t* device_ids, bht_sharded** out) {
  if (cfg_per_shard == nullptr || device_ids == nullptr || out == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_create: null argument");
  *out = nullptr;
  if (n_shards == 0 || n_shards > static_cast<uint32_t>(kMaxShards)) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_create: n_shards must be in [1, 256]");
  DeviceGuard guard;
  bht_sharded* s = new bht_sharded();
  s->cfg = *cfg_per_shard;
  uint64_t a = 0, b = 0;
  bht_shard_constants(cfg_per_shard->seed, &a, &b);
  s->alpha = static_cast<uint32_t>(a);
  s->beta = static_cast<uint32_t>(b);
  s->shards.resize(n_shards);
  bht_status st = BHT_OK;
  for (uint32_t g = 0; g < n_shards && st == BHT_OK; ++g) {
    Shard& sh = s->shards[g];
    sh.device = device_ids[g];
    cudaDeviceProp prop;
    cudaError_t e = cudaSetDevice(sh.device);
    if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, sh.device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sh.sent, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sh.done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      st = sh_cuda_fail(e, "bht_sharded_create");
      break;
    }
    sh.sm_count = prop.multiProcessorCount;
    st = bht_create(cfg_per_shard, sh.device, &sh.table);
  }
  // peer access between every pair of distinct devices that supports it (the copies fall back to staging otherwise)
  for (uint32_t g = 0; g < n_shards && st == BHT_OK; ++g)
    for (uint32_t d = 0; d < n_shards; ++d) {
      const int a_dev = s->shards[g].device, b_dev = s->shards[d].device;
      if (a_dev == b_dev) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, a_dev, b_dev) == cudaSuccess && can) {
        cudaSetDevice(a_dev);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b_dev, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) st = sh_cuda_fail(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();  // clear "already enabled"
      }
    }
  if (st != BHT_OK) {
    destroy_shards(s);
    delete s;
    return st;
  }
  *out = s;
  return BHT_OK;
}

bht_status bht_sharded_destroy(bht_sharded* s) {
  if (s == nullptr) return BHT_OK;
  DeviceGuard guard;
  destroy_shards(s);
  delete s;
  return BHT_OK;
}

uint32_t bht_sharded_count(const bht_sharded* s) { return s == nullptr ? 0u : static_cast<uint32_t>(s->shards.size()); }

bht_status bht_sharded_table(bht_sharded* s, uint32_t shard, bht_table** out) {
  if (s == nullptr || out == nullptr || shard >= s->shards.size()) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_table: bad argument");
  *out = s->shards[shard].table;
  return BHT_OK;
}

bht_status bht_sharded_clear(bht_sharded* s) {
  if (s == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_clear: null handle");
  DeviceGuard guard;
  for (Shard& sh : s->shards) SH_OK(bht_clear(sh.table, sh.stream));
  for (Shard& sh : s->shards) {
    SH_CUDA(cudaSetDevice(sh.device));
    SH_CUDA(cudaStreamSynchronize(sh.stream));
  }
  return BHT_OK;
}

bht_status bht_sharded_insert(bht_sharded* s, const uint32_t* const* keys, const uint32_t* const* values, const uint64_t* n,
                              bht_insert_result* result) {
  if (s == nullptr || keys == nullptr || n == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_insert: null argument");
  DeviceGuard guard;
  const uint32_t G = static_cast<uint32_t>(s->shards.size());
  std::vector<const uint32_t*> no_values(G, nullptr);
  if (values == nullptr) values = no_values.data();
  std::vector<uint64_t> counts;
  SH_OK(route_all(s, keys, values, n, true, false, counts));
  // receive layout on owner d: the runs of source 0, 1, ... G-1 back to back
  std::vector<uint64_t> recv_total(G, 0);
  for (uint32_t d = 0; d < G; ++d)
    for (uint32_t g = 0; g < G; ++g) recv_total[d] += counts[static_cast<size_t>(g) * G + d];
  for (uint32_t d = 0; d < G; ++d) {
    if (recv_total[d] > s->cfg.capacity) return sh_fail(BHT_CAPACITY_EXCEEDED, "build: key set exceeds table capacity");  // table.cpp:225, per shard
    Shard& owner = s->shards[d];
    SH_CUDA(cudaSetDevice(owner.device));
    SH_CUDA(owner.recv_keys.reserve(recv_total[d] * sizeof(uint32_t)));
    SH_CUDA(owner.recv_vals.reserve(recv_total[d] * sizeof(uint32_t)));
  }
  for (uint32_t g = 0; g < G; ++g) {
    Shard& src = s->shards[g];
    SH_CUDA(cudaSetDevice(src.device));
    uint64_t send_off = 0;
    for (uint32_t d = 0; d < G; ++d) {
      const uint64_t c = counts[static_cast<size_t>(g) * G + d];
      if (c != 0) {
        uint64_t recv_off = 0;
        for (uint32_t g2 = 0; g2 < g; ++g2) recv_off += counts[static_cast<size_t>(g2) * G + d];
        Shard& owner = s->shards[d];
        SH_CUDA(cudaMemcpyPeerAsync(owner.recv_keys.as<uint32_t>() + recv_off, owner.device, src.send_keys.as<uint32_t>() + send_off, src.device,
                                    c * sizeof(uint32_t), src.stream));
        SH_CUDA(cudaMemcpyPeerAsync(owner.recv_vals.as<uint32_t>() + recv_off, owner.device, src.send_vals.as<uint32_t>() + send_off, src.device,
                                    c * sizeof(uint32_t), src.stream));
      }
      send_off += c;
    }
    SH_CUDA(cudaEventRecord(src.sent, src.stream));
  }
  // every owner waits for all the senders, then inserts: the G bulk inserts run at the same time
  for (uint32_t d = 0; d < G; ++d) {
    Shard& owner = s->shards[d];
    SH_CUDA(cudaSetDevice(owner.device));
    for (uint32_t g = 0; g < G; ++g) SH_CUDA(cudaStreamWaitEvent(owner.stream, s->shards[g].sent, 0));
    if (recv_total[d] != 0)
      SH_OK(bht_insert(owner.table, owner.recv_keys.as<uint32_t>(), owner.recv_vals.as<uint32_t>(), recv_total[d], BHT_MEM_DEVICE, nullptr,
                       owner.stream));
    SH_CUDA(cudaEventRecord(owner.done, owner.stream));
  }
  bht_insert_result total{};
  total.first_failed_key = BHT_EMPTY_KEY;
  for (uint32_t d = 0; d < G; ++d) {
    Shard& owner = s->shards[d];
    bht_insert_result r{};
    if (recv_total[d] == 0) continue;  // nothing was sent to this shard
    SH_OK(bht_last_insert_result(owner.table, &r, owner.stream));  // synchronises the owner's stream
    total.attempted += recv_total[d];
    total.inserted += r.inserted;
    total.failed += r.failed;
    total.probes += r.probes;
    if (r.failed != 0 && total.first_failed_key == BHT_EMPTY_KEY) total.first_failed_key = r.first_failed_key;
  }
  // the senders' buffers are reused by the next call: make sure every copy out of them has finished
  for (uint32_t g = 0; g < G; ++g) {
    SH_CUDA(cudaSetDevice(s->shards[g].device));
    SH_CUDA(cudaStreamSynchronize(s->shards[g].stream));
  }
  total.success = total.inserted == total.attempted ? 1u : 0u;
  if (result != nullptr) *result = total;
  return BHT_OK;
}

bht_status bht_sharded_find(bht_sharded* s, const uint32_t* const* keys, uint32_t* const* out_values, const uint64_t* n,
                            bht_find_result* result) {
  if (s == nullptr || keys == nullptr || out_values == nullptr || n == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_find: null argument");
  DeviceGuard guard;
  const uint32_t G = static_cast<uint32_t>(s->shards.size());
  for (uint32_t g = 0; g < G; ++g)
    if (n[g] != 0 && out_values[g] == nullptr) return sh_fail(BHT_INVALID_ARGUMENT, "bht_sharded_find: null output slice");
  std::vector<uint64_t> counts;
  SH_OK(route_all(s, keys, nullptr, n, false, true, counts));
  std::vector<uint64_t> recv_total(G, 0);
  for (uint32_t d = 0; d < G; ++d)
    for (uint32_t g = 0; g < G; ++g) recv_total[d] += counts[static_cast<size_t>(g) * G + d];
  for (uint32_t d = 0; d < G; ++d) {
    Shard& owner = s->shards[d];
    SH_CUDA(cudaSetDevice(owner.device));
    SH_CUDA(owner.recv_keys.reserve(recv_total[d] * sizeof(uint32_t)));
    SH_CUDA(owner.recv_vals.reserve(recv_total[d] * sizeof(uint32_t)));  // the answers of the owned queries
  }
  for (uint32_t g = 0; g < G; ++g) {
    Shard& src = s->shards[g];
    SH_CUDA(cudaSetDevice(src.device));
    SH_CUDA(src.answers.reserve(n[g] * sizeof(uint32_t)));  // answers in routed order, before the un-permute
    uint64_t send_off = 0;
    for (uint32_t d = 0; d < G; ++d) {
      const uint64_t c = counts[static_cast<size_t>(g) * G + d];
      if (c != 0) {
        uint64_t recv_off = 0;
        for (uint32_t g2 = 0; g2 < g; ++g2) recv_off += counts[static_cast<size_t>(g2) * G + d];
        Shard& owner = s->shards[d];
        SH_CUDA(cudaMemcpyPeerAsync(owner.recv_keys.as<uint32_t>() + recv_off, owner.device, src.send_keys.as<uint32_t>() + send_off, src.device,
                                    c * sizeof(uint32_t), src.stream));
      }
      send_off += c;
    }
    SH_CUDA(cudaEventRecord(src.sent, src.stream));
  }
  bht_find_result total{};
  for (uint32_t d = 0; d < G; ++d) {
    Shard& owner = s->shards[d];
    SH_CUDA(cudaSetDevice(owner.device));
    for (uint32_t g = 0; g < G; ++g) SH_CUDA(cudaStreamWaitEvent(owner.stream, s->shards[g].sent, 0));
    if (recv_total[d] == 0) {
      SH_CUDA(cudaEventRecord(owner.done, owner.stream));
      continue;
    }
    if (result != nullptr) {  // per-shard statistics are read back shard by shard (the call synchronises the owner's stream)
      bht_find_result r{};
      SH_OK(bht_find(owner.table, owner.recv_keys.as<uint32_t>(), owner.recv_vals.as<uint32_t>(), recv_total[d], BHT_MEM_DEVICE, &r, owner.stream));
      total.queries += r.queries;
      total.hits += r.hits;
      total.probes += r.probes;
      total.value_sum += r.value_sum;
    } else {
      SH_OK(bht_find(owner.table, owner.recv_keys.as<uint32_t>(), owner.recv_vals.as<uint32_t>(), recv_total[d], BHT_MEM_DEVICE, nullptr,
                     owner.stream));
    }
    // the answer runs go back to where the queries came from, into the routed order of the source
    uint64_t recv_off = 0;
    for (uint32_t g = 0; g < G; ++g) {
      const uint64_t c = counts[static_cast<size_t>(g) * G + d];
      if (c != 0) {
        uint64_t send_off = 0;
        for (uint32_t d2 = 0; d2 < d; ++d2) send_off += counts[static_cast<size_t>(g) * G + d2];
        Shard& src = s->shards[g];
        SH_CUDA(cudaMemcpyPeerAsync(src.answers.as<uint32_t>() + send_off, src.device, owner.recv_vals.as<uint32_t>() + recv_off, owner.device,
                                    c * sizeof(uint32_t), owner.stream));
      }
      recv_off += c;
    }
    SH_CUDA(cudaEventRecord(owner.done, owner.stream));
  }
  for (uint32_t g = 0; g < G; ++g) {
    Shard& src = s->shards[g];
    if (n[g] == 0) continue;
    SH_CUDA(cudaSetDevice(src.device));
    for (uint32_t d = 0; d < G; ++d) SH_CUDA(cudaStreamWaitEvent(src.stream, s->shards[d].done, 0));
    SH_CUDA(launch_unpermute(src.answers.as<uint32_t>(), src.send_index.as<uint32_t>(), n[g], out_values[g], src.sm_count, src.stream));
  }
  for (uint32_t g = 0; g < G; ++g) {
    SH_CUDA(cudaSetDevice(s->shards[g].device));
    SH_CUDA(cudaStreamSynchronize(s->shards[g].stream));
  }
  if (result != nullptr) *result = total;
  return BHT_OK;
}

}  // extern "C"
