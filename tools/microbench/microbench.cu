// microbench.cu — calibration of the two primitives the hash-table path is made of, on this GPU:
//   gather   random 128-byte-aligned 128-byte lines (8 lanes x 16 B, like a b=16 bucket probe)
//   cas      one 64-bit atomicCAS per lane at a random 8-byte slot
//   exch     one 64-bit atomicExch per lane at a random 8-byte slot
//   gcas     gather of a line followed by a CAS into that line (the insert pattern)
// over a table of `mb` megabytes.  Prints GB/s (gather) or G ops/s.   nvcc -arch=sm_100a -O3 microbench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16; return x;
}

template <int ILP>
__global__ void __launch_bounds__(256) gather_kernel(const uint4* __restrict__ table, uint32_t n_lines, uint32_t per_thread, unsigned long long* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t tile = tid >> 3, sub = tid & 7;
  uint32_t acc = 0;
  for (uint32_t i = 0; i < per_thread; i += ILP) {
    uint4 v[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      const uint32_t line = static_cast<uint32_t>((static_cast<uint64_t>(mix(tile * 0x9E3779B9u + i + j)) * n_lines) >> 32);
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(table + static_cast<uint64_t>(line) * 8 + sub));
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// mode 0 = CAS(expect current garbage -> fails, no write), 1 = CAS that succeeds (table pre-filled with ~0), 2 = EXCH
template <int MODE>
__global__ void __launch_bounds__(256) atomic_kernel(unsigned long long* table, uint32_t n_slots, uint32_t per_thread, unsigned long long* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < per_thread; ++i) {
    const uint32_t slot = static_cast<uint32_t>((static_cast<uint64_t>(mix(tid * 0x9E3779B9u + i * 0x7F4A7C15u)) * n_slots) >> 32);
    if (MODE == 2) acc += atomicExch(table + slot, static_cast<unsigned long long>(tid) << 32 | i);
    else acc += atomicCAS(table + slot, ~0ull, static_cast<unsigned long long>(tid) << 32 | i);
  }
  if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

// the insert pattern: 8 lanes read a line, then lane 0 of the tile CASes one slot of it (dependent)
__global__ void __launch_bounds__(256) gather_cas_kernel(unsigned long long* table, uint32_t n_lines, uint32_t per_thread, unsigned long long* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t tile = tid >> 3, sub = tid & 7;
  unsigned long long acc = 0;
  for (uint32_t i = 0; i < per_thread; ++i) {
    const uint32_t line = static_cast<uint32_t>((static_cast<uint64_t>(mix(tile * 0x9E3779B9u + i)) * n_lines) >> 32);
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(reinterpret_cast<const uint4*>(table) + static_cast<uint64_t>(line) * 8 + sub));
    const uint32_t slot = (v.x ^ i) & 15;
    if (sub == 0) acc += atomicCAS(table + static_cast<uint64_t>(line) * 16 + slot, ~0ull, static_cast<unsigned long long>(tid) << 32 | i);
  }
  if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

static float time_ms(void (*launch)(void*), void* ctx, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(ctx); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); launch(ctx); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

struct Ctx { void* table; uint32_t n_lines; uint32_t per_thread; int grid; unsigned long long* sink; int ilp; int mode; };

int main(int argc, char** argv) {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  unsigned long long* sink; cudaMalloc(&sink, 8); cudaMemset(sink, 0, 8);
  const int sizes_mb[] = {32, 444, 4440};
  printf("device %s, %d SMs\n", prop.name, sms);
  for (int mb : sizes_mb) {
    const uint64_t bytes = static_cast<uint64_t>(mb) * 1000000ull / 128 * 128;
    void* table; if (cudaMalloc(&table, bytes) != cudaSuccess) { printf("alloc %d MB failed\n", mb); continue; }
    const uint32_t n_lines = static_cast<uint32_t>(bytes / 128);
    for (int occ : {4, 8}) {
      Ctx c{table, n_lines, 512, sms * occ, sink, 0, 0};
      cudaMemset(table, 0xFF, bytes);
      const double lines = static_cast<double>(c.grid) * 256 / 8 * c.per_thread;
      float ms;
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; gather_kernel<1><<<c->grid, 256>>>((const uint4*)c->table, c->n_lines, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  gather ilp1 : %8.1f GB/s  (%.2f G lines/s)\n", mb, occ, lines * 128 / ms / 1e6, lines / ms / 1e6);
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; gather_kernel<4><<<c->grid, 256>>>((const uint4*)c->table, c->n_lines, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  gather ilp4 : %8.1f GB/s  (%.2f G lines/s)\n", mb, occ, lines * 128 / ms / 1e6, lines / ms / 1e6);
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; gather_kernel<8><<<c->grid, 256>>>((const uint4*)c->table, c->n_lines, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  gather ilp8 : %8.1f GB/s  (%.2f G lines/s)\n", mb, occ, lines * 128 / ms / 1e6, lines / ms / 1e6);
      c.per_thread = 64;
      const double ops = static_cast<double>(c.grid) * 256 * c.per_thread;
      cudaMemset(table, 0x11, bytes);
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; atomic_kernel<0><<<c->grid, 256>>>((unsigned long long*)c->table, c->n_lines * 16, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  cas (fail)  : %8.2f G ops/s\n", mb, occ, ops / ms / 1e6);
      cudaMemset(table, 0xFF, bytes);
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; atomic_kernel<1><<<c->grid, 256>>>((unsigned long long*)c->table, c->n_lines * 16, c->per_thread, c->sink); }, &c, 1);
      printf("table %5d MB  ctas/sm %d  cas (mixed) : %8.2f G ops/s\n", mb, occ, ops / ms / 1e6);
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; atomic_kernel<2><<<c->grid, 256>>>((unsigned long long*)c->table, c->n_lines * 16, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  exch        : %8.2f G ops/s\n", mb, occ, ops / ms / 1e6);
      cudaMemset(table, 0xFF, bytes);
      c.per_thread = 256;
      const double glines = static_cast<double>(c.grid) * 256 / 8 * c.per_thread;
      ms = time_ms([](void* p) { Ctx* c = (Ctx*)p; gather_cas_kernel<<<c->grid, 256>>>((unsigned long long*)c->table, c->n_lines, c->per_thread, c->sink); }, &c, 3);
      printf("table %5d MB  ctas/sm %d  gather+cas  : %8.2f G keys/s (%.1f GB/s of lines)\n", mb, occ, glines / ms / 1e6, glines * 128 / ms / 1e6);
    }
    cudaFree(table);
  }
  return 0;
}
