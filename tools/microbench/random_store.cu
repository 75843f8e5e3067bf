// random_store.cu — rate of random 8-byte stores (one per lane, each to a different 128-byte line) over a table of `mb`
// megabytes, with and without a preceding L2 atomicAdd on a 16-bit-per-bucket counter array (the "choose by counters,
// then store" build of the balanced tables).   nvcc -arch=sm_100a -O3 random_store.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16; return x;
}

template <int MODE>  // 0: store only; 1: two counter reads + atomicAdd + store
__global__ void __launch_bounds__(256) k(unsigned long long* table, uint32_t* cnt, uint32_t n_buckets, uint32_t per_thread) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < per_thread; ++i) {
    const uint32_t key = mix(tid * 0x9E3779B9u + i);
    const uint32_t b0 = static_cast<uint32_t>((static_cast<uint64_t>(key) * n_buckets) >> 32);
    uint32_t slot = key & 15u, b = b0;
    if (MODE == 1) {
      const uint32_t b1 = static_cast<uint32_t>((static_cast<uint64_t>(mix(key)) * n_buckets) >> 32);
      const uint32_t c0 = __ldcg(cnt + (b0 >> 1)), c1 = __ldcg(cnt + (b1 >> 1));
      b = ((c0 >> (16 * (b0 & 1))) & 0xFFFF) <= ((c1 >> (16 * (b1 & 1))) & 0xFFFF) ? b0 : b1;
      const uint32_t old = atomicAdd(cnt + (b >> 1), 1u << (16 * (b & 1)));
      slot = (old >> (16 * (b & 1))) & 15u;
    }
    table[static_cast<uint64_t>(b) * 16 + slot] = (static_cast<unsigned long long>(i) << 32) | key;
  }
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atol(argv[1]) : 444;
  const uint32_t n_buckets = static_cast<uint32_t>(mb * 1000000 / 128);
  unsigned long long* table; uint32_t* cnt;
  cudaMalloc(&table, static_cast<size_t>(n_buckets) * 128);
  cudaMalloc(&cnt, (n_buckets / 2 + 1) * 4);
  cudaMemset(table, 0xFF, static_cast<size_t>(n_buckets) * 128);
  const int grid = 148 * 8, per = 160;  // ~48.5 M stores
  const double ops = double(grid) * 256 * per;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cnt, 0, (n_buckets / 2 + 1) * 4);
      cudaEventRecord(a);
      if (mode == 0) k<0><<<grid, 256>>>(table, cnt, n_buckets, per); else k<1><<<grid, 256>>>(table, cnt, n_buckets, per);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) std::printf("%s over %zu MB: %.3f ms for %.1f M keys = %.1f G keys/s\n", mode ? "2 counter reads + atomicAdd + 8-byte store" : "8-byte store only", mb, ms, ops / 1e6, ops / ms / 1e6);
    }
  }
  return 0;
}
