// warp_rank.cu — cost of ranking 32 keys among equals inside a warp, the primitive of an atomic-free partition:
//   match   __match_any_sync on a D-valued digit + popc                      (one MATCH.ANY)
//   ballot  log2(D) ballots + mask algebra (the K11 way)
//   atoms   shared-memory atomicAdd on a D-entry histogram (returns the rank; what the routers use today)
// Prints warp-steps per second per SM and the implied cycles per warp-step.   nvcc -arch=sm_100a -O3 warp_rank.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16; return x;
}

template <int MODE, int DBITS>
__global__ void __launch_bounds__(256) rank_kernel(uint32_t iters, unsigned long long* sink) {
  __shared__ uint32_t hist[8][1 << DBITS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (int i = lane; i < (1 << DBITS); i += 32) hist[warp][i] = 0;
  __syncwarp();
  uint32_t x = mix(blockIdx.x * 256 + threadIdx.x), acc = 0;
  for (uint32_t it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t d = x >> (32 - DBITS);
    if (MODE == 0) {
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
      const uint32_t rank = __popc(peers & lt);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) { base = hist[warp][d]; hist[warp][d] = base + __popc(peers); }  // private counter: plain RMW
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      acc += base + rank;
      __syncwarp();
    } else if (MODE == 1) {
      uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < DBITS; ++k) {
        const uint32_t mk = __ballot_sync(0xFFFFFFFFu, (d >> k) & 1u);
        peers &= ((d >> k) & 1u) ? mk : ~mk;
      }
      const uint32_t rank = __popc(peers & lt);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) { base = hist[warp][d]; hist[warp][d] = base + __popc(peers); }
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      acc += base + rank;
      __syncwarp();
    } else {
      acc += atomicAdd(&hist[warp][d], 1u);
    }
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int MODE, int DBITS>
void run(const char* name) {
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const uint32_t iters = 20000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148 * 8;
  rank_kernel<MODE, DBITS><<<grid, 256>>>(100, sink);
  cudaEventRecord(a);
  rank_kernel<MODE, DBITS><<<grid, 256>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double steps = double(grid) * 8 * iters;  // warp-steps
  const double per_sm_cycles = (ms * 1e-3 * 1.965e9) / (steps / 148);
  std::printf("%-7s D=%4d: %7.2f G keys/s, %6.2f SM-cycles per warp-step (32 keys)\n", name, 1 << DBITS, steps * 32 / (ms * 1e-3) / 1e9, per_sm_cycles);
  cudaFree(sink);
}

int main() {
  run<0, 5>("match"); run<1, 5>("ballot"); run<2, 5>("atoms");
  run<0, 8>("match"); run<1, 8>("ballot"); run<2, 8>("atoms");
  run<0, 9>("match"); run<1, 9>("ballot"); run<2, 9>("atoms");
  return 0;
}
