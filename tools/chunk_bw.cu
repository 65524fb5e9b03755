// chunk_bw.cu -- what HBM delivers for the AOT traversal's access pattern:
// contiguous chunks of C bytes (an out-list window) at random 4-byte-aligned
// places of a multi-GB array, read with coalesced 128-byte warp loads.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/chunk_bw tools/chunk_bw.cu
//   build/chunk_bw [array GiB = 4]
//
// Every warp of a persistent grid (5 CTAs x 8 warps per SM, the count
// kernel's residency) walks its own random chunks with UNROLL 128-byte rounds
// in flight, across chunk boundaries (the memory system's limit for the
// pattern, not the limit of a particular loop).  Printed per chunk size:
// useful GB/s (bytes the warps asked for).  DESIGN §4 compares the C4 count
// kernel's DRAM throughput with the row for its mean window.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

// FLAVOR 0: ld.global.nc (allocates in L1), 1: ld.global.nc.L1::no_allocate, 2: ld.global.cg (L2 only)
template <int FLAVOR>
__device__ __forceinline__ uint32_t load(const uint32_t* p) {
  uint32_t v;
  if constexpr (FLAVOR == 0) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  if constexpr (FLAVOR == 1) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  if constexpr (FLAVOR == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int UNROLL, int FLAVOR>
__global__ void __launch_bounds__(256, 5) k_chunks(const uint32_t* __restrict__ a, uint64_t words, uint32_t lg_rounds,
                                                   uint32_t rounds_per_warp, unsigned long long* sink) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t span = words - (32ull << lg_rounds) - 32;
  uint32_t acc = 0;
  for (uint32_t r0 = 0; r0 < rounds_per_warp; r0 += UNROLL) {
    uint32_t x[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const uint32_t r = r0 + k;
      const uint32_t chunk = r >> lg_rounds, within = r & ((1u << lg_rounds) - 1);
      uint32_t h = (uint32_t(warp) * 0x9E3779B1u + chunk) * 0x85EBCA6Bu;  // cheap per-chunk hash (the loop must stay load-bound)
      h ^= h >> 15;
      h *= 0xC2B2AE35u;
      h ^= h >> 16;
      const uint64_t start = (uint64_t(h) * span) >> 32;  // 4-byte aligned, like a window
      x[k] = load<FLAVOR>(a + start + 32 * within + lane);
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) acc += x[k];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  const uint64_t words = uint64_t(gib * (1ull << 30)) / 4;
  uint32_t* a;
  unsigned long long* sink;
  if (cudaMalloc(&a, words * 4) != cudaSuccess) return 1;
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, words * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 5;
  const uint64_t warps = uint64_t(grid) * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::printf("array %.1f GiB, %d CTAs x 8 warps, random 4-byte-aligned chunks\n", gib, grid);
  // the count kernel keeps 5 CTAs x 42 KB of shared memory per SM, which leaves the L1 ~18 KB
  for (int smem_kb : {0, 24, 31, 38, 42}) {
    for (int flavor = 0; flavor < (smem_kb == 0 || smem_kb == 42 ? 3 : 1); ++flavor) {
      for (int unroll : {6, 12}) {
        for (uint32_t lg : {1u, 3u, 5u}) {
          const uint32_t bytes = 128u << lg;
          const uint32_t rounds = 12 * 2048;  // per warp: 3 MiB
          float best = 1e30f;
          auto launch = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 42 * 1024);
            kern<<<grid, 256, smem_kb * 1024>>>(a, words, lg, rounds, sink);
          };
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (unroll == 6) {
              if (flavor == 0) launch(k_chunks<6, 0>);
              if (flavor == 1) launch(k_chunks<6, 1>);
              if (flavor == 2) launch(k_chunks<6, 2>);
            } else {
              if (flavor == 0) launch(k_chunks<12, 0>);
              if (flavor == 1) launch(k_chunks<12, 1>);
              if (flavor == 2) launch(k_chunks<12, 2>);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
          }
          const double gb = double(warps) * rounds * 128 / 1e9;
          static const char* names[] = {"ld.global.nc", "nc.L1::no_allocate", "ld.global.cg"};
          std::printf("smem %2d KB/CTA  %-18s  in flight %2d  chunk %6u B  %8.1f GB/s\n", smem_kb, names[flavor], unroll, bytes,
                      gb / (best * 1e-3));
        }
      }
    }
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
