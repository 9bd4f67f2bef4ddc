// TMEM read / write throughput per SM on the B200 (tcgen05.ld / tcgen05.st, 32x32b shapes):
// W warps (a multiple of 4: W/4 per TMEM lane quarter) each load or store 32 columns x 32
// lanes (4 KB) per instruction, with `depth` instructions in flight before each wait.
// Prints bytes per SM clock. The backward's B stage reads S^T and dP^T (128 KB per key
// block) and C' reads dV_j / dK_j (128 KB): this is the rate those phases run against.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include "../paper_2502_07590_b200/csrc/dsv_common.cuh"
using namespace dsv;

template <int MODE, int DEPTH>   // MODE 0: ld x32, 1: ld x16, 2: st x16
__global__ void __launch_bounds__(512, 1) k(unsigned long long* cyc, uint32_t* sink, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&taddr_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = taddr_s;
  const int quarter = warp & 3, slice = (warp >> 2) % 4;    // up to 4 warps per quarter share columns
  const uint32_t base = t + ((uint32_t)(quarter * 32) << 16) + slice * 128;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        uint32_t r[32];
        tmem_ld32(base + (d & 3) * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= r[i];
      }
      tmem_ld_wait();
    } else if constexpr (MODE == 1) {
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) {
        uint32_t r[16];
        tmem_ld16(base + (d & 7) * 16, r);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc ^= r[i];
      }
      tmem_ld_wait();
    } else {
      uint32_t r[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = acc + i + it;
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) tmem_st16(base + (d & 7) * 16, r);
      tmem_st_wait();
      acc += r[3];
    }
  }
  const unsigned long long c1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 512);
}

template <int MODE, int DEPTH>
static void run(const char* name, int warps) {
  const int blocks = 148, iters = 2000;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, blocks * 8);
  cudaMalloc(&sink, blocks * warps * 32 * 4);
  k<MODE, DEPTH><<<blocks, warps * 32>>>(cyc, sink, iters);
  k<MODE, DEPTH><<<blocks, warps * 32>>>(cyc, sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += (double)h[i] / blocks;
  const double bytes_per_instr = MODE == 0 ? 4096.0 : 2048.0;
  const double bytes = (double)warps * iters * DEPTH * bytes_per_instr;
  printf("%-22s warps %2d depth %d: %7.1f B/clk/SM  (%s)\n", name, warps, DEPTH, bytes / mean,
         cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<0, 1>("ld 32x32b.x32", 4);
  run<0, 2>("ld 32x32b.x32", 4);
  run<0, 4>("ld 32x32b.x32", 4);
  run<0, 1>("ld 32x32b.x32", 16);
  run<0, 2>("ld 32x32b.x32", 16);
  run<0, 4>("ld 32x32b.x32", 16);
  run<1, 2>("ld 32x32b.x16", 16);
  run<1, 4>("ld 32x32b.x16", 16);
  run<2, 1>("st 32x32b.x16", 4);
  run<2, 4>("st 32x32b.x16", 16);
  return 0;
}
