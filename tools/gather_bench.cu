// Microbenchmark: gathering 128 random 256-byte rows (one K block) into shared memory on B200.
// Variants: TMA tile::gather4 (1 issuing lane / 32 issuing lanes), cp.async 16B from 4 warps,
// contiguous TMA tile (upper bound). Every CTA streams NT tiles through a 4-stage ring.
#include <cuda.h>
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2502_07590_b200/csrc/dsv_common.cuh"
using namespace dsv;
constexpr int ROWS = 128, D = 128, TILE = ROWS * D * 2, ST = 4, NT = 256;

__global__ void __launch_bounds__(128) k_gather4(const __grid_constant__ CUtensorMap tm, const int* idx, int nrows, int all_lanes, long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~1023ull);
  __shared__ uint64_t full[ST];
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1); fence_barrier_init(); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int t = 0; t < NT; ++t) {
      const int s = t % ST;
      if (t >= ST) mbar_wait(&full[s], ((t / ST) - 1) & 1);
      const int* ir = idx + ((blockIdx.x * NT + t) % 1024) * ROWS;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], TILE);
      __syncwarp();
      uint8_t* dst = buf + s * TILE;
      if (all_lanes) {
        int4 r = *(const int4*)(ir + lane * 4);
        for (int a = 0; a < 2; ++a) tma_gather4(dst + a * 16384 + lane * 512, &tm, &full[s], a * 64, r.x, r.y, r.z, r.w);
      } else if (lane == 0) {
        for (int g = 0; g < 32; ++g) {
          int4 r = *(const int4*)(ir + g * 4);
          for (int a = 0; a < 2; ++a) tma_gather4(dst + a * 16384 + g * 512, &tm, &full[s], a * 64, r.x, r.y, r.z, r.w);
        }
      }
      __syncwarp();
    }
    for (int t = NT - ST; t < NT; ++t) mbar_wait(&full[t % ST], (t / ST) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = buf[threadIdx.x];
}

__global__ void __launch_bounds__(128) k_tile(const __grid_constant__ CUtensorMap tm, int nrows, long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~1023ull);
  __shared__ uint64_t full[ST];
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 0; t < NT; ++t) {
      const int s = t % ST;
      if (t >= ST) mbar_wait(&full[s], ((t / ST) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], TILE);
      int row0 = ((blockIdx.x * NT + t) * 128) % (nrows - 128);
      for (int a = 0; a < 2; ++a) tma_load_2d(buf + s * TILE + a * 16384, &tm, &full[s], a * 64, row0);
    }
    for (int t = NT - ST; t < NT; ++t) mbar_wait(&full[t % ST], (t / ST) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = buf[0];
}

// cp.async 16B gathers: NTHR threads; row = 16 chunks of 16 B placed with the 128B swizzle.
template <int NTHR>
__global__ void __launch_bounds__(NTHR) k_cpasync(const __nv_bfloat16* K, const int* idx, long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~1023ull);
  const int tid = threadIdx.x;
  for (int t = 0; t < NT + ST - 1; ++t) {
    if (t < NT) {
      const int s = t % ST;
      const int* ir = idx + ((blockIdx.x * NT + t) % 1024) * ROWS;
      uint8_t* dst = buf + s * TILE;
#pragma unroll
      for (int i = 0; i < 2048 / NTHR; ++i) {
        const int c = i * NTHR + tid;       // chunk id 0..2047
        const int r = c >> 4, ch = c & 15;
        const int key = __ldg(ir + r);
        const char* src = (const char*)(K + (long long)key * D) + ch * 16;
        uint32_t d = smem_u32(dst + (ch >> 3) * 16384 + sw128_off(r, ch & 7));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" :: "n"(ST - 1));
    __syncthreads();
  }
  if (tid == 0) sink[blockIdx.x] = buf[0];
}


// LDG.128 -> STS.128 through registers, NTHR threads, U chunks in flight per thread.
template <int NTHR, int U>
__global__ void __launch_bounds__(NTHR) k_ldgsts(const __nv_bfloat16* K, const int* idx, long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~1023ull);
  const int tid = threadIdx.x;
  constexpr int PER = 2048 / NTHR;
  for (int t = 0; t < NT; ++t) {
    const int s = t % ST;
    const int* ir = idx + ((blockIdx.x * NT + t) % 1024) * ROWS;
    uint8_t* dst = buf + s * TILE;
#pragma unroll
    for (int i0 = 0; i0 < PER; i0 += U) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = (i0 + u) * NTHR + tid; const int r = c >> 4, ch = c & 15;
        const int key = __ldg(ir + r);
        v[u] = __ldg((const int4*)((const char*)(K + (long long)key * D) + ch * 16));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = (i0 + u) * NTHR + tid; const int r = c >> 4, ch = c & 15;
        *(int4*)(dst + (ch >> 3) * 16384 + sw128_off(r, ch & 7)) = v[u];
      }
    }
  }
  __syncthreads();
  if (tid == 0) sink[blockIdx.x] = buf[0];
}
// cp.async with a deeper ring (NS stages of 32 KB)
template <int NTHR, int NS>
__global__ void __launch_bounds__(NTHR) k_cpasync_deep(const __nv_bfloat16* K, const int* idx, long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~1023ull);
  const int tid = threadIdx.x;
  for (int t = 0; t < NT + NS - 1; ++t) {
    if (t < NT) {
      const int s = t % NS;
      const int* ir = idx + ((blockIdx.x * NT + t) % 1024) * ROWS;
      uint8_t* dst = buf + s * TILE;
#pragma unroll
      for (int i = 0; i < 2048 / NTHR; ++i) {
        const int c = i * NTHR + tid;
        const int r = c >> 4, ch = c & 15;
        const int key = __ldg(ir + r);
        const char* src = (const char*)(K + (long long)key * D) + ch * 16;
        uint32_t d = smem_u32(dst + (ch >> 3) * 16384 + sw128_off(r, ch & 7));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" :: "n"(NS - 1));
  }
  __syncthreads();
  if (tid == 0) sink[blockIdx.x] = buf[0];
}
int main() {
  const long long nrows = 32000 * 2;  // two heads of K
  __nv_bfloat16* K; cudaMalloc(&K, nrows * D * 2); cudaMemset(K, 0, nrows * D * 2);
  std::vector<int> h(1024 * ROWS); std::mt19937 g(1);
  for (auto& x : h) x = g() % nrows;
  int* idx; cudaMalloc(&idx, h.size() * 4); cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  long long* sink; cudaMalloc(&sink, 148 * 64 * 8);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fp;
  CUtensorMap tg, tt;
  cuuint64_t dims[2] = {D, (cuuint64_t)nrows}, str[1] = {D * 2};
  cuuint32_t box1[2] = {64, 1}, box2[2] = {64, 128}, es[2] = {1, 1};
  enc(&tg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, str, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = ST * TILE + 1024;
  cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cpasync<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cpasync<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldgsts<256,4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldgsts<512,4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldgsts<256,8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int smem6 = 6 * TILE + 1024;
  cudaFuncSetAttribute(k_cpasync_deep<128,6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
  cudaFuncSetAttribute(k_cpasync_deep<256,6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
  cudaFuncSetAttribute(k_cpasync_deep<512,6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148;
  const double bytes = (double)grid * NT * TILE;
  const char* names[] = {"gather4 1 lane", "gather4 32 lanes", "cp.async 128 thr", "cp.async 256 thr", "tma tile",
     "ldg/sts 256x4", "ldg/sts 512x4", "ldg/sts 256x8", "cp.async 128 6st", "cp.async 256 6st", "cp.async 512 6st"};
  for (int v = 0; v < 11; ++v) {
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      if (v == 0) k_gather4<<<grid, 128, smem>>>(tg, idx, nrows, 0, sink);
      if (v == 1) k_gather4<<<grid, 128, smem>>>(tg, idx, nrows, 1, sink);
      if (v == 2) k_cpasync<128><<<grid, 128, smem>>>(K, idx, sink);
      if (v == 3) k_cpasync<256><<<grid, 256, smem>>>(K, idx, sink);
      if (v == 4) k_tile<<<grid, 128, smem>>>(tt, nrows, sink);
      if (v == 5) k_ldgsts<256,4><<<grid, 256, smem>>>(K, idx, sink);
      if (v == 6) k_ldgsts<512,4><<<grid, 512, smem>>>(K, idx, sink);
      if (v == 7) k_ldgsts<256,8><<<grid, 256, smem>>>(K, idx, sink);
      if (v == 8) k_cpasync_deep<128,6><<<grid, 128, smem6>>>(K, idx, sink);
      if (v == 9) k_cpasync_deep<256,6><<<grid, 256, smem6>>>(K, idx, sink);
      if (v == 10) k_cpasync_deep<512,6><<<grid, 512, smem6>>>(K, idx, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it == 2) printf("%-18s: %.3f ms  %7.1f GB/s  %5.1f B/clk/SM @1.9GHz  per-tile %.0f ns  err=%s\n", names[v],
                          ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / 1.9e9, ms * 1e6 / NT,
                          cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
