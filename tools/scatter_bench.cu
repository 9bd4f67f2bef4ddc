// Microbenchmark: fp32 scatter-add of 128 random rows x 128 floats (one dK or dV block) into an
// L2-resident [64000 x 128] accumulator. Variants:
//   0: thread-per-row red.v4 (what the first backward does)
//   1: coalesced red.v4 (8 lanes per row, 4 rows per warp instruction) after a smem transpose
//   2: cp.reduce.async.bulk (TMA) of one 512-byte row per instruction from shared memory
//   3: plain coalesced st.global.v4 (upper bound, not a reduction)
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_2502_07590_b200/csrc/dsv_common.cuh"
using namespace dsv;
constexpr int NT = 256;  // blocks per CTA

template <int NTH>
__global__ void __launch_bounds__(NTH) k_rowred(float* acc, const int* idx, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* stage = reinterpret_cast<float*>(sm);  // [128][128] fp32 = 64 KB
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = 0; t < NT; ++t) {
    const int* ir = idx + ((blockIdx.x * NT + t) % 1024) * 128;
    float v = 1.0f + t;
    if (mode == 0) {
      float* row = acc + (long long)ir[tid] * 128;
#pragma unroll 4
      for (int c = 0; c < 128; c += 4) red_add_v4(row + c, v, v, v, v);
    } else if (mode == 1 || mode == 3) {
      // each warp: its 32 rows; 8 lanes per row -> 4 rows per instruction
#pragma unroll 2
      for (int rr = 0; rr < 32; rr += 4) {
        const int r = (warp * 32 + rr + (lane >> 3)) & 127;
        float* row = acc + (long long)ir[r] * 128;
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          float* p = row + c + (lane & 7) * 4;
          if (mode == 1) red_add_v4(p, v, v, v, v);
          else *reinterpret_cast<float4*>(p) = make_float4(v, v, v, v);
        }
      }
    } else if (mode == 9 || mode == 10 || mode == 11) {
      // the backward's round: thread-per-row fp32 staging, bulk reduce per row, wait for
      // the smem reads before the next round (9: rows padded to 528 B, 10: 512 B rows,
      // 11: padded, waits deferred by one round = two buffers in flight)
      const int stride = mode == 10 ? 512 : 528;
      uint8_t* srow = sm + tid * stride + ((mode == 11 && (t & 1)) ? 0 : 0);
      if (mode != 11 || true) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          *reinterpret_cast<float4*>(srow + c * 16) = make_float4(v, v, v, v);
      }
      fence_proxy_async_smem();
      __syncthreads();
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;"
                   :: "l"(acc + (long long)ir[tid] * 128), "r"(smem_u32(srow)) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    } else if (mode == 7 || mode == 8) {
      // bulk reduces kept in flight (no per-iteration wait): 512 B rows (7) or 4 x 128 B (8)
      float* srow = stage + tid * 128;
      if (t == 0) {
        for (int c = 0; c < 128; c += 4) *reinterpret_cast<float4*>(srow + c) = make_float4(1.f, 1.f, 1.f, 1.f);
        fence_proxy_async_smem();
      }
      if (mode == 7) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;"
                     :: "l"(acc + (long long)ir[tid] * 128), "r"(smem_u32(srow)) : "memory");
      } else {
        for (int q = 0; q < 4; ++q)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;"
                       :: "l"(acc + (long long)ir[tid] * 128 + q * 32), "r"(smem_u32(srow + q * 32)) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
      if (t == NT - 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
      // stage rows in smem, one bulk reduce per row
      float* srow = stage + tid * 128;
#pragma unroll 4
      for (int c = 0; c < 128; c += 4) *reinterpret_cast<float4*>(srow + c) = make_float4(v, v, v, v);
      fence_proxy_async_smem();
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;"
                   :: "l"(acc + (long long)ir[tid] * 128), "r"(smem_u32(srow)) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
}

int main() {
  const long long nrows = 64000;
  float* acc; cudaMalloc(&acc, nrows * 128 * 4); cudaMemset(acc, 0, nrows * 128 * 4);
  std::vector<int> h(1024 * 128); std::mt19937 g(1);
  for (auto& x : h) x = g() % nrows;
  int* idx; cudaMalloc(&idx, h.size() * 4); cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_rowred<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"row-per-thread red.v4", "coalesced red.v4", "bulk reduce 512B", "coalesced store", "coal red 256thr(2x)", "coal red 512thr(4x)", "coal store 512thr(4x)", "bulk red 512B inflight", "bulk red 4x128B inflight", "round padded 528", "round 512"};
  for (int grid_mult = 1; grid_mult <= 2; ++grid_mult) {
    const int grid = 148 * grid_mult;
    const double bytes = (double)grid * NT * 128 * 128 * 4;
    for (int v = 0; v < 11; ++v) {
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        if (v < 4) k_rowred<128><<<grid, 128, v == 2 ? 65536 : 0>>>(acc, idx, v);
        if (v == 4) k_rowred<256><<<grid, 256, 0>>>(acc, idx, 1);
        if (v == 5) k_rowred<512><<<grid, 512, 0>>>(acc, idx, 1);
        if (v == 6) k_rowred<512><<<grid, 512, 0>>>(acc, idx, 3);
        if (v == 7 || v == 8) k_rowred<128><<<grid, 128, 65536>>>(acc, idx, v);
        if (v == 9 || v == 10) k_rowred<128><<<grid, 128, 70000>>>(acc, idx, v);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it == 2) printf("grid %3d %-22s: %.3f ms  %7.1f GB/s  per-block %.0f ns  err=%s\n", grid, names[v], ms,
                            (v == 4 ? 2 : (v == 5 || v == 6) ? 4 : 1) * bytes / ms / 1e6, ms * 1e6 / NT / grid_mult, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  // verify the in-flight bulk reduce really accumulates: sum(acc) == rows * 128 * 1.0
  for (int v = 7; v <= 8; ++v) {
    cudaMemset(acc, 0, nrows * 128 * 4);
    k_rowred<128><<<148, 128, 65536>>>(acc, idx, v);
    std::vector<float> hacc(nrows * 128);
    cudaMemcpy(hacc.data(), acc, hacc.size() * 4, cudaMemcpyDeviceToHost);
    double sum = 0; for (float x : hacc) sum += x;
    printf("verify mode %d: sum %.0f expected %.0f\n", v, sum, 148.0 * NT * 128 * 128);
  }
  return 0;
}
