// Phase breakdown of the K2 top-k kernel at the c2 shape (6240 rows x 32000, k = 3200).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/topk_phase tools/topk_phase.cu
#define DSV_TOPK_PROF 1
#include "../paper_2502_07590_b200/csrc/topk.cu"
#include <cstdio>
#include <random>
#include <vector>
__global__ void lowrank_scores(const float* q, const float* k, float* s, int rows, int L) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)rows * L) return;
  const int r = (int)(t / L), c = (int)(t % L);
  float acc = 0.f;
  for (int i = 0; i < 16; ++i) acc += q[r * 16 + i] * k[c * 16 + i];
  s[t] = acc;
}
int main(int argc, char** argv) {
  const int rows = 6240, L = 32000, k = 3200;
  const bool lowrank = argc > 1;   // scores = q . k^T with r = 16 (the layer's K1b output)
  std::vector<float> h((size_t)rows * L);
  std::mt19937 g(1); std::normal_distribution<float> nd;
  float* d; cudaMalloc(&d, h.size() * 4);
  if (!lowrank) {
    for (auto& x : h) x = nd(g);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  } else {
    std::vector<float> hq(rows * 16), hk(L * 16);
    for (auto& x : hq) x = nd(g);
    for (auto& x : hk) x = nd(g);
    float *dq, *dk; cudaMalloc(&dq, hq.size() * 4); cudaMalloc(&dk, hk.size() * 4);
    cudaMemcpy(dq, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
    lowrank_scores<<<(unsigned)(((long long)rows * L + 255) / 256), 256>>>(dq, dk, d, rows, L);
    cudaDeviceSynchronize();
  }
  int* kk; cudaMalloc(&kk, 4); cudaMemcpy(kk, &k, 4, cudaMemcpyHostToDevice);
  int* idx; cudaMalloc(&idx, (size_t)rows * k * 4);
  float* thr; cudaMalloc(&thr, rows * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_topk_prof, z, sizeof(z));
    cudaEventRecord(a);
    dsv_topk_launch(d, L, rows, L, kk, rows, idx, k, thr, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long p[16]; cudaMemcpyFromSymbol(p, g_topk_prof, sizeof(p));
    unsigned int slow = 0; cudaMemcpyFromSymbol(&slow, g_topk_slow, 4);
    unsigned int z0 = 0; cudaMemcpyToSymbol(g_topk_slow, &z0, 4);
    printf("[slow-path rows: %u] ", slow);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dsv::topk::topk_rows_kernel<true>, 256,
                                                  dsv_topk_smem_bytes(L));
    const int nrows0 = (rows + 148 * per_sm - 1) / (148 * per_sm);
    printf("%.3f ms (%s) CTAs/SM %d, cycles/row for CTA0 (%d rows):", ms, cudaGetErrorString(cudaGetLastError()),
           per_sm, nrows0);
    const char* nm[] = {"sample", "band", "pass1", "check", "select", "mark", "emit", "sync"};
    for (int i = 0; i < 8; ++i) printf(" %s=%llu", nm[i], p[i] / nrows0);
    printf("\n");
  }
  return 0;
}
