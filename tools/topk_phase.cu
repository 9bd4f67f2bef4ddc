// Phase breakdown of the K2 top-k kernel at the c2 shape (6240 rows x 32000, k = 3200).
#define DSV_TOPK_PROF 1
#ifdef ABL
#define DSV_TOPK_ABLATE 1
#endif
#include "../paper_2502_07590_b200/csrc/topk.cu"
#include "../paper_2502_07590_b200/csrc/topk_stream.cu"
#include <cstdio>
#include <random>
#include <vector>
int main() {
  const int rows = 6240, L = 32000, k = 3200;
  std::vector<float> h((size_t)rows * L);
  std::mt19937 g(1); std::normal_distribution<float> nd;
  for (auto& x : h) x = nd(g);
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
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
    printf("%.3f ms (%s) cycles/row for CTA0 (42 rows):", ms, cudaGetErrorString(cudaGetLastError()));
    const char* nm[] = {"load", "sample", "pass1", "bandchk", "refine", "cand", "emit", "sync", "p1loop", "p1scan"};
    for (int i = 0; i < 10; ++i) printf(" %s=%llu", nm[i], p[i] / 42);
    printf("\n");
  }
  return 0;
}
