// rows_simt.cu — CUDA-core kernels for the general (ragged / per-query) case.
//
// * dsv_scores_f32: batched fp32 score product C[b] = A[b] . B[b]^T for small
//   inner width r (the low-rank predictor scores, reference
//   pkg/src/dynsparse/selection.py:149 `q_block @ k_lr[c0:c1].T`). Summation
//   runs t = 0..r-1 with fmaf, so the result is deterministic; it feeds K2.
// * sparse attention over arbitrary per-(head, query) CSR index lists
//   (reference pkg/src/dynsparse/attention.py:176-183, the ragged per-row
//   loop, and the autograd of pkg/src/dynsparse/trainer.py:110-117).
//   One warp per (head, query); fp32 math; online softmax; LSE saved for the
//   backward, which recomputes P and scatter-adds dK/dV with fp32 atomics.
// These are the GPU correctness path for index sets the tensor-core kernels do
// not tile (per-query lists, theta-oracle sets, groups < 64 queries).

#include "dsv_common.cuh"

namespace dsv {
namespace simt {

template <typename T> DSV_DEV float ld_f(const T* p);
template <> DSV_DEV float ld_f<float>(const float* p) { return __ldg(p); }
template <> DSV_DEV float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// C[b, i, j] = sum_t A[b, i, t] * B[b, j, t]; A: [nb, R, r] (row stride lda),
// B: [nb, Lk, r] (row stride ldb), C: [nb, R, Lk] (row stride ldc). Any r: the
// inner loop runs in chunks of 64 but always in t order 0..r-1 (fmaf).
constexpr int kScRows = 16, kScT = 32;
template <typename T>
__global__ void __launch_bounds__(256)
scores_kernel(const T* __restrict__ A, long long lda, long long a_bs,
              const T* __restrict__ B, long long ldb, long long b_bs,
              float* __restrict__ C, long long ldc, long long c_bs, int R, int Lk, int r) {
  __shared__ float sA[kScRows * kScT];
  const int b = blockIdx.z;
  const int i0 = blockIdx.y * kScRows;
  const int j = blockIdx.x * 256 + threadIdx.x;
  const T* Ab = A + b * a_bs;
  const T* Bb = B + b * b_bs;
  float acc[kScRows];
#pragma unroll
  for (int ii = 0; ii < kScRows; ++ii) acc[ii] = 0.f;
  for (int t0 = 0; t0 < r; t0 += kScT) {
    const int tn = min(kScT, r - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kScRows * kScT; e += 256) {
      const int ii = e / kScT, t = e % kScT;
      sA[e] = (i0 + ii < R && t < tn) ? ld_f(Ab + (long long)(i0 + ii) * lda + t0 + t) : 0.f;
    }
    __syncthreads();
    if (j < Lk) {
      float bj[kScT];
#pragma unroll
      for (int t = 0; t < kScT; ++t) bj[t] = (t < tn) ? ld_f(Bb + (long long)j * ldb + t0 + t) : 0.f;
#pragma unroll
      for (int ii = 0; ii < kScRows; ++ii) {
#pragma unroll
        for (int t = 0; t < kScT; ++t)
          if (t < tn) acc[ii] = fmaf(sA[ii * kScT + t], bj[t], acc[ii]);
      }
    }
  }
  if (j >= Lk) return;
  float* Cb = C + b * c_bs;
  const int iend = min(kScRows, R - i0);
#pragma unroll
  for (int ii = 0; ii < kScRows; ++ii)
    if (ii < iend) Cb[(long long)(i0 + ii) * ldc + j] = acc[ii];
}

// ---------------------------------------------------------------- attention
// q: [H, Lq, dk], k: [H, Lk, dk], v: [H, Lk, dv]; ptr: [H*Lq + 1] (int64), cols: int32 key ids
// (cols == nullptr: every key). A is the arithmetic type: fp32 for bf16 / fp32 inputs, fp64
// for the reference-precision path (host fp64 callers: the reference computes in the input
// dtype, pkg/src/dynsparse/attention.py:95-109 / 153-187).
template <typename T, typename A> DSV_DEV A ld_a(const T* p) { return (A)ld_f(p); }
template <> DSV_DEV double ld_a<double, double>(const double* p) { return __ldg(p); }
DSV_DEV float ex_a(float x) { return __expf(x); }
DSV_DEV double ex_a(double x) { return exp(x); }
DSV_DEV float lg_a(float x) { return logf(x); }
DSV_DEV double lg_a(double x) { return log(x); }

template <typename T, typename A, int NE>  // NE = ceil(max(dk, dv) / 32) elements per lane
__global__ void __launch_bounds__(256)
attn_rows_fwd_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                     const long long* __restrict__ ptr, const int* __restrict__ cols,
                     int H, int Lq, int Lk, int dk, int dv, A scale,
                     A* __restrict__ o, A* __restrict__ lse) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= H * Lq) return;
  const int h = gw / Lq;
  const T* qr = q + (long long)gw * dk;
  A qv[NE], acc[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    qv[e] = (c < dk) ? ld_a<T, A>(qr + c) : A(0);
    acc[e] = A(0);
  }
  A m = -INFINITY, l = A(0);
  const long long p0 = cols ? ptr[gw] : 0, p1 = cols ? ptr[gw + 1] : Lk;
  const T* kh = k + (long long)h * Lk * dk;
  const T* vh = v + (long long)h * Lk * dv;
  for (long long p = p0; p < p1; ++p) {
    const int key = cols ? cols[p] : (int)p;
    const T* kr = kh + (long long)key * dk;
    A s = A(0);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      if (c < dk) s = fma(qv[e], ld_a<T, A>(kr + c), s);
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o2);
    s *= scale;
    const A mn = fmax(m, s);
    const A alpha = ex_a(m - mn);
    const A pw = ex_a(s - mn);
    l = l * alpha + pw;
    const T* vr = vh + (long long)key * dv;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      acc[e] = acc[e] * alpha + ((c < dv) ? pw * ld_a<T, A>(vr + c) : A(0));
    }
    m = mn;
  }
  const A inv = A(1) / l;
  A* orow = o + (long long)gw * dv;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dv) orow[c] = acc[e] * inv;
  }
  if (lane == 0) lse[gw] = m + lg_a(l);
}

template <typename T, typename A, int NE>
__global__ void __launch_bounds__(256)
attn_rows_bwd_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                     const A* __restrict__ o, const A* __restrict__ lse,
                     const T* __restrict__ dout,
                     const long long* __restrict__ ptr, const int* __restrict__ cols,
                     int H, int Lq, int Lk, int dk, int dv, A scale,
                     A* __restrict__ dq, A* __restrict__ dkacc, A* __restrict__ dvacc) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= H * Lq) return;
  const int h = gw / Lq;
  A qv[NE], dov[NE], dqa[NE];
  A delta = A(0);
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    qv[e] = (c < dk) ? ld_a<T, A>(q + (long long)gw * dk + c) : A(0);
    dov[e] = (c < dv) ? ld_a<T, A>(dout + (long long)gw * dv + c) : A(0);
    delta += (c < dv) ? dov[e] * o[(long long)gw * dv + c] : A(0);
    dqa[e] = A(0);
  }
#pragma unroll
  for (int o2 = 16; o2; o2 >>= 1) delta += __shfl_xor_sync(0xffffffffu, delta, o2);
  const A lrow = lse[gw];
  const long long p0 = cols ? ptr[gw] : 0, p1 = cols ? ptr[gw + 1] : Lk;
  const long long hk = (long long)h * Lk * dk, hv = (long long)h * Lk * dv;
  for (long long p = p0; p < p1; ++p) {
    const int key = cols ? cols[p] : (int)p;
    const T* kr = k + hk + (long long)key * dk;
    const T* vr = v + hv + (long long)key * dv;
    A s = A(0), dp = A(0);
    A kv[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      kv[e] = (c < dk) ? ld_a<T, A>(kr + c) : A(0);
      s = fma(qv[e], kv[e], s);
      dp = fma(dov[e], (c < dv) ? ld_a<T, A>(vr + c) : A(0), dp);
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o2);
      dp += __shfl_xor_sync(0xffffffffu, dp, o2);
    }
    const A pw = ex_a(s * scale - lrow);
    const A ds = pw * (dp - delta) * scale;
    A* dkr = dkacc + hk + (long long)key * dk;
    A* dvr = dvacc + hv + (long long)key * dv;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      if (c < dk) {
        dqa[e] = fma(ds, kv[e], dqa[e]);
        atomicAdd(dkr + c, ds * qv[e]);
      }
      if (c < dv) atomicAdd(dvr + c, pw * dov[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dk) dq[(long long)gw * dk + c] = dqa[e];
  }
}

}  // namespace simt
}  // namespace dsv

using namespace dsv::simt;

int dsv_scores_f32_launch(const void* A, long long lda, long long a_bs, const void* B,
                          long long ldb, long long b_bs, float* C, long long ldc, long long c_bs,
                          int nbatch, int R, int Lk, int r, int bf16_in, cudaStream_t st) {
  if (r < 1) return 1;
  dim3 grid((Lk + 255) / 256, (R + kScRows - 1) / kScRows, nbatch);
  const size_t sm = 0;
  if (bf16_in)
    scores_kernel<__nv_bfloat16><<<grid, 256, sm, st>>>(
        (const __nv_bfloat16*)A, lda, a_bs, (const __nv_bfloat16*)B, ldb, b_bs, C, ldc, c_bs, R,
        Lk, r);
  else
    scores_kernel<float><<<grid, 256, sm, st>>>((const float*)A, lda, a_bs, (const float*)B, ldb,
                                                b_bs, C, ldc, c_bs, R, Lk, r);
  return (int)cudaGetLastError();
}

template <typename T, typename A>
static int rows_fwd(const void* q, const void* k, const void* v, const long long* ptr,
                    const int* cols, int H, int Lq, int Lk, int dk, int dv, A scale, A* o, A* lse,
                    cudaStream_t st) {
  const long long warps = (long long)H * Lq;
  const int blocks = (int)((warps * 32 + 255) / 256);
  const T *Q = (const T*)q, *K = (const T*)k, *V = (const T*)v;
  const int d = dk > dv ? dk : dv;
#define DSV_ROWS_FWD(NE) \
  attn_rows_fwd_kernel<T, A, NE><<<blocks, 256, 0, st>>>(Q, K, V, ptr, cols, H, Lq, Lk, dk, dv, scale, o, lse)
  switch ((d + 31) / 32) {
    case 1: DSV_ROWS_FWD(1); break;
    case 2: DSV_ROWS_FWD(2); break;
    case 3: case 4: DSV_ROWS_FWD(4); break;
    case 5: case 6: case 7: case 8: DSV_ROWS_FWD(8); break;
    default: return 1;
  }
#undef DSV_ROWS_FWD
  return (int)cudaGetLastError();
}

template <typename T, typename A>
static int rows_bwd(const void* q, const void* k, const void* v, const A* o, const A* lse,
                    const void* dout, const long long* ptr, const int* cols, int H, int Lq, int Lk,
                    int dk, int dv, A scale, A* dq, A* dka, A* dva, cudaStream_t st) {
  const long long warps = (long long)H * Lq;
  const int blocks = (int)((warps * 32 + 255) / 256);
  const T *Q = (const T*)q, *K = (const T*)k, *V = (const T*)v, *DO = (const T*)dout;
  const int d = dk > dv ? dk : dv;
#define DSV_ROWS_BWD(NE) \
  attn_rows_bwd_kernel<T, A, NE><<<blocks, 256, 0, st>>>(Q, K, V, o, lse, DO, ptr, cols, H, Lq, Lk, dk, dv, scale, dq, dka, dva)
  switch ((d + 31) / 32) {
    case 1: DSV_ROWS_BWD(1); break;
    case 2: DSV_ROWS_BWD(2); break;
    case 3: case 4: DSV_ROWS_BWD(4); break;
    case 5: case 6: case 7: case 8: DSV_ROWS_BWD(8); break;
    default: return 1;
  }
#undef DSV_ROWS_BWD
  return (int)cudaGetLastError();
}

int dsv_rows_fwd_launch(const void* q, const void* k, const void* v, const long long* ptr,
                        const int* cols, int H, int Lq, int Lk, int d, float scale, int bf16_in,
                        float* o, float* lse, cudaStream_t st) {
  return bf16_in ? rows_fwd<__nv_bfloat16, float>(q, k, v, ptr, cols, H, Lq, Lk, d, d, scale, o, lse, st)
                 : rows_fwd<float, float>(q, k, v, ptr, cols, H, Lq, Lk, d, d, scale, o, lse, st);
}

int dsv_rows_bwd_launch(const void* q, const void* k, const void* v, const float* o,
                        const float* lse, const void* dout, const long long* ptr, const int* cols,
                        int H, int Lq, int Lk, int d, float scale, int bf16_in, float* dq,
                        float* dk, float* dv, cudaStream_t st) {
  return bf16_in ? rows_bwd<__nv_bfloat16, float>(q, k, v, o, lse, dout, ptr, cols, H, Lq, Lk, d, d,
                                                  scale, dq, dk, dv, st)
                 : rows_bwd<float, float>(q, k, v, o, lse, dout, ptr, cols, H, Lq, Lk, d, d, scale,
                                          dq, dk, dv, st);
}

int dsv_rows_fwd_f64_launch(const double* q, const double* k, const double* v, const long long* ptr,
                            const int* cols, int H, int Lq, int Lk, int dk, int dv, double scale,
                            double* o, double* lse, cudaStream_t st) {
  return rows_fwd<double, double>(q, k, v, ptr, cols, H, Lq, Lk, dk, dv, scale, o, lse, st);
}

int dsv_rows_bwd_f64_launch(const double* q, const double* k, const double* v, const double* o,
                            const double* lse, const double* dout, const long long* ptr,
                            const int* cols, int H, int Lq, int Lk, int dk, int dv, double scale,
                            double* dq, double* dka, double* dva, cudaStream_t st) {
  return rows_bwd<double, double>(q, k, v, o, lse, dout, ptr, cols, H, Lq, Lk, dk, dv, scale, dq,
                                  dka, dva, st);
}
