// predictor.cu — predictor training step on device.
//
// Reference: pkg/src/dynsparse/predictor.py:103-194 (`_cos_terms`, `_norm_terms`,
// `loss_and_grads`). With A_hat = Q_lr K_lr^T ([R, S], R sampled query rows) and the
// target T ([R, S]), the loss gradient G = dL/dA_hat is, row by row, a combination of the
// two matrices: G[i, :] = u_i T[i, :] + w_i A_hat[i, :] (cosine term: per-row u, w from
// |a_i|, |t_i|, a_i . t_i; norm term: one global coefficient on (A_hat - T)). So the step
// never materialises A_hat or G: three streaming passes over T, each recomputing A_hat
// entries (r-term fp64 dots; K_lr stays L2-resident):
//   1. row statistics       |a_i|^2, |t_i|^2, a_i . t_i, |a_i - t_i|^2          (row CTAs)
//   2. G K_lr  [R, r]       sum_s (u_i t_is + w_i a_is) k_s                     (row CTAs)
//   3. G^T Q_lr [S, r]      sum_i (u_i t_is + w_i a_is) q_i  (column CTAs, T rows staged)
// All accumulation is fp64 (the reference trains in fp64); T is read as fp32 or fp64.

#include <type_traits>
#include "dsv_common.cuh"

namespace dsv {
namespace pred {

constexpr int kThreads = 256;
constexpr int kMaxR = 64;     // low-rank width supported (d_lr <= 64)

template <typename TT>
DSV_DEV double ld_t(const TT* p) { return (double)__ldg(p); }

DSV_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) t += red[w];
  return t;
}

// pass 1: per row i the four sums
template <typename TT, int RM>
__global__ void __launch_bounds__(kThreads)
row_stats_kernel(const double* __restrict__ qlr, const double* __restrict__ klr, const TT* __restrict__ T,
                 long long ldt, int R, int S, int r, double* __restrict__ stats) {
  __shared__ double qs[kMaxR];
  __shared__ double red[kThreads / 32];
  for (int i = blockIdx.x; i < R; i += gridDim.x) {
    for (int j = threadIdx.x; j < r; j += kThreads) qs[j] = qlr[(long long)i * r + j];
    __syncthreads();
    double a2 = 0, t2 = 0, at = 0, d2 = 0;
    const TT* trow = T + (long long)i * ldt;
    for (int s = threadIdx.x; s < S; s += kThreads) {
      const double* kr = klr + (long long)s * r;
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < RM; ++j) if (j < r) a = fma(qs[j], kr[j], a);
      const double t = ld_t(trow + s);
      a2 = fma(a, a, a2);
      t2 = fma(t, t, t2);
      at = fma(a, t, at);
      d2 = fma(a - t, a - t, d2);
    }
    a2 = block_sum(a2, red);
    t2 = block_sum(t2, red);
    at = block_sum(at, red);
    d2 = block_sum(d2, red);
    if (threadIdx.x == 0) {
      stats[4 * i + 0] = a2; stats[4 * i + 1] = t2; stats[4 * i + 2] = at; stats[4 * i + 3] = d2;
    }
    __syncthreads();
  }
}

// pass 2: G1[i, :] = sum_s (u_i t_is + w_i a_is) k_s
template <typename TT, int RM>
__global__ void __launch_bounds__(kThreads)
g_klr_kernel(const double* __restrict__ qlr, const double* __restrict__ klr, const TT* __restrict__ T,
             long long ldt, int R, int S, int r, const double* __restrict__ uw, double* __restrict__ g1) {
  __shared__ double qs[kMaxR];
  __shared__ double part[kThreads / 32][kMaxR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = blockIdx.x; i < R; i += gridDim.x) {
    for (int j = threadIdx.x; j < r; j += kThreads) qs[j] = qlr[(long long)i * r + j];
    __syncthreads();
    const double u = uw[2 * i], w = uw[2 * i + 1];
    double acc[RM];
#pragma unroll
    for (int j = 0; j < RM; ++j) acc[j] = 0.0;
    const TT* trow = T + (long long)i * ldt;
    for (int s = threadIdx.x; s < S; s += kThreads) {
      const double* kr = klr + (long long)s * r;
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < RM; ++j) if (j < r) a = fma(qs[j], kr[j], a);
      const double g = fma(u, ld_t(trow + s), w * a);
#pragma unroll
      for (int j = 0; j < RM; ++j) if (j < r) acc[j] = fma(g, kr[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < RM; ++j) {
      if (j >= r) break;
      double v = acc[j];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) part[warp][j] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < r; j += kThreads) {
      double v = 0.0;
      for (int ww = 0; ww < kThreads / 32; ++ww) v += part[ww][j];
      g1[(long long)i * r + j] = v;
    }
    __syncthreads();
  }
}

// pass 3: G2[s, :] = sum_i (u_i t_is + w_i a_is) q_i  (thread = column s)
template <typename TT, int RM>
__global__ void __launch_bounds__(kThreads)
g_qlr_kernel(const double* __restrict__ qlr, const double* __restrict__ klr, const TT* __restrict__ T,
             long long ldt, int R, int S, int r, const double* __restrict__ uw, double* __restrict__ g2) {
  constexpr int kRows = 32;   // query rows staged per round
  __shared__ double qs[kRows][kMaxR];
  __shared__ double us[kRows], ws[kRows];
  const int s = blockIdx.x * kThreads + threadIdx.x;
  double kr[RM], acc[RM];
#pragma unroll
  for (int j = 0; j < RM; ++j) { kr[j] = (s < S && j < r) ? klr[(long long)s * r + j] : 0.0; acc[j] = 0.0; }
  for (int i0 = 0; i0 < R; i0 += kRows) {
    const int nr = min(kRows, R - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * r; e += kThreads) qs[e / r][e % r] = qlr[(long long)(i0 + e / r) * r + e % r];
    for (int e = threadIdx.x; e < nr; e += kThreads) { us[e] = uw[2 * (i0 + e)]; ws[e] = uw[2 * (i0 + e) + 1]; }
    __syncthreads();
    if (s < S) {
      for (int ii = 0; ii < nr; ++ii) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < RM; ++j) if (j < r) a = fma(qs[ii][j], kr[j], a);
        const double g = fma(us[ii], ld_t(T + (long long)(i0 + ii) * ldt + s), ws[ii] * a);
#pragma unroll
        for (int j = 0; j < RM; ++j) if (j < r) acc[j] = fma(g, qs[ii][j], acc[j]);
      }
    }
  }
  if (s < S) {
#pragma unroll
    for (int j = 0; j < RM; ++j) if (j < r) g2[(long long)s * r + j] = acc[j];
  }
}

}  // namespace pred
}  // namespace dsv

// stage: 0 = row stats, 1 = G K_lr, 2 = G^T Q_lr; t_f64: target is fp64 (else fp32)
int dsv_pred_pass_launch(int stage, const double* qlr, const double* klr, const void* T, int t_f64,
                         long long ldt, int R, int S, int r, const double* uw, double* out,
                         cudaStream_t st) {
  using namespace dsv::pred;
  if (r > kMaxR) return (int)cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int rgrid = R < 8 * sms ? R : 8 * sms;
  const int cgrid = (S + kThreads - 1) / kThreads;
  auto run = [&](auto tag, auto rm) {
    using TT = decltype(tag);
    constexpr int RM = decltype(rm)::value;
    const TT* t = static_cast<const TT*>(T);
    if (stage == 0) row_stats_kernel<TT, RM><<<rgrid, kThreads, 0, st>>>(qlr, klr, t, ldt, R, S, r, out);
    else if (stage == 1) g_klr_kernel<TT, RM><<<rgrid, kThreads, 0, st>>>(qlr, klr, t, ldt, R, S, r, uw, out);
    else g_qlr_kernel<TT, RM><<<cgrid, kThreads, 0, st>>>(qlr, klr, t, ldt, R, S, r, uw, out);
  };
  using R16 = std::integral_constant<int, 16>;
  using R64 = std::integral_constant<int, kMaxR>;
  if (t_f64) { if (r <= 16) run(double{}, R16{}); else run(double{}, R64{}); }
  else { if (r <= 16) run(float{}, R16{}); else run(float{}, R64{}); }
  return (int)cudaGetLastError();
}
