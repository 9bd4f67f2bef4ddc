// profiler.cu — critical-KV mass counts for the sampled sparsity profiler.
//
// Reference: pkg/src/dynsparse/profiler.py:48-79 `measure_block_sparsity` (sampled query
// rows scored against all keys, softmax, then attention.py:118-140 `critical_kv_oracle`:
// per row the shortest descending-score prefix whose mass reaches theta, ties toward the
// lower index; target = min(theta, total mass) - 1e-9) and attention.py:143-150
// `head_sparsity` (mean of (S - |I_q|) / S).
//
// One CTA (1024 threads) per row, persistent over rows; the row's fp32 logits are staged in
// shared memory when they fit. Arithmetic mirrors the reference in fp64: l_i = x_i / sqrt_d,
// l_i -= max, e_i = exp(l_i), p_i = e_i / sum(e). The prefix length is found without a
// sort: key-space bucket refinement over the logits' order keys (p is monotone in x), each
// level carrying per-bucket counts and fp64 masses; at a single key value x* with
// per-entry mass tau the prefix takes ceil((target - mass above) / tau) of the ties.
// Output: n_keep per row (int32).

#include "dsv_common.cuh"

namespace dsv {
namespace prof {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kBuckets = 1024;

DSV_DEV uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
DSV_DEV float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

struct alignas(16) Smem {
  double mass[kBuckets];
  uint32_t cnt[kBuckets];
  double wd[kWarps];
  uint32_t wu[kWarps];
  float wf[kWarps];
  double s_target, s_above_mass;
  uint32_t s_lo, s_hi, s_above_cnt, s_done, s_result;
};

DSV_DEV double block_sum_d(Smem& S, double v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) S.wd[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kWarps; ++w) t += S.wd[w];
  return t;
}

DSV_DEV float block_max_f(Smem& S, float v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) S.wf[warp] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int w = 0; w < kWarps; ++w) t = fmaxf(t, S.wf[w]);
  return t;
}

template <bool kSmem>
__global__ void __launch_bounds__(kThreads, 1)
critical_counts_kernel(const float* __restrict__ logits, long long ld, int rows, int L,
                       double sqrt_d, double theta, int* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  float* buf = reinterpret_cast<float*>(smem_raw + sizeof(Smem));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* g = logits + (long long)row * ld;
    const float* x = kSmem ? buf : g;
    if constexpr (kSmem) {
      for (int i = tid; i < L; i += kThreads) buf[i] = __ldg(g + i);
      __syncthreads();
    }
    float mx = -INFINITY;
    for (int i = tid; i < L; i += kThreads) mx = fmaxf(mx, x[i]);
    mx = block_max_f(S, mx);
    const double lmax = (double)mx / sqrt_d;
    auto e_of = [&](float v) { return exp((double)v / sqrt_d - lmax); };
    double se = 0.0;
    for (int i = tid; i < L; i += kThreads) se += e_of(x[i]);
    const double total = block_sum_d(S, se);
    double sp = 0.0;
    for (int i = tid; i < L; i += kThreads) sp += e_of(x[i]) / total;
    const double mass_all = block_sum_d(S, sp);
    // key range of the row
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int i = tid; i < L; i += kThreads) { const uint32_t k = f2key(x[i]); kmin = min(kmin, k); kmax = max(kmax, k); }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    __syncthreads();
    if (tid == 0) {
      S.s_lo = 0xffffffffu; S.s_hi = 0u; S.s_above_cnt = 0; S.s_above_mass = 0.0; S.s_done = 0;
      S.s_target = fmin(theta, mass_all) - 1e-9;
      if (S.s_target <= 0.0) { S.s_result = 1u; S.s_done = 1; }   // searchsorted -> 0
    }
    __syncthreads();
    if (lane == 0) { atomicMin(&S.s_lo, kmin); atomicMax(&S.s_hi, kmax); }
    __syncthreads();
    for (int level = 0; level < 8 && !S.s_done; ++level) {
      const uint32_t lo = S.s_lo, hi = S.s_hi;
      const uint64_t span = (uint64_t)(hi - lo) + 1ull;
      const uint32_t nb = span < (uint64_t)kBuckets ? (uint32_t)span : (uint32_t)kBuckets;
      const uint64_t m = ((uint64_t)nb << 32) / span;   // bucket(x) = ((x - lo) * m) >> 32
      for (int b = tid; b < kBuckets; b += kThreads) { S.mass[b] = 0.0; S.cnt[b] = 0u; }
      __syncthreads();
      for (int i = tid; i < L; i += kThreads) {
        const uint32_t k = f2key(x[i]);
        if (k >= lo && k <= hi) {
          const uint32_t b = (uint32_t)(((uint64_t)(k - lo) * m) >> 32);
          atomicAdd(&S.cnt[b], 1u);
          atomicAdd(&S.mass[b], e_of(x[i]) / total);
        }
      }
      __syncthreads();
      if (warp == 0) {
        // walk buckets from the top: lane owns 32 consecutive buckets, lanes descend
        const double above_m = S.s_above_mass;
        double lm = 0.0;
        uint32_t lc = 0;
        const int b0 = kBuckets - 32 * (lane + 1);   // this lane's buckets: b0 .. b0 + 31
        for (int i = 0; i < 32; ++i) { lm += S.mass[b0 + i]; lc += S.cnt[b0 + i]; }
        double cm = lm;      // inclusive prefix (higher buckets first)
        uint32_t cc = lc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double tm = __shfl_up_sync(0xffffffffu, cm, o);
          const uint32_t tc = __shfl_up_sync(0xffffffffu, cc, o);
          if (lane >= o) { cm += tm; cc += tc; }
        }
        // the target clamped to the mass this level actually holds (the fp64 sums of a
        // bucket and of its refinement may differ in the last bits)
        const double level_m = __shfl_sync(0xffffffffu, cm, 31);
        const double target = fmin(S.s_target, above_m + level_m);
        double before_m = above_m + cm - lm;
        uint32_t before_c = cc - lc;
        if (before_m < target && target <= above_m + cm) {
          int pick = b0;
          for (int i = 31; i >= 0; --i) {
            const double mb = S.mass[b0 + i];
            if (S.cnt[b0 + i] && before_m + mb >= target) { pick = b0 + i; break; }
            before_m += mb;
            before_c += S.cnt[b0 + i];
          }
          const uint64_t bb = (uint64_t)pick;
          const unsigned long long f0 = ((bb << 32) + m - 1) / m;
          const unsigned long long f1 = (((bb + 1) << 32) + m - 1) / m;
          const uint32_t nlo = lo + (uint32_t)f0;
          const uint32_t nhi = lo + (uint32_t)min(f1 - 1ull, (unsigned long long)(hi - lo));
          S.s_above_mass = before_m;
          S.s_above_cnt += before_c;
          if (nlo >= nhi) {
            // single key value: take ceil((target - above) / tau) of its entries
            const double tau = exp((double)key2f(nlo) / sqrt_d - lmax) / total;
            const uint32_t c = S.cnt[pick];
            double need = tau > 0.0 ? ceil((target - before_m) / tau) : (double)c;
            need = fmin(fmax(need, 1.0), (double)c);
            S.s_result = S.s_above_cnt + (uint32_t)need;
            S.s_done = 1;
          }
          S.s_lo = nlo;
          S.s_hi = nhi;
        }
      }
      __syncthreads();
    }
    if (tid == 0) {
      uint32_t r = S.s_done ? S.s_result : S.s_above_cnt + 1u;
      out[row] = (int)min(r, (uint32_t)L);
    }
    __syncthreads();
  }
}

}  // namespace prof
}  // namespace dsv

int dsv_critical_counts_launch(const float* logits, long long ld, int rows, int L, double sqrt_d,
                               double theta, int* out, cudaStream_t st) {
  using namespace dsv::prof;
  if (rows <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = rows < 2 * sms ? rows : 2 * sms;
  const size_t base = sizeof(Smem);
  const size_t need = base + (size_t)L * 4;
  if (need <= 200 * 1024) {
    cudaFuncSetAttribute(critical_counts_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    critical_counts_kernel<true><<<grid, kThreads, need, st>>>(logits, ld, rows, L, sqrt_d, theta, out);
  } else {
    cudaFuncSetAttribute(critical_counts_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)base);
    critical_counts_kernel<false><<<grid, kThreads, base, st>>>(logits, ld, rows, L, sqrt_d, theta, out);
  }
  return (int)cudaGetLastError();
}
