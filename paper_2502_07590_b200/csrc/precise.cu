// precise.cu — the reference-precision (fp64) path of the reference-named API.
//
// The reference computes in the caller's dtype, float64 by default (pkg/src/dynsparse/
// validate.py:10-25 `as_matrix`). Host fp64/fp32 callers of the drop-in API therefore get
// fp64 device arithmetic here, so the reference's own tolerances (1e-9 .. 1e-12) hold:
//
//   gemm_f64_kernel         predictor.py:94-100 `project` (X W), selection.py:149 / 204 / 222
//                           score tiles (Q_lr K_lr^T), attention.py:112-115 logits (/ sqrt(d))
//   softmax_rows_f64_kernel attention.py:88-92 `_stable_softmax_rows` (max-subtracted)
//   topk_f64_kernel         selection.py:118-175 / 178-242: exact per-row top-k, ties toward
//                           the lower index, indices ascending, threshold = k-th largest
//                           (fp64 order keys; -0.0 == +0.0 like numpy's comparisons)
//   sorted_stats_kernel     attention.py:118-140 `critical_kv_oracle` (descending order, ties
//                           toward the lower index, sequential cumsum exactly as np.cumsum,
//                           searchsorted(csum, min(theta, total) - eps, 'left') + 1) and
//                           attention.py:208-212 `analyze_distribution` top-fraction mass
//   histogram_f64_kernel    attention.py:214-216 np.histogram over given (log-spaced) edges
//
// None of this is on the bf16 hot path (the layer's K1-K3 kernels); it is the precision path
// for the numpy-in / numpy-out API, still entirely on the GPU (no CPU fallback).

#include "dsv_common.cuh"

namespace dsv {
namespace prec {

DSV_DEV uint64_t d2key(double x) {
  uint64_t u = (uint64_t)__double_as_longlong(x);
  if (u == 0x8000000000000000ull) u = 0ull;            // -0.0 == +0.0
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
DSV_DEV double key2d(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// ------------------------------------------------------------------ GEMM (fp64, CUDA cores)
// C[b][m][n] = (sum_{t=0}^{K-1} A[b](m, t) * B[b](t, n)) / div, fma in t order (deterministic;
// exact whenever the products and partial sums are, e.g. identity / zero / integer operands).
// A(m, t) = A[m * sam + t * sat], B(t, n) = B[t * sbt + n * sbn]: any strides (transposes are
// free). 64 x 64 outputs per CTA, 256 threads, 4 x 4 per thread, K staged 16 at a time.
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256)
gemm_f64_kernel(const double* __restrict__ A, long long sam, long long sat, long long a_bs,
                const double* __restrict__ B, long long sbt, long long sbn, long long b_bs,
                double* __restrict__ C, long long ldc, long long c_bs, int M, int N, int K,
                double div) {
  __shared__ double sA[kGK][kGT + 1];
  __shared__ double sB[kGK][kGT + 1];
  const int b = blockIdx.z;
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const double* Ab = A + b * a_bs;
  const double* Bb = B + b * b_bs;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int t0 = 0; t0 < K; t0 += kGK) {
    __syncthreads();
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int t = e / kGT, mm = e % kGT;
      const int gm = m0 + mm, gt = t0 + t;
      sA[t][mm] = (gm < M && gt < K) ? Ab[gm * sam + gt * sat] : 0.0;
      const int gn = n0 + mm;
      sB[t][mm] = (gn < N && gt < K) ? Bb[gt * sbt + gn * sbn] : 0.0;
    }
    __syncthreads();
    const int tn = min(kGK, K - t0);
    for (int t = 0; t < tn; ++t) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[t][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = sB[t][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
  }
  double* Cb = C + b * c_bs;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn < N) Cb[gm * ldc + gn] = (div == 1.0) ? acc[i][j] : acc[i][j] / div;
    }
  }
}

// ------------------------------------------------------------------ block helpers (256 thr)
template <int NT>
DSV_DEV double block_reduce(double v, double* red, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : v + w;
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < NT / 32; ++w) t = is_max ? fmax(t, red[w]) : t + red[w];
  return t;
}

// ------------------------------------------------------------------ row softmax (in place)
// x[r] <- exp(x[r] - max x[r]) / sum (attention.py:88-92).
__global__ void __launch_bounds__(256)
softmax_rows_f64_kernel(double* __restrict__ x, long long ld, int R, int N) {
  __shared__ double red[8];
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    double* row = x + r * ld;
    double m = -INFINITY;
    for (int i = threadIdx.x; i < N; i += 256) m = fmax(m, row[i]);
    m = block_reduce<256>(m, red, true);
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += 256) {
      const double w = exp(row[i] - m);
      row[i] = w;
      s += w;
    }
    s = block_reduce<256>(s, red, false);
    const double inv_s = s;
    for (int i = threadIdx.x; i < N; i += 256) row[i] = row[i] / inv_s;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ exact top-k (fp64 rows)
// Radix select of the k-th largest order key (8 digits of 8 bits), then an ordered emit:
// every key > v*, plus the first (k - #greater) keys == v* in index order, written ascending.
// One CTA (256 threads) per row, persistent over rows. Row r uses k = kp[r / rows_per_k].
constexpr int kTT = 256;
__global__ void __launch_bounds__(kTT)
topk_f64_kernel(const double* __restrict__ S, long long lds, int R, int L,
                const int* __restrict__ kp, int rows_per_k, int* __restrict__ out,
                long long ldo, double* __restrict__ thr) {
  __shared__ unsigned hist[256];
  __shared__ unsigned wcnt[2][kTT / 32];
  __shared__ unsigned s_b, s_above;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int row = blockIdx.x; row < R; row += gridDim.x) {
    const double* x = S + (long long)row * lds;
    const int k = kp[row / rows_per_k];
    uint64_t prefix = 0;
    unsigned remaining = (unsigned)k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      const uint64_t mask_hi = (shift == 56) ? 0ull : (~0ull << (shift + 8));
      hist[tid] = 0u;
      __syncthreads();
      for (int i = tid; i < L; i += kTT) {
        const uint64_t key = d2key(x[i]);
        if ((key & mask_hi) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (warp == 0) {
        // lane l owns buckets 255 - 8l .. 248 - 8l (descending); find the bucket holding the
        // remaining-th largest key
        unsigned c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { c[j] = hist[255 - 8 * lane - j]; tot += c[j]; }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned excl = incl - tot;
        const unsigned hit = __ballot_sync(0xffffffffu, excl < remaining && incl >= remaining);
        if (lane == __ffs(hit) - 1) {
          unsigned run = excl;
          int j = 0;
          while (run + c[j] < remaining) { run += c[j]; ++j; }
          s_b = 255u - 8u * lane - j;
          s_above = run;
        }
      }
      __syncthreads();
      prefix |= (uint64_t)s_b << shift;
      remaining -= s_above;
      __syncthreads();
    }
    const uint64_t kth = prefix;
    const unsigned need = remaining;     // ties at v* to take, in index order (>= 1)
    unsigned base = 0, ties = 0;
    for (int c0 = 0; c0 < L && base < (unsigned)k; c0 += kTT) {
      const int i = c0 + tid;
      uint64_t key = 0;
      if (i < L) key = d2key(x[i]);
      const bool gt = i < L && key > kth;
      const bool eq = i < L && key == kth;
      const unsigned lt_mask = (1u << lane) - 1u;
      const unsigned eqm = __ballot_sync(0xffffffffu, eq);
      if (lane == 0) wcnt[0][warp] = __popc(eqm);
      __syncthreads();
      unsigned eq_before = ties, eq_tot = 0;
      for (int w = 0; w < kTT / 32; ++w) {
        if (w < warp) eq_before += wcnt[0][w];
        eq_tot += wcnt[0][w];
      }
      const bool keep = gt || (eq && eq_before + __popc(eqm & lt_mask) < need);
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) wcnt[1][warp] = __popc(km);
      __syncthreads();
      unsigned k_before = base, k_tot = 0;
      for (int w = 0; w < kTT / 32; ++w) {
        if (w < warp) k_before += wcnt[1][w];
        k_tot += wcnt[1][w];
      }
      if (keep) out[(long long)row * ldo + k_before + __popc(km & lt_mask)] = i;
      base += k_tot;
      ties += eq_tot;
      __syncthreads();
    }
    if (tid == 0) thr[row] = key2d(kth);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ sorted-row statistics
// Per row of non-negative fp64 scores: sort (value descending, index ascending) by a bitonic
// network over (order key, index) pairs — in shared memory when the padded row fits, else in
// the caller's global scratch (one slab per CTA) — then one thread walks the sorted row:
//   total  = sequential sum (np.cumsum's order), n_keep = #{csum < min(theta, total) - eps} + 1
//   (capped at L; theta <= 0 skips it), topmass = sum of the first top_n values.
constexpr int kST = 1024;
__device__ __forceinline__ bool before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kST)
sorted_stats_kernel(const double* __restrict__ S, long long lds, int R, int L, int Lpad,
                    double theta, double eps, int top_n, int* __restrict__ n_keep,
                    double* __restrict__ topmass, uint64_t* __restrict__ gkeys,
                    uint32_t* __restrict__ gidx) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t* keys;
  uint32_t* idx;
  if (gkeys) {
    keys = gkeys + (long long)blockIdx.x * Lpad;
    idx = gidx + (long long)blockIdx.x * Lpad;
  } else {
    keys = reinterpret_cast<uint64_t*>(sm);
    idx = reinterpret_cast<uint32_t*>(sm + (size_t)Lpad * 8);
  }
  for (int row = blockIdx.x; row < R; row += gridDim.x) {
    const double* x = S + (long long)row * lds;
    for (int i = threadIdx.x; i < Lpad; i += kST) {
      keys[i] = (i < L) ? d2key(x[i]) : 0ull;
      idx[i] = (i < L) ? (uint32_t)i : 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= Lpad; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < (Lpad >> 1); t += kST) {
          const int lo = 2 * stride * (t / stride) + (t % stride);
          const int hi = lo + stride;
          const bool fwd = (lo & size) == 0;    // this run sorts in the 'before' order
          const uint64_t ka = keys[lo], kb = keys[hi];
          const uint32_t ia = idx[lo], ib = idx[hi];
          const bool swap = fwd ? before(kb, ib, ka, ia) : before(ka, ia, kb, ib);
          if (swap) {
            keys[lo] = kb; keys[hi] = ka;
            idx[lo] = ib; idx[hi] = ia;
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      double total = 0.0, top = 0.0;
      for (int i = 0; i < L; ++i) {
        const double v = key2d(keys[i]);
        total += v;
        if (i < top_n) top += v;
      }
      if (topmass) topmass[row] = top;
      if (n_keep) {
        int n = L;
        if (theta > 0.0) {
          const double target = fmin(theta, total) - eps;
          double c = 0.0;
          int cnt = 0;
          for (int i = 0; i < L; ++i) {
            c += key2d(keys[i]);
            if (c < target) ++cnt; else break;
          }
          n = min(cnt + 1, L);
        }
        n_keep[row] = n;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ histogram
// counts[b] += #{v : edges[b] <= v < edges[b+1]} (last bin closed), np.histogram semantics.
__global__ void __launch_bounds__(256)
histogram_f64_kernel(const double* __restrict__ S, long long lds, int R, int N,
                     const double* __restrict__ edges, int nb,
                     unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned sh[];
  for (int b = threadIdx.x; b < nb; b += 256) sh[b] = 0u;
  __syncthreads();
  const double lo = edges[0], hi = edges[nb];
  const long long total = (long long)R * N;
  for (long long e = (long long)blockIdx.x * 256 + threadIdx.x; e < total;
       e += (long long)gridDim.x * 256) {
    const double v = S[(e / N) * lds + e % N];
    if (!(v >= lo && v <= hi)) continue;
    int a = 0, b = nb;                  // largest a with edges[a] <= v
    while (b - a > 1) {
      const int m = (a + b) >> 1;
      if (edges[m] <= v) a = m; else b = m;
    }
    atomicAdd(&sh[a], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += 256)
    if (sh[b]) atomicAdd(&counts[b], (unsigned long long)sh[b]);
}

// ------------------------------------------------------------------ index-set statistics
// Per query q (one warp): |E_q & O_q| of two sorted CSR lists and the score masses
// sum_{j in E_q} S[q][j], sum_{j in O_q} S[q][j] (predictor.py:262-281 prediction_accuracy).
__global__ void __launch_bounds__(256)
set_stats_f64_kernel(const double* __restrict__ S, long long lds, int Q,
                     const long long* __restrict__ ep, const int* __restrict__ ec,
                     const long long* __restrict__ op, const int* __restrict__ oc,
                     int* __restrict__ inter, double* __restrict__ emass,
                     double* __restrict__ omass) {
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= Q) return;
  const double* row = S + (long long)q * lds;
  const long long e0 = ep[q], e1 = ep[q + 1], o0 = op[q], o1 = op[q + 1];
  int cnt = 0;
  double em = 0.0, om = 0.0;
  for (long long p = e0 + lane; p < e1; p += 32) {
    const int key = ec[p];
    em += row[key];
    long long a = o0, b = o1;                 // lower_bound of key in the oracle list
    while (a < b) {
      const long long m = (a + b) >> 1;
      if (oc[m] < key) a = m + 1; else b = m;
    }
    cnt += (a < o1 && oc[a] == key) ? 1 : 0;
  }
  for (long long p = o0 + lane; p < o1; p += 32) om += row[oc[p]];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    em += __shfl_xor_sync(0xffffffffu, em, o);
    om += __shfl_xor_sync(0xffffffffu, om, o);
  }
  if (lane == 0) {
    inter[q] = cnt;
    emass[q] = em;
    omass[q] = om;
  }
}

}  // namespace prec
}  // namespace dsv

using namespace dsv::prec;

static int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int dsv_gemm_f64_launch(const double* A, long long sam, long long sat, long long a_bs,
                        const double* B, long long sbt, long long sbn, long long b_bs, double* C,
                        long long ldc, long long c_bs, int M, int N, int K, int nbatch, double div,
                        cudaStream_t st) {
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, nbatch);
  gemm_f64_kernel<<<grid, 256, 0, st>>>(A, sam, sat, a_bs, B, sbt, sbn, b_bs, C, ldc, c_bs, M, N,
                                        K, div);
  return (int)cudaGetLastError();
}

int dsv_softmax_rows_f64_launch(double* x, long long ld, int R, int N, cudaStream_t st) {
  const int grid = R < 8 * sm_count() ? R : 8 * sm_count();
  softmax_rows_f64_kernel<<<grid, 256, 0, st>>>(x, ld, R, N);
  return (int)cudaGetLastError();
}

int dsv_topk_f64_launch(const double* S, long long lds, int R, int L, const int* kp, int rows_per_k,
                        int* out, long long ldo, double* thr, cudaStream_t st) {
  const int grid = R < 8 * sm_count() ? R : 8 * sm_count();
  topk_f64_kernel<<<grid, kTT, 0, st>>>(S, lds, R, L, kp, rows_per_k, out, ldo, thr);
  return (int)cudaGetLastError();
}

size_t dsv_sorted_stats_smem(int Lpad) { return (size_t)Lpad * 12; }

int dsv_sorted_stats_launch(const double* S, long long lds, int R, int L, int Lpad, double theta,
                            double eps, int top_n, int* n_keep, double* topmass, void* scratch,
                            int scratch_ctas, cudaStream_t st) {
  const size_t smem = dsv_sorted_stats_smem(Lpad);
  if (!scratch) {
    if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
    cudaFuncSetAttribute(sorted_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    const int grid = R < sm_count() ? R : sm_count();
    sorted_stats_kernel<<<grid, kST, smem, st>>>(S, lds, R, L, Lpad, theta, eps, top_n, n_keep,
                                                 topmass, nullptr, nullptr);
  } else {
    const int grid = R < scratch_ctas ? R : scratch_ctas;
    uint64_t* keys = reinterpret_cast<uint64_t*>(scratch);
    uint32_t* idx = reinterpret_cast<uint32_t*>(keys + (size_t)scratch_ctas * Lpad);
    sorted_stats_kernel<<<grid, kST, 0, st>>>(S, lds, R, L, Lpad, theta, eps, top_n, n_keep,
                                              topmass, keys, idx);
  }
  return (int)cudaGetLastError();
}

int dsv_histogram_f64_launch(const double* S, long long lds, int R, int N, const double* edges,
                             int nb, unsigned long long* counts, cudaStream_t st) {
  const long long total = (long long)R * N;
  long long blocks = (total + 255) / 256;
  if (blocks > 4LL * sm_count()) blocks = 4LL * sm_count();
  if (blocks < 1) blocks = 1;
  histogram_f64_kernel<<<(int)blocks, 256, (size_t)nb * 4, st>>>(S, lds, R, N, edges, nb, counts);
  return (int)cudaGetLastError();
}

int dsv_set_stats_f64_launch(const double* S, long long lds, int Q, const long long* ep,
                             const int* ec, const long long* op, const int* oc, int* inter,
                             double* emass, double* omass, cudaStream_t st) {
  const long long threads = (long long)Q * 32;
  set_stats_f64_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(S, lds, Q, ep, ec, op, oc,
                                                                         inter, emass, omass);
  return (int)cudaGetLastError();
}
