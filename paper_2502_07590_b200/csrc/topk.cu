// topk.cu — K2: exact per-row top-k selection over fp32 approximate scores.
//
// Semantics (reference: pkg/src/dynsparse/selection.py:82-115 `_merge_block`,
// :166-174 emit, :178-242 `twopass_select`):
//   * keep the k largest scores of a row; ties at the k-th value resolve toward
//     the lower column index;
//   * indices are emitted in ascending order;
//   * the threshold is the k-th largest score (= min of the kept scores);
//   * -0.0 compares equal to +0.0 (numpy semantics).
//
// B200 design: one CTA (1024 threads) per row. The row is staged once into
// shared memory as order-preserving uint32 keys (128 KB at L=32000). The
// k-th key T is found by iterative bucket refinement in key space: a histogram
// of min(2048, span) linear buckets over [lo, hi] narrows the range by ~2^11
// per level (<= 3 levels for 32-bit keys); once the bucket holding T has few
// members they are compacted into a candidate buffer and later levels run on
// that buffer only. The emit is the two-pass scheme of twopass_select: per-warp
// counts of (key > T) and (key == T) over contiguous index segments, a block
// scan, then an ordered compaction with warp ballots — so ascending output
// needs no sort. HBM traffic = one read of the row + k*4 bytes of indices.
// Rows longer than the shared-memory budget re-read keys from global/L2.

#include "dsv_common.cuh"

namespace dsv {
namespace topk {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kBuckets = 2048;
constexpr int kCandCap = 8192;

DSV_DEV uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;  // -0.0 == +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
DSV_DEV float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

struct alignas(16) Smem {
  uint32_t hist[kBuckets];
  uint32_t cand[kCandCap];
  uint32_t wa[kWarps], wb[kWarps], wc[kWarps];
  uint32_t s_lo, s_hi, s_need, s_ncand, s_T, s_mode;
  uint32_t s_gt_total;
};

template <bool kSmem>
struct Src {
  const uint32_t* keys;   // smem keys (kSmem)
  const float* row;       // global row (!kSmem)
  DSV_DEV uint32_t operator()(int i) const {
    if constexpr (kSmem) return keys[i];
    else return f2key(__ldg(row + i));
  }
};

DSV_DEV uint32_t warp_sum(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DSV_DEV uint32_t warp_min(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
DSV_DEV uint32_t warp_max(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <bool kSmem>
__global__ void __launch_bounds__(kThreads, 1)
topk_rows_kernel(const float* __restrict__ scores, long long ld, int L,
                 const int* __restrict__ k_per_head, int rows_per_head,
                 int* __restrict__ out_idx, long long out_ld, float* __restrict__ out_thr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Smem));

  const int row = blockIdx.x;
  const int k = k_per_head[row / rows_per_head];
  const float* src_row = scores + (long long)row * ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- stage keys (vectorised) + running min/max
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  if constexpr (kSmem) {
    const bool vec = ((reinterpret_cast<uintptr_t>(src_row) & 15) == 0);
    if (vec) {
      const int n4 = L >> 2;
      const float4* r4 = reinterpret_cast<const float4*>(src_row);
      uint4* k4 = reinterpret_cast<uint4*>(keys);
      for (int i = tid; i < n4; i += kThreads) {
        float4 v = __ldg(r4 + i);
        uint4 q = make_uint4(f2key(v.x), f2key(v.y), f2key(v.z), f2key(v.w));
        k4[i] = q;
        kmin = min(min(min(kmin, q.x), min(q.y, q.z)), q.w);
        kmax = max(max(max(kmax, q.x), max(q.y, q.z)), q.w);
      }
      for (int i = (n4 << 2) + tid; i < L; i += kThreads) {
        uint32_t q = f2key(__ldg(src_row + i));
        keys[i] = q; kmin = min(kmin, q); kmax = max(kmax, q);
      }
    } else {
      for (int i = tid; i < L; i += kThreads) {
        uint32_t q = f2key(__ldg(src_row + i));
        keys[i] = q; kmin = min(kmin, q); kmax = max(kmax, q);
      }
    }
  } else {
    for (int i = tid; i < L; i += kThreads) {
      uint32_t q = f2key(__ldg(src_row + i));
      kmin = min(kmin, q); kmax = max(kmax, q);
    }
  }
  kmin = warp_min(kmin); kmax = warp_max(kmax);
  if (lane == 0) { S.wa[warp] = kmin; S.wb[warp] = kmax; }
  __syncthreads();
  if (warp == 0) {
    uint32_t a = S.wa[lane], b = S.wb[lane];
    a = warp_min(a); b = warp_max(b);
    if (lane == 0) {
      S.s_lo = a; S.s_hi = b; S.s_need = (uint32_t)k; S.s_mode = 0; S.s_ncand = 0;
    }
  }
  __syncthreads();

  Src<kSmem> src{keys, src_row};

  // ---- iterative bucket refinement for T = k-th largest key
  for (int level = 0; level < 8; ++level) {
    const uint32_t lo = S.s_lo, hi = S.s_hi, need = S.s_need, mode = S.s_mode;
    if (lo == hi) break;
    const uint64_t span = (uint64_t)(hi - lo) + 1ull;
    const uint32_t nb = span < (uint64_t)kBuckets ? (uint32_t)span : (uint32_t)kBuckets;
    for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
    __syncthreads();
    const int n = mode ? (int)S.s_ncand : L;
    for (int i = tid; i < n; i += kThreads) {
      const uint32_t key = mode ? S.cand[i] : src(i);
      if (key >= lo && key <= hi) {
        const uint32_t b = (uint32_t)(((uint64_t)(key - lo) * nb) / span);
        atomicAdd(&S.hist[b], 1u);
      }
    }
    __syncthreads();
    // suffix scan: locate bucket b* with sum_{b>b*} < need <= sum_{b>=b*}
    // each thread owns 2 consecutive buckets (kBuckets = 2 * kThreads)
    {
      const uint32_t h0 = S.hist[2 * tid], h1 = S.hist[2 * tid + 1];
      uint32_t tot = h0 + h1;
      // inclusive suffix sum across threads: reverse-order warp scan
      uint32_t v = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v += t;
      }
      if (lane == 0) S.wc[warp] = v;  // warp total
      __syncthreads();
      uint32_t after = 0;  // sum of buckets in warps with higher index
      for (int w = warp + 1; w < kWarps; ++w) after += S.wc[w];
      const uint32_t incl = v + after;        // sum of buckets >= 2*tid
      const uint32_t excl = incl - tot;       // sum of buckets > 2*tid+1
      // bucket 2*tid+1: above = excl, at = h1 ; bucket 2*tid: above = excl + h1, at = h0
      int bstar = -1; uint32_t above = 0, at = 0;
      if (excl < need && need <= excl + h1) { bstar = 2 * tid + 1; above = excl; at = h1; }
      else if (excl + h1 < need && need <= incl) { bstar = 2 * tid; above = excl + h1; at = h0; }
      if (bstar >= 0 && bstar < (int)nb) {
        const uint64_t b = (uint64_t)bstar;
        const uint32_t nlo = lo + (uint32_t)((b * span + nb - 1) / nb);
        const uint32_t nhi = lo + (uint32_t)(((b + 1) * span + nb - 1) / nb) - 1u;
        S.s_lo = nlo; S.s_hi = nhi; S.s_need = need - above;
        S.wa[0] = at;  // members of the chosen bucket
      }
    }
    __syncthreads();
    if (!mode && S.wa[0] <= (uint32_t)kCandCap && S.s_lo != S.s_hi) {
      // compact the chosen bucket's members into the candidate buffer
      const uint32_t nlo = S.s_lo, nhi = S.s_hi;
      if (tid == 0) S.s_ncand = 0;
      __syncthreads();
      for (int base = warp * 32; base < L; base += kThreads) {
        const int i = base + lane;
        uint32_t key = (i < L) ? src(i) : 0u;
        const bool in = (i < L) && key >= nlo && key <= nhi;
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        uint32_t off = 0;
        if (lane == 0 && m) off = atomicAdd(&S.s_ncand, (uint32_t)__popc(m));
        off = __shfl_sync(0xffffffffu, off, 0);
        if (in) S.cand[off + __popc(m & ((1u << lane) - 1u))] = key;
      }
      __syncthreads();
      if (tid == 0) S.s_mode = 1;
      __syncthreads();
    }
  }
  __syncthreads();
  const uint32_t T = S.s_lo;

  // ---- emit pass 1: per-warp counts of (> T) and (== T) over contiguous segments
  const int seg = (((L + kWarps - 1) / kWarps) + 31) & ~31;
  const int s0 = warp * seg, s1 = min(L, s0 + seg);
  uint32_t ngt = 0, neq = 0;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const uint32_t key = (i < s1) ? src(i) : 0u;
    const bool valid = i < s1;
    ngt += __popc(__ballot_sync(0xffffffffu, valid && key > T));
    neq += __popc(__ballot_sync(0xffffffffu, valid && key == T));
  }
  if (lane == 0) { S.wa[warp] = ngt; S.wb[warp] = neq; }
  __syncthreads();
  if (warp == 0) {
    // exclusive scans over the 32 warps
    uint32_t g = S.wa[lane], e = S.wb[lane];
    uint32_t gi = g, ei = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t1 = __shfl_up_sync(0xffffffffu, gi, o);
      uint32_t t2 = __shfl_up_sync(0xffffffffu, ei, o);
      if (lane >= o) { gi += t1; ei += t2; }
    }
    const uint32_t gtot = __shfl_sync(0xffffffffu, gi, 31);
    const uint32_t need_eq = (uint32_t)k - gtot;
    const uint32_t gex = gi - g, eex = ei - e;
    S.wa[lane] = gex + min(eex, need_eq);  // kept elements before this warp
    S.wb[lane] = eex;                       // ties before this warp
    if (lane == 0) S.s_gt_total = gtot;
  }
  __syncthreads();
  const uint32_t need_eq = (uint32_t)k - S.s_gt_total;
  uint32_t kept = S.wa[warp];
  uint32_t eqs = S.wb[warp];
  int* orow = out_idx + (long long)row * out_ld;
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = s0; base < s1; base += 32) {
    const int i = base + lane;
    const bool valid = i < s1;
    const uint32_t key = valid ? src(i) : 0u;
    const uint32_t mgt = __ballot_sync(0xffffffffu, valid && key > T);
    const uint32_t meq = __ballot_sync(0xffffffffu, valid && key == T);
    const bool is_eq = (meq >> lane) & 1u;
    const bool keep_eq = is_eq && (eqs + __popc(meq & lt)) < need_eq;
    const uint32_t mkeep = mgt | __ballot_sync(0xffffffffu, keep_eq);
    if ((mkeep >> lane) & 1u) orow[kept + __popc(mkeep & lt)] = i;
    kept += __popc(mkeep);
    eqs += __popc(meq);
  }
  if (tid == 0) out_thr[row] = key2f(T);
}

}  // namespace topk
}  // namespace dsv

// --------------------------------------------------------------- launchers
size_t dsv_topk_smem_bytes(int L) {
  const size_t base = sizeof(dsv::topk::Smem);
  const size_t need = base + (size_t)L * 4;
  return need <= 227 * 1024 ? need : base;
}

int dsv_topk_launch(const float* scores, long long ld, int rows, int L, const int* k_per_head,
                    int rows_per_head, int* out_idx, long long out_ld, float* out_thr,
                    cudaStream_t stream) {
  using namespace dsv::topk;
  const size_t base = sizeof(Smem);
  const size_t need = base + (size_t)L * 4;
  if (rows <= 0) return 0;
  if (need <= 227 * 1024) {
    cudaFuncSetAttribute(topk_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)need);
    topk_rows_kernel<true><<<rows, kThreads, need, stream>>>(
        scores, ld, L, k_per_head, rows_per_head, out_idx, out_ld, out_thr);
  } else {
    cudaFuncSetAttribute(topk_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)base);
    topk_rows_kernel<false><<<rows, kThreads, base, stream>>>(
        scores, ld, L, k_per_head, rows_per_head, out_idx, out_ld, out_thr);
  }
  return (int)cudaGetLastError();
}
