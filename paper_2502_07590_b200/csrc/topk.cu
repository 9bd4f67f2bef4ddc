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
// B200 design: persistent CTAs (1024 threads, one row at a time, grid = #SMs).
// A row is brought into shared memory with one cp.async.bulk copy (the next
// row of the CTA is prefetched into L2 while the current one is processed).
// Three passes over the row in shared memory:
//   1. histogram: 2048 buckets linear in the score value over a range taken
//      from a strided sample (bucket = clamp(int(fma(v, a, b)))): monotone in
//      v, so the bucket b* holding the k-th value T follows from a suffix scan;
//      bell-shaped rows spread over many buckets, so smem atomics rarely collide;
//   2. per contiguous warp segment: count the entries in buckets > b* (all kept)
//      and compact the bucket-b* entries (value, index) into a candidate list;
//      T is then found exactly among the candidates by key-space bucket
//      refinement (<= 3 levels for 32-bit order keys), and the candidates give
//      each warp segment its (> T, == T) counts;
//   3. ordered compaction with warp ballots: keep v > T, and v == T while the
//      tie budget k - #(> T) lasts in index order (twopass_select's emit) —
//      ascending output, no sort. Float compares give -0.0 == +0.0.
// Rows whose T-bucket is too large (massive ties, non-finite ranges) fall back
// to key-space refinement over the whole row and a counting pass. Rows too long for
// shared memory go to the streaming kernel in topk_stream.cu.
// HBM traffic per row = one read of the row + k*4 bytes of indices.

#include "dsv_common.cuh"

// Optional phase profiling (tools/topk_phase.cu): cycles per phase, CTA 0 thread 0.
#ifdef DSV_TOPK_PROF
__device__ unsigned long long g_topk_prof[16];
#define TOPK_MARK(n) do { if (threadIdx.x == 0 && blockIdx.x == 0) { const long long _t = clock64(); \
    g_topk_prof[n] += _t - _prof_t; _prof_t = _t; } } while (0)
#else
#define TOPK_MARK(n) do { } while (0)
#endif

namespace dsv {
namespace topk {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kBuckets = 2048;
constexpr int kCandCap = 4096;
constexpr int kSample = 8192;
constexpr int kCandW = kCandCap / kWarps;   // per-warp candidate staging (pass 1)

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
  uint32_t cand[kCandCap];       // candidate order keys
  uint32_t cidx[kCandCap];       // candidate column ids
  uint32_t wa[kWarps], wb[kWarps], wc[kWarps], wd[kWarps];
  uint32_t s_lo, s_hi, s_need, s_ncand, s_mode, s_gt_total, s_cmin, s_cmax, s_kband;
  float s_vmin, s_vmax;
  uint64_t bar;
};

template <bool kSmem>
struct Src {
  const float* vals;   // smem row (kSmem) or global row
  DSV_DEV float val(int i) const {
    if constexpr (kSmem) return vals[i];
    else return __ldg(vals + i);
  }
  DSV_DEV uint32_t key(int i) const { return f2key(val(i)); }
};

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

// Value-space bucket: correctly rounded fma and saturating conversion keep it
// monotone non-decreasing in v (also for +-inf outside the sampled range).
DSV_DEV int vbucket(float v, float a, float b) {
  return min(max(__float2int_rz(__fmaf_rn(v, a, b)), 0), kBuckets - 1);
}

// Keep-mask addressing: plain (bit i&31 of word i>>5) or the pass-1 vec4 layout
// (chunk of 128 columns = 4 words; column 128c + 4l + j -> word 4c + j, bit l).
DSV_DEV uint32_t mword(uint32_t i, bool vec4) {
  return vec4 ? ((i >> 7) << 2) + (i & 3) : (i >> 5);
}
DSV_DEV uint32_t mbit(uint32_t i, bool vec4) {
  return vec4 ? 1u << ((i & 127) >> 2) : 1u << (i & 31);
}

// Locate bucket b* with sum_{b>b*} hist < need <= sum_{b>=b*} hist. Each thread owns
// buckets 2t, 2t+1. Returns through smem: wa[0] = b*, wb[0] = count above, wc[0]=count at.
DSV_DEV void find_bucket(Smem& S, uint32_t need, int tid, int lane, int warp) {
  const uint32_t h0 = S.hist[2 * tid], h1 = S.hist[2 * tid + 1];
  const uint32_t tot = h0 + h1;
  uint32_t v = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v += t;
  }
  if (lane == 0) S.wc[warp] = v;       // warp totals
  __syncthreads();
  // exclusive suffix over warps: sum of totals of warps > warp
  uint32_t wt = S.wc[lane];
  uint32_t suf = wt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_down_sync(0xffffffffu, suf, o);
    if (lane + o < 32) suf += t;
  }
  const uint32_t after = __shfl_sync(0xffffffffu, suf - wt, warp);
  const uint32_t incl = v + after;     // sum of buckets >= 2 tid
  const uint32_t excl = incl - tot;    // sum of buckets > 2 tid + 1
  __syncthreads();
  if (excl < need && need <= excl + h1) { S.wa[0] = 2 * tid + 1; S.wb[0] = excl; S.wc[0] = h1; }
  else if (excl + h1 < need && need <= incl) { S.wa[0] = 2 * tid; S.wb[0] = excl + h1; S.wc[0] = h0; }
  __syncthreads();
}

// Key-space refinement: [s_lo, s_hi] holds T, s_need-th largest inside; source is
// the candidate buffer (s_mode == 1) or the whole row.
template <bool kSmem>
DSV_DEV void refine(Smem& S, const Src<kSmem>& src, int L, int tid, int lane, int warp) {
  for (int level = 0; level < 40; ++level) {
    const uint32_t lo = S.s_lo, hi = S.s_hi, need = S.s_need, mode = S.s_mode;
    if (lo == hi) return;
    const uint64_t span = (uint64_t)(hi - lo) + 1ull;
    const uint32_t nb = span < (uint64_t)kBuckets ? (uint32_t)span : (uint32_t)kBuckets;
    for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
    __syncthreads();
    const int n = mode ? (int)S.s_ncand : L;
    for (int i = tid; i < n; i += kThreads) {
      const uint32_t key = mode ? S.cand[i] : src.key(i);
      if (key >= lo && key <= hi)
        atomicAdd(&S.hist[(uint32_t)(((uint64_t)(key - lo) * nb) / span)], 1u);
    }
    __syncthreads();
    find_bucket(S, need, tid, lane, warp);
    const uint64_t b = S.wa[0];
    const uint32_t nlo = lo + (uint32_t)((b * span + nb - 1) / nb);
    const uint32_t nhi = lo + (uint32_t)(((b + 1) * span + nb - 1) / nb) - 1u;
    const uint32_t above = S.wb[0];
    __syncthreads();
    if (tid == 0) { S.s_lo = nlo; S.s_hi = nhi; S.s_need = need - above; }
    __syncthreads();
  }
}

template <bool kSmem>
__global__ void __launch_bounds__(kThreads, 1)
topk_rows_kernel(const float* __restrict__ scores, long long ld, int rows, int L,
                 const int* __restrict__ k_per_head, int rows_per_head,
                 int* __restrict__ out_idx, long long out_ld, float* __restrict__ out_thr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  float* buf = reinterpret_cast<float*>(smem_raw + sizeof(Smem));
  const int nw = (L + 31) >> 5;                        // 32-column mask words
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Smem) + (kSmem ? (size_t)L * 4 : 0));
  uint32_t* bmask = mask + ((L + 127) / 128 * 4 + 4);   // band-candidate bits (pass 1)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool bulk = kSmem && (((ld * 4) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(scores) & 15) == 0) && L >= 4;
  const int n4 = L >> 2;
  // bulk L2 prefetch of later rows needs 16-byte aligned row starts
  const bool row_al16 = (((ld * 4) & 15) == 0) && ((reinterpret_cast<uintptr_t>(scores) & 15) == 0);
  const int seg = (((L + kWarps - 1) / kWarps) + 127) & ~127;  // contiguous warp segments (x128)
  const int s0 = warp * seg, s1 = min(L, s0 + seg);
  const uint32_t lt = (1u << lane) - 1u;
  const int sstride = max(1, L / kSample) | 1;             // odd: conflict-free sample reads
  const bool vec4 = false;   // plain keep-mask layout (see mword / mbit)
  if (tid == 0) { mbar_init(&S.bar, 1); fence_barrier_init(); }
  __syncthreads();
  uint32_t phase = 0;
  bool inflight = false;   // this row's bulk copy was issued during the previous row
#ifdef DSV_TOPK_PROF
  long long _prof_t = clock64();
#endif

  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const int k = k_per_head[row / rows_per_head];
    const float* grow = scores + (long long)row * ld;
    if (tid == 0 && row + 2 * (int)gridDim.x < rows && n4 > 0 && row_al16)
      prefetch_l2(scores + (long long)(row + 2 * gridDim.x) * ld, (uint32_t)n4 * 16u);

    // ---- stage the row (raw fp32) in shared memory
    if constexpr (kSmem) {
      if (bulk) {
        if (tid == 0 && !inflight) {
          fence_proxy_async_smem();   // previous row's generic reads before the async write
          mbar_arrive_expect_tx(&S.bar, (uint32_t)n4 * 16u);
          bulk_load(buf, grow, (uint32_t)n4 * 16u, &S.bar);
        }
        inflight = false;
        for (int i = (n4 << 2) + tid; i < L; i += kThreads) buf[i] = __ldg(grow + i);
        mbar_wait(&S.bar, phase);
        phase ^= 1;
      } else {
        for (int i = tid; i < L; i += kThreads) buf[i] = __ldg(grow + i);
      }
      __syncthreads();
    }
    Src<kSmem> src{kSmem ? buf : grow};
    TOPK_MARK(0);

    // ---- value range from a strided sample (any range is correct; a good one is fast)
    {
      const int i = (int)(((long long)tid * L) / kThreads);
      const float v = i < L ? src.val(i) : src.val(0);
      float mn = v, mx = v;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) { S.wa[warp] = __float_as_uint(mn); S.wb[warp] = __float_as_uint(mx); }
      for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
      __syncthreads();
      if (warp == 0) {
        mn = __uint_as_float(S.wa[lane]);
        mx = __uint_as_float(S.wb[lane]);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
          S.s_vmin = mn; S.s_vmax = mx; S.s_ncand = 0; S.s_mode = 0;
          S.s_cmin = 0xffffffffu; S.s_cmax = 0u;
        }
      }
      __syncthreads();
    }
    const float vmin = S.s_vmin, vmax = S.s_vmax;
    bool fast = isfinite(vmin) && isfinite(vmax) && vmax > vmin;
    const float ba = fast ? (float)kBuckets / (vmax - vmin) : 0.f;
    const float bb = -vmin * ba;
    uint32_t n_above = 0;   // this warp's entries in buckets > B_hi
    if (fast) {
      // ---- sample histogram (kSample strided entries) -> bucket band [B_lo, B_hi]
      //      expected to hold T: ~k*kSample/L sample entries lie above T, +- 4 sigma.
#pragma unroll
      for (int j = 0; j < kSample / kThreads; ++j) {
        const int i = min((tid + j * kThreads) * sstride, L - 1);
        atomicAdd(&S.hist[vbucket(src.val(i), ba, bb)], 1u);
      }
      __syncthreads();
      {
        const float t = (float)k * (float)kSample / (float)L;
        const float m = 4.f * sqrtf(fmaxf(t * (1.f - t / kSample), 1.f)) + 2.f;
        const float tm = t - m, tp = t + m;
        const uint32_t h0 = S.hist[2 * tid], h1 = S.hist[2 * tid + 1];
        uint32_t v = h0 + h1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_down_sync(0xffffffffu, v, o);
          if (lane + o < 32) v += x;
        }
        if (lane == 0) S.wc[warp] = v;
        if (tid == 0) { S.wa[0] = kBuckets - 1; S.wb[0] = 0; }   // defaults: B_hi = top, B_lo = 0
        __syncthreads();
        const uint32_t wt = S.wc[lane];
        uint32_t suf = wt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o);
          if (lane + o < 32) suf += x;
        }
        const uint32_t after = __shfl_sync(0xffffffffu, suf - wt, warp);
        // C(b) = samples in buckets >= b, for b = 2 tid, 2 tid + 1, 2 tid + 2
        const float c0 = (float)(v + after), c1 = c0 - (float)h0, c2 = c1 - (float)h1;
        __syncthreads();
        if (tm > 0.f) {
          if (c1 <= tm && c0 > tm) S.wa[0] = 2 * tid;
          if (c2 <= tm && c1 > tm) S.wa[0] = 2 * tid + 1;
        }
        if (tp < (float)kSample) {
          if (c0 >= tp && c1 < tp) S.wb[0] = 2 * tid;
          if (c1 >= tp && c2 < tp) S.wb[0] = 2 * tid + 1;
        }
        __syncthreads();
      }
      const int b_hi = (int)S.wa[0], b_lo = min((int)S.wb[0], b_hi);
      // value band: above <=> v > hi_v, candidate <=> lo_v <= v <= hi_v (any choice is
      // exact after the band check below; bucket edges make it tight)
      const float hi_v = b_hi >= kBuckets - 1 ? INFINITY : vmin + (float)(b_hi + 1) / ba;
      const float lo_v = b_lo <= 0 ? -INFINITY : vmin + (float)b_lo / ba;
      TOPK_MARK(1);
      // ---- pass 1: per contiguous warp segment, above-mask words and band candidates
      //      (staged per warp: no shared counter, so no cross-warp atomic contention)
      uint32_t cmin = 0xffffffffu, cmax = 0u, wcnt = 0;
      uint32_t* wcand = S.cand + warp * kCandW;
      uint32_t* wcidx = S.cidx + warp * kCandW;
      // 128 columns per warp step: one 16-byte shared load per lane; the above-mask words
      // (plain bit order) are assembled from per-lane nibbles with three shuffles
      for (int base = s0; base < s1; base += 128) {
        const int i0 = base + 4 * lane;
        float4 v;
        if (kSmem && i0 + 3 < s1) {
          v = reinterpret_cast<const float4*>(src.vals)[i0 >> 2];
        } else {
          v.x = i0 < s1 ? src.val(i0) : 0.f;
          v.y = i0 + 1 < s1 ? src.val(i0 + 1) : 0.f;
          v.z = i0 + 2 < s1 ? src.val(i0 + 2) : 0.f;
          v.w = i0 + 3 < s1 ? src.val(i0 + 3) : 0.f;
        }
        const bool ok0 = i0 < s1, ok1 = i0 + 1 < s1, ok2 = i0 + 2 < s1, ok3 = i0 + 3 < s1;
        const bool g0 = ok0 && v.x > hi_v, g1 = ok1 && v.y > hi_v, g2 = ok2 && v.z > hi_v, g3 = ok3 && v.w > hi_v;
        const uint32_t gt = (uint32_t)g0 | ((uint32_t)g1 << 1) | ((uint32_t)g2 << 2) | ((uint32_t)g3 << 3);
        n_above += __popc(gt);
        uint32_t wv = gt << (4 * (lane & 7));
        wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
        wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
        wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
        if ((lane & 7) == 0 && base + 32 * (lane >> 3) < s1) mask[(base >> 5) + (lane >> 3)] = wv;
        const bool n0 = ok0 && !g0 && v.x >= lo_v, n1 = ok1 && !g1 && v.y >= lo_v;
        const bool n2 = ok2 && !g2 && v.z >= lo_v, n3 = ok3 && !g3 && v.w >= lo_v;
        uint32_t bw = ((uint32_t)n0 | ((uint32_t)n1 << 1) | ((uint32_t)n2 << 2) | ((uint32_t)n3 << 3))
                      << (4 * (lane & 7));
        bw |= __shfl_xor_sync(0xffffffffu, bw, 1);
        bw |= __shfl_xor_sync(0xffffffffu, bw, 2);
        bw |= __shfl_xor_sync(0xffffffffu, bw, 4);
        if ((lane & 7) == 0 && base + 32 * (lane >> 3) < s1) bmask[(base >> 5) + (lane >> 3)] = bw;
      }
      __syncwarp();
      // band candidates from this warp's band-mask words: lane j takes word j of each
      // 32-word group, a warp scan of the popcounts gives the slots
      for (int w0 = s0 >> 5; w0 < ((s1 + 31) >> 5); w0 += 32) {
        const int w = w0 + lane;
        uint32_t m = w < ((s1 + 31) >> 5) ? bmask[w] : 0u;
        const uint32_t c = __popc(m);
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += x;
        }
        uint32_t slot = wcnt + inc - c;
        while (m) {
          const int i = w * 32 + __ffs(m) - 1;
          m &= m - 1;
          const uint32_t key = f2key(src.val(i));
          if (slot < (uint32_t)kCandW) { wcand[slot] = key; wcidx[slot] = (uint32_t)i; }
          ++slot;
          cmin = min(cmin, key);
          cmax = max(cmax, key);
        }
        wcnt += __shfl_sync(0xffffffffu, inc, 31);
      }
      TOPK_MARK(8);
#pragma unroll
      for (int o = 16; o; o >>= 1) n_above += __shfl_xor_sync(0xffffffffu, n_above, o);   // per-lane counts
      cmin = warp_min(cmin);
      cmax = warp_max(cmax);
      if (lane == 0) {
        atomicMin(&S.s_cmin, cmin);
        atomicMax(&S.s_cmax, cmax);
        S.wc[warp] = n_above;
        S.wd[warp] = wcnt;
      }
      __syncthreads();
      if (warp == 0) {
        uint32_t tot = S.wc[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const uint32_t c = S.wd[lane];
        uint32_t ci = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_up_sync(0xffffffffu, ci, o);
          if (lane >= o) ci += x;
        }
        const bool over = __any_sync(0xffffffffu, c > (uint32_t)kCandW);
        S.wb[lane] = ci - c;                   // compacted base of this warp's candidates
        const uint32_t nc = __shfl_sync(0xffffffffu, ci, 31);
        if (lane == 0) {
          const bool ok = !over && tot < (uint32_t)k && (uint32_t)k <= tot + nc;
          S.s_mode = ok ? 1u : 2u;
          S.s_ncand = nc;
          S.s_lo = S.s_cmin; S.s_hi = S.s_cmax;
          S.s_need = (uint32_t)k - tot; S.s_kband = (uint32_t)k - tot;
        }
      }
      __syncthreads();
      fast = S.s_mode == 1;
      if (fast) {
        // compact the per-warp staging into one list (destinations never overlap a
        // later warp's source region: each warp holds <= kCandW entries)
        uint32_t kk[kCandW / 32], ii[kCandW / 32];
        const uint32_t cb = S.wb[warp];
#pragma unroll
        for (int j = 0; j < kCandW / 32; ++j) {
          const uint32_t q = j * 32 + lane;
          kk[j] = q < wcnt ? wcand[q] : 0u;
          ii[j] = q < wcnt ? wcidx[q] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kCandW / 32; ++j) {
          const uint32_t q = j * 32 + lane;
          if (q < wcnt) { S.cand[cb + q] = kk[j]; S.cidx[cb + q] = ii[j]; }
        }
        TOPK_MARK(9);
        // the row buffer is no longer needed on the fast path: start the next row's load
        if constexpr (kSmem) {
          if (bulk && tid == 0 && row + (int)gridDim.x < rows) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&S.bar, (uint32_t)n4 * 16u);
            bulk_load(buf, scores + (long long)(row + gridDim.x) * ld, (uint32_t)n4 * 16u, &S.bar);
          }
          inflight = bulk && row + (int)gridDim.x < rows;
        }
      }
      __syncthreads();
      TOPK_MARK(2);
    }
    if (!fast) {
      // whole-row key-space refinement (ties-heavy or non-finite rows)
      uint32_t kmin = 0xffffffffu, kmax = 0u;
      for (int i = tid; i < L; i += kThreads) {
        const uint32_t q = src.key(i);
        kmin = min(kmin, q);
        kmax = max(kmax, q);
      }
      kmin = warp_min(kmin);
      kmax = warp_max(kmax);
      __syncthreads();
      if (lane == 0) { S.wa[warp] = kmin; S.wb[warp] = kmax; }
      __syncthreads();
      if (warp == 0) {
        const uint32_t a = warp_min(S.wa[lane]), b = warp_max(S.wb[lane]);
        if (lane == 0) { S.s_lo = a; S.s_hi = b; S.s_need = (uint32_t)k; S.s_mode = 0; }
      }
      __syncthreads();
    }
    TOPK_MARK(3);
    refine<kSmem>(S, src, L, tid, lane, warp);
    TOPK_MARK(4);
    const uint32_t T = S.s_lo;
    const float Tf = key2f(T);

    int* orow = out_idx + (long long)row * out_ld;
    if (fast) {
      // ---- kept candidates join the above-mask: key > T, then the first ties in index order
      if (tid == 0) { S.s_gt_total = 0; S.s_cmin = 0; }      // reused: #cand > T, #ties
      __syncthreads();
      const int nc = (int)min(S.s_ncand, (uint32_t)kCandCap);
      uint32_t cgt = 0, ceq = 0;
      for (int c = tid; c < nc; c += kThreads) {
        const uint32_t key = S.cand[c];
        if (key > T) { const uint32_t i = S.cidx[c]; atomicOr(&mask[mword(i, vec4)], mbit(i, vec4)); ++cgt; }
        else if (key == T) ++ceq;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        cgt += __shfl_xor_sync(0xffffffffu, cgt, o);
        ceq += __shfl_xor_sync(0xffffffffu, ceq, o);
      }
      if (lane == 0 && (cgt | ceq)) { atomicAdd(&S.s_gt_total, cgt); atomicAdd(&S.s_cmin, ceq); }
      __syncthreads();
      const uint32_t need_eq = S.s_kband - S.s_gt_total;   // k - #above - #(cand > T)
      const uint32_t nties = S.s_cmin;
      for (int c = tid; c < nc; c += kThreads) {
        if (S.cand[c] != T) continue;
        const uint32_t i = S.cidx[c];
        uint32_t rank = 0;
        if (nties > need_eq)
          for (int c2 = 0; c2 < nc; ++c2) rank += (S.cand[c2] == T && S.cidx[c2] < i);
        if (rank < need_eq) atomicOr(&mask[mword(i, vec4)], mbit(i, vec4));
      }
      __syncthreads();
      TOPK_MARK(5);
      // ---- ordered emit from the keep-mask: block scan of per-thread popcounts
      //      (vec4 layout: one thread per 128-column chunk = 4 words)
      const int gw = vec4 ? 4 : 1;                      // words per unit
      const int nu = vec4 ? (L + 127) / 128 : nw;       // units
      const int upt = (nu + kThreads - 1) / kThreads;
      const int u0 = tid * upt, u1 = min(nu, u0 + upt);
      uint32_t cnt = 0;
      for (int u = u0; u < u1; ++u)
        for (int j = 0; j < gw; ++j) cnt += __popc(mask[u * gw + j]);
      uint32_t inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
      }
      if (lane == 31) S.wc[warp] = inc;
      __syncthreads();
      uint32_t wbase = 0;
      if (lane < warp) wbase = S.wc[lane];
#pragma unroll
      for (int o = 16; o; o >>= 1) wbase += __shfl_xor_sync(0xffffffffu, wbase, o);
      uint32_t pos = wbase + inc - cnt;
      for (int u = u0; u < u1; ++u) {
        if (vec4) {
          const uint32_t m0 = mask[4 * u], m1 = mask[4 * u + 1], m2 = mask[4 * u + 2], m3 = mask[4 * u + 3];
          uint32_t any = m0 | m1 | m2 | m3;
          while (any) {
            const int l = __ffs(any) - 1;
            any &= any - 1;
            const int c0 = u * 128 + 4 * l;
            if ((m0 >> l) & 1u) orow[pos++] = c0;
            if ((m1 >> l) & 1u) orow[pos++] = c0 + 1;
            if ((m2 >> l) & 1u) orow[pos++] = c0 + 2;
            if ((m3 >> l) & 1u) orow[pos++] = c0 + 3;
          }
        } else {
          uint32_t m = mask[u];
          while (m) {
            const int bit = __ffs(m) - 1;
            orow[pos++] = u * 32 + bit;
            m &= m - 1;
          }
        }
      }
    } else {
      // ---- slow path: per-warp (> T, == T) counts by a scan, then ordered compaction
      uint32_t ngt = 0, neq = 0;
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        const bool valid = i < s1;
        const float v = valid ? src.val(i) : 0.f;
        ngt += __popc(__ballot_sync(0xffffffffu, valid && v > Tf));
        neq += __popc(__ballot_sync(0xffffffffu, valid && v == Tf));
      }
      __syncthreads();
      if (lane == 0) { S.wa[warp] = ngt; S.wb[warp] = neq; }
      __syncthreads();
      if (warp == 0) {
        const uint32_t g = S.wa[lane], e = S.wb[lane];
        uint32_t gi = g, ei = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t1 = __shfl_up_sync(0xffffffffu, gi, o);
          const uint32_t t2 = __shfl_up_sync(0xffffffffu, ei, o);
          if (lane >= o) { gi += t1; ei += t2; }
        }
        const uint32_t gtot = __shfl_sync(0xffffffffu, gi, 31);
        const uint32_t need_eq = (uint32_t)k - gtot;
        const uint32_t gex = gi - g, eex = ei - e;
        S.wa[lane] = gex + min(eex, need_eq);  // kept entries before this warp
        S.wb[lane] = eex;                       // ties before this warp
        if (lane == 0) S.s_gt_total = gtot;
      }
      __syncthreads();
      const uint32_t need_eq = (uint32_t)k - S.s_gt_total;
      uint32_t kept = S.wa[warp];
      uint32_t eqs = S.wb[warp];
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        const bool valid = i < s1;
        const float v = valid ? src.val(i) : 0.f;
        const uint32_t mgt = __ballot_sync(0xffffffffu, valid && v > Tf);
        const uint32_t meq = __ballot_sync(0xffffffffu, valid && v == Tf);
        const bool keep_eq = ((meq >> lane) & 1u) && (eqs + __popc(meq & lt)) < need_eq;
        const uint32_t mkeep = mgt | __ballot_sync(0xffffffffu, keep_eq);
        if ((mkeep >> lane) & 1u) orow[kept + __popc(mkeep & lt)] = i;
        kept += __popc(mkeep);
        eqs += __popc(meq);
      }
    }
    if (tid == 0) out_thr[row] = Tf;
    TOPK_MARK(6);
    __syncthreads();   // buffers reused by the next row
    TOPK_MARK(7);
  }
}

}  // namespace topk
}  // namespace dsv

size_t dsv_topk_smem_bytes(int L) {
  const size_t mask = 2 * (((size_t)L + 127) / 128 * 4 + 4) * 4;   // keep + band masks
  const size_t base = sizeof(dsv::topk::Smem) + mask;
  const size_t need = base + (size_t)L * 4;
  return need <= 227 * 1024 ? need : base;
}

int dsv_topk_stream_launch(const float*, long long, int, int, const int*, int, int*, long long,
                           float*, cudaStream_t);

int dsv_topk_launch(const float* scores, long long ld, int rows, int L, const int* k_per_head,
                    int rows_per_head, int* out_idx, long long out_ld, float* out_thr,
                    cudaStream_t stream) {
  using namespace dsv::topk;
  if (rows <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = rows < sms ? rows : sms;
  const size_t mask = 2 * (((size_t)L + 127) / 128 * 4 + 4) * 4;   // keep + band masks
  const size_t base = sizeof(Smem) + mask;
  const size_t need = base + (size_t)L * 4;
  if (base > 227 * 1024) return (int)cudaErrorInvalidValue;
  if (need > 227 * 1024)   // the row does not fit in shared memory: streaming kernel
    return dsv_topk_stream_launch(scores, ld, rows, L, k_per_head, rows_per_head, out_idx, out_ld,
                                  out_thr, stream);
  cudaFuncSetAttribute(topk_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)need);
  topk_rows_kernel<true><<<grid, kThreads, need, stream>>>(
      scores, ld, rows, L, k_per_head, rows_per_head, out_idx, out_ld, out_thr);
  return (int)cudaGetLastError();
}
