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
// This file: rows too long for the shared-memory kernel (topk.cu), e.g. L = 131072
// (c3/c4) and 524288 (c5). Small CTAs (256 threads, several per SM, persistent over
// rows) stream each row twice from HBM/L2:
//   1. a 4096-entry strided sample gives a value band [lo, hi] expected to hold the
//      k-th value T (value-linear histogram, +- 4 sigma of the binomial sample count);
//   A. pass A (float4, four loads in flight): count entries > hi and histogram the
//      in-band entries by order key (1024 linear buckets) — shared atomics on ~5% of
//      the row, nothing stored; the bucket holding T narrows the band ~1000x;
//   B. pass B: entries above the narrowed band set their bit in a shared keep-mask
//      (plain bit order from per-lane nibbles), entries inside it (a handful) are
//      appended with ballots;
//   3. T is found exactly among those candidates, candidates > T join the mask and
//      the first ties in column order fill the remaining budget;
//   4. the mask is emitted in ascending column order (warp-coalesced).
// Rows where a band check fails take a whole-row key-space selection and an ordered
// two-pass compaction. HBM traffic per row: two reads + k * 4 bytes of indices.

#include "dsv_common.cuh"

#ifdef DSV_TOPKS_PROF
__device__ unsigned int g_topks_slow;
#endif

namespace dsv {
namespace topks {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMinBlocks = 4;                 // CTAs per SM the kernel is built for
constexpr int kBuckets = 1024;                // sample histogram
constexpr int kSample = 4096;
constexpr int kCandCap = 4096;
constexpr int kCandW = kCandCap / kWarps;     // per-warp candidate region

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
  uint32_t cand[kCandCap];        // candidate order keys
  uint32_t cidx[kCandCap];        // candidate columns
  uint32_t wsum[kWarps];
  uint32_t wcnt[kWarps];          // candidates per warp region
  uint32_t ncand, nabove;
  uint32_t b_hi, b_lo;
  uint32_t prefix, need, neq;     // radix-select state
};

// Value-space bucket: correctly rounded fma and saturating conversion keep it
// monotone non-decreasing in v.
DSV_DEV int vbucket(float v, float a, float b) {
  return min(max(__float2int_rz(__fmaf_rn(v, a, b)), 0), kBuckets - 1);
}

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix
// and the total through *total.
DSV_DEV uint32_t block_excl_scan(Smem& S, uint32_t v, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  __syncthreads();
  if (lane == 31) S.wsum[warp] = inc;
  __syncthreads();
  uint32_t base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t s = S.wsum[w];
    base += w < warp ? s : 0u;
    tot += s;
  }
  *total = tot;
  return base + inc - v;
}

// Key-space bucketing of [lo, lo + span): bucket(x) = ((x - lo) * M) >> 32 with
// M = floor(nb 2^32 / span) — monotone, < nb, exact (one key per bucket) when
// span <= nb, and a multiply instead of a 64-bit division per key.
struct KMap {
  uint32_t lo;
  uint64_t m;
  DSV_DEV uint32_t bucket(uint32_t key) const { return (uint32_t)(((uint64_t)(key - lo) * m) >> 32); }
  // offset (from lo) of the first key that maps to bucket b: ceil(b 2^32 / m)
  DSV_DEV uint64_t first(uint64_t b) const { return ((b << 32) + m - 1) / m; }
};
DSV_DEV uint32_t nbuckets(uint64_t span) {
  return span < (uint64_t)kBuckets ? (uint32_t)span : (uint32_t)kBuckets;
}
DSV_DEV KMap kmap(uint32_t lo, uint32_t hi) {
  const uint64_t span = (uint64_t)(hi - lo) + 1ull;
  return KMap{lo, ((uint64_t)nbuckets(span) << 32) / span};
}

// Exact selection in key space: the need-th largest key among the keys fed by
// `feed` (called with a per-key visitor), all of which lie in [lo, hi]. Each level
// histograms [lo, hi] linearly into <= kBuckets buckets (keys of a narrow value
// band spread evenly, so the shared-memory atomics rarely collide) and keeps the
// bucket holding the need-th key; a level whose buckets are single keys ends it.
// With `prefilled`, S.hist already holds the first level's histogram. Leaves
// S.prefix = T, S.need = how many keys equal to T are kept, S.neq = how many keys
// equal T in total.
template <typename Feed>
DSV_DEV void key_select(Smem& S, uint32_t need, uint32_t lo, uint32_t hi, bool prefilled, Feed feed) {
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int level = 0; level < 8; ++level) {
    const KMap km = kmap(lo, hi);
    if (level > 0 || !prefilled) {
      for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
      __syncthreads();
      feed([&](uint32_t key) {
        if (key >= lo && key <= hi) atomicAdd(&S.hist[km.bucket(key)], 1u);
      });
      __syncthreads();
    }
    // C(b) = keys in buckets >= b; thread owns buckets 4 tid .. 4 tid + 3
    uint32_t h[4], own = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) { h[i] = S.hist[4 * tid + i]; own += h[i]; }
    uint32_t total;
    const uint32_t before = block_excl_scan(S, own, &total);
    uint32_t c = total - before;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t cn = c - h[i];
      if (cn < need && need <= c) {
        const uint64_t bb = 4 * tid + i;
        S.prefix = lo + (uint32_t)km.first(bb);                                // new lo
        S.b_hi = lo + (uint32_t)min((unsigned long long)(km.first(bb + 1) - 1ull), (unsigned long long)(hi - lo));   // new hi
        S.need = need - cn;
        S.neq = h[i];
      }
      c = cn;
    }
    __syncthreads();
    lo = S.prefix;
    hi = S.b_hi;
    need = S.need;
    if (lo == hi) return;          // single key: S.prefix = T, S.neq = its count
  }
}

template <bool kVec>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
topk_rows_kernel(const float* __restrict__ scores, long long ld, int rows, int L,
                 const int* __restrict__ k_per_head, int rows_per_head,
                 int* __restrict__ out_idx, long long out_ld, float* __restrict__ out_thr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Smem));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = (L + 31) >> 5;                  // 32-column mask words
  const int n4 = kVec ? (L >> 2) : 0;            // full float4 chunks
  const uint32_t lt = (1u << lane) - 1u;

  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const int k = k_per_head[row / rows_per_head];
    const float* grow = scores + (long long)row * ld;
    int* orow = out_idx + (long long)row * out_ld;
    if (kVec && tid == 0 && row + (int)gridDim.x < rows)   // next row of this CTA into L2
      prefetch_l2(scores + (long long)(row + gridDim.x) * ld, (uint32_t)(n4 * 16));
    if (k >= L) {
      // keep everything; threshold = row minimum
      float mn = INFINITY;
      for (int i = tid; i < L; i += kThreads) { orow[i] = i; mn = fminf(mn, __ldg(grow + i)); }
#pragma unroll
      for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (lane == 0) S.wsum[warp] = __float_as_uint(mn);
      __syncthreads();
      if (tid == 0) {
        float m = INFINITY;
        for (int w = 0; w < kWarps; ++w) m = fminf(m, __uint_as_float(S.wsum[w]));
        out_thr[row] = m == 0.f ? 0.f : m;
      }
      __syncthreads();
      continue;
    }
    if (k <= 0) {
      if (tid == 0) out_thr[row] = INFINITY;
      continue;
    }

    // ---- 1. strided sample: range, histogram, band [b_lo, b_hi]
    float sv[kSample / kThreads];
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kSample / kThreads; ++j) {
      const int i = (int)(((long long)(tid + j * kThreads) * L) / kSample);
      sv[j] = __ldg(grow + min(i, L - 1));
      mn = fminf(mn, sv[j]);
      mx = fmaxf(mx, sv[j]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
    for (int w = tid; w < nw; w += kThreads) mask[w] = 0;
    if (tid == 0) { S.ncand = 0; S.nabove = 0; }
    __syncthreads();
    if (lane == 0) S.wsum[warp] = __float_as_uint(mn);
    __syncthreads();
    float bmn = INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) bmn = fminf(bmn, __uint_as_float(S.wsum[w]));
    __syncthreads();
    if (lane == 0) S.wsum[warp] = __float_as_uint(mx);
    __syncthreads();
    float bmx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) bmx = fmaxf(bmx, __uint_as_float(S.wsum[w]));
    bool fast = isfinite(bmn) && isfinite(bmx) && bmx > bmn;
    float hi_v = INFINITY, lo_v = -INFINITY;
    if (fast) {
      const float ba = (float)kBuckets / (bmx - bmn), bb = -bmn * ba;
#pragma unroll
      for (int j = 0; j < kSample / kThreads; ++j) atomicAdd(&S.hist[vbucket(sv[j], ba, bb)], 1u);
      __syncthreads();
      // suffix counts C(b) = samples in buckets >= b; thread owns buckets 4t..4t+3
      const float t = (float)k * (float)kSample / (float)L;
      const float m = 4.f * sqrtf(fmaxf(t * (1.f - t / kSample), 1.f)) + 2.f;
      const float tm = t - m, tp = t + m;
      uint32_t h[4], own = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) { h[i] = S.hist[4 * tid + i]; own += h[i]; }
      uint32_t total;
      const uint32_t before = block_excl_scan(S, own, &total);   // buckets < 4 tid
      // C(4t + i) = total - before - sum(h[0..i-1])
      if (tid == 0) { S.b_hi = kBuckets - 1; S.b_lo = 0; }
      __syncthreads();
      float c = (float)(total - before);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float cn = c - (float)h[i];   // C(b + 1)
        const uint32_t b = 4 * tid + i;
        if (tm > 0.f && cn <= tm && c > tm) S.b_hi = b;
        if (tp < (float)kSample && c >= tp && cn < tp) S.b_lo = b;
        c = cn;
      }
      __syncthreads();
      const int b_hi = (int)S.b_hi, b_lo = min((int)S.b_lo, b_hi);
      hi_v = b_hi >= kBuckets - 1 ? INFINITY : bmn + (float)(b_hi + 1) / ba;
      lo_v = b_lo <= 0 ? -INFINITY : bmn + (float)b_lo / ba;
    }
    __syncthreads();
    for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;   // first selection level
    __syncthreads();

    uint32_t T = 0;
    uint32_t kneed = (uint32_t)k;                 // rank of T among band-B entries
    if (fast) {
      // ---- A. count entries > hi, histogram the band by order key (no stores)
      const uint32_t kloA = f2key(lo_v), khiA = f2key(hi_v);
      const KMap kmA = kmap(kloA, khiA);
      uint32_t nab = 0;
      if constexpr (kVec) {
        constexpr int kU = 4;
        const float4* g4 = reinterpret_cast<const float4*>(grow);
        const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        for (int qb = tid; qb < n4; qb += kU * kThreads) {
          float4 vb[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int q = qb + u * kThreads;
            vb[u] = q < n4 ? __ldg(g4 + q) : ninf;
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const float vv[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (vv[e] > hi_v) ++nab;
              else if (vv[e] >= lo_v) atomicAdd(&S.hist[kmA.bucket(f2key(vv[e]))], 1u);
            }
          }
        }
      }
      for (int i = 4 * n4 + tid; i < L; i += kThreads) {
        const float v = __ldg(grow + i);
        if (v > hi_v) ++nab;
        else if (v >= lo_v) atomicAdd(&S.hist[kmA.bucket(f2key(v))], 1u);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) nab += __shfl_xor_sync(0xffffffffu, nab, o);
      if (lane == 0) atomicAdd(&S.nabove, nab);
      __syncthreads();
      // the bucket holding the (k - #above)-th largest band entry -> band B
      const uint32_t nA = S.nabove;
      {
        uint32_t h[4], own = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) { h[i] = S.hist[4 * tid + i]; own += h[i]; }
        uint32_t total;
        const uint32_t before = block_excl_scan(S, own, &total);
        fast = nA < (uint32_t)k && (uint32_t)k <= nA + total;
        const uint32_t need = (uint32_t)k - nA;
        uint32_t c = total - before;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t cn = c - h[i];
          if (fast && cn < need && need <= c) {
            const uint64_t bb = 4 * tid + i;
            S.prefix = kloA + (uint32_t)kmA.first(bb);
            S.b_hi = kloA + (uint32_t)min((unsigned long long)(kmA.first(bb + 1) - 1ull),
                                          (unsigned long long)(khiA - kloA));
            S.need = need - cn;
          }
          c = cn;
        }
        __syncthreads();
      }
      if (fast) {
        lo_v = key2f(S.prefix);
        hi_v = key2f(S.b_hi);
        kneed = S.need;
      }
      __syncthreads();
      for (int b = tid; b < kBuckets; b += kThreads) S.hist[b] = 0;
      if (tid == 0) S.nabove = 0;
      __syncthreads();
    }
    if (fast) {
      // ---- B. above-mask bits (plain order: word (4 q0)/32 + m holds lanes 8m..8m+7
      //      of a warp's 128-column chunk, 4 bits each) and band-B candidates, appended
      //      with ballots and histogrammed for the first key-selection level on the way
      const uint32_t klo = f2key(lo_v), khi = f2key(hi_v);
      const KMap km0 = kmap(klo, khi);
      uint32_t nab = 0, wc = 0;                  // wc: this warp's candidates (uniform)
      uint32_t* wcand = S.cand + warp * kCandW;
      uint32_t* wcidx = S.cidx + warp * kCandW;
      auto put = [&](uint32_t slot, float v, int i) {
        const uint32_t key = f2key(v);
        if (slot < (uint32_t)kCandW) { wcand[slot] = key; wcidx[slot] = (uint32_t)i; }
        atomicAdd(&S.hist[km0.bucket(key)], 1u);
      };
      if constexpr (kVec) {
        // kU float4 loads per lane in flight before any is consumed
        constexpr int kU = 4;
        const float4* g4 = reinterpret_cast<const float4*>(grow);
        const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        for (int qb = warp * 32; qb < n4; qb += kU * kThreads) {
          float4 vb[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int q = qb + u * kThreads + lane;
            vb[u] = q < n4 ? __ldcs(g4 + q) : ninf;
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int q0 = qb + u * kThreads, q = q0 + lane;
            if (q0 >= n4) break;
            const float4 v = vb[u];
            const bool g0 = v.x > hi_v, g1 = v.y > hi_v, g2 = v.z > hi_v, g3 = v.w > hi_v;
            const uint32_t gt = (uint32_t)g0 | ((uint32_t)g1 << 1) | ((uint32_t)g2 << 2) | ((uint32_t)g3 << 3);
            nab += __popc(gt);
            uint32_t wv = gt << (4 * (lane & 7));
            wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
            wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
            wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
            if ((lane & 7) == 0 && q < n4) mask[(q0 >> 3) + (lane >> 3)] = wv;
            const bool i0 = !g0 && v.x >= lo_v, i1 = !g1 && v.y >= lo_v;
            const bool i2 = !g2 && v.z >= lo_v, i3 = !g3 && v.w >= lo_v;
            const uint32_t b0 = __ballot_sync(0xffffffffu, i0), b1 = __ballot_sync(0xffffffffu, i1);
            const uint32_t b2 = __ballot_sync(0xffffffffu, i2), b3 = __ballot_sync(0xffffffffu, i3);
            const uint32_t c0 = __popc(b0), c01 = c0 + __popc(b1), c012 = c01 + __popc(b2);
            const uint32_t wtot = c012 + __popc(b3);
            if (i0) put(wc + __popc(b0 & lt), v.x, 4 * q);
            if (i1) put(wc + c0 + __popc(b1 & lt), v.y, 4 * q + 1);
            if (i2) put(wc + c01 + __popc(b2 & lt), v.z, 4 * q + 2);
            if (i3) put(wc + c012 + __popc(b3 & lt), v.w, 4 * q + 3);
            wc += wtot;
          }
        }
      }
      __syncthreads();   // plain mask-word stores above before the tail's atomicOr
      // scalar part: the tail (or the whole row without 16-byte alignment)
      for (int i0 = 4 * n4 + warp * 32; i0 < L; i0 += kThreads) {
        const int i = i0 + lane;
        const float v = i < L ? __ldcs(grow + i) : -INFINITY;
        const bool g = v > hi_v, in = !g && v >= lo_v && i < L;
        if (g) { atomicOr(&mask[i >> 5], 1u << (i & 31)); ++nab; }
        const uint32_t bi = __ballot_sync(0xffffffffu, in);
        if (in) put(wc + __popc(bi & lt), v, i);
        wc += __popc(bi);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) nab += __shfl_xor_sync(0xffffffffu, nab, o);
      if (lane == 0) { atomicAdd(&S.nabove, nab); S.wcnt[warp] = wc; }
      __syncthreads();
      const uint32_t nabove = S.nabove;
      uint32_t nc = 0, wmax = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) { nc += S.wcnt[w]; wmax = max(wmax, S.wcnt[w]); }
      fast = wmax <= (uint32_t)kCandW && nabove < (uint32_t)k && (uint32_t)k <= nabove + nc;
      (void)kneed;
      if (fast) {
        // ---- 3. exact T among the candidates
        // candidate slot c lives in warp region c / kCandW, valid below that warp's count
        auto valid = [&](int c) { return (uint32_t)(c % kCandW) < S.wcnt[c / kCandW]; };
        key_select(S, (uint32_t)k - nabove, klo, khi, true, [&](auto visit) {
          for (int c = tid; c < kCandCap; c += kThreads)
            if (valid(c)) visit(S.cand[c]);
        });
        T = S.prefix;
        const uint32_t keep_eq = S.need, n_eq = S.neq;
        for (int c = tid; c < kCandCap; c += kThreads) {
          if (!valid(c)) continue;
          const uint32_t key = S.cand[c];
          bool keep = key > T;
          if (key == T) {
            if (n_eq <= keep_eq) {
              keep = true;
            } else {
              const uint32_t i = S.cidx[c];
              uint32_t rank = 0;
              for (int c2 = 0; c2 < kCandCap; ++c2)
                rank += (valid(c2) && S.cand[c2] == T && S.cidx[c2] < i);
              keep = rank < keep_eq;
            }
          }
          if (keep) { const uint32_t i = S.cidx[c]; atomicOr(&mask[i >> 5], 1u << (i & 31)); }
        }
        __syncthreads();
        // ---- 4. ordered emit: warp w owns a contiguous range of mask words, lane j
        //      the j-th word of each 32-word group (warp scan of the popcounts)
        const int wpw = (nw + kWarps - 1) / kWarps;
        const int a0 = min(nw, warp * wpw), a1 = min(nw, a0 + wpw);
        uint32_t wcnt = 0;
        for (int w = a0 + lane; w < a1; w += 32) wcnt += __popc(mask[w]);
#pragma unroll
        for (int o = 16; o; o >>= 1) wcnt += __shfl_xor_sync(0xffffffffu, wcnt, o);
        uint32_t tot;
        uint32_t base = block_excl_scan(S, lane == 0 ? wcnt : 0u, &tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int g0 = a0; g0 < a1; g0 += 32) {
          const int w = g0 + lane;
          uint32_t m = w < a1 ? mask[w] : 0u;
          const uint32_t c = __popc(m);
          uint32_t inc = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += x;
          }
          uint32_t pos = base + inc - c;
          while (m) {
            orow[pos++] = w * 32 + __ffs(m) - 1;
            m &= m - 1;
          }
          base += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
    }
    if (!fast) {
#ifdef DSV_TOPKS_PROF
      if (tid == 0) atomicAdd(&g_topks_slow, 1u);
#endif
      // ---- slow path: whole-row radix select, then ordered two-pass compaction over
      //      contiguous warp segments
      uint32_t kmn = 0xffffffffu, kmx = 0u;
      for (int i = tid; i < L; i += kThreads) {
        const uint32_t key = f2key(__ldg(grow + i));
        kmn = min(kmn, key);
        kmx = max(kmx, key);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
        kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
      }
      __syncthreads();
      if (tid == 0) { S.b_lo = 0xffffffffu; S.b_hi = 0u; }
      __syncthreads();
      if (lane == 0) { atomicMin(&S.b_lo, kmn); atomicMax(&S.b_hi, kmx); }
      __syncthreads();
      key_select(S, (uint32_t)k, S.b_lo, S.b_hi, false, [&](auto visit) {
        for (int i = tid; i < L; i += kThreads) visit(f2key(__ldg(grow + i)));
      });
      T = S.prefix;
      const uint32_t keep_eq = S.need;
      const int seg = (((L + kWarps - 1) / kWarps) + 31) & ~31;
      const int s0 = warp * seg, s1 = min(L, s0 + seg);
      uint32_t ngt = 0, neq = 0;
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < s1 ? f2key(__ldg(grow + i)) : 0u;
        ngt += __popc(__ballot_sync(0xffffffffu, i < s1 && key > T));
        neq += __popc(__ballot_sync(0xffffffffu, i < s1 && key == T));
      }
      // exclusive prefixes over warps of (gt, eq)
      uint32_t tot_gt, tot_eq;
      const uint32_t gbase = block_excl_scan(S, lane == 0 ? ngt : 0u, &tot_gt);
      const uint32_t ebase = block_excl_scan(S, lane == 0 ? neq : 0u, &tot_eq);
      uint32_t gb = __shfl_sync(0xffffffffu, gbase, 0), eb = __shfl_sync(0xffffffffu, ebase, 0);
      uint32_t kept = gb + min(eb, keep_eq);
      uint32_t eqs = eb;
      for (int base = s0; base < s1; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < s1 ? f2key(__ldg(grow + i)) : 0u;
        const uint32_t mgt = __ballot_sync(0xffffffffu, i < s1 && key > T);
        const uint32_t meq = __ballot_sync(0xffffffffu, i < s1 && key == T);
        const bool keq = ((meq >> lane) & 1u) && (eqs + __popc(meq & lt)) < keep_eq;
        const uint32_t mkeep = mgt | __ballot_sync(0xffffffffu, keq);
        if ((mkeep >> lane) & 1u) orow[kept + __popc(mkeep & lt)] = i;
        kept += __popc(mkeep);
        eqs += __popc(meq);
      }
    }
    if (tid == 0) out_thr[row] = key2f(T);
    __syncthreads();   // shared state reused by the next row
  }
}

}  // namespace topks
}  // namespace dsv

size_t dsv_topk_stream_smem_bytes(int L) {
  return sizeof(dsv::topks::Smem) + (((size_t)L + 31) / 32) * 4;   // keep-mask
}

int dsv_topk_stream_launch(const float* scores, long long ld, int rows, int L,
                           const int* k_per_head, int rows_per_head, int* out_idx,
                           long long out_ld, float* out_thr, cudaStream_t stream) {
  using namespace dsv::topks;
  if (rows <= 0) return 0;
  const size_t smem = dsv_topk_stream_smem_bytes(L);
  if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = ((ld * 4) % 16 == 0) && ((reinterpret_cast<uintptr_t>(scores) & 15) == 0);
  auto kern = vec ? topk_rows_kernel<true> : topk_rows_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  per_sm = per_sm < 1 ? 1 : per_sm;
  const long long want = (long long)sms * per_sm;
  const int grid = (int)(rows < want ? rows : want);
  kern<<<grid, kThreads, smem, stream>>>(scores, ld, rows, L, k_per_head, rows_per_head, out_idx,
                                         out_ld, out_thr);
  return (int)cudaGetLastError();
}
