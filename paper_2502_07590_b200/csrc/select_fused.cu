// select_fused.cu — K1b + K2 fused: proxy scores recomputed on tcgen05, exact top-k per
// row, no [H, G, L] fp32 score matrix in HBM.
//
// Semantics: those of K2 (topk.cu; reference pkg/src/dynsparse/selection.py:82-115
// `_merge_block`, :166-174 emit, :178-242 `twopass_select`) applied to the scores of K1b
// (reference selection.py:149, Q_lr[proxies] . K_lr^T per head). The score of (row, key)
// is one tcgen05 kind::f16 M=128 N=128 K=16 MMA on the same bf16 operands as the unfused
// K1b GEMM (gemm_tc.cu), whose first MMA of the k-block is this instruction and whose
// other three add products of the zero padding (exact zeros); the values are identical —
// at most the sign of an exactly-zero score differs, which the selection does not see
// (-0.0 == +0.0) — so the fused selection equals the unfused one bit for bit.
//
// Why: the unfused path writes H G L fp32 scores and K2 reads them twice (c2: 0.8 GB
// written + 1.6 GB read; c5: 206 GB + 412 GB). Here the scores are recomputed per pass —
// one MMA per 128 x 128 tile (r <= 16) from TMA-fed shared memory (32B-swizzled 4 KB
// tiles, 16 in flight), B (K_lr) tiles L2
// resident — and each pass touches only TMEM, registers and shared memory.
//
// CTA = one 128-row tile of one head's proxy rows x a contiguous key range; a cluster
// of S CTAs splits the key range of one row tile (S = 1..6, the fewest waves of resident
// clusters per unit of per-CTA work; per-pass partials are combined through distributed
// shared memory). Warp 0: TMA
// producer (B ring), warp 1: MMA issuer (4 TMEM accumulators x 128 columns), warps 2..:
// epilogue, each TMEM lane quadrant covered by kEpiWarps/4 warps that split a tile's
// 128 columns. Per row, passes over the key range (all rows advance together):
//   MINMAX / SHIST (a 16-tile strided sample): value-linear 128-bucket histogram of the
//       sample -> a key band [klo, khi] expected to hold the k-th value T;
//   FULL (repeat): count keys > khi and histogram the band key-linearly (128 buckets),
//       or, once the bucket holding T has <= kCap entries, collect them; T is exact when
//       the bucket is one key value or after the candidate pass;
//   EMIT: bit masks (s > T) and (s == T) per 32 columns staged in shared memory, then a
//       warp per row emits ascending column indices, ties at T in column order up to the
//       row's quota (ties resolve toward lower indices), coalesced per row.
// Single-pass mode (a workspace is given; the default): after the sample passes, ONE
// COLLECT pass writes per row a bitmap of the keys at or above the band and stashes the
// band entries (column, order key); select_finish_kernel (a CTA per row) finds T among
// the band by radix select and emits from the bitmap; row tiles whose band missed T are
// re-run with the passes above (list mode).
// Scores are compared as floats: with the order key f2key (-0.0 == +0.0, monotone) every
// band edge is converted to the float with that key (the one key without a float, the
// image of -0.0, is handled explicitly). Columns past L are NaN (no comparison holds).

#include <cuda.h>
#include <stdint.h>
#include "dsv_common.cuh"

__device__ unsigned long long g_fsel_prof[64][8];
#ifdef DSV_FSEL_PROF
#define FPROF_AT(p, e) do { if (blockIdx.x == 0 && (p) < 64) g_fsel_prof[(p)][(e)] = dsv::globaltimer_ns(); } while (0)
#else
#define FPROF_AT(p, e) do { } while (0)
#endif

namespace dsv {
namespace fsel {

constexpr int BM = 128, BN = 128, BK = 16;   // one K=16 MMA per tile (rank r <= 16)
constexpr int kStages = 8;                    // B (K_lr) tiles in flight (4 KB each)
constexpr int kScratch = 36;                  // words per epilogue thread: one 32-column chunk (padded)
constexpr int kAcc = 4;                       // TMEM accumulators (4 x 128 columns)
#ifndef DSV_FSEL_EPI_WARPS
#define DSV_FSEL_EPI_WARPS 16
#endif
constexpr int kEpiWarps = DSV_FSEL_EPI_WARPS;
constexpr int kParts = kEpiWarps / 4;         // threads per row
constexpr int kCols = BN / kParts;            // columns per thread per tile
static_assert(kEpiWarps == 4 || kEpiWarps == 8 || kEpiWarps == 16,
              "epilogue warps: 1, 2 or 4 per TMEM lane quadrant (32-column multiples, part_above)");
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int kBuckets = 128;
// histogram row stride (words): padded so that lanes = rows hitting the same bucket index
// land in different shared-memory banks
constexpr int kHistStride = kBuckets + 1;
constexpr int kCap = 128;                     // candidates per row (cluster-wide) = bucket words
constexpr int kSampleTiles = 48;
constexpr int kFlushTiles = 8;                // tiles per emission flush (1024 columns)
constexpr int kStageStride = kFlushTiles * 8 + 1;   // words per row (padded)
constexpr uint32_t KEY_LO = 0x007FFFFFu;      // key of -inf
constexpr uint32_t KEY_HI = 0xFF800000u;      // key of +inf
constexpr uint32_t KEY_NEG0 = 0x7FFFFFFFu;    // the key no float maps to (-0.0 -> +0.0)

#ifndef DSV_FSEL_SLEEP
#define DSV_FSEL_SLEEP 0
#endif
#if DSV_FSEL_SLEEP
#define FSEL_WAIT mbar_wait_sleep
#else
#define FSEL_WAIT mbar_wait
#endif

enum : uint32_t { ST_REFINE = 0, ST_CAND = 1, ST_DONE = 2 };
enum : uint32_t { P_MINMAX = 0, P_SHIST = 1, P_FULL = 2, P_EMIT = 3, P_EXIT = 4, P_COLLECT = 5 };
// launch modes: exact multi-pass (classic), single collect pass + select_finish_kernel (fast),
// classic restricted to the row tiles the finish kernel flagged (list)
enum : int { M_CLASSIC = 0, M_FAST = 1, M_LIST = 2 };

struct SL {
  static constexpr int kA = 0;
  static constexpr int kB = kA + BM * BK * 2;
  static constexpr int kU = kB + kStages * BN * BK * 2;              // hist / candidates
  static constexpr int kStage = kU + ((BM * kHistStride * 4 + 15) / 16) * 16;  // emission masks
  static constexpr int kRows = kStage + ((BM * kStageStride * 4 + 15) / 16) * 16;
  static constexpr int kRowArrays = 20;                              // see Rows
  static constexpr int kScr = kRows + kRowArrays * BM * 4;          // band-element scratch
  static constexpr int kBar = kScr + kEpiThreads * kScratch * 4;
  static constexpr int kBytes = kBar + 512 + 1024;
};

struct Bars {
  uint64_t full[kStages], empty[kStages], acc_full[kAcc], acc_empty[kAcc], a_full;
  uint32_t tmem;
  uint32_t pass, ntiles, flag, nfull;
};

// per-row state, structure of arrays (BM entries each)
struct Rows {
  uint32_t* k; uint32_t* klo; uint32_t* khi; uint32_t* above; uint32_t* state;
  uint32_t* T; uint32_t* pos; uint32_t* quota; uint32_t* taken; uint32_t* ncand;
  float* smin; float* smax;
  uint32_t* cta_above;             // this CTA's count > khi (sum over parts)
  float* cta_min; float* cta_max;
  uint32_t* part_above;            // [kParts][BM] (kParts <= 4)
};

DSV_DEV Rows rows_of(uint8_t* base) {
  uint32_t* u = reinterpret_cast<uint32_t*>(base);
  Rows r;
  r.k = u; r.klo = u + BM; r.khi = u + 2 * BM; r.above = u + 3 * BM; r.state = u + 4 * BM;
  r.T = u + 5 * BM; r.pos = u + 6 * BM; r.quota = u + 7 * BM; r.taken = u + 8 * BM;
  r.ncand = u + 9 * BM;
  r.smin = reinterpret_cast<float*>(u + 10 * BM); r.smax = reinterpret_cast<float*>(u + 11 * BM);
  r.cta_above = u + 12 * BM;
  r.cta_min = reinterpret_cast<float*>(u + 13 * BM); r.cta_max = reinterpret_cast<float*>(u + 14 * BM);
  r.part_above = u + 15 * BM;      // 4 x BM
  return r;
}

DSV_DEV uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
DSV_DEV float key2f(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
// float h with (s > h) <=> key(s) > k, for every non-NaN s
DSV_DEV float upper_f(uint32_t k) { return k == KEY_NEG0 ? __uint_as_float(0x80000001u) : key2f(k); }

// K-major operand, 32-byte rows (16 bf16 along K), 32B-swizzled (TMA SWIZZLE_32B), 8-row
// groups 256 B apart
DSV_DEV uint64_t sdesc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (Blackwell)
  d |= (uint64_t)6 << 61;                 // SWIZZLE_32B
  return d;
}

// ------------------------------------------------------------------ cluster helpers
DSV_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DSV_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
DSV_DEV uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
DSV_DEV uint32_t ld_dsmem(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
DSV_DEV uint32_t ld_shared_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
// a partial of cluster rank `rank` (read after a cluster barrier, which orders it): the own
// CTA's through a plain shared-memory load, a peer's through DSMEM
DSV_DEV uint32_t ld_peer(const uint32_t* p, uint32_t rank, uint32_t me) {
  return rank == me ? ld_shared_u32(p) : ld_dsmem(dsmem_addr(p, rank));
}

// key range of cluster rank s: tiles [s nt / S, (s + 1) nt / S)
DSV_DEV int range_lo(int nt, int S, int s) { return (int)(((long long)nt * s) / S); }
// i-th sample tile of a range [t0, t1)
// 1/8 of the range, at least 8 and at most kSampleTiles tiles
// (a twice denser sample in the single-pass mode shrank the band 27% but its histogram pass,
// ~2 us per tile on shared-memory atomics, cost more than the band saved: 0.483 vs 0.463 ms)
__host__ __device__ __forceinline__ int sample_count(int n, int mode = 0) {
  const int div = 8;
  (void)mode;
  const int a = n / div < kSampleTiles ? n / div : kSampleTiles;
  const int b = a > 8 ? a : 8;
  return n < b ? n : b;
}
DSV_DEV int sample_tile(int t0, int n, int ns, int i) { return t0 + (int)(((long long)i * n) / ns); }

// tile processed at step i of the current pass
DSV_DEV int pass_tile(uint32_t pass, int t0, int n, int i, int mode) {
  if (pass == P_MINMAX || pass == P_SHIST) return sample_tile(t0, n, sample_count(n, mode), i);
  return t0 + i;
}

template <int N>
DSV_DEV void tmem_ld_cols(uint32_t taddr, uint32_t (&v)[N]) {
  static_assert(N % 32 == 0, "columns per thread must be a multiple of 32");
#pragma unroll
  for (int c = 0; c < N / 32; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[c * 32 + i] = r[i];
  }
}

// ------------------------------------------------------------------ pass finalize
// One warp per row, after the pass's partials are complete cluster-wide. Lane l owns
// histogram buckets 4l .. 4l+3 (summed over the cluster's CTAs); "cum(b)" = entries in
// buckets >= b.
DSV_DEV uint32_t warp_sum(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// inclusive suffix sum over lanes (lane l: sum of lanes l..31)
DSV_DEV uint32_t warp_suffix(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v += y;
  }
  return v;
}

// Sample-rank band of the SHIST pass around the k-th value's expected rank tgt = k ns / L
// (the same for every row of a CTA: one head, one k): half-width 4 sigma (+4) when a miss
// only costs another FULL pass; 5.5 sigma (+8) for the single collect pass, where a miss
// re-runs the tile. Computed once per CTA and pass (double divisions and a square root).
struct SampleBand { double hi_rank, lo_rank; };
DSV_DEV SampleBand sample_band(uint32_t k, uint32_t ns, int L, int mode) {
  const double tgt = (double)k * ns / L;
  const double sig = sqrt(fmax(tgt * (1.0 - tgt / ns), 0.0));
  const double marg = mode == M_FAST ? 5.5 * sig + 8.0 : 4.0 * sig + 4.0;
  return {tgt - marg, tgt + marg};
}

DSV_DEV void finalize_row(Rows& R, uint32_t* U, int r, int lane, uint32_t pass, uint32_t S,
                          uint32_t me, SampleBand band, int L, int mode) {
  const uint32_t st = R.state[r];
  if (pass == P_MINMAX) {
    // lane s reads CTA s's partials (the cluster's loads in flight together)
    float a = __int_as_float(0x7f800000), b = __int_as_float(0xff800000);
    if ((uint32_t)lane < S) {
      a = __uint_as_float(ld_peer(reinterpret_cast<uint32_t*>(R.cta_min) + r, lane, me));
      b = __uint_as_float(ld_peer(reinterpret_cast<uint32_t*>(R.cta_max) + r, lane, me));
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {          // S <= 8
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      R.smin[r] = a;
      R.smax[r] = b;
    }
    return;
  }
  if (st == ST_DONE) return;
  const uint32_t* hrow = U + r * kHistStride + 4 * lane;
  uint32_t c[4] = {0u, 0u, 0u, 0u};
  if (pass == P_SHIST || st == ST_REFINE) {
    // all of a group of four CTAs' loads issued before any add: each add would otherwise
    // hold the next DSMEM load behind a full round trip
    for (uint32_t s0 = 0; s0 < S; s0 += 4) {
      uint32_t v[4][4];
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[s][q] = s0 + s < S ? ld_peer(hrow + q, s0 + s, me) : 0u;
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] += v[s][q];
    }
  }
  const uint32_t lsum = c[0] + c[1] + c[2] + c[3];
  const uint32_t excl = warp_suffix(lsum, lane) - lsum;     // entries in higher lanes' buckets
  if (pass == P_SHIST) {
    const float lo = R.smin[r], hi = R.smax[r];
    const double hi_rank = band.hi_rank, lo_rank = band.lo_rank;
    // highest bucket with cum > hi_rank / cum >= lo_rank
    int bh = -1, bl = -1;
    uint32_t cum = excl;
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      cum += c[q];
      if (bh < 0 && cum > hi_rank) bh = 4 * lane + q;
      if (bl < 0 && cum >= lo_rank) bl = 4 * lane + q;
    }
    int b_hi = bh, b_lo = bl;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      b_hi = max(b_hi, __shfl_xor_sync(0xffffffffu, b_hi, o));
      b_lo = max(b_lo, __shfl_xor_sync(0xffffffffu, b_lo, o));
    }
    if (lane == 0) {
      uint32_t klo = KEY_LO, khi = KEY_HI;
      if (hi > lo) {
        const float va = (float)kBuckets / (hi - lo);
        if (b_hi >= 0 && b_hi < kBuckets - 1) khi = f2key(lo + (float)(b_hi + 1) / va);
        if (b_lo > 0) klo = f2key(lo + (float)b_lo / va);
        if (klo > khi) { klo = KEY_LO; khi = KEY_HI; }
        klo = max(klo, KEY_LO);
        khi = min(khi, KEY_HI);
      } else if (hi == lo) {
        klo = khi = f2key(lo);
      }
      R.klo[r] = klo;
      R.khi[r] = khi;
    }
    return;
  }
  // ---- P_FULL
  const uint32_t k = R.k[r];
  uint32_t above = 0;
  for (uint32_t s = 0; s < S; ++s) above += ld_peer(R.cta_above + r, s, me);
  const uint32_t klo = R.klo[r], khi = R.khi[r];
  if (st == ST_REFINE) {
    const uint32_t band = __shfl_sync(0xffffffffu, excl + lsum, 0);
    if (above >= k) {                                   // T above the band
      if (lane == 0) { R.klo[r] = khi + 1; R.khi[r] = KEY_HI; }
      return;
    }
    if (above + band < k) {                             // T below the band
      if (lane == 0) { R.khi[r] = klo - 1; R.klo[r] = KEY_LO; }
      return;
    }
    // the bucket holding T: entries above it < k <= entries above it + its count
    int pick = -1;
    uint32_t pick_above = 0, pick_cnt = 0;
    uint32_t cum = above + excl;
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      if (pick < 0 && c[q] > 0 && cum < k && cum + c[q] >= k) { pick = 4 * lane + q; pick_above = cum; pick_cnt = c[q]; }
      cum += c[q];
    }
    const uint32_t who = __ballot_sync(0xffffffffu, pick >= 0);
    const int src = __ffs(who) - 1;
    pick = __shfl_sync(0xffffffffu, pick, src);
    pick_above = __shfl_sync(0xffffffffu, pick_above, src);
    pick_cnt = __shfl_sync(0xffffffffu, pick_cnt, src);
    const uint64_t span = (uint64_t)(khi - klo) + 1ull;
    const uint64_t nb = span < (uint64_t)kBuckets ? span : (uint64_t)kBuckets;
    const uint64_t mult = (nb << 32) / span;
    const uint64_t bb = (uint64_t)pick;
    const uint64_t f0 = ((bb << 32) + mult - 1) / mult;
    const uint64_t f1 = (((bb + 1) << 32) + mult - 1) / mult;
    const uint32_t nlo = klo + (uint32_t)f0;
    const uint64_t top = f1 - 1 < (uint64_t)(khi - klo) ? f1 - 1 : (uint64_t)(khi - klo);
    const uint32_t nhi = klo + (uint32_t)top;
    uint32_t nst = ST_REFINE;
    if (nlo == nhi) {
      // T is this single key: per-CTA counts > T (its count above the old band top plus
      // its entries in buckets above `pick`) and == T (its entries in `pick`)
      const uint32_t need = k - pick_above;
      uint32_t pos = 0, eq_before = 0, my_quota = 0;
      for (uint32_t s = 0; s <= me; ++s) {
        uint32_t part = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (4 * lane + q > pick) part += ld_peer(hrow + q, s, me);
        const uint32_t gt = warp_sum(part) + ld_peer(R.cta_above + r, s, me);
        const uint32_t eq = ld_peer(U + r * kHistStride + pick, s, me);
        const uint32_t qv = eq_before >= need ? 0u : min(eq, need - eq_before);
        if (s < me) pos += gt + qv; else my_quota = qv;
        eq_before += eq;
      }
      nst = ST_DONE;
      if (lane == 0) { R.T[r] = nlo; R.pos[r] = pos; R.quota[r] = my_quota; }
    } else if (pick_cnt <= (uint32_t)kCap) {
      nst = ST_CAND;
    }
    if (lane == 0) { R.klo[r] = nlo; R.khi[r] = nhi; R.state[r] = nst; }
    return;
  }
  // ---- ST_CAND: T = the (k - above)-th largest of the band's candidates (all CTAs)
  // lane holds candidates lane + 32 q of the concatenated per-CTA lists
  uint32_t cv[4], cs[4];
  uint32_t n = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) { cv[q] = 0u; cs[q] = 0xffffffffu; }
  for (uint32_t s = 0; s < S; ++s) {
    const uint32_t ns = min(ld_peer(R.ncand + r, s, me), (uint32_t)kCap);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = (uint32_t)(lane + 32 * q);
      if (i >= n && i < n + ns && i < (uint32_t)kCap) { cv[q] = ld_peer(U + r * kHistStride + (i - n), s, me); cs[q] = s; }
    }
    n += ns;
  }
  if (n > (uint32_t)kCap) n = kCap;
  const uint32_t m = k - above;                         // rank of T among the candidates
  uint32_t gt[4] = {0u, 0u, 0u, 0u}, eq[4] = {0u, 0u, 0u, 0u};
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t y = __shfl_sync(0xffffffffu, cv[j >> 5], j & 31);
#pragma unroll
    for (int q = 0; q < 4; ++q) { gt[q] += y > cv[q]; eq[q] += y == cv[q]; }
  }
  uint32_t T = 0;
  bool mine = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i = (uint32_t)(lane + 32 * q);
    if (i < n && gt[q] < m && m <= gt[q] + eq[q]) { T = cv[q]; mine = true; }
  }
  const uint32_t who = __ballot_sync(0xffffffffu, mine);
  T = __shfl_sync(0xffffffffu, T, __ffs(who) - 1);
  uint32_t gl = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) gl += (lane + 32 * q < (int)n && cv[q] > T) ? 1u : 0u;
  const uint32_t need = m - warp_sum(gl);                // ties at T kept, in column order
  uint32_t pos = 0, eq_before = 0, my_quota = 0;
  for (uint32_t s = 0; s <= me; ++s) {
    uint32_t g = 0, e = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (cs[q] == s) { g += cv[q] > T; e += cv[q] == T; }
    }
    g = warp_sum(g) + ld_peer(R.cta_above + r, s, me);
    e = warp_sum(e);
    const uint32_t qv = eq_before >= need ? 0u : min(e, need - eq_before);
    if (s < me) pos += g + qv; else my_quota = qv;
    eq_before += e;
  }
  if (lane == 0) { R.T[r] = T; R.pos[r] = pos; R.quota[r] = my_quota; R.state[r] = ST_DONE; }
}

__global__ void __launch_bounds__(kThreads, 1)
select_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int G, int L, int n_mt, const int* __restrict__ kcount,
                    int* __restrict__ out_idx, long long ldo, float* __restrict__ out_thr,
                    int mode, uint32_t* __restrict__ bitmap, int nwords, uint2* __restrict__ stash,
                    int cap, uint32_t* __restrict__ counts, const int* __restrict__ tile_fail) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  Bars& B = *reinterpret_cast<Bars*>(smem + SL::kBar);
  uint32_t* U = reinterpret_cast<uint32_t*>(smem + SL::kU);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + SL::kStage);
  Rows R = rows_of(smem + SL::kRows);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t S = gridDim.x / (uint32_t)(n_mt);   // cluster size (grid = n_mt x S)
  const uint32_t me = S > 1 ? cluster_rank() : 0u;
  const int tile_id = blockIdx.x / S;
  if (mode == M_LIST && tile_fail[tile_id] == 0) return;   // every CTA of the cluster agrees
  const int h = tile_id / ((G + BM - 1) / BM);
  const int m0 = (tile_id - h * ((G + BM - 1) / BM)) * BM;
  const int nt = (L + BN - 1) / BN;
  const int t0 = range_lo(nt, S, me), t1 = range_lo(nt, S, me + 1);
  const int nrange = t1 - t0;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      for (int s = 0; s < kStages; ++s) { mbar_init(&B.full[s], 1); mbar_init(&B.empty[s], 1); }
      for (int a = 0; a < kAcc; ++a) { mbar_init(&B.acc_full[a], 1); mbar_init(&B.acc_empty[a], kEpiWarps); }
      mbar_init(&B.a_full, 1);
      B.pass = P_MINMAX;
      B.nfull = 0;
      B.ntiles = sample_count(nrange, mode);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&B.tmem, 512);
  }
  // row state
  for (int r = threadIdx.x; r < BM; r += kThreads) {
    const bool live = m0 + r < G;
    const int kh = kcount[h];
    R.k[r] = (uint32_t)(kh < 1 ? 1 : (kh > L ? L : kh));
    R.klo[r] = KEY_LO; R.khi[r] = KEY_HI; R.above[r] = 0;
    R.state[r] = live ? ST_REFINE : ST_DONE;
    R.T[r] = 0; R.pos[r] = 0; R.quota[r] = 0; R.taken[r] = 0; R.ncand[r] = 0;
  }
  for (int i = threadIdx.x; i < BM * kHistStride; i += kThreads) U[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;

  // cluster-wide sample size (valid columns of every CTA's sample tiles)
  uint32_t ns_total = 0;
  for (uint32_t s = 0; s < S; ++s) {
    const int a0 = range_lo(nt, S, s), n = range_lo(nt, S, s + 1) - a0, cnt = sample_count(n, mode);
    for (int i = 0; i < cnt; ++i) ns_total += (uint32_t)min(BN, L - sample_tile(a0, n, cnt, i) * BN);
  }
  const SampleBand band = sample_band(R.k[0], ns_total, L, mode);   // every row: one head's k
  uint32_t seq = 0;    // tiles through the pipeline so far (same count in every role)
  const bool prof = threadIdx.x == 64;
  (void)prof;
  for (int np = 0;; ++np) {
    __syncthreads();
    const uint32_t pass = B.pass;
    const int ntl = (int)B.ntiles;
    if (pass == P_EXIT) break;
    if (prof) FPROF_AT(np, 0);

    if (warp == 0) {
      // ------------------------------------------------------------ TMA producer
      if (lane == 0) {
        if (seq == 0) {
          mbar_arrive_expect_tx(&B.a_full, BM * BK * 2);
          tma_load_3d(smem + SL::kA, &tmA, &B.a_full, 0, m0, h);
        }
        for (int i = 0; i < ntl; ++i, ++seq) {
          const int t = pass_tile(pass, t0, nrange, i, mode);
          const int s = seq % kStages;
          if (seq >= (uint32_t)kStages) FSEL_WAIT(&B.empty[s], ((seq / kStages) - 1) & 1);
          mbar_arrive_expect_tx(&B.full[s], BN * BK * 2);
          tma_load_3d(smem + SL::kB + s * (BN * BK * 2), &tmB, &B.full[s], 0, t * BN, h);
        }
      } else {
        seq += ntl;
      }
      __syncwarp();
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      if (lane == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
        if (seq == 0) mbar_wait(&B.a_full, 0);
        const uint32_t sa = smem_u32(smem + SL::kA);
        for (int i = 0; i < ntl; ++i, ++seq) {
          const int s = seq % kStages, a = seq % kAcc;
          FSEL_WAIT(&B.full[s], (seq / kStages) & 1);
          if (seq >= (uint32_t)kAcc) FSEL_WAIT(&B.acc_empty[a], ((seq / kAcc) - 1) & 1);
          tc_fence_after();
          const uint32_t sb = smem_u32(smem + SL::kB + s * (BN * BK * 2));
          mma_ss(tmem + a * BN, sdesc_sw32(sa), sdesc_sw32(sb), idesc, 0u);
          mma_commit(&B.empty[s]);
          mma_commit(&B.acc_full[a]);
        }
      } else {
        seq += ntl;
      }
      __syncwarp();
    } else {
      // ------------------------------------------------------------ epilogue
      const int ew = warp - 2;
      const int q = warp & 3;                 // TMEM lane quadrant of this warp
      const int part = ew >> 2;               // column slice of each tile
      const int row = q * 32 + lane;
      const uint32_t st = R.state[row];
      const uint32_t klo = R.klo[row], khi = R.khi[row];
      const float hi_f = st == ST_DONE ? __int_as_float(0x7f800000) : upper_f(khi);
      const float lo_f = st == ST_DONE ? __int_as_float(0x7fc00000) : key2f(klo);
      const uint64_t span = (uint64_t)(khi - klo) + 1ull;
      const uint64_t nb = span < (uint64_t)kBuckets ? span : (uint64_t)kBuckets;
      const uint64_t mult = (nb << 32) / span;
      const float T_f = key2f(R.T[row]);
      const bool emit_live = st == ST_DONE && m0 + row < G;
      float va = 0.f, vb = 0.f;               // SHIST mapping: bucket = va * s + vb
      if (pass == P_SHIST) {
        const float lo = R.smin[row], hi = R.smax[row];
        va = (hi > lo) ? (float)kBuckets / (hi - lo) : 0.f;
        vb = -lo * va;
      }
      uint32_t cnt = 0;
      float mn = __int_as_float(0x7f800000), mx = __int_as_float(0xff800000);
      uint32_t* hist = U + row * kHistStride;
      uint32_t* cand = U + row * kHistStride;    // candidates reuse the row's histogram space
      uint32_t* scr = reinterpret_cast<uint32_t*>(smem + SL::kScr) + (threadIdx.x - 64) * kScratch;
      int ft = 0, flush_t0 = t0;
      const bool warp_idle = __all_sync(0xffffffffu, st == ST_DONE);

      for (int i = 0; i < ntl; ++i, ++seq) {
        const int t = pass_tile(pass, t0, nrange, i, mode);
        const int a = seq % kAcc;
        mbar_wait(&B.acc_full[a], (seq / kAcc) & 1);
        tc_fence_after();
        if (prof && i == 0) FPROF_AT(np, 1);
        uint32_t v[kCols];
        tmem_ld_cols<kCols>(tmem + ((uint32_t)(q * 32) << 16) + a * BN + part * kCols, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.acc_empty[a]);
        const int col0 = t * BN + part * kCols;
        if (col0 + kCols > L) {
#pragma unroll
          for (int j = 0; j < kCols; ++j) if (col0 + j >= L) v[j] = 0x7fc00000u;   // NaN
        }
        if (pass == P_FULL) {
          if (!warp_idle) {
            // per 32 columns: count above the band (predicated adds) and a band bit mask;
            // the band entries (rare after the first refinement) are handled per set bit
#pragma unroll
            for (int c = 0; c < kCols / 32; ++c) {
              // four independent partial masks: no serial dependency through one register
              uint32_t gm[4] = {0u, 0u, 0u, 0u}, bm[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float s = __uint_as_float(v[c * 32 + j]);
                const bool gt = s > hi_f;
                if (gt) gm[j & 3] |= 1u << j;
                if (!gt && s >= lo_f) bm[j & 3] |= 1u << j;
              }
              cnt += __popc((gm[0] | gm[1]) | (gm[2] | gm[3]));
              const uint32_t band = (bm[0] | bm[1]) | (bm[2] | bm[3]);
              if (band) {
                // the chunk goes to this thread's scratch row (conflict-free 16-byte
                // stores), then only its band entries are visited
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  *reinterpret_cast<uint4*>(scr + j) = make_uint4(v[c * 32 + j], v[c * 32 + j + 1],
                                                                  v[c * 32 + j + 2], v[c * 32 + j + 3]);
                uint32_t bb = band;
                if (st == ST_REFINE) {
                  do {
                    const int j = __ffs(bb) - 1;
                    bb &= bb - 1;
                    const uint32_t key = f2key(__uint_as_float(scr[j]));
                    atomicAdd(hist + (uint32_t)(((uint64_t)(key - klo) * mult) >> 32), 1u);
                  } while (bb);
                } else {
                  const uint32_t slot0 = atomicAdd(R.ncand + row, (uint32_t)__popc(bb));
                  uint32_t slot = slot0;
                  do {
                    const int j = __ffs(bb) - 1;
                    bb &= bb - 1;
                    if (slot < (uint32_t)kCap) cand[slot] = f2key(__uint_as_float(scr[j]));
                    ++slot;
                  } while (bb);
                }
              }
            }
          }
        } else if (pass == P_COLLECT) {
          // one pass for the fast mode: bit (s >= lo) per column into the row's bitmap (the
          // keys above the band are kept whatever T is), and every band entry (col, key)
          // appended to this CTA's stash segment of the row; select_finish_kernel picks T
          // among the stash and emits from the bitmap
          if (!warp_idle && st != ST_DONE) {
            const long long grow = (long long)h * G + m0 + row;
            uint32_t* brow = bitmap + grow * nwords;
            uint2* srow = stash + (grow * S + me) * cap;
#pragma unroll
            for (int c = 0; c < kCols / 32; ++c) {
              uint32_t gm[4] = {0u, 0u, 0u, 0u}, bm[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float s = __uint_as_float(v[c * 32 + j]);
                const bool gt = s > hi_f;
                if (gt) gm[j & 3] |= 1u << j;
                if (!gt && s >= lo_f) bm[j & 3] |= 1u << j;
              }
              const uint32_t gt = (gm[0] | gm[1]) | (gm[2] | gm[3]);
              const uint32_t band = (bm[0] | bm[1]) | (bm[2] | bm[3]);
              const int cbase = col0 + c * 32;
              if ((cbase >> 5) < nwords) brow[cbase >> 5] = gt | band;
              if (band) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  *reinterpret_cast<uint4*>(scr + j) = make_uint4(v[c * 32 + j], v[c * 32 + j + 1],
                                                                  v[c * 32 + j + 2], v[c * 32 + j + 3]);
                uint32_t bb = band;
                uint32_t slot = atomicAdd(R.ncand + row, (uint32_t)__popc(bb));
                do {
                  const int j = __ffs(bb) - 1;
                  bb &= bb - 1;
                  if (slot < (uint32_t)cap)
                    srow[slot] = make_uint2((uint32_t)(cbase + j), f2key(__uint_as_float(scr[j])));
                  ++slot;
                } while (bb);
              }
            }
          }
        } else if (pass == P_EMIT) {
          // masks (s > T) and (s == T), 32 columns per word
#pragma unroll
          for (int w = 0; w < kCols / 32; ++w) {
            uint32_t gm[4] = {0u, 0u, 0u, 0u}, em[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float s = __uint_as_float(v[w * 32 + j]);
              if (s > T_f) gm[j & 3] |= 1u << j;
              if (s == T_f) em[j & 3] |= 1u << j;
            }
            const uint32_t gt = (gm[0] | gm[1]) | (gm[2] | gm[3]);
            const uint32_t eq = (em[0] | em[1]) | (em[2] | em[3]);
            const int wi = part * (kCols / 32) + w;
            stage[row * kStageStride + ft * 8 + wi] = emit_live ? gt : 0u;
            stage[row * kStageStride + ft * 8 + 4 + wi] = emit_live ? eq : 0u;
          }
          ++ft;
          if (ft == kFlushTiles || i == ntl - 1) {
            named_bar_sync(1, kEpiThreads);
            // flush: warp per row, lane = one 32-column word
            constexpr int kRowsPerWarp = BM / kEpiWarps;
            for (int rr = 0; rr < kRowsPerWarp; ++rr) {
              const int r = ew * kRowsPerWarp + rr;
              if (m0 + r >= G) continue;
              const int wt = lane >> 2, wi = lane & 3;
              uint32_t gt = 0, eq = 0;
              if (wt < ft) {
                gt = stage[r * kStageStride + wt * 8 + wi];
                eq = stage[r * kStageStride + wt * 8 + 4 + wi];
              }
              const uint32_t quota = R.quota[r], taken = R.taken[r];
              const uint32_t ec = __popc(eq);
              uint32_t ex = ec;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, ex, o);
                if (lane >= o) ex += y;
              }
              const uint32_t eq_before = taken + ex - ec;
              const uint32_t take = eq_before >= quota ? 0u : min(ec, quota - eq_before);
              uint32_t keep = 0;
              if (take == ec) {
                keep = eq;
              } else {
                uint32_t x = eq;
                for (uint32_t c = 0; c < take; ++c) { const uint32_t lb = x & (0u - x); keep |= lb; x ^= lb; }
              }
              uint32_t word = gt | keep;
              const uint32_t c = __popc(word);
              uint32_t cx = c;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, cx, o);
                if (lane >= o) cx += y;
              }
              const uint32_t total = __shfl_sync(0xffffffffu, cx, 31);
              uint32_t tk = take;
#pragma unroll
              for (int o = 16; o; o >>= 1) tk += __shfl_xor_sync(0xffffffffu, tk, o);
              uint32_t p = R.pos[r] + cx - c;
              int* orow = out_idx + ((long long)h * G + m0 + r) * ldo;
              const int cbase = (flush_t0 + wt) * BN + wi * 32;
              while (word) {
                const int b = __ffs(word) - 1;
                orow[p++] = cbase + b;
                word &= word - 1;
              }
              __syncwarp();
              if (lane == 0) { R.pos[r] += total; R.taken[r] = taken + tk; }
              __syncwarp();
            }
            named_bar_sync(1, kEpiThreads);
            flush_t0 = t0 + i + 1;
            ft = 0;
          }
        } else if (pass == P_MINMAX) {
#pragma unroll
          for (int j = 0; j < kCols; ++j) {
            const float s = __uint_as_float(v[j]);
            mn = fminf(mn, s);
            mx = fmaxf(mx, s);
          }
        } else {   // P_SHIST
          if (m0 + row < G) {
#pragma unroll
            for (int j = 0; j < kCols; ++j) {
              const float s = __uint_as_float(v[j]);
              if (s == s) {
                // bucket ~ floor(s va + vb) without F2I (a quarter-rate unit shared with the
                // MUFU): clamp in float, round (t - 0.5) to nearest with the 1.5 * 2^23 add;
                // an edge value may land one bucket low — the band is an estimate, a miss is
                // detected and re-run exactly
                const float t = fminf(fmaxf(__fmaf_rn(s, va, vb), 0.f), (float)kBuckets - 0.5f);
                const int b = (int)(__float_as_uint(__fadd_rn(t - 0.5f, 12582912.f)) - 0x4B400000u);
                atomicAdd(hist + b, 1u);
              }
            }
          }
        }
      }
      // partials of this pass -> per-CTA totals
      if (prof) FPROF_AT(np, 2);
      if (pass == P_FULL) R.part_above[part * BM + row] = cnt;
      if (pass == P_MINMAX) {
        reinterpret_cast<float*>(R.part_above)[part * BM + row] = mn;
        reinterpret_cast<float*>(stage)[part * BM + row] = mx;
      }
      named_bar_sync(1, kEpiThreads);
      if (pass == P_COLLECT && part == 0 && m0 + row < G) {
        const long long grow = (long long)h * G + m0 + row;
        counts[grow * S + me] = R.ncand[row];
        if (me == 0) reinterpret_cast<uint2*>(counts + (long long)gridDim.x * BM)[grow] =
            make_uint2(R.klo[row], R.khi[row]);       // the band, for the finish kernel
      }
      if (part == 0) {
        if (pass == P_FULL) {
          uint32_t c = 0;
          for (int p = 0; p < kParts; ++p) c += R.part_above[p * BM + row];
          R.cta_above[row] = c;
        } else if (pass == P_MINMAX) {
          float a = __int_as_float(0x7f800000), b = __int_as_float(0xff800000);
          for (int p = 0; p < kParts; ++p) {
            a = fminf(a, reinterpret_cast<float*>(R.part_above)[p * BM + row]);
            b = fmaxf(b, reinterpret_cast<float*>(stage)[p * BM + row]);
          }
          R.cta_min[row] = a;
          R.cta_max[row] = b;
        }
      }
    }

    // ---------------------------------------------------------------- pass end
    if (prof) FPROF_AT(np, 3);
    if (S > 1) cluster_sync(); else __syncthreads();
    if (prof) FPROF_AT(np, 4);
    if (warp >= 2 && pass != P_EMIT && pass != P_COLLECT) {
      for (int r = warp - 2; r < BM; r += kEpiWarps)
        finalize_row(R, U, r, lane, pass, S, me, band, L, mode);
    }
    if (prof) FPROF_AT(np, 5);
    if (S > 1) cluster_sync(); else __syncthreads();
    if (prof) FPROF_AT(np, 6);
    // clear this CTA's partials for the next pass; choose the next pass
    if (warp >= 2) {
      const int et = threadIdx.x - 64;
      for (int i = et; i < BM * kHistStride; i += kEpiThreads) U[i] = 0;
      for (int r = et; r < BM; r += kEpiThreads) R.ncand[r] = 0;
      if (et == 0) B.flag = 0;
      named_bar_sync(1, kEpiThreads);
      if (et < BM && R.state[et] != ST_DONE) atomicOr(&B.flag, 1u);
      named_bar_sync(1, kEpiThreads);
      if (et == 0) {
        uint32_t next, n;
        if (pass == P_MINMAX) { next = P_SHIST; n = sample_count(nrange, mode); }
        else if (pass == P_SHIST && mode == M_FAST) { next = P_COLLECT; n = nrange; }
        else if (pass == P_COLLECT) { next = P_EXIT; n = 0; }
        else if (pass == P_SHIST || pass == P_FULL) {
          // (FULL passes are bounded: each narrows the key range 128x; the cap only
          // guards against a hang)
          const uint32_t cap = 64u;
          if (B.flag && B.nfull < cap) { next = P_FULL; n = nrange; ++B.nfull; } else { next = P_EMIT; n = nrange; }
        } else { next = P_EXIT; n = 0; }
        B.pass = next;
        B.ntiles = n;
      }
    }
    if (prof) { FPROF_AT(np, 7); }
    if (pass == P_EMIT) {
      // thresholds (one CTA of the cluster writes them)
      if (warp >= 2 && me == 0) {
        const int et = threadIdx.x - 64;
        if (et < BM && m0 + et < G) out_thr[(long long)h * G + m0 + et] = key2f(R.T[et]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
  if (S > 1) cluster_sync();   // no CTA exits while a peer may still read its shared memory
}


// ------------------------------------------------------------------ fast-mode finish
// One warp per (head, proxy) row, after the collect pass: the row's bitmap marks every key
// with s >= lo (all of S CTAs' key ranges) and the stash segments hold the band entries
// (lo <= s <= hi) as (column, order key). With n_ge set bits and B band entries,
// above = n_ge - B keys lie above the band, so T is the m-th largest band key, m = k - above
// (1 <= m <= B when the band brackets T). Ties at T are kept in column order up to the
// quota: need = m - #(band > T); when more band entries equal T, the need-th smallest tie
// column bounds the kept ones. Dropped band entries are cleared from the bitmap, which then
// holds exactly the k kept keys; a warp-wide scan over its words emits them ascending.
// A row whose band missed T or overflowed its stash flags its row tile for the exact
// multi-pass re-run (M_LIST launch).
constexpr int kFinThreads = 256;
constexpr int kFinDigit = 11;                        // radix digit (2048-bucket histogram)
constexpr int kFinBuckets = 1 << kFinDigit;

struct FinShared {
  uint32_t hist[kFinBuckets];
  uint32_t red[2][kFinThreads / 32];
  uint32_t b, above, cnt;
};

// m-th largest (1-based) key among n entries passing `keyf`, all keys in [kmin, kmin + range]:
// radix select on key - kmin with 11-bit digits from the top of the range (two rounds for
// the band's ~2^22-ulp spread). *rem = m minus the number of entries strictly above it;
// *eq = the number equal to it (the last round's digit resolves the key exactly, so its
// bucket count is that number).
template <typename AtF, typename KeyF>
DSV_DEV uint32_t block_select(AtF at, uint32_t n, uint32_t m, uint32_t kmin, uint32_t range,
                              FinShared& F, KeyF keyf, uint32_t* rem, uint32_t* eq) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = kFinBuckets / kFinThreads;    // buckets per thread (8)
  const int top = range ? 31 - __clz(range) : 0;
  uint32_t prefix = 0, remaining = m;
  for (int sh = top + 1 - kFinDigit; sh > -kFinDigit; sh -= kFinDigit) {
    const int shift = sh > 0 ? sh : 0;
    const uint32_t mask_hi = sh + kFinDigit >= 32 ? 0u : (0xffffffffu << (sh + kFinDigit));
#pragma unroll
    for (int j = 0; j < kPer; ++j) F.hist[tid * kPer + j] = 0u;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kFinThreads) {
      uint32_t key;
      if (keyf(at(i), key)) {
        const uint32_t x = key - kmin;
        if ((x & mask_hi) == prefix) atomicAdd(&F.hist[(x >> shift) & (kFinBuckets - 1)], 1u);
      }
    }
    __syncthreads();
    // thread t owns buckets (top down) kFinBuckets-1-kPer*t ..; block scan of their counts
    uint32_t c[kPer], tot = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) { c[j] = F.hist[kFinBuckets - 1 - kPer * tid - j]; tot += c[j]; }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) F.red[0][warp] = incl;
    __syncthreads();
    uint32_t wb = 0;
#pragma unroll
    for (int w = 0; w < kFinThreads / 32; ++w) wb += w < warp ? F.red[0][w] : 0u;
    incl += wb;
    const uint32_t excl = incl - tot;
    if (excl < remaining && incl >= remaining) {
      uint32_t run = excl;
      int j = 0;
      while (run + c[j] < remaining) { run += c[j]; ++j; }
      F.b = kFinBuckets - 1 - kPer * tid - j;
      F.above = run;
      F.cnt = c[j];
    }
    __syncthreads();
    prefix |= F.b << shift;
    remaining -= F.above;
    __syncthreads();
  }
  *rem = remaining;
  *eq = F.cnt;
  return prefix + kmin;
}

DSV_DEV uint32_t block_sum(uint32_t v, FinShared& F) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) F.red[1][warp] = v;
  __syncthreads();
  uint32_t t = 0;
#pragma unroll
  for (int w = 0; w < kFinThreads / 32; ++w) t += F.red[1][w];
  __syncthreads();
  return t;
}

// One CTA (256 threads) per (head, proxy) row, after the collect pass: the row's bitmap marks
// every key with s >= lo (all S key ranges) and the stash segments hold the band entries
// (lo <= s <= hi) as (column, order key). With n_ge set bits and B band entries,
// above = n_ge - B keys lie above the band, so T is the m-th largest band key, m = k - above
// (1 <= m <= B when the band brackets T). Ties at T are kept in column order up to the
// quota: need = m - #(band > T); when more band entries equal T, the need-th smallest tie
// column bounds the kept ones. Dropped band entries are cleared from the shared copy of the
// bitmap, which then holds exactly the k kept keys, emitted ascending by a block scan.
// A row whose band missed T (or overflowed its stash) flags its row tile for the exact
// multi-pass re-run (M_LIST launch).
template <bool kStaged>
DSV_DEV void finish_row(FinShared& F, uint8_t* fin_smem, long long row, int G, int L,
                        uint32_t S, const int* __restrict__ kcount,
                        const uint32_t* __restrict__ bitmap, int nwords,
                        const uint2* __restrict__ stash, int cap, const uint32_t (&segn)[8],
                        uint32_t B, const uint2* __restrict__ bandlim, int* __restrict__ out_idx,
                        long long ldo, float* __restrict__ out_thr, int* fail, int smem_cap);

__global__ void __launch_bounds__(kFinThreads)
select_finish_kernel(int H, int G, int L, uint32_t S, const int* __restrict__ kcount,
                     const uint32_t* __restrict__ bitmap, int nwords,
                     const uint2* __restrict__ stash, int cap, const uint32_t* __restrict__ counts,
                     const uint2* __restrict__ bandlim, int* __restrict__ out_idx, long long ldo,
                     float* __restrict__ out_thr, int* __restrict__ tile_fail, int smem_cap) {
  __shared__ FinShared F;
  extern __shared__ __align__(16) uint8_t fin_smem[];
  const long long row = blockIdx.x;
  const int h = (int)(row / G), g = (int)(row % G);
  int* fail = tile_fail + h * ((G + BM - 1) / BM) + g / BM;
  uint32_t segn[8];
  uint32_t B = 0;
  bool over = false;
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s) {
    segn[s] = 0;
    if (s >= S) continue;
    const uint32_t n = counts[row * S + s];
    over |= n > (uint32_t)cap;
    segn[s] = n > (uint32_t)cap ? (uint32_t)cap : n;
    B += segn[s];
  }
  if (over) {
    if (threadIdx.x == 0) atomicExch(fail, 1);
    return;
  }
  // (the branch is uniform per CTA; each body reads its band entries one way)
  if (B <= (uint32_t)smem_cap)
    finish_row<true>(F, fin_smem, row, G, L, S, kcount, bitmap, nwords, stash, cap, segn, B,
                     bandlim, out_idx, ldo, out_thr, fail, smem_cap);
  else
    finish_row<false>(F, fin_smem, row, G, L, S, kcount, bitmap, nwords, stash, cap, segn, B,
                      bandlim, out_idx, ldo, out_thr, fail, smem_cap);
}

template <bool kStaged>
DSV_DEV void finish_row(FinShared& F, uint8_t* fin_smem, long long row, int G, int L,
                        uint32_t S, const int* __restrict__ kcount,
                        const uint32_t* __restrict__ bitmap, int nwords,
                        const uint2* __restrict__ stash, int cap, const uint32_t (&segn)[8],
                        uint32_t B, const uint2* __restrict__ bandlim, int* __restrict__ out_idx,
                        long long ldo, float* __restrict__ out_thr, int* fail, int smem_cap) {
  const int tid = threadIdx.x;
  const int nw4 = (nwords + 3) & ~3;
  uint32_t* bits = reinterpret_cast<uint32_t*>(fin_smem);
  uint2* sband = reinterpret_cast<uint2*>(bits + nw4);
  const int h = (int)(row / G);
  const int kh = kcount[h];
  const uint32_t k = (uint32_t)(kh < 1 ? 1 : (kh > L ? L : kh));
  // stage the bitmap and (when they fit) the band entries in shared memory
  const uint4* brow = reinterpret_cast<const uint4*>(bitmap + row * nwords);
  uint32_t nge = 0;
  if ((nwords & 3) == 0 && ((row * nwords) & 3) == 0) {
    for (int w = tid; w < nwords / 4; w += kFinThreads) {
      const uint4 x = brow[w];
      reinterpret_cast<uint4*>(bits)[w] = x;
      nge += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
  } else {
    const uint32_t* b1 = bitmap + row * nwords;
    for (int w = tid; w < nwords; w += kFinThreads) {
      const uint32_t x = b1[w];
      bits[w] = x;
      nge += __popc(x);
    }
  }
  const uint2* gbase = stash + row * S * cap;
  uint32_t sstart[8];
  {
    uint32_t off = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) { sstart[s] = off; off += segn[s]; }
  }
  if (kStaged) {
    // band entries: four loads in flight per thread before their shared-memory stores
    for (uint32_t s = 0; s < S; ++s) {
      const uint2* src = gbase + (size_t)s * cap;
      for (uint32_t i0 = 0; i0 < segn[s]; i0 += 4 * kFinThreads) {
        uint2 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t i = i0 + j * kFinThreads + tid;
          if (i < segn[s]) v[j] = src[i];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t i = i0 + j * kFinThreads + tid;
          if (i < segn[s]) sband[sstart[s] + i] = v[j];
        }
      }
    }
  }
  // entry i of the row's band: shared copy, or its stash segment (rows too large to stage)
  auto at = [&](uint32_t i) -> uint2 {
    if (kStaged) return sband[i];
    uint32_t s = 0;
    while (s + 1 < S && i >= sstart[s + 1]) ++s;
    return gbase[(size_t)s * cap + (i - sstart[s])];
  };
  nge = block_sum(nge, F);       // (its barriers also publish the staged copies)
  const uint32_t above = nge - B;
  if (nge < B || above >= k || above + B < k) {
    if (tid == 0) atomicExch(fail, 1);
    return;
  }
  const uint32_t m = k - above;
  const uint2 lim = bandlim[row];
  uint32_t need, eq;
  const uint32_t T = block_select(at, B, m, lim.x, lim.y - lim.x, F,
                                  [](uint2 e, uint32_t& key) { key = e.y; return true; }, &need,
                                  &eq);
  uint32_t col_max = 0xffffffffu;
  if (eq > need) {
    uint32_t dummy, dummy2;
    const uint32_t cmin = ~(uint32_t)(L - 1);         // ~col lies in [~(L-1), ~0]
    col_max = ~block_select(at, B, need, cmin, (uint32_t)(L - 1), F,
                            [T](uint2 e, uint32_t& key) { key = ~e.x; return e.y == T; }, &dummy,
                            &dummy2);
  }
  for (uint32_t i = tid; i < B; i += kFinThreads) {
    const uint2 e = at(i);
    if (!(e.y > T || (e.y == T && e.x <= col_max))) atomicAnd(bits + (e.x >> 5), ~(1u << (e.x & 31)));
  }
  __syncthreads();
  // emit: thread t owns a contiguous run of words; block exclusive scan of their popcounts
  const int wpt = (nwords + kFinThreads - 1) / kFinThreads;
  const int w0 = tid * wpt, w1 = min(nwords, w0 + wpt);
  uint32_t c = 0;
  for (int w = w0; w < w1; ++w) c += __popc(bits[w]);
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) F.red[1][warp] = incl;
  __syncthreads();
  uint32_t wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kFinThreads / 32; ++w) {
    if (w < warp) wbase += F.red[1][w];
    total += F.red[1][w];
  }
  if (total != k) {                    // cannot happen when the band brackets T; be exact
    if (tid == 0) atomicExch(fail, 1);
    return;
  }
  // indices go to shared memory (the band's space, no longer read) when they fit, then out
  // in coalesced 16-byte stores; a thread's own run of scattered stores would touch a
  // separate sector per lane
  int* grow = out_idx + row * ldo;
  const bool stage_out = (long long)k * 4 <= (long long)smem_cap * 8;
  int* op = (stage_out ? reinterpret_cast<int*>(sband) : grow) + (wbase + incl - c);
  for (int w = w0; w < w1; ++w) {
    uint32_t word = bits[w];
    const int cb = w * 32;
    while (word) {
      *op++ = cb + __ffs(word) - 1;
      word &= word - 1;
    }
  }
  if (tid == 0) out_thr[row] = key2f(T);
  if (stage_out) {
    __syncthreads();
    const int* so = reinterpret_cast<const int*>(sband);
    if ((reinterpret_cast<uintptr_t>(grow) & 15) == 0) {
      for (uint32_t i = tid; i < k / 4; i += kFinThreads)
        reinterpret_cast<int4*>(grow)[i] = reinterpret_cast<const int4*>(so)[i];
      for (uint32_t i = (k & ~3u) + tid; i < k; i += kFinThreads) grow[i] = so[i];
    } else {
      for (uint32_t i = tid; i < k; i += kFinThreads) grow[i] = so[i];
    }
  }
}
}  // namespace fsel
}  // namespace dsv

int dsv_select_fused_smem_bytes() { return dsv::fsel::SL::kBytes; }

// Clusters of S select_fused_kernel CTAs (one per SM: ~221 KB of shared memory) that can be
// resident at once on the current device (cudaOccupancyMaxActiveClusters: a cluster must fit
// in one GPC, so 4-CTA clusters leave SMs unused where a GPC's count is not a multiple of 4).
// 0 when it cannot be queried (no device).
int dsv_select_fused_clusters_query(int S) {
  using namespace dsv::fsel;
  if (S < 1 || S > 8) return 0;
  if (cudaFuncSetAttribute(select_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           SL::kBytes) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(S * 64), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = SL::kBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, select_fused_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int dsv_debug_select_timeline_copy(void* dst, int bytes) {
  const int n = (int)sizeof(g_fsel_prof) < bytes ? (int)sizeof(g_fsel_prof) : bytes;
  if (cudaMemcpyFromSymbol(dst, g_fsel_prof, n) != cudaSuccess) return -1;
  return n;
}

// grid = n_mt row tiles x S key-range CTAs (cluster of S along x)
static int launch_select(const CUtensorMap* ta, const CUtensorMap* tb, int H, int G, int L,
                         const int* kcount, int* out_idx, long long ldo, float* out_thr, int S,
                         int mode, uint32_t* bitmap, int nwords, uint2* stash, int cap,
                         uint32_t* counts, const int* tile_fail, cudaStream_t st) {
  using namespace dsv::fsel;
  const int n_mt = H * ((G + BM - 1) / BM);
  auto kern = select_fused_kernel;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SL::kBytes);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_mt * S), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = SL::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, *ta, *tb, G, L, n_mt, kcount, out_idx, ldo, out_thr,
                                 mode, bitmap, nwords, stash, cap, counts, tile_fail);
}

// fast-mode workspace: [tile_fail n_mt ints | counts rows*S u32 | bitmap rows*nwords u32 |
// stash rows*S*cap uint2], each part 256-byte aligned; cap (band entries per row and CTA)
// is what the remaining bytes hold
static long long align256(long long x) { return (x + 255) & ~255LL; }

static long long fixed_ws_bytes(int H, int G, int L, int S) {
  const long long rows = (long long)H * G, n_mt = (long long)H * ((G + 127) / 128);
  return align256(n_mt * 4) + align256(n_mt * S * 128 * 4 + rows * 8) +
         align256(rows * ((L + 31) / 32) * 4);
}

// Expected band entries per (row, CTA): the sample passes pick a band of +-(5.5 sigma + 8)
// sample ranks around the k-th (binomial sigma of the sample count above it), widened to
// the 128-bucket grid of the sample histogram; cap = twice that (0 = the single pass is
// not worthwhile: the band would hold too large a share of the keys, or too many bytes).
long long dsv_select_fused_ws_bytes(int H, int G, int L, int k_max, int S) {
  using namespace dsv::fsel;
  const int nt = (L + BN - 1) / BN;
  const int n = (nt + S - 1) / S;
  const double ns = (double)S * sample_count(n, 1) * BN;
  const double pk = fmin((double)k_max, (double)(L - k_max)) / L;
  const double sig = sqrt(fmax(ns * pk * (1.0 - pk), 0.0));
  const double frac = 2.0 * (5.5 * sig + 8.0) / ns + 4.0 / kBuckets;
  if (frac > 0.15) return 0;
  const long long band = (long long)(frac * L / S) + 64;
  const long long cap = ((2 * band + 255) / 256) * 256;
  const long long rows = (long long)H * G;
  const long long bytes = fixed_ws_bytes(H, G, L, S) + align256(rows * S * cap * 8);
  return bytes > (1LL << 30) ? 0 : bytes;
}

int dsv_select_fused_launch(const CUtensorMap* ta, const CUtensorMap* tb, int H, int G, int L,
                            const int* kcount, int* out_idx, long long ldo, float* out_thr,
                            int S, void* ws, long long ws_bytes, cudaStream_t st) {
  using namespace dsv::fsel;
  const long long rows = (long long)H * G, n_mt = (long long)H * ((G + BM - 1) / BM);
  const long long fixed = fixed_ws_bytes(H, G, L, S);
  const long long capl = ws ? (ws_bytes - fixed) / (rows * S * 8) : 0;
  if (capl < 256)
    return launch_select(ta, tb, H, G, L, kcount, out_idx, ldo, out_thr, S, M_CLASSIC, nullptr, 0,
                         nullptr, 0, nullptr, nullptr, st);
  const int cap = (int)(capl > (1 << 24) ? (1 << 24) : capl);
  const int nwords = (L + 31) / 32;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  int* tile_fail = reinterpret_cast<int*>(p);
  p += align256(n_mt * 4);
  // counts [rows][S] (row tiles x BM x S words reserved: the kernel addresses the band limits
  // [rows] uint2 right after gridDim.x * BM words) then the band limits
  uint32_t* counts = reinterpret_cast<uint32_t*>(p);
  const uint2* bandlim = reinterpret_cast<const uint2*>(counts + n_mt * S * BM);
  p += align256(n_mt * S * 128 * 4 + rows * 8);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(p);
  p += align256(rows * nwords * 4);
  uint2* stash = reinterpret_cast<uint2*>(p);
  cudaMemsetAsync(tile_fail, 0, n_mt * 4, st);
  int rc = launch_select(ta, tb, H, G, L, kcount, out_idx, ldo, out_thr, S, M_FAST, bitmap, nwords,
                         stash, cap, counts, tile_fail, st);
  if (rc) return rc;
  // one CTA per row: its bitmap and band entries staged in shared memory (<= 36 KB with the
  // static part, so six CTAs share an SM); rows with more band entries read them from the
  // workspace
  const int nw4 = (nwords + 3) & ~3;
  long long smem_cap = (36 * 1024 - 8400 - nw4 * 4) / 8;
  if (smem_cap > (long long)S * cap) smem_cap = (long long)S * cap;
  if (smem_cap < 0) smem_cap = 0;
  const size_t fin_smem = (size_t)nw4 * 4 + (size_t)smem_cap * 8;
  if (fin_smem > 200 * 1024) return (int)cudaErrorInvalidValue;
  cudaFuncSetAttribute(select_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)fin_smem);
  select_finish_kernel<<<(unsigned)rows, kFinThreads, fin_smem, st>>>(
      H, G, L, (uint32_t)S, kcount, bitmap, nwords, stash, cap, counts, bandlim, out_idx, ldo,
      out_thr, tile_fail, (int)smem_cap);
  rc = (int)cudaGetLastError();
  if (rc) return rc;
  // exact multi-pass re-run of flagged row tiles (its CTAs exit at once when none is)
  return launch_select(ta, tb, H, G, L, kcount, out_idx, ldo, out_thr, S, M_LIST, nullptr, 0,
                       nullptr, 0, nullptr, tile_fail, st);
}
