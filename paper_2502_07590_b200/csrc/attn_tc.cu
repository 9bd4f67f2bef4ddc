// attn_tc.cu — K3: block-sparse flash attention on tcgen05/TMEM (sm_100a).
//
// Query tile = one voxel group (<= 128 queries sharing one critical-KV list;
// reference pkg/src/dynsparse/grouping.py:196-216 `grouped_sparse_attention`,
// which expands to pkg/src/dynsparse/attention.py:153-187 `sparse_attention`:
// softmax over the selected logits only, logits divided by sqrt(d)).
// Backward semantics follow the autograd of pkg/src/dynsparse/trainer.py:110-117
// (gather -> einsum -> softmax -> einsum): dQ per query, dK/dV scatter-added
// over every query that selected a key.
//
// Layout in HBM: Q, K, V, O, dO as bf16 [H, L, D] (rows of D contiguous);
// group members int32 [G, 128] (padded with the last member), index lists int32
// [H, G, ldk] ascending, k per head int32 [H]; LSE fp32 [H, L] in the log2
// domain of the scaled logits (lse2 = max + log2(sum)).
//
// Both kernels are persistent: one CTA per SM draws 128-query tiles (a voxel group, or a
// 128-query slice of a larger ladder group sharing its index row) from a global atomic
// counter in head-major order, so the K/V of the one or two heads in flight stay
// L2-resident; every role keeps running block counters for its barrier parities, so the
// next tile's loads and first MMAs overlap the current tile's tail. Gather producers issue
// 16-byte cp.async copies of the selected K/V rows straight into 128B-swizzled UMMA tiles
// (measured on B200: ~50 B/clk/SM for random 256 B rows, vs ~8 for TMA tile::gather4).
// Forward, 800 threads: warps 0-15 softmax (4 per TMEM lane quarter, one 32-key slice
// each), warp 16 tcgen05.mma issuer + TMEM owner, warps 17-24 producers (K ring and V ring
// 3 deep each, three S/P buffers in TMEM, S issued three blocks ahead). The row max is
// exchanged for key block 0 only (lazy max: later blocks exponentiate against it, a tile
// whose scores exceed it by 2^64 is flagged and re-run with the per-block exchange); P
// (bf16) overwrites the warp's own S columns; O += P V reads P from TMEM (A operand) and
// V from shared memory (MN-major B); the producers also zero the backward's dK/dV
// accumulators for this tile's share.
// Backward, 864 threads: warps 0-15 row workers (4 per TMEM lane quarter), warp 16 MMA
// issuer, warps 17-18 producers, warps 19-26 dK/dV scatter. Transposed (keys in TMEM
// lanes): S^T = K_j Q^T, dP^T = V_j dO^T; workers (one key per thread) form P^T, dS^T in
// TMEM and dS in smem; then dQ += dS K_j, dV_j = P^T dO, dK_j = dS^T Q; dV_j / dK_j rows
// are staged through shared memory and scatter-added with row-contiguous red.v4 (the fp32
// L2 reduction rate bounds the kernel). Once the tile queue is exhausted the CTAs convert
// the finished heads' dK/dV accumulators to bf16 (per-head completion counters).
// Optional row-address tables send O / dQ / dK / dV rows to their token owners' peer
// buffers (head-parallel CP) from the same epilogue stores.

#include <cuda.h>
#include "dsv_common.cuh"

namespace dsv {
namespace attn {

constexpr int BQ = 128;   // queries per tile
constexpr int BKV = 128;  // keys per block
#ifndef DSV_PROD_WARPS
#define DSV_PROD_WARPS 8
#endif
constexpr int kProdWarps = DSV_PROD_WARPS;    // forward gather producers
constexpr int kProdThreads = kProdWarps * 32;

template <int D, int NT = kProdThreads>
struct Gather {
  static constexpr int kCPR = D / 8;                          // 16-byte chunks per row
  static constexpr int kPer = 128 * kCPR / NT;                // chunks per thread per tile
  static constexpr int kRowStep = NT / kCPR;                  // rows between a thread's chunks
  static constexpr int kTile = 128 * D * 2;
};

// Issue the cp.async copies of one 128-row tile (rows[i] = absolute row id of
// this thread's i-th chunk) into a 128B-swizzled K-major tile (atom = 64 cols).
template <int D, int NT = kProdThreads>
DSV_DEV void issue_tile(uint8_t* tile, const __nv_bfloat16* base,
                        const int (&rows)[Gather<D, NT>::kPer], int ptid) {
  using G = Gather<D, NT>;
  const int q = ptid % G::kCPR, r0 = ptid / G::kCPR;
  const uint32_t t0 = smem_u32(tile) + (q >> 3) * (128 * 128);
#pragma unroll
  for (int i = 0; i < G::kPer; ++i)
    cp_async16(t0 + sw128_off(r0 + i * G::kRowStep, q & 7), base + (long long)rows[i] * D + q * 8);
}

// ====================================================================== fwd
#ifndef DSV_FWD_KSTAGES
#define DSV_FWD_KSTAGES 3
#endif
constexpr int kFwdKStages = DSV_FWD_KSTAGES;                     // K_j frees after S_j
#ifndef DSV_FWD_VSTAGES
#define DSV_FWD_VSTAGES 3
#endif
constexpr int kFwdStages = DSV_FWD_VSTAGES;                      // V ring (frees after PV_j)
constexpr int kFwdSBufs = 3;                                     // S/P buffers in TMEM
#ifndef DSV_FWD_SOFT_WGS
#define DSV_FWD_SOFT_WGS 4
#endif
constexpr int kFwdSoftWGs = DSV_FWD_SOFT_WGS;                    // warps 0-15
// each softmax warp owns one 32-key slice of a 128-key block per TMEM lane quarter
static_assert(kFwdSoftWGs * 32 == BKV, "forward: four softmax warpgroups (32-key slices)");
constexpr int kFwdSoftThreads = kFwdSoftWGs * 128;
constexpr int kFwdMmaWarp = kFwdSoftWGs * 4;
constexpr int kFwdProdWarp0 = kFwdMmaWarp + 1;
constexpr int kFwdThreads = (kFwdProdWarp0 + kProdWarps) * 32;   // 800

template <int D>
struct FwdSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + kFwdKStages * kTile;
  static constexpr int kMax = kV + kFwdStages * kTile;   // [4 slices][128] fp32 row exchange
  static constexpr int kBar = kMax + kFwdSoftWGs * 128 * 4;
  // Q + 3 K + 3 V tiles (D = 128: 224 KB) leave no room for alignment slack: the dynamic
  // shared window starts 1024-aligned (checked at kernel entry)
  static constexpr int kBytes = kBar + 256 + (kFwdKStages + kFwdStages >= 6 && D == 128 ? 0 : 1024);
  static constexpr bool kSlack = !(kFwdKStages + kFwdStages >= 6 && D == 128);
  static_assert(kBytes <= 232448, "forward shared memory over 227 KB");
};

struct FwdBars {
  uint64_t q_full;
  uint64_t k_full[kFwdKStages], k_empty[kFwdKStages];     // K_j is free once S_j is done,
  uint64_t v_full[kFwdStages], v_empty[kFwdStages];       // V_j only after PV_j
  // per S/P buffer, so no barrier can run two phases ahead of its waiter
  uint64_t s_full[kFwdSBufs], p_full[kFwdSBufs], pv_done[kFwdSBufs];
  uint64_t o_final;
  uint64_t q_empty, o_empty;  // persistent CTAs: Q / the O accumulator free for the next tile
  uint64_t tq_full[2], tq_empty[2];  // tile-id queue (dynamic schedule)
  int tq[2];
  uint32_t tmem;
  uint32_t ovf;             // lazy-max pass: some score exceeded the row's reference max by > 2^64
};
static_assert(sizeof(FwdBars) <= 256, "forward barriers over their 256 B");

#ifndef DSV_FWD_LAZY
#define DSV_FWD_LAZY 1     // 0: exchange the row max every key block (the exact-max pass only)
#endif
constexpr float kLazyLimit = 64.f;   // log2 headroom of the lazy-max pass
// Optional in-kernel timeline (variant builds with -DDSV_BWD_PROF / -DDSV_FWD_PROF):
// clock64 stamps of each role's phase boundaries for the first kProfCtas CTAs of the
// backward (or forward) kernel, read back by dsv_debug_timeline.
constexpr int kProfCtas = 8, kProfBlocks = 32, kProfEv = 12;
__device__ long long g_bwd_prof[kProfCtas][kProfBlocks][kProfEv];
#define PROF_STAMP(j, e) do { if (blockIdx.x < kProfCtas && (j) < kProfBlocks) g_bwd_prof[blockIdx.x][j][e] = clock64(); } while (0)
#ifdef DSV_BWD_PROF
#define PROF(j, e) PROF_STAMP(j, e)
#else
#define PROF(j, e) do {} while (0)
#endif
#ifdef DSV_FWD_PROF
#define FPROF(j, e) PROF_STAMP(j, e)
#else
#define FPROF(j, e) do {} while (0)
#endif

// Softmax pass 1: row max of the raw scores of one S buffer (two TMEM loads in flight,
// 3-input max).
template <bool kMasked>
DSV_DEV float softmax_max_pass(uint32_t tS, int kv) {
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < BKV / 32; c += 2) {
    uint32_t r0[32], r1[32];
    tmem_ld32(tS + c * 32, r0);
    tmem_ld32(tS + (c + 1) * 32, r1);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float a0 = __uint_as_float(r0[i]), a1 = __uint_as_float(r0[i + 1]);
      float b0 = __uint_as_float(r1[i]), b1 = __uint_as_float(r1[i + 1]);
      if constexpr (kMasked) {
        if (c * 32 + i >= kv) a0 = -INFINITY;
        if (c * 32 + i + 1 >= kv) a1 = -INFINITY;
        if ((c + 1) * 32 + i >= kv) b0 = -INFINITY;
        if ((c + 1) * 32 + i + 1 >= kv) b1 = -INFINITY;
      }
      mx = fmax3f(mx, a0, a1);
      mx = fmax3f(mx, b0, b1);
    }
  }
  return mx;
}

// All exponentials on the MUFU: with the lazy max (no per-block exchange) all-MUFU measured
// fastest at c2 (1.431 ms vs 1.440 / 1.447 / 1.451 / 1.474 ms with one pair in 16 / 6 / 8 / 4
// on an FMA-pipe polynomial, round 1, tools/fwd_bench.py).
#ifndef DSV_P_CHUNKS
#define DSV_P_CHUNKS 2        // 32-column chunks loaded per TMEM wait in pass 2
#endif
// P for one 32-column chunk of raw scores: 2^(s*scale_log2 - m) (packed FMAs, MUFU ex2).
template <bool kMasked>
DSV_DEV void softmax_p_chunk(const uint32_t (&r)[32], uint32_t tdst, f32x2 sc2, f32x2 nm2, int c,
                             int kv, f32x2& lsum2) {
  uint32_t pk[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const f32x2 x = ffma2(f2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), sc2, nm2);
    const float2 xv = f2u(x);
    float2 p = make_float2(fast_exp2(xv.x), fast_exp2(xv.y));
    if constexpr (kMasked) {
      if (c * 32 + 2 * i >= kv) p.x = 0.f;
      if (c * 32 + 2 * i + 1 >= kv) p.y = 0.f;
    }
    lsum2 = fadd2(lsum2, f2(p.x, p.y));
    pk[i] = pack_bf16(p.x, p.y);
  }
  tmem_st16(tdst, pk);
}

// Softmax pass 2 over one S buffer: P = 2^(s*scale_log2 - m) (bf16) written over
// the S columns already read (chunk c -> columns [16c, 16c+16)); returns the row sum.
template <bool kMasked>
DSV_DEV float softmax_p_pass(uint32_t tS, float scale_log2, float m, int kv) {
  const f32x2 sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m, -m);
  f32x2 lsum2 = f2(0.f, 0.f);
#pragma unroll 1
  for (int c = 0; c < BKV / 32; c += DSV_P_CHUNKS) {
    uint32_t r0[32];
    tmem_ld32(tS + c * 32, r0);
    if constexpr (DSV_P_CHUNKS == 2) {
      uint32_t r1[32];
      tmem_ld32(tS + (c + 1) * 32, r1);
      tmem_ld_wait();
      softmax_p_chunk<kMasked>(r0, tS + c * 16, sc2, nm2, c, kv, lsum2);
      softmax_p_chunk<kMasked>(r1, tS + (c + 1) * 16, sc2, nm2, c + 1, kv, lsum2);
    } else {
      tmem_ld_wait();
      softmax_p_chunk<kMasked>(r0, tS + c * 16, sc2, nm2, c, kv, lsum2);
    }
  }
  const float2 l = f2u(lsum2);
  return l.x + l.y;
}

// Forward structure. All four softmax warpgroups work on every key block: warp w
// owns TMEM lanes 32 (w % 4).. (query rows) and key columns [32 (w / 4), +32), so a
// block's softmax is spread over 16 warps and the row max is exchanged through
// shared memory once per block. With one O accumulator the
// TMEM holds three S/P buffers, and the MMA issues S_{j+3} right after PV_j: the
// softmax of block j+1 never waits for PV_j to drain. O is rescaled (lazily, when
// the running max grows by > 2^8) only after PV_{j-1} has completed.
//
// Persistent CTAs: each CTA walks tiles blockIdx.x, +gridDim.x, ... with every role
// keeping running block counters, so the producers gather the next tile's Q and first
// K/V blocks and the MMA warp computes its first S blocks while the softmax warps finish
// the current tile (q_empty: every S of a tile has read Q; o_empty: the softmax epilogue
// has read O out of TMEM). Lazy max (below) flags a tile whose scores exceed its
// reference max by > 2^64 into ovf_list; the launcher re-runs those tiles with the exact
// per-block max in list mode (list = ovf_list, read after the first launch).
// Index-list row of a (head, tile): tiles are the 128-query pieces of the voxel groups; a group
// larger than 128 queries spans several tiles that share its row (tile_grp: tile -> group,
// nullptr = one tile per group), so idx / kcount_hg are [H, Gs, ...] over the Gs groups.
// Rows written to other ranks' buffers (HCP output redistribution fused into the kernels'
// epilogues): row (h, tok) of a [H, L, D] bf16 result goes to tab[h * n + tok / chunk] +
// (tok % chunk) * D — peer-mapped addresses of the token owners' regions. tab == nullptr:
// not used.
struct RowOut {
  const long long* tab;
  int n, chunk;
};
template <int D>
DSV_DEV __nv_bfloat16* row_out(const RowOut& ro, int h, int tok) {
  const int o = tok / ro.chunk;
  return reinterpret_cast<__nv_bfloat16*>(ro.tab[h * ro.n + o]) + (long long)(tok - o * ro.chunk) * D;
}

DSV_DEV long long sel_row(int tile, int G, const int* tile_grp, int Gs) {
  const int h = tile / G, g = tile - h * G;
  return (long long)h * Gs + (tile_grp ? __ldg(tile_grp + g) : g);
}

// Backward: the dK/dV fp32 -> bf16 conversion done by the persistent CTAs once the tile
// queue is exhausted (the kernel's tail, where CTAs would otherwise idle while the last
// tiles finish). head_done[h] counts the finished tiles of head h (scatter warps publish
// them after a fence); a CTA converts a slice of head h once all its tiles are done.
// head_done == nullptr: no conversion (the caller converts).
struct KvOut {
  __nv_bfloat16* dk;        // bf16 [H, Lk, D] (local outputs), or
  __nv_bfloat16* dv;
  RowOut dk_rows, dv_rows;  // row addresses at the token owners (tab != nullptr)
  int* head_done;           // [H] finished tiles per head; [H] = slice counter (zeroed)
  int H, tiles_per_head;
};
constexpr int kConvSlices = 32;   // conversion work items per head

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1)
sparse_fwd_kernel(const __nv_bfloat16* __restrict__ Qg, const __nv_bfloat16* __restrict__ Kg,
                  const __nv_bfloat16* __restrict__ Vg, const int* __restrict__ grp_rows,
                  const int* __restrict__ grp_size, const int* __restrict__ idx, long long ldk,
                  const int* __restrict__ kcount, const int* __restrict__ kcount_hg, int G,
                  int Lq, int Lk, float scale_log2, __nv_bfloat16* __restrict__ O,
                  float* __restrict__ lse, int n_tiles, const unsigned* __restrict__ list,
                  unsigned* __restrict__ ovf_list, unsigned* __restrict__ sched,
                  float4* __restrict__ zero_buf, long long zero_n4,
                  const int* __restrict__ tile_grp, int Gs, RowOut oremote) {
  using SL = FwdSmem<D>;
  using GT = Gather<D>;
  constexpr int ST = kFwdStages, KST = kFwdKStages, NS = kFwdSBufs;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = SL::kSlack ? aligned_smem(smem_raw) : smem_raw;
  if (!SL::kSlack && (smem_u32(smem_raw) & 1023u)) __trap();    // see FwdSmem
  FwdBars& B = *reinterpret_cast<FwdBars*>(smem + SL::kBar);
  uint8_t* sQ = smem + SL::kQ;
  uint8_t* sK = smem + SL::kK;
  uint8_t* sV = smem + SL::kV;
  float* sMax = reinterpret_cast<float*>(smem + SL::kMax);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work items: tiles blockIdx.x, +gridDim.x, ... of all n_tiles (lazy max), or in list
  // mode the flagged tiles list[1 + i] (exact per-block max)
  const bool list_mode = list != nullptr;
  const bool lazy = DSV_FWD_LAZY && !list_mode;
  const int n_work = list_mode ? (int)list[0] : n_tiles;
  if ((int)blockIdx.x >= n_work) return;                       // uniform
  // normal mode: tiles drawn from a global atomic counter (one producer lane feeds a
  // 2-slot shared-memory queue every thread reads; keeps the CTAs in step like the
  // hardware block scheduler); list mode: a static split of the flagged list
  auto tile_of = [&](int it) -> int {
    if (list_mode) {
      const long long i = (long long)blockIdx.x + (long long)it * gridDim.x;
      return i < n_work ? (int)list[1 + i] : -1;
    }
    const int slot = it & 1;
    mbar_wait(&B.tq_full[slot], (it >> 1) & 1);
    const int t = *reinterpret_cast<volatile int*>(&B.tq[slot]);
    mbar_arrive(&B.tq_empty[slot]);
    return t;
  };
  auto draw_tile = [&](int it) {
    if (list_mode) return;
    const int slot = it & 1;
    if (it >= 2) mbar_wait(&B.tq_empty[slot], ((it >> 1) - 1) & 1);
    const unsigned t = atomicAdd(sched, 1u);
    B.tq[slot] = t < (unsigned)n_tiles ? (int)t : -1;
    mbar_arrive(&B.tq_full[slot]);
  };

  auto init_bars = [&]() {
    mbar_init(&B.q_full, kProdThreads);
    mbar_init(&B.q_empty, 1);
    mbar_init(&B.o_empty, kFwdSoftThreads);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&B.tq_full[t], 1);
      mbar_init(&B.tq_empty[t], kFwdThreads);
    }
    for (int s = 0; s < KST; ++s) { mbar_init(&B.k_full[s], kProdThreads / 2); mbar_init(&B.k_empty[s], 1); }
    for (int s = 0; s < ST; ++s) { mbar_init(&B.v_full[s], kProdThreads / 2); mbar_init(&B.v_empty[s], 1); }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&B.s_full[s], 1);
      mbar_init(&B.p_full[s], kFwdSoftThreads);
      mbar_init(&B.pv_done[s], 1);
    }
    mbar_init(&B.o_final, 1);
    B.ovf = 0u;
    fence_barrier_init();
  };
  if (warp == kFwdMmaWarp) {
    if (lane == 0) init_bars();
    __syncwarp();
    tmem_alloc(&B.tmem, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;
  const uint32_t tS0 = tmem, tO = tmem + NS * 128;   // S/P buffer b at tS0 + 128 b

  // Lazy max: the row max is exchanged between the 16 softmax warps for key block 0
  // only; later blocks exponentiate against it without a barrier, each warp checking
  // that its scores stay within 2^64 of it (P, O and the row sums are fp32 / bf16 with
  // 2^127 range, and relative precision does not depend on the scale). A tile where some
  // score exceeds that is flagged for the exact pass (list mode), which exchanges the max
  // every block and rescales O when it grows by > 2^8.

  if (warp >= kFwdProdWarp0) {
    // ------------------------------------------------------------ producers
    // Two groups of 4 warps: one streams K tiles, the other V tiles, each through its
    // own 3-deep ring (K_j frees as soon as S_j is computed, so K runs ahead while V
    // waits for the PV products). cp.async copies arrive on the stage's "full"
    // barrier asynchronously (cp.async.mbarrier.arrive.noinc, one per thread).
    using GH = Gather<D, kProdThreads / 2>;
    const int ptid = threadIdx.x - kFwdProdWarp0 * 32;
    const bool is_v = ptid >= kProdThreads / 2;
    const int gtid = is_v ? ptid - kProdThreads / 2 : ptid;
    const int r0 = gtid / GH::kCPR;
    const __nv_bfloat16* src = is_v ? Vg : Kg;
    uint8_t* ring = is_v ? sV : sK;
    uint64_t* full = is_v ? B.v_full : B.k_full;
    uint64_t* empty = is_v ? B.v_empty : B.k_empty;
    const int nst = is_v ? ST : KST;
    int rows[GH::kPer];
    int kb = 0;                                      // blocks through this ring so far
    for (int it = 0;; ++it) {
      if (ptid == 0) draw_tile(it);
      const int tile = tile_of(it);
      if (tile < 0) break;
      const int h = tile / G, g = tile - h * G;
      const int kh = kcount_hg ? kcount_hg[sel_row(tile, G, tile_grp, Gs)] : kcount[h];
      const int nblk = (kh + BKV - 1) / BKV;
      const int* irow = idx + sel_row(tile, G, tile_grp, Gs) * ldk;
      const int* mrow = grp_rows + (long long)g * BQ;
      {   // Q of this tile, once every S of the previous tile has read the last one
        const int qr0 = ptid / GT::kCPR;
        int qrows[GT::kPer];
#pragma unroll
        for (int i = 0; i < GT::kPer; ++i) qrows[i] = h * Lq + __ldg(mrow + qr0 + i * GT::kRowStep);
        if (it > 0) mbar_wait(&B.q_empty, (it - 1) & 1);
        issue_tile<D>(sQ, Qg, qrows, ptid);
        cp_async_arrive_noinc(&B.q_full);
      }
      if (zero_buf != nullptr) {
        // zero this tile's share of the backward's dK/dV accumulators: HBM writes that
        // run under the gather-bound forward instead of a separate fill pass
        const long long per = (zero_n4 + n_tiles - 1) / n_tiles;
        const long long z0 = (long long)tile * per, z1 = min(zero_n4, z0 + per);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (long long i = z0 + ptid; i < z1; i += kProdThreads) zero_buf[i] = z;
      }
      const int kbase = h * Lk;
      for (int j = 0; j < nblk; ++j, ++kb) {
        const int st = kb % nst;
#pragma unroll
        for (int i = 0; i < GH::kPer; ++i)
          rows[i] = kbase + __ldg(irow + min(j * BKV + r0 + i * GH::kRowStep, kh - 1));
        if (kb >= nst) mbar_wait(&empty[st], ((kb / nst) - 1) & 1);
        if (gtid == 0) FPROF(j, is_v ? 6 : 5);
        issue_tile<D, kProdThreads / 2>(ring + st * SL::kTile, src, rows, gtid);
        cp_async_arrive_noinc(&full[st]);
      }
    }
    cp_async_wait<0>();
  } else if (warp == kFwdMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // order: S_0 S_1 S_2 PV_0 S_3 PV_1 S_4 ... (S_{j+3} reuses the buffer PV_j just read)
    constexpr uint32_t idS = idesc_bf16_f32(128, BKV, 0, 0);
    constexpr uint32_t idO = idesc_bf16_f32(128, D, 0, 1);
    const uint32_t aQ = smem_u32(sQ);
    int gb = 0;                                      // blocks of this CTA's earlier tiles
    for (int it = 0;; ++it) {
    const int tile = tile_of(it);
    if (tile < 0) break;
    const int h = tile / G;
    const int kh = kcount_hg ? kcount_hg[sel_row(tile, G, tile_grp, Gs)] : kcount[h];
    const int nblk = (kh + BKV - 1) / BKV;
    auto issue_s = [&](int s) {
      const int gs = gb + s, st = gs % KST;
      mbar_wait(&B.k_full[st], (gs / KST) & 1);
      tc_fence_after();
      if (lane == 0) FPROF(s, 0);
      if (elect_one()) {
        const uint32_t aK = smem_u32(sK + st * SL::kTile);
        const uint32_t dS = tS0 + (gs % NS) * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          mma_ss(dS, sdesc_sw128(aQ + off, 16, 1024), sdesc_sw128(aK + off, 16, 1024), idS, kk > 0);
        }
        mma_commit(&B.s_full[gs % NS]);
        mma_commit(&B.k_empty[st]);
        if (s == nblk - 1) mma_commit(&B.q_empty);   // the tile's last read of Q
      }
      __syncwarp();
    };
    mbar_wait(&B.q_full, it & 1);
    for (int s = 0; s < NS && s < nblk; ++s) issue_s(s);
    for (int j = 0; j < nblk; ++j) {
      const int gj = gb + j, st = gj % ST;
      mbar_wait(&B.p_full[gj % NS], (gj / NS) & 1);
      mbar_wait(&B.v_full[st], (gj / ST) & 1);
      if (j == 0 && it > 0) mbar_wait(&B.o_empty, (it - 1) & 1);   // O read out
      tc_fence_after();
      if (lane == 0) FPROF(j, 1);
      if (elect_one()) {
        const uint32_t aV = smem_u32(sV + st * SL::kTile);
        const uint32_t tP = tS0 + (gj % NS) * 128;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_ts(tO, tP + (kk >> 1) * 32 + (kk & 1) * 8, sdesc_sw128(aV + kk * 2048, 128 * 128, 1024),
                 idO, (j > 0 || kk > 0));   // P of keys [32c, +32) sits in S columns [32c, +16)
        mma_commit(&B.v_empty[st]);
        mma_commit(&B.pv_done[gj % NS]);
        if (j == nblk - 1) mma_commit(&B.o_final);
      }
      __syncwarp();
      if (j + NS < nblk) issue_s(j + NS);
    }
    gb += nblk;
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    // warp w: TMEM lanes 32 (w % 4).. (query rows), key columns [32 (w / 4), +32)
    const int cq = warp >> 2, wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    constexpr int kOc = D / kFwdSoftWGs;              // O columns per warp (rescale, store)
    int gb = 0;
    for (int it = 0;; ++it) {
    const int tile = tile_of(it);
    if (tile < 0) break;
    const int h = tile / G, g = tile - h * G;
    const int kh = kcount_hg ? kcount_hg[sel_row(tile, G, tile_grp, Gs)] : kcount[h];
    const int nblk = (kh + BKV - 1) / BKV;
    const int* mrow = grp_rows + (long long)g * BQ;
    float m_run = -INFINITY, l_run = 0.f;
    bool ovf_local = false;
    for (int j = 0; j < nblk; ++j) {
      const int gj = gb + j;
      const int kv = min(BKV, kh - j * BKV);
      const uint32_t tS = tS0 + (gj % NS) * 128 + lane_off;
      mbar_wait(&B.s_full[gj % NS], (gj / NS) & 1);
      tc_fence_after();
      if (warp == 0 && lane == 0) FPROF(j, 2);
      uint32_t r[32];
      tmem_ld32(tS + cq * 32, r);
      tmem_ld_wait();
      if (warp == 0 && lane == 0) FPROF(j, 7);
      float mx = -INFINITY;
      if (kv == BKV) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) mx = fmax3f(mx, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (cq * 32 + i < kv) mx = fmaxf(mx, __uint_as_float(r[i]));
      }
      if (lazy && j > 0) {
        // no exchange: this warp's 32 columns against the row's block-0 max
        ovf_local |= mx * scale_log2 > m_run + kLazyLimit;
      } else {
      // row max over the four column slices, through shared memory (one buffer: a
      // second barrier frees it before the next exchange)
      float* xch = sMax;
      xch[cq * 128 + row] = mx;
      if (warp == 0 && lane == 0) FPROF(j, 8);
      named_bar_sync(1, kFwdSoftThreads);
      mx = fmax3f(fmaxf(xch[row], xch[128 + row]), xch[256 + row], xch[384 + row]) * scale_log2;
      named_bar_sync(1, kFwdSoftThreads);
      if (warp == 0 && lane == 0) FPROF(j, 3);
      if (j == 0) {
        m_run = mx;
      } else if (__any_sync(0xffffffffu, mx > m_run + 8.f)) {
        // rescale O (this warp's D/4 columns) once PV_{j-1} has landed. The decision is
        // warp-uniform: tcgen05.ld/st are warp-collective, so every lane takes the branch
        // and a row whose max did not grow rescales by alpha = 1.
        mbar_wait(&B.pv_done[(gj - 1) % NS], ((gj - 1) / NS) & 1);
        tc_fence_after();
        mx = fmaxf(mx, m_run);
        const float alpha = fast_exp2(m_run - mx);
        l_run *= alpha;
#pragma unroll 1
        for (int c = cq * kOc; c < (cq + 1) * kOc; c += 16) {
          uint32_t o[16];
          tmem_ld16(tO + lane_off + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tO + lane_off + c, o);
        }
        m_run = mx;
      }
      }
      // P = 2^(s scale_log2 - m) for keys [32 cq, +32): bf16 into columns [32 cq, +16),
      // i.e. over this warp's own scores (already in registers) — no other warp reads
      // them, so the lazy-max blocks need no barrier at all
      const f32x2 sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m_run, -m_run);
      f32x2 lsum2 = f2(0.f, 0.f);
      if (kv == BKV) softmax_p_chunk<false>(r, tS + cq * 32, sc2, nm2, cq, kv, lsum2);
      else softmax_p_chunk<true>(r, tS + cq * 32, sc2, nm2, cq, kv, lsum2);
      const float2 ls = f2u(lsum2);
      l_run += ls.x + ls.y;
      if (warp == 0 && lane == 0) FPROF(j, 9);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&B.p_full[gj % NS]);
      if (warp == 0 && lane == 0) FPROF(j, 4);
    }
    // ---------------- epilogue: combine the slices' row sums, normalise, store
    mbar_wait(&B.o_final, it & 1);
    tc_fence_after();
    float* lx = sMax;
    if (__any_sync(0xffffffffu, ovf_local) && lane == 0) B.ovf = 1u;
    named_bar_sync(1, kFwdSoftThreads);
    lx[cq * 128 + row] = l_run;
    named_bar_sync(1, kFwdSoftThreads);
    const float denom = (lx[row] + lx[128 + row]) + (lx[256 + row] + lx[384 + row]);
    if (threadIdx.x == 0 && B.ovf) {                 // flag the tile for the exact pass
      B.ovf = 0u;
      ovf_list[1 + atomicAdd(ovf_list, 1u)] = (unsigned)tile;
    }
    named_bar_sync(1, kFwdSoftThreads);               // sMax / flag free for the next tile
    const float inv = denom > 0.f ? 1.f / denom : 0.f;
    const int gsz = grp_size[g];
    const int tok = mrow[row];
    __nv_bfloat16* orow = O + ((long long)h * Lq + tok) * D;
    __nv_bfloat16* rrow = oremote.tab ? row_out<D>(oremote, h, tok) : nullptr;
#pragma unroll 1
    for (int c = cq * kOc; c < (cq + 1) * kOc; c += 16) {
      uint32_t o[16];
      tmem_ld16(tO + lane_off + c, o);
      tmem_ld_wait();
      if (row < gsz) {
#pragma unroll
        for (int i = 0; i < 16; i += 8) {
          const uint4 pk =
              make_uint4(pack_bf16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv),
                         pack_bf16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv),
                         pack_bf16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv),
                         pack_bf16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv));
          *reinterpret_cast<uint4*>(orow + c + i) = pk;
          if (rrow) *reinterpret_cast<uint4*>(rrow + c + i) = pk;   // the token owner (NVLink)
        }
      }
    }
    if (cq == 0 && row < gsz) lse[(long long)h * Lq + tok] = m_run + __log2f(denom);
    tc_fence_before();
    mbar_arrive(&B.o_empty);                          // O is out of TMEM
    gb += nblk;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFwdMmaWarp) tmem_dealloc(tmem, 512);
}

// ====================================================================== bwd
// Per KV block j (keys in TMEM lanes; TMEM columns: tA | tB | tC | tDq):
//   A_j  MMA   S^T = K_j Q^T -> tA, dP^T = V_j dO^T -> tB            (V_j free after)
//   B_j  work  P^T, dS^T (bf16) -> tC[0,64), tC[64,128); dS -> smem (MN-major)
//   C_j  MMA   dQ += dS K_j -> tDq (K_j free), dV_j = P^T dO -> tA, dK_j = dS^T Q -> tB
//   C'_j work  dV_j -> staging half 0, dK_j -> staging half 1 (bf16); TMEM is released
//              as soon as both are in registers
//   D_j  scat  staging -> coalesced red.global.add.v4.f32 into the fp32 accumulators
// The fp32 adds into L2 (~5.5 TB/s on B200, measured for both red.v4 and TMA bulk
// reductions) bound the backward on random selections: 128 KB of adds per block.
// So the scatter warps only scatter — loads have their own warps — and each staging
// half is freed on its own, which keeps the reduction stream busy while A..C' of
// the next block run underneath it.
// Staging rounds each per-block contribution to bf16 like P and dS already are;
// the accumulation itself stays fp32.
#ifndef DSV_BWD_WORK_WARPS
#define DSV_BWD_WORK_WARPS 16
#endif
constexpr int kBwdWork = DSV_BWD_WORK_WARPS;        // multiple of 4 (TMEM lane quarters)
constexpr int kBwdWPQ = kBwdWork / 4;              // worker warps per lane quarter
constexpr int kBwdWorkThreads = kBwdWork * 32;
constexpr int kBwdMmaWarp = kBwdWork;
constexpr int kBwdLoadWarp0 = kBwdWork + 1;
constexpr int kBwdLoadWarps = 2;
constexpr int kBwdLoadThreads = kBwdLoadWarps * 32;
constexpr int kBwdScatWarp0 = kBwdLoadWarp0 + kBwdLoadWarps;
#ifndef DSV_BWD_SCAT_WARPS
#define DSV_BWD_SCAT_WARPS 8
#endif
constexpr int kBwdScatWarps = DSV_BWD_SCAT_WARPS;
static_assert(kBwdWork % 4 == 0 && 128 % kBwdScatWarps == 0,
              "worker warps: a multiple of 4 (TMEM lane quarters); scatter warps divide 128 rows");
constexpr int kBwdScatThreads = kBwdScatWarps * 32;
constexpr int kBwdThreads = (kBwdScatWarp0 + kBwdScatWarps) * 32;   // 864 by default


template <int D>
struct BwdSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kdO = kQ + kTile;
  static constexpr int kdS = kdO + kTile;                 // [128 keys][128 q] bf16 (MN-major A)
  static constexpr int kK = kdS + 128 * 128 * 2;
  static constexpr int kV = kK + kTile;
  static constexpr int kStg = kV + kTile;                 // [2 halves][128 rows][D] bf16
  static constexpr int kLse = kStg + 2 * 128 * D * 2;
  static constexpr int kDelta = kLse + 512;
  static constexpr int kBar = kDelta + 512;
  static constexpr int kBytes = kBar + 256 + 1024;
  static_assert(kBytes <= 232448, "backward shared memory over 227 KB");
};

struct BwdBars {
  uint64_t q_full, k_full, v_full, k_empty, v_empty;
  uint64_t sdp_full, pds_full, mma_done, tmem_free;
  uint64_t q_empty, dq_empty;                             // persistent CTAs: Q/dO, dQ free
  uint64_t tq_full[4], tq_empty[4];                       // tile-id queue (dynamic schedule)
  int tq[4];
  uint64_t stg_full[2], stg_free[2];                      // [0] = dV half, [1] = dK half
  uint32_t tmem;
};
static_assert(sizeof(BwdBars) <= 256, "backward barriers over their 256 B");

// byte offset of 16-byte chunk q of staging row p (rows of D bf16, XOR-swizzled)
template <int D>
DSV_DEV uint32_t stg_off(int p, int q) {
  constexpr int kC = D / 8;   // chunks per row
  return (uint32_t)(p * (D * 2) + ((q ^ (p & (kC - 1))) << 4));
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
sparse_bwd_kernel(const __nv_bfloat16* __restrict__ Qg, const __nv_bfloat16* __restrict__ dOg,
                  const __nv_bfloat16* __restrict__ Kg, const __nv_bfloat16* __restrict__ Vg,
                  const __nv_bfloat16* __restrict__ Og, const float* __restrict__ lse,
                  const int* __restrict__ grp_rows, const int* __restrict__ grp_size,
                  const int* __restrict__ idx, long long ldk, const int* __restrict__ kcount,
                  const int* __restrict__ kcount_hg, int G, int Lq, int Lk, float scale,
                  float scale_log2,
                  __nv_bfloat16* __restrict__ dQ, float* __restrict__ dK, float* __restrict__ dV,
                  int n_tiles, unsigned* __restrict__ sched, const int* __restrict__ tile_grp,
                  int Gs, RowOut dqremote, KvOut kv) {
  using SL = BwdSmem<D>;
  using GT = Gather<D, kBwdLoadThreads>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  BwdBars& B = *reinterpret_cast<BwdBars*>(smem + SL::kBar);
  uint8_t* sQ = smem + SL::kQ;
  uint8_t* sdO = smem + SL::kdO;
  uint8_t* sdS = smem + SL::kdS;
  uint8_t* sK = smem + SL::kK;
  uint8_t* sV = smem + SL::kV;
  uint8_t* sStg = smem + SL::kStg;
  float* sLse = reinterpret_cast<float*>(smem + SL::kLse);
  float* sDelta = reinterpret_cast<float*>(smem + SL::kDelta);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kCh = D / 32;                              // 32-column chunks per tensor
  // persistent CTAs: tiles blockIdx.x, +gridDim.x, ...; every role keeps running block
  // counters (gj) for the barrier parities, so the next tile's Q/dO and first K/V loads
  // and its first MMAs overlap the current tile's last blocks and dQ epilogue
  // Tiles are handed out dynamically (a global atomic counter, like the hardware block
  // scheduler): with a static round-robin split the CTAs drift apart over their ~40
  // tiles, more heads' dK/dV accumulators are live at once and fall out of L2. One
  // producer lane draws the ids into a 4-slot shared queue that every thread reads.
  auto tile_of = [&](int it) -> int {
    const int slot = it & 3;
    mbar_wait(&B.tq_full[slot], (it >> 2) & 1);
    const int t = *reinterpret_cast<volatile int*>(&B.tq[slot]);
    mbar_arrive(&B.tq_empty[slot]);
    return t;
  };
  auto draw_tile = [&](int it) {                   // the scheduler lane, ahead of everyone
    const int slot = it & 3;
    if (it >= 4) mbar_wait(&B.tq_empty[slot], ((it >> 2) - 1) & 1);
    const unsigned t = atomicAdd(sched, 1u);
    B.tq[slot] = t < (unsigned)n_tiles ? (int)t : -1;
    mbar_arrive(&B.tq_full[slot]);                  // release: the id is visible to waiters
  };
#define DSV_BWD_TILE()                                                    \
    const int tile = tile_of(it);                                           \
    if (tile < 0) break;                                                    \
    const int h = tile / G, g = tile - h * G;                               \
    const int kh = kcount_hg ? kcount_hg[sel_row(tile, G, tile_grp, Gs)] : kcount[h];                 \
    const int nblk = (kh + BKV - 1) / BKV;                                  \
    const int* irow = idx + sel_row(tile, G, tile_grp, Gs) * ldk;                   \
    const int* mrow = grp_rows + (long long)g * BQ;                         \
    (void)irow; (void)mrow; (void)nblk

  if (warp == kBwdMmaWarp) {
    if (lane == 0) {
      mbar_init(&B.q_full, kBwdLoadThreads);
      mbar_init(&B.k_full, kBwdLoadThreads);
      mbar_init(&B.v_full, kBwdLoadThreads);
      mbar_init(&B.k_empty, 1);
      mbar_init(&B.v_empty, 1);
      mbar_init(&B.sdp_full, 1);
      mbar_init(&B.pds_full, kBwdWorkThreads);
      mbar_init(&B.mma_done, 1);
      mbar_init(&B.tmem_free, kBwdWorkThreads);
      mbar_init(&B.q_empty, 1);
      mbar_init(&B.dq_empty, kBwdWorkThreads);
      for (int t = 0; t < 4; ++t) {
        mbar_init(&B.tq_full[t], 1);
        mbar_init(&B.tq_empty[t], kBwdThreads);
      }
      for (int t = 0; t < 2; ++t) {
        mbar_init(&B.stg_full[t], kBwdWorkThreads);   // every worker, once per half
        mbar_init(&B.stg_free[t], kBwdScatThreads);
      }
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&B.tmem, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;
  const uint32_t tA = tmem, tB = tmem + 128, tC = tmem + 256, tDq = tmem + 384;

  if (warp >= kBwdScatWarp0) {
    // ------------------------------------------------------------ scatter
    constexpr int RPW = 128 / kBwdScatWarps;        // staging rows per scatter warp
    const int pw = warp - kBwdScatWarp0;            // rows [RPW pw, RPW pw + RPW)
    const int stid = threadIdx.x - kBwdScatWarp0 * 32;
    int gj = 0;
    int prev_h = -1, pending = 0;
    // publish the finished tiles of head prev_h: every scatter thread's reductions are
    // performed (fence), then one release add (the tail conversion acquires it)
    auto flush = [&]() {
      __threadfence();
      named_bar_sync(2, kBwdScatThreads);
      if (stid == 0) red_release_add(kv.head_done + prev_h, pending);
      pending = 0;
    };
    for (int it = 0;; ++it) {
    DSV_BWD_TILE();
    if (kv.head_done != nullptr && prev_h >= 0 && h != prev_h) flush();
    prev_h = h;
    const long long hoff = (long long)h * Lk * D;
    for (int jb = 0; jb < nblk; ++jb, ++gj) {
      const int kv = min(BKV, kh - jb * BKV);
      const int myrow = pw * RPW + (lane % RPW);
      const int mykey = myrow < kv ? __ldg(irow + jb * BKV + myrow) : 0;
#pragma unroll 1
      for (int t = 0; t < 2; ++t) {
        mbar_wait(&B.stg_full[t], gj & 1);
        if (stid == 0) PROF(jb, 8 + t);
        float* acc = (t == 0 ? dV : dK) + hoff;
        const uint8_t* stg = sStg + t * (128 * D * 2);
        if constexpr (D == 128) {
#pragma unroll 4
          for (int rr = 0; rr < RPW; ++rr) {
            const int p = pw * RPW + rr;
            const int key = __shfl_sync(0xffffffffu, mykey, rr);
            if (p < kv) {
              const uint2 v = *reinterpret_cast<const uint2*>(stg + stg_off<D>(p, lane >> 1) + (lane & 1) * 8);
              red_add_v4(acc + (long long)key * D + lane * 4, bf16lo(v.x), bf16hi(v.x),
                         bf16lo(v.y), bf16hi(v.y));
            }
          }
        } else {
#pragma unroll 4
          for (int rr = 0; rr < RPW; rr += 2) {
            const int p = pw * RPW + rr + (lane >> 4);
            const int key = __shfl_sync(0xffffffffu, mykey, rr + (lane >> 4));
            if (p < kv) {
              const int e = (lane & 15) * 4;
              const uint2 v = *reinterpret_cast<const uint2*>(stg + stg_off<D>(p, e >> 3) + ((e >> 2) & 1) * 8);
              red_add_v4(acc + (long long)key * D + e, bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y));
            }
          }
        }
        mbar_arrive(&B.stg_free[t]);
      }
      if (stid == 0) PROF(jb, 10);
    }
    ++pending;
    }
    if (kv.head_done != nullptr && pending > 0) flush();
  } else if (warp >= kBwdLoadWarp0) {
    // ------------------------------------------------------------ gather producers
    const int ptid = threadIdx.x - kBwdLoadWarp0 * 32;
    const int r0 = ptid / GT::kCPR;
    int rows[GT::kPer];
    int gj = 0;
    for (int it = 0;; ++it) {
    if (ptid == 0) draw_tile(it);
    DSV_BWD_TILE();
    const int qbase = h * Lq;
#pragma unroll
    for (int i = 0; i < GT::kPer; ++i) rows[i] = qbase + __ldg(mrow + r0 + i * GT::kRowStep);
    if (it > 0) mbar_wait(&B.q_empty, (it - 1) & 1);   // the previous tile's MMAs are done with Q/dO
    issue_tile<D, kBwdLoadThreads>(sQ, Qg, rows, ptid);
    issue_tile<D, kBwdLoadThreads>(sdO, dOg, rows, ptid);
    cp_async_arrive_noinc(&B.q_full);
    const int kbase = h * Lk;
    for (int j = 0; j < nblk; ++j, ++gj) {
#pragma unroll
      for (int i = 0; i < GT::kPer; ++i)
        rows[i] = kbase + __ldg(irow + min(j * BKV + r0 + i * GT::kRowStep, kh - 1));
      if (gj > 0) mbar_wait(&B.v_empty, (gj - 1) & 1);
      if (ptid == 0) PROF(j, 0);
      issue_tile<D, kBwdLoadThreads>(sV, Vg, rows, ptid);
      cp_async_arrive_noinc(&B.v_full);
      if (gj > 0) mbar_wait(&B.k_empty, (gj - 1) & 1);
      if (ptid == 0) PROF(j, 1);
      issue_tile<D, kBwdLoadThreads>(sK, Kg, rows, ptid);
      cp_async_arrive_noinc(&B.k_full);
    }
    }
    cp_async_wait<0>();
  } else if (warp == kBwdMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idST = idesc_bf16_f32(128, 128, 0, 0);   // K_j . Q^T, V_j . dO^T
    constexpr uint32_t idTS = idesc_bf16_f32(128, D, 0, 1);     // P^T|dS^T (tmem) . dO|Q (MN)
    constexpr uint32_t idDQ = idesc_bf16_f32(128, D, 1, 1);     // dS(MN smem) . K_j(MN)
    const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), adS = smem_u32(sdS);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    int gj = 0;
    for (int it = 0;; ++it) {
    DSV_BWD_TILE();
    mbar_wait(&B.q_full, it & 1);
    for (int j = 0; j < nblk; ++j, ++gj) {
      mbar_wait(&B.k_full, gj & 1);
      mbar_wait(&B.v_full, gj & 1);
      if (gj > 0) mbar_wait(&B.tmem_free, (gj - 1) & 1);
      tc_fence_after();
      if (lane == 0) PROF(j, 2);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          mma_ss(tA, sdesc_sw128(aK + off, 16, 1024), sdesc_sw128(aQ + off, 16, 1024), idST, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          mma_ss(tB, sdesc_sw128(aV + off, 16, 1024), sdesc_sw128(adO + off, 16, 1024), idST, kk > 0);
        }
        mma_commit(&B.sdp_full);
        mma_commit(&B.v_empty);
      }
      __syncwarp();
      mbar_wait(&B.pds_full, gj & 1);
      if (j == 0 && it > 0) mbar_wait(&B.dq_empty, (it - 1) & 1);   // dQ read out of TMEM
      tc_fence_after();
      if (lane == 0) PROF(j, 3);
      if (elect_one()) {
        // dQ += dS K_j    (A = dS MN-major in smem, B = K_j MN-major)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tDq, sdesc_sw128(adS + kk * 2048, 128 * 128, 1024),
                 sdesc_sw128(aK + kk * 2048, 128 * 128, 1024), idDQ, (j | kk) != 0);
        mma_commit(&B.k_empty);
        // dV_j = P^T dO -> tA, dK_j = dS^T Q -> tB  (A from TMEM, K = 128 queries)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tA, tC + kk * 8, sdesc_sw128(adO + kk * 2048, 128 * 128, 1024), idTS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tB, tC + 64 + kk * 8, sdesc_sw128(aQ + kk * 2048, 128 * 128, 1024), idTS, kk > 0);
        mma_commit(&B.mma_done);
        if (j == nblk - 1) mma_commit(&B.q_empty);     // the tile's last read of Q / dO
      }
      __syncwarp();
    }
    }
  } else {
    // ------------------------------------------------------------ workers
    const int quarter = warp & 3, cg = warp >> 2;   // TMEM lane quarter, 32-column slice
    const int row = quarter * 32 + lane;            // query row (prologue/epilogue), key row (blocks)
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int gj = 0;
    for (int it = 0;; ++it) {
    DSV_BWD_TILE();
    const int gsz = grp_size[g];
    const int tok = mrow[row];
    if (it > 0) named_bar_sync(1, kBwdWorkThreads);   // every worker is past the last tile
    if (cg == 0) {
      // prologue: lse2 and Delta = rowsum(dO * O) for this query row
      float dlt = 0.f, l2 = INFINITY;
      if (row < gsz) {
        const uint4* o4 = reinterpret_cast<const uint4*>(Og + ((long long)h * Lq + tok) * D);
        const uint4* d4 = reinterpret_cast<const uint4*>(dOg + ((long long)h * Lq + tok) * D);
#pragma unroll 4
        for (int i = 0; i < D / 8; ++i) {
          const uint4 a = __ldg(o4 + i), b = __ldg(d4 + i);
          dlt += bf16lo(a.x) * bf16lo(b.x) + bf16hi(a.x) * bf16hi(b.x);
          dlt += bf16lo(a.y) * bf16lo(b.y) + bf16hi(a.y) * bf16hi(b.y);
          dlt += bf16lo(a.z) * bf16lo(b.z) + bf16hi(a.z) * bf16hi(b.z);
          dlt += bf16lo(a.w) * bf16lo(b.w) + bf16hi(a.w) * bf16hi(b.w);
        }
        l2 = lse[(long long)h * Lq + tok];
      }
      sLse[row] = l2;
      sDelta[row] = dlt * scale;                    // dS = P (dP scale - Delta scale)
    }
    named_bar_sync(1, kBwdWorkThreads);
    // staging of one 32-column chunk (fp32 registers -> bf16 staging row)
    auto stage = [&](const uint32_t (&r)[32], int t, int c) {
      uint8_t* srow = sStg + t * (128 * D * 2);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(srow + stg_off<D>(row, c * 4 + q)) = make_uint4(
            pack_bf16(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1])),
            pack_bf16(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3])),
            pack_bf16(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5])),
            pack_bf16(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7])));
    };
    for (int j = 0; j < nblk; ++j, ++gj) {
      const int kv = min(BKV, kh - j * BKV);
      const bool kvalid = row < kv;
      mbar_wait(&B.sdp_full, gj & 1);
      tc_fence_after();
      if (threadIdx.x == 0) PROF(j, 4);
      // ---- B: 16-query halves of this warp's 32-query slices, for its 32 keys
#pragma unroll 1
      for (int hs = cg * 2; hs < 8; hs += 2 * kBwdWPQ) {
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        const int q0 = (hs + hf) * 16;
        uint32_t rs[16], rd[16];
        tmem_ld16(tA + lane_off + q0, rs);
        tmem_ld16(tB + lane_off + q0, rd);
        tmem_ld_wait();
        uint32_t pp[8], dd[8];
        if (kvalid) {
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float4 l = *reinterpret_cast<const float4*>(sLse + q0 + 2 * i);
            const float4 dl = *reinterpret_cast<const float4*>(sDelta + q0 + 2 * i);
            const float p0 = fast_exp2(fmaf(__uint_as_float(rs[2 * i]), scale_log2, -l.x));
            const float p1 = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 1]), scale_log2, -l.y));
            const float p2 = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 2]), scale_log2, -l.z));
            const float p3 = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 3]), scale_log2, -l.w));
            pp[i] = pack_bf16(p0, p1);
            pp[i + 1] = pack_bf16(p2, p3);
            dd[i] = pack_bf16(p0 * fmaf(__uint_as_float(rd[2 * i]), scale, -dl.x),
                              p1 * fmaf(__uint_as_float(rd[2 * i + 1]), scale, -dl.y));
            dd[i + 1] = pack_bf16(p2 * fmaf(__uint_as_float(rd[2 * i + 2]), scale, -dl.z),
                                  p3 * fmaf(__uint_as_float(rd[2 * i + 3]), scale, -dl.w));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) pp[i] = dd[i] = 0u;
        }
        tmem_st8(tC + lane_off + (q0 >> 1), pp);
        tmem_st8(tC + 64 + lane_off + (q0 >> 1), dd);
        // dS row (this key) into the MN-major dS tile: atom q0/64, 16-byte chunks
        uint8_t* base = sdS + (q0 >> 6) * (128 * 128);
        const int ch = (q0 & 63) >> 3;
        *reinterpret_cast<uint4*>(base + sw128_off(row, ch)) = make_uint4(dd[0], dd[1], dd[2], dd[3]);
        *reinterpret_cast<uint4*>(base + sw128_off(row, ch + 1)) = make_uint4(dd[4], dd[5], dd[6], dd[7]);
      }
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&B.pds_full);
      if (threadIdx.x == 0) PROF(j, 5);
      // ---- C': dV_j | dK_j 32-column chunks -> bf16 staging halves. Tasks n = cg,
      // cg + WPQ, ... of the 2 * kCh per quarter (t = n / kCh, chunk n % kCh); TMEM is
      // released after the last TMEM read, before that chunk is staged.
      mbar_wait(&B.mma_done, gj & 1);
      tc_fence_after();
      if (threadIdx.x == 0) PROF(j, 6);
      int cur_t = 0;
#pragma unroll 1
      for (int n = cg; n < 2 * kCh; n += kBwdWPQ) {
        const int t = n / kCh, c = n % kCh;
        uint32_t r[32];
        tmem_ld32((t == 0 ? tA : tB) + lane_off + c * 32, r);
        tmem_ld_wait();
        if (n + kBwdWPQ >= 2 * kCh) {
          tc_fence_before();
          mbar_arrive(&B.tmem_free);                // last TMEM read of this block
          if (threadIdx.x == 0) PROF(j, 7);
        }
        if (t != cur_t) { mbar_arrive(&B.stg_full[0]); cur_t = 1; }
        if (n - kBwdWPQ < 0 || (n - kBwdWPQ) / kCh != t) {
          if (gj > 0) mbar_wait(&B.stg_free[t], (gj - 1) & 1);   // first chunk of half t
        }
        stage(r, t, c);
      }
      if (cur_t == 0) mbar_arrive(&B.stg_full[0]);
      mbar_arrive(&B.stg_full[1]);
    }
    // ---------------- dQ epilogue (query rows); the last mma_done covered dQ
    __nv_bfloat16* qrow = dqremote.tab ? row_out<D>(dqremote, h, tok)   // the token owner
                                       : dQ + ((long long)h * Lq + tok) * D;
#pragma unroll 1
    for (int c = cg; c < D / 32; c += kBwdWPQ) {
      uint32_t r[32];
      tmem_ld32(tDq + lane_off + c * 32, r);
      tmem_ld_wait();
      if (row < gsz) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(qrow + c * 32 + i) = make_uint4(
              pack_bf16(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
              pack_bf16(__uint_as_float(r[i + 2]), __uint_as_float(r[i + 3])),
              pack_bf16(__uint_as_float(r[i + 4]), __uint_as_float(r[i + 5])),
              pack_bf16(__uint_as_float(r[i + 6]), __uint_as_float(r[i + 7])));
      }
    }
    tc_fence_before();
    mbar_arrive(&B.dq_empty);                          // dQ is out of TMEM
    }
  }
#undef DSV_BWD_TILE
  tc_fence_before();
  __syncthreads();
  if (warp == kBwdMmaWarp) tmem_dealloc(tmem, 512);
  if (kv.head_done == nullptr) return;
  // ---- tail: convert dK / dV slices of finished heads (items handed out in head order)
  volatile int* s_item = reinterpret_cast<volatile int*>(sLse);
  const int total = kv.H * kConvSlices;
  const int rps = (Lk + kConvSlices - 1) / kConvSlices;
  constexpr int kC4 = D / 4;
  for (;;) {
    if (threadIdx.x == 0) {
      const int item = atomicAdd(kv.head_done + kv.H, 1);
      if (item < total) {
        const int* done = kv.head_done + item / kConvSlices;
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_gpu(done) < kv.tiles_per_head) {
          __nanosleep(256);
          if (globaltimer_ns() - t0 > 4000000000ull) __trap();   // watchdog
        }
      }
      *s_item = item;
    }
    __syncthreads();
    const int item = *s_item;
    __syncthreads();
    if (item >= total) break;
    const int hh = item / kConvSlices, sl = item - hh * kConvSlices;
    const int r0 = sl * rps, r1 = min(Lk, r0 + rps);
    const long long base = (long long)hh * Lk * D;
    for (int i = threadIdx.x; i < (r1 - r0) * kC4; i += kBwdThreads) {
      const int row = r0 + i / kC4, c = (i % kC4) * 4;
      const float4 a = __ldcg(reinterpret_cast<const float4*>(dK + base + (long long)row * D + c));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(dV + base + (long long)row * D + c));
      __nv_bfloat16* ok = kv.dk_rows.tab ? row_out<D>(kv.dk_rows, hh, row) : kv.dk + base + (long long)row * D;
      __nv_bfloat16* ov = kv.dv_rows.tab ? row_out<D>(kv.dv_rows, hh, row) : kv.dv + base + (long long)row * D;
      *reinterpret_cast<uint2*>(ok + c) = make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w));
      *reinterpret_cast<uint2*>(ov + c) = make_uint2(pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
    }
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   long long n) {
  long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(in + i);
    *reinterpret_cast<uint2*>(out + i) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  } else {
    for (; i < n; ++i) out[i] = __float2bfloat16_rn(in[i]);
  }
}

// fp32 [H, L, D] rows -> bf16 rows at their token owners (RowOut), one warp per row (D = 64
// or 128: 2 or 4 floats per lane).
template <int D>
__global__ void f32_to_bf16_rows_kernel(const float* __restrict__ in, long long rows, int L,
                                        RowOut out) {
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int h = (int)(r / L), tok = (int)(r - (long long)h * L);
  __nv_bfloat16* dst = row_out<D>(out, h, tok);
  if constexpr (D == 128) {
    const float4 v = reinterpret_cast<const float4*>(in + r * D)[lane];
    reinterpret_cast<uint2*>(dst)[lane] = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  } else {
    const float2 v = reinterpret_cast<const float2*>(in + r * D)[lane];
    reinterpret_cast<uint32_t*>(dst)[lane] = pack_bf16(v.x, v.y);
  }
}

}  // namespace attn
}  // namespace dsv

using namespace dsv::attn;

template <int D>
static int fwd_launch(const void* q, const void* k, const void* v, const int* grp_rows,
                      const int* grp_size, const int* idx, long long ldk, const int* kcount,
                      const int* kcount_hg, int H, int G, int Lq, int Lk, float scale_log2, void* O,
                      float* lse, unsigned* work, float* zero_buf, long long zero_floats,
                      const int* tile_grp, int Gs, RowOut oremote, cudaStream_t st) {
  auto kern = sparse_fwd_kernel<D>;
  const int smem = FwdSmem<D>::kBytes;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int n_tiles = H * G;
  // persistent grid: one CTA per SM (DSV_FWD_GRID=tiles: one CTA per tile, same kernel)
  static const bool per_tile = [] {
    const char* e = getenv("DSV_FWD_GRID");
    return e && e[0] == 't';
  }();
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = per_tile ? n_tiles : (n_tiles < sms ? n_tiles : sms);
  unsigned* sched = work + n_tiles + 1;              // tile counter after the flag list
  cudaMemsetAsync(work, 0, sizeof(unsigned), st);
  cudaMemsetAsync(sched, 0, sizeof(unsigned), st);
  kern<<<grid, kFwdThreads, smem, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                     (const __nv_bfloat16*)v, grp_rows, grp_size, idx, ldk,
                                     kcount, kcount_hg, G, Lq, Lk, scale_log2,
                                     (__nv_bfloat16*)O, lse, n_tiles, nullptr, work, sched,
                                     reinterpret_cast<float4*>(zero_buf), zero_floats / 4,
                                     tile_grp, Gs, oremote);
  // tiles flagged by the lazy max: exact per-block max (CTAs exit at once when none)
  const int g2 = n_tiles < sms ? n_tiles : sms;
  kern<<<g2, kFwdThreads, smem, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                   (const __nv_bfloat16*)v, grp_rows, grp_size, idx, ldk,
                                   kcount, kcount_hg, G, Lq, Lk, scale_log2,
                                   (__nv_bfloat16*)O, lse, n_tiles, work, nullptr, nullptr,
                                   nullptr, 0, tile_grp, Gs, oremote);
  return (int)cudaGetLastError();
}

int dsv_attn_fwd_tc_launch(const void* q, const void* k, const void* v, const int* grp_rows,
                           const int* grp_size, const int* idx, long long ldk, const int* kcount,
                           const int* kcount_hg, int H, int G, int Lq, int Lk, int D,
                           float scale_log2, void* O, float* lse, unsigned* work,
                           float* zero_buf, long long zero_floats, const int* tile_grp, int Gs,
                           const long long* o_tab, int o_n, int o_chunk, cudaStream_t st) {
  const RowOut ro{o_tab, o_n, o_chunk};
  if (D == 128)
    return fwd_launch<128>(q, k, v, grp_rows, grp_size, idx, ldk, kcount, kcount_hg, H, G, Lq, Lk,
                           scale_log2, O, lse, work, zero_buf, zero_floats, tile_grp, Gs, ro, st);
  if (D == 64)
    return fwd_launch<64>(q, k, v, grp_rows, grp_size, idx, ldk, kcount, kcount_hg, H, G, Lq, Lk,
                          scale_log2, O, lse, work, zero_buf, zero_floats, tile_grp, Gs, ro, st);
  return 1;
}

template <int D>
static int bwd_launch(const void* q, const void* k, const void* v, const void* O, const void* dO,
                      const float* lse, const int* grp_rows, const int* grp_size, const int* idx,
                      long long ldk, const int* kcount, const int* kcount_hg, int H, int G, int Lq,
                      int Lk, float scale,
                      float scale_log2, void* dQ, float* dK, float* dV, unsigned* sched,
                      const int* tile_grp, int Gs, RowOut dqremote, KvOut kv, cudaStream_t st) {
  auto kern = sparse_bwd_kernel<D>;
  const int smem = BwdSmem<D>::kBytes;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int n_tiles = H * G;
  static const bool per_tile = [] {          // DSV_BWD_GRID=tiles: one CTA per tile
    const char* e = getenv("DSV_BWD_GRID");
    return e && e[0] == 't';
  }();
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = per_tile ? n_tiles : (n_tiles < sms ? n_tiles : sms);
  cudaMemsetAsync(sched, 0, sizeof(unsigned), st);
  if (kv.head_done != nullptr) {
    kv.H = H;
    kv.tiles_per_head = G;
    cudaMemsetAsync(kv.head_done, 0, (H + 1) * sizeof(int), st);
  }
  kern<<<grid, kBwdThreads, smem, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)dO,
                                      (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
                                      (const __nv_bfloat16*)O, lse, grp_rows, grp_size, idx, ldk,
                                      kcount, kcount_hg, G, Lq, Lk, scale, scale_log2,
                                      (__nv_bfloat16*)dQ, dK, dV, n_tiles, sched, tile_grp, Gs,
                                      dqremote, kv);
  return (int)cudaGetLastError();
}

int dsv_attn_bwd_tc_launch(const void* q, const void* k, const void* v, const void* O,
                           const void* dO, const float* lse, const int* grp_rows,
                           const int* grp_size, const int* idx, long long ldk, const int* kcount,
                           const int* kcount_hg, int H, int G, int Lq, int Lk, int D, float scale,
                           float scale_log2, void* dQ, float* dK, float* dV, unsigned* sched,
                           const int* tile_grp, int Gs, const long long* dq_tab, int dq_n,
                           int dq_chunk, void* dkdv_out, const long long* dk_tab,
                           const long long* dv_tab, int kv_n, int kv_chunk, int* conv_ws,
                           cudaStream_t st) {
  const RowOut ro{dq_tab, dq_n, dq_chunk};
  KvOut kv{};
  if (conv_ws != nullptr && (dkdv_out != nullptr || (dk_tab != nullptr && dv_tab != nullptr))) {
    kv.dk = reinterpret_cast<__nv_bfloat16*>(dkdv_out);
    kv.dv = kv.dk ? kv.dk + (long long)H * Lk * D : nullptr;
    kv.dk_rows = RowOut{dk_tab, kv_n, kv_chunk};
    kv.dv_rows = RowOut{dv_tab, kv_n, kv_chunk};
    kv.head_done = conv_ws;
  }
  if (D == 128)
    return bwd_launch<128>(q, k, v, O, dO, lse, grp_rows, grp_size, idx, ldk, kcount, kcount_hg, H,
                           G, Lq, Lk, scale, scale_log2, dQ, dK, dV, sched, tile_grp, Gs, ro, kv,
                           st);
  if (D == 64)
    return bwd_launch<64>(q, k, v, O, dO, lse, grp_rows, grp_size, idx, ldk, kcount, kcount_hg, H,
                          G, Lq, Lk, scale, scale_log2, dQ, dK, dV, sched, tile_grp, Gs, ro, kv, st);
  return 1;
}

int dsv_debug_timeline_copy(void* dst, int bytes) {
  const int n = (int)sizeof(g_bwd_prof) < bytes ? (int)sizeof(g_bwd_prof) : bytes;
  if (cudaMemcpyFromSymbol(dst, g_bwd_prof, n) != cudaSuccess) return -1;
  return n;
}

int dsv_f32_to_bf16_rows_launch(const float* in, int H, int L, int D, const long long* tab, int n,
                                int chunk, cudaStream_t st) {
  const long long rows = (long long)H * L;
  if (rows <= 0) return 0;
  const RowOut ro{tab, n, chunk};
  const unsigned blocks = (unsigned)((rows * 32 + 255) / 256);
  if (D == 128) f32_to_bf16_rows_kernel<128><<<blocks, 256, 0, st>>>(in, rows, L, ro);
  else if (D == 64) f32_to_bf16_rows_kernel<64><<<blocks, 256, 0, st>>>(in, rows, L, ro);
  else return 1;
  return (int)cudaGetLastError();
}

int dsv_f32_to_bf16_launch(const float* in, void* out, long long n, cudaStream_t st) {
  if (n <= 0) return 0;
  const long long threads = (n + 3) / 4;
  f32_to_bf16_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(in, (__nv_bfloat16*)out, n);
  return (int)cudaGetLastError();
}
