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
// Forward CTA (one per (head, group); 192 threads):
//   warp 0   : TMA producer — Q tile via tile::gather4 on the member rows, then
//              per 128-key block the selected K and V rows via gather4 into a
//              2-stage ring (128B swizzle, two 64-column atoms for D=128);
//   warp 1   : tcgen05.mma issuer — S_j = Q K_j^T into one of two TMEM S
//              buffers, then O += P_{j-1} V_{j-1} (P read from TMEM aliased over
//              S, or from shared memory in the kPTmem=false variant);
//   warps 2-5: softmax — one query row per thread: tcgen05.ld of S, online
//              max with lazy rescale (only when the max grows by > 2^8), P to
//              TMEM/smem as bf16, O correction in TMEM when rescaling, and the
//              final O/l epilogue + LSE.
// Backward CTA (transposed formulation, keys in TMEM lanes):
//   S^T = K_j Q^T and dP^T = V_j dO^T (M = keys), workers (one key row per
//   thread) form P^T and dS^T in TMEM, dV_j = P^T dO and dK_j = dS^T Q read
//   their A operand from TMEM, dQ += dS K_j reads dS from shared memory;
//   dK_j / dV_j rows are scatter-added into fp32 accumulators with red.v4.

#include <cuda.h>
#include "dsv_common.cuh"

namespace dsv {
namespace attn {

constexpr int BQ = 128;   // queries per tile
constexpr int BKV = 128;  // keys per block
constexpr int kThreads = 192;
constexpr int kStages = 2;

template <int D>
struct FwdSmem {
  static constexpr int kAtoms = D / 64;
  static constexpr int kTile = 128 * D * 2;          // one 128-row operand tile
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kP = kV + kStages * kTile;     // only used when P lives in smem
  static constexpr int kBar = kP + 128 * 128 * 2;
  static constexpr int kBytes = kBar + 256 + 1024;
};

struct FwdBars {
  uint64_t q_full;
  uint64_t k_full[kStages], v_full[kStages], kv_empty[kStages];
  uint64_t s_full[2], p_full[2];
  uint64_t o_ready, o_final;
  uint32_t tmem;
};

// Gather 128 rows (row ids from `rows`, 4 per lane) of a [*, D] bf16 tensor
// into a 128B-swizzled tile: atom a holds columns [64a, 64a+64).
template <int D>
DSV_DEV void gather_tile(uint8_t* tile, const CUtensorMap* tm, uint64_t* bar, int lane,
                         int r0, int r1, int r2, int r3) {
#pragma unroll
  for (int a = 0; a < D / 64; ++a)
    tma_gather4(tile + a * (128 * 128) + lane * 512, tm, bar, a * 64, r0, r1, r2, r3);
}

template <int D, bool kPTmem>
__global__ void __launch_bounds__(kThreads, 1)
sparse_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const int* __restrict__ grp_rows,
                  const int* __restrict__ grp_size, const int* __restrict__ idx, long long ldk,
                  const int* __restrict__ kcount, int G, int Lq, int Lk, float scale_log2,
                  __nv_bfloat16* __restrict__ O, float* __restrict__ lse) {
  using SL = FwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  FwdBars& B = *reinterpret_cast<FwdBars*>(smem + SL::kBar);
  uint8_t* sQ = smem + SL::kQ;
  uint8_t* sK = smem + SL::kK;
  uint8_t* sV = smem + SL::kV;
  uint8_t* sP = smem + SL::kP;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x / G, g = blockIdx.x - h * G;
  const int kh = kcount[h];
  const int nblk = (kh + BKV - 1) / BKV;
  const int* irow = idx + ((long long)h * G + g) * ldk;
  const int* mrow = grp_rows + (long long)g * BQ;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
      mbar_init(&B.q_full, 1);
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&B.k_full[s], 1); mbar_init(&B.v_full[s], 1); mbar_init(&B.kv_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) { mbar_init(&B.s_full[s], 1); mbar_init(&B.p_full[s], 128); }
      mbar_init(&B.o_ready, 1);
      mbar_init(&B.o_final, 1);
      fence_barrier_init();
    }
  } else if (warp == 1) {
    tmem_alloc(&B.tmem, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;
  const uint32_t tS0 = tmem, tO = tmem + 256;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    {
      const int4 m4 = *reinterpret_cast<const int4*>(mrow + lane * 4);
      const int base = h * Lq;
      if (lane == 0) mbar_arrive_expect_tx(&B.q_full, SL::kTile);
      __syncwarp();
      gather_tile<D>(sQ, &tmQ, &B.q_full, lane, base + m4.x, base + m4.y, base + m4.z, base + m4.w);
    }
    const int kbase = h * Lk;
    for (int j = 0; j < nblk; ++j) {
      const int st = j % kStages;
      if (j >= kStages) mbar_wait(&B.kv_empty[st], ((j / kStages) - 1) & 1);
      const int p = j * BKV + lane * 4;
      int r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) r[i] = kbase + __ldg(irow + min(p + i, kh - 1));
      if (lane == 0) {
        mbar_arrive_expect_tx(&B.k_full[st], SL::kTile);
        mbar_arrive_expect_tx(&B.v_full[st], SL::kTile);
      }
      __syncwarp();
      gather_tile<D>(sK + st * SL::kTile, &tmK, &B.k_full[st], lane, r[0], r[1], r[2], r[3]);
      gather_tile<D>(sV + st * SL::kTile, &tmV, &B.v_full[st], lane, r[0], r[1], r[2], r[3]);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idS = idesc_bf16_f32(128, BKV, 0, 0);
    constexpr uint32_t idO = idesc_bf16_f32(128, D, 0, 1);
    const uint32_t aQ = smem_u32(sQ);
    mbar_wait(&B.q_full, 0);
    for (int j = 0; j <= nblk; ++j) {
      if (j < nblk) {
        const int st = j % kStages;
        mbar_wait(&B.k_full[st], (j / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aK = smem_u32(sK + st * SL::kTile);
          const uint32_t dS = tS0 + (j & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
            mma_ss(dS, sdesc_sw128(aQ + off, 16, 1024), sdesc_sw128(aK + off, 16, 1024), idS,
                   kk > 0);
          }
          mma_commit(&B.s_full[j & 1]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jp = j - 1, st = jp % kStages;
        mbar_wait(&B.p_full[jp & 1], (jp >> 1) & 1);
        mbar_wait(&B.v_full[st], (jp / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aV = smem_u32(sV + st * SL::kTile);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t bd = sdesc_sw128(aV + kk * 2048, 128 * 128, 1024);
            if constexpr (kPTmem) {
              mma_ts(tO, tS0 + (jp & 1) * 128 + kk * 8, bd, idO, (jp | kk) != 0);
            } else {
              const uint32_t aP = smem_u32(sP) + (kk >> 2) * (128 * 128) + (kk & 3) * 32;
              mma_ss(tO, sdesc_sw128(aP, 16, 1024), bd, idO, (jp | kk) != 0);
            }
          }
          mma_commit(&B.kv_empty[st]);
          mma_commit(&B.o_ready);
          if (jp == nblk - 1) mma_commit(&B.o_final);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int sb = j & 1;
      const int kv = min(BKV, kh - j * BKV);
      mbar_wait(&B.s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      float sv[BKV];
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tS0 + sb * 128 + lane_off + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(r[i]);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < BKV; ++i) {
        if (i >= kv) sv[i] = -INFINITY;
        mx = fmaxf(mx, sv[i]);
      }
      mx *= scale_log2;
      if (j == 0) {
        m_run = mx;
      } else if (mx > m_run + 8.f) {
        // O correction: wait for PV_{j-1}, rescale O and l by 2^(m_run - mx)
        mbar_wait(&B.o_ready, (j - 1) & 1);
        tc_fence_after();
        const float alpha = fast_exp2(m_run - mx);
        l_run *= alpha;
#pragma unroll 1
        for (int c = 0; c < D / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(tO + lane_off + c * 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st16(tO + lane_off + c * 16, r);
        }
        tmem_st_wait();
        m_run = mx;
      }
      if constexpr (!kPTmem) {
        // single smem P buffer: PV_{j-1} must have consumed it
        if (j >= 1) mbar_wait(&B.o_ready, (j - 1) & 1);
      }
      float lsum = 0.f;
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = fast_exp2(fmaf(sv[c * 32 + 2 * i], scale_log2, -m_run));
          const float p1 = fast_exp2(fmaf(sv[c * 32 + 2 * i + 1], scale_log2, -m_run));
          pk[i] = pack_bf16(p0, p1);
          lsum += bf16lo(pk[i]) + bf16hi(pk[i]);
        }
        if constexpr (kPTmem) {
          tmem_st16(tS0 + sb * 128 + lane_off + c * 16, pk);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = c * 4 + q;  // 16-byte chunk index along keys (0..15)
            uint8_t* dst = sP + (chunk >> 3) * (128 * 128) + sw128_off(row, chunk & 7);
            *reinterpret_cast<uint4*>(dst) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      }
      l_run += lsum;
      if constexpr (kPTmem) tmem_st_wait();
      else fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&B.p_full[sb]);
    }
    // ---------------- epilogue
    mbar_wait(&B.o_final, 0);
    tc_fence_after();
    const int gsz = grp_size[g];
    const int tok = mrow[row];
    const float inv = 1.f / l_run;
    __nv_bfloat16* orow = O + ((long long)h * Lq + tok) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tO + lane_off + c * 32, r);
      tmem_ld_wait();
      if (row < gsz) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = make_uint4(
              pack_bf16(__uint_as_float(r[i]) * inv, __uint_as_float(r[i + 1]) * inv),
              pack_bf16(__uint_as_float(r[i + 2]) * inv, __uint_as_float(r[i + 3]) * inv),
              pack_bf16(__uint_as_float(r[i + 4]) * inv, __uint_as_float(r[i + 5]) * inv),
              pack_bf16(__uint_as_float(r[i + 6]) * inv, __uint_as_float(r[i + 7]) * inv));
      }
    }
    if (row < gsz) lse[(long long)h * Lq + tok] = m_run + __log2f(l_run);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ====================================================================== bwd
template <int D>
struct BwdSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kdO = kQ + kTile;
  static constexpr int kdS = kdO + kTile;                 // [128 keys][128 q] bf16
  static constexpr int kK = kdS + 128 * 128 * 2;
  static constexpr int kStagesB = (kK + 4 * kTile + 1024 + 256 + 1024 <= 232448) ? 2 : 1;
  static constexpr int kV = kK + kStagesB * kTile;
  static constexpr int kLse = kV + kStagesB * kTile;
  static constexpr int kDelta = kLse + 512;
  static constexpr int kBar = kDelta + 512;
  static constexpr int kBytes = kBar + 256 + 1024;
};

struct BwdBars {
  uint64_t q_full;
  uint64_t k_full[2], v_full[2], kv_empty[2];
  uint64_t sdp_full, pds_full, dvdk_full, tmem_free, dq_done;
  uint32_t tmem;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
sparse_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                  const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const __nv_bfloat16* __restrict__ Og, const __nv_bfloat16* __restrict__ dOg,
                  const float* __restrict__ lse, const int* __restrict__ grp_rows,
                  const int* __restrict__ grp_size, const int* __restrict__ idx, long long ldk,
                  const int* __restrict__ kcount, int G, int Lq, int Lk, float scale,
                  float scale_log2, __nv_bfloat16* __restrict__ dQ, float* __restrict__ dK,
                  float* __restrict__ dV) {
  using SL = BwdSmem<D>;
  constexpr int ST = SL::kStagesB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  BwdBars& B = *reinterpret_cast<BwdBars*>(smem + SL::kBar);
  uint8_t* sQ = smem + SL::kQ;
  uint8_t* sdO = smem + SL::kdO;
  uint8_t* sdS = smem + SL::kdS;
  uint8_t* sK = smem + SL::kK;
  uint8_t* sV = smem + SL::kV;
  float* sLse = reinterpret_cast<float*>(smem + SL::kLse);
  float* sDelta = reinterpret_cast<float*>(smem + SL::kDelta);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x / G, g = blockIdx.x - h * G;
  const int kh = kcount[h];
  const int nblk = (kh + BKV - 1) / BKV;
  const int* irow = idx + ((long long)h * G + g) * ldk;
  const int* mrow = grp_rows + (long long)g * BQ;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmQ); prefetch_tmap(&tmdO); prefetch_tmap(&tmK); prefetch_tmap(&tmV);
      mbar_init(&B.q_full, 1);
      for (int s = 0; s < 2; ++s) {
        mbar_init(&B.k_full[s], 1); mbar_init(&B.v_full[s], 1); mbar_init(&B.kv_empty[s], 1);
      }
      mbar_init(&B.sdp_full, 1);
      mbar_init(&B.pds_full, 128);
      mbar_init(&B.dvdk_full, 1);
      mbar_init(&B.tmem_free, 128);
      mbar_init(&B.dq_done, 1);
      fence_barrier_init();
    }
  } else if (warp == 1) {
    tmem_alloc(&B.tmem, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;
  const uint32_t tA = tmem, tB = tmem + 128, tC = tmem + 256, tDq = tmem + 384;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    {
      const int4 m4 = *reinterpret_cast<const int4*>(mrow + lane * 4);
      const int base = h * Lq;
      if (lane == 0) mbar_arrive_expect_tx(&B.q_full, 2 * SL::kTile);
      __syncwarp();
      gather_tile<D>(sQ, &tmQ, &B.q_full, lane, base + m4.x, base + m4.y, base + m4.z, base + m4.w);
      gather_tile<D>(sdO, &tmdO, &B.q_full, lane, base + m4.x, base + m4.y, base + m4.z, base + m4.w);
    }
    const int kbase = h * Lk;
    for (int j = 0; j < nblk; ++j) {
      const int st = j % ST;
      if (j >= ST) mbar_wait(&B.kv_empty[st], ((j / ST) - 1) & 1);
      const int p = j * BKV + lane * 4;
      int r[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) r[i] = kbase + __ldg(irow + min(p + i, kh - 1));
      if (lane == 0) {
        mbar_arrive_expect_tx(&B.k_full[st], SL::kTile);
        mbar_arrive_expect_tx(&B.v_full[st], SL::kTile);
      }
      __syncwarp();
      gather_tile<D>(sK + st * SL::kTile, &tmK, &B.k_full[st], lane, r[0], r[1], r[2], r[3]);
      gather_tile<D>(sV + st * SL::kTile, &tmV, &B.v_full[st], lane, r[0], r[1], r[2], r[3]);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idST = idesc_bf16_f32(128, 128, 0, 0);   // K_j . Q^T, V_j . dO^T
    constexpr uint32_t idDV = idesc_bf16_f32(128, D, 0, 1);     // P^T(tmem) . dO(MN)
    constexpr uint32_t idDK = idesc_bf16_f32(128, 64, 0, 1);    // dS^T(tmem) . Q(MN), 64 cols
    constexpr uint32_t idDQ = idesc_bf16_f32(128, D, 1, 1);     // dS(MN smem) . K_j(MN)
    const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), adS = smem_u32(sdS);
    mbar_wait(&B.q_full, 0);
    for (int j = 0; j < nblk; ++j) {
      const int st = j % ST;
      const uint32_t aK = smem_u32(sK + st * SL::kTile), aV = smem_u32(sV + st * SL::kTile);
      mbar_wait(&B.k_full[st], (j / ST) & 1);
      mbar_wait(&B.v_full[st], (j / ST) & 1);
      if (j > 0) mbar_wait(&B.tmem_free, (j - 1) & 1);
      tc_fence_after();
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
      }
      __syncwarp();
      mbar_wait(&B.pds_full, j & 1);
      tc_fence_after();
      if (elect_one()) {
        // dV_j = P^T dO   (A = P^T in TMEM cols tA[0,64), K = 128 queries)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tC, tA + kk * 8, sdesc_sw128(adO + kk * 2048, 128 * 128, 1024), idDV, kk > 0);
        // dK_j = dS^T Q   (A = dS^T in TMEM cols tB[0,64)); N split in 64-column halves
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_ts(tA + 64, tB + kk * 8, sdesc_sw128(aQ + kk * 2048, 128 * 128, 1024), idDK, kk > 0);
          if constexpr (D == 128)
            mma_ts(tB + 64, tB + kk * 8, sdesc_sw128(aQ + 128 * 128 + kk * 2048, 128 * 128, 1024),
                   idDK, kk > 0);
        }
        mma_commit(&B.dvdk_full);
        // dQ += dS K_j    (A = dS MN-major in smem, B = K_j MN-major)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tDq, sdesc_sw128(adS + kk * 2048, 128 * 128, 1024),
                 sdesc_sw128(aK + kk * 2048, 128 * 128, 1024), idDQ, (j | kk) != 0);
        mma_commit(&B.dq_done);
        mma_commit(&B.kv_empty[st]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ workers
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;   // query row in prologue/epilogue; key row per block
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int gsz = grp_size[g];
    const int tok = mrow[row];
    {
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
      sDelta[row] = dlt;
      named_bar_sync(1, 128);
    }
    for (int j = 0; j < nblk; ++j) {
      const int kv = min(BKV, kh - j * BKV);
      const bool kvalid = row < kv;
      const int key = kvalid ? __ldg(irow + j * BKV + row) : 0;
      mbar_wait(&B.sdp_full, j & 1);
      tc_fence_after();
      if (j > 0) mbar_wait(&B.dq_done, (j - 1) & 1);   // dQ_{j-1} done reading sdS
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t rs[32], rd[32];
        tmem_ld32(tA + lane_off + c * 32, rs);
        tmem_ld32(tB + lane_off + c * 32, rd);
        tmem_ld_wait();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int q0 = c * 32 + 2 * i;
          float p0 = fast_exp2(fmaf(__uint_as_float(rs[2 * i]), scale_log2, -sLse[q0]));
          float p1 = fast_exp2(fmaf(__uint_as_float(rs[2 * i + 1]), scale_log2, -sLse[q0 + 1]));
          float d0 = p0 * (__uint_as_float(rd[2 * i]) - sDelta[q0]) * scale;
          float d1 = p1 * (__uint_as_float(rd[2 * i + 1]) - sDelta[q0 + 1]) * scale;
          if (!kvalid) { p0 = p1 = d0 = d1 = 0.f; }
          pp[i] = pack_bf16(p0, p1);
          dd[i] = pack_bf16(d0, d1);
        }
        tmem_st16(tA + lane_off + c * 16, pp);
        tmem_st16(tB + lane_off + c * 16, dd);
        // dS row (this key) into the MN-major dS tile: atom c/2, chunks (c%2)*4..+3
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint8_t* dst = sdS + (c >> 1) * (128 * 128) + sw128_off(row, (c & 1) * 4 + q);
          *reinterpret_cast<uint4*>(dst) = make_uint4(dd[4 * q], dd[4 * q + 1], dd[4 * q + 2], dd[4 * q + 3]);
        }
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&B.pds_full);
      // ---- scatter dV_j, dK_j rows of this key into the fp32 accumulators
      mbar_wait(&B.dvdk_full, j & 1);
      tc_fence_after();
      float* dvrow = dV + ((long long)h * Lk + key) * D;
      float* dkrow = dK + ((long long)h * Lk + key) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t rv[32], rk[32];
        tmem_ld32(tC + lane_off + c * 32, rv);
        // dK columns [0,64) live in tA[64,128), [64,128) in tB[64,128)
        tmem_ld32((c < 2 ? tA : tB) + 64 + lane_off + (c & 1) * 32, rk);
        tmem_ld_wait();
        if (kvalid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            red_add_v4(dvrow + c * 32 + i, __uint_as_float(rv[i]), __uint_as_float(rv[i + 1]),
                       __uint_as_float(rv[i + 2]), __uint_as_float(rv[i + 3]));
            red_add_v4(dkrow + c * 32 + i, __uint_as_float(rk[i]), __uint_as_float(rk[i + 1]),
                       __uint_as_float(rk[i + 2]), __uint_as_float(rk[i + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&B.tmem_free);
    }
    // ---------------- dQ epilogue (query rows)
    mbar_wait(&B.dq_done, (nblk - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* qrow = dQ + ((long long)h * Lq + tok) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
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

}  // namespace attn
}  // namespace dsv

using namespace dsv::attn;

template <int D, bool PT>
static int fwd_launch(const CUtensorMap* tq, const CUtensorMap* tk, const CUtensorMap* tv,
                      const int* grp_rows, const int* grp_size, const int* idx, long long ldk,
                      const int* kcount, int H, int G, int Lq, int Lk, float scale_log2,
                      void* O, float* lse, cudaStream_t st) {
  auto kern = sparse_fwd_kernel<D, PT>;
  const int smem = FwdSmem<D>::kBytes;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<H * G, kThreads, smem, st>>>(*tq, *tk, *tv, grp_rows, grp_size, idx, ldk, kcount, G, Lq,
                                      Lk, scale_log2, (__nv_bfloat16*)O, lse);
  return (int)cudaGetLastError();
}

int dsv_attn_fwd_tc_launch(const CUtensorMap* tq, const CUtensorMap* tk, const CUtensorMap* tv,
                           const int* grp_rows, const int* grp_size, const int* idx,
                           long long ldk, const int* kcount, int H, int G, int Lq, int Lk, int D,
                           float scale_log2, int p_in_tmem, void* O, float* lse,
                           cudaStream_t st) {
  if (D == 128)
    return p_in_tmem ? fwd_launch<128, true>(tq, tk, tv, grp_rows, grp_size, idx, ldk, kcount, H, G, Lq, Lk, scale_log2, O, lse, st)
                     : fwd_launch<128, false>(tq, tk, tv, grp_rows, grp_size, idx, ldk, kcount, H, G, Lq, Lk, scale_log2, O, lse, st);
  if (D == 64)
    return p_in_tmem ? fwd_launch<64, true>(tq, tk, tv, grp_rows, grp_size, idx, ldk, kcount, H, G, Lq, Lk, scale_log2, O, lse, st)
                     : fwd_launch<64, false>(tq, tk, tv, grp_rows, grp_size, idx, ldk, kcount, H, G, Lq, Lk, scale_log2, O, lse, st);
  return 1;
}

template <int D>
static int bwd_launch(const CUtensorMap* tq, const CUtensorMap* tdo, const CUtensorMap* tk,
                      const CUtensorMap* tv, const void* O, const void* dO, const float* lse,
                      const int* grp_rows, const int* grp_size, const int* idx, long long ldk,
                      const int* kcount, int H, int G, int Lq, int Lk, float scale,
                      float scale_log2, void* dQ, float* dK, float* dV, cudaStream_t st) {
  auto kern = sparse_bwd_kernel<D>;
  const int smem = BwdSmem<D>::kBytes;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<H * G, kThreads, smem, st>>>(*tq, *tdo, *tk, *tv, (const __nv_bfloat16*)O,
                                      (const __nv_bfloat16*)dO, lse, grp_rows, grp_size, idx, ldk,
                                      kcount, G, Lq, Lk, scale, scale_log2, (__nv_bfloat16*)dQ,
                                      dK, dV);
  return (int)cudaGetLastError();
}

int dsv_attn_bwd_tc_launch(const CUtensorMap* tq, const CUtensorMap* tdo, const CUtensorMap* tk,
                           const CUtensorMap* tv, const void* O, const void* dO, const float* lse,
                           const int* grp_rows, const int* grp_size, const int* idx,
                           long long ldk, const int* kcount, int H, int G, int Lq, int Lk, int D,
                           float scale, float scale_log2, void* dQ, float* dK, float* dV,
                           cudaStream_t st) {
  if (D == 128)
    return bwd_launch<128>(tq, tdo, tk, tv, O, dO, lse, grp_rows, grp_size, idx, ldk, kcount, H, G,
                           Lq, Lk, scale, scale_log2, dQ, dK, dV, st);
  if (D == 64)
    return bwd_launch<64>(tq, tdo, tk, tv, O, dO, lse, grp_rows, grp_size, idx, ldk, kcount, H, G,
                          Lq, Lk, scale, scale_log2, dQ, dK, dV, st);
  return 1;
}

int dsv_f32_to_bf16_launch(const float* in, void* out, long long n, cudaStream_t st) {
  if (n <= 0) return 0;
  const long long threads = (n + 3) / 4;
  f32_to_bf16_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(in, (__nv_bfloat16*)out, n);
  return (int)cudaGetLastError();
}
