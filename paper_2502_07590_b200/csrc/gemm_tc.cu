// gemm_tc.cu — K1: tcgen05/TMEM GEMM for the low-rank predictor.
//
//   C[b, m, n] = sum_k A[b, m, k] * B[b, n, k]     (bf16 in, fp32 accumulate)
//
// Used twice on the hot path:
//  * K1a projection  X[L, H*d] . Wt[2*r*H, H*d]^T -> [Q_lr | K_lr] (reference
//    pkg/src/dynsparse/predictor.py:94-100 `project`, applied at :238-239 for
//    both W_q and W_k, batched over all heads in one GEMM);
//  * K1b proxy scores Q_lr[proxies] . K_lr^T per head (K = r = 16; reference
//    pkg/src/dynsparse/selection.py:149), fp32 out for K2.
//
// Structure: one 128 x BN output tile per CTA; warp 0 (one elected lane) is the
// TMA producer over a STAGES-deep ring of 128B-swizzled K-major A/B tiles,
// warp 1 (one elected lane) issues tcgen05.mma (M=128, N=BN, K=16) into a TMEM
// accumulator, then all four warps drain TMEM (tcgen05.ld 32x32b) and store.

#include <cuda.h>
#include "dsv_common.cuh"

namespace dsv {
namespace gemm {

constexpr int BM = 128, BK = 64;

template <int BN, int STAGES, bool kTmaStore = false>
struct SmemLayout {
  static constexpr int kA = BM * BK * 2;
  static constexpr int kB = BN * BK * 2;
  static constexpr int kStage = kA + kB;
  static constexpr int kOut = kTmaStore ? 2 * BM * 32 * 4 : 0;   // two 128 x 32 fp32 slices
  static constexpr int kBytes = STAGES * kStage + kOut + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int STAGES, bool kF32Out, bool kTmaStore = false>
__global__ void __launch_bounds__(128)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmC,
            void* __restrict__ C, int M, int N, int K, long long ldc, long long c_bs) {
  using SL = SmemLayout<BN, STAGES, kTmaStore>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  uint8_t* sOut = smem + STAGES * SL::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SL::kStage + SL::kOut);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // N tiles fastest: the CTAs sharing one A tile run together, so A streams from
  // DRAM once (the projection's X is 196 MB at c2; B = Wt stays in L2)
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, b = blockIdx.z;
  const int nk = (K + BK - 1) / BK;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
      mbar_init(accum, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(empty + s, ph ^ 1);
      uint8_t* sa = smem + s * SL::kStage;
      uint8_t* sb = sa + SL::kA;
      mbar_arrive_expect_tx(full + s, SL::kStage);
      tma_load_3d(sa, &tmA, full + s, kb * BK, m0, b);
      tma_load_3d(sb, &tmB, full + s, kb * BK, n0, b);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, 0, 0);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(full + s, ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * SL::kStage);
      const uint32_t sb = sa + SL::kA;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        const uint64_t ad = sdesc_sw128(sa + kk * 32, 16, 1024);
        const uint64_t bd = sdesc_sw128(sb + kk * 32, 16, 1024);
        mma_ss(tmem, ad, bd, idesc, (kb | kk) != 0);
      }
      mma_commit(empty + s);
    }
    mma_commit(accum);
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> global
  mbar_wait(accum, 0);
  tc_fence_after();
  const int row = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  if constexpr (kTmaStore) {
    // 32-column slices: TMEM -> 128B-swizzled smem (conflict-free 16-byte stores) ->
    // one TMA tensor store per slice, two slices in flight; TMA clips the edges.
    const int r = warp * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(trow + c * 32, v);
      tmem_ld_wait();
      uint8_t* buf = sOut + (c & 1) * (BM * 32 * 4);
      if (c >= 2) {
        if (threadIdx.x == 0) bulk_wait_read1();
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint4*>(buf + r * 128 + ((q ^ (r & 7)) << 4)) =
            make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        tma_store_3d(&tmC, buf, n0 + c * 32, m0, b);
        bulk_commit();
      }
    }
    if (threadIdx.x == 0) bulk_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, kTmemCols);
    return;
  }
  const bool vec_ok = kF32Out ? ((ldc & 3) == 0) : ((ldc & 7) == 0);
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    uint32_t r[32];
    tmem_ld32(trow + c, r);
    tmem_ld_wait();
    if (row >= M) continue;
    const int col = n0 + c;
    if constexpr (kF32Out) {
      float* out = reinterpret_cast<float*>(C) + (long long)b * c_bs + (long long)row * ldc + col;
      if (vec_ok && col + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(out + j) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                          __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
      } else {
        for (int j = 0; j < 32; ++j)
          if (col + j < N) out[j] = __uint_as_float(r[j]);
      }
    } else {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(C) + (long long)b * c_bs +
                           (long long)row * ldc + col;
      if (vec_ok && col + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8)
          *reinterpret_cast<uint4*>(out + j) = make_uint4(
              pack_bf16(__uint_as_float(r[j]), __uint_as_float(r[j + 1])),
              pack_bf16(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])),
              pack_bf16(__uint_as_float(r[j + 4]), __uint_as_float(r[j + 5])),
              pack_bf16(__uint_as_float(r[j + 6]), __uint_as_float(r[j + 7])));
      } else {
        for (int j = 0; j < 32; ++j)
          if (col + j < N) out[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gemm
}  // namespace dsv

template <int BN, int STAGES, bool F32, bool TMA_ST = false>
static int launch_gemm(const CUtensorMap* ta, const CUtensorMap* tb, const CUtensorMap* tc, void* C,
                       int M, int N, int K, long long ldc, long long c_bs, int nbatch,
                       cudaStream_t st) {
  using namespace dsv::gemm;
  const int smem = SmemLayout<BN, STAGES, TMA_ST>::kBytes;
  auto kern = gemm_kernel<BN, STAGES, F32, TMA_ST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, nbatch);
  kern<<<grid, 128, smem, st>>>(*ta, *tb, tc ? *tc : *ta, C, M, N, K, ldc, c_bs);
  return (int)cudaGetLastError();
}

int dsv_gemm_launch(const CUtensorMap* ta, const CUtensorMap* tb, const CUtensorMap* tc, void* C,
                    int M, int N, int K, long long ldc, long long c_bs, int nbatch, int f32_out,
                    int bn, cudaStream_t st) {
  if (K <= dsv::gemm::BK) {   // one k-block (proxy scores, K = r): small CTAs, several per SM
    if (f32_out && tc) return launch_gemm<128, 1, true, true>(ta, tb, tc, C, M, N, K, ldc, c_bs, nbatch, st);
    return f32_out ? launch_gemm<128, 1, true>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st)
                   : launch_gemm<128, 1, false>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st);
  }
  if (bn == 256) {
    return f32_out ? launch_gemm<256, 4, true>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st)
                   : launch_gemm<256, 4, false>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st);
  }
  // 128-wide tiles (narrow N, or few output tiles such as the projection of one rank's
  // L/N tokens): 3 stages, two CTAs per SM
  return f32_out ? launch_gemm<128, 3, true>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st)
                 : launch_gemm<128, 3, false>(ta, tb, nullptr, C, M, N, K, ldc, c_bs, nbatch, st);
}
