// scores_tc.cu — K1b: proxy approximate scores S_h = Q_lr[proxies] . K_lr^T on tcgen05.
//
// Reference: pkg/src/dynsparse/selection.py:149 (`q_block @ k_lr[c0:c1].T`) applied to
// the group proxies (grouping.py:184-193 selects one set per voxel from its proxy).
// Output: fp32 scores [H][G][L] (row = proxy, contiguous over keys) for K2.
//
// The product is tiny in FLOPs (2*G*L*r per head) and bound by the 4*H*G*L bytes it
// writes. The MMA is issued "transposed" — M = 128 keys, N = the head's proxies —
// so each epilogue thread owns one key (TMEM lane) and, column by column, the 32
// lanes of a warp store 32 consecutive keys of one proxy row: every store is a
// fully coalesced 128-byte line, straight from tcgen05.ld registers.
// Persistent CTAs walk (head, proxy chunk, key tile) units; key tiles are gathered
// by cp.async into the no-swizzle K-major UMMA layout through a 4-stage ring, and
// two TMEM accumulators let the epilogue of tile i overlap the MMA of tile i+1.

#include "dsv_common.cuh"

namespace dsv {
namespace scores {

constexpr int kThreads = 256;   // warp 0: MMA, warps 1-3: loaders, warps 4-7: epilogue
constexpr int kStages = 4;
constexpr int kMaxN = 256;

// no-swizzle K-major canonical layout for r = 16 (two 8-column core-matrix halves):
// row p, half c at (p/8)*256 + c*128 + (p%8)*16
DSV_DEV uint32_t ns_off(int p, int c) { return (uint32_t)((p >> 3) * 256 + c * 128 + (p & 7) * 16); }

DSV_DEV uint64_t sdesc_noswz(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;    // LBO: next 8-column K half
  d |= (uint64_t)(256 >> 4) << 32;    // SBO: next 8-row group
  d |= (uint64_t)1 << 46;             // version
  return d;                           // layout type 0 = SWIZZLE_NONE
}

struct Bars {
  uint64_t a_full[kStages], a_empty[kStages], acc_full[2], acc_empty[2], b_full;
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreads, 1)
proxy_scores_kernel(const __nv_bfloat16* __restrict__ Qp, long long ldq, long long q_bs,
                    const __nv_bfloat16* __restrict__ Klr, long long ldk, long long k_bs,
                    float* __restrict__ out, long long ldo, long long o_bs,
                    int H, int G, int L, int chunk_n, int nchunks) {
  __shared__ __align__(1024) uint8_t sA[kStages][128 * 32];
  __shared__ __align__(1024) uint8_t sB[kMaxN * 32];
  __shared__ Bars B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (L + 127) / 128;
  const long long units = (long long)H * nchunks * ntiles;
  const long long per = (units + gridDim.x - 1) / gridDim.x;
  const long long u0 = blockIdx.x * per, u1 = min(units, u0 + per);
  const int N = chunk_n;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kStages; ++s) { mbar_init(&B.a_full[s], 64); mbar_init(&B.a_empty[s], 1); }
      for (int s = 0; s < 2; ++s) { mbar_init(&B.acc_full[s], 1); mbar_init(&B.acc_empty[s], 128); }
      mbar_init(&B.b_full, 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc(&B.tmem, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem;

  // B (proxy chunk) is reloaded whenever (head, chunk) changes; all roles agree on the
  // unit sequence so they can track it locally. Loading B is done by the epilogue warps
  // between units under the b_full / acc barriers (rare: once per (head, chunk)).
  if (warp >= 1 && warp <= 2) {
    // ------------------------------------------------------------ A loaders (64 thr)
    const int t = threadIdx.x - 32;         // 0..63
    int it = 0;
    for (long long u = u0; u < u1; ++u, ++it) {
      const int kt = (int)(u % ntiles);
      const long long hc = u / ntiles;
      const int h = (int)(hc / nchunks);
      const int s = it % kStages;
      if (it >= kStages) mbar_wait(&B.a_empty[s], ((it / kStages) - 1) & 1);
      const __nv_bfloat16* kb = Klr + (long long)h * k_bs;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = i * 64 + t;          // 0..255: row c/2, half c%2
        const int p = c >> 1, half = c & 1;
        const int key = min(kt * 128 + p, L - 1);
        cp_async16(smem_u32(sA[s]) + ns_off(p, half), kb + (long long)key * ldk + half * 8);
      }
      cp_async_arrive_noinc(&B.a_full[s]);
    }
    cp_async_wait<0>();
  } else if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
    int it = 0;
    long long cur_hc = -1;
    uint32_t bphase = 0;
    for (long long u = u0; u < u1; ++u, ++it) {
      const long long hc = u / ntiles;
      if (hc != cur_hc) {                   // new B chunk: wait for the epilogue to load it
        mbar_wait(&B.b_full, bphase);
        bphase ^= 1;
        cur_hc = hc;
      }
      const int s = it % kStages, ab = it & 1;
      mbar_wait(&B.a_full[s], (it / kStages) & 1);
      if (it >= 2) mbar_wait(&B.acc_empty[ab], ((it >> 1) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        mma_ss(tmem + ab * 256, sdesc_noswz(smem_u32(sA[s])), sdesc_noswz(smem_u32(sB)), idesc, 0);
        mma_commit(&B.a_empty[s]);
        mma_commit(&B.acc_full[ab]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (128 thr)
    const int e = threadIdx.x - 128;        // TMEM lane = key within the tile
    const int wq = warp & 3;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    int it = 0;
    long long cur_hc = -1;
    for (long long u = u0; u < u1; ++u, ++it) {
      const int kt = (int)(u % ntiles);
      const long long hc = u / ntiles;
      const int h = (int)(hc / nchunks), ch = (int)(hc % nchunks);
      const int p0 = ch * N;
      if (hc != cur_hc) {
        // every earlier MMA (the last read of sB) completed: this warp group already
        // consumed acc_full of tile it-1, and tcgen05 MMAs complete in issue order
        named_bar_sync(1, 128);
        const __nv_bfloat16* qb = Qp + (long long)h * q_bs;
        for (int c = e; c < N * 2; c += 128) {
          const int p = c >> 1, half = c & 1;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (p0 + p < G) v = *reinterpret_cast<const uint4*>(qb + (long long)(p0 + p) * ldq + half * 8);
          *reinterpret_cast<uint4*>(sB + ns_off(p, half)) = v;
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (e == 0) mbar_arrive(&B.b_full);
        cur_hc = hc;
      }
      const int ab = it & 1;
      mbar_wait(&B.acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
      const int key = kt * 128 + e;
      float* ob = out + (long long)h * o_bs + key;
#pragma unroll 1
      for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ab * 256 + lane_off + c, r);
        tmem_ld_wait();
        if (key < L) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (p0 + c + j < G && c + j < N) ob[(long long)(p0 + c + j) * ldo] = __uint_as_float(r[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&B.acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace scores
}  // namespace dsv

int dsv_proxy_scores_launch(const void* Qp, long long ldq, long long q_bs, const void* Klr,
                            long long ldk, long long k_bs, float* out, long long ldo,
                            long long o_bs, int H, int G, int L, cudaStream_t st) {
  using namespace dsv::scores;
  const int nchunks = (G + kMaxN - 1) / kMaxN;
  const int n = ((G + nchunks - 1) / nchunks + 15) / 16 * 16;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (long long)H * nchunks * ((L + 127) / 128);
  const int grid = (int)(units < sms ? units : sms);
  proxy_scores_kernel<<<grid, kThreads, 0, st>>>((const __nv_bfloat16*)Qp, ldq, q_bs,
                                                 (const __nv_bfloat16*)Klr, ldk, k_bs, out, ldo,
                                                 o_bs, H, G, L, n, nchunks);
  return (int)cudaGetLastError();
}
