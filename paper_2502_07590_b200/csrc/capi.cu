// capi.cu — the extern "C" boundary (include/dsv.h): argument validation, TMA
// descriptor encoding and kernel dispatch. No allocation, no exceptions.

#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/dsv.h"
#include "dsv_common.cuh"

// kernels (defined in the other translation units)
size_t dsv_topk_smem_bytes(int L);
int dsv_topk_launch(const float*, long long, int, int, const int*, int, int*, long long, float*,
                    cudaStream_t);
int dsv_scores_f32_launch(const void*, long long, long long, const void*, long long, long long,
                          float*, long long, long long, int, int, int, int, int, cudaStream_t);
int dsv_rows_fwd_launch(const void*, const void*, const void*, const long long*, const int*, int,
                        int, int, int, float, int, float*, float*, cudaStream_t);
int dsv_rows_bwd_launch(const void*, const void*, const void*, const float*, const float*,
                        const void*, const long long*, const int*, int, int, int, int, float, int,
                        float*, float*, float*, cudaStream_t);
int dsv_critical_counts_launch(const float*, long long, int, int, double, double, int*, cudaStream_t);
int dsv_varint_launch(int, const int*, long long, const int*, int, int, long long*, unsigned char*, int*,
                      cudaStream_t);
int dsv_pred_pass_launch(int, const double*, const double*, const void*, int, long long, int, int,
                         int, const double*, double*, cudaStream_t);
int dsv_gemm_launch(const CUtensorMap*, const CUtensorMap*, const CUtensorMap*, void*, int, int, int, long long,
                    long long, int, int, int, cudaStream_t);
int dsv_attn_fwd_tc_launch(const void*, const void*, const void*, const int*, const int*,
                           const int*, long long, const int*, const int*, int, int, int, int, int,
                           float, void*, float*, unsigned*, float*, long long, const int*, int,
                           const long long*, int, int, cudaStream_t);
int dsv_attn_bwd_tc_launch(const void*, const void*, const void*, const void*, const void*,
                           const float*, const int*, const int*, const int*, long long,
                           const int*, const int*, int, int, int, int, int, float, float, void*,
                           float*, float*, unsigned*, const int*, int, const long long*, int, int,
                           void*, const long long*, const long long*, int, int, int*,
                           cudaStream_t);
int dsv_f32_to_bf16_rows_launch(const float*, int, int, int, const long long*, int, int,
                                cudaStream_t);
int dsv_f32_to_bf16_launch(const float*, void*, long long, cudaStream_t);
int dsv_select_fused_launch(const CUtensorMap*, const CUtensorMap*, int, int, int, const int*, int*,
                            long long, float*, int, void*, long long, cudaStream_t);
long long dsv_select_fused_ws_bytes(int, int, int, int, int);
int dsv_select_fused_clusters_query(int);
int dsv_lse_merge_launch(float*, const float*, float*, const void*, const float*, long long, int,
                         int, void*, cudaStream_t);
int dsv_accum_bf16_launch(float*, const void*, long long, int, void*, cudaStream_t);
int dsv_accum_f32_launch(float*, float*, long long, int, cudaStream_t);
int dsv_proxy_scores_launch(const void*, long long, long long, const void*, long long, long long,
                            float*, long long, long long, int, int, int, cudaStream_t);
int dsv_gemm_f64_launch(const double*, long long, long long, long long, const double*, long long,
                        long long, long long, double*, long long, long long, int, int, int, int,
                        double, cudaStream_t);
int dsv_softmax_rows_f64_launch(double*, long long, int, int, cudaStream_t);
int dsv_topk_f64_launch(const double*, long long, int, int, const int*, int, int*, long long,
                        double*, cudaStream_t);
int dsv_rows_fwd_f64_launch(const double*, const double*, const double*, const long long*,
                            const int*, int, int, int, int, int, double, double*, double*,
                            cudaStream_t);
int dsv_rows_bwd_f64_launch(const double*, const double*, const double*, const double*,
                            const double*, const double*, const long long*, const int*, int, int,
                            int, int, int, double, double*, double*, double*, cudaStream_t);
size_t dsv_sorted_stats_smem(int);
int dsv_sorted_stats_launch(const double*, long long, int, int, int, double, double, int, int*,
                            double*, void*, int, cudaStream_t);
int dsv_histogram_f64_launch(const double*, long long, int, int, const double*, int,
                             unsigned long long*, cudaStream_t);
int dsv_set_stats_f64_launch(const double*, long long, int, const long long*, const int*,
                             const long long*, const int*, int*, double*, double*, cudaStream_t);

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(int rc, const char* what) {
  if (rc == 0) return DSV_OK;
  return fail(DSV_ECUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)rc));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 tensor map with up to 3 dims: dims[0] innermost (elements), strides in bytes for
// dims 1..rank-1, 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box,
              CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[5];
  cuuint64_t gs[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) { gd[i] = dims[i]; bx[i] = box[i]; es[i] = 1; }
  for (int i = 0; i + 1 < rank; ++i) gs[i] = strides_bytes[i];
  CUresult r = fn(m, dt, rank, const_cast<void*>(base), gd, gs, bx,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int dsv_version(void) { return 100; }
const char* dsv_last_error(void) { return g_err; }

int dsv_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int dsv_gemm_bf16(const void* A, long long lda, long long a_bs, const void* B, long long ldb,
                  long long b_bs, void* C, int c_dtype, long long ldc, long long c_bs, int M,
                  int N, int K, int nbatch, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || nbatch <= 0) return fail(DSV_EINVAL, "gemm: empty shape");
  if (!al16(A) || !al16(B)) return fail(DSV_EINVAL, "gemm: operands must be 16-byte aligned");
  if ((lda * 2) % 16 || (ldb * 2) % 16 || (a_bs * 2) % 16 || (b_bs * 2) % 16)
    return fail(DSV_EINVAL, "gemm: operand strides must be multiples of 16 bytes");
  if (c_dtype != DSV_DTYPE_F32 && c_dtype != DSV_DTYPE_BF16)
    return fail(DSV_EINVAL, "gemm: bad output dtype");
  int bn = (N >= 256 && K > 64) ? 256 : 128;
  if (bn == 256 && (long long)((M + 127) / 128) * ((N + 255) / 256) * nbatch < 2LL * dsv_device_sm_count())
    bn = 128;   // too few 128 x 256 tiles to fill the GPU twice

  CUtensorMap ta, tb;
  {
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)M, (uint64_t)nbatch};
    const uint64_t st[2] = {(uint64_t)lda * 2, (uint64_t)(nbatch > 1 ? a_bs : (long long)M * lda) * 2};
    const uint32_t box[3] = {64, 128, 1};
    if (!make_map(&ta, A, 3, dims, st, box)) return fail(DSV_EINVAL, "gemm: tensor map A");
  }
  {
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)nbatch};
    const uint64_t st[2] = {(uint64_t)ldb * 2, (uint64_t)(nbatch > 1 ? b_bs : (long long)N * ldb) * 2};
    const uint32_t box[3] = {64, (uint32_t)bn, 1};
    if (!make_map(&tb, B, 3, dims, st, box)) return fail(DSV_EINVAL, "gemm: tensor map B");
  }
  // fp32 output of a one-k-block GEMM (the proxy scores): TMA tensor stores of
  // 32-column swizzled slices instead of row-per-thread stores
  CUtensorMap tc;
  const CUtensorMap* tcp = nullptr;
  if (c_dtype == DSV_DTYPE_F32 && K <= 64 && al16(C) && (ldc * 4) % 16 == 0 &&
      (nbatch == 1 || (c_bs * 4) % 16 == 0)) {
    const uint64_t dims[3] = {(uint64_t)N, (uint64_t)M, (uint64_t)nbatch};
    const uint64_t st[2] = {(uint64_t)ldc * 4, (uint64_t)(nbatch > 1 ? c_bs : (long long)M * ldc) * 4};
    const uint32_t box[3] = {32, 128, 1};
    if (make_map(&tc, C, 3, dims, st, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32)) tcp = &tc;
  }
  return cuda_status(dsv_gemm_launch(&ta, &tb, tcp, C, M, N, K, ldc, c_bs, nbatch,
                                     c_dtype == DSV_DTYPE_F32, bn, S(stream)),
                     "gemm launch");
}

int dsv_project(const void* X, const void* Wt, void* out, int L, int d_model, int n_out,
                void* stream) {
  if (L <= 0 || d_model <= 0 || n_out <= 0) return fail(DSV_EINVAL, "project: empty shape");
  return dsv_gemm_bf16(X, d_model, 0, Wt, d_model, 0, out, DSV_DTYPE_BF16, n_out, 0, L, n_out,
                       d_model, 1, stream);
}

int dsv_scores_f32(const void* A, long long lda, long long a_bs, const void* B, long long ldb,
                   long long b_bs, float* C, long long ldc, long long c_bs, int nbatch, int R,
                   int Lk, int r, int in_dtype, void* stream) {
  if (R <= 0 || Lk <= 0 || nbatch <= 0) return fail(DSV_EINVAL, "scores: empty shape");
  if (r < 1) return fail(DSV_EINVAL, "scores: inner width %d < 1", r);
  return cuda_status(dsv_scores_f32_launch(A, lda, a_bs, B, ldb, b_bs, C, ldc, c_bs, nbatch, R,
                                           Lk, r, in_dtype == DSV_DTYPE_BF16, S(stream)),
                     "scores launch");
}

int dsv_proxy_scores(const void* q_prox, long long ldq, long long q_bs, const void* k_lr,
                     long long ldk, long long k_bs, float* out, long long ldo, long long o_bs,
                     int H, int G, int L, int r, void* stream) {
  if (H <= 0 || G <= 0 || L <= 0) return fail(DSV_EINVAL, "proxy_scores: empty shape");
  if (r != 16) return fail(DSV_EUNSUPPORTED, "proxy_scores: predictor rank %d (tcgen05 path: 16)", r);
  if ((ldq * 2) % 16 || (q_bs * 2) % 16 || (ldk * 2) % 16 || (k_bs * 2) % 16 || !al16(q_prox) ||
      !al16(k_lr))
    return fail(DSV_EINVAL, "proxy_scores: rows must be 16-byte aligned");
  return cuda_status(dsv_proxy_scores_launch(q_prox, ldq, q_bs, k_lr, ldk, k_bs, out, ldo, o_bs, H,
                                             G, L, S(stream)),
                     "proxy_scores launch");
}

extern "C" int dsv_select_fused_max_clusters(int S) {
  // per-device cache of the occupancy query (the only mutable state: mutex-guarded)
  static std::mutex mu;
  static int cache[64][9];
  static bool init = false;
  if (S < 1 || S > 8) return 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!init) {
    for (auto& row : cache) for (int& v : row) v = -1;
    init = true;
  }
  if (cache[dev][S] < 0) cache[dev][S] = dsv_select_fused_clusters_query(S);
  return cache[dev][S];
}

static int select_split(int H, int G, int L, int split) {
  // key-range split per 128-row tile (a cluster of `split` CTAs, 1..6): fewest waves per
  // unit of per-CTA work, at least one 128-key tile per CTA. Waves count the clusters that can be
  // resident at once (a cluster fits in one GPC; measured: 36 4-CTA clusters at c2 with 12
  // heads took two waves, 0.40 ms against 0.375 at S = 2); ties keep the smaller split
  // (fewer cross-CTA merges)
  const int n_mt = H * ((G + 127) / 128), nt = (L + 127) / 128;
  int ns = split;
  if (ns <= 0) {
    int sms = dsv_device_sm_count();
    if (sms <= 0) sms = 148;        // no device visible: size for a B200
    double best = 1e30;
    for (int s = 1; s <= 6 && s <= nt; ++s) {
      const int mc = dsv_select_fused_max_clusters(s);
      const int per_wave = mc > 0 ? mc : sms / s;
      const double cost = (double)((n_mt + per_wave - 1) / per_wave) / s;
      if (cost < best - 1e-9) { best = cost; ns = s; }
    }
  }
  return ns;
}

long long dsv_select_fused_workspace_size(int H, int G, int L, int k_max, int split) {
  if (H <= 0 || G <= 0 || L <= 0 || k_max < 1 || k_max > L) return 0;
  const int ns = select_split(H, G, L, split);
  if (ns < 1 || ns > 8) return 0;
  return dsv_select_fused_ws_bytes(H, G, L, k_max, ns);
}

int dsv_select_fused(const void* q_prox, long long ldq, long long q_bs, const void* k_lr,
                     long long ldk, long long k_bs, int H, int G, int L, int r,
                     const int* k_per_head, int* out_idx, long long out_ld, float* out_thr,
                     int split, void* workspace, long long ws_bytes, void* stream) {
  if (H <= 0 || G <= 0 || L <= 0) return fail(DSV_EINVAL, "select_fused: empty shape");
  if (r < 1 || r > 16) return fail(DSV_EUNSUPPORTED, "select_fused: predictor rank %d (1..16)", r);
  if (!al16(q_prox) || !al16(k_lr) || (ldq * 2) % 16 || (ldk * 2) % 16 || (q_bs * 2) % 16 ||
      (k_bs * 2) % 16)
    return fail(DSV_EINVAL, "select_fused: rows must be 16-byte aligned");
  CUtensorMap ta, tb;
  {
    const uint64_t dims[3] = {(uint64_t)r, (uint64_t)G, (uint64_t)H};
    const uint64_t st[2] = {(uint64_t)ldq * 2, (uint64_t)(H > 1 ? q_bs : (long long)G * ldq) * 2};
    const uint32_t box[3] = {16, 128, 1};
    if (!make_map(&ta, q_prox, 3, dims, st, box, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_32B))
      return fail(DSV_EINVAL, "select_fused: tensor map Q");
  }
  {
    const uint64_t dims[3] = {(uint64_t)r, (uint64_t)L, (uint64_t)H};
    const uint64_t st[2] = {(uint64_t)ldk * 2, (uint64_t)(H > 1 ? k_bs : (long long)L * ldk) * 2};
    const uint32_t box[3] = {16, 128, 1};
    if (!make_map(&tb, k_lr, 3, dims, st, box, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_32B))
      return fail(DSV_EINVAL, "select_fused: tensor map K");
  }
  const int nt = (L + 127) / 128;
  const int ns = select_split(H, G, L, split);
  if (ns < 1 || ns > 8 || ns > nt) return fail(DSV_EINVAL, "select_fused: split %d", ns);
  return cuda_status(dsv_select_fused_launch(&ta, &tb, H, G, L, k_per_head, out_idx, out_ld,
                                             out_thr, ns, workspace, ws_bytes, S(stream)),
                     "select_fused launch");
}

int dsv_topk(const float* scores, long long ld, int rows, int L, const int* k_per_head,
             int rows_per_head, int* out_idx, long long out_ld, float* out_thr, void* stream) {
  if (rows < 0 || L < 1 || rows_per_head < 1) return fail(DSV_EINVAL, "topk: bad shape");
  if (ld < L) return fail(DSV_EINVAL, "topk: row stride %lld < L=%d", ld, L);
  return cuda_status(dsv_topk_launch(scores, ld, rows, L, k_per_head, rows_per_head, out_idx,
                                     out_ld, out_thr, S(stream)),
                     "topk launch");
}

int dsv_sparse_fwd(const void* q, const void* k, const void* v, const int* grp_rows,
                   const int* grp_size, const int* idx, long long ldk, const int* kcount,
                   const int* kcount_hg, int H, int G, int Lq, int Lk, int D, float scale,
                   void* out, float* lse, unsigned* work, long long work_words, float* zero_buf,
                   long long zero_floats, const int* tile_grp, int n_groups,
                   const long long* o_tab, int o_n, int o_chunk, void* stream) {
  if (D != 64 && D != 128) return fail(DSV_EUNSUPPORTED, "sparse_fwd: head dim %d not 64/128", D);
  if (o_tab && (o_n < 1 || o_chunk < 1 || (long long)o_n * o_chunk < Lq))
    return fail(DSV_EINVAL, "sparse_fwd: o_tab needs n * chunk >= Lq");
  if (tile_grp && n_groups <= 0) return fail(DSV_EINVAL, "sparse_fwd: tile_grp needs n_groups > 0");
  if (H <= 0 || G <= 0 || Lq <= 0 || Lk <= 0 || ldk < 0)
    return fail(DSV_EINVAL, "sparse_fwd: empty shape");
  if (!al16(q) || !al16(k) || !al16(v) || !al16(out) || !al16(grp_rows))
    return fail(DSV_EINVAL, "sparse_fwd: pointers must be 16-byte aligned");
  if (!work || work_words < (long long)H * G + 2)
    return fail(DSV_EINVAL, "sparse_fwd: workspace needs H*G + 2 words");
  if (zero_buf && (zero_floats < 0 || zero_floats % 4 || !al16(zero_buf)))
    return fail(DSV_EINVAL, "sparse_fwd: zero_buf must be 16-byte aligned, a multiple of 4 floats");
  const float scale_log2 = scale * 1.4426950408889634f;
  return cuda_status(dsv_attn_fwd_tc_launch(q, k, v, grp_rows, grp_size, idx, ldk, kcount,
                                            kcount_hg, H, G, Lq, Lk, D, scale_log2, out, lse,
                                            work, zero_buf, zero_buf ? zero_floats : 0, tile_grp,
                                            tile_grp ? n_groups : G, o_tab, o_n, o_chunk,
                                            S(stream)),
                     "sparse_fwd launch");
}

int dsv_sparse_bwd_convert(const void* q, const void* k, const void* v, const void* out,
                           const void* dout, const float* lse, const int* grp_rows,
                           const int* grp_size, const int* idx, long long ldk, const int* kcount,
                           const int* kcount_hg, int H, int G, int Lq, int Lk, int D, float scale,
                           void* dq, float* dk_acc, float* dv_acc, unsigned* work,
                           const int* tile_grp, int n_groups, const long long* dq_tab, int dq_n,
                           int dq_chunk, void* dkdv_out, const long long* dk_tab,
                           const long long* dv_tab, int kv_n, int kv_chunk, int* conv_ws,
                           void* stream) {
  if (D != 64 && D != 128) return fail(DSV_EUNSUPPORTED, "sparse_bwd: head dim %d not 64/128", D);
  if (conv_ws) {
    if (!dkdv_out && !(dk_tab && dv_tab))
      return fail(DSV_EINVAL, "sparse_bwd: conversion needs dkdv_out or both row tables");
    if (dkdv_out && !al16(dkdv_out)) return fail(DSV_EINVAL, "sparse_bwd: dkdv_out must be 16-byte aligned");
    if (!dkdv_out && (kv_n < 1 || kv_chunk < 1 || (long long)kv_n * kv_chunk < Lk))
      return fail(DSV_EINVAL, "sparse_bwd: dk/dv tables need n * chunk >= Lk");
  }
  if (dq_tab && (dq_n < 1 || dq_chunk < 1 || (long long)dq_n * dq_chunk < Lq))
    return fail(DSV_EINVAL, "sparse_bwd: dq_tab needs n * chunk >= Lq");
  if (tile_grp && n_groups <= 0) return fail(DSV_EINVAL, "sparse_bwd: tile_grp needs n_groups > 0");
  if (H <= 0 || G <= 0 || Lq <= 0 || Lk <= 0 || ldk < 0)
    return fail(DSV_EINVAL, "sparse_bwd: empty shape");
  if (!al16(q) || !al16(k) || !al16(v) || !al16(out) || !al16(dout) || !al16(dq) ||
      !al16(dk_acc) || !al16(dv_acc) || !al16(grp_rows))
    return fail(DSV_EINVAL, "sparse_bwd: pointers must be 16-byte aligned");
  if (!work) return fail(DSV_EINVAL, "sparse_bwd: null workspace");
  const float scale_log2 = scale * 1.4426950408889634f;
  return cuda_status(dsv_attn_bwd_tc_launch(q, k, v, out, dout, lse, grp_rows, grp_size, idx, ldk,
                                            kcount, kcount_hg, H, G, Lq, Lk, D, scale, scale_log2,
                                            dq, dk_acc, dv_acc, work, tile_grp,
                                            tile_grp ? n_groups : G, dq_tab, dq_n, dq_chunk,
                                            dkdv_out, dk_tab, dv_tab, kv_n, kv_chunk, conv_ws,
                                            S(stream)),
                     "sparse_bwd launch");
}

int dsv_sparse_bwd(const void* q, const void* k, const void* v, const void* out,
                   const void* dout, const float* lse, const int* grp_rows, const int* grp_size,
                   const int* idx, long long ldk, const int* kcount, const int* kcount_hg, int H,
                   int G, int Lq, int Lk, int D, float scale, void* dq, float* dk_acc,
                   float* dv_acc, unsigned* work, const int* tile_grp, int n_groups,
                   const long long* dq_tab, int dq_n, int dq_chunk, void* stream) {
  return dsv_sparse_bwd_convert(q, k, v, out, dout, lse, grp_rows, grp_size, idx, ldk, kcount,
                                kcount_hg, H, G, Lq, Lk, D, scale, dq, dk_acc, dv_acc, work,
                                tile_grp, n_groups, dq_tab, dq_n, dq_chunk, nullptr, nullptr,
                                nullptr, 0, 0, nullptr, stream);
}

int dsv_rows_fwd(const void* q, const void* k, const void* v, const long long* ptr,
                 const int* cols, int H, int Lq, int Lk, int D, float scale, int in_dtype,
                 float* out, float* lse, void* stream) {
  if (D < 1 || D > 256) return fail(DSV_EUNSUPPORTED, "rows_fwd: head dim %d outside [1, 256]", D);
  if (H <= 0 || Lq <= 0 || Lk <= 0) return fail(DSV_EINVAL, "rows_fwd: empty shape");
  return cuda_status(dsv_rows_fwd_launch(q, k, v, ptr, cols, H, Lq, Lk, D, scale,
                                         in_dtype == DSV_DTYPE_BF16, out, lse, S(stream)),
                     "rows_fwd launch");
}

int dsv_rows_bwd(const void* q, const void* k, const void* v, const float* out, const float* lse,
                 const void* dout, const long long* ptr, const int* cols, int H, int Lq, int Lk,
                 int D, float scale, int in_dtype, float* dq, float* dk_acc, float* dv_acc,
                 void* stream) {
  if (D < 1 || D > 256) return fail(DSV_EUNSUPPORTED, "rows_bwd: head dim %d outside [1, 256]", D);
  if (H <= 0 || Lq <= 0 || Lk <= 0) return fail(DSV_EINVAL, "rows_bwd: empty shape");
  return cuda_status(dsv_rows_bwd_launch(q, k, v, out, lse, dout, ptr, cols, H, Lq, Lk, D, scale,
                                         in_dtype == DSV_DTYPE_BF16, dq, dk_acc, dv_acc, S(stream)),
                     "rows_bwd launch");
}

int dsv_f32_to_bf16_rows(const float* in, int H, int L, int D, const long long* tab, int n,
                         int chunk, void* stream) {
  if (D != 64 && D != 128) return fail(DSV_EUNSUPPORTED, "f32_to_bf16_rows: D must be 64 or 128");
  if (!in || !tab || n < 1 || chunk < 1 || (long long)n * chunk < L)
    return fail(DSV_EINVAL, "f32_to_bf16_rows: bad arguments");
  return cuda_status(dsv_f32_to_bf16_rows_launch(in, H, L, D, tab, n, chunk, S(stream)),
                     "f32_to_bf16_rows launch");
}

int dsv_f32_to_bf16(const float* in, void* out, long long n, void* stream) {
  return cuda_status(dsv_f32_to_bf16_launch(in, out, n, S(stream)), "f32_to_bf16 launch");
}

int dsv_ring_lse_merge(float* acc, const float* lse_in, float* lse_out, const void* part,
                       const float* lse_part, long long rows, int D, int first, void* out,
                       void* stream) {
  if (rows < 0 || (D != 64 && D != 128)) return fail(DSV_EINVAL, "ring_lse_merge: D must be 64 or 128");
  if (!acc || !lse_out || !part || !lse_part || (!first && !lse_in))
    return fail(DSV_EINVAL, "ring_lse_merge: null operand");
  if (!al16(acc) || !al16(part) || (out && !al16(out)))
    return fail(DSV_EINVAL, "ring_lse_merge: rows must be 16-byte aligned");
  return cuda_status(dsv_lse_merge_launch(acc, lse_in, lse_out, part, lse_part, rows, D, first, out,
                                          S(stream)), "ring_lse_merge launch");
}

int dsv_ring_accum_bf16(float* acc, const void* x, long long n, int first, void* out, void* stream) {
  if (n < 0 || n % 8) return fail(DSV_EINVAL, "ring_accum_bf16: n must be a multiple of 8");
  if (!al16(acc) || !al16(x) || (out && !al16(out)))
    return fail(DSV_EINVAL, "ring_accum_bf16: operands must be 16-byte aligned");
  return cuda_status(dsv_accum_bf16_launch(acc, x, n, first, out, S(stream)), "ring_accum_bf16 launch");
}

int dsv_ring_accum_f32(float* acc, float* part, long long n, int first, void* stream) {
  if (n < 0 || n % 4) return fail(DSV_EINVAL, "ring_accum_f32: n must be a multiple of 4");
  if (!al16(acc) || !al16(part)) return fail(DSV_EINVAL, "ring_accum_f32: operands must be 16-byte aligned");
  return cuda_status(dsv_accum_f32_launch(acc, part, n, first, S(stream)), "ring_accum_f32 launch");
}

}  // extern "C"

// ------------------------------------------------------------ gather rows
namespace {
// one warp per row; 16-byte vectors when every row start is 16-byte aligned
template <bool kVec>
__global__ void __launch_bounds__(256)
gather_rows_kernel(const uint8_t* __restrict__ src, long long sstride, const int* __restrict__ rows,
                   int n, int row_bytes, uint8_t* __restrict__ out, long long ostride) {
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < n; r += (long long)gridDim.x * 8) {
    const uint8_t* s = src + (long long)rows[r] * sstride;
    uint8_t* o = out + r * ostride;
    if constexpr (kVec) {
      for (int w = lane; w < row_bytes / 16; w += 32)
        reinterpret_cast<uint4*>(o)[w] = __ldg(reinterpret_cast<const uint4*>(s) + w);
    } else {
      for (int w = lane; w < row_bytes / 4; w += 32)
        reinterpret_cast<uint32_t*>(o)[w] = __ldg(reinterpret_cast<const uint32_t*>(s) + w);
    }
  }
}
}  // namespace

// Job-table copy: blockIdx.x = job, blockIdx.y = split; each thread moves 16-byte
// chunks, four in flight. HBM- or NVLink-bound; the stores may target peer memory.
__global__ void __launch_bounds__(256) copy_jobs_kernel(const dsv_copy_job* __restrict__ jobs) {
  const dsv_copy_job j = jobs[blockIdx.x];
  const uint32_t cpr = (uint32_t)(j.row_bytes >> 4);
  const uint32_t total = (uint32_t)j.rows * cpr;
  const uint32_t step = gridDim.y * blockDim.x;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(j.src);
  uint8_t* dst = reinterpret_cast<uint8_t*>(j.dst);
  auto saddr = [&](uint32_t c) {
    const uint32_t r = c / cpr, w = c - r * cpr;
    return reinterpret_cast<const uint4*>(src + (long long)r * j.src_stride + (w << 4));
  };
  auto daddr = [&](uint32_t c) {
    const uint32_t r = c / cpr, w = c - r * cpr;
    return reinterpret_cast<uint4*>(dst + (long long)r * j.dst_stride + (w << 4));
  };
  uint32_t c = blockIdx.y * blockDim.x + threadIdx.x;
  for (; c + 3 * step < total; c += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(saddr(c + u * step));
#pragma unroll
    for (int u = 0; u < 4; ++u) *daddr(c + u * step) = v[u];
  }
  for (; c < total; c += step) *daddr(c) = __ldcs(saddr(c));
}

int dsv_debug_timeline_copy(void* dst, int bytes);
int dsv_debug_select_timeline_copy(void* dst, int bytes);
extern "C" int dsv_debug_select_timeline(void* host_dst, int bytes) {
  if (!host_dst || bytes <= 0) return fail(DSV_EINVAL, "debug_select_timeline: bad buffer");
  return dsv_debug_select_timeline_copy(host_dst, bytes);
}
extern "C" int dsv_debug_timeline(void* host_dst, int bytes) {
  if (!host_dst || bytes <= 0) return fail(DSV_EINVAL, "debug_timeline: bad buffer");
  return dsv_debug_timeline_copy(host_dst, bytes);
}

extern "C" int dsv_pred_pass(int stage, const double* q_lr, const double* k_lr, const void* target,
                             int target_dtype, long long ldt, int R, int n_keys, int r, const double* uw,
                             double* out, void* stream) {
  if (stage < 0 || stage > 2) return fail(DSV_EINVAL, "pred_pass: stage must be 0, 1 or 2");
  if (R < 1 || n_keys < 1 || r < 1 || r > 64 || ldt < n_keys) return fail(DSV_EINVAL, "pred_pass: bad shape");
  if (target_dtype != DSV_DTYPE_F32 && target_dtype != DSV_DTYPE_F64)
    return fail(DSV_EINVAL, "pred_pass: target must be fp32 or fp64");
  if (stage > 0 && !uw) return fail(DSV_EINVAL, "pred_pass: stages 1-2 need the row coefficients");
  return cuda_status(dsv_pred_pass_launch(stage, q_lr, k_lr, target, target_dtype == DSV_DTYPE_F64,
                                          ldt, R, n_keys, r, uw, out, S(stream)),
                     "pred_pass launch");
}

extern "C" int dsv_varint_index_bytes(const int* idx, long long ld, const int* counts, int k_uniform,
                                      int rows, long long* out_len, int* err, void* stream) {
  if (rows < 0 || ld < 0 || (!counts && k_uniform < 0) || !err) return fail(DSV_EINVAL, "varint_index_bytes: bad arguments");
  return cuda_status(dsv_varint_launch(0, idx, ld, counts, k_uniform, rows, out_len, nullptr, err, S(stream)),
                     "varint_index_bytes launch");
}

extern "C" int dsv_varint_encode(const int* idx, long long ld, const int* counts, int k_uniform, int rows,
                                 const long long* row_off, unsigned char* out, int* err, void* stream) {
  if (rows < 0 || ld < 0 || (!counts && k_uniform < 0) || !err || !out) return fail(DSV_EINVAL, "varint_encode: bad arguments");
  return cuda_status(dsv_varint_launch(1, idx, ld, counts, k_uniform, rows,
                                       const_cast<long long*>(row_off), out, err, S(stream)),
                     "varint_encode launch");
}

extern "C" int dsv_critical_counts(const float* scores, long long ld, int rows, int L,
                                   double sqrt_d, double theta, int* out, void* stream) {
  if (rows < 0 || L < 1 || ld < L) return fail(DSV_EINVAL, "critical_counts: bad shape");
  if (!(theta > 0.0 && theta <= 1.0)) return fail(DSV_EINVAL, "critical_counts: theta must lie in (0, 1]");
  if (!(sqrt_d > 0.0)) return fail(DSV_EINVAL, "critical_counts: sqrt_d must be positive");
  return cuda_status(dsv_critical_counts_launch(scores, ld, rows, L, sqrt_d, theta, out, S(stream)),
                     "critical_counts launch");
}

extern "C" int dsv_copy_jobs_threads(const dsv_copy_job* jobs, int njobs, int splits, int threads,
                                     void* stream) {
  if (njobs <= 0) return DSV_OK;
  if (!jobs || splits < 1 || splits > 1024 || (threads != 128 && threads != 256))
    return fail(DSV_EINVAL, "copy_jobs_threads: bad job table, split count or block size");
  dim3 grid(njobs, splits);
  copy_jobs_kernel<<<grid, threads, 0, S(stream)>>>(jobs);
  return cuda_status((int)cudaGetLastError(), "copy_jobs launch");
}

extern "C" int dsv_copy_jobs(const dsv_copy_job* jobs, int njobs, int splits, void* stream) {
  if (njobs <= 0) return DSV_OK;
  if (!jobs || splits < 1 || splits > 1024)
    return fail(DSV_EINVAL, "copy_jobs: bad job table or split count");
  dim3 grid(njobs, splits);
  copy_jobs_kernel<<<grid, 256, 0, S(stream)>>>(jobs);
  return cuda_status((int)cudaGetLastError(), "copy_jobs launch");
}

// ---------------------------------------------------------------- peer memory (NVLink)
// One buffer per rank, mapped into every peer process with CUDA IPC (public runtime API;
// replaces torch's private symmetric-memory module). The device barrier orders the copy
// kernels' peer writes: rank r stores its arrival epoch into slot r of every peer's slot
// array (system-scope release after a system fence), then waits until all of its own slots
// reached the epoch (acquire). Epochs live in device memory, so a captured graph's replays
// keep counting.
namespace {
__global__ void peer_barrier_kernel(unsigned* const* __restrict__ peer_slots,
                                    unsigned* __restrict__ my_slots, unsigned* __restrict__ epoch,
                                    int world, int rank) {
  // lane r signals peer r and waits for peer r, all lanes at once (world <= 32): a release
  // (fence.acq_rel.sys + relaxed store) orders every write issued before this kernel on the
  // stream — the exchange copies into peer memory — before the flag; the acquire loads make
  // the peers' writes visible before the kernels after this one. One thread storing and
  // polling the peers in turn measured 20-25 us per barrier.
  const int lane = threadIdx.x;
  const unsigned e = *epoch + 1u;
  if (lane < world) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(peer_slots[lane] + rank), "r"(e) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_slots + lane) : "memory");
    } while ((int)(v - e) < 0);
  }
  __syncwarp();
  if (lane == 0) *epoch = e;
}
}  // namespace

extern "C" int dsv_peer_alloc(long long bytes, void** ptr, void* handle) {
  if (bytes <= 0 || !ptr || !handle) return fail(DSV_EINVAL, "peer_alloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e != cudaSuccess) return cuda_status((int)e, "peer_alloc cudaMalloc");
  e = cudaMemset(p, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_status((int)e, "peer_alloc cudaIpcGetMemHandle");
  }
  *ptr = p;
  return DSV_OK;
}

extern "C" int dsv_peer_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return fail(DSV_EINVAL, "peer_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_status((int)cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess),
                     "peer_open cudaIpcOpenMemHandle");
}

extern "C" int dsv_peer_close(void* ptr) {
  return cuda_status((int)cudaIpcCloseMemHandle(ptr), "peer_close");
}

extern "C" int dsv_peer_free(void* ptr) { return cuda_status((int)cudaFree(ptr), "peer_free"); }

extern "C" int dsv_peer_barrier(unsigned* const* peer_slots, unsigned* my_slots, unsigned* epoch,
                                int world, int rank, void* stream) {
  if (world < 1 || world > 32 || rank < 0 || rank >= world || !peer_slots || !my_slots || !epoch)
    return fail(DSV_EINVAL, "peer_barrier: bad arguments (world 1..32)");
  peer_barrier_kernel<<<1, 32, 0, S(stream)>>>(peer_slots, my_slots, epoch, world, rank);
  return cuda_status((int)cudaGetLastError(), "peer_barrier launch");
}

// ---------------------------------------------------------------- selective KV (SCP) over NVLink
// Every rank of an SCP group keeps full-length per-head buffers [hs][L][D] (K, V bf16; dK, dV
// fp32) addressed by global token and mapped into its peers. The critical-key mark of this
// rank's span (bool [hs][L]) decides, per (head, key row) outside the own span, whether the
// row is pulled from its owner's buffer (forward) and whether its gradient rows are added
// into the owner's accumulators (backward). Counts never leave the device.
namespace {
template <bool kPush>
__global__ void __launch_bounds__(256)
scp_rows_kernel(const unsigned char* __restrict__ mark, int hs, int L, int span0, int span_len,
                const long long* __restrict__ peer_a, const long long* __restrict__ peer_b,
                void* __restrict__ own_a, void* __restrict__ own_b, int D,
                unsigned long long* __restrict__ count) {
  const long long nrows = (long long)hs * L;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  unsigned long long got = 0;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows;
       r += warps) {
    const int tok = (int)(r % L);
    if (!mark[r] || (tok >= span0 && tok < span0 + span_len)) continue;
    const int owner = tok / span_len;
    ++got;
    if (!kPush) {                 // K, V rows (bf16) from the owner into the own buffers
      const uint4* sa = reinterpret_cast<const uint4*>(peer_a[owner]) + r * D / 8;
      const uint4* sb = reinterpret_cast<const uint4*>(peer_b[owner]) + r * D / 8;
      uint4* da = reinterpret_cast<uint4*>(own_a) + r * D / 8;
      uint4* db = reinterpret_cast<uint4*>(own_b) + r * D / 8;
      for (int i = lane; i < D / 8; i += 32) { da[i] = sa[i]; db[i] = sb[i]; }
    } else {                      // dK, dV rows (fp32) added into the owner's accumulators
      const float4* sa = reinterpret_cast<const float4*>(own_a) + r * D / 4;
      const float4* sb = reinterpret_cast<const float4*>(own_b) + r * D / 4;
      float* da = reinterpret_cast<float*>(peer_a[owner]) + r * D;
      float* db = reinterpret_cast<float*>(peer_b[owner]) + r * D;
      for (int i = lane; i < D / 4; i += 32) {
        const float4 x = sa[i], y = sb[i];
        dsv::red_add_v4(da + 4 * i, x.x, x.y, x.z, x.w);
        dsv::red_add_v4(db + 4 * i, y.x, y.y, y.z, y.w);
      }
    }
  }
  if (count && lane == 0 && got) atomicAdd(count, got);
}
}  // namespace

extern "C" int dsv_scp_pull(const unsigned char* mark, int hs, int L, int span0, int span_len,
                            const long long* peer_k, const long long* peer_v, void* k_full,
                            void* v_full, int D, unsigned long long* count, void* stream) {
  if (hs <= 0 || L <= 0 || span_len <= 0 || L % span_len || D % 8 || !mark || !peer_k || !peer_v)
    return fail(DSV_EINVAL, "scp_pull: bad arguments");
  scp_rows_kernel<false><<<148 * 8, 256, 0, S(stream)>>>(mark, hs, L, span0, span_len, peer_k,
                                                         peer_v, k_full, v_full, D, count);
  return cuda_status((int)cudaGetLastError(), "scp_pull launch");
}

extern "C" int dsv_scp_push(const unsigned char* mark, int hs, int L, int span0, int span_len,
                            const long long* peer_dk, const long long* peer_dv, void* dk_full,
                            void* dv_full, int D, void* stream) {
  if (hs <= 0 || L <= 0 || span_len <= 0 || L % span_len || D % 4 || !mark || !peer_dk || !peer_dv)
    return fail(DSV_EINVAL, "scp_push: bad arguments");
  scp_rows_kernel<true><<<148 * 8, 256, 0, S(stream)>>>(mark, hs, L, span0, span_len, peer_dk,
                                                        peer_dv, dk_full, dv_full, D, nullptr);
  return cuda_status((int)cudaGetLastError(), "scp_push launch");
}

extern "C" int dsv_gather_rows(const void* src, long long src_stride, const int* rows, int n,
                               int row_bytes, void* out, long long out_stride, void* stream) {
  if (n <= 0) return DSV_OK;
  if (row_bytes % 4 || src_stride % 4 || out_stride % 4)
    return fail(DSV_EINVAL, "gather_rows: byte sizes must be multiples of 4");
  const bool vec = row_bytes % 16 == 0 && src_stride % 16 == 0 && out_stride % 16 == 0 &&
                   al16(src) && al16(out);
  const int blocks = (int)((n + 7) / 8 < 148 * 16 ? (n + 7) / 8 : 148 * 16);
  if (vec)
    gather_rows_kernel<true><<<blocks, 256, 0, S(stream)>>>((const uint8_t*)src, src_stride, rows, n,
                                                            row_bytes, (uint8_t*)out, out_stride);
  else
    gather_rows_kernel<false><<<blocks, 256, 0, S(stream)>>>((const uint8_t*)src, src_stride, rows, n,
                                                             row_bytes, (uint8_t*)out, out_stride);
  return cuda_status((int)cudaGetLastError(), "gather_rows launch");
}

// ---------------------------------------------------------------- fp64 precision path
namespace {
int pad_pow2(int L) {
  int p = 2;
  while (p < L) p <<= 1;
  return p;
}
constexpr size_t kSortSmemMax = 200 * 1024;
constexpr int kSortScratchCtas = 64;
}  // namespace

extern "C" int dsv_gemm_f64(const double* A, long long sam, long long sat, long long a_bs,
                            const double* B, long long sbt, long long sbn, long long b_bs,
                            double* C, long long ldc, long long c_bs, int M, int N, int K,
                            int nbatch, double div, void* stream) {
  if (M <= 0 || N <= 0 || nbatch <= 0) return fail(DSV_EINVAL, "gemm_f64: empty shape");
  if (K < 0) return fail(DSV_EINVAL, "gemm_f64: negative inner dimension");
  if (!A || !B || !C) return fail(DSV_EINVAL, "gemm_f64: null operand");
  if (!(div != 0.0)) return fail(DSV_EINVAL, "gemm_f64: zero divisor");
  return cuda_status(dsv_gemm_f64_launch(A, sam, sat, a_bs, B, sbt, sbn, b_bs, C, ldc, c_bs, M, N,
                                         K, nbatch, div, S(stream)), "gemm_f64 launch");
}

extern "C" int dsv_softmax_rows_f64(double* x, long long ld, int R, int N, void* stream) {
  if (R <= 0 || N <= 0 || ld < N) return fail(DSV_EINVAL, "softmax_rows_f64: bad shape");
  return cuda_status(dsv_softmax_rows_f64_launch(x, ld, R, N, S(stream)), "softmax_rows_f64 launch");
}

extern "C" int dsv_topk_f64(const double* Sc, long long lds, int R, int L, const int* k_per,
                            int rows_per_k, int* out, long long ldo, double* thr, void* stream) {
  if (R <= 0 || L <= 0 || lds < L || rows_per_k <= 0) return fail(DSV_EINVAL, "topk_f64: bad shape");
  if (!Sc || !k_per || !out || !thr) return fail(DSV_EINVAL, "topk_f64: null operand");
  return cuda_status(dsv_topk_f64_launch(Sc, lds, R, L, k_per, rows_per_k, out, ldo, thr, S(stream)),
                     "topk_f64 launch");
}

extern "C" int dsv_rows_fwd_f64(const double* q, const double* k, const double* v,
                                const long long* ptr, const int* cols, int H, int Lq, int Lk,
                                int Dk, int Dv, double scale, double* out, double* lse,
                                void* stream) {
  if (Dk < 1 || Dk > 256 || Dv < 1 || Dv > 256)
    return fail(DSV_EUNSUPPORTED, "rows_fwd_f64: head dims (%d, %d) outside [1, 256]", Dk, Dv);
  if (H <= 0 || Lq <= 0 || Lk <= 0) return fail(DSV_EINVAL, "rows_fwd_f64: empty shape");
  return cuda_status(dsv_rows_fwd_f64_launch(q, k, v, ptr, cols, H, Lq, Lk, Dk, Dv, scale, out, lse,
                                             S(stream)), "rows_fwd_f64 launch");
}

extern "C" int dsv_rows_bwd_f64(const double* q, const double* k, const double* v,
                                const double* out, const double* lse, const double* dout,
                                const long long* ptr, const int* cols, int H, int Lq, int Lk,
                                int Dk, int Dv, double scale, double* dq, double* dk_acc,
                                double* dv_acc, void* stream) {
  if (Dk < 1 || Dk > 256 || Dv < 1 || Dv > 256)
    return fail(DSV_EUNSUPPORTED, "rows_bwd_f64: head dims (%d, %d) outside [1, 256]", Dk, Dv);
  if (H <= 0 || Lq <= 0 || Lk <= 0) return fail(DSV_EINVAL, "rows_bwd_f64: empty shape");
  return cuda_status(dsv_rows_bwd_f64_launch(q, k, v, out, lse, dout, ptr, cols, H, Lq, Lk, Dk, Dv,
                                             scale, dq, dk_acc, dv_acc, S(stream)),
                     "rows_bwd_f64 launch");
}

extern "C" long long dsv_sorted_stats_scratch_bytes(int R, int L) {
  if (R <= 0 || L <= 0) return 0;
  const int Lpad = pad_pow2(L);
  if (dsv_sorted_stats_smem(Lpad) <= kSortSmemMax) return 0;
  const int ctas = R < kSortScratchCtas ? R : kSortScratchCtas;
  return (long long)ctas * Lpad * 12;
}

extern "C" int dsv_sorted_stats_f64(const double* Sc, long long lds, int R, int L, double theta,
                                    double eps, int top_n, int* n_keep, double* topmass,
                                    void* scratch, long long scratch_bytes, void* stream) {
  if (R <= 0 || L <= 0 || lds < L) return fail(DSV_EINVAL, "sorted_stats_f64: bad shape");
  if (L > (1 << 30)) return fail(DSV_EUNSUPPORTED, "sorted_stats_f64: row too long");
  const int Lpad = pad_pow2(L);
  const long long need = dsv_sorted_stats_scratch_bytes(R, L);
  if (need > 0 && (!scratch || scratch_bytes < need))
    return fail(DSV_EINVAL, "sorted_stats_f64: rows of %d keys need %lld bytes of scratch", L, need);
  const int ctas = need > 0 ? (R < kSortScratchCtas ? R : kSortScratchCtas) : 0;
  return cuda_status(dsv_sorted_stats_launch(Sc, lds, R, L, Lpad, theta, eps, top_n, n_keep, topmass,
                                             need > 0 ? scratch : nullptr, ctas, S(stream)),
                     "sorted_stats_f64 launch");
}

extern "C" int dsv_histogram_f64(const double* Sc, long long lds, int R, int N, const double* edges,
                                 int nb, unsigned long long* counts, void* stream) {
  if (R < 0 || N < 0 || nb < 1 || nb > 16384) return fail(DSV_EINVAL, "histogram_f64: bad shape");
  if (R == 0 || N == 0) return DSV_OK;
  return cuda_status(dsv_histogram_f64_launch(Sc, lds, R, N, edges, nb, counts, S(stream)),
                     "histogram_f64 launch");
}

extern "C" int dsv_set_stats_f64(const double* Sc, long long lds, int Q, const long long* est_ptr,
                                 const int* est_cols, const long long* ora_ptr,
                                 const int* ora_cols, int* inter, double* est_mass,
                                 double* ora_mass, void* stream) {
  if (Q <= 0) return fail(DSV_EINVAL, "set_stats_f64: no queries");
  if (!Sc || !est_ptr || !ora_ptr || !inter || !est_mass || !ora_mass)
    return fail(DSV_EINVAL, "set_stats_f64: null operand");
  return cuda_status(dsv_set_stats_f64_launch(Sc, lds, Q, est_ptr, est_cols, ora_ptr, ora_cols, inter,
                                              est_mass, ora_mass, S(stream)), "set_stats_f64 launch");
}
