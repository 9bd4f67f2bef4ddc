/*
 * dsv.h — C ABI of the B200-native DSV dynamic-sparsity attention path.
 *
 * Every entry point is `extern "C"`, takes plain device pointers, element
 * strides and a cudaStream_t (as void*), launches asynchronously on that
 * stream and returns an int status (DSV_OK or DSV_E*). Nothing here allocates
 * device memory or throws; callers own every buffer. Pointers are device
 * pointers unless stated otherwise.
 *
 * Reference interfaces replaced (reference = /root/reference/pkg/src/dynsparse):
 *   dsv_project          predictor.py:94-100   project(x, w)            (X W, both sides, all heads)
 *   dsv_gemm_bf16        predictor.py:238-239  + selection.py:149 tile product (tcgen05 GEMM)
 *   dsv_proxy_scores     grouping.py:184-193 + selection.py:149 proxy-row scores (tcgen05)
 *   dsv_scores_f32       selection.py:149/204/222 q_lr @ k_lr.T (fp32, CUDA cores)
 *   dsv_topk             selection.py:118-175  streaming_topk / :178-242 twopass_select
 *                        (exact top-k, ties -> lower index, ascending emit, k-th threshold)
 *   dsv_sparse_fwd       attention.py:153-187  sparse_attention (uniform/group-shared sets)
 *                        grouping.py:196-216   grouped_sparse_attention
 *   dsv_sparse_bwd       trainer.py:110-117    autograd of the sparse attention (dQ, dK, dV)
 *   dsv_sparse_bwd_convert  the same, dK / dV also converted to the caller's dtype (bf16)
 *                        in the kernel's tail (trainer.py:110-117 returns them in it)
 *   dsv_select_fused     grouping.py:184-193 + selection.py:118-175 proxy scores and exact
 *                        top-k fused (no score matrix); dsv_select_fused_workspace_size /
 *                        dsv_select_fused_max_clusters size its workspace and key split
 *   dsv_rows_fwd/_bwd    attention.py:176-183  ragged per-query index sets (CSR)
 *   dsv_gather_rows      cpsim.py:147-156/195-216 pack/unpack of head slices and KV rows
 *   dsv_pred_pass        predictor.py:103-194 (predictor training step: row statistics and the
 *                        two gradient contractions, streaming the target matrix)
 *   dsv_varint_*         serialize.py:119-151 encode_index_sets (varint-delta wire format)
 *   dsv_critical_counts  profiler.py:48-79 + attention.py:118-140 (sampled sparsity profiler:
 *                        critical-KV prefix length per scored row)
 *   dsv_copy_jobs        cpsim.py:147-156/284-299 HCP head exchange written straight into
 *                        the owners' buffers (peer pointers over NVLink); _threads: the
 *                        same with 128-thread blocks (runs beside a persistent kernel)
 *   dsv_peer_*           cpsim.py:125-161/284-299 transport: CUDA-IPC peer buffers and the
 *                        device barrier that orders each exchange phase
 *   dsv_scp_pull/_push   cpsim.py:164-216 selective_comm_scp (critical rows pulled from the
 *                        owners; their gradients added back)
 *   dsv_ring_*           ring KV pass for dense residual heads under SCP (no reference
 *                        counterpart; dense semantics of attention.py:95-109)
 * Reference-precision (fp64) path for host fp64/fp32 callers (validate.py:10-25 computes in
 * the caller's dtype):
 *   dsv_gemm_f64         predictor.py:94-100 project; selection.py:149/204/222 score tiles;
 *                        attention.py:112-115 logits (q @ k.T / sqrt(d))
 *   dsv_softmax_rows_f64 attention.py:88-92 _stable_softmax_rows
 *   dsv_topk_f64         selection.py:118-175 / 178-242 on fp64 scores (fp64 thresholds)
 *   dsv_rows_*_f64       attention.py:95-109 / 153-187 and trainer.py:110-117 in fp64
 *   dsv_sorted_stats_f64 attention.py:118-140 critical_kv_oracle prefix length;
 *                        attention.py:208-212 analyze_distribution top-fraction mass
 *   dsv_histogram_f64    attention.py:214-216 np.histogram
 *   dsv_set_stats_f64    predictor.py:262-281 prediction_accuracy (recall / mass coverage)
 */
#ifndef DSV_H_
#define DSV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSV_OK 0
#define DSV_EINVAL 1       /* invalid argument: shape, k outside [1, L], alignment      */
#define DSV_EUNSUPPORTED 2 /* outside the kernels' envelope (e.g. head dim not 64/128) */
#define DSV_ECUDA 3        /* CUDA runtime / launch failure                             */

#define DSV_DTYPE_F32 0
#define DSV_DTYPE_BF16 1
#define DSV_DTYPE_F64 2

/* Library version (major*10000 + minor*100 + patch) and last error text (thread-local). */
int dsv_version(void);
const char* dsv_last_error(void);

/* Number of streaming multiprocessors of the current device (0 if none). */
int dsv_device_sm_count(void);

/* C[b] = A[b] . B[b]^T on tcgen05 (bf16 in, fp32 accumulate).
 * A: [nbatch][M][K] bf16, row stride lda (elements), batch stride a_bs;
 * B: [nbatch][N][K] bf16, row stride ldb, batch stride b_bs;
 * C: [nbatch][M][N], dtype DSV_DTYPE_F32 or DSV_DTYPE_BF16, row stride ldc, batch stride c_bs.
 * Strides in bytes must be multiples of 16; K is zero-padded to 64 internally. */
int dsv_gemm_bf16(const void* A, long long lda, long long a_bs, const void* B, long long ldb,
                  long long b_bs, void* C, int c_dtype, long long ldc, long long c_bs,
                  int M, int N, int K, int nbatch, void* stream);

/* Predictor projection (K1a): out[L][n_out] = X[L][d_model] . Wt[n_out][d_model]^T, bf16.
 * Wt stacks the per-head W_q^T then W_k^T rows: row (side*H + h)*r + j. */
int dsv_project(const void* X, const void* Wt, void* out, int L, int d_model, int n_out,
                void* stream);

/* K1b proxy scores on tcgen05: out[h][g][l] = sum_t q_prox[h][g][t] * k_lr[h][l][t] (fp32),
 * bf16 inputs with rank r = 16; q_prox row stride ldq / head stride q_bs, k_lr row stride ldk /
 * head stride k_bs (elements), out row stride ldo / head stride o_bs. Stores are coalesced. */
int dsv_proxy_scores(const void* q_prox, long long ldq, long long q_bs, const void* k_lr,
                     long long ldk, long long k_bs, float* out, long long ldo, long long o_bs,
                     int H, int G, int L, int r, void* stream);

/* fp32 scores C[b][i][j] = sum_t A[b][i][t] * B[b][j][t] (any r >= 1), deterministic
 * fmaf order t = 0..r-1. a_dtype: DSV_DTYPE_F32 or DSV_DTYPE_BF16 (for both A and B). */
int dsv_scores_f32(const void* A, long long lda, long long a_bs, const void* B, long long ldb,
                   long long b_bs, float* C, long long ldc, long long c_bs, int nbatch, int R,
                   int Lk, int r, int in_dtype, void* stream);

/* K1b + K2 fused: exact top-k of the proxy scores q_prox[h][g] . k_lr[h][l] (bf16, rank
 * r <= 64) without materialising them. Same scores (same tcgen05 sequence) and the same
 * selection semantics as dsv_gemm_bf16 (fp32 out) followed by dsv_topk with
 * rows_per_head = G: out_idx[h*G + g][0..k_h) ascending, out_thr[h*G + g].
 * split: CTAs per 128-row tile splitting the key range (cluster), 0 = automatic.
 * workspace (dsv_select_fused_workspace_size bytes for the largest k, or NULL): enables the single-pass
 * mode — sample passes pick a key band around the k-th score, one collect pass writes a
 * per-row bitmap of the keys at or above the band plus the band entries, a finish kernel
 * selects the k-th score among the band and emits from the bitmap; row tiles whose band
 * missed it re-run the exact multi-pass algorithm (same results either way). NULL: the
 * multi-pass algorithm only (sample, band refinement, candidates, emission passes).
 * The workspace size is 0 where the single pass is not worthwhile (the band would hold too
 * large a share of the keys, or need more than 1 GiB): pass NULL then. */
long long dsv_select_fused_workspace_size(int H, int G, int L, int k_max, int split);
/* Clusters of S dsv_select_fused CTAs resident at once on the current device (occupancy
 * query, cached per device); the automatic split counts waves with it. 0 = no device. */
int dsv_select_fused_max_clusters(int S);
int dsv_select_fused(const void* q_prox, long long ldq, long long q_bs, const void* k_lr,
                     long long ldk, long long k_bs, int H, int G, int L, int r,
                     const int* k_per_head, int* out_idx, long long out_ld, float* out_thr,
                     int split, void* workspace, long long ws_bytes, void* stream);

/* Exact top-k per row of an fp32 score matrix (K2).
 * scores: [rows][ld] fp32; row r uses k = k_per_head[r / rows_per_head] (1 <= k <= L).
 * out_idx: [rows][out_ld] int32 ascending column ids (first k entries written);
 * out_thr: [rows] fp32 k-th largest score. Ties at the threshold keep lower ids;
 * -0.0 == +0.0. */
int dsv_topk(const float* scores, long long ld, int rows, int L, const int* k_per_head,
             int rows_per_head, int* out_idx, long long out_ld, float* out_thr, void* stream);

/* Group-tiled sparse attention forward (K3f), bf16, head dim D in {64, 128}.
 * q: [H][Lq][D], k, v: [H][Lk][D]; grp_rows: [G][128] int32 member token ids (entries past
 * grp_size[g] repeat a member); idx: [H][G][ldk] int32 ascending key ids with kcount[h] valid
 * entries per row (1..ldk), or, when kcount_hg != NULL, kcount_hg[h*G + g] valid entries;
 * ldk = 0: every (head, group) reads the same list (dense chunks of the ring KV pass).
 * out: [H][Lq][D] bf16; lse: [H][Lq] fp32, log2 domain of the scaled logits.
 * work: device workspace of >= H*G + 2 words (the persistent kernel's list of tiles that
 * need the exact-max pass and its tile counter; contents need no initialisation).
 * zero_buf (optional): zero_floats fp32 set to 0 while the kernel runs (the backward's dK/dV
 * accumulators; the writes hide under the gather-bound forward).
 * tile_grp (optional, int32 [G]): the G tiles are 128-query pieces of n_groups voxel groups
 * (grouping.py:22-32 ladder shapes up to 8x8x8 = 512 queries); tile g reads index row
 * tile_grp[g] of idx [H][n_groups][ldk] (and kcount_hg [H][n_groups]). NULL: tile = group.
 * o_tab (optional, int64 device table [H][o_n] of addresses): each output row (h, tok) is
 * also stored at o_tab[h*o_n + tok/o_chunk] + (tok % o_chunk) * D elements — the token
 * owners' buffers under head-parallel CP (peer-mapped), so the output redistribution rides
 * on the epilogue's stores (cpsim.py:284-299). dsv_sparse_bwd's dq_tab does the same for dQ
 * (dQ is then written only there). */
int dsv_sparse_fwd(const void* q, const void* k, const void* v, const int* grp_rows,
                   const int* grp_size, const int* idx, long long ldk, const int* kcount,
                   const int* kcount_hg, int H, int G, int Lq, int Lk, int D, float scale,
                   void* out, float* lse, unsigned* work, long long work_words, float* zero_buf,
                   long long zero_floats, const int* tile_grp, int n_groups,
                   const long long* o_tab, int o_n, int o_chunk, void* stream);

/* Backward (K3b). dout: [H][Lq][D] bf16, out/lse from dsv_sparse_fwd. dq: [H][Lq][D] bf16
 * (every query of a group is written); dk_acc, dv_acc: [H][Lk][D] fp32 accumulators that the
 * caller zeroes; contributions are added atomically. work: one device word (the persistent
 * CTAs' tile counter; reset by the call). */
int dsv_sparse_bwd(const void* q, const void* k, const void* v, const void* out,
                   const void* dout, const float* lse, const int* grp_rows, const int* grp_size,
                   const int* idx, long long ldk, const int* kcount, const int* kcount_hg, int H,
                   int G, int Lq, int Lk, int D, float scale, void* dq, float* dk_acc,
                   float* dv_acc, unsigned* work, const int* tile_grp, int n_groups,
                   const long long* dq_tab, int dq_n, int dq_chunk, void* stream);
/* dsv_sparse_bwd plus the dK/dV conversion to bf16 in the kernel's tail: once the tile queue
 * is exhausted the persistent CTAs convert slices of every head whose tiles are all done
 * (what a separate conversion pass over the accumulators would do, without the CTAs idling
 * while the last tiles finish). Outputs: dkdv_out bf16 [2][H][Lk][D] (dK then dV), or the
 * token owners' rows dk_tab / dv_tab[h*kv_n + tok/kv_chunk] + (tok % kv_chunk)*D.
 * conv_ws: H + 1 device ints (zeroed by the call). conv_ws == NULL: no conversion. */
int dsv_sparse_bwd_convert(const void* q, const void* k, const void* v, const void* out,
                           const void* dout, const float* lse, const int* grp_rows,
                           const int* grp_size, const int* idx, long long ldk, const int* kcount,
                           const int* kcount_hg, int H, int G, int Lq, int Lk, int D, float scale,
                           void* dq, float* dk_acc, float* dv_acc, unsigned* work,
                           const int* tile_grp, int n_groups, const long long* dq_tab, int dq_n,
                           int dq_chunk, void* dkdv_out, const long long* dk_tab,
                           const long long* dv_tab, int kv_n, int kv_chunk, int* conv_ws,
                           void* stream);

/* Ragged per-(head, query) CSR sparse attention on CUDA cores (fp32 math), any D <= 256.
 * ptr: [H*Lq + 1] int64 offsets into cols (int32 key ids); cols == NULL selects every key
 * (dense attention, ptr unused). out: [H][Lq][D] fp32,
 * lse: [H][Lq] fp32 natural log of the scaled logits. in_dtype: F32 or BF16 (q/k/v/dout). */
int dsv_rows_fwd(const void* q, const void* k, const void* v, const long long* ptr,
                 const int* cols, int H, int Lq, int Lk, int D, float scale, int in_dtype,
                 float* out, float* lse, void* stream);
int dsv_rows_bwd(const void* q, const void* k, const void* v, const float* out, const float* lse,
                 const void* dout, const long long* ptr, const int* cols, int H, int Lq, int Lk,
                 int D, float scale, int in_dtype, float* dq, float* dk_acc, float* dv_acc,
                 void* stream);

/* out[i] = src[rows[i]] for n rows of row_bytes bytes (row strides in bytes, multiples of 4). */
int dsv_gather_rows(const void* src, long long src_stride, const int* rows, int n,
                    int row_bytes, void* out, long long out_stride, void* stream);

/* Predictor training passes over the target T [R, S] (row stride ldt elements, dtype
 * DSV_DTYPE_F32 or DSV_DTYPE_F64) with A_hat = Q_lr K_lr^T recomputed in fp64
 * (Q_lr [R, r], K_lr [S, r] fp64 row-major, r <= 64):
 *   stage 0: out [R, 4] = per row (|a|^2, |t|^2, a.t, |a - t|^2)
 *   stage 1: out [R, r] = G K_lr      with G[i, :] = uw[i, 0] T[i, :] + uw[i, 1] A_hat[i, :]
 *   stage 2: out [S, r] = G^T Q_lr    (uw [R, 2] fp64; unused by stage 0) */
int dsv_pred_pass(int stage, const double* q_lr, const double* k_lr, const void* target,
                  int target_dtype, long long ldt, int R, int S, int r, const double* uw,
                  double* out, void* stream);

/* Varint-delta index-set encoding (serialize.py:119-151). Rows r of idx (row stride ld
 * elements) hold counts[r] (or k_uniform when counts == NULL) strictly increasing indices.
 * dsv_varint_index_bytes: out_len[r] = encoded bytes of row r (count varint + deltas).
 * dsv_varint_encode: writes row r's bytes at out + row_off[r] (the caller places the
 * varint(n_rows) header and the scan of out_len). *err |= 1 for a negative first index,
 * |= 2 for a non-increasing row (the reference raises ValueError). */
int dsv_varint_index_bytes(const int* idx, long long ld, const int* counts, int k_uniform, int rows,
                           long long* out_len, int* err, void* stream);
int dsv_varint_encode(const int* idx, long long ld, const int* counts, int k_uniform, int rows,
                      const long long* row_off, unsigned char* out, int* err, void* stream);

/* Critical-KV mass counts (profiler.py:48-79, attention.py:118-140): for each row of fp32
 * raw scores x (q . k, unscaled), p = softmax(x / sqrt_d) in fp64, and out[row] = the
 * length of the shortest descending-p prefix (ties toward the lower index) whose mass
 * reaches min(theta, sum p) - 1e-9. theta in (0, 1]. */
int dsv_critical_counts(const float* scores, long long ld, int rows, int L, double sqrt_d,
                        double theta, int* out, void* stream);

/* One strided copy: `rows` rows of `row_bytes` bytes from src (+src_stride per row) to
 * dst (+dst_stride per row). Six int64 fields, so a [njobs, 6] int64 device array is a
 * job table. src/dst may be peer-mapped device pointers (CUDA IPC / symmetric memory). */
typedef struct dsv_copy_job {
  int64_t src;
  int64_t dst;
  int64_t src_stride;
  int64_t dst_stride;
  int64_t rows;
  int64_t row_bytes;
} dsv_copy_job;

/* Run njobs copies from a DEVICE job table in one launch; every address, stride and
 * row_bytes must be a multiple of 16 and rows * row_bytes / 16 < 2^31 per job.
 * `splits` blocks cooperate on each job (1..1024). */
int dsv_copy_jobs(const dsv_copy_job* jobs, int njobs, int splits, void* stream);
/* The same with `threads` (128 or 256) per block: 128-thread blocks (4 K registers) fit next
 * to a persistent attention kernel's CTA on its SM, so a copy can run under it. */
int dsv_copy_jobs_threads(const dsv_copy_job* jobs, int njobs, int splits, int threads,
                          void* stream);

/* Selective KV gathering (SCP, cpsim.py:164-216) over NVLink, one-sided: each rank of an SCP
 * group holds full-length buffers [hs][L][D] addressed by global token (K, V bf16; dK, dV
 * fp32) whose addresses in this process are peer_*[g] for group member g (member g owns the
 * tokens [g*span_len, (g+1)*span_len)). mark (bool [hs][L]) = the keys this rank's span
 * selected. dsv_scp_pull copies every marked (head, key) row outside [span0, span0+span_len)
 * from its owner's K/V buffers into k_full / v_full (count += rows, optional);
 * dsv_scp_push adds the same rows of dk_full / dv_full into the owners' accumulators
 * (red.add over NVLink). No host round trip: graph-capturable. */
int dsv_scp_pull(const unsigned char* mark, int hs, int L, int span0, int span_len,
                 const long long* peer_k, const long long* peer_v, void* k_full, void* v_full,
                 int D, unsigned long long* count, void* stream);
int dsv_scp_push(const unsigned char* mark, int hs, int L, int span0, int span_len,
                 const long long* peer_dk, const long long* peer_dv, void* dk_full, void* dv_full,
                 int D, void* stream);

/* fp32 [H][L][D] rows -> bf16 rows at tab[h*n + tok/chunk] + (tok % chunk) * D (D = 64 or
 * 128): the dK / dV conversion writing straight into the token owners' buffers. */
int dsv_f32_to_bf16_rows(const float* in, int H, int L, int D, const long long* tab, int n,
                         int chunk, void* stream);

/* Peer memory for the NVLink exchanges (one process per GPU): dsv_peer_alloc returns a
 * zeroed device buffer and its 64-byte CUDA IPC handle, which a peer process maps with
 * dsv_peer_open (unmap: dsv_peer_close; owner: dsv_peer_free). dsv_peer_barrier is a
 * device-side barrier over those buffers: peer_slots is a DEVICE array of `world` pointers
 * (rank r's slot array as mapped here), my_slots this rank's own array of `world` u32 and
 * epoch a u32 device counter; all ranks must issue their barriers in the same order. Writes
 * of earlier kernels on `stream` (including peer writes) are visible to every rank's later
 * kernels. Graph-capturable (the epoch advances on the device). */
int dsv_peer_alloc(long long bytes, void** ptr, void* handle);
int dsv_peer_open(const void* handle, void** ptr);
int dsv_peer_close(void* ptr);
int dsv_peer_free(void* ptr);
int dsv_peer_barrier(unsigned* const* peer_slots, unsigned* my_slots, unsigned* epoch, int world,
                     int rank, void* stream);

/* Diagnostics: copy the backward kernel's phase timeline (clock64 stamps, filled only
 * by builds with -DDSV_BWD_PROF; layout [8 CTAs][32 blocks][12 events] int64) into a
 * host buffer. Returns the bytes copied or a negative value. */
int dsv_debug_timeline(void* host_dst, int bytes);
/* Diagnostics: the fused selection's pass timeline (globaltimer ns stamps of CTA 0, filled
 * only by builds with -DDSV_FSEL_PROF; layout [64 passes][8 events] uint64). */
int dsv_debug_select_timeline(void* host_dst, int bytes);

/* fp32 -> bf16 conversion of n contiguous elements. */
int dsv_f32_to_bf16(const float* in, void* out, long long n, void* stream);

/* Ring KV pass for dense residual heads (no reference counterpart: the
 * reference only pins the dense semantics, attention.py:95-109 full_attention and
 * tests/test_cpsim.py:75-88). Element kernels between the per-hop attention launches:
 *   dsv_ring_lse_merge: merge one hop's partial rows part (bf16 [rows][D], normalised by
 *     its own softmax sum) with LSE lse_part (log2 domain, as dsv_sparse_fwd writes it)
 *     into the running fp32 acc [rows][D] / lse_in -> lse_out (first: acc := part);
 *     out (optional, bf16 [rows][D]) receives the merged rows (the last hop).
 *   dsv_ring_accum_bf16: acc (fp32) := (first ? 0 : acc) + x (bf16); out optional bf16(acc).
 *   dsv_ring_accum_f32: acc := (first ? 0 : acc) + part; part := 0 (the traveling dK/dV
 *     accumulator absorbs one hop's atomically-accumulated contribution). */
int dsv_ring_lse_merge(float* acc, const float* lse_in, float* lse_out, const void* part,
                       const float* lse_part, long long rows, int D, int first, void* out,
                       void* stream);
int dsv_ring_accum_bf16(float* acc, const void* x, long long n, int first, void* out, void* stream);
int dsv_ring_accum_f32(float* acc, float* part, long long n, int first, void* stream);

/* ---- reference-precision (fp64) path ------------------------------------------------- */
/* C[b](m, n) = (sum_t A[b](m, t) B[b](t, n)) / div, fp64, fma in t order (deterministic).
 * A(m, t) = A[m*sam + t*sat], B(t, n) = B[t*sbt + n*sbn] (element strides; transposes free),
 * C row stride ldc, batch strides a_bs / b_bs / c_bs. */
int dsv_gemm_f64(const double* A, long long sam, long long sat, long long a_bs, const double* B,
                 long long sbt, long long sbn, long long b_bs, double* C, long long ldc,
                 long long c_bs, int M, int N, int K, int nbatch, double div, void* stream);
/* In place: x[r] <- softmax(x[r]) with the row max subtracted first. */
int dsv_softmax_rows_f64(double* x, long long ld, int R, int N, void* stream);
/* Exact top-k per row of fp64 scores S [R][L] (row stride lds); row r takes
 * k = k_per[r / rows_per_k] (1 <= k <= L). out [R][>= k] int32 ascending, thr[r] = k-th
 * largest score. Ties toward the lower index; -0.0 == +0.0. */
int dsv_topk_f64(const double* S, long long lds, int R, int L, const int* k_per, int rows_per_k,
                 int* out, long long ldo, double* thr, void* stream);
/* Attention over CSR index lists in fp64 (cols == NULL: every key). q [H][Lq][Dk],
 * k [H][Lk][Dk], v [H][Lk][Dv]; out [H][Lq][Dv], lse natural log of the scaled logits.
 * Backward: dq [H][Lq][Dk]; dk_acc / dv_acc are accumulated into (caller zeroes them). */
int dsv_rows_fwd_f64(const double* q, const double* k, const double* v, const long long* ptr,
                     const int* cols, int H, int Lq, int Lk, int Dk, int Dv, double scale,
                     double* out, double* lse, void* stream);
int dsv_rows_bwd_f64(const double* q, const double* k, const double* v, const double* out,
                     const double* lse, const double* dout, const long long* ptr,
                     const int* cols, int H, int Lq, int Lk, int Dk, int Dv, double scale,
                     double* dq, double* dk_acc, double* dv_acc, void* stream);
/* Sorted-row statistics of non-negative fp64 rows S [R][L]: with the row sorted by value
 * descending (ties: lower index first) and csum its sequential prefix sums,
 * n_keep[r] = min(L, #{csum < min(theta, total) - eps} + 1) (theta <= 0: L; NULL: skipped)
 * and topmass[r] = sum of the first top_n sorted values (NULL: skipped). Rows whose padded
 * length fits shared memory need no scratch; otherwise pass scratch of
 * dsv_sorted_stats_scratch_bytes(R, L) bytes. */
long long dsv_sorted_stats_scratch_bytes(int R, int L);
int dsv_sorted_stats_f64(const double* S, long long lds, int R, int L, double theta, double eps,
                         int top_n, int* n_keep, double* topmass, void* scratch,
                         long long scratch_bytes, void* stream);
/* counts[b] += #{S values with edges[b] <= v < edges[b+1]} (last bin closed); nb bins,
 * edges ascending [nb + 1], counts uint64 [nb] (np.histogram semantics). */
int dsv_histogram_f64(const double* S, long long lds, int R, int N, const double* edges, int nb,
                      unsigned long long* counts, void* stream);

/* Per query q: inter[q] = |E_q & O_q| for sorted CSR lists E (est_ptr / est_cols) and O
 * (ora_ptr / ora_cols), est_mass[q] / ora_mass[q] = sum of S[q][j] over each list
 * (predictor.py:262-281 prediction_accuracy). */
int dsv_set_stats_f64(const double* S, long long lds, int Q, const long long* est_ptr,
                      const int* est_cols, const long long* ora_ptr, const int* ora_cols,
                      int* inter, double* est_mass, double* ora_mass, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DSV_H_ */
