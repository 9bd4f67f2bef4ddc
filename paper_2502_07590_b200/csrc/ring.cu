// ring.cu — element kernels of the ring KV pass for dense residual heads (SURVEY §2.1
// "ring KV exchange only for residual dense blocks", §8(e)): the LSE merge of per-hop
// partial outputs, the fp32 accumulation of per-hop dQ partials, and the traveling dK/dV
// accumulator update. All three are HBM-bound streams (one read of each operand, one
// write): 16-byte vectors, grid = a multiple of the SM count, grid-stride loops.

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dsv_common.cuh"

namespace dsv {
namespace ring {

constexpr int kThreads = 256;

inline int grid_for(long long work, int per_block) {
  long long b = (work + per_block - 1) / per_block;
  const long long cap = 148LL * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

__device__ __forceinline__ void unpack8(uint4 u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  u.x = pack_bf16(f[0], f[1]);
  u.y = pack_bf16(f[2], f[3]);
  u.z = pack_bf16(f[4], f[5]);
  u.w = pack_bf16(f[6], f[7]);
  return u;
}

// One (row, 8-element chunk) per thread-iteration. LSE in the log2 domain (the attention
// kernels' convention). acc/lse_in hold the running merge; part/lse_part one hop's
// partial (normalised by its own sum); the merged LSE goes to lse_out (a separate buffer:
// every chunk of a row reads lse_in). first: acc := part. out (optional): bf16 of the
// merged rows, written on the last hop.
__global__ void __launch_bounds__(kThreads)
lse_merge_kernel(float* __restrict__ acc, const float* __restrict__ lse_in,
                 float* __restrict__ lse_out, const __nv_bfloat16* __restrict__ part,
                 const float* __restrict__ lse_part, long long rows, int D, int first,
                 __nv_bfloat16* __restrict__ out) {
  const int cpr = D / 8;                              // 8-element chunks per row
  const long long total = rows * cpr;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / cpr;
    const int c = (int)(i - row * cpr);
    const float b = lse_part[row];
    float p[8], a[8];
    unpack8(reinterpret_cast<const uint4*>(part + row * D)[c], p);
    float4* ap = reinterpret_cast<float4*>(acc + row * D) + 2 * c;
    float l_new;
    if (first) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = p[j];
      l_new = b;
    } else {
      const float la = lse_in[row];
      const float4 a0 = ap[0], a1 = ap[1];
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      const float m = fmaxf(la, b);
      if (m == -INFINITY) {
        l_new = -INFINITY;                            // neither side saw a key
      } else {
        const float wa = exp2f(la - m), wb = exp2f(b - m);
        const float s = wa + wb, inv = 1.0f / s;
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = (a[j] * wa + p[j] * wb) * inv;
        l_new = m + log2f(s);
      }
    }
    ap[0] = make_float4(a[0], a[1], a[2], a[3]);
    ap[1] = make_float4(a[4], a[5], a[6], a[7]);
    if (out) reinterpret_cast<uint4*>(out + row * D)[c] = pack8(a);
    if (c == 0) lse_out[row] = l_new;
  }
}

// acc (fp32) := (first ? 0 : acc) + x (bf16); out (optional) = bf16(acc). n % 8 == 0.
__global__ void __launch_bounds__(kThreads)
accum_bf16_kernel(float* __restrict__ acc, const __nv_bfloat16* __restrict__ x, long long n8,
                  int first, __nv_bfloat16* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (long long)gridDim.x * blockDim.x) {
    float p[8], a[8];
    unpack8(reinterpret_cast<const uint4*>(x)[i], p);
    float4* ap = reinterpret_cast<float4*>(acc) + 2 * i;
    if (first) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = p[j];
    } else {
      const float4 a0 = ap[0], a1 = ap[1];
      a[0] = a0.x + p[0]; a[1] = a0.y + p[1]; a[2] = a0.z + p[2]; a[3] = a0.w + p[3];
      a[4] = a1.x + p[4]; a[5] = a1.y + p[5]; a[6] = a1.z + p[6]; a[7] = a1.w + p[7];
    }
    if (!out || !first) {
      ap[0] = make_float4(a[0], a[1], a[2], a[3]);
      ap[1] = make_float4(a[4], a[5], a[6], a[7]);
    }
    if (out) reinterpret_cast<uint4*>(out)[i] = pack8(a);
  }
}

// acc := (first ? 0 : acc) + part; part := 0 (ready for the next hop's atomic adds).
__global__ void __launch_bounds__(kThreads)
accum_f32_kernel(float4* __restrict__ acc, float4* __restrict__ part, long long n4, int first) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 p = part[i];
    if (!first) {
      const float4 a = acc[i];
      p.x += a.x; p.y += a.y; p.z += a.z; p.w += a.w;
    }
    acc[i] = p;
    part[i] = z;
  }
}

}  // namespace ring
}  // namespace dsv

using namespace dsv::ring;

int dsv_lse_merge_launch(float* acc, const float* lse_in, float* lse_out, const void* part,
                         const float* lse_part, long long rows, int D, int first, void* out,
                         cudaStream_t st) {
  if (rows <= 0) return 0;
  lse_merge_kernel<<<grid_for(rows * (D / 8), kThreads), kThreads, 0, st>>>(
      acc, lse_in, lse_out, (const __nv_bfloat16*)part, lse_part, rows, D, first,
      (__nv_bfloat16*)out);
  return (int)cudaGetLastError();
}

int dsv_accum_bf16_launch(float* acc, const void* x, long long n, int first, void* out,
                          cudaStream_t st) {
  if (n <= 0) return 0;
  accum_bf16_kernel<<<grid_for(n / 8, kThreads), kThreads, 0, st>>>(
      acc, (const __nv_bfloat16*)x, n / 8, first, (__nv_bfloat16*)out);
  return (int)cudaGetLastError();
}

int dsv_accum_f32_launch(float* acc, float* part, long long n, int first, cudaStream_t st) {
  if (n <= 0) return 0;
  accum_f32_kernel<<<grid_for(n / 4, kThreads), kThreads, 0, st>>>(
      (float4*)acc, (float4*)part, n / 4, first);
  return (int)cudaGetLastError();
}
