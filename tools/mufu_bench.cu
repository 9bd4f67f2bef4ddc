// MUFU ex2 vs FMA-pipe polynomial exp2 throughput per SM (B200), and the mix.
#include <cstdio>
#include "../paper_2502_07590_b200/csrc/dsv_common.cuh"
using namespace dsv;

// degree-3 minimax 2^x on the FMA pipe (Cody-Waite split via the 1.5 * 2^23 magic add), the
// variant the kernels once mixed with MUFU ex2 (kept here for the throughput comparison)
__device__ __forceinline__ f32x2 exp2_poly2(f32x2 x) {
  float2 v = f2u(x);
  v.x = fmaxf(v.x, -125.f);
  v.y = fmaxf(v.y, -125.f);
  const f32x2 magic = f2(12582912.f, 12582912.f);
  const f32x2 xc = f2(v.x, v.y);
  const f32x2 t = fadd2(xc, magic);
  const f32x2 jf = fadd2(t, f2(-12582912.f, -12582912.f));
  const f32x2 fr = ffma2(jf, f2(-1.f, -1.f), xc);
  f32x2 p = ffma2(fr, f2(0.05517044f, 0.05517044f), f2(0.2426081f, 0.2426081f));
  p = ffma2(fr, p, f2(0.69326096f, 0.69326096f));
  p = ffma2(fr, p, f2(0.99992834f, 0.99992834f));
  const float2 q = f2u(p), tt = f2u(t);
  return f2(__int_as_float(__float_as_int(q.x) + (__float_as_int(tt.x) << 23)),
            __int_as_float(__float_as_int(q.y) + (__float_as_int(tt.y) << 23)));
}

template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  f32x2 b[4];
  for (int i = 0; i < 4; ++i) b[i] = f2(a[2 * i], a[2 * i + 1]);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fast_exp2(a[i]) - 1.0f;
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) { b[i] = exp2_poly2(b[i]); b[i] = fadd2(b[i], f2(-1.f, -1.f)); }
    } else if (MODE == 3) {
      // bf16x2 packing throughput (cvt.rn.bf16x2.f32 = F2FP)
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const uint32_t pk = pack_bf16(a[i], a[i + 1]);
        a[i] = __uint_as_float(pk) + 1.0f;
        a[i + 1] = __uint_as_float(pk ^ 0x10001u) + 1.0f;
      }
    } else if (MODE == 4) {
      // the same with integer round-to-nearest-even + PRMT
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        uint32_t u0 = __float_as_uint(a[i]), u1 = __float_as_uint(a[i + 1]);
        u0 += 0x7fffu + ((u0 >> 16) & 1u);
        u1 += 0x7fffu + ((u1 >> 16) & 1u);
        const uint32_t pk = __byte_perm(u0, u1, 0x7632);
        a[i] = __uint_as_float(pk) + 1.0f;
        a[i + 1] = __uint_as_float(pk ^ 0x10001u) + 1.0f;
      }
    } else if (MODE == 5 || MODE == 6) {
      // the forward's P chunk: 32 scores -> 16 bf16x2 + row-sum (MODE 6: all MUFU)
      uint32_t r[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(a[i & 7] - 0.01f * i);
      const f32x2 sc2 = f2(1.44f, 1.44f), nm2 = f2(-3.f, -3.f);
      f32x2 lsum2 = f2(0.f, 0.f);
      uint32_t acc = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const f32x2 x = ffma2(f2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), sc2, nm2);
        float2 p;
        if (MODE == 5 && (i & 3) == 3) {
          p = f2u(exp2_poly2(x));
        } else {
          const float2 xv = f2u(x);
          p = make_float2(fast_exp2(xv.x), fast_exp2(xv.y));
        }
        lsum2 = fadd2(lsum2, f2(p.x, p.y));
        acc ^= pack_bf16(p.x, p.y);
      }
      const float2 l = f2u(lsum2);
      a[it & 7] += l.x + l.y + __uint_as_float(acc & 0x3f800000u) * 1e-30f;
      // 32 exp2 per iteration here (vs 8 in the other modes)
    } else {
      // 3 MUFU pairs : 1 poly pair
#pragma unroll
      for (int i = 0; i < 6; ++i) a[i] = fast_exp2(a[i]) - 1.0f;
      b[3] = fadd2(exp2_poly2(b[3]), f2(-1.f, -1.f));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  for (int i = 0; i < 4; ++i) { float2 v = f2u(b[i]); s += v.x + v.y; }
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* o; cudaMalloc(&o, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, grid = 148 * 2, thr = 512;
  const char* names[] = {"MUFU ex2", "poly exp2 (FFMA2)", "3 MUFU : 1 poly", "F2FP pack (per value)", "int RNE+PRMT (per value)", "P chunk 3:1 (x4 exps)", "P chunk MUFU only (x4)"};
  for (int m = 0; m < 7; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<grid, thr>>>(o, iters);
      if (m == 1) k<1><<<grid, thr>>>(o, iters);
      if (m == 2) k<2><<<grid, thr>>>(o, iters);
      if (m == 3) k<3><<<grid, thr>>>(o, iters);
      if (m == 4) k<4><<<grid, thr>>>(o, iters);
      if (m == 5) k<5><<<grid, thr>>>(o, iters);
      if (m == 6) k<6><<<grid, thr>>>(o, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)grid * thr * iters * 8;   // exp2 evaluations
      if (rep == 1) printf("%-20s %.3f ms  %.1f exp2/clk/SM (at %d MHz)\n", names[m], ms,
                           ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
