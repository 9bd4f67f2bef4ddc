// serialize.cu — index-set wire formats on device.
//
// Reference: pkg/src/dynsparse/serialize.py:119-151 `encode_index_sets`: varint(n_rows),
// then per row varint(count) and the varint deltas of the strictly increasing indices
// (first value as is), 7 bits per byte, low bits first, 0x80 = continuation. At c5 the
// per-rank index sets are ~2.6 GB as int32; the delta varints of sorted critical sets
// are ~1-2 bytes each, so encoding on the GPU before an offload to host memory cuts the
// PCIe bytes 2-4x. Two passes, one warp per row: byte lengths (and validation), then
// the bytes at offsets from a scan of the lengths (warp scan of per-element lengths).

#include "dsv_common.cuh"

namespace dsv {
namespace ser {

DSV_DEV int vlen(uint32_t v) {   // bytes of the unsigned varint of v (>= 1)
  return v < (1u << 7) ? 1 : v < (1u << 14) ? 2 : v < (1u << 21) ? 3 : v < (1u << 28) ? 4 : 5;
}

DSV_DEV int row_count(const int* counts, int k_uniform, int row) {
  return counts ? counts[row] : k_uniform;
}

// element j's delta (first value as is); err bit 1: negative first value, bit 2: not
// strictly increasing
DSV_DEV uint32_t delta_of(const int* r, int j, int* err) {
  const int v = r[j];
  if (j == 0) {
    if (v < 0) atomicOr(err, 1);
    return (uint32_t)v;
  }
  const int d = v - r[j - 1];
  if (d <= 0) atomicOr(err, 2);
  return (uint32_t)d;
}

__global__ void row_bytes_kernel(const int* __restrict__ idx, long long ld, const int* __restrict__ counts,
                                 int k_uniform, int rows, long long* __restrict__ out_len, int* err) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int n = row_count(counts, k_uniform, row);
    const int* r = idx + (long long)row * ld;
    long long len = 0;
    for (int j = lane; j < n; j += 32) len += vlen(delta_of(r, j, err));
#pragma unroll
    for (int o = 16; o; o >>= 1) len += __shfl_xor_sync(0xffffffffu, len, o);
    if (lane == 0) out_len[row] = len + vlen((uint32_t)n);
  }
}

DSV_DEV void put_varint(uint8_t* p, uint32_t v) {
  while (v >= 0x80u) { *p++ = (uint8_t)(v | 0x80u); v >>= 7; }
  *p = (uint8_t)v;
}

__global__ void encode_kernel(const int* __restrict__ idx, long long ld, const int* __restrict__ counts,
                              int k_uniform, int rows, const long long* __restrict__ row_off,
                              uint8_t* __restrict__ out, int* err) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int n = row_count(counts, k_uniform, row);
    const int* r = idx + (long long)row * ld;
    long long pos = row_off[row];
    if (lane == 0) put_varint(out + pos, (uint32_t)n);
    pos += vlen((uint32_t)n);
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const uint32_t d = j < n ? delta_of(r, j, err) : 0u;
      const int l = j < n ? vlen(d) : 0;
      int inc = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
      }
      if (j < n) put_varint(out + pos + inc - l, d);
      pos += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

}  // namespace ser
}  // namespace dsv

int dsv_varint_launch(int stage, const int* idx, long long ld, const int* counts, int k_uniform,
                      int rows, long long* lens_or_offsets, unsigned char* out, int* err,
                      cudaStream_t st) {
  using namespace dsv::ser;
  if (rows <= 0) return 0;
  const int threads = 256, wpb = threads / 32;
  const int grid = (rows + wpb - 1) / wpb < 65535 ? (rows + wpb - 1) / wpb : 65535;
  if (stage == 0)
    row_bytes_kernel<<<grid, threads, 0, st>>>(idx, ld, counts, k_uniform, rows, lens_or_offsets, err);
  else
    encode_kernel<<<grid, threads, 0, st>>>(idx, ld, counts, k_uniform, rows, lens_or_offsets, out, err);
  return (int)cudaGetLastError();
}
