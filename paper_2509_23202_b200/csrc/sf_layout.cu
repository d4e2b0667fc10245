// Scale-factor layout conversion and device dequantize.
//
// sf_swizzle:   MfpTensor.scale_codes (row-major [rows, K/G], formats.py:314-316)
//               -> the 128x4-atom layout tcgen05 block-scaled MMA reads (weight prep, K3).
// sf_unswizzle: inverse (hand device results back as a reference MfpTensor).
// dequantize:   formats.py:424-442, ts * scale * fp4 (fp32 out) -- a checker, not the hot path.
#include "common.cuh"

namespace mrfp4 {
namespace {

// One thread per output byte of the padded swizzled buffer (coalesced writes).
__global__ void k_sf_swizzle(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t rows,
                             int64_t cols, int64_t col_blocks, int64_t total) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t atom = o >> 9, within = o & 511;
    const int64_t rb = atom / col_blocks, cb = atom % col_blocks;
    const int64_t r = rb * 128 + ((within >> 2) & 3) * 32 + (within >> 4);
    const int64_t c = cb * 4 + (within & 3);
    dst[o] = (r < rows && c < cols) ? src[r * cols + c] : (uint8_t)0;
  }
}

__global__ void k_sf_unswizzle(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t rows,
                               int64_t cols, int64_t col_blocks) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[i] = src[sf_offset(r, c, col_blocks)];
  }
}

__device__ __forceinline__ float fp4_value(uint32_t code) {
  const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  const float v = mag[code & 7];
  return (code & 8) ? -v : v;
}

template <int G>
__global__ void k_dequantize(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ sf,
                             const float* __restrict__ ts, int64_t rows, int64_t cols, int64_t col_blocks,
                             float* __restrict__ out) {
  const int64_t total = rows * cols;
  const float t = *ts;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const uint32_t byte = codes[r * (cols >> 1) + (c >> 1)];
    const uint32_t code = (c & 1) ? (byte >> 4) : (byte & 15u);
    const uint32_t s = sf[sf_offset(r, c / G, col_blocks)];
    const float scale = G == 32 ? (s == 0 ? 5.877471754111438e-39f : __uint_as_float(s << 23)) : e4m3_value(s);
    out[i] = t * scale * fp4_value(code);  // same association as formats.py:441
  }
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

int launch_sf_swizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  const int64_t cb = ceil_div(cols, 4);
  const int64_t total = ceil_div(rows, 128) * 128 * cb * 4;
  k_sf_swizzle<<<grid_for(total), 256, 0, s>>>(src, dst, rows, cols, cb, total);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_sf_unswizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  k_sf_unswizzle<<<grid_for(rows * cols), 256, 0, s>>>(src, dst, rows, cols, ceil_div(cols, 4));
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_dequantize(const uint8_t* codes, const uint8_t* sf, const float* ts, int64_t rows, int64_t cols, int fmt,
                      float* out, cudaStream_t s) {
  const int G = fmt == MRFP4_FMT_MXFP4 ? 32 : 16;
  const int64_t cb = ceil_div(cols / G, 4);
  if (G == 32)
    k_dequantize<32><<<grid_for(rows * cols), 256, 0, s>>>(codes, sf, ts, rows, cols, cb, out);
  else
    k_dequantize<16><<<grid_for(rows * cols), 256, 0, s>>>(codes, sf, ts, rows, cols, cb, out);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

}  // namespace mrfp4
