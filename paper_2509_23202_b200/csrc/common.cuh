// Shared helpers for the mrfp4 sm_100a kernels (B200).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../../include/mrfp4.h"

namespace mrfp4 {

// ---------------------------------------------------------------------------
// Scale-factor layout consumed by tcgen05 block-scaled MMA (cuBLAS "blocked"
// layout): 128-row x 4-column atoms of 512 bytes, atoms K-contiguous.
// offset(r, c) = ((r/128)*ceil(C/4) + c/4)*512 + (r%32)*16 + ((r/32)%4)*4 + c%4
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t sf_offset(int64_t r, int64_t c, int64_t col_blocks) {
  return ((r >> 7) * col_blocks + (c >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (c & 3);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Value of an E4M3 (unsigned, bias 7) scale code as fp32 (exact).
__device__ __forceinline__ float e4m3_value(uint32_t code) {
  const uint32_t e = code >> 3, m = code & 7u;
  const float sub = (float)m * 0.001953125f;                  // m * 2^-9
  const float nrm = __uint_as_float(((e + 120u) << 23) | (m << 20));
  return e == 0 ? sub : nrm;
}

__device__ __forceinline__ void atomic_or_status(uint32_t* status, uint32_t bits) {
  if (status) atomicOr(status, bits);
}

}  // namespace mrfp4
