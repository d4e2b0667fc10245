// TMA read bandwidth vs box row width: one producer thread per SM streams a contiguous
// range of a 512 MB buffer through an S-stage ring (wait full -> re-issue), no consumer work.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

template <int S>
__global__ void k_stream(const __grid_constant__ CUtensorMap tm, int rows_per_box, int box_bytes, int64_t nboxes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  const int64_t per = (nboxes + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < nboxes ? b0 + per : nboxes;
  int64_t issued = b0;
  for (int s = 0; s < S && issued < b1; ++s, ++issued) {
    mbar_arrive_expect_tx(&full[s], box_bytes);
    tma_load_2d(smem + s * box_bytes, &tm, &full[s], 0, (int)(issued * rows_per_box));
  }
  uint32_t ph = 0;
  int s = 0;
  for (int64_t b = b0; b < b1; ++b) {
    mbar_wait(&full[s], (ph >> s) & 1);
    ph ^= 1u << s;
    if (issued < b1) {
      mbar_arrive_expect_tx(&full[s], box_bytes);
      tma_load_2d(smem + s * box_bytes, &tm, &full[s], 0, (int)(issued * rows_per_box));
      ++issued;
    }
    s = s + 1 == S ? 0 : s + 1;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t bytes = 512ull << 20;
  void* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  void* fl; cudaMalloc(&fl, 256 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int row_bytes, rows, swz; } cfgs[] = {{64, 128, 2}, {64, 32, 2}, {128, 64, 3}, {128, 128, 3}, {128, 256, 3}, {64, 256, 2}};
  for (auto c : cfgs) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)c.row_bytes, (cuuint64_t)(bytes / c.row_bytes)};
    cuuint64_t strides[1] = {(cuuint64_t)c.row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)c.row_bytes, (cuuint32_t)c.rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        c.swz == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int box_bytes = c.row_bytes * c.rows;
    const int64_t nboxes = bytes / box_bytes;
    for (int S : {4, 12}) {
      auto kern = S == 4 ? k_stream<4> : k_stream<12>;
      const int smem = S * box_bytes + 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        cudaMemset(fl, it, 256 << 20);
        cudaEventRecord(e0);
        kern<<<148, 32, smem>>>(tm, c.rows, box_bytes, nboxes);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("rows of %3d B x %3d (box %5d B), S=%2d: %.1f GB/s  %s\n", c.row_bytes, c.rows, box_bytes, S,
             bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
