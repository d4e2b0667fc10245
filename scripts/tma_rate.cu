// Microbenchmark: per-SM TMA load throughput (L2-resident source) for GEMM-like boxes.
// One CTA per SM (grid = #SMs), one producer thread, a ring of S stages of BOX_BYTES each,
// a consumer warp that waits on `full` and immediately frees the slot.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. scripts/tma_rate.cu -o tma_rate -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

struct Cfg { int rows; int inner; int swz; int stages; int per_stage; int iters; int kdepth; };

__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, Cfg c, int row_span,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int box = c.rows * c.inner;
  if (threadIdx.x == 0) {
    for (int i = 0; i < c.stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < c.iters; ++it) {
      mbar_wait(&empty[st], ph ^ 1);
      mbar_arrive_expect_tx(&full[st], box * c.per_stage * c.kdepth);
      for (int j = 0; j < c.per_stage; ++j) {
        const int r = ((blockIdx.x * 7 + it * c.per_stage + j) * c.rows) % row_span;
        if (c.kdepth > 1) {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem + (st * c.per_stage + j) * box * c.kdepth)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[st])), "r"(0), "r"(r), "r"(0)
              : "memory");
        } else {
          tma_load_2d(smem + (st * c.per_stage + j) * box, &tm, &full[st], 0, r);
        }
      }
      if (++st == c.stages) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < c.iters; ++it) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == c.stages) { st = 0; ph ^= 1; }
    }
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 16u << 20;  // 16 MB source (L2-resident)
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  Cfg cfgs[] = {
      {128, 128, 1, 6, 2, 2000, 1}, {128, 128, 1, 3, 2, 2000, 2}, {128, 128, 1, 2, 2, 2000, 2}, {128, 128, 1, 4, 2, 2000, 2},
      {128, 128, 1, 2, 2, 2000, 3}, {128, 128, 1, 6, 4, 1000, 1}, {128, 128, 1, 1, 2, 2000, 4}, {256, 128, 1, 3, 2, 2000, 1},
  };
  for (const Cfg& c : cfgs) {
    const int inner = c.inner;
    const int64_t rows_total = bytes / 4096;      // tensor viewed as [rows_total, 4096 B]
    CUtensorMap tm;
    CUresult r;
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = c.swz ? (inner == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)
                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (c.kdepth > 1) {  // [k-block][row][128 B] view of a [rows, 4096 B] matrix
      cuuint64_t dims[3] = {128, (cuuint64_t)rows_total, 32};
      cuuint64_t strides[2] = {4096, 128};
      cuuint32_t box[3] = {128, (cuuint32_t)c.rows, (cuuint32_t)c.kdepth};
      r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[2] = {4096, (cuuint64_t)rows_total};
      cuuint64_t strides[1] = {4096};
      cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)c.rows};
      r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    const int smem = c.stages * c.per_stage * c.rows * inner * c.kdepth + 1024;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int span = (int)(rows_total - c.rows);
    k_tma<<<nsm, 64, smem>>>(tm, c, span, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_tma<<<nsm, 64, smem>>>(tm, c, span, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double per_sm = (double)c.iters * c.per_stage * c.rows * inner * c.kdepth;
    printf("box %3dx%3dBx%d swz=%d stages=%2d x%d (%3d KB in flight): %6.1f B/cycle/SM, %6.1f GB/s/SM, chip %7.0f GB/s %s\n",
           c.rows, inner, c.kdepth, c.swz, c.stages, c.per_stage, c.stages * c.per_stage * c.rows * inner * c.kdepth / 1024,
           per_sm / cyc, per_sm / (ms * 1e-3) / 1e9, per_sm * nsm / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
