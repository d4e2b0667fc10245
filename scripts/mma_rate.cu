// Microbenchmark: sustained tcgen05.mma issue rate per SM on B200 (sm_100a).
// One CTA per SM; one elected thread issues `iters` MMAs on fixed SMEM operands
// (no loads), then commits and waits.  Reports cycles/MMA and chip TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. scripts/mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"

using namespace mrfp4::sm100;

template <int KIND, int N, bool WITH_CP>  // KIND 0: bf16 f16-kind, 1: mxf4nvf4 4X, 2: mxf4nvf4 2X
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 32) {
    const uint32_t a_s = smem_u32(smem), b_s = smem_u32(smem + 16384);
    const uint64_t adesc = smem_desc(a_s, 16, 1024, 2), bdesc = smem_desc(b_s, 16, 1024, 2);
    const uint32_t sf_t = tmem + 256;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (WITH_CP && (i & 3) == 0) {
        for (int a = 0; a < 6; ++a) tc_cp_32x128b_warpx4(sf_t + 4 * a, smem_desc(smem_u32(smem + 32768 + 512 * a), 0, 128, 0));
      }
      if constexpr (KIND == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(i));
      } else if constexpr (KIND == 1) {
        tc_mma_fp4<16>(tmem, adesc, bdesc, idesc_fp4(128, N, false, 0, 0), sf_t, sf_t + 16, i);
      } else {
        tc_mma_fp4<32>(tmem, adesc, bdesc, idesc_fp4(128, N, true, 0, 0), sf_t, sf_t + 16, i);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int KIND, int N, bool CP>
void run(const char* name, double flops_per_mma) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_rate<KIND, N, CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  k_rate<KIND, N, CP><<<sms, 128, 65536>>>(64, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<KIND, N, CP><<<sms, 128, 65536>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t err = cudaGetLastError();
  printf("%-28s N=%3d cp=%d: %7.1f cycles/MMA, %8.1f TFLOP/s chip (%.3f ms) %s\n", name, N, (int)CP,
         (double)cyc / iters, flops_per_mma * iters * sms / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<0, 256, false>("bf16 kind::f16 K16", 2.0 * 128 * 256 * 16);
  run<0, 128, false>("bf16 kind::f16 K16", 2.0 * 128 * 128 * 16);
  run<1, 256, false>("nvfp4 mxf4nvf4 4X K64", 2.0 * 128 * 256 * 64);
  run<1, 128, false>("nvfp4 mxf4nvf4 4X K64", 2.0 * 128 * 128 * 64);
  run<2, 256, false>("mxfp4 mxf4nvf4 2X K64", 2.0 * 128 * 256 * 64);
  run<2, 128, false>("mxfp4 mxf4nvf4 2X K64", 2.0 * 128 * 128 * 64);
  run<1, 256, true>("nvfp4 4X + 6 UTCCP/4 MMA", 2.0 * 128 * 256 * 64);
  run<2, 256, true>("mxfp4 2X + 6 UTCCP/4 MMA", 2.0 * 128 * 256 * 64);
  return 0;
}
