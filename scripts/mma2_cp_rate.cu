// Microbenchmark: can the scale factors go SMEM -> TMEM by tcgen05.cp.cta_group::2 (issued by the
// MMA thread, in order with the MMAs: no stager warps, no cross-CTA release) without slowing the
// 2-CTA block-scaled MMA stream?  All SMs (74 pairs), fixed SMEM operands, per "stage" of 8 MMAs
// (K = 512): NCP tcgen05.cp.cta_group::2.32x128b.warpx4 atoms into one of two TMEM SF slots, then
// 8 MMAs reading that slot, commit per stage, wait on the commit of two stages back.
// NVFP4 needs 24 atoms per stage (8 SFA + 16 SFB), MXFP4 12.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. scripts/mma2_cp_rate.cu -o mma2_cp_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"

using namespace mrfp4::sm100;

template <int VEC, int NCP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4], fin;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) {
    uint32_t x = (i + 7919u * blockIdx.x) * 2654435761u;
    x ^= x >> 13;
    // operands random, SF region (last 32 KB) = valid scale codes (0x38 = 1.0 e4m3, 127 = 1.0 e8m0)
    reinterpret_cast<uint32_t*>(smem)[i] = i >= 98304 / 4 ? (VEC == 16 ? 0x38383838u : 0x7F7F7F7Fu) : x;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    mbar_init(&fin, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_2sm(&holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  constexpr int kSlotCols = VEC == 16 ? 96 : 48;
  if (rank == 0 && warp == 1) {
    const uint32_t el = elect_lane();
    long long t0 = clock64();
    uint64_t g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int it = 0; it < iters; ++it) {
      const int slot = it & 1, sb = it % 3;
      const uint32_t sf_t = tmem + 256 + slot * kSlotCols;
      if (el) {
#pragma unroll
        for (int a = 0; a < NCP; ++a)
          tc_cp_32x128b_warpx4_2sm(sf_t + 4 * (a % (kSlotCols / 4)),
                                   smem_desc(smem_u32(smem + 98304 + slot * 16384 + 512 * a), 0, 128, 0));
      }
      const uint32_t a_s = smem_u32(smem + sb * 32768), b_s = smem_u32(smem + sb * 32768 + 16384);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = smem_desc(a_s + (k & 3) * 32 + (k >> 2) * 8192, 16, 1024, 2);
        const uint64_t bd = smem_desc(b_s + (k & 3) * 32 + (k >> 2) * 8192, 16, 1024, 2);
        if constexpr (VEC == 16) {
          tc_mma_fp4_2sm_if<16>(el, tmem, ad, bd, idesc_fp4(256, 256, false, 0, 0), sf_t + 4 * k,
                                sf_t + 32 + 8 * k, (it | k) ? 1u : 0u);
        } else {
          const uint32_t sfid = (uint32_t)(k & 1) * 2u;
          tc_mma_fp4_2sm_if<32>(el, tmem, ad, bd, idesc_fp4(256, 256, true, sfid, sfid),
                                (sf_t + (k >> 1) * 4) | (sfid << 30), (sf_t + 16 + (k >> 1) * 8) | (sfid << 30),
                                (it | k) ? 1u : 0u);
        }
      }
      tc_commit_2sm_mc_if(el, &bar[it & 3], 0x3);
      if (it >= 2) mbar_wait(&bar[(it - 2) & 3], ((it - 2) >> 2) & 1);
    }
    tc_commit_2sm_mc_if(el, &fin, 0x3);
    mbar_wait(&fin, 0);
    long long t1 = clock64();
    uint64_t g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (blockIdx.x == 0 && el) {
      out[0] = t1 - t0;
      out[1] = g1 - g0;
    }
  } else if (rank == 1 && warp == 1 && (threadIdx.x & 31) == 0) {
    mbar_wait(&fin, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

template <int VEC, int NCP>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  auto k = k_rate<VEC, NCP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 8192;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<<<sms, 128, 131072>>>(64, d);
  cudaDeviceSynchronize();
  k<<<sms, 128, 131072>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long c[2] = {0, 0};
  cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
  printf("%-34s %7.1f cycles/MMA (ideal 128), %.0f MHz, %.0f TFLOP/s chip %s\n", name, (double)c[0] / (iters * 8.0),
         (double)c[0] / c[1] * 1e3, 2.0 * 256 * 256 * 64 * 8.0 * iters * (sms / 2) / (c[1] * 1e-9) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, 0>("nvfp4 8 MMA/stage, no cp");
  run<16, 12>("nvfp4 8 MMA + 12 cp");
  run<16, 24>("nvfp4 8 MMA + 24 cp (needed)");
  run<32, 0>("mxfp4 8 MMA/stage, no cp");
  run<32, 12>("mxfp4 8 MMA + 12 cp (needed)");
  run<32, 24>("mxfp4 8 MMA + 24 cp");
  return 0;
}
