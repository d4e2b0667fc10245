// Microbenchmark: sustained tcgen05.mma.cta_group::2 kind::mxf4nvf4 rate (M=256, N=256/128, K=64)
// on a CTA pair, fixed SMEM operands (no loads).  V0: back-to-back MMAs; V1: a commit to a
// multicast mbarrier every 4 MMAs (the GEMM's per-k-block commit), no waits; V2: V1 plus a
// wait on the commit of 2 k-blocks ago (ring back-pressure).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. scripts/mma2_rate.cu -o mma2_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"

using namespace mrfp4::sm100;

template <int V, int N, bool RANDOM = false, int SPIN = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(448, 1) k_rate2(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4], stop, fin;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) {
    uint32_t x = (i + 7919u * blockIdx.x) * 2654435761u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = RANDOM ? x : 0x22222222u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    mbar_init(&stop, 1);
    mbar_init(&fin, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_2sm(&holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (V >= 7 && warp < 4) {  // valid scale factors (E8M0 127 = 1.0) in every SF column
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = 0x7F7F7F7Fu;
    for (int c = 256; c < 512; c += 16) tmem_st_32x32b<16>(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp >= 4 && warp < 4 + SPIN) { if (V >= 5) mbar_wait_sleep(&stop, 0); else mbar_wait(&stop, 0); }  // idle warps polling an mbarrier
  if (rank == 0 && threadIdx.x == 32) {
    uint64_t g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int st = (V >= 3) ? it % 6 : 0;                  // V3+: kernel's per-stage SF slots (24 cols)
      const int sb = (V >= 4) ? it % 3 : 0;                  // V4+: rotating A/B stage buffers
      const uint32_t a_s = smem_u32(smem + sb * 32768), b_s = smem_u32(smem + sb * 32768 + 16384);
      const uint32_t sfa = tmem + 256 + st * 24, sfb = sfa + 8;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t sfid = (uint32_t)(k & 1) * 2u;
        const uint64_t ad = smem_desc(a_s + k * 32, 16, 1024, 2), bd = smem_desc(b_s + k * 32, 16, 1024, 2);
        tc_mma_fp4_2sm<32>(tmem, ad, bd, idesc_fp4(256, N, true, sfid, sfid), (sfa + (k >> 1) * 4) | (sfid << 30),
                           (sfb + (k >> 1) * 8) | (sfid << 30), (it | k) ? 1u : 0u);
      }
      if (V >= 1) tc_commit_2sm_mc(&bar[it & 3], 0x3);
      if (V >= 2 && it >= 2) mbar_wait(&bar[(it - 2) & 3], ((it - 2) >> 2) & 1);
    }
    tc_commit_2sm_mc(&fin, 0x3);
    long long t1 = clock64();
    uint64_t g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (blockIdx.x == 0) { cycles[0] = t1 - t0; cycles[1] = g1 - g0; }
  }
  if (threadIdx.x == 32) {
    mbar_wait(&fin, 0);
    mbar_arrive(&stop);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

template <int V, int N, bool RANDOM = false, int SPIN = 0>
void run(const char* name, int nclusters = 1) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  auto k = k_rate2<V, N, RANDOM, SPIN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  const int iters = 65536;
  k<<<2 * nclusters, 128 + 32 * SPIN, 98304>>>(iters, d);
  cudaDeviceSynchronize();
  k<<<2 * nclusters, 128 + 32 * SPIN, 98304>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long c[2] = {0, 0};
  cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
  printf("%-40s N=%3d clusters=%2d: %7.1f cycles/MMA (ideal %d), %.0f MHz, %.0f TFLOP/s chip-equiv %s\n", name, N,
         nclusters, (double)c[0] / (iters * 4), 128 * N / 256, (double)c[0] / c[1] * 1e3,
         2.0 * 256 * N * 64 * iters * 4 * nclusters / (c[1] * 1e-9) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 256>("2CTA back-to-back");
  run<0, 224>("2CTA back-to-back");
  run<0, 192>("2CTA back-to-back");
  run<0, 160>("2CTA back-to-back");
  run<0, 128>("2CTA back-to-back");
  run<4, 256, true>("V4 all SMs, random operands", 74);
  run<4, 224, true>("V4 all SMs, random operands", 74);
  run<4, 160, true>("V4 all SMs, random operands", 74);
  return 0;
}
