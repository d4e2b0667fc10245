// Microbenchmark: mbarrier / tcgen05.commit round trips on B200.
//  (1) single thread: [n MMAs] -> commit -> wait, repeated: commit latency
//  (2) producer/consumer ring of S stages: producer waits empty/arrives full, consumer
//      waits full, issues n MMAs (+ optional UTCCP), commits empty: cycles per stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

template <int S, int NMMA, int NCP>
__global__ void __launch_bounds__(128, 1) k_ring(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[S], empty[S], lat;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&lat, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  const uint64_t adesc = smem_desc(smem_u32(smem), 16, 1024, 2), bdesc = smem_desc(smem_u32(smem + 16384), 16, 1024, 2);
  if (warp == 0 && lane == 0) {  // producer
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive(&full[stage]);
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {  // consumer
    int stage = 0; uint32_t phase = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      for (int c = 0; c < NCP; ++c) tc_cp_32x128b_warpx4(tmem + 256 + 4 * c, smem_desc(smem_u32(smem + 32768 + 512 * c), 0, 128, 0));
      for (int k = 0; k < NMMA; ++k) tc_mma_fp4<32>(tmem, adesc, bdesc, idesc_fp4(128, 256, true, 0, 0), tmem + 256, tmem + 272, 1);
      tc_commit(&empty[stage]);
      if (++stage == S) { stage = 0; phase ^= 1; }
    }
    tc_commit(&lat);
    mbar_wait(&lat, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    // commit latency alone
    __syncwarp(1);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

__global__ void __launch_bounds__(128, 1) k_commit_lat(int iters, int nmma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  const uint64_t adesc = smem_desc(smem_u32(smem), 16, 1024, 2), bdesc = smem_desc(smem_u32(smem + 16384), 16, 1024, 2);
  if (threadIdx.x == 32) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int k = 0; k < nmma; ++k) tc_mma_fp4<32>(tmem, adesc, bdesc, idesc_fp4(128, 256, true, 0, 0), tmem + 256, tmem + 272, 1);
      tc_commit(&bar);
      mbar_wait(&bar, i & 1);
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int S, int NMMA, int NCP>
void ring(int sms) {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_ring<S, NMMA, NCP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 2000;
  k_ring<S, NMMA, NCP><<<sms, 128, 65536>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("ring S=%d mma/stage=%d cp/stage=%d: %7.1f cycles/stage (MMA floor %d) %s\n", S, NMMA, NCP, (double)c / iters,
         NMMA * 128, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_commit_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int n : {0, 1, 4}) {
    k_commit_lat<<<sms, 128, 65536>>>(500, n, d);
    cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("commit->wait round trip with %d MMAs: %7.1f cycles %s\n", n, (double)c / 500, cudaGetErrorString(cudaGetLastError()));
  }
  ring<4, 0, 0>(sms); ring<4, 0, 6>(sms); ring<4, 4, 0>(sms); ring<4, 4, 6>(sms); ring<4, 4, 12>(sms);
  ring<2, 4, 6>(sms); ring<8, 4, 6>(sms); ring<4, 2, 6>(sms);
  return 0;
}
