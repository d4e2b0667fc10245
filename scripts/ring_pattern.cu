// Ring pipeline (S=4) with the GEMM kernel's exact MMA operand pattern, to find what slows it.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

// V bits: 1 = per-stage A/B buffers, 2 = per-k desc advance, 4 = per-stage SF slot (24 cols),
//         8 = sf_id cycling, 16 = 192 threads w/ idle epilogue warps waiting on a barrier
template <int V>
__global__ void __launch_bounds__(192, 1) k_ring(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[4], empty[4], done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive(&full[stage]);
      if (++stage == 4) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t a_s = smem_u32(smem) + ((V & 1) ? stage * 16384 : 0);
      const uint32_t b_s = smem_u32(smem + 65536) + ((V & 1) ? stage * 32768 : 0);
      const uint32_t sfa_t = tmem + 256 + ((V & 4) ? stage * 24 : 0);
      const uint32_t sfb_t = sfa_t + 8;
      for (int k = 0; k < 4; ++k) {
        const uint32_t off = (V & 2) ? k * 32 : 0;
        const uint32_t sfid = (V & 8) ? (uint32_t)(k & 1) * 2u : 0u;
        const int atom = (V & 8) ? (k >> 1) : 0;
        tc_mma_fp4<32>(tmem, smem_desc(a_s + off, 16, 1024, 2), smem_desc(b_s + off, 16, 1024, 2),
                       idesc_fp4(128, 256, true, sfid, sfid), (sfa_t + atom * 4) | (sfid << 30),
                       (sfb_t + atom * 8) | (sfid << 30), (i | k) != 0);
      }
      tc_commit(&empty[stage]);
      if (++stage == 4) { stage = 0; phase ^= 1; }
    }
    tc_commit(&done);
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  } else if ((V & 16) && warp >= 2) {
    mbar_wait(&done, 0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int V>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_ring<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k_ring<V><<<1, 192, 200000>>>(2000, d);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("V=%2d (stages=%d desc=%d sfslot=%d sfid=%d epi=%d): %7.1f cycles/stage %s\n", V, V & 1, !!(V & 2), !!(V & 4),
         !!(V & 8), !!(V & 16), (double)c / 2000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>(); run<1>(); run<2>(); run<4>(); run<8>(); run<16>(); run<3>(); run<12>(); run<15>(); run<31>();
  return 0;
}
