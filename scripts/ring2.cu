// cp + MMA interplay in a 4-stage ring (1 CTA, 2 roles), kernel-exact SF column pattern (MXFP4, 1-CTA, N=256).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

// MODE: 0 = no cp; 1 = 6 cp/stage into per-stage slot, MMAs read same stage's SF;
//       2 = cps into slot of next stage (MMAs read SF copied one stage earlier);
//       3 = 6 cp/stage into a slot never read by MMAs (MMAs read a fixed preloaded slot)
//       4 = 2 cp/stage only (SFA), SFB fixed
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];   // A: 4x16KB @0, B: 4x32KB @64KB, SF: 4 x 3KB @192KB
  __shared__ uint64_t full[4], empty[4], done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (196608 + 12288) / 4; i += blockDim.x) {
    uint32_t x = i * 2654435761u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = i >= 196608 / 4 ? 0x7E7F807Fu : x;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&done, 1); fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1); mbar_arrive(&full[stage]);
      if (++stage == 4) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    // preload all SF slots once
    for (int s = 0; s < 5; ++s)
      for (int c = 0; c < 6; ++c) tc_cp_32x128b_warpx4(tmem + 256 + s * 24 + 4 * c, smem_desc(smem_u32(smem + 196608 + c * 512), 0, 128, 0));
    int stage = 0; uint32_t phase = 0;
    long long t0 = 0;
    for (int i = 0; i < iters; ++i) {
      if (i == 100) t0 = clock64();
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t sf_read = tmem + 256 + ((MODE == 3 || MODE == 4) ? 4 * 24 : stage * 24);
      const uint32_t sf_cp = tmem + 256 + (MODE == 2 ? ((stage + 1) & 3) * 24 : MODE == 3 ? 4 * 24 + 0 : stage * 24);
      const uint32_t cs = smem_u32(smem + 196608 + stage * 3072);
      if (MODE >= 1 && MODE <= 3) {
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          tc_cp_32x128b_warpx4(sf_cp + a * 4, smem_desc(cs + a * 512, 0, 128, 0));
#pragma unroll
          for (int j = 0; j < 2; ++j) tc_cp_32x128b_warpx4(sf_cp + 8 + a * 8 + j * 4, smem_desc(cs + 1024 + (j * 2 + a) * 512, 0, 128, 0));
        }
      }
      if (MODE == 5) {
#pragma unroll
        for (int c = 0; c < 6; ++c) tc_cp_32x128b_warpx4(sf_cp + 4 * c, smem_desc(cs + c * 512, 0, 128, 0));
      }
      if (MODE == 6) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + 96 + 8 * c), "l"(smem_desc(cs, 2048, 256, 0)) : "memory");
      }
      if (MODE == 7) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
          asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + 256 + 96 + 4 * c), "l"(smem_desc(cs, 0, 128, 0)) : "memory");
      }
      if (MODE == 4) {
        tc_cp_32x128b_warpx4(tmem + 256 + stage * 24, smem_desc(cs, 0, 128, 0));
        tc_cp_32x128b_warpx4(tmem + 256 + stage * 24 + 4, smem_desc(cs + 512, 0, 128, 0));
      }
      const uint32_t a_s = smem_u32(smem) + stage * 16384, b_s = smem_u32(smem) + 65536 + stage * 32768;
#pragma unroll
      for (int kk = 0; kk < (MODE == 5 ? 0 : 4); ++kk) {
        const uint32_t sfid = (uint32_t)(kk & 1) * 2u; const int atom = kk >> 1;
        tc_mma_fp4<32>(tmem, smem_desc(a_s + kk * 32, 16, 1024, 2), smem_desc(b_s + kk * 32, 16, 1024, 2),
                       idesc_fp4(128, 256, true, sfid, sfid), (sf_read + atom * 4) | (sfid << 30),
                       (sf_read + 8 + atom * 8) | (sfid << 30), 1);
      }
      tc_commit(&empty[stage]);
      if (++stage == 4) { stage = 0; phase ^= 1; }
    }
    tc_commit(&done); mbar_wait(&done, 0);
    if (blockIdx.x == 0) out[0] = (unsigned long long)(clock64() - t0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE> void run(const char* nm) {
  unsigned long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 12288);
  k<MODE><<<148, 128, 196608 + 12288>>>(1100, d); cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d %-45s %7.1f cycles/stage (floor 512) %s\n", MODE, nm, c / 1000.0, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("no cp"); run<1>("6 cp -> same-stage slot, MMAs read it"); run<2>("6 cp -> next-stage slot (prefetch)");
  run<3>("6 cp -> unread slot"); run<4>("2 cp (SFA only)");
  run<5>("6 cp, no MMA"); run<6>("3 x 128x256b cp + 4 MMA"); run<7>("6 x 128x128b cp + 4 MMA");
  return 0;
}
