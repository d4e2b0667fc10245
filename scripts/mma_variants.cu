// Which MMA operand pattern slows tcgen05.mma kind::mxf4nvf4 (MXFP4 2X, M128 N256 K64)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

template <int V>
__global__ void __launch_bounds__(128, 1) k_var(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = (V == 7 || V == 10 || V == 12) ? (uint32_t)(i * 2654435761u) : (V == 11 ? 0u : 0x22222222u);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  if (V >= 9) {
    // valid scale factors: E8M0 127 (=1.0) in a 512-B smem atom, copied to the SF columns
    for (int i = threadIdx.x; i < 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + 180224)[i] = 0x7F7F7F7Fu;
    __syncthreads();
    if (threadIdx.x == 32) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int c = 0; c < 8; ++c) tc_cp_32x128b_warpx4(tmem + 256 + 4 * c, smem_desc(smem_u32(smem + 180224), 0, 128, 0));
      tc_commit(&bar); mbar_wait(&bar, 0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 32) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int k = i & 3;
      uint32_t off = (V == 1 || V == 4) ? k * 32 : 0;
      const int st = (V == 5 || V == 7) ? ((i >> 2) & 3) : (V == 8 ? ((i >> 2) & 1) : 0);
      const uint64_t adesc = smem_desc(smem_u32(smem) + st * 16384 + off, 16, 1024, 2);
      const uint64_t bdesc = smem_desc(smem_u32(smem + 65536) + st * 32768 + off, 16, 1024, 2);
      uint32_t sfid = (V == 2 || V == 4) ? (uint32_t)(k & 1) * 2 : 0;
      uint32_t atom = (V == 3 || V == 4) ? (k >> 1) : 0;
      const uint32_t sfa = (tmem + 256 + atom * 4) | (sfid << 30);
      const uint32_t sfb = (tmem + 272 + atom * 8) | (sfid << 30);
      tc_mma_fp4<32>(tmem, adesc, bdesc, idesc_fp4(128, 256, true, sfid, sfid), sfa, sfb, (V == 6) ? (k != 0) : 1);
    }
    tc_commit(&bar); mbar_wait(&bar, V >= 9 ? 1 : 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int V>
void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_var<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  k_var<V><<<sms, 128, 196608>>>(4096, d);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("V%d %-40s %7.1f cycles/MMA %s\n", V, name, (double)c / 4096, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("baseline same addr");
  run<1>("A/B desc start += k*32B");
  run<2>("sf_id cycling 0/2");
  run<3>("SF atom column per k");
  run<4>("all of 1+2+3 (kernel pattern)");
  run<5>("A/B stage buffers rotate over 4 stages");
  run<6>("accumulate=0 every 4th");
  run<7>("4-stage rotate, random data");
  run<8>("2-stage rotate");
  run<9>("valid SF (1.0), data 0x22");
  run<10>("valid SF (1.0), random data");
  run<11>("valid SF (1.0), zero data");
  return 0;
}
