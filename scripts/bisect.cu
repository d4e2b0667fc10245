// Bisect: the 1-CTA GEMM mainloop skeleton with knobs, single CTA, no loads, valid-ish SF.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2509_23202_b200/csrc/sm100.cuh"
using namespace mrfp4::sm100;

struct Args { int num_kb; int num_tiles; long long K; unsigned long long* dbg; };

// KNOB bits: 1 = epilogue tile handshake (tfull/tempty), 2 = producer int64 math, 4 = nk from K (dynamic)
template <int KNOB>
__global__ void __launch_bounds__(192, 1) k_bis(Args g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int S = 4, kABytes = 16384, kBBytes = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 196608 + 8192);
  uint64_t* empty = full + S; uint64_t* tfull = empty + S; uint64_t* tempty = tfull + 1;
  uint32_t* holder = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1); mbar_init(tempty, 4); fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(holder, 512);
  // KNOB 8: fill operand SMEM with pseudo-random FP4 codes; KNOB 16: valid SF (E8M0 ~2^0) in all slots
  if (KNOB & 8)
    for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) {
      uint32_t x = i * 2654435761u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      reinterpret_cast<uint32_t*>(smem)[i] = x;
    }
  if (KNOB & 16)
    for (int i = threadIdx.x; i < 12288 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + 196608)[i] = 0x7E7F807Fu;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem_base = *holder;
  if ((KNOB & 16) && threadIdx.x == 32) {
    for (int c = 0; c < 24; ++c) tc_cp_32x128b_warpx4(tmem_base + 256 + 4 * c, smem_desc(smem_u32(smem + 196608), 0, 128, 0));
  }
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int tile = 0; tile < g.num_tiles; ++tile)
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive(&full[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0, acc_phase = 0;
      for (int tile = 0; tile < g.num_tiles; ++tile) {
        if (KNOB & 1) { mbar_wait(tempty, acc_phase ^ 1); tc_fence_after(); }
        for (int kb = 0; kb < g.num_kb; ++kb) {
          if (tile == 0 && kb < 64) g.dbg[kb] = clock64();
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sfa_t = tmem_base + 256 + stage * 24;
          const uint32_t sfb_t = sfa_t + 8;
          const uint32_t cpa_t = (KNOB & 64) ? tmem_base + 256 + ((stage + 1) & 3) * 24 : sfa_t;
          const uint32_t cpb_t = cpa_t + 8;
          if (KNOB & 32) {
#pragma unroll
            for (int a = 0; a < 2; ++a) {
              tc_cp_32x128b_warpx4(cpa_t + a * 4, smem_desc(smem_u32(smem + 196608 + 1024 * stage + a * 512), 0, 128, 0));
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tc_cp_32x128b_warpx4(cpb_t + a * 8 + j * 4, smem_desc(smem_u32(smem + 200704 + 2048 * stage + (j * 2 + a) * 512), 0, 128, 0));
            }
          }
          const uint32_t a_s = smem_u32(smem + stage * kABytes);
          const uint32_t b_s = smem_u32(smem + 65536 + stage * kBBytes);
          int nk = 4;
          if (KNOB & 4) nk = (int)((g.K - (long long)kb * 256) / 64 < 4 ? (g.K - (long long)kb * 256) / 64 : 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k >= nk) break;
            const int atom = k >> 1;
            const uint32_t sfid = (uint32_t)(k & 1) * 2u;
            tc_mma_fp4<32>(tmem_base, smem_desc(a_s + k * 32, 16, 1024, 2), smem_desc(b_s + k * 32, 16, 1024, 2),
                           idesc_fp4(128, 256, true, sfid, sfid), (sfa_t + atom * 4) | (sfid << 30),
                           (sfb_t + atom * 8) | (sfid << 30), (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (KNOB & 1) tc_commit(tfull);
        acc_phase ^= 1;
      }
    }
  } else if (KNOB & 1) {
    uint32_t acc_phase = 0;
    for (int tile = 0; tile < g.num_tiles; ++tile) {
      mbar_wait(tfull, acc_phase); tc_fence_after(); tc_fence_before(); __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem_base, 512); }
}

template <int KNOB>
void run(int smem_bytes) {
  unsigned long long* d; cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(k_bis<KNOB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  Args g{56, 2, 14336, d};
  k_bis<KNOB><<<1, 192, smem_bytes>>>(g);
  cudaDeviceSynchronize();
  unsigned long long t[64]; cudaMemcpy(t, d, 64 * 8, cudaMemcpyDeviceToHost);
  printf("KNOB=%d smem=%d: per-kb %llu %llu %llu %llu  %s\n", KNOB, smem_bytes, t[11] - t[10], t[21] - t[20], t[31] - t[30],
         t[41] - t[40], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<32>(215000); run<40>(215000); run<48>(215000); run<56>(215000); run<24>(215000);
  return 0;
}
