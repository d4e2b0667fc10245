// (1) mma.sync m16n8k16 bf16->f32 issue throughput per SM on B200 (legacy tensor path).
// (2) exactness: Hadamard-32 of bf16 rows by two chained HMMAs vs the fp32 FWHT (RN per stage).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ void hmma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int NW>
__global__ void k_rate(int iters, float* out) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, 7u};
  uint32_t b[2] = {0x3f803f80u, 0xbf803f80u};
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hmma(c[j], a, b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// H32 Sylvester entry sign: (-1)^popc(i & j)
__host__ __device__ inline float hsign(int i, int j) { return (__builtin_popcount(i & j) & 1) ? -1.f : 1.f; }

// rows of 32 bf16; one warp handles 16 rows (one m-tile) per iteration
__global__ void k_cmp(const __nv_bfloat16* x, int rows, unsigned long long* mism, float* ymma, float* yfw) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  // B fragments: B[k][n] = H[k][n]; thread holds B[2t..2t+1][g] and B[2t+8..2t+9][g] for each (ktile, ntile)
  uint32_t bf[2][4][2];
  for (int kt = 0; kt < 2; ++kt)
    for (int nt = 0; nt < 4; ++nt)
      for (int r = 0; r < 2; ++r) {
        const int k0 = kt * 16 + 2 * t + 8 * r, n = nt * 8 + g;
        __nv_bfloat162 v = __floats2bfloat162_rn(hsign(k0, n), hsign(k0 + 1, n));
        bf[kt][nt][r] = *reinterpret_cast<uint32_t*>(&v);
      }
  for (int m0 = warp * 16; m0 < rows; m0 += nwarps * 16) {
    // A fragment: a0 = (row g, k 2t..2t+1), a1 = (row g+8, ...), a2 = (row g, k 2t+8..), a3 = (row g+8, k 2t+8..)
    float c[4][4] = {};
    for (int kt = 0; kt < 2; ++kt) {
      uint32_t a[4];
      const uint32_t* xr0 = reinterpret_cast<const uint32_t*>(x + (size_t)(m0 + g) * 32 + kt * 16);
      const uint32_t* xr1 = reinterpret_cast<const uint32_t*>(x + (size_t)(m0 + g + 8) * 32 + kt * 16);
      a[0] = xr0[t]; a[1] = xr1[t]; a[2] = xr0[t + 4]; a[3] = xr1[t + 4];
      for (int nt = 0; nt < 4; ++nt) hmma(c[nt], a, bf[kt][nt]);
    }
    for (int nt = 0; nt < 4; ++nt) {
      ymma[(size_t)(m0 + g) * 32 + nt * 8 + 2 * t] = c[nt][0];
      ymma[(size_t)(m0 + g) * 32 + nt * 8 + 2 * t + 1] = c[nt][1];
      ymma[(size_t)(m0 + g + 8) * 32 + nt * 8 + 2 * t] = c[nt][2];
      ymma[(size_t)(m0 + g + 8) * 32 + nt * 8 + 2 * t + 1] = c[nt][3];
    }
  }
  // FWHT reference: one row per thread
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = __bfloat162float(x[(size_t)r * 32 + i]);
    for (int h = 1; h < 32; h <<= 1)
      for (int i = 0; i < 32; ++i)
        if (!(i & h)) { float a = v[i], b = v[i + h]; v[i] = __fadd_rn(a, b); v[i + h] = __fsub_rn(a, b); }
    for (int i = 0; i < 32; ++i) yfw[(size_t)r * 32 + i] = v[i];
  }
}

int main() {
  float* out; cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  k_rate<8><<<148, 256>>>(iters, out);
  for (int bs : {128, 256, 512}) {
    cudaEventRecord(e0);
    k_rate<8><<<148 * 4, bs>>>(iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * 4 * (bs / 32) * iters * 8;
    printf("block %d: %.3f ms, %.1f HMMA/clk/SM @1.9GHz, %.1f TFLOP/s\n", bs, ms, mmas / (ms * 1e-3) / 148 / 1.9e9,
           mmas * 4096 / (ms * 1e-3) / 1e12);
  }
  const int rows = 1 << 20;
  __nv_bfloat16* hx = (__nv_bfloat16*)malloc((size_t)rows * 32 * 2);
  srand(1);
  for (size_t i = 0; i < (size_t)rows * 32; ++i) {
    double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
    double z = sqrt(-2 * log(u1)) * cos(6.283185307 * u2);
    int mode = (i / 32 / 4096) % 4;
    if (mode == 1) z = (u1 < 0.5 ? 1 : -1) * log(u2) * 3;          // Laplace
    if (mode == 2) z *= ldexp(1.0, (rand() % 24) - 12);            // wide dynamic range
    if (mode == 3 && rand() % 64 == 0) z *= 1000;                    // outliers
    hx[i] = __float2bfloat16((float)z);
  }
  __nv_bfloat16* dx; float *ym, *yf;
  cudaMalloc(&dx, (size_t)rows * 64); cudaMalloc(&ym, (size_t)rows * 128); cudaMalloc(&yf, (size_t)rows * 128);
  cudaMemcpy(dx, hx, (size_t)rows * 64, cudaMemcpyHostToDevice);
  k_cmp<<<148, 256>>>(dx, rows, nullptr, ym, yf);
  cudaDeviceSynchronize();
  float* hm = (float*)malloc((size_t)rows * 128); float* hf = (float*)malloc((size_t)rows * 128);
  cudaMemcpy(hm, ym, (size_t)rows * 128, cudaMemcpyDeviceToHost);
  cudaMemcpy(hf, yf, (size_t)rows * 128, cudaMemcpyDeviceToHost);
  size_t mism[4] = {0, 0, 0, 0}, exact_mism[4] = {0, 0, 0, 0}, fw_mism[4] = {0, 0, 0, 0};
  for (size_t i = 0; i < (size_t)rows * 32; ++i) {
    int mode = (i / 32 / 4096) % 4;
    // exact value in double
    size_t r = i / 32; int j = i % 32;
    double s = 0;
    for (int k = 0; k < 32; ++k) s += (double)__bfloat162float(hx[r * 32 + k]) * hsign(k, j);
    if (hm[i] != hf[i]) ++mism[mode];
    if ((double)hm[i] != s) ++exact_mism[mode];
    if ((double)hf[i] != s) ++fw_mism[mode];
  }
  printf("H32 mma vs fwht mismatches per mode (gauss, laplace, wide, outlier): %zu %zu %zu %zu of %d each\n",
         mism[0], mism[1], mism[2], mism[3], rows * 8);
  printf("mma vs exact mismatches: %zu %zu %zu %zu\n", exact_mism[0], exact_mism[1], exact_mism[2], exact_mism[3]);
  printf("fwht vs exact mismatches: %zu %zu %zu %zu\n", fw_mism[0], fw_mism[1], fw_mism[2], fw_mism[3]);
  return 0;
}
