// Offline MSE scale search on the GPU:
//   optimize_group_scales (/root/reference/pkg/src/microfp/quantizers.py:263-327).
// The host driver (quantize.py::_mse_optimize) runs the reference's alternating search --
// per-group candidate passes and, for NVFP4, the 128-point tensor-scale scan -- and sums
// group errors exactly as numpy does; these kernels do the per-group work in float64 with
// the reference's arithmetic:
//   candidate raw   cand[c] * raw0                      (quantizers.py:294)
//   scale code      fp_scale_encode(raw / s_global)     (quantizers.py:157-167; formats.py:220-262)
//   group error     ((B - eff * fp4(B / eff))**2).sum(-1), numpy's pairwise order for 16 / 32
//                   terms (8 accumulators, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)))
//                                                       (quantizers.py:257-260, :211-215)
//   argmin          first minimum over candidates        (quantizers.py:297)
#include <cmath>

#include "common.cuh"

namespace mrfp4 {
namespace {

// E4M3 RNE of a positive double onto codes 0..126 (formats.py:239-251, :81-91), saturating.
__device__ __forceinline__ uint32_t e4m3_code64(double v) {
  if (!(v < 432.0)) return 126u;
  if (v < 0.015625) return (uint32_t)__double2int_rn(v * 512.0);
  int e;
  const double fr = frexp(v, &e);
  int m = __double2int_rn((fr * 2.0 - 1.0) * 8.0);
  int E = e - 1;
  if (m == 8) { m = 0; E += 1; }
  return (uint32_t)(((E + 7) << 3) | m);
}

__device__ __forceinline__ double e4m3_value64(uint32_t c) {
  const int E = (int)(c >> 3), m = (int)(c & 7u);
  return E == 0 ? ldexp((double)m, -9) : ldexp(1.0 + m / 8.0, E - 7);
}

// Signed FP4 grid value of u (formats.py:94-113: ties 0.25 / 1.25 / 2.5 / 5 down, 0.75 / 1.75
// / 3.5 up; saturate at 6) and its 4-bit code (sign only when the magnitude is non-zero).
__device__ __forceinline__ double fp4_round64(double u, uint32_t& code) {
  const double a = fabs(u);
  const uint32_t idx = (a > 0.25) + (a > 0.75) + (a == 0.75) + (a > 1.25) + (a > 1.75) + (a == 1.75) + (a > 2.5) +
                       (a > 3.5) + (a == 3.5) + (a > 5.0);
  const double g[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  const bool neg = signbit(u);
  code = idx | ((neg && idx) ? 8u : 0u);
  return neg ? -g[idx] : g[idx];
}

// numpy pairwise_sum for n in {16, 32}: 8 accumulators, then a fixed tree.
template <int G>
__device__ __forceinline__ double group_err(const double (&v)[G], double eff) {
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t c;
    const double d = v[j] - eff * fp4_round64(v[j] / eff, c);
    r[j] = d * d;
  }
#pragma unroll
  for (int i = 8; i < G; i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t c;
      const double d = v[i + j] - eff * fp4_round64(v[i + j] / eff, c);
      r[j] += d * d;
    }
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

template <int G>
__device__ __forceinline__ void load_group(const double* y, int64_t g, double (&v)[G]) {
  const double2* p = reinterpret_cast<const double2*>(y + g * G);
#pragma unroll
  for (int i = 0; i < G / 2; ++i) {
    const double2 t = p[i];
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}

// One candidate pass (quantizers.py:288-302) at tensor scale ts = f32(sg * factor).
template <int G, int FMT>
__global__ void __launch_bounds__(128) k_mse_pass(const double* __restrict__ y, int64_t ngroups,
                                                  const double* __restrict__ cand, int ncand,
                                                  const double* __restrict__ raw0, double sg, double ts,
                                                  uint8_t* __restrict__ sc, double* __restrict__ dec,
                                                  double* __restrict__ gerr, uint8_t* __restrict__ codes,
                                                  uint32_t* status) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups; g += (int64_t)gridDim.x * blockDim.x) {
    double v[G];
    load_group<G>(y, g, v);
    const double r0 = raw0[g];
    double best = 0.0, bdec = 1.0;
    uint32_t bcode = 0, bad = 0;
    for (int c = 0; c < ncand; ++c) {
      const double enc = (cand[c] * r0) / sg;
      uint32_t code;
      double d;
      if constexpr (FMT == MRFP4_FMT_MXFP4) {
        const double e = fmin(fmax(rint(log2(enc)), -127.0), 127.0);   // formats.py:225
        code = (uint32_t)(e + 127.0);
        d = ldexp(1.0, (int)e);
      } else {
        code = e4m3_code64(enc);
        d = e4m3_value64(code);
      }
      const double eff = ts * d;
      if (!(eff > 0.0)) {   // B / 0: the reference raises DataError (fp4_round_codes, formats.py:101-102)
        bad |= MRFP4_STATUS_SCALE_UNDERFLOW;
        continue;
      }
      const double err = group_err<G>(v, eff);
      if (!(err <= 1.79e308)) bad |= MRFP4_STATUS_NONFINITE;
      if (c == 0 || err < best) {
        best = err;
        bcode = code;
        bdec = d;
      }
    }
    sc[g] = (uint8_t)bcode;
    dec[g] = bdec;
    gerr[g] = best;
    const double eff = ts * bdec;
#pragma unroll
    for (int i = 0; i < G; i += 2) {
      uint32_t c0, c1;
      fp4_round64(v[i] / eff, c0);
      fp4_round64(v[i + 1] / eff, c1);
      codes[g * (G / 2) + i / 2] = (uint8_t)(c0 | (c1 << 4));
    }
    if (bad) atomicOr(status, bad);
  }
}

// Group errors at a fixed assignment (quantizers.py:304-306, total_err's per-group terms).
template <int G>
__global__ void __launch_bounds__(128) k_mse_group_err(const double* __restrict__ y, int64_t ngroups,
                                                       const double* __restrict__ dec, double ts,
                                                       double* __restrict__ gerr, uint32_t* status) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups; g += (int64_t)gridDim.x * blockDim.x) {
    double v[G];
    load_group<G>(y, g, v);
    const double eff = ts * dec[g];
    if (!(eff > 0.0)) {
      atomicOr(status, MRFP4_STATUS_SCALE_UNDERFLOW);
      gerr[g] = 0.0;
      continue;
    }
    gerr[g] = group_err<G>(v, eff);
  }
}

// numpy's pairwise_sum (umath loops: n < 8 sequential from 0; n <= 128 eight accumulators
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; larger n split at
// n2 = n/2 rounded down to a multiple of 8).  Bit-identical to np.sum of a float64 array.
__device__ double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

__global__ void k_np_pairwise_segments(const double* __restrict__ a, const int64_t* __restrict__ starts,
                                       const int64_t* __restrict__ lens, int64_t nseg, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = np_pairwise(a + starts[i], lens[i]);
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 128), (int64_t)sms * 16));
}

// apply_blockwise for float64 X (transforms.py:77-91): y[r, b + j] = sum_i x[r, b + i] * M[i][j],
// M = (H_k / sqrt(k))^T with entries +-RN64(1 / RN64(sqrt(k))), summed in index order as an fma
// chain (see mrfp4.h: the reference's BLAS order for k = 16, where every product is exact).
__global__ void __launch_bounds__(256) k_rotate_f64(const double* __restrict__ x, int64_t M, int64_t K, int64_t ldx,
                                                    int hk, double c, double* __restrict__ y) {
  const int64_t total = M * K;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = o / K, col = o - r * K;
    const double* xr = x + r * ldx;
    if (hk == 0) {
      y[o] = xr[col];
      continue;
    }
    const int j = (int)(col % hk);
    const int64_t b = col - j;
    double acc = xr[b] * c;                       // i = 0: H[0][j] = +1
    for (int i = 1; i < hk; ++i) acc = fma(xr[b + i], (__popc(i & j) & 1) ? -c : c, acc);
    y[o] = acc;
  }
}

}  // namespace

int launch_mse_pass(const double* y, int64_t ngroups, int fmt, const double* cand, int ncand, const double* raw0,
                    double sg, double ts, uint8_t* sc, double* dec, double* gerr, uint8_t* codes, uint32_t* status,
                    cudaStream_t s) {
  const int grid = grid_for(ngroups);
  if (fmt == MRFP4_FMT_MXFP4)
    k_mse_pass<32, MRFP4_FMT_MXFP4><<<grid, 128, 0, s>>>(y, ngroups, cand, ncand, raw0, sg, ts, sc, dec, gerr, codes,
                                                          status);
  else
    k_mse_pass<16, MRFP4_FMT_NVFP4><<<grid, 128, 0, s>>>(y, ngroups, cand, ncand, raw0, sg, ts, sc, dec, gerr, codes,
                                                          status);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_mse_group_err(const double* y, int64_t ngroups, int fmt, const double* dec, double ts, double* gerr,
                         uint32_t* status, cudaStream_t s) {
  const int grid = grid_for(ngroups);
  if (fmt == MRFP4_FMT_MXFP4)
    k_mse_group_err<32><<<grid, 128, 0, s>>>(y, ngroups, dec, ts, gerr, status);
  else
    k_mse_group_err<16><<<grid, 128, 0, s>>>(y, ngroups, dec, ts, gerr, status);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_rotate_f64(const double* x, int64_t M, int64_t K, int64_t ldx, int hk, double* y, cudaStream_t s) {
  const double c = hk ? 1.0 / std::sqrt((double)hk) : 1.0;   // _sylvester(k) / np.sqrt(k)
  k_rotate_f64<<<grid_for(M * K), 256, 0, s>>>(x, M, K, ldx, hk, c, y);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_np_pairwise_segments(const double* a, const int64_t* starts, const int64_t* lens, int64_t nseg,
                                double* out, cudaStream_t s) {
  k_np_pairwise_segments<<<grid_for(nseg), 128, 0, s>>>(a, starts, lens, nseg, out);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

}  // namespace mrfp4

// ---------------------------------------------------------------------------
// GPTQ column solver: one lazy block of _gptq_core
// (/root/reference/pkg/src/microfp/gptq.py:148-167) for all rows at once.  Rows are
// independent given T and the column scales, so a thread owns one row: the block's columns
// i1 .. i1+B-1 of its row sit in shared memory ([B][threads], conflict-free), the block of the
// upper factor T ([B][B]) is shared by the CTA.  Per column i, in the reference's float64
// arithmetic (no FMA contraction):
//     codes, vals = fp4_round_codes(w_i / s_i); q = s_i * vals          (:141-145)
//     e = (w_i - q) / T[i, i];  w_j -= e * T[i, j]  for i < j < B          (:160-164)
// The caller applies the lazy trailing update W[:, i2:] -= Err @ T[i1:i2, i2:] (:165-166) as a
// float64 GEMM.
// ---------------------------------------------------------------------------
namespace mrfp4 {
namespace {

constexpr int kGptqThreads = 64;
constexpr int kGptqMaxB = 128;

__global__ void __launch_bounds__(kGptqThreads, 1)
    k_gptq_block(double* __restrict__ W, const double* __restrict__ S, const double* __restrict__ T, int64_t rows,
                 int64_t d, int i1, int B, double* __restrict__ Q, uint8_t* __restrict__ codes,
                 double* __restrict__ Err) {
  extern __shared__ __align__(16) double gsm[];
  double* Tb = gsm;                          // [B][B] block of T (row i, column j)
  double* Wb = gsm + kGptqMaxB * kGptqMaxB;  // [B][kGptqThreads]
  const int tid = threadIdx.x;
  for (int x = tid; x < B * B; x += blockDim.x) {
    const int i = x / B, j = x - i * B;
    Tb[i * B + j] = T[(int64_t)(i1 + i) * d + i1 + j];
  }
  const int64_t r = (int64_t)blockIdx.x * kGptqThreads + tid;
  const bool live = r < rows;
  if (live)
    for (int j = 0; j < B; ++j) Wb[j * kGptqThreads + tid] = W[r * d + i1 + j];
  __syncthreads();
  if (!live) return;
  const double* Sr = S + r * d + i1;
  for (int i = 0; i < B; ++i) {
    const double wi = Wb[i * kGptqThreads + tid];
    const double si = Sr[i];
    uint32_t c;
    const double q = __dmul_rn(si, fp4_round64(__ddiv_rn(wi, si), c));
    const double e = __ddiv_rn(__dsub_rn(wi, q), Tb[i * B + i]);
    Q[r * d + i1 + i] = q;
    codes[r * d + i1 + i] = (uint8_t)c;
    Err[r * kGptqMaxB + i] = e;
    const double* Ti = Tb + i * B;
#pragma unroll 4
    for (int j = i + 1; j < B; ++j) {
      double* wj = Wb + j * kGptqThreads + tid;
      *wj = __dsub_rn(*wj, __dmul_rn(e, Ti[j]));
    }
  }
}

}  // namespace

int launch_gptq_block(double* W, const double* S, const double* T, int64_t rows, int64_t d, int i1, int B, double* Q,
                      uint8_t* codes, double* Err, cudaStream_t s) {
  if (B < 1 || B > kGptqMaxB) return MRFP4_EINVAL;
  const size_t smem = (size_t)(kGptqMaxB * kGptqMaxB + kGptqMaxB * kGptqThreads) * sizeof(double);
  static std::atomic<int> attr[kMaxDevices];
  if (per_device_once(attr, [&] {
        return cudaFuncSetAttribute(k_gptq_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                       cudaSuccess ? 1 : -1;
      }) < 0)
    return MRFP4_ECUDA;
  const int grid = (int)ceil_div(rows, kGptqThreads);
  k_gptq_block<<<grid, kGptqThreads, smem, s>>>(W, S, T, rows, d, i1, B, Q, codes, Err);
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

}  // namespace mrfp4
