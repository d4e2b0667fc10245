// K1: fused online activation quantization for sm_100a.
//
// Replaces quantize_rtn(X, spec, transform=TransformSpec.hadamard(k))
// (/root/reference/pkg/src/microfp/quantizers.py:247-255) on the GPU:
//   rotate   transforms.py:77-91   y = X_blk @ (H_k/sqrt(k))^T, Sylvester order
//   scales   quantizers.py:170-208 absmax/6, zero group -> 1.0, NVFP4 global s_T,
//                                   MXFP4 tensor scale f32(4/3)
//   codes    formats.py:220-251    E8M0 = clamp(rint(log2 raw)), E4M3 RNE (sat 448)
//   elements quantizers.py:211-215 + formats.py:94-113  RNE onto E2M1, -0 -> 0
//   packing  formats.py:377-382    low nibble = even element
//
// Work decomposition: one thread owns 32 contiguous elements of one row
// (4 x 16-byte loads for bf16).  Hadamard blocks of k <= 32 are rotated fully in
// registers; k = 64 / 128 add one / two butterfly stages across 2 / 4 lanes.
// A CTA covers 64 rows x 128 columns (4 threads per row).
//
// Exactness: the rotation is an fp32 FWHT (exact whenever the block sum fits in
// 24 bits -- always for k in {16, 64} scaling, typically for bf16 inputs).  All
// downstream decisions reproduce the reference's float64 arithmetic on the
// rotated value y = S * c:  scale codes are decided from an fp32 estimate and
// re-decided in float64 whenever the estimate is within 2^-18 of a rounding
// threshold; element codes are decided twice with u*(1 +- 2^-18) and any element
// whose two roundings disagree is re-decided from u = RN64(y / eff) exactly as
// numpy does (quantizers.py:213).
#include <algorithm>

#include "common.cuh"

namespace mrfp4 {

namespace {

constexpr int kSeg = 32;
constexpr int kSegsPerRow = 4;
constexpr int kRowsPerCta = 64;
constexpr int kThreads = kRowsPerCta * kSegsPerRow;  // 256

struct AQParams {
  const void* x;
  int64_t M, K, ldx;
  uint8_t* codes;
  uint8_t* sf;
  float* tensor_scale;
  uint32_t* status;
  uint32_t* gmax;          // NVFP4: max |S| over the tensor, fp32 bits (atomicMax)
  int64_t sf_cols;         // K / G
  int64_t sf_col_blocks;   // ceil(sf_cols / 4)
  int64_t rows_pad;        // ceil(M / 128) * 128
  double c64;              // RN64(1 / RN64(sqrt(k)))  (transforms.py:65: H / np.sqrt(k))
  float c32;
};

// ---------------------------------------------------------------------------
// loads
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bf16x2_to_f32(uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xFFFF0000u);
}

template <int IN>
__device__ __forceinline__ void load_seg(const void* base, int64_t off, int nvalid, float (&v)[kSeg]) {
  if (nvalid == 0) {
#pragma unroll
    for (int i = 0; i < kSeg; ++i) v[i] = 0.f;
    return;
  }
  if constexpr (IN == MRFP4_DT_F32) {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const float*>(base) + off);
    uint4 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (j < 4 || nvalid == kSeg) ? __ldg(p + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[4 * j + 0] = __uint_as_float(r[j].x);
      v[4 * j + 1] = __uint_as_float(r[j].y);
      v[4 * j + 2] = __uint_as_float(r[j].z);
      v[4 * j + 3] = __uint_as_float(r[j].w);
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + off);
    uint4 r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = (j < 2 || nvalid == kSeg) ? __ldg(p + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t w[4] = {r[j].x, r[j].y, r[j].z, r[j].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if constexpr (IN == MRFP4_DT_BF16) {
          bf16x2_to_f32(w[t], v[8 * j + 2 * t], v[8 * j + 2 * t + 1]);
        } else {
          __half2 h = *reinterpret_cast<const __half2*>(&w[t]);
          float2 f = __half22float2(h);
          v[8 * j + 2 * t] = f.x;
          v[8 * j + 2 * t + 1] = f.y;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fast Walsh-Hadamard transform (unnormalized, Sylvester natural order)
// ---------------------------------------------------------------------------
template <int HK>
__device__ __forceinline__ void fwht(float (&v)[kSeg], int lane) {
  constexpr int kIn = HK < kSeg ? HK : kSeg;
#pragma unroll
  for (int h = 1; h < kIn; h <<= 1) {
#pragma unroll
    for (int i = 0; i < kSeg; ++i) {
      if ((i & h) == 0) {
        const float a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
    }
  }
  // Cross-lane stages: block element index bit 5 (k>=64) lives in lane bit 0,
  // bit 6 (k=128) in lane bit 1.  Lower partner keeps a+b, upper keeps a-b.
  if constexpr (HK >= 64) {
    const float sg = (lane & 1) ? -1.f : 1.f;
#pragma unroll
    for (int i = 0; i < kSeg; ++i) {
      const float p = __shfl_xor_sync(0xffffffffu, v[i], 1);
      v[i] = fmaf(sg, v[i], p);
    }
  }
  if constexpr (HK >= 128) {
    const float sg = (lane & 2) ? -1.f : 1.f;
#pragma unroll
    for (int i = 0; i < kSeg; ++i) {
      const float p = __shfl_xor_sync(0xffffffffu, v[i], 2);
      v[i] = fmaf(sg, v[i], p);
    }
  }
}

// max |v| over [lo, lo+n); NaN/Inf-propagating for rotated data, bit-exact for raw.
template <int HK, int N>
__device__ __forceinline__ uint32_t group_absmax_bits(const float (&v)[kSeg], int lo) {
  if constexpr (HK == 0) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) m = max(m, __float_as_uint(v[lo + i]) & 0x7fffffffu);
    return m;  // NaN/Inf bit patterns are the largest
  } else {
    // After a Hadamard, a non-finite input makes every output of its block
    // non-finite, so a max seeded with the first element stays non-finite.
    float m = fabsf(v[lo]);
#pragma unroll
    for (int i = 1; i < N; ++i) m = fmaxf(m, fabsf(v[lo + i]));
    return __float_as_uint(m) & 0x7fffffffu;
  }
}

// ---------------------------------------------------------------------------
// exact (float64) decisions, mirroring numpy
// ---------------------------------------------------------------------------
// E4M3 RNE of a positive double onto codes 0..126 (formats.py:239-251, :81-91).
__device__ __noinline__ uint32_t e4m3_rne64(double v) {
  if (!(v < 432.0)) return 126u;                       // >= mid(416,448) (tie -> even 126)
  if (v < 0.015625) {                                  // subnormal range m * 2^-9
    return (uint32_t)__double2int_rn(v * 512.0);       // rint: ties to even m; 8 -> code 8 = 2^-6
  }
  int e;
  const double fr = frexp(v, &e);                      // v = fr * 2^e, fr in [0.5, 1)
  const double q = (fr * 2.0 - 1.0) * 8.0;             // mantissa fraction * 8, exact
  int m = __double2int_rn(q);
  int E = e - 1;
  if (m == 8) { m = 0; E += 1; }
  return (uint32_t)(((E + 7) << 3) | m);
}

// E8M0 exponent of raw = RN64(a64 / 6): clamp(rint(log2 raw), -127, 127)  (formats.py:225).
__device__ __noinline__ int e8m0_exp_exact(float amax_s, double c64) {
  const double a64 = (double)amax_s * c64;
  const double raw = a64 / 6.0;
  double e = rint(log2(raw));
  e = fmin(fmax(e, -127.0), 127.0);
  return (int)e;
}

// NVFP4 scale code from the float64 chain RN64(RN64(a64/6)/s_T)  (quantizers.py:162,187).
__device__ __noinline__ uint32_t e4m3_code_exact(float amax_s, double c64, double st64) {
  const double a64 = (double)amax_s * c64;
  const double raw = a64 / 6.0;
  return e4m3_rne64(raw / st64);
}

// FP4 code of y = RN64(S * c64) against eff = ts * dec, exactly as numpy: u = RN64(y / eff).
__device__ __noinline__ uint32_t fp4_code_exact(float s, double c64, float ts, float dec) {
  const double y = (double)s * c64;
  const double eff = (double)ts * (double)dec;
  const double u = y / eff;
  const double a = fabs(u);
  uint32_t idx = (a > 0.25) + (a > 0.75) + (a == 0.75) + (a > 1.25) + (a > 1.75) + (a == 1.75) +
                 (a > 2.5) + (a > 3.5) + (a == 3.5) + (a > 5.0);
  // signbit(u) & idx > 0 -> sign nibble (formats.py:110); u = -0.0 keeps code 0
  return idx | ((signbit(u) && idx) ? 8u : 0u);
}

// ---------------------------------------------------------------------------
// hardware conversions
// ---------------------------------------------------------------------------
// 8 floats -> 8 E2M1 codes (satfinite, RNE), element 0 in the low nibble.
__device__ __forceinline__ uint32_t cvt_e2m1x8(const float (&u)[8]) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(r)
      : "f"(u[0]), "f"(u[1]), "f"(u[2]), "f"(u[3]), "f"(u[4]), "f"(u[5]), "f"(u[6]), "f"(u[7]));
  return r;
}

// A nibble whose magnitude rounded to 0 must be 0x0, not 0x8 (formats.py:110).
__device__ __forceinline__ uint32_t fix_neg_zero(uint32_t w) {
  const uint32_t mag = w & 0x77777777u;
  const uint32_t nz = (mag + 0x77777777u) & 0x88888888u;  // bit 3 of each nibble set iff mag > 0
  return mag | (w & nz);
}

__device__ __forceinline__ uint32_t cvt_e4m3(float x) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(x));
  return r & 0xFFu;
}

// ---------------------------------------------------------------------------
// group scale selection
// ---------------------------------------------------------------------------
struct GroupScale {
  uint32_t code;
  float ts;      // tensor scale (f32 value)
  float dec;     // decoded group scale (exact in fp32)
  float f;       // ~ c / (ts * dec), fp32
  bool slow_all; // force the exact element path (tiny scales)
};

__device__ __forceinline__ GroupScale mx_group_scale(uint32_t amax_bits, const AQParams& p, float kraw) {
  GroupScale g;
  int e = 0;
  if (amax_bits != 0) {
    const float raw32 = __uint_as_float(amax_bits) * kraw;   // ~ RN64(a/6), <= 1 ulp off
    const uint32_t rb = __float_as_uint(raw32);
    const int bexp = (int)(rb >> 23);
    const int d = (int)(rb & 0x7FFFFFu) - 0x3504F3;          // mantissa of sqrt(2)
    if (bexp == 0 || bexp == 255 || (d <= 64 && d >= -64)) {
      e = e8m0_exp_exact(__uint_as_float(amax_bits), p.c64);
    } else {
      e = bexp - 127 + (d > 0);
    }
    e = min(max(e, -127), 127);
  }
  g.code = (uint32_t)(e + 127);
  g.ts = 1.33333337306976318359375f;                          // f32(4/3), quantizers.py:34,191
  g.dec = e >= -126 ? __uint_as_float((uint32_t)(e + 127) << 23) : 5.877471754111438e-39f;  // 2^e
  const float eff = g.ts * g.dec;
  g.f = p.c32 * __frcp_rn(eff);
  g.slow_all = e < -100;
  return g;
}

__device__ __forceinline__ GroupScale nv_group_scale(uint32_t amax_bits, const AQParams& p, float kenc,
                                                     float st32, double st64, uint32_t zero_code) {
  GroupScale g;
  uint32_t code;
  if (amax_bits == 0) {
    code = zero_code;
  } else {
    const float enc32 = __uint_as_float(amax_bits) * kenc;   // ~ RN64(RN64(a/6)/s_T)
    const uint32_t eb = __float_as_uint(enc32);
    // E4M3 midpoints have <= 5 significant bits: low 19 mantissa bits are zero.
    const bool near = ((eb + 64u) & 0x7FFFFu) < 128u;
    if (near || eb >= 0x7f800000u || eb < 0x38800000u /* < 2^-14 */) {
      code = e4m3_code_exact(__uint_as_float(amax_bits), p.c64, st64);
    } else {
      code = cvt_e4m3(enc32);
    }
  }
  g.code = code;
  g.ts = st32;
  g.dec = e4m3_value(code);
  const float eff = st32 * g.dec;
  g.f = eff > 0.f ? p.c32 * __frcp_rn(eff) : 0.f;
  g.slow_all = eff < 1e-30f;
  return g;
}

// Quantize 8 consecutive rotated values S[lo..lo+8) against one group scale.
__device__ __forceinline__ uint32_t quantize8(const float (&v)[kSeg], int lo, const GroupScale& g,
                                              const AQParams& p) {
  constexpr float kEps = 3.814697265625e-06f;  // 2^-18
  const float fhi = g.f * (1.f + kEps), flo = g.f * (1.f - kEps);
  float uh[8], ul[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    uh[t] = v[lo + t] * fhi;
    ul[t] = v[lo + t] * flo;
  }
  const uint32_t wh = fix_neg_zero(cvt_e2m1x8(uh));
  const uint32_t wl = fix_neg_zero(cvt_e2m1x8(ul));
  uint32_t w = wh;
  uint32_t diff = wh ^ wl;
  if (g.slow_all) diff = 0xFFFFFFFFu;
  if (diff) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if ((diff >> (4 * t)) & 0xFu) {
        const uint32_t c = fp4_code_exact(v[lo + t], p.c64, g.ts, g.dec);
        w = (w & ~(0xFu << (4 * t))) | (c << (4 * t));
      }
    }
  }
  return w;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int IN, int HK>
__device__ __forceinline__ int load_and_rotate(const AQParams& p, int64_t row, int64_t col0,
                                               float (&v)[kSeg], int lane) {
  int nvalid = 0;
  if (row < p.M && col0 < p.K) nvalid = (col0 + kSeg <= p.K) ? kSeg : (int)(p.K - col0);
  load_seg<IN>(p.x, row * p.ldx + col0, nvalid, v);
  if constexpr (HK > 0) fwht<HK>(v, lane);
  return nvalid;
}

// NVFP4 phase 1: max |S| over the whole tensor (quantizers.py:198-200 needs it first).
template <int IN, int HK>
__global__ void __launch_bounds__(kThreads) k_tensor_absmax(AQParams p) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t row = (int64_t)blockIdx.y * kRowsPerCta + (tid >> 2);
  const int64_t col0 = ((int64_t)blockIdx.x * kSegsPerRow + (tid & 3)) * kSeg;
  float v[kSeg];
  const int nvalid = load_and_rotate<IN, HK>(p, row, col0, v, lane);
  uint32_t m = 0;
  if (nvalid) m = group_absmax_bits<HK, kSeg>(v, 0);  // zero-padded half segments are harmless
  m = __reduce_max_sync(0xffffffffu, m);
  __shared__ uint32_t smax[kThreads / 32];
  if (lane == 0) smax[tid >> 5] = m;
  __syncthreads();
  if (tid < 32) {
    uint32_t x = tid < kThreads / 32 ? smax[tid] : 0u;
    x = __reduce_max_sync(0xffffffffu, x);
    if (tid == 0 && x) {
      atomicMax(p.gmax, min(x, 0x7fc00000u));
      if (x >= 0x7f800000u) atomic_or_status(p.status, MRFP4_STATUS_NONFINITE);
    }
  }
}

template <int IN, int FMT, int HK>
__global__ void __launch_bounds__(kThreads, 3) k_act_quant(AQParams p) {
  constexpr int G = FMT == MRFP4_FMT_MXFP4 ? 32 : 16;
  constexpr int NG = kSeg / G;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t row = (int64_t)blockIdx.y * kRowsPerCta + (tid >> 2);
  const int64_t seg = (int64_t)blockIdx.x * kSegsPerRow + (tid & 3);
  const int64_t col0 = seg * kSeg;

  // Per-launch constants (uniform).
  float kscale;          // MXFP4: ~c/6 ; NVFP4: ~c/6/s_T
  float st32 = 1.f;
  double st64 = 1.0;
  uint32_t zero_code = 0;
  if constexpr (FMT == MRFP4_FMT_NVFP4) {
    const float smax = __uint_as_float(*p.gmax);         // max |S| over the tensor
    const double top = (double)smax * p.c64 / 6.0;      // absmax.max() / FP4_MAX
    st32 = top > 0.0 ? __double2float_rn(top / 448.0) : 1.0f;  // f32(top / E4M3 max)
    st64 = (double)st32;
    zero_code = e4m3_rne64(1.0 / st64);                  // raw = 1.0 sentinel (quantizers.py:187)
    kscale = __double2float_rn(p.c64 / 6.0 / st64);
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *p.tensor_scale = st32;
  } else {
    kscale = __double2float_rn(p.c64 / 6.0);
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *p.tensor_scale = 1.33333337306976318359375f;
  }

  float v[kSeg];
  const int nvalid = load_and_rotate<IN, HK>(p, row, col0, v, lane);

  const bool row_in_pad = row < p.rows_pad;
  if (nvalid == 0) {
    // Zero the padding of the swizzled scale buffer (rows >= M, columns >= K/G).
    if (row_in_pad) {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int64_t c = seg * NG + g;
        if (c < p.sf_col_blocks * 4) p.sf[sf_offset(row, c, p.sf_col_blocks)] = 0;
      }
    }
    return;
  }

  uint32_t words[kSeg / 8];
  uint32_t sfc[NG];
  uint32_t bad = 0;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const uint32_t ab = group_absmax_bits<HK, G>(v, g * G);
    const bool real = g * G < nvalid;  // a trailing half segment pads group 1 with zeros
    if (real && ab >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
    GroupScale gs;
    if constexpr (FMT == MRFP4_FMT_NVFP4) {
      gs = nv_group_scale(ab, p, kscale, st32, st64, zero_code);
      if (real && gs.code == 0) bad |= MRFP4_STATUS_SCALE_UNDERFLOW;
    } else {
      gs = mx_group_scale(ab, p, kscale);
    }
    sfc[g] = gs.code;
#pragma unroll
    for (int j = 0; j < G / 8; ++j) words[g * (G / 8) + j] = quantize8(v, g * G + 8 * j, gs, p);
  }
  if (bad) atomic_or_status(p.status, bad);

  // codes: 16 bytes (or 8 for a trailing half segment) at codes[row, col0/2]
  uint8_t* cdst = p.codes + row * (p.K >> 1) + (col0 >> 1);
  if (nvalid == kSeg) {
    if ((p.K & 31) == 0) {
      *reinterpret_cast<uint4*>(cdst) = make_uint4(words[0], words[1], words[2], words[3]);
    } else {
      reinterpret_cast<uint2*>(cdst)[0] = make_uint2(words[0], words[1]);
      reinterpret_cast<uint2*>(cdst)[1] = make_uint2(words[2], words[3]);
    }
  } else {
    *reinterpret_cast<uint2*>(cdst) = make_uint2(words[0], words[1]);
  }
  // scale codes straight into the swizzled layout
  if constexpr (NG == 1) {
    p.sf[sf_offset(row, seg, p.sf_col_blocks)] = (uint8_t)sfc[0];
  } else {
    const int64_t c0 = seg * 2;                  // c0 even -> c0, c0+1 share a 16-bit word
    const uint32_t hi = (nvalid == kSeg) ? sfc[1] : 0u;
    *reinterpret_cast<uint16_t*>(p.sf + sf_offset(row, c0, p.sf_col_blocks)) =
        (uint16_t)(sfc[0] | (hi << 8));
  }
}

template <int IN, int FMT>
int dispatch_hk(const AQParams& p, int hk, dim3 grid, cudaStream_t s) {
  switch (hk) {
#define MRFP4_CASE(K)                                                            \
  case K:                                                                        \
    if (FMT == MRFP4_FMT_NVFP4) k_tensor_absmax<IN, K><<<grid, kThreads, 0, s>>>(p); \
    k_act_quant<IN, FMT, K><<<grid, kThreads, 0, s>>>(p);                        \
    break;
    MRFP4_CASE(0)
    MRFP4_CASE(16)
    MRFP4_CASE(32)
    MRFP4_CASE(64)
    MRFP4_CASE(128)
#undef MRFP4_CASE
    default:
      return MRFP4_EUNSUPPORTED;
  }
  return MRFP4_OK;
}

template <int IN>
int dispatch_fmt(const AQParams& p, int fmt, int hk, dim3 grid, cudaStream_t s) {
  return fmt == MRFP4_FMT_MXFP4 ? dispatch_hk<IN, MRFP4_FMT_MXFP4>(p, hk, grid, s)
                                : dispatch_hk<IN, MRFP4_FMT_NVFP4>(p, hk, grid, s);
}

}  // namespace

// Host launcher; arguments validated by the C-ABI layer (capi.cu).
int launch_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int hk,
                     uint8_t* codes, uint8_t* sf, float* tensor_scale, uint32_t* status,
                     void* workspace, cudaStream_t s) {
  AQParams p;
  p.x = x;
  p.M = M;
  p.K = K;
  p.ldx = ldx;
  p.codes = codes;
  p.sf = sf;
  p.tensor_scale = tensor_scale;
  p.status = status;
  p.gmax = static_cast<uint32_t*>(workspace);
  const int G = fmt == MRFP4_FMT_MXFP4 ? 32 : 16;
  p.sf_cols = K / G;
  p.sf_col_blocks = ceil_div(p.sf_cols, 4);
  p.rows_pad = ceil_div(M, 128) * 128;
  p.c64 = hk ? 1.0 / sqrt((double)hk) : 1.0;
  p.c32 = (float)p.c64;
  // Columns: enough segments to cover K and the padded scale columns.
  const int64_t segs = std::max(ceil_div(K, kSeg), ceil_div(p.sf_col_blocks * 4, kSeg / G));
  dim3 grid((unsigned)ceil_div(segs, kSegsPerRow), (unsigned)ceil_div(p.rows_pad, kRowsPerCta));
  if (fmt == MRFP4_FMT_NVFP4) {
    if (cudaMemsetAsync(p.gmax, 0, sizeof(uint32_t), s) != cudaSuccess) return MRFP4_ECUDA;
  }
  int rc;
  switch (x_dtype) {
    case MRFP4_DT_BF16: rc = dispatch_fmt<MRFP4_DT_BF16>(p, fmt, hk, grid, s); break;
    case MRFP4_DT_F16: rc = dispatch_fmt<MRFP4_DT_F16>(p, fmt, hk, grid, s); break;
    case MRFP4_DT_F32: rc = dispatch_fmt<MRFP4_DT_F32>(p, fmt, hk, grid, s); break;
    default: return MRFP4_EUNSUPPORTED;
  }
  if (rc != MRFP4_OK) return rc;
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

}  // namespace mrfp4
