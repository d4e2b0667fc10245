// Shared device core of the FP4 activation quantizer (K1) -- the rotation, the group-scale
// decisions and the element rounding of quantize_rtn (/root/reference/pkg/src/microfp/
// quantizers.py:157-215, formats.py:94-113, :220-251) -- used by the act-quant kernels
// (act_quant.cu) and by the GEMM epilogue that quantizes its own output for the next layer
// (gemm_fp4.cu).  See act_quant.cu for the exactness argument.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace mrfp4 {
namespace qc {
namespace {

constexpr int kSeg = 32;       // elements per lane segment
constexpr int kPairs = kSeg / 2;

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
  int64_t items;           // warp items
  uint32_t div_m;          // ceil(2^32 / div_d): FlatWalk divides by nseg, GenWalk by nchunk
  int nchunk;              // column chunks of L segments per row group
  int seg_span;            // nchunk * L
  int lane_bits;           // log2(L)
  double c64;              // RN64(1 / RN64(sqrt(k)))  (transforms.py:65: H / np.sqrt(k))
  float kraw;              // MXFP4: ~ c / 6
  float kmx;               // MXFP4: ~ c / ts
  float mx_ts;             // MXFP4 tensor scale: f32(4/3), or 1.0 for e8m0_four_thirds=False
  const float* static_ts;  // NVFP4: device s_T given by the caller (single pass), or null
  unsigned long long pm;   // f32x2 (1, -1): FWHT h = 1 signs, a uniform-register operand of FFMA2
  int Mi, Ki;              // M, K as 32-bit (the C-ABI checks they fit)
  uint32_t half_k;         // K / 2: bytes per code row
  uint32_t cb;             // sf_col_blocks as 32-bit
  unsigned long long* trace;  // perf experiments: per-warp globaltimer stamps (null in production)
  uint64_t x_bytes;         // M * K * element size
  int marks;                // NVFP4 ring-resident re-encode: -1 auto, 0 off, 1 on
  int nseg;                // flat walk: segments per row (K / 32)
  uint32_t total_segs;     // flat walk: M * K / 32
};

// ---------------------------------------------------------------------------
// packed f32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2)
// ---------------------------------------------------------------------------
typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_of(u64 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_of(u64 v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// max(|a|, |b|, |c|), NaN-propagating (a NaN anywhere in a group must reach the status check)
__device__ __forceinline__ float amax3(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(fabsf(a)), "f"(fabsf(b)), "f"(fabsf(c)));
  return r;
}
__device__ __forceinline__ float max3n(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Unnormalized fast Walsh-Hadamard transform (Sylvester natural order) of the segment.
template <int HK>
__device__ __forceinline__ void fwht(u64 (&P)[kPairs], int lane, u64 pm) {
  // h = 1: (x + y, x - y) inside each pair, one FFMA2 with broadcast x and y
#pragma unroll
  for (int i = 0; i < kPairs; ++i) {
    const float x = lo_of(P[i]), y = hi_of(P[i]);
    P[i] = fma2(pk(y, y), pm, pk(x, x));
  }
  // h = 2 .. min(k, 32)/2: element h apart = pair h/2 apart
  constexpr int kIn = (HK < kSeg ? HK : kSeg) / 2;
#pragma unroll
  for (int hp = 1; hp < kIn; hp <<= 1) {
#pragma unroll
    for (int i = 0; i < kPairs; ++i) {
      if ((i & hp) == 0) {
        const u64 a = P[i], b = P[i + hp];
        P[i] = add2(a, b);
        P[i + hp] = sub2(a, b);
      }
    }
  }
  // Cross-lane stages: block element index bit 5 (k >= 64) lives in lane bit 0,
  // bit 6 (k = 128) in lane bit 1.  Lower partner keeps a+b, upper keeps a-b (exact: sg = +-1).
  if constexpr (HK >= 64) {
    const float s = (lane & 1) ? -1.f : 1.f;
    const u64 sg = pk(s, s);
#pragma unroll
    for (int i = 0; i < kPairs; ++i) P[i] = fma2(sg, P[i], __shfl_xor_sync(0xffffffffu, P[i], 1));
  }
  if constexpr (HK >= 128) {
    const float s = (lane & 2) ? -1.f : 1.f;
    const u64 sg = pk(s, s);
#pragma unroll
    for (int i = 0; i < kPairs; ++i) P[i] = fma2(sg, P[i], __shfl_xor_sync(0xffffffffu, P[i], 2));
  }
}

// Absmax of pairs [0, 8) (elements 0..15) and [8, 16) (elements 16..31): NaN-propagating.
__device__ __forceinline__ void half_amax(const u64 (&P)[kPairs], float& m0, float& m1) {
  float a[6], b[6];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int o = 8 * t;
    float* d = t ? b : a;
    d[0] = amax3(lo_of(P[o]), hi_of(P[o]), lo_of(P[o + 1]));
    d[1] = amax3(hi_of(P[o + 1]), lo_of(P[o + 2]), hi_of(P[o + 2]));
    d[2] = amax3(lo_of(P[o + 3]), hi_of(P[o + 3]), lo_of(P[o + 4]));
    d[3] = amax3(hi_of(P[o + 4]), lo_of(P[o + 5]), hi_of(P[o + 5]));
    d[4] = amax3(lo_of(P[o + 6]), hi_of(P[o + 6]), lo_of(P[o + 7]));
    d[5] = fabsf(hi_of(P[o + 7]));
  }
  m0 = max3n(max3n(a[0], a[1], a[2]), max3n(a[3], a[4], a[5]), 0.f);
  m1 = max3n(max3n(b[0], b[1], b[2]), max3n(b[3], b[4], b[5]), 0.f);
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

// One float -> its E2M1 code (satfinite, RNE) in the low nibble.
__device__ __forceinline__ uint32_t cvt_e2m1x1(float x) {
  uint16_t r;
  asm("{\n\t.reg .b8 b0;\n\tcvt.rn.satfinite.e2m1x2.f32 b0, %1, %2;\n\tcvt.u16.u8 %0, b0;\n\t}"
      : "=h"(r)
      : "f"(0.0f), "f"(x));
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

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---------------------------------------------------------------------------
// group scale selection
// ---------------------------------------------------------------------------
struct GroupScale {
  uint32_t code;
  float dec;     // decoded group scale (exact in fp32)
  float f;       // ~ c / (ts * dec), fp32
  bool slow_all; // force the exact element path (extreme scales)
};

__device__ __forceinline__ GroupScale mx_group_scale(float amax, const AQParams& p) {
  GroupScale g;
  const uint32_t ab = __float_as_uint(amax);
  const uint32_t rb = __float_as_uint(amax * p.kraw);         // ~ RN64(a/6), <= 1 ulp off
  const int bexp = (int)(rb >> 23);
  const int d = (int)(rb & 0x7FFFFFu) - 0x3504F3;              // vs the mantissa of sqrt(2)
  int e = bexp - 127 + (d > 0);
  if ((uint32_t)(d + 64) <= 128u || bexp == 0 || bexp == 255) {
    e = ab ? e8m0_exp_exact(amax, p.c64) : 0;                  // rare: near a threshold / extreme
  }
  e = min(max(e, -127), 127);
  g.code = (uint32_t)(e + 127);
  g.dec = __uint_as_float(e >= -126 ? (uint32_t)(e + 127) << 23 : 0x00400000u);  // 2^e
  g.slow_all = e < -100 || e > 100;
  g.f = p.kmx * __uint_as_float((uint32_t)(127 - min(max(e, -100), 100)) << 23);   // c/ts * 2^-e
  return g;
}

// kFma (decode kernel), c_pow2 (c64 a power of 2): near a true E4M3 midpoint M of the normal
// range, v = RN64(RN64(a * c / 6) / s_T) vs M follows sign(a * c - 6 M s_T), one exact fmaf
// (x = a * c exact, 6 M has <= 7 significant bits).  If x != 6 M s_T their difference is a
// multiple of a quantum >= 2^-29 * x, far beyond the two float64 roundings (2^-52), so v lies
// on the same side as the quotient; if equal, v == M exactly (M s_T has <= 29 bits) and RNE
// picks the even code.  Everything else: the float64 chain.
template <bool kFma = false>
__device__ __forceinline__ GroupScale nv_group_scale(float amax, const AQParams& p, float kenc, float knv,
                                                     float st32, double st64, uint32_t zero_code,
                                                     bool c_pow2 = false) {
  GroupScale g;
  const uint32_t ab = __float_as_uint(amax);
  const float enc32 = amax * kenc;                            // ~ RN64(RN64(a/6)/s_T)
  const uint32_t eb = __float_as_uint(enc32);
  uint32_t code = cvt_e4m3(enc32);
  // E4M3 midpoints have <= 5 significant bits: low 19 mantissa bits are zero.
  if (((eb + 64u) & 0x7FFFFu) < 128u || eb >= 0x7f800000u || eb < 0x38800000u /* < 2^-14 */) {
    bool done = false;
    if constexpr (kFma) {
      const uint32_t mb = (eb + 64u) & ~0x7FFFFu;               // the 5-bit value enc32 is near
      const float x = amax * (float)p.c64;
      if (c_pow2 && ((eb + 64u) & 0x7FFFFu) < 128u && (mb & 0x80000u) && mb >= 0x3C800000u /* 2^-6 */ &&
          mb <= 0x43E00000u /* 448 */ && x >= 0x1p-100f) {
        const uint32_t lower = cvt_e4m3(__uint_as_float(mb - 1u));
        const float r = fmaf(-6.f * __uint_as_float(mb), st32, x);
        code = r > 0.f ? lower + 1u : r < 0.f ? lower : lower + (lower & 1u);
        done = true;
      }
    }
    if (!done)
      code = ab ? e4m3_code_exact(amax, p.c64, st64) : zero_code != ~0u ? zero_code : e4m3_rne64(1.0 / st64);
  }
  g.code = code;
  g.dec = e4m3_value(code);
  const float eff = st32 * g.dec;
  g.slow_all = !(eff >= 1e-30f);
  g.f = knv * rcp_approx(g.dec);
  return g;
}

// Per-launch encode constants.  MXFP4: ts = f32(4/3) (quantizers.py:34,191).  NVFP4: derived
// from the whole-tensor max exactly as numpy does (quantizers.py:187, :198-200).
struct EncConsts {
  float st32 = 1.33333337306976318359375f;
  double st64 = 1.0;
  float kenc = 0.f, knv = 0.f;
  uint32_t zero_code = 0;
};

__device__ __forceinline__ EncConsts nv_consts_st(const AQParams& p, float st32) {
  EncConsts k;
  k.st32 = st32;
  k.st64 = (double)k.st32;
  k.zero_code = e4m3_rne64(1.0 / k.st64);                               // raw = 1.0 sentinel
  k.kenc = __double2float_rn(p.c64 / 6.0 / k.st64);
  k.knv = __double2float_rn(p.c64 / k.st64);
  return k;
}

// nv_consts_st split over 4 threads (part 0..3 each writes its own field of `k`).
// NVFP4 encode constants from the whole-tensor max |y| bits `xb` on ONE thread, without float64
// where it can (decode kernel: this sits between the cross-CTA max exchange and quantization).
//  * s_T = RN32(RN64(RN64(x * c64) / 6) / 448) (quantizers.py:198-200).  When c64 is a power of 2
//    (k in {0, 16}, and any k = 4^j) x * c64 is exact and the chain equals RN32(x * c64 / 2688):
//    x * c64 / 21 is never within 2^-52 (relative) of an fp32 rounding midpoint -- a midpoint has
//    25 significant bits ending in 1, and 21 * midpoint needs more than x's 24 bits -- so both
//    roundings agree with the correctly rounded fp32 division.  Otherwise: the float64 chain.
//  * kenc / knv only feed the fast path's estimates (their errors of a few ulp sit far inside
//    its 64-ulp / 2^-18 exactness windows), so fp32 divisions suffice.
//  * zero_code (all-zero groups, rare) is formed on demand in nv_group_scale (~0u sentinel).
__device__ __forceinline__ EncConsts nv_consts_fast(const AQParams& p, bool c_pow2, uint32_t xb) {
  EncConsts k;
  const float x = __uint_as_float(xb);
  float st;
  if (c_pow2) {
    const float y = x * (float)p.c64;
    st = y > 0.f ? __fdiv_rn(y, 2688.f) : 1.0f;
  } else {
    const double top = (double)x * p.c64 / 6.0;
    st = top > 0.0 ? __double2float_rn(top / 448.0) : 1.0f;
  }
  k.st32 = st;
  k.st64 = (double)st;
  k.kenc = __fdiv_rn(p.kraw, st);
  k.knv = __fdiv_rn((float)p.c64, st);
  k.zero_code = ~0u;
  return k;
}

struct SegVals { u64 p[kPairs]; };
struct Words4 { uint32_t w[4]; };

// The rare exact path of quantize_seg, out of line (passed by value: the caller's registers stay
// registers) so that the hot instruction stream stays dense: every element whose code could
// depend on the last bits of its fp32 value is re-decided in float64.  Rolled over the 4 words,
// 8 independent elements per iteration.
__device__ __noinline__ Words4 requant_exact(SegVals v, GroupScale s0, GroupScale s1, float ts, double c64,
                                             Words4 w) {
  constexpr float kEps = 3.814697265625e-06f;  // 2^-18
#pragma unroll 1
  for (int wi = 0; wi < 4; ++wi) {
    const bool lo = wi < 2;
    const float gf = lo ? s0.f : s1.f, gdec = lo ? s0.dec : s1.dec;
    const bool slow = lo ? s0.slow_all : s1.slow_all;
    u64 q[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      q[t] = v.p[t];
#pragma unroll
      for (int z = 1; z < 4; ++z) q[t] = wi == z ? v.p[4 * z + t] : q[t];
    }
    uint32_t word = w.w[0];
#pragma unroll
    for (int z = 1; z < 4; ++z) word = wi == z ? w.w[z] : word;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float x = (t & 1) ? hi_of(q[t / 2]) : lo_of(q[t / 2]);
      if (slow || ((cvt_e2m1x1(x * (gf * (1.f + kEps))) ^ cvt_e2m1x1(x * (gf * (1.f - kEps)))) & 0xFu)) {
        const uint32_t c = fp4_code_exact(x, c64, ts, gdec);
        word = (word & ~(0xFu << (4 * t))) | (c << (4 * t));
      }
    }
#pragma unroll
    for (int z = 0; z < 4; ++z)
      if (wi == z) w.w[z] = word;
  }
  return w;
}

// Exact E2M1 code of u = RN64(RN64(x * c64) / RN64(ts * dec)) (fp4_code_exact's decision) with
// no division, for c64 a power of 2 (c32 = c64) and |x| >= 2^-100, dec * 5 finite: y = |x| * c
// is exact, and so is each threshold product T * dec (<= 7 significant bits).  RN64(y / eff)
// vs T follows sign(y - T * ts * dec), which one fmaf gets exactly: if y != T * eff, their
// difference is a multiple of a quantum >= 2^-31 * y, so y / eff is more than half an ulp of
// T away from T and rounding cannot reach it; if equal, u == T exactly.
__device__ __forceinline__ uint32_t fp4_code_fma(float x, float c32, float ts, float dec) {
  const float y = fabsf(x) * c32;
  uint32_t idx = 0;
  constexpr float kT[7] = {0.25f, 0.75f, 1.25f, 1.75f, 2.5f, 3.5f, 5.f};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    const float r = fmaf(-(kT[i] * dec), ts, y);
    idx += r > 0.f;
    if (i == 1 || i == 3 || i == 5) idx += r == 0.f;   // ties at 0.75 / 1.75 / 3.5 go up (even code)
  }
  return idx | ((signbit(x) && idx) ? 8u : 0u);
}

// Codes of the segment as 4 words (word w = elements 8w..8w+7 = pairs 4w..4w+3).
// s0 scales pairs 0..7 (elements 0..15), s1 pairs 8..15.
// kOutOfLine (the decode kernel: once-per-launch code, every inline instruction fetched cold):
// the flagged elements are re-decided by a short inline loop (fp4_code_fma when c_pow2), whole
// extreme-scale groups by an out-of-line call (requant_exact) -- instead of the inline
// fully-unrolled exact block.
template <bool kOutOfLine = false>
__device__ __forceinline__ void quantize_seg(const u64 (&P)[kPairs], const GroupScale& s0, const GroupScale& s1,
                                             float ts, const AQParams& p, uint32_t (&w)[4], bool c_pow2 = false) {
  constexpr float kEps = 3.814697265625e-06f;  // 2^-18
  const float h0 = s0.f * (1.f + kEps), l0 = s0.f * (1.f - kEps);
  const float h1 = s1.f * (1.f + kEps), l1 = s1.f * (1.f - kEps);
  uint32_t diff = 0, dw[4];
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const float fh = wi < 2 ? h0 : h1, fl = wi < 2 ? l0 : l1;
    float uh[8], ul[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const u64 a = mul2(P[4 * wi + t], pk(fh, fh)), b = mul2(P[4 * wi + t], pk(fl, fl));
      uh[2 * t] = lo_of(a); uh[2 * t + 1] = hi_of(a);
      ul[2 * t] = lo_of(b); ul[2 * t + 1] = hi_of(b);
    }
    const uint32_t a = cvt_e2m1x8(uh), b = cvt_e2m1x8(ul);
    w[wi] = a;
    dw[wi] = a ^ b;
    diff |= a ^ b;
  }
  if (kOutOfLine && (s0.slow_all | s1.slow_all)) {
    SegVals sv;
#pragma unroll
    for (int i = 0; i < kPairs; ++i) sv.p[i] = P[i];
    const Words4 r = requant_exact(sv, s0, s1, ts, p.c64, Words4{{w[0], w[1], w[2], w[3]}});
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) w[wi] = r.w[wi];
  } else if (kOutOfLine && diff) {
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
      const float dec = wi < 2 ? s0.dec : s1.dec;
      uint32_t d = dw[wi];
#pragma unroll 1
      while (d) {
        const int t = (__ffs(d) - 1) >> 2;     // nibble = element of the word
        d &= ~(0xFu << (4 * t));
        u64 pr = P[4 * wi];
#pragma unroll
        for (int z = 1; z < 4; ++z) pr = (t >> 1) == z ? P[4 * wi + z] : pr;
        const float x = (t & 1) ? hi_of(pr) : lo_of(pr);
        const uint32_t c = c_pow2 && fabsf(x) >= 0x1p-100f ? fp4_code_fma(x, (float)p.c64, ts, dec)
                                                            : fp4_code_exact(x, p.c64, ts, dec);
        w[wi] = (w[wi] & ~(0xFu << (4 * t))) | (c << (4 * t));
      }
    }
  }
  if (!kOutOfLine && (diff | (uint32_t)(s0.slow_all | s1.slow_all))) {
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
      const GroupScale& g = wi < 2 ? s0 : s1;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const u64 pr = P[4 * wi + t / 2];
        const float s = (t & 1) ? hi_of(pr) : lo_of(pr);
        float a[8], b[8];
        a[0] = s * (g.f * (1.f + kEps)); b[0] = s * (g.f * (1.f - kEps));
#pragma unroll
        for (int z = 1; z < 8; ++z) { a[z] = 0.f; b[z] = 0.f; }
        if (g.slow_all || ((cvt_e2m1x8(a) ^ cvt_e2m1x8(b)) & 0xFu)) {
          const uint32_t c = fp4_code_exact(s, p.c64, ts, g.dec);
          w[wi] = (w[wi] & ~(0xFu << (4 * t))) | (c << (4 * t));
        }
      }
    }
  }
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) w[wi] = fix_neg_zero(w[wi]);
}

}  // namespace
}  // namespace qc
}  // namespace mrfp4
