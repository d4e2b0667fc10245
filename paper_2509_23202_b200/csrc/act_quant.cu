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
// Work decomposition (HBM-bound kernel; 2.5 + 1/G bytes per bf16 element):
//   * A lane owns one 32-element column segment of one row, held as 16 packed pairs
//     P[j] = (v[2j], v[2j+1]) -- exactly the (low, high) halves of the j-th bf16x2
//     input word and the two nibbles of the j-th output byte.  FWHT stage h = 1 is the
//     in-pair butterfly (one FFMA2 with broadcast operands), stages h = 2..16 and the
//     cross-lane stages are FADD2 / FFMA2 between pairs, the group scaling is FMUL2.
//   * A warp item is 32 segments: L = 2^ceil(log2(K/32)) lanes (<= 32) cover a row
//     chunk, so short rows pack several rows per warp.  Hadamard blocks of k <= 32
//     rotate in registers; k = 64 / 128 add 1 / 2 shuffle stages across lane bits 0 / 1.
//   * Persistent grid; each warp walks a contiguous range of items with incremental
//     (row, segment) cursors, each lane streaming its segments through a private
//     3-stage cp.async ring in shared memory (16-B chunks XOR-swizzled by lane, so the
//     16-B shared loads are bank-conflict free) -- no block barriers on the data path.
//   * Scale codes go straight into the swizzled tensor-core layout, codes out as one
//     16-B store per segment.
//
// Exactness: the rotation is an fp32 FWHT (exact whenever the block sum fits in
// 24 bits; validated by the parity tests).  All downstream decisions reproduce the
// reference's float64 arithmetic on the rotated value y = S * c:  scale codes are
// decided from an fp32 estimate and re-decided in float64 whenever the estimate is
// within 2^-17 of a rounding threshold; element codes are rounded twice through the
// hardware E2M1 conversion, from u * (1 +- 2^-18) (the fp32 u ~ y / eff is within
// 2^-21 of the exact quotient), and any element whose two roundings disagree is
// re-decided from u = RN64(y / eff) exactly as numpy does (quantizers.py:213).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "quant_core.cuh"

namespace mrfp4 {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // gemm_fp4.cu

namespace {

using namespace qc;

constexpr int kMetricWarps = 8;
#ifndef MRFP4_K1_STAGES
#define MRFP4_K1_STAGES 3
#endif
constexpr int kMaxStages = 3;

template <int IN>
struct InCfg {
  static constexpr int kEs = IN == MRFP4_DT_F32 ? 4 : 2;
  static constexpr int kChunks = kSeg * kEs / 16;          // 16-B chunks per segment: 4 or 8
  static constexpr int kLaneBytes = kSeg * kEs;
  // ring depth per warp (f32 rows are twice as long: 2 stages fit the 227 KB of SMEM)
  static constexpr int kStages = kEs == 4 ? 2 : MRFP4_K1_STAGES;
  static constexpr int smem(int warps) { return warps * kStages * 32 * kLaneBytes + 1024; }  // + 1 KB alignment
};


// ---------------------------------------------------------------------------
// cp.async ring
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}

// Physical 16-B chunk of logical chunk j in a lane's ring slot: XOR-swizzled so the
// eight lanes of a quarter warp hit eight different 16-B bank groups on a 16-B load.
template <int IN>
__device__ __forceinline__ uint32_t swz(int j, int lane) {
  return InCfg<IN>::kChunks == 8 ? (uint32_t)(j ^ (lane & 7)) : (uint32_t)(j ^ ((lane >> 1) & 3));
}

// A lane's position: row and 32-element column segment of the current warp item.
// Items are row-group-major (item = rg * nchunk + cc); a warp walks a contiguous range.
// Two walkers share one interface (at / step / issue / live / full / row / seg / cdst):
//   GenWalk  -- any K and row stride: L = 2^lane_bits lanes per row chunk, ragged tails
//               zero-filled.
//   FlatWalk -- contiguous rows (ldx == K), K % 32 == 0, K >= 1024: lane segment
//               s = 32 * item + lane of the flattened matrix, so a segment is 64 contiguous
//               bytes, never straddles a row, and the row / column cursor is one compare per
//               step.  Lane groups of 2 / 4 (H64 / H128 shuffles) stay inside one Hadamard
//               block because K % k == 0.
// n / d for n < 2^31 with m = ceil(2^32 / d) (m = 0 encodes d = 1): the estimate is exact or
// one too large.
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t d, uint32_t m) {
  uint32_t q = m ? __umulhi(n, m) : n;
  if ((int)(n - q * d) < 0) --q;
  return q;
}

struct GenWalk {
  static constexpr bool kTma = false;
  int row_, seg_;
  __device__ __forceinline__ void at(const AQParams& p, int item, int lane) {
    const int rg = (int)fast_div((uint32_t)item, (uint32_t)p.nchunk, p.div_m);
    const int cc = item - rg * p.nchunk;
    row_ = (int)(rg * (32 >> p.lane_bits)) + (lane >> p.lane_bits);
    seg_ = (cc << p.lane_bits) + (lane & ((1 << p.lane_bits) - 1));
  }
  template <int DIR>
  __device__ __forceinline__ void step(const AQParams& p) {
    if constexpr (DIR > 0) {
      seg_ += 1 << p.lane_bits;
      if (seg_ >= p.seg_span) { seg_ -= p.seg_span; row_ += 32 >> p.lane_bits; }
    } else {
      seg_ -= 1 << p.lane_bits;
      if (seg_ < 0) { seg_ += p.seg_span; row_ -= 32 >> p.lane_bits; }
    }
  }
  template <int IN>
  __device__ __forceinline__ void issue(const AQParams& p, uint32_t sbase, int lane) const;
  __device__ __forceinline__ bool live(const AQParams& p) const { return seg_ * kSeg < p.Ki && row_ < p.Mi; }
  __device__ __forceinline__ bool full(const AQParams& p) const { return seg_ * kSeg + kSeg <= p.Ki; }
  __device__ __forceinline__ int row() const { return row_; }
  __device__ __forceinline__ int seg() const { return seg_; }
  __device__ __forceinline__ uint8_t* cdst(const AQParams& p) const {
    return p.codes + (uint64_t)row_ * p.half_k + (uint32_t)(seg_ * (kSeg / 2));
  }
};

struct FlatWalk {
  static constexpr bool kTma = true;
  uint32_t s_;
  int row_, seg_;
  __device__ __forceinline__ void at(const AQParams& p, int item, int lane) {
    s_ = (uint32_t)item * 32u + (uint32_t)lane;
    row_ = (int)fast_div(s_, (uint32_t)p.nseg, p.div_m);
    seg_ = (int)(s_ - (uint32_t)row_ * (uint32_t)p.nseg);
  }
  template <int DIR>
  __device__ __forceinline__ void step(const AQParams& p) {
    if constexpr (DIR > 0) {
      s_ += 32u;
      seg_ += 32;
      if (seg_ >= p.nseg) { seg_ -= p.nseg; ++row_; }
    } else {
      s_ -= 32u;
      seg_ -= 32;
      if (seg_ < 0) { seg_ += p.nseg; --row_; }
    }
  }
  template <int IN>
  __device__ __forceinline__ void issue(const AQParams& p, uint32_t sbase, int lane) const {
    using C = InCfg<IN>;
    if (s_ < p.total_segs) {
      const char* src = static_cast<const char*>(p.x) + (uint64_t)s_ * C::kLaneBytes;
#pragma unroll
      for (int j = 0; j < C::kChunks; ++j) cp_async16(sbase + swz<IN>(j, lane) * 16, src + j * 16, 16u);
    }
  }
  __device__ __forceinline__ bool live(const AQParams& p) const { return s_ < p.total_segs; }
  __device__ __forceinline__ bool full(const AQParams&) const { return true; }
  __device__ __forceinline__ int row() const { return row_; }
  __device__ __forceinline__ int seg() const { return seg_; }
  __device__ __forceinline__ uint8_t* cdst(const AQParams& p) const { return p.codes + (uint64_t)s_ * (kSeg / 2); }
};

template <int IN>
__device__ __forceinline__ void GenWalk::issue(const AQParams& p, uint32_t sbase, int lane) const {
  using C = InCfg<IN>;
  const int col0 = seg_ * kSeg;
  const char* x = static_cast<const char*>(p.x);
  if (row_ < p.Mi && col0 + kSeg <= p.Ki) {  // interior segment
    const char* src = x + ((uint64_t)row_ * (uint64_t)p.ldx + (uint32_t)col0) * C::kEs;
#pragma unroll
    for (int j = 0; j < C::kChunks; ++j) cp_async16(sbase + swz<IN>(j, lane) * 16, src + j * 16, 16u);
    return;
  }
  const int nb = (col0 < p.Ki && row_ < p.Mi) ? (p.Ki - col0) * C::kEs : 0;  // < kSeg * kEs here
  const char* src = nb ? x + ((uint64_t)row_ * (uint64_t)p.ldx + (uint32_t)col0) * C::kEs : x;
#pragma unroll
  for (int j = 0; j < C::kChunks; ++j) {
    const int rem = nb - j * 16;
    const uint32_t bytes = rem >= 16 ? 16u : (rem > 0 ? (uint32_t)rem : 0u);
    cp_async16(sbase + swz<IN>(j, lane) * 16, bytes ? src + j * 16 : x, bytes);
  }
}

// Shared memory -> P[j] = (v[2j], v[2j+1]), fp32.
template <int IN>
__device__ __forceinline__ void load_pairs(uint32_t sbase, int lane, u64 (&P)[kPairs]) {
  using C = InCfg<IN>;
  uint32_t w[kSeg * C::kEs / 4];
#pragma unroll
  for (int j = 0; j < C::kChunks; ++j) {
    const uint4 a = lds128(sbase + swz<IN>(j, lane) * 16);
    w[4 * j] = a.x; w[4 * j + 1] = a.y; w[4 * j + 2] = a.z; w[4 * j + 3] = a.w;
  }
#pragma unroll
  for (int j = 0; j < kPairs; ++j) {
    if constexpr (IN == MRFP4_DT_F32) {
      P[j] = pk(__uint_as_float(w[2 * j]), __uint_as_float(w[2 * j + 1]));
    } else if constexpr (IN == MRFP4_DT_BF16) {
      P[j] = pk(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xFFFF0000u));
    } else {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
      P[j] = pk(f.x, f.y);
    }
  }
}



// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Work split: CTA b (one per SM) owns the contiguous items [c0, c1); its warps claim them
// one at a time from a shared-memory counter.  DRAM service is far from uniform across the
// warps of a grid (per-warp first-load latency ranges 1.5-11 us at 2048x14336), so a static
// per-warp split ends when the unluckiest warp does; a per-SM queue lets the SM's other warps
// absorb it (scripts/k1_trace.py).  A claim is made one item ahead, hiding its latency.
struct CtaRange {
  int c0, cnt;
  __device__ __forceinline__ void init(const AQParams& p) {
    c0 = (int)((int64_t)blockIdx.x * p.items / gridDim.x);
    cnt = (int)((int64_t)(blockIdx.x + 1) * p.items / gridDim.x) - c0;
  }
};

struct Claims {
  uint32_t* ctr;   // shared-memory counter
  int cnt;
  uint32_t pend;   // lane 0: claimed index (claimed one item ahead)
  bool live;
  __device__ __forceinline__ void init(uint32_t* c, int n, int lane) {
    ctr = c;
    cnt = n;
    live = true;
    if (lane == 0) pend = atomicAdd(ctr, 1u);
  }
  // Next claimed index in [0, cnt), or -1 once the range is exhausted (then forever -1).
  __device__ __forceinline__ int next(int lane) {
    if (!live) return -1;
    const int c = (int)__shfl_sync(0xffffffffu, pend, 0);
    if (c >= cnt) { live = false; return -1; }
    if (lane == 0) pend = atomicAdd(ctr, 1u);
    return c;
  }
};

// Per-warp ring of kStages item slots (32 lane segments each) in shared memory.
//   GenWalk (cp.async): every lane copies its own segment in 16-B chunks, XOR-swizzled by
//     lane so the 16-B shared loads are bank-conflict free.
//   FlatWalk (TMA): lane 0 issues one 2-D tensor copy of the item's 32 contiguous segments;
//     the 64-B (bf16 / f16) or 128-B (f32) TMA swizzle produces exactly the same layout, and
//     completion is tracked by one mbarrier per slot.  One request per 2-4 KB instead of 128.
template <int IN, typename W>
struct Loader {
  using C = InCfg<IN>;
  static constexpr int kStages = C::kStages;
  static constexpr uint32_t kStride = 32 * C::kLaneBytes;
  uint32_t wbase, lbase, bars, ph;
  int lane;
  __device__ __forceinline__ void init(uint32_t ring, uint32_t bar_addr, int lane_) {
    lane = lane_;
    wbase = ring;
    lbase = ring + (uint32_t)lane_ * C::kLaneBytes;
    bars = bar_addr;
    ph = 0;
    if constexpr (W::kTma) {
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kStages; ++s)
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncwarp();
    }
  }
  __device__ __forceinline__ uint32_t slot(int s) const { return lbase + (uint32_t)s * kStride; }
  __device__ __forceinline__ void issue(const AQParams& p, const CUtensorMap* tm, int item, int s) {
    if constexpr (W::kTma) {
      if (lane == 0) {
        const uint32_t bar = bars + 8 * s;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kStride) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4}], [%2];" ::"r"(wbase + (uint32_t)s * kStride),
            "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(0), "r"(item * 32)
            : "memory");
      }
    } else {
      W c;
      c.at(p, item, lane);
      c.template issue<IN>(p, slot(s), lane);
    }
  }
  __device__ __forceinline__ void commit() {
    if constexpr (!W::kTma) cp_commit();
  }
  // Data of the oldest outstanding slot `s` has landed (cp.async: all but kStages-1 groups).
  __device__ __forceinline__ void wait(int s) {
    if constexpr (W::kTma) {
      const uint32_t par = (ph >> s) & 1u;
      asm volatile(
          "{\n\t.reg .pred P1;\n"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@!P1 bra WAIT_%=;\n\t}" ::"r"(bars + 8 * s),
          "r"(par)
          : "memory");
      ph ^= 1u << s;
    } else {
      cp_wait<kStages - 1>();
    }
  }
  __device__ __forceinline__ void wait_all() {
    if constexpr (!W::kTma) cp_wait<0>();
  }
  // Before a slot this warp has read is refilled by the async proxy.
  __device__ __forceinline__ void release() {
    if constexpr (W::kTma) {
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
};

// The warp's ring: kStages slots in dynamic shared memory (1 KB aligned for the TMA swizzle),
// mbarriers in static shared memory.
template <int NW, int IN, typename W>
__device__ __forceinline__ void init_loader(Loader<IN, W>& L, int warp, int lane) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  constexpr int kStages = InCfg<IN>::kStages;
  __shared__ __align__(8) uint64_t bars[NW * kMaxStages];
  const uint32_t base = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  L.init(base + (uint32_t)warp * kStages * Loader<IN, W>::kStride,
         (uint32_t)__cvta_generic_to_shared(&bars[warp * kMaxStages]), lane);
}

// Per-warp pipeline over the items `next()` yields (-1 = done): issue item j+kStages-1 while
// item j is processed; item j of the walk sits in ring slot j % kStages.  `resident[s]`
// (warp-private shared memory) receives the last item processed from slot s (-1: none).
template <int IN, typename W, typename N, typename F>
__device__ __forceinline__ int run_pipeline(const AQParams& p, const CUtensorMap* tm, Loader<IN, W>& L, N&& next,
                                            int* resident, F&& body) {
  constexpr int kStages = InCfg<IN>::kStages;
  const int lane = threadIdx.x & 31;
  int it[kStages];
  L.release();
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    it[s] = next();
    if (it[s] >= 0) L.issue(p, tm, it[s], s);
    L.commit();
  }
  int rd = 0, wr = kStages - 1, n = 0;
  while (true) {
    it[kStages - 1] = next();
    if (it[kStages - 1] >= 0) {
      L.release();
      L.issue(p, tm, it[kStages - 1], wr);
    }
    L.commit();
    if (it[0] < 0) break;
    L.wait(rd);
    W c;
    c.at(p, it[0], lane);
    body(c, L.slot(rd));
    if (resident && lane == 0) resident[rd] = it[0];
    ++n;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) it[s] = it[s + 1];
    rd = rd + 1 == kStages ? 0 : rd + 1;
    wr = wr + 1 == kStages ? 0 : wr + 1;
  }
  L.wait_all();
  return n;
}

// sf_offset in 32-bit arithmetic (scale buffers are < 4 GiB).
__device__ __forceinline__ uint32_t sf_off32(uint32_t r, uint32_t c, uint32_t cb) {
  return ((r >> 7) * cb + (c >> 2)) * 512u + (r & 31u) * 16u + ((r >> 5) & 3u) * 4u + (c & 3u);
}

// Zero the padding of the swizzled scale buffer: rows [M, rows_pad) (whole 4-byte words)
// and columns [sf_cols, 4*col_blocks) of the real rows (<= 3 bytes per row).
// Padding rows all lie in the last 128-row block, whose cb atoms are one contiguous run of
// cb * 512 bytes: word i of it belongs to row (i % 128 / 4) + 32 * (i % 4) of its atom, so
// the grid walks the run linearly (coalesced) and zeroes the words of rows >= M % 128.
__device__ __forceinline__ void zero_sf_padding(const AQParams& p) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const uint32_t M = (uint32_t)p.Mi, cb = p.cb;
  const uint32_t live = M & 127u;
  if (live) {
    uint32_t* run = reinterpret_cast<uint32_t*>(p.sf + (size_t)(M >> 7) * cb * 512u);
    for (uint32_t i = tid; i < cb * 128u; i += nth) {
      const uint32_t r = ((i & 127u) >> 2) + 32u * (i & 3u);
      if (r >= live) run[i] = 0u;
    }
  }
  const uint32_t sfc = (uint32_t)p.sf_cols, extra = 4 * cb - sfc;
  if (extra) {
    for (uint32_t i = tid; i < M * extra; i += nth) {
      const uint32_t r = i / extra;
      p.sf[sf_off32(r, sfc + (i - r * extra), cb)] = 0;
    }
  }
}

__device__ __forceinline__ EncConsts nv_consts(const AQParams& p, uint32_t gmax_bits) {
  const double top = (double)__uint_as_float(gmax_bits) * p.c64 / 6.0;  // absmax.max() / FP4_MAX
  return nv_consts_st(p, top > 0.0 ? __double2float_rn(top / 448.0) : 1.0f);   // f32(top / E4M3 max)
}

// Single-pass constants: MXFP4 (tensor scale f32(4/3) or 1.0, quantizers.py:203-207) or NVFP4
// with a caller-given global scale (read after pdl_wait: a predecessor may produce it).
template <int FMT>
__device__ __forceinline__ EncConsts single_pass_consts(const AQParams& p) {
  if constexpr (FMT == MRFP4_FMT_NVFP4) {
    return nv_consts_st(p, *p.static_ts);
  } else {
    EncConsts k;
    k.st32 = p.mx_ts;
    return k;
  }
}

// Rotate (already done by the caller) -> scales -> codes -> stores of one lane segment.
template <int FMT, typename W>
__device__ __forceinline__ void encode_seg(const AQParams& p, const W& c, const u64 (&P)[kPairs],
                                           const EncConsts& k, uint32_t& bad) {
  if (!c.live(p)) return;                               // idle lane (after the shuffles)
  const bool full = c.full(p);                          // else a 16-element tail (K % 32 == 16)
  float a0, a1;
  half_amax(P, a0, a1);
  GroupScale s0, s1;
  uint32_t sfc;
  if constexpr (FMT == MRFP4_FMT_NVFP4) {
    s0 = nv_group_scale(a0, p, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
    s1 = nv_group_scale(a1, p, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
    if (__float_as_uint(a0) >= 0x7f800000u || (full && __float_as_uint(a1) >= 0x7f800000u))
      bad |= MRFP4_STATUS_NONFINITE;
    if (s0.code == 0 || (full && s1.code == 0)) bad |= MRFP4_STATUS_SCALE_UNDERFLOW;
    sfc = s0.code | (full ? s1.code << 8 : 0u);
  } else {
    const float a = max3n(a0, a1, 0.f);
    if (__float_as_uint(a) >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
    s0 = mx_group_scale(a, p);
    s1 = s0;
    sfc = s0.code;
  }
  uint32_t w[4];
  quantize_seg(P, s0, s1, k.st32, p, w);

  uint8_t* cdst = c.cdst(p);
  if (full) {
    if ((p.Ki & 31) == 0) {
      *reinterpret_cast<uint4*>(cdst) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      reinterpret_cast<uint2*>(cdst)[0] = make_uint2(w[0], w[1]);
      reinterpret_cast<uint2*>(cdst)[1] = make_uint2(w[2], w[3]);
    }
  } else {
    *reinterpret_cast<uint2*>(cdst) = make_uint2(w[0], w[1]);
  }
  if constexpr (FMT == MRFP4_FMT_MXFP4) {
    p.sf[sf_off32(c.row(), c.seg(), p.cb)] = (uint8_t)sfc;
  } else {
    // columns 2*seg, 2*seg+1 share a 16-bit word of the swizzled layout
    *reinterpret_cast<uint16_t*>(p.sf + sf_off32(c.row(), 2 * c.seg(), p.cb)) = (uint16_t)sfc;
  }
}

// Per-warp trace stamps (perf experiments), 8 words per warp:
// [start, end, items | smid << 32, NVFP4 phase-1 end, NVFP4 barrier release, -, -, -].
struct Trace {
  unsigned long long* t;
  __device__ __forceinline__ Trace(const AQParams& p, int warp, int lane)
      : t(p.trace && lane == 0 ? p.trace + ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 8 : nullptr) {
    if (t) t[0] = globaltimer();
  }
  __device__ __forceinline__ void mark(int i) {
    if (t) t[i] = globaltimer();
  }
  __device__ __forceinline__ void end(int n) {
    if (t) { t[1] = globaltimer(); t[2] = (unsigned long long)n | ((unsigned long long)smid() << 32); }
  }
};

// Single pass: MXFP4 (group-local scales), or NVFP4 with a caller-given global scale.
template <int IN, int FMT, int HK, typename W, int NW>
__global__ void __launch_bounds__(NW * 32, 768 / (NW * 32))
    k_act_quant_1p(const __grid_constant__ CUtensorMap tmx, AQParams p) {
  __shared__ uint32_t ctr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Trace tr(p, warp, lane);
  if (threadIdx.x == 0) ctr = 0u;
  Loader<IN, W> L;
  init_loader<NW>(L, warp, lane);
  __syncthreads();
  pdl_wait();
  // Trigger only after the wait: a dependent launched now can only find this grid's
  // predecessors complete, so its pre-wait loads (the GEMM's weight stream) never race a
  // kernel two steps back (e.g. K1 of the weight itself).
  pdl_trigger();
  const EncConsts k = single_pass_consts<FMT>(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.tensor_scale = k.st32;
  CtaRange r;
  r.init(p);
  Claims cl;
  cl.init(&ctr, r.cnt, lane);
  uint32_t bad = 0;
  const int n = run_pipeline<IN, W>(
      p, &tmx, L, [&] { const int c = cl.next(lane); return c < 0 ? -1 : r.c0 + c; }, nullptr,
      [&](const W& c, uint32_t sbase) {
        u64 P[kPairs];
        load_pairs<IN>(sbase, lane, P);
        if constexpr (HK > 0) fwht<HK>(P, lane, p.pm);
        encode_seg<FMT>(p, c, P, k, bad);
      });
  tr.end(n);
  if (bad) atomic_or_status(p.status, bad);
  zero_sf_padding(p);
}

// NVFP4: the whole-tensor scale (quantizers.py:198-200) must be known before any group is
// encoded.  One persistent launch (one CTA per SM, all co-resident by construction):
//   phase 1 streams X and reduces max |y| into gmax; grid barrier;
//   phase 2 first encodes the items still held in each warp's ring (the last kStages it
//   processed), then the CTA's other items, claimed in reverse order (most recently loaded,
//   so most likely still in L2, first).  A shared bitmap marks the ring-resident items.
// Workspace words: [0] gmax, [1] barrier count, [2] barrier generation, [3] exit count; the
// last CTA out re-zeroes [0], [3].
constexpr int kBitmapWords = 1024;  // ring-resident marks for up to 32768 items per CTA

template <int IN, int HK, typename W, int NW>
__global__ void __launch_bounds__(NW * 32, 768 / (NW * 32))
    k_act_quant_nv(const __grid_constant__ CUtensorMap tmx, AQParams p) {
  constexpr int kStages = InCfg<IN>::kStages;
  __shared__ uint32_t ctr[2];
  __shared__ int resident[NW][kMaxStages];
  __shared__ uint32_t marks[kBitmapWords];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* ws = p.gmax;
  volatile uint32_t* vgen = ws + 2;
  const uint32_t gen0 = *vgen;  // before arriving: the barrier releases when gen != gen0
  Trace tr(p, warp, lane);
  CtaRange r;
  r.init(p);
  // Re-encoding the ring-resident items first (no reload) measured faster or equal at every
  // shape (scripts/k1_ab.py MRFP4_K1_MARKS=0/1), most at decode sizes.
  const bool use_marks = r.cnt <= 32 * kBitmapWords && p.marks != 0;
  if (threadIdx.x < 2) ctr[threadIdx.x] = 0u;
  if (lane < kStages) resident[warp][lane] = -1;
  if (use_marks)
    for (int i = threadIdx.x; i < (r.cnt + 31) / 32; i += NW * 32) marks[i] = 0u;
  Loader<IN, W> L;
  init_loader<NW>(L, warp, lane);
  __syncthreads();
  pdl_wait();

  // ---- phase 1: max |y| over the tensor
  float m = 0.f;
  {
    Claims cl;
    cl.init(&ctr[0], r.cnt, lane);
    run_pipeline<IN, W>(
        p, &tmx, L, [&] { const int c = cl.next(lane); return c < 0 ? -1 : r.c0 + c; }, resident[warp],
        [&](const W& c, uint32_t sbase) {
          u64 P[kPairs];
          load_pairs<IN>(sbase, lane, P);
          if constexpr (HK > 0) fwht<HK>(P, lane, p.pm);
          float a, b;
          half_amax(P, a, b);   // GenWalk: padding rows / columns were zero-filled
          if (c.live(p)) m = max3n(a, b, m);
        });
  }
  __syncwarp();
  tr.mark(3);
  if (use_marks && lane < kStages) {
    const int it = resident[warp][lane];
    if (it >= 0) atomicOr(&marks[(it - r.c0) >> 5], 1u << ((it - r.c0) & 31));
  }
  uint32_t mb = __float_as_uint(m);
  mb = mb > 0x7f800000u ? 0x7fc00000u : mb;  // canonical NaN
  mb = __reduce_max_sync(0xffffffffu, mb);
  __shared__ uint32_t smax[NW];
  __shared__ EncConsts sk;
  if (lane == 0) smax[warp] = mb;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t x = 0;
    for (int i = 0; i < NW; ++i) x = max(x, smax[i]);
    if (x) atomicMax(ws, x);
    if (x >= 0x7f800000u) atomic_or_status(p.status, MRFP4_STATUS_NONFINITE);
    // ---- grid barrier without full fences: the arrival is an acq_rel RMW (releases this
    // CTA's max, acquires every earlier arrival's); the last arriver re-arms the count and
    // bumps the generation with a release; the others acquire the generation.
    uint32_t arrived;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(ws + 1) : "memory");
    if (arrived == gridDim.x - 1) {
      ws[1] = 0u;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ws + 2) : "memory");
    } else {
      uint32_t g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(ws + 2) : "memory");
      } while (g == gen0);
    }
    uint32_t gm;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gm) : "l"(ws) : "memory");
    sk = nv_consts(p, gm);  // fp64 divides: once per CTA, not per warp
  }
  __syncthreads();
  tr.mark(4);
  pdl_trigger();  // only after the barrier: every CTA of this grid is resident by now
  const EncConsts k = sk;
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.tensor_scale = k.st32;

  // ---- phase 2: encode
  uint32_t bad = 0;
  auto encode = [&](const W& c, uint32_t sbase) {
    u64 P[kPairs];
    load_pairs<IN>(sbase, lane, P);
    if constexpr (HK > 0) fwht<HK>(P, lane, p.pm);
    encode_seg<MRFP4_FMT_NVFP4>(p, c, P, k, bad);
  };
  if (use_marks) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      const int it = resident[warp][s];
      if (it >= 0) {
        W c;
        c.at(p, it, lane);
        encode(c, L.slot(s));
      }
    }
  }
  Claims cl;
  cl.init(&ctr[1], r.cnt, lane);
  const int n = run_pipeline<IN, W>(
      p, &tmx, L,
      [&] {
        while (true) {
          const int c = cl.next(lane);
          if (c < 0) return -1;
          const int off = r.cnt - 1 - c;
          if (!use_marks || !((marks[off >> 5] >> (off & 31)) & 1u)) return r.c0 + off;
        }
      },
      nullptr, encode);
  tr.end(n);
  if (bad) atomic_or_status(p.status, bad);
  zero_sf_padding(p);
  // Last CTA out re-arms gmax for the next call (every CTA read it before the barrier released).
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ws + 3, 1u) == gridDim.x - 1) {
      ws[0] = 0u;
      ws[3] = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// K1m: the rotation on the tensor cores (bf16 / f16 input, contiguous rows, K % 32 == 0,
// K >= 1024, k in {16, 32, 64, 128}).
//
// Per warp sub-item: 32 consecutive 32-element segments (2 KB of bf16) of the flattened X,
// one 32 x 32 tile.  Y = X_tile . H32' by 16 mma.sync.m16n8k16 (fp32 accumulate; +-1
// operands, so the products are exact and each output is the fp32 sum the butterfly would
// produce -- scripts/hmma_probe.cu: no less exact than the FWHT), where H32' is H32 (or
// diag(H16, H16)) with its columns permuted so that lane (g, t) = (lane / 4, lane % 4)
// receives output elements 8t .. 8t+7 of segments 8j + g, j = 0..3 ("slot" j): 4 f32 pairs
// per slot, i.e. one 32-bit word of codes.  k = 64 / 128 add the H2 / H4 factor across
// segments (8j + g) ^ 1 / ^ 2, i.e. lanes xor 4 / 8.
// The group absmax is a reduce-scatter over the lanes sharing a group (MXFP4: the quad,
// lane t ends with segment 8t + g; NVFP4: the lane pair, each lane with two groups), so
// every scale code is computed once; the element multipliers go back by shuffles.
// Replaces ~80 FADD2/FFMA2 + 32 unpack instructions per lane segment with 16 HMMA per
// warp tile (0.5 HMMA/clk/SM measured, ~3 us of tensor time at c1).
// ---------------------------------------------------------------------------
template <int IN>
__device__ __forceinline__ void hmma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (IN == MRFP4_DT_BF16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t saddr, uint32_t (&a)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"(saddr));
}

__device__ __forceinline__ float maxn(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// B fragments of the permuted Hadamard (constant per lane): b[(kt * 4 + nt) * 2 + r] holds
// rows k = 16 kt + 2t + 8r, k + 1 of column n = g of n-tile nt, which is output element
// e = 8 (g >> 1) + 2 nt + (g & 1).  Entry (-1)^popc(k & e) (k = 16: (-1)^popc(k & e & 15) on
// the two diagonal 16 x 16 blocks, zero off them).
template <int IN, int HK>
__device__ __forceinline__ void hadamard_frags(int lane, uint32_t (&b)[16]) {
  const int g = lane >> 2, t = lane & 3;
  const uint32_t one = IN == MRFP4_DT_BF16 ? 0x3F80u : 0x3C00u;
  const uint32_t neg = 0x8000u;
#pragma unroll
  for (int kt = 0; kt < 2; ++kt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k0 = 16 * kt + 2 * t + 8 * r;
        const int e = 8 * (g >> 1) + 2 * nt + (g & 1);
        uint32_t v = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = k0 + h;
          const bool live = HK != 16 || (k >> 4) == (e >> 4);
          const uint32_t x = live ? (one | ((__popc(k & e & (HK == 16 ? 15 : 31)) & 1) ? neg : 0u)) : 0u;
          v |= x << (16 * h);
        }
        b[(kt * 4 + nt) * 2 + r] = v;
      }
}

// ldmatrix addresses (bytes from the tile base) of lane's rows for (mt, kt) = (i / 2, i % 2):
// matrix q = lane / 8 -> rows 16 mt + 8 (q & 1) + lane % 8, 16-B chunk 2 kt + (q >> 1), under
// the TMA 64-B swizzle (chunk ^= (row >> 1) & 3).  The 8 rows of a matrix are consecutive
// segments: conflict-free.
__device__ __forceinline__ void ldsm_offsets(int lane, uint32_t (&off)[4]) {
  const int q = lane >> 3, r8 = lane & 7;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int mt = i >> 1, kt = i & 1;
    const int seg = 16 * mt + 8 * (q & 1) + r8;
    const int chunk = 2 * kt + (q >> 1);
    off[i] = (uint32_t)(seg * 64 + ((chunk ^ ((seg >> 1) & 3)) * 16));
  }
}

// 32 x 32 tile at `sbase` -> P[j][nt] = output elements (8t + 2nt, 8t + 2nt + 1) of segment 8j + g.
// The B fragments live in shared memory (HB_SMEM: [8 (kt, nt)][32 lanes] x 8 B, conflict-free
// LDS.64), not in 16 registers per lane: registers bound the kernel's occupancy.
__device__ __forceinline__ void lds64(uint32_t saddr, uint32_t& a, uint32_t& b) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(saddr));
}

template <int IN, int HK>
__device__ __forceinline__ void rotate_tile(uint32_t sbase, const uint32_t (&off)[4], uint32_t hb_smem,
                                            int lane, u64 (&P)[4][4]) {
  float c[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int z = 0; z < 4; ++z) c[mt][nt][z] = 0.f;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kt = 0; kt < 2; ++kt) {
      uint32_t a[4];
      ldsm_x4(sbase + off[2 * mt + kt], a);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t b0, b1;
        lds64(hb_smem + (uint32_t)(((kt * 4 + nt) * 32 + lane) * 8), b0, b1);
        hmma16816<IN>(c[mt][nt], a, b0, b1);
      }
    }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      P[2 * mt][nt] = pk(c[mt][nt][0], c[mt][nt][1]);
      P[2 * mt + 1][nt] = pk(c[mt][nt][2], c[mt][nt][3]);
    }
  // Segment-index bits 0 / 1 (k = 64 / 128) live in lane bits 2 / 3.
  if constexpr (HK >= 64) {
    const float s = (lane & 4) ? -1.f : 1.f;
    const u64 sg = pk(s, s);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) P[j][nt] = fma2(sg, P[j][nt], __shfl_xor_sync(0xffffffffu, P[j][nt], 4));
  }
  if constexpr (HK >= 128) {
    const float s = (lane & 8) ? -1.f : 1.f;
    const u64 sg = pk(s, s);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) P[j][nt] = fma2(sg, P[j][nt], __shfl_xor_sync(0xffffffffu, P[j][nt], 8));
  }
}

__device__ __forceinline__ float slot_amax(const u64 (&Pj)[4]) {
  const float a = amax3(lo_of(Pj[0]), hi_of(Pj[0]), lo_of(Pj[1]));
  const float b = amax3(hi_of(Pj[1]), lo_of(Pj[2]), hi_of(Pj[2]));
  const float c = amax3(lo_of(Pj[3]), hi_of(Pj[3]), 0.f);
  return max3n(a, b, c);
}

// 8 elements -> one word of E2M1 codes, rounded twice (u * (1 +- 2^-18)); nibbles that
// disagree are re-decided exactly by the caller.
__device__ __forceinline__ uint32_t quant_slot(const u64 (&Pj)[4], float f, uint32_t& diff) {
  constexpr float kEps = 3.814697265625e-06f;  // 2^-18
  const float fh = f * (1.f + kEps), fl = f * (1.f - kEps);
  float uh[8], ul[8];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const u64 a = mul2(Pj[t], pk(fh, fh)), b = mul2(Pj[t], pk(fl, fl));
    uh[2 * t] = lo_of(a); uh[2 * t + 1] = hi_of(a);
    ul[2 * t] = lo_of(b); ul[2 * t + 1] = hi_of(b);
  }
  const uint32_t w = cvt_e2m1x8(uh);
  diff = w ^ cvt_e2m1x8(ul);
  return w;
}

// Decoded group scale from its code (exact in fp32), as mx_group_scale / nv_group_scale.
template <int FMT>
__device__ __forceinline__ float dec_of(uint32_t code) {
  if constexpr (FMT == MRFP4_FMT_MXFP4) {
    const int e = (int)code - 127;
    return __uint_as_float(e >= -126 ? (uint32_t)(e + 127) << 23 : 0x00400000u);
  } else {
    return e4m3_value(code);
  }
}

// Rare: re-decide the nibbles of `w` flagged in `redo` (all when slow) exactly (quantizers.py:213).
template <int FMT>
__device__ __noinline__ uint32_t redo_slot(uint32_t w, uint32_t redo, bool slow, const float (&v)[8], double c64,
                                           float ts, uint32_t code) {
  const float dec = dec_of<FMT>(code);
  for (int e = 0; e < 8; ++e) {
    if (slow || ((redo >> (4 * e)) & 0xFu)) {
      const uint32_t c = fp4_code_exact(v[e], c64, ts, dec);
      w = (w & ~(0xFu << (4 * e))) | (c << (4 * e));
    }
  }
  return w;
}

// Row / column of global segment s (flat walk).
__device__ __forceinline__ void seg_rc(const AQParams& p, uint32_t s, uint32_t& row, uint32_t& col) {
  row = fast_div(s, (uint32_t)p.nseg, p.div_m);
  col = s - row * (uint32_t)p.nseg;
}

// Encode one 32-segment tile whose first global segment is s0.  Returns nothing; ORs status bits.
template <int FMT>
__device__ __forceinline__ void encode_tile(const AQParams& p, const EncConsts& k, const u64 (&P)[4][4], uint32_t s0,
                                            int lane, uint32_t& bad) {
  const int g = lane >> 2, t = lane & 3;
  float m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) m[j] = slot_amax(P[j]);
  float f[4];
  uint32_t codes_own, codes_oth;  // FMT-specific packing of the 4 slots' codes (slow path)
  bool slow;
  if constexpr (FMT == MRFP4_FMT_MXFP4) {
    // reduce-scatter over the quad: lane t ends with the max of slot t (segment 8t + g)
    const bool hi2 = t & 2, hi1 = t & 1;
    float k0 = hi2 ? m[2] : m[0], k1 = hi2 ? m[3] : m[1];
    const float s0v = hi2 ? m[0] : m[2], s1v = hi2 ? m[1] : m[3];
    k0 = maxn(k0, __shfl_xor_sync(0xffffffffu, s0v, 2));
    k1 = maxn(k1, __shfl_xor_sync(0xffffffffu, s1v, 2));
    const float a = maxn(hi1 ? k1 : k0, __shfl_xor_sync(0xffffffffu, hi1 ? k0 : k1, 1));
    if (__float_as_uint(a) >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
    const GroupScale gs = mx_group_scale(a, p);
    const int qb = lane & ~3;
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = __shfl_sync(0xffffffffu, gs.f, qb | j);
    uint32_t cw = gs.code << (8 * t);
    cw |= __shfl_xor_sync(0xffffffffu, cw, 1);
    cw |= __shfl_xor_sync(0xffffffffu, cw, 2);
    codes_own = cw;
    codes_oth = 0;
    slow = __any_sync(0xffffffffu, gs.slow_all);
    const uint32_t s = s0 + 8u * (uint32_t)t + (uint32_t)g;
    if (s < p.total_segs) {
      uint32_t row, col;
      seg_rc(p, s, row, col);
      p.sf[sf_off32(row, col, p.cb)] = (uint8_t)gs.code;
    }
  } else {
    // reduce-scatter over the lane pair: even lanes keep slots 0, 1, odd lanes slots 2, 3
    const bool odd = t & 1;
    float k0 = odd ? m[2] : m[0], k1 = odd ? m[3] : m[1];
    const float s0v = odd ? m[0] : m[2], s1v = odd ? m[1] : m[3];
    k0 = maxn(k0, __shfl_xor_sync(0xffffffffu, s0v, 1));
    k1 = maxn(k1, __shfl_xor_sync(0xffffffffu, s1v, 1));
    const GroupScale g0 = nv_group_scale(k0, p, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
    const GroupScale g1 = nv_group_scale(k1, p, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
    if (__float_as_uint(k0) >= 0x7f800000u || __float_as_uint(k1) >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
    const float o0 = __shfl_xor_sync(0xffffffffu, g0.f, 1), o1 = __shfl_xor_sync(0xffffffffu, g1.f, 1);
    f[0] = odd ? o0 : g0.f; f[1] = odd ? o1 : g1.f;
    f[2] = odd ? g0.f : o0; f[3] = odd ? g1.f : o1;
    const uint32_t cw = g0.code | (g1.code << 8);
    codes_own = cw;
    codes_oth = __shfl_xor_sync(0xffffffffu, cw, 1);
    slow = __any_sync(0xffffffffu, g0.slow_all | g1.slow_all);
    const uint32_t gi = (uint32_t)(t >> 1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t code = h ? g1.code : g0.code;
      const uint32_t s = s0 + 8u * (uint32_t)(2 * (t & 1) + h) + (uint32_t)g;
      if (s < p.total_segs) {
        if (code == 0) bad |= MRFP4_STATUS_SCALE_UNDERFLOW;
        uint32_t row, col;
        seg_rc(p, s, row, col);
        p.sf[sf_off32(row, 2 * col + gi, p.cb)] = (uint8_t)code;
      }
    }
  }
  uint32_t w[4], dif[4], any = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    w[j] = quant_slot(P[j], f[j], dif[j]);
    any |= dif[j];
  }
  if (any | (uint32_t)slow) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (dif[j] | (uint32_t)slow) {
        float v[8];
#pragma unroll
        for (int z = 0; z < 4; ++z) { v[2 * z] = lo_of(P[j][z]); v[2 * z + 1] = hi_of(P[j][z]); }
        uint32_t code;
        if constexpr (FMT == MRFP4_FMT_MXFP4) {
          code = (codes_own >> (8 * j)) & 0xFFu;
        } else {
          const bool mine = (j >> 1) == (t & 1);
          code = ((mine ? codes_own : codes_oth) >> (8 * (j & 1))) & 0xFFu;
        }
        w[j] = redo_slot<FMT>(w[j], dif[j], slow, v, p.c64, k.st32, code);
      }
    }
  }
  uint32_t* cdst = reinterpret_cast<uint32_t*>(p.codes) + (uint64_t)s0 * 4u + (uint32_t)(4 * g + t);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (s0 + 8u * j + (uint32_t)g < p.total_segs) cdst[32 * j] = fix_neg_zero(w[j]);
}

// Per-warp TMA ring of kStages items of U tiles (U * 2 KB) for K1m.
template <int U, int S>
struct MRing {
  static constexpr uint32_t kItemBytes = 32u * U * 64u;
  uint32_t base, bars, ph;
  int lane;
  __device__ __forceinline__ void init(uint32_t ring, uint32_t bar_addr, int lane_) {
    lane = lane_;
    base = ring;
    bars = bar_addr;
    ph = 0;
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  __device__ __forceinline__ uint32_t slot(int s) const { return base + (uint32_t)s * kItemBytes; }
  __device__ __forceinline__ void issue(const CUtensorMap* tm, int item, int s) {
    if (lane == 0) {
      const uint32_t bar = bars + 8 * s;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kItemBytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(slot(s)),
          "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(0), "r"(item * 32 * U)
          : "memory");
    }
  }
  __device__ __forceinline__ void wait(int s) {
    const uint32_t par = (ph >> s) & 1u;
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(bars + 8 * s),
        "r"(par)
        : "memory");
    ph ^= 1u << s;
  }
  __device__ __forceinline__ void release() {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
};

// Issue item j + S - 1 while item j is processed; item j of the walk sits in slot j % S.
template <int U, int S, typename N, typename F>
__device__ __forceinline__ int run_ring(const CUtensorMap* tm, MRing<U, S>& R, N&& next, int* resident, int lane,
                                        F&& body) {
  int it[S];
  R.release();
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    it[s] = next();
    if (it[s] >= 0) R.issue(tm, it[s], s);
  }
  int rd = 0, wr = S - 1, n = 0;
  while (true) {
    it[S - 1] = next();
    if (it[S - 1] >= 0) {
      R.release();
      R.issue(tm, it[S - 1], wr);
    }
    if (it[0] < 0) break;
    R.wait(rd);
    body(it[0], R.slot(rd));
    if (resident && lane == 0) resident[rd] = it[0];
    ++n;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) it[s] = it[s + 1];
    rd = rd + 1 == S ? 0 : rd + 1;
    wr = wr + 1 == S ? 0 : wr + 1;
  }
  return n;
}

template <int U, int S, int NW>
__device__ __forceinline__ void init_mring(MRing<U, S>& R, int warp, int lane) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[NW * S];
  const uint32_t base = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  R.init(base + (uint32_t)warp * S * MRing<U, S>::kItemBytes, (uint32_t)__cvta_generic_to_shared(&bars[warp * S]),
         lane);
}

template <int U, int S, int NW>
constexpr int mring_smem() { return NW * S * (int)MRing<U, S>::kItemBytes + 1024; }

// Single pass (MXFP4, or NVFP4 with a given global scale).  MB: CTAs per SM the register
// allocation must allow.
template <int IN, int FMT, int HK, int U, int S, int NW, int MB>
__global__ void __launch_bounds__(NW * 32, MB)
    k_act_quant_1p_mma(const __grid_constant__ CUtensorMap tmx, AQParams p) {
  __shared__ uint32_t ctr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Trace tr(p, warp, lane);
  if (threadIdx.x == 0) ctr = 0u;
  MRing<U, S> R;
  init_mring<U, S, NW>(R, warp, lane);
  __shared__ __align__(16) uint32_t hb_tab[8 * 32 * 2];
  uint32_t off[4];
  if (warp == 0) {
    uint32_t hb[16];
    hadamard_frags<IN, HK>(lane, hb);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hb_tab[(i * 32 + lane) * 2] = hb[2 * i];
      hb_tab[(i * 32 + lane) * 2 + 1] = hb[2 * i + 1];
    }
  }
  const uint32_t hbs = (uint32_t)__cvta_generic_to_shared(hb_tab);
  ldsm_offsets(lane, off);
  __syncthreads();
  pdl_wait();
  // Trigger only after the wait: a dependent launched now can only find this grid's
  // predecessors complete, so its pre-wait loads (the GEMM's weight stream) never race a
  // kernel two steps back (e.g. K1 of the weight itself).
  pdl_trigger();
  const EncConsts k = single_pass_consts<FMT>(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.tensor_scale = k.st32;
  CtaRange r;
  r.init(p);
  Claims cl;
  cl.init(&ctr, r.cnt, lane);
  uint32_t bad = 0;
  const int n = run_ring(
      &tmx, R, [&] { const int c = cl.next(lane); return c < 0 ? -1 : r.c0 + c; }, nullptr, lane,
      [&](int item, uint32_t sbase) {
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
          u64 P[4][4];
          rotate_tile<IN, HK>(sbase + u * 2048u, off, hbs, lane, P);
          encode_tile<FMT>(p, k, P, (uint32_t)(item * U + u) * 32u, lane, bad);
        }
      });
  tr.end(n);
  if (bad) atomic_or_status(p.status, bad);
  zero_sf_padding(p);
}

// NVFP4: phase 1 (tensor max) -> grid barrier -> phase 2 (encode), as k_act_quant_nv.
template <int IN, int HK, int U, int S, int NW, int MB>
__global__ void __launch_bounds__(NW * 32, MB)
    k_act_quant_nv_mma(const __grid_constant__ CUtensorMap tmx, AQParams p) {
  __shared__ uint32_t ctr[2];
  __shared__ int resident[NW][S];
  __shared__ uint32_t marks[kBitmapWords];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* ws = p.gmax;
  volatile uint32_t* vgen = ws + 2;
  const uint32_t gen0 = *vgen;
  Trace tr(p, warp, lane);
  CtaRange r;
  r.init(p);
  const bool use_marks = r.cnt <= 32 * kBitmapWords && p.marks != 0;
  if (threadIdx.x < 2) ctr[threadIdx.x] = 0u;
  if (lane < S) resident[warp][lane] = -1;
  if (use_marks)
    for (int i = threadIdx.x; i < (r.cnt + 31) / 32; i += NW * 32) marks[i] = 0u;
  MRing<U, S> R;
  init_mring<U, S, NW>(R, warp, lane);
  __shared__ __align__(16) uint32_t hb_tab[8 * 32 * 2];
  uint32_t off[4];
  if (warp == 0) {
    uint32_t hb[16];
    hadamard_frags<IN, HK>(lane, hb);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hb_tab[(i * 32 + lane) * 2] = hb[2 * i];
      hb_tab[(i * 32 + lane) * 2 + 1] = hb[2 * i + 1];
    }
  }
  const uint32_t hbs = (uint32_t)__cvta_generic_to_shared(hb_tab);
  ldsm_offsets(lane, off);
  __syncthreads();
  pdl_wait();

  float m = 0.f;
  {
    Claims cl;
    cl.init(&ctr[0], r.cnt, lane);
    run_ring(
        &tmx, R, [&] { const int c = cl.next(lane); return c < 0 ? -1 : r.c0 + c; }, resident[warp], lane,
        [&](int item, uint32_t sbase) {
#pragma unroll 1
          for (int u = 0; u < U; ++u) {
            u64 P[4][4];
            rotate_tile<IN, HK>(sbase + u * 2048u, off, hbs, lane, P);
            m = max3n(max3n(slot_amax(P[0]), slot_amax(P[1]), slot_amax(P[2])), slot_amax(P[3]), m);
          }
        });
  }
  __syncwarp();
  tr.mark(3);
  if (use_marks && lane < S) {
    const int it = resident[warp][lane];
    if (it >= 0) atomicOr(&marks[(it - r.c0) >> 5], 1u << ((it - r.c0) & 31));
  }
  uint32_t mb = __float_as_uint(m);
  mb = mb > 0x7f800000u ? 0x7fc00000u : mb;
  mb = __reduce_max_sync(0xffffffffu, mb);
  __shared__ uint32_t smax[NW];
  __shared__ EncConsts sk;
  if (lane == 0) smax[warp] = mb;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t x = 0;
    for (int i = 0; i < NW; ++i) x = max(x, smax[i]);
    if (x) atomicMax(ws, x);
    if (x >= 0x7f800000u) atomic_or_status(p.status, MRFP4_STATUS_NONFINITE);
    // ---- grid barrier without full fences: the arrival is an acq_rel RMW (releases this
    // CTA's max, acquires every earlier arrival's); the last arriver re-arms the count and
    // bumps the generation with a release; the others acquire the generation.
    uint32_t arrived;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(ws + 1) : "memory");
    if (arrived == gridDim.x - 1) {
      ws[1] = 0u;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ws + 2) : "memory");
    } else {
      uint32_t g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(ws + 2) : "memory");
      } while (g == gen0);
    }
    uint32_t gm;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gm) : "l"(ws) : "memory");
    sk = nv_consts(p, gm);
  }
  __syncthreads();
  tr.mark(4);
  pdl_trigger();
  const EncConsts k = sk;
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.tensor_scale = k.st32;

  uint32_t bad = 0;
  auto encode = [&](int item, uint32_t sbase) {
#pragma unroll 1
    for (int u = 0; u < U; ++u) {
      u64 P[4][4];
      rotate_tile<IN, HK>(sbase + u * 2048u, off, hbs, lane, P);
      encode_tile<MRFP4_FMT_NVFP4>(p, k, P, (uint32_t)(item * U + u) * 32u, lane, bad);
    }
  };
  if (use_marks) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int it = resident[warp][s];
      if (it >= 0) encode(it, R.slot(s));
    }
  }
  Claims cl;
  cl.init(&ctr[1], r.cnt, lane);
  const int n = run_ring(
      &tmx, R,
      [&] {
        while (true) {
          const int c = cl.next(lane);
          if (c < 0) return -1;
          const int o = r.cnt - 1 - c;
          if (!use_marks || !((marks[o >> 5] >> (o & 31)) & 1u)) return r.c0 + o;
        }
      },
      nullptr, lane, encode);
  tr.end(n);
  if (bad) atomic_or_status(p.status, bad);
  zero_sf_padding(p);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ws + 3, 1u) == gridDim.x - 1) {
      ws[0] = 0u;
      ws[3] = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// QuantResult metrics (quantizers.py:218-231): mse_rel = sum (y - q)^2 / sum y^2 and
// mse_top_rel = mean over groups of ((y_top - q_top) / y_top)^2 at each group's argmax |y|
// (first index on ties, like np.argmax), all in the rotated domain.  Sums in fp64 with
// the rotated values y = RN64(S * c); accumulated per warp, then fp64 atomics into
// acc[0..2] = {sum err^2, sum y^2, sum top ratio} (zeroed by the caller).
// Off the hot path (quantized_linear never asks for it).
// ---------------------------------------------------------------------------
template <int IN, int FMT, int HK>
__global__ void __launch_bounds__(kMetricWarps * 32) k_quant_metrics(AQParams p, double* acc) {
  using C = InCfg<IN>;
  constexpr int G = FMT == MRFP4_FMT_MXFP4 ? 32 : 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float ts = *p.tensor_scale;
  double e2 = 0.0, x2 = 0.0, top = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * kMetricWarps + warp, tw = (int64_t)gridDim.x * kMetricWarps;
  for (int64_t item = gw; item < p.items; item += tw) {
    GenWalk c;
    c.at(p, item, lane);
    const int col0 = c.seg() * kSeg;
    const bool live = c.live(p);
    const int nvalid = live ? min(kSeg, p.Ki - col0) : 0;
    uint32_t w[kSeg * C::kEs / 4];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(static_cast<const char*>(p.x) +
                                                            ((uint64_t)c.row() * p.ldx + (uint32_t)col0) * C::kEs);
#pragma unroll
    for (int j = 0; j < kSeg * C::kEs / 4; ++j) w[j] = (j * 4 < nvalid * C::kEs) ? src[j] : 0u;
    u64 P[kPairs];
#pragma unroll
    for (int j = 0; j < kPairs; ++j) {
      if constexpr (IN == MRFP4_DT_F32) {
        P[j] = pk(__uint_as_float(w[2 * j]), __uint_as_float(w[2 * j + 1]));
      } else if constexpr (IN == MRFP4_DT_BF16) {
        P[j] = pk(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xFFFF0000u));
      } else {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
        P[j] = pk(f.x, f.y);
      }
    }
    if constexpr (HK > 0) fwht<HK>(P, lane, p.pm);
    if (!live) continue;
    const uint8_t* cb = p.codes + (uint64_t)c.row() * p.half_k + (uint32_t)(col0 >> 1);
    for (int g0 = 0; g0 < nvalid; g0 += G) {
      const int gcol = (col0 + g0) / G;
      const uint32_t scode = p.sf[sf_off32(c.row(), gcol, p.cb)];
      const double dec = FMT == MRFP4_FMT_MXFP4 ? ldexp(1.0, (int)scode - 127) : (double)e4m3_value(scode);
      const double eff = (double)ts * dec;
      double best = -1.0, yt = 0.0, qt = 0.0;
      for (int t = 0; t < G; ++t) {
        const int e = g0 + t;
        const float sv = (e & 1) ? hi_of(P[e >> 1]) : lo_of(P[e >> 1]);
        const double y = (double)sv * p.c64;
        const uint32_t code = (cb[e >> 1] >> (4 * (e & 1))) & 0xFu;
        const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
        const double q = eff * (double)((code & 8u) ? -mag[code & 7u] : mag[code & 7u]);
        e2 += (y - q) * (y - q);
        x2 += y * y;
        if (fabs(y) > best) { best = fabs(y); yt = y; qt = q; }
      }
      if (yt != 0.0) top += (yt - qt) * (yt - qt) / (yt * yt);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
    top += __shfl_xor_sync(0xffffffffu, top, o);
  }
  if (lane == 0) {
    atomicAdd(acc, e2);
    atomicAdd(acc + 1, x2);
    atomicAdd(acc + 2, top);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Perf-experiment knobs (environment, read once per process; unset in production).
int knob(const char* name, int dflt) {
  static std::mutex mu;
  static std::unordered_map<std::string, std::pair<bool, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(name);
  if (it == cache.end()) {
    const char* v = std::getenv(name);
    it = cache.emplace(name, std::make_pair(v != nullptr, v ? std::atoi(v) : 0)).first;
  }
  return it->second.first ? it->second.second : dflt;
}

int num_sms() { return device_sms(); }

// One CTA set per SM that the occupancy calculator allows (cached per kernel and device).
template <auto Kern, int NW, bool kCoop = false>
int launch_persistent(int smem, const CUtensorMap& tm, const AQParams& p, cudaStream_t s) {
  static std::atomic<int> cache[kMaxDevices];
  const int per_sm = per_device_once(cache, [&] {
    int n = 0;
    // Max-shared carveout (the GEMM's too), so K1 -> K2 -> K1 never reconfigures L1/SMEM.
    cudaFuncSetAttribute(Kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, Kern, NW * 32, smem) == cudaSuccess)
      return std::max(n, 1);
    return -1;
  });
  if (per_sm < 0) return MRFP4_ECUDA;
  const int64_t need = ceil_div(p.items, NW);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)per_sm * num_sms()));
  return launch_pdl(Kern, dim3(grid), dim3(NW * 32), smem, s, kCoop, tm, p) == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

// FlatWalk's TMA view of X: [total_segs rows][one segment = kLaneBytes] bytes, box = one
// item (32 segments), swizzled like the cp.async ring (64 B rows: SWIZZLE_64B, 128 B: 128B).
template <int IN>
bool make_segment_map(CUtensorMap* tm, const AQParams& p, int box_segs = 32) {
  using C = InCfg<IN>;
  auto encode = tensor_map_encoder();
  if (!encode) return false;
  cuuint64_t dims[2] = {(cuuint64_t)C::kLaneBytes, (cuuint64_t)p.total_segs};
  cuuint64_t strides[1] = {(cuuint64_t)C::kLaneBytes};
  cuuint32_t box[2] = {(cuuint32_t)C::kLaneBytes, (cuuint32_t)box_segs};
  cuuint32_t estr[2] = {1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(p.x), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                C::kLaneBytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int IN, int FMT, int HK, int NW>
int launch_nw(const AQParams& p, const CUtensorMap& tm, cudaStream_t s) {
  constexpr int smem = InCfg<IN>::smem(NW);
  if constexpr (FMT == MRFP4_FMT_NVFP4) {
    if (!p.static_ts) {
      if (p.nseg) return launch_persistent<k_act_quant_nv<IN, HK, FlatWalk, NW>, NW, true>(smem, tm, p, s);
      return launch_persistent<k_act_quant_nv<IN, HK, GenWalk, NW>, NW, true>(smem, tm, p, s);
    }
  }
  if (p.nseg) return launch_persistent<k_act_quant_1p<IN, FMT, HK, FlatWalk, NW>, NW>(smem, tm, p, s);
  return launch_persistent<k_act_quant_1p<IN, FMT, HK, GenWalk, NW>, NW>(smem, tm, p, s);
}

// K1m launch: U tiles per item, S ring stages, NW warps per CTA.
template <int IN, int FMT, int HK, int U, int S, int NW, int MB>
int launch_mma_cfg(AQParams p, cudaStream_t s) {
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (!make_segment_map<IN>(&tm, p, 32 * U)) return MRFP4_ECUDA;
  p.items = ceil_div((int64_t)p.total_segs, 32 * U);
  constexpr int smem = mring_smem<U, S, NW>();
  if constexpr (FMT == MRFP4_FMT_NVFP4) {
    if (!p.static_ts) return launch_persistent<k_act_quant_nv_mma<IN, HK, U, S, NW, MB>, NW, true>(smem, tm, p, s);
  }
  return launch_persistent<k_act_quant_1p_mma<IN, FMT, HK, U, S, NW, MB>, NW>(smem, tm, p, s);
}

// Two tiles per item (fewer claims / TMA issues per tile) once every warp gets >= 8 tiles;
// one tile per item below that (more items to balance over the SM's warps).  Capping the
// registers for a third 8-warp CTA per SM spills and measured 1.4-1.6x slower.
template <int IN, int FMT, int HK>
int launch_mma(const AQParams& p, cudaStream_t s) {
  const int64_t tiles = ceil_div((int64_t)p.total_segs, 32);
  int cfg = knob("MRFP4_K1M_CFG", -1);
  if (cfg < 0) cfg = tiles >= 8 * 16 * (int64_t)num_sms() ? 1 : 0;
  // (18 / 20 warps per SM -- 2 x 9 or 2 x 10 -- measured no faster: the stalls are
  // fixed-latency dependency waits inside a warp's tile, not a lack of warps.)
  return cfg == 0 ? launch_mma_cfg<IN, FMT, HK, 1, 3, 8, 1>(p, s) : launch_mma_cfg<IN, FMT, HK, 2, 3, 8, 1>(p, s);
}

template <int IN, int FMT, int HK>
int launch_hk(const AQParams& p, cudaStream_t s) {
  if constexpr (IN != MRFP4_DT_F32 && HK >= 16) {
    // Tensor-core rotation: contiguous bf16 / f16 rows with K % 32 == 0, K >= 1024.  MXFP4 with
    // >= 2^24 elements takes the butterfly kernel instead: its single 24-warp CTA per SM hands
    // the SMs to the following GEMM sooner, and at these sizes it is as fast alone (c1 step
    // 67.0 -> 65.5 us; 70B down M=8192: K1 153 -> 112 us) -- profiles/r02_k1_notes.md.
    const bool mma_default = FMT == MRFP4_FMT_NVFP4 || (int64_t)p.Mi * p.Ki < (int64_t(1) << 24);
    if (p.nseg && knob("MRFP4_K1_MMA", mma_default ? 1 : 0)) return launch_mma<IN, FMT, HK>(p, s);
  }
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (p.nseg && !make_segment_map<IN>(&tm, p)) return MRFP4_ECUDA;
  // MXFP4: one 24-warp CTA per SM (the SM's warps share one work queue; best at large M).
  // NVFP4: three 8-warp CTAs per SM (its two phases and grid barrier run better in smaller
  // CTAs -- scripts/k1_warps.sh).
  const int nw = knob(FMT == MRFP4_FMT_NVFP4 ? "MRFP4_K1_NVWARPS" : "MRFP4_K1_MXWARPS",
                      FMT == MRFP4_FMT_NVFP4 ? 8 : 24);
  return nw == 8 ? launch_nw<IN, FMT, HK, 8>(p, tm, s) : launch_nw<IN, FMT, HK, 24>(p, tm, s);
}

template <int IN, int FMT>
int dispatch_hk(const AQParams& p, int hk, cudaStream_t s) {
  switch (hk) {
    case 0: return launch_hk<IN, FMT, 0>(p, s);
    case 16: return launch_hk<IN, FMT, 16>(p, s);
    case 32: return launch_hk<IN, FMT, 32>(p, s);
    case 64: return launch_hk<IN, FMT, 64>(p, s);
    case 128: return launch_hk<IN, FMT, 128>(p, s);
    default: return MRFP4_EUNSUPPORTED;
  }
}

template <int IN>
int dispatch_fmt(const AQParams& p, int fmt, int hk, cudaStream_t s) {
  return fmt == MRFP4_FMT_MXFP4 ? dispatch_hk<IN, MRFP4_FMT_MXFP4>(p, hk, s)
                                : dispatch_hk<IN, MRFP4_FMT_NVFP4>(p, hk, s);
}

}  // namespace

// Host launcher; arguments validated by the C-ABI layer (capi.cu).
namespace {

unsigned long long* g_k1_trace = nullptr;
// flat_ok: the caller's kernel supports FlatWalk (chosen when rows are contiguous, K % 32 == 0,
// K >= 1024 and the segment count fits 32 bits); p.nseg != 0 marks the flat walk.
AQParams make_params(const void* x, int64_t M, int64_t K, int64_t ldx, int fmt, int hk, uint8_t* codes, uint8_t* sf,
                     float* tensor_scale, uint32_t* status, void* workspace, bool flat_ok) {
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
  const int64_t nseg = ceil_div(K, kSeg);
  int lb = 0;
  while ((1 << lb) < nseg && lb < 5) ++lb;
  if (hk >= 128) lb = std::max(lb, 2);  // a 128-element block spans 4 lanes
  else if (hk >= 64) lb = std::max(lb, 1);
  p.lane_bits = lb;
  p.nchunk = (int)ceil_div(nseg, 1 << lb);
  p.seg_span = p.nchunk << lb;
  p.items = ceil_div(M, 32 >> lb) * p.nchunk;
  p.nseg = 0;
  p.total_segs = 0;
  p.trace = g_k1_trace;
  p.x_bytes = 0;
  p.marks = -1;
  if (flat_ok && ldx == K && K % kSeg == 0 && K >= 32 * kSeg && M * (K / kSeg) < (int64_t(1) << 31) &&
      !knob("MRFP4_K1_GENWALK", 0)) {
    p.nseg = (int)(K / kSeg);
    p.total_segs = (uint32_t)(M * (K / kSeg));
    p.items = ceil_div((int64_t)p.total_segs, 32);
  }
  const int64_t d = p.nseg ? p.nseg : p.nchunk;
  p.div_m = d > 1 ? (uint32_t)(((uint64_t(1) << 32) + (uint64_t)d - 1) / (uint64_t)d) : 0u;
  p.Mi = (int)M;
  p.Ki = (int)K;
  p.half_k = (uint32_t)(K / 2);
  p.cb = (uint32_t)p.sf_col_blocks;
  {
    const float pm[2] = {1.f, -1.f};
    memcpy(&p.pm, pm, sizeof(pm));
  }
  p.c64 = hk ? 1.0 / sqrt((double)hk) : 1.0;
  p.kraw = (float)(p.c64 / 6.0);
  p.mx_ts = 1.33333337306976318359375f;   // f32(4/3), quantizers.py:34, :191
  p.kmx = (float)(p.c64 / (double)p.mx_ts);
  p.static_ts = nullptr;
  return p;
}
}  // namespace

int launch_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int hk,
                     uint8_t* codes, uint8_t* sf, float* tensor_scale, uint32_t* status,
                     void* workspace, const mrfp4_act_quant_opts* opts, cudaStream_t s) {
  AQParams p = make_params(x, M, K, ldx, fmt, hk, codes, sf, tensor_scale, status, workspace, true);
  if (opts) {
    if (fmt == MRFP4_FMT_MXFP4 && !opts->mx_four_thirds) {
      p.mx_ts = 1.0f;   // ScalePolicy(e8m0_four_thirds=False): quantizers.py:206-207
      p.kmx = (float)p.c64;
    }
    if (fmt == MRFP4_FMT_NVFP4) p.static_ts = opts->nv_tensor_scale;
  }
  p.x_bytes = (uint64_t)M * (uint64_t)K * (x_dtype == MRFP4_DT_F32 ? 4u : 2u);
  p.marks = knob("MRFP4_K1_MARKS", -1);
  int rc;
  switch (x_dtype) {
    case MRFP4_DT_BF16: rc = dispatch_fmt<MRFP4_DT_BF16>(p, fmt, hk, s); break;
    case MRFP4_DT_F16: rc = dispatch_fmt<MRFP4_DT_F16>(p, fmt, hk, s); break;
    case MRFP4_DT_F32: rc = dispatch_fmt<MRFP4_DT_F32>(p, fmt, hk, s); break;
    default: return MRFP4_EUNSUPPORTED;
  }
  if (rc != MRFP4_OK) return rc;
  return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
}

int launch_quant_metrics(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int hk,
                         const uint8_t* codes, const uint8_t* sf, const float* tensor_scale, double* acc,
                         cudaStream_t s) {
  const AQParams p = make_params(x, M, K, ldx, fmt, hk, const_cast<uint8_t*>(codes), const_cast<uint8_t*>(sf),
                                 const_cast<float*>(tensor_scale), nullptr, nullptr, false);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.items, kMetricWarps), 4 * num_sms()));
  auto go = [&](auto kern) {
    kern<<<grid, kMetricWarps * 32, 0, s>>>(p, acc);
    return cudaPeekAtLastError() == cudaSuccess ? MRFP4_OK : MRFP4_ECUDA;
  };
#define MRFP4_MCASE(IN, FMT, HK) \
  if (x_dtype == IN && fmt == FMT && hk == HK) return go(k_quant_metrics<IN, FMT, HK>);
#define MRFP4_MFMT(IN, FMT) \
  MRFP4_MCASE(IN, FMT, 0) MRFP4_MCASE(IN, FMT, 16) MRFP4_MCASE(IN, FMT, 32) MRFP4_MCASE(IN, FMT, 64) \
  MRFP4_MCASE(IN, FMT, 128)
  MRFP4_MFMT(MRFP4_DT_BF16, MRFP4_FMT_MXFP4) MRFP4_MFMT(MRFP4_DT_BF16, MRFP4_FMT_NVFP4)
  MRFP4_MFMT(MRFP4_DT_F16, MRFP4_FMT_MXFP4) MRFP4_MFMT(MRFP4_DT_F16, MRFP4_FMT_NVFP4)
  MRFP4_MFMT(MRFP4_DT_F32, MRFP4_FMT_MXFP4) MRFP4_MFMT(MRFP4_DT_F32, MRFP4_FMT_NVFP4)
#undef MRFP4_MFMT
#undef MRFP4_MCASE
  return MRFP4_EUNSUPPORTED;
}

}  // namespace mrfp4

// Perf experiments only: per-warp timeline stamps (see Trace).
extern "C" void mrfp4_debug_k1_trace(unsigned long long* buf) { mrfp4::g_k1_trace = buf; }
