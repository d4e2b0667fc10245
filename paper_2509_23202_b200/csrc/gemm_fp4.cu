// K2: block-scaled FP4 x FP4 GEMM on the 5th-gen tensor cores (sm_100a).
//
// Computes the quantized linear Q(X H) Q(W H)^T of PAPER.md:337 -- in the
// reference only defined by composition, dequantize(Aq) @ dequantize(Wq).T
// (/root/reference/pkg/src/microfp/formats.py:424-442):
//     D[m, n] = ts_A * ts_W * sum_k (sfA[m, k/G] * a[m, k]) * (sfB[n, k/G] * w[n, k])
//
// Structure (one CTA per SM, persistent over 128 x BN output tiles):
//   warp 0      TMA producer: A/B code tiles via cp.async.bulk.tensor (128-B swizzle),
//               scale-factor atoms via cp.async.bulk, into a kStages-deep mbarrier ring
//   warp 1      TMEM allocator + single-thread MMA issuer: tcgen05.cp moves the
//               stage's scale factors SMEM -> TMEM, then tcgen05.mma
//               kind::mxf4nvf4.block_scale (scale_vec::4X ue4m3 for NVFP4,
//               ::2X ue8m0 for MXFP4) accumulates in TMEM; tcgen05.commit frees
//               the stage
//   warps 2-5   epilogue: tcgen05.ld 32 columns at a time, * ts_A*ts_W, -> bf16/f32
//               global stores
// Scale factors occupy a per-stage TMEM region so a stage's SF are only
// overwritten after the MMAs that read them committed (same ring as SMEM).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "quant_core.cuh"
#include "sm100.cuh"

namespace mrfp4 {
namespace {

constexpr int BM = 128;
constexpr int BK = 256;         // FP4 elements per k-block
constexpr int BK_BYTES = BK / 2;
constexpr int UMMA_K = 64;      // FP4 elements per tcgen05.mma
constexpr int kThreads = 192;

template <int VEC, int BN>
struct Cfg {
  static constexpr int kAtomsPerKb = BK / VEC / 4;  // 128x4 SF atoms per k-block: 4 (NVFP4) / 2 (MXFP4)
  static constexpr int kNB = BN / 128;              // 128-row SF blocks of B per tile
  static constexpr int kStages = 4;
  static constexpr int kABytes = BM * BK_BYTES;
  static constexpr int kBBytes = BN * BK_BYTES;
  static constexpr int kSfaBytes = kAtomsPerKb * 512;
  static constexpr int kSfbBytes = kNB * kAtomsPerKb * 512;
  static constexpr int kSfaCols = kAtomsPerKb * 4;
  static constexpr int kSfbCols = kNB * kAtomsPerKb * 4;
  static constexpr int kAccCols = BN;
  static constexpr int kTmemCols = 512;
  static_assert(kAccCols + kStages * (kSfaCols + kSfbCols) <= kTmemCols, "TMEM budget");
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kStages * kABytes;
  static constexpr int kOffSfa = kOffB + kStages * kBBytes;
  static constexpr int kOffSfb = kOffSfa + kStages * kSfaBytes;
  static constexpr int kOffBar = kOffSfb + kStages * kSfbBytes;
  static constexpr int kSmem = kOffBar + 256 + 1024;  // barriers + 1024-B alignment slack
};

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

struct GemmArgs {
  const uint8_t* b;       // weight codes [N, K/2] (L2 prefetch of upcoming panels)
  const uint8_t* a_sf;
  const uint8_t* b_sf;
  const float* a_ts;
  const float* b_ts;
  void* d;
  int64_t M, N, K, ldd;
  int64_t sf_col_blocks;  // ceil(K / VEC / 4)
  int64_t b_row_blocks;   // ceil(N / 128)
  int num_m_blk, num_n_blk, num_kb;
  int tail_mmas;  // MMAs in the last k-block (0 = full)
  int preissue;   // 2-CTA kernel: issue the first weight stages before the PDL wait
  int splits;     // 1-CTA kernel: K splits per output tile (> 1: fp32 partials to `ws`)
  int kb_per;     // k-blocks per split
  float* ws;      // [splits][M][N] fp32 partial sums (splits > 1)
  size_t ws_bytes;
  unsigned long long* dbg;  // perf experiments: per-k-block MMA-thread timestamps of CTA 0
  int debug;  // perf experiments: 1 = no operand loads, 2 = no MMAs (0 in production)
  // Fused next-layer MXFP4 quantization of the bf16 output (OUT == kOutMxq, 2-CTA kernel):
  // the epilogue rounds each output row to bf16, rotates it by H_k (k = q_hk in {0, 16, 32})
  // and writes the next layer's E2M1 codes [M, N/2] + swizzled E8M0 scales, exactly what K1
  // would produce from the bf16 output (quantizers.py:247-255).  d (bf16 Y) may be null.
  uint8_t* q_codes;
  uint8_t* q_sf;
  float* q_ts;        // the next layer's tensor scale: f32(4/3) (quantizers.py:191, :206-207) or the NVFP4 s_T
  const float* q_static_ts;  // NVFP4 next layer: the given (static) global scale s_T
  uint32_t* q_status;
  uint32_t q_cb;      // scale column blocks of the next layer: N / G / 4
  int64_t q_rows_pad; // ceil(M / 128) * 128
  qc::AQParams qp;    // c64 / kraw / kmx / pm of the next layer's rotation
  // Fused output all-gather (SURVEY.md 8(f) row f1, 2-CTA kernel, bf16): every output row
  // segment is stored to each of npeer destinations (peer-mapped over NVLink on a multi-GPU
  // node; each already offset to this rank's column block of that rank's full output).
  int npeer;
  void* peer_d[8];
  // 1-CTA split-K: per-tile arrival counters (zero between calls); the last split of a tile to
  // finish sums all splits' partials in split order (deterministic) and writes the output,
  // replacing the separate reduce kernel.  Null: the reduce kernel runs.
  uint32_t* sk_cnt;
};
constexpr size_t kSplitkHeader = 4096;   // counters, ahead of the fp32 partials in the workspace
constexpr int kOutMxq = 100;  // internal OUT tags (not ABI dtypes): bf16 output quantized for the next
constexpr int kOutNvq = 101;  // layer in MXFP4 / in NVFP4 with a static global scale
__host__ __device__ constexpr bool is_quant_out(int out) { return out == kOutMxq || out == kOutNvq; }

// Swizzled scale-factor offset (128 x 4 atoms), 32-bit.
__device__ __forceinline__ uint32_t sf_off32q(uint32_t r, uint32_t c, uint32_t cb) {
  return ((r >> 7) * cb + (c >> 2)) * 512u + (r & 31u) * 16u + ((r >> 5) & 3u) * 4u + (c & 3u);
}



// Advance a shared-memory descriptor's start-address field (bits [0,14), address >> 4)
// by `x` 16-byte units.  No carry can leave the field (SMEM < 228 KB), so only the low
// word changes: one IADD instead of re-encoding the descriptor.
__device__ __forceinline__ uint64_t desc_add(uint64_t d, uint32_t x) {
  uint64_t r;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tadd.u32 lo, lo, %2;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r)
      : "l"(d), "r"(x));
  return r;
}

// Issue MMAs k in [K0, K1) of one k-block.  The issuing thread's per-MMA work is kept
// to a few integer adds on precomputed stage descriptors: with the descriptors
// re-encoded per MMA the single issuing thread (dependent uniform-datapath chains)
// could not keep up with the tensor pipe (measured ~170-200 vs 128 cycles per MMA).
//   ad, bd   SMEM descriptors of this stage's A / B tiles at k = 0
//   sfa, sfb TMEM column of this stage's scale-factor slots
template <int VEC, int K0, int K1, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_mmas(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t sfa, uint32_t sfb,
                                           bool first) {
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    constexpr int kStepDesc = (UMMA_K / 2) >> 4;  // 32 B of K per MMA
    const uint32_t atom = VEC == 16 ? k : (k >> 1);
    const uint32_t sfid = VEC == 16 ? 0u : (uint32_t)(k & 1) * 2u;
    const uint32_t idesc = sm100::idesc_fp4(M, N, VEC == 32, sfid, sfid);
    const uint32_t acc = (K0 == 0 && k == 0 && first) ? 0u : 1u;
    const uint64_t adk = desc_add(ad, k * kStepDesc), bdk = desc_add(bd, k * kStepDesc);
    const uint32_t sa = sfa + (atom * 4 + (sfid << 30)), sb = sfb + (atom * kNB * 4 + (sfid << 30));
    if constexpr (PAIR)
      sm100::tc_mma_fp4_2sm<VEC>(d_tmem, adk, bdk, idesc, sa, sb, acc);
    else
      sm100::tc_mma_fp4<VEC>(d_tmem, adk, bdk, idesc, sa, sb, acc);
  }
}

// Warp-converged 2-CTA variant: all lanes run it, lane `el` issues.
template <int VEC, int K0, int K1, int M, int N, int kNB>
__device__ __forceinline__ void issue_mmas_warp(uint32_t el, uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t sfa,
                                                uint32_t sfb, bool first) {
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    constexpr int kStepDesc = (UMMA_K / 2) >> 4;
    const uint32_t atom = VEC == 16 ? k : (k >> 1);
    const uint32_t sfid = VEC == 16 ? 0u : (uint32_t)(k & 1) * 2u;
    const uint32_t idesc = sm100::idesc_fp4(M, N, VEC == 32, sfid, sfid);
    const uint32_t acc = (K0 == 0 && k == 0 && first) ? 0u : 1u;
    sm100::tc_mma_fp4_2sm_if<VEC>(el, d_tmem, desc_add(ad, k * kStepDesc), desc_add(bd, k * kStepDesc), idesc,
                                  sfa + (atom * 4 + (sfid << 30)), sfb + (atom * kNB * 4 + (sfid << 30)), acc);
  }
}

template <int VEC, int NK, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_kblock(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t sfa, uint32_t sfb,
                                             bool first) {
  issue_mmas<VEC, 0, NK, M, N, kNB, PAIR>(d_tmem, ad, bd, sfa, sfb, first);
}

template <int VEC, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_kblock_any(int nk, uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t sfa,
                                                 uint32_t sfb, bool first) {
  switch (nk) {
    case 4: issue_kblock<VEC, 4, M, N, kNB, PAIR>(d_tmem, ad, bd, sfa, sfb, first); break;
    case 3: issue_kblock<VEC, 3, M, N, kNB, PAIR>(d_tmem, ad, bd, sfa, sfb, first); break;
    case 2: issue_kblock<VEC, 2, M, N, kNB, PAIR>(d_tmem, ad, bd, sfa, sfb, first); break;
    case 1: issue_kblock<VEC, 1, M, N, kNB, PAIR>(d_tmem, ad, bd, sfa, sfb, first); break;
    default: break;
  }
}

// 256-bit global store (sm_100): 8 words to a 32-byte aligned address.
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* r) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// 32 consecutive accumulator columns of one output row -> global (bf16 or f32).
template <int OUT>
__device__ __forceinline__ void store_row32(const GemmArgs& g, int64_t row, int64_t col, const uint32_t (&r)[32],
                                            float alpha) {
  if constexpr (OUT == MRFP4_DT_BF16) {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g.d) + row * g.ldd + col;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (col + 8 * j < g.N) {
        uint32_t w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 2 * t]) * alpha,
                                                   __uint_as_float(r[8 * j + 2 * t + 1]) * alpha);
          w[t] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(dst + 8 * j) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  } else {
    float* dst = static_cast<float*>(g.d) + row * g.ldd + col;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (col + 4 * j < g.N) {
        *reinterpret_cast<float4*>(dst + 4 * j) =
            make_float4(__uint_as_float(r[4 * j]) * alpha, __uint_as_float(r[4 * j + 1]) * alpha,
                        __uint_as_float(r[4 * j + 2]) * alpha, __uint_as_float(r[4 * j + 3]) * alpha);
      }
    }
  }
}

template <int VEC, int BN, int OUT>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_fp4(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
  using C = Cfg<VEC, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // perf experiments (per-CTA globaltimer stamps, load/MMA knock-out modes) exist only in
  // MRFP4_TRACE builds (scripts/build_variant.sh): compiled out of the production kernel
#ifdef MRFP4_TRACE
  const int dbg_mode = g.debug;
  unsigned long long* const dbg_buf = g.dbg;
#else
  constexpr int dbg_mode = 0;
  unsigned long long* const dbg_buf = nullptr;
#endif
  auto mark = [&](int i) { if (dbg_buf) dbg_buf[blockIdx.x * 8 + i] = globaltimer(); };
  if (threadIdx.x == 0) mark(0);
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(tfull, 1);
    sm100::mbar_init(tempty, 4);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc(tmem_holder, C::kTmemCols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) mark(1);
  pdl_trigger();

  const int num_units = g.num_m_blk * g.num_n_blk * g.splits;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      auto stage_bytes = [&](int kb, int n_blk) {
        const int atoms = (int)imin64(C::kAtomsPerKb, g.sf_col_blocks - (int64_t)kb * C::kAtomsPerKb);
        int nbv = 0;
#pragma unroll
        for (int j = 0; j < C::kNB; ++j) nbv += ((int64_t)n_blk * C::kNB + j < g.b_row_blocks);
        return C::kABytes + C::kBBytes + (uint32_t)atoms * 512u * (1u + nbv);
      };
      auto load_weight = [&](int stage, int kb, int n_blk) {
        const int atoms = (int)imin64(C::kAtomsPerKb, g.sf_col_blocks - (int64_t)kb * C::kAtomsPerKb);
        const int64_t katom = (int64_t)kb * C::kAtomsPerKb;
        sm100::tma_load_2d(smem + C::kOffB + stage * C::kBBytes, &tmB, &full[stage], kb * BK_BYTES, n_blk * BN);
#pragma unroll
        for (int j = 0; j < C::kNB; ++j) {
          const int64_t rb = (int64_t)n_blk * C::kNB + j;
          if (rb < g.b_row_blocks)
            sm100::bulk_load(smem + C::kOffSfb + stage * C::kSfbBytes + j * C::kAtomsPerKb * 512,
                             g.b_sf + (rb * g.sf_col_blocks + katom) * 512, atoms * 512u, &full[stage]);
        }
      };
      // The weight half of the first unit's first stages does not depend on the act-quant
      // kernel: issue it before the PDL wait so the weight stream overlaps K1's tail.
      int pre = 0;
      if (blockIdx.x < num_units && dbg_mode == 0) {
        const int tile = blockIdx.x / g.splits, split = blockIdx.x - tile * g.splits;
        const int n_blk = tile / g.num_m_blk;
        const int kb0 = split * g.kb_per, kb1 = min(g.num_kb, kb0 + g.kb_per);
        pre = min(kb1 - kb0, C::kStages);
        for (int i = 0; i < pre; ++i) {
          sm100::mbar_arrive_expect_tx(&full[i], stage_bytes(kb0 + i, n_blk));   // A + B, all of it
          load_weight(i, kb0 + i, n_blk);
        }
      }
      pdl_wait();  // A, its scale factors and tensor scale come from the act-quant kernel
      mark(2);
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int tile = unit / g.splits, split = unit - tile * g.splits;
        const int m_blk = tile % g.num_m_blk, n_blk = tile / g.num_m_blk;
        const int kb0 = split * g.kb_per, kb1 = min(g.num_kb, kb0 + g.kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          const bool preissued = unit == (int)blockIdx.x && kb - kb0 < pre;
          if (!preissued) sm100::mbar_wait(&empty[stage], phase ^ 1);
          const int atoms = (int)imin64(C::kAtomsPerKb, g.sf_col_blocks - (int64_t)kb * C::kAtomsPerKb);
          if (dbg_mode == 1 || dbg_mode == 3 || dbg_mode == 4 || dbg_mode == 5) {
            sm100::mbar_arrive(&full[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (!preissued) {
            sm100::mbar_arrive_expect_tx(&full[stage], stage_bytes(kb, n_blk));
            load_weight(stage, kb, n_blk);
          }
          sm100::tma_load_2d(smem + C::kOffA + stage * C::kABytes, &tmA, &full[stage], kb * BK_BYTES, m_blk * BM);
          const int64_t katom = (int64_t)kb * C::kAtomsPerKb;
          sm100::bulk_load(smem + C::kOffSfa + stage * C::kSfaBytes,
                           g.a_sf + ((int64_t)m_blk * g.sf_col_blocks + katom) * 512, atoms * 512u, &full[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      const uint64_t adesc0 = sm100::smem_desc(sm100::smem_u32(smem + C::kOffA), 16, 1024, 2);
      const uint64_t bdesc0 = sm100::smem_desc(sm100::smem_u32(smem + C::kOffB), 16, 1024, 2);
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int split = unit % g.splits;
        const int kb0 = split * g.kb_per, kb1 = min(g.num_kb, kb0 + g.kb_per);
        sm100::mbar_wait(tempty, acc_phase ^ 1);
        sm100::tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          if (kb == kb0 && unit == (int)blockIdx.x) mark(3);
          sm100::tc_fence_after();
          const uint32_t sfa_t = tmem_base + C::kAccCols + stage * (C::kSfaCols + C::kSfbCols);
          const uint32_t sfb_t = sfa_t + C::kSfaCols;
          const uint32_t sfa_s = sm100::smem_u32(smem + C::kOffSfa + stage * C::kSfaBytes);
          const uint32_t sfb_s = sm100::smem_u32(smem + C::kOffSfb + stage * C::kSfbBytes);
#pragma unroll
          for (int a = 0; a < C::kAtomsPerKb; ++a) {
            if (dbg_mode < 5 || (dbg_mode == 6 && kb < C::kStages)) {
              sm100::tc_cp_32x128b_warpx4(sfa_t + a * 4, sm100::smem_desc(sfa_s + a * 512, 0, 128, 0));
#pragma unroll
              for (int j = 0; j < C::kNB; ++j)
                sm100::tc_cp_32x128b_warpx4(sfb_t + a * C::kNB * 4 + j * 4,
                                            sm100::smem_desc(sfb_s + (j * C::kAtomsPerKb + a) * 512, 0, 128, 0));
            }
          }
          const uint64_t ad = desc_add(adesc0, (uint32_t)(stage * (C::kABytes >> 4)));
          const uint64_t bd = desc_add(bdesc0, (uint32_t)(stage * (C::kBBytes >> 4)));
          if (dbg_mode == 2 || dbg_mode == 4) {
          } else if (kb + 1 < g.num_kb || g.tail_mmas == 0) {
            issue_kblock<VEC, BK / UMMA_K, BM, BN, C::kNB, false>(tmem_base, ad, bd, sfa_t, sfb_t, kb == kb0);
          } else {
            issue_kblock_any<VEC, BM, BN, C::kNB, false>(g.tail_mmas, tmem_base, ad, bd, sfa_t, sfb_t, kb == kb0);
          }
          sm100::tc_commit(&empty[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        sm100::tc_commit(tfull);
        acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    pdl_wait();
    const float alpha = __ldg(g.a_ts) * __ldg(g.b_ts);
    uint32_t acc_phase = 0;
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
      const int tile = unit / g.splits, split = unit - tile * g.splits;
      const int m_blk = tile % g.num_m_blk, n_blk = tile / g.num_m_blk;
      sm100::mbar_wait(tfull, acc_phase);
      if (threadIdx.x == 64 && unit == (int)blockIdx.x) mark(4);
      sm100::tc_fence_after();
      const int64_t row = (int64_t)m_blk * BM + q * 32 + lane;
      // Split-K: lanes past M skip the TMEM read entirely when the whole warp is past M.
      const bool warp_live = (int64_t)m_blk * BM + q * 32 < g.M;
#pragma unroll 1
      for (int c = 0; c < ((dbg_mode >= 3 && dbg_mode <= 5) || !warp_live ? 0 : BN); c += 64) {
        uint32_t r[2][32];   // two 32-column TMEM loads per wait
        sm100::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + c, r[0]);
        sm100::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + c + 32, r[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = (int64_t)n_blk * BN + c + 32 * h;
          if (row < g.M) {
            if (g.splits == 1) {
              store_row32<OUT>(g, row, col, r[h], alpha);
            } else {  // fp32 partial, unscaled: ws[split][row][col]
              float* dst = g.ws + ((int64_t)split * g.M + row) * g.N + col;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (col + 4 * j < g.N)
                  *reinterpret_cast<float4*>(dst + 4 * j) =
                      make_float4(__uint_as_float(r[h][4 * j]), __uint_as_float(r[h][4 * j + 1]),
                                  __uint_as_float(r[h][4 * j + 2]), __uint_as_float(r[h][4 * j + 3]));
            }
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(tempty);
      acc_phase ^= 1;
      if (g.splits > 1 && g.sk_cnt) {
        // ---- in-kernel split-K reduction.  Every unit is resident at once (units <= SMs, one
        // CTA each, checked by the host), so the tile's splits wait for each other and then each
        // reduces 1/splits of the tile, summing ALL splits' partials in split order (the same
        // order, hence the same bits, as a separate reduce kernel).  Counter pair per tile:
        // [0] partials written, [1] slices reduced; the last slice re-arms both.
        uint32_t* cnt = g.sk_cnt + 2 * tile;
        const int et = threadIdx.x - 64;   // epilogue thread 0..127 (warps 2-5)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          mark(5);
          __threadfence();   // cumulative over the epilogue's stores ordered by the bar.sync
          atomicAdd(cnt, 1u);
          uint32_t seen;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
          } while (seen < (uint32_t)g.splits);
          mark(6);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        __threadfence();
        const int64_t r0 = (int64_t)m_blk * BM, c0 = (int64_t)n_blk * BN;
        const int rows = (int)imin64(BM, g.M - r0), c4 = (int)imin64(BN, g.N - c0) / 4;
        const int total = rows * c4, chunk = (total + g.splits - 1) / g.splits;
        const int e_end = min(total, (split + 1) * chunk);
        for (int e = split * chunk + et; e < e_end; e += 128) {
          const int rr = e / c4, cc = (e - rr * c4) * 4;
          const int64_t off = (r0 + rr) * g.N + c0 + cc;
          float4 acc = make_float4(-0.f, -0.f, -0.f, -0.f);   // -0 + x == x bit for bit
          for (int s0 = 0; s0 < g.splits; s0 += 8) {
            float4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (s0 + j < g.splits) v[j] = __ldcg(reinterpret_cast<const float4*>(g.ws + (int64_t)(s0 + j) * g.M * g.N + off));
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (s0 + j < g.splits) { acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w; }
          }
          if constexpr (OUT == MRFP4_DT_BF16) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * alpha, acc.y * alpha);
            __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * alpha, acc.w * alpha);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(g.d) + (r0 + rr) * g.ldd + c0 + cc) = pk;
          } else {
            *reinterpret_cast<float4*>(static_cast<float*>(g.d) + (r0 + rr) * g.ldd + c0 + cc) =
                make_float4(acc.x * alpha, acc.y * alpha, acc.z * alpha, acc.w * alpha);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) mark(7);
        if (et == 0 && atomicAdd(cnt + 1, 1u) == (uint32_t)g.splits - 1) {
          cnt[0] = 0u;   // every split has passed its wait: re-arm for the next call
          cnt[1] = 0u;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}


// ---------------------------------------------------------------------------
// 2-CTA (cta_group::2) kernel: a CTA pair computes a 256 x 256 output tile, persistent
// over tiles.  K advances in 512-wide stages (two 128-B K slices per row).
//   warp 0      TMA producer (both CTAs): one 3-D box of 128 rows x 2 slices each for A
//               and B, and 3-D boxes of this CTA's scale-factor atoms (SFA for its 128
//               rows, SFB for all 256 rows) -- all cta_group::2, so every byte of both
//               CTAs is counted on the LEADER's mbarriers (`full` for A/B, `sf_full` for
//               the SF slot).  Out-of-range boxes (M / N / K tails) are zero-filled by TMA.
//   warp 1      TMEM allocator (both) + MMA issuer (leader, whole warp converged, one
//               elected lane issues): per stage, tcgen05.cp.cta_group::2 copies both CTAs'
//               SF atoms SMEM -> their own TMEM SF slot, then 8 x tcgen05.mma.cta_group::2
//               M=256 N=256 K=64 read them; cp and MMA are issued by the same thread, so the
//               tensor pipe orders them -- no cross-CTA handoff, no cluster-scope fence.
//               Commits go multicast to both CTAs (`empty` A/B stage, `sf_empty` SF slot).
//               (scripts/mma2_cp_rate.cu: 12 atom copies per 8 MMAs are free, 24 -- NVFP4 --
//               cost ~11% when the MMAs are back to back; before this the SF went through
//               stager warps + a MEMBAR.ALL.GPU per stage on the peer.)
//   warps 2-9   epilogue (per CTA): TMEM -> regs -> * ts_A*ts_W -> bf16 (released to the
//               next tile's MMAs before the global stores) / f32 -> global
// A/B SMEM stages and SF slots are decoupled: 3 A/B stages of 64 KB (~97 B/cycle/SM of
// TMA throughput measured for this box shape) and 2-3 SF slots (SMEM and TMEM), sized so
// NVFP4's SF (96 TMEM columns per stage) fit next to the 256-column accumulator.
// ---------------------------------------------------------------------------
template <int VEC>
struct Cfg2 {
#ifndef MRFP4_K2_BK
#define MRFP4_K2_BK 256
#endif
#ifndef MRFP4_K2_STAGES
#define MRFP4_K2_STAGES 6
#endif
#ifndef MRFP4_K2_SFSLOTS
#define MRFP4_K2_SFSLOTS 5
#endif
  // 256-wide stages, 6 deep (16-KB boxes per operand per CTA, the shape of cuBLASLt's
  // 256x256x256 2-SM block-scaled kernel), with the scale factors on their own producer warp:
  // a slot is recycled after 4 MMAs.  70B up NVFP4 K2: 194 -> 163 us (91% of 4x bf16);
  // 3 x 512-wide stages with one producer thread for A/B and SF: 196 us; 256-wide with one
  // producer thread: 262 us (the thread could not issue fast enough) -- profiles/r02_k2_notes.md.
  static constexpr int kBK = MRFP4_K2_BK;                        // FP4 elements per stage
  static constexpr int kSlices = kBK / BK;                       // 128-B K slices per stage
  static constexpr int kMmas = kBK / UMMA_K;                     // MMAs per stage
  static constexpr int kAtoms = kBK / VEC / 4;                   // SF atoms (128 rows x 4 cols) per stage
  static constexpr int kStages = MRFP4_K2_STAGES;                // A/B stages
  static constexpr int kSfSlots = MRFP4_K2_SFSLOTS;              // SF slots (SMEM and TMEM)
  static constexpr int kABytes = 128 * kBK / 2;
  static constexpr int kBBytes = 128 * kBK / 2;
  static constexpr int kSfaBytes = kAtoms * 512;
  static constexpr int kSfbBytes = 2 * kAtoms * 512;
  static constexpr int kSfaCols = kAtoms * 4;
  static constexpr int kSfbCols = 2 * kAtoms * 4;
  static constexpr int kSfCols = kSfaCols + kSfbCols;          // TMEM columns per SF slot
  static constexpr int kAccCols = 256;
  static constexpr int kTmemCols = 512;
  static_assert(kAccCols + kSfSlots * kSfCols <= kTmemCols, "TMEM budget");
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kStages * kABytes;
  static constexpr int kOffSfa = kOffB + kStages * kBBytes;
  static constexpr int kOffSfb = kOffSfa + kSfSlots * kSfaBytes;
  static constexpr int kOffBar = kOffSfb + kSfSlots * kSfbBytes;
  static constexpr int kSmem = kOffBar + 512 + 1024;
  static_assert(kSmem <= 232448, "SMEM budget");
#ifndef MRFP4_K2_SFWARP
#define MRFP4_K2_SFWARP 1
#endif
#ifndef MRFP4_K2_BWARP
#define MRFP4_K2_BWARP 0
#endif
  static constexpr bool kSfWarp = MRFP4_K2_SFWARP;   // scale factors issued by their own producer warp (2)
  static constexpr bool kBWarp = kSfWarp && MRFP4_K2_BWARP;   // B codes by their own producer warp (3)
  static constexpr int kEpiWarp0 = 2 + kSfWarp + kBWarp;
  static constexpr int kEpiWarps = 8;   // 2 per TMEM lane quadrant, 128 accumulator columns each
  static constexpr int kThreads2 = 32 * (kEpiWarp0 + kEpiWarps);
};

// 3-D TMA load (box {128 B, 128 rows, kSlices}) whose completion bytes are counted on the
// LEADER CTA's mbarrier (cta_group::2).
__device__ __forceinline__ void tma_load_3d_2sm(void* smem_dst, const CUtensorMap* desc, uint32_t leader_mbar,
                                                int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sm100::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(leader_mbar), "r"(0), "r"(c1), "r"(c2)
      : "memory");
}

// Warp-converged MMAs k in [K0, K1) of a 512-wide stage (k-step k: K slice k / 4, 32-B
// offset k % 4 inside the 128-B swizzled row).
template <int VEC, int K0, int K1>
__device__ __forceinline__ void issue_stage_mmas(uint32_t el, uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t sfa,
                                                 uint32_t sfb, bool first) {
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    constexpr uint32_t kSliceDesc = (128 * BK_BYTES) >> 4;   // 16 KB between K slices
    const uint32_t off = (uint32_t)(k >> 2) * kSliceDesc + (uint32_t)(k & 3) * 2u;
    const uint32_t atom = VEC == 16 ? k : (k >> 1);
    const uint32_t sfid = VEC == 16 ? 0u : (uint32_t)(k & 1) * 2u;
    const uint32_t idesc = sm100::idesc_fp4(256, 256, VEC == 32, sfid, sfid);
    const uint32_t acc = (K0 == 0 && k == 0 && first) ? 0u : 1u;
    sm100::tc_mma_fp4_2sm_if<VEC>(el, d_tmem, desc_add(ad, off), desc_add(bd, off), idesc,
                                  sfa + (atom * 4 + (sfid << 30)), sfb + (atom * 8 + (sfid << 30)), acc);
  }
}

template <int VEC>
__device__ __forceinline__ void issue_stage_tail(int nk, uint32_t el, uint32_t d_tmem, uint64_t ad, uint64_t bd,
                                                 uint32_t sfa, uint32_t sfb, bool first) {
  switch (nk) {  // MMAs in the last stage (0 = full)
    case 1: issue_stage_mmas<VEC, 0, 1>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 2: issue_stage_mmas<VEC, 0, 2>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 3: issue_stage_mmas<VEC, 0, 3>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 4: issue_stage_mmas<VEC, 0, 4>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 5: issue_stage_mmas<VEC, 0, 5>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 6: issue_stage_mmas<VEC, 0, 6>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    case 7: issue_stage_mmas<VEC, 0, 7>(el, d_tmem, ad, bd, sfa, sfb, first); break;
    default: issue_stage_mmas<VEC, 0, 8>(el, d_tmem, ad, bd, sfa, sfb, first); break;
  }
}

// Next-layer quantization of one output row's 128 bf16 columns (4 segments of 32) -- the K1
// arithmetic (quant_core.cuh) on the values K1 would read back from Y: MXFP4 (OUT == kOutMxq),
// or NVFP4 against a given global scale (kOutNvq; the whole-Y max would need all of Y first).
// Rotation: k <= 32 inside each segment; k = 64 / 128 span 2 / 4 segments of the row, so the
// cross-segment butterfly stages (block element bits 5, 6) run in registers after the 32-point
// transforms -- the FWHT stage order of K1.  Padding rows [M, rows_pad) get zero scale bytes.
template <int OUT, int HKQ>
__device__ __forceinline__ void quant_next_row(const GemmArgs& g, const qc::EncConsts& k, int64_t row, int64_t col0,
                                               const uint32_t (&pkd)[64]) {
  using namespace qc;
  constexpr bool kNv = OUT == kOutNvq;
  constexpr int G = kNv ? 16 : 32;
  if (row >= g.M) {
    if (row < g.q_rows_pad)
#pragma unroll
      for (int c = 0; c < 128 / G; ++c) g.q_sf[sf_off32q((uint32_t)row, (uint32_t)(col0 / G + c), g.q_cb)] = 0;
    return;
  }
  uint32_t bad = 0;
  auto encode = [&](const u64 (&P)[kPairs], int c) {
    float a0, a1;
    half_amax(P, a0, a1);
    GroupScale s0, s1;
    if constexpr (kNv) {
      s0 = nv_group_scale(a0, g.qp, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
      s1 = nv_group_scale(a1, g.qp, k.kenc, k.knv, k.st32, k.st64, k.zero_code);
      if (__float_as_uint(a0) >= 0x7f800000u || __float_as_uint(a1) >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
      if (s0.code == 0 || s1.code == 0) bad |= MRFP4_STATUS_SCALE_UNDERFLOW;
    } else {
      const float a = max3n(a0, a1, 0.f);
      if (__float_as_uint(a) >= 0x7f800000u) bad |= MRFP4_STATUS_NONFINITE;
      s0 = mx_group_scale(a, g.qp);
      s1 = s0;
    }
    uint32_t w4[4];
    quantize_seg(P, s0, s1, k.st32, g.qp, w4);
    *reinterpret_cast<uint4*>(g.q_codes + row * (g.N >> 1) + ((col0 + 32 * c) >> 1)) =
        make_uint4(w4[0], w4[1], w4[2], w4[3]);
    if constexpr (kNv)   // columns 2c, 2c+1 of the 16-element groups share a 16-bit word of the layout
      *reinterpret_cast<uint16_t*>(g.q_sf + sf_off32q((uint32_t)row, (uint32_t)(col0 / 16 + 2 * c), g.q_cb)) =
          (uint16_t)(s0.code | (s1.code << 8));
    else
      g.q_sf[sf_off32q((uint32_t)row, (uint32_t)(col0 / 32 + c), g.q_cb)] = (uint8_t)s0.code;
  };
  auto unpack = [&](u64 (&P)[kPairs], int c) {
#pragma unroll
    for (int j = 0; j < kPairs; ++j) {
      const uint32_t w = pkd[16 * c + j];
      P[j] = pk(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
    }
  };
  if constexpr (HKQ <= 32) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      u64 P[kPairs];
      unpack(P, c);
      if constexpr (HKQ > 0) fwht<HKQ>(P, 0, g.qp.pm);
      encode(P, c);
    }
  } else {
    u64 P[4][kPairs];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      unpack(P[c], c);
      fwht<32>(P[c], 0, g.qp.pm);
    }
#pragma unroll
    for (int c = 0; c < 4; c += 2)          // bit 5: segments (c, c + 1)
#pragma unroll
      for (int j = 0; j < kPairs; ++j) {
        const u64 a = P[c][j], b = P[c + 1][j];
        P[c][j] = add2(a, b);
        P[c + 1][j] = sub2(a, b);
      }
    if constexpr (HKQ >= 128) {
#pragma unroll
      for (int c = 0; c < 2; ++c)           // bit 6: segments (c, c + 2)
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
          const u64 a = P[c][j], b = P[c + 2][j];
          P[c][j] = add2(a, b);
          P[c + 2][j] = sub2(a, b);
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) encode(P[c], c);
  }
  if (bad) atomic_or_status(g.q_status, bad);
}

// Work of one cluster, identical for all roles of both CTAs: whole 256 x 256 tiles,
// tile = cluster + i * clusters (m-block fastest, so concurrent pairs share weight panels in L2).
// (A stream-K tail -- splitting a sparse last wave's k-stages across pairs with fp32
// partials -- was implemented and measured slower than this schedule in every case tried on
// B200, e.g. 256x14336x8192: 46.0 vs 34.9 us, and removed.)
struct Work {
  int tile, kb0, kb1;
};

struct WorkIter {
  int c, C, i;
  __device__ __forceinline__ WorkIter(const GemmArgs&, int cluster, int nclusters) : c(cluster), C(nclusters), i(0) {}
  __device__ __forceinline__ bool next(const GemmArgs& g, Work& w) {
    const int t = c + i * C;
    if (t >= g.num_m_blk * g.num_n_blk) return false;
    ++i;
    w = Work{t, 0, g.num_kb};
    return true;
  }
};

// Flattened (tile, k-stage) sequence of one cluster's work.
struct StageIter {
  WorkIter it;
  Work w;
  int kb, nm;
  bool live;
  const GemmArgs& g;
  __device__ __forceinline__ StageIter(const GemmArgs& g_, int cluster, int nclusters, int num_m_blk)
      : it(g_, cluster, nclusters), nm(num_m_blk), g(g_) {
    live = it.next(g, w);
    kb = live ? w.kb0 : 0;
  }
  __device__ __forceinline__ int m_blk() const { return w.tile % nm; }
  __device__ __forceinline__ int n_blk() const { return w.tile / nm; }
  __device__ __forceinline__ void advance() {
    if (++kb >= w.kb1) {
      live = it.next(g, w);
      kb = live ? w.kb0 : 0;
    }
  }
};

// Ring position: slot index and parity, advanced once per stage.
struct Ring {
  int idx = 0;
  uint32_t ph = 0;
  template <int N>
  __device__ __forceinline__ void next() {
    if (++idx == N) { idx = 0; ph ^= 1; }
  }
};

template <int VEC, int OUT, int HKQ = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2<VEC>::kThreads2, 1)
    k_gemm_fp4_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmSfa, const __grid_constant__ CUtensorMap tmSfb, GemmArgs g) {
  using C = Cfg2<VEC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);   // leader's: A/B of both CTAs landed
  uint64_t* empty = full + C::kStages;                               // A/B stage free (MMAs committed)
  uint64_t* sf_full = empty + C::kStages;                            // leader's: SF slot of both CTAs landed
  uint64_t* sf_empty = sf_full + C::kSfSlots;                        // SF slot (SMEM + TMEM) free
  uint64_t* tfull = sf_empty + C::kSfSlots;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Kernel parameters into registers once (asm "memory" clobbers would force reloads).
  const int num_m_blk = g.num_m_blk, num_kb = g.num_kb, tail_mmas = g.tail_mmas;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmSfa);
    sm100::tma_prefetch_desc(&tmSfb);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);    // the leader producer's expect_tx (bytes of both CTAs)
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kSfSlots; ++s) {
      sm100::mbar_init(&sf_full[s], 1);
      sm100::mbar_init(&sf_empty[s], 1);
    }
    sm100::mbar_init(tfull, 1);
    sm100::mbar_init(tempty, 2 * C::kEpiWarps);  // epilogue warps x 2 CTAs
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc_2sm(tmem_holder, C::kTmemCols);
  sm100::tc_fence_before();
  __syncwarp();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------- producer
      // Two independent streams, each bounded by its own ring: A/B codes (3 stages) and scale
      // factors (2-3 slots); whichever has a free slot is issued next.  The weight (B) of the
      // first stages does not depend on the act-quant kernel: it is issued BEFORE the PDL
      // wait, so its latency hides behind K1's tail; A and the scale factors follow.
      Ring ab, sf;
      StageIter abq(g, cluster, nclusters, num_m_blk), sfq(g, cluster, nclusters, num_m_blk);
      auto arm = [&](uint64_t* bar, uint32_t bytes) {
        if (leader) sm100::mbar_arrive_expect_tx(bar, 2u * bytes);   // this CTA's and the peer's bytes
      };
      auto load_ab = [&](bool a_part, bool b_part) {
        const int kb = abq.kb, mb = abq.m_blk(), nb = abq.n_blk();
        const uint32_t bar = sm100::leader_bar(&full[ab.idx]);
        if (b_part)
          tma_load_3d_2sm(smem + C::kOffB + ab.idx * C::kBBytes, &tmB, bar, nb * 256 + (int)rank * 128,
                          kb * C::kSlices);
        if (a_part)
          tma_load_3d_2sm(smem + C::kOffA + ab.idx * C::kABytes, &tmA, bar, mb * 256 + (int)rank * 128,
                          kb * C::kSlices);
      };
      auto load_sf = [&] {
        const int kb = sfq.kb, mb = sfq.m_blk(), nb = sfq.n_blk();
        arm(&sf_full[sf.idx], C::kSfaBytes + C::kSfbBytes);
        const uint32_t bar = sm100::leader_bar(&sf_full[sf.idx]);
        // SF boxes {256 B, 2 * kAtoms half-atoms, 1 | 2 row blocks}: this CTA's 128 rows of A,
        // both 128-row blocks of the tile's B (each CTA's MMA half needs all 256 N columns).
        tma_load_3d_2sm(smem + C::kOffSfa + sf.idx * C::kSfaBytes, &tmSfa, bar, 2 * C::kAtoms * kb, mb * 2 + (int)rank);
        tma_load_3d_2sm(smem + C::kOffSfb + sf.idx * C::kSfbBytes, &tmSfb, bar, 2 * C::kAtoms * kb, nb * 2);
        sfq.advance();
        sf.next<C::kSfSlots>();
      };
      // PDL pre-issue: the weight half of the first A/B stages
      int pre = 0;
      if (g.preissue && !C::kBWarp) {
        StageIter q2 = abq;
        for (; pre < C::kStages && q2.live; ++pre) {
          arm(&full[pre], C::kABytes + C::kBBytes);
          tma_load_3d_2sm(smem + C::kOffB + pre * C::kBBytes, &tmB, sm100::leader_bar(&full[pre]),
                          q2.n_blk() * 256 + (int)rank * 128, q2.kb * C::kSlices);
          q2.advance();
        }
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) {   // A of the pre-issued stages (their slots were never used)
        load_ab(true, false);
        abq.advance();
        ab.next<C::kStages>();
      }
      if constexpr (C::kSfWarp) {
        while (abq.live) {
          sm100::mbar_wait(&empty[ab.idx], ab.ph ^ 1);
          arm(&full[ab.idx], C::kABytes + C::kBBytes);
          load_ab(true, !C::kBWarp);
          abq.advance();
          ab.next<C::kStages>();
        }
      } else {
        while (abq.live || sfq.live) {
          if (sfq.live && sm100::mbar_test(&sf_empty[sf.idx], sf.ph ^ 1)) {
            load_sf();
          } else if (abq.live && sm100::mbar_test(&empty[ab.idx], ab.ph ^ 1)) {
            arm(&full[ab.idx], C::kABytes + C::kBBytes);
            load_ab(true, true);
            abq.advance();
            ab.next<C::kStages>();
          }
        }
      }
    }
  } else if (C::kBWarp && warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------ B producer
      // The weight stream on its own thread (it does not depend on the act-quant kernel: no
      // PDL wait); the A producer arms `full` with both operands' bytes.
      Ring ab;
      StageIter q(g, cluster, nclusters, num_m_blk);
      while (q.live) {
        sm100::mbar_wait(&empty[ab.idx], ab.ph ^ 1);
        tma_load_3d_2sm(smem + C::kOffB + ab.idx * C::kBBytes, &tmB, sm100::leader_bar(&full[ab.idx]),
                        q.n_blk() * 256 + (int)rank * 128, q.kb * C::kSlices);
        q.advance();
        ab.next<C::kStages>();
      }
    }
  } else if (C::kSfWarp && warp == 2) {
    if (lane == 0) {
      // ---------------------------------------------------------- SF producer
      // The scale-factor stream on its own thread: its slot waits and small TMA issues never
      // delay the A/B stream (and vice versa).
      Ring sf;
      StageIter sfq(g, cluster, nclusters, num_m_blk);
      pdl_wait();   // SFA comes from the act-quant kernel
      while (sfq.live) {
        sm100::mbar_wait(&sf_empty[sf.idx], sf.ph ^ 1);
        const int kb = sfq.kb, mb = sfq.m_blk(), nb = sfq.n_blk();
        if (leader) sm100::mbar_arrive_expect_tx(&sf_full[sf.idx], 2u * (C::kSfaBytes + C::kSfbBytes));
        const uint32_t bar = sm100::leader_bar(&sf_full[sf.idx]);
        tma_load_3d_2sm(smem + C::kOffSfa + sf.idx * C::kSfaBytes, &tmSfa, bar, 2 * C::kAtoms * kb, mb * 2 + (int)rank);
        tma_load_3d_2sm(smem + C::kOffSfb + sf.idx * C::kSfbBytes, &tmSfb, bar, 2 * C::kAtoms * kb, nb * 2);
        sfq.advance();
        sf.next<C::kSfSlots>();
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------------------------------------------------- MMA issuer
      // The whole warp runs the loop (converged, uniform descriptors); one elected lane
      // issues.  A stage's SF copies and 8 MMAs (~1000 cycles of tensor work) are queued
      // before the thread waits for the next stage, so barrier latency never starves the pipe.
      // An SF slot's TMEM columns are rewritten only after sf_full of its next use, which the
      // producer arms only after sf_empty (the previous use's MMAs completed).
      const uint32_t el = sm100::elect_lane();
      Ring ab, sf;
      uint32_t acc_phase = 0;
      const uint64_t adesc0 = sm100::smem_desc(sm100::smem_u32(smem + C::kOffA), 16, 1024, 2);
      const uint64_t bdesc0 = sm100::smem_desc(sm100::smem_u32(smem + C::kOffB), 16, 1024, 2);
      const uint32_t sfa_s0 = sm100::smem_u32(smem + C::kOffSfa), sfb_s0 = sm100::smem_u32(smem + C::kOffSfb);
      const uint32_t sf0 = tmem_base + C::kAccCols;
      WorkIter it(g, cluster, nclusters);
      Work w;
#ifdef MRFP4_TRACE
      // perf experiments (scripts/k2_timeline.py): per-stage clock64 of cluster 0's MMA thread
      unsigned long long* tr = (g.dbg && cluster == 0 && lane == 0) ? g.dbg : nullptr;
      int tn = 0;
      auto stamp = [&](int tag) { if (tr && tn < 8192) { tr[2 * tn] = clock64(); tr[2 * tn + 1] = tag; ++tn; } };
#else
      auto stamp = [](int) {};
#endif
      while (it.next(g, w)) {
        stamp(0);
        sm100::mbar_wait_cluster(tempty, acc_phase ^ 1);   // both CTAs' epilogues (remote arrivals)
        stamp(1);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          sm100::mbar_wait(&sf_full[sf.idx], sf.ph);
          stamp(2);
          sm100::mbar_wait(&full[ab.idx], ab.ph);
          stamp(3);
          sm100::tc_fence_after();
          const uint32_t sfa_t = sf0 + sf.idx * C::kSfCols, sfb_t = sfa_t + C::kSfaCols;
          const uint32_t sfa_s = sfa_s0 + sf.idx * C::kSfaBytes, sfb_s = sfb_s0 + sf.idx * C::kSfbBytes;
#pragma unroll
          for (int a = 0; a < C::kAtoms; ++a) {   // TMEM SFB order: atom-major, then 128-row block
            sm100::tc_cp_32x128b_warpx4_2sm_if(el, sfa_t + a * 4, sm100::smem_desc(sfa_s + a * 512, 0, 128, 0));
#pragma unroll
            for (int j = 0; j < 2; ++j)
              sm100::tc_cp_32x128b_warpx4_2sm_if(el, sfb_t + (2 * a + j) * 4,
                                                 sm100::smem_desc(sfb_s + (j * C::kAtoms + a) * 512, 0, 128, 0));
          }
          const uint64_t ad = desc_add(adesc0, (uint32_t)(ab.idx * (C::kABytes >> 4)));
          const uint64_t bd = desc_add(bdesc0, (uint32_t)(ab.idx * (C::kBBytes >> 4)));
#ifdef MRFP4_TRACE
          if (g.debug == 2) {   // load pipeline only: no MMA (commits arrive at once)
          } else
#endif
          if (kb + 1 < num_kb || tail_mmas == 0)
            issue_stage_mmas<VEC, 0, C::kMmas>(el, tmem_base, ad, bd, sfa_t, sfb_t, kb == w.kb0);
          else
            issue_stage_tail<VEC>(tail_mmas, el, tmem_base, ad, bd, sfa_t, sfb_t, kb == w.kb0);
          sm100::tc_commit_2sm_mc_if(el, &empty[ab.idx], 0x3);
          sm100::tc_commit_2sm_mc_if(el, &sf_empty[sf.idx], 0x3);
          stamp(4);
          ab.next<C::kStages>();
          sf.next<C::kSfSlots>();
        }
        sm100::tc_commit_2sm_mc_if(el, tfull, 0x3);
        acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------ epilogue (both CTAs)
    // Warp w reads TMEM lane quadrant w % 4 (hardware rule), columns [h*128, h*128+128).
    // bf16 output: the 128 columns are pulled into registers (as bf16 pairs) and the
    // accumulator is released BEFORE the global stores, so the next tile's MMAs start
    // while this tile's output is being written.
    const int q = warp & 3, h = (warp - C::kEpiWarp0) >> 2;
    pdl_wait();
    const float alpha = __ldg(g.a_ts) * __ldg(g.b_ts);
    qc::EncConsts qk;   // the next layer's encode constants (MXFP4: ts = f32(4/3))
    if constexpr (OUT == kOutNvq) qk = qc::nv_consts_st(g.qp, __ldg(g.q_static_ts));
    if constexpr (is_quant_out(OUT))
      if (blockIdx.x == 0 && warp == C::kEpiWarp0 && lane == 0) *g.q_ts = qk.st32;
    uint32_t acc_phase = 0;
    auto release_acc = [&] {
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) sm100::mbar_arrive(tempty);
        else sm100::mbar_arrive_remote_relaxed(tempty, 0);
      }
    };
    WorkIter it(g, cluster, nclusters);
    Work w;
    while (it.next(g, w)) {
      const int m_blk = w.tile % num_m_blk, n_blk = w.tile / num_m_blk;
      sm100::mbar_wait(tfull, acc_phase);
      sm100::tc_fence_after();
      acc_phase ^= 1;
      const int64_t row = (int64_t)m_blk * 256 + rank * 128 + q * 32 + lane;
      const int64_t col0 = (int64_t)n_blk * 256 + h * 128;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + h * 128;
      if constexpr (OUT == MRFP4_DT_BF16 || is_quant_out(OUT)) {
        uint32_t pkd[64];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          sm100::tmem_ld_32x32b_x32(taddr + c * 32, r);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]) * alpha, __uint_as_float(r[2 * j + 1]) * alpha);
            pkd[16 * c + j] = *reinterpret_cast<uint32_t*>(&b2);
          }
        }
        release_acc();
        if constexpr (is_quant_out(OUT)) {
          if (col0 < g.N) quant_next_row<OUT, HKQ>(g, qk, row, col0, pkd);
          if (!g.d) continue;
        }
        if (row < g.M) {
          const int nd = g.npeer > 0 ? g.npeer : 1;
#pragma unroll 1
          for (int pd = 0; pd < nd; ++pd) {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g.npeer > 0 ? g.peer_d[pd] : g.d) + row * g.ldd + col0;
            // 32-B stores: whole L2 sectors per lane (16-B stores from 32 rows at once were
            // partial-sector writes that stalled the next tile's pipeline by ~5K cycles).
            if ((g.ldd & 15) == 0 && col0 + 128 <= g.N) {
#pragma unroll
              for (int j = 0; j < 8; ++j) st_global_v8(dst + 16 * j, pkd + 8 * j);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (col0 + 8 * j < g.N)
                  *reinterpret_cast<uint4*>(dst + 8 * j) = make_uint4(pkd[4 * j], pkd[4 * j + 1], pkd[4 * j + 2], pkd[4 * j + 3]);
            }
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          sm100::tmem_ld_32x32b_x32(taddr + c * 32, r);
          sm100::tmem_ld_wait();
          if (row < g.M) store_row32<OUT>(g, row, col0 + c * 32, r, alpha);
        }
        release_acc();
      }
    }
  }
  sm100::tc_fence_before();
  __syncwarp();
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_2sm(tmem_base, C::kTmemCols);
  }
}

// ---------------------------------------------------------------- host side
}  // namespace
extern int g_force_grid;
namespace {

PFN_cuTensorMapEncodeTiled_v12000 driver_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor maps are pure functions of their arguments (address, shape, box, swizzle): a launch
// re-using the buffers of an earlier one (every decode step, every layer of a model) gets the
// same 128-B descriptor from this cache instead of re-encoding it on the host.  Bounded
// (cleared past 4096 entries), mutex-guarded.
struct MapKey {
  uint64_t w[20];
  bool operator==(const MapKey& o) const { return memcmp(w, o.w, sizeof(w)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t v : k.w) h = (h ^ v) * 1099511628211ull;
    return (size_t)h;
  }
};

CUresult cached_encode(CUtensorMap* tm, CUtensorMapDataType dt, cuuint32_t rank, void* addr, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* estr,
                       CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                       CUtensorMapFloatOOBfill oob) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  if (rank < 1 || rank > 3) return driver_encode_fn()(tm, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
  MapKey k{};
  k.w[0] = (uint64_t)dt | ((uint64_t)rank << 8) | ((uint64_t)il << 16) | ((uint64_t)sw << 24) | ((uint64_t)l2 << 32) |
           ((uint64_t)oob << 40);
  k.w[1] = reinterpret_cast<uint64_t>(addr);
  for (cuuint32_t i = 0; i < rank; ++i) {
    k.w[2 + i] = dims[i];
    k.w[5 + i] = i + 1 < rank ? strides[i] : 0;
    k.w[8 + i] = box[i];
    k.w[11 + i] = estr[i];
  }
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(k);
    if (it != cache.end()) {
      *tm = it->second;
      return CUDA_SUCCESS;
    }
  }
  const CUresult r = driver_encode_fn()(tm, dt, rank, addr, dims, strides, box, estr, il, sw, l2, oob);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 4096) cache.clear();
    cache.emplace(k, *tm);
  }
  return r;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  return driver_encode_fn() ? &cached_encode : nullptr;
}

}  // namespace
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return get_encode_fn(); }
namespace {

bool make_code_map(CUtensorMap* tm, const uint8_t* ptr, int64_t rows, int64_t K, int box_rows) {
  auto encode = get_encode_fn();
  if (!encode) return false;
  cuuint64_t dims[2] = {(cuuint64_t)(K / 2), (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(K / 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK_BYTES, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Codes [rows, K/2] viewed as [K/256 slices][rows][128 B] (3-D, K % 256 == 0): one box =
// `slices` consecutive 128-B K slices of `box_rows` rows, 128-B swizzled.
bool make_code_map3(CUtensorMap* tm, const uint8_t* ptr, int64_t rows, int64_t K, int box_rows, int slices) {
  auto encode = get_encode_fn();
  if (!encode) return false;
  cuuint64_t dims[3] = {(cuuint64_t)BK_BYTES, (cuuint64_t)rows, (cuuint64_t)(K / BK)};
  cuuint64_t strides[2] = {(cuuint64_t)(K / 2), (cuuint64_t)BK_BYTES};
  cuuint32_t box[3] = {(cuuint32_t)BK_BYTES, (cuuint32_t)box_rows, (cuuint32_t)slices};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Swizzled scale factors [row_blocks][col_blocks atoms of 512 B] viewed as 3-D
// {256 B, 2 * col_blocks half-atoms, row_blocks}: a box {256, 2 * atoms, nrb} is `atoms`
// consecutive K atoms of `nrb` consecutive 128-row blocks (row blocks / atoms past the end
// are zero-filled, and still counted as transaction bytes).
bool make_sf_map(CUtensorMap* tm, const uint8_t* ptr, int64_t row_blocks, int64_t col_blocks, int atoms, int nrb) {
  auto encode = get_encode_fn();
  if (!encode) return false;
  cuuint64_t dims[3] = {256, (cuuint64_t)(2 * col_blocks), (cuuint64_t)row_blocks};
  cuuint64_t strides[2] = {256, (cuuint64_t)(col_blocks * 512)};
  cuuint32_t box[3] = {256, (cuuint32_t)(2 * atoms), (cuuint32_t)nrb};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Split-K plan for `tiles` output tiles of `num_kb` k-blocks: about one unit per SM, at
// least 2 k-blocks per split.
void splitk_plan(int tiles, int num_kb, int* splits, int* kb_per);

int num_sms() { return device_sms(); }

template <int VEC, int BN, int OUT>
int launch(const uint8_t* a, const uint8_t* b, const GemmArgs& args0, cudaStream_t s) {
  using C = Cfg<VEC, BN>;
  static std::atomic<int> attr[kMaxDevices];   // per device: the attribute is per context
  if (per_device_once(attr, [] {
        return cudaFuncSetAttribute(k_gemm_fp4<VEC, BN, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmem) == cudaSuccess ? 1 : -1;
      }) < 0)
    return MRFP4_ECUDA;
  GemmArgs g = args0;
  CUtensorMap tmA, tmB;
  if (!make_code_map(&tmA, a, g.M, g.K, BM) || !make_code_map(&tmB, b, g.N, g.K, BN)) return MRFP4_ECUDA;
  g.num_m_blk = (int)ceil_div(g.M, BM);
  g.num_n_blk = (int)ceil_div(g.N, BN);
  g.num_kb = (int)ceil_div(g.K, BK);
  g.tail_mmas = (int)((g.K % BK) / UMMA_K);
  g.sf_col_blocks = ceil_div(g.K / VEC, 4);
  g.b_row_blocks = ceil_div(g.N, 128);
  const int tiles = g.num_m_blk * g.num_n_blk;
  // Small M (weight-bandwidth bound): split K so every SM streams a slice of the weight.
  g.splits = 1;
  g.kb_per = g.num_kb;
  if (g.ws) {
    int sp = 1, per = g.num_kb;
    splitk_plan(tiles, g.num_kb, &sp, &per);
    if (sp > 1 && g.ws_bytes >= kSplitkHeader + (size_t)sp * g.M * g.N * sizeof(float) &&
        tiles <= (int)(kSplitkHeader / (2 * sizeof(uint32_t))) && tiles * sp <= num_sms() && g_force_grid == 0 && g.N % 4 == 0 &&
        g.ldd % 4 == 0) {
      g.splits = sp;
      g.kb_per = per;
      g.sk_cnt = reinterpret_cast<uint32_t*>(g.ws);
      g.ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(g.ws) + kSplitkHeader);
    }
  }
  const int units = tiles * g.splits;
  int grid = std::min(units, num_sms());
  if (g_force_grid > 0) grid = std::min(grid, g_force_grid);
  // split-K reduces inside the kernel (every split waits for its tile's others): co-residency
  if (launch_pdl(k_gemm_fp4<VEC, BN, OUT>, dim3(grid), dim3(kThreads), C::kSmem, s, g.splits > 1, tmA, tmB, g) !=
      cudaSuccess)
    return MRFP4_ECUDA;
  return MRFP4_OK;
}

template <int VEC, int OUT, int HKQ = 0>
int launch2(const uint8_t* a, const uint8_t* b, const GemmArgs& args0, cudaStream_t s) {
  using C = Cfg2<VEC>;
  static std::atomic<int> attr[kMaxDevices];
  if (per_device_once(attr, [] {
        return cudaFuncSetAttribute(k_gemm_fp4_2sm<VEC, OUT, HKQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::kSmem) == cudaSuccess ? 1 : -1;
      }) < 0)
    return MRFP4_ECUDA;
  GemmArgs g = args0;
  CUtensorMap tmA, tmB, tmSfa, tmSfb;
  const int64_t sfc = g.K / VEC;
  if (!make_code_map3(&tmA, a, g.M, g.K, 128, C::kSlices) || !make_code_map3(&tmB, b, g.N, g.K, 128, C::kSlices) ||
      !make_sf_map(&tmSfa, g.a_sf, ceil_div(g.M, 128), ceil_div(sfc, 4), C::kAtoms, 1) ||
      !make_sf_map(&tmSfb, g.b_sf, ceil_div(g.N, 128), ceil_div(sfc, 4), C::kAtoms, 2))
    return MRFP4_ECUDA;
  g.num_m_blk = (int)ceil_div(g.M, 256);
  g.num_n_blk = (int)ceil_div(g.N, 256);
  g.num_kb = (int)ceil_div(g.K, C::kBK);
  g.tail_mmas = (int)((g.K % C::kBK) / UMMA_K);
  g.sf_col_blocks = ceil_div(sfc, 4);
  g.b_row_blocks = ceil_div(g.N, 128);
  const int tiles = g.num_m_blk * g.num_n_blk;
  int nclu = std::min(tiles, num_sms() / 2);
  if (g_force_grid > 0) nclu = std::min(nclu, std::max(1, g_force_grid / 2));
  return launch_pdl(k_gemm_fp4_2sm<VEC, OUT, HKQ>, dim3(2 * nclu), dim3(C::kThreads2), C::kSmem, s, false, tmA, tmB, tmSfa,
                    tmSfb, g) ==
                 cudaSuccess
             ? MRFP4_OK
             : MRFP4_ECUDA;
}

void splitk_plan(int tiles, int num_kb, int* splits, int* kb_per) {
  int sp = 1;
  static const int min_kb = [] {   // k-blocks per split, at least (MRFP4_SK_MINKB: experiments)
    const char* e = getenv("MRFP4_SK_MINKB");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  if (tiles * 2 <= num_sms()) sp = std::min(std::max(1, num_sms() / tiles), std::max(1, num_kb / min_kb));
  const int per = (int)ceil_div(num_kb, sp);
  *kb_per = per;
  *splits = (int)ceil_div(num_kb, per);
}

}  // namespace

// Workspace bytes mrfp4_gemm uses for split-K at this shape (0 when it does not split).
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const bool pair = (K % 256 == 0) && M > 128;
  if (pair) {
    return 0;
  }
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, 256));
  int sp = 1, per = 1;
  splitk_plan(tiles, (int)ceil_div(K, BK), &sp, &per);
  return sp > 1 ? kSplitkHeader + (size_t)sp * M * N * sizeof(float) : 0;
}

int g_debug_mode = 0;
unsigned long long* g_debug_buf = nullptr;
int g_force_grid = 0;
int g_force_kernel = 0;  // 0 auto, 1 = 1-CTA kernel, 2 = 2-CTA kernel
int g_preissue = 1;

int launch_gemm_fp4(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
                    const float* b_ts, void* d, int d_dtype, int64_t M, int64_t N, int64_t K, int64_t ldd, int fmt,
                    void* ws, size_t ws_bytes, cudaStream_t s) {
  GemmArgs g{};
  g.b = b;
  g.preissue = g_preissue;
  g.ws = static_cast<float*>(ws);
  g.ws_bytes = ws_bytes;
  g.debug = g_debug_mode;
  g.dbg = g_debug_buf;
  g.a_sf = a_sf;
  g.b_sf = b_sf;
  g.a_ts = a_ts;
  g.b_ts = b_ts;
  g.d = d;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldd = ldd;
  // The 2-CTA kernel streams 512-wide K stages as 3-D boxes of 128-B slices: K % 256 == 0.
  const bool pair = (K % 256 == 0) && (g_force_kernel ? g_force_kernel == 2 : M > 128);
  if (pair) {
    if (fmt == MRFP4_FMT_NVFP4)
      return d_dtype == MRFP4_DT_BF16 ? launch2<16, MRFP4_DT_BF16>(a, b, g, s) : launch2<16, MRFP4_DT_F32>(a, b, g, s);
    return d_dtype == MRFP4_DT_BF16 ? launch2<32, MRFP4_DT_BF16>(a, b, g, s) : launch2<32, MRFP4_DT_F32>(a, b, g, s);
  }
  if (fmt == MRFP4_FMT_NVFP4) {
    return d_dtype == MRFP4_DT_BF16 ? launch<16, 256, MRFP4_DT_BF16>(a, b, g, s)
                                    : launch<16, 256, MRFP4_DT_F32>(a, b, g, s);
  }
  return d_dtype == MRFP4_DT_BF16 ? launch<32, 256, MRFP4_DT_BF16>(a, b, g, s)
                                  : launch<32, 256, MRFP4_DT_F32>(a, b, g, s);
}

// K2 storing its bf16 output straight into several (peer) output buffers: the all-gather
// of the N-sharded linear fused into the epilogue (2-CTA kernel only).
int launch_gemm_peers(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                      const uint8_t* b_sf, const float* b_ts, void* const* dsts, int ndst, int64_t M, int64_t N,
                      int64_t K, int64_t ldd, int fmt, cudaStream_t s) {
  GemmArgs g{};
  g.b = b;
  g.preissue = g_preissue;
  g.a_sf = a_sf;
  g.b_sf = b_sf;
  g.a_ts = a_ts;
  g.b_ts = b_ts;
  g.d = dsts[0];
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldd = ldd;
  g.npeer = ndst;
  for (int i = 0; i < ndst; ++i) g.peer_d[i] = dsts[i];
  return fmt == MRFP4_FMT_NVFP4 ? launch2<16, MRFP4_DT_BF16>(a, b, g, s) : launch2<32, MRFP4_DT_BF16>(a, b, g, s);
}

// K2 with the next layer's act-quant fused into the epilogue (2-CTA kernel only): MXFP4, or
// NVFP4 against a given global scale (next_static_ts).
int launch_gemm_quant_next(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                           const uint8_t* b_sf, const float* b_ts, void* y, int64_t ldy, int64_t M, int64_t N,
                           int64_t K, int fmt, int next_fmt, int next_hk, const float* next_static_ts,
                           uint8_t* q_codes, uint8_t* q_sf, float* q_ts, uint32_t* q_status, cudaStream_t s) {
  GemmArgs g{};
  g.b = b;
  g.preissue = g_preissue;
  g.a_sf = a_sf;
  g.b_sf = b_sf;
  g.a_ts = a_ts;
  g.b_ts = b_ts;
  g.d = y;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldd = y ? ldy : N;
  g.q_codes = q_codes;
  g.q_sf = q_sf;
  g.q_ts = q_ts;
  g.q_status = q_status;
  g.q_static_ts = next_static_ts;
  g.q_cb = (uint32_t)(N / (next_fmt == MRFP4_FMT_NVFP4 ? 64 : 128));
  g.q_rows_pad = ceil_div(M, 128) * 128;
  const double c64 = next_hk ? 1.0 / std::sqrt((double)next_hk) : 1.0;
  g.qp.c64 = c64;
  g.qp.kraw = (float)(c64 / 6.0);
  g.qp.kmx = (float)(c64 / (double)1.33333337306976318359375f);
  const float pm[2] = {1.f, -1.f};
  memcpy(&g.qp.pm, pm, sizeof(pm));
  auto go = [&](auto vec_tag, auto out_tag) {
    constexpr int V = decltype(vec_tag)::value, O = decltype(out_tag)::value;
    switch (next_hk) {
      case 16: return launch2<V, O, 16>(a, b, g, s);
      case 32: return launch2<V, O, 32>(a, b, g, s);
      case 64: return launch2<V, O, 64>(a, b, g, s);
      case 128: return launch2<V, O, 128>(a, b, g, s);
      default: return launch2<V, O, 0>(a, b, g, s);
    }
  };
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  using Mx = std::integral_constant<int, kOutMxq>;
  using Nv = std::integral_constant<int, kOutNvq>;
  if (next_fmt == MRFP4_FMT_NVFP4)
    return fmt == MRFP4_FMT_NVFP4 ? go(I16{}, Nv{}) : go(I32{}, Nv{});
  return fmt == MRFP4_FMT_NVFP4 ? go(I16{}, Mx{}) : go(I32{}, Mx{});
}

}  // namespace mrfp4

// Perf experiments only (deliberately not in include/mrfp4.h): 1 = skip operand loads, 2 = skip MMAs.
extern "C" void mrfp4_debug_gemm_grid(int g) { mrfp4::g_force_grid = g; }

extern "C" void mrfp4_debug_gemm_timestamps(unsigned long long* dev_buf) { mrfp4::g_debug_buf = dev_buf; }

extern "C" void mrfp4_debug_gemm_preissue(int on) { mrfp4::g_preissue = on; }

extern "C" int mrfp4_debug_gemm_kernel(int which) {
  const int old = mrfp4::g_force_kernel;
  mrfp4::g_force_kernel = which;
  return old;
}

extern "C" int mrfp4_debug_gemm_mode(int mode) {
  const int old = mrfp4::g_debug_mode;
  mrfp4::g_debug_mode = mode;
  return old;
}
