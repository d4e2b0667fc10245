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
#include <mutex>

#include "common.cuh"
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
  unsigned long long* dbg;  // perf experiments: per-k-block MMA-thread timestamps of CTA 0
  int debug;  // perf experiments: 1 = no operand loads, 2 = no MMAs (0 in production)
};



// Issue the NK tcgen05.mma of one k-block (compile-time count: no runtime control flow
// in the issue path -- a data-dependent loop bound here measurably slows issue).
template <int VEC, int NK, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_kblock(uint32_t d_tmem, uint32_t a_s, uint32_t b_s, uint32_t sfa_t, uint32_t sfb_t,
                                             bool first) {
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int atom = VEC == 16 ? k : (k >> 1);
    const uint32_t sfid = VEC == 16 ? 0u : (uint32_t)(k & 1) * 2u;
    const uint64_t adesc = sm100::smem_desc(a_s + k * (UMMA_K / 2), 16, 1024, 2);
    const uint64_t bdesc = sm100::smem_desc(b_s + k * (UMMA_K / 2), 16, 1024, 2);
    const uint32_t idesc = sm100::idesc_fp4(M, N, VEC == 32, sfid, sfid);
    const uint32_t acc = (first && k == 0) ? 0u : 1u;
    if constexpr (PAIR)
      sm100::tc_mma_fp4_2sm<VEC>(d_tmem, adesc, bdesc, idesc, (sfa_t + atom * 4) | (sfid << 30),
                                 (sfb_t + atom * kNB * 4) | (sfid << 30), acc);
    else
      sm100::tc_mma_fp4<VEC>(d_tmem, adesc, bdesc, idesc, (sfa_t + atom * 4) | (sfid << 30),
                             (sfb_t + atom * kNB * 4) | (sfid << 30), acc);
  }
}

// MMAs k in [K0, K1) of a k-block (K0 > 0: always accumulate).
template <int VEC, int K0, int K1, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_kblock_from(uint32_t d_tmem, uint32_t a_s, uint32_t b_s, uint32_t sfa_t,
                                                  uint32_t sfb_t, bool first) {
#pragma unroll
  for (int k = K0; k < K1; ++k) {
    const int atom = VEC == 16 ? k : (k >> 1);
    const uint32_t sfid = VEC == 16 ? 0u : (uint32_t)(k & 1) * 2u;
    const uint64_t adesc = sm100::smem_desc(a_s + k * (UMMA_K / 2), 16, 1024, 2);
    const uint64_t bdesc = sm100::smem_desc(b_s + k * (UMMA_K / 2), 16, 1024, 2);
    const uint32_t idesc = sm100::idesc_fp4(M, N, VEC == 32, sfid, sfid);
    const uint32_t acc = (first && k == 0) ? 0u : 1u;
    if constexpr (PAIR)
      sm100::tc_mma_fp4_2sm<VEC>(d_tmem, adesc, bdesc, idesc, (sfa_t + atom * 4) | (sfid << 30),
                                 (sfb_t + atom * kNB * 4) | (sfid << 30), acc);
    else
      sm100::tc_mma_fp4<VEC>(d_tmem, adesc, bdesc, idesc, (sfa_t + atom * 4) | (sfid << 30),
                             (sfb_t + atom * kNB * 4) | (sfid << 30), acc);
  }
}

template <int VEC, int M, int N, int kNB, bool PAIR>
__device__ __forceinline__ void issue_kblock_any(int nk, uint32_t d_tmem, uint32_t a_s, uint32_t b_s, uint32_t sfa_t,
                                                 uint32_t sfb_t, bool first) {
  switch (nk) {
    case 4: issue_kblock<VEC, 4, M, N, kNB, PAIR>(d_tmem, a_s, b_s, sfa_t, sfb_t, first); break;
    case 3: issue_kblock<VEC, 3, M, N, kNB, PAIR>(d_tmem, a_s, b_s, sfa_t, sfb_t, first); break;
    case 2: issue_kblock<VEC, 2, M, N, kNB, PAIR>(d_tmem, a_s, b_s, sfa_t, sfb_t, first); break;
    case 1: issue_kblock<VEC, 1, M, N, kNB, PAIR>(d_tmem, a_s, b_s, sfa_t, sfb_t, first); break;
    default: break;
  }
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
  pdl_trigger();

  const int num_tiles = g.num_m_blk * g.num_n_blk;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      pdl_wait();  // A, its scale factors and tensor scale come from the act-quant kernel
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile % g.num_m_blk, n_blk = tile / g.num_m_blk;
        for (int kb = 0; kb < g.num_kb; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          const int atoms = (int)imin64(C::kAtomsPerKb, g.sf_col_blocks - (int64_t)kb * C::kAtomsPerKb);
          int nbv = 0;
#pragma unroll
          for (int j = 0; j < C::kNB; ++j) nbv += ((int64_t)n_blk * C::kNB + j < g.b_row_blocks);
          const uint32_t bytes = C::kABytes + C::kBBytes + (uint32_t)atoms * 512u * (1u + nbv);
          if (g.debug == 1 || g.debug == 3 || g.debug == 4 || g.debug == 5) {
            sm100::mbar_arrive(&full[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          sm100::mbar_arrive_expect_tx(&full[stage], bytes);
          sm100::tma_load_2d(smem + C::kOffA + stage * C::kABytes, &tmA, &full[stage], kb * BK_BYTES, m_blk * BM);
          sm100::tma_load_2d(smem + C::kOffB + stage * C::kBBytes, &tmB, &full[stage], kb * BK_BYTES, n_blk * BN);
          const int64_t katom = (int64_t)kb * C::kAtomsPerKb;
          sm100::bulk_load(smem + C::kOffSfa + stage * C::kSfaBytes,
                           g.a_sf + ((int64_t)m_blk * g.sf_col_blocks + katom) * 512, atoms * 512u, &full[stage]);
#pragma unroll
          for (int j = 0; j < C::kNB; ++j) {
            const int64_t rb = (int64_t)n_blk * C::kNB + j;
            if (rb < g.b_row_blocks)
              sm100::bulk_load(smem + C::kOffSfb + stage * C::kSfbBytes + j * C::kAtomsPerKb * 512,
                               g.b_sf + (rb * g.sf_col_blocks + katom) * 512, atoms * 512u, &full[stage]);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        sm100::mbar_wait(tempty, acc_phase ^ 1);
        sm100::tc_fence_after();
        for (int kb = 0; kb < g.num_kb; ++kb) {
          if (g.dbg && blockIdx.x == 0 && tile == 0 && kb < 64) g.dbg[2 * kb] = clock64();
          sm100::mbar_wait(&full[stage], phase);
          if (g.dbg && blockIdx.x == 0 && tile == 0 && kb < 64) g.dbg[2 * kb + 1] = clock64();
          sm100::tc_fence_after();
          const uint32_t sfa_t = tmem_base + C::kAccCols + stage * (C::kSfaCols + C::kSfbCols);
          const uint32_t sfb_t = sfa_t + C::kSfaCols;
          const uint32_t sfa_s = sm100::smem_u32(smem + C::kOffSfa + stage * C::kSfaBytes);
          const uint32_t sfb_s = sm100::smem_u32(smem + C::kOffSfb + stage * C::kSfbBytes);
#pragma unroll
          for (int a = 0; a < C::kAtomsPerKb; ++a) {
            if (g.debug < 5 || (g.debug == 6 && kb < C::kStages)) {
              sm100::tc_cp_32x128b_warpx4(sfa_t + a * 4, sm100::smem_desc(sfa_s + a * 512, 0, 128, 0));
#pragma unroll
              for (int j = 0; j < C::kNB; ++j)
                sm100::tc_cp_32x128b_warpx4(sfb_t + a * C::kNB * 4 + j * 4,
                                            sm100::smem_desc(sfb_s + (j * C::kAtomsPerKb + a) * 512, 0, 128, 0));
            }
          }
          const uint32_t a_s = sm100::smem_u32(smem + C::kOffA + stage * C::kABytes);
          const uint32_t b_s = sm100::smem_u32(smem + C::kOffB + stage * C::kBBytes);
          if (g.debug == 2 || g.debug == 4) {
          } else if (kb + 1 < g.num_kb || g.tail_mmas == 0) {
            issue_kblock<VEC, BK / UMMA_K, BM, BN, C::kNB, false>(tmem_base, a_s, b_s, sfa_t, sfb_t, kb == 0);
          } else {
            issue_kblock_any<VEC, BM, BN, C::kNB, false>(g.tail_mmas, tmem_base, a_s, b_s, sfa_t, sfb_t, kb == 0);
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
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % g.num_m_blk, n_blk = tile / g.num_m_blk;
      sm100::mbar_wait(tfull, acc_phase);
      sm100::tc_fence_after();
      const int64_t row = (int64_t)m_blk * BM + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < ((g.debug >= 3 && g.debug <= 5) ? 0 : BN); c += 32) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + c, r);
        sm100::tmem_ld_wait();
        const int64_t col = (int64_t)n_blk * BN + c;
        if (row < g.M) store_row32<OUT>(g, row, col, r, alpha);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}


// ---------------------------------------------------------------------------
// 2-CTA (cta_group::2) kernel: a CTA pair computes a 256 x 256 output tile.
//   warp 0      TMA producer (both CTAs): own 128 rows of A and of B (cta_group::2
//               loads counted on the leader's `full` barrier) and this CTA's scale
//               factors (SFA for its 128 rows, SFB for all 256 rows) on its own `sf_full`
//   warp 1      TMEM allocator (both) + MMA issuer (leader, one thread):
//               tcgen05.mma.cta_group::2 M=256 N=256 K=64, commit multicast to both CTAs
//   warps 2-5   scale-factor stagers (per CTA, one per TMEM lane quadrant): SMEM -> regs
//               -> tcgen05.st into the stage's TMEM slot, then arrive on the leader's
//               leader's `full` barrier.  (tcgen05.cp costs ~86 tensor-pipe cycles per 512-B
//               atom -- 60-120% of the MMA time -- so the copy is moved off the pipe.)
//   warps 6-9   epilogue (per CTA): TMEM -> regs -> * ts_A*ts_W -> bf16/f32 -> global
// ---------------------------------------------------------------------------
template <int VEC>
struct Cfg2 {
  static constexpr int kAtomsPerKb = BK / VEC / 4;           // SF atoms (128 rows x 4 cols) per k-block
  static constexpr int kStages = VEC == 16 ? 5 : 6;
  static constexpr int kABytes = 128 * BK_BYTES;
  static constexpr int kBBytes = 128 * BK_BYTES;
  static constexpr int kSfaBytes = kAtomsPerKb * 512;
  static constexpr int kSfbBytes = 2 * kAtomsPerKb * 512;
  static constexpr int kSfaCols = kAtomsPerKb * 4;
  static constexpr int kSfbCols = 2 * kAtomsPerKb * 4;
  static constexpr int kSfCols = kSfaCols + kSfbCols;          // TMEM columns per stage slot
  static constexpr int kAccCols = 256;
  static constexpr int kTmemCols = 512;
  static_assert(kAccCols + kStages * kSfCols <= kTmemCols, "TMEM budget");
  static constexpr int kOffA = 0;
  static constexpr int kOffB = kOffA + kStages * kABytes;
  static constexpr int kOffSfa = kOffB + kStages * kBBytes;
  static constexpr int kOffSfb = kOffSfa + kStages * kSfaBytes;
  static constexpr int kOffBar = kOffSfb + kStages * kSfbBytes;
  static constexpr int kSmem = kOffBar + 512 + 1024;
  static constexpr int kThreads2 = 320;
};

template <int VEC, int OUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    k_gemm_fp4_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB, GemmArgs g) {
  using C = Cfg2<VEC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // full[s] (leader's): both CTAs' A/B bytes landed AND both CTAs' scale factors staged in TMEM
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty = full + C::kStages;                               // stage free (MMA committed)
  uint64_t* sf_full = empty + C::kStages;                            // this CTA's SF landed in SMEM
  uint64_t* tfull = sf_full + C::kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Kernel parameters into registers once (asm "memory" clobbers would force reloads).
  const int num_m_blk = g.num_m_blk, num_n_blk = g.num_n_blk, num_kb = g.num_kb, tail_mmas = g.tail_mmas;
  const int num_tiles = num_m_blk * num_n_blk;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int64_t sf_col_blocks = g.sf_col_blocks, b_row_blocks = g.b_row_blocks, a_row_blocks = (g.M + 127) / 128;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmSFA);
    sm100::tma_prefetch_desc(&tmSFB);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 9);      // leader producer (A/B bytes) + 4 stager warps x 2 CTAs
      sm100::mbar_init(&empty[s], 1);
      sm100::mbar_init(&sf_full[s], 1);
    }
    sm100::mbar_init(tfull, 1);
    sm100::mbar_init(tempty, 8);          // 4 epilogue warps x 2 CTAs
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
      pdl_wait();  // A, its scale factors and tensor scale come from the act-quant kernel
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters) {
        const int m_blk = tile % num_m_blk, n_blk = tile / num_m_blk;
        for (int kb = 0; kb < num_kb; ++kb) {
          unsigned long long* dbg = (g.dbg && blockIdx.x == 0 && tile == cluster && kb < 32) ? g.dbg + 256 + 2 * kb : nullptr;
          if (dbg) dbg[0] = clock64();
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (dbg) dbg[1] = clock64();
          {
            // Scale factors: contiguous 512-B atoms per 128-row block -> 1-D bulk copies
            // (K tail: copy only the atoms that exist; the rest of the slot is never read
            // by an issued MMA).  Row blocks past the end of A / B are skipped.
            const int64_t katom = (int64_t)kb * C::kAtomsPerKb;
            const uint32_t nat = (uint32_t)imin64(C::kAtomsPerKb, sf_col_blocks - katom) * 512u;
            const int64_t ra = (int64_t)m_blk * 2 + rank;
            const int64_t rb0 = (int64_t)n_blk * 2;
            const uint32_t bytes = (ra < a_row_blocks ? nat : 0u) + (rb0 < b_row_blocks ? nat : 0u) +
                                   (rb0 + 1 < b_row_blocks ? nat : 0u);
            sm100::mbar_arrive_expect_tx(&sf_full[stage], bytes);
            if (ra < a_row_blocks)
              sm100::bulk_load(smem + C::kOffSfa + stage * C::kSfaBytes, g.a_sf + (ra * sf_col_blocks + katom) * 512,
                               nat, &sf_full[stage]);
#pragma unroll
            for (int j = 0; j < 2; ++j)
              if (rb0 + j < b_row_blocks)
                sm100::bulk_load(smem + C::kOffSfb + stage * C::kSfbBytes + j * C::kSfaBytes,
                                 g.b_sf + ((rb0 + j) * sf_col_blocks + katom) * 512, nat, &sf_full[stage]);
          }
          if (leader) sm100::mbar_arrive_expect_tx(&full[stage], 2u * (C::kABytes + C::kBBytes));
          const uint32_t lb = sm100::leader_bar(&full[stage]);
          sm100::tma_load_2d_2sm(smem + C::kOffA + stage * C::kABytes, &tmA, lb, kb * BK_BYTES,
                                 m_blk * 256 + (int)rank * 128);
          sm100::tma_load_2d_2sm(smem + C::kOffB + stage * C::kBBytes, &tmB, lb, kb * BK_BYTES,
                                 n_blk * 256 + (int)rank * 128);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      int ntl = 0;
      for (int tile = cluster; tile < num_tiles; tile += nclusters, ++ntl) {
        if (g.dbg && blockIdx.x == 0 && ntl < 4) {
          uint64_t gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          g.dbg[400 + 4 * ntl] = clock64(); g.dbg[401 + 4 * ntl] = gt;
        }
        sm100::mbar_wait(tempty, acc_phase ^ 1);
        if (g.dbg && blockIdx.x == 0 && ntl < 4) g.dbg[402 + 4 * ntl] = clock64();
        sm100::tc_fence_after();
        sm100::mbar_wait(&full[stage], phase);
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::tc_fence_after();
          const uint32_t sfa_t = tmem_base + C::kAccCols + stage * C::kSfCols;
          const uint32_t sfb_t = sfa_t + C::kSfaCols;
          const uint32_t a_s = sm100::smem_u32(smem + C::kOffA + stage * C::kABytes);
          const uint32_t b_s = sm100::smem_u32(smem + C::kOffB + stage * C::kBBytes);
          const int cur = stage;
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          if (kb + 1 < num_kb) {
            // Issue 3 MMAs, then wait for the next stage while they execute (keeps the
            // shallow tcgen05 issue queue non-empty across the barrier wait).
            issue_kblock<VEC, 3, 256, 256, 2, true>(tmem_base, a_s, b_s, sfa_t, sfb_t, kb == 0);
            sm100::mbar_wait(&full[stage], phase);
            issue_kblock_from<VEC, 3, 4, 256, 256, 2, true>(tmem_base, a_s, b_s, sfa_t, sfb_t, false);
          } else if (tail_mmas == 0) {
            issue_kblock<VEC, BK / UMMA_K, 256, 256, 2, true>(tmem_base, a_s, b_s, sfa_t, sfb_t, kb == 0);
          } else {
            issue_kblock_any<VEC, 256, 256, 2, true>(tail_mmas, tmem_base, a_s, b_s, sfa_t, sfb_t, kb == 0);
          }
          sm100::tc_commit_2sm_mc(&empty[cur], 0x3);
        }
        sm100::tc_commit_2sm_mc(tfull, 0x3);
        if (g.dbg && blockIdx.x == 0 && ntl < 4) g.dbg[403 + 4 * ntl] = clock64();
        acc_phase ^= 1;
      }
      if (g.dbg && blockIdx.x == 0) {
        uint64_t gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g.dbg[420] = clock64(); g.dbg[421] = gt; g.dbg[422] = ntl;
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------ scale-factor stagers (both CTAs)
    // TMEM slot layout (replicated over the 4 lane quadrants, as tcgen05.cp.warpx4
    // would produce): lane 32q+l, column c+j of a 128-row atom holds the 4 scale
    // codes of row l+32j -- i.e. bytes [16l, 16l+16) of the 512-B SMEM atom.
    const int q = warp & 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      for (int kb = 0; kb < num_kb; ++kb) {
        unsigned long long* dbg = (g.dbg && blockIdx.x == 0 && q == 0 && lane == 0 && tile == cluster && kb < 32) ? g.dbg + 128 + 4 * kb : nullptr;
        if (dbg) dbg[0] = clock64();
        sm100::mbar_wait(&sf_full[stage], phase);
        if (dbg) dbg[1] = clock64();
        const uint8_t* sa = smem + C::kOffSfa + stage * C::kSfaBytes + lane * 16;
        const uint8_t* sb = smem + C::kOffSfb + stage * C::kSfbBytes + lane * 16;
        uint32_t ra[C::kSfaCols], rb[C::kSfbCols];
#pragma unroll
        for (int a = 0; a < C::kAtomsPerKb; ++a) {
          const uint4 va = *reinterpret_cast<const uint4*>(sa + a * 512);
          ra[4 * a + 0] = va.x; ra[4 * a + 1] = va.y; ra[4 * a + 2] = va.z; ra[4 * a + 3] = va.w;
#pragma unroll
          for (int j = 0; j < 2; ++j) {  // TMEM order: atom-major, then 128-row block
            const uint4 vb = *reinterpret_cast<const uint4*>(sb + (j * C::kAtomsPerKb + a) * 512);
            rb[8 * a + 4 * j + 0] = vb.x; rb[8 * a + 4 * j + 1] = vb.y;
            rb[8 * a + 4 * j + 2] = vb.z; rb[8 * a + 4 * j + 3] = vb.w;
          }
        }
        const uint32_t t0 = tmem_base + ((uint32_t)(q * 32) << 16) + C::kAccCols + stage * C::kSfCols;
        sm100::tmem_st_32x32b<C::kSfaCols>(t0, ra);
        if constexpr (C::kSfbCols == 32) {
          sm100::tmem_st_32x32b<16>(t0 + C::kSfaCols, rb);
          sm100::tmem_st_32x32b<16>(t0 + C::kSfaCols + 16, rb + 16);
        } else {
          sm100::tmem_st_32x32b<C::kSfbCols>(t0 + C::kSfaCols, rb);
        }
        if (dbg) dbg[2] = clock64();
        sm100::tmem_st_wait();
        if (dbg) dbg[3] = clock64();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) sm100::mbar_arrive(&full[stage]);
          else sm100::mbar_arrive_remote(&full[stage], 0);
        }
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    pdl_wait();
    const float alpha = __ldg(g.a_ts) * __ldg(g.b_ts);
    uint32_t acc_phase = 0;
    for (int tile = cluster; tile < num_tiles; tile += nclusters) {
      const int m_blk = tile % num_m_blk, n_blk = tile / num_m_blk;
      sm100::mbar_wait(tfull, acc_phase);
      sm100::tc_fence_after();
      const int64_t row = (int64_t)m_blk * 256 + rank * 128 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + c, r);
        sm100::tmem_ld_wait();
        const int64_t col = (int64_t)n_blk * 256 + c;
        if (row < g.M) store_row32<OUT>(g, row, col, r, alpha);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) sm100::mbar_arrive(tempty);
        else sm100::mbar_arrive_remote(tempty, 0);
      }
      acc_phase ^= 1;
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

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
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

// Swizzled scale factors viewed as [128-row blocks][col_blocks * 64] uint64 (one 512-B atom = 64 x u64).
bool make_sf_map(CUtensorMap* tm, const uint8_t* sf, int64_t rows, int64_t sf_cols, int atoms, int box_rows) {
  auto encode = get_encode_fn();
  if (!encode) return false;
  const int64_t rb = ceil_div(rows, 128), cb = ceil_div(sf_cols, 4);
  cuuint64_t dims[2] = {(cuuint64_t)(cb * 64), (cuuint64_t)rb};
  cuuint64_t strides[1] = {(cuuint64_t)(cb * 512)};
  cuuint32_t box[2] = {(cuuint32_t)(atoms * 64), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(sf), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int VEC, int BN, int OUT>
int launch(const uint8_t* a, const uint8_t* b, const GemmArgs& args0, cudaStream_t s) {
  using C = Cfg<VEC, BN>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_gemm_fp4<VEC, BN, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return MRFP4_ECUDA;
    attr_set = true;
  }
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
  int grid = std::min(tiles, num_sms());
  if (g_force_grid > 0) grid = std::min(grid, g_force_grid);
  return launch_pdl(k_gemm_fp4<VEC, BN, OUT>, dim3(grid), dim3(kThreads), C::kSmem, s, tmA, tmB, g) == cudaSuccess
             ? MRFP4_OK
             : MRFP4_ECUDA;
}

template <int VEC, int OUT>
int launch2(const uint8_t* a, const uint8_t* b, const GemmArgs& args0, cudaStream_t s) {
  using C = Cfg2<VEC>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(k_gemm_fp4_2sm<VEC, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
        cudaSuccess)
      return MRFP4_ECUDA;
    attr_set = true;
  }
  GemmArgs g = args0;
  CUtensorMap tmA, tmB, tmSFA, tmSFB;
  const int64_t sfc = g.K / VEC;
  if (!make_code_map(&tmA, a, g.M, g.K, 128) || !make_code_map(&tmB, b, g.N, g.K, 128) ||
      !make_sf_map(&tmSFA, g.a_sf, g.M, sfc, C::kAtomsPerKb, 1) ||
      !make_sf_map(&tmSFB, g.b_sf, g.N, sfc, C::kAtomsPerKb, 2))
    return MRFP4_ECUDA;
  g.num_m_blk = (int)ceil_div(g.M, 256);
  g.num_n_blk = (int)ceil_div(g.N, 256);
  g.num_kb = (int)ceil_div(g.K, BK);
  g.tail_mmas = (int)((g.K % BK) / UMMA_K);
  g.sf_col_blocks = ceil_div(sfc, 4);
  g.b_row_blocks = ceil_div(g.N, 128);
  const int tiles = g.num_m_blk * g.num_n_blk;
  const int clusters = std::min(tiles, num_sms() / 2);
  int nclu = clusters;
  if (g_force_grid > 0) nclu = std::min(nclu, std::max(1, g_force_grid / 2));
  return launch_pdl(k_gemm_fp4_2sm<VEC, OUT>, dim3(2 * nclu), dim3(C::kThreads2), C::kSmem, s, tmA, tmB, tmSFA,
                    tmSFB, g) == cudaSuccess
             ? MRFP4_OK
             : MRFP4_ECUDA;
}

}  // namespace

int g_debug_mode = 0;
unsigned long long* g_debug_buf = nullptr;
int g_force_grid = 0;
int g_force_kernel = 0;  // 0 auto, 1 = 1-CTA kernel, 2 = 2-CTA kernel

int launch_gemm_fp4(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
                    const float* b_ts, void* d, int d_dtype, int64_t M, int64_t N, int64_t K, int64_t ldd, int fmt,
                    cudaStream_t s) {
  GemmArgs g{};
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
  const bool pair = g_force_kernel ? g_force_kernel == 2 : M > 128;
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

}  // namespace mrfp4

// Perf experiments only (deliberately not in include/mrfp4.h): 1 = skip operand loads, 2 = skip MMAs.
extern "C" void mrfp4_debug_gemm_grid(int g) { mrfp4::g_force_grid = g; }

extern "C" void mrfp4_debug_gemm_timestamps(unsigned long long* dev_buf) { mrfp4::g_debug_buf = dev_buf; }

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
