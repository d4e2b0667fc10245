/*
 * mrfp4.h -- C ABI of libmrfp4.so, the B200 (sm_100a) MR-GPTQ FP4 quantized-linear path.
 *
 * The reference (microfp 0.1.0, /root/reference/pkg/src/microfp) exposes this hot path
 * as a Python API, not an FFI.  Each entry point below replaces one reference call
 * (paths relative to /root/reference):
 *
 *   mrfp4_act_quant     quantize_rtn(X, FormatSpec.mxfp4()|nvfp4(), transform=TransformSpec.hadamard(k))
 *                       pkg/src/microfp/quantizers.py:247-255 (with transforms.py:77-91,
 *                       quantizers.py:170-215, formats.py:94-113/220-251/393-416)
 *   mrfp4_sf_swizzle    MfpTensor.scale_codes (row-major, formats.py:314-316, :327) ->
 *                       tensor-core scale layout; used by weight prep (MfpTensor -> device)
 *   mrfp4_sf_unswizzle  inverse, to hand results back as a reference MfpTensor
 *   mrfp4_gemm          dequantize(Aq) @ dequantize(Wq).T  (formats.py:424-442)
 *   mrfp4_dequantize    dequantize(t) (formats.py:424-442) on the device, for checks
 *
 * Conventions
 *   - All buffers are device pointers allocated by the caller; the library never
 *     allocates on the hot path.  `stream` is a cudaStream_t (NULL = legacy default).
 *   - Calls are stream-ordered and thread-safe.  Host-side argument checks return
 *     a status synchronously; data errors found on the device (non-finite input,
 *     NVFP4 E4M3 scale underflow -- both DataError in the reference,
 *     quantizers.py:99-100, formats.py:101-102) are OR-ed into the caller's
 *     device `status` word as MRFP4_STATUS_* bits.
 *   - mrfp4_last_error() returns a thread-local message for the last failing call.
 *
 * Layouts
 *   codes : uint8 [rows, K/2], row-major, element 2j in the low nibble of byte j
 *           (identical to MfpTensor.codes, formats.py:377-382).
 *   sf    : uint8, swizzled 128x4-atom layout, size mrfp4_sf_bytes(rows, K/G);
 *           offset(r,c) = ((r/128)*ceil(C/4) + c/4)*512 + (r%32)*16 + ((r/32)%4)*4 + c%4,
 *           padding rows/columns are zero.
 *   MXFP4 : G = 32, E8M0 scale codes, tensor scale f32(4/3)      (formats.py:302-303)
 *   NVFP4 : G = 16, E4M3 scale codes, whole-tensor global scale   (formats.py:306-307)
 */
#ifndef MRFP4_H_
#define MRFP4_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRFP4_ABI_VERSION 3

/* return codes */
#define MRFP4_OK 0
#define MRFP4_EINVAL 1         /* bad shape / argument      -> DataError  */
#define MRFP4_EUNSUPPORTED 2   /* unsupported configuration -> DataError  */
#define MRFP4_ECUDA 3          /* CUDA launch/runtime error -> RuntimeError */

/* formats */
#define MRFP4_FMT_MXFP4 0
#define MRFP4_FMT_NVFP4 1

/* element dtypes (inputs / outputs) */
#define MRFP4_DT_BF16 0
#define MRFP4_DT_F16 1
#define MRFP4_DT_F32 2
#define MRFP4_DT_F64 3   /* mrfp4_rotate_f64 only (the reference's own float64 inputs) */

/* device status bits */
#define MRFP4_STATUS_NONFINITE 1u        /* NaN/Inf in the input (quantizers.py:99-100) */
#define MRFP4_STATUS_SCALE_UNDERFLOW 2u  /* NVFP4 group scale code 0 -> eff = 0 (formats.py:101-102) */

int mrfp4_abi_version(void);
const char* mrfp4_last_error(void);

/* Group size of a format (32 or 16), or 0 for an unknown format. */
int mrfp4_group_size(int fmt);

/* Bytes of a swizzled scale-factor buffer for a [rows, sf_cols] scale matrix. */
size_t mrfp4_sf_bytes(int64_t rows, int64_t sf_cols);

/* Device workspace needed by mrfp4_act_quant (NVFP4: 16 bytes -- the tensor max and the
 * counters of the in-kernel grid barrier).  It must be zero-filled once before first use;
 * every successful call leaves it re-armed, so one workspace serves a stream's calls in
 * order (not concurrent calls). */
size_t mrfp4_act_quant_workspace(int64_t M, int64_t K, int fmt);

/*
 * Fused online activation quantization (K1): y = X (.) blockdiag(H_k/sqrt(k)) ->
 * group absmax -> scale codes written straight into the swizzled layout ->
 * E2M1 codes, 2 per byte.  had_k in {0 (no rotation), 16, 32, 64, 128}.
 * x: [M, K] with row stride ldx elements (ldx*elt_size % 16 == 0), dtype x_dtype.
 * tensor_scale: device float, receives f32(4/3) (MXFP4) or the NVFP4 global scale.
 * NVFP4 runs both passes (whole-tensor max, then encode) in one persistent launch with a
 * grid barrier.
 * Kernels are launched with programmatic dependent launch (PDL); set MRFP4_PDL=0 in
 * the environment to launch them with plain stream ordering.
 */
int mrfp4_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx,
                    int fmt, int had_k,
                    uint8_t* codes, uint8_t* sf, float* tensor_scale,
                    uint32_t* status, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Scale-policy options of mrfp4_act_quant_ex (NULL = the ScalePolicy() defaults of
 * quantize_rtn, i.e. exactly mrfp4_act_quant):
 *   mx_four_thirds   MXFP4 only.  1: tensor scale f32(4/3) (quantizers.py:34, :191, :206-207);
 *                    0: tensor scale 1.0 -- ScalePolicy(e8m0_four_thirds=False).  The E8M0 scale
 *                    codes are the same; the element codes are rounded against 2^e.
 *   nv_tensor_scale  NVFP4 only.  NULL: the global scale s_T is derived from the whole tensor's
 *                    max (quantizers.py:195-200; two-phase launch).  Otherwise a device float s_T
 *                    used as given (a static / calibrated activation scale):
 *                    scale codes = E4M3(raw / s_T) saturating at 448, elements saturating at +-6,
 *                    exactly prepare_scales' arithmetic with that s_global (quantizers.py:157-167,
 *                    :211-215).  Single pass, no workspace, rows independent.
 */
typedef struct mrfp4_act_quant_opts {
  int mx_four_thirds;
  const float* nv_tensor_scale;
} mrfp4_act_quant_opts;

int mrfp4_act_quant_ex(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx,
                       int fmt, int had_k,
                       uint8_t* codes, uint8_t* sf, float* tensor_scale,
                       uint32_t* status, void* workspace, size_t workspace_bytes,
                       const mrfp4_act_quant_opts* opts, void* stream);

/*
 * apply_blockwise(X, TransformSpec.hadamard(k)) (transforms.py:77-91) for float64 X, as the
 * reference computes it: y[., j] = sum_i x[., i] * M[i][j] with M = (H_k / sqrt(k))^T, summed
 * in index order (i = 0 .. k-1, one rounding per term, as an fma chain).  For k = 16 every
 * product is exact (1/sqrt(16) = 1/4) and this is the order OpenBLAS' dgemm kernel uses for the
 * reference's X.reshape(rows, K/k, k) @ M at every shape tried (bit-identical in the dev
 * container); for k in {32, 64, 128} the reference's own result depends on which BLAS kernel
 * the shape selects (its summation order changes with the shape), so it is not reproducible in
 * general: this order matches it for some shapes, and is within a few ulp elsewhere.  k = 0: copy.
 * x: [M, K] float64 row stride ldx; y: [M, K] float64, contiguous.
 */
int mrfp4_rotate_f64(const double* x, int64_t M, int64_t K, int64_t ldx, int had_k, double* y, void* stream);

/* QuantResult metrics of an act-quant result (quantizers.py:218-231): accumulates into the
 * caller-zeroed device acc[3] = {sum (y-q)^2, sum y^2, sum over groups of the squared relative
 * error at the group's argmax |y|} (fp64, rotated domain); mse_rel = acc[0] / acc[1],
 * mse_top_rel = acc[2] / (M * K / G).  Off the hot path. */
int mrfp4_quant_metrics(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int had_k,
                        const uint8_t* codes, const uint8_t* sf, const float* tensor_scale, double* acc,
                        void* stream);

/* Row-major [rows, sf_cols] scale codes <-> swizzled layout (padding written as 0). */
int mrfp4_sf_swizzle(const uint8_t* sf_rowmajor, uint8_t* sf_swizzled,
                     int64_t rows, int64_t sf_cols, void* stream);
int mrfp4_sf_unswizzle(const uint8_t* sf_swizzled, uint8_t* sf_rowmajor,
                       int64_t rows, int64_t sf_cols, void* stream);

/*
 * Block-scaled FP4 x FP4 GEMM (K2) on tcgen05.mma kind::mxf4nvf4:
 *   D[M,N] = a_ts * b_ts * sum_k (sfA * a) (sfB * b)      (both operands K-major)
 * a: [M, K/2] codes + swizzled sf; b: [N, K/2] codes + swizzled sf (the weight);
 * a_ts, b_ts: device float tensor scales; d: [M, N] row stride ldd, dtype d_dtype
 * (MRFP4_DT_BF16 or MRFP4_DT_F32).  Requires K % 64 == 0, N % 8 == 0.
 * workspace: device scratch of mrfp4_gemm_workspace() bytes, zero-filled once before first
 * use (a 4 KB header of per-tile arrival counters that every call leaves zero again; do not
 * share one workspace between concurrent streams).  Small M: split-K fp32 partials, summed in
 * split order by the last split of each tile to finish (one kernel, deterministic).  Large M:
 * no workspace (0 bytes).  NULL or too small: no split (correct, slower).
 */
size_t mrfp4_gemm_workspace(int64_t M, int64_t N, int64_t K, int fmt);
int mrfp4_gemm(const uint8_t* a, const uint8_t* a_sf, const float* a_ts,
               const uint8_t* b, const uint8_t* b_sf, const float* b_ts,
               void* d, int d_dtype, int64_t M, int64_t N, int64_t K, int64_t ldd,
               int fmt, void* workspace, size_t workspace_bytes, void* stream);

/* Device dequantize (formats.py:424-442): out[r,c] = ts * scale * fp4, fp32 output. */
int mrfp4_dequantize(const uint8_t* codes, const uint8_t* sf, const float* tensor_scale,
                     int64_t rows, int64_t cols, int fmt, float* out, void* stream);

/*
 * K2 of an N-sharded linear with the output all-gather fused into its epilogue (SURVEY.md
 * 8(f) row f1): D = a . b^T (bf16) stored row segment by row segment into EACH of the ndst
 * (<= 8) destinations -- on a multi-GPU node, the peer-mapped full-output buffers of every rank
 * (e.g. torch symmetric memory over NVLink), each pointer already offset to this rank's column
 * block; row stride ldd (the full N).  Replaces mrfp4_gemm + the NCCL all-gather of the bf16
 * output.  The caller synchronizes the ranks afterwards.  Requires M > 128, K % 256 == 0.
 */
int mrfp4_gemm_peers(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
                     const float* b_ts, void* const* dsts, int ndst, int64_t M, int64_t N, int64_t K, int64_t ldd,
                     int fmt, void* stream);

/*
 * K2 with the NEXT layer's act-quant fused into its epilogue: computes
 * Y = bf16(a . b^T) as mrfp4_gemm does and, from those bf16 values, the MXFP4 quantization
 * quantize_rtn(Y, FormatSpec.mxfp4(), transform=hadamard(next_had_k)) (quantizers.py:247-255)
 * -- E2M1 codes [M, N/2], swizzled E8M0 scales [M, N/32] (padding rows zeroed) and the tensor
 * scale f32(4/3) -- bit-identical to mrfp4_act_quant on Y.  y_bf16 may be NULL (Y not stored).
 * Requires M > 128, K % 256 == 0, N % 128 == 0, next_had_k in {0, 16, 32, 64, 128}; status: bit 1 =
 * non-finite Y.  A whole-Y NVFP4 tensor scale cannot be fused (it needs all of Y before any group
 * is encoded): mrfp4_gemm_quant_next_ex takes a static one.
 */
int mrfp4_gemm_quant_next(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                          const uint8_t* b_sf, const float* b_ts, void* y_bf16, int64_t ldy, int64_t M, int64_t N,
                          int64_t K, int fmt, int next_had_k, uint8_t* next_codes, uint8_t* next_sf,
                          float* next_tensor_scale, uint32_t* status, void* stream);
/* The same for either next-layer format: next_fmt MXFP4 (as above), or NVFP4 against the given
 * device global scale next_static_ts (a static / calibrated s_T, see mrfp4_act_quant_opts) --
 * identical to mrfp4_act_quant_ex on Y with opts.nv_tensor_scale = next_static_ts.  next_had_k in
 * {0, 16, 32, 64, 128} (64 / 128: the cross-segment stages run in the epilogue thread, which
 * holds 128 consecutive output columns).  next_sf: scale codes [M, N/G] (G = 16 or 32). */
int mrfp4_gemm_quant_next_ex(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                             const uint8_t* b_sf, const float* b_ts, void* y_bf16, int64_t ldy, int64_t M, int64_t N,
                             int64_t K, int fmt, int next_fmt, int next_had_k, const float* next_static_ts,
                             uint8_t* next_codes, uint8_t* next_sf, float* next_tensor_scale, uint32_t* status,
                             void* stream);

/*
 * Offline MSE scale search (replaces the numpy loops of
 * optimize_group_scales, quantizers.py:263-327).  y: the rotated matrix in float64, viewed as
 * ngroups contiguous groups of 32 (MXFP4) / 16 (NVFP4) values, 16-byte aligned.
 *
 * mrfp4_mse_pass -- one candidate pass (quantizers.py:288-302): for every group, the
 *   candidate raw scales cand[c] * raw0[g] (c < ncand; the reference's [1.0] + 128 multipliers)
 *   are encoded against s_global (fp_scale_encode, formats.py:220-262), each scored by
 *   sum((y - eff * fp4(y / eff))^2) with eff = ts * decoded in numpy's pairwise order, and the
 *   first minimum is kept: scale_codes[g], decoded[g], group_err[g], and the group's packed
 *   E2M1 codes (low nibble first) in codes[g * G / 2 ..].
 * mrfp4_mse_group_err -- group errors at fixed decoded scales and tensor scale ts (the terms
 *   of total_err, quantizers.py:304-306).
 * Device status bits: 2 = a candidate scale decodes to 0 (the reference raises DataError),
 * 1 = non-finite error.  The caller sums group_err in numpy's order.
 */
int mrfp4_mse_pass(const double* y, int64_t ngroups, int fmt, const double* cand, int ncand, const double* raw0,
                   double s_global, double ts, uint8_t* scale_codes, double* decoded, double* group_err,
                   uint8_t* codes, uint32_t* status, void* stream);
int mrfp4_mse_group_err(const double* y, int64_t ngroups, int fmt, const double* decoded, double ts,
                        double* group_err, uint32_t* status, void* stream);
/*
 * Decode-sized quantized linear in one kernel (M <= 32 tokens) -- replaces
 * dequantize(quantize_rtn(X, spec, H_k)) @ dequantize(Wq).T (quantizers.py:247-255,
 * formats.py:424-442) like mrfp4_act_quant + mrfp4_gemm: the activation rotate + quantize runs
 * inside the GEMM CTAs (the CTAs of one cluster cover all of K, so the NVFP4 whole-tensor max is
 * their slice maxima combined over DSMEM -- no grid barrier), and the FP4 GEMM puts the
 * weight on the 128-row MMA side (D^T = W . Xq^T, N = 16 | 32 tokens).  Same result as
 * mrfp4_act_quant + mrfp4_gemm up to fp32 summation order.  x: [M, K] contiguous bf16 / f16;
 * w: [N, K/2] codes + swizzled scales + device tensor scale; d: [M, N] (row stride ldd) bf16 /
 * f32.  Two variants, chosen by shape: one thread-block cluster per 128-row weight tile, its
 * CTAs splitting K (<= 8) with the NVFP4 whole-tensor max and the K-split partial sums combined
 * over distributed shared memory (when row tiles x splits fit one wave); or, for wider weights
 * with small M * K, persistent CTAs that each quantize the whole activation into shared memory
 * and stream whole weight tiles.  No workspace, no grid-wide synchronization.  Requires
 * K % 256 == 0, N % 128 == 0, had_k in {0, 16, 32, 64, 128}; returns MRFP4_EUNSUPPORTED for shapes
 * neither variant takes (use mrfp4_act_quant + mrfp4_gemm; mrfp4_linear_decode_ctas() == 0).
 * workspace: unused (mrfp4_linear_decode_workspace() returns 0).  status: optional device word for
 * the DataError bits.
 */
size_t mrfp4_linear_decode_workspace(int64_t M, int64_t N, int64_t K);
/* CTAs mrfp4_linear_decode launches for this shape (0: not a decode shape it takes). */
int mrfp4_linear_decode_ctas(int64_t M, int64_t N, int64_t K);
int mrfp4_linear_decode(const void* x, int x_dtype, int64_t M, int64_t K, int fmt, int had_k, const uint8_t* w,
                        const uint8_t* w_sf, const float* w_ts, int64_t N, void* d, int d_dtype, int64_t ldd,
                        void* workspace, size_t workspace_bytes, uint32_t* status, void* stream);

/*
 * GPTQ column solver, one lazy block (replaces the inner loop of
 * _gptq_core, gptq.py:148-167): for columns i1 .. i1+block-1 (block <= 128) of the permuted
 * weight W [rows, d] (float64, row-major, updated in place), column scales S [rows, d] and the
 * upper inverse-Cholesky factor T [d, d]: per column, codes / q = fp4_round_codes(w / s) (E2M1
 * code per element, written unpacked to codes [rows, d]; q to Q [rows, d]), e = (w - q) / T[i, i]
 * to err [rows, 128] (column i - i1), and w_j -= e * T[i, j] for the block's later columns -- the
 * reference's float64 operations, unfused.  The caller applies W[:, i1+block:] -= err @ T[block
 * rows, i1+block:] (gptq.py:165-166).
 */
int mrfp4_gptq_block(double* W, const double* S, const double* T, int64_t rows, int64_t d, int i1, int block,
                     double* Q, uint8_t* codes, double* err, void* stream);

/* out[i] = numpy's pairwise sum (np.sum) of a[starts[i] .. starts[i] + lens[i]) -- the segment
 * sums the MSE driver combines on the host in numpy's order (bit-identical totals). */
int mrfp4_pairwise_sums(const double* a, const int64_t* starts, const int64_t* lens, int64_t nseg, double* out,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MRFP4_H_ */
