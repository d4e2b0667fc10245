// extern "C" boundary of libmrfp4.so (declared in include/mrfp4.h).
// Host-side validation mirrors the reference's DataError conditions
// (/root/reference/pkg/src/microfp/quantizers.py:95-111) and returns a status;
// kernels report data errors through the caller's device status word.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "common.cuh"

namespace mrfp4 {
int launch_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int hk, uint8_t* codes,
                     uint8_t* sf, float* tensor_scale, uint32_t* status, void* workspace,
                     const mrfp4_act_quant_opts* opts, cudaStream_t s);
int launch_linear_decode(const void* x, int x_dtype, int64_t M, int64_t K, int fmt, int hk, const uint8_t* w,
                         const uint8_t* w_sf, const float* w_ts, int64_t N, void* d, int d_dtype, int64_t ldd,
                         void* ws, size_t ws_bytes, uint32_t* status, cudaStream_t s);
size_t decode_workspace_bytes(int64_t M, int64_t N, int64_t K);
bool decode_plan(int64_t M, int64_t N, int64_t K, int* splits, int* kb_per);
bool decode_p_plan(int64_t M, int64_t N, int64_t K, int* grid);
int launch_gptq_block(double* W, const double* S, const double* T, int64_t rows, int64_t d, int i1, int B, double* Q,
                      uint8_t* codes, double* Err, cudaStream_t s);
int launch_rotate_f64(const double* x, int64_t M, int64_t K, int64_t ldx, int hk, double* y, cudaStream_t s);
int launch_gemm_fp4(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
                    const float* b_ts, void* d, int d_dtype, int64_t M, int64_t N, int64_t K, int64_t ldd, int fmt,
                    void* ws, size_t ws_bytes, cudaStream_t s);
size_t gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
int launch_quant_metrics(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int hk,
                         const uint8_t* codes, const uint8_t* sf, const float* tensor_scale, double* acc,
                         cudaStream_t s);
int launch_sf_swizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, cudaStream_t s);
int launch_sf_unswizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, cudaStream_t s);
int launch_dequantize(const uint8_t* codes, const uint8_t* sf, const float* ts, int64_t rows, int64_t cols, int fmt,
                      float* out, cudaStream_t s);
int launch_gemm_quant_next(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                           const uint8_t* b_sf, const float* b_ts, void* y, int64_t ldy, int64_t M, int64_t N,
                           int64_t K, int fmt, int next_fmt, int next_hk, const float* next_static_ts,
                           uint8_t* q_codes, uint8_t* q_sf, float* q_ts, uint32_t* q_status, cudaStream_t s);
int launch_gemm_peers(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                      const uint8_t* b_sf, const float* b_ts, void* const* dsts, int ndst, int64_t M, int64_t N,
                      int64_t K, int64_t ldd, int fmt, cudaStream_t s);
int launch_np_pairwise_segments(const double* a, const int64_t* starts, const int64_t* lens, int64_t nseg,
                                double* out, cudaStream_t s);
int launch_mse_pass(const double* y, int64_t ngroups, int fmt, const double* cand, int ncand, const double* raw0,
                    double sg, double ts, uint8_t* sc, double* dec, double* gerr, uint8_t* codes, uint32_t* status,
                    cudaStream_t s);
int launch_mse_group_err(const double* y, int64_t ngroups, int fmt, const double* dec, double ts, double* gerr,
                         uint32_t* status, cudaStream_t s);
}  // namespace mrfp4

namespace mrfp4 {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MRFP4_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Cooperative launch of the grid-synchronizing kernels: opt-in (MRFP4_COOP=1).  A cooperative
// launch cannot also be a programmatic dependent launch, which costs ~4 us per decode-sized
// layer (c0: 21.5 -> 25.6 us, scripts/c0_coop_probe.sh).  By default the grids are sized by the
// occupancy calculator to be co-resident on the whole GPU; deployments that share SMs (MPS
// partitions, green contexts, concurrent persistent kernels) should set MRFP4_COOP=1, which makes
// an over-subscribed launch fail instead of hang.
bool coop_enabled() {
  static const bool on = [] {
    const char* e = getenv("MRFP4_COOP");
    return e && e[0] == '1';
  }();
  return on;
}
}  // namespace mrfp4

namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(int rc, const char* what) {
  if (rc == MRFP4_OK) return MRFP4_OK;
  if (rc == MRFP4_ECUDA) {
    cudaError_t e = cudaGetLastError();
    return fail(rc, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  }
  return fail(rc, "%s: unsupported configuration", what);
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int elt_size(int dt) { return dt == MRFP4_DT_F32 ? 4 : (dt == MRFP4_DT_BF16 || dt == MRFP4_DT_F16) ? 2 : 0; }
}  // namespace

extern "C" {

int mrfp4_abi_version(void) { return MRFP4_ABI_VERSION; }

const char* mrfp4_last_error(void) { return g_err.c_str(); }

int mrfp4_group_size(int fmt) { return fmt == MRFP4_FMT_MXFP4 ? 32 : fmt == MRFP4_FMT_NVFP4 ? 16 : 0; }

size_t mrfp4_sf_bytes(int64_t rows, int64_t sf_cols) {
  if (rows <= 0 || sf_cols <= 0) return 0;
  return (size_t)(mrfp4::ceil_div(rows, 128) * 128 * mrfp4::ceil_div(sf_cols, 4) * 4);
}

size_t mrfp4_act_quant_workspace(int64_t, int64_t, int fmt) { return fmt == MRFP4_FMT_NVFP4 ? 16 : 0; }

int mrfp4_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int had_k, uint8_t* codes,
                    uint8_t* sf, float* tensor_scale, uint32_t* status, void* workspace, size_t workspace_bytes,
                    void* stream) {
  return mrfp4_act_quant_ex(x, x_dtype, M, K, ldx, fmt, had_k, codes, sf, tensor_scale, status, workspace,
                            workspace_bytes, nullptr, stream);
}

int mrfp4_act_quant_ex(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int had_k,
                       uint8_t* codes, uint8_t* sf, float* tensor_scale, uint32_t* status, void* workspace,
                       size_t workspace_bytes, const mrfp4_act_quant_opts* opts, void* stream) {
  const int G = mrfp4_group_size(fmt);
  if (G == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  const int es = elt_size(x_dtype);
  if (es == 0) return fail(MRFP4_EUNSUPPORTED, "unsupported input dtype %d", x_dtype);
  if (M < 1 || K < 1) return fail(MRFP4_EINVAL, "expected a non-empty 2-D matrix");  // quantizers.py:97-98
  if (M > INT32_MAX / 2 || K > INT32_MAX / 2 || (M * K) / 32 > (int64_t)UINT32_MAX)
    return fail(MRFP4_EUNSUPPORTED, "matrix too large for one call (split the rows)");
  if (K % G) return fail(MRFP4_EINVAL, "columns (%lld) not divisible by group size (%d)", (long long)K, G);
  if (had_k != 0 && had_k != 16 && had_k != 32 && had_k != 64 && had_k != 128)
    return fail(MRFP4_EUNSUPPORTED, "unsupported Hadamard block %d (GPU path: 16, 32, 64, 128)", had_k);
  if (had_k && K % had_k)
    return fail(MRFP4_EINVAL, "columns (%lld) not divisible by transform block (%d)", (long long)K, had_k);
  if (ldx < K) return fail(MRFP4_EINVAL, "row stride %lld < columns %lld", (long long)ldx, (long long)K);
  if (!x || !codes || !sf || !tensor_scale) return fail(MRFP4_EINVAL, "null buffer");
  if (((uint64_t)ldx * es) % 16 || !aligned(x, 16))
    return fail(MRFP4_EUNSUPPORTED, "input rows must be 16-byte aligned");
  if (!aligned(codes, 16) || !aligned(sf, 2)) return fail(MRFP4_EUNSUPPORTED, "output buffers must be 16-byte aligned");
  const bool nv_static = fmt == MRFP4_FMT_NVFP4 && opts && opts->nv_tensor_scale;
  if (nv_static && !aligned(opts->nv_tensor_scale, 4)) return fail(MRFP4_EINVAL, "misaligned nv_tensor_scale");
  if (fmt == MRFP4_FMT_NVFP4 && !nv_static &&
      (workspace == nullptr || workspace_bytes < 16 || !aligned(workspace, 4)))
    return fail(MRFP4_EINVAL, "NVFP4 needs a 16-byte, 4-byte aligned, zero-initialised device workspace");
  const int rc = mrfp4::launch_act_quant(x, x_dtype, M, K, ldx, fmt, had_k, codes, sf, tensor_scale, status,
                                         workspace, opts, static_cast<cudaStream_t>(stream));
  return cuda_status(rc, "mrfp4_act_quant");
}

int mrfp4_rotate_f64(const double* x, int64_t M, int64_t K, int64_t ldx, int had_k, double* y, void* stream) {
  if (M < 1 || K < 1) return fail(MRFP4_EINVAL, "expected a non-empty 2-D matrix");
  if (had_k != 0 && had_k != 16 && had_k != 32 && had_k != 64 && had_k != 128)
    return fail(MRFP4_EUNSUPPORTED, "unsupported Hadamard block %d (GPU path: 16, 32, 64, 128)", had_k);
  if (had_k && K % had_k)
    return fail(MRFP4_EINVAL, "columns (%lld) not divisible by transform block (%d)", (long long)K, had_k);
  if (ldx < K || !x || !y) return fail(MRFP4_EINVAL, "bad arguments");
  return cuda_status(mrfp4::launch_rotate_f64(x, M, K, ldx, had_k, y, static_cast<cudaStream_t>(stream)),
                     "mrfp4_rotate_f64");
}

int mrfp4_linear_decode_ctas(int64_t M, int64_t N, int64_t K) {
  if (M < 1 || M > 32 || K % 256 || K < 256 || N % 128) return 0;
  int sp, per, grid;
  if (mrfp4::decode_plan(M, N, K, &sp, &per)) return (int)(N / 128) * sp;
  if (mrfp4::decode_p_plan(M, N, K, &grid)) return grid;   // persistent wide-weight variant
  return 0;
}

size_t mrfp4_linear_decode_workspace(int64_t M, int64_t N, int64_t K) {
  if (M < 1 || M > 32 || K % 256 || N % 128) return 0;
  return mrfp4::decode_workspace_bytes(M, N, K);
}

int mrfp4_linear_decode(const void* x, int x_dtype, int64_t M, int64_t K, int fmt, int had_k, const uint8_t* w,
                        const uint8_t* w_sf, const float* w_ts, int64_t N, void* d, int d_dtype, int64_t ldd,
                        void* workspace, size_t workspace_bytes, uint32_t* status, void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (!x || !w || !w_sf || !w_ts || !d) return fail(MRFP4_EINVAL, "null buffer");
  if (d_dtype != MRFP4_DT_BF16 && d_dtype != MRFP4_DT_F32) return fail(MRFP4_EUNSUPPORTED, "output dtype");
  if (ldd < N) return fail(MRFP4_EINVAL, "bad output row stride");
  if (!aligned(x, 16) || !aligned(w, 16) || !aligned(w_sf, 16))
    return fail(MRFP4_EUNSUPPORTED, "buffers must be 16-byte aligned");
  const int rc = mrfp4::launch_linear_decode(x, x_dtype, M, K, fmt, had_k, w, w_sf, w_ts, N, d, d_dtype, ldd,
                                             workspace, workspace_bytes, status, static_cast<cudaStream_t>(stream));
  if (rc == MRFP4_EUNSUPPORTED)
    return fail(MRFP4_EUNSUPPORTED, "not a decode shape (M <= 32, K %% 256 == 0, N %% 128 == 0, k <= 32, "
                                    "M * K <= 2^18, M * K / 8 splits <= 16K elements, bf16 / f16 input)");
  return cuda_status(rc, "mrfp4_linear_decode");
}

int mrfp4_gptq_block(double* W, const double* S, const double* T, int64_t rows, int64_t d, int i1, int block,
                     double* Q, uint8_t* codes, double* err, void* stream) {
  if (rows < 1 || d < 1 || i1 < 0 || block < 1 || block > 128 || i1 + block > d)
    return fail(MRFP4_EINVAL, "bad GPTQ block (rows %lld, d %lld, i1 %d, block %d; block <= 128)", (long long)rows,
                (long long)d, i1, block);
  if (!W || !S || !T || !Q || !codes || !err) return fail(MRFP4_EINVAL, "null buffer");
  return cuda_status(mrfp4::launch_gptq_block(W, S, T, rows, d, i1, block, Q, codes, err,
                                              static_cast<cudaStream_t>(stream)),
                     "mrfp4_gptq_block");
}

int mrfp4_quant_metrics(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int fmt, int had_k,
                        const uint8_t* codes, const uint8_t* sf, const float* tensor_scale, double* acc,
                        void* stream) {
  const int G = mrfp4_group_size(fmt);
  if (G == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  const int es = elt_size(x_dtype);
  if (es == 0) return fail(MRFP4_EUNSUPPORTED, "unsupported input dtype %d", x_dtype);
  if (M < 1 || K < 1 || K % G || (had_k && K % had_k) || ldx < K) return fail(MRFP4_EINVAL, "bad dimensions");
  if (!x || !codes || !sf || !tensor_scale || !acc) return fail(MRFP4_EINVAL, "null buffer");
  if (((uint64_t)ldx * es) % 16 || !aligned(x, 16)) return fail(MRFP4_EUNSUPPORTED, "input rows must be 16-byte aligned");
  return cuda_status(mrfp4::launch_quant_metrics(x, x_dtype, M, K, ldx, fmt, had_k, codes, sf, tensor_scale, acc,
                                                 static_cast<cudaStream_t>(stream)),
                     "mrfp4_quant_metrics");
}

int mrfp4_sf_swizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, void* stream) {
  if (rows < 1 || cols < 1 || !src || !dst) return fail(MRFP4_EINVAL, "bad scale matrix");
  return cuda_status(mrfp4::launch_sf_swizzle(src, dst, rows, cols, static_cast<cudaStream_t>(stream)),
                     "mrfp4_sf_swizzle");
}

int mrfp4_sf_unswizzle(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, void* stream) {
  if (rows < 1 || cols < 1 || !src || !dst) return fail(MRFP4_EINVAL, "bad scale matrix");
  return cuda_status(mrfp4::launch_sf_unswizzle(src, dst, rows, cols, static_cast<cudaStream_t>(stream)),
                     "mrfp4_sf_unswizzle");
}

size_t mrfp4_gemm_workspace(int64_t M, int64_t N, int64_t K, int fmt) {
  if (mrfp4_group_size(fmt) == 0 || M < 1 || N < 1 || K < 1) return 0;
  return mrfp4::gemm_workspace_bytes(M, N, K);
}

int mrfp4_gemm(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
               const float* b_ts, void* d, int d_dtype, int64_t M, int64_t N, int64_t K, int64_t ldd, int fmt,
               void* workspace, size_t workspace_bytes, void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (d_dtype != MRFP4_DT_BF16 && d_dtype != MRFP4_DT_F32)
    return fail(MRFP4_EUNSUPPORTED, "output dtype must be bf16 or f32");
  if (M < 1 || N < 1 || K < 1) return fail(MRFP4_EINVAL, "empty GEMM");
  if (K % 64) return fail(MRFP4_EUNSUPPORTED, "K (%lld) must be a multiple of 64", (long long)K);
  if (N % 8) return fail(MRFP4_EUNSUPPORTED, "N (%lld) must be a multiple of 8", (long long)N);
  if (ldd < N) return fail(MRFP4_EINVAL, "ldd < N");
  if (!a || !a_sf || !a_ts || !b || !b_sf || !b_ts || !d) return fail(MRFP4_EINVAL, "null buffer");
  if (!aligned(a, 16) || !aligned(b, 16) || !aligned(a_sf, 16) || !aligned(b_sf, 16) || !aligned(d, 16) ||
      (ldd * elt_size(d_dtype)) % 16)
    return fail(MRFP4_EUNSUPPORTED, "GEMM buffers must be 16-byte aligned");
  if (workspace && !aligned(workspace, 16)) return fail(MRFP4_EINVAL, "GEMM workspace must be 16-byte aligned");
  const int rc = mrfp4::launch_gemm_fp4(a, a_sf, a_ts, b, b_sf, b_ts, d, d_dtype, M, N, K, ldd, fmt, workspace,
                                        workspace ? workspace_bytes : 0, static_cast<cudaStream_t>(stream));
  return cuda_status(rc, "mrfp4_gemm");
}

int mrfp4_dequantize(const uint8_t* codes, const uint8_t* sf, const float* tensor_scale, int64_t rows, int64_t cols,
                     int fmt, float* out, void* stream) {
  const int G = mrfp4_group_size(fmt);
  if (G == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (rows < 1 || cols < 1 || cols % G || cols % 2) return fail(MRFP4_EINVAL, "bad dimensions");
  if (!codes || !sf || !tensor_scale || !out) return fail(MRFP4_EINVAL, "null buffer");
  return cuda_status(mrfp4::launch_dequantize(codes, sf, tensor_scale, rows, cols, fmt, out,
                                              static_cast<cudaStream_t>(stream)),
                     "mrfp4_dequantize");
}

}  // extern "C"

int mrfp4_mse_pass(const double* y, int64_t ngroups, int fmt, const double* cand, int ncand, const double* raw0,
                   double s_global, double ts, uint8_t* scale_codes, double* decoded, double* group_err,
                   uint8_t* codes, uint32_t* status, void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (ngroups < 1 || ncand < 1) return fail(MRFP4_EINVAL, "empty MSE search");
  if (!(s_global > 0.0) || !(ts > 0.0)) return fail(MRFP4_EINVAL, "scales must be positive");
  if (!y || !cand || !raw0 || !scale_codes || !decoded || !group_err || !codes || !status)
    return fail(MRFP4_EINVAL, "null buffer");
  if (!aligned(y, 16)) return fail(MRFP4_EUNSUPPORTED, "y must be 16-byte aligned");
  return cuda_status(mrfp4::launch_mse_pass(y, ngroups, fmt, cand, ncand, raw0, s_global, ts, scale_codes, decoded,
                                            group_err, codes, status, static_cast<cudaStream_t>(stream)),
                     "mrfp4_mse_pass");
}

int mrfp4_mse_group_err(const double* y, int64_t ngroups, int fmt, const double* decoded, double ts,
                        double* group_err, uint32_t* status, void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (ngroups < 1) return fail(MRFP4_EINVAL, "empty MSE search");
  if (!(ts > 0.0)) return fail(MRFP4_EINVAL, "tensor scale must be positive");
  if (!y || !decoded || !group_err || !status) return fail(MRFP4_EINVAL, "null buffer");
  if (!aligned(y, 16)) return fail(MRFP4_EUNSUPPORTED, "y must be 16-byte aligned");
  return cuda_status(mrfp4::launch_mse_group_err(y, ngroups, fmt, decoded, ts, group_err, status,
                                                 static_cast<cudaStream_t>(stream)),
                     "mrfp4_mse_group_err");
}

int mrfp4_gemm_quant_next(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                          const uint8_t* b_sf, const float* b_ts, void* y_bf16, int64_t ldy, int64_t M, int64_t N,
                          int64_t K, int fmt, int next_had_k, uint8_t* next_codes, uint8_t* next_sf,
                          float* next_tensor_scale, uint32_t* status, void* stream) {
  return mrfp4_gemm_quant_next_ex(a, a_sf, a_ts, b, b_sf, b_ts, y_bf16, ldy, M, N, K, fmt, MRFP4_FMT_MXFP4,
                                  next_had_k, nullptr, next_codes, next_sf, next_tensor_scale, status, stream);
}

int mrfp4_gemm_quant_next_ex(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b,
                             const uint8_t* b_sf, const float* b_ts, void* y_bf16, int64_t ldy, int64_t M, int64_t N,
                             int64_t K, int fmt, int next_fmt, int next_had_k, const float* next_static_ts,
                             uint8_t* next_codes, uint8_t* next_sf, float* next_tensor_scale, uint32_t* status,
                             void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (mrfp4_group_size(next_fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown next-layer format %d", next_fmt);
  if (M < 1 || N < 1 || K < 1) return fail(MRFP4_EINVAL, "empty GEMM");
  if (M <= 128 || K % 256)
    return fail(MRFP4_EUNSUPPORTED, "fused next-layer quantization needs M > 128 and K %% 256 == 0 (2-CTA GEMM)");
  if (N % 128) return fail(MRFP4_EUNSUPPORTED, "fused next-layer quantization needs N %% 128 == 0");
  if (next_had_k != 0 && next_had_k != 16 && next_had_k != 32 && next_had_k != 64 && next_had_k != 128)
    return fail(MRFP4_EUNSUPPORTED, "fused next-layer quantization: Hadamard block must be 0, 16, 32, 64 or 128");
  if (next_fmt == MRFP4_FMT_NVFP4 && !next_static_ts)
    return fail(MRFP4_EUNSUPPORTED, "fused NVFP4 next-layer quantization needs a static global scale "
                                    "(the whole-output max is not known inside the GEMM)");
  if (y_bf16 && (ldy < N || ldy % 16)) return fail(MRFP4_EINVAL, "bad output row stride");
  if (!a || !a_sf || !a_ts || !b || !b_sf || !b_ts || !next_codes || !next_sf || !next_tensor_scale || !status)
    return fail(MRFP4_EINVAL, "null buffer");
  if (!aligned(next_codes, 16) || !aligned(next_sf, 2)) return fail(MRFP4_EUNSUPPORTED, "codes must be 16-byte aligned");
  return cuda_status(mrfp4::launch_gemm_quant_next(a, a_sf, a_ts, b, b_sf, b_ts, y_bf16, ldy, M, N, K, fmt, next_fmt,
                                                   next_had_k, next_static_ts, next_codes, next_sf, next_tensor_scale,
                                                   status, static_cast<cudaStream_t>(stream)),
                     "mrfp4_gemm_quant_next_ex");
}

int mrfp4_pairwise_sums(const double* a, const int64_t* starts, const int64_t* lens, int64_t nseg, double* out,
                        void* stream) {
  if (nseg < 1) return fail(MRFP4_EINVAL, "no segments");
  if (!a || !starts || !lens || !out) return fail(MRFP4_EINVAL, "null buffer");
  return cuda_status(mrfp4::launch_np_pairwise_segments(a, starts, lens, nseg, out, static_cast<cudaStream_t>(stream)),
                     "mrfp4_pairwise_sums");
}

int mrfp4_gemm_peers(const uint8_t* a, const uint8_t* a_sf, const float* a_ts, const uint8_t* b, const uint8_t* b_sf,
                     const float* b_ts, void* const* dsts, int ndst, int64_t M, int64_t N, int64_t K, int64_t ldd,
                     int fmt, void* stream) {
  if (mrfp4_group_size(fmt) == 0) return fail(MRFP4_EUNSUPPORTED, "unknown format %d", fmt);
  if (M < 1 || N < 1 || K < 1) return fail(MRFP4_EINVAL, "empty GEMM");
  if (M <= 128 || K % 256)
    return fail(MRFP4_EUNSUPPORTED, "peer-store GEMM needs M > 128 and K %% 256 == 0 (2-CTA GEMM)");
  if (N % 8) return fail(MRFP4_EUNSUPPORTED, "N (%lld) must be a multiple of 8", (long long)N);
  if (ndst < 1 || ndst > 8 || !dsts) return fail(MRFP4_EINVAL, "1..8 destinations");
  if (ldd < N || ldd % 16) return fail(MRFP4_EINVAL, "ldd must be >= N and a multiple of 16");
  for (int i = 0; i < ndst; ++i)
    if (!dsts[i] || !aligned(dsts[i], 32)) return fail(MRFP4_EINVAL, "destinations must be 32-byte aligned");
  if (!a || !a_sf || !a_ts || !b || !b_sf || !b_ts) return fail(MRFP4_EINVAL, "null buffer");
  return cuda_status(mrfp4::launch_gemm_peers(a, a_sf, a_ts, b, b_sf, b_ts, dsts, ndst, M, N, K, ldd, fmt,
                                              static_cast<cudaStream_t>(stream)),
                     "mrfp4_gemm_peers");
}
