// Shared helpers for the mrfp4 sm_100a kernels (B200).
#pragma once
#include <atomic>
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../../include/mrfp4.h"

namespace mrfp4 {

// ---------------------------------------------------------------------------
// Scale-factor layout consumed by tcgen05 block-scaled MMA (cuBLAS "blocked"
// layout): 128-row x 4-column atoms of 512 bytes, atoms K-contiguous.
// offset(r, c) = ((r/128)*ceil(C/4) + c/4)*512 + (r%32)*16 + ((r/32)%4)*4 + c%4
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__host__ __device__ __forceinline__ int64_t sf_offset(int64_t r, int64_t c, int64_t col_blocks) {
  return ((r >> 7) * col_blocks + (c >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (c & 3);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Value of an E4M3 (unsigned, bias 7) scale code as fp32 (exact).
__device__ __forceinline__ float e4m3_value(uint32_t code) {
  const uint32_t e = code >> 3, m = code & 7u;
  const float sub = (float)m * 0.001953125f;                  // m * 2^-9
  const float nrm = __uint_as_float(((e + 120u) << 23) | (m << 20));
  return e == 0 ? sub : nrm;
}

__device__ __forceinline__ void atomic_or_status(uint32_t* status, uint32_t bits) {
  if (status) atomicOr(status, bits);
}

// Programmatic dependent launch (PDL).  Every kernel is launched with programmatic
// stream serialization, so it may start while its predecessor in the stream is still
// running: pdl_wait() blocks until the predecessor grid has completed and its writes
// are visible, and MUST precede any read of data a predecessor may produce.
// pdl_trigger() lets the successor's CTAs launch (they still wait in pdl_wait()).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Per-device host state.  Kernel attributes (max dynamic SMEM, carveout) and occupancy are
// per device, so every cache is an array indexed by the calling thread's current device.
// Entries are atomics: concurrent first calls may both compute the (idempotent) value.
// ---------------------------------------------------------------------------
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
inline int device_sms() {
  static std::atomic<int> n[kMaxDevices];
  const int d = current_device();
  int v = n[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
    n[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
// Runs `init()` (returning > 0 on success, <= 0 on failure) once per device for the cache
// `slot` (one static array per kernel instantiation) and returns its cached result.
template <typename F>
inline int per_device_once(std::atomic<int> (&slot)[kMaxDevices], F&& init) {
  const int d = current_device();
  int v = slot[d].load(std::memory_order_acquire);
  if (v == 0) {
    v = init();
    if (v == 0) v = -1;
    slot[d].store(v, std::memory_order_release);
  }
  return v;
}

// Launch `kern` on `s` with the PDL attribute (disabled when MRFP4_PDL=0 in the environment).
// `cooperative`: the kernel spin-waits on other CTAs of its grid (the NVFP4 act-quant grid
// barrier, the split-K GEMM's in-kernel reduction).  Its grid is sized from the occupancy
// calculator so every CTA is co-resident on an otherwise idle GPU; with MRFP4_COOP=1 the launch
// is also made cooperative, so that under MPS, green contexts or a concurrent persistent kernel
// it fails (cudaErrorCooperativeLaunchTooLarge -> MRFP4_ECUDA) instead of hanging.  If the
// driver refuses the cooperative + PDL combination, it is retried cooperative only.
bool pdl_enabled();
bool coop_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       bool cooperative, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cooperative && coop_enabled()) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n++].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess && n == 2 && e != cudaErrorCooperativeLaunchTooLarge) {
    (void)cudaGetLastError();
    attr[0] = attr[1];
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, args...);
  }
  return e;
}

}  // namespace mrfp4
