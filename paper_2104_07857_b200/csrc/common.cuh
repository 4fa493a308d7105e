// Shared helpers for libzinf (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstddef>
#include <string>
#include <utility>

#include "../../include/zinf.h"

namespace zi {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

// After a kernel launch: map a launch failure to ZI_ECUDA with context.
inline int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  return cuda_status(e, what);
}

// ---------------------------------------------------- programmatic dependent launch
// The step's kernels launch with cudaLaunchAttributeProgrammaticStreamSerialization
// (launch_pdl): the next kernel in the stream is launched while this one drains, runs
// its prologue (barrier init, TMEM alloc, descriptor prefetch) and then waits in
// pdl_sync() until every predecessor grid has completed and its memory is visible, so
// the ordering is that of a plain stream; only launch latency and setup overlap. Each
// kernel calls pdl_sync() before its first global-memory access (read or write), and
// pdl_sync() also lets this kernel's own dependents launch. Without the attribute
// (ZI_PDL=0, or a plain <<<>>> launch) both instructions are no-ops.
__device__ __forceinline__ void pdl_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();

// every libzinf kernel launch is counted (zi_launch_count: the engine's launches per step)
void count_launches(int n = 1);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  count_launches();
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline bool aligned(const void* p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

inline int grid_for(size_t work_items, int block, int max_blocks_per_sm = 8) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  size_t want = (work_items + block - 1) / block;
  size_t cap = (size_t)sms * max_blocks_per_sm;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

// ---------------------------------------------------------------- half types
template <int KIND> struct Half;
template <> struct Half<ZI_HALF_FP16> {
  using T = __half;
  static __device__ __forceinline__ float widen(uint16_t b) {
    return __half2float(__ushort_as_half(b));
  }
  static __device__ __forceinline__ uint16_t narrow(float x) {
    return __half_as_ushort(__float2half_rn(x));
  }
};
template <> struct Half<ZI_HALF_BF16> {
  using T = __nv_bfloat16;
  static __device__ __forceinline__ float widen(uint16_t b) {
    return __uint_as_float(((uint32_t)b) << 16);
  }
  static __device__ __forceinline__ uint16_t narrow(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
};

// Streaming (evict-first) vector loads/stores: every byte of the optimizer
// stream is touched exactly once per step.
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(uint2* p, uint2 v) { __stcs(p, v); }

// Adam update with the oracle's exact operation order (oracle/adam.py).
__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g,
                                      const zi_adam_consts& c) {
  m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, g));
  v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(c.omb2, __fmul_rn(g, g)));
  const float mh = __fdiv_rn(m, c.bc1);
  const float vh = __fdiv_rn(v, c.bc2);
  const float den = __fadd_rn(__fsqrt_rn(vh), c.eps);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(c.lr, mh), den));
}

// tanh on the SFU (tanh.approx.f32, max relative error ~2^-11). GELU results
// are rounded to bf16 (2^-8), so the approximation is below the output
// precision and keeps the GELU kernels / epilogues HBM-bound, not issue-bound.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float GELU_C = 0.7978845608028654f, GELU_A = 0.044715f;

__device__ __forceinline__ float gelu_tanh(float z) {
  return 0.5f * z * (1.f + tanh_fast(GELU_C * (z + GELU_A * z * z * z)));
}

// gelu_tanh(z) and gelu_tanh'(z) from one tanh (the fc1 forward saving GELU')
__device__ __forceinline__ void gelu_and_grad(float z, float& g, float& gp) {
  const float th = tanh_fast(GELU_C * (z + GELU_A * z * z * z));
  g = 0.5f * z * (1.f + th);
  gp = 0.5f * (1.f + th) + 0.5f * z * (1.f - th * th) * GELU_C * (1.f + 3.f * GELU_A * z * z);
}

__device__ __forceinline__ float gelu_tanh_grad(float z) {
  const float th = tanh_fast(GELU_C * (z + GELU_A * z * z * z));
  return 0.5f * (1.f + th) + 0.5f * z * (1.f - th * th) * GELU_C * (1.f + 3.f * GELU_A * z * z);
}

}  // namespace zi

#define ZI_CHECK_ARG(cond, ...)           \
  do {                                    \
    if (!(cond)) {                        \
      zi::set_error(__VA_ARGS__);         \
      return ZI_EINVAL;                   \
    }                                     \
  } while (0)

#define ZI_CUDA(call, what)                              \
  do {                                                   \
    int _s = zi::cuda_status((call), what);              \
    if (_s != ZI_OK) return _s;                          \
  } while (0)
