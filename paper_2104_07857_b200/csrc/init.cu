// Shard-local parameter init and half/fp32 casts.
//
// zi_init_uniform: "partitioned immediately after its initialization ...
// never fully instantiated on a single" GPU (PAPER §7.2):
// each rank generates only the elements of its own shard with a counter RNG
// (splitmix64 of (key, element index)), bit-identical to
// oracle/numerics.py:uniform_init, and writes the fp32 master and the RNE
// half working copy in one pass.
#include "common.cuh"

namespace zi {

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int KIND>
__global__ void __launch_bounds__(256)
init_uniform_kernel(float* __restrict__ master, uint16_t* __restrict__ ph, size_t n, uint64_t key,
                    uint64_t start, float scale) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t z = key + (start + i + 1) * 0x9E3779B97F4A7C15ULL;
    const int64_t k = (int64_t)(splitmix_mix(z) >> 40);
    const float v = (float)(int32_t)(2 * k + 1 - (1LL << 24));
    const float x = __fmul_rn(v, scale);
    if (master) master[i] = x;
    if (ph) ph[i] = Half<KIND>::narrow(x);
  }
}

template <int KIND>
__global__ void __launch_bounds__(256)
fill_kernel(float* __restrict__ master, uint16_t* __restrict__ ph, size_t n, float value) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const uint16_t h = Half<KIND>::narrow(value);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (master) master[i] = value;
    if (ph) ph[i] = h;
  }
}

template <int KIND>
__global__ void __launch_bounds__(256)
f32_to_half_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = Half<KIND>::narrow(src[i]);
}

template <int KIND>
__global__ void __launch_bounds__(256)
half_to_f32_kernel(const uint16_t* __restrict__ src, float* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = Half<KIND>::widen(src[i]);
}

}  // namespace zi

#define ZI_DISPATCH_HALF(kind, KERNEL, ...)                                 \
  do {                                                                     \
    zi::count_launches();                                                   \
    if ((kind) == ZI_HALF_BF16) KERNEL<ZI_HALF_BF16><<<grid, 256, 0, s>>>(__VA_ARGS__); \
    else KERNEL<ZI_HALF_FP16><<<grid, 256, 0, s>>>(__VA_ARGS__);           \
  } while (0)

extern "C" {

int zi_init_uniform(float* master, void* p_half, size_t n, uint64_t key, uint64_t start_index,
                    float scale, int half_kind, void* stream) {
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16, "zi_init_uniform: bad half_kind");
  if (n == 0 || (!master && !p_half)) return ZI_OK;
  const int grid = zi::grid_for(n, 256);
  cudaStream_t s = (cudaStream_t)stream;
  ZI_DISPATCH_HALF(half_kind, zi::init_uniform_kernel, master, static_cast<uint16_t*>(p_half), n,
                   key, start_index, scale);
  return zi::launch_status("zi_init_uniform");
}

int zi_fill(float* master, void* p_half, size_t n, float value, int half_kind, void* stream) {
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16, "zi_fill: bad half_kind");
  if (n == 0 || (!master && !p_half)) return ZI_OK;
  const int grid = zi::grid_for(n, 256);
  cudaStream_t s = (cudaStream_t)stream;
  ZI_DISPATCH_HALF(half_kind, zi::fill_kernel, master, static_cast<uint16_t*>(p_half), n, value);
  return zi::launch_status("zi_fill");
}

int zi_cast_f32_to_half(const float* src, void* dst, size_t n, int half_kind, void* stream) {
  ZI_CHECK_ARG(src && dst, "zi_cast_f32_to_half: NULL");
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16, "zi_cast_f32_to_half: bad half_kind");
  if (n == 0) return ZI_OK;
  const int grid = zi::grid_for(n, 256);
  cudaStream_t s = (cudaStream_t)stream;
  ZI_DISPATCH_HALF(half_kind, zi::f32_to_half_kernel, src, static_cast<uint16_t*>(dst), n);
  return zi::launch_status("zi_cast_f32_to_half");
}

int zi_cast_half_to_f32(const void* src, float* dst, size_t n, int half_kind, void* stream) {
  ZI_CHECK_ARG(src && dst, "zi_cast_half_to_f32: NULL");
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16, "zi_cast_half_to_f32: bad half_kind");
  if (n == 0) return ZI_OK;
  const int grid = zi::grid_for(n, 256);
  cudaStream_t s = (cudaStream_t)stream;
  ZI_DISPATCH_HALF(half_kind, zi::half_to_f32_kernel, static_cast<const uint16_t*>(src), dst, n);
  return zi::launch_status("zi_cast_half_to_f32");
}

}  // extern "C"
