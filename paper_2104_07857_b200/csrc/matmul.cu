// zi_matmul_fixed: C = A B (+ bias) in fp32 or fp64 with a fixed summation order.
//
// The SPEC harness must give bit-identical digests across world
// sizes and placements (AC-9) and reduces "in fixed order everywhere"
// (SPEC.md:786,789). cuBLAS does not promise that: its fp32 algorithm (split-K or
// not) depends on the workspace it finds, so the same product can round differently
// from one process state to the next. Here each output is one thread's sequential
// k = 0..K-1 fma chain, then + bias: the result depends only on the operands. The
// harness matrices are tiny (tens of rows/columns), so this is latency-, not
// throughput-bound; it is not used on the bf16 GPT path.
#include "common.cuh"

namespace zi {

template <typename T>
__device__ __forceinline__ T fma_rn(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_rn<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_rn<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T>
__global__ void __launch_bounds__(256)
matmul_fixed_kernel(const T* __restrict__ A, int64_t sam, int64_t sak, const T* __restrict__ B,
                    int64_t sbk, int64_t sbn, const T* __restrict__ bias, T* __restrict__ C,
                    int64_t scm, int64_t scn, int M, int N, int K) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)M * N) return;
  const int m = (int)(idx / N), n = (int)(idx % N);
  const T* a = A + m * sam;
  const T* b = B + n * sbn;
  T acc = T(0);
  for (int k = 0; k < K; ++k) acc = fma_rn<T>(a[k * sak], b[k * sbk], acc);
  if (bias) acc = acc + bias[n];
  C[m * scm + n * scn] = acc;
}

}  // namespace zi

extern "C" {

int zi_matmul_fixed(const void* A, int64_t sam, int64_t sak, const void* B, int64_t sbk,
                    int64_t sbn, const void* bias, void* C, int64_t scm, int64_t scn, int M,
                    int N, int K, int dtype, void* stream) {
  ZI_CHECK_ARG(A && B && C, "zi_matmul_fixed: NULL operand");
  ZI_CHECK_ARG(M >= 0 && N >= 0 && K >= 0, "zi_matmul_fixed: negative size");
  ZI_CHECK_ARG(dtype == ZI_DT_F32 || dtype == ZI_DT_F64, "zi_matmul_fixed: dtype must be f32/f64");
  if ((int64_t)M * N == 0) return ZI_OK;
  const int64_t total = (int64_t)M * N;
  const int grid = (int)((total + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  zi::count_launches();
  if (dtype == ZI_DT_F32)
    zi::matmul_fixed_kernel<float><<<grid, 256, 0, s>>>(
        (const float*)A, sam, sak, (const float*)B, sbk, sbn, (const float*)bias, (float*)C, scm,
        scn, M, N, K);
  else
    zi::matmul_fixed_kernel<double><<<grid, 256, 0, s>>>(
        (const double*)A, sam, sak, (const double*)B, sbk, sbn, (const double*)bias, (double*)C,
        scm, scn, M, N, K);
  return zi::launch_status("zi_matmul_fixed");
}

}  // extern "C"
