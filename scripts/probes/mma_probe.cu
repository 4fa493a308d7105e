// Throughput of back-to-back tcgen05.mma (cta_group::1, kind::f16, M = 128) for N = 64 /
// 128 / 256 from one issuing thread, operands in shared memory (contents irrelevant).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_2104_07857_b200/csrc
//        -o mma_probe mma_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "tc.cuh"
using namespace zi::tc;

template <int N, int MODE>   // MODE 0: A, B K-major smem; 1: B MN-major; 2: A in TMEM, B MN-major
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* a = sm;                // 128 x 64 bf16, SW128 K-major
  uint8_t* b = sm + 16384;        // N x 64 bf16
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16_f32(128, N, false, MODE >= 1);
    const uint64_t da = sdesc_sw128(smem_u32(a), 16);
    const uint64_t db = MODE >= 1 ? sdesc_sw128(smem_u32(b), 64 * 128) : sdesc_sw128(smem_u32(b), 16);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (MODE == 2) umma_bf16_ts(tmem, tmem + 256 + 8 * k, db + 128 * k, id, 1u);
        else umma_bf16(tmem, da + 2 * k, MODE == 1 ? db + 128 * k : db + 2 * k, id, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int N, int MODE>
void run(long long* d, int iters) {
  const int sm = 16384 + 65536;
  cudaFuncSetAttribute(probe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  probe<N, MODE><<<148, 128, sm>>>(d, iters);
  probe<N, MODE><<<148, 128, sm>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148;
  const double flop = 2.0 * 128 * N * 16 * 4 * iters;
  printf("mode %d M=128 N=%3d K=16: %.1f cycles per MMA, %.0f flop/clk/SM (%s)\n", N, MODE, cyc / (4.0 * iters),
         flop / cyc, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, 0>(d, 4000);
  run<128, 0>(d, 4000);
  run<256, 0>(d, 4000);
  run<64, 1>(d, 4000);
  run<128, 1>(d, 4000);
  run<128, 2>(d, 4000);
  run<256, 2>(d, 4000);
  return 0;
}
