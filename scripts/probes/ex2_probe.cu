// MUFU exp2 throughput on one B200: ex2.approx.f32 (1 result per lane) vs
// ex2.approx.f16x2 (2 results per lane) vs ex2.approx.ftz.bf16x2. Prints results / clk / SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/ex2_probe scripts/probes/ex2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

constexpr int IT = 4096;

__global__ void k_f32(float* out, float seed) {
  float a0 = seed * threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < IT; ++i) {
    asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a0));
    asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a1));
    asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a2));
    asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a3));
  }
  if (a0 + a1 + a2 + a3 == 12345.f) out[0] = a0;
}

__global__ void k_f16x2(float* out, float seed) {
  uint32_t a[4];
  for (int j = 0; j < 4; ++j) {
    __half2 h = __floats2half2_rn(-seed * (threadIdx.x + j), -seed);
    a[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[j]));
  }
  if ((a[0] ^ a[1] ^ a[2] ^ a[3]) == 0x12345) out[0] = 1.f;
}

__global__ void k_bf16x2(float* out, float seed) {
  uint32_t a[4];
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(-seed * (threadIdx.x + j), -seed);
    a[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[j]));
  }
  if ((a[0] ^ a[1] ^ a[2] ^ a[3]) == 0x12345) out[0] = 1.f;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512;
  for (int kind = 0; kind < 3; ++kind) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_f32<<<blocks, threads>>>(out, 0.001f);
      else if (kind == 1) k_f16x2<<<blocks, threads>>>(out, 0.001f);
      else k_bf16x2<<<blocks, threads>>>(out, 0.001f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double res = (double)blocks * threads * IT * 4 * (kind ? 2 : 1);
      const double instr = (double)blocks * threads * IT * 4;
      if (rep == 2)
        printf("%s: %.3f ms, %.1f G results/s, %.2f lane-instr/ns/SM (%.1f results per SM per ns)\n",
               kind == 0 ? "ex2.f32" : kind == 1 ? "ex2.f16x2" : "ex2.bf16x2", ms, res / ms / 1e6,
               instr / ms / 1e6 / sms, res / ms / 1e6 / sms);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
