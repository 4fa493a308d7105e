// Memory-centric tiling: one row-block tile of a tiled linear,
// forward and backward, behind the names of SURVEY §8(b)
// (zi_linear_tile_fwd / zi_linear_tile_bwd). The GEMMs are zi_gemm_sk / zi_gemm (tcgen05
// + TMEM, TMA-fed, 2-SM pair tiles); the tile's bias gradient is a deterministic
// fp32 column sum over the tile's strided column block of the upstream grad.
#include "common.cuh"

namespace zi {

// db[n] = sum_m dy[m * ld + n]; 64 columns per CTA, 8 warps over rows in a
// fixed order, then the 8 partials folded in warp order: deterministic.
__global__ void __launch_bounds__(256)
tile_colsum_kernel(const __nv_bfloat16* __restrict__ dy, int M, int N, int ld,
                   float* __restrict__ db) {
  __shared__ float part[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 64 + 2 * lane;
  float s0 = 0.f, s1 = 0.f;
  if (c + 1 < N && (ld & 1) == 0) {
    for (int m = warp; m < M; m += 8) {
      const __nv_bfloat162 v =
          *reinterpret_cast<const __nv_bfloat162*>(dy + (size_t)m * ld + c);
      s0 += __bfloat162float(v.x);
      s1 += __bfloat162float(v.y);
    }
  } else {
    for (int m = warp; m < M; m += 8) {
      if (c < N) s0 += __bfloat162float(dy[(size_t)m * ld + c]);
      if (c + 1 < N) s1 += __bfloat162float(dy[(size_t)m * ld + c + 1]);
    }
  }
  part[warp][2 * lane] = s0;
  part[warp][2 * lane + 1] = s1;
  __syncthreads();
  if (threadIdx.x < 64) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[w][threadIdx.x];
    const int n = blockIdx.x * 64 + threadIdx.x;
    if (n < N) db[n] = s;
  }
}

}  // namespace zi

extern "C" {

// dW of tiles whose shapes meet zi_gemm_sk's contract (16-byte rows: N, ld multiples of 8)
// runs on the stream-K kernel with whole tiles (no workspace); others on zi_gemm.
static bool sk_ok(int N, int lda, int ldb, int ldd, const void* a, const void* b, const void* d) {
  return N % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0 && ldd % 8 == 0 && zi::aligned(a, 16) &&
         zi::aligned(b, 16) && zi::aligned(d, 16);
}

// The forward stays on zi_gemm's 256 x 512 wide pair tiles: at K = 16384 the stream-K
// kernel's 16-row raster re-reads 3.2 GB of DRAM per config-4 tile against 1.76 GB
// (ncu), 1488 vs 1593 TFLOPS; the backward's dW runs 18 % faster on zi_gemm_sk.
int zi_linear_tile_fwd(const void* x, const void* w_t, const void* b_t, void* y, int M, int K,
                       int N_t, int ldx, int ldw, int ldy, void* stream) {
  return zi_gemm(x, 0, ldx, w_t, 0, ldw, b_t, y, 0, 0, ldy, M, N_t, K, stream);
}

int zi_linear_tile_bwd(const void* x, int ldx, const void* w_t, int ldw, const void* dy_t,
                       int lddy, void* dw_t, int lddw, float* dx_acc, int lddx, float* db_t,
                       int M, int K, int N_t, void* stream) {
  ZI_CHECK_ARG(x && w_t && dy_t && M > 0 && K > 0 && N_t > 0,
               "zi_linear_tile_bwd: bad arguments");
  int st;
  if (dw_t) {   // dW_t[n, k] = sum_m dy_t[m, n] x[m, k]   (both operands MN-major)
    if (sk_ok(K, lddy, ldx, lddw, dy_t, x, dw_t) && N_t % 8 == 0)
      st = zi_gemm_sk(dy_t, 1, lddy, x, 1, ldx, nullptr, dw_t, lddw, 0, nullptr, 0, nullptr, 0,
                      ZI_EPI_PLAIN, N_t, K, M, nullptr, 0, stream);
    else
      st = zi_gemm(dy_t, 1, lddy, x, 1, ldx, nullptr, dw_t, 0, 0, lddw, N_t, K, M, stream);
    if (st) return st;
  }
  if (dx_acc) { // dx[m, k] += sum_n dy_t[m, n] W_t[n, k]  (fp32, tiles accumulate in order)
    st = zi_gemm(dy_t, 0, lddy, w_t, 1, ldw, nullptr, dx_acc, 1, 1, lddx, M, K, N_t, stream);
    if (st) return st;
  }
  if (db_t) {
    zi::count_launches();
    zi::tile_colsum_kernel<<<(N_t + 63) / 64, 256, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)dy_t, M, N_t, lddy, db_t);
    return zi::launch_status("zi_linear_tile_bwd(db)");
  }
  return ZI_OK;
}

}  // extern "C"
