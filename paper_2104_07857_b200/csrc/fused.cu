// Fused HBM-bound kernels of the GPT block around the GEMMs (bf16 activations,
// fp32 math). Each reads its inputs once and writes its outputs once; column
// reductions (LayerNorm gamma/beta grads, bias grads) are deterministic:
// per-CTA fp32 partials reduced in a fixed order by zi_colsum_finish.
//
//   zi_ln_fwd        y = LN(x) * w + b            (+ x2 = x + r fused residual)
//   zi_ln_bwd        dx = LN'(dy) (+ dres), partial dgamma / dbeta
//   zi_bias_grad     partial column sums of dy (bias gradient)
//   zi_gelu_bwd      du = gelu'(u) * da, partial column sums of du
//   zi_colsum_finish partials [P x N] -> out[N] (bf16 RNE or fp32), fixed order
//   zi_softmax_ce    per-row logsumexp, loss, dlogits = (softmax - onehot) * scale
#include <type_traits>

#include "common.cuh"

namespace zi {
namespace fused {

__device__ __forceinline__ float bf(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t tobf(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }

template <int N>
__device__ __forceinline__ void ld_row(const uint16_t* p, float* f) {
  // N elements (multiple of 4) -> fp32, 8- or 4-element vector loads
  if constexpr (N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        f[8 * i + 2 * j] = bf(u[j] & 0xFFFF);
        f[8 * i + 2 * j + 1] = bf(u[j] >> 16);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      const uint2 v = reinterpret_cast<const uint2*>(p)[i];
      f[4 * i] = bf(v.x & 0xFFFF); f[4 * i + 1] = bf(v.x >> 16);
      f[4 * i + 2] = bf(v.y & 0xFFFF); f[4 * i + 3] = bf(v.y >> 16);
    }
  }
}

template <int N>
__device__ __forceinline__ void st_row(uint16_t* p, const float* f) {
  if constexpr (N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      uint4 v;
      v.x = tobf(f[8 * i]) | ((uint32_t)tobf(f[8 * i + 1]) << 16);
      v.y = tobf(f[8 * i + 2]) | ((uint32_t)tobf(f[8 * i + 3]) << 16);
      v.z = tobf(f[8 * i + 4]) | ((uint32_t)tobf(f[8 * i + 5]) << 16);
      v.w = tobf(f[8 * i + 6]) | ((uint32_t)tobf(f[8 * i + 7]) << 16);
      reinterpret_cast<uint4*>(p)[i] = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      uint2 v;
      v.x = tobf(f[4 * i]) | ((uint32_t)tobf(f[4 * i + 1]) << 16);
      v.y = tobf(f[4 * i + 2]) | ((uint32_t)tobf(f[4 * i + 3]) << 16);
      reinterpret_cast<uint2*>(p)[i] = v;
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row-group LayerNorm: TPR threads per row, 8 contiguous columns each
// (H = 8 * TPR); a 256-thread CTA holds 256 / TPR rows. Row statistics are
// reduced with shuffles (TPR <= 32) or shuffles + shared memory.
template <int TPR>
__device__ __forceinline__ float row_reduce(float v, float* sm) {
#pragma unroll
  for (int o = (TPR < 32 ? TPR : 32) / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if constexpr (TPR > 32) {
    constexpr int W = TPR / 32;              // warps per row
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sm[wid] = v;
    __syncthreads();
    const int base = (wid / W) * W;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < W; ++k) t += sm[base + k];
    __syncthreads();
    v = t;
  }
  return v;
}

// CTA size: 256 threads, or one whole row when a row needs more (H = 4096 / 8192)
template <int TPR>
struct RowCta {
  static constexpr int NT = TPR > 256 ? TPR : 256;
  static constexpr int RPC = NT / TPR;
};

template <int TPR>
__global__ void __launch_bounds__(RowCta<TPR>::NT)
ln_fwd_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ r,
              uint16_t* __restrict__ xsum, const uint16_t* __restrict__ w,
              const uint16_t* __restrict__ b, uint16_t* __restrict__ y, float* __restrict__ mean,
              float* __restrict__ rstd, int T, float eps) {
  constexpr int H = 8 * TPR, RPC = RowCta<TPR>::RPC;
  __shared__ float sm[32];
  const int t = threadIdx.x % TPR;
  float wf[8], bv[8];
  ld_row<8>(w + t * 8, wf);
  ld_row<8>(b + t * 8, bv);
  for (int row0 = blockIdx.x * RPC; row0 < T; row0 += gridDim.x * RPC) {
    const int row = row0 + threadIdx.x / TPR;
    const bool live = row < T;
    const size_t off = (size_t)(live ? row : 0) * H + t * 8;
    float v[8];
    ld_row<8>(x + off, v);
    if (r != nullptr) {
      float rv[8];
      ld_row<8>(r + off, rv);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(__float2bfloat16_rn(v[i] + rv[i]));
      if (live) st_row<8>(xsum + off, v);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    const float mu = row_reduce<TPR>(s, sm) * (1.0f / H);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float d = v[i] - mu;
      q += d * d;
    }
    const float rs = rsqrtf(row_reduce<TPR>(q, sm) * (1.0f / H) + eps);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * wf[i] + bv[i];
    if (live) {
      st_row<8>(y + off, v);
      if (t == 0) {
        mean[row] = mu;
        rstd[row] = rs;
      }
    }
  }
}

// dx = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)) with dxh = dy * w,
// plus dres (residual gradient) if given.
template <int TPR>
__global__ void __launch_bounds__(RowCta<TPR>::NT)
ln_bwd_dx_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                 const uint16_t* __restrict__ w, const float* __restrict__ mean,
                 const float* __restrict__ rstd, const uint16_t* __restrict__ dres,
                 uint16_t* __restrict__ dx, int T) {
  constexpr int H = 8 * TPR, RPC = RowCta<TPR>::RPC;
  __shared__ float sm[32];
  const int t = threadIdx.x % TPR;
  float wf[8];
  ld_row<8>(w + t * 8, wf);
  for (int row0 = blockIdx.x * RPC; row0 < T; row0 += gridDim.x * RPC) {
    const int row = row0 + threadIdx.x / TPR;
    const bool live = row < T;
    const int rr = live ? row : 0;
    const size_t off = (size_t)rr * H + t * 8;
    float g[8], xv[8];
    ld_row<8>(dy + off, g);
    ld_row<8>(x + off, xv);
    const float mu = mean[rr], rs = rstd[rr];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      g[i] *= wf[i];                 // dxh
      xv[i] = (xv[i] - mu) * rs;     // xh
      s1 += g[i];
      s2 += g[i] * xv[i];
    }
    const float m1 = row_reduce<TPR>(s1, sm) * (1.0f / H);
    const float m2 = row_reduce<TPR>(s2, sm) * (1.0f / H);
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = rs * (g[i] - m1 - xv[i] * m2);
    if (dres != nullptr) {
      float rv[8];
      ld_row<8>(dres + off, rv);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] += rv[i];
    }
    if (live) st_row<8>(dx + off, o);
  }
}

// Column reductions (bias grads, GELU-bwd + bias grad, LayerNorm dgamma/dbeta).
// CTA = 64 columns (8 threads x 8) x 32 row groups; blockIdx.y = chunk of rows.
// Each thread folds rows rg, rg+32, ... of its chunk; the CTA folds its 32 row
// groups in order into one partial row; the last CTA of a column block (atomic
// counter, self-resetting so CUDA graphs replay it) folds the chunk partials in
// chunk order and writes the result. Deterministic, one launch, no finish kernel.
//   MODE 0: out0 = sum a                          (bias grad)
//   MODE 1: du = gelu_tanh'(u) * a -> d; out0 = sum du   (GELU bwd + fc1 bias grad)
//   MODE 2: out0 = sum a * (u - mean) * rstd, out1 = sum a   (LN dgamma, dbeta)
constexpr int CR_COLS = 64, CR_RG = 32;

template <int MODE>
__global__ void __launch_bounds__(256)
colred_kernel(const uint16_t* __restrict__ a, const uint16_t* __restrict__ u,
              uint16_t* __restrict__ d, const float* __restrict__ mean,
              const float* __restrict__ rstd, float* __restrict__ part, int* __restrict__ counters,
              void* __restrict__ out0, void* __restrict__ out1, int out_f32, int T, int N,
              int rows_per) {
  constexpr int NO = MODE == 2 ? 2 : 1;
  __shared__ float red[NO][CR_RG][CR_COLS + 1];
  __shared__ int last;
  const int cx = threadIdx.x & 7, rg = threadIdx.x >> 3;
  const int c8 = blockIdx.x * CR_COLS + cx * 8;
  const bool colok = c8 < N;
  const int r0 = blockIdx.y * rows_per, r1 = min(T, r0 + rows_per);
  float acc[NO][8];
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[o][j] = 0.f;
  if (colok) {
#pragma unroll 4
    for (int row = r0 + rg; row < r1; row += CR_RG) {
      const size_t off = (size_t)row * N + c8;
      float v[8];
      ld_row<8>(a + off, v);
      if (MODE == 1) {
        float uv[8];
        ld_row<8>(u + off, uv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float z = uv[j];
          const float c = 0.7978845608028654f;
          const float th = tanhf(c * (z + 0.044715f * z * z * z));
          const float dg = 0.5f * (1.f + th) + 0.5f * z * (1.f - th * th) * c * (1.f + 3.f * 0.044715f * z * z);
          v[j] = __bfloat162float(__float2bfloat16_rn(v[j] * dg));
        }
        st_row<8>(d + off, v);
      }
      if (MODE == 2) {
        float xv[8];
        ld_row<8>(u + off, xv);
        const float mu = mean[row], rs = rstd[row];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[0][j] += v[j] * (xv[j] - mu) * rs;
          acc[NO - 1][j] += v[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[0][j] += v[j];
      }
    }
  }
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int j = 0; j < 8; ++j) red[o][rg][cx * 8 + j] = acc[o][j];
  __syncthreads();
  // fold the 32 row groups (fixed order) -> this chunk's partial row
  if (threadIdx.x < CR_COLS * NO) {
    const int o = threadIdx.x / CR_COLS, col = threadIdx.x % CR_COLS;
    const int gc = blockIdx.x * CR_COLS + col;
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < CR_RG; ++k) t += red[o][k][col];
    if (gc < N) part[((size_t)o * gridDim.y + blockIdx.y) * N + gc] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[blockIdx.x], 1) == (int)gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < CR_COLS * NO) {
    const int o = threadIdx.x / CR_COLS, col = threadIdx.x % CR_COLS;
    const int gc = blockIdx.x * CR_COLS + col;
    if (gc < N) {
      float t = 0.f;
      for (int p = 0; p < (int)gridDim.y; ++p) t += __ldcg(&part[((size_t)o * gridDim.y + p) * N + gc]);
      void* dst = o == 0 ? out0 : out1;
      if (out_f32) static_cast<float*>(dst)[gc] = t;
      else static_cast<uint16_t*>(dst)[gc] = tobf(t);
    }
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0;   // ready for the next launch / replay
}

// One CTA per row of V logits (bf16, in place): lse, loss_row = lse - l[t],
// dlogits = (exp(l - lse) - [j == t]) * scale written back as bf16.
__global__ void __launch_bounds__(512)
softmax_ce_kernel(uint16_t* __restrict__ logits, const int64_t* __restrict__ tgt,
                  float* __restrict__ loss_rows, int V, float scale) {
  const size_t row = blockIdx.x;
  uint16_t* L = logits + row * (size_t)V;
  __shared__ float red_m[16], red_s[16];
  float m = -INFINITY, s = 0.f;
  const int V8 = (V % 8 == 0) ? V / 8 : 0;
  for (int i = threadIdx.x; i < V8; i += blockDim.x) {
    float f[8];
    ld_row<8>(L + 8 * i, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (f[j] > m) {
        s *= __expf(m - f[j]);
        m = f[j];
      }
      s += __expf(f[j] - m);
    }
  }
  for (int i = V8 * 8 + threadIdx.x; i < V; i += blockDim.x) {
    const float f = bf(L[i]);
    if (f > m) { s *= __expf(m - f); m = f; }
    s += __expf(f - m);
  }
  // block reduce (m, s)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { red_m[wid] = m; red_s[wid] = s; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    m = lane < nw ? red_m[lane] : -INFINITY;
    s = lane < nw ? red_s[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (lane == 0) { red_m[0] = m; red_s[0] = s; }
  }
  __syncthreads();
  const float lse = red_m[0] + __logf(red_s[0]);
  const int t = (int)tgt[row];
  if (threadIdx.x == 0) loss_rows[row] = lse - bf(L[t]);
  __syncthreads();  // everyone read L[t] before it is overwritten
  for (int i = threadIdx.x; i < V8; i += blockDim.x) {
    float f[8];
    ld_row<8>(L + 8 * i, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = 8 * i + j;
      f[j] = (__expf(f[j] - lse) - (col == t ? 1.f : 0.f)) * scale;
    }
    st_row<8>(L + 8 * i, f);
  }
  for (int i = V8 * 8 + threadIdx.x; i < V; i += blockDim.x)
    L[i] = tobf((__expf(bf(L[i]) - lse) - (i == t ? 1.f : 0.f)) * scale);
}

__global__ void sum_kernel(const float* __restrict__ v, int n, float scale, float* __restrict__ out) {
  // single block, fixed-order tree: deterministic
  __shared__ float sm[1024];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0] * scale;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
  }
  return sms;
}

}  // namespace fused
}  // namespace zi

using namespace zi::fused;

#define TPR_DISPATCH(H, KERNEL, GRID, STREAM, ...)                                        \
  switch ((H) / 8) {                                                                       \
    case 16: KERNEL<16><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;                     \
    case 32: KERNEL<32><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;                     \
    case 64: KERNEL<64><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;                     \
    case 128: KERNEL<128><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;                   \
    case 256: KERNEL<256><<<GRID, 256, 0, STREAM>>>(__VA_ARGS__); break;                   \
    case 512: KERNEL<512><<<GRID, 512, 0, STREAM>>>(__VA_ARGS__); break;                   \
    case 1024: KERNEL<1024><<<GRID, 1024, 0, STREAM>>>(__VA_ARGS__); break;                \
    default: zi::set_error("LayerNorm: hidden size %d not in {128..8192, power of 2}", H); \
      return ZI_EINVAL;                                                                    \
  }

static int ln_grid(int T, int H) {
  const int tpr = H / 8;
  const int rpc = tpr >= 256 ? 1 : 256 / tpr;
  const int need = (T + rpc - 1) / rpc;
  const int cap = sm_count() * 8;
  return need < cap ? need : cap;
}

extern "C" {

int zi_ln_fwd(const void* x, const void* resid, void* xsum, const void* w, const void* b, void* y,
              float* mean, float* rstd, int T, int H, float eps, void* stream) {
  ZI_CHECK_ARG(x && w && b && y && mean && rstd && T > 0, "zi_ln_fwd: bad arguments");
  ZI_CHECK_ARG(!resid || xsum, "zi_ln_fwd: resid needs xsum");
  cudaStream_t s = (cudaStream_t)stream;
  ZI_CHECK_ARG(H >= 128 && H <= 8192 && (H & (H - 1)) == 0, "zi_ln_fwd: H must be 128..8192, power of 2");
  const int grid = ln_grid(T, H);
  TPR_DISPATCH(H, ln_fwd_kernel, grid, s, (const uint16_t*)x, (const uint16_t*)resid,
               (uint16_t*)xsum, (const uint16_t*)w, (const uint16_t*)b, (uint16_t*)y, mean, rstd,
               T, eps);
  return zi::launch_status("zi_ln_fwd");
}

// work layout: [0, 1024) int counters (zeroed once, self-resetting), then partials
static int launch_colred(int mode, const void* a, const void* u, void* d, const float* mean,
                         const float* rstd, void* out0, void* out1, int out_f32, float* work,
                         size_t work_elems, int T, int N, cudaStream_t s, const char* name) {
  ZI_CHECK_ARG(N % 8 == 0, "%s: N must be a multiple of 8", name);
  const int cblocks = (N + CR_COLS - 1) / CR_COLS;
  ZI_CHECK_ARG(cblocks <= 1024, "%s: N too large for the counter block", name);
  int chunks = (sm_count() * 4 + cblocks - 1) / cblocks;
  const int max_chunks = (T + CR_RG - 1) / CR_RG;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  const int rows_per = (T + chunks - 1) / chunks;
  chunks = (T + rows_per - 1) / rows_per;
  const size_t need = 1024 + (size_t)(mode == 2 ? 2 : 1) * chunks * N;
  ZI_CHECK_ARG(work_elems >= need, "%s: work needs %zu floats", name, need);
  int* counters = reinterpret_cast<int*>(work);
  float* part = work + 1024;
  dim3 grid(cblocks, chunks);
  const uint16_t* A = static_cast<const uint16_t*>(a);
  const uint16_t* U = static_cast<const uint16_t*>(u);
  uint16_t* D = static_cast<uint16_t*>(d);
  if (mode == 0)
    colred_kernel<0><<<grid, 256, 0, s>>>(A, U, D, mean, rstd, part, counters, out0, out1, out_f32, T, N, rows_per);
  else if (mode == 1)
    colred_kernel<1><<<grid, 256, 0, s>>>(A, U, D, mean, rstd, part, counters, out0, out1, out_f32, T, N, rows_per);
  else
    colred_kernel<2><<<grid, 256, 0, s>>>(A, U, D, mean, rstd, part, counters, out0, out1, out_f32, T, N, rows_per);
  return zi::launch_status(name);
}

int zi_ln_bwd(const void* dy, const void* x, const void* w, const float* mean, const float* rstd,
              const void* dres, void* dx, void* dgamma, void* dbeta, int grads_f32, float* work,
              size_t work_elems, int T, int H, void* stream) {
  ZI_CHECK_ARG(dy && x && w && mean && rstd && dx && dgamma && dbeta && work, "zi_ln_bwd: NULL");
  ZI_CHECK_ARG(H >= 128 && H <= 8192 && (H & (H - 1)) == 0, "zi_ln_bwd: H must be 128..8192, power of 2");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = ln_grid(T, H);
  TPR_DISPATCH(H, ln_bwd_dx_kernel, grid, s, (const uint16_t*)dy, (const uint16_t*)x,
               (const uint16_t*)w, mean, rstd, (const uint16_t*)dres, (uint16_t*)dx, T);
  int st = zi::launch_status("zi_ln_bwd(dx)");
  if (st) return st;
  return launch_colred(2, dy, x, nullptr, mean, rstd, dgamma, dbeta, grads_f32, work, work_elems,
                       T, H, s, "zi_ln_bwd(gamma/beta)");
}

int zi_bias_grad(const void* dy, const void* u, void* du, void* db, int db_f32, float* work,
                 size_t work_elems, int T, int N, void* stream) {
  ZI_CHECK_ARG(dy && db && work && T > 0 && N > 0, "zi_bias_grad: bad arguments");
  ZI_CHECK_ARG(!u || du, "zi_bias_grad: gelu backward needs du");
  return launch_colred(u ? 1 : 0, dy, u, du, nullptr, nullptr, db, nullptr, db_f32, work,
                       work_elems, T, N, (cudaStream_t)stream, "zi_bias_grad");
}

int zi_softmax_ce(void* logits, const int64_t* targets, float* loss_rows, float* loss, int T, int V,
                  float scale, void* stream) {
  ZI_CHECK_ARG(logits && targets && loss_rows && loss && T > 0 && V > 0, "zi_softmax_ce: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  softmax_ce_kernel<<<T, 512, 0, s>>>((uint16_t*)logits, targets, loss_rows, V, scale);
  int st = zi::launch_status("zi_softmax_ce");
  if (st) return st;
  sum_kernel<<<1, 1024, 0, s>>>(loss_rows, T, 1.0f / T, loss);
  return zi::launch_status("zi_softmax_ce(sum)");
}

}  // extern "C"
