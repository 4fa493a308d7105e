// Fused HBM-bound kernels of the GPT block around the GEMMs (bf16 activations,
// fp32 math). Each reads its inputs once and writes its outputs once; column
// reductions (LayerNorm gamma/beta grads, bias grads) are deterministic:
// per-CTA fp32 partials reduced in a fixed order.
//
//   zi_ln_fwd      y = LN(x) * w + b            (+ x2 = x + r fused residual)
//   zi_ln_bwd      dx = LN'(dy) (+ dres); dgamma, dbeta and optionally the
//                  column sums of dres (a bias gradient) from the same pass
//   zi_gelu_fwd    y = gelu_tanh(u)
//   zi_bias_grad   column sums of dy, or du = gelu'(u) * dy and sums of du
//   zi_softmax_ce  per-row logsumexp, loss, dlogits = (softmax - onehot) * scale
#include <cstdlib>
#include <type_traits>

#include "bulk.cuh"
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

// two fp32 -> one bf16x2 word (a low, b high), RNE: one F2FP.PACK_AB instead of two
// conversions and a byte permute (same bits as tobf)
__device__ __forceinline__ uint32_t bf2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

template <int N>
__device__ __forceinline__ void st_row(uint16_t* p, const float* f) {
  if constexpr (N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      uint4 v;
      v.x = bf2(f[8 * i], f[8 * i + 1]);
      v.y = bf2(f[8 * i + 2], f[8 * i + 3]);
      v.z = bf2(f[8 * i + 4], f[8 * i + 5]);
      v.w = bf2(f[8 * i + 6], f[8 * i + 7]);
      reinterpret_cast<uint4*>(p)[i] = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      uint2 v;
      v.x = bf2(f[4 * i], f[4 * i + 1]);
      v.y = bf2(f[4 * i + 2], f[4 * i + 3]);
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
  zi::pdl_sync();
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

// Warp-per-row LayerNorm forward for H = 256 * VPL (H <= 2048): each lane owns VPL
// 8-column vectors (vector k at columns 256k + 8 * lane, so every k is one coalesced
// 512-byte segment per warp), all of a row's loads are issued before the first use,
// and the row statistics are warp shuffles only: no CTA barriers, so many rows'
// loads are in flight per SM (the CTA-per-row kernel stalls on __syncthreads).
// Same math as ln_fwd_kernel: bf16-rounded residual sum, two-pass mean / variance.
template <int VPL, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
ln_fwd_warp_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ r,
                   uint16_t* __restrict__ xsum, const uint16_t* __restrict__ w,
                   const uint16_t* __restrict__ b, uint16_t* __restrict__ y,
                   float* __restrict__ mean, float* __restrict__ rstd, int T, float eps) {
  zi::pdl_sync();
  constexpr int H = 256 * VPL;
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < T; row += nwarps) {
    const size_t base = (size_t)row * H + lane * 8;
    uint4 xv[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) xv[k] = *reinterpret_cast<const uint4*>(x + base + k * 256);
    if (r != nullptr) {
      uint4 rv[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) rv[k] = *reinterpret_cast<const uint4*>(r + base + k * 256);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        float a[8], c[8];
        ld_row<8>(reinterpret_cast<const uint16_t*>(&xv[k]), a);
        ld_row<8>(reinterpret_cast<const uint16_t*>(&rv[k]), c);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] + c[i];
        st_row<8>(reinterpret_cast<uint16_t*>(&xv[k]), a);     // bf16(x + r)
        *reinterpret_cast<uint4*>(xsum + base + k * 256) = xv[k];
      }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      float a[8];
      ld_row<8>(reinterpret_cast<const uint16_t*>(&xv[k]), a);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i];
    }
    const float mu = warp_sum(s) * (1.0f / H);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      float a[8];
      ld_row<8>(reinterpret_cast<const uint16_t*>(&xv[k]), a);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = a[i] - mu;
        q += d * d;
      }
    }
    const float rs = rsqrtf(warp_sum(q) * (1.0f / H) + eps);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      float a[8], wf[8], bv[8];
      ld_row<8>(reinterpret_cast<const uint16_t*>(&xv[k]), a);
      ld_row<8>(w + lane * 8 + k * 256, wf);
      ld_row<8>(b + lane * 8 + k * 256, bv);
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = (a[i] - mu) * rs * wf[i] + bv[i];
      uint4 o;
      st_row<8>(reinterpret_cast<uint16_t*>(&o), a);
      *reinterpret_cast<uint4*>(y + base + k * 256) = o;
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
}

// LayerNorm backward in one pass over dy, x (and dres):
//   dx = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)) with dxh = dy * w, + dres;
//   per-CTA column partials of dgamma = sum dy * xh, dbeta = sum dy and, when
//   asked, of sum dres (the bias gradient of the linear that produced dres).
// Rows stream through a LNB_STAGES-deep shared-memory ring filled by bulk
// async copies (one per input per stage, RPC contiguous rows), so the loads of
// the next stages are in flight while this one is reduced. The CTA folds its
// row slots in order and writes one partial row per set to
// part[set][blockIdx.x][H]; ln_fold_kernel sums the partials in CTA order.
constexpr int LNB_NT = 512, LNB_STAGES = 4;
template <int TPR>
struct LnbCta {
  static constexpr int NT = TPR > LNB_NT ? TPR : LNB_NT;
  static constexpr int RPC = NT / TPR;
};

template <int TPR, bool DRES>
constexpr size_t lnb_smem() {
  return (size_t)LNB_STAGES * (DRES ? 3 : 2) * LnbCta<TPR>::RPC * 8 * TPR * 2 + 64;
}

template <int TPR, bool DRES, bool RSUM>
__global__ void __launch_bounds__(LnbCta<TPR>::NT, LnbCta<TPR>::NT > LNB_NT ? 1 : 2)
ln_bwd_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
              const uint16_t* __restrict__ w, const float* __restrict__ mean,
              const float* __restrict__ rstd, const uint16_t* __restrict__ dres,
              uint16_t* __restrict__ dx, float* __restrict__ part, int T) {
  zi::pdl_sync();
  constexpr int H = 8 * TPR, RPC = LnbCta<TPR>::RPC, NT = LnbCta<TPR>::NT;
  constexpr int NIN = DRES ? 3 : 2, NS = RSUM ? 3 : 2;
  constexpr int ROWS_E = RPC * H;                    // elements per input per stage
  extern __shared__ __align__(128) uint16_t ring[];  // [stage][input][RPC * H]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)LNB_STAGES * NIN * ROWS_E);
  __shared__ float sm[32];
  const int t = threadIdx.x % TPR, slot = threadIdx.x / TPR;
  const int G = gridDim.x, ngroups = (T + RPC - 1) / RPC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < LNB_STAGES; ++s) bulk::mbar_init(&full[s], 1);
    bulk::fence_init();
  }
  __syncthreads();
  auto issue = [&](int i) {                          // thread 0: fill stage i % STAGES
    const int g = blockIdx.x + i * G;
    if (g >= ngroups) return;
    const int s = i % LNB_STAGES;
    const uint32_t bytes = (uint32_t)min(RPC, T - g * RPC) * H * 2;
    const size_t off = (size_t)g * RPC * H;
    uint16_t* st = ring + (size_t)s * NIN * ROWS_E;
    bulk::mbar_expect_tx(&full[s], NIN * bytes);
    bulk::g2s(st, dy + off, bytes, &full[s]);
    bulk::g2s(st + ROWS_E, x + off, bytes, &full[s]);
    if (DRES) bulk::g2s(st + 2 * ROWS_E, dres + off, bytes, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < LNB_STAGES; ++i) issue(i);
  float wf[8];
  ld_row<8>(w + t * 8, wf);
  float acc[NS][8];
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[k][i] = 0.f;
  // row statistics loaded one stage ahead (as in ln_bwd_split_kernel)
  float mu_n = 0.f, rs_n = 0.f;
  {
    const int row0 = blockIdx.x * RPC + slot;
    if (row0 < T) {
      mu_n = mean[row0];
      rs_n = rstd[row0];
    }
  }
  for (int i = 0;; ++i) {
    const int g = blockIdx.x + i * G;
    if (g >= ngroups) break;
    const int s = i % LNB_STAGES;
    const int row = g * RPC + slot;
    const bool live = row < T;
    const float mu = mu_n, rs = rs_n;
    {
      const int rn = (g + G) * RPC + slot;
      if (rn < T) {
        mu_n = mean[rn];
        rs_n = rstd[rn];
      }
    }
    bulk::mbar_wait(&full[s], (i / LNB_STAGES) & 1);
    const uint16_t* st = ring + (size_t)s * NIN * ROWS_E + slot * H + t * 8;
    float gv[8], xv[8], rv[8];
    ld_row<8>(st, gv);
    ld_row<8>(st + ROWS_E, xv);
    if (DRES) ld_row<8>(st + 2 * ROWS_E, rv);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      xv[k] = (xv[k] - mu) * rs;     // xh
      if (live) {
        acc[0][k] += gv[k] * xv[k];
        acc[1][k] += gv[k];
        if (RSUM) acc[NS - 1][k] += rv[k];
      }
      gv[k] *= wf[k];                // dxh
      s1 += gv[k];
      s2 += gv[k] * xv[k];
    }
    const float m1 = row_reduce<TPR>(s1, sm) * (1.0f / H);
    const float m2 = row_reduce<TPR>(s2, sm) * (1.0f / H);
    float o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      o[k] = rs * (gv[k] - m1 - xv[k] * m2);
      if (DRES) o[k] += rv[k];
    }
    if (live) st_row<8>(dx + (size_t)row * H + t * 8, o);
    __syncthreads();                 // stage s fully read: refill it
    if (threadIdx.x == 0) issue(i + LNB_STAGES);
  }
  // this CTA's partial rows: fold the RPC row slots in order (the ring is idle now:
  // every issued stage was consumed above)
  if constexpr (RPC == 1) {
#pragma unroll
    for (int k = 0; k < NS; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) part[((size_t)k * gridDim.x + blockIdx.x) * H + t * 8 + q] = acc[k][q];
  } else {
    float* red = reinterpret_cast<float*>(ring);     // RPC * H floats <= one stage
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) red[slot * H + t * 8 + q] = acc[k][q];
      __syncthreads();
      for (int c = threadIdx.x; c < H; c += NT) {
        float sum = 0.f;
        for (int q = 0; q < RPC; ++q) sum += red[q * H + c];
        part[((size_t)k * gridDim.x + blockIdx.x) * H + c] = sum;
      }
    }
  }
}

// LayerNorm backward for H = 2048 / 4096 / 8192 in two phases per ring stage, so the
// row statistics need no CTA-wide reductions: a stage holds R = 8192 / H rows of dy, x
// (and dres), filled by one bulk copy per input; 512 threads.
//   phase 1 (warp layout): W = H / 512 warps per row, each lane 16 columns, reduce
//     s1 = sum dxh and s2 = sum dxh * xh with shuffles; one (s1, s2) pair per warp and
//     the row's (mean, rstd) go to shared memory;
//   phase 2 (column layout): thread t owns CPT = H / 512 columns of every row (a warp
//     writes 32 * CPT contiguous elements of dx), sums the W pairs in warp order,
//     writes dx and accumulates its columns of dgamma / dbeta (/ sum dres) in row order.
// One __syncthreads between the phases and one to release the stage: 2 per R rows,
// against 5 per 2 rows for ln_bwd_kernel's CTA-wide row reductions. Deterministic: fixed
// per-row summation order, the CTA's rows in order, CTA partials folded in order.
// NT = 512: one CTA per SM with a 192 KB ring; NT = 256 (H <= 4096): two CTAs per SM
// with 96 KB rings each.
template <int H, bool DRES, int NT>
struct Lns {
  static constexpr int NW = NT / 32, W = H / 512, R = NW / W, CPT = H / NT;
  static constexpr int NIN = DRES ? 3 : 2;
  static constexpr int STAGE = NIN * R * H;                 // bf16 elements per stage
  static constexpr int NSTG = DRES ? 4 : 6;
  static constexpr int MINB = NT == 512 ? 1 : 2;
  static constexpr size_t SMEM = (size_t)NSTG * STAGE * 2 + NSTG * 8 + 16 * 16 + 64;
  static_assert(R >= 1, "a stage holds at least one row");
};

template <int H, bool DRES, bool RSUM, int NT>
__global__ void __launch_bounds__(NT, (Lns<H, DRES, NT>::MINB))
ln_bwd_split_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                    const uint16_t* __restrict__ w, const float* __restrict__ mean,
                    const float* __restrict__ rstd, const uint16_t* __restrict__ dres,
                    uint16_t* __restrict__ dx, float* __restrict__ part, int T) {
  zi::pdl_sync();
  using L = Lns<H, DRES, NT>;
  constexpr int R = L::R, W = L::W, CPT = L::CPT, NS = RSUM ? 3 : 2;
  constexpr int VE = CPT < 8 ? CPT : 8;                     // elements per vector access
  constexpr int NV = CPT / VE;                              // accesses per row
  extern __shared__ __align__(128) uint16_t ring[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)L::NSTG * L::STAGE);
  float2* red = reinterpret_cast<float2*>(full + L::NSTG);  // [16] per-warp (s1, s2)
  float2* stat = red + 16;                                  // [R] (mean, rstd)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, ngroups = (T + R - 1) / R;
  if (tid == 0) {
    for (int s = 0; s < L::NSTG; ++s) bulk::mbar_init(&full[s], 1);
    bulk::fence_init();
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int g = blockIdx.x + i * G;
    if (g >= ngroups) return;
    const int s = i % L::NSTG;
    const uint32_t bytes = (uint32_t)min(R, T - g * R) * H * 2;
    const size_t off = (size_t)g * R * H;
    uint16_t* st = ring + (size_t)s * L::STAGE;
    bulk::mbar_expect_tx(&full[s], L::NIN * bytes);
    bulk::g2s(st, dy + off, bytes, &full[s]);
    bulk::g2s(st + R * H, x + off, bytes, &full[s]);
    if (DRES) bulk::g2s(st + 2 * R * H, dres + off, bytes, &full[s]);
  };
  if (tid == 0)
    for (int i = 0; i < L::NSTG; ++i) issue(i);
  // phase-1 role: row pr of the stage, columns [pw * 512, +512): lane's 16 at
  // pw * 512 + k * 256 + lane * 8, k = 0, 1
  const int pr = warp / W, pw = warp % W;
  float g1[16];
  ld_row<8>(w + pw * 512 + lane * 8, g1);
  ld_row<8>(w + pw * 512 + 256 + lane * 8, g1 + 8);
  // phase-2 role: columns a * 512 * VE + tid * VE + [0, VE), a < NV
  float g2[CPT];
#pragma unroll
  for (int a = 0; a < NV; ++a) ld_row<VE>(w + (a * NT + tid) * VE, g2 + a * VE);
  float acc[NS][CPT];
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[k][c] = 0.f;
  // the row statistics are loaded one stage ahead: a load issued just before its use
  // left ~20 % of the warps' stall samples on the first (x - mean) (ncu,
  // profiles/r2_ln_bwd_split_ncu.md)
  float mu_n = 0.f, rs_n = 0.f;
  if (blockIdx.x < ngroups && pr < min(R, T - (int)blockIdx.x * R)) {
    mu_n = mean[blockIdx.x * R + pr];
    rs_n = rstd[blockIdx.x * R + pr];
  }
  for (int i = 0;; ++i) {
    const int g = blockIdx.x + i * G;
    if (g >= ngroups) break;
    const int s = i % L::NSTG;
    const int rows = min(R, T - g * R);
    const uint16_t* st = ring + (size_t)s * L::STAGE;
    const float mu = mu_n, rs = rs_n;
    if (g + G < ngroups && pr < min(R, T - (g + G) * R)) {
      mu_n = mean[(g + G) * R + pr];
      rs_n = rstd[(g + G) * R + pr];
    }
    bulk::mbar_wait(&full[s], (i / L::NSTG) & 1);
    if (pr < rows) {
      const uint16_t* gy = st + pr * H + pw * 512 + lane * 8;
      const uint16_t* gx = gy + R * H;
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float yv[8], xv[8];
        ld_row<8>(gy + k * 256, yv);
        ld_row<8>(gx + k * 256, xv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = yv[j] * g1[8 * k + j];
          s1 += d;
          s2 += d * ((xv[j] - mu) * rs);
        }
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        red[warp] = make_float2(s1, s2);
        if (pw == 0) stat[pr] = make_float2(mu, rs);
      }
    }
    __syncthreads();
    for (int r = 0; r < rows; ++r) {
      float m1 = 0.f, m2 = 0.f;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const float2 p = red[r * W + q];
        m1 += p.x;
        m2 += p.y;
      }
      m1 *= 1.0f / H;
      m2 *= 1.0f / H;
      const float2 ms = stat[r];
      const size_t grow = (size_t)(g * R + r) * H;
#pragma unroll
      for (int a = 0; a < NV; ++a) {
        const int col = (a * NT + tid) * VE;
        float yv[VE], xv[VE], rv[VE], o[VE];
        ld_row<VE>(st + r * H + col, yv);
        ld_row<VE>(st + R * H + r * H + col, xv);
        if (DRES) ld_row<VE>(st + 2 * R * H + r * H + col, rv);
#pragma unroll
        for (int j = 0; j < VE; ++j) {
          const float xh = (xv[j] - ms.x) * ms.y;
          const float d = yv[j] * g2[a * VE + j];
          acc[0][a * VE + j] += yv[j] * xh;
          acc[1][a * VE + j] += yv[j];
          if (RSUM) acc[NS - 1][a * VE + j] += rv[j];
          o[j] = ms.y * (d - m1 - xh * m2);
          if (DRES) o[j] += rv[j];
        }
        st_row<VE>(dx + grow + col, o);
      }
    }
    __syncthreads();                     // stage s and red / stat read by everyone
    if (tid == 0) issue(i + L::NSTG);
  }
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int j = 0; j < VE; ++j)
        part[((size_t)k * gridDim.x + blockIdx.x) * H + (a * NT + tid) * VE + j] = acc[k][a * VE + j];
}

// part[set][P][H] -> out_set[H] (bf16 RNE or fp32); per column, P is split into
// FOLD_SUB ordered runs summed by separate threads, then combined in run order:
// deterministic for a fixed P, and ~P / FOLD_SUB dependent loads per thread.
constexpr int FOLD_SUB = 32;
__global__ void __launch_bounds__(32 * FOLD_SUB)
ln_fold_kernel(const float* __restrict__ part, int P, int H, void* __restrict__ o0,
               void* __restrict__ o1, void* __restrict__ o2, int out_f32) {
  zi::pdl_sync();
  __shared__ float sm[FOLD_SUB][33];
  const int set = blockIdx.y, lane = threadIdx.x & 31, sub = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (col < H) {
    const int per = (P + FOLD_SUB - 1) / FOLD_SUB, p0 = sub * per, p1 = min(P, p0 + per);
    const float* src = part + (size_t)set * P * H + col;
#pragma unroll 4
    for (int p = p0; p < p1; ++p) s += __ldcg(src + (size_t)p * H);
  }
  sm[sub][lane] = s;
  __syncthreads();
  if (sub == 0 && col < H) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < FOLD_SUB; ++k) t += sm[k][lane];
    void* dst = set == 0 ? o0 : (set == 1 ? o1 : o2);
    if (out_f32) static_cast<float*>(dst)[col] = t;
    else static_cast<uint16_t*>(dst)[col] = tobf(t);
  }
}

// zi_fold_sets: up to ZI_FOLD_MAX_SETS independent folds in one launch (blockIdx.y = set),
// each exactly ln_fold_kernel's order: FOLD_SUB ordered runs, combined in run order.
struct FoldSets {
  zi_fold_set s[ZI_FOLD_MAX_SETS];
  int out_f32;
};
__global__ void __launch_bounds__(32 * FOLD_SUB)
fold_sets_kernel(const __grid_constant__ FoldSets f) {
  zi::pdl_sync();
  __shared__ float sm[FOLD_SUB][33];
  const zi_fold_set& d = f.s[blockIdx.y];
  const int lane = threadIdx.x & 31, sub = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  if (blockIdx.x * 32 >= d.N) return;            // whole CTA past this set's columns
  float s = 0.f;
  if (col < d.N) {
    const int per = (d.P + FOLD_SUB - 1) / FOLD_SUB, p0 = sub * per, p1 = min(d.P, p0 + per);
    const float* src = d.part + col;
#pragma unroll 4
    for (int p = p0; p < p1; ++p) s += __ldcg(src + (size_t)p * d.N);
  }
  sm[sub][lane] = s;
  __syncthreads();
  if (sub == 0 && col < d.N) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < FOLD_SUB; ++k) t += sm[k][lane];
    if (f.out_f32) static_cast<float*>(d.out)[col] = t;
    else static_cast<uint16_t*>(d.out)[col] = tobf(t);
  }
}

// y = gelu_tanh(u), 8 bf16 per thread per step (n % 8 == 0), grid-stride.
__global__ void __launch_bounds__(256)
gelu_fwd_kernel(const uint16_t* __restrict__ u, uint16_t* __restrict__ y, size_t n8) {
  zi::pdl_sync();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8;
       i += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    ld_row<8>(u + 8 * i, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = gelu_tanh(v[j]);
    st_row<8>(y + 8 * i, v);
  }
}

// Column reductions (bias grads, GELU-bwd + bias grad) over rows streamed
// through an NSTG-deep bulk-copy ring. CTA (column block, row chunk): C
// columns (8 per thread, C/8 threads), rows [r0, r1) in stages of R rows; one
// bulk copy per row and input. Each thread accumulates its 8 columns over the
// chunk in row order and writes one partial row part[chunk][N]; the fold kernel
// then sums the chunks in order: deterministic for a fixed grid.
//   MODE 0: out = sum_rows a                               (bias grad)
//   MODE 1: du = gelu_tanh'(u) * a -> d; out = sum_rows du (GELU bwd + fc1 bias grad)
constexpr int CRW_MAX_COLS = 4096;

template <int MODE, int NSTG>
__global__ void __launch_bounds__(CRW_MAX_COLS / 8)
colrow_kernel(const uint16_t* __restrict__ a, const uint16_t* __restrict__ u,
              uint16_t* __restrict__ d, float* __restrict__ part, int T, int N, int C, int R,
              int rows_per) {
  zi::pdl_sync();
  constexpr int NIN = MODE == 1 ? 2 : 1;
  extern __shared__ __align__(128) uint16_t ring[];   // [stage][input][R][C]
  const int SE = R * C;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NSTG * NIN * SE);
  const int c0 = blockIdx.x * C, W = min(C, N - c0);
  const int r0 = blockIdx.y * rows_per, r1 = min(T, r0 + rows_per);
  const int nst = r1 > r0 ? (r1 - r0 + R - 1) / R : 0;
  const int t = threadIdx.x;
  const bool colok = t * 8 < W;
  if (t == 0) {
    for (int s = 0; s < NSTG; ++s) bulk::mbar_init(&full[s], 1);
    bulk::fence_init();
  }
  __syncthreads();
  auto issue = [&](int i) {                          // thread 0: rows of stage i
    if (i >= nst) return;
    const int s = i % NSTG, rb = r0 + i * R, rows = min(R, r1 - rb);
    const uint32_t bytes = (uint32_t)W * 2;
    bulk::mbar_expect_tx(&full[s], NIN * rows * bytes);
    uint16_t* st = ring + (size_t)s * NIN * SE;
    for (int j = 0; j < rows; ++j) {
      const size_t off = (size_t)(rb + j) * N + c0;
      bulk::g2s(st + j * C, a + off, bytes, &full[s]);
      if (MODE == 1) bulk::g2s(st + SE + j * C, u + off, bytes, &full[s]);
    }
  };
  if (t == 0)
    for (int i = 0; i < NSTG; ++i) issue(i);
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  for (int i = 0; i < nst; ++i) {
    const int s = i % NSTG, rb = r0 + i * R, rows = min(R, r1 - rb);
    bulk::mbar_wait(&full[s], (i / NSTG) & 1);
    if (colok) {
      const uint16_t* st = ring + (size_t)s * NIN * SE + t * 8;
      for (int j = 0; j < rows; ++j) {
        float v[8];
        ld_row<8>(st + j * C, v);
        if (MODE == 1) {
          float uv[8];
          ld_row<8>(st + SE + j * C, uv);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            v[k] = __bfloat162float(__float2bfloat16_rn(v[k] * gelu_tanh_grad(uv[k])));
          st_row<8>(d + (size_t)(rb + j) * N + c0 + t * 8, v);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += v[k];
      }
    }
    __syncthreads();                                 // stage s read by everyone: refill
    if (t == 0) issue(i + NSTG);
  }
  if (colok) {
#pragma unroll
    for (int k = 0; k < 8; ++k) part[(size_t)blockIdx.y * N + c0 + t * 8 + k] = acc[k];
  }
}

// One CTA per row of V logits (bf16, in place): lse, loss_row = lse - l[t],
// dlogits = (exp(l - lse) - [j == t]) * scale written back as bf16.
__global__ void __launch_bounds__(512)
softmax_ce_kernel(uint16_t* __restrict__ logits, const int64_t* __restrict__ tgt,
                  float* __restrict__ loss_rows, int V, float scale) {
  zi::pdl_sync();
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

// Persistent, row-staged variant (V % 8 == 0, two rows fit in shared memory): one CTA
// per SM streams its rows through a 2-deep ring of whole bf16 rows filled by one bulk
// copy each, so row r+1 lands while row r is worked on, and the logits are read from
// HBM once (the CTA-per-row kernel reads them twice with one 16-byte load per thread
// in flight). The row work is issue-bound, so it is kept to ~8 instructions per
// logit: max on packed bf16 pairs (exact), then e = 2^(l*log2e - max*log2e) (one
// FFMA + one MUFU) summed in fp32 and parked as fp16 over the row in shared memory,
// then dlogits = e * (scale / sum) with the target's -scale applied once by the
// thread that owns it. lse = max + log(sum) from the fp32 sum, as in the CTA-per-row
// kernel (same loss; dlogits differ by the fp16 parking of e: relative 2^-11, under
// the bf16 output rounding).
constexpr int CE_NT = 1024;
__device__ __forceinline__ float ce_block_reduce(float v, float* red, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int k = 1; k < CE_NT / 32; ++k) r = is_max ? fmaxf(r, red[k]) : r + red[k];
  return r;   // red is rewritten only after the caller's next __syncthreads
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(CE_NT, 1)
softmax_ce_ring_kernel(uint16_t* __restrict__ logits, const int64_t* __restrict__ tgt,
                       float* __restrict__ loss_rows, int T, int V, int Vpad, float scale) {
  zi::pdl_sync();
  extern __shared__ __align__(128) uint16_t rowbuf[];     // [2][Vpad] bf16 + 2 mbarriers
  uint64_t* full = reinterpret_cast<uint64_t*>(rowbuf + 2 * (size_t)Vpad);
  __shared__ float red_m[CE_NT / 32], red_s[CE_NT / 32];
  constexpr float LOG2E = 1.4426950408889634f;
  const int V8 = V / 8;
  const uint32_t bytes = (uint32_t)V * 2;
  if (threadIdx.x == 0) {
    bulk::mbar_init(&full[0], 1);
    bulk::mbar_init(&full[1], 1);
    bulk::fence_init();
  }
  __syncthreads();
  auto issue = [&](int it) {                      // thread 0: row of iteration it
    const size_t row = (size_t)blockIdx.x + (size_t)it * gridDim.x;
    if (row >= (size_t)T) return;
    const int b = it & 1;
    bulk::mbar_expect_tx(&full[b], bytes);
    bulk::g2s(rowbuf + b * (size_t)Vpad, logits + row * V, bytes, &full[b]);
  };
  if (threadIdx.x == 0) {
    issue(0);
    issue(1);
  }
  for (int it = 0;; ++it) {
    const size_t row = (size_t)blockIdx.x + (size_t)it * gridDim.x;
    if (row >= (size_t)T) break;
    const int b = it & 1;
    const int t = (int)tgt[row];
    bulk::mbar_wait(&full[b], (it >> 1) & 1);
    uint16_t* R = rowbuf + b * (size_t)Vpad;
    uint4* S = reinterpret_cast<uint4*>(R);
    const float lt = threadIdx.x == 0 ? bf(R[t]) : 0.f;   // read before the barrier in the
                                                           // max reduce: e overwrites R below
    __nv_bfloat162 mx = __float2bfloat162_rn(-INFINITY);
    for (int i = threadIdx.x; i < V8; i += CE_NT) {
      const uint4 w = S[i];
      mx = __hmax2(mx, __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.x),
                               *reinterpret_cast<const __nv_bfloat162*>(&w.y)));
      mx = __hmax2(mx, __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w.z),
                               *reinterpret_cast<const __nv_bfloat162*>(&w.w)));
    }
    const float m = ce_block_reduce(fmaxf(__low2float(mx), __high2float(mx)), red_m, true);
    const float ml = m * LOG2E;
    float sum = 0.f;
    for (int i = threadIdx.x; i < V8; i += CE_NT) {
      float f[8];
      ld_row<8>(reinterpret_cast<const uint16_t*>(S + i), f);
      uint32_t h[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float e0 = ex2_approx(fmaf(f[2 * j], LOG2E, -ml));
        const float e1 = ex2_approx(fmaf(f[2 * j + 1], LOG2E, -ml));
        sum += e0;
        sum += e1;
        const __half2 hv = __floats2half2_rn(e0, e1);
        h[j] = *reinterpret_cast<const uint32_t*>(&hv);
      }
      S[i] = make_uint4(h[0], h[1], h[2], h[3]);  // e parked as fp16 in place (own chunk)
    }
    sum = ce_block_reduce(sum, red_s, false);
    if (threadIdx.x == 0) loss_rows[row] = m + __logf(sum) - lt;
    const float c = scale / sum;
    uint16_t* L = logits + row * V;
    for (int i = threadIdx.x; i < V8; i += CE_NT) {
      const uint4 w = S[i];
      const uint32_t h[4] = {w.x, w.y, w.z, w.w};
      float f[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&h[j]));
        f[2 * j] = e.x * c;
        f[2 * j + 1] = e.y * c;
      }
      if (i == (t >> 3)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] -= (j == (t & 7)) ? scale : 0.f;
      }
      st_row<8>(L + 8 * i, f);
    }
    __syncthreads();                              // row buffer b and red_* fully read
    if (threadIdx.x == 0) issue(it + 2);
  }
}

__global__ void sum_kernel(const float* __restrict__ v, int n, float scale, float* __restrict__ out) {
  zi::pdl_sync();
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
    case 16: zi::launch_pdl(KERNEL<16>, dim3(GRID), dim3(256), 0, STREAM, __VA_ARGS__); break;                     \
    case 32: zi::launch_pdl(KERNEL<32>, dim3(GRID), dim3(256), 0, STREAM, __VA_ARGS__); break;                     \
    case 64: zi::launch_pdl(KERNEL<64>, dim3(GRID), dim3(256), 0, STREAM, __VA_ARGS__); break;                     \
    case 128: zi::launch_pdl(KERNEL<128>, dim3(GRID), dim3(256), 0, STREAM, __VA_ARGS__); break;                   \
    case 256: zi::launch_pdl(KERNEL<256>, dim3(GRID), dim3(256), 0, STREAM, __VA_ARGS__); break;                   \
    case 512: zi::launch_pdl(KERNEL<512>, dim3(GRID), dim3(512), 0, STREAM, __VA_ARGS__); break;                   \
    case 1024: zi::launch_pdl(KERNEL<1024>, dim3(GRID), dim3(1024), 0, STREAM, __VA_ARGS__); break;                \
    default: zi::set_error("LayerNorm: hidden size %d not in {128..8192, power of 2}", H); \
      return ZI_EINVAL;                                                                    \
  }

// ZI_LN_BWD_LEGACY=1: the CTA-reduction LayerNorm backward for every H (A/B only)
static bool ln_bwd_legacy() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZI_LN_BWD_LEGACY");
    v = e && atoi(e) ? 1 : 0;
  }
  return v == 1;
}

static int ln_grid(int T, int H) {
  const int tpr = H / 8;
  const int rpc = tpr >= 256 ? 1 : 256 / tpr;
  const int need = (T + rpc - 1) / rpc;
  const int cap = sm_count() * 8;
  return need < cap ? need : cap;
}

template <int TPR, bool DRES, bool RSUM>
static int launch_ln_bwd3(int grid, cudaStream_t s, const uint16_t* dy, const uint16_t* x,
                          const uint16_t* w, const float* mean, const float* rstd,
                          const uint16_t* dres, uint16_t* dx, float* part, int T) {
  constexpr size_t smem = lnb_smem<TPR, DRES>();
  static bool attr = false;
  if (!attr) {
    ZI_CUDA(cudaFuncSetAttribute(ln_bwd_kernel<TPR, DRES, RSUM>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "cudaFuncSetAttribute(ln_bwd)");
    attr = true;
  }
  zi::launch_pdl(ln_bwd_kernel<TPR, DRES, RSUM>, dim3(grid), dim3(LnbCta<TPR>::NT), smem, s, dy, x, w, mean, rstd, dres,
                                                                     dx, part, T);
  return ZI_OK;
}

template <int H, bool DRES, bool RSUM, int NT>
static int launch_ln_split3(int grid, cudaStream_t s, const uint16_t* dy, const uint16_t* x,
                            const uint16_t* w, const float* mean, const float* rstd,
                            const uint16_t* dres, uint16_t* dx, float* part, int T) {
  constexpr size_t smem = Lns<H, DRES, NT>::SMEM;
  static bool attr = false;
  if (!attr) {
    ZI_CUDA(cudaFuncSetAttribute(ln_bwd_split_kernel<H, DRES, RSUM, NT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "cudaFuncSetAttribute(ln_bwd_split)");
    attr = true;
  }
  zi::launch_pdl(ln_bwd_split_kernel<H, DRES, RSUM, NT>, dim3(grid), dim3(NT), smem, s, dy, x, w,
                 mean, rstd, dres, dx, part, T);
  return ZI_OK;
}

template <int H, int NT>
static int launch_ln_split(int grid, cudaStream_t s, bool rsum, const uint16_t* dy,
                           const uint16_t* x, const uint16_t* w, const float* mean,
                           const float* rstd, const uint16_t* dres, uint16_t* dx, float* part,
                           int T) {
  if (rsum) return launch_ln_split3<H, true, true, NT>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
  if (dres) return launch_ln_split3<H, true, false, NT>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
  return launch_ln_split3<H, false, false, NT>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
}

template <int TPR>
static int launch_ln_bwd(int grid, cudaStream_t s, bool rsum, const uint16_t* dy,
                         const uint16_t* x, const uint16_t* w, const float* mean,
                         const float* rstd, const uint16_t* dres, uint16_t* dx, float* part,
                         int T) {
  if (rsum) return launch_ln_bwd3<TPR, true, true>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
  if (dres) return launch_ln_bwd3<TPR, true, false>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
  return launch_ln_bwd3<TPR, false, false>(grid, s, dy, x, w, mean, rstd, dres, dx, part, T);
}

// The row pass of zi_ln_bwd: dx, and the CTA partials of dgamma / dbeta (/ sum dres)
// as part[set][P][H]; returns P (the grid) through *nparts.
static int ln_bwd_rows(const void* dy, const void* x, const void* w, const float* mean,
                       const float* rstd, const void* dres, void* dx, bool rs, float* part,
                       size_t part_elems, int T, int H, int* nparts, cudaStream_t s) {
  ZI_CHECK_ARG(zi::aligned(dy, 16) && zi::aligned(x, 16) && zi::aligned(dx, 16) &&
               (!dres || zi::aligned(dres, 16)), "zi_ln_bwd: rows must be 16-byte aligned");
  ZI_CHECK_ARG(H >= 128 && H <= 8192 && (H & (H - 1)) == 0, "zi_ln_bwd: H must be 128..8192, power of 2");
  const int tpr = H / 8;
  const bool split = H >= 2048 && !ln_bwd_legacy();
  // (256-thread CTAs, two per SM with 96 KB rings, measured 9 % slower than one 512-thread
  // CTA with a 192 KB ring: 40.6 vs 37.2 us on 8192 x 2048)
  const int snt = 512;
  const int rpc = split ? snt * 16 / H : (tpr >= LNB_NT ? 1 : LNB_NT / tpr);
  int grid = (split ? (snt == 256 ? 2 : 1) : (tpr > LNB_NT ? 1 : 2)) * sm_count();
  if (grid > (T + rpc - 1) / rpc) grid = (T + rpc - 1) / rpc;
  const int sets = rs ? 3 : 2;
  ZI_CHECK_ARG(part_elems >= (size_t)sets * grid * H, "zi_ln_bwd: partials need %zu floats",
               (size_t)sets * grid * H);
  auto DY = (const uint16_t*)dy, X = (const uint16_t*)x, W = (const uint16_t*)w,
       DR = (const uint16_t*)dres;
  auto DX = (uint16_t*)dx;
  int st = ZI_OK;
  if (split) {
    if (H == 2048) st = launch_ln_split<2048, 512>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T);
    else if (H == 4096) st = launch_ln_split<4096, 512>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T);
    else st = launch_ln_split<8192, 512>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T);
  } else switch (tpr) {
    case 16: st = launch_ln_bwd<16>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 32: st = launch_ln_bwd<32>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 64: st = launch_ln_bwd<64>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 128: st = launch_ln_bwd<128>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 256: st = launch_ln_bwd<256>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 512: st = launch_ln_bwd<512>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
    case 1024: st = launch_ln_bwd<1024>(grid, s, rs, DY, X, W, mean, rstd, DR, DX, part, T); break;
  }
  if (st) return st;
  *nparts = grid;
  return zi::launch_status("zi_ln_bwd(dx)");
}

extern "C" {

int zi_ln_fwd(const void* x, const void* resid, void* xsum, const void* w, const void* b, void* y,
              float* mean, float* rstd, int T, int H, float eps, void* stream) {
  ZI_CHECK_ARG(x && w && b && y && mean && rstd && T > 0, "zi_ln_fwd: bad arguments");
  ZI_CHECK_ARG(!resid || xsum, "zi_ln_fwd: resid needs xsum");
  cudaStream_t s = (cudaStream_t)stream;
  ZI_CHECK_ARG(H >= 128 && H <= 8192 && (H & (H - 1)) == 0, "zi_ln_fwd: H must be 128..8192, power of 2");
  if (H >= 512 && H <= 2048) {   // warp per row: 8 rows per 256-thread CTA
    const int grid = (T + 7) / 8;
    auto X = (const uint16_t*)x, R = (const uint16_t*)resid, W = (const uint16_t*)w,
         B = (const uint16_t*)b;
    auto XS = (uint16_t*)xsum, Y = (uint16_t*)y;
    if (H == 512) zi::launch_pdl(ln_fwd_warp_kernel<2>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
    else if (H == 1024) zi::launch_pdl(ln_fwd_warp_kernel<4>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
    else {
      // register budget for 3 resident CTAs (80 registers, a small spill): 24 warps per SM
      // keep more row loads in flight than 16 (8192 x 2048: fwd 15.9 vs 21.4 us, with the
      // residual 26.4 vs 33.8 us); ZI_LNF_MINB=1/2/4 for A/B
      static int minb = -1;
      if (minb < 0) {
        const char* e = getenv("ZI_LNF_MINB");
        minb = e ? atoi(e) : 3;
      }
      if (minb == 3) zi::launch_pdl(ln_fwd_warp_kernel<8, 3>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
      else if (minb == 2) zi::launch_pdl(ln_fwd_warp_kernel<8, 2>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
      else if (minb == 4) zi::launch_pdl(ln_fwd_warp_kernel<8, 4>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
      else zi::launch_pdl(ln_fwd_warp_kernel<8>, dim3(grid), dim3(256), 0, s, X, R, XS, W, B, Y, mean, rstd, T, eps);
    }
    return zi::launch_status("zi_ln_fwd");
  }
  const int grid = ln_grid(T, H);
  TPR_DISPATCH(H, ln_fwd_kernel, grid, s, (const uint16_t*)x, (const uint16_t*)resid,
               (uint16_t*)xsum, (const uint16_t*)w, (const uint16_t*)b, (uint16_t*)y, mean, rstd,
               T, eps);
  return zi::launch_status("zi_ln_fwd");
}

// work layout: [0, 1024) reserved (zero), then the fp32 partial rows
static int launch_colred(int mode, const void* a, const void* u, void* d, void* out, int out_f32,
                         float* work, size_t work_elems, int T, int N, cudaStream_t s,
                         const char* name) {
  ZI_CHECK_ARG(N % 8 == 0, "%s: N must be a multiple of 8", name);
  ZI_CHECK_ARG(zi::aligned(a, 16) && (!u || zi::aligned(u, 16)) && (!d || zi::aligned(d, 16)),
               "%s: rows must be 16-byte aligned", name);
  const int cblocks = (N + CRW_MAX_COLS - 1) / CRW_MAX_COLS;
  const int C = ((N + cblocks - 1) / cblocks + 7) / 8 * 8;
  const int nt = C / 8;
  const int nin = mode == 1 ? 2 : 1;
  int R = 16384 / (C * 2);
  R = R < 1 ? 1 : (R > 8 ? 8 : R);
  // ring depth: the bulk copies in flight per SM set the bandwidth (~3 us of HBM latency
  // under load x 44 GB/s per SM needs >= 130 KB in flight), so fill ~190 KB per SM
  const size_t stage_bytes = (size_t)nin * R * C * 2;
  int per_sm = 2;   // enough bytes in flight per SM; more CTAs only add partial rows
  if (4 * stage_bytes * per_sm > 200000) per_sm = 1;
  const int nstg = 8 * stage_bytes * per_sm <= 197000 ? 8 : (6 * stage_bytes * per_sm <= 197000 ? 6 : 4);
  const size_t smem = (size_t)nstg * stage_bytes + 64;
  int chunks = (sm_count() * per_sm + cblocks - 1) / cblocks;
  const int max_chunks = (T + R - 1) / R;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  const int rows_per = ((T + chunks - 1) / chunks + R - 1) / R * R;
  chunks = (T + rows_per - 1) / rows_per;
  ZI_CHECK_ARG(work_elems >= 1024 + (size_t)chunks * N, "%s: work needs %zu floats", name,
               1024 + (size_t)chunks * N);
  float* part = work + 1024;
  static bool attr = false;
  if (!attr) {
    for (auto k : {colrow_kernel<0, 4>, colrow_kernel<0, 6>, colrow_kernel<0, 8>,
                   colrow_kernel<1, 4>, colrow_kernel<1, 6>, colrow_kernel<1, 8>})
      ZI_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
              "cudaFuncSetAttribute(colrow)");
    attr = true;
  }
  dim3 grid(cblocks, chunks);
  const uint16_t* A = static_cast<const uint16_t*>(a);
  const uint16_t* U = static_cast<const uint16_t*>(u);
  uint16_t* D = static_cast<uint16_t*>(d);
#define ZI_COLROW(MODE, NS) zi::launch_pdl(colrow_kernel<MODE, NS>, dim3(grid), dim3(nt), smem, s, A, U, D, part, T, N, C, R, rows_per)
  if (mode == 0) {
    if (nstg == 8) ZI_COLROW(0, 8); else if (nstg == 6) ZI_COLROW(0, 6); else ZI_COLROW(0, 4);
  } else {
    if (nstg == 8) ZI_COLROW(1, 8); else if (nstg == 6) ZI_COLROW(1, 6); else ZI_COLROW(1, 4);
  }
#undef ZI_COLROW
  int st = zi::launch_status(name);
  if (st) return st;
  zi::launch_pdl(ln_fold_kernel, dim3(dim3((N + 31) / 32, 1)), dim3(32 * FOLD_SUB), 0, s, part, chunks, N, out, nullptr,
                                                                 nullptr, out_f32);
  return zi::launch_status(name);
}

int zi_ln_bwd(const void* dy, const void* x, const void* w, const float* mean, const float* rstd,
              const void* dres, void* dx, void* dgamma, void* dbeta, void* dres_sum, int grads_f32,
              float* work, size_t work_elems, int T, int H, void* stream) {
  ZI_CHECK_ARG(dy && x && w && mean && rstd && dx && dgamma && dbeta && work, "zi_ln_bwd: NULL");
  ZI_CHECK_ARG(!dres_sum || dres, "zi_ln_bwd: dres_sum needs dres");
  ZI_CHECK_ARG(work_elems > 1024, "zi_ln_bwd: work too small");
  cudaStream_t s = (cudaStream_t)stream;
  // work[0, 1024) holds the column-reduction counters (must stay zero); partials follow
  float* part = work + 1024;
  const int sets = dres_sum ? 3 : 2;
  int grid = 0;
  int st = ln_bwd_rows(dy, x, w, mean, rstd, dres, dx, dres_sum != nullptr, part, work_elems - 1024,
                       T, H, &grid, s);
  if (st) return st;
  zi::launch_pdl(ln_fold_kernel, dim3(dim3((H + 31) / 32, sets)), dim3(32 * FOLD_SUB), 0, s, part, grid, H, dgamma, dbeta, dres_sum,
                                                          grads_f32);
  return zi::launch_status("zi_ln_bwd(fold)");
}

int zi_ln_bwd_partials(const void* dy, const void* x, const void* w, const float* mean,
                       const float* rstd, const void* dres, void* dx, int dres_sum, float* part,
                       size_t part_elems, int T, int H, int* nparts, void* stream) {
  ZI_CHECK_ARG(dy && x && w && mean && rstd && dx && part && nparts, "zi_ln_bwd_partials: NULL");
  ZI_CHECK_ARG(!dres_sum || dres, "zi_ln_bwd_partials: dres_sum needs dres");
  return ln_bwd_rows(dy, x, w, mean, rstd, dres, dx, dres_sum != 0, part, part_elems, T, H, nparts,
                     (cudaStream_t)stream);
}

int zi_fold_sets(const zi_fold_set* sets, int n, int out_f32, void* stream) {
  ZI_CHECK_ARG(sets && n >= 1 && n <= ZI_FOLD_MAX_SETS, "zi_fold_sets: 1..%d sets", ZI_FOLD_MAX_SETS);
  FoldSets f = {};
  int maxn = 0;
  for (int i = 0; i < n; ++i) {
    ZI_CHECK_ARG(sets[i].part && sets[i].out && sets[i].P > 0 && sets[i].N > 0,
                 "zi_fold_sets: bad set %d", i);
    f.s[i] = sets[i];
    if (sets[i].N > maxn) maxn = sets[i].N;
  }
  f.out_f32 = out_f32;
  zi::launch_pdl(fold_sets_kernel, dim3((maxn + 31) / 32, n), dim3(32 * FOLD_SUB), 0,
                 (cudaStream_t)stream, f);
  return zi::launch_status("zi_fold_sets");
}

int zi_colsum_fold(const float* part, int P, int N, void* out, int out_f32, void* stream) {
  ZI_CHECK_ARG(part && out && P > 0 && N > 0, "zi_colsum_fold: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  zi::launch_pdl(ln_fold_kernel, dim3(dim3((N + 31) / 32, 1)), dim3(32 * FOLD_SUB), 0, s, part, P, N, out, nullptr,
                                                                 nullptr, out_f32);
  return zi::launch_status("zi_colsum_fold");
}

int zi_gelu_fwd(const void* u, void* y, size_t n, void* stream) {
  ZI_CHECK_ARG(u && y && n % 8 == 0, "zi_gelu_fwd: need n % 8 == 0");
  ZI_CHECK_ARG(zi::aligned(u, 16) && zi::aligned(y, 16), "zi_gelu_fwd: 16-byte aligned buffers");
  const size_t n8 = n / 8;
  size_t g = (n8 + 255) / 256;
  const size_t cap = (size_t)sm_count() * 8;
  if (g > cap) g = cap;
  if (g == 0) return ZI_OK;
  zi::launch_pdl(gelu_fwd_kernel, dim3((unsigned)g), dim3(256), 0, (cudaStream_t)stream, (const uint16_t*)u, (uint16_t*)y, n8);
  return zi::launch_status("zi_gelu_fwd");
}

int zi_bias_grad(const void* dy, const void* u, void* du, void* db, int db_f32, float* work,
                 size_t work_elems, int T, int N, void* stream) {
  ZI_CHECK_ARG(dy && db && work && T > 0 && N > 0, "zi_bias_grad: bad arguments");
  ZI_CHECK_ARG(!u || du, "zi_bias_grad: gelu backward needs du");
  return launch_colred(u ? 1 : 0, dy, u, du, db, db_f32, work, work_elems, T, N,
                       (cudaStream_t)stream, "zi_bias_grad");
}

int zi_softmax_ce(void* logits, const int64_t* targets, float* loss_rows, float* loss, int T, int V,
                  float scale, void* stream) {
  ZI_CHECK_ARG(logits && targets && loss_rows && loss && T > 0 && V > 0, "zi_softmax_ce: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  const int Vpad = (V + 63) / 64 * 64;                    // 128-byte aligned row slots
  const size_t ring_smem = 2 * (size_t)Vpad * 2 + 16;
  if (V % 8 == 0 && zi::aligned(logits, 16) && ring_smem <= 220 * 1024) {
    static bool attr = false;
    if (!attr) {
      ZI_CUDA(cudaFuncSetAttribute(softmax_ce_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   220 * 1024), "cudaFuncSetAttribute(softmax_ce)");
      attr = true;
    }
    const int grid = T < sm_count() ? T : sm_count();
    zi::launch_pdl(softmax_ce_ring_kernel, dim3(grid), dim3(CE_NT), ring_smem, s, (uint16_t*)logits, targets, loss_rows, T,
                                                           V, Vpad, scale);
  } else {
    zi::launch_pdl(softmax_ce_kernel, dim3(T), dim3(512), 0, s, (uint16_t*)logits, targets, loss_rows, V, scale);
  }
  int st = zi::launch_status("zi_softmax_ce");
  if (st) return st;
  zi::launch_pdl(sum_kernel, dim3(1), dim3(1024), 0, s, loss_rows, T, 1.0f / T, loss);
  return zi::launch_status("zi_softmax_ce(sum)");
}

}  // extern "C"
