// Causal multi-head attention of the GPT block on the 5th-gen tensor cores, forward and a
// deterministic backward ("reductions run in fixed order everywhere").
//
// Layout (the engine's, gpt.py): qkv is [B*S, 3*hd] bf16 row-major, head h of q / k / v at
// columns h*D, hd + h*D, 2*hd + h*D; o and do are [B*S, hd]; dqkv like qkv. lse / delta
// are fp32 [B*H*S] ((b*H + h)*S + s). D (head dim) in {64, 128}, S % 128 == 0.
//
// Every kernel is one CTA per 128-row tile of one (batch, head), 6 warps:
//   warp 0      TMA producer: 64 x 64 SWIZZLE_128B boxes of the operand tiles;
//   warp 1      TMEM allocator + the single thread issuing tcgen05.mma (M = 128, fp32
//               accumulators in TMEM, operands from shared memory);
//   warps 2..5  one thread per tile row (= TMEM lane): tcgen05.ld of score rows, the
//               softmax / gradient elementwise work, bf16 probability tiles written back
//               to shared memory for the next MMA, and the epilogue.
// The probability / gradient tiles a thread writes (its own row, K-major) are read by the
// next MMA either K-major or, reinterpreted, MN-major (tc.cuh), so no transposes exist.
//
//   forward   per q tile: S = Q K_j^T (double-buffered in TMEM, so S_{j+1} overlaps the
//             softmax of S_j) -> online softmax in the log2 domain -> P (bf16, smem) ->
//             O += P V_j (TMEM; rows rescaled in place when their running max moves).
//             Writes O and lse2 = m + log2(l).
//   dK / dV   per kv tile j (q tiles i >= j, in order): S^T = K Q_i^T, dP^T = V dO_i^T,
//             P^T = exp2(S^T c - lse2), dS^T = P^T (dP^T - delta), then dV += P^T dO_i and
//             dK += dS^T Q_i accumulate in TMEM.
//   dQ        per q tile i (kv tiles j <= i, in order): S, dP, P, dS as above (row form),
//             dQ += dS K_j in TMEM.
// No atomics: each output row is produced by one CTA that sums its terms in a fixed
// order, so the backward is bitwise reproducible run to run and across placements.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace zi {
namespace attn {

using namespace zi::tc;

constexpr int THREADS = 192;
constexpr int PB = 128 * 128 * 2;            // one 128 x 128 bf16 tile
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// 128 rows x D columns of a bf16 matrix (box 64 x 64) -> chunk regions of 16 KiB
template <int D>
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                          int col0, int row0) {
#pragma unroll
  for (int kc = 0; kc < D / 64; ++kc)
#pragma unroll
    for (int rh = 0; rh < 2; ++rh)
      tma_load_2d(dst + kc * 16384 + rh * 8192, map, bar, col0 + kc * 64, row0 + rh * 64);
}

// k-step kk (16 deep) of a 128-row tile read K-major / MN-major (tc.cuh convention)
__device__ __forceinline__ uint64_t kdesc(const uint8_t* base, int kk) {
  return sdesc_sw128(smem_u32(base) + (kk >> 2) * 16384 + (kk & 3) * 32, 16);
}
__device__ __forceinline__ uint64_t mndesc(const uint8_t* base, int kk) {
  return sdesc_sw128(smem_u32(base) + kk * 2048, 16384);
}

// 16-byte piece g (elements 8g .. 8g+7) of row r of a 128-row K-major tile
__device__ __forceinline__ void st_piece(uint8_t* tile, int r, int g, uint4 v) {
  *reinterpret_cast<uint4*>(tile + (g >> 3) * 16384 + r * 128 + (((g & 7) ^ (r & 7)) << 4)) = v;
}

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// D[128 x N] (+)= A B over `ksteps` 16-deep steps; A K-major, B K- or MN-major
template <bool B_MN>
__device__ __forceinline__ void mma_tile(uint32_t d, const uint8_t* a, const uint8_t* b,
                                         int ksteps, uint32_t idesc, bool accumulate) {
  for (int kk = 0; kk < ksteps; ++kk)
    umma_bf16(d, kdesc(a, kk), B_MN ? mndesc(b, kk) : kdesc(b, kk), idesc,
              (accumulate || kk > 0) ? 1u : 0u);
}

// one row of D fp32 TMEM columns (x scale) -> bf16 global (16-byte stores)
template <int D>
__device__ __forceinline__ void store_row(uint32_t taddr, float scale, __nv_bfloat16* dst) {
#pragma unroll
  for (int cc = 0; cc < D / 32; ++cc) {
    uint32_t o[32];
    tmem_ld32(taddr + cc * 32, o);
    uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint4 v;
      v.x = pack_bf16(u2f(o[8 * g + 0]) * scale, u2f(o[8 * g + 1]) * scale);
      v.y = pack_bf16(u2f(o[8 * g + 2]) * scale, u2f(o[8 * g + 3]) * scale);
      v.z = pack_bf16(u2f(o[8 * g + 4]) * scale, u2f(o[8 * g + 5]) * scale);
      v.w = pack_bf16(u2f(o[8 * g + 6]) * scale, u2f(o[8 * g + 7]) * scale);
      d4[g] = v;
    }
  }
}

__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               ::"r"(smem_u32(slot)), "r"(512) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free512(uint32_t tmem) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
               : "memory");
}

// ============================================================================ forward
template <int D>
struct Fwd {
  static constexpr int TB = 128 * D * 2;
  static constexpr int Q = 0, K = TB, V = 3 * TB, P = 5 * TB, BAR = 5 * TB + PB;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
fwd_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
           float* __restrict__ lse, int B, int H, int S, int hd, float sl2) {
  using L = Fwd<D>;
  constexpr int TB = L::TB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sQ = sm + L::Q, *sK = sm + L::K, *sV = sm + L::V, *sP = sm + L::P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = bar + 3, *v_full = bar + 5,
           *v_empty = bar + 7, *s_full = bar + 9, *s_free = bar + 11, *p_full = bar + 13,
           *pv_done = bar + 14;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 16);

  const int nq = S / 128, BH = B * H;
  const int i = nq - 1 - (int)blockIdx.x / BH;     // long causal rows first
  const int bh = (int)blockIdx.x % BH, b = bh / H, h = bh % H;
  const int nkv = i + 1, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1); mbar_init(&s_free[s], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t tS0 = tmem, tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, TB);
      load_tile<D>(sQ, &tm, q_full, h * D, row0 + i * 128);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], TB);
        load_tile<D>(sK + s * TB, &tm, &k_full[s], hd + h * D, row0 + j * 128);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], TB);
        load_tile<D>(sV + s * TB, &tm, &v_full[s], 2 * hd + h * D, row0 + j * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_o = idesc_bf16_f32(128, D, false, true);
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      fence_after_sync();
      mma_tile<false>(tS0, sQ, sK, D / 16, id_s, false);
      umma_commit(&k_empty[0]);
      umma_commit(&s_full[0]);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) {                       // S_{j+1} overlaps the softmax of S_j
          const int n = j + 1, sb = n & 1;
          if (n >= 2) mbar_wait(&s_free[sb], ((n - 2) >> 1) & 1);
          mbar_wait(&k_full[sb], (n >> 1) & 1);
          fence_after_sync();
          mma_tile<false>(tS0 + sb * 128, sQ, sK + sb * TB, D / 16, id_s, false);
          umma_commit(&k_empty[sb]);
          umma_commit(&s_full[sb]);
        }
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[j & 1], (j >> 1) & 1);
        fence_after_sync();
        mma_tile<true>(tO, sP, sV + (j & 1) * TB, 8, id_o, j > 0);
        umma_commit(&v_empty[j & 1]);
        umma_commit(pv_done);
      }
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      fence_after_sync();
      float x[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t t[32];
        tmem_ld32(tS0 + sb * 128 + lo + c * 32, t);
#pragma unroll
        for (int k = 0; k < 32; ++k) x[c * 32 + k] = u2f(t[k]) * sl2;
      }
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[sb]);
      if (j == i) {                              // diagonal tile: key index > query index
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) x[c] = -INFINITY;
      }
      float mx = m;
#pragma unroll
      for (int c = 0; c < 128; ++c) mx = fmaxf(mx, x[c]);
      const float alpha = ex2(m - mx);           // 0 on the first tile (m = -inf)
      uint32_t pk[64];
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const float p0 = ex2(x[2 * c] - mx), p1 = ex2(x[2 * c + 1] - mx);
        rs += p0 + p1;
        pk[c] = pack_bf16(p0, p1);
      }
      l = l * alpha + rs;
      m = mx;
      if (j >= 1) {
        mbar_wait(pv_done, (j - 1) & 1);         // O_{j-1} complete, P buffer free
        fence_after_sync();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(tO + lo + cc * 32, o);
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(u2f(o[k]) * alpha);
            tmem_st32(tO + lo + cc * 32, o);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < 16; ++g)
        st_piece(sP, r, g, make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]));
      fence_proxy_async_smem();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(pv_done, (nkv - 1) & 1);
    fence_after_sync();
    const size_t row = (size_t)row0 + i * 128 + r;
    store_row<D>(tO + lo, 1.f / l, out + row * hd + h * D);
    lse[(size_t)bh * S + i * 128 + r] = m + __log2f(l);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
}

// =================================================================== backward: dK, dV
template <int D>
struct Bkv {
  static constexpr int TB = 128 * D * 2;
  static constexpr int K = 0, V = TB, Q = 2 * TB, DO = 3 * TB, PT = 4 * TB, DST = 4 * TB + PB,
                       LD = 4 * TB + 2 * PB, BAR = LD + 2 * 256 * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_do,
                const float* __restrict__ lse, const float* __restrict__ delta,
                __nv_bfloat16* __restrict__ dqkv, int B, int H, int S, int hd, float sl2,
                float scale) {
  using L = Bkv<D>;
  constexpr int TB = L::TB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sK = sm + L::K, *sV = sm + L::V, *sQ = sm + L::Q, *sdO = sm + L::DO,
          *sPT = sm + L::PT, *sdST = sm + L::DST;
  float* sLD = reinterpret_cast<float*>(sm + L::LD);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *kv_full = bar, *qdo_full = bar + 1, *qdo_empty = bar + 2, *st_full = bar + 3,
           *st_free = bar + 4, *ps_full = bar + 5, *ps_empty = bar + 6, *acc_done = bar + 7;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);

  const int nq = S / 128, BH = B * H;
  const int j = (int)blockIdx.x / BH;            // kv tile; small j = many q tiles, first
  const int bh = (int)blockIdx.x % BH, b = bh / H, h = bh % H;
  const int nit = nq - j, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1); mbar_init(qdo_full, 1); mbar_init(qdo_empty, 1);
    mbar_init(st_full, 1); mbar_init(st_free, 4); mbar_init(ps_full, 4);
    mbar_init(ps_empty, 1); mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
    prefetch_map(&tm_do);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t tST = tmem, tdPT = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * TB);
      load_tile<D>(sK, &tm, kv_full, hd + h * D, row0 + j * 128);
      load_tile<D>(sV, &tm, kv_full, 2 * hd + h * D, row0 + j * 128);
      for (int it = 0; it < nit; ++it) {
        const int i = j + it;
        mbar_wait(qdo_empty, (it & 1) ^ 1);
        mbar_expect_tx(qdo_full, 2 * TB);
        load_tile<D>(sQ, &tm, qdo_full, h * D, row0 + i * 128);
        load_tile<D>(sdO, &tm_do, qdo_full, h * D, row0 + i * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_d = idesc_bf16_f32(128, D, false, true);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < nit; ++it) {
        mbar_wait(qdo_full, it & 1);
        if (it >= 1) mbar_wait(st_free, (it - 1) & 1);
        fence_after_sync();
        mma_tile<false>(tST, sK, sQ, D / 16, id_s, false);
        mma_tile<false>(tdPT, sV, sdO, D / 16, id_s, false);
        umma_commit(st_full);
        mbar_wait(ps_full, it & 1);
        fence_after_sync();
        mma_tile<true>(tdV, sPT, sdO, 8, id_d, it > 0);
        mma_tile<true>(tdK, sdST, sQ, 8, id_d, it > 0);
        umma_commit(qdo_empty);
        umma_commit(ps_empty);
      }
      umma_commit(acc_done);
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    for (int it = 0; it < nit; ++it) {
      const int i = j + it;
      float* Ls = sLD + (it & 1) * 256;
      Ls[r] = lse[(size_t)bh * S + i * 128 + r];
      Ls[128 + r] = delta[(size_t)bh * S + i * 128 + r];
      named_sync(1, 128);
      mbar_wait(st_full, it & 1);
      fence_after_sync();
      if (it >= 1) mbar_wait(ps_empty, (it - 1) & 1);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t s32[32], p32[32];
        tmem_ld32_nowait(tST + lo + c * 32, s32);
        tmem_ld32_nowait(tdPT + lo + c * 32, p32);
        tmem_wait_ld();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int q = c * 32 + k;
          float p0 = ex2(u2f(s32[k]) * sl2 - Ls[q]);
          float p1 = ex2(u2f(s32[k + 1]) * sl2 - Ls[q + 1]);
          if (it == 0) {                          // diagonal tile: query before key
            if (q < r) p0 = 0.f;
            if (q + 1 < r) p1 = 0.f;
          }
          const float d0 = p0 * (u2f(p32[k]) - Ls[128 + q]);
          const float d1 = p1 * (u2f(p32[k + 1]) - Ls[128 + q + 1]);
          pp[k >> 1] = pack_bf16(p0, p1);
          dd[k >> 1] = pack_bf16(d0, d1);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          st_piece(sPT, r, c * 4 + g, make_uint4(pp[4 * g], pp[4 * g + 1], pp[4 * g + 2], pp[4 * g + 3]));
          st_piece(sdST, r, c * 4 + g, make_uint4(dd[4 * g], dd[4 * g + 1], dd[4 * g + 2], dd[4 * g + 3]));
        }
      }
      fence_before_sync();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(st_free);
        mbar_arrive(ps_full);
      }
    }
    mbar_wait(acc_done, 0);
    fence_after_sync();
    const size_t row = (size_t)row0 + j * 128 + r;
    __nv_bfloat16* d = dqkv + row * 3 * hd;
    store_row<D>(tdV + lo, 1.f, d + 2 * hd + h * D);
    store_row<D>(tdK + lo, scale, d + hd + h * D);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
}

// ======================================================================= backward: dQ
template <int D>
struct Bq {
  static constexpr int TB = 128 * D * 2;
  static constexpr int Q = 0, DO = TB, K = 2 * TB, V = 4 * TB, DS = 6 * TB, BAR = 6 * TB + PB;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
bwd_dq_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_do,
              const float* __restrict__ lse, const float* __restrict__ delta,
              __nv_bfloat16* __restrict__ dqkv, int B, int H, int S, int hd, float sl2,
              float scale) {
  using L = Bq<D>;
  constexpr int TB = L::TB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sQ = sm + L::Q, *sdO = sm + L::DO, *sK = sm + L::K, *sV = sm + L::V, *sdS = sm + L::DS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *qdo_full = bar, *k_full = bar + 1, *k_empty = bar + 3, *v_full = bar + 5,
           *v_empty = bar + 7, *s_full = bar + 9, *s_free = bar + 10, *ds_full = bar + 11,
           *ds_empty = bar + 12, *acc_done = bar + 13;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 14);

  const int nq = S / 128, BH = B * H;
  const int i = nq - 1 - (int)blockIdx.x / BH;
  const int bh = (int)blockIdx.x % BH, b = bh / H, h = bh % H;
  const int nkv = i + 1, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(qdo_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1); mbar_init(s_free, 4); mbar_init(ds_full, 4);
    mbar_init(ds_empty, 1); mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
    prefetch_map(&tm_do);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qdo_full, 2 * TB);
      load_tile<D>(sQ, &tm, qdo_full, h * D, row0 + i * 128);
      load_tile<D>(sdO, &tm_do, qdo_full, h * D, row0 + i * 128);
      for (int jj = 0; jj < nkv; ++jj) {
        const int s = jj & 1;
        const uint32_t ph = (jj >> 1) & 1;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], TB);
        load_tile<D>(sK + s * TB, &tm, &k_full[s], hd + h * D, row0 + jj * 128);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], TB);
        load_tile<D>(sV + s * TB, &tm, &v_full[s], 2 * hd + h * D, row0 + jj * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_d = idesc_bf16_f32(128, D, false, true);
      mbar_wait(qdo_full, 0);
      for (int jj = 0; jj < nkv; ++jj) {
        const int s = jj & 1;
        const uint32_t ph = (jj >> 1) & 1;
        mbar_wait(&k_full[s], ph);
        mbar_wait(&v_full[s], ph);
        if (jj >= 1) mbar_wait(s_free, (jj - 1) & 1);
        fence_after_sync();
        mma_tile<false>(tS, sQ, sK + s * TB, D / 16, id_s, false);
        mma_tile<false>(tdP, sdO, sV + s * TB, D / 16, id_s, false);
        umma_commit(&v_empty[s]);
        umma_commit(s_full);
        mbar_wait(ds_full, jj & 1);
        fence_after_sync();
        mma_tile<true>(tdQ, sdS, sK + s * TB, 8, id_d, jj > 0);
        umma_commit(&k_empty[s]);
        umma_commit(ds_empty);
      }
      umma_commit(acc_done);
    }
    __syncwarp();
  } else {
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    const float lse_r = lse[(size_t)bh * S + i * 128 + r];
    const float del_r = delta[(size_t)bh * S + i * 128 + r];
    for (int jj = 0; jj < nkv; ++jj) {
      mbar_wait(s_full, jj & 1);
      fence_after_sync();
      if (jj >= 1) mbar_wait(ds_empty, (jj - 1) & 1);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t s32[32], p32[32];
        tmem_ld32_nowait(tS + lo + c * 32, s32);
        tmem_ld32_nowait(tdP + lo + c * 32, p32);
        tmem_wait_ld();
        uint32_t dd[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int kv = c * 32 + k;
          float p0 = ex2(u2f(s32[k]) * sl2 - lse_r);
          float p1 = ex2(u2f(s32[k + 1]) * sl2 - lse_r);
          if (jj == i) {                          // diagonal tile: key after query
            if (kv > r) p0 = 0.f;
            if (kv + 1 > r) p1 = 0.f;
          }
          dd[k >> 1] = pack_bf16(p0 * (u2f(p32[k]) - del_r), p1 * (u2f(p32[k + 1]) - del_r));
        }
#pragma unroll
        for (int g = 0; g < 4; ++g)
          st_piece(sdS, r, c * 4 + g, make_uint4(dd[4 * g], dd[4 * g + 1], dd[4 * g + 2], dd[4 * g + 3]));
      }
      fence_before_sync();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(s_free);
        mbar_arrive(ds_full);
      }
    }
    mbar_wait(acc_done, 0);
    fence_after_sync();
    const size_t row = (size_t)row0 + i * 128 + r;
    store_row<D>(tdQ + lo, scale, dqkv + row * 3 * hd + h * D);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
}

// delta[(b*H + h)*S + s] = sum_d dO[row, h*D + d] * O[row, h*D + d]  (fixed shuffle tree)
template <int D>
__global__ void delta_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dO,
                             float* __restrict__ delta, int H, int S, int hd) {
  const int row = blockIdx.x;                     // b*S + s
  const int t = threadIdx.x;                      // 8 elements each; D/8 threads per head
  const unsigned mask = __activemask();           // hd < 256: a partial warp
  const size_t off = (size_t)row * hd + t * 8;
  const uint4 a = *reinterpret_cast<const uint4*>(o + off);
  const uint4 g = *reinterpret_cast<const uint4*>(dO + off);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = __bfloat1622float2(a2[k]), y = __bfloat1622float2(g2[k]);
    acc = fmaf(x.x, y.x, acc);
    acc = fmaf(x.y, y.y, acc);
  }
#pragma unroll
  for (int w = D / 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(mask, acc, w);
  if ((t & (D / 8 - 1)) == 0) {
    const int h = t / (D / 8), b = row / S, s = row % S;
    delta[((size_t)b * H + h) * S + s] = acc;
  }
}

// ------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int encoder() {
  if (g_encode) return ZI_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  ZI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
          "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
  if (!fn || q != cudaDriverEntryPointSuccess) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZI_ECUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return ZI_OK;
}

// rows x cols bf16, row stride ld elements, 64 x 64 boxes, 128-byte swizzle
static int make_map(CUtensorMap* m, const void* base, int rows, int cols, int ld) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 64}, estr[2] = {1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return ZI_ECUDA;
  }
  return ZI_OK;
}

template <typename K>
static int set_smem(K kern, int bytes, bool& done) {
  if (!done) {
    ZI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
            "cudaFuncSetAttribute(attn smem)");
    done = true;
  }
  return ZI_OK;
}

static int check(const void* qkv, int B, int H, int S, int D, const char* who) {
  ZI_CHECK_ARG(qkv != nullptr, "%s: NULL qkv", who);
  ZI_CHECK_ARG(B >= 1 && H >= 1, "%s: bad B/H %d/%d", who, B, H);
  ZI_CHECK_ARG(S >= 128 && S % 128 == 0, "%s: S=%d must be a positive multiple of 128", who, S);
  ZI_CHECK_ARG(D == 64 || D == 128, "%s: head_dim %d must be 64 or 128", who, D);
  ZI_CHECK_ARG((size_t)B * S < (1u << 31), "%s: too many rows", who);
  return ZI_OK;
}

template <int D>
static int fwd(const void* qkv, void* out, float* lse, int B, int H, int S, cudaStream_t st) {
  const int hd = H * D;
  int rc = encoder();
  if (rc != ZI_OK) return rc;
  CUtensorMap tm;
  if ((rc = make_map(&tm, qkv, B * S, 3 * hd, 3 * hd)) != ZI_OK) return rc;
  static bool attr = false;
  if ((rc = set_smem(fwd_kernel<D>, Fwd<D>::BYTES, attr)) != ZI_OK) return rc;
  const float sl2 = LOG2E / sqrtf((float)D);
  fwd_kernel<D><<<B * H * (S / 128), THREADS, Fwd<D>::BYTES, st>>>(
      tm, static_cast<__nv_bfloat16*>(out), lse, B, H, S, hd, sl2);
  return launch_status("zi_attn_fwd");
}

template <int D>
static int bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* delta,
               void* dqkv, int B, int H, int S, cudaStream_t st) {
  const int hd = H * D;
  int rc = encoder();
  if (rc != ZI_OK) return rc;
  CUtensorMap tm, tdo;
  if ((rc = make_map(&tm, qkv, B * S, 3 * hd, 3 * hd)) != ZI_OK) return rc;
  if ((rc = make_map(&tdo, dout, B * S, hd, hd)) != ZI_OK) return rc;
  static bool a1 = false, a2 = false;
  if ((rc = set_smem(bwd_dkdv_kernel<D>, Bkv<D>::BYTES, a1)) != ZI_OK) return rc;
  if ((rc = set_smem(bwd_dq_kernel<D>, Bq<D>::BYTES, a2)) != ZI_OK) return rc;
  delta_kernel<D><<<B * S, hd / 8, 0, st>>>(static_cast<const __nv_bfloat16*>(out),
                                            static_cast<const __nv_bfloat16*>(dout), delta, H, S, hd);
  if ((rc = launch_status("zi_attn_bwd(delta)")) != ZI_OK) return rc;
  const float scale = 1.f / sqrtf((float)D), sl2 = LOG2E * scale;
  const int grid = B * H * (S / 128);
  auto* dq = static_cast<__nv_bfloat16*>(dqkv);
  bwd_dkdv_kernel<D><<<grid, THREADS, Bkv<D>::BYTES, st>>>(tm, tdo, lse, delta, dq, B, H, S, hd,
                                                            sl2, scale);
  if ((rc = launch_status("zi_attn_bwd(dkdv)")) != ZI_OK) return rc;
  bwd_dq_kernel<D><<<grid, THREADS, Bq<D>::BYTES, st>>>(tm, tdo, lse, delta, dq, B, H, S, hd, sl2,
                                                        scale);
  return launch_status("zi_attn_bwd(dq)");
}

}  // namespace attn
}  // namespace zi

extern "C" {

int zi_attn_fwd(const void* qkv, void* out, float* lse, int B, int H, int S, int head_dim,
                void* stream) {
  int rc = zi::attn::check(qkv, B, H, S, head_dim, "zi_attn_fwd");
  if (rc != ZI_OK) return rc;
  ZI_CHECK_ARG(out && lse, "zi_attn_fwd: NULL out/lse");
  ZI_CHECK_ARG(zi::aligned(qkv, 16) && zi::aligned(out, 16), "zi_attn_fwd: 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  return head_dim == 64 ? zi::attn::fwd<64>(qkv, out, lse, B, H, S, s)
                        : zi::attn::fwd<128>(qkv, out, lse, B, H, S, s);
}

int zi_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* delta,
                void* dqkv, int B, int H, int S, int head_dim, void* stream) {
  int rc = zi::attn::check(qkv, B, H, S, head_dim, "zi_attn_bwd");
  if (rc != ZI_OK) return rc;
  ZI_CHECK_ARG(out && dout && lse && delta && dqkv, "zi_attn_bwd: NULL argument");
  ZI_CHECK_ARG(zi::aligned(out, 16) && zi::aligned(dout, 16) && zi::aligned(dqkv, 16),
               "zi_attn_bwd: 16-byte alignment");
  ZI_CHECK_ARG(H * head_dim / 8 <= 1024, "zi_attn_bwd: hidden %d too wide", H * head_dim);
  cudaStream_t s = (cudaStream_t)stream;
  return head_dim == 64 ? zi::attn::bwd<64>(qkv, out, dout, lse, delta, dqkv, B, H, S, s)
                        : zi::attn::bwd<128>(qkv, out, dout, lse, delta, dqkv, B, H, S, s);
}

}  // extern "C"
