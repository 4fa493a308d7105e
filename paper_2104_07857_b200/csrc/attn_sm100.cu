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
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "bulk.cuh"
#include "common.cuh"
#include "tc.cuh"

namespace zi {
namespace attn {

using namespace zi::tc;

// warp 0 TMA; warp 1 the score MMAs (and TMEM allocation); warps 2..9 elementwise;
// warp 10 the accumulating MMAs (PV / dV-dK / dQ). Two issuing warps, so a score MMA
// never waits in program order behind an accumulate that waits for the other group's
// probabilities (one issuing thread serialised the two elementwise groups).
constexpr int THREADS = 352;
constexpr int ACC_WARP = 10;
constexpr int GW = 4;                        // warps per elementwise group (one per lane quadrant)
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ROWS x D bf16 (box 64 x 64) -> D/64 chunk regions of ROWS*128 bytes (tc.cuh layout)
template <int D, int ROWS>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                          int col0, int row0) {
#pragma unroll
  for (int kc = 0; kc < D / 64; ++kc)
#pragma unroll
    for (int rh = 0; rh < ROWS / 64; ++rh)
      tma_load_2d(dst + kc * ROWS * 128 + rh * 8192, map, bar, col0 + kc * 64, row0 + rh * 64);
}

// k-step kk (16 deep) of a ROWS-row tile read K-major / MN-major
template <int ROWS>
__device__ __forceinline__ uint64_t kdesc(const uint8_t* base, int kk) {
  return sdesc_sw128(smem_u32(base) + (kk >> 2) * ROWS * 128 + (kk & 3) * 32, 16);
}
template <int ROWS>
__device__ __forceinline__ uint64_t mndesc(const uint8_t* base, int kk) {
  return sdesc_sw128(smem_u32(base) + kk * 2048, ROWS * 128);
}

// 16-byte piece g (elements 8g .. 8g+7) of row r of a 128-row K-major tile
__device__ __forceinline__ void st_piece(uint8_t* tile, int r, int g, uint4 v) {
  *reinterpret_cast<uint4*>(tile + (g >> 3) * 16384 + r * 128 + (((g & 7) ^ (r & 7)) << 4)) = v;
}

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// D[128 x N] (+)= A B over KS 16-deep steps: A a 128-row K-major tile, B a BROWS-row tile
// (K- or MN-major). Descriptors are built once and stepped by constant offsets (the start
// address field holds bytes >> 4), so each MMA issues with no per-step address math.
template <int BROWS, bool B_MN, int KS>
__device__ __forceinline__ void mma_tile(uint32_t d, const uint8_t* a, const uint8_t* b,
                                         uint32_t idesc, bool accumulate) {
  const uint64_t da = kdesc<128>(a, 0);
  const uint64_t db = B_MN ? mndesc<BROWS>(b, 0) : kdesc<BROWS>(b, 0);
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const uint64_t oa = (uint64_t)((kk >> 2) * (128 * 128 >> 4) + (kk & 3) * 2);
    const uint64_t ob = B_MN ? (uint64_t)(kk * (2048 >> 4))
                             : (uint64_t)((kk >> 2) * (BROWS * 128 >> 4) + (kk & 3) * 2);
    umma_bf16(d, da + oa, db + ob, idesc, (accumulate || kk > 0) ? 1u : 0u);
  }
}

// CTA index -> (rank t of its tile, batch-head bh). CTAs run in groups of G batch-heads
// (G * nq CTAs, about one wave for G = 16): inside a group rank-major (t = 0 is the
// tile with the most causal work), so a wave holds every tile of its batch-heads and
// their K / V tiles are read from HBM once and then hit in L2. G = B*H is one group.
__device__ __forceinline__ void tile_order(int idx, int nq, int BH, int G, int& t, int& bh) {
  const int per = G * nq, grp = idx / per, r = idx - grp * per;
  const int g = min(G, BH - grp * G);              // the last group may be partial
  t = r / g;
  bh = grp * G + r % g;
}

// D[128 x N] (+)= A B over KS 16-deep steps with A (128 x 16*KS bf16) in TMEM at column
// a_tmem (8 columns per step) and B a BROWS-row MN-major tile in shared memory.
template <int BROWS, int KS>
__device__ __forceinline__ void mma_tile_ts(uint32_t d, uint32_t a_tmem, const uint8_t* b,
                                            uint32_t idesc, bool accumulate) {
  const uint64_t db = mndesc<BROWS>(b, 0);
#pragma unroll
  for (int kk = 0; kk < KS; ++kk)
    umma_bf16_ts(d, a_tmem + kk * 8, db + (uint64_t)(kk * (2048 >> 4)), idesc,
                 (accumulate || kk > 0) ? 1u : 0u);
}

// one lane of a converged warp (elect.sync): the tcgen05.mma issuer
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}"
               : "=r"(p));
  return p != 0;
}

// one row of NC fp32 TMEM columns (x scale) -> bf16 global (16-byte stores)
template <int NC>
__device__ __forceinline__ void store_row(uint32_t taddr, float scale, __nv_bfloat16* dst) {
#pragma unroll
  for (int cc = 0; cc < NC / 32; ++cc) {
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

// store_row plus the column sums of the stored (bf16-rounded) values over the warp's 32
// rows: a transpose-reduce butterfly (31 shuffles per 32 columns) leaves column c's sum in
// lane c, written to csum[c] (the 32-row block partial of a bias gradient). Fixed order.
template <int NC>
__device__ __forceinline__ void store_row_csum(uint32_t taddr, float scale, __nv_bfloat16* dst,
                                               float* csum, int lane) {
#pragma unroll 1
  for (int cc = 0; cc < NC / 32; ++cc) {
    uint32_t o[32];
    tmem_ld32(taddr + cc * 32, o);
    float v[32];
    uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[k] = pack_bf16(u2f(o[8 * g + 2 * k]) * scale, u2f(o[8 * g + 2 * k + 1]) * scale);
        v[8 * g + 2 * k] = __uint_as_float(w[k] << 16);
        v[8 * g + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
      }
      d4[g] = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int k = 0; k < off; ++k) {
        const float send = up ? v[k] : v[k + off];
        const float keep = up ? v[k + off] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    csum[cc * 32 + lane] = v[0];
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

// Every kernel walks its kv (or q) range in 64-column sub-tiles u = 0, 1, 2, ...; sub-tile
// u belongs to elementwise group g = u & 1 (warps 2..5 / 6..9: lane quadrant = warp & 3),
// which owns TMEM score slot g and shared tile slot g. The MMA thread issues the score
// MMAs of sub-tile u before it waits for group (u-1)&1's elementwise result, so the
// tensor core works on one sub-tile while the other group works on the previous one.

// ============================================================================ forward
// Two independent online softmaxes: group g folds the kv columns g*64..g*64+63 of every
// kv tile into its own (m_g, l_g, O_g); the epilogue merges the two.
// K and V half-tiles stream through separate rings: a K stage is released as soon as
// its score MMA completed, a V stage after its PV MMA, so K is fetched up to NSK
// sub-tiles ahead of the scores instead of waiting behind the PV of its stage (TMA
// latency under load is ~2 us, several sub-tiles). The epilogue's (m, l) exchange
// reuses the group's own P tile once its last PV completed.
template <int D>
struct Fwd {
  static constexpr int QB = 128 * D * 2, HB = 64 * D * 2, NSK = 5, NSV = 5;
  static constexpr int Q = 0, K = QB, V = K + NSK * HB, P = V + NSV * HB, BAR = P + 2 * 16384;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
fwd_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
           float* __restrict__ lse, int B, int H, int S, int hd, float sl2,
           unsigned long long* __restrict__ trace, int grp) {
  // trace (diagnostics, normally null): per CTA {sm, entry, operands in, last MMA issued,
  // softmax done, exit} in globaltimer ns
  unsigned long long* tr = trace ? trace + blockIdx.x * 6 : nullptr;
  if (tr && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[0] = smid;
    tr[1] = gtimer();
  }
  using L = Fwd<D>;
  constexpr int HB = L::HB, NSK = L::NSK, NSV = L::NSV;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sQ = sm + L::Q, *sK = sm + L::K, *sV = sm + L::V, *sP = sm + L::P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = k_full + NSK, *v_full = k_empty + NSK,
           *v_empty = v_full + NSV, *s_full = v_empty + NSV, *s_free = s_full + 2,
           *p_full = s_full + 4, *pv_done = s_full + 6;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s_full + 8);

  const int nq = S / 128, BH = B * H;
  int i, bh;                                       // long causal rows first
  tile_order((int)blockIdx.x, nq, BH, grp, i, bh);
  i = nq - 1 - i;
  const int b = bh / H, h = bh % H;
  const int nkv = i + 1, nsub = 2 * nkv, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NSK; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < NSV; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1); mbar_init(&s_free[g], GW);
      mbar_init(&p_full[g], GW); mbar_init(&pv_done[g], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  zi::pdl_sync();   // setup above overlapped the previous kernel's tail
  const uint32_t tmem = *tslot;        // S slot g at g*64; P_g (bf16) at 128 + g*32; O_g at 256 + g*128

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, L::QB);
      load_rows<D, 128>(sQ, &tm, q_full, h * D, row0 + i * 128);
      // K runs up to 2 sub-tiles ahead of V in issue order (the scores lead the PVs)
      int uk = 0, uv = 0;
      while (uv < nsub) {
        if (uk < nsub && uk < uv + 3) {
          const int st = uk % NSK;
          mbar_wait(&k_empty[st], ((uk / NSK) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], HB);
          load_rows<D, 64>(sK + st * HB, &tm, &k_full[st], hd + h * D, row0 + uk * 64);
          ++uk;
        } else {
          const int st = uv % NSV;
          mbar_wait(&v_empty[st], ((uv / NSV) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], HB);
          load_rows<D, 64>(sV + st * HB, &tm, &v_full[st], 2 * hd + h * D, row0 + uv * 64);
          ++uv;
        }
      }
    }
  } else if (warp == 1) {
    // scores: the whole warp waits; one elected lane issues each group of MMAs and commits.
    // S_u goes into group g's slot as soon as the group has loaded S_{u-2} (s_free).
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
    mbar_wait(q_full, 0);
    unsigned long long* ms = (tr && blockIdx.x == 0 && lane == 0)
                                 ? trace + gridDim.x * 6 + 2 * 64 * 6 : nullptr;
    for (int u = 0; u < nsub; ++u) {
      if (tr && lane == 0 && u == 1) tr[2] = gtimer();
      if (ms) ms[u * 4 + 0] = clock64();
      const int st = u % NSK, g = u & 1;
      mbar_wait(&k_full[st], (u / NSK) & 1);
      if (ms) ms[u * 4 + 1] = clock64();
      if (u >= 2) mbar_wait(&s_free[g], ((u - 2) >> 1) & 1);
      if (ms) ms[u * 4 + 2] = clock64();
      fence_after_sync();
      if (elect_one()) {
        mma_tile<64, false, D / 16>(tmem + g * 64, sQ, sK + st * HB, id_s, false);
        umma_commit(&s_full[g]);
        umma_commit(&k_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp == ACC_WARP) {
    // O_g += P V of sub-tile v once group g published P_v; frees the kv stage (its S
    // MMA completed before the group could load S_v)
    constexpr uint32_t id_o = idesc_bf16_f32(128, D, false, true);
    unsigned long long* ms = (tr && blockIdx.x == 0 && lane == 0)
                                 ? trace + gridDim.x * 6 + 2 * 64 * 6 : nullptr;
    for (int v = 0; v < nsub; ++v) {
      const int st = v % NSV, g = v & 1;
      mbar_wait(&v_full[st], (v / NSV) & 1);
      mbar_wait(&p_full[g], (v >> 1) & 1);
      if (ms) ms[v * 4 + 3] = clock64();
      fence_after_sync();
      if (elect_one()) {
        mma_tile_ts<64, 4>(tmem + 256 + g * 128, tmem + 128 + g * 32, sV + st * HB, id_o, v >= 2);
        umma_commit(&v_empty[st]);
        umma_commit(&pv_done[g]);
      }
      __syncwarp();
    }
    if (tr && lane == 0) tr[3] = gtimer();
  } else {
    const int g = (warp - 2) >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + g * 64 + lo, tO = tmem + 256 + g * 128 + lo;
    const uint32_t tP = tmem + 128 + g * 32 + lo;    // this thread's row of P_g
    float m = -INFINITY, l = 0.f;
    unsigned long long* fs = (tr && blockIdx.x == 0 && lane == 0 && (warp == 2 || warp == 6))
                                 ? trace + gridDim.x * 6 + g * 64 * 6 : nullptr;
    for (int jj = 0; jj < nkv; ++jj) {
      if (fs) fs[jj * 6 + 0] = clock64();
      mbar_wait(&s_full[g], jj & 1);
      if (fs) fs[jj * 6 + 1] = clock64();
      fence_after_sync();
      uint32_t t0[32], t1[32];
      tmem_ld32_nowait(tS, t0);
      tmem_ld32_nowait(tS + 32, t1);
      tmem_wait_ld();
      if (fs) fs[jj * 6 + 2] = clock64();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[g]);
      float x[64];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        x[k] = u2f(t0[k]);
        x[32 + k] = u2f(t1[k]);
      }
      if (jj == i) {                             // diagonal tile: key index > query index
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (g * 64 + c > r) x[c] = -INFINITY;
      }
      float mx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx[k] = x[k];
#pragma unroll
      for (int c = 8; c < 64; ++c) mx[c & 7] = fmaxf(mx[c & 7], x[c]);
      const float mrow = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
      // lazy rescale (FA4): move the reference max only when it grows by > 2^8
      float alpha = 1.f;
      if (mrow > m + 8.f) {                      // first live tile: m = -inf -> alpha = 0
        alpha = ex2(m - mrow);
        m = mrow;
      }
      const float nm = (m == -INFINITY) ? 0.f : -m;   // fully masked so far: p = 0
      uint32_t pk[32];
      float rs[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) rs[k] = 0.f;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float p0 = ex2(fmaf(x[2 * c], sl2, nm)), p1 = ex2(fmaf(x[2 * c + 1], sl2, nm));
        rs[c & 7] += p0 + p1;
        pk[c] = pack_bf16(p0, p1);
      }
      l = l * alpha + (((rs[0] + rs[1]) + (rs[2] + rs[3])) + ((rs[4] + rs[5]) + (rs[6] + rs[7])));
      if (fs) fs[jj * 6 + 3] = clock64();
      if (jj >= 1) {
        mbar_wait(&pv_done[g], (jj - 1) & 1);    // O_g stable, P_g free
        fence_after_sync();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(tO + cc * 32, o);
#pragma unroll
            for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(u2f(o[k]) * alpha);
            tmem_st32(tO + cc * 32, o);
          }
        }
      }
      if (fs) fs[jj * 6 + 4] = clock64();
      // P_g (bf16, two per column) into TMEM columns 128 + g*32: the PV MMA reads its A
      // operand from there, so P never touches shared memory (the forward is bound by
      // shared-memory bandwidth: operand reads of the N = 64 score MMAs, K / V fills)
      tmem_st32(tP, pk);
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
      if (fs) fs[jj * 6 + 5] = clock64();
    }
    // merge the two streams: O = (O_0 2^(m_0-M) + O_1 2^(m_1-M)) / (l_0 2^(m_0-M) + l_1 2^(m_1-M))
    // (m, l) exchange in the group's own P tile, free once its last PV completed
    mbar_wait(&pv_done[g], (nkv - 1) & 1);
    float* xg = reinterpret_cast<float*>(sP + g * 16384);
    xg[r] = m;
    xg[128 + r] = l;
    named_sync(1 + q4, 2 * 32);
    const float* x0 = reinterpret_cast<const float*>(sP);
    const float* x1 = reinterpret_cast<const float*>(sP + 16384);
    const float m0 = x0[r], l0 = x0[128 + r], m1 = x1[r], l1 = x1[128 + r];
    const float M = fmaxf(m0, m1);
    const float a0 = ex2(m0 - M), a1 = (m1 == -INFINITY) ? 0.f : ex2(m1 - M);
    const float Lt = l0 * a0 + l1 * a1, inv = 1.f / Lt;
    fence_after_sync();
    const size_t row = (size_t)row0 + i * 128 + r;
    __nv_bfloat16* dst = out + row * hd + h * D + g * (D / 2);
    const uint32_t o0 = tmem + 256 + lo + g * (D / 2), o1 = o0 + 128;
#pragma unroll 1
    for (int cc = 0; cc < D / 64; ++cc) {
      uint32_t x0[32], x1[32];
      tmem_ld32_nowait(o0 + cc * 32, x0);
      tmem_ld32_nowait(o1 + cc * 32, x1);
      tmem_wait_ld();
      uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float f[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          f[k] = fmaf(u2f(x0[8 * q + k]), a0, u2f(x1[8 * q + k]) * a1) * inv;
        d4[q] = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]),
                           pack_bf16(f[6], f[7]));
      }
    }
    if (g == 0) lse[(size_t)bh * S + i * 128 + r] = M + __log2f(Lt);
    if (tr && warp == 2 && lane == 0) tr[4] = gtimer();
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
  if (tr && threadIdx.x == 0) tr[5] = gtimer();
}

// ================================================================ forward, 2 Q tiles
// CTA = two adjacent q tiles (qa = 2t, qb = 2t + 1) of one (batch, head) sharing every
// K / V tile; 128-column kv tiles, so the score MMAs run at N = 128 (the N = 64 shape
// reaches only 2/3 of the tensor rate, scripts/probes/mma_probe.cu). TMEM: S_a, S_b
// (128 columns each; P_x, bf16, overwrites the first 64 columns of S_x once read), O_a,
// O_b. One MMA thread issues, per kv tile j: PV_a(j), S_a(j+1), PV_b(j), S_b(j+1) — so
// while softmax group x works on S_x(j) the tensor core runs the other tile's PV and S
// (ping-pong); a tile's S_x(j+1) follows its own PV_x(j) in issue order, which is what
// makes the P / S aliasing and the lazy O rescale safe (tcgen05 work of one thread
// completes in order: S_x(j) complete implies PV_x(j-1) complete).
template <int D>
struct Fwd2 {
  static constexpr int TB = 128 * D * 2, NSK = 3, NSV = 2;
  static constexpr int QA = 0, QBo = TB, K = 2 * TB, V = K + NSK * TB, BAR = V + NSV * TB;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(320, 1)
fwd2_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
            float* __restrict__ lse, int B, int H, int S, int hd, float sl2,
            unsigned long long* __restrict__ trace) {
  // trace (diagnostics, normally null): per CTA {sm, entry, operands in, last MMA issued,
  // softmax done, exit} in globaltimer ns; CTA 0: per kv tile, group x's
  // {wait start, S ready, max done, P published} and the MMA thread's
  // {PV_a issued, S_a issued, PV_b issued, S_b issued} in clock64
  unsigned long long* tr = trace ? trace + blockIdx.x * 6 : nullptr;
  if (tr && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[0] = smid;
    tr[1] = gtimer();
  }
  unsigned long long* fine = (trace && blockIdx.x == 0) ? trace + gridDim.x * 6 : nullptr;
  using L = Fwd2<D>;
  constexpr int TB = L::TB, NSK = L::NSK, NSV = L::NSV;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sQa = sm + L::QA, *sQb = sm + L::QBo, *sK = sm + L::K, *sV = sm + L::V;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *q_full = bar, *k_full = bar + 1, *k_empty = k_full + NSK, *v_full = k_empty + NSK,
           *v_empty = v_full + NSV, *s_full = v_empty + NSV, *p_full = s_full + 2,
           *pv_done = s_full + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s_full + 6);

  const int nq2 = S / 256, BH = B * H;
  const int t = nq2 - 1 - (int)blockIdx.x / BH;    // most causal work first
  const int bh = (int)blockIdx.x % BH, b = bh / H, h = bh % H;
  const int qa = 2 * t, nkv_a = qa + 1, nkv_b = qa + 2, row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NSK; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < NSV; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1); mbar_init(&p_full[x], GW); mbar_init(&pv_done[x], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  zi::pdl_sync();
  const uint32_t tmem = *tslot;        // S_x / P_x at x*128; O_x at 256 + x*128

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * TB);
      load_rows<D, 128>(sQa, &tm, q_full, h * D, row0 + qa * 128);
      load_rows<D, 128>(sQb, &tm, q_full, h * D, row0 + (qa + 1) * 128);
      int uk = 0, uv = 0;                          // K runs one tile ahead of V
      while (uv < nkv_b) {
        if (uk < nkv_b && uk <= uv + 1) {
          const int st = uk % NSK;
          mbar_wait(&k_empty[st], ((uk / NSK) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], TB);
          load_rows<D, 128>(sK + st * TB, &tm, &k_full[st], hd + h * D, row0 + uk * 128);
          ++uk;
        } else {
          const int st = uv % NSV;
          mbar_wait(&v_empty[st], ((uv / NSV) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], TB);
          load_rows<D, 128>(sV + st * TB, &tm, &v_full[st], 2 * hd + h * D, row0 + uv * 128);
          ++uv;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t id_o = idesc_bf16_f32(128, D, false, true);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int x, int j) {             // S_x(j) = Q_x K_j^T
      const int st = j % NSK;
      mbar_wait(&k_full[st], (j / NSK) & 1);
      fence_after_sync();
      if (elect_one()) {
        mma_tile<128, false, D / 16>(tmem + x * 128, x ? sQb : sQa, sK + st * TB, id_s, false);
        umma_commit(&s_full[x]);
        if (x == 1) umma_commit(&k_empty[st]);     // both tiles' scores of K_j issued
      }
      __syncwarp();
    };
    auto issue_pv = [&](int x, int j) {            // O_x += P_x(j) V_j
      const int st = j % NSV;
      mbar_wait(&v_full[st], (j / NSV) & 1);
      mbar_wait(&p_full[x], j & 1);
      fence_after_sync();
      if (elect_one()) {
        mma_tile_ts<128, 8>(tmem + 256 + x * 128, tmem + x * 128, sV + st * TB, id_o, j > 0);
        if (j == nkv_a - 1 + x) umma_commit(&pv_done[x]);   // the tile's last PV: O final
        if (x == 1) umma_commit(&v_empty[st]);
      }
      __syncwarp();
    };
    unsigned long long* mf = (fine && lane == 0) ? fine + 2 * 16 * 4 : nullptr;
    issue_s(0, 0);
    issue_s(1, 0);
    if (tr && lane == 0) tr[2] = gtimer();
    for (int j = 0; j < nkv_b; ++j) {
      if (j < nkv_a) {
        issue_pv(0, j);
        if (mf) mf[j * 4 + 0] = clock64();
        if (j + 1 < nkv_a) issue_s(0, j + 1);
        if (mf) mf[j * 4 + 1] = clock64();
      }
      issue_pv(1, j);
      if (mf) mf[j * 4 + 2] = clock64();
      if (j + 1 < nkv_b) issue_s(1, j + 1);
      if (mf) mf[j * 4 + 3] = clock64();
    }
    if (tr && lane == 0) tr[3] = gtimer();
  } else {
    // softmax group x = q tile qa + x; thread = row r of the tile (TMEM lane)
    const int x = (warp - 2) >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + x * 128 + lo, tO = tmem + 256 + x * 128 + lo;
    const int qi = qa + x, nkv = nkv_a + x;
    unsigned long long* gf = (fine && lane == 0 && q4 == 0) ? fine + x * 16 * 4 : nullptr;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      if (gf) gf[j * 4 + 0] = clock64();
      mbar_wait(&s_full[x], j & 1);
      if (gf) gf[j * 4 + 1] = clock64();
      fence_after_sync();
      const bool diag = j == qi;                   // key index > query index masked
      uint32_t sv[128];                            // the row's 128 scores, loaded once
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) tmem_ld32_nowait(tS + hh * 32, sv + hh * 32);
      tmem_wait_ld();
      if (diag) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      float mx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mx[k] = u2f(sv[k]);
#pragma unroll
      for (int c = 8; c < 128; ++c) mx[c & 7] = fmaxf(mx[c & 7], u2f(sv[c]));
      const float mrow = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * sl2;
      float alpha = 1.f;
      if (mrow > m + 8.f) {                        // lazy rescale (FA4); first tile: alpha 0
        alpha = ex2(m - mrow);
        m = mrow;
      }
      if (j >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // S_x(j) complete => PV_x(j-1) complete (same issuing thread): O_x is stable
#pragma unroll 1
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t o[32];
          tmem_ld32(tO + cc * 32, o);
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(u2f(o[k]) * alpha);
          tmem_st32(tO + cc * 32, o);
        }
      }
      if (gf) gf[j * 4 + 2] = clock64();
      const float nm = (m == -INFINITY) ? 0.f : -m;
      float rs[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) rs[k] = 0.f;
      // (exp2 on the FMA pipe for part of the row, FA4's trick, measured slower here: the
      // polynomial costs ~10 issue slots per element against one MUFU slot)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int k0 = hh * 64 + 2 * c;
          const float p0 = ex2(fmaf(u2f(sv[k0]), sl2, nm));
          const float p1 = ex2(fmaf(u2f(sv[k0 + 1]), sl2, nm));
          rs[c & 7] += p0 + p1;
          pk[c] = pack_bf16(p0, p1);
        }
        tmem_st32(tS + hh * 32, pk);                 // P over S columns already read
      }
      l = l * alpha + (((rs[0] + rs[1]) + (rs[2] + rs[3])) + ((rs[4] + rs[5]) + (rs[6] + rs[7])));
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[x]);
      if (gf) gf[j * 4 + 3] = clock64();
    }
    if (tr && x == 1 && warp == 6 && lane == 0) tr[4] = gtimer();
    mbar_wait(&pv_done[x], 0);                     // committed once, after the last PV
    fence_after_sync();
    const float inv = 1.f / l;
    const size_t row = (size_t)row0 + qi * 128 + r;
    store_row<D>(tO, inv, out + row * hd + h * D);
    lse[(size_t)bh * S + qi * 128 + r] = m + __log2f(l);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
  if (tr && threadIdx.x == 0) tr[5] = gtimer();
}

// =================================================================== backward: dK, dV
// CTA = kv tile j; sub-tiles over the q columns (q halves of tiles i >= j).
template <int D>
struct Bkv {
  // q / dO half-tile stages; P^T / dS^T live in TMEM, so the shared memory they took holds a
  // fourth stage (the Q / dO loads of sub-tile u+4 wait only for dV / dK of u)
  static constexpr int TB = 128 * D * 2, HB = 64 * D * 2, NST = 4;
  // LD: each stage's 64 lse and 64 delta values (bulk-copied with its q / dO halves)
  static constexpr int K = 0, V = TB, QD = 2 * TB, LD = QD + NST * 2 * HB, BAR = LD + NST * 512;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_do,
                const float* __restrict__ lse, const float* __restrict__ delta,
                __nv_bfloat16* __restrict__ dqkv, int B, int H, int S, int hd, float sl2,
                float scale, int grp, float* __restrict__ csum,
                unsigned long long* __restrict__ trace) {
  // trace (diagnostics, normally null), CTA 0 only, clock64 per sub-tile u:
  // [S warp: qd landed, st_free passed, issued] [acc warp: ps_full passed]
  // [group: st_full passed, ps_empty passed, published]
  unsigned long long* tk = (trace && blockIdx.x == 0) ? trace : nullptr;
  using L = Bkv<D>;
  constexpr int TB = L::TB, HB = L::HB, NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sK = sm + L::K, *sV = sm + L::V, *sQD = sm + L::QD, *sLD = sm + L::LD;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *kv_full = bar, *qd_full = bar + 1, *qd_empty = bar + 1 + NST,
           *st_full = bar + 1 + 2 * NST, *st_free = st_full + 2, *ps_full = st_full + 4,
           *ps_empty = st_full + 6, *acc_done = st_full + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(st_full + 9);

  const int nq = S / 128, BH = B * H;
  int j, bh;                                     // kv tile; small j = many q tiles, first
  tile_order((int)blockIdx.x, nq, BH, grp, j, bh);
  const int b = bh / H, h = bh % H;
  const int nsub = 2 * (nq - j), row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) { mbar_init(&qd_full[s], 1); mbar_init(&qd_empty[s], 1); }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&st_full[g], 1); mbar_init(&st_free[g], GW);
      mbar_init(&ps_full[g], GW); mbar_init(&ps_empty[g], 1);
    }
    mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
    prefetch_map(&tm_do);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  zi::pdl_sync();   // setup above overlapped the previous kernel's tail
  const uint32_t tmem = *tslot;   // slot g: S^T at g*128, dP^T at g*128 + 64; dV 256, dK 384

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * TB);
      load_rows<D, 128>(sK, &tm, kv_full, hd + h * D, row0 + j * 128);
      load_rows<D, 128>(sV, &tm, kv_full, 2 * hd + h * D, row0 + j * 128);
      for (int u = 0; u < nsub; ++u) {
        const int st = u % NST, r = row0 + j * 128 + u * 64;   // q rows of sub-tile u
        mbar_wait(&qd_empty[st], ((u / NST) & 1) ^ 1);
        mbar_expect_tx(&qd_full[st], 2 * HB + 512);
        load_rows<D, 64>(sQD + st * 2 * HB, &tm, &qd_full[st], h * D, r);
        load_rows<D, 64>(sQD + st * 2 * HB + HB, &tm_do, &qd_full[st], h * D, r);
        const size_t q0 = (size_t)bh * S + j * 128 + u * 64;
        bulk::g2s(sLD + st * 512, lse + q0, 256, &qd_full[st]);
        bulk::g2s(sLD + st * 512 + 256, delta + q0, 256, &qd_full[st]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
    mbar_wait(kv_full, 0);
    // S^T / dP^T of sub-tile u into slot g once dV / dK of u-2 have read its P^T / dS^T
    // (which overwrote S^T / dP^T u-2 in TMEM)
    for (int u = 0; u < nsub; ++u) {
      const int st = u % NST, g = u & 1;
      mbar_wait(&qd_full[st], (u / NST) & 1);
      if (tk && lane == 0) tk[u * 8 + 0] = clock64();
      if (u >= 2) mbar_wait(&ps_empty[g], ((u - 2) >> 1) & 1);
      if (tk && lane == 0) tk[u * 8 + 1] = clock64();
      fence_after_sync();
      if (elect_one()) {
        const uint8_t* q = sQD + st * 2 * HB;
        mma_tile<64, false, D / 16>(tmem + g * 128, sK, q, id_s, false);
        mma_tile<64, false, D / 16>(tmem + g * 128 + 64, sV, q + HB, id_s, false);
        umma_commit(&st_full[g]);
      }
      __syncwarp();
      if (tk && lane == 0) tk[u * 8 + 2] = clock64();
    }
  } else if (warp == ACC_WARP) {
    // dV += P^T dO, dK += dS^T Q of sub-tile v once group g published them
    constexpr uint32_t id_d = idesc_bf16_f32(128, D, false, true);
    for (int v = 0; v < nsub; ++v) {
      const int st = v % NST, g = v & 1;
      mbar_wait(&ps_full[g], (v >> 1) & 1);
      if (tk && lane == 0) tk[v * 8 + 3] = clock64();
      fence_after_sync();
      if (elect_one()) {
        const uint8_t* q = sQD + st * 2 * HB;
        mma_tile_ts<64, 4>(tmem + 256, tmem + g * 128, q + HB, id_d, v > 0);      // P^T
        mma_tile_ts<64, 4>(tmem + 384, tmem + g * 128 + 64, q, id_d, v > 0);  // dS^T
        umma_commit(&qd_empty[st]);
        umma_commit(&ps_empty[g]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(acc_done);
    __syncwarp();
  } else {
    // thread = kv row r of the tile; group g owns the sub-tiles u = 2*it + g (64 q each)
    const int g = (warp - 2) >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    const uint32_t tST = tmem + g * 128 + lo, tdPT = tST + 64;
    const int nit = nsub / 2;
    for (int it = 0; it < nit; ++it) {
      // lse / delta of the sub-tile's 64 queries, bulk-copied into the stage with its q /
      // dO halves (shared-memory broadcast reads instead of dependent global loads)
      const int u = 2 * it + g, ust = u % L::NST;
      const float4* lq = reinterpret_cast<const float4*>(sLD + ust * 512);
      const float4* dq4 = reinterpret_cast<const float4*>(sLD + ust * 512 + 256);
      mbar_wait(&st_full[g], it & 1);
      mbar_wait(&qd_full[ust], (u / L::NST) & 1);  // complete already (the MMA waited on it)
      unsigned long long* tg = (tk && lane == 0 && q4 == 0) ? tk + u * 8 : nullptr;
      if (tg) tg[4] = clock64();
      fence_after_sync();
      if (tg) tg[5] = clock64();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t s32[32], p32[32];
        tmem_ld32_nowait(tST + c * 32, s32);
        tmem_ld32_nowait(tdPT + c * 32, p32);
        float Ls[32], Ds[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 a = lq[c * 8 + k], d = dq4[c * 8 + k];
          Ls[4 * k] = a.x; Ls[4 * k + 1] = a.y; Ls[4 * k + 2] = a.z; Ls[4 * k + 3] = a.w;
          Ds[4 * k] = d.x; Ds[4 * k + 1] = d.y; Ds[4 * k + 2] = d.z; Ds[4 * k + 3] = d.w;
        }
        tmem_wait_ld();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int q = c * 32 + k;
          float p0 = ex2(fmaf(u2f(s32[k]), sl2, -Ls[k]));
          float p1 = ex2(fmaf(u2f(s32[k + 1]), sl2, -Ls[k + 1]));
          if (it == 0) {                          // diagonal tile: query before key
            if (g * 64 + q < r) p0 = 0.f;
            if (g * 64 + q + 1 < r) p1 = 0.f;
          }
          pp[k >> 1] = pack_bf16(p0, p1);
          dd[k >> 1] = pack_bf16(p0 * (u2f(p32[k]) - Ds[k]), p1 * (u2f(p32[k + 1]) - Ds[k + 1]));
        }
        // P^T / dS^T (bf16 pairs) over this thread's S^T / dP^T columns already read:
        // chunk c writes columns c*16 .. c*16+15, read by chunk 0
        tmem_st16_nowait(tST + c * 16, pp);
        tmem_st16_nowait(tdPT + c * 16, dd);
      }
      tmem_wait_st();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps_full[g]);
      if (tg) tg[6] = clock64();
    }
    mbar_wait(acc_done, 0);
    fence_after_sync();
    const size_t row = (size_t)row0 + j * 128 + r;
    __nv_bfloat16* d = dqkv + row * 3 * hd;
    if (csum == nullptr) {
      if (g == 0) store_row<D>(tmem + 256 + lo, 1.f, d + 2 * hd + h * D);
      else store_row<D>(tmem + 384 + lo, scale, d + hd + h * D);
    } else {   // + the qkv bias gradient's 32-row block partials of dV / dK
      float* cp = csum + ((size_t)row0 + j * 128 + q4 * 32) / 32 * (3 * hd);
      if (g == 0) store_row_csum<D>(tmem + 256 + lo, 1.f, d + 2 * hd + h * D, cp + 2 * hd + h * D, lane);
      else store_row_csum<D>(tmem + 384 + lo, scale, d + hd + h * D, cp + hd + h * D, lane);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_free512(tmem);
  }
}

// ======================================================================= backward: dQ
// CTA = q tile i; sub-tiles over the kv columns (kv halves of tiles j <= i).
template <int D>
struct Bq {
  // kv half stages; dS lives in TMEM (over S), so its former shared memory is a 5th stage
  static constexpr int TB = 128 * D * 2, HB = 64 * D * 2, NST = 5;
  static constexpr int Q = 0, DO = TB, KV = 2 * TB, BAR = KV + NST * 2 * HB;
  static constexpr int BYTES = BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
bwd_dq_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_do,
              const float* __restrict__ lse, const float* __restrict__ delta,
              __nv_bfloat16* __restrict__ dqkv, int B, int H, int S, int hd, float sl2,
              float scale, int grp, float* __restrict__ csum) {
  using L = Bq<D>;
  constexpr int TB = L::TB, HB = L::HB, NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  uint8_t *sQ = sm + L::Q, *sdO = sm + L::DO, *sKV = sm + L::KV;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t *qd_full = bar, *kv_full = bar + 1, *kv_empty = bar + 1 + NST,
           *s_full = bar + 1 + 2 * NST, *s_free = s_full + 2, *ds_full = s_full + 4,
           *ds_empty = s_full + 6, *acc_done = s_full + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(s_full + 9);

  const int nq = S / 128, BH = B * H;
  int i, bh;
  tile_order((int)blockIdx.x, nq, BH, grp, i, bh);
  i = nq - 1 - i;
  const int b = bh / H, h = bh % H;
  const int nsub = 2 * (i + 1), row0 = b * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(qd_full, 1);
    for (int s = 0; s < NST; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1); mbar_init(&s_free[g], GW);
      mbar_init(&ds_full[g], GW); mbar_init(&ds_empty[g], 1);
    }
    mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tm);
    prefetch_map(&tm_do);
  }
  if (warp == 1) tmem_alloc512(tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  zi::pdl_sync();   // setup above overlapped the previous kernel's tail
  const uint32_t tmem = *tslot;   // slot g: S at g*128, dP at g*128 + 64; dQ at 256

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qd_full, 2 * TB);
      load_rows<D, 128>(sQ, &tm, qd_full, h * D, row0 + i * 128);
      load_rows<D, 128>(sdO, &tm_do, qd_full, h * D, row0 + i * 128);
      for (int u = 0; u < nsub; ++u) {
        const int st = u % NST, r = row0 + u * 64;      // kv rows of sub-tile u
        mbar_wait(&kv_empty[st], ((u / NST) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * HB);
        load_rows<D, 64>(sKV + st * 2 * HB, &tm, &kv_full[st], hd + h * D, r);
        load_rows<D, 64>(sKV + st * 2 * HB + HB, &tm, &kv_full[st], 2 * hd + h * D, r);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
    mbar_wait(qd_full, 0);
    // S / dP of sub-tile u into slot g once dQ of u-2 has read its dS (over S u-2 in TMEM)
    for (int u = 0; u < nsub; ++u) {
      const int st = u % NST, g = u & 1;
      mbar_wait(&kv_full[st], (u / NST) & 1);
      if (u >= 2) mbar_wait(&ds_empty[g], ((u - 2) >> 1) & 1);
      fence_after_sync();
      if (elect_one()) {
        const uint8_t* kv = sKV + st * 2 * HB;
        mma_tile<64, false, D / 16>(tmem + g * 128, sQ, kv, id_s, false);
        mma_tile<64, false, D / 16>(tmem + g * 128 + 64, sdO, kv + HB, id_s, false);
        umma_commit(&s_full[g]);
      }
      __syncwarp();
    }
  } else if (warp == ACC_WARP) {
    // dQ += dS K of sub-tile v once group g published dS_v
    constexpr uint32_t id_d = idesc_bf16_f32(128, D, false, true);
    for (int v = 0; v < nsub; ++v) {
      const int st = v % NST, g = v & 1;
      mbar_wait(&ds_full[g], (v >> 1) & 1);
      fence_after_sync();
      if (elect_one()) {
        mma_tile_ts<64, 4>(tmem + 256, tmem + g * 128, sKV + st * 2 * HB, id_d, v > 0);
        umma_commit(&kv_empty[st]);
        umma_commit(&ds_empty[g]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(acc_done);
    __syncwarp();
  } else {
    const int g = (warp - 2) >> 2, q4 = warp & 3, r = q4 * 32 + lane;
    const uint32_t lo = (uint32_t)(q4 * 32) << 16;
    const uint32_t tSg = tmem + g * 128 + lo, tdPg = tSg + 64;
    const float nl = -lse[(size_t)bh * S + i * 128 + r];
    const float del = delta[(size_t)bh * S + i * 128 + r];
    const int nit = nsub / 2;
    for (int jj = 0; jj < nit; ++jj) {
      mbar_wait(&s_full[g], jj & 1);
      fence_after_sync();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t s32[32], p32[32];
        tmem_ld32_nowait(tSg + c * 32, s32);
        tmem_ld32_nowait(tdPg + c * 32, p32);
        tmem_wait_ld();
        uint32_t dd[16];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int kv = g * 64 + c * 32 + k;
          float p0 = ex2(fmaf(u2f(s32[k]), sl2, nl));
          float p1 = ex2(fmaf(u2f(s32[k + 1]), sl2, nl));
          if (jj == i) {                          // diagonal tile: key after query
            if (kv > r) p0 = 0.f;
            if (kv + 1 > r) p1 = 0.f;
          }
          dd[k >> 1] = pack_bf16(p0 * (u2f(p32[k]) - del), p1 * (u2f(p32[k + 1]) - del));
        }
        tmem_st16_nowait(tSg + c * 16, dd);   // dS over S columns chunk 0 has read
      }
      tmem_wait_st();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[g]);
    }
    mbar_wait(acc_done, 0);
    fence_after_sync();
    const size_t row = (size_t)row0 + i * 128 + r;
    if (csum == nullptr)
      store_row<D / 2>(tmem + 256 + lo + g * (D / 2), scale,
                       dqkv + row * 3 * hd + h * D + g * (D / 2));
    else
      store_row_csum<D / 2>(tmem + 256 + lo + g * (D / 2), scale,
                            dqkv + row * 3 * hd + h * D + g * (D / 2),
                            csum + ((size_t)row0 + i * 128 + q4 * 32) / 32 * (3 * hd) + h * D +
                                g * (D / 2), lane);
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
  zi::pdl_sync();
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
static unsigned long long* g_trace = nullptr;   // zi_attn_set_trace (diagnostics)

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

// batch-heads per CTA group (tile_order); default one group (rank-major over all
// batch-heads: measured 1-8 % faster than groups of 1-32, the K / V re-reads are not the
// bound); ZI_ATTN_GROUP=G for A/B
static int attn_group(int BH) {
  static int g = -1;
  if (g < 0) {
    const char* e = getenv("ZI_ATTN_GROUP");
    g = e ? atoi(e) : 0;
  }
  return (g <= 0 || g > BH) ? BH : g;
}

// ZI_ATTN_FWD2=0: the one-Q-tile forward everywhere (A/B)
static bool use_fwd2() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZI_ATTN_FWD2");
    v = (e && atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
}

template <int D>
static int fwd(const void* qkv, void* out, float* lse, int B, int H, int S, cudaStream_t st) {
  const int hd = H * D;
  int rc = encoder();
  if (rc != ZI_OK) return rc;
  CUtensorMap tm;
  if ((rc = make_map(&tm, qkv, B * S, 3 * hd, 3 * hd)) != ZI_OK) return rc;
  if (S % 256 == 0 && use_fwd2()) {   // two q tiles per CTA
    static bool attr2 = false;
    if ((rc = set_smem(fwd2_kernel<D>, Fwd2<D>::BYTES, attr2)) != ZI_OK) return rc;
    const float sl2 = LOG2E / sqrtf((float)D);
    zi::launch_pdl(fwd2_kernel<D>, dim3(B * H * (S / 256)), dim3(320), Fwd2<D>::BYTES, st, tm,
                   static_cast<__nv_bfloat16*>(out), lse, B, H, S, hd, sl2, g_trace);
    return launch_status("zi_attn_fwd");
  }
  static bool attr = false;
  if ((rc = set_smem(fwd_kernel<D>, Fwd<D>::BYTES, attr)) != ZI_OK) return rc;
  const float sl2 = LOG2E / sqrtf((float)D);
  zi::launch_pdl(fwd_kernel<D>, dim3(B * H * (S / 128)), dim3(THREADS), Fwd<D>::BYTES, st,
                 tm, static_cast<__nv_bfloat16*>(out), lse, B, H, S, hd, sl2, g_trace,
                 attn_group(B * H));
  return launch_status("zi_attn_fwd");
}

template <int D>
static int bwd(const void* qkv, const void* out, const void* dout, const float* lse, float* delta,
               void* dqkv, int B, int H, int S, float* csum, cudaStream_t st) {
  const int hd = H * D;
  int rc = encoder();
  if (rc != ZI_OK) return rc;
  CUtensorMap tm, tdo;
  if ((rc = make_map(&tm, qkv, B * S, 3 * hd, 3 * hd)) != ZI_OK) return rc;
  if ((rc = make_map(&tdo, dout, B * S, hd, hd)) != ZI_OK) return rc;
  static bool a1 = false, a2 = false;
  if ((rc = set_smem(bwd_dkdv_kernel<D>, Bkv<D>::BYTES, a1)) != ZI_OK) return rc;
  if ((rc = set_smem(bwd_dq_kernel<D>, Bq<D>::BYTES, a2)) != ZI_OK) return rc;
  if (out != nullptr) {   // else delta already holds rowsum(dO o O) (zi_gemm_sk_aux)
    zi::launch_pdl(delta_kernel<D>, dim3(B * S), dim3(hd / 8), 0, st, static_cast<const __nv_bfloat16*>(out),
                                              static_cast<const __nv_bfloat16*>(dout), delta, H, S, hd);
    if ((rc = launch_status("zi_attn_bwd(delta)")) != ZI_OK) return rc;
  }
  const float scale = 1.f / sqrtf((float)D), sl2 = LOG2E * scale;
  const int grid = B * H * (S / 128);
  auto* dq = static_cast<__nv_bfloat16*>(dqkv);
  // (a 128-column dK / dV variant with P^T / dS^T aliased into TMEM — N = 128 score MMAs,
  // no shared-memory round trip — measured 5 % slower: with TMEM full, the next q tile's
  // scores cannot overlap the elementwise work, so MMA and softmax serialise)
  zi::launch_pdl(bwd_dkdv_kernel<D>, dim3(grid), dim3(THREADS), Bkv<D>::BYTES, st, tm, tdo,
                 lse, delta, dq, B, H, S, hd, sl2, scale, attn_group(B * H), csum, g_trace);
  if ((rc = launch_status("zi_attn_bwd(dkdv)")) != ZI_OK) return rc;
  // (likewise a 128-column dQ variant with dS in TMEM, one score slot overlapped with the
  // previous tile's elementwise work: 4 % slower than the two 64-column groups)
  zi::launch_pdl(bwd_dq_kernel<D>, dim3(grid), dim3(THREADS), Bq<D>::BYTES, st, tm, tdo, lse,
                 delta, dq, B, H, S, hd, sl2, scale, attn_group(B * H), csum);
  return launch_status("zi_attn_bwd(dq)");
}

}  // namespace attn
}  // namespace zi

extern "C" {

int zi_attn_set_trace(void* buf) {
  zi::attn::g_trace = static_cast<unsigned long long*>(buf);
  return ZI_OK;
}

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
  return zi_attn_bwd_colsum(qkv, out, dout, lse, delta, dqkv, B, H, S, head_dim, nullptr, stream);
}

int zi_attn_bwd_colsum(const void* qkv, const void* out, const void* dout, const float* lse,
                       float* delta, void* dqkv, int B, int H, int S, int head_dim,
                       float* colsum_part, void* stream) {
  int rc = zi::attn::check(qkv, B, H, S, head_dim, "zi_attn_bwd");
  if (rc != ZI_OK) return rc;
  // out == NULL: delta already holds rowsum(dout o out) (the proj.dx GEMM's epilogue)
  ZI_CHECK_ARG(dout && lse && delta && dqkv, "zi_attn_bwd: NULL argument");
  ZI_CHECK_ARG(zi::aligned(out, 16) && zi::aligned(dout, 16) && zi::aligned(dqkv, 16),
               "zi_attn_bwd: 16-byte alignment");
  ZI_CHECK_ARG(H * head_dim / 8 <= 1024, "zi_attn_bwd: hidden %d too wide", H * head_dim);
  cudaStream_t s = (cudaStream_t)stream;
  return head_dim == 64 ? zi::attn::bwd<64>(qkv, out, dout, lse, delta, dqkv, B, H, S, colsum_part, s)
                        : zi::attn::bwd<128>(qkv, out, dout, lse, delta, dqkv, B, H, S, colsum_part, s);
}

}  // extern "C"
