// Stream-K GEMM for the GPT step's linears (the block's qkv / proj / fc1 / fc2 and the
// tied head, forward, input gradient and weight gradient), on the 5th-gen tensor cores.
//
//   D[m, n] = epi( sum_k A(m, k) * B(n, k) )
//
// A(m, k) is K-major (A[m*lda + k]) or M-major (A[k*lda + m]); B likewise. bf16
// operands, fp32 accumulation in TMEM; bf16 output with a fused epilogue (bias,
// bias + GELU with both outputs, bias + residual, GELU' of the fc1 pre-activation)
// or fp32 output (the tied head's weight gradient).
//
// Why a second GEMM next to gemm_sm100.cu's: at the GPT-1.3B shapes (K = 2048 ..
// 8192, N = 2048 .. 8192) a pair tile takes 10-40 us, so a whole-tile persistent
// schedule loses up to a wave to quantization (proj: 256 pair tiles on 74 CTA pairs =
// 3.46 waves -> 4; proj.dW: 64 tiles on 74 pairs), and a single TMEM accumulator
// exposes every tile's epilogue. This kernel:
//   * CTA pairs (cluster of 2) run tcgen05.mma.cta_group::2 on a 256 x 256 pair tile
//     (M = 256, N = 256, K = 16 per instruction), each CTA staging its 128 rows of A
//     and its half of B's 256 rows through a TMA ring (SWIZZLE_128B);
//   * two 256-column fp32 accumulators in TMEM, so the epilogue of item j runs while
//     the MMA works on item j + 1;
//   * hybrid stream-K schedule: with P pairs and T tiles of nk k-blocks, the first S
//     tiles (S = T mod P, or all T when T < P) are cut into S*nk k-block units
//     dealt out evenly, unit range [q*U/P, (q+1)*U/P) to pair q; the remaining T - S
//     tiles (a multiple of P) are whole tiles round-robin. Every pair does the same
//     work to within one k-block;
//   * a tile cut across pairs is finished by the pair holding its first k-block (it
//     reaches it last in its range); every other contributor q holds the tile's later
//     k-blocks at the *start* of its range, writes its fp32 partial to its own
//     workspace slot and raises a per-warp flag. The finisher adds the partials in
//     pair order (fixed, so the result is deterministic run to run) and runs the
//     epilogue. Each pair writes at most one partial (only its first item can start
//     mid-tile), so the workspace is one 128 x 256 fp32 slot per CTA;
//   * epilogue warps: TMEM -> registers (tcgen05.ld.32x32b, lane = row) -> math ->
//     SW128 staging boxes in shared memory -> TMA stores.
// No reference counterpart: the SPEC's step only names "the GEMM"
// (SPEC.md:649-667, 747-755); this is the build's B200 implementation of it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace zi {
namespace gsk {
using namespace zi::tc;

constexpr int BK = 64;
constexpr int A_BYTES = 128 * BK * 2;       // this CTA's 128 rows of A per k-block
constexpr int B_BYTES = 128 * BK * 2;       // this CTA's 128 of the pair tile's 256 B rows
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int MN_BOX_BYTES = 64 * BK * 2;   // one 64(mn) x 64(k) MN-major box
constexpr int BOX_BYTES = 32 * 128;         // staging box: 32 rows x 128 B (SW128)
constexpr int TMEM_COLS = 512;              // two 256-column fp32 accumulators
constexpr int SLOT_FLOATS = 128 * 256;      // one CTA's partial accumulator
constexpr int FLAG_BYTES = 1 << 16;         // flag area at the start of the workspace
constexpr int GROUP_M = 16;

constexpr int EPI_PLAIN = ZI_EPI_PLAIN, EPI_GELU = ZI_EPI_GELU, EPI_RESID = ZI_EPI_RESID,
              EPI_DGELU = ZI_EPI_DGELU, EPI_GELU_SAVE = ZI_EPI_GELU_SAVE, EPI_MUL = ZI_EPI_MUL,
              EPI_F32 = 16;

constexpr size_t smem_bytes(int NS, int EW, int BPW) {
  return (size_t)NS * STAGE_BYTES + (size_t)EW * BPW * BOX_BYTES + 1024 + 256;
}

// Optional epilogue side outputs (bf16 output only; nullptr = off):
//   csum:  column sums of the stored bf16 output per 32-row block, fp32 [ceil(M/32)][N]
//          (a bias gradient's partials; zi_colsum_fold sums the blocks in order);
//   delta: per (row, head) sum over the head's D columns of out * X (X = the attention
//          output O, out = dO): the attention backward's rowsum(dO o O), fp32 [B][H][S]
//          for row = b * S + s, head = column / D (D = 64 or 128).
struct Aux {
  float* csum;
  float* delta;
  int S, H, D;
};

// Work decomposition, identical in every warp of both CTAs of a pair.
struct Sched {
  int tiles_m, tiles_n, T, nk, P, S, group_m;
};

struct Item {
  int t, k0, k1, role;   // tile, k-block range [k0, k1), role
};
enum { ROLE_FULL = 0, ROLE_FINISH = 1, ROLE_PARTIAL = 2 };

__device__ __forceinline__ int sk_begin(const Sched& s, int q) {
  return (int)((long long)q * s.S * s.nk / s.P);
}

struct Iter {
  Sched s;
  int u, b, dpt;
  __device__ Iter(const Sched& sc, int p) : s(sc) {
    u = sk_begin(sc, p);
    b = sk_begin(sc, p + 1);
    dpt = sc.S + p;
  }
  __device__ bool next(Item& w) {
    if (u < b) {
      const int t = u / s.nk;
      const int k0 = u - t * s.nk;
      const int k1 = min(b - t * s.nk, s.nk);
      w.t = t; w.k0 = k0; w.k1 = k1;
      w.role = k0 > 0 ? ROLE_PARTIAL : (k1 < s.nk ? ROLE_FINISH : ROLE_FULL);
      u = t * s.nk + k1;
      return true;
    }
    if (dpt < s.T) {
      w.t = dpt; w.k0 = 0; w.k1 = s.nk; w.role = ROLE_FULL;
      dpt += s.P;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_m, int& mt,
                                            int& nt) {
  const int per_group = group_m * tiles_n;
  const int g = t / per_group;
  const int first = g * group_m;
  const int gm = min(tiles_m - first, group_m);
  const int r = t % per_group;
  mt = first + r % gm;
  nt = r / gm;
}

// Rows [r0, r0 + 128) of an operand for k-block k0 (K-major: one box of 128 rows;
// MN-major: two boxes of 64 mn x 64 k).
template <bool MN>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint32_t lbar,
                                          int k0, int r0) {
  if (!MN) {
    tma_load_2d_2sm(dst, map, lbar, k0, r0);
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) tma_load_2d_2sm(dst + j * MN_BOX_BYTES, map, lbar, r0 + 64 * j, k0);
  }
}

__device__ __forceinline__ float bf16f(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// 64 accumulator columns of one row (fp32 bits in v) through the bf16 epilogue,
// packed to 32 bf16x2 words. Columns past N compute values the TMA store clips.
template <int EPI>
__device__ __forceinline__ void epi_words(const uint32_t* v, int row, int col0, int M, int N,
                                          const __nv_bfloat16* __restrict__ bias,
                                          const uint16_t* __restrict__ X, int ldx, uint32_t* w) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = col0 + 8 * q;
    const bool in = c < N;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[8 * q + j]);
    if (bias != nullptr && in) {
      const uint4 bv = *reinterpret_cast<const uint4*>(bias + c);
      const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        f[2 * j] += bf16f(bw[j] & 0xFFFF);
        f[2 * j + 1] += bf16f(bw[j] >> 16);
      }
    }
    if (EPI == EPI_RESID || EPI == EPI_DGELU || EPI == EPI_MUL) {
      uint4 xv = make_uint4(0, 0, 0, 0);
      if (in && row < M) xv = *reinterpret_cast<const uint4*>(X + (size_t)row * ldx + c);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x0 = bf16f(xw[j] & 0xFFFF), x1 = bf16f(xw[j] >> 16);
        if (EPI == EPI_RESID) {
          f[2 * j] = rbf(f[2 * j]) + x0;
          f[2 * j + 1] = rbf(f[2 * j + 1]) + x1;
        } else if (EPI == EPI_MUL) {
          f[2 * j] = rbf(f[2 * j]) * x0;
          f[2 * j + 1] = rbf(f[2 * j + 1]) * x1;
        } else {
          f[2 * j] = rbf(f[2 * j]) * gelu_tanh_grad(x0);
          f[2 * j + 1] = rbf(f[2 * j + 1]) * gelu_tanh_grad(x1);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) w[4 * q + j] = pack_bf16(f[2 * j], f[2 * j + 1]);
  }
}

// 8 x 16 B of one row (lane) into a SW128 staging box: chunk j at j ^ (row % 8).
__device__ __forceinline__ void stage_row(uint8_t* box, int lane, const uint32_t* w) {
  const uint32_t base = smem_u32(box) + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t a = base + ((uint32_t)(j ^ (lane & 7)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[4 * j]),
                 "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3]) : "memory");
  }
}

// mbar_wait with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or ~1 ms passes) instead of re-polling, so the epilogue and producer
// warps that wait most of a tile draw no issue slots (or power) while they wait.
__device__ __forceinline__ void mbar_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  long long t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(a), "r"(parity), "r"(1000000u) : "memory");
    if (done) return;
    if (t0 == 0) t0 = clock64();
    else if (clock64() - t0 > 20000000000LL) __trap();
  }
}

// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}"
               : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CL CTAs per cluster: CL = 2 is one CTA pair on a 256 x 256 tile; CL = 4 is two pairs
// side by side along N (a 256 x 512 cluster tile) that share A: CTA c of pair j loads
// A rows [c*128 + j*64, +64) of the stage and multicasts them to CTA c of both pairs,
// so each A byte crosses from L2 once per cluster (25 % less L2 -> SM traffic).
// CL = 4 launches as a *preferred* cluster of 4 over regular clusters of 2: where a GPC
// has no room for 4 more CTAs the hardware forms two pairs instead, so every SM runs.
// The schedule is the same either way (blocks 4c .. 4c + 3 work on cluster tile items
// of preferred cluster c, pair (blockIdx / 2) % 2 on its half); only the A loads differ
// (a lone pair loads both 64-row halves itself), so the result does not depend on how
// the clusters formed.
// NS ring stages, EW epilogue warps (multiple of 4: EW / 4 warps share a TMEM lane
// quadrant, splitting its 256 columns), BPW staging boxes per epilogue warp.
template <bool A_MN, bool B_MN, int EPI, int NS, int EW, int BPW, int CL>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
gemm_sk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmD2,
               const __nv_bfloat16* __restrict__ bias, const uint16_t* __restrict__ X, int ldx,
               int M, int N, const Sched sc, float* __restrict__ ws_part,
               uint32_t* __restrict__ ws_flag, const Aux aux) {
  static_assert(CL == 2 || CL == 4, "clusters of one or two CTA pairs");
  constexpr int NPAIR = CL / 2;
  constexpr int CT_N = 256 * NPAIR;                  // cluster tile columns
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NS * A_BYTES;
  uint8_t* sOut = sB + NS * B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + EW * BPW * BOX_BYTES);
  uint64_t* empty = full + NS;
  uint64_t* tmem_full = empty + NS;     // [2]
  uint64_t* tmem_empty = tmem_full + 2; // [2], pair leader only: 2 * EW arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  // npair: pairs in this cluster as formed (CL = 4: 2, or 1 when it fell back to a pair);
  // pj: which half of the cluster tile this pair computes (fixed by blockIdx); prank:
  // the pair's index inside the formed cluster (multicast masks)
  const uint32_t npair = CL == 4 ? cluster_nctarank() >> 1 : 1;
  const uint32_t crank = rank & 1, prank = rank >> 1, lead = rank & ~1u;
  const uint32_t pj = CL == 4 ? (blockIdx.x >> 1) & 1 : 0;
  const uint32_t pos = blockIdx.x % CL;   // position in the (preferred) cluster: ws slots
  const bool leader = crank == 0;
  const int cid = blockIdx.x / CL;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], npair);        // every pair's MMAs released the slot
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 2 * EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&tmA);
    prefetch_map(&tmB);
    prefetch_map(&tmD);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before_sync();
  __syncthreads();
  cluster_sync();
  fence_after_sync();
  zi::pdl_sync();   // setup above overlapped the previous kernel's tail
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer (every CTA; bytes complete on its pair leader's full[s])
    if (lane == 0) {
      Iter itr(sc, cid);
      Item w;
      uint32_t it = 0;
      constexpr uint16_t AMASK = 0x5;     // CTA c of both pairs (shifted by c below)
      while (itr.next(w)) {
        int mt, nt;
        tile_coords(w.t, sc.tiles_m, sc.tiles_n, sc.group_m, mt, nt);
        const int m0 = mt * 256 + (int)crank * 128;
        const int n0 = nt * CT_N + (int)pj * 256 + (int)crank * 128;
        for (int kb = w.k0; kb < w.k1; ++kb, ++it) {
          const int s = it % NS;
          mbar_sleep(&empty[s], ((it / NS) & 1) ^ 1);
          const uint32_t lbar = map_to_rank(smem_u32(&full[s]), lead);
          if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
          if (NPAIR == 1) {
            load_rows<A_MN>(sA + s * A_BYTES, &tmA, lbar, kb * BK, m0);
          } else if (npair == 2) {   // one 64-row box (K-major {64 k, 64 rows}; MN-major {64 mn, 64 k})
            uint8_t* dst = sA + s * A_BYTES + prank * (A_BYTES / 2);
            const int r = m0 + (int)prank * 64;
            if (!A_MN) tma_load_2d_2sm_mc(dst, &tmA, lbar, kb * BK, r, (uint16_t)(AMASK << crank));
            else tma_load_2d_2sm_mc(dst, &tmA, lbar, r, kb * BK, (uint16_t)(AMASK << crank));
          } else {                   // a lone pair: both 64-row boxes, no multicast
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint8_t* dst = sA + s * A_BYTES + h * (A_BYTES / 2);
              if (!A_MN) tma_load_2d_2sm(dst, &tmA, lbar, kb * BK, m0 + 64 * h);
              else tma_load_2d_2sm(dst, &tmA, lbar, m0 + 64 * h, kb * BK);
            }
          }
          load_rows<B_MN>(sB + s * B_BYTES, &tmB, lbar, kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (each pair leader): the whole warp waits, one elected lane issues.
    // Descriptors are precomputed per ring slot; the k-steps add to the address field.
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256, A_MN, B_MN);
      constexpr uint64_t ka = A_MN ? (2 * 1024) >> 4 : 32 >> 4;   // per 16-deep k step
      constexpr uint64_t kb_ = B_MN ? (2 * 1024) >> 4 : 32 >> 4;
      const uint16_t ALL = (uint16_t)((1u << (2 * npair)) - 1);
      const uint16_t PAIR = (uint16_t)(0x3u << (2 * prank));
      const uint64_t da0 = sdesc_sw128(smem_u32(sA), A_MN ? MN_BOX_BYTES : 16);
      const uint64_t db0 = sdesc_sw128(smem_u32(sB), B_MN ? MN_BOX_BYTES : 16);
      Iter itr(sc, cid);
      Item w;
      uint32_t it = 0, j = 0;
      while (itr.next(w)) {
        const uint32_t acc = j & 1;
        mbar_wait(&tmem_empty[acc], ((j >> 1) & 1) ^ 1);
        fence_after_sync();
        const uint32_t d = tmem + acc * 256;
        for (int kb = w.k0; kb < w.k1; ++kb, ++it) {
          const int s = it % NS;
          mbar_wait(&full[s], (it / NS) & 1);
          fence_after_sync();
          if (elect_one()) {
            const uint64_t da = da0 + (uint64_t)((s * A_BYTES) >> 4);
            const uint64_t db = db0 + (uint64_t)((s * B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(d, da + k * ka, db + k * kb_, idesc, (kb != w.k0 || k != 0) ? 1u : 0u);
            umma_commit_2sm(&empty[s], ALL);   // the slot (and its multicast A) is free
          }
          __syncwarp();
        }
        if (elect_one()) umma_commit_2sm(&tmem_full[acc], PAIR);
        __syncwarp();
        ++j;
      }
    }
  } else {
    // ---- epilogue: warp e = warp - 2 reads TMEM lane quadrant q = warp % 4 (rows
    // 32q .. 32q + 31 of this CTA's 128) and columns [sub * CPW, (sub + 1) * CPW)
    const int e = warp - 2;
    const int q = warp & 3, sub = e >> 2;
    constexpr int CPW = 256 / (EW / 4);           // columns per warp
    constexpr int CH = CPW / 64;                  // 64-column chunks per warp
    static_assert(CH >= 1 && CPW % 64 == 0, "epilogue warp split");
    uint8_t* wbox = sOut + e * BPW * BOX_BYTES;
    uint32_t bsel = 0;
    auto next_box = [&]() -> uint8_t* {
      uint8_t* box = wbox + bsel * BOX_BYTES;
      bsel = bsel + 1 == BPW ? 0 : bsel + 1;
      if (lane == 0) bulk_wait_read<BPW - 1>();   // the box's previous store has read it
      __syncwarp();
      return box;
    };
    auto emit = [&](const CUtensorMap* map, const uint32_t* w, int c0, int r0) -> const uint8_t* {
      uint8_t* box = next_box();
      stage_row(box, lane, w);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map, box, c0, r0);
        bulk_commit();
      }
      return box;
    };
    float dsum = 0.f;   // aux.delta: this row's running sum over the current head
    Iter itr(sc, cid);
    Item w;
    uint32_t j = 0;
    while (itr.next(w)) {
      int mt, nt;
      tile_coords(w.t, sc.tiles_m, sc.tiles_n, sc.group_m, mt, nt);
      const uint32_t acc = j & 1;
      mbar_sleep(&tmem_full[acc], (j >> 1) & 1);
      fence_after_sync();
      const uint32_t base = tmem + acc * 256 + ((uint32_t)(q * 32) << 16);
      const int r0 = mt * 256 + (int)crank * 128 + q * 32;
      const int row = r0 + lane;
      if (w.role == ROLE_PARTIAL) {
        // lane-interleaved slot layout: float4 i of chunk c of lane l at ((c*16 + i)*32 + l);
        // the finisher's same warp and lane reads it back, and every warp access is 512
        // contiguous bytes
        float4* dst = reinterpret_cast<float4*>(ws_part + (size_t)blockIdx.x * SLOT_FLOATS) +
                      (size_t)e * (CH * 16 * 32) + lane;
#pragma unroll 1
        for (int c = 0; c < CH; ++c) {
          const int col = sub * CPW + c * 64;
          uint32_t v[64];
          tmem_ld32_nowait(base + col, v);
          tmem_ld32_nowait(base + col + 32, v + 32);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i)
            __stcg(dst + (c * 16 + i) * 32,
                   make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                               __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
        }
        fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tmem_empty[acc], lead);
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(ws_flag + (size_t)blockIdx.x * EW + e, 1u);
      } else {
        // contributors of a finished tile: clusters p+1 .. whose ranges start inside it
        int qlo = cid + 1, qhi = cid + 1;
        if (w.role == ROLE_FINISH) {
          const int tend = (w.t + 1) * sc.nk;
          while (qhi < sc.P && sk_begin(sc, qhi) < tend) ++qhi;
          if (lane == 0) {
            for (int qq = qlo; qq < qhi; ++qq) {
              if (sk_begin(sc, qq) == sk_begin(sc, qq + 1)) continue;   // empty range
              const uint32_t* f = ws_flag + (size_t)(CL * qq + pos) * EW + e;
              long long t0 = 0;
              while (ld_acquire(f) == 0) {
                if (t0 == 0) t0 = clock64();
                else if (clock64() - t0 > 20000000000LL) __trap();
              }
            }
          }
          __syncwarp();
        }
#pragma unroll 1
        for (int c = 0; c < CH; ++c) {
          const int col = sub * CPW + c * 64;
          uint32_t v[64];
          tmem_ld32_nowait(base + col, v);
          tmem_ld32_nowait(base + col + 32, v + 32);
          tmem_wait_ld();
          if (c == CH - 1) {   // accumulator drained: hand it back to the MMA
            fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tmem_empty[acc], lead);
          }
          for (int qq = qlo; qq < qhi; ++qq) {   // partials in cluster order
            if (sk_begin(sc, qq) == sk_begin(sc, qq + 1)) continue;
            const float4* s4 = reinterpret_cast<const float4*>(
                                   ws_part + (size_t)(CL * qq + pos) * SLOT_FLOATS) +
                               (size_t)e * (CH * 16 * 32) + (size_t)c * 16 * 32 + lane;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float4 p = __ldcg(s4 + i * 32);
              v[4 * i] = __float_as_uint(__uint_as_float(v[4 * i]) + p.x);
              v[4 * i + 1] = __float_as_uint(__uint_as_float(v[4 * i + 1]) + p.y);
              v[4 * i + 2] = __float_as_uint(__uint_as_float(v[4 * i + 2]) + p.z);
              v[4 * i + 3] = __float_as_uint(__uint_as_float(v[4 * i + 3]) + p.w);
            }
          }
          const int gcol = nt * CT_N + (int)pj * 256 + col;
          if (EPI == EPI_F32) {
            emit(&tmD, v, gcol, r0);
            emit(&tmD, v + 32, gcol + 32, r0);
          } else {
            uint32_t wd[32];
            epi_words<EPI>(v, row, gcol, M, N, bias, X, ldx, wd);
            uint32_t wg[EPI == EPI_GELU_SAVE ? 32 : 1];
            if (EPI == EPI_GELU_SAVE) {   // D <- GELU'(u), D2 <- GELU(u), one tanh each
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float g0, g1, d0, d1;
                gelu_and_grad(bf16f(wd[i] & 0xFFFF), g0, d0);
                gelu_and_grad(bf16f(wd[i] >> 16), g1, d1);
                wg[i] = pack_bf16(g0, g1);
                wd[i] = pack_bf16(d0, d1);
              }
            }
            const uint8_t* box = emit(&tmD, wd, gcol, r0);
            if (EPI == EPI_GELU_SAVE) emit(&tmD2, wg, gcol, r0);
            if (aux.csum != nullptr && r0 < M) {
              // column pair (2 lane, 2 lane + 1) of the 32 staged rows, summed in row
              // order (the box is SW128: row r's 16-byte chunk j at (j ^ (r % 8)) * 16)
              const uint32_t b0 = smem_u32(box) + ((lane & 3) << 2);
              float c0 = 0.f, c1 = 0.f;
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                uint32_t wv;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv)
                             : "r"(b0 + r * 128 + ((((uint32_t)lane >> 2) ^ (r & 7)) << 4)));
                if (r0 + r < M) {   // rows past M hold epilogue values of zero rows
                  c0 += bf16f(wv & 0xFFFF);
                  c1 += bf16f(wv >> 16);
                }
              }
              const int c = gcol + 2 * lane;
              if (c < N)
                *reinterpret_cast<float2*>(aux.csum + (size_t)(r0 >> 5) * N + c) = make_float2(c0, c1);
            }
            if (aux.delta != nullptr) {
              if (row < M && gcol < N) {
#pragma unroll
                for (int q8 = 0; q8 < 8; ++q8) {
                  const uint4 ov = *reinterpret_cast<const uint4*>(X + (size_t)row * ldx + gcol + 8 * q8);
                  const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    dsum = fmaf(bf16f(wd[4 * q8 + j] & 0xFFFF), bf16f(ow[j] & 0xFFFF), dsum);
                    dsum = fmaf(bf16f(wd[4 * q8 + j] >> 16), bf16f(ow[j] >> 16), dsum);
                  }
                }
              }
              if ((gcol + 64) % aux.D == 0) {   // the head's last 64 columns
                if (row < M && gcol < N) {
                  const int b = row / aux.S, sq = row - b * aux.S, h = gcol / aux.D;
                  aux.delta[((size_t)b * aux.H + h) * aux.S + sq] = dsum;
                }
                dsum = 0.f;
              }
            }
            if (EPI == EPI_GELU) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                wd[i] = pack_bf16(gelu_tanh(bf16f(wd[i] & 0xFFFF)), gelu_tanh(bf16f(wd[i] >> 16)));
              emit(&tmD2, wd, gcol, r0);
            }
          }
        }
        if (w.role == ROLE_FINISH && lane == 0) {   // flags back to 0 for the next launch
          for (int qq = qlo; qq < qhi; ++qq)
            if (sk_begin(sc, qq) != sk_begin(sc, qq + 1))
              ws_flag[(size_t)(CL * qq + pos) * EW + e] = 0u;
        }
      }
      ++j;
    }
    if (lane == 0) bulk_wait_all();   // every store landed before the CTA (and its smem) exits
    __syncwarp();
  }
  fence_before_sync();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS) : "memory");
  }
}

// --------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  if (g_encode) return ZI_OK;
  cudaDriverEntryPointQueryResult qr;
  void* fn = nullptr;
  ZI_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr),
          "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
  if (!fn || qr != cudaDriverEntryPointSuccess) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZI_ECUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return ZI_OK;
}

// Operand map: K-major dims {K, rows}, box {64, box_rows}; MN-major dims {rows, K},
// box {64, 64}.
static int make_operand_map(CUtensorMap* m, const void* base, int rows, int K, int ld, bool mn,
                            int box_rows) {
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (!mn) {
    dims[0] = (cuuint64_t)K; dims[1] = (cuuint64_t)rows;
    box[0] = BK; box[1] = (cuuint32_t)box_rows;
  } else {
    dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)K;
    box[0] = 64; box[1] = BK;
  }
  static int promo = -1;
  if (promo < 0) {
    const char* e = getenv("ZI_SK_PROMO");
    promo = e ? atoi(e) : 3;
  }
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(operand) failed (%d)", (int)r);
    return ZI_ECUDA;
  }
  return ZI_OK;
}

// Output map: box of 32 rows x 128 B (64 bf16 or 32 fp32 columns), SW128.
static int make_out_map(CUtensorMap* m, void* base, int rows, int cols, int ld, bool f32) {
  const cuuint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {f32 ? 32u : 64u, 32u}, estr[2] = {1, 1};
  CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(output) failed (%d)", (int)r);
    return ZI_ECUDA;
  }
  return ZI_OK;
}

static int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// Schedule for M x N x K on `clusters` clusters of CL CTAs (cluster tile 256 x 128*CL);
// split = false keeps whole tiles.
static Sched make_sched(int M, int N, int K, int clusters, int CL, bool split) {
  Sched s;
  s.tiles_m = (M + 255) / 256;
  s.tiles_n = (N + 128 * CL - 1) / (128 * CL);
  s.T = s.tiles_m * s.tiles_n;
  s.nk = (K + BK - 1) / BK;
  static int gm = -1;
  if (gm < 0) {
    const char* e = getenv("ZI_SK_GROUP");
    gm = e ? atoi(e) : GROUP_M;
  }
  s.group_m = gm;
  // Stream-K only with at least one whole wave of tiles and short K (<= 256 k-blocks).
  // Cut tiles put the pairs at different k offsets, so the k-slices of A and B are no
  // longer shared in L2 by pairs in lock step: with fewer tiles than pairs (every tile
  // cut; proj.dW measured +50 % DRAM reads) or a long-K GEMM whose operands exceed L2
  // (the tied head's dx, K = 50304) the extra DRAM reads cost more than the wave
  // quantization they remove.
  if (s.nk > 256 || s.T < clusters) split = false;
  // Stream-K over the last partial wave only (S = T mod P tiles, each cut across ~2-3
  // pairs) rather than P + T mod P tiles (each pair ~1.5 tiles): fewer tiles run at
  // staggered k offsets. In the 1.3B step +0.35 % (3 of 3 same-box interleaved rounds,
  // profiles/r2_gemm_power.md); ZI_SK_TAIL=0 restores P + T mod P.
  static int sk_tail = -1;
  if (sk_tail < 0) {
    const char* e = getenv("ZI_SK_TAIL");
    sk_tail = e ? atoi(e) : 1;
  }
  if (!split || s.T % clusters == 0) {
    s.P = s.T < clusters ? s.T : clusters;
    s.S = 0;
  } else {
    s.P = clusters;
    s.S = s.T < clusters ? s.T : (sk_tail ? 0 : clusters) + s.T % clusters;
  }
  return s;
}

constexpr int EW_ = 8;

// How many clusters of CL CTAs (one per SM) can be resident at once: a persistent
// grid larger than that would serialise, and the stream-K finisher spins on its
// contributors, which must all be resident. GPCs are not multiples of 4 SMs, so
// fewer than sms / 4 clusters of 4 fit.
template <int NS_, int BPW_, int CL>
static int max_clusters() {
  static int n = -1;
  if (n < 0) {
    auto kern = gemm_sk_kernel<false, false, EPI_PLAIN, NS_, EW_, BPW_, CL>;
    constexpr size_t SMEM = smem_bytes(NS_, EW_, BPW_);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) !=
        cudaSuccess)
      return 0;
    // CL = 4 launches preferred clusters of 4 over regular pairs, so every resident pair
    // runs: count resident pairs, two per preferred cluster
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 64);
    cfg.blockDim = dim3(64 + 32 * EW_);
    cfg.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = sm_count() / 2;
    }
    c = c * 2 / CL;
    n = c < sm_count() / CL ? c : sm_count() / CL;
  }
  return n;
}

static int sk_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    const char* e = getenv("ZI_SK_CFG");
    cfg = e ? atoi(e) : 6;
  }
  return cfg;
}

template <int CL>
static int resident_clusters() {
  return sk_cfg() == 4 ? max_clusters<4, 2, CL>() : max_clusters<6, 1, CL>();
}

template <bool A_MN, bool B_MN, int EPI, int NS_, int BPW_, int CL>
static int launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                      const CUtensorMap& md2, const void* bias, const void* X, int ldx, int M,
                      int N, const Sched& sc, float* part, uint32_t* flag, const Aux& aux,
                      cudaStream_t s) {
  auto kern = gemm_sk_kernel<A_MN, B_MN, EPI, NS_, EW_, BPW_, CL>;
  constexpr size_t SMEM = smem_bytes(NS_, EW_, BPW_);
  static_assert(SMEM <= 232448, "stream-K GEMM shared memory");
  static bool attr = false;
  if (!attr) {
    ZI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM),
            "cudaFuncSetAttribute(smem)");
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * sc.P);
  cfg.blockDim = dim3(64 + 32 * EW_);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = zi::pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (CL == 4) {   // clusters of 4 where a GPC has room, pairs elsewhere
    at[2].id = cudaLaunchAttributePreferredClusterDimension;
    at[2].val.preferredClusterDim.x = 4;
    at[2].val.preferredClusterDim.y = 1;
    at[2].val.preferredClusterDim.z = 1;
    cfg.numAttrs = 3;
  }
  zi::count_launches();
  ZI_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, md, md2, static_cast<const __nv_bfloat16*>(bias),
                             static_cast<const uint16_t*>(X), ldx, M, N, sc, part, flag, aux),
          "cudaLaunchKernelEx(zi_gemm_sk)");
  return launch_status("zi_gemm_sk");
}

// Ring depth / staging boxes: ZI_SK_CFG = 6 (6 stages, 1 box per warp; default) or 4
// (4 stages, 2 boxes).
template <bool A_MN, bool B_MN, int EPI, int CL>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                  const CUtensorMap& md2, const void* bias, const void* X, int ldx, int M, int N,
                  const Sched& sc, float* part, uint32_t* flag, const Aux& aux, cudaStream_t s) {
  if (sk_cfg() == 4)
    return launch_cfg<A_MN, B_MN, EPI, 4, 2, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
  return launch_cfg<A_MN, B_MN, EPI, 6, 1, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
}

template <bool A_MN, bool B_MN, int CL>
static int dispatch(int epi, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                    const CUtensorMap& md2, const void* bias, const void* X, int ldx, int M, int N,
                    const Sched& sc, float* part, uint32_t* flag, const Aux& aux, cudaStream_t s) {
  switch (epi) {
    case EPI_PLAIN: return launch<A_MN, B_MN, EPI_PLAIN, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_GELU: return launch<A_MN, B_MN, EPI_GELU, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_RESID: return launch<A_MN, B_MN, EPI_RESID, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_DGELU: return launch<A_MN, B_MN, EPI_DGELU, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_GELU_SAVE: return launch<A_MN, B_MN, EPI_GELU_SAVE, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_MUL: return launch<A_MN, B_MN, EPI_MUL, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
    case EPI_F32: return launch<A_MN, B_MN, EPI_F32, CL>(ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
  }
  set_error("zi_gemm_sk: unknown epilogue %d", epi);
  return ZI_EINVAL;
}

template <int CL>
static int dispatch_major(int a_mn, int b_mn, int epi, const CUtensorMap& ma, const CUtensorMap& mb,
                          const CUtensorMap& md, const CUtensorMap& md2, const void* bias,
                          const void* X, int ldx, int M, int N, const Sched& sc, float* part,
                          uint32_t* flag, const Aux& aux, cudaStream_t s) {
  if (a_mn) return dispatch<true, true, CL>(epi, ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
  if (b_mn) return dispatch<false, true, CL>(epi, ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
  return dispatch<false, false, CL>(epi, ma, mb, md, md2, bias, X, ldx, M, N, sc, part, flag, aux, s);
}

}  // namespace gsk
}  // namespace zi

extern "C" size_t zi_gemm_sk_workspace_bytes(void) {
  return (size_t)zi::gsk::FLAG_BYTES +
         (size_t)zi::gsk::sm_count() * zi::gsk::SLOT_FLOATS * sizeof(float);
}

extern "C" int zi_gemm_sk_aux(const void* A, int a_mn_major, int lda, const void* B,
                              int b_mn_major, int ldb, const void* bias, void* D, int ldd,
                              int d_f32, const void* X, int ldx, void* D2, int ldd2, int epi,
                              int M, int N, int K, void* ws, size_t ws_bytes, float* colsum_part,
                              float* delta, int delta_S, int delta_H, int delta_D, void* stream) {
  using namespace zi::gsk;
  ZI_CHECK_ARG(!(colsum_part || delta) || !d_f32, "zi_gemm_sk_aux: side outputs need bf16 output");
  ZI_CHECK_ARG(!colsum_part || zi::aligned(colsum_part, 8), "zi_gemm_sk_aux: colsum_part 8-byte aligned");
  ZI_CHECK_ARG(!delta || (epi == ZI_EPI_PLAIN && X && (delta_D == 64 || delta_D == 128) &&
                          delta_S > 0 && delta_H > 0 && N == delta_H * delta_D &&
                          M % delta_S == 0),
               "zi_gemm_sk_aux: delta needs the plain epilogue, X = O, D in {64, 128}, "
               "N = H * D and M = B * S");
  ZI_CHECK_ARG(A && B && D, "zi_gemm_sk: NULL operand");
  ZI_CHECK_ARG(M > 0 && N > 0 && K > 0, "zi_gemm_sk: empty shape");
  ZI_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0, "zi_gemm_sk: lda / ldb must be multiples of 8");
  ZI_CHECK_ARG(lda >= (a_mn_major ? M : K) && ldb >= (b_mn_major ? N : K) && ldd >= N,
               "zi_gemm_sk: leading dimension smaller than the row length");
  ZI_CHECK_ARG(zi::aligned(A, 16) && zi::aligned(B, 16) && zi::aligned(D, 16) &&
               (!bias || zi::aligned(bias, 16)), "zi_gemm_sk: 16-byte aligned buffers");
  ZI_CHECK_ARG(!(a_mn_major && !b_mn_major), "zi_gemm_sk: MN-major A needs MN-major B");
  ZI_CHECK_ARG(epi >= ZI_EPI_PLAIN && epi <= ZI_EPI_MUL, "zi_gemm_sk: unknown epilogue %d", epi);
  if (d_f32) {
    ZI_CHECK_ARG(epi == ZI_EPI_PLAIN && !bias, "zi_gemm_sk: fp32 output takes no epilogue");
    ZI_CHECK_ARG(ldd % 4 == 0 && N % 4 == 0, "zi_gemm_sk: fp32 output needs N, ldd % 4 == 0");
  } else {
    ZI_CHECK_ARG(ldd % 8 == 0 && N % 8 == 0, "zi_gemm_sk: bf16 output needs N, ldd % 8 == 0");
  }
  ZI_CHECK_ARG((epi != ZI_EPI_GELU && epi != ZI_EPI_GELU_SAVE) ||
               (D2 && ldd2 % 8 == 0 && ldd2 >= N && zi::aligned(D2, 16)),
               "zi_gemm_sk: GELU epilogue needs D2");
  ZI_CHECK_ARG((epi != ZI_EPI_RESID && epi != ZI_EPI_DGELU && epi != ZI_EPI_MUL && !delta) ||
               (X && ldx % 8 == 0 && ldx >= N && zi::aligned(X, 16)),
               "zi_gemm_sk: epilogue needs X");
  ZI_CHECK_ARG(!ws || ws_bytes >= zi_gemm_sk_workspace_bytes(),
               "zi_gemm_sk: workspace smaller than zi_gemm_sk_workspace_bytes()");
  ZI_CHECK_ARG(!ws || zi::aligned(ws, 256), "zi_gemm_sk: workspace must be 256-byte aligned");
  int st = get_encoder();
  if (st != ZI_OK) return st;
  static int env_split = -2, env_cl = -2;
  if (env_split == -2) {
    const char* e = getenv("ZI_GEMM_SPLIT");
    env_split = !e ? -1 : atoi(e);
    const char* c = getenv("ZI_SK_CL");
    env_cl = !c ? 4 : atoi(c);
  }
  // Default: preferred clusters of 4 (two pairs sharing A by multicast, 25 % less L2 -> SM
  // traffic) over regular pairs, so the SMs a GPC cannot group in fours still run pairs.
  // Under the 1 kW cap the step runs ~1.5 % faster than with plain pairs (fewer bytes
  // moved per flop: same clocks, more work; profiles/r2_gemm_cluster4.md). ZI_SK_CL=2:
  // pairs only (A/B).
  const int CL = (env_cl == 4 && M > 128) ? 4 : 2;
  CUtensorMap ma, mb, md, md2;
  if ((st = make_operand_map(&ma, A, M, K, lda, a_mn_major != 0, CL == 4 ? 64 : 128)) != ZI_OK)
    return st;
  if ((st = make_operand_map(&mb, B, N, K, ldb, b_mn_major != 0, 128)) != ZI_OK) return st;
  if ((st = make_out_map(&md, D, M, N, ldd, d_f32 != 0)) != ZI_OK) return st;
  if ((st = make_out_map(&md2, D2 ? D2 : D, M, N, D2 ? ldd2 : ldd, d_f32 != 0)) != ZI_OK) return st;
  const int clusters = CL == 4 ? resident_clusters<4>() : resident_clusters<2>();
  if (clusters <= 0) {
    zi::set_error("zi_gemm_sk: no resident cluster of %d CTAs", CL);
    return ZI_ECUDA;
  }
  const Sched sc = make_sched(M, N, K, clusters, CL, ws != nullptr && env_split != 0);
  uint32_t* flag = static_cast<uint32_t*>(ws);
  float* part = ws ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + FLAG_BYTES) : nullptr;
  const int e = d_f32 ? EPI_F32 : epi;
  cudaStream_t s = (cudaStream_t)stream;
  const Aux aux = {colsum_part, delta, delta_S, delta_H, delta_D};
  if (CL == 4)
    return dispatch_major<4>(a_mn_major, b_mn_major, e, ma, mb, md, md2, bias, X, ldx, M, N, sc,
                             part, flag, aux, s);
  return dispatch_major<2>(a_mn_major, b_mn_major, e, ma, mb, md, md2, bias, X, ldx, M, N, sc,
                           part, flag, aux, s);
}

extern "C" int zi_gemm_sk(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major,
                          int ldb, const void* bias, void* D, int ldd, int d_f32, const void* X,
                          int ldx, void* D2, int ldd2, int epi, int M, int N, int K, void* ws,
                          size_t ws_bytes, void* stream) {
  return zi_gemm_sk_aux(A, a_mn_major, lda, B, b_mn_major, ldb, bias, D, ldd, d_f32, X, ldx, D2,
                        ldd2, epi, M, N, K, ws, ws_bytes, nullptr, nullptr, 0, 0, 0, stream);
}
