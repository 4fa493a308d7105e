// Tiled-linear GEMMs on the 5th-gen tensor cores (PAPER §5.1.3).
//
//   D[m, n] = sum_k A(m, k) * B(n, k)  (+ bias[n])  (+ D if accumulating)
//
// A(m, k) is K-major (A[m*lda + k]) or M-major (A[k*lda + m]); B likewise
// (B[n*ldb + k] or B[k*ldb + n]). That covers a linear's forward
// y = x W^T + b (both K-major), its input gradient dx = dy W (B N-major) and
// its weight gradient dW = dy^T x (both MN-major). bf16 operands, fp32
// accumulation in TMEM, bf16 or fp32 output. Blackwell-native structure:
//   * persistent CTAs (one per SM), tiles 128 x 256 visited in GROUP_M-row
//     groups so the tiles in flight share A / B blocks in L2;
//   * warp 0: TMA producer. cp.async.bulk.tensor.2d fills a 4-stage ring of
//     128-byte-swizzled A / B tiles (K-major: box 64(k) x rows; MN-major:
//     boxes of 64(mn) x 64(k)), completion via mbarrier expect_tx;
//   * warp 1: TMEM allocator + the single MMA-issuing thread:
//     tcgen05.mma.cta_group::1.kind::f16 M=128 N=256 K=16 from smem
//     descriptors into one of two 256-column TMEM accumulators;
//     tcgen05.commit frees ring slots and publishes finished accumulators;
//   * warps 2..5: epilogue. tcgen05.ld.32x32b drains the accumulator (rows =
//     TMEM lanes), adds bias / the existing output, stores, and hands the
//     accumulator back, so the epilogue of tile i overlaps the mainloop of i+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

#include "common.cuh"

namespace zi {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;           // 16 KiB
constexpr int B_BYTES = BN * BK * 2;           // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int MN_BOX_BYTES = 64 * BK * 2;      // one 64(mn) x 64(k) MN-major box: 8 KiB
constexpr int TMEM_COLS = 512;                 // two 256-column fp32 accumulators
constexpr int THREADS = 192;
constexpr int GROUP_M = 16;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait for the phase with the given parity to complete; traps after ~10 s
// so a protocol bug fails loudly instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  long long t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (done) return;
    if (t0 == 0) t0 = clock64();
    else if (clock64() - t0 > 20000000000LL) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1)
      : "memory");
}

// Same load, written to the same smem offset in every CTA of `mask` and
// completing bytes on each destination CTA's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

// Shared-memory matrix descriptor (tcgen05), SWIZZLE_128B, version 1.
//  K-major : rows of 128 B (64 k), 8-row atoms -> SBO = 1024 B, LBO unused (16 B).
//  MN-major: 128 B lines of 64 mn per k-row, 8 k-rows per atom -> SBO = 1024 B
//            between k-groups, LBO = BK*128 B between 64-wide mn boxes.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16; bit 15/16 = A/B MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}

// Commit arriving on the barrier at the same offset in every CTA of `mask`
// (1-SM MMA + multicast TMA: a ring slot is free once every CTA consumed it).
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// two fp32 -> one bf16x2 word (a low, b high), RNE, a single cvt instruction
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mt, int& nt) {
  const int per_group = GROUP_M * tiles_n;
  const int g = t / per_group;
  const int first = g * GROUP_M;
  const int gm = min(tiles_m - first, GROUP_M);
  const int r = t % per_group;
  mt = first + r % gm;
  nt = r / gm;
}

// One operand tile (rows = BM or BN, 64 k) into smem at dst.
template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                             int k0, int r0) {
  if (!MN) {
    tma_load_2d(dst, map, bar, k0, r0);               // box {64 k, ROWS}
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)               // boxes {64 mn, 64 k}
      tma_load_2d(dst + j * MN_BOX_BYTES, map, bar, r0 + 64 * j, k0);
  }
}

// Epilogue for 32 accumulator columns of one row: + bias, (+ existing D), store.
template <bool OUT_F32, bool ACCUM>
__device__ __forceinline__ void store_chunk(const uint32_t* r, int row, int col0, int M, int N,
                                            const __nv_bfloat16* __restrict__ bias,
                                            void* __restrict__ Dout, int ldd, bool vec_ok) {
  if (row >= M || col0 >= N) return;
  constexpr int OB = OUT_F32 ? 4 : 2;
  float f[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int col = col0 + j;
    const float b = (bias != nullptr && col < N) ? __bfloat162float(bias[col]) : 0.f;
    f[j] = __uint_as_float(r[j]) + b;
  }
  uint8_t* dst = static_cast<uint8_t*>(Dout) + ((size_t)row * ldd + col0) * OB;
  const bool full_vec = vec_ok && col0 + 32 <= N;
  if (OUT_F32) {
    float* o = reinterpret_cast<float*>(dst);
    if (full_vec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 v = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
        if (ACCUM) {
          const float4 o4 = reinterpret_cast<const float4*>(o)[j];
          v.x += o4.x; v.y += o4.y; v.z += o4.z; v.w += o4.w;
        }
        reinterpret_cast<float4*>(o)[j] = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) o[j] = ACCUM ? o[j] + f[j] : f[j];
    }
  } else {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(dst);
    if (ACCUM) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) f[j] += __bfloat162float(o[j]);
    }
    if (full_vec) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 v;
        v.x = pack_bf16(f[8 * j + 0], f[8 * j + 1]);
        v.y = pack_bf16(f[8 * j + 2], f[8 * j + 3]);
        v.z = pack_bf16(f[8 * j + 4], f[8 * j + 5]);
        v.w = pack_bf16(f[8 * j + 6], f[8 * j + 7]);
        reinterpret_cast<uint4*>(o)[j] = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) o[j] = __float2bfloat16_rn(f[j]);
    }
  }
}

// Rows [r0, r0 + ROWS) of an operand, multicast to the whole cluster pair.
template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand_mc(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                                int k0, int r0, uint16_t mask) {
  if (!MN) {
    tma_load_2d_mc(dst, map, bar, k0, r0, mask);
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)
      tma_load_2d_mc(dst + j * MN_BOX_BYTES, map, bar, r0 + 64 * j, k0, mask);
  }
}

// CL = CTAs per cluster along M (1 or 2). With CL = 2 the pair computes a
// 256 x 256 output block: each CTA its own 128 rows of A, while the shared
// 256-row B tile is loaded half by each CTA and multicast to both — 32 KiB
// instead of 48 KiB of L2->SM traffic per CTA per k-block.
template <bool A_MN, bool B_MN, bool OUT_F32, bool ACCUM, int CL>
__global__ void __launch_bounds__(THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __nv_bfloat16* __restrict__ bias, void* __restrict__ Dout, int M, int N, int K,
            int ldd) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;      // [2] accumulator ready
  uint64_t* tmem_empty = tmem_full + 2;      // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;
  const int tiles_m = (M + BM * CL - 1) / (BM * CL), tiles_n = (N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;          // cluster tiles
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  constexpr uint16_t MASK = (1u << CL) - 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // every CTA of the cluster must release the slot
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CL > 1) cluster_sync();   // peers' barriers exist before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;  // global k-block counter across tiles (ring position)
      for (int t = cid; t < ntiles; t += ncl) {
        int mt, nt;
        tile_coords(t, tiles_m, tiles_n, mt, nt);
        const int m0 = (mt * CL + (int)crank) * BM;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], STAGE_BYTES);
          load_operand<A_MN, BM>(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
          if (CL == 1) {
            load_operand<B_MN, BN>(sB + s * B_BYTES, &tmB, &full[s], kb * BK, nt * BN);
          } else {
            constexpr int HB = BN / CL;
            load_operand_mc<B_MN, HB>(sB + s * B_BYTES + crank * (B_BYTES / CL), &tmB, &full[s],
                                      kb * BK, nt * BN + (int)crank * HB, MASK);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
      // per 16-deep k step: K-major advances 32 B inside the swizzle atom,
      // MN-major advances two 8-row k-groups (2 KiB)
      constexpr uint32_t kstep = 32;
      constexpr uint32_t kstep_mn = 2 * 1024;
      uint32_t it = 0, tcount = 0;
      for (int t = cid; t < ntiles; t += ncl, ++tcount) {
        const uint32_t acc = tcount & 1;
        mbar_wait(&tmem_empty[acc], ((tcount >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = A_MN ? sdesc_sw128(a0 + k * kstep_mn, MN_BOX_BYTES)
                                     : sdesc_sw128(a0 + k * kstep, 16);
            const uint64_t db = B_MN ? sdesc_sw128(b0 + k * kstep_mn, MN_BOX_BYTES)
                                     : sdesc_sw128(b0 + k * kstep, 16);
            umma_bf16(d, da, db, idesc, (kb | k) != 0);
          }
          if (CL == 1) umma_commit(&empty[s]);
          else umma_commit_mc(&empty[s], MASK);
        }
        umma_commit(&tmem_full[acc]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w owns TMEM lanes 32*(w%4) .. +31 (= tile rows)
    const int q = warp & 3;
    const bool vec_ok = (ldd % 8) == 0 && ((reinterpret_cast<uintptr_t>(Dout) & 15) == 0);
    uint32_t tcount = 0;
    for (int t = cid; t < ntiles; t += ncl, ++tcount) {
      int mt, nt;
      tile_coords(t, tiles_m, tiles_n, mt, nt);
      const uint32_t acc = tcount & 1;
      mbar_wait(&tmem_full[acc], (tcount >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = (mt * CL + (int)crank) * BM + q * 32 + lane;
      const int n0 = nt * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * BN + ((uint32_t)(q * 32) << 16) + c, r);
        store_chunk<OUT_F32, ACCUM>(r, row, n0 + c, M, N, bias, Dout, ldd, vec_ok);
      }
      // accumulator drained: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CL > 1) cluster_sync();   // no CTA leaves while its peer may still multicast into it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS) : "memory");
  }
}

// ------------------------------------------------------------ 2-SM variant
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 output block with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A
// and its own half (128 rows) of B — 32 KiB per k-block per CTA instead of
// 48 KiB, so six ring stages fit — and the leader CTA's single thread issues
// the MMA over both CTAs' shared memory. Each CTA's TMEM holds the fp32
// accumulators of its 128 rows; each CTA runs its own epilogue.
//   full[s]   leader only: both CTAs' TMA bytes land here (peer bit cleared)
//   empty[s]  both CTAs: the leader's commit multicasts the release
//   tmem_full both CTAs (multicast commit); tmem_empty leader only: 8 arrivals
//             (4 epilogue warps x 2 CTAs, the peer's remote)
namespace g2 {
constexpr int STAGES2 = 6;
constexpr int A2_BYTES = 128 * BK * 2;        // this CTA's 128 rows of A
constexpr int B2_BYTES = 128 * BK * 2;        // this CTA's half of the 256-row B tile
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr size_t SMEM2_BYTES = (size_t)STAGES2 * STAGE2_BYTES + 1024 + 256;
}  // namespace g2

__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map,
                                                uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

template <bool MN>
__device__ __forceinline__ void load_operand_2sm(uint8_t* dst, const CUtensorMap* map,
                                                 uint32_t leader_bar, int k0, int r0) {
  if (!MN) {
    tma_load_2d_2sm(dst, map, leader_bar, k0, r0);       // box {64 k, 128 rows}
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j)                           // boxes {64 mn, 64 k}
      tma_load_2d_2sm(dst + j * MN_BOX_BYTES, map, leader_bar, r0 + 64 * j, k0);
  }
}

__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t a, uint64_t b,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}

template <bool A_MN, bool B_MN, bool OUT_F32, bool ACCUM>
__global__ void __launch_bounds__(THREADS, 1)
gemm2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __nv_bfloat16* __restrict__ bias, void* __restrict__ Dout, int M, int N,
               int K, int ldd) {
  using namespace g2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A2_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES2 * B2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tmem_full = empty + STAGES2;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int nk = (K + BK - 1) / BK;
  const int tiles_m = (M + 255) / 256, tiles_n = (N + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {  // same warp id in both CTAs: a paired 2-SM allocation
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        int mt, nt;
        tile_coords(t, tiles_m, tiles_n, mt, nt);
        const int m0 = mt * 256 + (int)crank * 128;
        const int nb = nt * BN + (int)crank * 128;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES2;
          const uint32_t ph = (it / STAGES2) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t lbar = map_to_rank(smem_u32(&full[s]), 0);
          if (leader) mbar_expect_tx(&full[s], 2 * STAGE2_BYTES);
          load_operand_2sm<A_MN>(sA + s * A2_BYTES, &tmA, lbar, kb * BK, m0);
          load_operand_2sm<B_MN>(sB + s * B2_BYTES, &tmB, lbar, kb * BK, nb);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN, A_MN, B_MN);
      constexpr uint32_t kstep = 32, kstep_mn = 2 * 1024;
      uint32_t it = 0, tcount = 0;
      for (int t = cid; t < ntiles; t += ncl, ++tcount) {
        const uint32_t acc = tcount & 1;
        mbar_wait(&tmem_empty[acc], ((tcount >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES2;
          const uint32_t ph = (it / STAGES2) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + s * A2_BYTES), b0 = smem_u32(sB + s * B2_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = A_MN ? sdesc_sw128(a0 + k * kstep_mn, MN_BOX_BYTES)
                                     : sdesc_sw128(a0 + k * kstep, 16);
            const uint64_t db = B_MN ? sdesc_sw128(b0 + k * kstep_mn, MN_BOX_BYTES)
                                     : sdesc_sw128(b0 + k * kstep, 16);
            umma_bf16_2sm(d, da, db, idesc, (kb | k) != 0);
          }
          umma_commit_2sm(&empty[s]);
        }
        umma_commit_2sm(&tmem_full[acc]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const bool vec_ok = (ldd % 8) == 0 && ((reinterpret_cast<uintptr_t>(Dout) & 15) == 0);
    uint32_t tcount = 0;
    for (int t = cid; t < ntiles; t += ncl, ++tcount) {
      int mt, nt;
      tile_coords(t, tiles_m, tiles_n, mt, nt);
      const uint32_t acc = tcount & 1;
      mbar_wait(&tmem_full[acc], (tcount >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = mt * 256 + (int)crank * 128 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + acc * BN + ((uint32_t)(q * 32) << 16) + c, r);
        store_chunk<OUT_F32, ACCUM>(r, row, nt * BN + c, M, N, bias, Dout, ldd, vec_ok);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const uint32_t rb = map_to_rank(smem_u32(&tmem_empty[acc]), 0);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb)
                     : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS) : "memory");
  }
}

// ------------------------------------------------------- 2-SM wide variant (256 x 512)
// The 256 x 256 pair tile moves 32 KiB into each SM per 512 MMA cycles; on
// B200 that operand ingress, not the tensor pipe, bounds it (~64 % tensor
// active measured). A 256 x 512 pair tile issues two M=256 N=256 MMAs per
// k-step that share the A tile: 48 KiB per 1024 MMA cycles. The 512 fp32
// accumulator columns fill TMEM, so there is one accumulator: the epilogue of
// tile i runs while the producer already streams tile i+1 into the 4-stage
// ring, and the MMA restarts as soon as the accumulator is drained.
// Epilogues (bf16 out, bias optional):
//   EPI_PLAIN  D = acc + bias
//   EPI_GELU   D = u = bf16(acc + bias), D2 = bf16(gelu_tanh(u))     (fc1 forward)
//   EPI_RESID  D = bf16(bf16(acc + bias) + X)                          (fc2 forward + residual)
//   EPI_DGELU  D = bf16(bf16(acc) * gelu_tanh'(X))                     (fc2 dX -> fc1 du)
constexpr int EPI_PLAIN = ZI_EPI_PLAIN, EPI_GELU = ZI_EPI_GELU, EPI_RESID = ZI_EPI_RESID,
              EPI_DGELU = ZI_EPI_DGELU;
namespace g3 {
constexpr int BN3 = 512;
constexpr int A3_BYTES = 128 * BK * 2;        // this CTA's 128 rows of A
constexpr int B3_BYTES = 256 * BK * 2;        // this CTA's 256 of the pair tile's 512 B rows
constexpr int STAGE3_BYTES = A3_BYTES + B3_BYTES;
constexpr int OUT_BOX_BYTES = 32 * 64 * 2;    // one warp's 32 rows x 64 columns, bf16, SW128
// NS ring stages, EW epilogue warps, BPW staging boxes per epilogue warp
constexpr size_t smem3(int NS, int EW, int BPW) {
  return (size_t)NS * STAGE3_BYTES + (size_t)EW * BPW * OUT_BOX_BYTES + 1024 + 256;
}
constexpr int threads3(int EW) { return 64 + 32 * EW; }
}  // namespace g3

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float bf16f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// async-proxy (TMA) stores from shared memory
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 accumulator columns of one row through the fused epilogue, packed to 16
// bf16x2 words (w: D, g: the GELU output). Columns past N compute garbage that
// the TMA store clips; X is only read inside the matrix.
template <int EPI>
__device__ __forceinline__ void epi_words(const uint32_t* r, int row, int col0, int M, int N,
                                          const __nv_bfloat16* __restrict__ bias,
                                          const uint16_t* __restrict__ X, int ldx, uint32_t* w) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = col0 + 8 * q;
    const bool in = c < N;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[8 * q + j]);
    if (bias != nullptr && in) {
      const uint4 bv = *reinterpret_cast<const uint4*>(bias + c);
      const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        f[2 * j] += bf16f(bw[j] & 0xFFFF);
        f[2 * j + 1] += bf16f(bw[j] >> 16);
      }
    }
    if (EPI == EPI_RESID || EPI == EPI_DGELU) {
      uint4 xv = make_uint4(0, 0, 0, 0);
      if (in && row < M) xv = *reinterpret_cast<const uint4*>(X + (size_t)row * ldx + c);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x0 = bf16f(xw[j] & 0xFFFF), x1 = bf16f(xw[j] >> 16);
        if (EPI == EPI_RESID) {
          f[2 * j] = rbf(f[2 * j]) + x0;
          f[2 * j + 1] = rbf(f[2 * j + 1]) + x1;
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

// bf16x2 words u -> gelu_tanh(u), in place
__device__ __forceinline__ void gelu_words(uint32_t* w, int n) {
#pragma unroll
  for (int j = 0; j < n; ++j)
    w[j] = pack_bf16(gelu_tanh(bf16f(w[j] & 0xFFFF)), gelu_tanh(bf16f(w[j] >> 16)));
}

// One warp's 32 rows x 64 columns (w0: columns 0-31, w1: 32-63; lane = row) into a
// SW128 staging box: 16-byte chunk j of row r lives at chunk j ^ (r % 8).
__device__ __forceinline__ void stage_box(uint8_t* box, int lane, const uint32_t* w0,
                                          const uint32_t* w1) {
  const uint32_t base = smem_u32(box) + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t* w = j < 4 ? w0 + 4 * j : w1 + 4 * (j - 4);
    const uint32_t a = base + ((uint32_t)(j ^ (lane & 7)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3]) : "memory");
  }
}

// B rows [r0, r0 + ROWS) of a k-block for the 2-SM MMA (K-major: one box of ROWS
// rows; MN-major: ROWS / 64 boxes of 64 mn x 64 k).
template <bool MN, int ROWS>
__device__ __forceinline__ void load_rows_2sm(uint8_t* dst, const CUtensorMap* map,
                                              uint32_t leader_bar, int k0, int r0) {
  if (!MN) {
    tma_load_2d_2sm(dst, map, leader_bar, k0, r0);
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)
      tma_load_2d_2sm(dst + j * MN_BOX_BYTES, map, leader_bar, r0 + 64 * j, k0);
  }
}

// NP accumulator parts: the pair tile's 512 columns are computed by NP MMAs of
// N = 512 / NP per k-step (each CTA stages 256 / NP B rows per part), and the
// epilogue releases TMEM part by part, so the next tile's MMAs restart after
// only one part (128 columns at NP = 4) has been drained.
template <bool A_MN, bool B_MN, int EPI, int STAGES3, int EW, int BPW, int NP>
__global__ void __launch_bounds__(g3::threads3(EW), 1)
gemm2sm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmD2,
                    const __nv_bfloat16* __restrict__ bias, const uint16_t* __restrict__ X, int ldx,
                    int M, int N, int K, unsigned long long* __restrict__ prof) {
  using namespace g3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES3 * A3_BYTES;
  uint8_t* sOut = sB + STAGES3 * B3_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + EW * BPW * OUT_BOX_BYTES);
  uint64_t* empty = full + STAGES3;
  uint64_t* tmem_full = empty + STAGES3;
  uint64_t* tmem_empty = tmem_full + 1;                // [NP]: accumulator parts drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + NP);
  constexpr int PN = BN3 / NP;                 // output columns per part
  constexpr int PR = PN / 2;                   // B rows per part staged by each CTA
  constexpr int PART_BYTES = PR * BK * 2;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int nk = (K + BK - 1) / BK;
  const int tiles_m = (M + 255) / 256, tiles_n = (N + BN3 - 1) / BN3;
  const int ntiles = tiles_m * tiles_n;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES3; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    for (int p = 0; p < NP; ++p) mbar_init(&tmem_empty[p], 2 * EW);   // all epilogue warps, both CTAs
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        int mt, nt;
        tile_coords(t, tiles_m, tiles_n, mt, nt);
        const int m0 = mt * 256 + (int)crank * 128;
        const int nb = nt * BN3 + (int)crank * PR;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES3;
          const uint32_t ph = (it / STAGES3) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t lbar = map_to_rank(smem_u32(&full[s]), 0);
          if (leader) mbar_expect_tx(&full[s], 2 * STAGE3_BYTES);
          load_operand_2sm<A_MN>(sA + s * A3_BYTES, &tmA, lbar, kb * BK, m0);
#pragma unroll
          for (int p = 0; p < NP; ++p)
            load_rows_2sm<B_MN, PR>(sB + s * B3_BYTES + p * PART_BYTES, &tmB, lbar, kb * BK,
                                    nb + p * PN);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, PN, A_MN, B_MN);
      constexpr uint32_t kstep = 32, kstep_mn = 2 * 1024;
      // MMA of one stage into accumulator part p (columns p*PN .. +PN)
      auto mma_part = [&](int s, int p, bool first) {
        const uint32_t a0 = smem_u32(sA + s * A3_BYTES);
        const uint32_t b0 = smem_u32(sB + s * B3_BYTES + p * PART_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t da = A_MN ? sdesc_sw128(a0 + k * kstep_mn, MN_BOX_BYTES)
                                   : sdesc_sw128(a0 + k * kstep, 16);
          const uint64_t db = B_MN ? sdesc_sw128(b0 + k * kstep_mn, MN_BOX_BYTES)
                                   : sdesc_sw128(b0 + k * kstep, 16);
          umma_bf16_2sm(tmem + p * PN, da, db, idesc, (!first || k != 0) ? 1u : 0u);
        }
      };
      uint32_t it = 0, tcount = 0;
      for (int t = cid; t < ntiles; t += ncl, ++tcount) {
        // The epilogue drains the accumulator part by part. The first E k-blocks
        // (already in the ring) run on each part as soon as it is drained; their
        // ring slots are released after the last part consumed them.
        const int E = nk < STAGES3 ? nk : STAGES3;
#pragma unroll 1
        for (int p = 0; p < NP; ++p) {
          if (prof && tcount < 15 && p < 2) prof[(blockIdx.x * 16 + tcount) * 8 + 2 * p] = clock64();
          mbar_wait(&tmem_empty[p], (tcount & 1) ^ 1);
          if (prof && tcount < 15 && p < 2) prof[(blockIdx.x * 16 + tcount) * 8 + 2 * p + 1] = clock64();
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int kb = 0; kb < E; ++kb) {
            const int s = (it + kb) % STAGES3;
            if (p == 0) {
              mbar_wait(&full[s], ((it + kb) / STAGES3) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            mma_part(s, p, kb == 0);
            if (p == NP - 1) umma_commit_2sm(&empty[s]);
          }
        }
        it += E;
        for (int kb = E; kb < nk; ++kb, ++it) {
          const int s = it % STAGES3;
          mbar_wait(&full[s], (it / STAGES3) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int p = 0; p < NP; ++p) mma_part(s, p, false);
          umma_commit_2sm(&empty[s]);
        }
        umma_commit_2sm(tmem_full);
        if (prof && tcount < 15) prof[(blockIdx.x * 16 + tcount) * 8 + 4] = clock64();
      }
    }
    __syncwarp();
  } else {
    // Epilogue: TMEM -> registers (bias / GELU / residual) -> SW128 staging box in
    // shared memory -> TMA store. Each warp owns 32 rows and BPW staging boxes
    // used round-robin; a box is rewritten only once its previous store has
    // finished reading it (at most BPW - 1 stores pending). TMEM is released as
    // soon as a half is staged, so with BPW = 8 the stores of a tile drain
    // during the next tile's mainloop instead of stalling the MMA.
    // Warps 2 .. 2+EW-1: quadrant q = warp % 4 (TMEM lanes 32q .. 32q+31, the
    // only lanes a warp may read), sub = which share of each half's columns.
    const int q = warp & 3, sub = (warp - 2) >> 2;
    constexpr int JPW = (PN / 64) / (EW / 4);   // 64-column chunks per warp per part
    static_assert(JPW >= 1, "too many epilogue warps for the part width");
    uint8_t* wbox = sOut + (warp - 2) * BPW * OUT_BOX_BYTES;
    uint32_t bsel = 0, tcount = 0;
    auto emit = [&](const CUtensorMap* map, const uint32_t* w0, const uint32_t* w1, int c0, int r0) {
      uint8_t* box = wbox + bsel * OUT_BOX_BYTES;
      bsel = bsel + 1 == BPW ? 0 : bsel + 1;
      if (lane == 0) bulk_wait_read<BPW - 1>();
      __syncwarp();
      stage_box(box, lane, w0, w1);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map, box, c0, r0);
        bulk_commit();
      }
    };
    for (int t = cid; t < ntiles; t += ncl, ++tcount) {
      int mt, nt;
      tile_coords(t, tiles_m, tiles_n, mt, nt);
      mbar_wait(tmem_full, tcount & 1);
      if (prof && warp == 4 && lane == 0 && tcount < 15) prof[(blockIdx.x * 16 + tcount) * 8 + 5] = clock64();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int r0 = mt * 256 + (int)crank * 128 + q * 32;
      const int row = r0 + lane;
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16);
      const int cols = min(BN3, N - nt * BN3);
      // Per part: this warp's JPW x 64 columns TMEM -> registers -> epilogue math ->
      // packed bf16 words, one 64-column chunk at a time; the part is handed back to
      // the MMA warp before its (slower) staging + TMA stores. Holding the whole
      // tile in registers instead would need > 168 registers per thread, the most
      // 3 warps per scheduler can have.
      const bool live = r0 < M;
#pragma unroll 1
      for (int h = 0; h < NP; ++h) {
        uint32_t w[JPW][32];
#pragma unroll
        for (int j = 0; j < JPW; ++j) {
          const int c = h * PN + 64 * (sub * JPW + j);
          if (live && c < cols) {
            uint32_t v[64];
            tmem_ld32_nowait(base + c, v);
            tmem_ld32_nowait(base + c + 32, v + 32);
            tmem_wait_ld();
            const int col = nt * BN3 + c;
            epi_words<EPI>(v, row, col, M, N, bias, X, ldx, w[j]);
            epi_words<EPI>(v + 32, row, col + 32, M, N, bias, X, ldx, w[j] + 16);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (prof && warp == 4 && lane == 0 && tcount < 15 && h < 2) prof[(blockIdx.x * 16 + tcount) * 8 + 6 + h] = clock64();
        if (lane == 0) {
          const uint32_t rbar = map_to_rank(smem_u32(&tmem_empty[h]), 0);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar)
                       : "memory");
        }
#pragma unroll
        for (int j = 0; j < JPW; ++j) {
          const int c = h * PN + 64 * (sub * JPW + j);
          if (live && c < cols) {
            const int col = nt * BN3 + c;
            emit(&tmD, w[j], w[j] + 16, col, r0);
            if (EPI == EPI_GELU) {
              gelu_words(w[j], 32);
              emit(&tmD2, w[j], w[j] + 16, col, r0);
            }
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();   // every store landed before the CTA (and its smem) exits
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS) : "memory");
  }
}

// --------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
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

// Operand map. K-major: dims {K, rows}, box {64, box_rows}. MN-major (rows
// contiguous): dims {rows, K}, box {64, 64}. ld = elements between the
// starts of consecutive outer-dimension lines.
static int make_map(CUtensorMap* m, const void* base, int rows, int K, int ld, int box_rows,
                    bool mn_major) {
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (!mn_major) {
    dims[0] = (cuuint64_t)K; dims[1] = (cuuint64_t)rows;
    box[0] = BK; box[1] = (cuuint32_t)box_rows;
  } else {
    dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)K;
    box[0] = 64; box[1] = BK;
  }
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return ZI_ECUDA;
  }
  return ZI_OK;
}

// Output map for the TMA-store epilogue: bf16 rows x cols (ld elements), box of
// 64 columns x 32 rows (one epilogue warp's chunk), 128-byte swizzle.
static int make_out_map(CUtensorMap* m, void* base, int rows, int cols, int ld) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 32}, estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
    return ZI_ECUDA;
  }
  return ZI_OK;
}

// Pair CTAs along M (cluster of 2, multicast B). Measured on B200: correct but
// 1-5 % slower than unpaired (the two CTAs lock-step on every ring slot and
// smem per stage stays 48 KiB), so it is opt-in: ZI_GEMM_PAIR=1.
// Kernel choice: MODE_1SM (one CTA per 128x256 tile), MODE_PAIR (1-SM MMAs in
// a cluster of 2 sharing B by multicast), MODE_2SM (cta_group::2, 256x256 per
// CTA pair, 6 stages). ZI_GEMM_MODE=1sm|pair|2sm overrides the default.
enum { MODE_1SM = 0, MODE_PAIR = 1, MODE_2SM = 2 };
static inline int gemm_mode(int M) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("ZI_GEMM_MODE");
    env = !e ? -1 : (e[0] == 'p' ? MODE_PAIR : (e[0] == '2' ? MODE_2SM : MODE_1SM));
  }
  const int m = env >= 0 ? env : MODE_2SM;
  return (m != MODE_1SM && M <= BM) ? MODE_1SM : m;
}
static inline bool pair_m(int M) { return gemm_mode(M) != MODE_1SM; }

template <bool A_MN, bool B_MN, bool OUT_F32, bool ACCUM>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const void* bias, void* D, int M,
                  int N, int K, int ldd, cudaStream_t s) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int mode = gemm_mode(M);
  const int CL = mode == MODE_1SM ? 1 : 2;
  auto kern = mode == MODE_2SM ? gemm2sm_kernel<A_MN, B_MN, OUT_F32, ACCUM>
            : mode == MODE_PAIR ? gemm_kernel<A_MN, B_MN, OUT_F32, ACCUM, 2>
                                : gemm_kernel<A_MN, B_MN, OUT_F32, ACCUM, 1>;
  const size_t smem = mode == MODE_2SM ? g2::SMEM2_BYTES : SMEM_BYTES;
  static bool attr[3] = {false, false, false};
  if (!attr[mode]) {
    ZI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "cudaFuncSetAttribute(smem)");
    attr[mode] = true;
  }
  const int ntiles = ((M + BM * CL - 1) / (BM * CL)) * ((N + BN - 1) / BN);
  int grid = ntiles * CL < sms ? ntiles * CL : (sms / CL) * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  zi::count_launches();
  ZI_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, static_cast<const __nv_bfloat16*>(bias), D, M, N,
                             K, ldd), "cudaLaunchKernelEx(zi_gemm)");
  return launch_status("zi_gemm");
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

// 256 x 512 pair tiles or 256 x 256 ones: whole waves of pair tiles times the
// measured relative tile cost (256x512 ~2.35, 256x256 ~1.56: the wide tile is
// tensor-bound, the narrow one ingress-bound). ZI_GEMM_WIDE=0/1 forces it.
static bool use_wide(int M, int N) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("ZI_GEMM_WIDE");
    env = !e ? -1 : (e[0] == '1' ? 1 : 0);
  }
  if (env >= 0) return env == 1;
  if (M <= BM || N <= 256) return false;
  const int pairs = sm_count() / 2;
  const long tm = (M + 255) / 256;
  const long tw = tm * ((N + 511) / 512), tn = tm * ((N + 255) / 256);
  const double ew = (double)((tw + pairs - 1) / pairs) * 2.35;
  const double en = (double)((tn + pairs - 1) / pairs) * 1.56;
  return ew <= en;
}

// Diagnostics: when set (zi_gemm_set_profile), wide-tile launches record clock64()
// stamps per CTA and tile: [cta][tile<15][8] = MMA wait-half0 begin/end, wait-half1
// begin/end, tile committed; epilogue (warp q=0) accumulator seen, half 0 / 1 staged.
static unsigned long long* g_prof = nullptr;

template <bool A_MN, bool B_MN, int EPI, int NS, int EW, int BPW, int NP>
static int launch_wide_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const void* Bp, int ldb,
                           const void* bias, void* D,
                           int ldd, const void* X, int ldx, void* D2, int ldd2, int M, int N, int K,
                           cudaStream_t s) {
  auto kern = gemm2sm_wide_kernel<A_MN, B_MN, EPI, NS, EW, BPW, NP>;
  constexpr size_t SMEM3_BYTES = g3::smem3(NS, EW, BPW);
  CUtensorMap mbp;   // B box of this configuration's part rows (256 / NP per CTA)
  {
    int st0 = make_map(&mbp, Bp, N, K, ldb, 256 / NP, B_MN);
    if (st0 != ZI_OK) return st0;
  }
  static_assert(SMEM3_BYTES <= 232448, "wide GEMM shared memory");
  static bool attr = false;
  if (!attr) {
    ZI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM3_BYTES), "cudaFuncSetAttribute(smem)");
    attr = true;
  }
  CUtensorMap md, md2;
  int st;
  if ((st = make_out_map(&md, D, M, N, ldd)) != ZI_OK) return st;
  if ((st = make_out_map(&md2, D2 ? D2 : D, M, N, D2 ? ldd2 : ldd)) != ZI_OK) return st;
  const int sms = sm_count();
  const int ntiles = ((M + 255) / 256) * ((N + g3::BN3 - 1) / g3::BN3);
  const int grid = ntiles * 2 < sms ? ntiles * 2 : (sms / 2) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(g3::threads3(EW));
  cfg.dynamicSmemBytes = SMEM3_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  zi::count_launches();
  ZI_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mbp, md, md2, static_cast<const __nv_bfloat16*>(bias),
                             static_cast<const uint16_t*>(X), ldx, M, N, K, g_prof),
          "cudaLaunchKernelEx(zi_gemm wide)");
  return launch_status("zi_gemm(wide)");
}

// Staging configuration: (ring stages, boxes per warp). ZI_GEMM_STAGING=8|2 overrides.
template <bool A_MN, bool B_MN, int EPI>
static int launch_wide(const CUtensorMap& ma, const CUtensorMap& mb, const void* Bp, int ldb,
                       const void* bias, void* D,
                       int ldd, const void* X, int ldx, void* D2, int ldd2, int M, int N, int K,
                       cudaStream_t s) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("ZI_GEMM_STAGING");
    env = !e ? -1 : atoi(e);
  }
  // Measured on B200 (8192x8192x2048): halves + 8 epilogue warps + 4 stages is the
  // fastest; quarter parts (N = 128 MMAs) slow the mainloop by ~15 %.
  const int cfgno = env > 0 ? env : 2;
  if (cfgno == 3)   // quarters, 8 epilogue warps, 4 stages, 1 box each
    return launch_wide_cfg<A_MN, B_MN, EPI, 4, 8, 1, 4>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
  if (cfgno == 4)   // halves, 4 epilogue warps, 4 stages, 2 boxes each
    return launch_wide_cfg<A_MN, B_MN, EPI, 4, 4, 2, 2>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
  // halves, 8 epilogue warps, 4 stages, 1 box each
  return launch_wide_cfg<A_MN, B_MN, EPI, 4, 8, 1, 2>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
}

template <bool A_MN, bool B_MN>
static int dispatch_epi(int epi, const CUtensorMap& ma, const CUtensorMap& mb, const void* Bp,
                        int ldb, const void* bias,
                        void* D, int ldd, const void* X, int ldx, void* D2, int ldd2, int M, int N,
                        int K, cudaStream_t s) {
  switch (epi) {
    case EPI_PLAIN: return launch_wide<A_MN, B_MN, EPI_PLAIN>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
    case EPI_GELU: return launch_wide<A_MN, B_MN, EPI_GELU>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
    case EPI_RESID: return launch_wide<A_MN, B_MN, EPI_RESID>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
    case EPI_DGELU: return launch_wide<A_MN, B_MN, EPI_DGELU>(ma, mb, Bp, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
  }
  set_error("zi_gemm_ex: unknown epilogue %d", epi);
  return ZI_EINVAL;
}

}  // namespace gemm
}  // namespace zi

extern "C" int zi_gemm_set_profile(void* buf) {
  zi::gemm::g_prof = static_cast<unsigned long long*>(buf);
  return ZI_OK;
}

extern "C" int zi_gemm_ex(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major,
                          int ldb, const void* bias, void* D, int ldd, const void* X, int ldx,
                          void* D2, int ldd2, int epi, int M, int N, int K, void* stream) {
  using namespace zi::gemm;
  ZI_CHECK_ARG(A && B && D, "zi_gemm_ex: NULL operand");
  ZI_CHECK_ARG(M > 0 && N > 0 && K > 0 && N % 8 == 0, "zi_gemm_ex: need M, K > 0 and N % 8 == 0");
  ZI_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ldd % 8 == 0, "zi_gemm_ex: leading dims % 8");
  ZI_CHECK_ARG(lda >= (a_mn_major ? M : K) && ldb >= (b_mn_major ? N : K) && ldd >= N,
               "zi_gemm_ex: leading dimension smaller than the row length");
  ZI_CHECK_ARG(zi::aligned(A, 16) && zi::aligned(B, 16) && zi::aligned(D, 16) &&
               (!bias || zi::aligned(bias, 16)), "zi_gemm_ex: 16-byte aligned buffers");
  ZI_CHECK_ARG(epi != ZI_EPI_GELU || (D2 && ldd2 % 8 == 0 && ldd2 >= N && zi::aligned(D2, 16)),
               "zi_gemm_ex: GELU epilogue needs D2");
  ZI_CHECK_ARG((epi != ZI_EPI_RESID && epi != ZI_EPI_DGELU) ||
               (X && ldx % 8 == 0 && ldx >= N && zi::aligned(X, 16)),
               "zi_gemm_ex: epilogue needs X");
  ZI_CHECK_ARG(!(a_mn_major && !b_mn_major), "zi_gemm_ex: MN-major A needs MN-major B");
  int st = get_encoder();
  if (st != ZI_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (epi == ZI_EPI_PLAIN && !use_wide(M, N))
    return zi_gemm(A, a_mn_major, lda, B, b_mn_major, ldb, bias, D, 0, 0, ldd, M, N, K, stream);
  CUtensorMap ma, mb;
  if ((st = make_map(&ma, A, M, K, lda, BM, a_mn_major != 0)) != ZI_OK) return st;
  if ((st = make_map(&mb, B, N, K, ldb, BN / 2, b_mn_major != 0)) != ZI_OK) return st;
  if (a_mn_major)
    return dispatch_epi<true, true>(epi, ma, mb, B, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
  if (b_mn_major)
    return dispatch_epi<false, true>(epi, ma, mb, B, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
  return dispatch_epi<false, false>(epi, ma, mb, B, ldb, bias, D, ldd, X, ldx, D2, ldd2, M, N, K, s);
}

extern "C" int zi_gemm(const void* A, int a_mn_major, int lda, const void* B, int b_mn_major,
                       int ldb, const void* bias, void* D, int d_f32, int accumulate, int ldd,
                       int M, int N, int K, void* stream) {
  using namespace zi::gemm;
  ZI_CHECK_ARG(A && B && D, "zi_gemm: NULL operand");
  ZI_CHECK_ARG(M > 0 && N > 0 && K > 0, "zi_gemm: empty shape");
  ZI_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0, "zi_gemm: lda/ldb must be multiples of 8");
  ZI_CHECK_ARG(lda >= (a_mn_major ? M : K) && ldb >= (b_mn_major ? N : K) && ldd >= N,
               "zi_gemm: leading dimension smaller than the row length");
  ZI_CHECK_ARG(zi::aligned(A, 16) && zi::aligned(B, 16), "zi_gemm: operands must be 16-byte aligned");
  int st = get_encoder();
  if (st != ZI_OK) return st;
  CUtensorMap ma, mb;
  if ((st = make_map(&ma, A, M, K, lda, BM, a_mn_major != 0)) != ZI_OK) return st;
  // paired CTAs each load half of the 256-row B tile (multicast or 2-SM)
  const int b_box = pair_m(M) ? BN / 2 : BN;
  if ((st = make_map(&mb, B, N, K, ldb, b_box, b_mn_major != 0)) != ZI_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!d_f32 && !accumulate && pair_m(M) && use_wide(M, N) && (ldd % 8) == 0 && (N % 8) == 0 &&
      zi::aligned(D, 16) && (!bias || zi::aligned(bias, 16)) && !(a_mn_major && !b_mn_major)) {
    if (a_mn_major)
      return dispatch_epi<true, true>(EPI_PLAIN, ma, mb, B, ldb, bias, D, ldd, nullptr, 0, nullptr, 0, M, N, K, s);
    if (b_mn_major)
      return dispatch_epi<false, true>(EPI_PLAIN, ma, mb, B, ldb, bias, D, ldd, nullptr, 0, nullptr, 0, M, N, K, s);
    return dispatch_epi<false, false>(EPI_PLAIN, ma, mb, B, ldb, bias, D, ldd, nullptr, 0, nullptr, 0, M, N, K, s);
  }
  const int key = (a_mn_major ? 8 : 0) | (b_mn_major ? 4 : 0) | (d_f32 ? 2 : 0) | (accumulate ? 1 : 0);
  switch (key) {
    case 0: return launch<false, false, false, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 4: return launch<false, true, false, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 6: return launch<false, true, true, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 7: return launch<false, true, true, true>(ma, mb, bias, D, M, N, K, ldd, s);
    case 12: return launch<true, true, false, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 14: return launch<true, true, true, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 2: return launch<false, false, true, false>(ma, mb, bias, D, M, N, K, ldd, s);
    case 3: return launch<false, false, true, true>(ma, mb, bias, D, M, N, K, ldd, s);
    default:
      zi::set_error("zi_gemm: unsupported operand/output combination %d", key);
      return ZI_EINVAL;
  }
}

extern "C" int zi_linear_fwd(const void* x, const void* w, const void* bias, void* y, int M, int N,
                             int K, int ldx, int ldw, int ldy, void* stream) {
  return zi_gemm(x, 0, ldx, w, 0, ldw, bias, y, 0, 0, ldy, M, N, K, stream);
}
