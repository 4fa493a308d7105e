// Tied-embedding gradient in a fixed order (reductions in fixed order).
//
//   out[v, :] = half_RNE( acc[v, :] + sum_{t : tokens[t] == v, t ascending} dx[t, :] )
//
// acc is the head's fp32 contribution (dlogits^T hf, written by the head.dW GEMM); dx the
// gradient reaching the embedding lookup. A scatter-add (index_add_) would sum a row's
// tokens in whatever order its atomics land; here the tokens are counting-sorted by id
// with a stable rank (the number of earlier equal ids), so every row sums its tokens in
// sequence order and the gradient is bitwise reproducible.
//
//   count   counts[v] = #tokens with id v (integer atomics: order-free)
//   scan    offsets = exclusive prefix sum of counts (one CTA)
//   place   order[offsets[id_t] + rank_t] = t, rank_t = #{t' < t : id_t' == id_t}
//   rows    one CTA per vocabulary row: fold acc + dx rows in order, round, store
#include "common.cuh"

namespace zi {
namespace emb {

__global__ void count_kernel(const int64_t* __restrict__ tok, int T, int V, int* __restrict__ counts) {
  zi::pdl_sync();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) {
    const int64_t v = tok[t];
    if (v >= 0 && v < V) atomicAdd(&counts[v], 1);
  }
}

// exclusive scan of counts[0..V) into offsets[0..V] (offsets[V] = T); one CTA of 1024.
// Each thread's contiguous range is read 8 counts at a time, the 8 loads in flight together
// (not one dependent L2 round trip per element).
__global__ void __launch_bounds__(1024)
scan_kernel(const int* __restrict__ counts, int V, int* __restrict__ offsets) {
  zi::pdl_sync();
  __shared__ int part[1024];
  const int tid = threadIdx.x, per = (V + 1023) / 1024;
  const int lo = min(V, tid * per), hi = min(V, lo + per);
  int s = 0;
  for (int i = lo; i < hi; i += 8) {
    int c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = i + k < hi ? counts[i + k] : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k];
  }
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {           // Hillis-Steele inclusive scan
    const int x = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += x;
    __syncthreads();
  }
  int run = tid ? part[tid - 1] : 0;
  for (int i = lo; i < hi; i += 8) {
    int c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = i + k < hi ? counts[i + k] : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i + k < hi) offsets[i + k] = run;
      run += c[k];
    }
  }
  if (tid == 1023) offsets[V] = part[1023];
}

// stable placement; earlier tokens stream through shared memory in tiles of int32 ids.
// A CTA of 256 threads places 64 tokens, 4 threads per token each counting the equal ids
// in one quarter of the earlier range (integer sums: order-free), so T / 64 CTAs share
// the O(T^2 / 2) comparisons.
constexpr int PLACE_TILE = 8192, PLACE_TOK = 64, PLACE_SPLIT = 4;

__global__ void __launch_bounds__(PLACE_TOK * PLACE_SPLIT)
place_kernel(const int64_t* __restrict__ tok, int T, int V, const int* __restrict__ offsets,
             int* __restrict__ order) {
  zi::pdl_sync();
  __shared__ int st[PLACE_TILE];
  __shared__ int cnt[PLACE_SPLIT][PLACE_TOK];
  const int j = threadIdx.x % PLACE_TOK, q = threadIdx.x / PLACE_TOK;
  const int t = blockIdx.x * PLACE_TOK + j;
  const int v = t < T ? (int)tok[t] : -1;
  const int tmax = min(T, (int)((blockIdx.x + 1) * PLACE_TOK));   // the block's last t + 1
  int rank = 0;
  for (int k0 = 0; k0 < tmax; k0 += PLACE_TILE) {
    const int n = min(PLACE_TILE, T - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) st[i] = (int)tok[k0 + i];
    __syncthreads();
    const int kend = max(0, min(n, t - k0));
    const int qlen = (kend + PLACE_SPLIT - 1) / PLACE_SPLIT;
    const int a = min(kend, q * qlen), b = min(kend, a + qlen);
    for (int k = a; k < b; ++k) rank += (st[k] == v);
  }
  cnt[q][j] = rank;
  __syncthreads();
  if (q == 0) {
    rank = cnt[0][j] + cnt[1][j] + cnt[2][j] + cnt[3][j];
    if (t < T && v >= 0 && v < V) order[offsets[v] + rank] = t;
  }
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  const uint4 g = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 x = __bfloat1622float2(g2[q]);
    f[2 * q] = x.x;
    f[2 * q + 1] = x.y;
  }
}
__device__ __forceinline__ void load8(const __half* p, float* f) {
  const uint4 g = *reinterpret_cast<const uint4*>(p);
  const __half2* g2 = reinterpret_cast<const __half2*>(&g);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 x = __half22float2(g2[q]);
    f[2 * q] = x.x;
    f[2 * q + 1] = x.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <int KIND, typename TX>
__global__ void rows_kernel(const TX* __restrict__ dx, const float* __restrict__ acc,
                            const int* __restrict__ offsets, const int* __restrict__ order, int hd,
                            uint16_t* __restrict__ out) {
  zi::pdl_sync();
  const int v = blockIdx.x;
  const int e = threadIdx.x * 8;                 // 8 consecutive elements per thread
  if (e >= hd) return;
  const size_t base = (size_t)v * hd + e;
  const float4 a0 = *reinterpret_cast<const float4*>(acc + base);
  const float4 a1 = *reinterpret_cast<const float4*>(acc + base + 4);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int k0 = offsets[v], k1 = offsets[v + 1];
  for (int k = k0; k < k1; ++k) {                // the row's tokens in sequence order
    float f[8];
    load8(dx + (size_t)order[k] * hd + e, f);
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] += f[q];
  }
  const float r[8] = {a0.x + s[0], a0.y + s[1], a0.z + s[2], a0.w + s[3],
                      a1.x + s[4], a1.y + s[5], a1.z + s[6], a1.w + s[7]};
  uint4 o;
  o.x = (uint32_t)Half<KIND>::narrow(r[0]) | ((uint32_t)Half<KIND>::narrow(r[1]) << 16);
  o.y = (uint32_t)Half<KIND>::narrow(r[2]) | ((uint32_t)Half<KIND>::narrow(r[3]) << 16);
  o.z = (uint32_t)Half<KIND>::narrow(r[4]) | ((uint32_t)Half<KIND>::narrow(r[5]) << 16);
  o.w = (uint32_t)Half<KIND>::narrow(r[6]) | ((uint32_t)Half<KIND>::narrow(r[7]) << 16);
  *reinterpret_cast<uint4*>(out + base) = o;
}

// Embedding lookup of the step's forward: x[t, :] = RNE(wte[tokens[t], :] + wpe[t % S, :]),
// bf16 in and out, the sum in fp32 (torch's bf16 add: F.embedding(tok, wte) + wpe, bit
// for bit). One thread per 8 consecutive elements of a row; out-of-range ids read no wte
// row (their x row is wpe alone, like count_kernel skipping them).
__global__ void __launch_bounds__(256)
fwd_kernel(const int64_t* __restrict__ tok, int T, int S, const __nv_bfloat16* __restrict__ wte,
           const __nv_bfloat16* __restrict__ wpe, int V, int hd, uint16_t* __restrict__ x) {
  zi::pdl_sync();
  const int per_row = hd / 8;
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)T * per_row) return;
  const int t = (int)(i / per_row), e = (int)(i % per_row) * 8;
  const int64_t v = tok[t];
  float a[8], b[8];
  load8(wpe + (size_t)(t % S) * hd + e, b);
  if (v >= 0 && v < V) load8(wte + (size_t)v * hd + e, a);
  else for (int q = 0; q < 8; ++q) a[q] = 0.f;
  uint4 o;
  uint32_t* w = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    w[q] = (uint32_t)Half<ZI_HALF_BF16>::narrow(a[2 * q] + b[2 * q]) |
           ((uint32_t)Half<ZI_HALF_BF16>::narrow(a[2 * q + 1] + b[2 * q + 1]) << 16);
  *reinterpret_cast<uint4*>(x + (size_t)t * hd + e) = o;
}

// Position-embedding gradient: out[s, :] = sum_{b ascending} dx[b * S + s, :] in fp32,
// stored as fp32 (OUT = -1) or rounded RNE to half (OUT = half kind). Fixed order.
template <typename TX, int OUT>
__global__ void __launch_bounds__(256)
pos_grad_kernel(const TX* __restrict__ dx, int B, int S, int hd, void* __restrict__ out) {
  zi::pdl_sync();
  const int per_row = hd / 8;
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)S * per_row) return;
  const size_t off = (i / per_row) * (size_t)hd + (i % per_row) * 8;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int b = 0; b < B; ++b) {
    float f[8];
    load8(dx + (size_t)b * S * hd + off, f);
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] += f[q];
  }
  if constexpr (OUT < 0) {
    float* o = static_cast<float*>(out) + off;
    *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
  } else {
    uint4 o;
    uint32_t* w = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      w[q] = (uint32_t)Half<OUT>::narrow(s[2 * q]) | ((uint32_t)Half<OUT>::narrow(s[2 * q + 1]) << 16);
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(out) + off) = o;
  }
}

}  // namespace emb
}  // namespace zi

extern "C" {

int zi_embed_grad(const int64_t* tokens, int T, const void* dx, int dx_f32, const float* acc, int V,
                  int hd, void* out, int half_kind, int* work, void* stream) {
  ZI_CHECK_ARG(tokens && dx && acc && out && work, "zi_embed_grad: NULL argument");
  ZI_CHECK_ARG(T >= 1 && V >= 1 && hd >= 8 && hd % 8 == 0 && hd / 8 <= 1024,
               "zi_embed_grad: bad T/V/hd %d/%d/%d", T, V, hd);
  ZI_CHECK_ARG(half_kind == ZI_HALF_BF16 || half_kind == ZI_HALF_FP16,
               "zi_embed_grad: bad half_kind %d", half_kind);
  ZI_CHECK_ARG(zi::aligned(dx, 16) && zi::aligned(acc, 16) && zi::aligned(out, 16),
               "zi_embed_grad: 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  int* counts = work;              // [V]
  int* offsets = work + V;         // [V + 1]
  int* order = offsets + V + 1;    // [T]
  ZI_CUDA(cudaMemsetAsync(counts, 0, (size_t)V * sizeof(int), s), "zi_embed_grad: memset");
  zi::launch_pdl(zi::emb::count_kernel, dim3((T + 255) / 256), dim3(256), 0, s, tokens, T, V, counts);
  zi::launch_pdl(zi::emb::scan_kernel, dim3(1), dim3(1024), 0, s, counts, V, offsets);
  zi::launch_pdl(zi::emb::place_kernel, dim3((T + zi::emb::PLACE_TOK - 1) / zi::emb::PLACE_TOK),
                 dim3(zi::emb::PLACE_TOK * zi::emb::PLACE_SPLIT), 0, s, tokens, T, V, offsets, order);
  const int threads = ((hd / 8 + 31) / 32) * 32;
  auto* o = static_cast<uint16_t*>(out);
  const auto* xb = static_cast<const __nv_bfloat16*>(dx);
  const auto* xf = static_cast<const float*>(dx);
  if (half_kind == ZI_HALF_BF16) {
    if (dx_f32) zi::launch_pdl(zi::emb::rows_kernel<ZI_HALF_BF16, float>, dim3(V), dim3(threads), 0, s, xf, acc, offsets, order, hd, o);
    else zi::launch_pdl(zi::emb::rows_kernel<ZI_HALF_BF16, __nv_bfloat16>, dim3(V), dim3(threads), 0, s, xb, acc, offsets, order, hd, o);
  } else {
    if (dx_f32) zi::launch_pdl(zi::emb::rows_kernel<ZI_HALF_FP16, float>, dim3(V), dim3(threads), 0, s, xf, acc, offsets, order, hd, o);
    else zi::launch_pdl(zi::emb::rows_kernel<ZI_HALF_FP16, __nv_bfloat16>, dim3(V), dim3(threads), 0, s, xb, acc, offsets, order, hd, o);
  }
  return zi::launch_status("zi_embed_grad");
}

int zi_embed_fwd(const int64_t* tokens, int T, int S, const void* wte, const void* wpe, int V,
                 int hd, void* x, void* stream) {
  ZI_CHECK_ARG(tokens && wte && wpe && x, "zi_embed_fwd: NULL argument");
  ZI_CHECK_ARG(T >= 1 && S >= 1 && V >= 1 && hd >= 8 && hd % 8 == 0,
               "zi_embed_fwd: bad T/S/V/hd %d/%d/%d/%d", T, S, V, hd);
  ZI_CHECK_ARG(zi::aligned(wte, 16) && zi::aligned(wpe, 16) && zi::aligned(x, 16),
               "zi_embed_fwd: 16-byte alignment");
  const size_t n = (size_t)T * (hd / 8);
  zi::launch_pdl(zi::emb::fwd_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
                 (cudaStream_t)stream, tokens, T, S, static_cast<const __nv_bfloat16*>(wte),
                 static_cast<const __nv_bfloat16*>(wpe), V, hd, static_cast<uint16_t*>(x));
  return zi::launch_status("zi_embed_fwd");
}

int zi_pos_grad(const void* dx, int dx_kind, int B, int S, int hd, void* out, int out_kind,
                void* stream) {
  ZI_CHECK_ARG(dx && out, "zi_pos_grad: NULL argument");
  ZI_CHECK_ARG(B >= 1 && S >= 1 && hd >= 8 && hd % 8 == 0, "zi_pos_grad: bad B/S/hd %d/%d/%d",
               B, S, hd);
  ZI_CHECK_ARG(out_kind == -1 || out_kind == ZI_HALF_BF16 || out_kind == ZI_HALF_FP16,
               "zi_pos_grad: out_kind must be -1 (fp32) or a half kind, got %d", out_kind);
  ZI_CHECK_ARG(zi::aligned(dx, 16) && zi::aligned(out, 16), "zi_pos_grad: 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = (size_t)S * (hd / 8);
  const dim3 g((unsigned)((n + 255) / 256)), b(256);
  ZI_CHECK_ARG(dx_kind == -1 || dx_kind == ZI_HALF_BF16 || dx_kind == ZI_HALF_FP16,
               "zi_pos_grad: dx_kind must be -1 (fp32) or a half kind, got %d", dx_kind);
  const auto* xb = static_cast<const __nv_bfloat16*>(dx);
  const auto* xh = static_cast<const __half*>(dx);
  const auto* xf = static_cast<const float*>(dx);
  using namespace zi::emb;
  if (dx_kind == ZI_HALF_FP16) {
    if (out_kind < 0) zi::launch_pdl(pos_grad_kernel<__half, -1>, g, b, 0, s, xh, B, S, hd, out);
    else if (out_kind == ZI_HALF_BF16) zi::launch_pdl(pos_grad_kernel<__half, ZI_HALF_BF16>, g, b, 0, s, xh, B, S, hd, out);
    else zi::launch_pdl(pos_grad_kernel<__half, ZI_HALF_FP16>, g, b, 0, s, xh, B, S, hd, out);
  } else if (dx_kind < 0) {
    if (out_kind < 0) zi::launch_pdl(pos_grad_kernel<float, -1>, g, b, 0, s, xf, B, S, hd, out);
    else if (out_kind == ZI_HALF_BF16) zi::launch_pdl(pos_grad_kernel<float, ZI_HALF_BF16>, g, b, 0, s, xf, B, S, hd, out);
    else zi::launch_pdl(pos_grad_kernel<float, ZI_HALF_FP16>, g, b, 0, s, xf, B, S, hd, out);
  } else {
    if (out_kind < 0) zi::launch_pdl(pos_grad_kernel<__nv_bfloat16, -1>, g, b, 0, s, xb, B, S, hd, out);
    else if (out_kind == ZI_HALF_BF16) zi::launch_pdl(pos_grad_kernel<__nv_bfloat16, ZI_HALF_BF16>, g, b, 0, s, xb, B, S, hd, out);
    else zi::launch_pdl(pos_grad_kernel<__nv_bfloat16, ZI_HALF_FP16>, g, b, 0, s, xb, B, S, hd, out);
  }
  return zi::launch_status("zi_pos_grad");
}

}  // extern "C"
