// Partitioned optimizer kernels (HBM-bound, one pass over each byte).
//
//   zi_adam_step            chunked_adam_step chunk
//   zi_reduce_scatter_cast  reduce_scatter + cast/scale
//   zi_rs_adam              both fused: the per-layer update the engine runs
//
// Numerics: every float op is an explicit __f*_rn intrinsic in the oracle's
// order (oracle/adam.py, oracle/partition.py), so results are bit-exact with
// the CPU oracle. Contributions are folded left-to-right in fp32 in the
// order given (rank order).
//
// Memory: 8 elements per thread-iteration; fp32 arrays move as two 128-bit
// streaming accesses, half arrays as one. Algorithmic bytes per element:
// adam 30 (16 read + 14 write), rs_adam 2*K + 12 read + 14 write.
#include "common.cuh"

namespace zi {

constexpr int kMaxContrib = 64;
struct Contribs {
  const uint16_t* ptr[kMaxContrib];
};

template <int KIND>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  return (uint32_t)Half<KIND>::narrow(a) | ((uint32_t)Half<KIND>::narrow(b) << 16);
}

template <int KIND>
__device__ __forceinline__ void widen8(uint4 w, float* f) {
  const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[2 * j] = Half<KIND>::widen((uint16_t)(u[j] & 0xFFFF));
    f[2 * j + 1] = Half<KIND>::widen((uint16_t)(u[j] >> 16));
  }
}

__device__ __forceinline__ void load8(const float* base, size_t i8, float* f) {
  const float4 a = ld_stream(reinterpret_cast<const float4*>(base) + 2 * i8);
  const float4 b = ld_stream(reinterpret_cast<const float4*>(base) + 2 * i8 + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

__device__ __forceinline__ void store8(float* base, size_t i8, const float* f) {
  st_stream(reinterpret_cast<float4*>(base) + 2 * i8, make_float4(f[0], f[1], f[2], f[3]));
  st_stream(reinterpret_cast<float4*>(base) + 2 * i8 + 1, make_float4(f[4], f[5], f[6], f[7]));
}

template <int KIND>
__device__ __forceinline__ void store8_half(uint16_t* base, size_t i8, const float* f) {
  uint4 h;
  h.x = pack2<KIND>(f[0], f[1]);
  h.y = pack2<KIND>(f[2], f[3]);
  h.z = pack2<KIND>(f[4], f[5]);
  h.w = pack2<KIND>(f[6], f[7]);
  st_stream(reinterpret_cast<uint4*>(base) + i8, h);
}

// ------------------------------------------------------------------- Adam
template <int KIND>
__global__ void __launch_bounds__(256)
adam_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
            const float* __restrict__ g, uint16_t* __restrict__ ph, size_t n, size_t n8,
            zi_adam_consts c) {
  zi::pdl_sync();
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < n8; i += stride) {
    float pp[8], mm[8], vv[8], gg[8];
    load8(p, i, pp); load8(m, i, mm); load8(v, i, vv); load8(g, i, gg);
#pragma unroll
    for (int j = 0; j < 8; ++j) adam1(pp[j], mm[j], vv[j], gg[j], c);
    store8(p, i, pp); store8(m, i, mm); store8(v, i, vv);
    if (ph) store8_half<KIND>(ph, i, pp);
  }
  for (size_t i = n8 * 8 + tid; i < n; i += stride) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam1(pp, mm, vv, g[i], c);
    p[i] = pp; m[i] = mm; v[i] = vv;
    if (ph) ph[i] = Half<KIND>::narrow(pp);
  }
}

// ----------------------------------------------------- reduce-scatter (+Adam)
// Fold of K half contributions at [off, off + n) into fp32, times scale.
// Elements at global index >= clen read 0. If ADAM, the fp32 gradient feeds
// the Adam update of (p, m, v) and the half copy; g_out (nullable) gets it.
template <int KIND, bool ADAM>
__global__ void __launch_bounds__(256)
rs_kernel(Contribs cb, int K, size_t off, size_t n, size_t nvec8, size_t clen, float scale,
          float* __restrict__ out_or_g, float* __restrict__ p, float* __restrict__ m,
          float* __restrict__ v, uint16_t* __restrict__ ph, zi_adam_consts c,
          const zi_adam_consts* __restrict__ cdev) {
  zi::pdl_sync();
  if (ADAM && cdev != nullptr) c = *cdev;  // constants advanced on the device (CUDA graphs)
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < nvec8; i += stride) {
    float acc[8];
    {
      const uint4 w = ld_stream(reinterpret_cast<const uint4*>(cb.ptr[0] + off) + i);
      widen8<KIND>(w, acc);
    }
#pragma unroll 4
    for (int k = 1; k < K; ++k) {
      const uint4 w = ld_stream(reinterpret_cast<const uint4*>(cb.ptr[k] + off) + i);
      float f[8];
      widen8<KIND>(w, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], f[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __fmul_rn(acc[j], scale);
    if (!ADAM) {
      store8(out_or_g, i, acc);
    } else {
      if (out_or_g) store8(out_or_g, i, acc);
      float pp[8], mm[8], vv[8];
      load8(p, i, pp); load8(m, i, mm); load8(v, i, vv);
#pragma unroll
      for (int j = 0; j < 8; ++j) adam1(pp[j], mm[j], vv[j], acc[j], c);
      store8(p, i, pp); store8(m, i, mm); store8(v, i, vv);
      if (ph) store8_half<KIND>(ph, i, pp);
    }
  }
  for (size_t i = nvec8 * 8 + tid; i < n; i += stride) {
    const size_t gi = off + i;
    float acc = 0.f;
    for (int k = 0; k < K; ++k) {
      const float f = gi < clen ? Half<KIND>::widen(cb.ptr[k][gi]) : 0.f;
      acc = k == 0 ? f : __fadd_rn(acc, f);
    }
    acc = __fmul_rn(acc, scale);
    if (!ADAM) {
      out_or_g[i] = acc;
    } else {
      if (out_or_g) out_or_g[i] = acc;
      float pp = p[i], mm = m[i], vv = v[i];
      adam1(pp, mm, vv, acc, c);
      p[i] = pp; m[i] = mm; v[i] = vv;
      if (ph) ph[i] = Half<KIND>::narrow(pp);
    }
  }
}

// ZI_RS_WAVES (A/B): grid = that many waves of resident CTAs (default 1)
static int rs_waves() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("ZI_RS_WAVES");
    w = e ? atoi(e) : 1;
    if (w < 1) w = 1;
  }
  return w;
}

template <bool ADAM>
int launch_rs(const void* const* contribs, int K, size_t off, size_t n, size_t clen,
              float scale, int half_kind, float* out_or_g, float* p, float* m, float* v,
              void* p_half, const zi_adam_consts* c, void* stream, const char* name,
              const zi_adam_consts* cdev = nullptr) {
  ZI_CHECK_ARG(contribs != nullptr && K >= 1 && K <= kMaxContrib,
               "%s: need 1 <= n_contrib <= %d", name, kMaxContrib);
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16, "%s: bad half_kind", name);
  if (ADAM) ZI_CHECK_ARG(p && m && v && (c || cdev), "%s: NULL p/m/v/consts", name);
  else ZI_CHECK_ARG(out_or_g != nullptr, "%s: NULL out", name);
  if (n == 0) return ZI_OK;
  Contribs cb{};
  bool vec = (off % 8) == 0;
  for (int k = 0; k < K; ++k) {
    ZI_CHECK_ARG(contribs[k] != nullptr, "%s: contribs[%d] is NULL", name, k);
    cb.ptr[k] = static_cast<const uint16_t*>(contribs[k]);
    vec = vec && aligned(contribs[k], 16);
  }
  vec = vec && (!out_or_g || aligned(out_or_g, 16));
  if (ADAM) vec = vec && aligned(p, 16) && aligned(m, 16) && aligned(v, 16) &&
                  (!p_half || aligned(p_half, 16));
  const size_t valid = clen > off ? (clen - off < n ? clen - off : n) : 0;
  const size_t nvec8 = vec ? valid / 8 : 0;
  const zi_adam_consts cc = c ? *c : zi_adam_consts{};
  const int block = 256;
  // one wave of resident CTAs (64 registers: 4 per SM), each grid-striding: a grid of
  // 8 per SM ran as two waves with a ragged hand-over between them
  static int per_sm[2] = {0, 0};
  int& ps = per_sm[half_kind == ZI_HALF_BF16];
  if (ps == 0) {
    int b = 0;
    if (half_kind == ZI_HALF_BF16)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_kernel<ZI_HALF_BF16, ADAM>, block, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rs_kernel<ZI_HALF_FP16, ADAM>, block, 0);
    ps = b > 0 ? b : 8;
  }
  const int grid = grid_for(nvec8 + (n - nvec8 * 8), block, rs_waves() * ps);
  cudaStream_t s = (cudaStream_t)stream;
  uint16_t* ph = static_cast<uint16_t*>(p_half);
  // (two 8-element groups per thread-iteration, all 14 loads in flight, measured slower
  // in the step: 275 vs 249 us per launch at 118 vs 64 registers)
  if (half_kind == ZI_HALF_BF16)
    zi::launch_pdl(rs_kernel<ZI_HALF_BF16, ADAM>, dim3(grid), dim3(block), 0, s, cb, K, off, n, nvec8,
                   clen, scale, out_or_g, p, m, v, ph, cc, cdev);
  else
    zi::launch_pdl(rs_kernel<ZI_HALF_FP16, ADAM>, dim3(grid), dim3(block), 0, s, cb, K, off, n, nvec8,
                   clen, scale, out_or_g, p, m, v, ph, cc, cdev);
  return launch_status(name);
}

// t <- t + 1 on the device and the step's folded constants, exactly the
// host-side folding (oracle/adam.py AdamConsts.make): doubles rounded once.
__global__ void adam_advance_kernel(double lr, double b1, double b2, double eps, int* step,
                                    zi_adam_consts* out) {
  zi::pdl_sync();
  const int t = *step + 1;
  *step = t;
  zi_adam_consts c;
  c.lr = (float)lr;
  c.b1 = (float)b1;
  c.omb1 = (float)(1.0 - b1);
  c.b2 = (float)b2;
  c.omb2 = (float)(1.0 - b2);
  c.bc1 = (float)(1.0 - pow(b1, (double)t));
  c.bc2 = (float)(1.0 - pow(b2, (double)t));
  c.eps = (float)eps;
  *out = c;
}

// Generic SPEC reduce_scatter for full-precision contributions: fp32 inputs
// fold in fp32, fp64 in fp64 ("bit-exact in f64 ... and f32").
template <typename T>
__global__ void __launch_bounds__(256)
rs_full_kernel(Contribs cb, int K, size_t off, size_t n, size_t clen, T scale, T* __restrict__ out) {
  zi::pdl_sync();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const size_t gi = off + i;
    T acc = 0;
    for (int k = 0; k < K; ++k) {
      const T f = gi < clen ? reinterpret_cast<const T*>(cb.ptr[k])[gi] : T(0);
      acc = k == 0 ? f : acc + f;
    }
    out[i] = acc * scale;
  }
}

}  // namespace zi

extern "C" {

int zi_reduce_scatter(const void* const* contribs, int n_contrib, size_t shard_offset,
                      size_t shard_elems, size_t contrib_len, int dtype, double scale, void* out,
                      void* stream) {
  if (dtype == ZI_DT_F16 || dtype == ZI_DT_BF16)
    return zi_reduce_scatter_cast(contribs, n_contrib, shard_offset, shard_elems, contrib_len,
                                  (float)scale, dtype == ZI_DT_BF16 ? ZI_HALF_BF16 : ZI_HALF_FP16,
                                  static_cast<float*>(out), stream);
  ZI_CHECK_ARG(dtype == ZI_DT_F32 || dtype == ZI_DT_F64, "zi_reduce_scatter: bad dtype %d", dtype);
  ZI_CHECK_ARG(contribs && out && n_contrib >= 1 && n_contrib <= zi::kMaxContrib,
               "zi_reduce_scatter: bad arguments");
  if (shard_elems == 0) return ZI_OK;
  zi::Contribs cb{};
  for (int k = 0; k < n_contrib; ++k) {
    ZI_CHECK_ARG(contribs[k] != nullptr, "zi_reduce_scatter: contribs[%d] is NULL", k);
    cb.ptr[k] = static_cast<const uint16_t*>(contribs[k]);
  }
  const int grid = zi::grid_for(shard_elems, 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == ZI_DT_F32)
    zi::launch_pdl(zi::rs_full_kernel<float>, dim3(grid), dim3(256), 0, s, cb, n_contrib, shard_offset, shard_elems,
                                                   contrib_len, (float)scale, static_cast<float*>(out));
  else
    zi::launch_pdl(zi::rs_full_kernel<double>, dim3(grid), dim3(256), 0, s, cb, n_contrib, shard_offset, shard_elems,
                                                    contrib_len, scale, static_cast<double*>(out));
  return zi::launch_status("zi_reduce_scatter");
}


int zi_adam_step(float* p, float* m, float* v, const float* g, void* p_half, size_t n,
                 const zi_adam_consts* c, int half_kind, void* stream) {
  ZI_CHECK_ARG(p && m && v && g && c, "zi_adam_step: NULL argument");
  ZI_CHECK_ARG(half_kind == ZI_HALF_FP16 || half_kind == ZI_HALF_BF16,
               "zi_adam_step: bad half_kind %d", half_kind);
  if (n == 0) return ZI_OK;
  const bool vec = zi::aligned(p, 16) && zi::aligned(m, 16) && zi::aligned(v, 16) &&
                   zi::aligned(g, 16) && (!p_half || zi::aligned(p_half, 16));
  const size_t n8 = vec ? n / 8 : 0;
  const int block = 256;
  const int grid = zi::grid_for(n8 + (n - n8 * 8), block);
  cudaStream_t s = (cudaStream_t)stream;
  uint16_t* ph = static_cast<uint16_t*>(p_half);
  if (half_kind == ZI_HALF_BF16)
    zi::launch_pdl(zi::adam_kernel<ZI_HALF_BF16>, dim3(grid), dim3(block), 0, s, p, m, v, g, ph, n, n8, *c);
  else
    zi::launch_pdl(zi::adam_kernel<ZI_HALF_FP16>, dim3(grid), dim3(block), 0, s, p, m, v, g, ph, n, n8, *c);
  return zi::launch_status("zi_adam_step");
}

int zi_reduce_scatter_cast(const void* const* contribs, int n_contrib, size_t shard_offset,
                           size_t shard_elems, size_t contrib_len, float scale, int half_kind,
                           float* out, void* stream) {
  return zi::launch_rs<false>(contribs, n_contrib, shard_offset, shard_elems, contrib_len, scale,
                              half_kind, out, nullptr, nullptr, nullptr, nullptr, nullptr, stream,
                              "zi_reduce_scatter_cast");
}

int zi_rs_adam(const void* const* contribs, int n_contrib, size_t shard_offset, size_t shard_elems,
               size_t contrib_len, float scale, int half_kind, float* p, float* m, float* v,
               void* p_half, float* g_out, const zi_adam_consts* c, void* stream) {
  return zi::launch_rs<true>(contribs, n_contrib, shard_offset, shard_elems, contrib_len, scale,
                             half_kind, g_out, p, m, v, p_half, c, stream, "zi_rs_adam");
}

int zi_rs_adam_dc(const void* const* contribs, int n_contrib, size_t shard_offset,
                  size_t shard_elems, size_t contrib_len, float scale, int half_kind, float* p,
                  float* m, float* v, void* p_half, float* g_out, const zi_adam_consts* c_dev,
                  void* stream) {
  ZI_CHECK_ARG(c_dev != nullptr, "zi_rs_adam_dc: NULL device constants");
  return zi::launch_rs<true>(contribs, n_contrib, shard_offset, shard_elems, contrib_len, scale,
                             half_kind, g_out, p, m, v, p_half, nullptr, stream, "zi_rs_adam_dc",
                             c_dev);
}

int zi_adam_advance(double lr, double beta1, double beta2, double eps, int* step_dev,
                    zi_adam_consts* consts_dev, void* stream) {
  ZI_CHECK_ARG(step_dev && consts_dev, "zi_adam_advance: NULL device pointer");
  zi::launch_pdl(zi::adam_advance_kernel, dim3(1), dim3(1), 0, (cudaStream_t)stream, lr, beta1, beta2, eps, step_dev,
                                                            consts_dev);
  return zi::launch_status("zi_adam_advance");
}

}  // extern "C"
