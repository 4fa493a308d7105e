// Partition collectives over peer memory.
//
// zi_allgather: the bandwidth-centric fetch (PAPER §6.1 "allgather instead of
// a broadcast"). shards[r] is rank r's shard buffer — local, or a CUDA-IPC
// mapping of the peer's HBM reached over NVLink 5 / NVSwitch. Either one
// copy-engine transfer per rank (no SMs taken from the compute stream) or a
// single vectorised SM kernel that pulls every rank's shard.
//
// zi_barrier: flag-based cross-GPU barrier used to order the P2P
// reduce-scatter (which reads peers' gradient buckets) with the peers'
// producers, and the peers' next overwrite with our reads.
#include "common.cuh"

namespace zi {

constexpr int kMaxWorld = 64;
struct PtrTable {
  const uint8_t* ptr[kMaxWorld];
};
struct FlagTable {
  uint32_t* ptr[kMaxWorld];
};

// blockIdx.y = source rank; grid-stride over 16-byte words of its shard.
__global__ void __launch_bounds__(256)
gather_vec16(PtrTable src, uint8_t* __restrict__ dst, size_t shard_bytes, size_t full_bytes) {
  const int r = blockIdx.y;
  const size_t base = (size_t)r * shard_bytes;
  if (base >= full_bytes) return;
  size_t bytes = full_bytes - base < shard_bytes ? full_bytes - base : shard_bytes;
  const size_t n16 = bytes / 16;
  const uint4* s = reinterpret_cast<const uint4*>(src.ptr[r]);
  uint4* d = reinterpret_cast<uint4*>(dst + base);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread (peer latency ~2 us).
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(s + i), b = __ldcs(s + i + stride);
    uint4 c = __ldcs(s + i + 2 * stride), e = __ldcs(s + i + 3 * stride);
    __stcs(d + i, a); __stcs(d + i + stride, b);
    __stcs(d + i + 2 * stride, c); __stcs(d + i + 3 * stride, e);
  }
  for (; i < n16; i += stride) __stcs(d + i, __ldcs(s + i));
  for (size_t j = n16 * 16 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < bytes; j += stride)
    dst[base + j] = src.ptr[r][j];
}

// Unaligned fallback: element-wise (2/4/8-byte) copy.
template <typename T>
__global__ void __launch_bounds__(256)
gather_elem(PtrTable src, T* __restrict__ dst, size_t shard_elems, size_t full_elems) {
  const int r = blockIdx.y;
  const size_t base = (size_t)r * shard_elems;
  if (base >= full_elems) return;
  size_t n = full_elems - base < shard_elems ? full_elems - base : shard_elems;
  const T* s = reinterpret_cast<const T*>(src.ptr[r]);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[base + i] = s[i];
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// epoch_ctr != nullptr: the epoch is this channel's device counter + 1 (incremented
// here, in stream order), so a barrier captured in a CUDA graph gets a fresh epoch on
// every replay, identical on every rank (each rank runs the same barrier sequence).
__global__ void barrier_kernel(FlagTable f, int world, int rank, uint32_t epoch,
                               uint32_t* epoch_ctr) {
  if (epoch_ctr != nullptr) {
    __shared__ uint32_t e;
    if (threadIdx.x == 0) e = *epoch_ctr + 1;
    __syncthreads();
    epoch = e;
    if (threadIdx.x == 0) *epoch_ctr = e;
  }
  const int k = threadIdx.x;
  if (k < world) {
    __threadfence_system();
    st_release_sys(f.ptr[k] + rank, epoch);
    const long long t0 = clock64();
    while ((int)(ld_acquire_sys(f.ptr[rank] + k) - epoch) < 0) {
      // ~20 s at 2 GHz: a missing peer is a bug; fail loudly, never hang the GPU.
      if (clock64() - t0 > 40000000000LL) __trap();
      __nanosleep(64);
    }
  }
}

}  // namespace zi

extern "C" {

int zi_allgather(const void* const* shards, int world, size_t shard_elems, size_t elem_bytes,
                 void* full, size_t full_elems, int use_copy_engine, void* stream) {
  ZI_CHECK_ARG(shards && full, "zi_allgather: NULL argument");
  ZI_CHECK_ARG(world >= 1 && world <= zi::kMaxWorld, "zi_allgather: bad world %d", world);
  ZI_CHECK_ARG(elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8,
               "zi_allgather: elem_bytes must be 2/4/8");
  ZI_CHECK_ARG(full_elems <= shard_elems * (size_t)world,
               "zi_allgather: full_elems exceeds world*shard_elems");
  if (full_elems == 0 || shard_elems == 0) return ZI_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t shard_bytes = shard_elems * elem_bytes, full_bytes = full_elems * elem_bytes;
  if (use_copy_engine) {
    for (int r = 0; r < world; ++r) {
      const size_t base = (size_t)r * shard_bytes;
      if (base >= full_bytes) break;
      const size_t b = full_bytes - base < shard_bytes ? full_bytes - base : shard_bytes;
      if (shards[r] == static_cast<const uint8_t*>(full) + base) continue;  // in place
      ZI_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(full) + base, shards[r], b,
                              cudaMemcpyDefault, s), "zi_allgather: cudaMemcpyAsync");
    }
    return ZI_OK;
  }
  zi::PtrTable t{};
  bool vec = zi::aligned(full, 16) && shard_bytes % 16 == 0;
  for (int r = 0; r < world; ++r) {
    ZI_CHECK_ARG(shards[r] != nullptr, "zi_allgather: shards[%d] is NULL", r);
    t.ptr[r] = static_cast<const uint8_t*>(shards[r]);
    vec = vec && zi::aligned(shards[r], 16);
  }
  const int block = 256;
  const size_t per_rank = vec ? shard_bytes / 16 : shard_elems;
  int gx = zi::grid_for(per_rank, block, 8);
  gx = (gx + world - 1) / world;
  if (gx < 1) gx = 1;
  dim3 grid(gx, world);
  if (vec) {
    zi::gather_vec16<<<grid, block, 0, s>>>(t, static_cast<uint8_t*>(full), shard_bytes, full_bytes);
  } else if (elem_bytes == 2) {
    zi::gather_elem<uint16_t><<<grid, block, 0, s>>>(t, static_cast<uint16_t*>(full), shard_elems, full_elems);
  } else if (elem_bytes == 4) {
    zi::gather_elem<uint32_t><<<grid, block, 0, s>>>(t, static_cast<uint32_t*>(full), shard_elems, full_elems);
  } else {
    zi::gather_elem<uint64_t><<<grid, block, 0, s>>>(t, static_cast<uint64_t*>(full), shard_elems, full_elems);
  zi::count_launches();
  }
  return zi::launch_status("zi_allgather");
}

int zi_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, void* stream) {
  ZI_CHECK_ARG(flags != nullptr, "zi_barrier: NULL flags");
  ZI_CHECK_ARG(world >= 1 && world <= zi::kMaxWorld && rank >= 0 && rank < world,
               "zi_barrier: bad world/rank %d/%d", world, rank);
  if (world == 1) return ZI_OK;
  zi::FlagTable f{};
  for (int k = 0; k < world; ++k) {
    ZI_CHECK_ARG(flags[k] != nullptr, "zi_barrier: flags[%d] is NULL", k);
    f.ptr[k] = flags[k];
  }
  zi::barrier_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(f, world, rank, epoch, nullptr);
  zi::count_launches();
  return zi::launch_status("zi_barrier");
}

int zi_barrier_dev(uint32_t* const* flags, int world, int rank, uint32_t* epoch_ctr,
                   void* stream) {
  ZI_CHECK_ARG(flags != nullptr && epoch_ctr != nullptr, "zi_barrier_dev: NULL argument");
  ZI_CHECK_ARG(world >= 1 && world <= zi::kMaxWorld && rank >= 0 && rank < world,
               "zi_barrier_dev: bad world/rank %d/%d", world, rank);
  if (world == 1) return ZI_OK;
  zi::FlagTable f{};
  for (int k = 0; k < world; ++k) {
    ZI_CHECK_ARG(flags[k] != nullptr, "zi_barrier_dev: flags[%d] is NULL", k);
    f.ptr[k] = flags[k];
  }
  zi::barrier_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(f, world, rank, 0u, epoch_ctr);
  zi::count_launches();
  return zi::launch_status("zi_barrier_dev");
}

}  // extern "C"
