// zi_ctx: the native communicator context of one data-parallel rank.
//
// SURVEY.md §8(b) asks the C ABI for a context holding rank, world and device plus
// the peers' IPC-mapped buffers, so a binding can run the partitioned collectives
// with plain pointers. The context owns
//   * windows: a buffer of the same shape on every rank (the bf16 parameter arena,
//     a gradient-bucket ring, a barrier flag array). Each rank's CUDA-IPC handle and
//     byte offset are exchanged out of band (torch.distributed in comm.DistComm, or
//     any launcher) and handed to zi_ctx_add_window, which maps every peer
//     allocation once (cudaIpcMemLazyEnablePeerAccess: direct NVLink 5 loads and
//     stores between GPUs) and keeps the per-rank pointer table;
//   * barrier epochs: one device-side counter per flag window, advanced by the barrier
//     kernel itself, so zi_ctx_barrier needs no caller-side state, a barrier captured in
//     a CUDA graph stays correct on every replay, and barriers on different streams use
//     different windows.
// The data-path entry points are the SPEC collectives over a window:
//   zi_ctx_allgather           = SPEC allgather
//   zi_ctx_reduce_scatter_cast = SPEC reduce_scatter with the half->fp32 cast and
//                                1/N scale, folded in rank order
// Every call is asynchronous on the caller's stream; the context is guarded by a
// mutex, so one context may be shared by the threads of a rank.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

struct zi_ctx {
  int rank = 0, world = 1, device = 0;
  std::mutex mu;
  struct Window {
    std::vector<uint8_t*> ptr;   // [world] base of this window on each rank (ours is local)
  };
  static constexpr int kMaxWindows = 1024;
  uint32_t* epochs = nullptr;    // device: barrier epoch counter per window (graph-safe)
  std::vector<Window> windows;
  struct Mapping {
    unsigned char handle[64];
    void* base;
  };
  std::vector<Mapping> mapped;   // each peer allocation opened once
};

namespace {

int open_mapping(zi_ctx* c, const unsigned char* h, void** base) {
  for (auto& m : c->mapped)
    if (memcmp(m.handle, h, 64) == 0) {
      *base = m.base;
      return ZI_OK;
    }
  cudaIpcMemHandle_t ih;
  memcpy(&ih, h, 64);
  void* p = nullptr;
  ZI_CUDA(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  zi_ctx::Mapping m;
  memcpy(m.handle, h, 64);
  m.base = p;
  c->mapped.push_back(m);
  *base = p;
  return ZI_OK;
}

// Stream memory operations (driver API, resolved once through the runtime's entry-point
// query so libzinf needs no -lcuda): the barrier's writes and waits execute in the
// stream's front end, so a waiting rank holds no SM (it cannot starve the persistent
// tcgen05 GEMMs, or a peer context time-sharing the GPU).
PFN_cuStreamWriteValue32_v11070 g_write32 = nullptr;
PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;

int load_memops() {
  static std::once_flag once;
  static int st = ZI_OK;
  std::call_once(once, [] {
    void* w = nullptr;
    void* t = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !t) {
      st = ZI_ECUDA;
      return;
    }
    g_write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(w);
    g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(t);
  });
  if (st != ZI_OK) zi::set_error("cuStreamWriteValue32 / cuStreamWaitValue32 unavailable");
  return st;
}

}  // namespace

extern "C" {

int zi_ctx_create(int rank, int world, int device, zi_ctx** out) {
  ZI_CHECK_ARG(out != nullptr, "zi_ctx_create: NULL out");
  ZI_CHECK_ARG(world >= 1 && world <= 64 && rank >= 0 && rank < world,
               "zi_ctx_create: bad rank/world %d/%d", rank, world);
  ZI_CHECK_ARG(device >= 0, "zi_ctx_create: bad device %d", device);
  int ndev = 0;
  ZI_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  ZI_CHECK_ARG(device < ndev, "zi_ctx_create: device %d of %d", device, ndev);
  // libzinf links its own (static) CUDA runtime: make its current device on this thread
  // the rank's GPU, so zi_device_alloc / IPC mappings / launches agree with the caller's
  ZI_CUDA(cudaSetDevice(device), "cudaSetDevice");
  uint32_t* ep = nullptr;
  ZI_CUDA(cudaMalloc(&ep, zi_ctx::kMaxWindows * sizeof(uint32_t)), "cudaMalloc(epochs)");
  ZI_CUDA(cudaMemset(ep, 0, zi_ctx::kMaxWindows * sizeof(uint32_t)), "cudaMemset(epochs)");
  zi_ctx* c = new zi_ctx;
  c->epochs = ep;
  c->rank = rank;
  c->world = world;
  c->device = device;
  *out = c;
  return ZI_OK;
}

int zi_ctx_destroy(zi_ctx* c) {
  if (!c) return ZI_OK;
  int st = ZI_OK;
  {
    std::lock_guard<std::mutex> g(c->mu);
    for (auto& m : c->mapped) {
      cudaError_t e = cudaIpcCloseMemHandle(m.base);
      if (e != cudaSuccess && st == ZI_OK) st = zi::cuda_status(e, "cudaIpcCloseMemHandle");
    }
    c->mapped.clear();
  }
  if (c->epochs) cudaFree(c->epochs);
  delete c;
  return st;
}

int zi_ctx_info(const zi_ctx* c, int* rank, int* world, int* device) {
  ZI_CHECK_ARG(c != nullptr, "zi_ctx_info: NULL ctx");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (device) *device = c->device;
  return ZI_OK;
}

int zi_ctx_add_window(zi_ctx* c, void* local, const unsigned char* handles,
                      const uint64_t* offsets, int* win) {
  ZI_CHECK_ARG(c && local && win, "zi_ctx_add_window: NULL argument");
  ZI_CHECK_ARG((int)c->windows.size() < zi_ctx::kMaxWindows, "zi_ctx_add_window: too many windows");
  ZI_CHECK_ARG(c->world == 1 || (handles && offsets), "zi_ctx_add_window: NULL handles/offsets");
  std::lock_guard<std::mutex> g(c->mu);
  zi_ctx::Window w;
  w.ptr.resize(c->world);
  int dev_save = 0;
  ZI_CUDA(cudaGetDevice(&dev_save), "cudaGetDevice");
  ZI_CUDA(cudaSetDevice(c->device), "cudaSetDevice");
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) {
      w.ptr[r] = static_cast<uint8_t*>(local);
      continue;
    }
    void* base = nullptr;
    const int st = open_mapping(c, handles + (size_t)r * 64, &base);
    if (st != ZI_OK) {
      cudaSetDevice(dev_save);
      return st;
    }
    w.ptr[r] = static_cast<uint8_t*>(base) + offsets[r];
  }
  ZI_CUDA(cudaSetDevice(dev_save), "cudaSetDevice");
  c->windows.push_back(std::move(w));
  *win = (int)c->windows.size() - 1;
  return ZI_OK;
}

int zi_ctx_window_ptrs(zi_ctx* c, int win, void** ptrs) {
  ZI_CHECK_ARG(c && ptrs, "zi_ctx_window_ptrs: NULL argument");
  std::lock_guard<std::mutex> g(c->mu);
  ZI_CHECK_ARG(win >= 0 && win < (int)c->windows.size(), "zi_ctx_window_ptrs: bad window %d", win);
  for (int r = 0; r < c->world; ++r) ptrs[r] = c->windows[win].ptr[r];
  return ZI_OK;
}

int zi_ctx_allgather(zi_ctx* c, int win, size_t offset_bytes, size_t shard_elems, int dtype,
                     void* full, size_t full_elems, int use_copy_engine, void* stream) {
  ZI_CHECK_ARG(c != nullptr, "zi_ctx_allgather: NULL ctx");
  const size_t eb = dtype == ZI_DT_F32 ? 4 : dtype == ZI_DT_F64 ? 8
                  : (dtype == ZI_DT_F16 || dtype == ZI_DT_BF16) ? 2 : 0;
  ZI_CHECK_ARG(eb != 0, "zi_ctx_allgather: bad dtype %d", dtype);
  std::vector<const void*> src(c->world);
  {
    std::lock_guard<std::mutex> g(c->mu);
    ZI_CHECK_ARG(win >= 0 && win < (int)c->windows.size(), "zi_ctx_allgather: bad window %d", win);
    for (int r = 0; r < c->world; ++r) src[r] = c->windows[win].ptr[r] + offset_bytes;
  }
  return zi_allgather(src.data(), c->world, shard_elems, eb, full, full_elems, use_copy_engine,
                      stream);
}

int zi_ctx_reduce_scatter_cast(zi_ctx* c, int win, size_t offset_bytes, size_t contrib_len,
                               size_t shard_elems, float scale, int half_kind, float* shard_out,
                               void* stream) {
  ZI_CHECK_ARG(c != nullptr, "zi_ctx_reduce_scatter_cast: NULL ctx");
  std::vector<const void*> src(c->world);
  {
    std::lock_guard<std::mutex> g(c->mu);
    ZI_CHECK_ARG(win >= 0 && win < (int)c->windows.size(),
                 "zi_ctx_reduce_scatter_cast: bad window %d", win);
    for (int r = 0; r < c->world; ++r) src[r] = c->windows[win].ptr[r] + offset_bytes;
  }
  // rank order = fold order: bit-identical to the oracle's sequential sum
  return zi_reduce_scatter_cast(src.data(), c->world, (size_t)c->rank * shard_elems, shard_elems,
                                contrib_len, scale, half_kind, shard_out, stream);
}

int zi_ctx_barrier(zi_ctx* c, int flags_win, void* stream) {
  ZI_CHECK_ARG(c != nullptr, "zi_ctx_barrier: NULL ctx");
  std::vector<uint32_t*> f(c->world);
  {
    std::lock_guard<std::mutex> g(c->mu);
    ZI_CHECK_ARG(flags_win >= 0 && flags_win < (int)c->windows.size(),
                 "zi_ctx_barrier: bad window %d", flags_win);
    auto& w = c->windows[flags_win];
    for (int r = 0; r < c->world; ++r) f[r] = reinterpret_cast<uint32_t*>(w.ptr[r]);
  }
  // the epoch lives on the device (one counter per window): CUDA-graph replays of a
  // captured barrier advance it like eager calls do
  return zi_barrier_dev(f.data(), c->world, c->rank, c->epochs + flags_win, stream);
}

int zi_ctx_barrier_value(zi_ctx* c, int flags_win, int parity, void* stream) {
  ZI_CHECK_ARG(c != nullptr, "zi_ctx_barrier_value: NULL ctx");
  ZI_CHECK_ARG(parity == 0 || parity == 1, "zi_ctx_barrier_value: parity must be 0 or 1");
  const int st = load_memops();
  if (st != ZI_OK) return st;
  std::vector<uint8_t*> f(c->world);
  {
    std::lock_guard<std::mutex> g(c->mu);
    ZI_CHECK_ARG(flags_win >= 0 && flags_win < (int)c->windows.size(),
                 "zi_ctx_barrier_value: bad window %d", flags_win);
    for (int r = 0; r < c->world; ++r) f[r] = c->windows[flags_win].ptr[r];
  }
  CUstream s = reinterpret_cast<CUstream>(stream);
  const size_t set = (size_t)parity * c->world * 4;   // this barrier's slot set
  auto fail = [](const char* what, CUresult e) {
    zi::set_error("%s failed (%d)", what, (int)e);
    return ZI_ECUDA;
  };
  // arrive: 1 into our slot of every peer's set (the default write is preceded by a
  // memory fence: this stream's earlier writes are visible to the peer first) ...
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    const CUresult e = g_write32(s, reinterpret_cast<CUdeviceptr>(f[r] + set + 4 * (size_t)c->rank),
                                 1u, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (e != CUDA_SUCCESS) return fail("cuStreamWriteValue32", e);
  }
  // ... wait for every peer's arrival in our set, then reset it. A peer can run at most
  // one barrier ahead (it needs our arrival to pass this one), and that barrier uses the
  // other set; it writes this set again only after our next arrival, which is fenced
  // behind these resets.
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    const CUdeviceptr slot = reinterpret_cast<CUdeviceptr>(f[c->rank] + set + 4 * (size_t)r);
    CUresult e = g_wait32(s, slot, 1u, CU_STREAM_WAIT_VALUE_EQ);
    if (e != CUDA_SUCCESS) return fail("cuStreamWaitValue32", e);
    e = g_write32(s, slot, 0u, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (e != CUDA_SUCCESS) return fail("cuStreamWriteValue32", e);
  }
  return ZI_OK;
}

}  // extern "C"
