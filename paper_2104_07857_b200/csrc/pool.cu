// Native staging-buffer pool and the offload engine's named transfer calls.
//
// zi_pool_* is the BufferPool of the reference tier store (store.py:81-123):
// a fixed set of equally sized transfer buffers allocated once, handed out
// LIFO; acquire blocks (counting `waits`) or fails with ZI_EEXHAUSTED
// (PoolExhausted); release refuses foreign indices and over-release. Here
// the buffers are pinned (cudaHostAlloc) so staged copies run on the copy
// engines; pinned = 0 gives pageable malloc buffers for hosts without a GPU.
// The blocking wait happens in C with the caller's GIL released (ctypes), so
// store worker threads park here, not in Python.
//
// zi_h2d_async / zi_d2h_async are the cg / grad-offload lanes of SURVEY §8(b):
// one cudaMemcpyAsync on the caller's stream plus an optional completion
// event (the IoTicket analog, store.py:126-153).
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace zi {

struct Pool {
  size_t bytes = 0;
  int count = 0;
  bool blocking = true;
  bool pinned = true;
  std::vector<void*> bufs;
  std::vector<int> free_list;   // LIFO, as the reference's list.pop()
  uint64_t waits = 0;
  std::mutex mu;
  std::condition_variable cv;
};

static void free_buffers(Pool* p) {
  for (void* b : p->bufs) {
    if (!b) continue;
    if (p->pinned) cudaFreeHost(b);
    else std::free(b);
  }
  p->bufs.clear();
}

}  // namespace zi

extern "C" {

int zi_pool_create(size_t buffer_bytes, int buffer_count, int blocking, int pinned, void** pool) {
  ZI_CHECK_ARG(pool != nullptr, "zi_pool_create: pool is NULL");
  *pool = nullptr;
  ZI_CHECK_ARG(buffer_bytes >= 1 && buffer_count >= 1,
               "buffer size and count must be >= 1");
  auto* p = new zi::Pool();
  p->bytes = buffer_bytes;
  p->count = buffer_count;
  p->blocking = blocking != 0;
  p->pinned = pinned != 0;
  p->bufs.assign(buffer_count, nullptr);
  for (int i = 0; i < buffer_count; ++i) {
    if (p->pinned) {
      cudaError_t e = cudaHostAlloc(&p->bufs[i], buffer_bytes, cudaHostAllocPortable);
      if (e != cudaSuccess) {
        int st = zi::cuda_status(e, "zi_pool_create: cudaHostAlloc");
        zi::free_buffers(p);
        delete p;
        return st;
      }
    } else {
      // page-aligned (O_DIRECT file I/O into pool buffers needs 4 KiB alignment)
      p->bufs[i] = std::aligned_alloc(4096, (buffer_bytes + 4095) / 4096 * 4096);
      if (!p->bufs[i]) {
        zi::set_error("zi_pool_create: malloc of %zu bytes failed", buffer_bytes);
        zi::free_buffers(p);
        delete p;
        return ZI_ECAPACITY;
      }
    }
    p->free_list.push_back(i);
  }
  *pool = p;
  return ZI_OK;
}

int zi_pool_destroy(void* pool) {
  if (!pool) return ZI_OK;
  auto* p = static_cast<zi::Pool*>(pool);
  zi::free_buffers(p);
  delete p;
  return ZI_OK;
}

int zi_pool_buffer(void* pool, int index, void** ptr) {
  ZI_CHECK_ARG(pool && ptr, "zi_pool_buffer: NULL argument");
  auto* p = static_cast<zi::Pool*>(pool);
  ZI_CHECK_ARG(index >= 0 && index < p->count, "buffer does not belong to this pool");
  *ptr = p->bufs[index];
  return ZI_OK;
}

int zi_pool_acquire(void* pool, int* index) {
  ZI_CHECK_ARG(pool && index, "zi_pool_acquire: NULL argument");
  auto* p = static_cast<zi::Pool*>(pool);
  std::unique_lock<std::mutex> lk(p->mu);
  if (p->free_list.empty()) {
    if (!p->blocking) {
      zi::set_error("all transfer buffers in use");
      return ZI_EEXHAUSTED;
    }
    p->waits += 1;
    p->cv.wait(lk, [p] { return !p->free_list.empty(); });
  }
  *index = p->free_list.back();
  p->free_list.pop_back();
  return ZI_OK;
}

int zi_pool_release(void* pool, int index) {
  ZI_CHECK_ARG(pool != nullptr, "zi_pool_release: NULL pool");
  auto* p = static_cast<zi::Pool*>(pool);
  ZI_CHECK_ARG(index >= 0 && index < p->count, "buffer does not belong to this pool");
  {
    std::lock_guard<std::mutex> lk(p->mu);
    if ((int)p->free_list.size() >= p->count) {
      zi::set_error("pool over-released");
      return ZI_EINVAL;
    }
    p->free_list.push_back(index);
  }
  p->cv.notify_one();
  return ZI_OK;
}

int zi_pool_stats(void* pool, int* free_count, uint64_t* waits) {
  ZI_CHECK_ARG(pool != nullptr, "zi_pool_stats: NULL pool");
  auto* p = static_cast<zi::Pool*>(pool);
  std::lock_guard<std::mutex> lk(p->mu);
  if (free_count) *free_count = (int)p->free_list.size();
  if (waits) *waits = p->waits;
  return ZI_OK;
}

static int copy_then_record(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                            void* stream, void* event, const char* what) {
  ZI_CHECK_ARG(bytes == 0 || (dst && src), "%s: NULL pointer", what);
  cudaStream_t s = (cudaStream_t)stream;
  if (bytes) ZI_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, s), what);
  if (event) ZI_CUDA(cudaEventRecord((cudaEvent_t)event, s), "cudaEventRecord");
  return ZI_OK;
}

int zi_h2d_async(void* dst, const void* src, size_t bytes, void* stream, void* event) {
  return copy_then_record(dst, src, bytes, cudaMemcpyHostToDevice, stream, event, "zi_h2d_async");
}

int zi_d2h_async(void* dst, const void* src, size_t bytes, void* stream, void* event) {
  return copy_then_record(dst, src, bytes, cudaMemcpyDeviceToHost, stream, event, "zi_d2h_async");
}

}  // extern "C"
