// Error plumbing, pinned host allocation, async copies, events and CUDA IPC.
// Host tier of the offload engine (reference BufferPool / IoTicket,
// store.py:81-153): pinned cudaHostAlloc buffers + copy-engine transfers;
// tickets are CUDA events.
#include <atomic>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace zi {

static thread_local char g_err[1024] = "";

static std::atomic<long long> g_launch_count{0};
void count_launches(int n) { g_launch_count.fetch_add(n, std::memory_order_relaxed); }

bool pdl_enabled() {   // ZI_PDL=0: plain stream serialisation (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZI_PDL");
    v = (e && atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ZI_OK;
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  if (e == cudaErrorMemoryAllocation) return ZI_ECAPACITY;
  return ZI_ECUDA;
}

}  // namespace zi

extern "C" {

long long zi_launch_count(void) { return zi::g_launch_count.load(std::memory_order_relaxed); }


const char* zi_last_error(void) { return zi::g_err; }

int zi_version(void) { return 100; }

int zi_host_alloc(size_t bytes, void** out) {
  ZI_CHECK_ARG(out != nullptr, "zi_host_alloc: out is NULL");
  *out = nullptr;
  if (bytes == 0) return ZI_OK;
  ZI_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
  return ZI_OK;
}

int zi_host_free(void* p) {
  if (!p) return ZI_OK;
  ZI_CUDA(cudaFreeHost(p), "cudaFreeHost");
  return ZI_OK;
}

int zi_memcpy_async(void* dst, const void* src, size_t bytes, int kind, void* stream) {
  if (bytes == 0) return ZI_OK;
  ZI_CHECK_ARG(dst && src, "zi_memcpy_async: NULL pointer");
  cudaMemcpyKind k;
  switch (kind) {
    case 0: k = cudaMemcpyHostToDevice; break;
    case 1: k = cudaMemcpyDeviceToHost; break;
    case 2: k = cudaMemcpyDeviceToDevice; break;
    case 3: k = cudaMemcpyDefault; break;
    default: zi::set_error("zi_memcpy_async: bad kind %d", kind); return ZI_EINVAL;
  }
  ZI_CUDA(cudaMemcpyAsync(dst, src, bytes, k, (cudaStream_t)stream), "cudaMemcpyAsync");
  return ZI_OK;
}

int zi_event_create(void** ev) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_create: NULL");
  cudaEvent_t e;
  ZI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  *ev = (void*)e;
  return ZI_OK;
}

int zi_event_create_timed(void** ev) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_create_timed: NULL");
  cudaEvent_t e;
  ZI_CUDA(cudaEventCreate(&e), "cudaEventCreate");
  *ev = (void*)e;
  return ZI_OK;
}

int zi_event_record_external(void* ev, void* stream) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_record_external: NULL event");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ZI_CUDA(cudaStreamIsCapturing((cudaStream_t)stream, &cs), "cudaStreamIsCapturing");
  if (cs == cudaStreamCaptureStatusActive)   // an external record node in the graph
    ZI_CUDA(cudaEventRecordWithFlags((cudaEvent_t)ev, (cudaStream_t)stream, cudaEventRecordExternal),
            "cudaEventRecordWithFlags(external)");
  else
    ZI_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream), "cudaEventRecord");
  return ZI_OK;
}

int zi_event_elapsed_ms(void* ev0, void* ev1, float* ms) {
  ZI_CHECK_ARG(ev0 && ev1 && ms, "zi_event_elapsed_ms: NULL");
  ZI_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)ev0, (cudaEvent_t)ev1), "cudaEventElapsedTime");
  return ZI_OK;
}

int zi_event_destroy(void* ev) {
  if (!ev) return ZI_OK;
  ZI_CUDA(cudaEventDestroy((cudaEvent_t)ev), "cudaEventDestroy");
  return ZI_OK;
}

int zi_event_record(void* ev, void* stream) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_record: NULL event");
  ZI_CUDA(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream), "cudaEventRecord");
  return ZI_OK;
}

int zi_event_query(void* ev) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_query: NULL event");
  cudaError_t e = cudaEventQuery((cudaEvent_t)ev);
  if (e == cudaSuccess) return ZI_OK;
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();
    return ZI_ENOTFOUND;
  }
  return zi::cuda_status(e, "cudaEventQuery");
}

int zi_event_sync(void* ev) {
  ZI_CHECK_ARG(ev != nullptr, "zi_event_sync: NULL event");
  ZI_CUDA(cudaEventSynchronize((cudaEvent_t)ev), "cudaEventSynchronize");
  return ZI_OK;
}

int zi_stream_wait_event(void* stream, void* ev) {
  ZI_CHECK_ARG(ev != nullptr, "zi_stream_wait_event: NULL event");
  ZI_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0), "cudaStreamWaitEvent");
  return ZI_OK;
}

int zi_device_alloc(size_t bytes, void** out) {
  ZI_CHECK_ARG(out != nullptr, "zi_device_alloc: out is NULL");
  *out = nullptr;
  if (bytes == 0) return ZI_OK;
  ZI_CUDA(cudaMalloc(out, bytes), "cudaMalloc");
  return ZI_OK;
}

int zi_device_free(void* p) {
  if (!p) return ZI_OK;
  ZI_CUDA(cudaFree(p), "cudaFree");
  return ZI_OK;
}

int zi_ipc_get_handle(void* dptr, unsigned char handle[64]) {
  ZI_CHECK_ARG(dptr && handle, "zi_ipc_get_handle: NULL");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  ZI_CUDA(cudaIpcGetMemHandle(&h, dptr), "cudaIpcGetMemHandle");
  memcpy(handle, &h, 64);
  return ZI_OK;
}

int zi_ipc_open(const unsigned char handle[64], void** dptr) {
  ZI_CHECK_ARG(dptr && handle, "zi_ipc_open: NULL");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  ZI_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return ZI_OK;
}

int zi_ipc_close(void* dptr) {
  if (!dptr) return ZI_OK;
  ZI_CUDA(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
  return ZI_OK;
}

}  // extern "C"
