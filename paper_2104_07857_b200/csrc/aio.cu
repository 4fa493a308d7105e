// Native asynchronous file I/O for the NVMe tier (the DeepNVMe analog of PAPER §6.2 and
// the reference store's NVMe worker pool, store.py:442-560): a pool of worker threads
// moving byte ranges of .shard files between the file and pinned host buffers.
//
// A range [b0, b1) of a file is split at the 4 KiB block grid: the whole blocks in the
// middle go through an O_DIRECT descriptor (no page cache, DMA straight into the pinned
// buffer), the partial blocks at either edge through a buffered descriptor. The caller
// places the range's bytes at buf + (b0 % 4096), so the middle part is 4 KiB-aligned in
// memory as O_DIRECT requires; cudaHostAlloc buffers are page-aligned. Middle parts are
// cut into <= 8 MiB pieces served by all workers in parallel. Two writers may share an
// edge block (adjacent chunks): both write it through the page cache, which merges
// them; a later O_DIRECT read of that block sees the merged data (Linux writes dirty
// pages back before a direct read of the range).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace zi {

constexpr size_t kBlock = 4096, kPiece = 8u << 20;

struct AioReq {
  int remaining = 0;
  int err = 0;             // first errno (or -1 for a short read)
};

struct AioTask {
  uint64_t id;
  int fd;
  bool write;
  uint8_t* buf;
  size_t off, len;
};

struct Aio {
  std::mutex mu;
  std::condition_variable cv_task, cv_done;
  std::deque<AioTask> tasks;
  std::unordered_map<uint64_t, AioReq> reqs;
  std::vector<std::thread> workers;
  uint64_t next = 1;
  bool stop = false;
};

static void aio_worker(Aio* a) {
  for (;;) {
    AioTask t;
    {
      std::unique_lock<std::mutex> lk(a->mu);
      a->cv_task.wait(lk, [a] { return a->stop || !a->tasks.empty(); });
      if (a->stop && a->tasks.empty()) return;
      t = a->tasks.front();
      a->tasks.pop_front();
    }
    int err = 0;
    size_t done = 0;
    while (done < t.len) {
      const ssize_t r = t.write ? pwrite(t.fd, t.buf + done, t.len - done, t.off + done)
                                : pread(t.fd, t.buf + done, t.len - done, t.off + done);
      if (r < 0) {
        if (errno == EINTR) continue;
        err = errno;
        break;
      }
      if (r == 0) {         // EOF inside a requested range: truncated shard
        err = -1;
        break;
      }
      done += (size_t)r;
    }
    {
      std::lock_guard<std::mutex> lk(a->mu);
      AioReq& q = a->reqs[t.id];
      if (err && !q.err) q.err = err;
      if (--q.remaining == 0) a->cv_done.notify_all();
    }
  }
}

}  // namespace zi

extern "C" {

int zi_aio_create(int threads, void** eng) {
  ZI_CHECK_ARG(eng && threads >= 1 && threads <= 256, "zi_aio_create: bad arguments");
  auto* a = new zi::Aio();
  for (int i = 0; i < threads; ++i) a->workers.emplace_back(zi::aio_worker, a);
  *eng = a;
  return ZI_OK;
}

int zi_aio_destroy(void* eng) {
  if (!eng) return ZI_OK;
  auto* a = static_cast<zi::Aio*>(eng);
  {
    std::lock_guard<std::mutex> lk(a->mu);
    a->stop = true;
  }
  a->cv_task.notify_all();
  for (auto& t : a->workers) t.join();
  delete a;
  return ZI_OK;
}

// Opens `path` twice: fds[0] with O_DIRECT, fds[1] buffered (create: O_CREAT, 0644).
int zi_aio_open(const char* path, int write, int create, int* fds) {
  ZI_CHECK_ARG(path && fds, "zi_aio_open: NULL argument");
  const int base = (write ? O_RDWR : O_RDONLY) | (create ? O_CREAT : 0) | O_CLOEXEC;
  const int fd_b = open(path, base, 0644);
  if (fd_b < 0) {
    zi::set_error("zi_aio_open(%s): %s", path, strerror(errno));
    return errno == ENOENT ? ZI_ENOTFOUND : ZI_EIO;
  }
  const int fd_d = open(path, (base & ~O_CREAT) | O_DIRECT);
  if (fd_d < 0) {
    const int e = errno;
    close(fd_b);
    zi::set_error("zi_aio_open(%s, O_DIRECT): %s", path, strerror(e));
    return ZI_EIO;
  }
  fds[0] = fd_d;
  fds[1] = fd_b;
  return ZI_OK;
}

int zi_aio_close(const int* fds) {
  ZI_CHECK_ARG(fds != nullptr, "zi_aio_close: NULL");
  if (fds[0] >= 0) close(fds[0]);
  if (fds[1] >= 0) close(fds[1]);
  return ZI_OK;
}

int zi_aio_truncate(const int* fds, size_t size) {
  ZI_CHECK_ARG(fds != nullptr, "zi_aio_truncate: NULL");
  if (ftruncate(fds[1], (off_t)size) != 0) {
    zi::set_error("zi_aio_truncate: %s", strerror(errno));
    return ZI_EIO;
  }
  return ZI_OK;
}

// Queue the transfer of file bytes [b0, b1) <-> buf + (b0 % 4096) .. ; returns its id.
int zi_aio_submit(void* eng, const int* fds, int write, void* buf, size_t b0, size_t b1,
                  uint64_t* id) {
  using zi::kBlock;
  ZI_CHECK_ARG(eng && fds && buf && id && b1 >= b0, "zi_aio_submit: bad arguments");
  ZI_CHECK_ARG(((uintptr_t)buf % kBlock) == 0, "zi_aio_submit: buffer must be 4 KiB aligned");
  auto* a = static_cast<zi::Aio*>(eng);
  uint8_t* base = static_cast<uint8_t*>(buf) - (b0 / kBlock) * kBlock;   // file offset o -> base + o
  std::vector<zi::AioTask> parts;
  const size_t m0 = (b0 + kBlock - 1) / kBlock * kBlock, m1 = b1 / kBlock * kBlock;
  if (m0 >= m1) {                          // inside one block, or two partial ones
    if (b1 > b0) parts.push_back({0, fds[1], write != 0, base + b0, b0, b1 - b0});
  } else {
    if (m0 > b0) parts.push_back({0, fds[1], write != 0, base + b0, b0, m0 - b0});
    for (size_t o = m0; o < m1; o += zi::kPiece) {
      const size_t n = m1 - o < zi::kPiece ? m1 - o : zi::kPiece;
      parts.push_back({0, fds[0], write != 0, base + o, o, n});
    }
    if (b1 > m1) parts.push_back({0, fds[1], write != 0, base + m1, m1, b1 - m1});
  }
  {
    std::lock_guard<std::mutex> lk(a->mu);
    const uint64_t rid = a->next++;
    a->reqs[rid].remaining = (int)parts.size();
    for (auto& p : parts) {
      p.id = rid;
      a->tasks.push_back(p);
    }
    *id = rid;
    if (parts.empty()) a->cv_done.notify_all();
  }
  a->cv_task.notify_all();
  return ZI_OK;
}

int zi_aio_wait(void* eng, uint64_t id) {
  ZI_CHECK_ARG(eng != nullptr, "zi_aio_wait: NULL engine");
  auto* a = static_cast<zi::Aio*>(eng);
  std::unique_lock<std::mutex> lk(a->mu);
  auto it = a->reqs.find(id);
  ZI_CHECK_ARG(it != a->reqs.end(), "zi_aio_wait: unknown request %llu", (unsigned long long)id);
  a->cv_done.wait(lk, [&] { return a->reqs[id].remaining == 0; });
  const int err = a->reqs[id].err;
  a->reqs.erase(id);
  if (err == -1) {
    zi::set_error("zi_aio: short read (truncated shard)");
    return ZI_EIO;
  }
  if (err) {
    zi::set_error("zi_aio: %s", strerror(err));
    return ZI_EIO;
  }
  return ZI_OK;
}

}  // extern "C"
