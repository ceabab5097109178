// File tier of the multi-tier loader (§Multi-Tier Loading
// Subsystem P:572-602): SSD -> pinned DRAM -> GPU as one pipeline.
//
//   P:587  "direct file access (e.g. O_DIRECT) ... directly reading data into user space"
//   P:578  "fixed-size memory chunks" with "APIs for the allocation and deallocation"
//   P:601  "multiple I/O threads for reading data within each storage tier"
//   P:602  "I/O threads read storage chunks and enqueue their indices (offset and size)
//           for the I/O threads in the next tier"
//
// Per partition a ring of R pinned slots (one load window each, from a process-wide
// pinned chunk pool) sits between `io_threads` O_DIRECT readers and the GPU worker: a
// reader fills slot w % R once the GPU has finished consuming window w - R (CUDA event),
// then publishes "window w ready"; the worker issues that window's copy / kernel from the
// slot and records the slot's release event.  Storage reads, PCIe transfers and
// verification of different windows overlap; no tier waits for a whole partition.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <condition_variable>
#include <map>

#include "runtime.hpp"

namespace sllm {

void* host_alloc(uint64_t bytes, int gpu);

// ---- process-wide pinned chunk pool -------------------------------------
static std::mutex g_pool_mu;
static std::map<uint64_t, std::vector<void*>> g_pool_free;  // slot size -> free slots

static std::vector<void*> pool_acquire(size_t n, uint64_t bytes, int gpu) {
  std::vector<void*> out;
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto& fl = g_pool_free[bytes];
    while (out.size() < n && !fl.empty()) {
      out.push_back(fl.back());
      fl.pop_back();
    }
  }
  while (out.size() < n) out.push_back(host_alloc(bytes, gpu));  // grows once, then reused
  return out;
}

static void pool_release(const std::vector<void*>& slots, uint64_t bytes) {
  std::lock_guard<std::mutex> g(g_pool_mu);
  auto& fl = g_pool_free[bytes];
  fl.insert(fl.end(), slots.begin(), slots.end());
}

struct FileSource {
  std::string path;
  uint64_t base = 0, length = 0, window = 0, nwin = 0;  // window w = file bytes [base + w*window, ...) < length
  int R = 0;
  int fd_direct = -1, fd_buf = -1;
  std::vector<void*> slots;
  std::vector<cudaEvent_t> slot_ev;
  std::vector<uint64_t> ready;     // per slot: 1 + index of the window it holds (0 = none)
  std::vector<uint64_t> consumed;  // per slot: 1 + index of the last window the GPU consumed
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<uint64_t> next{0};
  std::atomic<bool> stop{false};
  std::string error;
  std::vector<std::thread> io;
  uint64_t bytes_read = 0;
  uint64_t wait_ns = 0;  // time the GPU worker spent blocked on storage (a per-tier time)
};

static void read_window(FileSource& f, uint64_t w, uint8_t* dst) {
  const uint64_t lo = f.base + w * f.window, hi = std::min(lo + f.window, f.length);
  const uint64_t direct_end = f.fd_direct >= 0 ? f.length / 4096 * 4096 : 0;
  uint64_t pos = lo;
  while (pos < hi) {
    const bool direct = pos + 4096 <= direct_end && (pos % 4096) == 0;
    const uint64_t end = direct ? std::min(hi, direct_end) : hi;
    ssize_t r = ::pread(direct ? f.fd_direct : f.fd_buf, dst + (pos - lo), end - pos, (off_t)pos);
    if (r <= 0) fail(SLLM_E_IO, "read failed on " + f.path + " at " + std::to_string(pos));
    pos += (uint64_t)r;
  }
}

static void io_main(FileSource* f, int gpu) {
  try {
    cudaSetDevice(gpu);
    bind_thread_to_gpu(gpu);  // readers fill slots on the GPU's node
    for (;;) {
      const uint64_t w = f->next.fetch_add(1);
      if (w >= f->nwin || f->stop) return;
      const int s = (int)(w % (uint64_t)f->R);
      if (w >= (uint64_t)f->R) {  // wait until the GPU has consumed window w - R from this slot
        std::unique_lock<std::mutex> lk(f->mu);
        f->cv.wait(lk, [&] { return f->stop || f->consumed[s] >= w - f->R + 1; });
        if (f->stop) return;
        lk.unlock();
        SLLM_CUDA(cudaEventSynchronize(f->slot_ev[s]));
      }
      read_window(*f, w, static_cast<uint8_t*>(f->slots[s]));
      {
        std::lock_guard<std::mutex> g(f->mu);
        f->ready[s] = w + 1;
        f->bytes_read += std::min(f->window, f->length - f->base - w * f->window);
      }
      f->cv.notify_all();
    }
  } catch (const std::exception& e) {
    std::lock_guard<std::mutex> g(f->mu);
    if (f->error.empty()) f->error = e.what();
    f->stop = true;
    f->cv.notify_all();
  }
}

void FileSourceDeleter::operator()(FileSource* f) const {
  if (!f) return;
  {
    std::lock_guard<std::mutex> g(f->mu);
    f->stop = true;
  }
  f->cv.notify_all();
  for (auto& t : f->io)
    if (t.joinable()) t.join();
  for (auto& e : f->slot_ev)
    if (e) {
      cudaEventSynchronize(e);
      cudaEventDestroy(e);
    }
  if (!f->slots.empty()) pool_release(f->slots, f->window);
  if (f->fd_direct >= 0) ::close(f->fd_direct);
  if (f->fd_buf >= 0) ::close(f->fd_buf);
  delete f;
}

FileSourcePtr file_source_open(const std::string& path, uint64_t lo, uint64_t length, uint64_t window, int io_threads,
                               int gpu) {
  FileSourcePtr f(new FileSource);
  f->path = path;
  f->base = lo;
  f->length = length;
  f->window = window;
  f->nwin = length > lo ? ceil_div(length - lo, window) : 0;
  f->fd_buf = ::open(path.c_str(), O_RDONLY);
  if (f->fd_buf < 0) fail(SLLM_E_IO, "cannot open " + path + ": " + strerror(errno));
  struct stat st;
  fstat(f->fd_buf, &st);
  if ((uint64_t)st.st_size < length) fail(SLLM_E_IO, path + " is shorter than its partition");
  f->fd_direct = ::open(path.c_str(), O_RDONLY | O_DIRECT);  // -1: buffered reads only
  if (io_threads <= 0) io_threads = 4;                        // 4 cores saturate
  f->R = (int)std::min<uint64_t>(std::max<uint64_t>(f->nwin, 1), (uint64_t)io_threads + 2);
  f->slots = pool_acquire((size_t)f->R, window, gpu);
  f->slot_ev.resize(f->R);
  for (auto& e : f->slot_ev) SLLM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  f->ready.assign(f->R, 0);
  f->consumed.assign(f->R, 0);
  const int n = (int)std::min<uint64_t>((uint64_t)io_threads, std::max<uint64_t>(f->nwin, 1));
  for (int t = 0; t < n; ++t) f->io.emplace_back(io_main, f.get(), gpu);
  return f;
}

const uint8_t* file_source_window(FileSource& f, uint64_t w) {
  const int s = (int)(w % (uint64_t)f.R);
  std::unique_lock<std::mutex> lk(f.mu);
  if (f.error.empty() && f.ready[s] != w + 1) {
    const auto t0 = std::chrono::steady_clock::now();
    f.cv.wait(lk, [&] { return !f.error.empty() || f.ready[s] == w + 1; });
    f.wait_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                     .count();
  }
  if (!f.error.empty()) fail(SLLM_E_IO, f.error);
  return static_cast<const uint8_t*>(f.slots[s]);
}

void file_source_consumed(FileSource& f, uint64_t w, cudaStream_t st) {
  const int s = (int)(w % (uint64_t)f.R);
  SLLM_CUDA(cudaEventRecord(f.slot_ev[s], st));
  {
    std::lock_guard<std::mutex> g(f.mu);
    f.consumed[s] = w + 1;
  }
  f.cv.notify_all();
}

uint64_t file_source_bytes(FileSource& f) {
  std::lock_guard<std::mutex> g(f.mu);
  return f.bytes_read;
}

uint64_t file_source_wait_ns(FileSource& f) {
  std::lock_guard<std::mutex> g(f.mu);
  return f.wait_ns;
}

}  // namespace sllm
