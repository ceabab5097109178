// File tier: convert() writes <dir>/part_<device>.bin + <dir>/index.bin;
// host_read_partition() is the SSD -> pinned-DRAM stage of the multi-tier pipeline
// ("direct file access (e.g. O_DIRECT)", "multiple I/O threads ...
// within each storage tier", P:680 chunked reads).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <thread>

#include "common.hpp"

namespace sllm {

static std::string part_path(const std::string& dir, int32_t device) {
  return dir + "/part_" + std::to_string(device) + ".bin";
}

static void write_all(const std::string& path, const uint8_t* p, uint64_t n) {
  int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) fail(SLLM_E_IO, "cannot create " + path + ": " + strerror(errno));
  uint64_t done = 0;
  while (done < n) {
    ssize_t w = ::pwrite(fd, p + done, std::min<uint64_t>(n - done, 1ull << 30), (off_t)done);
    if (w <= 0) {
      ::close(fd);
      fail(SLLM_E_IO, "write failed on " + path);
    }
    done += (uint64_t)w;
  }
  if (::close(fd) != 0) fail(SLLM_E_IO, "close failed on " + path);
}

void convert_files(const sllm_src_tensor* t, size_t n, uint64_t align, uint64_t block, const char* model_id,
                   const char* out_dir) {
  if (!out_dir) fail(SLLM_E_INVALID, "null output directory");
  std::unique_ptr<sllm_index> idx(plan(t, n, align, block, model_id));
  ::mkdir(out_dir, 0755);
  std::vector<std::unique_ptr<uint8_t, void (*)(void*)>> bufs;
  std::vector<void*> ptrs;
  for (auto& pr : idx->parts) {
    void* p = nullptr;
    if (posix_memalign(&p, 4096, pr.length) != 0) fail(SLLM_E_NOMEM, "cannot allocate partition buffer");
    bufs.emplace_back(static_cast<uint8_t*>(p), free);
    ptrs.push_back(p);
  }
  convert_into(t, n, idx.get(), ptrs.data());
  for (size_t p = 0; p < idx->parts.size(); ++p)
    write_all(part_path(out_dir, idx->parts[p].device), bufs[p].get(), idx->parts[p].length);
  std::vector<uint8_t> blob = serialize(*idx);
  write_all(std::string(out_dir) + "/index.bin", blob.data(), blob.size());
}

std::vector<uint8_t> read_file(const char* path) {
  if (!path) fail(SLLM_E_INVALID, "null path");
  int fd = ::open(path, O_RDONLY);
  if (fd < 0) fail(SLLM_E_IO, std::string("cannot open ") + path + ": " + strerror(errno));
  struct stat st;
  if (fstat(fd, &st) != 0) {
    ::close(fd);
    fail(SLLM_E_IO, std::string("cannot stat ") + path);
  }
  std::vector<uint8_t> b((size_t)st.st_size);
  size_t done = 0;
  while (done < b.size()) {
    ssize_t r = ::pread(fd, b.data() + done, b.size() - done, (off_t)done);
    if (r <= 0) {
      ::close(fd);
      fail(SLLM_E_IO, std::string("read failed on ") + path);
    }
    done += (size_t)r;
  }
  ::close(fd);
  return b;
}

// File -> pinned DRAM with `threads` readers, each pulling 16 MiB chunk indices from a
// shared counter (the paper's per-tier task queue).  O_DIRECT is used when the
// destination, the length and the chunk size are all 4 KiB aligned (bypassing the page
// cache); the unaligned tail (if any) is read through a buffered descriptor.
void read_partition(const char* dir, const sllm_index* idx, size_t p, void* dst, int threads) {
  if (!dir || !idx || !dst) fail(SLLM_E_INVALID, "null argument");
  if (p >= idx->parts.size()) fail(SLLM_E_LOOKUP, "partition index out of range");
  const PartRec& pr = idx->parts[p];
  std::string path = part_path(dir, pr.device);
  int fd_buf = ::open(path.c_str(), O_RDONLY);
  if (fd_buf < 0) fail(SLLM_E_IO, "cannot open " + path + ": " + strerror(errno));
  struct stat st;
  fstat(fd_buf, &st);
  if ((uint64_t)st.st_size < pr.length) {
    ::close(fd_buf);
    fail(SLLM_E_IO, path + " is shorter than the partition");
  }
  const uint64_t kChunk = 16ull << 20;
  bool direct_ok = (reinterpret_cast<uintptr_t>(dst) % 4096) == 0;
  int fd_dir = direct_ok ? ::open(path.c_str(), O_RDONLY | O_DIRECT) : -1;
  const uint64_t direct_len = fd_dir >= 0 ? pr.length / 4096 * 4096 : 0;
  uint64_t nch = ceil_div(pr.length, kChunk);
  if (threads <= 0) threads = 4;  // "with 4 CPU cores ... maximum bandwidth"
  threads = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(nch, 1));
  std::atomic<uint64_t> next{0};
  std::atomic<int> err{0};
  const int node = page_node(dst);  // readers run on the node of the destination pages
  auto body = [&] {
    bind_thread_to_node(node);
    for (uint64_t k; (k = next.fetch_add(1)) < nch && !err.load();) {
      uint64_t lo = k * kChunk, hi = std::min(lo + kChunk, pr.length);
      while (lo < hi) {
        bool use_direct = lo + 4096 <= direct_len;
        uint64_t end = use_direct ? std::min(hi, direct_len) : hi;
        ssize_t r = ::pread(use_direct ? fd_dir : fd_buf, static_cast<uint8_t*>(dst) + lo, end - lo, (off_t)lo);
        if (r <= 0) {
          err = 1;
          return;
        }
        lo += (uint64_t)r;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t) th.emplace_back(body);  // (never re-binds the caller)
  for (auto& t : th) t.join();
  if (fd_dir >= 0) ::close(fd_dir);
  ::close(fd_buf);
  if (err) fail(SLLM_E_IO, "read failed on " + path);
}

}  // namespace sllm
