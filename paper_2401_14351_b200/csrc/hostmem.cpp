// Pinned host memory -- the DRAM tier of the multi-tier loader (PAPER.md P:578-579
// "fixed-size memory chunks", P:588 / P:692 "pinned memory ... DMA without involving
// CPU").  Buffers are anonymous mappings (2 MiB transparent huge pages when available),
// placed on the GPU's NUMA node when the host has several (mbind via syscall; the image
// has no libnuma), first-touched by several threads, then page-locked and mapped into
// every device's address space with cudaHostRegister(Mapped | Portable) so they serve
// both the copy engine and the zero-copy kernels.  Falls back to cudaHostAlloc.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <map>

#include "runtime.hpp"

namespace sllm {

struct HostAlloc {
  uint64_t bytes;
  bool mmapped;     // true: mmap + cudaHostRegister; false: cudaHostAlloc
};
static std::mutex g_host_mu;
static std::map<void*, HostAlloc> g_host;

static void parallel_touch(uint8_t* p, uint64_t bytes, int node) {
  const uint64_t piece = 64ull << 20;
  uint64_t n = ceil_div(bytes, piece);
  int threads = (int)std::min<uint64_t>(n, (uint64_t)default_threads());
  std::vector<std::thread> th;
  std::atomic<uint64_t> next{0};
  auto body = [&] {
    bind_thread_to_node(node);  // first touch from the node the pages are bound to
    for (uint64_t i; (i = next.fetch_add(1)) < n;) {
      uint64_t lo = i * piece, len = std::min(piece, bytes - lo);
      std::memset(p + lo, 0, len);
    }
  };
  for (int t = 0; t < threads; ++t) th.emplace_back(body);  // (the caller's own affinity stays)
  for (auto& t : th) t.join();
}

void* host_alloc(uint64_t bytes, int gpu) {
  if (bytes == 0) fail(SLLM_E_INVALID, "zero-byte host allocation");
  const uint64_t len = align_up(bytes, 2ull << 20);
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p != MAP_FAILED) {
    madvise(p, len, MADV_HUGEPAGE);
    int node = -1;
    if (gpu >= 0 && numa_nodes() > 1) {
      node = gpu_numa_node(gpu);
      if (node >= 0 && node < 64) {
        unsigned long mask = 1ul << node;
        syscall(SYS_mbind, p, len, 2 /*MPOL_BIND*/, &mask, 64, 0);
      }
    }
    parallel_touch(static_cast<uint8_t*>(p), len, node);
    cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e == cudaSuccess) {
      std::lock_guard<std::mutex> g(g_host_mu);
      g_host[p] = HostAlloc{len, true};
      return p;
    }
    cudaGetLastError();
    munmap(p, len);
  }
  void* q = nullptr;
  SLLM_CUDA(cudaHostAlloc(&q, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  std::lock_guard<std::mutex> g(g_host_mu);
  g_host[q] = HostAlloc{bytes, false};
  return q;
}

void host_free(void* p) {
  if (!p) return;
  HostAlloc a{};
  {
    std::lock_guard<std::mutex> g(g_host_mu);
    auto it = g_host.find(p);
    if (it == g_host.end()) fail(SLLM_E_INVALID, "pointer was not returned by sllm_host_alloc");
    a = it->second;
    g_host.erase(it);
  }
  if (a.mmapped) {
    cudaHostUnregister(p);
    munmap(p, a.bytes);
  } else {
    cudaFreeHost(p);
  }
}

}  // namespace sllm
