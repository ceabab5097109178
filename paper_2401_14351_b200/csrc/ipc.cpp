// Cross-process tensor handles:
// the model manager exports each loaded partition's device base with a CUDA IPC handle;
// the inference process maps it and sets every tensor pointer to base + offset.
#include <cuda.h>

#include <map>

#include "runtime.hpp"

namespace sllm {

using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_range range_fn() {
  static PFN_range fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_range>(p);
    cudaGetLastError();
  });
  return fn;
}

static std::mutex g_ipc_mu;
struct Mapping {
  void* base;
  int refs;
};
struct Opened {
  std::string key;
  int count;
};
static std::map<std::string, Mapping> g_maps;  // handle bytes + device -> mapping (one per allocation)
static std::map<void*, Opened> g_open;         // returned pointer -> its mapping, times returned

void ipc_export(const void* ptr, uint64_t nbytes, sllm_ipc_region* out) {
  if (!ptr || !out) fail(SLLM_E_INVALID, "null argument");
  cudaPointerAttributes at{};
  SLLM_CUDA(cudaPointerGetAttributes(&at, ptr));
  if (at.type != cudaMemoryTypeDevice) fail(SLLM_E_INVALID, "not device memory");
  SLLM_CUDA(cudaSetDevice(at.device));
  PFN_range rf = range_fn();
  if (!rf) fail(SLLM_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (rf(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    fail(SLLM_E_CUDA, "cuMemGetAddressRange failed");
  const uint64_t off = reinterpret_cast<uint64_t>(ptr) - (uint64_t)base;
  if (off + nbytes > size) fail(SLLM_E_CAPACITY, "region extends past its allocation");
  cudaIpcMemHandle_t h;
  SLLM_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  sllm_ipc_region r{};
  std::memcpy(r.handle, &h, sizeof h);
  r.offset = off;
  r.nbytes = nbytes;
  r.gpu = at.device;
  *out = r;
}

// Several regions may live in one allocation (e.g. partitions carved from one caching-
// allocator segment): the allocation is mapped once and reference counted.
void* ipc_open(const sllm_ipc_region* r) {
  if (!r) fail(SLLM_E_INVALID, "null region");
  SLLM_CUDA(cudaSetDevice(r->gpu));
  std::string key(reinterpret_cast<const char*>(r->handle), 64);
  key.append(reinterpret_cast<const char*>(&r->gpu), sizeof r->gpu);  // mapped per importing device
  std::lock_guard<std::mutex> g(g_ipc_mu);
  auto it = g_maps.find(key);
  if (it == g_maps.end()) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, r->handle, sizeof h);
    void* base = nullptr;
    SLLM_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    it = g_maps.emplace(key, Mapping{base, 0}).first;
  }
  it->second.refs++;
  void* p = static_cast<uint8_t*>(it->second.base) + r->offset;
  auto o = g_open.emplace(p, Opened{key, 0}).first;  // the same region opened twice: counted
  o->second.count++;
  return p;
}

void ipc_close(void* p) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> g(g_ipc_mu);
    auto it = g_open.find(p);
    if (it == g_open.end()) fail(SLLM_E_INVALID, "pointer was not returned by sllm_ipc_open");
    auto m = g_maps.find(it->second.key);
    if (--it->second.count == 0) g_open.erase(it);
    if (--m->second.refs > 0) return;
    base = m->second.base;
    g_maps.erase(m);
  }
  SLLM_CUDA(cudaIpcCloseMemHandle(base));
}

}  // namespace sllm
