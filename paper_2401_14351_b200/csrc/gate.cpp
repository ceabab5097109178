// Stream gates: let a caller's stream wait for a load that is issued asynchronously by a
// worker thread (the inference process sets tensor pointers before the data has
// arrived; it synchronizes with the loader).  sllm_load_start enqueues, on the
// caller's stream and before returning, a wait for a 32-bit flag in pinned host memory
// to reach a fresh value; the load's last stream operation writes that value
// (cuStreamWriteValue32), and the worker thread also writes it from the host when it
// finishes or fails, so the caller's stream can never be left waiting.  Values only grow
// per slot, so a recycled slot never satisfies a stale wait early.
#include <cuda.h>

#include "runtime.hpp"

namespace sllm {

using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static constexpr int kSlots = 4096;
static std::mutex g_gate_mu;
static uint32_t* g_flags = nullptr;
static std::vector<int> g_free;
static std::vector<uint32_t> g_gen;
static PFN_wait32 g_wait = nullptr;
static PFN_write32 g_write = nullptr;
static bool g_init = false;

static void gate_init() {
  if (g_init) return;
  void* p = nullptr;
  SLLM_CUDA(cudaHostAlloc(&p, kSlots * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(p, 0, kSlots * sizeof(uint32_t));
  g_flags = static_cast<uint32_t*>(p);
  g_gen.assign(kSlots, 0);
  for (int i = kSlots - 1; i >= 0; --i) g_free.push_back(i);
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_wait = reinterpret_cast<PFN_wait32>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_write = reinterpret_cast<PFN_write32>(fn);
  cudaGetLastError();
  g_init = true;
}

Gate gate_acquire() {
  std::lock_guard<std::mutex> g(g_gate_mu);
  gate_init();
  if (g_free.empty()) fail(SLLM_E_CAPACITY, "too many loads in flight (stream gates exhausted)");
  Gate gt;
  gt.slot = g_free.back();
  g_free.pop_back();
  gt.value = ++g_gen[gt.slot];
  if (gt.value == 0) gt.value = ++g_gen[gt.slot];
  gt.host = g_flags + gt.slot;
  void* d = nullptr;
  SLLM_CUDA(cudaHostGetDevicePointer(&d, gt.host, 0));
  gt.dev = reinterpret_cast<uint64_t>(d);
  return gt;
}

void gate_release(const Gate& gt) {
  if (gt.slot < 0) return;
  std::lock_guard<std::mutex> g(g_gate_mu);
  g_free.push_back(gt.slot);
}

void gate_wait(cudaStream_t s, const Gate& gt) {
  if (g_wait) {
    CUresult r = g_wait(reinterpret_cast<CUstream>(s), (CUdeviceptr)gt.dev, gt.value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r == CUDA_SUCCESS) return;
  }
  SLLM_CUDA(launch_gate_spin(reinterpret_cast<const uint32_t*>(gt.dev), gt.value, s));
}

void gate_open_device(cudaStream_t s, const Gate& gt) {
  if (g_write && g_write(reinterpret_cast<CUstream>(s), (CUdeviceptr)gt.dev, gt.value, 0) == CUDA_SUCCESS) return;
  // fallback: the host opens the gate when the worker finishes (gate_open_host)
}

void gate_open_host(const Gate& gt) {
  if (gt.slot < 0) return;
  __atomic_store_n(gt.host, gt.value, __ATOMIC_RELEASE);
}

}  // namespace sllm
