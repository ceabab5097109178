// NVLink-SHARP multicast group for the replicated fan-out.
//
// The paper loads every replica of a multi-GPU model over its own PCIe link from the pinned
// pool.  With a fan-out each byte crosses PCIe once; the NVLS
// variant then lets the NVSwitch replicate it: one multicast object spans the group's GPUs,
// every GPU's replica is bound to it, and a single `multimem.st` from the loading kernel
// lands the 16-byte vector in every replica at once -- no NCCL kernels, no per-peer stores.
//
// Capability-gated at run time: creating the multicast object needs an NVSwitch fabric with
// multicast enabled (cuMulticastCreate fails on hosts without it, e.g. the 1-GPU VMs of this
// build: profiles/r01/probe_nvls.txt); sllm_comm_init_nvls then returns SLLM_E_INVALID and
// the caller keeps the P2P or NCCL fan-out.  One process drives every GPU of the group (the
// paper's model manager), so no handle export is needed.
#include <cuda.h>

#include "runtime.hpp"

namespace sllm {
namespace {

struct Drv {
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};

template <class F>
bool entry(F& f, const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  f = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry(d.GetErrorString, "cuGetErrorString") && entry(d.DeviceGet, "cuDeviceGet") &&
           entry(d.DeviceGetAttribute, "cuDeviceGetAttribute") && entry(d.MulticastCreate, "cuMulticastCreate") &&
           entry(d.MulticastAddDevice, "cuMulticastAddDevice") && entry(d.MulticastBindMem, "cuMulticastBindMem") &&
           entry(d.MulticastUnbind, "cuMulticastUnbind") &&
           entry(d.MulticastGetGranularity, "cuMulticastGetGranularity") && entry(d.MemCreate, "cuMemCreate") &&
           entry(d.MemRelease, "cuMemRelease") &&
           entry(d.MemGetAllocationGranularity, "cuMemGetAllocationGranularity") &&
           entry(d.MemAddressReserve, "cuMemAddressReserve") && entry(d.MemAddressFree, "cuMemAddressFree") &&
           entry(d.MemMap, "cuMemMap") && entry(d.MemUnmap, "cuMemUnmap") && entry(d.MemSetAccess, "cuMemSetAccess");
  });
  return d;
}

std::string cu_str(CUresult r) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return std::string(s ? s : "?") + " (" + std::to_string((int)r) + ")";
}

}  // namespace

// Owned by every comm handle of the group (shared_ptr): torn down when the last is freed.
struct NvlsGroup {
  std::vector<int> gpus;
  size_t size = 0;                         // bytes of every replica (granularity-aligned)
  CUmemGenericAllocationHandle mc = 0;     // the multicast object
  CUdeviceptr mc_va = 0;                   // its mapping (one address, every group GPU)
  std::vector<CUmemGenericAllocationHandle> mem;  // replica allocations, per GPU
  std::vector<CUdeviceptr> uva;            // replica unicast mappings, per GPU
  std::vector<uint32_t*> signal;           // per GPU: 2*R uint32 ready/done epochs (cudaMalloc)
  std::vector<bool> bound;
  ~NvlsGroup();
};

NvlsGroup::~NvlsGroup() {
  const Drv& d = drv();
  if (!d.ok) return;
  for (size_t i = 0; i < gpus.size(); ++i) {
    cudaSetDevice(gpus[i]);
    cudaDeviceSynchronize();
    if (i < signal.size() && signal[i]) cudaFree(signal[i]);
  }
  if (mc_va) {
    d.MemUnmap(mc_va, size);
    d.MemAddressFree(mc_va, size);
  }
  for (size_t i = 0; i < uva.size(); ++i)
    if (uva[i]) {
      d.MemUnmap(uva[i], size);
      d.MemAddressFree(uva[i], size);
    }
  for (size_t i = 0; i < bound.size(); ++i)
    if (bound[i]) {
      CUdevice dev;
      if (d.DeviceGet(&dev, gpus[i]) == CUDA_SUCCESS) d.MulticastUnbind(mc, dev, 0, size);
    }
  for (auto m : mem)
    if (m) d.MemRelease(m);
  if (mc) d.MemRelease(mc);
  cudaGetLastError();
}

// Build the group: multicast object over gpus[0..n-1], one replica of >= bytes per GPU bound
// to it, the multicast mapping, and per-GPU signal arrays (peer access enabled between the
// group's GPUs).  Throws SLLM_E_INVALID when the platform cannot do NVLS.
std::shared_ptr<NvlsGroup> nvls_group_create(const int32_t* gpus, int32_t n, uint64_t bytes) {
  if (!gpus || n < 1 || n > kMaxPeers + 1 || bytes == 0)
    fail(SLLM_E_INVALID, "bad NVLS group arguments (1..8 GPUs, bytes > 0)");
  const Drv& d = drv();
  if (!d.ok) fail(SLLM_E_INVALID, "NVLS: the driver has no multicast entry points");
  auto g = std::make_shared<NvlsGroup>();
  g->gpus.assign(gpus, gpus + n);
  std::vector<CUdevice> devs(n);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < i; ++k)
      if (gpus[k] == gpus[i]) fail(SLLM_E_INVALID, "NVLS: a GPU appears twice in the group");
    SLLM_CUDA(cudaSetDevice(gpus[i]));
    SLLM_CUDA(cudaFree(nullptr));  // primary context current on this thread
    CUresult r = d.DeviceGet(&devs[i], gpus[i]);
    if (r != CUDA_SUCCESS) fail(SLLM_E_CUDA, "cuDeviceGet: " + cu_str(r));
    int mc_ok = 0;
    r = d.DeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, devs[i]);
    if (r != CUDA_SUCCESS || !mc_ok)
      fail(SLLM_E_INVALID, "NVLS: GPU " + std::to_string(gpus[i]) + " does not support multicast objects");
  }
  // One process, so no shareable handle is needed; some drivers still insist on a type.
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                              CU_MEM_HANDLE_TYPE_FABRIC};
  std::string why;
  CUmemAllocationHandleType ht = CU_MEM_HANDLE_TYPE_NONE;
  bool created = false;
  for (CUmemAllocationHandleType t : types) {
    CUmulticastObjectProp mp{};
    mp.numDevices = (unsigned)n;
    mp.handleTypes = t;
    size_t gran = 0;
    CUresult r = d.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS || !gran) {
      why += " granularity(" + std::to_string((int)t) + "): " + cu_str(r) + ";";
      continue;
    }
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devs[0];
    ap.requestedHandleTypes = t;
    size_t ugran = 0;
    r = d.MemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS || !ugran) ugran = gran;
    const size_t a = std::max(gran, ugran);
    mp.size = align_up(bytes, a);
    r = d.MulticastCreate(&g->mc, &mp);
    if (r != CUDA_SUCCESS) {
      why += " cuMulticastCreate(handle type " + std::to_string((int)t) + "): " + cu_str(r) + ";";
      g->mc = 0;
      continue;
    }
    g->size = mp.size;
    ht = t;
    created = true;
    break;
  }
  if (!created) fail(SLLM_E_INVALID, "NVLS: this platform cannot create multicast objects --" + why);
  for (int i = 0; i < n; ++i) {
    CUresult r = d.MulticastAddDevice(g->mc, devs[i]);
    if (r != CUDA_SUCCESS) fail(SLLM_E_INVALID, "NVLS: cuMulticastAddDevice: " + cu_str(r));
  }
  g->mem.assign(n, 0);
  g->uva.assign(n, 0);
  g->bound.assign(n, false);
  g->signal.assign(n, nullptr);
  for (int i = 0; i < n; ++i) {
    SLLM_CUDA(cudaSetDevice(gpus[i]));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devs[i];
    ap.requestedHandleTypes = ht;
    CUresult r = d.MemCreate(&g->mem[i], g->size, &ap, 0);
    if (r != CUDA_SUCCESS) fail(SLLM_E_CAPACITY, "NVLS: cuMemCreate of a replica: " + cu_str(r));
    r = d.MulticastBindMem(g->mc, 0, g->mem[i], 0, g->size, 0);
    if (r != CUDA_SUCCESS) fail(SLLM_E_INVALID, "NVLS: cuMulticastBindMem: " + cu_str(r));
    g->bound[i] = true;
    r = d.MemAddressReserve(&g->uva[i], g->size, 0, 0, 0);
    if (r == CUDA_SUCCESS) r = d.MemMap(g->uva[i], g->size, 0, g->mem[i], 0);
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = devs[i];
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (r == CUDA_SUCCESS) r = d.MemSetAccess(g->uva[i], g->size, &acc, 1);
    if (r != CUDA_SUCCESS) fail(SLLM_E_CUDA, "NVLS: mapping a replica: " + cu_str(r));
  }
  CUresult r = d.MemAddressReserve(&g->mc_va, g->size, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = d.MemMap(g->mc_va, g->size, 0, g->mc, 0);
  std::vector<CUmemAccessDesc> acc(n);
  for (int i = 0; i < n; ++i) {
    acc[i] = CUmemAccessDesc{};
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = devs[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  if (r == CUDA_SUCCESS) r = d.MemSetAccess(g->mc_va, g->size, acc.data(), n);
  if (r != CUDA_SUCCESS) fail(SLLM_E_CUDA, "NVLS: mapping the multicast object: " + cu_str(r));
  // completion signals (the P2P group's protocol): per GPU, written by the peers over NVLink
  for (int i = 0; i < n; ++i) {
    SLLM_CUDA(cudaSetDevice(gpus[i]));
    void* s = nullptr;
    SLLM_CUDA(cudaMalloc(&s, 2 * (size_t)n * sizeof(uint32_t)));
    SLLM_CUDA(cudaMemset(s, 0, 2 * (size_t)n * sizeof(uint32_t)));
    g->signal[i] = static_cast<uint32_t*>(s);
    for (int k = 0; k < n; ++k)
      if (k != i) {
        int ok = 0;
        SLLM_CUDA(cudaDeviceCanAccessPeer(&ok, gpus[i], gpus[k]));
        if (!ok) fail(SLLM_E_INVALID, "NVLS: GPU " + std::to_string(gpus[i]) + " cannot access GPU " + std::to_string(gpus[k]));
        cudaError_t e = cudaDeviceEnablePeerAccess(gpus[k], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SLLM_CUDA(e);
        cudaGetLastError();
      }
  }
  for (int i = 0; i < n; ++i) {
    SLLM_CUDA(cudaSetDevice(gpus[i]));
    SLLM_CUDA(cudaDeviceSynchronize());
  }
  return g;
}

size_t nvls_size(const NvlsGroup& g) { return g.size; }
uint8_t* nvls_mc(const NvlsGroup& g) { return reinterpret_cast<uint8_t*>(g.mc_va); }
uint8_t* nvls_replica(const NvlsGroup& g, int i) { return reinterpret_cast<uint8_t*>(g.uva[i]); }
uint32_t* nvls_signal(const NvlsGroup& g, int i) { return g.signal[i]; }

}  // namespace sllm
