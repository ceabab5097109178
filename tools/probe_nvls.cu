// Probe: can this box build an NVLink-SHARP multicast object (cuMulticastCreate), bind a
// cuMemCreate allocation to it, map the multicast address and store through it with
// multimem.st (NVLS fan-out)?  With one GPU the group has one member;
// the unicast mapping must then hold what the multimem stores wrote.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_nvls tools/probe_nvls.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x)                                                                    \
  do {                                                                           \
    CUresult r_ = (x);                                                           \
    if (r_ != CUDA_SUCCESS) {                                                    \
      const char* s_ = nullptr;                                                  \
      cuGetErrorString(r_, &s_);                                                 \
      printf("{\"step\": \"%s\", \"error\": %d, \"msg\": \"%s\"}\n", #x, (int)r_, s_ ? s_ : "?"); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void mc_store(uint8_t* mc, size_t n) {
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n; i += (size_t)gridDim.x * blockDim.x * 16) {
    uint32_t a = (uint32_t)i, b = a ^ 0x5a5a5a5au, c = a * 2654435761u, d = ~a;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
  }
}

int main() {
  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CU(cuDevicePrimaryCtxRetain(&ctx, dev));
  CU(cuCtxSetCurrent(ctx));
  const CUmemAllocationHandleType types[2] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
  const char* tname[2] = {"fabric", "posix_fd"};
  for (int ti = 0; ti < 2; ++ti) {
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = 1;
    mp.handleTypes = types[ti];
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t n = 32ull << 20;
    mp.size = (n + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle mch;
    CUresult r = cuMulticastCreate(&mch, &mp);
    if (r != CUDA_SUCCESS) {
      printf("{\"handle\": \"%s\", \"cuMulticastCreate\": %d}\n", tname[ti], (int)r);
      continue;
    }
    CU(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof ap);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = dev;
    ap.requestedHandleTypes = types[ti];
    size_t ugran = 0;
    CU(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t sz = (mp.size + ugran - 1) / ugran * ugran;
    CUmemGenericAllocationHandle mem;
    CU(cuMemCreate(&mem, sz, &ap, 0));
    CU(cuMulticastBindMem(mch, 0, mem, 0, mp.size, 0));
    CUdeviceptr uva, mva;
    CU(cuMemAddressReserve(&uva, sz, 0, 0, 0));
    CU(cuMemMap(uva, sz, 0, mem, 0));
    CU(cuMemAddressReserve(&mva, mp.size, 0, 0, 0));
    CU(cuMemMap(mva, mp.size, 0, mch, 0));
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof acc);
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(uva, sz, &acc, 1));
    CU(cuMemSetAccess(mva, mp.size, &acc, 1));
    CU(cuMemsetD8(uva, 0, n));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mc_store<<<148, 256>>>(reinterpret_cast<uint8_t*>(mva), n);
    cudaEventRecord(b);
    cudaError_t ke = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<uint32_t> h(n / 4);
    CU(cuMemcpyDtoH(h.data(), uva, n));
    size_t bad = 0;
    for (size_t i = 0; i < n; i += 16) {
      uint32_t x = (uint32_t)i;
      const uint32_t* w = &h[i / 4];
      if (w[0] != x || w[1] != (x ^ 0x5a5a5a5au) || w[2] != x * 2654435761u || w[3] != ~x) ++bad;
    }
    char fh[64] = {};
    CUresult er = CUDA_ERROR_NOT_SUPPORTED;
    if (types[ti] == CU_MEM_HANDLE_TYPE_FABRIC) er = cuMemExportToShareableHandle(fh, mch, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    printf("{\"handle\": \"%s\", \"mc_granularity\": %zu, \"kernel\": \"%s\", \"bad_vectors\": %zu, \"ms\": %.4f, "
           "\"GBps_mc_store\": %.1f, \"export_mc_handle\": %d}\n",
           tname[ti], gran, cudaGetErrorString(ke), bad, ms, n / (ms * 1e-3) / 1e9, (int)er);
    cuMemUnmap(mva, mp.size);
    cuMemUnmap(uva, sz);
    cuMemAddressFree(mva, mp.size);
    cuMemAddressFree(uva, sz);
    cuMulticastUnbind(mch, dev, 0, mp.size);
    cuMemRelease(mem);
    cuMemRelease(mch);
  }
  return 0;
}
