// Where the time between a kernel's CUDA events and its own execution goes (diagnostic,
// never the product): for a kernel shaped like the ring kernel (148 CTAs x 320 threads,
// 196.8 KB dynamic shared memory) and for a plain one (0 B), launched alone between two
// events, report the event-to-event time and the in-kernel span (first CTA start to last
// CTA end, %globaltimer).  Their difference is launch + completion overhead.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/launch_gap tools/launch_gap.cu
//   build/launch_gap [spin_us]
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// every CTA spins for spin_ns, then marks [~min start, max end]
__global__ void spin_kernel(unsigned long long* kt, unsigned long long spin_ns, int touch) {
  extern __shared__ unsigned char smem[];
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) atomicMax(kt, ~t0);
  while (gt() - t0 < spin_ns) {
  }
  if (threadIdx.x == 0 && touch) smem[0] = 1;  // (only with dynamic shared memory)
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(kt + 1, gt());
}

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

int main(int argc, char** argv) {
  const unsigned long long spin_us = argc > 1 ? atoll(argv[1]) : 300;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int big = 12 * 16384 + 2 * 12 * 8;  // the ring kernel's dynamic shared memory
  CK(cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  unsigned long long* kt;
  CK(cudaMalloc(&kt, 16));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  // "after_copy": like the loader's kernel stream, st first waits for a 64 MiB host->device
  // copy on another stream (the event pair brackets only the kernel, as in the pipeline)
  cudaStream_t cs;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t landed;
  CK(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming));
  const size_t cbytes = 64ull << 20, big_copy = 1ull << 30;
  void *hsrc, *ddst;
  CK(cudaMallocHost(&hsrc, big_copy));
  CK(cudaMalloc(&ddst, big_copy));
  // variants: 0 plain (0 B smem), 1 ring-kernel smem, 2 after a 64 MiB copy on another
  // stream (waited), 3 while a 1 GiB host->device copy saturates PCIe on another stream,
  // 4 as 3 with (event, kernel, event) launched as one CUDA graph
  cudaGraphExec_t gexec = nullptr;
  for (int variant = 0; variant < 5; ++variant) {
    const int smem = variant == 0 ? 0 : big;
    const bool after_copy = variant == 2, during_copy = variant >= 3, graph = variant == 4;
    if (graph && !gexec) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      CK(cudaEventRecordWithFlags(a, st, cudaEventRecordExternal));
      spin_kernel<<<sms, 320, smem, st>>>(kt, spin_us * 1000, smem > 0);
      CK(cudaEventRecordWithFlags(b, st, cudaEventRecordExternal));
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&gexec, g, 0));
      CK(cudaGraphUpload(gexec, st));
    }
    std::vector<double> ev_us, span_us;
    for (int rep = 0; rep < 40; ++rep) {
      CK(cudaMemsetAsync(kt, 0, 16, st));
      if (after_copy) {
        CK(cudaMemcpyAsync(ddst, hsrc, cbytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(landed, cs));
        CK(cudaStreamWaitEvent(st, landed, 0));
      }
      if (during_copy) {  // the kernel starts ~2 ms into a ~19 ms copy
        CK(cudaMemcpyAsync(ddst, hsrc, big_copy, cudaMemcpyHostToDevice, cs));
        CK(cudaStreamSynchronize(st));
        const auto t0 = std::chrono::steady_clock::now();
        while (std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(2)) {
        }
      }
      if (graph) {
        CK(cudaGraphLaunch(gexec, st));
      } else {
        CK(cudaEventRecord(a, st));
        spin_kernel<<<sms, 320, smem, st>>>(kt, spin_us * 1000, smem > 0);
        CK(cudaEventRecord(b, st));
      }
      CK(cudaStreamSynchronize(st));
      CK(cudaStreamSynchronize(cs));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      unsigned long long h[2];
      CK(cudaMemcpy(h, kt, 16, cudaMemcpyDeviceToHost));
      if (rep < 5) continue;  // warm-up
      ev_us.push_back(ms * 1e3);
      span_us.push_back((h[1] - ~h[0]) * 1e-3);
    }
    std::sort(ev_us.begin(), ev_us.end());
    std::sort(span_us.begin(), span_us.end());
    const size_t m = ev_us.size() / 2;
    printf("{\"smem\": %d, \"after_copy\": %d, \"during_copy\": %d, \"graph\": %d, \"spin_us\": %llu, "
           "\"event_us_median\": %.2f, \"span_us_median\": %.2f, \"overhead_us_median\": %.2f, \"event_us_min\": %.2f, "
           "\"event_us_max\": %.2f}\n",
           smem, (int)after_copy, (int)during_copy, (int)graph, spin_us, ev_us[m], span_us[m], ev_us[m] - span_us[m],
           ev_us[0], ev_us.back());
  }
  return 0;
}
