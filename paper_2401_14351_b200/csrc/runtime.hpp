// Host runtime internals: per-GPU contexts, NCCL shim, load objects.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <functional>
#include <mutex>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include <cstdio>

#include "common.hpp"
#include "kernels.cuh"

namespace sllm {

// Host-side NVTX range around a load phase (SURVEY §5 tracing): "sllm.<phase> ...".  Free
// unless a tool (ncu --nvtx, nsys) injects NVTX; ncu selects e.g. only the verification
// launches with --nvtx --nvtx-include "regex:sllm\.verify\..*/" ('/' is ncu's range-nesting
// separator, so the names use '.').
struct NvtxRange {
  template <class... A>
  explicit NvtxRange(const char* fmt, A... a) {
    if constexpr (sizeof...(A) == 0) {
      nvtxRangePushA(fmt);
    } else {
      char b[96];
      snprintf(b, sizeof b, fmt, a...);
      nvtxRangePushA(b);
    }
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


[[noreturn]] void cuda_fail(cudaError_t e, const char* what);
#define SLLM_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) ::sllm::cuda_fail(_e, #call);  \
  } while (0)

constexpr int kMaxStreams = 8;
constexpr uint32_t kTile = 64u << 10;  // bytes per kernel work tile
constexpr uint64_t kWindowBytes = 64ull << 20;   // min bytes per copy submission / kernel launch
constexpr uint64_t kCopyWindowMaxBytes = 256ull << 20;  // max bytes per copy submission (large partitions)
constexpr uint64_t kVerifyBytes = 4096ull << 20;  // CE mode: max bytes per verification launch
                                                  // (span sweep r02: 2 -> 4 GiB spans, K4 0.91 -> 0.94 of HBM, step unchanged)
constexpr uint64_t kVerifyTailBytes = 512ull << 20;  // CE mode: min span once the load's end is near
constexpr uint64_t kAutoZeroCopyBytes = 256ull << 20;  // SLLM_MODE_AUTO: zero-copy below this per job
constexpr int kDefaultEngine = 1;  // MatParams.engine of sllm_load_config.engine == 0
constexpr uint64_t kScatterWindowBytes = 1024ull << 20;  // SCATTER_CE: bytes per staging slot / K3 launch
constexpr uint64_t kScatterTailBytes = 256ull << 20;     // SCATTER_CE: smallest window near the end
constexpr uint32_t kGranShift = 20;  // scatter granule table: one entry per MiB of partition
constexpr uint64_t kScatterFileWindowBytes = 256ull << 20;  // SCATTER_CE from files: storage-ring window

// Library-owned, per-GPU resources reused across loads (no allocation in the hot path).
// Every running partition job leases its own stream set, so concurrent jobs on one GPU
// (several partitions, several loads) never queue behind each other's waits and their
// per-launch timings stay their own.
struct StreamSet {
  cudaStream_t xfer[kMaxStreams] = {};
  cudaStream_t kern = nullptr;
  cudaStream_t comm = nullptr;
  // pinned host block of the job holding the set: its per-load tables go up in ONE async
  // copy and its result word comes back into it (grown on demand, kept for the next job)
  uint8_t* host = nullptr;
  size_t host_cap = 0;
  uint8_t* host_stage(size_t bytes);  // caller holds the set (exclusive), device set
};
struct DeviceCtx {
  int dev = -1;
  std::mutex mu;
  cudaStream_t misc = nullptr;                         // scratch frees after a load
  std::vector<std::unique_ptr<StreamSet>> sets;
  std::vector<StreamSet*> idle;
  StreamSet* acquire(int n_streams);                   // caller holds mu, device set
  void release(StreamSet* s);                          // caller holds mu
};
DeviceCtx& device_ctx(int dev);

// ---- file tier (filetier.cpp) --------------------------------------------------------
struct FileSource;
struct FileSourceDeleter {
  void operator()(FileSource* f) const;
};
using FileSourcePtr = std::unique_ptr<FileSource, FileSourceDeleter>;
// Start `io_threads` O_DIRECT readers filling a ring of pinned `window`-byte slots with
// windows of the partition file at `path`: window w = bytes [lo + w*window, ...) below
// `length` (lo > 0: a replicated load's slice).
FileSourcePtr file_source_open(const std::string& path, uint64_t lo, uint64_t length, uint64_t window, int io_threads,
                               int gpu);
const uint8_t* file_source_window(FileSource& f, uint64_t w);        // blocks until window w is in its slot
void file_source_consumed(FileSource& f, uint64_t w, cudaStream_t s);  // slot reusable once s passes here
uint64_t file_source_bytes(FileSource& f);
uint64_t file_source_wait_ns(FileSource& f);  // worker time blocked waiting for storage

// ---- NCCL (loaded with dlopen; only the calls the fan-out needs) -------------------
struct Nccl;
const Nccl& nccl();  // throws SLLM_E_NCCL if libnccl.so.2 cannot be loaded
void nccl_bcast_group(sllm_comm* comm, const std::vector<std::pair<uint64_t, uint64_t>>& ranges_by_root,
                      uint8_t* buf, cudaStream_t s);
void nccl_allgather_inplace(sllm_comm* comm, uint64_t lo, uint64_t count, uint8_t* buf, cudaStream_t s);
int comm_nranks(const sllm_comm* c);
int comm_local_members(const sllm_comm* c);  // ranks of c's P2P group living in this process
int comm_rank(const sllm_comm* c);
int comm_device(const sllm_comm* c);
bool comm_is_peers(const sllm_comm* c);
uint8_t* comm_peer_base(const sllm_comm* c, int q);
uint32_t* comm_peer_signal(const sllm_comm* c, int q);
uint64_t comm_timeout_ns(const sllm_comm* c);
uint32_t comm_next_epoch(sllm_comm* c);
uint8_t* comm_mc(const sllm_comm* c);  // NVLS: multicast address of replica byte 0 (else null)
// In-process peer groups (every rank's handle lives in this process): stream ordering by
// CUDA events, no device-side waits (fanout.cpp).
enum PeerEvent { kPeerReady = 0, kPeerDone = 1 };
bool comm_in_process(const sllm_comm* c);
void comm_record(sllm_comm* c, PeerEvent which, cudaStream_t s);      // this rank's event, on s
void comm_wait_peers(sllm_comm* c, PeerEvent which, cudaStream_t s);  // s waits on every peer's
bool comm_local_barrier(sllm_comm* c);  // host rendezvous of the in-process ranks; false on timeout
bool comm_host_wait();                  // SLLM_PEER_WAIT=host: multi-process peers waited for on the host
// host wait until own[q] >= epoch for every peer q (SLLM_E_PEER after the group timeout)
void comm_wait_flags_host(sllm_comm* c, const uint32_t* own, uint32_t epoch);

// ---- NVLS multicast group (nvls.cpp) -------------------------------------------------
struct NvlsGroup;
std::shared_ptr<NvlsGroup> nvls_group_create(const int32_t* gpus, int32_t n, uint64_t bytes);
size_t nvls_size(const NvlsGroup& g);
uint8_t* nvls_mc(const NvlsGroup& g);
uint8_t* nvls_replica(const NvlsGroup& g, int i);
uint32_t* nvls_signal(const NvlsGroup& g, int i);

// GPUDirect Storage reads (gds.cpp): file bytes [lo, hi) -> dst + lo on `gpu`, `threads`
// cuFile readers; landed(a, b) on the calling thread as the contiguous landed prefix grows.
void gds_read(const std::string& path, int gpu, uint8_t* dst, uint64_t lo, uint64_t hi, uint64_t window, int threads,
              const std::function<void(uint64_t, uint64_t)>& landed, uint64_t* wait_ns);

// out[g] = index of the last segment with off <= g << shift, g = 0..ceil(len >> shift)
// (segs sorted by off, segs[0].off == 0) -- MatParams.gran_seg.
inline void gran_table(const std::vector<Seg>& segs, uint64_t len, uint32_t shift, std::vector<uint32_t>& out) {
  const uint64_t n = ((len + (1ull << shift) - 1) >> shift) + 1;
  out.assign(n, 0);
  size_t s = 0;
  for (uint64_t g = 0; g < n; ++g) {
    while (s + 1 < segs.size() && segs[s + 1].off <= (g << shift)) ++s;
    out[g] = (uint32_t)s;
  }
}
cudaStream_t comm_stream(sllm_comm* c, int s);

}  // namespace sllm
