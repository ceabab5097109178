// Replicated-model fan-out over NVLink 5 / NVSwitch with NCCL.
//
// The paper loads multi-GPU models "from pinned memory pool" over "parallel PCIe links"
// and has no GPU-to-GPU path.  For a replicated checkpoint the
// B200 build lets every byte cross PCIe once: rank r reads slice r over its own link,
// and each chunk round is broadcast from its owner to every other GPU (grouped
// ncclBroadcast, one root per slice) while the next PCIe chunk is in flight -- or, with
// round-robin chunk ownership, gathered by one in-place ncclAllGather per round.
//
// libnccl.so.2 (NCCL 2.28, shipped with PyTorch) is opened with dlopen so the library
// loads on hosts without NCCL; only the handful of calls below are bound.
#include <dlfcn.h>

#include <condition_variable>
#include <map>

#include "nccl.h"
#include "runtime.hpp"

namespace sllm {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static std::mutex g_nccl_mu;
static Nccl g_nccl;
static bool g_nccl_ok = false;

template <class F>
static void bind(void* h, F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) fail(SLLM_E_NCCL, std::string("libnccl is missing ") + name);
}

const Nccl& nccl() {
  std::lock_guard<std::mutex> g(g_nccl_mu);
  if (g_nccl_ok) return g_nccl;
  const char* env = getenv("SLLM_NCCL_LIBRARY");
  void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(SLLM_E_NCCL, std::string("cannot load NCCL: ") + dlerror());
  g_nccl.h = h;
  bind(h, g_nccl.GetUniqueId, "ncclGetUniqueId");
  bind(h, g_nccl.CommInitRank, "ncclCommInitRank");
  bind(h, g_nccl.CommInitAll, "ncclCommInitAll");
  bind(h, g_nccl.CommDestroy, "ncclCommDestroy");
  bind(h, g_nccl.Broadcast, "ncclBroadcast");
  bind(h, g_nccl.AllGather, "ncclAllGather");
  bind(h, g_nccl.GroupStart, "ncclGroupStart");
  bind(h, g_nccl.GroupEnd, "ncclGroupEnd");
  bind(h, g_nccl.GetErrorString, "ncclGetErrorString");
  g_nccl_ok = true;
  return g_nccl;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SLLM_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// Ranks of one P2P group that live in the same process (several GPUs driven by one process,
// or tests with several replicas on one GPU) order each other with CUDA events instead of
// device-side flag waits: rank r records its `ready` event once its stores into every replica
// are done and its `done` event once it has verified what it received, and a peer's stream
// waits on those events (cudaStreamWaitEvent, across devices too).  No kernel of one rank
// then waits for a kernel of another, so the ranks may share a GPU -- kernels that spin on a
// flag another rank writes must not (nothing guarantees both run at once; on B200 such
// ranks as processes on one GPU raised Xid 109).  An event wait only orders after the
// record already queued, so the in-process ranks rendezvous on the host at two points of
// every load: after each has recorded `ready` (before anyone waits on it) and after each
// has recorded `done` (before the next load's wait on it).  One rank per process (the
// deployment, peers mapped with CUDA IPC) uses the device-side signals instead.
struct LocalGroup {
  std::mutex mu;
  std::condition_variable cv;
  int members = 0;
  int count = 0;
  uint64_t gen = 0;
  std::vector<cudaEvent_t> ev[2];  // [kPeerReady / kPeerDone][rank], owned by the rank's handle
};
static std::mutex g_groups_mu;
static std::map<std::vector<uint32_t*>, std::weak_ptr<LocalGroup>> g_groups;

}  // namespace sllm

struct sllm_comm {
  ncclComm_t comm = nullptr;  // NCCL communicator (SLLM_FANOUT_BCAST)
  int nranks = 0, rank = 0, dev = 0;
  // peer group (SLLM_FANOUT_P2P): every rank's replica base and signal array, as device
  // pointers valid in this process; streams owned by the group so that several ranks on
  // one GPU (tests) never queue behind each other's peer waits
  bool peers = false;
  std::vector<uint8_t*> base;
  std::vector<uint32_t*> signal;
  uint32_t epoch = 0;
  uint64_t timeout_ns = 0;
  cudaStream_t streams[sllm::kMaxStreams + 2] = {};  // transfer, kernel, host-wait poll
  uint32_t* poll = nullptr;                            // pinned copy of the own signal words (host wait)
  std::shared_ptr<sllm::LocalGroup> local;  // the in-process ranks of this peer group
  cudaEvent_t ev[2] = {};                    // this rank's ready / done events (in-process groups)
  // NVLS group (SLLM_FANOUT_NVLS): the multicast object and the library-owned replicas it
  // binds (shared by the group's handles); mc = the multicast address of replica byte 0
  std::shared_ptr<sllm::NvlsGroup> nvls;
  uint8_t* mc = nullptr;
};

namespace sllm {

int comm_nranks(const sllm_comm* c) { return c->nranks; }
int comm_local_members(const sllm_comm* c) {
  if (!c || !c->local) return 1;
  std::lock_guard<std::mutex> g(c->local->mu);
  return c->local->members;
}
int comm_rank(const sllm_comm* c) { return c->rank; }
int comm_device(const sllm_comm* c) { return c->dev; }
bool comm_is_peers(const sllm_comm* c) { return c->peers; }
uint8_t* comm_peer_base(const sllm_comm* c, int q) { return c->base[q]; }
uint32_t* comm_peer_signal(const sllm_comm* c, int q) { return c->signal[q]; }
uint8_t* comm_mc(const sllm_comm* c) { return c->mc; }
uint64_t comm_timeout_ns(const sllm_comm* c) { return c->timeout_ns; }
uint32_t comm_next_epoch(sllm_comm* c) {
  if (++c->epoch == 0) ++c->epoch;  // 0 is the signal arrays' initial value
  return c->epoch;
}
bool comm_in_process(const sllm_comm* c) {
  if (!c || !c->local || c->nranks < 2) return false;
  std::lock_guard<std::mutex> g(c->local->mu);
  return c->local->members == c->nranks;
}

void comm_record(sllm_comm* c, PeerEvent which, cudaStream_t s) { SLLM_CUDA(cudaEventRecord(c->ev[which], s)); }

void comm_wait_peers(sllm_comm* c, PeerEvent which, cudaStream_t s) {
  std::vector<cudaEvent_t> evs;
  {
    std::lock_guard<std::mutex> g(c->local->mu);
    evs = c->local->ev[which];
  }
  for (int q = 0; q < (int)evs.size(); ++q)
    if (q != c->rank) {
      if (!evs[q]) fail(SLLM_E_PEER, "peer rank " + std::to_string(q) + " of this process has no handle");
      SLLM_CUDA(cudaStreamWaitEvent(s, evs[q], 0));
    }
}

bool comm_local_barrier(sllm_comm* c) {
  LocalGroup* g = c->local.get();
  if (!g) return true;
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->members <= 1) return true;
  const uint64_t my = g->gen;
  if (++g->count == g->members) {
    g->count = 0;
    ++g->gen;
    g->cv.notify_all();
    return true;
  }
  // a rank that never arrives (its load was not started): give up after the group timeout
  if (!g->cv.wait_for(lk, std::chrono::nanoseconds(c->timeout_ns), [&] { return g->gen != my; })) {
    --g->count;
    return false;
  }
  return true;
}

// This rank's share of the in-process group's events (created on the rank's GPU, current).
static void join_local_events(sllm_comm* c) {
  for (int w = 0; w < 2; ++w) SLLM_CUDA(cudaEventCreateWithFlags(&c->ev[w], cudaEventDisableTiming));
  std::lock_guard<std::mutex> lg(c->local->mu);
  for (auto& v : c->local->ev) {
    if ((int)v.size() < c->nranks) v.resize(c->nranks, nullptr);
  }
  for (int w = 0; w < 2; ++w) c->local->ev[w][c->rank] = c->ev[w];
}

// SLLM_PEER_WAIT=host: a one-process-per-rank group waits for its peers' flags on the host
// (the load's worker thread polls its own signal words with a small device->host copy)
// instead of with a device-side wait kernel.  No kernel then waits for another process's
// kernel, so the ranks may share a GPU (the multi-process wiring tested on one GPU); the
// flags themselves are written as in the default mode (peer_signal_kernel).
bool comm_host_wait() {
  static const bool host = [] {
    const char* e = getenv("SLLM_PEER_WAIT");
    return e && std::string(e) == "host";
  }();
  return host;
}

void comm_wait_flags_host(sllm_comm* c, const uint32_t* own, uint32_t epoch) {
  if (c->nranks <= 1) return;
  if (!c->poll) SLLM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->poll), 4 * (size_t)c->nranks, cudaHostAllocDefault));
  cudaStream_t s = comm_stream(c, kMaxStreams + 1);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    SLLM_CUDA(cudaMemcpyAsync(c->poll, own, 4 * (size_t)c->nranks, cudaMemcpyDeviceToHost, s));
    SLLM_CUDA(cudaStreamSynchronize(s));
    int missing = -1;
    for (int q = 0; q < c->nranks && missing < 0; ++q)
      if (q != c->rank && (int32_t)(c->poll[q] - epoch) < 0) missing = q;
    if (missing < 0) return;
    if ((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count() >
        c->timeout_ns)
      fail(SLLM_E_PEER, "P2P fan-out: peer rank " + std::to_string(missing) +
                            " did not signal completion within the timeout (host wait)");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

cudaStream_t comm_stream(sllm_comm* c, int s) {  // s = 0..kMaxStreams-1 transfer, kMaxStreams kernel, +1 poll
  if (!c->streams[s]) SLLM_CUDA(cudaStreamCreateWithFlags(&c->streams[s], cudaStreamNonBlocking));
  return c->streams[s];
}

// One round: ranges_by_root[q] = [lo, hi) broadcast from rank q (empty = no message).
void nccl_bcast_group(sllm_comm* c, const std::vector<std::pair<uint64_t, uint64_t>>& ranges, uint8_t* buf,
                      cudaStream_t s) {
  const Nccl& n = nccl();
  nccl_check(n.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < (int)ranges.size(); ++q) {
    uint64_t lo = ranges[q].first, hi = ranges[q].second;
    if (hi <= lo) continue;
    ncclResult_t r = n.Broadcast(buf + lo, buf + lo, hi - lo, ncclUint8, q, c->comm, s);
    if (r != ncclSuccess) {
      n.GroupEnd();
      nccl_check(r, "ncclBroadcast");
    }
  }
  nccl_check(n.GroupEnd(), "ncclGroupEnd");
}

// One full all-gather round (SLLM_FANOUT_ALLGATHER): rank q's chunk sits at
// buf + lo + q*count, so the gather is in place (sendbuff = recvbuff + rank*count).
void nccl_allgather_inplace(sllm_comm* c, uint64_t lo, uint64_t count, uint8_t* buf, cudaStream_t s) {
  nccl_check(nccl().AllGather(buf + lo + (uint64_t)c->rank * count, buf + lo, count, ncclUint8, c->comm, s),
             "ncclAllGather");
}

}  // namespace sllm

using namespace sllm;

void sllm_comm_unique_id_internal(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  if (!id128) fail(SLLM_E_INVALID, "null id buffer");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof id);
}

sllm_comm* sllm_comm_init_rank_internal(const void* id128, int32_t nranks, int32_t rank, int32_t gpu) {
  if (!id128 || nranks < 1 || rank < 0 || rank >= nranks || gpu < 0) fail(SLLM_E_INVALID, "bad communicator arguments");
  const Nccl& n = nccl();
  SLLM_CUDA(cudaSetDevice(gpu));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  std::unique_ptr<sllm_comm> c(new sllm_comm);
  nccl_check(n.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  c->nranks = nranks;
  c->rank = rank;
  c->dev = gpu;
  return c.release();
}

void sllm_comm_init_all_internal(const int32_t* gpus, int32_t n, sllm_comm** out) {
  if (!gpus || n < 1 || !out) fail(SLLM_E_INVALID, "bad communicator arguments");
  const Nccl& nc = nccl();
  std::vector<ncclComm_t> comms(n);
  std::vector<int> devs(gpus, gpus + n);
  nccl_check(nc.CommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
  for (int i = 0; i < n; ++i) {
    out[i] = new sllm_comm;
    out[i]->comm = comms[i];
    out[i]->nranks = n;
    out[i]->rank = i;
    out[i]->dev = gpus[i];
  }
}

// P2P peer group (no NCCL): SURVEY §8(f) rank 4 -- the fan-out fused into the loading
// kernel, stores over NVLink straight into every peer's replica.
sllm_comm* sllm_comm_init_peers_internal(int32_t nranks, int32_t rank, int32_t gpu, void* const* peer_base,
                                         uint32_t* const* peer_signal, uint64_t timeout_ms) {
  if (nranks < 1 || nranks > kMaxPeers + 1 || rank < 0 || rank >= nranks || gpu < 0 || !peer_base || !peer_signal)
    fail(SLLM_E_INVALID, "bad peer-group arguments (1 <= nranks <= 8, 0 <= rank < nranks)");
  SLLM_CUDA(cudaSetDevice(gpu));
  std::unique_ptr<sllm_comm> c(new sllm_comm);
  c->nranks = nranks;
  c->rank = rank;
  c->dev = gpu;
  c->peers = true;
  c->timeout_ns = (timeout_ms ? timeout_ms : 60000ull) * 1000000ull;
  for (int q = 0; q < nranks; ++q) {
    if (!peer_base[q] || !peer_signal[q]) fail(SLLM_E_INVALID, "null peer base / signal");
    if (reinterpret_cast<uintptr_t>(peer_base[q]) & 15) fail(SLLM_E_INVALID, "peer base must be 16-byte aligned");
    if (reinterpret_cast<uintptr_t>(peer_signal[q]) & 3) fail(SLLM_E_INVALID, "peer signal must be 4-byte aligned");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, peer_base[q]) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      fail(SLLM_E_INVALID, "peer base " + std::to_string(q) + " is not device memory visible to this process");
    }
    if (at.device != gpu) {  // a replica on another GPU: this GPU must be able to store into it
      int ok = 0;
      SLLM_CUDA(cudaDeviceCanAccessPeer(&ok, gpu, at.device));
      if (!ok) fail(SLLM_E_INVALID, "GPU " + std::to_string(gpu) + " cannot access peer GPU " + std::to_string(at.device));
      cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SLLM_CUDA(e);
      cudaGetLastError();
    }
    c->base.push_back(static_cast<uint8_t*>(peer_base[q]));
    c->signal.push_back(peer_signal[q]);
  }
  if (nranks > 1) {  // join (or start) this process's share of the group
    std::lock_guard<std::mutex> g(g_groups_mu);
    auto& w = g_groups[c->signal];
    c->local = w.lock();
    if (!c->local) w = c->local = std::make_shared<LocalGroup>();
    {
      std::lock_guard<std::mutex> lg(c->local->mu);
      ++c->local->members;
    }
    join_local_events(c.get());
  }
  return c.release();
}

// NVLS group: one process, GPUs gpus[0..n-1]; handle i is rank i on
// gpus[i].  The fan-out runs the P2P group's protocol (slices, ready/done epochs, received
// ranges verified by K4) with every vector stored once through the multicast address.
void sllm_comm_init_nvls_internal(const int32_t* gpus, int32_t n, uint64_t bytes, uint64_t timeout_ms,
                                  sllm_comm** out) {
  if (!out) fail(SLLM_E_INVALID, "null out");
  std::shared_ptr<NvlsGroup> g = nvls_group_create(gpus, n, bytes);
  auto local = std::make_shared<LocalGroup>();
  local->members = n;
  std::vector<std::unique_ptr<sllm_comm>> cs;
  for (int i = 0; i < n; ++i) {
    std::unique_ptr<sllm_comm> c(new sllm_comm);
    c->nranks = n;
    c->rank = i;
    c->dev = gpus[i];
    c->peers = true;
    c->timeout_ns = (timeout_ms ? timeout_ms : 60000ull) * 1000000ull;
    for (int q = 0; q < n; ++q) {
      c->base.push_back(nvls_replica(*g, q));
      c->signal.push_back(nvls_signal(*g, q));
    }
    c->nvls = g;
    c->mc = nvls_mc(*g);
    if (n > 1) {
      c->local = local;
      SLLM_CUDA(cudaSetDevice(gpus[i]));
      join_local_events(c.get());
    }
    cs.push_back(std::move(c));
  }
  for (int i = 0; i < n; ++i) out[i] = cs[i].release();
}

void sllm_comm_replica_internal(const sllm_comm* c, void** base, uint64_t* bytes) {
  if (!c || !base) fail(SLLM_E_INVALID, "null argument");
  if (!c->peers) fail(SLLM_E_INVALID, "an NCCL communicator is not bound to a replica");
  *base = c->base[c->rank];
  if (bytes) *bytes = c->nvls ? nvls_size(*c->nvls) : 0;
}

void sllm_comm_free_internal(sllm_comm* c) {
  if (!c) return;
  if (c->comm && g_nccl_ok) g_nccl.CommDestroy(c->comm);
  if (c->local) {  // this rank's events leave the group's table (its loads are complete)
    std::lock_guard<std::mutex> lg(c->local->mu);
    for (auto& v : c->local->ev)
      if (c->rank < (int)v.size() && (v[c->rank] == c->ev[0] || v[c->rank] == c->ev[1])) v[c->rank] = nullptr;
  }
  if (c->local && c->nvls) {  // (an NVLS group's local share is not in the registry)
    std::lock_guard<std::mutex> lg(c->local->mu);
    --c->local->members;
  } else if (c->local) {
    std::lock_guard<std::mutex> g(g_groups_mu);
    {
      std::lock_guard<std::mutex> lg(c->local->mu);
      --c->local->members;
    }
    auto it = g_groups.find(c->signal);
    c->local.reset();
    if (it != g_groups.end() && it->second.expired()) g_groups.erase(it);
  }
  if (c->peers) {
    cudaSetDevice(c->dev);
    for (auto& s : c->streams)
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->poll) cudaFreeHost(c->poll);
  }
  delete c;
}
