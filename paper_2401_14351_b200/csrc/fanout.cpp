// Replicated-model fan-out over NVLink 5 / NVSwitch with NCCL.
//
// The paper loads multi-GPU models "from pinned memory pool" over "parallel PCIe links"
// and has no GPU-to-GPU path.  For a replicated checkpoint the
// B200 build lets every byte cross PCIe once: rank r reads slice r over its own link,
// and each chunk round is broadcast from its owner to every other GPU (grouped
// ncclBroadcast, one root per slice) while the next PCIe chunk is in flight.
//
// libnccl.so.2 (NCCL 2.28, shipped with PyTorch) is opened with dlopen so the library
// loads on hosts without NCCL; only the handful of calls below are bound.
#include <dlfcn.h>

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
  bind(h, g_nccl.GroupStart, "ncclGroupStart");
  bind(h, g_nccl.GroupEnd, "ncclGroupEnd");
  bind(h, g_nccl.GetErrorString, "ncclGetErrorString");
  g_nccl_ok = true;
  return g_nccl;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SLLM_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace sllm

struct sllm_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, dev = 0;
};

namespace sllm {

int comm_nranks(const sllm_comm* c) { return c->nranks; }
int comm_rank(const sllm_comm* c) { return c->rank; }
int comm_device(const sllm_comm* c) { return c->dev; }

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

void sllm_comm_free_internal(sllm_comm* c) {
  if (!c) return;
  if (c->comm && g_nccl_ok) g_nccl.CommDestroy(c->comm);
  delete c;
}
