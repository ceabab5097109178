// NUMA placement of the DRAM tier's host work: pinned pages are
// bound to the node of the GPU they feed (hostmem.cpp, mbind) and the threads that touch
// them -- the per-partition load workers, the first-touch threads, the storage readers and
// the converter's fill / checksum threads -- run on that node's CPUs, so on a multi-socket
// 8-GPU server no byte of a partition crosses the socket interconnect on its way to its
// GPU's PCIe link ("parallel DRAM-to-GPU PCIe links").  No-ops on hosts with
// one node (sysfs only: the image has no libnuma).
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "runtime.hpp"

namespace sllm {

// sysfs root ("/sys"; SLLM_SYSFS_ROOT points the host tests at a fake node tree)
static const std::string& sysfs() {
  static const std::string root = [] {
    const char* e = getenv("SLLM_SYSFS_ROOT");
    return std::string(e && *e ? e : "/sys");
  }();
  return root;
}

int numa_nodes() {
  static const int n = [] {
    int k = 0;
    for (int i = 0; i < 1024; ++i) {
      std::string p = sysfs() + "/devices/system/node/node" + std::to_string(i);
      if (access(p.c_str(), F_OK) != 0) break;
      ++k;
    }
    return k;
  }();
  return n;
}

int gpu_numa_node(int gpu) {
  char bus[32] = {};
  if (gpu < 0 || cudaDeviceGetPCIBusId(bus, sizeof bus, gpu) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  std::string b(bus);
  for (auto& ch : b) ch = (char)tolower(ch);
  // cudaDeviceGetPCIBusId returns "0000:d1:00.0"; sysfs uses the same form
  FILE* f = fopen((sysfs() + "/bus/pci/devices/" + b + "/numa_node").c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

// "0-15,32-47" -> the CPU set
bool parse_cpulist(const std::string& s, cpu_set_t* set) {
  CPU_ZERO(set);
  size_t i = 0;
  bool any = false;
  while (i < s.size()) {
    size_t j = i;
    while (j < s.size() && isdigit((unsigned char)s[j])) ++j;
    if (j == i) { ++i; continue; }
    long a = std::stol(s.substr(i, j - i)), b = a;
    if (j < s.size() && s[j] == '-') {
      size_t k = j + 1;
      while (k < s.size() && isdigit((unsigned char)s[k])) ++k;
      if (k > j + 1) b = std::stol(s.substr(j + 1, k - j - 1));
      j = k;
    }
    for (long c = a; c <= b && c < CPU_SETSIZE; ++c) {
      CPU_SET((int)c, set);
      any = true;
    }
    i = j;
  }
  return any;
}

static bool node_cpus(int node, cpu_set_t* set) {
  FILE* f = fopen((sysfs() + "/devices/system/node/node" + std::to_string(node) + "/cpulist").c_str(), "r");
  if (!f) return false;
  char buf[4096] = {};
  const size_t n = fread(buf, 1, sizeof buf - 1, f);
  fclose(f);
  return parse_cpulist(std::string(buf, n), set);
}

// Pin the calling thread to the CPUs of `node`, intersected with the process's allowed set
// -- the main thread's mask, not the calling thread's: a pooled load worker bound to one
// node for one job is re-bound to another node for the next (its own mask would intersect
// to nothing).  An unknown node, or one with no allowed CPU, unbinds the thread (process
// mask).  Returns true if the affinity was set.
bool bind_thread_to_node(int node) {
  if (numa_nodes() <= 1) return false;
  cpu_set_t want, allowed, both;
  if (sched_getaffinity(getpid(), sizeof allowed, &allowed) != 0) return false;
  both = allowed;
  if (node >= 0 && node_cpus(node, &want)) {
    CPU_AND(&both, &want, &allowed);
    if (CPU_COUNT(&both) == 0) both = allowed;
  }
  return sched_setaffinity(0, sizeof both, &both) == 0;
}

bool bind_thread_to_gpu(int gpu) { return numa_nodes() > 1 && bind_thread_to_node(gpu_numa_node(gpu)); }

// Node holding the page at p (get_mempolicy(MPOL_F_NODE | MPOL_F_ADDR)), -1 if unknown.
int page_node(const void* p) {
  int node = -1;
  if (syscall(SYS_get_mempolicy, &node, nullptr, 0, const_cast<void*>(p), 3 /*MPOL_F_NODE|MPOL_F_ADDR*/) != 0)
    return -1;
  return node;
}

}  // namespace sllm
