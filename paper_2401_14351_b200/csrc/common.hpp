// Internal declarations shared by the library's translation units.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "sllm.h"

namespace sllm {

// Thrown inside the library, converted to sllm_status at the ABI boundary (abi.cpp).
struct Error : std::runtime_error {
  sllm_status code;
  Error(sllm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(sllm_status c, const std::string& m) { throw Error(c, m); }

void set_last_error(const std::string& m);

// Largest alignment / checksum block (Q8): keeps the kernels' unfolded 64-bit
// Fletcher partial sums (word index < 2^26 times a 16-byte vector sum < 2^34, 16 per tile)
// below 2^64.
constexpr uint64_t kMaxBlock = 256ull << 20;

inline bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

int dtype_width(int32_t dtype);  // 0 for unknown codes

// NUMA (numa.cpp)
int numa_nodes();
int gpu_numa_node(int gpu);            // -1 if unknown
bool bind_thread_to_node(int node);    // calling thread -> that node's CPUs (multi-node hosts)
bool bind_thread_to_gpu(int gpu);      // ... the node of `gpu`'s PCIe root
int page_node(const void* p);          // node holding the page at p, -1 if unknown

struct TensorRec {
  std::string name;
  int32_t device;
  int32_t part;      // index into Index::parts
  int32_t dtype;
  int32_t ndim;
  int64_t shape[SLLM_MAX_NDIM];
  uint64_t offset;
  uint64_t nbytes;
};

struct PartRec {
  int32_t device;
  uint64_t length;
  uint64_t n_tensors;
  uint64_t n_blocks;
  std::vector<uint64_t> checksums;   // n_blocks entries
  std::vector<uint32_t> by_offset;   // tensor ids of this partition sorted by offset
};

}  // namespace sllm

struct sllm_index {
  uint64_t align = 0, block = 0;
  std::string model_id;
  std::vector<sllm::PartRec> parts;
  std::vector<sllm::TensorRec> tensors;
  // name -> tensor id; keys view tensors[i].name (the tensor table is sized once, never
  // reallocated after the names are entered)
  std::unordered_map<std::string_view, uint32_t> by_name;
  uint64_t payload = 0;
  uint64_t serial = 0;  // process-unique id (device-side caches key on it)
  bool sealed = false;
};

namespace sllm {

// format.cpp
sllm_index* plan(const sllm_src_tensor* t, size_t n, uint64_t align, uint64_t block, const char* model_id);
void seal(sllm_index* idx, const void* const* part_bufs);
std::vector<uint8_t> serialize(const sllm_index& idx);
sllm_index* parse(const uint8_t* blob, size_t len);
uint64_t fletcher64(const uint8_t* p, uint64_t nbytes);
int default_threads();

}  // namespace sllm

namespace sllm {
void convert_into(const sllm_src_tensor* t, size_t n, sllm_index* idx, void* const* part_bufs);
}
