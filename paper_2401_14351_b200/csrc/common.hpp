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
  std::string_view name;  // NUL-terminated, in the owning index's name arena
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

// Name -> tensor id: open addressing over a power-of-two table of (hash, id + 1) slots, the
// keys being views into the tensor table (one probe array, no node allocation per name: the
// index parse of an 1,120-tensor adapter spent most of its time in per-name heap work).
class NameTable {
 public:
  static constexpr uint32_t kNone = ~0u;
  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    slots_.assign(cap, Slot{0, 0});
    mask_ = cap - 1;
  }
  // false if the name is already present
  bool insert(std::string_view k, uint32_t id, const std::vector<TensorRec>& t) {
    const uint64_t h = hash(k);
    for (size_t i = h & mask_;; i = (i + 1) & mask_) {
      Slot& s = slots_[i];
      if (!s.id1) {
        s = Slot{h, id + 1};
        return true;
      }
      if (s.h == h && t[s.id1 - 1].name == k) return false;
    }
  }
  uint32_t find(std::string_view k, const std::vector<TensorRec>& t) const {
    if (slots_.empty()) return kNone;
    const uint64_t h = hash(k);
    for (size_t i = h & mask_;; i = (i + 1) & mask_) {
      const Slot& s = slots_[i];
      if (!s.id1) return kNone;
      if (s.h == h && t[s.id1 - 1].name == k) return s.id1 - 1;
    }
  }
  static uint64_t hash(std::string_view k) {  // 8 bytes per step
    uint64_t h = 0x9E3779B97F4A7C15ull ^ k.size();
    size_t i = 0;
    for (; i + 8 <= k.size(); i += 8) {
      uint64_t w;
      std::memcpy(&w, k.data() + i, 8);
      h = (h ^ w) * 0xBF58476D1CE4E5B9ull;
      h ^= h >> 31;
    }
    uint64_t w = 0;
    std::memcpy(&w, k.data() + i, k.size() - i);
    h = (h ^ w) * 0x94D049BB133111EBull;
    return h ^ (h >> 29);
  }

 private:
  struct Slot {
    uint64_t h;
    uint32_t id1;  // tensor id + 1 (0 = empty)
  };
  std::vector<Slot> slots_;
  size_t mask_ = 0;
};

}  // namespace sllm

struct sllm_index {
  sllm_index() = default;
  sllm_index(const sllm_index&) = delete;  // the tensor names view `names`
  sllm_index& operator=(const sllm_index&) = delete;
  uint64_t align = 0, block = 0;
  std::string model_id;
  std::vector<sllm::PartRec> parts;
  std::vector<sllm::TensorRec> tensors;
  // every tensor name, NUL-terminated, back to back: reserved once before the names are
  // appended, so the views in `tensors` stay valid
  std::string names;
  sllm::NameTable by_name;  // name -> tensor id
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
