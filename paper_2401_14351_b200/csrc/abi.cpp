// extern "C" boundary of libsllm.so (include/sllm.h): argument checks, exception ->
// sllm_status translation and the thread-local last-error message.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.hpp"

namespace sllm {
static thread_local std::string t_last_error;
void set_last_error(const std::string& m) { t_last_error = m; }

// defined in the other translation units
void* host_alloc(uint64_t bytes, int gpu);
void host_free(void* p);
void convert_files(const sllm_src_tensor* t, size_t n, uint64_t align, uint64_t block, const char* model_id,
                   const char* out_dir);
std::vector<uint8_t> read_file(const char* path);
void read_partition(const char* dir, const sllm_index* idx, size_t p, void* dst, int threads);
void block_checksums_device(const void* src, uint64_t len, uint64_t block, uint64_t* out, int ctas, cudaStream_t st);
uint64_t materialise_device(const sllm_index* idx, size_t p, const void* src, void* const* dst_tensor, int ctas,
                            cudaStream_t st, float* kernel_ms);
}  // namespace sllm

sllm_load* sllm_load_create_internal(const sllm_index*, const sllm_load_config*, const void* const*, const int32_t*,
                                     void* const*, void* const*, void* const*, sllm_comm*, const char*, int32_t, bool capture = false);
void sllm_load_replay_internal(sllm_load*, void* const*);
sllm_status sllm_load_wait_internal(sllm_load*, sllm_load_report*);
void sllm_load_tensor_internal(const sllm_load*, const char*, sllm_tensor_handle*);
void sllm_load_block_checksums_internal(sllm_load*, size_t, const uint64_t**);
void sllm_load_free_internal(sllm_load*);
void sllm_device_trim_internal(int32_t gpu, uint64_t keep_bytes);
namespace sllm {
uint64_t fanout_unit(uint64_t chunk, int32_t fanout);
}
void sllm_comm_unique_id_internal(void*);
sllm_comm* sllm_comm_init_rank_internal(const void*, int32_t, int32_t, int32_t);
void sllm_comm_init_all_internal(const int32_t*, int32_t, sllm_comm**);
sllm_comm* sllm_comm_init_peers_internal(int32_t, int32_t, int32_t, void* const*, uint32_t* const*, uint64_t);
void sllm_comm_free_internal(sllm_comm*);
void sllm_comm_init_nvls_internal(const int32_t*, int32_t, uint64_t, uint64_t, sllm_comm**);
void sllm_comm_replica_internal(const sllm_comm*, void**, uint64_t*);
namespace sllm {
sllm_cache* cache_create(uint64_t capacity, int gpu, int pin);
void cache_acquire(sllm_cache* c, const char* dir, int io_threads, const sllm_index** index, void* const** bufs,
                   int32_t* hit);
void cache_release(sllm_cache* c, const char* dir);
void cache_stats(sllm_cache* c, sllm_cache_stats* s);
void cache_destroy(sllm_cache* c);
}  // namespace sllm

using namespace sllm;

template <class F>
static sllm_status guard(F&& f) {
  try {
    f();
    return SLLM_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return SLLM_E_NOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SLLM_E_INVALID;
  } catch (...) {
    set_last_error("unknown internal error");
    return SLLM_E_INVALID;
  }
}

// Entry points that select devices (cudaSetDevice on the caller's thread) restore the
// caller's current device on exit: the device is per-thread driver state shared with every
// other CUDA runtime in the process (PyTorch's included), so a load onto GPU 1 must not
// leave the caller's thread on GPU 1.
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = -1;
    }
  }
  ~DeviceGuard() {
    int now = -1;
    if (dev >= 0 && (cudaGetDevice(&now) != cudaSuccess || now != dev)) cudaSetDevice(dev);
    cudaGetLastError();
  }
};

template <class F>
static sllm_status guard_dev(F&& f) {
  DeviceGuard dg;
  return guard(std::forward<F>(f));
}

extern "C" {

const char* sllm_last_error(void) { return t_last_error.c_str(); }
int32_t sllm_abi_version(void) { return SLLM_ABI_VERSION; }

sllm_status sllm_plan(const sllm_src_tensor* tensors, size_t n, uint64_t align, uint64_t block, const char* model_id,
                      sllm_index** out) {
  return guard([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = plan(tensors, n, align, block, model_id);
  });
}

sllm_status sllm_convert_into(const sllm_src_tensor* tensors, size_t n, sllm_index* idx, void* const* part_bufs) {
  return guard([&] {
    if (!idx) fail(SLLM_E_INVALID, "null index");
    if (n && !tensors) fail(SLLM_E_INVALID, "null tensors");
    convert_into(tensors, n, idx, part_bufs);
  });
}

sllm_status sllm_index_seal(sllm_index* idx, const void* const* part_bufs) {
  return guard([&] {
    if (!idx) fail(SLLM_E_INVALID, "null index");
    seal(idx, part_bufs);
  });
}

sllm_status sllm_convert(const sllm_src_tensor* tensors, size_t n, uint64_t align, uint64_t block, const char* model_id,
                         const char* out_dir) {
  return guard([&] { convert_files(tensors, n, align, block, model_id, out_dir); });
}

sllm_status sllm_index_serialize(const sllm_index* idx, void* buf, size_t cap, size_t* len) {
  return guard([&] {
    if (!idx || !len) fail(SLLM_E_INVALID, "null argument");
    std::vector<uint8_t> b = serialize(*idx);
    *len = b.size();
    if (!buf) return;
    if (cap < b.size()) fail(SLLM_E_CAPACITY, "serialization buffer too small");
    std::memcpy(buf, b.data(), b.size());
  });
}

sllm_status sllm_index_open(const char* path, sllm_index** out) {
  return guard([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    std::vector<uint8_t> b = read_file(path);
    *out = parse(b.data(), b.size());
  });
}

sllm_status sllm_index_from_memory(const void* blob, size_t len, sllm_index** out) {
  return guard([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = parse(static_cast<const uint8_t*>(blob), len);
  });
}

void sllm_index_close(sllm_index* idx) { delete idx; }

sllm_status sllm_index_counts(const sllm_index* idx, size_t* n_tensors, size_t* n_partitions) {
  return guard([&] {
    if (!idx) fail(SLLM_E_INVALID, "null index");
    if (n_tensors) *n_tensors = idx->tensors.size();
    if (n_partitions) *n_partitions = idx->parts.size();
  });
}

sllm_status sllm_index_get_info(const sllm_index* idx, sllm_index_info* out) {
  return guard([&] {
    if (!idx || !out) fail(SLLM_E_INVALID, "null argument");
    sllm_index_info i{};
    i.align = idx->align;
    i.block = idx->block;
    i.payload_bytes = idx->payload;
    i.n_partitions = idx->parts.size();
    i.n_tensors = idx->tensors.size();
    i.model_id = idx->model_id.c_str();
    *out = i;
  });
}

sllm_status sllm_index_partition(const sllm_index* idx, size_t p, int32_t* device_id, uint64_t* length,
                                 uint64_t* n_blocks, uint64_t* n_tensors) {
  return guard([&] {
    if (!idx) fail(SLLM_E_INVALID, "null index");
    if (p >= idx->parts.size()) fail(SLLM_E_LOOKUP, "partition index out of range");
    const PartRec& pr = idx->parts[p];
    if (device_id) *device_id = pr.device;
    if (length) *length = pr.length;
    if (n_blocks) *n_blocks = pr.n_blocks;
    if (n_tensors) *n_tensors = pr.n_tensors;
  });
}

sllm_status sllm_index_block_checksums(const sllm_index* idx, size_t p, const uint64_t** table) {
  return guard([&] {
    if (!idx || !table) fail(SLLM_E_INVALID, "null argument");
    if (p >= idx->parts.size()) fail(SLLM_E_LOOKUP, "partition index out of range");
    *table = idx->parts[p].checksums.data();
  });
}

sllm_status sllm_index_tensor(const sllm_index* idx, size_t i, sllm_tensor_info* out) {
  return guard([&] {
    if (!idx || !out) fail(SLLM_E_INVALID, "null argument");
    if (i >= idx->tensors.size()) fail(SLLM_E_LOOKUP, "tensor index out of range");
    const TensorRec& t = idx->tensors[i];
    sllm_tensor_info o{};
    o.name = t.name.data();  // NUL-terminated in the index's name arena
    o.device_id = t.device;
    o.partition = t.part;
    o.dtype = t.dtype;
    o.ndim = t.ndim;
    std::memcpy(o.shape, t.shape, sizeof o.shape);
    o.offset = t.offset;
    o.nbytes = t.nbytes;
    *out = o;
  });
}

sllm_status sllm_index_find(const sllm_index* idx, const char* name, size_t* i) {
  return guard([&] {
    if (!idx || !name || !i) fail(SLLM_E_INVALID, "null argument");
    const uint32_t id = idx->by_name.find(name, idx->tensors);
    if (id == NameTable::kNone) fail(SLLM_E_LOOKUP, std::string("unknown tensor '") + name + "'");
    *i = id;
  });
}

sllm_status sllm_tensor_address(const sllm_index* idx, const char* name, const uint64_t* base_by_partition,
                                int32_t* device_id, uint64_t* addr) {
  return guard([&] {
    if (!idx || !name || !base_by_partition || !addr) fail(SLLM_E_INVALID, "null argument");
    const uint32_t id = idx->by_name.find(name, idx->tensors);
    if (id == NameTable::kNone) fail(SLLM_E_LOOKUP, std::string("unknown tensor '") + name + "'");
    const TensorRec& t = idx->tensors[id];
    if (device_id) *device_id = t.device;
    *addr = base_by_partition[t.part] + t.offset;  // P:549 base + offset
  });
}

sllm_status sllm_fletcher64_host(const void* data, uint64_t nbytes, uint64_t* out) {
  return guard([&] {
    if ((!data && nbytes) || !out) fail(SLLM_E_INVALID, "null argument");
    *out = fletcher64(static_cast<const uint8_t*>(data), nbytes);
  });
}

sllm_status sllm_chunk_count(uint64_t length, uint64_t chunk, uint64_t* n_chunks) {
  return guard([&] {
    if (!chunk || !n_chunks) fail(SLLM_E_INVALID, "chunk size must be positive");
    *n_chunks = ceil_div(length, chunk);
  });
}

sllm_status sllm_replica_slices(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t* lo_hi) {
  return guard([&] {
    if (!chunk || nranks < 1 || !lo_hi) fail(SLLM_E_INVALID, "bad slice arguments");
    const uint64_t k = ceil_div(length, chunk);
    for (int32_t r = 0; r < nranks; ++r) {
      uint64_t c0 = k * (uint64_t)r / (uint64_t)nranks, c1 = k * (uint64_t)(r + 1) / (uint64_t)nranks;
      lo_hi[2 * r] = std::min(c0 * chunk, length);
      lo_hi[2 * r + 1] = std::min(c1 * chunk, length);
    }
  });
}

sllm_status sllm_replica_round(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t round, uint64_t* lo_hi,
                               uint64_t* n_rounds) {
  return guard([&] {
    if (!chunk || nranks < 1 || !lo_hi) fail(SLLM_E_INVALID, "bad round arguments");
    std::vector<uint64_t> sl(2 * (size_t)nranks);
    if (sllm_replica_slices(length, chunk, nranks, sl.data()) != SLLM_OK) fail(SLLM_E_INVALID, "slice plan failed");
    uint64_t rounds = 0;
    for (int32_t q = 0; q < nranks; ++q) rounds = std::max(rounds, ceil_div(sl[2 * q + 1] - sl[2 * q], chunk));
    if (n_rounds) *n_rounds = rounds;
    if (round >= rounds) fail(SLLM_E_LOOKUP, "round out of range");
    for (int32_t q = 0; q < nranks; ++q) {
      uint64_t a = sl[2 * q] + round * chunk;
      bool has = a < sl[2 * q + 1];
      lo_hi[2 * q] = has ? a : 0;
      lo_hi[2 * q + 1] = has ? std::min(a + chunk, sl[2 * q + 1]) : 0;
    }
  });
}

sllm_status sllm_allgather_round(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t round, uint64_t* lo_hi,
                                 uint64_t* n_rounds, int32_t* full) {
  return guard([&] {
    if (!chunk || nranks < 1 || !lo_hi) fail(SLLM_E_INVALID, "bad round arguments");
    const uint64_t R = (uint64_t)nranks, nch = ceil_div(length, chunk), rounds = ceil_div(nch, R);
    if (n_rounds) *n_rounds = rounds;
    if (round >= rounds) fail(SLLM_E_LOOKUP, "round out of range");
    bool all = true;
    for (uint64_t q = 0; q < R; ++q) {
      const uint64_t k = round * R + q;
      const uint64_t a = k < nch ? k * chunk : 0, b = k < nch ? std::min(a + chunk, length) : 0;
      lo_hi[2 * q] = a;
      lo_hi[2 * q + 1] = b;
      all = all && b - a == chunk;
    }
    if (full) *full = all ? 1 : 0;
  });
}

sllm_status sllm_gpu_numa_node(int32_t gpu, int32_t* node) {
  return guard([&] {
    if (!node || gpu < 0) fail(SLLM_E_INVALID, "bad argument");
    *node = gpu_numa_node(gpu);
  });
}

sllm_status sllm_host_numa_node(const void* p, int32_t* node) {
  return guard([&] {
    if (!p || !node) fail(SLLM_E_INVALID, "null argument");
    *node = page_node(p);
  });
}

sllm_status sllm_fanout_unit(uint64_t chunk, int32_t fanout, uint64_t* unit) {
  return guard([&] {
    if (!chunk || !unit) fail(SLLM_E_INVALID, "bad fan-out unit arguments");
    *unit = fanout_unit(chunk, fanout);
  });
}

sllm_status sllm_host_alloc(uint64_t bytes, int32_t gpu, void** p) {
  return guard([&] {
    if (!p) fail(SLLM_E_INVALID, "null out");
    *p = host_alloc(bytes, gpu);
  });
}

void sllm_host_free(void* p) {
  guard([&] { host_free(p); });
}

sllm_status sllm_host_register(void* p, uint64_t bytes) {
  return guard([&] {
    if (!p || !bytes) fail(SLLM_E_INVALID, "null/empty buffer");
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(SLLM_E_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    }
  });
}

sllm_status sllm_host_unregister(void* p) {
  return guard([&] {
    cudaError_t e = cudaHostUnregister(p);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(SLLM_E_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
    }
  });
}

sllm_status sllm_host_read_partition(const char* dir, const sllm_index* idx, size_t p, void* dst, int32_t threads) {
  return guard([&] { read_partition(dir, idx, p, dst, threads); });
}

sllm_status sllm_comm_unique_id(void* id128) {
  return guard([&] { sllm_comm_unique_id_internal(id128); });
}

sllm_status sllm_comm_init_rank(const void* id128, int32_t nranks, int32_t rank, int32_t gpu, sllm_comm** out) {
  return guard_dev([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = sllm_comm_init_rank_internal(id128, nranks, rank, gpu);
  });
}

sllm_status sllm_comm_init_all(const int32_t* gpus, int32_t n, sllm_comm** out) {
  return guard_dev([&] { sllm_comm_init_all_internal(gpus, n, out); });
}

sllm_status sllm_comm_init_peers(int32_t nranks, int32_t rank, int32_t gpu, void* const* peer_base,
                                 uint32_t* const* peer_signal, uint64_t timeout_ms, sllm_comm** out) {
  return guard_dev([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = sllm_comm_init_peers_internal(nranks, rank, gpu, peer_base, peer_signal, timeout_ms);
  });
}

sllm_status sllm_comm_init_nvls(const int32_t* gpus, int32_t n, uint64_t bytes, uint64_t timeout_ms, sllm_comm** out) {
  return guard_dev([&] { sllm_comm_init_nvls_internal(gpus, n, bytes, timeout_ms, out); });
}

sllm_status sllm_comm_replica(const sllm_comm* c, void** base, uint64_t* bytes) {
  return guard([&] { sllm_comm_replica_internal(c, base, bytes); });
}

void sllm_comm_free(sllm_comm* c) {
  guard_dev([&] { sllm_comm_free_internal(c); });
}

sllm_status sllm_cache_create(uint64_t capacity, int32_t gpu, int32_t pin, sllm_cache** out) {
  return guard([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = cache_create(capacity, gpu, pin);
  });
}

sllm_status sllm_cache_acquire(sllm_cache* c, const char* dir, int32_t io_threads, const sllm_index** index,
                               void* const** part_bufs, int32_t* hit) {
  return guard([&] { cache_acquire(c, dir, io_threads, index, part_bufs, hit); });
}

sllm_status sllm_cache_release(sllm_cache* c, const char* dir) {
  return guard([&] { cache_release(c, dir); });
}

sllm_status sllm_cache_get_stats(sllm_cache* c, sllm_cache_stats* out) {
  return guard([&] { cache_stats(c, out); });
}

void sllm_cache_destroy(sllm_cache* c) {
  guard([&] { cache_destroy(c); });
}


sllm_status sllm_load_start(const sllm_index* idx, const sllm_load_config* cfg, const void* const* host_src,
                            const int32_t* gpu, void* const* dst_base, void* const* dst_tensor, void* const* stream,
                            sllm_comm* comm, sllm_load** out) {
  return guard_dev([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = sllm_load_create_internal(idx, cfg, host_src, gpu, dst_base, dst_tensor, stream, comm, nullptr, 0);
  });
}

sllm_status sllm_load_files_start(const sllm_index* idx, const sllm_load_config* cfg, const char* dir, const int32_t* gpu,
                                  void* const* dst_base, void* const* dst_tensor, void* const* stream, int32_t io_threads,
                                  sllm_comm* comm, sllm_load** out) {
  return guard_dev([&] {
    if (!out || !dir) fail(SLLM_E_INVALID, "null argument");
    *out = sllm_load_create_internal(idx, cfg, nullptr, gpu, dst_base, dst_tensor, stream, comm, dir, io_threads);
  });
}

sllm_status sllm_load_capture(const sllm_index* idx, const sllm_load_config* cfg, const void* const* host_src,
                              const int32_t* gpu, void* const* dst_base, void* const* dst_tensor, sllm_load** out) {
  return guard_dev([&] {
    if (!out) fail(SLLM_E_INVALID, "null out");
    *out = sllm_load_create_internal(idx, cfg, host_src, gpu, dst_base, dst_tensor, nullptr, nullptr, nullptr, 0, true);
  });
}

sllm_status sllm_load_replay(sllm_load* load, void* const* stream) {
  return guard_dev([&] {
    if (!load) fail(SLLM_E_INVALID, "null load");
    sllm_load_replay_internal(load, stream);
  });
}

sllm_status sllm_load_wait(sllm_load* load, sllm_load_report* rep) {
  sllm_status st = SLLM_OK;
  sllm_status g = guard_dev([&] {
    if (!load) fail(SLLM_E_INVALID, "null load");
    st = sllm_load_wait_internal(load, rep);
  });
  return g != SLLM_OK ? g : st;
}

sllm_status sllm_load_tensor(const sllm_load* load, const char* name, sllm_tensor_handle* h) {
  return guard([&] {
    if (!load) fail(SLLM_E_INVALID, "null load");
    sllm_load_tensor_internal(load, name, h);
  });
}

sllm_status sllm_load_block_checksums(const sllm_load* load, size_t p, const uint64_t** table) {
  return guard_dev([&] {
    if (!load || !table) fail(SLLM_E_INVALID, "null argument");
    sllm_load_block_checksums_internal(const_cast<sllm_load*>(load), p, table);
  });
}

void sllm_load_free(sllm_load* load) {
  if (load) guard_dev([&] { sllm_load_free_internal(load); });
}

sllm_status sllm_device_trim(int32_t gpu, uint64_t keep_bytes) {
  return guard_dev([&] { sllm_device_trim_internal(gpu, keep_bytes); });
}

sllm_status sllm_block_checksums_device(const void* src_dev, uint64_t len, uint64_t block, uint64_t* out_dev,
                                        int32_t ctas, void* stream) {
  return guard_dev([&] { block_checksums_device(src_dev, len, block, out_dev, ctas, static_cast<cudaStream_t>(stream)); });
}

sllm_status sllm_materialise_device(const sllm_index* idx, size_t p, const void* src_dev, void* const* dst_tensor,
                                    int32_t ctas, void* stream, uint64_t* bad_block, float* kernel_ms) {
  return guard_dev([&] {
    uint64_t bad = materialise_device(idx, p, src_dev, dst_tensor, ctas, static_cast<cudaStream_t>(stream), kernel_ms);
    if (bad_block) *bad_block = bad;
    if (bad != ~0ull) fail(SLLM_E_CHECKSUM, "checksum mismatch in partition " + std::to_string(p) + ", block " +
                                                std::to_string(bad));
  });
}

}  // extern "C"

namespace sllm {
void ipc_export(const void* ptr, uint64_t nbytes, sllm_ipc_region* out);
void* ipc_open(const sllm_ipc_region* r);
void ipc_close(void* p);
}  // namespace sllm

extern "C" {

sllm_status sllm_ipc_export(const void* dev_ptr, uint64_t nbytes, sllm_ipc_region* out) {
  return guard_dev([&] { ipc_export(dev_ptr, nbytes, out); });
}

sllm_status sllm_ipc_open(const sllm_ipc_region* region, void** dev_ptr) {
  return guard_dev([&] {
    if (!dev_ptr) fail(SLLM_E_INVALID, "null out");
    *dev_ptr = ipc_open(region);
  });
}

sllm_status sllm_ipc_close(void* dev_ptr) {
  return guard_dev([&] { ipc_close(dev_ptr); });
}

}  // extern "C"
