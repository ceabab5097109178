// Loading-optimized checkpoint format: layout planner, partition writer, block
// checksums and the binary index codec.
//
//   PAPER.md P:545-547 (§Loading-Optimized Checkpoints): "tensors for each GPU are
//   grouped in partitions ... contain only the binary data ... a tensor index file ...
//   maps tensor names to a tuple of GPU id, offset, and size ... The tensors are
//   aligned with memory word sizes".  SPEC.md S:43-91 (convert / read_index).
//   Readings Q1-Q7 and the index record layout: DESIGN.md §Format.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <thread>

#include "common.hpp"

namespace sllm {

static constexpr uint64_t kM = 0xFFFFFFFFull;
static const char kMagic[8] = {'S', 'L', 'L', 'M', 'I', 'D', 'X', '1'};
static constexpr uint32_t kVersion = 1;
static constexpr uint32_t kFlagChecksums = 1;

int dtype_width(int32_t dt) {
  switch (dt) {
    case SLLM_F16: case SLLM_BF16: case SLLM_I16: return 2;
    case SLLM_F32: case SLLM_I32: return 4;
    case SLLM_I8: case SLLM_U8: case SLLM_BOOL: case SLLM_F8_E4M3: case SLLM_F8_E5M2: return 1;
    case SLLM_I64: case SLLM_F64: return 8;
    default: return 0;
  }
}

int default_threads() {
  unsigned n = std::thread::hardware_concurrency();
  return n ? (int)std::min(n, 32u) : 4;
}

static std::atomic<uint64_t> g_serial{1};

// ---------------------------------------------------------------------------------
// Fletcher-64 over little-endian u32 words, modulus 2^32-1 (Q8).  Sequential
// recurrence s1 += w, s2 += s1 with lazy end-around-carry folding every 2^15 words:
// from s1, s2 < 2^32, after m <= 2^15 words s1 < 2^48 and s2 < 2^62, so no overflow.
// ---------------------------------------------------------------------------------
static inline uint64_t fold(uint64_t x) {
  x = (x & kM) + (x >> 32);
  x = (x & kM) + (x >> 32);
  return x >= kM ? x - kM : x;
}

uint64_t fletcher64(const uint8_t* p, uint64_t nbytes) {
  uint64_t s1 = 0, s2 = 0;
  uint64_t nw = nbytes / 4;
  while (nw) {
    uint64_t m = std::min<uint64_t>(nw, 1u << 15);
    for (uint64_t k = 0; k < m; ++k) {
      uint32_t w;
      std::memcpy(&w, p + 4 * k, 4);
      s1 += w;
      s2 += s1;
    }
    s1 = fold(s1);
    s2 = fold(s2);
    p += 4 * m;
    nw -= m;
  }
  uint64_t tail = nbytes % 4;
  if (tail) {
    uint32_t w = 0;
    std::memcpy(&w, p, tail);
    s1 = fold(s1 + w);
    s2 = fold(s2 + s1);
  }
  return (s2 << 32) | s1;
}

// Run fn(i) for i in [0, n) on up to `threads` threads (dynamic scheduling).
template <class F>
static void parallel_for(size_t n, int threads, F fn) {
  if (n == 0) return;
  threads = std::max(1, std::min<int>(threads, (int)n));
  std::atomic<size_t> next{0};
  auto body = [&] {
    for (size_t i; (i = next.fetch_add(1)) < n;) fn(i);
  };
  std::vector<std::thread> pool;  // (worker threads only: jobs may re-bind their thread's NUMA affinity)
  for (int t = 0; t < threads; ++t) pool.emplace_back(body);
  for (auto& th : pool) th.join();
}

// Converter threads fill / checksum a partition's pinned buffer from the CPUs of the node its
// pages live on (numa.cpp; no-op on single-node hosts).
static void follow_pages(const void* buf) {
  static thread_local const void* last = nullptr;
  if (numa_nodes() <= 1 || buf == last) return;
  last = buf;
  bind_thread_to_node(page_node(buf));
}

// ---------------------------------------------------------------------------------
// Layout: devices ascending; per device, source order,
// offset = align_up(cursor, A), cursor = offset + size; L_d = align_up(cursor, A).
// ---------------------------------------------------------------------------------
static void check_params(uint64_t align, uint64_t block) {
  if (!is_pow2(align) || align < 16) fail(SLLM_E_INVALID, "alignment must be a power of two >= 16");
  if (block != 0 && (!is_pow2(block) || block % align))
    fail(SLLM_E_INVALID, "block size must be 0 or a power of two multiple of the alignment");
  // DESIGN.md Q8: the device kernels fold their 64-bit Fletcher partial sums once per
  // stage / tile; blocks up to kMaxBlock keep every unfolded sum below 2^64
  if (align > kMaxBlock || block > kMaxBlock) fail(SLLM_E_INVALID, "alignment / block size above 256 MiB");
}

static void finish_index(sllm_index* idx) {
  // per-partition tensor lists sorted by offset (used by the scatter planner)
  for (auto& p : idx->parts) p.by_offset.clear();
  for (uint32_t i = 0; i < idx->tensors.size(); ++i) idx->parts[idx->tensors[i].part].by_offset.push_back(i);
  auto by_off = [&](uint32_t a, uint32_t b) { return idx->tensors[a].offset < idx->tensors[b].offset; };
  for (auto& p : idx->parts)  // (source order is offset order for converter-written indexes)
    if (!std::is_sorted(p.by_offset.begin(), p.by_offset.end(), by_off))
      std::stable_sort(p.by_offset.begin(), p.by_offset.end(), by_off);
  idx->serial = g_serial.fetch_add(1);
}

sllm_index* plan(const sllm_src_tensor* t, size_t n, uint64_t align, uint64_t block, const char* model_id) {
  check_params(align, block);
  if (n && !t) fail(SLLM_E_INVALID, "null tensor array");
  std::unique_ptr<sllm_index> idx(new sllm_index);
  idx->align = align;
  idx->block = block;
  idx->model_id = model_id ? model_id : "";
  std::vector<int32_t> devs;
  idx->tensors.resize(n);
  idx->by_name.reserve(n);
  size_t name_bytes = 0;
  for (size_t i = 0; i < n; ++i) name_bytes += (t[i].name ? std::strlen(t[i].name) : 0) + 1;
  idx->names.reserve(name_bytes);  // (no reallocation below: the views stay valid)
  for (size_t i = 0; i < n; ++i) {
    const sllm_src_tensor& s = t[i];
    if (!s.name || !s.name[0]) fail(SLLM_E_CONVERSION, "empty tensor name");
    TensorRec& r = idx->tensors[i];
    const size_t at = idx->names.size(), len = std::strlen(s.name);
    idx->names.append(s.name, len + 1);
    r.name = std::string_view(idx->names.data() + at, len);
    const std::string name(r.name);
    if (!idx->by_name.insert(r.name, (uint32_t)i, idx->tensors))
      fail(SLLM_E_CONVERSION, "duplicate tensor name '" + name + "'");
    int w = dtype_width(s.dtype);
    if (!w) fail(SLLM_E_CONVERSION, "unknown dtype for '" + name + "'");
    if (s.device_id < 0) fail(SLLM_E_CONVERSION, "negative device id for '" + name + "'");
    if (s.ndim < 0 || s.ndim > SLLM_MAX_NDIM || (s.ndim > 0 && !s.shape))
      fail(SLLM_E_CONVERSION, "bad rank for '" + name + "'");
    unsigned __int128 numel = 1;
    r.device = s.device_id;
    r.dtype = s.dtype;
    r.ndim = s.ndim;
    std::memset(r.shape, 0, sizeof r.shape);
    for (int k = 0; k < s.ndim; ++k) {
      if (s.shape[k] <= 0) fail(SLLM_E_CONVERSION, "non-positive dimension in '" + name + "'");
      r.shape[k] = s.shape[k];
      numel *= (uint64_t)s.shape[k];
      if (numel >> 62) fail(SLLM_E_CONVERSION, "tensor too large: '" + name + "'");
    }
    if ((unsigned __int128)s.nbytes != numel * (unsigned)w)
      fail(SLLM_E_CONVERSION, "payload of '" + name + "' != prod(shape) * width");
    r.nbytes = s.nbytes;
    devs.push_back(s.device_id);
  }
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  std::unordered_map<int32_t, int32_t> part_of;
  for (size_t p = 0; p < devs.size(); ++p) {
    part_of[devs[p]] = (int32_t)p;
    PartRec pr{};
    pr.device = devs[p];
    idx->parts.push_back(pr);
  }
  std::vector<uint64_t> cursor(devs.size(), 0);
  for (auto& r : idx->tensors) {  // source order within each device
    int32_t p = part_of[r.device];
    r.part = p;
    r.offset = align_up(cursor[p], align);
    cursor[p] = r.offset + r.nbytes;
    idx->parts[p].n_tensors++;
    idx->payload += r.nbytes;
  }
  for (size_t p = 0; p < devs.size(); ++p) {
    PartRec& pr = idx->parts[p];
    pr.length = align_up(cursor[p], align);
    pr.n_blocks = block ? ceil_div(pr.length, block) : 0;
    pr.checksums.assign(pr.n_blocks, 0);
  }
  finish_index(idx.get());
  return idx.release();
}

void seal(sllm_index* idx, const void* const* part_bufs) {
  if (!part_bufs && !idx->parts.empty()) fail(SLLM_E_INVALID, "null partition buffer array");
  if (idx->block) {
    struct Job { size_t p; uint64_t j; };
    std::vector<Job> jobs;
    for (size_t p = 0; p < idx->parts.size(); ++p)
      if (part_bufs[p])  // NULL: partition not held by this process, table left as is
        for (uint64_t j = 0; j < idx->parts[p].n_blocks; ++j) jobs.push_back({p, j});
    parallel_for(jobs.size(), default_threads(), [&](size_t i) {
      const PartRec& pr = idx->parts[jobs[i].p];
      uint64_t lo = jobs[i].j * idx->block;
      uint64_t len = std::min(idx->block, pr.length - lo);
      follow_pages(part_bufs[jobs[i].p]);
      idx->parts[jobs[i].p].checksums[jobs[i].j] =
          fletcher64(static_cast<const uint8_t*>(part_bufs[jobs[i].p]) + lo, len);
    });
  }
  idx->sealed = true;
}

// Copy every tensor's payload to its slot, zero every other byte (Q3) and compute the
// block checksums -- fused per checksum block: a worker fills block j (tensor pieces and
// padding, in offset order) and checksums it while it is still in its core's cache, so
// the partition bytes are written once and never re-read from DRAM (a separate seal pass
// would read all of them again).
void convert_into(const sllm_src_tensor* t, size_t n, sllm_index* idx, void* const* part_bufs) {
  if (n != idx->tensors.size()) fail(SLLM_E_INVALID, "tensor count differs from the plan");
  if (!part_bufs && !idx->parts.empty()) fail(SLLM_E_INVALID, "null partition buffer array");
  for (size_t p = 0; p < idx->parts.size(); ++p)
    if (!part_bufs[p]) fail(SLLM_E_INVALID, "null partition buffer");
  for (size_t i = 0; i < n; ++i) {
    const TensorRec& r = idx->tensors[i];
    if (std::strcmp(t[i].name ? t[i].name : "", r.name.data()) || t[i].nbytes != r.nbytes)
      fail(SLLM_E_CONVERSION, "tensor " + std::to_string(i) + " differs from the plan");
    if (!t[i].data) fail(SLLM_E_INVALID, "null data for '" + std::string(r.name) + "'");
  }
  const uint64_t B = idx->block ? idx->block : (4ull << 20);  // work unit: one checksum block
  struct Job { size_t p; uint64_t j; };
  std::vector<Job> jobs;
  for (size_t p = 0; p < idx->parts.size(); ++p)
    for (uint64_t j = 0; j < ceil_div(idx->parts[p].length, B); ++j) jobs.push_back({p, j});
  parallel_for(jobs.size(), default_threads(), [&](size_t i) {
    PartRec& pr = idx->parts[jobs[i].p];
    uint8_t* base = static_cast<uint8_t*>(part_bufs[jobs[i].p]);
    follow_pages(base);
    const uint64_t lo = jobs[i].j * B, hi = std::min(lo + B, pr.length);
    // first tensor (in offset order) that ends after lo
    auto it = std::partition_point(pr.by_offset.begin(), pr.by_offset.end(), [&](uint32_t ti) {
      return idx->tensors[ti].offset + idx->tensors[ti].nbytes <= lo;
    });
    uint64_t cur = lo;
    for (; it != pr.by_offset.end(); ++it) {
      const TensorRec& r = idx->tensors[*it];
      if (r.offset >= hi) break;
      const uint64_t a = std::max(r.offset, lo), b = std::min(r.offset + r.nbytes, hi);
      if (a > cur) std::memset(base + cur, 0, a - cur);
      std::memcpy(base + a, static_cast<const uint8_t*>(t[*it].data) + (a - r.offset), b - a);
      cur = b;
    }
    if (hi > cur) std::memset(base + cur, 0, hi - cur);
    if (idx->block) pr.checksums[jobs[i].j] = fletcher64(base + lo, hi - lo);
  });
  idx->sealed = true;
}

// ---------------------------------------------------------------------------------
// Index codec (DESIGN.md §Index format; "little-endian binary record stream
// with a magic number and format_version=1").
// ---------------------------------------------------------------------------------
namespace {
struct Writer {
  std::vector<uint8_t> b;
  template <class T> void put(T v) {
    uint8_t tmp[sizeof(T)];
    std::memcpy(tmp, &v, sizeof(T));
    b.insert(b.end(), tmp, tmp + sizeof(T));
  }
  void bytes(const void* p, size_t n) { b.insert(b.end(), (const uint8_t*)p, (const uint8_t*)p + n); }
  void pad8() { b.resize(align_up(b.size(), 8), 0); }
};

struct Reader {
  const uint8_t* b;
  size_t pos, limit;
  const uint8_t* take(size_t n) {
    if (n > limit - pos) fail(SLLM_E_FORMAT, "truncated index at byte " + std::to_string(pos));
    const uint8_t* p = b + pos;
    pos += n;
    return p;
  }
  template <class T> T get() {
    T v;
    std::memcpy(&v, take(sizeof(T)), sizeof(T));
    return v;
  }
  void pad8() {
    size_t n = align_up(pos, 8) - pos;
    const uint8_t* p = take(n);
    for (size_t i = 0; i < n; ++i)
      if (p[i]) fail(SLLM_E_FORMAT, "non-zero padding");
  }
};
}  // namespace

std::vector<uint8_t> serialize(const sllm_index& idx) {
  Writer w;
  w.bytes(kMagic, 8);
  w.put<uint32_t>(kVersion);
  w.put<uint32_t>(idx.block ? kFlagChecksums : 0);
  w.put<uint64_t>(idx.align);
  w.put<uint64_t>(idx.block);
  w.put<uint32_t>((uint32_t)idx.parts.size());
  w.put<uint32_t>((uint32_t)idx.tensors.size());
  w.put<uint64_t>(idx.payload);
  w.put<uint32_t>((uint32_t)idx.model_id.size());
  w.bytes(idx.model_id.data(), idx.model_id.size());
  w.pad8();
  for (const auto& p : idx.parts) {
    w.put<int32_t>(p.device);
    w.put<uint32_t>(0);
    w.put<uint64_t>(p.length);
    w.put<uint64_t>(p.n_tensors);
    w.put<uint64_t>(p.n_blocks);
  }
  for (const auto& r : idx.tensors) {
    w.put<uint32_t>((uint32_t)r.name.size());
    w.bytes(r.name.data(), r.name.size());
    w.put<int32_t>(r.device);
    w.put<uint8_t>((uint8_t)r.dtype);
    w.put<uint8_t>((uint8_t)r.ndim);
    w.put<uint16_t>(0);
    w.put<uint64_t>(r.offset);
    w.put<uint64_t>(r.nbytes);
    for (int k = 0; k < r.ndim; ++k) w.put<int64_t>(r.shape[k]);
    w.pad8();
  }
  if (idx.block)
    for (const auto& p : idx.parts)
      for (uint64_t c : p.checksums) w.put<uint64_t>(c);
  w.put<uint64_t>(fletcher64(w.b.data(), w.b.size()));
  w.put<uint64_t>(w.b.size() + 8);
  return std::move(w.b);
}

static bool valid_utf8(const uint8_t* s, size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {  // ASCII fast path, 8 bytes at a time
    uint64_t w;
    std::memcpy(&w, s + i, 8);
    if (w & 0x8080808080808080ull) break;
  }
  while (i < n) {
    uint8_t c = s[i];
    size_t k;
    uint32_t cp;
    if (c < 0x80) { ++i; continue; }
    else if ((c & 0xE0) == 0xC0) { k = 1; cp = c & 0x1F; }
    else if ((c & 0xF0) == 0xE0) { k = 2; cp = c & 0x0F; }
    else if ((c & 0xF8) == 0xF0) { k = 3; cp = c & 0x07; }
    else return false;
    for (size_t j = 1; j <= k; ++j) {
      if (i + j >= n || (s[i + j] & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (s[i + j] & 0x3F);
    }
    if ((k == 1 && cp < 0x80) || (k == 2 && cp < 0x800) || (k == 3 && (cp < 0x10000 || cp > 0x10FFFF)) ||
        (cp >= 0xD800 && cp <= 0xDFFF))
      return false;
    i += k + 1;
  }
  return true;
}

sllm_index* parse(const uint8_t* blob, size_t n) {
  if (!blob && n) fail(SLLM_E_INVALID, "null index blob");
  if (n < 16 + 56) fail(SLLM_E_FORMAT, "index too short (" + std::to_string(n) + " bytes)");
  if (n % 8) fail(SLLM_E_FORMAT, "index length not a multiple of 8");
  uint64_t cs_stored, total;
  std::memcpy(&cs_stored, blob + n - 16, 8);
  std::memcpy(&total, blob + n - 8, 8);
  if (total != n) fail(SLLM_E_FORMAT, "trailer length differs from the file length");
  if (fletcher64(blob, n - 16) != cs_stored) fail(SLLM_E_FORMAT, "index self-checksum mismatch");
  Reader r{blob, 0, n - 16};
  if (std::memcmp(r.take(8), kMagic, 8)) fail(SLLM_E_FORMAT, "bad magic");
  uint32_t version = r.get<uint32_t>(), flags = r.get<uint32_t>();
  uint64_t A = r.get<uint64_t>(), B = r.get<uint64_t>();
  uint32_t n_parts = r.get<uint32_t>(), n_tensors = r.get<uint32_t>();
  uint64_t payload = r.get<uint64_t>();
  uint32_t mid_len = r.get<uint32_t>();
  if (version != kVersion) fail(SLLM_E_FORMAT, "unsupported version");
  if (flags & ~kFlagChecksums) fail(SLLM_E_FORMAT, "unknown flag bits");
  if (!is_pow2(A) || A < 16) fail(SLLM_E_FORMAT, "bad alignment");
  bool has_cs = flags & kFlagChecksums;
  if (has_cs ? (!is_pow2(B) || B % A) : B != 0) fail(SLLM_E_FORMAT, "bad block size");
  if (A > kMaxBlock || B > kMaxBlock) fail(SLLM_E_FORMAT, "alignment / block size above 256 MiB");
  std::unique_ptr<sllm_index> idx(new sllm_index);
  idx->align = A;
  idx->block = B;
  const uint8_t* mid = r.take(mid_len);
  if (!valid_utf8(mid, mid_len)) fail(SLLM_E_FORMAT, "model id not UTF-8");
  idx->model_id.assign((const char*)mid, mid_len);
  r.pad8();
  std::unordered_map<int32_t, int32_t> part_of;
  for (uint32_t p = 0; p < n_parts; ++p) {
    PartRec pr{};
    pr.device = r.get<int32_t>();
    if (r.get<uint32_t>() != 0) fail(SLLM_E_FORMAT, "non-zero reserved field");
    pr.length = r.get<uint64_t>();
    pr.n_tensors = r.get<uint64_t>();
    pr.n_blocks = r.get<uint64_t>();
    if (pr.device < 0 || (p && pr.device <= idx->parts.back().device))
      fail(SLLM_E_FORMAT, "partition device ids not strictly ascending");
    if (pr.length == 0 || pr.length % A) fail(SLLM_E_FORMAT, "partition length not a positive multiple of A");
    if (pr.n_blocks != (has_cs ? ceil_div(pr.length, B) : 0)) fail(SLLM_E_FORMAT, "block count mismatch");
    if (pr.n_tensors == 0) fail(SLLM_E_FORMAT, "partition without tensors");
    part_of[pr.device] = (int32_t)p;
    idx->parts.push_back(std::move(pr));
  }
  std::vector<uint64_t> count(n_parts, 0);
  uint64_t sum = 0;
  // every tensor record takes >= 32 bytes: a count the blob cannot hold is rejected before
  // anything is sized by it
  if ((uint64_t)n_tensors * 32 > r.limit - r.pos) fail(SLLM_E_FORMAT, "tensor count exceeds the index length");
  idx->tensors.reserve(n_tensors);
  idx->by_name.reserve(n_tensors);
  idx->names.reserve(r.limit - r.pos);  // every name (+ its NUL) fits the bytes left: no reallocation
  for (uint32_t i = 0; i < n_tensors; ++i) {
    TensorRec t{};
    uint32_t nl = r.get<uint32_t>();
    if (nl == 0) fail(SLLM_E_FORMAT, "empty tensor name");
    const uint8_t* nm = r.take(nl);
    if (!valid_utf8(nm, nl)) fail(SLLM_E_FORMAT, "tensor name not UTF-8");
    const size_t at = idx->names.size();
    idx->names.append((const char*)nm, nl);
    idx->names.push_back('\0');
    t.name = std::string_view(idx->names.data() + at, nl);
    t.device = r.get<int32_t>();
    t.dtype = r.get<uint8_t>();
    t.ndim = r.get<uint8_t>();
    if (r.get<uint16_t>() != 0) fail(SLLM_E_FORMAT, "non-zero reserved field");
    t.offset = r.get<uint64_t>();
    t.nbytes = r.get<uint64_t>();
    auto it = part_of.find(t.device);
    if (it == part_of.end()) fail(SLLM_E_FORMAT, "tensor '" + std::string(t.name) + "' on an unknown device");
    t.part = it->second;
    int w = dtype_width(t.dtype);
    if (!w) fail(SLLM_E_FORMAT, "unknown dtype code");
    if (t.ndim > SLLM_MAX_NDIM) fail(SLLM_E_FORMAT, "rank above 8");
    unsigned __int128 numel = 1;
    for (int k = 0; k < t.ndim; ++k) {
      t.shape[k] = r.get<int64_t>();
      if (t.shape[k] <= 0) fail(SLLM_E_FORMAT, "non-positive dimension in '" + std::string(t.name) + "'");
      numel *= (uint64_t)t.shape[k];
      if (numel >> 62) fail(SLLM_E_FORMAT, "tensor too large");
    }
    r.pad8();
    if (numel * (unsigned)w != (unsigned __int128)t.nbytes) fail(SLLM_E_FORMAT, "size of '" + std::string(t.name) + "' != prod(shape) * width");
    if (t.offset % A) fail(SLLM_E_FORMAT, "offset of '" + std::string(t.name) + "' not aligned");
    const PartRec& pr = idx->parts[t.part];
    if (t.offset > pr.length || t.nbytes > pr.length - t.offset) fail(SLLM_E_FORMAT, "'" + std::string(t.name) + "' extends past its partition");
    count[t.part]++;
    sum += t.nbytes;
    idx->tensors.push_back(t);
    if (!idx->by_name.insert(t.name, i, idx->tensors))
      fail(SLLM_E_FORMAT, "duplicate tensor name '" + std::string(t.name) + "'");
  }
  for (uint32_t p = 0; p < n_parts; ++p)
    if (count[p] != idx->parts[p].n_tensors) fail(SLLM_E_FORMAT, "partition tensor count mismatch");
  if (sum != payload) fail(SLLM_E_FORMAT, "payload_bytes mismatch");
  idx->payload = payload;
  finish_index(idx.get());
  for (const auto& pr : idx->parts)
    for (size_t k = 1; k < pr.by_offset.size(); ++k) {
      const TensorRec& a = idx->tensors[pr.by_offset[k - 1]];
      const TensorRec& b = idx->tensors[pr.by_offset[k]];
      if (b.offset < a.offset + a.nbytes) fail(SLLM_E_FORMAT, "overlapping tensors '" + std::string(a.name) + "' and '" + std::string(b.name) + "'");
    }
  {  // the checksum tables must fit the bytes left before the trailer (n_blocks comes from L_d)
    unsigned __int128 need = 0;
    for (const auto& pr : idx->parts) need += (unsigned __int128)pr.n_blocks * 8;
    if (need > r.limit - r.pos) fail(SLLM_E_FORMAT, "checksum tables exceed the index length");
  }
  for (auto& pr : idx->parts) {
    pr.checksums.resize(pr.n_blocks);
    for (auto& c : pr.checksums) {
      c = r.get<uint64_t>();
      if ((c & kM) == kM || (c >> 32) == kM) fail(SLLM_E_FORMAT, "non-canonical block checksum");
    }
  }
  if (r.pos != n - 16) fail(SLLM_E_FORMAT, "records do not end at the trailer");
  idx->sealed = true;
  return idx.release();
}

}  // namespace sllm
