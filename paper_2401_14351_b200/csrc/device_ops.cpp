// Device-resident entry points of the kernels (K4 checksum, K3 scatter) for partitions
// already in HBM -- also how bench.py measures them standalone against the HBM roofline.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "runtime.hpp"

namespace sllm {

// Kernel engine of the standalone entry points: kDefaultEngine, or SLLM_STANDALONE_ENGINE
// = ldg | tma | tma_store (a measurement knob for A/B runs of the same kernel family).
static int standalone_engine() {
  const char* e = getenv("SLLM_STANDALONE_ENGINE");
  if (!e || !*e) return kDefaultEngine;
  if (!strcmp(e, "ldg")) return 0;
  if (!strcmp(e, "tma")) return 1;
  if (!strcmp(e, "tma_store")) return 2;
  fail(SLLM_E_INVALID, std::string("SLLM_STANDALONE_ENGINE: unknown engine '") + e + "'");
}

void block_checksums_device(const void* src, uint64_t len, uint64_t block, uint64_t* out, int ctas,
                            cudaStream_t st) {
  if (!src || !out || !block) fail(SLLM_E_INVALID, "null argument");
  if (len % 16) fail(SLLM_E_INVALID, "length must be a multiple of 16");
  if (!is_pow2(block) || block < 16) fail(SLLM_E_INVALID, "block must be a power of two >= 16");
  if (len == 0) return;
  const uint64_t nb = ceil_div(len, block);
  const uint32_t tile = (uint32_t)std::min<uint64_t>(kTile, block);
  void* scratch = nullptr;
  const size_t acc_bytes = align_up(nb * sizeof(BlockAcc), 256);
  SLLM_CUDA(cudaMallocAsync(&scratch, acc_bytes + 256 + 256, st));
  uint8_t* b = static_cast<uint8_t*>(scratch);
  Seg* seg = reinterpret_cast<Seg*>(b + acc_bytes);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(b + acc_bytes + 128);
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(b + acc_bytes + 256);
  SLLM_CUDA(cudaMemsetAsync(b, 0, acc_bytes + 512, st));
  SLLM_CUDA(launch_init_seg(seg, len, st));  // (a pageable upload would synchronise the stream)
  MatParams mp{};
  mp.src = static_cast<const uint8_t*>(src);
  mp.lo = 0;
  mp.hi = len;
  mp.segs = seg;
  mp.seg_begin = 0;
  mp.seg_end = 1;
  mp.tile = tile;
  mp.block = block;
  mp.part_len = len;
  mp.acc = reinterpret_cast<BlockAcc*>(b);
  mp.cs_out = out;
  mp.bad = bad;
  mp.engine = standalone_engine();
  if (!getenv("SLLM_STATIC_UNITS")) mp.ticket = ticket;  // dynamic unit distribution (base 0)
  static const bool ktime = getenv("SLLM_KTIME") != nullptr;  // diagnostic: in-kernel span on stderr
  if (ktime) mp.ktime = reinterpret_cast<unsigned long long*>(b + acc_bytes + 320);
  SLLM_CUDA(launch_materialise(mp, MatKind::kChecksumOnly, ctas > 0 ? ctas : 0, st));
  if (ktime) {
    unsigned long long kt[4];
    SLLM_CUDA(cudaMemcpyAsync(kt, mp.ktime, sizeof(kt), cudaMemcpyDeviceToHost, st));
    SLLM_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "sllm-ktime bytes=%llu span_ms=%.4f end_spread_us=%.2f\n", (unsigned long long)len,
            (kt[3] - ~kt[0]) * 1e-6, (kt[3] - ~kt[2]) * 1e-3);
  }
  SLLM_CUDA(cudaFreeAsync(scratch, st));
}

uint64_t materialise_device(const sllm_index* idx, size_t p, const void* src, void* const* dst_tensor, int ctas,
                            cudaStream_t st, float* kernel_ms) {
  if (!idx || !src || !dst_tensor) fail(SLLM_E_INVALID, "null argument");
  if (p >= idx->parts.size()) fail(SLLM_E_LOOKUP, "partition index out of range");
  const PartRec& pr = idx->parts[p];
  std::vector<Seg> segs;
  uint64_t cur = 0;
  for (uint32_t ti : pr.by_offset) {
    const TensorRec& t = idx->tensors[ti];
    if (!dst_tensor[ti] || (reinterpret_cast<uintptr_t>(dst_tensor[ti]) & 15))
      fail(SLLM_E_INVALID, "destination of '" + std::string(t.name) + "' is null or not 16-byte aligned");
    if (t.offset > cur) segs.push_back(Seg{cur, t.offset - cur, nullptr, 0});
    uint64_t end16 = align_up(t.offset + t.nbytes, 16);
    segs.push_back(Seg{t.offset, end16 - t.offset, static_cast<uint8_t*>(dst_tensor[ti]), t.nbytes});
    cur = end16;
  }
  if (pr.length > cur) segs.push_back(Seg{cur, pr.length - cur, nullptr, 0});
  const uint64_t nb = std::max<uint64_t>(pr.n_blocks, 1);
  const size_t seg_bytes = align_up(segs.size() * sizeof(Seg), 256);
  const size_t acc_bytes = align_up(nb * sizeof(BlockAcc), 256);
  const size_t tab = align_up(nb * 8, 256);
  std::vector<uint32_t> gran;
  gran_table(segs, pr.length, kGranShift, gran);
  const size_t gran_bytes = align_up(gran.size() * 4, 256);
  void* scratch = nullptr;
  SLLM_CUDA(cudaMallocAsync(&scratch, seg_bytes + acc_bytes + tab + 256 + gran_bytes + 256, st));
  uint8_t* b = static_cast<uint8_t*>(scratch);
  Seg* d_segs = reinterpret_cast<Seg*>(b);
  BlockAcc* d_acc = reinterpret_cast<BlockAcc*>(b + seg_bytes);
  uint64_t* d_expect = reinterpret_cast<uint64_t*>(b + seg_bytes + acc_bytes);
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(b + seg_bytes + acc_bytes + tab);
  uint32_t* d_gran = reinterpret_cast<uint32_t*>(b + seg_bytes + acc_bytes + tab + 256);
  unsigned long long* d_ticket = reinterpret_cast<unsigned long long*>(b + seg_bytes + acc_bytes + tab + 256 + gran_bytes);
  SLLM_CUDA(cudaMemsetAsync(d_ticket, 0, 8, st));
  SLLM_CUDA(cudaMemcpyAsync(d_gran, gran.data(), gran.size() * 4, cudaMemcpyHostToDevice, st));
  SLLM_CUDA(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(Seg), cudaMemcpyHostToDevice, st));
  SLLM_CUDA(cudaMemsetAsync(d_acc, 0, acc_bytes, st));
  SLLM_CUDA(cudaMemsetAsync(d_bad, 0xFF, 8, st));
  const bool check = idx->block != 0;
  if (check) SLLM_CUDA(cudaMemcpyAsync(d_expect, pr.checksums.data(), pr.n_blocks * 8, cudaMemcpyHostToDevice, st));
  MatParams mp{};
  mp.src = static_cast<const uint8_t*>(src);
  mp.lo = 0;
  mp.hi = pr.length;
  mp.segs = d_segs;
  mp.seg_begin = 0;
  mp.seg_end = (uint32_t)segs.size();
  mp.gran_seg = d_gran;
  mp.gran_shift = kGranShift;
  mp.tile = idx->block ? (uint32_t)std::min<uint64_t>(kTile, idx->block) : kTile;
  mp.block = idx->block ? idx->block : kTile;
  mp.part_len = pr.length;
  mp.acc = d_acc;
  mp.expect = check ? d_expect : nullptr;
  mp.bad = d_bad;
  mp.engine = standalone_engine();
  if (!getenv("SLLM_STATIC_UNITS")) mp.ticket = d_ticket;  // dynamic unit distribution (base 0)
  cudaEvent_t ev[2] = {};
  if (kernel_ms)
    for (auto& e : ev) SLLM_CUDA(cudaEventCreate(&e));
  if (kernel_ms) SLLM_CUDA(cudaEventRecord(ev[0], st));
  SLLM_CUDA(launch_materialise(mp, check ? MatKind::kCopyChecksum : MatKind::kCopyOnly, ctas > 0 ? ctas : 0, st));
  if (kernel_ms) SLLM_CUDA(cudaEventRecord(ev[1], st));
  unsigned long long bad = ~0ull;
  SLLM_CUDA(cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, st));
  SLLM_CUDA(cudaStreamSynchronize(st));
  if (kernel_ms) {
    SLLM_CUDA(cudaEventElapsedTime(kernel_ms, ev[0], ev[1]));
    for (auto& e : ev) cudaEventDestroy(e);
  }
  SLLM_CUDA(cudaFreeAsync(scratch, st));
  return bad;
}

}  // namespace sllm
