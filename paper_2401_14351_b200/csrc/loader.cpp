// The load path: one host worker thread per partition drives a chunk pipeline on a
// few CUDA streams of its GPU.
//
//   PAPER.md P:576-602 (§Multi-Tier Loading Subsystem): chunk-based data management,
//   "parallel DRAM-to-GPU PCIe links", pinned memory ("one thread is enough" P:692),
//   a task-queue pipeline of (offset, size) chunk indices;
//   "divides each partition into chunks with equal size (except for the last one)";
//   tensors are base + offset; sync returns when all data is loaded.
//
// On B200 the task queue between the DRAM tier and the GPU is the CUDA stream itself:
// chunk k is issued on stream k mod S (copy-engine DMA or a zero-copy kernel), its
// verification/scatter kernel follows on the same stream, and the next chunk's transfer
// proceeds on the other stream(s) -- the pipeline "avoids synchronization for all data
// on each storage tier" without host round trips.
#include <algorithm>
#include <condition_variable>
#include <deque>
#include <functional>
#include <thread>
#include <cstdlib>
#include <set>

#include "runtime.hpp"

namespace sllm {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what) {
  fail(SLLM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------------
// Device contexts
// ------------------------------------------------------------------------------------
static std::mutex g_ctx_mu;
static std::vector<std::unique_ptr<DeviceCtx>> g_ctx;

DeviceCtx& device_ctx(int dev) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if (dev < 0) fail(SLLM_E_INVALID, "negative GPU ordinal");
  if ((size_t)dev >= g_ctx.size()) g_ctx.resize(dev + 1);
  if (!g_ctx[dev]) {
    g_ctx[dev].reset(new DeviceCtx);
    g_ctx[dev]->dev = dev;
  }
  return *g_ctx[dev];
}

StreamSet* DeviceCtx::acquire(int n) {
  if (!misc) {  // first use: keep stream-ordered allocations (scratch, staging) cached between loads
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    SLLM_CUDA(cudaStreamCreateWithFlags(&misc, cudaStreamNonBlocking));
  }
  StreamSet* ss = nullptr;
  if (!idle.empty()) {
    ss = idle.back();
    idle.pop_back();
  } else {
    sets.emplace_back(new StreamSet);
    ss = sets.back().get();
  }
  for (int s = 0; s < n; ++s)
    if (!ss->xfer[s]) SLLM_CUDA(cudaStreamCreateWithFlags(&ss->xfer[s], cudaStreamNonBlocking));
  if (!ss->kern) SLLM_CUDA(cudaStreamCreateWithFlags(&ss->kern, cudaStreamNonBlocking));
  if (!ss->comm) SLLM_CUDA(cudaStreamCreateWithFlags(&ss->comm, cudaStreamNonBlocking));
  return ss;
}

uint8_t* StreamSet::host_stage(size_t bytes) {
  if (bytes > host_cap) {
    if (host) cudaFreeHost(host);
    host = nullptr;
    host_cap = 0;
    size_t cap = 64u << 10;
    while (cap < bytes) cap *= 2;
    void* h = nullptr;
    SLLM_CUDA(cudaHostAlloc(&h, cap, cudaHostAllocPortable));
    host = static_cast<uint8_t*>(h);
    host_cap = cap;
  }
  return host;
}

void DeviceCtx::release(StreamSet* s) {
  if (s) idle.push_back(s);
}

// ------------------------------------------------------------------------------------
// Busy set (concurrent loads of the same destinations are rejected)
// ------------------------------------------------------------------------------------
static std::mutex g_busy_mu;
static std::set<const void*> g_busy;

// ------------------------------------------------------------------------------------
// Load objects
// ------------------------------------------------------------------------------------
struct PartJob {
  size_t p = 0;
  int gpu = 0;
  // caller-stream ordering: `eager` jobs make the caller's stream wait on ev[1] before
  // sllm_load_start returns (once the job has enqueued all its work); the others (file
  // tier, in-process P2P groups: their issue waits on storage / on the peers) at wait()
  bool eager = false, issue_signalled = false, issue_ok = false;
  const uint8_t* src = nullptr;      // host pointer (pinned)
  const uint8_t* src_dev = nullptr;  // its device-visible alias (zero-copy modes)
  uint8_t* dst_base = nullptr;
  cudaStream_t origin = nullptr;
  std::string file;                  // file tier: <dir>/part_<device>.bin (else empty)
  int io_threads = 0;
  FileSourcePtr fsrc;                // file tier: reader threads + pinned slot ring
  // fan-out slice of this rank (whole partition when not replicated)
  uint64_t lo = 0, hi = 0;
  // P2P fan-out: the peers' replicas (device pointers valid here), this load's epoch
  uint8_t* peers[kMaxPeers] = {};
  uint32_t n_peers = 0;
  uint8_t* mc = nullptr;             // NVLS fan-out: multicast address of replica byte 0
  uint32_t epoch = 0;
  uint32_t h_err = 0;                // peer-wait result (0 = every peer signalled)
  uint32_t* d_err = nullptr;
  uint8_t* h_result = nullptr;  // pinned copy of {d_bad, d_err} (the set's host block)
  std::vector<Seg> segs;
  std::vector<uint32_t> chunk_seg;  // first segment of each chunk of [0, L)
  std::vector<uint32_t> gran_seg;   // scatter: last segment with off <= g MiB (MatParams.gran_seg)
  uint32_t* d_gran_seg = nullptr;
  // device scratch (one cudaMallocAsync block)
  void* scratch = nullptr;
  uint8_t* staging = nullptr;  // SCATTER_CE ring: n_streams slots of chunk_bytes (per job)
  Seg* d_segs = nullptr;
  BlockAcc* d_acc = nullptr;
  uint64_t* d_expect = nullptr;
  uint64_t* d_cs = nullptr;
  unsigned long long* d_bad = nullptr;
  unsigned long long* d_ktime = nullptr;  // profile 3 / SLLM_KTIME: MatParams.ktime slots
  unsigned long long* h_ktime = nullptr;  // their pinned copy (read back behind the load)
  // dynamic unit distribution (MatParams.ticket): one zeroed counter per launching stream,
  // with the tickets its earlier launches drew (launches on one stream run in order)
  unsigned long long* d_tickets = nullptr;
  std::vector<std::pair<cudaStream_t, uint64_t>> ticket_base;
  cudaEvent_t ev[4] = {};  // start, end, setup, origin
  // results
  std::vector<uint64_t> h_cs;
  bool h_cs_valid = false;
  unsigned long long h_bad = ~0ull;
  sllm_status status = SLLM_OK;
  std::string error;
  uint64_t t_issue_ns = 0;
  float t_dev_ms = 0.f;
  uint64_t chunks = 0, launches = 0, copies = 0, transferred = 0, fanout = 0;
  uint64_t storage_bytes = 0, storage_wait_ns = 0;  // file tier
  // profile: (start, end) event pairs around kernel launches / copies
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev, cev;
  std::vector<uint64_t> kev_bytes;  // bytes covered by each timed kernel launch
  uint64_t kernel_bytes = 0;
  double kernel_ms = 0, copy_ms = 0, kernel_span_ms = 0;
  // captured loads (sllm_load_capture): the job's work as one CUDA graph, replayed by
  // sllm_load_replay; its tables / result word live in a pinned block of its own
  bool capture = false;
  cudaGraphExec_t exec = nullptr;
  uint8_t* gstage = nullptr;
  cudaStream_t rstream = nullptr;  // replay stream when the caller passes none
  bool finished = false;           // run_job_guarded returned (guarded by sllm_load::issue_mu)
  std::vector<cudaStream_t> used;  // streams this job queued work on (drained on failure)
  StreamSet* ss = nullptr;         // leased from the GPU's DeviceCtx for the job's lifetime
};

}  // namespace sllm

struct sllm_load {
  const sllm_index* idx = nullptr;
  sllm_load_config cfg{};
  sllm_comm* comm = nullptr;
  std::vector<sllm::PartJob> jobs;
  std::vector<void*> dst_tensor;  // scatter modes: per tensor
  std::vector<const void*> busy_keys;
  std::chrono::steady_clock::time_point t0;
  bool joined = false;
  sllm_status result = SLLM_OK;
  sllm_load_report rep{};
  std::mutex issue_mu;                 // jobs report "all my work is enqueued" (or failed)
  std::condition_variable issue_cv;
  // captured load: replays issued / the last one reported by wait
  bool graph = false;
  uint64_t replays = 0;
  bool replay_pending = false;
  std::chrono::steady_clock::time_point t_replay;
  uint64_t t_replay_issue_ns = 0;
};

namespace sllm {

static uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Segments of partition p: every tensor [off, align16(off+size)) -> its destination,
// every gap between tensors (padding) -> checksum only.  Contiguous modes use a single
// segment [0, L) -> dst_base.
static void build_segments(const sllm_index& idx, PartJob& j, bool scatter, const std::vector<void*>& dst_tensor,
                           uint64_t chunk) {
  const PartRec& pr = idx.parts[j.p];
  j.segs.clear();
  if (!scatter) {
    j.segs.push_back(Seg{0, pr.length, j.dst_base, pr.length});
  } else {
    uint64_t cur = 0;
    for (uint32_t ti : pr.by_offset) {
      const TensorRec& t = idx.tensors[ti];
      if (t.offset > cur) j.segs.push_back(Seg{cur, t.offset - cur, nullptr, 0});
      uint64_t end16 = align_up(t.offset + t.nbytes, 16);
      j.segs.push_back(Seg{t.offset, end16 - t.offset, static_cast<uint8_t*>(dst_tensor[ti]), t.nbytes});
      cur = end16;
    }
    if (pr.length > cur) j.segs.push_back(Seg{cur, pr.length - cur, nullptr, 0});
  }
  uint64_t nch = ceil_div(pr.length, chunk);
  j.chunk_seg.assign(nch + 1, 0);
  size_t s = 0;
  for (uint64_t k = 0; k < nch; ++k) {
    uint64_t lo = k * chunk;
    while (s + 1 < j.segs.size() && j.segs[s + 1].off <= lo) ++s;
    j.chunk_seg[k] = (uint32_t)s;
  }
  j.chunk_seg[nch] = (uint32_t)j.segs.size();
  j.gran_seg.clear();
  if (scatter) gran_table(j.segs, pr.length, kGranShift, j.gran_seg);
}

// Work tile: 64 KiB, or the checksum block when smaller (tiles never straddle blocks).
static uint32_t tile_for(const sllm_index& idx) {
  return idx.block ? (uint32_t)std::min<uint64_t>(kTile, idx.block) : kTile;
}

// 0 = one grid of ring CTAs per GPU (two per SM, resolved by launch_materialise): every window's kernel spreads
// over the whole GPU, splitting checksum blocks across CTAs when a window is small.
static int default_ctas(int /*mode*/) { return 0; }

static std::pair<cudaEvent_t, cudaEvent_t> timed_begin(bool on, cudaStream_t st) {
  std::pair<cudaEvent_t, cudaEvent_t> e{nullptr, nullptr};
  if (!on) return e;
  SLLM_CUDA(cudaEventCreate(&e.first));
  SLLM_CUDA(cudaEventCreate(&e.second));
  SLLM_CUDA(cudaEventRecord(e.first, st));
  return e;
}

static void timed_end(std::pair<cudaEvent_t, cudaEvent_t> e, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& out,
                      cudaStream_t st) {
  if (!e.first) return;
  SLLM_CUDA(cudaEventRecord(e.second, st));
  out.push_back(e);
}

constexpr size_t kMaxKtime = 1024;  // timed launches per job with in-kernel timestamps
constexpr size_t kTicketSlots = kMaxStreams + 2;  // transfer streams, kernel stream, comm stream

// Units are handed out dynamically (tickets) unless SLLM_STATIC_UNITS is set (A/B knob).
static bool dynamic_units() {
  static const bool on = getenv("SLLM_STATIC_UNITS") == nullptr;
  return on;
}

static void launch(PartJob& j, bool prof, const MatParams& mp0, MatKind kind, int ctas, cudaStream_t st) {
  MatParams mp = mp0;
  if (prof && j.d_ktime && j.kev.size() < kMaxKtime) mp.ktime = j.d_ktime + 4 * j.kev.size();
  size_t slot = 0;
  while (slot < j.ticket_base.size() && j.ticket_base[slot].first != st) ++slot;
  if (slot == j.ticket_base.size() && slot < kTicketSlots) j.ticket_base.push_back({st, 0});
  if (j.d_tickets && slot < j.ticket_base.size()) {
    mp.ticket = j.d_tickets + slot;
    mp.ticket_base = j.ticket_base[slot].second;
  }
  auto e = timed_begin(prof, st);
  uint64_t drawn = 0;
  SLLM_CUDA(launch_materialise(mp, kind, ctas, st, &drawn));
  if (mp.ticket) j.ticket_base[slot].second += drawn;
  timed_end(e, j.kev, st);
  if (prof) {
    j.kernel_bytes += mp.hi - mp.lo;
    j.kev_bytes.push_back(mp.hi - mp.lo);
  }
  j.launches++;
}

// Streams of one job: S transfer streams (copy engine or zero-copy kernels) and one
// kernel stream for the verify / scatter kernels that follow a copy-engine transfer, so
// the copy engine always has the next chunk queued (no per-chunk kernel in its way).
struct Pipe {
  cudaStream_t xfer[kMaxStreams] = {};
  int S = 1;
  cudaStream_t kern = nullptr;
  cudaEvent_t copied = nullptr;            // chunk k landed (recorded, then waited at once)
  std::vector<cudaEvent_t> freed;          // SCATTER_CE: staging slot reusable
  int nslot = 0;
  uint64_t slot_bytes = 0;                 // SCATTER_CE: one window of chunks
  uint64_t window = 1;                     // chunks per submission (kernel launch)
  uint64_t v_k0 = 0, v_k1 = 0;             // CE: landed chunks not yet verified [v_k0, v_k1)
  std::vector<std::pair<uint64_t, uint64_t>> plan;  // SCATTER_CE from pinned DRAM: window chunk ranges
};

// sllm_load_config.engine -> MatParams.engine (0 LDG tiles, 1 TMA ring + STG, 2 TMA ring +
// TMA bulk stores).  Default: kDefaultEngine.
static int kernel_engine(int cfg_engine) {
  switch (cfg_engine) {
    case 1: return 1;
    case 2: return 0;
    case 3: return 2;
    default: return kDefaultEngine;
  }
}

static MatParams window_params(const sllm_index& idx, const sllm_load_config& cfg, const PartJob& j, uint64_t k0,
                               uint64_t k1, uint64_t lo, uint64_t hi) {
  const bool check = cfg.verify && idx.block;
  MatParams mp{};
  mp.lo = lo;
  mp.hi = hi;
  mp.segs = j.d_segs;
  mp.gran_seg = j.d_gran_seg;
  mp.gran_shift = kGranShift;
  mp.seg_begin = j.chunk_seg[k0];
  const uint64_t nch = j.chunk_seg.size() - 1;
  mp.seg_end = k1 < nch ? std::min<uint32_t>(j.chunk_seg[k1] + 1, (uint32_t)j.segs.size()) : (uint32_t)j.segs.size();
  mp.tile = tile_for(idx);
  mp.block = idx.block ? idx.block : kTile;
  mp.part_len = idx.parts[j.p].length;
  mp.acc = j.d_acc;
  mp.expect = check ? j.d_expect : nullptr;
  mp.cs_out = check ? j.d_cs : nullptr;
  mp.bad = j.d_bad;
  mp.engine = kernel_engine(cfg.engine);
  mp.n_peers = j.n_peers;
  for (uint32_t k = 0; k < j.n_peers; ++k) mp.peer[k] = j.peers[k];
  mp.mc = j.mc;
  return mp;
}

// Copy chunks [k0, k1) (chunk k = partition bytes [k*C, min((k+1)*C, L))) from the pinned
// source to dst + (k*C - lo) on stream xs.  The chunks of a window are contiguous on both
// sides, so the window is ONE cudaMemcpyAsync of [k0*C, min(k1*C, L)): one host call per
// >= 64 MiB instead of one per chunk (per-chunk calls at 1 MiB chunks made the host issue
// loop the bottleneck: 41.8 GB/s, profiles/r01/sweep_opt67b.jsonl), and the copy engine
// splits it into its own transfers.  (The batched-copy runtime entry point is not used:
// it is closed on the B200 pool this build is measured on.)
static void copy_window(PartJob& j, int prof, uint8_t* dst, const uint8_t* wsrc, uint64_t lo, uint64_t k0, uint64_t k1,
                        uint64_t C, uint64_t L, cudaStream_t xs) {
  const uint64_t a = k0 * C, b = std::min(k1 * C, L);
  if (b <= a) return;
  auto e = timed_begin(prof >= 2, xs);  // copies are timed only at profile level 2
  SLLM_CUDA(cudaMemcpyAsync(dst + (a - lo), wsrc + (a - lo), b - a, cudaMemcpyHostToDevice, xs));
  timed_end(e, j.cev, xs);
  j.copies++;
}

// Unit of the NCCL fan-outs' slicing and rounds: a whole copy window (>= kWindowBytes of
// chunks), so every round is one copy submission and one grouped broadcast /
// all-gather per root instead of one per chunk; the chunk stays the copy engine's
// transfer unit inside it.  The P2P fan-out and unreplicated loads slice by chunk.
uint64_t fanout_unit(uint64_t chunk, int32_t fanout) {
  if (fanout != SLLM_FANOUT_BCAST && fanout != SLLM_FANOUT_ALLGATHER) return chunk;
  return std::max<uint64_t>(1, kWindowBytes / chunk) * chunk;
}

// Largest verification span (kVerifyBytes; SLLM_VERIFY_SPAN_MIB: measurement knob).
static uint64_t verify_span_bytes() {
  static const uint64_t v = [] {
    const char* e = getenv("SLLM_VERIFY_SPAN_MIB");
    return (e && atoll(e) > 0) ? (uint64_t)atoll(e) << 20 : kVerifyBytes;
  }();
  return v;
}

// Smallest span once the end of the load is near (CE / fan-out / GDS verification): the K4
// after the final copy covers at most this much.  kVerifyTailBytes for large partitions; an
// eighth of the partition (>= one copy window) for small ones, so a latency-bound load
// (e.g. an 828 MB LoRA adapter, 15 ms) does not end with a 300+ MB verification pass.
static uint64_t verify_tail_bytes(uint64_t L) {
  return std::min<uint64_t>(kVerifyTailBytes, std::max<uint64_t>(kWindowBytes, L / 8));
}

// Issue the window of chunks [k0, k1) of job j: the copy engine moves every chunk (one
// submission), then ONE verify / scatter launch covers the window; zero-copy
// modes issue one kernel for the window.  Returns the stream whose completion means
// "the window is in place and verified" (the fan-out orders its broadcast after it).
static cudaStream_t issue_window(const sllm_index& idx, const sllm_load_config& cfg, PartJob& j, Pipe& P, uint64_t w,
                                 uint64_t k0, uint64_t k1, bool last) {
  NvtxRange nv("sllm.window p=%zu w=%llu chunks=[%llu,%llu)", j.p, (unsigned long long)w, (unsigned long long)k0,
               (unsigned long long)k1);
  const bool check = cfg.verify && idx.block;
  const int prof = cfg.profile;
  const int ctas = cfg.ctas > 0 ? cfg.ctas : default_ctas(cfg.mode);
  const uint64_t C = cfg.chunk_bytes, L = idx.parts[j.p].length;
  const uint64_t lo = k0 * C, hi = std::min(k1 * C, L);
  MatParams mp = window_params(idx, cfg, j, k0, k1, lo, hi);
  cudaStream_t xs = P.xfer[w % P.S];
  cudaStream_t done = xs;
  // Source of the window: the pinned partition, or (file tier) the pinned ring slot the
  // storage readers filled with this window (UVA: the slot's device alias is its address).
  const uint8_t* wsrc = j.fsrc ? file_source_window(*j.fsrc, w) : j.src + lo;
  const uint8_t* wsrc_dev = j.fsrc ? wsrc : j.src_dev + lo;
  switch (cfg.mode) {
    case SLLM_MODE_CE:
      copy_window(j, prof, j.dst_base + lo, wsrc, lo, k0, k1, C, L, xs);
      if (j.n_peers || j.mc) {
        // P2P / NVLS fan-out: one kernel per landed window reads it back from the rank's own
        // replica, verifies it and stores it into every peer replica over NVLink (NVLS: one
        // multicast store per vector)
        SLLM_CUDA(cudaEventRecord(P.copied, xs));
        SLLM_CUDA(cudaStreamWaitEvent(P.kern, P.copied, 0));
        mp.src = j.dst_base;
        mp.src_origin = 0;
        mp.host_src = 0;
        mp.no_seg_store = 1;
        launch(j, prof, mp, check ? MatKind::kCopyChecksum : MatKind::kCopyOnly, ctas, P.kern);
        done = P.kern;
      } else if (check) {
        SLLM_CUDA(cudaEventRecord(P.copied, xs));
        SLLM_CUDA(cudaStreamWaitEvent(P.kern, P.copied, 0));
        // K4 runs per verification span of landed windows: up to kVerifyBytes per launch
        // (few, long launches that keep every SM streaming), and once the pending span is
        // at least kVerifyTailBytes and as long as what is still to come, at once -- spans
        // shrink towards the end, so the tail after the last copy is one K4 of at most
        // ~kVerifyTailBytes (~0.1 ms at HBM rate).  The copies never wait.
        if (P.v_k1 == P.v_k0) P.v_k0 = k0;
        P.v_k1 = k1;
        const uint64_t pending = std::min(P.v_k1 * C, L) - P.v_k0 * C;
        if (last || pending >= verify_span_bytes() || (pending >= verify_tail_bytes(L) && pending >= L - hi)) {
          NvtxRange nvv("sllm.verify.span [%llu,%llu)", (unsigned long long)(P.v_k0 * C),
                        (unsigned long long)std::min(P.v_k1 * C, L));
          MatParams vp = window_params(idx, cfg, j, P.v_k0, P.v_k1, P.v_k0 * C, std::min(P.v_k1 * C, L));
          vp.src = j.dst_base;
          vp.src_origin = 0;
          vp.host_src = 0;
          launch(j, prof, vp, MatKind::kChecksumOnly, ctas, P.kern);
          P.v_k0 = P.v_k1 = 0;
        }
        done = P.kern;
      }
      break;
    case SLLM_MODE_ZEROCOPY:
    case SLLM_MODE_SCATTER_ZC:
      // (P2P fan-out: the same kernel also stores every vector into the peer replicas)
      mp.src = wsrc_dev;
      mp.src_origin = lo;
      mp.host_src = 1;
      launch(j, prof, mp, check ? MatKind::kCopyChecksum : MatKind::kCopyOnly, ctas, xs);
      break;
    case SLLM_MODE_SCATTER_CE: {
      const int slot = (int)(w % (uint64_t)P.nslot);
      uint8_t* stage = j.staging + (uint64_t)slot * P.slot_bytes;
      if (w >= (uint64_t)P.nslot) SLLM_CUDA(cudaStreamWaitEvent(xs, P.freed[slot], 0));
      copy_window(j, prof, stage, wsrc, lo, k0, k1, C, L, xs);
      SLLM_CUDA(cudaEventRecord(P.copied, xs));
      SLLM_CUDA(cudaStreamWaitEvent(P.kern, P.copied, 0));
      mp.src = stage;
      mp.src_origin = lo;
      mp.host_src = 0;
      launch(j, prof, mp, check ? MatKind::kCopyChecksum : MatKind::kCopyOnly, ctas, P.kern);
      SLLM_CUDA(cudaEventRecord(P.freed[slot], P.kern));
      done = P.kern;
      break;
    }
    default:
      fail(SLLM_E_INVALID, "unknown mode");
  }
  if (j.fsrc) file_source_consumed(*j.fsrc, w, xs);  // the slot is free once xs is past its reader
  j.chunks += k1 - k0;
  j.transferred += hi - lo;
  return done;
}

// Checksum-only verification of bytes that arrived through the fan-out.
static void verify_range(const sllm_index& idx, const sllm_load_config& cfg, PartJob& j, uint64_t lo, uint64_t hi,
                         cudaStream_t st) {
  NvtxRange nv("sllm.verify.range [%llu,%llu)", (unsigned long long)lo, (unsigned long long)hi);
  MatParams mp{};
  mp.src = j.dst_base;
  mp.lo = lo;
  mp.hi = hi;
  mp.segs = j.d_segs;
  mp.seg_begin = 0;
  mp.seg_end = 1;  // contiguous single segment
  mp.tile = tile_for(idx);
  mp.block = idx.block;
  mp.part_len = idx.parts[j.p].length;
  mp.acc = j.d_acc;
  mp.expect = j.d_expect;
  mp.cs_out = j.d_cs;
  mp.bad = j.d_bad;
  mp.engine = kernel_engine(cfg.engine);
  launch(j, cfg.profile != 0, mp, MatKind::kChecksumOnly, cfg.ctas > 0 ? cfg.ctas : 0, st);
}

// s0 waits for the work queued so far on every stream of `tails`.
static void join_streams(const std::vector<cudaStream_t>& tails, cudaStream_t s0) {
  for (cudaStream_t t : tails) {
    cudaEvent_t e;
    SLLM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SLLM_CUDA(cudaEventRecord(e, t));
    SLLM_CUDA(cudaStreamWaitEvent(s0, e, 0));
    SLLM_CUDA(cudaEventDestroy(e));  // destruction is deferred until the event completes
  }
}

static void run_job(sllm_load* L, PartJob& j) {
  NvtxRange nv("sllm.partition p=%zu gpu=%d", j.p, j.gpu);
  const sllm_index& idx = *L->idx;
  const sllm_load_config& cfg = L->cfg;
  const PartRec& pr = idx.parts[j.p];
  const uint64_t t0 = now_ns();
  SLLM_CUDA(cudaSetDevice(j.gpu));
  bind_thread_to_gpu(j.gpu);  // the worker runs next to its GPU's PCIe root and pinned pages
  DeviceCtx& dc = device_ctx(j.gpu);
  {
    std::lock_guard<std::mutex> g(dc.mu);
    j.ss = dc.acquire(cfg.n_streams);
  }
  Pipe P;
  P.S = cfg.n_streams;
  const bool p2p = cfg.fanout == SLLM_FANOUT_P2P || cfg.fanout == SLLM_FANOUT_NVLS;  // (same group protocol)
  for (int s = 0; s < P.S; ++s) P.xfer[s] = p2p ? comm_stream(L->comm, s) : j.ss->xfer[s];
  P.kern = p2p ? comm_stream(L->comm, kMaxStreams) : j.ss->kern;
  P.nslot = std::max(3, P.S + 1);
  // Chunks are the copy engine's transfer unit; kernels and copy submissions are
  // grouped per window of >= kWindowBytes so small chunks do not make the host issue
  // loop (one API call per chunk) the bottleneck.
  // SCATTER_CE stages whole windows in HBM and scatters each with one K3 launch: larger
  // windows there (kScatterWindowBytes) make fewer, longer launches; the staging ring is
  // never larger than the partition.
  // (the file tier keeps kScatterFileWindowBytes: its windows are storage-ring slots)
  const bool files = !j.file.empty();
  uint64_t scatter_win = files ? kScatterFileWindowBytes : kScatterWindowBytes;
  if (const char* e = getenv("SLLM_SCATTER_WINDOW_MIB"))  // measurement knob (A/B runs)
    if (atoll(e) > 0 && !files) scatter_win = (uint64_t)atoll(e) << 20;
  // Copy windows (one cudaMemcpyAsync each): a 16th of the partition, between kWindowBytes
  // and kCopyWindowMaxBytes -- 256 MiB windows shave ~0.8 ms (0.3 %) off a 13.3 GB load
  // against 64 MiB ones (per-copy start cost, profiles/r02/window_sweep.jsonl), while a
  // small partition (an 828 MB adapter) keeps 64 MiB windows so its first K4 starts early.
  uint64_t copy_win = files ? kWindowBytes
                            : std::min(kCopyWindowMaxBytes, std::max(kWindowBytes, align_up(pr.length / 16, kWindowBytes)));
  if (const char* e = getenv("SLLM_WINDOW_MIB"))  // measurement knob (A/B runs)
    if (atoll(e) > 0 && !files) copy_win = (uint64_t)atoll(e) << 20;
  const uint64_t win_bytes = cfg.mode == SLLM_MODE_SCATTER_CE ? scatter_win : copy_win;
  const bool nccl_fanout = cfg.fanout == SLLM_FANOUT_BCAST || cfg.fanout == SLLM_FANOUT_ALLGATHER;
  P.window = nccl_fanout ? fanout_unit(cfg.chunk_bytes, cfg.fanout) / cfg.chunk_bytes
                         : std::max<uint64_t>(1, win_bytes / cfg.chunk_bytes);
  const uint64_t nch_all = std::max<uint64_t>(1, ceil_div(pr.length, cfg.chunk_bytes));
  if (cfg.mode == SLLM_MODE_SCATTER_CE && !files) {
    // windows of P.window chunks, halving over the last two windows' worth of chunks down
    // to kScatterTailBytes, so the K3 that runs after the final copy is short
    // (a partition of fewer than four full windows gets windows of a quarter of it, >= the
    // tail size, so its first K3 starts early as well)
    const uint64_t wmin = std::min<uint64_t>(P.window, std::max<uint64_t>(1, kScatterTailBytes / cfg.chunk_bytes));
    const uint64_t wide = std::min(P.window, std::max(wmin, ceil_div(nch_all, 4)));
    uint64_t widest = 1;
    for (uint64_t k0 = 0; k0 < nch_all;) {
      const uint64_t rem = nch_all - k0;
      const uint64_t n = std::min(rem, rem > 2 * wide ? wide : std::max(wmin, (rem + 1) / 2));
      P.plan.emplace_back(k0, k0 + n);
      widest = std::max(widest, n);
      k0 += n;
    }
    P.slot_bytes = widest * cfg.chunk_bytes;
    P.nslot = (int)std::min<uint64_t>((uint64_t)P.nslot, P.plan.size());
  } else {
    P.slot_bytes = std::min(P.window, nch_all) * cfg.chunk_bytes;
    P.nslot = (int)std::min<uint64_t>((uint64_t)P.nslot, ceil_div(nch_all, P.window));
  }
  if (!j.file.empty() && cfg.mode != SLLM_MODE_GDS)  // (a replicated load reads only its slice [lo, hi) from storage)
    j.fsrc = file_source_open(j.file, j.lo, j.hi, P.window * cfg.chunk_bytes, j.io_threads, j.gpu);
  SLLM_CUDA(cudaEventCreateWithFlags(&P.copied, cudaEventDisableTiming));
  if (cfg.mode == SLLM_MODE_SCATTER_CE) {
    P.freed.resize(P.nslot);
    for (auto& e : P.freed) SLLM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t s0 = P.xfer[0];
  j.used.assign(P.xfer, P.xfer + P.S);
  j.used.push_back(P.kern);
  if (nccl_fanout) j.used.push_back(j.ss->comm);
  const uint64_t nb = pr.n_blocks;
  const size_t seg_bytes = align_up(j.segs.size() * sizeof(Seg), 256);
  const size_t acc_bytes = align_up(std::max<uint64_t>(nb, 1) * sizeof(BlockAcc), 256);
  const size_t tab_bytes = align_up(std::max<uint64_t>(nb, 1) * 8, 256);
  const size_t gran_bytes = align_up(j.gran_seg.size() * 4, 256);
  // Device scratch: [segs | granule table | expected checksums | result word] is uploaded
  // in ONE async copy from the set's pinned block, [block accumulators | computed
  // checksums] is zeroed by one memset -- two setup operations ahead of the first chunk.
  const size_t up_bytes = seg_bytes + gran_bytes + tab_bytes + 256;
  static const bool ktime = getenv("SLLM_KTIME") != nullptr;
  const size_t kt_bytes = (cfg.profile == 3 || (cfg.profile && ktime)) ? kMaxKtime * 4 * sizeof(unsigned long long) : 0;
  const size_t tk_bytes = dynamic_units() ? align_up(kTicketSlots * sizeof(unsigned long long), 256) : 0;
  const size_t zero_bytes = acc_bytes + tab_bytes + kt_bytes + tk_bytes;
  const size_t total = up_bytes + zero_bytes;
  if (j.origin) SLLM_CUDA(cudaStreamWaitEvent(s0, j.ev[3], 0));  // recorded by sllm_load_start
  SLLM_CUDA(cudaMallocAsync(&j.scratch, total, s0));
  if (cfg.mode == SLLM_MODE_SCATTER_CE) {
    void* st = nullptr;
    SLLM_CUDA(cudaMallocAsync(&st, (size_t)P.nslot * P.slot_bytes, s0));
    j.staging = static_cast<uint8_t*>(st);
  }
  uint8_t* h = nullptr;
  if (j.capture) {  // the graph's upload node reads this block at every replay: the job owns it
    SLLM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&j.gstage), up_bytes + 256, cudaHostAllocDefault));
    h = j.gstage;
  } else {
    h = j.ss->host_stage(up_bytes + 256 + kt_bytes);
  }
  j.h_result = h + up_bytes;  // 16 bytes: first failing block, peer-wait result
  std::memcpy(h, j.segs.data(), j.segs.size() * sizeof(Seg));
  if (!j.gran_seg.empty()) std::memcpy(h + seg_bytes, j.gran_seg.data(), j.gran_seg.size() * 4);
  if (nb) std::memcpy(h + seg_bytes + gran_bytes, pr.checksums.data(), nb * 8);
  std::memset(h + seg_bytes + gran_bytes + tab_bytes, 0xFF, 8);      // first failing block: none
  std::memset(h + seg_bytes + gran_bytes + tab_bytes + 8, 0, 248);  // peer-wait result: 0
  uint8_t* base = static_cast<uint8_t*>(j.scratch);
  j.d_segs = reinterpret_cast<Seg*>(base);
  if (!j.gran_seg.empty()) j.d_gran_seg = reinterpret_cast<uint32_t*>(base + seg_bytes);
  j.d_expect = reinterpret_cast<uint64_t*>(base + seg_bytes + gran_bytes);
  j.d_bad = reinterpret_cast<unsigned long long*>(base + seg_bytes + gran_bytes + tab_bytes);
  j.d_err = reinterpret_cast<uint32_t*>(j.d_bad + 1);
  j.d_acc = reinterpret_cast<BlockAcc*>(base + up_bytes);
  j.d_cs = reinterpret_cast<uint64_t*>(base + up_bytes + acc_bytes);
  j.d_ktime = kt_bytes ? reinterpret_cast<unsigned long long*>(base + up_bytes + acc_bytes + tab_bytes) : nullptr;
  j.h_ktime = kt_bytes ? reinterpret_cast<unsigned long long*>(h + up_bytes + 256) : nullptr;
  j.d_tickets = tk_bytes ? reinterpret_cast<unsigned long long*>(base + up_bytes + acc_bytes + tab_bytes + kt_bytes)
                         : nullptr;
  j.ticket_base.clear();
  if (j.capture) {
    // everything from the table upload to the result word becomes the job's graph (the
    // scratch / staging allocations above are done first: a replay reuses them)
    SLLM_CUDA(cudaStreamSynchronize(s0));
    SLLM_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  }
  SLLM_CUDA(cudaMemcpyAsync(base, h, up_bytes, cudaMemcpyHostToDevice, s0));
  SLLM_CUDA(cudaMemsetAsync(base + up_bytes, 0, zero_bytes, s0));
  SLLM_CUDA(cudaEventRecord(j.ev[0], s0));
  const bool in_process = p2p && comm_in_process(L->comm);  // peers ordered by events, not device waits
  if (p2p) {  // no store into a peer replica before every peer is done verifying the previous load
    const int R = comm_nranks(L->comm), me = comm_rank(L->comm);
    if (in_process) {
      comm_wait_peers(L->comm, kPeerDone, s0);
    } else if (comm_host_wait()) {
      comm_wait_flags_host(L->comm, comm_peer_signal(L->comm, me) + R, j.epoch - 1);
    } else {
      SLLM_CUDA(launch_peer_wait(comm_peer_signal(L->comm, me) + R, R, me, j.epoch - 1, comm_timeout_ns(L->comm),
                                 j.d_err, s0));
      if (R > 1) j.launches++;
    }
  }
  SLLM_CUDA(cudaEventRecord(j.ev[2], s0));
  for (int s = 1; s < P.S; ++s) SLLM_CUDA(cudaStreamWaitEvent(P.xfer[s], j.ev[2], 0));
  SLLM_CUDA(cudaStreamWaitEvent(P.kern, j.ev[2], 0));

  const uint64_t C = cfg.chunk_bytes;
  std::vector<cudaStream_t> tails;  // streams to join at the end
  for (int s = 1; s < P.S; ++s) tails.push_back(P.xfer[s]);
  tails.push_back(P.kern);
  if (nccl_fanout) {
    // Replicated load: this rank moves its chunks over PCIe; every chunk
    // round is then spread over NVLink -- BCAST: grouped broadcasts, one root per slice;
    // ALLGATHER: chunks owned round-robin, one in-place all-gather per full round (the
    // ragged last round falls back to grouped broadcasts).
    const bool ag = cfg.fanout == SLLM_FANOUT_ALLGATHER;
    const int R = comm_nranks(L->comm), me = comm_rank(L->comm);
    std::vector<uint64_t> lohi(2 * R);
    uint64_t rounds = 0;
    int32_t full = 0;
    const uint64_t U = fanout_unit(C, cfg.fanout);  // round unit: a whole window of chunks
    auto schedule = [&](uint64_t r, uint64_t* n) {
      return ag ? sllm_allgather_round(pr.length, U, R, r, lohi.data(), n, &full)
                : sllm_replica_round(pr.length, U, R, r, lohi.data(), n);
    };
    if (schedule(0, &rounds) != SLLM_OK && pr.length) fail(SLLM_E_INVALID, "fan-out schedule failed");
    cudaEvent_t evk;
    SLLM_CUDA(cudaEventCreateWithFlags(&evk, cudaEventDisableTiming));
    cudaStream_t cs = j.ss->comm;
    SLLM_CUDA(cudaStreamWaitEvent(cs, j.ev[2], 0));
    // Verification of what the round moved (K4 on the comm stream, after the collective).
    // ZC: the rank's own chunks are verified inside K2; only received chunks are checked,
    // per round.  CE: own and received chunks alike are verified in spans -- per root
    // slice (BCAST) or over the partition (ALLGATHER rounds are contiguous) -- with the CE
    // pipeline's span rule (<= kVerifyBytes per launch, shrinking towards the end), so a
    // load is verified by a few long K4 launches instead of one per chunk and root.
    const bool check = cfg.verify && idx.block;
    const bool spans = check && cfg.mode == SLLM_MODE_CE;
    sllm_load_config cfg_own = cfg;
    if (spans) cfg_own.verify = 0;
    struct Span { uint64_t lo = 0, hi = 0, end = 0; };
    std::vector<Span> sp(ag ? 1 : R);
    if (ag) {
      sp[0].end = pr.length;
    } else {
      std::vector<uint64_t> sl(2 * R);
      if (sllm_replica_slices(pr.length, U, R, sl.data()) != SLLM_OK) fail(SLLM_E_INVALID, "bad slices");
      for (int q = 0; q < R; ++q) sp[q].end = sl[2 * q + 1];
    }
    auto extend = [&](Span& v, uint64_t a, uint64_t b) {
      if (v.hi == v.lo) v.lo = a;
      v.hi = b;
      const uint64_t pending = v.hi - v.lo, remaining = v.end - v.hi;
      if (remaining == 0 || pending >= verify_span_bytes() || (pending >= verify_tail_bytes(pr.length) && pending >= remaining)) {
        verify_range(idx, cfg, j, v.lo, v.hi, cs);
        v.lo = v.hi = 0;
      }
    };
    for (uint64_t r = 0; r < rounds; ++r) {
      NvtxRange nvr("sllm.fanout.round %llu", (unsigned long long)r);
      full = 0;
      if (schedule(r, nullptr) != SLLM_OK) fail(SLLM_E_INVALID, "fan-out schedule failed");
      std::vector<std::pair<uint64_t, uint64_t>> ranges(R);
      for (int q = 0; q < R; ++q) ranges[q] = {lohi[2 * q], lohi[2 * q + 1]};
      if (ranges[me].second > ranges[me].first) {  // this rank's own unit of the round: PCIe
        const uint64_t lo = ranges[me].first, hi = ranges[me].second;
        cudaStream_t done = issue_window(idx, cfg_own, j, P, r, lo / C, ceil_div(hi, C), true);
        SLLM_CUDA(cudaEventRecord(evk, done));
        SLLM_CUDA(cudaStreamWaitEvent(cs, evk, 0));
      }
      for (int q = 0; q < R; ++q)
        if (q != me && ranges[q].second > ranges[q].first) j.fanout += ranges[q].second - ranges[q].first;
      if (ag && full) {  // NVLink: one in-place all-gather of the round's R whole chunks
        nccl_allgather_inplace(L->comm, ranges[0].first, U, j.dst_base, cs);
      } else {
        nccl_bcast_group(L->comm, ranges, j.dst_base, cs);  // NVLink: every root's chunk to every rank
      }
      if (spans) {
        for (int q = 0; q < R; ++q)
          if (ranges[q].second > ranges[q].first) extend(sp[ag ? 0 : q], ranges[q].first, ranges[q].second);
      } else if (check) {
        if (ag && full) {  // the round is contiguous: what arrived is around our chunk
          if (me > 0) verify_range(idx, cfg, j, ranges[0].first, ranges[me].first, cs);
          if (me + 1 < R) verify_range(idx, cfg, j, ranges[me].second, ranges[R - 1].second, cs);
        } else {
          for (int q = 0; q < R; ++q)
            if (q != me && ranges[q].second > ranges[q].first) verify_range(idx, cfg, j, ranges[q].first, ranges[q].second, cs);
        }
      }
    }
    tails.push_back(cs);
    SLLM_CUDA(cudaEventDestroy(evk));
  } else if (p2p) {
    // Replicated load, fan-out fused into the loading kernels: this
    // rank moves its slice [lo, hi) over PCIe and its kernels store it into every replica.
    const uint64_t nch_hi = ceil_div(j.hi, C);
    for (uint64_t k0 = j.lo / C, w = 0; k0 < nch_hi; k0 += P.window, ++w)
      issue_window(idx, cfg, j, P, w, k0, std::min(k0 + P.window, nch_hi), k0 + P.window >= nch_hi);
    join_streams(tails, s0);
    tails.clear();
    const int R = comm_nranks(L->comm), me = comm_rank(L->comm);
    // Signal array of rank q (2R words): ready[r] = last epoch whose stores rank r has
    // completed into q's replica, done[r] = last epoch rank r has finished (its replica is
    // free for the next epoch's stores).  Every store of this rank's kernels -> visible to
    // the peers (ready), then wait for theirs, verify what arrived, publish done.
    // (In-process ranks: the same protocol with CUDA events, see fanout.cpp.)
    PeerSignal ready{}, done{};
    for (int q = 0; q < R; ++q)
      if (q != me) {
        ready.remote[ready.n++] = comm_peer_signal(L->comm, q) + me;
        done.remote[done.n++] = comm_peer_signal(L->comm, q) + R + me;
      }
    const char* lost = "P2P fan-out: a peer rank of this process did not reach the fan-out within the timeout";
    if (in_process) {
      comm_record(L->comm, kPeerReady, s0);
      if (!comm_local_barrier(L->comm)) fail(SLLM_E_PEER, lost);  // every ready event recorded before any wait
      comm_wait_peers(L->comm, kPeerReady, s0);
    } else {
      SLLM_CUDA(launch_peer_signal(ready, j.epoch, s0));
      // (a group split over processes with several ranks in this one: those ranks still queue
      // every ready signal before any wait, so no wait sits ahead of a peer's signal)
      comm_local_barrier(L->comm);
      if (comm_host_wait()) {
        comm_wait_flags_host(L->comm, comm_peer_signal(L->comm, me), j.epoch);
      } else {
        SLLM_CUDA(launch_peer_wait(comm_peer_signal(L->comm, me), R, me, j.epoch, comm_timeout_ns(L->comm), j.d_err, s0));
      }
    }
    j.fanout = pr.length - (j.hi - j.lo);
    if (cfg.verify && idx.block) {  // what arrived over NVLink is verified like what came over PCIe
      if (j.lo > 0) verify_range(idx, cfg, j, 0, j.lo, s0);
      if (j.hi < pr.length) verify_range(idx, cfg, j, j.hi, pr.length, s0);
    }
    if (in_process) {
      comm_record(L->comm, kPeerDone, s0);
      if (!comm_local_barrier(L->comm)) fail(SLLM_E_PEER, lost);  // ... and every done event before the next load
    } else {
      SLLM_CUDA(launch_peer_signal(done, j.epoch, s0));
      comm_local_barrier(L->comm);  // (same: every done signal before the next load's done wait)
      if (R > 1) j.launches += comm_host_wait() ? 2 : 3;  // ready signal, [ready wait,] done signal
    }
  } else {
    const uint64_t nch = ceil_div(pr.length, C);
    if (!P.plan.empty()) {  // SCATTER_CE from pinned DRAM: the window plan (every window fits a slot)
      for (uint64_t w = 0; w < P.plan.size(); ++w)
        issue_window(idx, cfg, j, P, w, P.plan[w].first, P.plan[w].second, w + 1 == P.plan.size());
    } else if (cfg.mode == SLLM_MODE_GDS) {
      NvtxRange nvg("sllm.gds p=%zu", j.p);
      // storage -> HBM with cuFile (gds.cpp); the landed prefix is verified in K4 spans on
      // the kernel stream with the CE pipeline's span rule
      SLLM_CUDA(cudaStreamSynchronize(s0));  // scratch and tables are in place before K4 runs
      const bool check = cfg.verify && idx.block;
      uint64_t v_lo = 0, v_hi = 0;
      gds_read(j.file, j.gpu, j.dst_base, 0, pr.length, P.window * C, j.io_threads > 0 ? j.io_threads : 4,
               [&](uint64_t a, uint64_t b) {
                 if (!check) return;
                 if (v_hi == v_lo) v_lo = a;
                 v_hi = b;
                 const uint64_t pending = v_hi - v_lo, remaining = pr.length - v_hi;
                 if (remaining == 0 || pending >= verify_span_bytes() || (pending >= verify_tail_bytes(pr.length) && pending >= remaining)) {
                   verify_range(idx, cfg, j, v_lo, v_hi, P.kern);
                   v_lo = v_hi = 0;
                 }
               },
               &j.storage_wait_ns);
      j.transferred = j.storage_bytes = pr.length;
      j.chunks = nch;
    } else {
      for (uint64_t k0 = 0, w = 0; k0 < nch; k0 += P.window, ++w)
        issue_window(idx, cfg, j, P, w, k0, std::min(k0 + P.window, nch), k0 + P.window >= nch);
    }
  }
  // join every stream into s0, then let the caller's stream wait for the load
  join_streams(tails, s0);
  SLLM_CUDA(cudaEventRecord(j.ev[1], s0));
  // the result word comes back into the pinned block behind the load (no extra round trip)
  SLLM_CUDA(cudaMemcpyAsync(j.h_result, j.d_bad, 16, cudaMemcpyDeviceToHost, s0));
  if (j.d_ktime && !j.kev.empty())  // profile 3: the timed launches' in-kernel stamps
    SLLM_CUDA(cudaMemcpyAsync(j.h_ktime, j.d_ktime, 4 * sizeof(unsigned long long) * std::min(j.kev.size(), kMaxKtime),
                              cudaMemcpyDeviceToHost, s0));
  if (j.capture) {  // the job's graph: instantiated here, run by sllm_load_replay
    cudaGraph_t g = nullptr;
    SLLM_CUDA(cudaStreamEndCapture(s0, &g));
    const cudaError_t e = cudaGraphInstantiate(&j.exec, g, 0);
    cudaGraphDestroy(g);
    SLLM_CUDA(e);
    cudaEventDestroy(P.copied);
    for (auto& ev : P.freed) cudaEventDestroy(ev);
    j.t_issue_ns = now_ns() - t0;
    std::lock_guard<std::mutex> lk(L->issue_mu);
    j.issue_ok = j.issue_signalled = true;
    return;
  }
  {  // every command of this job is enqueued: the caller's stream may now wait on ev[1]
    std::lock_guard<std::mutex> g(L->issue_mu);
    j.issue_ok = j.issue_signalled = true;
  }
  L->issue_cv.notify_all();
  j.t_issue_ns = now_ns() - t0;
  SLLM_CUDA(cudaStreamSynchronize(s0));  // the load (ev[1]) and its result word
  if (j.staging) {
    // The SCATTER_CE staging ring is not part of the loaded model: back to the stream-ordered
    // pool as soon as the load is done (reusable by the next load at no cost; re-growing a
    // trimmed pool per load measured 4x slower, profiles/r01/staging_trim_ab.json).  The pool
    // keeps it cached until sllm_device_trim releases idle memory to the inference engine.
    SLLM_CUDA(cudaFreeAsync(j.staging, s0));
    j.staging = nullptr;
  }
  if (j.fsrc) {  // (GDS: set by the read loop)
    j.storage_bytes = file_source_bytes(*j.fsrc);
    j.storage_wait_ns = file_source_wait_ns(*j.fsrc);
  }
  j.fsrc.reset();  // file tier: readers are done, slots go back to the pinned pool
  uint64_t tail[2] = {};
  std::memcpy(tail, j.h_result, 16);  // first failing block, peer-wait result
  j.h_bad = tail[0];
  j.h_err = (uint32_t)tail[1];
  SLLM_CUDA(cudaEventElapsedTime(&j.t_dev_ms, j.ev[0], j.ev[1]));
  static const bool dump = getenv("SLLM_PROFILE_DUMP") != nullptr;  // per-launch timeline on stderr
  std::vector<unsigned long long> kt;
  j.kernel_span_ms = 0;
  if (j.d_ktime && !j.kev.empty()) {  // in-kernel timestamps (the job's work is complete)
    kt.assign(j.h_ktime, j.h_ktime + 4 * std::min(j.kev.size(), kMaxKtime));
    for (size_t i = 0; i + 3 < kt.size(); i += 4)
      if (kt[i + 3]) j.kernel_span_ms += (kt[i + 3] - ~kt[i]) * 1e-6;  // (a launch with no bytes has no marks)
  }
  for (auto* v : {&j.kev, &j.cev}) {
    double sum = 0;
    for (size_t i = 0; i < v->size(); ++i) {
      auto& e = (*v)[i];
      float ms = 0;
      SLLM_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      sum += ms;
      if (dump) {
        float at = 0;
        SLLM_CUDA(cudaEventElapsedTime(&at, j.ev[0], e.first));
        if (v == &j.kev) {
          fprintf(stderr, "sllm-prof p=%zu kernel=%zu start_ms=%.4f ms=%.4f bytes=%llu GBps=%.1f", j.p, i, at, ms,
                  (unsigned long long)j.kev_bytes[i], j.kev_bytes[i] / (ms * 1e6));
          if (4 * i + 3 < kt.size()) {  // kernel span (first CTA start .. last CTA end), CTA start / end spread
            const unsigned long long s0 = ~kt[4 * i], s1 = kt[4 * i + 1], e0 = ~kt[4 * i + 2], e1 = kt[4 * i + 3];
            fprintf(stderr, " span_ms=%.4f start_spread_us=%.2f end_spread_us=%.2f", (e1 - s0) * 1e-6,
                    (s1 - s0) * 1e-3, (e1 - e0) * 1e-3);
          }
          fprintf(stderr, "\n");
        } else
          fprintf(stderr, "sllm-prof p=%zu copy=%zu start_ms=%.4f ms=%.4f\n", j.p, i, at, ms);
      }
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    (v == &j.kev ? j.kernel_ms : j.copy_ms) = sum;
    v->clear();
    j.kev_bytes.clear();
  }
  cudaEventDestroy(P.copied);
  for (auto& e : P.freed) cudaEventDestroy(e);
  SLLM_CUDA(cudaGetLastError());
  if (j.h_err) fail(SLLM_E_PEER, "P2P fan-out: peer rank " + std::to_string(j.h_err - 1) +
                                     " did not signal completion within the timeout");
}

// Worker threads of the partition jobs, kept for the next load (a thread start and join per
// partition per load cost ~50 us of a 0.44 ms toy load).  A job runs for its whole load and
// the jobs of an in-process P2P group wait for each other, so a job never queues behind
// another: run() starts a thread whenever fewer threads are idle than jobs are pending.
// Threads are detached; at most kMaxIdle stay parked; the pool is never destroyed (threads
// parked at exit are simply ended with the process).
class WorkerPool {
 public:
  void run(std::function<void()> f) {
    std::lock_guard<std::mutex> g(mu_);
    q_.push_back(std::move(f));
    if (idle_ < q_.size()) {
      try {
        std::thread([this] { loop(); }).detach();
      } catch (...) {  // the job never runs: take it back, the caller fails it
        q_.pop_back();
        throw;
      }
    }
    cv_.notify_one();
  }

 private:
  static constexpr size_t kMaxIdle = 16;
  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      ++idle_;
      cv_.wait(lk, [&] { return !q_.empty(); });
      --idle_;
      std::function<void()> f = std::move(q_.front());
      q_.pop_front();
      lk.unlock();
      f();
      f = nullptr;
      lk.lock();
      if (idle_ >= kMaxIdle) return;
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  size_t idle_ = 0;
};

static WorkerPool& worker_pool() {
  static WorkerPool* pool = new WorkerPool;  // intentionally never destroyed (see above)
  return *pool;
}

static void run_job_guarded(sllm_load* L, PartJob& j) {
  try {
    run_job(L, j);
  } catch (const Error& e) {
    j.status = e.code;
    j.error = e.what();
  } catch (const std::exception& e) {
    j.status = SLLM_E_INVALID;
    j.error = e.what();
  }
  if (j.status != SLLM_OK && j.gpu >= 0) {
    // a failure part-way through issuing: let what was queued finish before the scratch,
    // staging and events it uses can be released by sllm_load_free
    cudaSetDevice(j.gpu);
    if (j.capture)  // (a failure inside a capture: end it so the streams can be reused)
      for (cudaStream_t st : j.used) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
          cudaGraph_t g = nullptr;
          cudaStreamEndCapture(st, &g);
          if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();
      }
    for (cudaStream_t st : j.used) cudaStreamSynchronize(st);
    cudaGetLastError();
  }
  if (j.ss) {  // every stream of the set is idle now (synchronized above or in run_job)
    DeviceCtx& dc = device_ctx(j.gpu);
    std::lock_guard<std::mutex> g(dc.mu);
    dc.release(j.ss);
    j.ss = nullptr;
  }
  {  // a job that failed before enqueueing everything still unblocks sllm_load_start
    std::lock_guard<std::mutex> g(L->issue_mu);
    j.issue_signalled = true;
    j.finished = true;
  }
  L->issue_cv.notify_all();
}

}  // namespace sllm

using namespace sllm;

void sllm_load_free_internal(sllm_load* L);

sllm_load* sllm_load_create_internal(const sllm_index* idx, const sllm_load_config* cfg_in, const void* const* host_src,
                                     const int32_t* gpu, void* const* dst_base, void* const* dst_tensor,
                                     void* const* stream, sllm_comm* comm, const char* dir, int32_t io_threads,
                                     bool capture) {
  NvtxRange nv(capture ? "sllm.load_capture" : "sllm.load_start");
  if (!idx) fail(SLLM_E_INVALID, "null index");
  if (!idx->sealed) fail(SLLM_E_INVALID, "index is planned but not sealed");
  sllm_load_config cfg{};
  if (cfg_in) cfg = *cfg_in;
  else cfg.verify = 1;
  if (cfg.chunk_bytes == 0) cfg.chunk_bytes = 16ull << 20;
  if (cfg.n_streams == 0) cfg.n_streams = 2;
  if (cfg.n_streams < 1 || cfg.n_streams > kMaxStreams) fail(SLLM_E_INVALID, "n_streams must be in 1..8");
  if (cfg.mode < SLLM_MODE_CE || cfg.mode > SLLM_MODE_GDS) fail(SLLM_E_INVALID, "unknown mode");
  if (cfg.mode == SLLM_MODE_GDS && !dir) fail(SLLM_E_INVALID, "SLLM_MODE_GDS reads partition files (sllm_load_files_start)");
  if (cfg.mode == SLLM_MODE_GDS && cfg.fanout != SLLM_FANOUT_NONE) fail(SLLM_E_INVALID, "SLLM_MODE_GDS has no fan-out");
  if (cfg.mode == SLLM_MODE_GDS && !(getenv("SLLM_ENABLE_GDS") && atoi(getenv("SLLM_ENABLE_GDS")) == 1))
    // cuFileDriverOpen never returns on hosts without nvidia-fs where its compatibility mode
    // cannot probe the PCI topology (the VMs of this build: profiles/r01/gds_probe.log), and a
    // hung driver open cannot be cancelled -- so GPUDirect Storage is opt-in per host.
    fail(SLLM_E_INVALID, "SLLM_MODE_GDS is opt-in: set SLLM_ENABLE_GDS=1 on hosts with a working cuFile (nvidia-fs)");
  // AUTO: the copy engine unless every job moves less than kAutoZeroCopyBytes over PCIe from
  // device-mapped memory -- then the zero-copy kernel, whose lower fixed cost wins for small
  // loads (measured crossover).  Resolved below once the jobs are known.
  const bool auto_mode = cfg.mode == SLLM_MODE_AUTO;
  if (auto_mode) cfg.mode = SLLM_MODE_CE;
  if (cfg.profile < 0 || cfg.profile > 3) fail(SLLM_E_INVALID, "profile must be 0, 1, 2 or 3");
  if (cfg.engine < 0 || cfg.engine > 3) fail(SLLM_E_INVALID, "unknown kernel engine");
  if (cfg.reserved) fail(SLLM_E_INVALID, "reserved config field must be 0");
  if (cfg.chunk_bytes % tile_for(*idx)) fail(SLLM_E_INVALID, "chunk size must be a multiple of the 64 KiB work tile");
  if (idx->block && cfg.chunk_bytes % idx->block) fail(SLLM_E_INVALID, "chunk size must be a multiple of the block size");
  if (cfg.chunk_bytes % idx->align) fail(SLLM_E_INVALID, "chunk size must be a multiple of the alignment");
  const bool scatter = cfg.mode == SLLM_MODE_SCATTER_CE || cfg.mode == SLLM_MODE_SCATTER_ZC;
  const bool group_fanout = cfg.fanout == SLLM_FANOUT_P2P || cfg.fanout == SLLM_FANOUT_NVLS;
  if (cfg.fanout == SLLM_FANOUT_BCAST || group_fanout || cfg.fanout == SLLM_FANOUT_ALLGATHER) {
    if (!comm) fail(SLLM_E_INVALID, "fan-out needs a communicator");
    if (!group_fanout && comm_is_peers(comm))
      fail(SLLM_E_INVALID, "SLLM_FANOUT_BCAST/ALLGATHER need an NCCL communicator (sllm_comm_init_rank/_all)");
    if (cfg.fanout == SLLM_FANOUT_NVLS && !comm_mc(comm))
      fail(SLLM_E_INVALID, "SLLM_FANOUT_NVLS needs an NVLS group (sllm_comm_init_nvls)");
    if (cfg.fanout == SLLM_FANOUT_P2P && comm_mc(comm))
      fail(SLLM_E_INVALID, "an NVLS group's replicas take multicast stores only: use SLLM_FANOUT_NVLS");
    if (cfg.fanout == SLLM_FANOUT_NVLS && cfg.engine == 2) fail(SLLM_E_INVALID, "the NVLS fan-out needs the TMA engine");
    if (cfg.fanout == SLLM_FANOUT_ALLGATHER && dir)
      fail(SLLM_E_INVALID, "SLLM_FANOUT_ALLGATHER loads from pinned sources only (its chunks are strided)");
    if (cfg.fanout == SLLM_FANOUT_P2P && !comm_is_peers(comm))
      fail(SLLM_E_INVALID, "SLLM_FANOUT_P2P needs a peer group (sllm_comm_init_peers)");
    if (cfg.fanout == SLLM_FANOUT_P2P && cfg.engine == 2) fail(SLLM_E_INVALID, "the P2P fan-out needs the TMA engine");
    if (idx->parts.size() != 1) fail(SLLM_E_INVALID, "fan-out needs a single-partition (replicated) index");
    if (scatter) fail(SLLM_E_INVALID, "fan-out supports the contiguous modes only");
  } else if (cfg.fanout != SLLM_FANOUT_NONE) {
    fail(SLLM_E_INVALID, "unknown fan-out");
  }
  if (capture) {  // a captured load replays one fixed sequence of device work
    if (dir || cfg.mode == SLLM_MODE_GDS) fail(SLLM_E_INVALID, "sllm_load_capture loads from pinned sources only");
    if (cfg.fanout != SLLM_FANOUT_NONE) fail(SLLM_E_INVALID, "sllm_load_capture has no fan-out");
    cfg.profile = 0;
    stream = nullptr;  // (the replay takes the streams)
  }
  if ((!host_src && !dir) || !gpu) fail(SLLM_E_INVALID, "null host_src / gpu array");
  if (scatter && !dst_tensor) fail(SLLM_E_INVALID, "scatter modes need dst_tensor");
  if (!scatter && !dst_base) fail(SLLM_E_INVALID, "contiguous modes need dst_base");

  std::unique_ptr<sllm_load> L(new sllm_load);
  L->idx = idx;
  L->cfg = cfg;
  L->graph = capture;
  L->comm = comm;
  L->t0 = std::chrono::steady_clock::now();
  if (scatter) L->dst_tensor.assign(dst_tensor, dst_tensor + idx->tensors.size());
  for (size_t p = 0; p < idx->parts.size(); ++p) {
    if (dir ? gpu[p] < 0 : !host_src[p]) continue;
    PartJob j;
    j.p = p;
    j.gpu = gpu[p];
    if (dir) {
      j.file = std::string(dir) + "/part_" + std::to_string(idx->parts[p].device) + ".bin";
      j.io_threads = io_threads;
    } else {
      j.src = static_cast<const uint8_t*>(host_src[p]);
    }
    j.dst_base = dst_base ? static_cast<uint8_t*>(dst_base[p]) : nullptr;
    j.origin = stream ? static_cast<cudaStream_t>(stream[p]) : nullptr;
    if (!scatter && !j.dst_base) fail(SLLM_E_INVALID, "null dst_base for a loaded partition");
    if (cfg.fanout != SLLM_FANOUT_NONE && comm_device(comm) != j.gpu)
      fail(SLLM_E_INVALID, "communicator belongs to another GPU");
    j.lo = 0;
    j.hi = idx->parts[p].length;
    if (cfg.fanout != SLLM_FANOUT_NONE) {  // this rank's slice: the only bytes it reads from the host
      const int R = comm_nranks(comm), me = comm_rank(comm);
      std::vector<uint64_t> lohi(2 * R);
      const uint64_t U = fanout_unit(cfg.chunk_bytes, cfg.fanout);
      if (sllm_replica_slices(j.hi, U, R, lohi.data()) != SLLM_OK) fail(SLLM_E_INVALID, "bad slices");
      j.lo = lohi[2 * me];
      j.hi = lohi[2 * me + 1];
      if (cfg.fanout == SLLM_FANOUT_ALLGATHER) {  // units me, me+R, me+2R, ... (strided)
        j.lo = std::min((uint64_t)me * U, idx->parts[p].length);
        j.hi = idx->parts[p].length;
      }
    }
    if (group_fanout) {
      if (j.dst_base != comm_peer_base(comm, comm_rank(comm)))
        fail(SLLM_E_INVALID, "P2P / NVLS fan-out: dst_base must be this rank's replica of the group");
      if (cfg.fanout == SLLM_FANOUT_NVLS) {
        j.mc = comm_mc(comm);
      } else {
        for (int q = 0; q < comm_nranks(comm); ++q)
          if (q != comm_rank(comm)) j.peers[j.n_peers++] = comm_peer_base(comm, q);
      }
    }
    if (j.dst_base && (reinterpret_cast<uintptr_t>(j.dst_base) & 15)) fail(SLLM_E_INVALID, "dst_base must be 16-byte aligned");
    if (scatter) {
      for (uint32_t ti : idx->parts[p].by_offset) {
        if (!dst_tensor[ti]) fail(SLLM_E_INVALID, "null destination for tensor '" + std::string(idx->tensors[ti].name) + "'");
        if (reinterpret_cast<uintptr_t>(dst_tensor[ti]) & 15)
          fail(SLLM_E_INVALID, "destination of '" + std::string(idx->tensors[ti].name) + "' is not 16-byte aligned");
      }
    }
    SLLM_CUDA(cudaSetDevice(j.gpu));
    if (!dir) {
      // the source must be page-locked host memory ("pinned memory ... DMA")
      // (with a fan-out only the rank's slice needs to be pinned: check where it starts)
      const uint64_t probe = j.hi > j.lo ? j.lo : 0;
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, j.src + probe) != cudaSuccess || at.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        fail(SLLM_E_INVALID, "partition source is not pinned host memory (use sllm_host_alloc / sllm_host_register)");
      }
      j.src_dev = at.devicePointer ? static_cast<const uint8_t*>(at.devicePointer) - probe : nullptr;
      if ((cfg.mode == SLLM_MODE_ZEROCOPY || cfg.mode == SLLM_MODE_SCATTER_ZC) && !j.src_dev)
        fail(SLLM_E_INVALID, "zero-copy modes need host memory mapped into the device address space");
      // the zero-copy kernels read the source with 16-byte vector loads / TMA bulk copies from
      // window starts (multiples of the chunk size): a misaligned source would fault the
      // context, so it is refused here (AUTO then keeps the copy engine)
      if ((cfg.mode == SLLM_MODE_ZEROCOPY || cfg.mode == SLLM_MODE_SCATTER_ZC) &&
          (reinterpret_cast<uintptr_t>(j.src_dev) & 15))
        fail(SLLM_E_INVALID, "zero-copy modes need a 16-byte aligned host source");
    }
    build_segments(*idx, j, scatter, L->dst_tensor, cfg.chunk_bytes);
    j.capture = capture;
    L->jobs.push_back(std::move(j));
  }
  // busy set
  if (auto_mode) {
    bool zc = !L->jobs.empty();
    for (auto& j : L->jobs)
      zc = zc && (j.hi - j.lo) < kAutoZeroCopyBytes &&
           (!j.file.empty() || (j.src_dev && !(reinterpret_cast<uintptr_t>(j.src_dev) & 15)));
    if (zc) cfg.mode = L->cfg.mode = SLLM_MODE_ZEROCOPY;
  }
  {
    std::lock_guard<std::mutex> g(g_busy_mu);
    std::vector<const void*> keys;
    for (auto& j : L->jobs) {
      if (j.dst_base) keys.push_back(j.dst_base);
      if (scatter)
        for (uint32_t ti : idx->parts[j.p].by_offset) keys.push_back(L->dst_tensor[ti]);
    }
    for (const void* k : keys)
      if (g_busy.count(k)) fail(SLLM_E_BUSY, "destination is already being loaded");
    for (const void* k : keys) g_busy.insert(k);
    L->busy_keys = std::move(keys);
  }
  // Caller-stream ordering is fixed here, on the caller's thread, before returning: the
  // load starts after work already queued on stream[p], and stream[p] waits for the load.
  try {
    for (auto& j : L->jobs) {
      SLLM_CUDA(cudaSetDevice(j.gpu));
      for (auto& e : j.ev) SLLM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDefault));
      if (j.origin) {
        SLLM_CUDA(cudaEventRecord(j.ev[3], j.origin));
        // (a group whose issue waits for its peers -- in-process ranks, host-polled flags --
        // orders the caller's stream in sllm_load_wait, so sllm_load_start stays asynchronous)
        j.eager = j.file.empty() && !(group_fanout && (comm_local_members(comm) > 1 || comm_host_wait()));
      }
    }
  } catch (...) {
    std::lock_guard<std::mutex> g(g_busy_mu);
    for (const void* k : L->busy_keys) g_busy.erase(k);
    for (auto& j : L->jobs) {
      for (auto& e : j.ev)
        if (e) cudaEventDestroy(e);
    }
    throw;
  }
  if (group_fanout)  // one epoch per collective load, taken in call order
    for (auto& j : L->jobs) j.epoch = comm_next_epoch(comm);
  for (auto& j : L->jobs) {
    sllm_load* Lp = L.get();
    PartJob* jp = &j;
    try {
      worker_pool().run([Lp, jp] { run_job_guarded(Lp, *jp); });
    } catch (const std::exception& e) {  // no thread for this job: it fails, the load stays valid
      std::lock_guard<std::mutex> g(L->issue_mu);
      j.status = SLLM_E_INVALID;
      j.error = std::string("cannot start a load worker thread: ") + e.what();
      j.issue_signalled = j.finished = true;
    }
  }
  if (capture) {  // every job's graph is built before sllm_load_capture returns
    {
      std::unique_lock<std::mutex> lk(L->issue_mu);
      L->issue_cv.wait(lk, [&] {
        for (auto& j : L->jobs)
          if (!j.finished) return false;
        return true;
      });
    }
    for (auto& j : L->jobs)
      if (j.status != SLLM_OK) {
        const sllm_status st = j.status;
        const std::string err = j.error;
        sllm_load_free_internal(L.release());
        fail(st, err);
      }
    return L.release();
  }
  // Caller-stream ordering without a device-side gate: a stream waiting for work that is not
  // yet enqueued can block, through the few hardware queues the context's streams share,
  // work this or another load enqueues later (a deadlock seen with concurrent gated loads).
  // So the caller's stream waits on ev[1] only once the job has enqueued everything -- the
  // host issue of a pinned-source job takes well under the transfer time.
  {
    std::unique_lock<std::mutex> lk(L->issue_mu);
    L->issue_cv.wait(lk, [&] {
      for (auto& j : L->jobs)
        if (j.eager && !j.issue_signalled) return false;
      return true;
    });
  }
  for (auto& j : L->jobs)
    if (j.eager && j.issue_ok) {
      cudaSetDevice(j.gpu);
      if (cudaStreamWaitEvent(j.origin, j.ev[1], 0) != cudaSuccess) cudaGetLastError();
    }
  return L.release();
}

// Captured load: the last replay's completion and verification result (idempotent until the
// next replay).
static void join_replay(sllm_load* L) {
  if (!L->replay_pending) return;
  L->replay_pending = false;
  sllm_load_report& r = L->rep;
  r = sllm_load_report{};
  r.bad_partition = -1;
  r.bad_block = ~0ull;
  r.mode = L->cfg.mode;
  sllm_status st = SLLM_OK;
  for (auto& j : L->jobs) {
    cudaSetDevice(j.gpu);
    cudaError_t e = cudaEventSynchronize(j.ev[1]);
    float ms = 0;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, j.ev[0], j.ev[1]);
    if (e != cudaSuccess && st == SLLM_OK) {
      cudaGetLastError();
      st = SLLM_E_CUDA;
      set_last_error(std::string("replay: ") + cudaGetErrorString(e));
    }
    uint64_t tail[2] = {};
    std::memcpy(tail, j.h_result, 16);  // written by the graph's last node
    j.h_bad = tail[0];
    j.h_cs_valid = false;
    for (uint32_t ti : L->idx->parts[j.p].by_offset) r.payload_bytes += L->idx->tensors[ti].nbytes;
    r.transferred_bytes += j.transferred;
    r.chunks += j.chunks;
    r.kernel_launches += j.launches;
    r.copy_calls += j.copies;
    r.t_device_ms_max = std::max(r.t_device_ms_max, (double)ms);
    if (st == SLLM_OK && j.h_bad != ~0ull && r.bad_partition < 0) {
      r.bad_partition = (int32_t)j.p;
      r.bad_block = j.h_bad;
    }
  }
  r.t_issue_ns_max = L->t_replay_issue_ns;
  if (st == SLLM_OK && r.bad_partition >= 0) {
    st = SLLM_E_CHECKSUM;
    set_last_error("checksum mismatch in partition " + std::to_string(r.bad_partition) + ", block " +
                   std::to_string(r.bad_block));
  }
  r.t_total_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() -
                                                                                L->t_replay).count();
  L->result = st;
}

static void join_load(sllm_load* L) {
  if (L->graph) return join_replay(L);
  if (L->joined) return;
  {
    std::unique_lock<std::mutex> lk(L->issue_mu);
    L->issue_cv.wait(lk, [&] {
      for (auto& j : L->jobs)
        if (!j.finished) return false;
      return true;
    });
  }
  L->joined = true;
  for (auto& j : L->jobs)  // file tier / in-process P2P: the caller's stream is ordered here
    if (j.origin && !j.eager && j.issue_ok) {
      cudaSetDevice(j.gpu);
      if (cudaStreamWaitEvent(j.origin, j.ev[1], 0) != cudaSuccess) cudaGetLastError();
    }
  {
    std::lock_guard<std::mutex> g(g_busy_mu);
    for (const void* k : L->busy_keys) g_busy.erase(k);
    L->busy_keys.clear();
  }
  sllm_load_report& r = L->rep;
  r = sllm_load_report{};
  r.bad_partition = -1;
  r.bad_block = ~0ull;
  r.mode = L->cfg.mode;
  sllm_status st = SLLM_OK;
  std::string err;
  for (auto& j : L->jobs) {
    for (uint32_t ti : L->idx->parts[j.p].by_offset) r.payload_bytes += L->idx->tensors[ti].nbytes;
    r.transferred_bytes += j.transferred;
    r.fanout_bytes += j.fanout;
    r.chunks += j.chunks;
    r.kernel_launches += j.launches;
    r.copy_calls += j.copies;
    r.t_issue_ns_max = std::max(r.t_issue_ns_max, j.t_issue_ns);
    r.t_device_ms_max = std::max(r.t_device_ms_max, (double)j.t_dev_ms);
    r.t_kernel_ms_sum += j.kernel_ms;
    r.t_kernel_span_ms_sum += j.kernel_span_ms;
    r.t_copy_ms_sum += j.copy_ms;
    r.kernel_bytes += j.kernel_bytes;
    r.storage_bytes += j.storage_bytes;
    r.t_storage_wait_ns_max = std::max(r.t_storage_wait_ns_max, j.storage_wait_ns);
    if (j.status != SLLM_OK && st == SLLM_OK) {
      st = j.status;
      err = j.error;
    }
    if (j.status == SLLM_OK && j.h_bad != ~0ull && r.bad_partition < 0) {
      r.bad_partition = (int32_t)j.p;
      r.bad_block = j.h_bad;
    }
  }
  if (st == SLLM_OK && r.bad_partition >= 0) {
    st = SLLM_E_CHECKSUM;
    err = "checksum mismatch in partition " + std::to_string(r.bad_partition) + ", block " + std::to_string(r.bad_block);
  }
  r.t_total_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - L->t0).count();
  L->result = st;
  if (st != SLLM_OK) set_last_error(err);
}

sllm_status sllm_load_wait_internal(sllm_load* L, sllm_load_report* rep) {
  NvtxRange nv("sllm.load_wait");
  join_load(L);
  if (rep) *rep = L->rep;
  if (L->result != SLLM_OK) {
    for (auto& j : L->jobs)
      if (j.status != SLLM_OK) { set_last_error(j.error); break; }
    if (L->result == SLLM_E_CHECKSUM)
      set_last_error("checksum mismatch in partition " + std::to_string(L->rep.bad_partition) + ", block " +
                     std::to_string(L->rep.bad_block));
  }
  return L->result;
}

void sllm_load_tensor_internal(const sllm_load* L, const char* name, sllm_tensor_handle* h) {
  if (!name || !h) fail(SLLM_E_INVALID, "null argument");
  const uint32_t id = L->idx->by_name.find(name, L->idx->tensors);
  if (id == NameTable::kNone) fail(SLLM_E_LOOKUP, std::string("unknown tensor '") + name + "'");
  const TensorRec& t = L->idx->tensors[id];
  const PartJob* job = nullptr;
  for (auto& j : L->jobs)
    if ((int32_t)j.p == t.part) job = &j;
  if (!job) fail(SLLM_E_LOOKUP, "tensor '" + std::string(t.name) + "' belongs to a partition this load does not handle");
  sllm_tensor_handle o{};
  o.gpu = job->gpu;
  o.dtype = t.dtype;
  o.ndim = t.ndim;
  std::memcpy(o.shape, t.shape, sizeof o.shape);
  o.ptr = L->dst_tensor.empty() ? (void*)(job->dst_base + t.offset) : L->dst_tensor[id];
  o.nbytes = t.nbytes;
  *h = o;
}

void sllm_load_block_checksums_internal(sllm_load* L, size_t p, const uint64_t** table) {
  join_load(L);
  for (auto& j : L->jobs) {
    if (j.p != p) continue;
    if (!j.h_cs_valid) {
      j.h_cs.assign(L->idx->parts[p].n_blocks, 0);
      if (!j.h_cs.empty() && j.d_cs) {
        SLLM_CUDA(cudaSetDevice(j.gpu));
        SLLM_CUDA(cudaMemcpy(j.h_cs.data(), j.d_cs, j.h_cs.size() * 8, cudaMemcpyDeviceToHost));
      }
      j.h_cs_valid = true;
    }
    *table = j.h_cs.data();
    return;
  }
  fail(SLLM_E_LOOKUP, "partition not handled by this load");
}

void sllm_load_free_internal(sllm_load* L) {
  join_load(L);
  if (L->graph) {  // the destinations were reserved for the captured load's lifetime
    std::lock_guard<std::mutex> g(g_busy_mu);
    for (const void* k : L->busy_keys) g_busy.erase(k);
    L->busy_keys.clear();
  }
  for (auto& j : L->jobs) {
    if (j.gpu >= 0) cudaSetDevice(j.gpu);
    DeviceCtx& dc = device_ctx(j.gpu);
    if (j.exec) cudaGraphExecDestroy(j.exec);
    if (j.rstream) cudaStreamDestroy(j.rstream);
    if (j.scratch) cudaFreeAsync(j.scratch, dc.misc);
    if (j.staging) cudaFreeAsync(j.staging, dc.misc);
    if (j.gstage) cudaFreeHost(j.gstage);  // (join_load above waited for the last replay)
    for (auto& e : j.ev)
      if (e) cudaEventDestroy(e);
  }
  delete L;
}

// One replay of a captured load: per job, one graph launch on its stream between two timing
// events (the second also marks completion for sllm_load_wait).
void sllm_load_replay_internal(sllm_load* L, void* const* stream) {
  if (!L->graph) fail(SLLM_E_INVALID, "not a captured load (sllm_load_capture)");
  if (L->replay_pending) fail(SLLM_E_BUSY, "the previous replay has not been waited for");
  const uint64_t t0 = now_ns();
  L->t_replay = std::chrono::steady_clock::now();
  L->replay_pending = true;  // (set first: a failure part-way still gets the launched graphs waited for)
  for (auto& j : L->jobs) {
    SLLM_CUDA(cudaSetDevice(j.gpu));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream[j.p]) : nullptr;
    if (!st) {
      if (!j.rstream) SLLM_CUDA(cudaStreamCreateWithFlags(&j.rstream, cudaStreamNonBlocking));
      st = j.rstream;
    }
    SLLM_CUDA(cudaEventRecord(j.ev[0], st));
    SLLM_CUDA(cudaGraphLaunch(j.exec, st));
    SLLM_CUDA(cudaEventRecord(j.ev[1], st));
  }
  L->replays++;
  L->t_replay_issue_ns = now_ns() - t0;
}

void sllm_device_trim_internal(int32_t gpu, uint64_t keep_bytes) {
  if (gpu < 0) fail(SLLM_E_INVALID, "bad GPU ordinal");
  SLLM_CUDA(cudaSetDevice(gpu));
  cudaMemPool_t pool;
  SLLM_CUDA(cudaDeviceGetDefaultMemPool(&pool, gpu));
  SLLM_CUDA(cudaDeviceSynchronize());  // frees queued by finished loads have taken effect
  SLLM_CUDA(cudaMemPoolTrimTo(pool, (size_t)keep_bytes));
}
