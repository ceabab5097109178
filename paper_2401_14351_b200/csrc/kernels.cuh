// Device-side data structures shared by kernels.cu (device code) and loader.cpp (host).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sllm {

// A 16-byte aligned byte range of a partition and where its bytes go.
//   [off, off+len)  partition bytes covered (off, len multiples of 16)
//   dst             device pointer receiving byte `off` (nullptr: checksum only -- padding)
//   valid           bytes of [off, off+valid) that belong to the tensor (<= len); the rest
//                   of the last 16-byte vector is partition padding and is not stored.
struct Seg {
  uint64_t off;
  uint64_t len;
  uint8_t* dst;
  uint64_t valid;
};

// Per-block checksum accumulator (closed form of Q8):
//   a = sum w_i,  b = sum i*w_i (i = word index in the block, per 16 B vector i0*sum4),
//   c = sum k*w_{i0+k} within each vector;  s1 = a,  s2 = n*a - b - c  (all mod 2^32-1).
struct BlockAcc {
  unsigned long long a, b, c, tiles_done;
};

constexpr int kMaxPeers = 7;  // P2P fan-out: up to 8 GPUs (an NVSwitch node)

// One launch of the materialise/checksum kernel covers partition bytes [lo, hi).
struct MatParams {
  const uint8_t* src;        // address holding partition byte `src_origin` (host-mapped or device)
  uint64_t src_origin;
  uint64_t lo, hi;           // multiples of 16; lo is a multiple of `tile`
  const Seg* segs;           // segments covering [lo, hi), sorted by off
  uint32_t seg_begin, seg_end;
  // optional (scatter modes): gran_seg[g] = last segment with off <= g << gran_shift, for
  // g = 0..ceil(L >> gran_shift); bounds each unit's segment search to one granule's segments
  const uint32_t* gran_seg;
  uint32_t gran_shift;
  uint32_t tile;             // bytes per work tile (divides block; multiple of 16)
  uint64_t block;            // checksum block size B (0 = no checksum)
  uint64_t part_len;         // L_p
  BlockAcc* acc;             // n_blocks accumulators (zeroed before the load)
  const uint64_t* expect;    // expected block checksums, or nullptr
  uint64_t* cs_out;          // computed block checksums, or nullptr
  unsigned long long* bad;   // min failing block index (init UINT64_MAX)
  int host_src;              // 1: src is host-mapped pinned memory (zero-copy over PCIe)
  int engine;                // 0: LDG/STG tiles; 1: TMA bulk loads through a shared-memory ring,
                             // STG stores; 2: as 1 with TMA bulk stores out of the ring
  uint32_t split;            // TMA engine: units per checksum block (set by the launcher)
  // TMA engine fine tail (set by the launcher): the first n_coarse units are whole units,
  // the rest of the range is cut into units of unit / fine bytes (fine = 1: no tail)
  uint32_t fine;
  uint64_t n_coarse;
  // P2P fan-out (TMA engine, contiguous single segment): every stored vector of partition
  // offset x also goes to peer[k] + x -- device pointers to the other GPUs' replicas,
  // written over NVLink -- and, with no_seg_store, only there (CE: the source is the
  // rank's own replica, already in place).
  uint32_t n_peers;
  uint32_t no_seg_store;
  uint8_t* peer[kMaxPeers];
  // NVLS fan-out: multicast address of partition byte 0 -- every vector is stored once with
  // multimem.st and lands in every replica of the group (own included); no per-segment store
  uint8_t* mc;
  // diagnostic (profile dumps with SLLM_KTIME=1, else nullptr): 4 words per launch, zeroed
  // before it -- [0] = ~min CTA start, [1] = max CTA start, [2] = ~min CTA end, [3] = max
  // CTA end (%globaltimer ns; the complements let one atomicMax serve min and max)
  unsigned long long* ktime;
  // TMA engine work distribution: nullptr = static (CTA b takes units b, b + grid, ...);
  // else CTA b takes unit b first and then unit grid + (atomicAdd(ticket, 1) - ticket_base)
  // until that is past the launch's last unit.  Every launch draws exactly `units` tickets
  // (each CTA draws one past the end), so consecutive launches on one stream share one
  // counter by advancing ticket_base (launch_materialise reports the count).
  unsigned long long* ticket;
  unsigned long long ticket_base;
};

enum class MatKind : int {
  kChecksumOnly = 0,   // K4: read a device buffer, checksum only
  kCopyChecksum = 1,   // K2/K3: read (host-mapped or device), store per segment, checksum
  kCopyOnly = 2        // K2/K3 with verify off
};

// Launch on `stream` with `grid` CTAs.  Returns cudaGetLastError(); *tickets (optional) =
// tickets the launch draws from p.ticket (0 when it does not use one).
cudaError_t launch_materialise(const MatParams& p, MatKind kind, int grid, cudaStream_t stream,
                               uint64_t* tickets = nullptr);

// P2P fan-out completion: publish `epoch` into one slot of every peer's
// signal array (system-scope release, after every store of the preceding kernels), and
// wait until every peer has published at least `epoch` into this GPU's own array
// (system-scope acquire).  A peer that has not signalled after timeout_ns sets
// *err = 1 + its rank and the wait returns (no hang).
struct PeerSignal {
  uint32_t* remote[kMaxPeers];  // &signal_q[me] for every peer q
  uint32_t n;
};
cudaError_t launch_peer_signal(const PeerSignal& s, uint32_t epoch, cudaStream_t stream);
// Write the single whole-buffer segment {0, len, null, 0} of a device-resident checksum
// pass (no host staging copy on the stream: a pageable upload would synchronise it).
cudaError_t launch_init_seg(Seg* seg, uint64_t len, cudaStream_t stream);
cudaError_t launch_peer_wait(const uint32_t* own, int nranks, int me, uint32_t epoch, uint64_t timeout_ns,
                             uint32_t* err, cudaStream_t stream);


}  // namespace sllm
