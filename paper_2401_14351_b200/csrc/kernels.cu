// sm_100a kernels of the load path:
//   K2  zero-copy read of host-mapped pinned memory (PCIe, SM-issued 16 B loads) -> HBM,
//       with the block checksum fused;
//   K3  index-driven scatter: partition bytes (staging chunk in HBM, or host-mapped) ->
//       per-tensor buffers, checksum fused;
//   K4  checksum-only pass over a device buffer (CE-contiguous mode verification).
// All three are one template: a persistent grid walks fixed-size tiles of the launch's
// byte range; inside a tile it walks the index-derived segments (tensor bytes or
// padding) with coalesced 16-byte vectors, U loads in flight per thread.
//
// Checksum (Q8): Fletcher-64 per block of B bytes,
// evaluated in closed form so tiles/threads may add their terms in any order:
//   s1 = sum_i w_i,  s2 = sum_i (n - i) w_i = n*sum w - sum_v i0_v*sum4_v - sum_v (w1+2w2+3w3)_v
// (v = 16-byte vector whose first word has block index i0_v).  Per-thread partials are
// folded mod 2^32-1 after every segment, reduced over the CTA with warp shuffles, and
// added atomically into the block's accumulator; the CTA finishing a block's last tile
// finalises it and compares against the index's table.
#include <atomic>
#include <cstdlib>

#include "kernels.cuh"

namespace sllm {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 16;                       // 16 x 16 B in flight per thread
constexpr unsigned long long kM = 0xFFFFFFFFull;  // 2^32 - 1

__device__ __forceinline__ unsigned long long fold(unsigned long long x) {
  x = (x & kM) + (x >> 32);
  x = (x & kM) + (x >> 32);
  return x >= kM ? x - kM : x;
}

#ifndef SLLM_HOST_L2_PREFETCH
#define SLLM_HOST_L2_PREFETCH 0
#endif

template <bool kHostSrc>
__device__ __forceinline__ uint4 load16(const uint8_t* p) {
  uint4 r;
  if (kHostSrc) {
    // host-mapped pinned memory over PCIe: plain global load, no L1 allocation
#if SLLM_HOST_L2_PREFETCH == 256  // A/B knob: ask the L2 for 256-byte fills of the host lines
    asm("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#else
    asm("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#endif
  } else {
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  }
  return r;
}

// NVLS: one store through the multicast address reaches every replica bound to it (the
// 32-bit lanes are moved, never converted: an .f32 store is a bit copy)
__device__ __forceinline__ void mc_store16(uint8_t* p, const uint4& v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// L2 evict-first hints (profiles/r02/l2_hints/, ncu + bench A/B on one box): on the ring's
// TMA bulk loads of the store kernels (K3 / K2 / fan-out) the read bytes leave L2 first and
// the stores keep it -- K3 4.26 -> 4.19 ms per 26.6 GB, in-pipeline K3 0.899 -> 0.907
// in-kernel; on K4 (read only) the hint costs ~1 % (0.622 -> 0.627 ms per 4 GiB), and on the
// stores it costs 3 % (K3 4.39 ms), on host-mapped sources (K2) 1 %.  SLLM_LD_HINT: 0 never,
// 1 every ring kernel, 2 (default) store kernels reading HBM only; SLLM_ST_HINT=1 puts the hint
// on the stores (A/B knobs).
#ifndef SLLM_ST_HINT
#define SLLM_ST_HINT 0
#endif
#ifndef SLLM_LD_HINT
#define SLLM_LD_HINT 2
#endif
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void store16(uint8_t* p, const uint4& v) {
#if SLLM_ST_HINT
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(evict_first_policy()) : "memory");
#else
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
#endif
}

// Store the first n (< 16) bytes of v at p (tensor tail; the rest of the vector is padding).
__device__ __forceinline__ void store_partial(uint8_t* p, const uint4& v, uint32_t n) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (uint32_t k = 0; k < 16; ++k)
    if (k < n) p[k] = (uint8_t)(w[k / 4] >> (8 * (k % 4)));
}

template <bool kStore, bool kCheck, bool kHostSrc>
__global__ void __launch_bounds__(kThreads) materialise_kernel(const MatParams p) {
  __shared__ uint32_t s_seg;
  __shared__ unsigned long long s_red[3][kThreads / 32];
  const int tid = threadIdx.x;
  const uint64_t T = p.tile;
  const uint64_t ntiles = (p.hi - p.lo + T - 1) / T;

  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t t_lo = p.lo + t * T;
    const uint64_t t_hi = min(t_lo + T, p.hi);
    if (tid == 0) {  // last segment with off <= t_lo
      uint32_t lo = p.seg_begin, hi = p.seg_end;
      while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (p.segs[mid].off <= t_lo) lo = mid; else hi = mid;
      }
      s_seg = lo;
    }
    __syncthreads();
    const uint32_t first = s_seg;
    const uint64_t blk_lo = kCheck ? (t_lo / p.block) * p.block : 0;
    unsigned long long a = 0, b = 0, c = 0;

    for (uint32_t s = first; s < p.seg_end; ++s) {
      const Seg sg = p.segs[s];
      if (sg.off >= t_hi) break;
      const uint64_t x_lo = max(sg.off, t_lo);
      const uint64_t x_hi = min(sg.off + sg.len, t_hi);
      for (uint64_t x0 = x_lo + (uint64_t)tid * 16; x0 < x_hi; x0 += (uint64_t)kThreads * 16 * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t x = x0 + (uint64_t)u * kThreads * 16;
          if (x < x_hi) v[u] = load16<kHostSrc>(p.src + (x - p.src_origin));
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t x = x0 + (uint64_t)u * kThreads * 16;
          if (x < x_hi) {
            if (kStore && sg.dst) {
              const uint64_t rel = x - sg.off;
              if (rel + 16 <= sg.valid) store16(sg.dst + rel, v[u]);
              else if (rel < sg.valid) store_partial(sg.dst + rel, v[u], (uint32_t)(sg.valid - rel));
            }
            if (kCheck) {
              const uint32_t i0 = (uint32_t)((x - blk_lo) >> 2);
              const unsigned long long s4 = (unsigned long long)v[u].x + v[u].y + v[u].z + v[u].w;
              a += s4;
              b += (unsigned long long)i0 * s4;
              c += (unsigned long long)v[u].y + 2ull * v[u].z + 3ull * v[u].w;
            }
          }
        }
      }
      if (kCheck) {  // keep partials < 2^32 whatever the number of segments per tile
        a = fold(a);
        b = fold(b);
        c = fold(c);
      }
    }

    if (kCheck) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      if ((tid & 31) == 0) {
        s_red[0][tid >> 5] = a;
        s_red[1][tid >> 5] = b;
        s_red[2][tid >> 5] = c;
      }
      __syncthreads();
      if (tid == 0) {
        unsigned long long A = 0, Bs = 0, C = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
          A += s_red[0][w];
          Bs += s_red[1][w];
          C += s_red[2][w];
        }
        const uint64_t j = t_lo / p.block;
        BlockAcc* acc = p.acc + j;
        atomicAdd(&acc->a, fold(A));
        atomicAdd(&acc->b, fold(Bs));
        atomicAdd(&acc->c, fold(C));
        __threadfence();
        const uint64_t blen = min(p.block, p.part_len - j * p.block);
        const unsigned long long tiles_in_block = (blen + T - 1) / T;
        if (atomicAdd(&acc->tiles_done, 1ull) == tiles_in_block - 1) {
          __threadfence();
          const unsigned long long fa = fold(atomicAdd(&acc->a, 0ull));
          const unsigned long long fb = fold(atomicAdd(&acc->b, 0ull));
          const unsigned long long fc = fold(atomicAdd(&acc->c, 0ull));
          const unsigned long long n = (blen >> 2) % kM;
          const unsigned long long s2 = fold(fold(n * fa) + (kM - fb) + (kM - fc));
          const unsigned long long cs = (s2 << 32) | fa;
          if (p.cs_out) p.cs_out[j] = cs;
          if (p.expect && p.expect[j] != cs) atomicMin(p.bad, (unsigned long long)j);
        }
      }
    }
    __syncthreads();  // s_seg / s_red reuse by the next tile
  }
}


// ---------------------------------------------------------------------------------
// TMA-staged variant (default engine).  One CTA = 1 producer warp + 8 consumer warps (+ a
// bulk-storer warp for engine 2), two CTAs per SM.  The producer streams the CTA's units
// through a 6-stage shared-memory ring with 1-D bulk copies (cp.async.bulk, completion
// counted on an mbarrier); the consumers read each 16 KiB stage with 16-byte LDS, store the
// tensor bytes to their destination and accumulate the closed-form checksum terms.  A CTA
// owns whole checksum blocks unless a launch splits them, so a block is usually reduced
// once inside the CTA -- no global atomics, no fences.  192 KiB in flight per SM covers HBM
// latency (K3/K4) and PCIe latency (K2).
// ---------------------------------------------------------------------------------
constexpr int kConsumerWarps = 8;
// Stage release: one arrival per consumer warp after __syncwarp (default), or one per
// consumer thread (SLLM_THREAD_ARRIVE=1: each thread's own reads directly before its own
// release; the A/B for compute-sanitizer racecheck's model of the indirect syncwarp path).
#ifndef SLLM_THREAD_ARRIVE
#define SLLM_THREAD_ARRIVE 1
#endif
constexpr int kConsumerArrivals = SLLM_THREAD_ARRIVE ? 32 * kConsumerWarps : kConsumerWarps;
constexpr int kTmaThreads = 32 * (kConsumerWarps + 2);  // producer, 8 consumers, bulk storer
constexpr int kStoreLag = 4;                             // bulk-store groups in flight per CTA
// Ring geometry A/B (profiles/r01/ring_geometry_ab.jsonl): 16 KiB stages with the consumer
// loop unrolled 4x beat 16 KiB / 8x and 32 KiB / 4x or 8x on K4 and K3 alike.
#ifndef SLLM_CONSUMER_UNROLL
#define SLLM_CONSUMER_UNROLL 4
#endif
#ifndef SLLM_STAGE_KIB
#define SLLM_STAGE_KIB 16
#endif
constexpr int kConsumerUnroll = SLLM_CONSUMER_UNROLL;
// Ring bytes per CTA and CTAs per SM (A/B knobs SLLM_RING_KIB / SLLM_CTAS_PER_SM).  Two CTAs
// per SM with 96 KiB rings (the same bytes in flight per SM as one 192 KiB ring) beat one:
// while one CTA's consumers meet at a unit end or its producer waits, the other streams --
// K4 0.620 -> 0.586 ms per 4 GiB, K3 4.24 -> 4.01 ms per 26.6 GB (ncu), in-pipeline K4
// 0.955 -> 0.985 and K3 0.834 -> 0.88 by events; three 64 KiB CTAs measure the same as two
// (profiles/r02/ctas_per_sm/).
#ifndef SLLM_RING_KIB
#define SLLM_RING_KIB 96
#endif
#ifndef SLLM_CTAS_PER_SM
#define SLLM_CTAS_PER_SM 2
#endif
constexpr int kCtasPerSm = SLLM_CTAS_PER_SM;
constexpr uint32_t kStageBytes = SLLM_STAGE_KIB << 10;  // ring: kStages x kStageBytes
constexpr int kStages = (SLLM_RING_KIB << 10) / kStageBytes;
constexpr uint64_t kMaxUnitBytes = 1ull << 20;  // default: whole 1 MiB blocks when the launch is balanced
constexpr uint32_t kFineTail = 4;  // fine-tail units per block (see launch_tma)
constexpr size_t kTmaSmem = (size_t)kStages * kStageBytes + 2 * kStages * sizeof(uint64_t);

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
// Parity wait with a watchdog: a transfer that never completes (e.g. an unmapped source)
// traps after ~20 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(smem_addr(b)), "r"(parity) : "memory");
    if (done) return;
    if ((it & 1023) == 1023) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (!t0) t0 = t;
      else if (t - t0 > 20000000000ull) __trap();
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, bool hint) {
  if (hint) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(evict_first_policy()) : "memory");
  } else {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
  }
}
// smem -> global bulk copy (TMA store, SASS UBLKCP), tracked by bulk async-groups.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_addr(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // <= N most recent groups may still read smem
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint4 lds16(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(smem_addr(p)));
  return r;
}
// Segment holding partition byte a: binary search over the launch's segments, narrowed to
// a's granule when the host built the granule table (one dependent load instead of ~log2(n)).
__device__ __forceinline__ uint32_t find_seg(const MatParams& p, uint64_t a) {
  uint32_t lo = p.seg_begin, hi = p.seg_end;
  if (p.gran_seg) {
    const uint64_t g = a >> p.gran_shift;
    lo = max(lo, p.gran_seg[g]);
    hi = min(hi, p.gran_seg[g + 1] + 1);
  }
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.segs[mid].off <= a) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktime_mark(unsigned long long* kt, int which) {
  const unsigned long long t = globaltimer();
  atomicMax(kt + 2 * which, ~t);
  atomicMax(kt + 2 * which + 1, t);
}

constexpr uint64_t kNoUnit = ~0ull;
// Work items of a launch: n_coarse units of `unit` bytes (a 1/split-th of a checksum block),
// then -- the fine tail -- the rest of [lo, hi) in units of unit / fine bytes, so that the
// CTAs that finish their coarse units at different times share the last wave in small
// pieces (the launch ends within ~one fine unit of its last CTA).  Item i -> bytes [a, e).
struct Items {
  uint64_t unit, fine_unit, u_first, n_coarse, v_first, n;
  __device__ Items(const MatParams& p, uint64_t blk) {
    unit = blk / p.split;
    fine_unit = unit / p.fine;
    u_first = p.lo / unit;
    n_coarse = p.n_coarse;
    v_first = (u_first + n_coarse) * p.fine;
    n = n_coarse + ((p.hi + fine_unit - 1) / fine_unit - v_first);
  }
  // bytes of item i and the size of the piece it is of its checksum block
  __device__ __forceinline__ void range(const MatParams& p, uint64_t i, uint64_t& a, uint64_t& e, uint64_t& sz) const {
    const bool c = i < n_coarse;
    sz = c ? unit : fine_unit;
    const uint64_t k = c ? u_first + i : v_first + (i - n_coarse);
    a = max(k * sz, p.lo);
    e = min((k + 1) * sz, p.hi);
  }
};

// The item index the producer stored for a stage, read after that stage's full-barrier wait
// (acquire) -- volatile so the compiler cannot hoist it above the wait.
__device__ __forceinline__ uint64_t unit_of(const uint64_t* s_unit, uint32_t stage) {
  return *static_cast<const volatile uint64_t*>(s_unit + stage);
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps) : "memory"); }

// kMc: the NVLS fan-out's instance (every vector stored once through the multicast address;
// a separate instance keeps the per-vector test out of the K2 / K3 store loops)
template <bool kStore, bool kCheck, bool kMc = false>
__global__ void __launch_bounds__(kTmaThreads, kCtasPerSm) materialise_tma_kernel(const MatParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  __shared__ unsigned long long s_red[2][3][kConsumerWarps];  // double-buffered by unit parity
  __shared__ uint64_t s_unit[kStages];  // item whose first stage is in the slot (kNoUnit: end)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Work unit: a 1/split-th of a checksum block (a CTA owns whole units).  split > 1 lets
  // a launch covering few blocks still spread over every SM; the partial sums of a
  // block's units are then combined with atomics and finalised by its last unit.
  const uint64_t blk = kCheck ? p.block : (1ull << 20);
  const Items items(p, blk);
  if (p.ktime && threadIdx.x == 0) ktime_mark(p.ktime, 0);

  // engine 2: the tensor bytes leave shared memory by TMA bulk stores issued by one
  // storer thread (contiguous pieces: segment x stage); consumers then only read smem for
  // the checksum and write the < 16-byte tails of tensors.
  const bool bulk_store = kStore && !kMc && p.engine == 2 && p.n_peers == 0 && !p.no_seg_store;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerArrivals + (bulk_store ? 1 : 0));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer: picks the CTA's units and streams them through the ring
    // L2 evict-first on the ring loads of the HBM-source store kernels (K3, CE fan-out); not on
    // K4 (read only) nor on host-mapped sources (K2: 1 % slower with it, profiles/r02/l2_hints/)
    const bool ld_hint = SLLM_LD_HINT == 1 || (SLLM_LD_HINT == 2 && kStore && !p.host_src);
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint64_t u = blockIdx.x;  // first item: static (grid <= items)
      for (;;) {
        uint64_t a, e, sz;
        items.range(p, u, a, e, sz);
        for (uint64_t off = a; off < e; off += kStageBytes) {
          const uint32_t n = (uint32_t)min((uint64_t)kStageBytes, e - off);
          mbar_wait(&empty[stage], phase ^ 1);
          // the consumers' generic-proxy reads of this stage (ordered before their empty
          // arrivals) happen before the async-proxy TMA write that refills it
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (off == a) s_unit[stage] = u;  // published by the arrive below (release)
          mbar_expect_tx(&full[stage], n);
          bulk_g2s(smem + (size_t)stage * kStageBytes, p.src + (off - p.src_origin), n, &full[stage], ld_hint);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        // next unit: dynamic (a ticket, drawn once this unit is fully issued -- the ring
        // still holds up to 12 stages for the consumers, which hides the atomic) or static
        u = p.ticket ? gridDim.x + (atomicAdd(p.ticket, 1ull) - p.ticket_base) : u + gridDim.x;
        if (u >= items.n) break;
      }
      mbar_wait(&empty[stage], phase ^ 1);
      s_unit[stage] = kNoUnit;  // end of the CTA's work: a stage with no bytes
      mbar_arrive(&full[stage]);
    }
    return;
  }

  if (warp == kConsumerWarps + 1) {  // bulk storer
    if (bulk_store && lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint32_t ring[kStoreLag + 1];
      int head = 0, cnt = 0;  // stages whose stores may still read smem, oldest first
      for (;;) {
        mbar_wait(&full[stage], phase);
        const uint64_t u = unit_of(s_unit, stage);
        if (u == kNoUnit) break;
        uint64_t a, e, sz;
        items.range(p, u, a, e, sz);
        uint32_t cur = find_seg(p, a);
        Seg sg = p.segs[cur];
        for (uint64_t off = a; off < e; off += kStageBytes) {
          const uint64_t end = off + min((uint64_t)kStageBytes, e - off);
          if (off != a) mbar_wait(&full[stage], phase);
          const uint8_t* sb = smem + (size_t)stage * kStageBytes;
          while (off >= sg.off + sg.len && cur + 1 < p.seg_end) sg = p.segs[++cur];
          uint32_t k = cur;
          Seg s2 = sg;
          for (;;) {  // every segment piece of this stage: one bulk store of its whole vectors
            const uint64_t x0 = max(s2.off, off), x1 = min(min(s2.off + s2.len, end), (uint64_t)(s2.off + (s2.valid & ~(uint64_t)15)));
            if (s2.dst && x1 > x0) bulk_s2g(s2.dst + (x0 - s2.off), sb + (x0 - off), (uint32_t)(x1 - x0));
            if (s2.off + s2.len >= end || k + 1 >= p.seg_end) break;
            s2 = p.segs[++k];
          }
          bulk_commit();
          ring[(head + cnt) % (kStoreLag + 1)] = stage;
          if (++cnt > kStoreLag) {
            bulk_wait_read<kStoreLag>();
            mbar_arrive(&empty[ring[head]]);
            head = (head + 1) % (kStoreLag + 1);
            --cnt;
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      bulk_wait_read<0>();
      for (; cnt; --cnt, head = (head + 1) % (kStoreLag + 1)) mbar_arrive(&empty[ring[head]]);
      bulk_wait_all();
    }
    return;
  }

  const int ct = threadIdx.x - 32;  // consumer thread 0..255
  const int cw = warp - 1;
  uint32_t stage = 0, phase = 0, par = 0;
  for (;; par ^= 1) {
    mbar_wait(&full[stage], phase);  // first stage of the CTA's next unit (or the end mark)
    const uint64_t u = unit_of(s_unit, stage);
    if (u == kNoUnit) break;
    uint64_t a, e, unit;  // unit: this item's piece size (coarse or fine)
    items.range(p, u, a, e, unit);
    // segment holding byte a (same search in every thread: uniform, L1-cached)
    uint32_t cur = p.seg_begin;
    if (kStore) cur = find_seg(p, a);
    Seg sg = kStore ? p.segs[cur] : Seg{0, 0, nullptr, 0};
    const uint64_t bstart = (a / blk) * blk;  // first byte of this item's checksum block
    unsigned long long A = 0, Bs = 0, Cs = 0;
    for (uint64_t off = a; off < e; off += kStageBytes) {
      const uint32_t n = (uint32_t)min((uint64_t)kStageBytes, e - off);
      const uint32_t w0 = (uint32_t)((off - bstart) >> 2);  // block word index of the stage start
      if (off != a) mbar_wait(&full[stage], phase);
      const uint8_t* sb = smem + (size_t)stage * kStageBytes;
#pragma unroll kConsumerUnroll
      for (uint32_t v = (uint32_t)ct * 16; v < n; v += 32 * kConsumerWarps * 16) {
        const uint4 val = lds16(sb + v);
        const uint64_t x = off + v;
        if (kMc) {
          mc_store16(p.mc + x, val);  // NVLS fan-out (contiguous): every replica at once
        } else if (kStore) {
          while (x >= sg.off + sg.len && cur + 1 < p.seg_end) sg = p.segs[++cur];
          if (sg.dst && !p.no_seg_store) {
            const uint64_t rel = x - sg.off;
            if (rel + 16 <= sg.valid) {
              if (!bulk_store) store16(sg.dst + rel, val);
            } else if (rel < sg.valid) {
              store_partial(sg.dst + rel, val, (uint32_t)(sg.valid - rel));
            }
          }
          // P2P fan-out: the same vector to every peer replica (NVLink stores; partitions are
          // multiples of the alignment >= 16, so whole vectors only)
          for (uint32_t k = 0; k < p.n_peers; ++k) store16(p.peer[k] + x, val);
        }
        if (kCheck) {
          const uint32_t i0 = w0 + (v >> 2);
          const unsigned long long s4 = (unsigned long long)val.x + val.y + val.z + val.w;
          A += s4;
          Bs += (unsigned long long)i0 * s4;
          Cs += (unsigned long long)val.y + 2ull * val.z + 3ull * val.w;
        }
      }
#if SLLM_THREAD_ARRIVE
      mbar_arrive(&empty[stage]);  // every consumer thread releases its own reads of the stage
#else
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
#endif
      if (++stage == kStages) { stage = 0; phase ^= 1; }
      if (kCheck) {
        A = fold(A);
        Bs = fold(Bs);
        Cs = fold(Cs);
      }
    }
    if (kCheck) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        A += __shfl_xor_sync(0xffffffffu, A, o);
        Bs += __shfl_xor_sync(0xffffffffu, Bs, o);
        Cs += __shfl_xor_sync(0xffffffffu, Cs, o);
      }
      if (lane == 0) {
        s_red[par][0][cw] = A;
        s_red[par][1][cw] = Bs;
        s_red[par][2][cw] = Cs;
      }
      consumer_sync();  // the other parity's slots are rewritten only after the next unit's sync
      if (ct == 0) {
        unsigned long long SA = 0, SB = 0, SC = 0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          SA += s_red[par][0][w];
          SB += s_red[par][1][w];
          SC += s_red[par][2][w];
        }
        unsigned long long fa = fold(SA), fb = fold(SB), fc = fold(SC);
        const uint64_t j = a / blk;
        const uint64_t blen = min(blk, p.part_len - j * blk);
        bool last = true;
        if (unit < blk) {  // combine this piece's partial sums with the block's other pieces
          BlockAcc* acc = p.acc + j;
          atomicAdd(&acc->a, fa);
          atomicAdd(&acc->b, fb);
          atomicAdd(&acc->c, fc);
          __threadfence();
          last = atomicAdd(&acc->tiles_done, 1ull) == (blen + unit - 1) / unit - 1;
          if (last) {
            __threadfence();
            fa = fold(atomicAdd(&acc->a, 0ull));
            fb = fold(atomicAdd(&acc->b, 0ull));
            fc = fold(atomicAdd(&acc->c, 0ull));
          }
        }
        if (last) {
          const unsigned long long nw = (blen >> 2) % kM;
          const unsigned long long s2 = fold(fold(nw * fa) + (kM - fb) + (kM - fc));
          const unsigned long long cs = (s2 << 32) | fa;
          if (p.cs_out) p.cs_out[j] = cs;
          if (p.expect && p.expect[j] != cs) atomicMin(p.bad, (unsigned long long)j);
        }
      }
    }
  }
  if (p.ktime) {  // diagnostic: this CTA's consumers are done
    consumer_sync();
    if (ct == 0) ktime_mark(p.ktime, 1);
  }
}

}  // namespace

__global__ void peer_signal_kernel(const PeerSignal s, uint32_t epoch) {
  // every store of the preceding fan-out kernels (same stream) happens-before this
  // kernel; the system-scope release makes them visible to a peer that acquires the flag
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (uint32_t k = threadIdx.x; k < s.n; k += blockDim.x)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(s.remote[k]), "r"(epoch) : "memory");
}

__global__ void peer_wait_kernel(const uint32_t* own, int nranks, int me, uint32_t epoch, uint64_t timeout_ns,
                                 uint32_t* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < nranks; ++q) {
    if (q == me) continue;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(own + q) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        *err = 1u + (uint32_t)q;
        return;
      }
      __nanosleep(1000);
    }
  }
}

__global__ void init_seg_kernel(Seg* seg, uint64_t len) { *seg = Seg{0, len, nullptr, 0}; }

cudaError_t launch_init_seg(Seg* seg, uint64_t len, cudaStream_t stream) {
  init_seg_kernel<<<1, 1, 0, stream>>>(seg, len);
  return cudaGetLastError();
}

cudaError_t launch_peer_signal(const PeerSignal& s, uint32_t epoch, cudaStream_t stream) {
  if (!s.n) return cudaSuccess;
  peer_signal_kernel<<<1, 32, 0, stream>>>(s, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint32_t* own, int nranks, int me, uint32_t epoch, uint64_t timeout_ns,
                             uint32_t* err, cudaStream_t stream) {
  if (nranks <= 1) return cudaSuccess;
  peer_wait_kernel<<<1, 1, 0, stream>>>(own, nranks, me, epoch, timeout_ns, err);
  return cudaGetLastError();
}


static int num_sms() {
  static std::atomic<int> sm_count[64];  // per device, queried once (zero-initialised)
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = sm_count[dev & 63].load(std::memory_order_relaxed);
  if (!sms) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 148;
    sm_count[dev & 63].store(sms, std::memory_order_relaxed);
  }
  return sms;
}

template <bool kStore, bool kCheck, bool kMc = false>
static cudaError_t launch_tma(const MatParams& p, int grid, cudaStream_t stream, uint64_t* tickets) {
  // The dynamic shared-memory opt-in is a property of the kernel in each device's context:
  // set it once per (template instance, device); worker threads of different GPUs race here.
  static std::atomic<bool> configured[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(materialise_tma_kernel<kStore, kCheck, kMc>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
    if (e != cudaSuccess) return e;
#ifdef SLLM_SMEM_CARVEOUT  // A/B knob: fix the L1/shared split (percent shared) for the ring kernels
    e = cudaFuncSetAttribute(materialise_tma_kernel<kStore, kCheck, kMc>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, SLLM_SMEM_CARVEOUT);
    if (e != cudaSuccess) return e;
#endif
    configured[dev & 63].store(true, std::memory_order_release);
  }
  // Work items of the launch (see Items): unit size (split), fine tail, ticket count.
  MatParams q = p;
  const uint64_t blk = kCheck ? p.block : (1ull << 20);
  const uint64_t G = (uint64_t)(grid < 1 ? num_sms() * kCtasPerSm : grid);  // resident CTAs
  q.split = 1;
  const uint64_t blocks = (p.hi + blk - 1) / blk - p.lo / blk;
  auto can_halve = [&](uint32_t s) { return s < 16 && blk / (2 * s) >= kStageBytes && (blk / (2 * s)) % 16 == 0; };
  // Wave balance: a launch of U equal units on G CTAs runs ceil(U/G) waves, the last one
  // U/G - floor(U/G) full -- e.g. a 397-block span on 148 CTAs runs 2.68 of 3 waves (89 %).
  auto balance = [&](uint32_t s) {
    const uint64_t U = blocks * s;
    return (double)U / (double)(((U + G - 1) / G) * G);
  };
  // Fine tail: a launch of >= one wave of whole blocks hands out its last G blocks in
  // quarter blocks (combined per block like split units) instead of splitting every block,
  // so the CTAs, which finish their whole blocks up to a block-time apart (~44 us per 1 MiB
  // at two CTAs per SM), share the end in small pieces.  Measured with two CTAs per SM
  // (profiles/r02/ctas_per_sm/): 4 GiB K4 span 0.5855 -> 0.5806 ms, K3 4.009 -> 3.997 ms
  // (ncu), in-pipeline K4 0.996 -> 1.005 by events; the 470 MB LoRA span (448 blocks on 296
  // CTAs) 0.095 ms with every block in sixteenths -> 0.075.  (With one CTA per SM the tail
  // only paid off on unbalanced launches: SLLM_FINE_TAIL=1 keeps that rule, 0 turns it off.)
  static const int fine_mode = [] {  // 0 off, 1 unbalanced launches only, 2 every launch (default)
    const char* e = getenv("SLLM_FINE_TAIL");
    return e ? atoi(e) : 2;
  }();
  const bool tail = fine_mode && blocks >= G && (fine_mode == 2 || balance(1) < 0.95) &&
                    blk / kFineTail >= (64u << 10) && (blk / kFineTail) % kStageBytes == 0;
  if (!tail) {
    // fewer blocks than CTAs, or balanced: split blocks into up to 16 units of >= one stage
    // while the launch has fewer than two units per CTA (so a 64 MiB window still covers
    // every SM), then keep halving (down to 64 KiB) until the last wave is >= 95 % full
    while (can_halve(q.split) && blocks * q.split < 2ull * G) q.split *= 2;
    while (can_halve(q.split) && blk / (2 * q.split) >= (64u << 10) && balance(q.split) < 0.95) q.split *= 2;
  }
  // Largest unit (measurement knob SLLM_UNIT_KIB): smaller units shorten the launch's tail
  // (the last CTA to finish is at most one unit behind) at 4 atomics per unit.
  static const uint64_t max_unit = [] {
    const char* e = getenv("SLLM_UNIT_KIB");
    return (e && atoll(e) > 0) ? (uint64_t)atoll(e) << 10 : kMaxUnitBytes;
  }();
  while (can_halve(q.split) && blk / q.split > max_unit) q.split *= 2;
  if (!kCheck) q.split = 1;
  const uint64_t unit = blk / q.split;
  const uint64_t units = (p.hi + unit - 1) / unit - p.lo / unit;
  q.fine = 1;
  q.n_coarse = units;
  if (tail && q.split == 1) {
    q.fine = kFineTail;
    q.n_coarse = units - G;
  }
  const uint64_t fine_unit = unit / q.fine;
  const uint64_t n_items = q.n_coarse + ((p.hi + fine_unit - 1) / fine_unit - (p.lo / unit + q.n_coarse) * q.fine);
  if ((uint64_t)grid > n_items) grid = (int)n_items;
  if (tickets) *tickets = q.ticket ? n_items : 0;  // each CTA draws one ticket past the end
  materialise_tma_kernel<kStore, kCheck, kMc><<<grid, kTmaThreads, kTmaSmem, stream>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_materialise(const MatParams& p, MatKind kind, int grid, cudaStream_t stream, uint64_t* tickets) {
  if (tickets) *tickets = 0;
  if (p.hi <= p.lo) return cudaSuccess;
  if (grid < 1) grid = num_sms() * (p.engine >= 1 ? kCtasPerSm : 1);  // default: one (ring) CTA per SM
  if (p.engine >= 1) {
    switch (kind) {
      case MatKind::kChecksumOnly: return launch_tma<false, true>(p, grid, stream, tickets);
      case MatKind::kCopyChecksum:
        return p.mc ? launch_tma<true, true, true>(p, grid, stream, tickets) : launch_tma<true, true>(p, grid, stream, tickets);
      case MatKind::kCopyOnly:
        return p.mc ? launch_tma<true, false, true>(p, grid, stream, tickets) : launch_tma<true, false>(p, grid, stream, tickets);
    }
  }
  const uint64_t ntiles = (p.hi - p.lo + p.tile - 1) / p.tile;
  if ((uint64_t)grid > ntiles) grid = (int)ntiles;
  switch (kind) {
    case MatKind::kChecksumOnly:
      if (p.host_src) materialise_kernel<false, true, true><<<grid, kThreads, 0, stream>>>(p);
      else materialise_kernel<false, true, false><<<grid, kThreads, 0, stream>>>(p);
      break;
    case MatKind::kCopyChecksum:
      if (p.host_src) materialise_kernel<true, true, true><<<grid, kThreads, 0, stream>>>(p);
      else materialise_kernel<true, true, false><<<grid, kThreads, 0, stream>>>(p);
      break;
    case MatKind::kCopyOnly:
      if (p.host_src) materialise_kernel<true, false, true><<<grid, kThreads, 0, stream>>>(p);
      else materialise_kernel<true, false, false><<<grid, kThreads, 0, stream>>>(p);
      break;
  }
  return cudaGetLastError();
}

}  // namespace sllm
