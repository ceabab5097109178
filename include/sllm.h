/* sllm.h -- C ABI of the B200-native loading-optimized checkpoint loader.
 *
 * The operations follow the paper's statement of the loading problem
 * (ServerlessLLM, arXiv 2401.14351; PAPER.md = /root/reference/PAPER.md):
 *   - convert a checkpoint into one aligned, metadata-free partition per GPU plus a
 *     tensor index "that maps tensor names to a tuple of GPU id, offset, and size"
 *     (§Loading-Optimized Checkpoints);
 *   - open the index;
 *   - the model manager "allocates memory on GPUs and loads the binary data" through
 *     chunk-based, pipelined transfers from pinned memory;
 *   - tensor address = base + offset;
 *   - a synchronization "returns when all data is loaded into GPUs".
 * Integrity checking (per-block Fletcher-64) is the build's addition (Q8).
 *
 * Conventions (apply to every function):
 *   - every call returns sllm_status; SLLM_OK == 0.  Outputs go through out-params,
 *     which are left untouched on failure.  No exception or abort crosses the ABI;
 *     sllm_last_error() returns a thread-local message for the last failure on the
 *     calling thread (valid until that thread's next failing call).
 *   - "host pointer" = CPU virtual address; "device pointer" = CUDA device address.
 *   - integers are byte counts unless stated; all on-disk data is little-endian.
 *   - ownership: the CALLER owns source buffers (pinned host memory) and every
 *     destination (device memory, typically allocated through PyTorch).  The LIBRARY
 *     owns sllm_index / sllm_load / sllm_comm objects and their internal scratch
 *     (staging rings, device checksum tables, streams, worker threads), released by
 *     the matching *_close / *_free call.
 *   - thread safety: an sllm_index is immutable after open/seal and may be shared by
 *     threads; one sllm_load object must not be used from two threads at once.
 *   - current device: calls that work on GPUs (load, comm, ipc, device helpers) may select
 *     devices internally but restore the calling thread's current CUDA device before
 *     returning.
 */
#ifndef SLLM_H_
#define SLLM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SLLM_API __attribute__((visibility("default")))
#else
#define SLLM_API
#endif

#define SLLM_ABI_VERSION 1
#define SLLM_MAX_NDIM 8

typedef enum {
  SLLM_OK = 0,
  SLLM_E_INVALID = 1,     /* bad argument: null pointer, bad alignment/block/chunk, bad mode   */
  SLLM_E_CONVERSION = 2,  /* duplicate/empty name, payload != prod(shape)*width, bad dtype */
  SLLM_E_FORMAT = 3,      /* bad magic/version/flags, truncated, overlap, misaligned   */
  SLLM_E_LOOKUP = 4,      /* unknown tensor name / index out of range                     */
  SLLM_E_CAPACITY = 5,    /* destination or buffer too small                                    */
  SLLM_E_IO = 6,          /* file open/read/write failure                                       */
  SLLM_E_CUDA = 7,        /* a CUDA runtime call failed (message names it)                      */
  SLLM_E_NCCL = 8,        /* an NCCL call failed or libnccl could not be loaded                 */
  SLLM_E_CHECKSUM = 9,    /* a loaded block's Fletcher-64 differs from the index               */
  SLLM_E_BUSY = 10,       /* the destination set is already being loaded                 */
  SLLM_E_NOMEM = 11,      /* host allocation / pinning failed                                   */
  SLLM_E_PEER = 12        /* P2P fan-out: a peer did not signal completion within the timeout   */
} sllm_status;

/* dtype codes (Q12: loading is dtype-agnostic -- the dtype fixes the
 * element width the converter checks against the payload size, and the view type).  Widths:
 * F16/BF16/I16 2, F32/I32 4, F64/I64 8, I8/U8/BOOL/F8_E4M3/F8_E5M2 1. */
typedef enum {
  SLLM_F16 = 0, SLLM_BF16 = 1, SLLM_F32 = 2, SLLM_I8 = 3, SLLM_U8 = 4, SLLM_I64 = 5,
  SLLM_I32 = 6, SLLM_F64 = 7, SLLM_I16 = 8, SLLM_BOOL = 9, SLLM_F8_E4M3 = 10, SLLM_F8_E5M2 = 11
} sllm_dtype;

typedef struct sllm_index sllm_index; /* parsed / planned index (opaque)                  */
typedef struct sllm_load sllm_load;   /* one in-flight load (opaque)                       */
typedef struct sllm_comm sllm_comm;   /* NCCL communicator for the replicated fan-out      */

SLLM_API const char* sllm_last_error(void);
SLLM_API int32_t sllm_abi_version(void);

/* ------------------------------------------------------------------------------------
 * Converter (host only).  SPEC S:43 convert(src, align); layout per PAPER.md P:545-547:
 * for each device ascending, tensors in source order, offset = align_up(cursor, align),
 * partition length L_d = align_up(last end, align), padding bytes 0x00 (Q1-Q5).
 * ------------------------------------------------------------------------------------ */
typedef struct {
  const char* name;      /* NUL-terminated UTF-8, unique, non-empty                         */
  int32_t device_id;     /* logical partition id (>= 0); "target GPU" of P:462              */
  int32_t dtype;         /* sllm_dtype                                                      */
  int32_t ndim;          /* 0..8; 0 = scalar                                                */
  const int64_t* shape;  /* ndim positive dims (may be NULL when ndim == 0)                 */
  const void* data;      /* host pointer to nbytes of payload; may be NULL for sllm_plan    */
  uint64_t nbytes;       /* must equal prod(shape) * width(dtype)                           */
} sllm_src_tensor;

/* Plan the layout of n tensors (no bytes move).  align: power of two >= 16.  block:
 * checksum block size, power of two multiple of align, or 0 for "no checksums".  The
 * returned index has zeroed checksum tables until sllm_index_seal / sllm_convert_into.
 * align and block are at most 256 MiB (the device kernels' unfolded Fletcher sums stay below
 * 2^64; Q8); sllm_index_open rejects larger values with SLLM_E_FORMAT.
 * Errors: SLLM_E_INVALID (align/block), SLLM_E_CONVERSION (names, sizes, dtype, dims). */
SLLM_API sllm_status sllm_plan(const sllm_src_tensor* tensors, size_t n, uint64_t align, uint64_t block,
                      const char* model_id, sllm_index** out);

/* Fill caller-provided partition buffers (host pointers, part_bufs[p] of length >= L_p for
 * partition p in ascending device order) from tensors[i].data -- the same tensors, same
 * order as given to sllm_plan -- zero all padding, then seal (compute block checksums).
 * Multi-threaded.  Errors: SLLM_E_INVALID (null data / buffer), SLLM_E_CONVERSION. */
SLLM_API sllm_status sllm_convert_into(const sllm_src_tensor* tensors, size_t n, sllm_index* plan,
                              void* const* part_bufs);

/* Compute every block checksum of a planned index from partition buffers the caller has
 * already filled (plan -> fill -> seal).  part_bufs[p]: host pointer, >= L_p bytes, or
 * NULL to leave partition p's table untouched (a process that holds only its own
 * partition).  Multi-threaded. */
SLLM_API sllm_status sllm_index_seal(sllm_index* index, const void* const* part_bufs);

/* convert() to files: <out_dir>/part_<device>.bin and <out_dir>/index.bin. */
SLLM_API sllm_status sllm_convert(const sllm_src_tensor* tensors, size_t n, uint64_t align, uint64_t block,
                         const char* model_id, const char* out_dir);

/* Serialize the index (binary format of DESIGN.md §Index format).  If buf is NULL or cap
 * is too small, *len receives the required size and SLLM_E_CAPACITY is returned (unless
 * buf is NULL, which returns SLLM_OK with *len set). */
SLLM_API sllm_status sllm_index_serialize(const sllm_index* index, void* buf, size_t cap, size_t* len);

/* ------------------------------------------------------------------------------------
 * Index (S:52 read_index, S:61 tensor_address).
 * ------------------------------------------------------------------------------------ */
typedef struct {
  uint64_t align, block, payload_bytes;
  uint64_t n_partitions, n_tensors;
  const char* model_id;  /* owned by the index */
} sllm_index_info;

typedef struct {
  const char* name;      /* owned by the index */
  int32_t device_id;
  int32_t partition;     /* position of the tensor's partition in ascending device order */
  int32_t dtype;
  int32_t ndim;
  int64_t shape[SLLM_MAX_NDIM];
  uint64_t offset;       /* byte offset inside the partition (multiple of align) */
  uint64_t nbytes;
} sllm_tensor_info;

/* Parse + fully validate (every check of DESIGN.md §Index format -> SLLM_E_FORMAT). */
SLLM_API sllm_status sllm_index_open(const char* path, sllm_index** out);
SLLM_API sllm_status sllm_index_from_memory(const void* blob, size_t len, sllm_index** out);
SLLM_API void sllm_index_close(sllm_index* index);
SLLM_API sllm_status sllm_index_get_info(const sllm_index* index, sllm_index_info* out);
/* SURVEY §8(b) sllm_index_counts: number of tensors and of partitions (either out may be NULL). */
SLLM_API sllm_status sllm_index_counts(const sllm_index* index, size_t* n_tensors, size_t* n_partitions);
/* Partition p (0..n_partitions-1, ascending device id). */
SLLM_API sllm_status sllm_index_partition(const sllm_index* index, size_t p, int32_t* device_id,
                                 uint64_t* length, uint64_t* n_blocks, uint64_t* n_tensors);
/* Pointer to partition p's n_blocks block checksums (owned by the index). */
SLLM_API sllm_status sllm_index_block_checksums(const sllm_index* index, size_t p, const uint64_t** table);
/* Tensor i in global source order. */
SLLM_API sllm_status sllm_index_tensor(const sllm_index* index, size_t i, sllm_tensor_info* out);
SLLM_API sllm_status sllm_index_find(const sllm_index* index, const char* name, size_t* i); /* SLLM_E_LOOKUP */
/* P:549 base + offset: base_by_partition[p] is partition p's base address (any address
 * space; the library never dereferences it). */
SLLM_API sllm_status sllm_tensor_address(const sllm_index* index, const char* name, const uint64_t* base_by_partition,
                                int32_t* device_id, uint64_t* addr);

/* Fletcher-64 (Q8) of a host buffer; nbytes need not be a multiple of 4
 * (tail zero-padded).  Host-only helper used by the converter. */
SLLM_API sllm_status sllm_fletcher64_host(const void* data, uint64_t nbytes, uint64_t* out);

/* Chunk plan (equal chunks except the last): number of chunks of `chunk` bytes
 * covering `length` bytes. */
SLLM_API sllm_status sllm_chunk_count(uint64_t length, uint64_t chunk, uint64_t* n_chunks);
/* Replicated fan-out slices: cut [0, length) into nranks contiguous,
 * chunk-aligned slices; lo_hi receives 2*nranks values {lo_0, hi_0, lo_1, hi_1, ...}.
 * Slices are balanced in whole chunks; trailing slices may be empty. */
SLLM_API sllm_status sllm_replica_slices(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t* lo_hi);
/* Fan-out round schedule (the one sllm_load_wait's replicated path executes): round r
 * broadcasts, from every rank q, the r-th chunk of q's slice.  lo_hi receives 2*nranks
 * values {lo_q, hi_q} (hi_q == lo_q: rank q sends nothing in this round); *n_rounds (may
 * be NULL) receives the number of rounds, max over q of ceil(|slice_q| / chunk).
 * SLLM_E_LOOKUP if round >= n_rounds. */
SLLM_API sllm_status sllm_replica_round(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t round,
                                        uint64_t* lo_hi, uint64_t* n_rounds);
/* Unit of the NCCL fan-outs' slices and rounds for a load with chunk size `chunk` and fan-out
 * `fanout`: BCAST / ALLGATHER slice the partition and run their rounds in whole copy windows
 * of chunks (max(1, 64 MiB / chunk) chunks -- one copy submission and one grouped
 * broadcast / all-gather per round instead of one per chunk); every other fan-out: `chunk`.
 * The loader calls sllm_replica_slices / sllm_replica_round / sllm_allgather_round with this
 * unit in place of the chunk. */
SLLM_API sllm_status sllm_fanout_unit(uint64_t chunk, int32_t fanout, uint64_t* unit);
/* All-gather schedule of SLLM_FANOUT_ALLGATHER ("in-place ncclAllGather is the
 * equal-count alternative"): chunk k of the partition belongs to rank k mod nranks, so
 * round r is the contiguous run of chunks [r*nranks, (r+1)*nranks) and rank q contributes
 * chunk r*nranks + q.  lo_hi receives 2*nranks values {lo_q, hi_q} (hi_q == lo_q: rank q
 * has no chunk in this round); *n_rounds (may be NULL) = ceil(ceil(length/chunk)/nranks);
 * *full (may be NULL) = 1 when every rank has a whole chunk in the round -- the loader then
 * issues one in-place ncclAllGather of `chunk` bytes per rank, else (the ragged last round)
 * grouped ncclBroadcasts of each chunk from its owner.  SLLM_E_LOOKUP if round >= n_rounds. */
SLLM_API sllm_status sllm_allgather_round(uint64_t length, uint64_t chunk, int32_t nranks, uint64_t round,
                                          uint64_t* lo_hi, uint64_t* n_rounds, int32_t* full);

/* ------------------------------------------------------------------------------------
 * Pinned host memory (the DRAM tier).  Page-locked, mapped into the
 * device address space (zero-copy capable) and portable across devices.  gpu >= 0
 * places the pages on that GPU's NUMA node when the system has several nodes.
 * ------------------------------------------------------------------------------------ */
SLLM_API sllm_status sllm_host_alloc(uint64_t bytes, int32_t gpu, void** p);
SLLM_API void sllm_host_free(void* p);
/* NUMA placement: *node = the NUMA node of GPU `gpu`'s PCIe root (sysfs), or -1
 * when the host does not report one; sllm_host_numa_node: the node holding the page at host
 * address p (get_mempolicy), -1 if unknown.  The library binds the pages of sllm_host_alloc
 * (gpu >= 0) to that node, and runs the threads touching them -- first touch, per-partition
 * load workers, storage readers, converter fill / checksum threads -- on its CPUs when the
 * host has several nodes. */
SLLM_API sllm_status sllm_gpu_numa_node(int32_t gpu, int32_t* node);
SLLM_API sllm_status sllm_host_numa_node(const void* p, int32_t* node);
/* Page-lock + map caller-owned memory (e.g. a NumPy array) so it can be a load source. */
SLLM_API sllm_status sllm_host_register(void* p, uint64_t bytes);
SLLM_API sllm_status sllm_host_unregister(void* p);
/* File -> pinned DRAM tier: read <dir>/part_<device>.bin of partition p into dst (host
 * pointer, >= L_p bytes), O_DIRECT when possible, `threads` readers (0 = default). */
SLLM_API sllm_status sllm_host_read_partition(const char* dir, const sllm_index* index, size_t p, void* dst,
                                     int32_t threads);

/* ------------------------------------------------------------------------------------
 * Pinned model cache: the DRAM tier as a pool of whole models with LRU eviction (PAPER.md
 * P:578-579).  Thread-safe.
 * ------------------------------------------------------------------------------------ */
typedef struct sllm_cache sllm_cache;
typedef struct {
  uint64_t capacity, used;       /* bytes (each partition rounded up to 2 MiB)              */
  uint64_t models;               /* resident (or being read) models                          */
  uint64_t hits, misses, evictions;
} sllm_cache_stats;
/* capacity: bytes of host memory the cache may hold.  gpu >= 0: NUMA placement as
 * sllm_host_alloc.  pin = 1: page-locked, device-mapped memory (a load source); pin = 0:
 * plain page-aligned memory (host-only use). */
SLLM_API sllm_status sllm_cache_create(uint64_t capacity, int32_t gpu, int32_t pin, sllm_cache** out);
/* The model converted into <dir> (index.bin + part_<device>.bin).  Hit: the resident copy,
 * marked most recently used.  Miss: its bytes are reserved by evicting least recently used
 * models that nobody holds, then every partition is read with `io_threads` O_DIRECT
 * readers (0 = 4) outside the cache lock; concurrent acquirers of the same model wait for
 * that read.  Outputs (owned by the cache, valid until the matching release): *index, and
 * *part_bufs = n_partitions host pointers (partition p at part_bufs[p]); *hit (may be
 * NULL) = 1 on a hit.  The model is held (never evicted) until sllm_cache_release.
 * SLLM_E_CAPACITY: the model does not fit even after evicting every unheld model. */
SLLM_API sllm_status sllm_cache_acquire(sllm_cache* cache, const char* dir, int32_t io_threads,
                                        const sllm_index** index, void* const** part_bufs, int32_t* hit);
/* Drop one hold of <dir>; SLLM_E_LOOKUP if it is not held. */
SLLM_API sllm_status sllm_cache_release(sllm_cache* cache, const char* dir);
SLLM_API sllm_status sllm_cache_get_stats(sllm_cache* cache, sllm_cache_stats* out);
/* Frees every resident model (held or not: the caller must have finished its loads). */
SLLM_API void sllm_cache_destroy(sllm_cache* cache);

/* ------------------------------------------------------------------------------------
 * Load (S:115 load()).
 * ------------------------------------------------------------------------------------ */
typedef enum {
  SLLM_MODE_CE = 0,         /* copy engine per chunk into base+off, then checksum kernel     */
  SLLM_MODE_ZEROCOPY = 1,   /* SM-issued 16 B reads of host-mapped memory -> base+off, fused checksum */
  SLLM_MODE_SCATTER_CE = 2, /* copy engine into a staging ring, then index-driven scatter kernel */
  SLLM_MODE_SCATTER_ZC = 3, /* SM-issued host reads scattered straight into per-tensor buffers */
  SLLM_MODE_AUTO = 4,       /* contiguous: ZEROCOPY when every partition (fan-out: slice) this
                               call moves is < 256 MiB and device-mapped, else CE; the report's
                               `mode` says which ran */
  SLLM_MODE_GDS = 5         /* sllm_load_files_start only, contiguous, no fan-out: GPUDirect
                               Storage -- `io_threads` cuFileRead readers move part_<d>.bin
                               straight into base+off (no pinned DRAM tier), K4 verifies the
                               landed prefix in spans.  libcufile.so.0 is loaded lazily; without
                               the nvidia-fs driver cuFile serves the reads in its compatibility
                               mode.  SLLM_E_IO if cuFile cannot be opened or a read fails.
                               Opt-in: SLLM_E_INVALID unless the environment sets
                               SLLM_ENABLE_GDS=1 (cuFileDriverOpen hangs, uncancellably, on
                               hosts where cuFile cannot probe the PCI topology). */
} sllm_mode;

/* Replicated checkpoint (one partition, every GPU gets a full replica): rank r of n moves
 * only its slice (sllm_replica_slices) over its own PCIe link; the other GPUs receive it
 *   BCAST : by grouped ncclBroadcast per chunk round over NVLink (sllm_comm_init_rank/_all);
 *   P2P   : inside the loading kernel itself -- the zero-copy kernel (ZEROCOPY) or the
 *           per-window verify kernel (CE) stores every 16-byte vector into the rank's own
 *           replica and, over NVLink, into every peer replica at the same offset; then a
 *           device-side signal/wait exchange (system-scope release/acquire flags) orders
 *           the peers' stores before each rank verifies what it received
 *           (sllm_comm_init_peers);
 *   ALLGATHER: by one in-place ncclAllGather per round of nranks chunks (NCCL communicator).
 *           Here rank r's PCIe share is not a contiguous slice but every chunk k with
 *           k mod nranks == r (sllm_allgather_round), so the whole partition must be pinned;
 *           pinned sources only (not sllm_load_files_start).
 *   NVLS  : as P2P, but every vector is stored ONCE through an NVLink-
 *           SHARP multicast address (multimem.st) and the NVSwitch writes it into every
 *           replica of the group; the group and its replicas come from sllm_comm_init_nvls.
 * Every rank's received bytes are verified against the index like its own (K4). */
typedef enum { SLLM_FANOUT_NONE = 0, SLLM_FANOUT_BCAST = 1, SLLM_FANOUT_P2P = 2, SLLM_FANOUT_ALLGATHER = 3,
               SLLM_FANOUT_NVLS = 4 } sllm_fanout;

typedef struct {
  uint64_t chunk_bytes; /* multiple of the index block size (and of align); 0 = 16 MiB    */
  int32_t n_streams;    /* internal streams per GPU, 1..8 (0 = 2)                           */
  int32_t mode;         /* sllm_mode                                                        */
  int32_t fanout;       /* sllm_fanout; BCAST/ALLGATHER/P2P require a comm and a 1-partition index */
  int32_t verify;       /* 1 = check every block's Fletcher-64 against the index            */
  int32_t ctas;         /* CTAs per kernel launch (0 = mode default)                        */
  int32_t profile;      /* 1 = time every kernel launch with CUDA events, 2 = also copies,
                           3 = as 1 plus in-kernel spans (%globaltimer: first CTA start .. last
                           CTA end of each timed launch, 2 atomics per CTA)                  */
  int32_t engine;       /* kernel engine: 0 = default (TMA), 1 = TMA bulk-load ring + vector stores,
                           2 = LDG/STG register tiles, 3 = TMA bulk-load ring + TMA bulk stores */
  int32_t reserved;     /* must be 0                                                        */
} sllm_load_config;

typedef struct {
  uint64_t payload_bytes;      /* sum of tensor sizes in the partitions this call loaded    */
  uint64_t transferred_bytes;  /* host->device bytes moved by this process (PCIe)           */
  uint64_t fanout_bytes;       /* bytes received through the NVLink fan-out                 */
  uint64_t chunks;             /* chunks issued                                             */
  uint64_t kernel_launches;    /* library kernels launched                                  */
  uint64_t copy_calls;         /* cudaMemcpyAsync calls issued                              */
  uint64_t t_total_ns;         /* host clock, sllm_load_start entry -> sllm_load_wait exit  */
  uint64_t t_issue_ns_max;     /* longest per-partition host issue time                     */
  double t_device_ms_max;      /* longest per-partition device time (CUDA events)           */
  double t_kernel_ms_sum;      /* profile: summed device time of the load's kernel launches */
  double t_copy_ms_sum;        /* profile: summed device time of its cudaMemcpyAsync calls */
  uint64_t kernel_bytes;       /* profile: partition bytes covered by those kernel launches */
  int32_t bad_partition;       /* -1 when OK                                                */
  int32_t mode;
  uint64_t bad_block;          /* UINT64_MAX when OK                                        */
  uint64_t storage_bytes;      /* file tier: bytes read from the partition files            */
  uint64_t t_storage_wait_ns_max; /* file tier: longest time a partition's GPU worker waited for
                                     storage (0 = storage never the bottleneck)              */
  double t_kernel_span_ms_sum; /* profile 3: summed in-kernel spans of the timed launches (the
                                  CUDA-event times above also hold launch and completion)   */
} sllm_load_report;

/* Communicator for SLLM_FANOUT_BCAST and SLLM_FANOUT_ALLGATHER.  One process per GPU: rank 0 calls
 * sllm_comm_unique_id, the caller distributes the 128 bytes (e.g. via torch.distributed),
 * every rank calls sllm_comm_init_rank.  Single process, several GPUs: sllm_comm_init_all
 * (one comm per listed GPU; handle i belongs to gpus[i]).  libnccl.so.2 is loaded lazily. */
SLLM_API sllm_status sllm_comm_unique_id(void* id128);
SLLM_API sllm_status sllm_comm_init_rank(const void* id128, int32_t nranks, int32_t rank, int32_t gpu, sllm_comm** out);
SLLM_API sllm_status sllm_comm_init_all(const int32_t* gpus, int32_t n, sllm_comm** out /* n handles */);
/* Peer group for SLLM_FANOUT_P2P (fan-out fused into the loading
 * kernel over NVLink peer memory, no NCCL).  Collective: every rank of the group creates
 * its handle with the same arrays and then issues the same sequence of P2P loads.
 *   nranks        : 1..8 (one NVSwitch node); rank: this process's rank; gpu: its device.
 *   peer_base[q]  : device pointer, valid in THIS process, to rank q's replica (>= L bytes,
 *                   16-byte aligned): peer_base[rank] is this rank's own destination (it
 *                   must be dst_base[0] of every P2P load), the others come from
 *                   sllm_ipc_open of the peers' sllm_ipc_export (or plain pointers when
 *                   the ranks share a process).  The group is bound to these replicas.
 *   peer_signal[q]: device pointer (valid here) to rank q's signal array of 2*nranks
 *                   uint32 words, zero-filled once before the first load and owned by rank
 *                   q: ready[r] (rank r's stores into q's replica are complete for that
 *                   epoch) and done[r] (rank r finished that load; its replica may be
 *                   overwritten by the next one), so back-to-back loads need no host barrier.
 *   timeout_ms    : how long a rank waits for its peers' completion signals before the
 *                   load fails with SLLM_E_PEER (0 = 60000).
 * A P2P load completes only when every rank's load has run.  Ranks of one group that share
 * a process order each other with CUDA events (no signal words, no device-side waits; they
 * rendezvous on the host so every event is recorded before it is waited on, and a rank that
 * never arrives fails the others with SLLM_E_PEER after timeout_ms), and their caller
 * streams are ordered after the load in sllm_load_wait, not in sllm_load_start.  Ranks in
 * separate processes wait for each other's signal words with a device-side wait kernel, or,
 * with the environment variable SLLM_PEER_WAIT=host, on the host (the load's worker polls its
 * own signal words; the caller's stream is then ordered after the load in sllm_load_wait)
 * -- required when the ranks share a GPU: a kernel spinning on another process's flag must
 * not share a GPU with the kernel that sets it.
 * The handle owns its streams; sllm_comm_free releases them (never the replicas). */
SLLM_API sllm_status sllm_comm_init_peers(int32_t nranks, int32_t rank, int32_t gpu, void* const* peer_base,
                                          uint32_t* const* peer_signal, uint64_t timeout_ms, sllm_comm** out);
/* NVLS multicast group for SLLM_FANOUT_NVLS (the fan-out fused into the
 * loading kernel, replicated by the NVSwitch).  One process drives every GPU of the group
 * (P:721-727): handle i is rank i on gpus[i] (n = 1..8, distinct).  The library creates one
 * multicast object (cuMulticastCreate), allocates and binds a replica of >= `bytes` on every
 * GPU (cuMemCreate; the replica is LIBRARY-owned, freed with the last handle of the group:
 * sllm_comm_replica gives its address) and maps the multicast address.  Loads of the group
 * pass dst_base[0] = that replica.  timeout_ms as in sllm_comm_init_peers (0 = 60000).
 * Capability-gated: SLLM_E_INVALID (message names the failing driver call) when a GPU lacks
 * multicast support or the platform cannot create the object (no NVSwitch / NVLS fabric) --
 * keep the P2P or NCCL fan-out then.  SLLM_E_CAPACITY when a replica cannot be allocated. */
SLLM_API sllm_status sllm_comm_init_nvls(const int32_t* gpus, int32_t n, uint64_t bytes, uint64_t timeout_ms,
                                         sllm_comm** out /* n handles */);
/* The replica a P2P / NVLS group handle is bound to: *base = this rank's replica (device
 * pointer), *bytes (may be NULL) = its size for an NVLS group (library-owned), 0 for a P2P
 * group (caller-owned).  SLLM_E_INVALID for an NCCL communicator. */
SLLM_API sllm_status sllm_comm_replica(const sllm_comm* comm, void** base, uint64_t* bytes);
SLLM_API void sllm_comm_free(sllm_comm* comm);

/* Start loading (asynchronous: returns once worker threads are launched).
 *   index          : opened/sealed index (must outlive the load).
 *   cfg            : NULL = defaults (16 MiB chunks, 2 streams, CE, verify).
 *   host_src[p]    : host pointer to partition p's bytes (pinned via sllm_host_alloc /
 *                    sllm_host_register or cudaHostAlloc), or NULL = partition not
 *                    loaded by this call.  For FANOUT_BCAST only the rank's slice is read.
 *                    ZEROCOPY / SCATTER_ZC read it with 16-byte vector loads and TMA bulk
 *                    copies: its device alias must be 16-byte aligned (else SLLM_E_INVALID;
 *                    AUTO keeps the copy engine for a misaligned source).
 *   gpu[p]         : CUDA device ordinal for partition p (ignored if host_src[p] NULL).
 *   dst_base[p]    : device pointer, >= L_p bytes (contiguous modes and FANOUT); the
 *                    tensors are views base+offset.  May be NULL in scatter modes.
 *   dst_tensor[i]  : scatter modes only: device pointer to tensor i's own buffer (>= its
 *                    nbytes, 16-byte aligned), global source order; NULL entries for
 *                    tensors of unloaded partitions.  NULL array for contiguous modes.
 *   stream[p]      : optional caller cudaStream_t (as void*) for partition p.  The load is
 *                    ordered after work already queued on it, and the stream is made to
 *                    wait for the load's completion (an event wait, enqueued once the load's
 *                    own work is all enqueued -- before this call returns), so work queued on
 *                    it after sllm_load_start sees the loaded bytes.  (sllm_load_files_start
 *                    and P2P groups with several ranks in one process enqueue that wait in
 *                    sllm_load_wait instead: their issue waits on storage / on the peers.)
 *                    NULL array/entry = no ordering.
 *   comm           : NULL unless cfg->fanout is BCAST / ALLGATHER (NCCL communicator) or
 *                    P2P (peer group); with BCAST or P2P, host_src[0] needs to hold (pinned)
 *                    only the rank's own slice [lo_r, hi_r) of sllm_replica_slices: bytes
 *                    outside it are never read (ALLGATHER: the rank's chunks k = r mod n).
 * Returns SLLM_E_BUSY if one of dst_base/dst_tensor is the target of an unfinished load.
 * Tensor contents are defined only after sllm_load_wait returns SLLM_OK (Q17). */
SLLM_API sllm_status sllm_load_start(const sllm_index* index, const sllm_load_config* cfg,
                            const void* const* host_src, const int32_t* gpu,
                            void* const* dst_base, void* const* dst_tensor,
                            void* const* stream, sllm_comm* comm, sllm_load** out);

/* Start loading straight from the partition files <dir>/part_<device>.bin -- the whole
 * multi-tier pipeline SSD -> pinned DRAM -> GPU: `io_threads`
 * (0 = 4) readers fill a ring of pinned 64 MiB slots from a process-wide pool
 * with O_DIRECT reads, each slot's window is copied / verified / scattered exactly
 * as in sllm_load_start, and a slot is refilled once the GPU has consumed it.
 *   gpu[p] : CUDA ordinal for partition p, or < 0 to skip that partition.
 *   comm   : as in sllm_load_start: with a fan-out (replicated checkpoint) this rank reads
 *            only its slice of part_<d>.bin from storage and the rest arrives over NVLink,
 *            so the group reads every byte from storage once.
 *   other arguments as in sllm_load_start.  SLLM_E_IO names the file. */
SLLM_API sllm_status sllm_load_files_start(const sllm_index* index, const sllm_load_config* cfg, const char* dir,
                                           const int32_t* gpu, void* const* dst_base, void* const* dst_tensor,
                                           void* const* stream, int32_t io_threads, sllm_comm* comm, sllm_load** out);

/* Captured load (latency-bound small checkpoints; CUDA graphs instead of
 * a per-load host issue sequence).  sllm_load_capture plans the load exactly as
 * sllm_load_start (same arguments, pinned sources, no fan-out, no files, no profiling) and
 * records each partition's whole device work -- table upload, accumulator reset, the copy
 * windows, the verify / scatter launches, the result read-back -- as one CUDA graph per
 * partition, without moving any byte.  sllm_load_replay then loads the checkpoint again by
 * launching those graphs (one cudaGraphLaunch per partition, no index walk, no worker
 * hand-off, no per-window API calls) for repeated loads of the same checkpoint into the same
 * destinations from the same pinned source (the graphs hold the source, destination and
 * table addresses and the checkpoint's expected checksums): e.g. an adapter kept resident in
 * the pinned pool and re-loaded into its GPU slot whenever it is needed again (P:1253 LoRA
 * loading); another checkpoint -- another adapter -- is another captured load.
 *   sllm_load_replay: stream[p] = the caller's cudaStream_t (as void*) for partition p, the
 *     replay queued on it (ordered after its earlier work; later work on it sees the bytes),
 *     or NULL array / entry = a library stream.  SLLM_E_BUSY if the previous replay has not
 *     been waited for.  The sources must hold the checkpoint's bytes when the replay runs.
 *   sllm_load_wait reports the last replay (verification result, device time); tensor
 *   handles and block checksums refer to the last waited replay.
 * The destinations stay reserved (SLLM_E_BUSY for other loads) until sllm_load_free, which
 * waits for the last replay and frees the graphs. */
SLLM_API sllm_status sllm_load_capture(const sllm_index* index, const sllm_load_config* cfg,
                                       const void* const* host_src, const int32_t* gpu,
                                       void* const* dst_base, void* const* dst_tensor, sllm_load** out);
SLLM_API sllm_status sllm_load_replay(sllm_load* load, void* const* stream);

/* Block until every chunk (and fan-out round) has landed and been verified.  Returns
 * SLLM_E_CHECKSUM with rep->bad_partition / rep->bad_block naming the first failing
 * block, or the first CUDA/NCCL error.  Idempotent (returns the same status again).
 * rep may be NULL. */
SLLM_API sllm_status sllm_load_wait(sllm_load* load, sllm_load_report* rep);

/* {gpu, device pointer, dtype, shape} of a tensor of this load; valid right after start
 * (pointers may be set before the data arrives). */
typedef struct {
  int32_t gpu;
  int32_t dtype;
  int32_t ndim;
  int32_t reserved;
  int64_t shape[SLLM_MAX_NDIM];
  void* ptr;
  uint64_t nbytes;
} sllm_tensor_handle;
SLLM_API sllm_status sllm_load_tensor(const sllm_load* load, const char* name, sllm_tensor_handle* h);

/* Device-computed block checksums of partition p from the last wait (host copy owned by
 * the load; n_blocks entries; entries of blocks not verified by this process are 0). */
SLLM_API sllm_status sllm_load_block_checksums(const sllm_load* load, size_t p, const uint64_t** table);

/* Free worker state and scratch; waits for completion first.  Never frees caller memory. */
SLLM_API void sllm_load_free(sllm_load* load);

/* Release idle device memory the library keeps cached on `gpu` -- the stream-ordered pool
 * holding per-load scratch and SCATTER_CE staging rings (up to 3 x 1 GiB), which finished
 * loads return to the pool for the next load to reuse -- down to keep_bytes.  Synchronizes
 * the device first; memory of loads still in flight is untouched.  For an inference engine
 * that needs the HBM back (the GPU is shared with inference after the load).
 * Errors: SLLM_E_INVALID for a negative ordinal, SLLM_E_CUDA if the device or pool call fails. */
SLLM_API sllm_status sllm_device_trim(int32_t gpu, uint64_t keep_bytes);

/* ------------------------------------------------------------------------------------
 * Cross-process tensor handles (the inference process
 * "acquires the base addresses for each GPU (i.e., CUDA IPC handles) from the model
 * manager" and computes base + offset).  The exporter (loader process) publishes each
 * partition's device base; the importer maps it and builds its tensors from the index.
 * ------------------------------------------------------------------------------------ */
typedef struct {
  uint8_t handle[64];  /* cudaIpcMemHandle_t of the allocation that holds the region       */
  uint64_t offset;     /* region start minus that allocation's base                         */
  uint64_t nbytes;     /* region length                                                     */
  int32_t gpu;         /* CUDA ordinal of the exporting device                              */
  int32_t reserved;
} sllm_ipc_region;
/* dev_ptr: device pointer inside a cudaMalloc'd allocation (e.g. a torch tensor). */
SLLM_API sllm_status sllm_ipc_export(const void* dev_ptr, uint64_t nbytes, sllm_ipc_region* out);
/* Map an exported region into this (other) process in the context of device region->gpu
 * (the exporter's GPU as exported; set it to the importing GPU to reach a peer's memory
 * over NVLink, e.g. for a P2P peer group); *dev_ptr = its start.
 * The mapping stays valid until sllm_ipc_close; the exporter must keep the memory alive. */
SLLM_API sllm_status sllm_ipc_open(const sllm_ipc_region* region, void** dev_ptr);
SLLM_API sllm_status sllm_ipc_close(void* dev_ptr);

/* ------------------------------------------------------------------------------------
 * Device-resident helpers (the kernels on their own; used for HBM-roofline measurement
 * and by users who already hold partition bytes in device memory).
 * ------------------------------------------------------------------------------------ */
/* Fletcher-64 of every `block`-byte block of a device buffer (len multiple of 16).
 * out_dev: device pointer to ceil(len/block) uint64.  Asynchronous on `stream`. */
SLLM_API sllm_status sllm_block_checksums_device(const void* src_dev, uint64_t len, uint64_t block, uint64_t* out_dev,
                                        int32_t ctas, void* stream);
/* Scatter partition p, already resident at src_dev (device pointer, L_p bytes), into the
 * per-tensor buffers dst_tensor[i] (as in sllm_load_start), verifying every block against
 * the index.  Synchronous; SLLM_E_CHECKSUM names the first bad block in *bad_block.
 * kernel_ms (NULL = not timed): device time of the K3 launch alone, from CUDA events
 * recorded on `stream` immediately around it (table uploads and the result read excluded). */
SLLM_API sllm_status sllm_materialise_device(const sllm_index* index, size_t p, const void* src_dev,
                                    void* const* dst_tensor, int32_t ctas, void* stream, uint64_t* bad_block,
                                    float* kernel_ms);

#ifdef __cplusplus
}
#endif
#endif /* SLLM_H_ */
