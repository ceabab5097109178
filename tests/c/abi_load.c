/* A plain-C client of libsllm.so: no Python, no torch -- only include/sllm.h and the CUDA
 * runtime for device memory.  Plans a small checkpoint (odd sizes, a scalar, a 66-byte
 * vector), fills pinned partitions through the converter's in-memory sink, serialises and
 * re-opens the index, loads every partition in each mode, and checks every device byte,
 * every tensor handle (base + offset) and the device checksums against the index.
 * Exit code 0 = pass.  Built and run by tests/test_c_abi.py. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "sllm.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    sllm_status s_ = (x);                                                          \
    if (s_ != SLLM_OK) {                                                           \
      fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, (int)s_,     \
              sllm_last_error());                                                  \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CUDA(x)                                                                    \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

enum { NT = 7 };

int main(void) {
  /* two logical devices (partitions), both loaded onto GPU 0 */
  static const char* names[NT] = {"emb", "w0", "b0", "odd.vec", "odd.scalar", "w1", "head"};
  static const int32_t dev[NT] = {0, 0, 0, 0, 1, 1, 1};
  static const int64_t shp[NT][2] = {{1000, 384}, {384, 384}, {384, 0}, {33, 0}, {0, 0}, {512, 700}, {3, 5}};
  static const int32_t nd[NT] = {2, 2, 1, 1, 0, 2, 2};
  sllm_src_tensor t[NT];
  uint8_t* data[NT];
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < NT; ++i) {
    uint64_t n = 2;
    for (int d = 0; d < nd[i]; ++d) n *= (uint64_t)shp[i][d];
    data[i] = (uint8_t*)malloc(n);
    for (uint64_t k = 0; k < n; ++k) { /* xorshift bytes */
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      data[i][k] = (uint8_t)x;
    }
    t[i].name = names[i];
    t[i].device_id = dev[i];
    t[i].dtype = SLLM_F16;
    t[i].ndim = nd[i];
    t[i].shape = shp[i];
    t[i].data = data[i];
    t[i].nbytes = n;
  }
  sllm_index* plan = NULL;
  CHECK(sllm_plan(t, NT, 4096, 64 << 10, "c-abi", &plan));
  size_t ntens = 0, nparts = 0;
  CHECK(sllm_index_counts(plan, &ntens, &nparts));
  if (ntens != NT || nparts != 2) { fprintf(stderr, "counts %zu %zu\n", ntens, nparts); return 1; }
  void* host[2];
  uint64_t len[2];
  for (size_t p = 0; p < nparts; ++p) {
    int32_t did; uint64_t nb, ntp;
    CHECK(sllm_index_partition(plan, p, &did, &len[p], &nb, &ntp));
    CHECK(sllm_host_alloc(len[p], 0, &host[p]));
  }
  CHECK(sllm_convert_into(t, NT, plan, host));
  /* round trip through the serialised index, as a separate process would see it */
  size_t blen = 0;
  CHECK(sllm_index_serialize(plan, NULL, 0, &blen));
  void* blob = malloc(blen);
  CHECK(sllm_index_serialize(plan, blob, blen, &blen));
  sllm_index* idx = NULL;
  CHECK(sllm_index_from_memory(blob, blen, &idx));

  void* dbase[2];
  for (size_t p = 0; p < nparts; ++p) CUDA(cudaMalloc(&dbase[p], len[p]));
  const int32_t gpu[2] = {0, 0};
  const int modes[2] = {SLLM_MODE_CE, SLLM_MODE_ZEROCOPY};
  for (int m = 0; m < 2; ++m) {
    for (size_t p = 0; p < nparts; ++p) CUDA(cudaMemset(dbase[p], 0xEE, len[p]));
    sllm_load_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.chunk_bytes = 128 << 10;
    cfg.n_streams = 2;
    cfg.mode = modes[m];
    cfg.verify = 1;
    sllm_load* ld = NULL;
    CHECK(sllm_load_start(idx, &cfg, (const void* const*)host, gpu, dbase, NULL, NULL, NULL, &ld));
    sllm_load_report rep;
    CHECK(sllm_load_wait(ld, &rep));
    for (size_t p = 0; p < nparts; ++p) {
      uint8_t* back = (uint8_t*)malloc(len[p]);
      CUDA(cudaMemcpy(back, dbase[p], len[p], cudaMemcpyDeviceToHost));
      if (memcmp(back, host[p], len[p]) != 0) { fprintf(stderr, "mode %d partition %zu differs\n", m, p); return 1; }
      free(back);
      const uint64_t* got = NULL;
      const uint64_t* want = NULL;
      int32_t did; uint64_t L, nb, ntp;
      CHECK(sllm_index_partition(idx, p, &did, &L, &nb, &ntp));
      CHECK(sllm_load_block_checksums(ld, p, &got));
      CHECK(sllm_index_block_checksums(idx, p, &want));
      if (memcmp(got, want, nb * 8) != 0) { fprintf(stderr, "checksums differ\n"); return 1; }
    }
    for (int i = 0; i < NT; ++i) { /* handle = base + offset, contents = source tensor */
      sllm_tensor_handle h;
      CHECK(sllm_load_tensor(ld, names[i], &h));
      sllm_tensor_info ti;
      size_t k;
      CHECK(sllm_index_find(idx, names[i], &k));
      CHECK(sllm_index_tensor(idx, k, &ti));
      if ((uint8_t*)h.ptr != (uint8_t*)dbase[ti.partition] + ti.offset || h.nbytes != t[i].nbytes) {
        fprintf(stderr, "handle of %s\n", names[i]);
        return 1;
      }
      uint8_t* back = (uint8_t*)malloc(h.nbytes);
      CUDA(cudaMemcpy(back, h.ptr, h.nbytes, cudaMemcpyDeviceToHost));
      if (memcmp(back, data[i], h.nbytes) != 0) { fprintf(stderr, "tensor %s differs\n", names[i]); return 1; }
      free(back);
    }
    if (rep.payload_bytes == 0 || rep.bad_partition != -1) { fprintf(stderr, "report\n"); return 1; }
    sllm_load_free(ld);
  }
  /* captured load: no byte moves at capture; two replays load every partition again */
  {
    sllm_load_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.chunk_bytes = 128 << 10;
    cfg.verify = 1;
    for (size_t p = 0; p < nparts; ++p) CUDA(cudaMemset(dbase[p], 0xEE, len[p]));
    sllm_load* cap = NULL;
    CHECK(sllm_load_capture(idx, &cfg, (const void* const*)host, gpu, dbase, NULL, &cap));
    for (int r = 0; r < 3; ++r) {
      for (size_t p = 0; p < nparts; ++p) {
        uint8_t* back = (uint8_t*)malloc(len[p]);
        CUDA(cudaMemcpy(back, dbase[p], len[p], cudaMemcpyDeviceToHost));
        const int loaded = memcmp(back, host[p], len[p]) == 0;
        free(back);
        if (loaded != (r > 0)) { fprintf(stderr, "capture: replay %d partition %zu\n", r, p); return 1; }
      }
      if (r == 2) break;
      for (size_t p = 0; p < nparts && r == 1; ++p) CUDA(cudaMemset(dbase[p], 0x11, len[p]));
      CHECK(sllm_load_replay(cap, NULL));
      sllm_load_report rep;
      CHECK(sllm_load_wait(cap, &rep));
      if (rep.payload_bytes == 0 || rep.bad_partition != -1) { fprintf(stderr, "capture report\n"); return 1; }
    }
    sllm_load_free(cap);
  }
  /* a corrupted source byte is reported as (partition, block) */
  ((uint8_t*)host[1])[70000] ^= 1;
  {
    sllm_load_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.chunk_bytes = 128 << 10;
    cfg.verify = 1;
    sllm_load* ld = NULL;
    CHECK(sllm_load_start(idx, &cfg, (const void* const*)host, gpu, dbase, NULL, NULL, NULL, &ld));
    sllm_load_report rep;
    sllm_status st = sllm_load_wait(ld, &rep);
    if (st != SLLM_E_CHECKSUM || rep.bad_partition != 1 || rep.bad_block != 70000 / (64 << 10)) {
      fprintf(stderr, "fault: status %d partition %d block %llu\n", (int)st, rep.bad_partition,
              (unsigned long long)rep.bad_block);
      return 1;
    }
    sllm_load_free(ld);
  }
  for (size_t p = 0; p < nparts; ++p) {
    cudaFree(dbase[p]);
    sllm_host_free(host[p]);
  }
  sllm_index_close(idx);
  sllm_index_close(plan);
  free(blob);
  for (int i = 0; i < NT; ++i) free(data[i]);
  printf("c-abi ok\n");
  return 0;
}
