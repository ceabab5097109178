/* Host-side exerciser of libsllm.so for AddressSanitizer / UBSan builds (no GPU needed):
 * plan + convert_into + seal + serialize for random checkpoints, then parse every
 * truncation of every index and thousands of single-byte corruptions (each must fail
 * cleanly with SLLM_E_FORMAT or parse to an identical re-serialisation), tensor lookups,
 * addresses, conversion errors, and the pinned-cache policy with pin = 0.
 * Run by tests/test_sanitizers.py against an -fsanitize=address,undefined build. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>

#include "sllm.h"

static uint64_t rng = 0x243F6A8885A308D3ull;
static uint64_t next_u64(void) {
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return rng;
}

#define FAILIF(c, ...)                 \
  do {                                 \
    if (c) {                           \
      fprintf(stderr, __VA_ARGS__);    \
      fprintf(stderr, "\n");           \
      exit(1);                         \
    }                                  \
  } while (0)

static const int32_t kWidth[6] = {2, 2, 4, 1, 1, 8};

int main(int argc, char** argv) {
  const char* tmpdir = argc > 1 ? argv[1] : "/tmp";
  long parsed_ok = 0, rejected = 0;
  for (int round = 0; round < 40; ++round) {
    const int n = 1 + (int)(next_u64() % 60);
    sllm_src_tensor* t = calloc((size_t)n, sizeof *t);
    int64_t(*shape)[4] = calloc((size_t)n, sizeof *shape);
    char(*names)[32] = calloc((size_t)n, sizeof *names);
    uint8_t** data = calloc((size_t)n, sizeof *data);
    for (int i = 0; i < n; ++i) {
      snprintf(names[i], sizeof names[i], "r%d.t%d", round, i);
      t[i].name = names[i];
      t[i].device_id = (int32_t)(next_u64() % 3) * 2; /* sparse ids 0, 2, 4 */
      t[i].dtype = (int32_t)(next_u64() % 6);
      t[i].ndim = (int32_t)(next_u64() % 4);
      uint64_t numel = 1;
      for (int d = 0; d < t[i].ndim; ++d) {
        shape[i][d] = 1 + (int64_t)(next_u64() % 37);
        numel *= (uint64_t)shape[i][d];
      }
      t[i].shape = shape[i];
      t[i].nbytes = numel * (uint64_t)kWidth[t[i].dtype];
      data[i] = malloc(t[i].nbytes);
      for (uint64_t k = 0; k < t[i].nbytes; ++k) data[i][k] = (uint8_t)next_u64();
      t[i].data = data[i];
    }
    const uint64_t align = 16ull << (next_u64() % 9);          /* 16 .. 4096 */
    const uint64_t block = (next_u64() % 4 == 0) ? 0 : align << (next_u64() % 4);
    sllm_index* plan = NULL;
    FAILIF(sllm_plan(t, (size_t)n, align, block, "fuzz", &plan) != SLLM_OK, "plan: %s", sllm_last_error());
    size_t nt = 0, np = 0;
    sllm_index_counts(plan, &nt, &np);
    FAILIF(nt != (size_t)n, "count");
    void** bufs = calloc(np, sizeof *bufs);
    for (size_t p = 0; p < np; ++p) {
      int32_t dev;
      uint64_t L, nb, ntp;
      sllm_index_partition(plan, p, &dev, &L, &nb, &ntp);
      bufs[p] = malloc(L ? L : 1);
      memset(bufs[p], 0xA5, L);
    }
    FAILIF(sllm_convert_into(t, (size_t)n, plan, bufs) != SLLM_OK, "convert_into: %s", sllm_last_error());
    FAILIF(sllm_index_seal(plan, (const void* const*)bufs) != SLLM_OK, "seal");
    size_t len = 0;
    sllm_index_serialize(plan, NULL, 0, &len);
    uint8_t* blob = malloc(len);
    FAILIF(sllm_index_serialize(plan, blob, len, &len) != SLLM_OK, "serialize");
    /* every truncation must be rejected */
    for (size_t cut = 0; cut < len; cut += 1 + (len > 4000 ? next_u64() % 7 : 0)) {
      sllm_index* x = NULL;
      FAILIF(sllm_index_from_memory(blob, cut, &x) == SLLM_OK, "truncation %zu accepted", cut);
      ++rejected;
    }
    /* single-byte corruptions: reject, or parse to something that re-serialises to the input */
    uint8_t* mut = malloc(len);
    for (int k = 0; k < 300; ++k) {
      memcpy(mut, blob, len);
      mut[next_u64() % len] ^= (uint8_t)(1 + next_u64() % 255);
      sllm_index* x = NULL;
      if (sllm_index_from_memory(mut, len, &x) == SLLM_OK) {
        size_t l2 = 0;
        sllm_index_serialize(x, NULL, 0, &l2);
        uint8_t* b2 = malloc(l2);
        sllm_index_serialize(x, b2, l2, &l2);
        FAILIF(l2 != len || memcmp(b2, mut, len) != 0, "accepted corruption does not round-trip");
        free(b2);
        sllm_index_close(x);
        ++parsed_ok;
      } else {
        ++rejected;
      }
    }
    /* lookups and addresses */
    sllm_index* idx = NULL;
    FAILIF(sllm_index_from_memory(blob, len, &idx) != SLLM_OK, "parse");
    uint64_t bases[8] = {1u << 20, 2u << 20, 3u << 20, 4u << 20, 5u << 20, 6u << 20, 7u << 20, 8u << 20};
    for (int i = 0; i < n; ++i) {
      size_t k = 0;
      FAILIF(sllm_index_find(idx, names[i], &k) != SLLM_OK || k != (size_t)i, "find");
      sllm_tensor_info ti;
      sllm_index_tensor(idx, k, &ti);
      int32_t dev;
      uint64_t addr;
      FAILIF(sllm_tensor_address(idx, names[i], bases, &dev, &addr) != SLLM_OK, "address");
      FAILIF(addr != bases[ti.partition] + ti.offset, "address value");
      FAILIF(memcmp((uint8_t*)bufs[ti.partition] + ti.offset, data[i], t[i].nbytes) != 0, "bytes");
    }
    size_t k = 0;
    FAILIF(sllm_index_find(idx, "missing", &k) != SLLM_E_LOOKUP, "lookup error");
    /* conversion errors: duplicate name, size mismatch */
    if (n > 1) {
      t[1].name = t[0].name;
      sllm_index* bad = NULL;
      FAILIF(sllm_plan(t, (size_t)n, align, block, "", &bad) != SLLM_E_CONVERSION, "duplicate accepted");
      t[1].name = names[1];
      t[0].nbytes += 1;
      FAILIF(sllm_plan(t, (size_t)n, align, block, "", &bad) != SLLM_E_CONVERSION, "size mismatch accepted");
      t[0].nbytes -= 1;
    }
    /* files + cache (pin = 0): convert to a directory, acquire twice, release */
    if (round % 8 == 0) {
      char dir[512];
      snprintf(dir, sizeof dir, "%s/fuzz_ckpt_%d", tmpdir, round);
      FAILIF(sllm_convert(t, (size_t)n, align, block, "fuzz", dir) != SLLM_OK, "convert: %s", sllm_last_error());
      sllm_cache* cache = NULL;
      FAILIF(sllm_cache_create(64ull << 20, -1, 0, &cache) != SLLM_OK, "cache");
      const sllm_index* ci = NULL;
      void* const* cb = NULL;
      int32_t hit = -1;
      FAILIF(sllm_cache_acquire(cache, dir, 2, &ci, &cb, &hit) != SLLM_OK || hit != 0, "acquire: %s", sllm_last_error());
      FAILIF(sllm_cache_acquire(cache, dir, 2, &ci, &cb, &hit) != SLLM_OK || hit != 1, "re-acquire");
      for (size_t p = 0; p < np; ++p) {
        int32_t dev;
        uint64_t L, nb, ntp;
        sllm_index_partition(ci, p, &dev, &L, &nb, &ntp);
        FAILIF(memcmp(cb[p], bufs[p], L) != 0, "cache bytes");
      }
      sllm_cache_release(cache, dir);
      sllm_cache_release(cache, dir);
      FAILIF(sllm_cache_release(cache, dir) != SLLM_E_LOOKUP, "over-release");
      sllm_cache_destroy(cache);
    }
    sllm_index_close(idx);
    sllm_index_close(plan);
    free(mut);
    free(blob);
    for (size_t p = 0; p < np; ++p) free(bufs[p]);
    free(bufs);
    for (int i = 0; i < n; ++i) free(data[i]);
    free(data);
    free(names);
    free(shape);
    free(t);
  }
  printf("host fuzz ok: %ld rejected, %ld accepted round-trips\n", rejected, parsed_ok);
  return 0;
}
