/* Multi-threaded twin of synth/payload.py: fills host
 * buffers with the counter-based splitmix64 payload.  Input generation only --
 * no layout, index, checksum or chunking arithmetic lives here. */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define JOB_BYTES (4ULL << 20)

static inline uint64_t splitmix64(uint64_t z) {
  z += GOLDEN;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct { uint8_t* dst; uint64_t lo, hi, key; } job_t;  /* byte range [lo,hi) of one tensor */
typedef struct { job_t* jobs; size_t njobs; size_t next; pthread_mutex_t mu; } pool_t;

static void run_job(const job_t* j) {
  uint64_t k = j->lo / 8;
  uint64_t b = j->lo;
  for (; b + 8 <= j->hi; b += 8, ++k) {
    uint64_t w = splitmix64(j->key + k * GOLDEN);
    memcpy(j->dst + b, &w, 8); /* x86-64 is little-endian */
  }
  if (b < j->hi) {
    uint64_t w = splitmix64(j->key + k * GOLDEN);
    memcpy(j->dst + b, &w, (size_t)(j->hi - b));
  }
}

static void* worker(void* arg) {
  pool_t* p = (pool_t*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    size_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->njobs) return NULL;
    run_job(&p->jobs[i]);
  }
}

int synth_fill_many(size_t n, void* const* dsts, const uint64_t* sizes, uint64_t seed,
                    const uint64_t* es, int nthreads) {
  size_t njobs = 0;
  for (size_t i = 0; i < n; ++i) njobs += (size_t)((sizes[i] + JOB_BYTES - 1) / JOB_BYTES);
  if (njobs == 0) return 0;
  job_t* jobs = (job_t*)malloc(njobs * sizeof(job_t));
  if (!jobs) return 1;
  size_t q = 0;
  for (size_t i = 0; i < n; ++i) {
    uint64_t key = splitmix64(seed ^ splitmix64(es[i]));
    for (uint64_t lo = 0; lo < sizes[i]; lo += JOB_BYTES) {
      uint64_t hi = lo + JOB_BYTES < sizes[i] ? lo + JOB_BYTES : sizes[i];
      jobs[q++] = (job_t){(uint8_t*)dsts[i], lo, hi, key};
    }
  }
  pool_t pool = {jobs, njobs, 0, PTHREAD_MUTEX_INITIALIZER};
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > njobs) nthreads = (int)njobs;
  pthread_t* th = (pthread_t*)malloc((size_t)nthreads * sizeof(pthread_t));
  int started = 0;
  for (int t = 1; t < nthreads; ++t)
    if (pthread_create(&th[t], NULL, worker, &pool) == 0) ++started; else break;
  worker(&pool);
  for (int t = 1; t <= started; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
