// Pinned DRAM model cache with whole-model LRU (SURVEY §8(f) rank 4 sibling; PAPER.md
// P:578-579 "pinned memory pool", "allocates pinned memory ... for the model
// checkpoints", P:1416 keeps popular checkpoints in host memory; SPEC S:102-108,
// S:140-148 pool with alloc/free and LRU of whole models).
//
// acquire(dir) returns the partitions of the model stored under <dir> (index.bin +
// part_<d>.bin, the converter's output) resident in page-locked, device-mapped host memory
// -- ready to be a load source.  A miss reserves the model's bytes, evicting the least
// recently used models nobody holds, then reads every partition with the O_DIRECT
// readers of the file tier outside the cache lock; concurrent acquirers of the same model
// wait for that one read.  An acquired model is never evicted until released.
#include <condition_variable>
#include <list>
#include <map>

#include "common.hpp"

namespace sllm {

void* host_alloc(uint64_t bytes, int gpu);
void host_free(void* p);
std::vector<uint8_t> read_file(const char* path);
void read_partition(const char* dir, const sllm_index* idx, size_t p, void* dst, int threads);

}  // namespace sllm

struct sllm_cache {
  struct Entry {
    sllm_index* idx = nullptr;
    std::vector<void*> bufs;
    uint64_t bytes = 0;
    int refs = 0;
    bool ready = false;
    std::list<std::string>::iterator pos;  // in `lru`, front = most recently acquired
  };
  uint64_t capacity = 0, used = 0, hits = 0, misses = 0, evictions = 0;
  int gpu = -1;
  bool pin = true;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::string, Entry> models;
  std::list<std::string> lru;
};

namespace sllm {

static void* cache_alloc(const sllm_cache& c, uint64_t n) {
  if (c.pin) return host_alloc(n, c.gpu);
  void* p = nullptr;  // pin = 0: plain page-aligned memory (host-only use, CPU tests)
  if (posix_memalign(&p, 4096, align_up(std::max<uint64_t>(n, 1), 4096)) != 0) fail(SLLM_E_NOMEM, "cache allocation");
  return p;
}

static void cache_free(const sllm_cache& c, void* p) {
  if (!p) return;
  if (c.pin) host_free(p);
  else free(p);
}

static void drop(sllm_cache& c, std::map<std::string, sllm_cache::Entry>::iterator it) {
  for (void* b : it->second.bufs) cache_free(c, b);
  delete it->second.idx;
  c.used -= it->second.bytes;
  c.lru.erase(it->second.pos);
  c.models.erase(it);
}

sllm_cache* cache_create(uint64_t capacity, int gpu, int pin) {
  if (capacity == 0) fail(SLLM_E_INVALID, "zero cache capacity");
  std::unique_ptr<sllm_cache> c(new sllm_cache);
  c->capacity = capacity;
  c->gpu = gpu;
  c->pin = pin != 0;
  return c.release();
}

void cache_acquire(sllm_cache* c, const char* dir, int io_threads, const sllm_index** index, void* const** bufs,
                   int32_t* hit) {
  if (!c || !dir || !index || !bufs) fail(SLLM_E_INVALID, "null argument");
  const std::string key(dir);
  std::unique_ptr<sllm_index> parsed;  // a miss's index, read and parsed outside the lock
  std::unique_lock<std::mutex> g(c->mu);
  for (;;) {
    auto it = c->models.find(key);
    if (it == c->models.end()) {
      if (parsed) break;
      g.unlock();  // storage read + parse: hits on other models are not held up by it
      std::vector<uint8_t> blob = read_file((key + "/index.bin").c_str());
      parsed.reset(parse(blob.data(), blob.size()));
      g.lock();
      continue;  // look again: another acquirer may have started this model meanwhile
    }
    if (!it->second.ready) {  // another thread is reading it: wait, then look again
      c->cv.wait(g);
      continue;
    }
    it->second.refs++;
    c->lru.splice(c->lru.begin(), c->lru, it->second.pos);
    c->hits++;
    *index = it->second.idx;
    *bufs = it->second.bufs.data();
    if (hit) *hit = 1;
    return;
  }
  // miss: reserve the bytes (evicting unheld models, LRU first)
  sllm_index* idx = parsed.release();
  uint64_t need = 0;
  for (auto& pr : idx->parts) need += align_up(pr.length, 2ull << 20);
  if (need > c->capacity) {
    delete idx;
    fail(SLLM_E_CAPACITY, "model " + key + " (" + std::to_string(need) + " B) exceeds the cache capacity");
  }
  for (auto l = c->lru.end(); c->used + need > c->capacity && l != c->lru.begin();) {
    --l;  // walk from the least recently used end
    auto it = c->models.find(*l);
    if (it->second.refs == 0 && it->second.ready) {
      ++l;  // stays valid: drop() erases only the victim's list node
      drop(*c, it);
      c->evictions++;
    }
  }
  if (c->used + need > c->capacity) {
    delete idx;
    fail(SLLM_E_CAPACITY, "cache full: models in use hold " + std::to_string(c->used) + " B of " +
                              std::to_string(c->capacity) + " B");
  }
  c->lru.push_front(key);
  sllm_cache::Entry& e = c->models[key];
  e.idx = idx;
  e.bytes = need;
  e.refs = 1;
  e.pos = c->lru.begin();
  c->used += need;
  c->misses++;
  g.unlock();
  // storage -> pinned DRAM, outside the lock (other models stay available meanwhile)
  std::vector<void*> got(idx->parts.size(), nullptr);
  try {
    for (size_t p = 0; p < idx->parts.size(); ++p) {
      got[p] = cache_alloc(*c, idx->parts[p].length);
      read_partition(dir, idx, p, got[p], io_threads);
    }
  } catch (...) {
    g.lock();
    auto it = c->models.find(key);
    it->second.bufs = got;
    it->second.ready = true;  // so drop() accounting is uniform
    drop(*c, it);
    c->cv.notify_all();
    throw;
  }
  g.lock();
  sllm_cache::Entry& done = c->models[key];
  done.bufs = got;
  done.ready = true;
  *index = done.idx;
  *bufs = done.bufs.data();
  if (hit) *hit = 0;
  c->cv.notify_all();
}

void cache_release(sllm_cache* c, const char* dir) {
  if (!c || !dir) fail(SLLM_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  auto it = c->models.find(dir);
  if (it == c->models.end() || !it->second.ready || it->second.refs == 0)
    fail(SLLM_E_LOOKUP, std::string("model ") + dir + " is not held");
  it->second.refs--;
}

void cache_stats(sllm_cache* c, sllm_cache_stats* s) {
  if (!c || !s) fail(SLLM_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(c->mu);
  s->capacity = c->capacity;
  s->used = c->used;
  s->models = c->models.size();
  s->hits = c->hits;
  s->misses = c->misses;
  s->evictions = c->evictions;
}

void cache_destroy(sllm_cache* c) {
  if (!c) return;
  {
    std::lock_guard<std::mutex> g(c->mu);
    while (!c->models.empty()) drop(*c, c->models.begin());
  }
  delete c;
}

}  // namespace sllm
