// Host test of the NUMA thread binding (numa.cpp) against a fake sysfs node tree
// (SLLM_SYSFS_ROOT): node0 = CPU argv[1], node1 = CPU argv[2].  One thread is bound to
// node 0, then re-bound to node 1 (a pooled load worker moving to another GPU's job), then
// unbound (unknown node, missing node); the main thread's mask never changes.
#include "../../paper_2401_14351_b200/csrc/numa.cpp"

#include <cstdlib>
#include <thread>

static int fails = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                      \
    }                                                               \
  } while (0)

static cpu_set_t mask_of(pid_t t) {
  cpu_set_t m;
  CPU_ZERO(&m);
  sched_getaffinity(t, sizeof m, &m);
  return m;
}
static cpu_set_t only(int c) {
  cpu_set_t m;
  CPU_ZERO(&m);
  CPU_SET(c, &m);
  return m;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const int c0 = atoi(argv[1]), c1 = atoi(argv[2]);
  using namespace sllm;
  EXPECT(numa_nodes() == 2);
  cpu_set_t l;
  EXPECT(parse_cpulist("0-3,8,10-11\n", &l) && CPU_COUNT(&l) == 7 && CPU_ISSET(3, &l) && CPU_ISSET(8, &l) &&
         !CPU_ISSET(9, &l) && CPU_ISSET(11, &l));
  EXPECT(!parse_cpulist("\n", &l));
  const cpu_set_t main_before = mask_of(0);
  std::thread t([&] {
    EXPECT(bind_thread_to_node(0));
    cpu_set_t m = mask_of(0), want = only(c0);
    EXPECT(CPU_EQUAL(&m, &want));
    EXPECT(bind_thread_to_node(1));  // re-bound to the other node
    m = mask_of(0);
    want = only(c1);
    EXPECT(CPU_EQUAL(&m, &want));
    EXPECT(bind_thread_to_node(-1));  // unknown node: back to the process mask
    m = mask_of(0);
    EXPECT(CPU_EQUAL(&m, &main_before));
    EXPECT(bind_thread_to_node(1));
    EXPECT(bind_thread_to_node(7));  // no such node: process mask
    m = mask_of(0);
    EXPECT(CPU_EQUAL(&m, &main_before));
  });
  t.join();
  const cpu_set_t main_after = mask_of(0);
  EXPECT(CPU_EQUAL(&main_before, &main_after));
  if (fails) return 1;
  std::printf("numa bind ok\n");
  return 0;
}
