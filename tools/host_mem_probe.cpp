// Host memory probe for the drop-in API's result vectors: why value-
// initialising a 64 MB std::vector<float> costs what it does on the box.
// g++ -O2 -std=c++20 tools/host_mem_probe.cpp -o build/host_mem_probe -L... -lagq_cuda
#include <malloc.h>
#include <sys/resource.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../include/agq_cuda.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static long minflt() {
  rusage u;
  getrusage(RUSAGE_SELF, &u);
  return u.ru_minflt;
}
template <class F>
static double med(F&& f, int reps = 15) {
  const long f0 = minflt();
  std::vector<double> t;
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    f();
    t.push_back(now() - t0);
  }
  std::sort(t.begin(), t.end());
  std::printf("[%ld faults/rep] ", (minflt() - f0) / reps);
  return t[t.size() / 2] * 1e3;
}

int main() {
  mallopt(M_MMAP_MAX, 0);
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
  const size_t n = 4096ull * 4096ull;
  std::vector<float> keep(n, 1.0f), src(n, 2.0f);
  std::vector<float> a(n);
  std::printf("memset same buffer: %.3f ms\n", med([&] { std::memset(a.data(), 0, n * 4); }));
  std::printf("alloc+zero+free same size: %.3f ms\n",
              med([&] { std::vector<float> v(n); asm volatile("" ::"r"(v.data()) : "memory"); }));
  std::printf("alternate two (move-assign): %.3f ms\n", med([&] {
                std::vector<float> v(n);
                keep = std::move(v);
              }));
  std::printf("alternate two + pool copy into new: zero %.3f ms\n", med([&] {
                std::vector<float> v(n);
                agq_host_copy(v.data(), src.data(), n * 4);
                keep = std::move(v);
              }));
  double z = 0, c = 0;
  for (int r = 0; r < 15; ++r) {
    const double t0 = now();
    std::vector<float> v(n);
    const double t1 = now();
    agq_host_copy(v.data(), src.data(), n * 4);
    const double t2 = now();
    keep = std::move(v);
    z += t1 - t0;
    c += t2 - t1;
  }
  std::printf("  split: zero %.3f ms, pool copy %.3f ms\n", z / 15 * 1e3, c / 15 * 1e3);
  std::printf("pool copy only (warm dst): %.3f ms\n",
              med([&] { agq_host_copy(a.data(), src.data(), n * 4); }));
  return 0;
}
