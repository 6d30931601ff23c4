// End-to-end timing of the C++ drop-in API (include/agq_b200/*.hpp) as a
// reference-side caller uses it: host std::vector in, host std::vector out
// (quantize.hpp:78-189, collective.hpp:128-147; tools/agq.cpp:119-120 calls
// quantize_blockwise + dequantize_blockwise exactly like this), beside the
// reference's own CPU implementation of the same calls (oracle/_ref, loaded
// with dlopen so this binary links only libagq_cuda.so).
//
// Workload C1: 4096 x 4096 FP32 values of make_rng(1, 0x1D) (the reference
// CLI's `--seed 1 --normal 16777216`), INT4 block 128. Also the FP8
// local_accumulate of a 2^24-element gradient. Prints one JSON object.
//
// usage: dropin_bench [ref_lib_path]
#include <dlfcn.h>
#include <malloc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../include/agq_b200/agq.hpp"

namespace {
double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
template <class F>
double median_time(F&& f, int reps) {
  std::vector<double> t;
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    f();
    t.push_back(now() - t0);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}
using RefQ = int (*)(const float*, size_t, int, uint32_t, int, uint8_t*, float*, char*, size_t);
using RefD = int (*)(const uint8_t*, const float*, size_t, int, uint32_t, int, float*, char*,
                     size_t);
using RefA = int (*)(const uint8_t*, const float*, size_t, uint32_t, const float*, int, uint8_t*,
                     float*, char*, size_t);
}  // namespace

int main(int argc, char** argv) {
  // Steady state of a long-running caller: freed vectors stay in the heap and
  // are reused (no mmap/munmap and first-touch page faults per call). Applies
  // to both arms; the API returns its results in new std::vectors.
  mallopt(M_MMAP_MAX, 0);
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
  const std::size_t n = 4096ull * 4096ull;
  std::vector<float> x(n);
  if (agq_fill_input(1, 0x1D, 0, AGQ_INPUT_NORMAL, 0.0, 1.0, AGQ_F32, x.data(), n) != AGQ_OK) {
    std::printf("{\"error\": \"fill\"}\n");
    return 1;
  }
  // warm-up (CUDA context, pipeline staging, kernels)
  auto q = agq::quantize_blockwise(x, 4);
  auto back = agq::dequantize_blockwise(q);
  const int reps = 15;
  const double tq = median_time([&] { q = agq::quantize_blockwise(x, 4); }, reps);
  const double td = median_time([&] { back = agq::dequantize_blockwise(q); }, reps);
  // the C-ABI host entry points into caller-owned (warm) buffers: the
  // library's path without the API's result-vector construction
  std::vector<uint8_t> pc(n);
  std::vector<float> pscales(n / 128), pout(n);
  double st[4], sq[4], sd[4];
  agq_host_pipeline_stats(st, 1);
  const double tq_abi = median_time([&] {
    agq_quantize_host(x.data(), n, 4, 128, 0, pc.data(), pscales.data());
  }, reps);
  agq_host_pipeline_stats(sq, 1);
  const double td_abi = median_time([&] {
    agq_dequantize_host(pc.data(), pscales.data(), n, 4, 128, 0, pout.data());
  }, reps);
  agq_host_pipeline_stats(sd, 1);
  // the staging copy rate the pipelines run at (caller memory -> other
  // memory through the library's copy threads): the host-memory bound
  const double t_copy = median_time([&] { agq_host_copy(pout.data(), x.data(), 4 * n); }, reps);
  // what the API's value-initialised result vectors cost on this host alone
  const double t_alloc_f32 = median_time([&] { std::vector<float> v(n); asm volatile("" ::"r"(v.data()) : "memory"); }, reps);
  const double t_alloc_u8 = median_time([&] { std::vector<uint8_t> v(n); asm volatile("" ::"r"(v.data()) : "memory"); }, reps);

  // where the API's dequantize time goes: the same steps as
  // dequantize_blockwise, timed one by one
  double parts[3] = {0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    std::vector<float> v(n);
    const double t1 = now();
    agq_dequantize_host(q.codes.data(), q.scales.data(), n, 4, 128, 0, v.data());
    const double t2 = now();
    back = std::move(v);
    const double t3 = now();
    parts[0] += t1 - t0;
    parts[1] += t2 - t1;
    parts[2] += t3 - t2;
  }

  // the same with the split entry the API uses (begin, zero, finish)
  double jparts[3] = {0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    agq_host_job* job = nullptr;
    agq_dequantize_host_begin(q.codes.data(), q.scales.data(), n, 4, 128, 0, &job);
    const double t1 = now();
    std::vector<float> v(n);
    const double t2 = now();
    agq_host_job_finish(job, v.data(), nullptr);
    const double t3 = now();
    back = std::move(v);
    jparts[0] += t1 - t0;
    jparts[1] += t2 - t1;
    jparts[2] += t3 - t2;
  }

  double qparts[3] = {0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    const double t0 = now();
    agq_host_job* job = nullptr;
    agq_quantize_host_begin(x.data(), n, 4, 128, 0, &job);
    const double t1 = now();
    agq::QuantizedTensor t;
    t.codes.resize(n);
    t.scales.resize(n / 128);
    const double t2 = now();
    agq_host_job_finish(job, t.codes.data(), t.scales.data());
    const double t3 = now();
    q = std::move(t);
    qparts[0] += t1 - t0;
    qparts[1] += t2 - t1;
    qparts[2] += t3 - t2;
  }

  // FP8 local_accumulate: 2^24-element gradient, FP32 local
  const std::size_t na = 1u << 24;
  std::vector<float> g0(na), loc(na);
  agq_fill_input(7, 0x1D, 0, AGQ_INPUT_NORMAL, 0.0, 1e-3, AGQ_F32, g0.data(), na);
  agq_fill_input(7, 0x1D, 1, AGQ_INPUT_NORMAL, 0.0, 1e-3, AGQ_F32, loc.data(), na);
  const auto main_g = agq::quantize_blockwise(g0, 8, 128, agq::CodecKind::Fp8E4M3);
  auto acc = agq::local_accumulate(main_g, loc);
  const double ta = median_time([&] { acc = agq::local_accumulate(main_g, loc); }, reps);

  // the reference's own implementation of the same calls (one thread)
  double rq = -1, rd = -1, ra = -1;
  bool same = false, same_q = false, same_acc = false;
  if (argc > 1) {
    if (void* h = dlopen(argv[1], RTLD_NOW | RTLD_LOCAL)) {
      auto fq = reinterpret_cast<RefQ>(dlsym(h, "ref_quantize"));
      auto fd = reinterpret_cast<RefD>(dlsym(h, "ref_dequantize"));
      auto fa = reinterpret_cast<RefA>(dlsym(h, "ref_local_accumulate"));
      std::vector<uint8_t> rc(n);
      std::vector<float> rs(n / 128), ro(n);
      char err[256];
      rq = median_time([&] { fq(x.data(), n, 4, 128, 0, rc.data(), rs.data(), err, 256); }, 3);
      rd = median_time([&] { fd(rc.data(), rs.data(), n, 4, 128, 0, ro.data(), err, 256); }, 3);
      same_q = rc == q.codes && rs == q.scales;
      same = same_q && std::memcmp(ro.data(), back.data(), n * 4) == 0;
      std::vector<uint8_t> ac(na);
      std::vector<float> as(na / 128);
      ra = median_time([&] {
        fa(main_g.codes.data(), main_g.scales.data(), na, 128, loc.data(), 0, ac.data(), as.data(),
           err, 256);
      }, 3);
      same_acc = ac == acc.codes && as == acc.scales;
    }
  }
  // bytes the API must move over PCIe (one code byte per element, FP32 I/O)
  const double nb = (double)n / 128;
  const double q_h2d = 4.0 * n, q_d2h = n + 4 * nb, d_h2d = n + 4 * nb, d_d2h = 4.0 * n;
  const double a_h2d = na + 4.0 * na / 128 + 4.0 * na, a_d2h = na + 4.0 * na / 128;
  std::printf(
      "{\"config\": \"C1 through the C++ drop-in API: agq::quantize_blockwise(4096x4096 fp32 "
      "std::vector, 4) + agq::dequantize_blockwise; FP8 local_accumulate 2^24\", "
      "\"elements\": %zu, \"quantize_ms\": %.3f, \"dequantize_ms\": %.3f, "
      "\"roundtrip_ms\": %.3f, \"accumulate_ms\": %.3f, "
      "\"quantize_h2d_bytes\": %.0f, \"quantize_d2h_bytes\": %.0f, "
      "\"dequantize_h2d_bytes\": %.0f, \"dequantize_d2h_bytes\": %.0f, "
      "\"accumulate_h2d_bytes\": %.0f, \"accumulate_d2h_bytes\": %.0f, "
      "\"ref_quantize_ms\": %.3f, \"ref_dequantize_ms\": %.3f, \"ref_accumulate_ms\": %.3f, "
      "\"ref_threads\": 1, \"allocator\": \"glibc heap, no mmap/trim (vectors reused, both arms)\", "
      "\"abi_pipeline_quantize_ms\": {\"inside\": %.3f, \"host_copies\": %.3f, \"wait_device\": %.3f}, "
      "\"abi_pipeline_dequantize_ms\": {\"inside\": %.3f, \"host_copies\": %.3f, \"wait_device\": %.3f}, "
      "\"alloc_zero_f32_ms\": %.3f, \"alloc_zero_u8_ms\": %.3f, "
      "\"abi_quantize_host_ms\": %.3f, \"abi_dequantize_host_ms\": %.3f, "
      "\"host_copy_GBs\": %.2f, "
      "\"api_dequantize_parts_ms\": {\"alloc_zero\": %.3f, \"host_call\": %.3f, \"assign_free\": %.3f}, "
      "\"api_dequantize_job_parts_ms\": {\"begin\": %.3f, \"alloc_zero\": %.3f, \"finish\": %.3f}, "
      "\"api_quantize_job_parts_ms\": {\"begin\": %.3f, \"alloc_zero\": %.3f, \"finish\": %.3f}, "
      "\"quantize_bitexact_vs_ref\": %s, \"bitexact_vs_ref\": %s, \"accumulate_bitexact_vs_ref\": %s}\n",
      n, tq * 1e3, td * 1e3, (tq + td) * 1e3, ta * 1e3, q_h2d, q_d2h, d_h2d, d_d2h, a_h2d, a_d2h,
      rq * 1e3, rd * 1e3, ra * 1e3, sq[0] * 1e3 / reps, sq[1] * 1e3 / reps,
      sq[2] * 1e3 / reps, sd[0] * 1e3 / reps, sd[1] * 1e3 / reps, sd[2] * 1e3 / reps,
      t_alloc_f32 * 1e3, t_alloc_u8 * 1e3, tq_abi * 1e3, td_abi * 1e3,
      4.0 * n / t_copy / 1e9, parts[0] * 1e3 / reps, parts[1] * 1e3 / reps, parts[2] * 1e3 / reps,
      jparts[0] * 1e3 / reps, jparts[1] * 1e3 / reps, jparts[2] * 1e3 / reps,
      qparts[0] * 1e3 / reps, qparts[1] * 1e3 / reps, qparts[2] * 1e3 / reps, same_q ? "true" : "false", same ? "true" : "false", same_acc ? "true" : "false");
  return 0;
}
