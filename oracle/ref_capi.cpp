// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/agq (quantize.hpp, fp8.hpp, tensor_io.hpp,
// collective.hpp, rng.hpp). `oracle/Makefile` compiles this one file against
// those headers where they lie into oracle/_ref/libagq_ref.so. Nothing here
// restates the algorithm: every entry point calls the reference function of
// the same name, so the shared object IS the reference, and tests / the bench
// cpu_baseline / golden-vector generation can load it through ctypes.
//
// dbca.hpp / layers.hpp are not compiled (they need Eigen, absent here); the
// policy planner is restated in oracle/agq_oracle.c instead.
#include <cstring>  // collective.hpp uses std::memcpy without including it

#include <algorithm>
#include <cstdint>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "agq/collective.hpp"
#include "agq/fp8.hpp"
#include "agq/quantize.hpp"
#include "agq/rng.hpp"
#include "agq/tensor_io.hpp"

namespace {

// Status codes shared with the product C-ABI (include/agq_cuda.h).
constexpr int kOk = 0;
constexpr int kInvalidArgument = 1;
constexpr int kRuntimeError = 2;

int fail(const std::exception& e, int code, char* err, std::size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

template <typename F>
int guarded(char* err, std::size_t errlen, F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument& e) {
    return fail(e, kInvalidArgument, err, errlen);
  } catch (const std::exception& e) {
    return fail(e, kRuntimeError, err, errlen);
  }
}

agq::QuantizedTensor make_q(const std::uint8_t* codes, const float* scales,
                            std::size_t n, int bits, std::uint32_t block,
                            int codec) {
  agq::QuantizedTensor q;
  q.codes.assign(codes, codes + n);
  const std::size_t nb = block ? (n + block - 1) / block : 0;
  q.scales.assign(scales, scales + nb);
  q.bit_width = bits;
  q.block_size = block;
  q.codec_kind = static_cast<agq::CodecKind>(codec);
  q.shape = {static_cast<std::uint64_t>(n)};
  return q;
}

}  // namespace

extern "C" {

// ---- scalar formats (fp8.hpp) -------------------------------------------
std::uint8_t ref_fp8_encode(double v, int* overflow) {
  const auto r = agq::fp8_encode(v);
  if (overflow) *overflow = r.overflow ? 1 : 0;
  return r.value.byte;
}
double ref_fp8_decode(std::uint8_t b) { return agq::fp8_decode(agq::Fp8Value{b}); }
std::uint8_t ref_fp4_encode(double v) { return agq::fp4_encode(v); }
double ref_fp4_decode(std::uint8_t c) { return agq::fp4_decode(c); }
double ref_code_unit_value(int codec, int bits, std::uint8_t code) {
  return agq::code_unit_value(static_cast<agq::CodecKind>(codec), bits, code);
}
float ref_round_bf16(float x) { return agq::round_bf16(x); }
float ref_round_fp16(float x) { return agq::round_fp16(x); }

// ---- RNG (rng.hpp + libstdc++ normal_distribution<float>) ----------------
// kind 0: normal(0, scale); 1: uniform(lo, hi) float. Same draws as
// InputSpec::materialize (agq.cpp:47-65) and the test fixtures.
void ref_fill_normal(std::uint64_t root, std::uint64_t stream,
                     std::uint64_t index, float mean, float stddev,
                     float* out, std::size_t n) {
  agq::Rng rng = agq::make_rng(root, stream, index);
  std::normal_distribution<float> g(mean, stddev);
  for (std::size_t i = 0; i < n; ++i) out[i] = g(rng);
}
// Plain Rng(seed) as used by test_codec.cpp:15-22 random_floats.
void ref_fill_normal_seed(std::uint64_t seed, float stddev, float* out,
                          std::size_t n) {
  agq::Rng rng(seed);
  std::normal_distribution<float> g(0.0f, stddev);
  for (std::size_t i = 0; i < n; ++i) out[i] = g(rng);
}
std::uint64_t ref_derive_seed(std::uint64_t root, std::uint64_t stream,
                              std::uint64_t index) {
  return agq::derive_seed(root, stream, index);
}

// ---- block codec (quantize.hpp) ------------------------------------------
int ref_quantize(const float* x, std::size_t n, int bits, std::uint32_t block,
                 int codec, std::uint8_t* codes, float* scales, char* err,
                 std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto q = agq::quantize_blockwise(
        std::span<const float>(x, n), bits, block,
        static_cast<agq::CodecKind>(codec));
    std::copy(q.codes.begin(), q.codes.end(), codes);
    std::copy(q.scales.begin(), q.scales.end(), scales);
  });
}

int ref_dequantize(const std::uint8_t* codes, const float* scales,
                   std::size_t n, int bits, std::uint32_t block, int codec,
                   float* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto q = make_q(codes, scales, n, bits, block, codec);
    const auto v = agq::dequantize_blockwise(q);
    std::copy(v.begin(), v.end(), out);
  });
}

// Multi-threaded harness over the reference's single-threaded functions:
// block-aligned disjoint ranges, one reference call per thread (blocks are
// independent, quantize.hpp:103-136). Used only as the CPU baseline timing.
int ref_quantize_mt(const float* x, std::size_t n, int bits,
                    std::uint32_t block, int codec, std::uint8_t* codes,
                    float* scales, int threads) {
  const std::size_t nb = (n + block - 1) / block;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::vector<int> status(threads, 0);
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const std::size_t b0 = nb * t / threads, b1 = nb * (t + 1) / threads;
      const std::size_t e0 = std::min(n, b0 * block), e1 = std::min(n, b1 * block);
      if (e0 >= e1) return;
      try {
        const auto q = agq::quantize_blockwise(
            std::span<const float>(x + e0, e1 - e0), bits, block,
            static_cast<agq::CodecKind>(codec));
        std::copy(q.codes.begin(), q.codes.end(), codes + e0);
        std::copy(q.scales.begin(), q.scales.end(), scales + b0);
      } catch (...) {
        status[t] = 1;
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int s : status)
    if (s) return kInvalidArgument;
  return kOk;
}

int ref_dequantize_mt(const std::uint8_t* codes, const float* scales,
                      std::size_t n, int bits, std::uint32_t block, int codec,
                      float* out, int threads) {
  const std::size_t nb = (n + block - 1) / block;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::vector<int> status(threads, 0);
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const std::size_t b0 = nb * t / threads, b1 = nb * (t + 1) / threads;
      const std::size_t e0 = std::min(n, b0 * block), e1 = std::min(n, b1 * block);
      if (e0 >= e1) return;
      try {
        const auto q = make_q(codes + e0, scales + b0, e1 - e0, bits, block, codec);
        const auto v = agq::dequantize_blockwise(q);
        std::copy(v.begin(), v.end(), out + e0);
      } catch (...) {
        status[t] = 1;
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int s : status)
    if (s) return kInvalidArgument;
  return kOk;
}

// ---- packing and dump format (tensor_io.hpp) -----------------------------
std::size_t ref_pack_codes(const std::uint8_t* codes, std::size_t n, int bits,
                           std::uint8_t* out) {
  const std::vector<std::uint8_t> c(codes, codes + n);
  const auto p = agq::pack_codes(c, bits);
  std::copy(p.begin(), p.end(), out);
  return p.size();
}

int ref_unpack_codes(const std::uint8_t* bytes, std::size_t nbytes, int bits,
                     std::size_t count, std::uint8_t* out, char* err,
                     std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const std::vector<std::uint8_t> b(bytes, bytes + nbytes);
    const auto c = agq::unpack_codes(b, bits, count);
    std::copy(c.begin(), c.end(), out);
  });
}

// Writes the AGQT dump of quantize_blockwise(x, ...) with the given shape
// into `out` (capacity cap); returns the byte count or -1 on error.
long long ref_dump_quantized(const float* x, std::size_t n, int bits,
                             std::uint32_t block, int codec,
                             const std::uint64_t* shape, int ndim,
                             std::uint8_t* out, std::size_t cap) {
  try {
    std::vector<std::uint64_t> s(shape, shape + ndim);
    const auto q = agq::quantize_blockwise(std::span<const float>(x, n), bits,
                                           block,
                                           static_cast<agq::CodecKind>(codec),
                                           s);
    std::stringstream ss;
    agq::dump_tensor(q, ss);
    const std::string bytes = ss.str();
    if (bytes.size() > cap) return -1;
    std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
  } catch (...) {
    return -1;
  }
}

// ---- gradient path (collective.hpp) --------------------------------------
int ref_local_accumulate(const std::uint8_t* codes, const float* scales,
                         std::size_t n, std::uint32_t block, const float* local,
                         int precision, std::uint8_t* out_codes,
                         float* out_scales, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto main = make_q(codes, scales, n, 8, block, 2);
    const auto r = agq::local_accumulate(
        main, std::span<const float>(local, n),
        static_cast<agq::AccumulatePrecision>(precision));
    std::copy(r.codes.begin(), r.codes.end(), out_codes);
    std::copy(r.scales.begin(), r.scales.end(), out_scales);
  });
}

int ref_local_accumulate_mt(const std::uint8_t* codes, const float* scales,
                            std::size_t n, std::uint32_t block,
                            const float* local, int precision,
                            std::uint8_t* out_codes, float* out_scales,
                            int threads) {
  const std::size_t nb = (n + block - 1) / block;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  std::vector<int> status(threads, 0);
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const std::size_t b0 = nb * t / threads, b1 = nb * (t + 1) / threads;
      const std::size_t e0 = std::min(n, b0 * block), e1 = std::min(n, b1 * block);
      if (e0 >= e1) return;
      try {
        const auto main = make_q(codes + e0, scales + b0, e1 - e0, 8, block, 2);
        const auto r = agq::local_accumulate(
            main, std::span<const float>(local + e0, e1 - e0),
            static_cast<agq::AccumulatePrecision>(precision));
        std::copy(r.codes.begin(), r.codes.end(), out_codes + e0);
        std::copy(r.scales.begin(), r.scales.end(), out_scales + b0);
      } catch (...) {
        status[t] = 1;
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int s : status)
    if (s) return kInvalidArgument;
  return kOk;
}

int ref_chunk_assignment(std::size_t n, std::uint32_t block, int workers,
                         std::uint64_t* ranges /* 2*workers */, char* err,
                         std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto a = agq::ChunkAssignment::block_aligned(n, block, workers);
    for (int r = 0; r < workers; ++r) {
      ranges[2 * r] = a.ranges[r].first;
      ranges[2 * r + 1] = a.ranges[r].second;
    }
  });
}

namespace {
std::vector<agq::WorkerState> make_workers(int world, std::size_t n,
                                           std::uint32_t block,
                                           const std::uint8_t* const* codes,
                                           const float* const* scales) {
  std::vector<agq::WorkerState> w;
  for (int r = 0; r < world; ++r)
    w.push_back(agq::WorkerState::make(
        r, world, make_q(codes[r], scales[r], n, 8, block, 2)));
  return w;
}
}  // namespace

// protocol: 0 decomposed, 1 naive. Output is worker 0's tensor (all outputs
// are identical for the decomposed protocol; the naive one assigns the same
// gathered tensor to all). trace_out (optional, 6 u64 per event: phase
// (0 a2a / 1 all_gather / 2 reduce_scatter), sender, receiver, chunk_start,
// chunk_len, payload_bytes); *n_events receives the count.
int ref_allreduce(int protocol, int world, std::size_t n, std::uint32_t block,
                  const std::uint8_t* const* codes, const float* const* scales,
                  const int* schedule, std::uint8_t* out_codes,
                  float* out_scales, std::uint64_t* overflow_elements,
                  std::uint64_t* trace_out, std::size_t trace_cap,
                  std::size_t* n_events, int* outputs_identical, char* err,
                  std::size_t errlen) {
  return guarded(err, errlen, [&] {
    auto workers = make_workers(world, n, block, codes, scales);
    std::vector<int> sched;
    if (schedule) sched.assign(schedule, schedule + world);
    const auto res = protocol == 0 ? agq::allreduce_decomposed(workers, sched)
                                   : agq::allreduce_naive_fp8(workers, sched);
    const auto& o = res.outputs.at(0);
    std::copy(o.codes.begin(), o.codes.end(), out_codes);
    std::copy(o.scales.begin(), o.scales.end(), out_scales);
    if (overflow_elements) *overflow_elements = res.overflow_elements;
    int same = 1;
    for (const auto& x : res.outputs)
      if (x.codes != o.codes || x.scales != o.scales) same = 0;
    if (outputs_identical) *outputs_identical = same;
    if (n_events) *n_events = res.trace.events.size();
    if (trace_out) {
      std::size_t k = 0;
      for (const auto& e : res.trace.events) {
        if (k >= trace_cap) break;
        const std::uint64_t phase = e.phase == "all_to_all"  ? 0
                                    : e.phase == "all_gather" ? 1
                                                              : 2;
        const std::uint64_t row[6] = {phase, (std::uint64_t)e.sender,
                                      (std::uint64_t)e.receiver, e.chunk_start,
                                      e.chunk_len, e.payload_bytes};
        std::memcpy(trace_out + 6 * k, row, sizeof(row));
        ++k;
      }
    }
  });
}

int ref_allreduce_oracle(int world, std::size_t n, std::uint32_t block,
                         const std::uint8_t* const* codes,
                         const float* const* scales, float* out, char* err,
                         std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const auto workers = make_workers(world, n, block, codes, scales);
    const auto v = agq::allreduce_oracle(workers);
    std::copy(v.begin(), v.end(), out);
  });
}

}  // extern "C"
