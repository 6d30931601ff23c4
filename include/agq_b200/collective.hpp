// Drop-in for agq/collective.hpp: FP8 gradient accumulation and the simulated
// data-parallel all-reduce protocols with the reference's API
// (/root/reference/proj/include/agq/collective.hpp:20-467). The arithmetic
// (dequantize, fp32 reduce in ascending sender rank, fresh-scale requantize;
// the naive FP8 ring) runs on the GPU through the C ABI; the message trace is
// the protocol's deterministic schedule, built on the host.
//
// For real ranks (one process per GPU) use agq_allreduce_fp8 (include/agq_cuda.h).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "quantize.hpp"

namespace agq {

struct ChunkAssignment {
  std::vector<std::pair<std::size_t, std::size_t>> ranges;

  static ChunkAssignment block_aligned(std::size_t n, std::uint32_t block, int workers) {
    if (workers < 1) throw std::invalid_argument("need at least one worker");
    std::vector<std::uint64_t> r(2 * static_cast<std::size_t>(workers));
    detail::throw_status(agq_chunk_assignment(n, block, workers, r.data()));
    ChunkAssignment a;
    for (int w = 0; w < workers; ++w) a.ranges.emplace_back(r[2 * w], r[2 * w + 1]);
    return a;
  }
};

struct Message {
  std::string phase;
  int sender = 0;
  std::size_t chunk_start = 0;
  std::vector<std::uint8_t> codes;
  std::vector<float> scales;
};

struct TraceEvent {
  std::string phase;
  int sender = 0;
  int receiver = 0;
  std::size_t chunk_start = 0;
  std::size_t chunk_len = 0;
  std::size_t payload_bytes = 0;
};

struct MessageTrace {
  std::vector<TraceEvent> events;

  std::size_t total_bytes() const {
    std::size_t t = 0;
    for (const auto& e : events) t += e.payload_bytes;
    return t;
  }

  void write_jsonl(std::ostream& os) const {  // one object per line, same keys
    for (const auto& e : events)
      os << "{\"chunk_len\":" << e.chunk_len << ",\"chunk_start\":" << e.chunk_start
         << ",\"payload_bytes\":" << e.payload_bytes << ",\"phase\":\"" << e.phase
         << "\",\"receiver\":" << e.receiver << ",\"sender\":" << e.sender << "}\n";
  }
};

struct WorkerState {
  int rank = 0;
  QuantizedTensor main_gradient;
  std::vector<std::deque<Message>> inbox;
  std::uint64_t overflow_events = 0;

  static WorkerState make(int rank, int world, const QuantizedTensor& gradient) {
    if (gradient.codec_kind != CodecKind::Fp8E4M3)
      throw std::invalid_argument("worker gradients are FP8 E4M3 tensors");
    WorkerState w;
    w.rank = rank;
    w.main_gradient = gradient;
    w.inbox.resize(world);
    return w;
  }
};

enum class AccumulatePrecision { Fp32 = AGQ_ACC_FP32, Bf16 = AGQ_ACC_BF16, Fp16 = AGQ_ACC_FP16 };

// Round to bf16 with ties to even on the fp32 bit pattern.
inline float round_bf16(float x) {
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Round to fp16 with ties to even; saturates at |x| >= 65520 to +-65504.
inline float round_fp16(float x) {
  if (x == 0.0f || !std::isfinite(x)) return x;
  const double m = std::fabs(static_cast<double>(x));
  const double sgn = x < 0.0f ? -1.0 : 1.0;
  if (m >= 65520.0) return static_cast<float>(sgn * 65504.0);
  const int e = m < 0x1p-14 ? -14 : std::ilogb(m);
  return static_cast<float>(sgn * std::ldexp(std::nearbyint(std::ldexp(m, 10 - e)), e - 10));
}

inline QuantizedTensor local_accumulate(const QuantizedTensor& main,
                                        std::span<const float> local_grad,
                                        AccumulatePrecision precision = AccumulatePrecision::Fp32) {
  if (main.codec_kind != CodecKind::Fp8E4M3)
    throw std::invalid_argument("main gradient must be FP8 E4M3");
  if (main.num_elements() != local_grad.size())
    throw std::invalid_argument("local gradient shape mismatch");
  detail::validate_structure(main);  // dequantize_blockwise(main) validates first
  // the transfers and kernels run while the result is built
  detail::HostJob job;
  detail::throw_status(agq_local_accumulate_host_begin(
      main.codes.data(), main.scales.data(), main.num_elements(), main.block_size,
      local_grad.data(), static_cast<int>(precision), job.out()));
  QuantizedTensor out;
  out.bit_width = main.bit_width;
  out.block_size = main.block_size;
  out.codec_kind = main.codec_kind;
  out.shape = main.shape;
  out.codes.resize(main.codes.size());
  out.scales.resize(main.scales.size());
  if (job)
    job.finish(out.codes.data(), out.scales.data());
  else
    detail::throw_status(agq_local_accumulate_host(main.codes.data(), main.scales.data(),
                                                   main.num_elements(), main.block_size,
                                                   local_grad.data(), static_cast<int>(precision),
                                                   out.codes.data(), out.scales.data()));
  return out;
}

struct CollectiveResult {
  std::vector<QuantizedTensor> outputs;
  MessageTrace trace;
  std::vector<std::uint64_t> overflow_events;
  std::uint64_t overflow_elements = 0;
};

namespace detail {

inline void check_workers(const std::vector<WorkerState>& workers) {
  if (workers.empty()) throw std::invalid_argument("no workers");
  const auto& shape = workers.front().main_gradient.shape;
  const auto block = workers.front().main_gradient.block_size;
  for (const auto& w : workers) {
    if (w.main_gradient.shape != shape || w.main_gradient.block_size != block)
      throw std::invalid_argument("all-reduce aborted: main gradient shapes must match");
    validate(w.main_gradient);
  }
}

inline void check_schedule(const std::vector<int>& schedule, int world) {
  if (!schedule.empty() && static_cast<int>(schedule.size()) != world)
    throw std::invalid_argument("schedule must permute all workers");
}

inline std::size_t payload(std::size_t begin, std::size_t end, std::uint32_t block) {
  return (end - begin) + 4 * ((end + block - 1) / block - begin / block);
}

inline CollectiveResult run_simulated(std::vector<WorkerState>& workers, int protocol) {
  check_workers(workers);
  const int world = static_cast<int>(workers.size());
  const auto& proto = workers.front().main_gradient;
  std::vector<const std::uint8_t*> codes(world);
  std::vector<const float*> scales(world);
  for (int r = 0; r < world; ++r) {
    codes[r] = workers[r].main_gradient.codes.data();
    scales[r] = workers[r].main_gradient.scales.data();
  }
  QuantizedTensor out = proto;
  std::uint64_t overflow = 0;
  std::vector<std::uint64_t> events(world, 0);
  throw_status(agq_allreduce_simulated_host(world, codes.data(), scales.data(),
                                            proto.num_elements(), proto.block_size, protocol,
                                            out.codes.data(), out.scales.data(), &overflow,
                                            events.data()));
  CollectiveResult res;
  res.outputs.assign(world, out);
  res.overflow_elements = overflow;
  res.overflow_events = events;
  for (int r = 0; r < world; ++r) workers[r].overflow_events += events[r];
  return res;
}

}  // namespace detail

inline std::vector<float> allreduce_oracle(const std::vector<WorkerState>& workers) {
  detail::check_workers(workers);
  std::vector<float> acc(workers.front().main_gradient.num_elements(), 0.0f);
  for (const auto& w : workers) {
    const auto v = dequantize_blockwise(w.main_gradient);
    for (std::size_t i = 0; i < acc.size(); ++i) acc[i] += v[i];
  }
  return acc;
}

inline CollectiveResult allreduce_decomposed(std::vector<WorkerState>& workers,
                                             const std::vector<int>& schedule = {}) {
  detail::check_workers(workers);
  const int world = static_cast<int>(workers.size());
  detail::check_schedule(schedule, world);
  CollectiveResult res = detail::run_simulated(workers, 0);
  const auto& q = workers.front().main_gradient;
  const auto a = ChunkAssignment::block_aligned(q.num_elements(), q.block_size, world);
  for (int s = 0; s < world; ++s)  // all-to-all: chunk r of every sender to r
    for (int r = 0; r < world; ++r) {
      const auto [b, e] = a.ranges[r];
      if (r == s || b == e) continue;
      res.trace.events.push_back({"all_to_all", s, r, b, e - b, detail::payload(b, e, q.block_size)});
    }
  for (int s = 0; s < world; ++s) {  // all-gather of every reduced chunk
    const auto [b, e] = a.ranges[s];
    if (b == e) continue;
    for (int r = 0; r < world; ++r)
      if (r != s)
        res.trace.events.push_back({"all_gather", s, r, b, e - b, detail::payload(b, e, q.block_size)});
  }
  return res;
}

inline CollectiveResult allreduce_naive_fp8(std::vector<WorkerState>& workers,
                                            const std::vector<int>& schedule = {}) {
  detail::check_workers(workers);
  const int world = static_cast<int>(workers.size());
  detail::check_schedule(schedule, world);
  CollectiveResult res = detail::run_simulated(workers, 1);
  const auto& q = workers.front().main_gradient;
  const auto a = ChunkAssignment::block_aligned(q.num_elements(), q.block_size, world);
  for (int step = 0; step < world - 1; ++step)  // ring reduce-scatter
    for (int r = 0; r < world; ++r) {
      const auto [b, e] = a.ranges[((r - step) % world + world) % world];
      if (b == e) continue;
      res.trace.events.push_back({"reduce_scatter", r, (r + 1) % world, b, e - b,
                                  detail::payload(b, e, q.block_size)});
    }
  for (int chunk = 0; chunk < world; ++chunk) {
    const int owner = world == 1 ? 0 : (chunk - 1 + world) % world;
    const auto [b, e] = a.ranges[chunk];
    if (b == e) continue;
    for (int r = 0; r < world; ++r)
      if (r != owner)
        res.trace.events.push_back({"all_gather", owner, r, b, e - b,
                                    detail::payload(b, e, q.block_size)});
  }
  return res;
}

enum class Protocol { Decomposed, Naive, Oracle };

inline const char* protocol_name(Protocol p) {
  switch (p) {
    case Protocol::Decomposed: return "decomposed";
    case Protocol::Naive: return "naive";
    case Protocol::Oracle: return "oracle";
  }
  return "?";
}

struct ProtocolRun {
  CollectiveResult collective;
  std::vector<float> oracle_values;
  Protocol protocol = Protocol::Decomposed;
};

inline ProtocolRun run_protocol_trace(std::vector<WorkerState>& workers, Protocol protocol,
                                      const std::vector<int>& schedule = {}) {
  ProtocolRun run;
  run.protocol = protocol;
  if (protocol == Protocol::Decomposed) run.collective = allreduce_decomposed(workers, schedule);
  if (protocol == Protocol::Naive) run.collective = allreduce_naive_fp8(workers, schedule);
  if (protocol == Protocol::Oracle) run.oracle_values = allreduce_oracle(workers);
  return run;
}

}  // namespace agq
