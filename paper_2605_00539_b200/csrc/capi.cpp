// C ABI of libagq_cuda.so (include/agq_cuda.h): argument checks with the
// reference's exception texts, dispatch to the sm_100a kernels, host-buffer
// entry points for the C++ drop-in API, the DBCA bit-width planner.
#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "../../include/agq_cuda.h"

namespace agqh {
// kernels (act_codec.cu, grad_codec.cu, collective.cu)
agq_status quantize_device(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                           int codec, void* codes, int layout, float* scales, agq_errors* err,
                           cudaStream_t s);
agq_status dequantize_device(const void* codes, int layout, const float* scales, uint64_t n,
                             int bits, uint32_t block, int codec, void* out, int out_dtype,
                             int validate, agq_errors* err, cudaStream_t s);
agq_status quantize_grouped_device(const agq_segment* segs, int nseg, int x_dtype, int bits,
                                   int codec, agq_errors* err, cudaStream_t s);
agq_status dequantize_grouped_device(const agq_segment* segs, int nseg, int out_dtype, int bits,
                                     int codec, int validate, agq_errors* err, cudaStream_t s);
agq_status pack_device(const uint8_t* codes, uint64_t n, int bits, uint8_t* packed,
                       cudaStream_t s);
agq_status unpack_device(const uint8_t* packed, uint64_t n, int bits, uint8_t* codes,
                         cudaStream_t s);
agq_status accumulate_device(const uint8_t* codes, const float* scales, const void* local,
                             int local_dtype, uint64_t n, uint32_t block, int prec, uint8_t* oc,
                             float* os, agq_errors* err, cudaStream_t s);
agq_status reduce_requant_device(int np, const uint8_t* const* pc, const float* const* ps,
                                 uint64_t len, uint32_t block, int nout, uint8_t* const* oc,
                                 float* const* os, long long blk_base, agq_errors* err,
                                 cudaStream_t s);
agq_status naive_ring_device(int world, const uint8_t* const* codes, const float* const* scales,
                             uint64_t n, uint32_t block, const uint64_t* d_ranges, uint8_t* oc,
                             float* os, agq_errors* err, unsigned long long* events,
                             cudaStream_t s);
agq_status comm_unique_id(unsigned char id[128]);
agq_status comm_init(agq_comm** out, const unsigned char id[128], int nranks, int rank,
                     int device);
agq_status comm_p2p_export(agq_comm* c, uint64_t capacity, unsigned char handle[256]);
agq_status comm_p2p_open(agq_comm* c, const unsigned char* handles);
agq_status comm_p2p_buffers(agq_comm* c, uint8_t** codes, float** scales);
agq_status comm_destroy(agq_comm* c);
agq_status comm_set_timeout(agq_comm* c, double seconds);
agq_status comm_last_trace(agq_comm* c, agq_trace_event* events, int cap, int* count,
                           unsigned long long* moved);
int comm_rank(const agq_comm* c);
int comm_size(const agq_comm* c);
agq_status allreduce_naive(agq_comm* c, uint8_t* codes, float* scales, uint64_t n,
                           uint32_t block, agq_errors* err, unsigned long long* events,
                           cudaStream_t s);
agq_status allreduce_fp8(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                         int algo, agq_errors* err, cudaStream_t s);
agq_status allreduce_bf16_nccl(agq_comm* c, void* data, uint64_t n, cudaStream_t s);

namespace {
thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

agq_status set_error(agq_status st, const char* msg) {
  g_err = msg ? msg : "";
  return st;
}

agq_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return AGQ_OK;
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(AGQ_ERR_CUDA, m.c_str());
}

void chunk_ranges(uint64_t n, uint32_t block, int workers, uint64_t* ranges) {
  // collective.hpp:23-39 ChunkAssignment::block_aligned
  const uint64_t blocks = (n + block - 1) / block;
  uint64_t next = 0;
  for (int r = 0; r < workers; ++r) {
    const uint64_t share = blocks / workers + ((uint64_t)r < blocks % workers ? 1 : 0);
    const uint64_t begin = std::min<uint64_t>(n, next * block);
    next += share;
    const uint64_t end = std::min<uint64_t>(n, next * block);
    ranges[2 * r] = begin;
    ranges[2 * r + 1] = end;
  }
}

namespace {

agq_status check_args(int bits, uint32_t block, int codec) {
  // quantize.hpp:64-74
  if (bits < 4 || bits > 8) {
    std::string m = "bit_width must be in [4, 8], got " + std::to_string(bits);
    return set_error(AGQ_ERR_INVALID_ARGUMENT, m.c_str());
  }
  if (block == 0) return set_error(AGQ_ERR_INVALID_ARGUMENT, "block_size must be >= 1");
  if (codec == AGQ_CODEC_FP8_E4M3 && bits != 8)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "fp8_e4m3 requires bit_width 8");
  if (codec == AGQ_CODEC_FP4_E2M1 && bits != 4)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "fp4_e2m1 requires bit_width 4");
  if (codec < 0 || codec > 2) return set_error(AGQ_ERR_INVALID_ARGUMENT, "unknown codec kind");
  return AGQ_OK;
}

agq_status check_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "no CUDA device (the AGoQ kernels have no CPU path)");
  return AGQ_OK;
}

// Per-device cached workspace for the host entry points.
struct Workspace {
  std::mutex mu;
  void* dev = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
};
Workspace g_ws[64];

Workspace& workspace() {
  int dev = 0;
  cudaGetDevice(&dev);
  return g_ws[dev & 63];
}

agq_status ws_reserve(Workspace& w, size_t bytes) {
  if (!w.stream) {
    cudaError_t e = cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "workspace stream");
  }
  if (w.bytes >= bytes) return AGQ_OK;
  if (w.dev) cudaFree(w.dev);
  w.dev = nullptr;
  w.bytes = 0;
  cudaError_t e = cudaMalloc(&w.dev, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "workspace");
  w.bytes = bytes;
  return AGQ_OK;
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

agq_errors none_errors() {
  agq_errors e;
  e.nonfinite_block = LLONG_MAX;
  e.bad_scale_block = LLONG_MAX;
  e.bad_code_index = LLONG_MAX;
  e.nonfinite_local = LLONG_MAX;
  e.overflow_block = LLONG_MAX;
  e.saturated = 0;
  return e;
}

}  // namespace
}  // namespace agqh

using namespace agqh;

extern "C" {

const char* agq_version(void) { return "agoq-b200 0.1 (sm_100a)"; }
const char* agq_last_error(void) { return g_err.c_str(); }
unsigned long long agq_launch_count(void) { return g_launches.load(); }

int agq_device_ok(void) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

agq_status agq_errors_reset(agq_errors* d_err, agq_stream_t stream) {
  if (!d_err) return AGQ_OK;
  static const agq_errors none = none_errors();
  return cuda_fail(cudaMemcpyAsync(d_err, &none, sizeof(none), cudaMemcpyHostToDevice,
                                   (cudaStream_t)stream),
                   "errors_reset");
}

agq_status agq_errors_message(const agq_errors* h, int op, char* msg, size_t msglen) {
  std::string m;
  agq_status st = AGQ_OK;
  auto inv = [&](const std::string& s) { st = AGQ_ERR_INVALID_ARGUMENT; m = s; };
  auto rt = [&](const std::string& s) { st = AGQ_ERR_RUNTIME; m = s; };
  switch (op) {
    case AGQ_OP_QUANTIZE:
      if (h->nonfinite_block != LLONG_MAX)
        inv("non-finite input element in block " + std::to_string(h->nonfinite_block));
      break;
    case AGQ_OP_DEQUANTIZE:
      if (h->bad_code_index != LLONG_MAX)
        inv("quantized tensor: code out of range at " + std::to_string(h->bad_code_index));
      else if (h->bad_scale_block != LLONG_MAX)
        inv("quantized tensor: bad scale at block " + std::to_string(h->bad_scale_block));
      break;
    case AGQ_OP_ACCUMULATE:
      if (h->bad_scale_block != LLONG_MAX)
        inv("quantized tensor: bad scale at block " + std::to_string(h->bad_scale_block));
      else if (h->nonfinite_local != LLONG_MAX)
        inv("non-finite local gradient element");
      else if (h->nonfinite_block != LLONG_MAX)
        inv("non-finite input element in block " + std::to_string(h->nonfinite_block));
      break;
    case AGQ_OP_ALLREDUCE:
      // key = (sender << 40) | block: the lowest sender's lowest bad block
      if (h->bad_scale_block != LLONG_MAX)
        inv("quantized tensor: bad scale at block " +
            std::to_string(h->bad_scale_block & ((1LL << 40) - 1)));
      else if (h->overflow_block == -1)
        rt("all-reduce aborted: peer did not arrive (timeout)");
      else if (h->overflow_block != LLONG_MAX)
        rt("all-reduce aborted: fp32 overflow during local reduce");
      break;
    default:
      break;
  }
  if (msg && msglen) {
    std::strncpy(msg, m.c_str(), msglen - 1);
    msg[msglen - 1] = 0;
  }
  if (st) set_error(st, m.c_str());
  return st;
}

uint64_t agq_num_blocks(uint64_t n, uint32_t block) { return block ? (n + block - 1) / block : 0; }
uint64_t agq_packed_bytes(uint64_t n, int bits) { return (n * (uint64_t)bits + 7) / 8; }

agq_status agq_check_codec_args(int bits, uint32_t block, int codec) {
  return check_args(bits, block, codec);
}

agq_status agq_quantize(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                        int codec, void* codes, int layout, float* scales, agq_errors* d_err,
                        agq_stream_t stream) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  return quantize_device(x, x_dtype, n, bits, block, codec, codes, layout, scales, d_err,
                         (cudaStream_t)stream);
}

agq_status agq_dequantize(const void* codes, int layout, const float* scales, uint64_t n,
                          int bits, uint32_t block, int codec, void* out, int out_dtype,
                          int validate, agq_errors* d_err, agq_stream_t stream) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (validate && !d_err)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "validate needs an error record");
  return dequantize_device(codes, layout, scales, n, bits, block, codec, out, out_dtype,
                           validate, d_err, (cudaStream_t)stream);
}

agq_status agq_quantize_grouped(const agq_segment* segs, int nseg, int x_dtype, int bits,
                                int codec, agq_errors* d_err, agq_stream_t stream) {
  if (agq_status st = check_args(bits, 128, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (nseg < 0) return set_error(AGQ_ERR_INVALID_ARGUMENT, "negative segment count");
  return quantize_grouped_device(segs, nseg, x_dtype, bits, codec, d_err, (cudaStream_t)stream);
}

agq_status agq_dequantize_grouped(const agq_segment* segs, int nseg, int out_dtype, int bits,
                                  int codec, int validate, agq_errors* d_err,
                                  agq_stream_t stream) {
  if (agq_status st = check_args(bits, 128, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (nseg < 0) return set_error(AGQ_ERR_INVALID_ARGUMENT, "negative segment count");
  if (validate && !d_err)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "validate needs an error record");
  return dequantize_grouped_device(segs, nseg, out_dtype, bits, codec, validate, d_err,
                                   (cudaStream_t)stream);
}

agq_status agq_pack_codes(const uint8_t* codes, uint64_t n, int bits, uint8_t* packed,
                          agq_stream_t stream) {
  if (agq_status st = check_args(bits, 128, 0)) return st;
  return pack_device(codes, n, bits, packed, (cudaStream_t)stream);
}

agq_status agq_unpack_codes(const uint8_t* packed, uint64_t n, int bits, uint8_t* codes,
                            agq_stream_t stream) {
  if (agq_status st = check_args(bits, 128, 0)) return st;
  return unpack_device(packed, n, bits, codes, (cudaStream_t)stream);
}

agq_status agq_fp8_accumulate(const uint8_t* codes, const float* scales, const void* local,
                              int local_dtype, uint64_t n, uint32_t block, int precision,
                              uint8_t* out_codes, float* out_scales, agq_errors* d_err,
                              agq_stream_t stream) {
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (!d_err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "accumulate needs an error record");
  return accumulate_device(codes, scales, local, local_dtype, n, block, precision, out_codes,
                           out_scales, d_err, (cudaStream_t)stream);
}

agq_status agq_fp8_reduce_requant(int npieces, const uint8_t* const* piece_codes,
                                  const float* const* piece_scales, uint64_t len,
                                  uint32_t block, int nout, uint8_t* const* out_codes,
                                  float* const* out_scales, agq_errors* d_err,
                                  agq_stream_t stream) {
  if (npieces < 1 || npieces > AGQ_MAX_WORLD || nout < 1 || nout > AGQ_MAX_WORLD)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "piece/output count out of range");
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (!d_err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "reduce needs an error record");
  return reduce_requant_device(npieces, piece_codes, piece_scales, len, block, nout, out_codes,
                               out_scales, 0, d_err, (cudaStream_t)stream);
}

agq_status agq_chunk_assignment(uint64_t n, uint32_t block, int workers, uint64_t* ranges) {
  if (workers < 1) return set_error(AGQ_ERR_INVALID_ARGUMENT, "need at least one worker");
  if (block == 0) return set_error(AGQ_ERR_INVALID_ARGUMENT, "block_size must be >= 1");
  chunk_ranges(n, block, workers, ranges);
  return AGQ_OK;
}

agq_status agq_allreduce_simulated(int world, const uint8_t* const* codes,
                                   const float* const* scales, uint64_t n, uint32_t block,
                                   uint8_t* out_codes, float* out_scales, agq_errors* d_err,
                                   agq_stream_t stream) {
  if (world < 1) return set_error(AGQ_ERR_INVALID_ARGUMENT, "no workers");
  // Results do not depend on the chunk partition (per-block reduction in
  // ascending sender rank), so one reduce over the whole tensor reproduces
  // every owner's chunk at once.
  return agq_fp8_reduce_requant(world, codes, scales, n, block, 1, &out_codes, &out_scales,
                                d_err, stream);
}

agq_status agq_allreduce_naive_simulated(int world, const uint8_t* const* codes,
                                         const float* const* scales, uint64_t n, uint32_t block,
                                         uint8_t* out_codes, float* out_scales,
                                         agq_errors* d_err, unsigned long long* d_events,
                                         agq_stream_t stream) {
  if (world < 1 || world > AGQ_MAX_WORLD) return set_error(AGQ_ERR_INVALID_ARGUMENT, "no workers");
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (!d_err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "naive protocol needs an error record");
  std::vector<uint64_t> rg(2 * world);
  chunk_ranges(n, block, world, rg.data());
  uint64_t* d_rg = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMallocAsync(&d_rg, rg.size() * 8, s);
  if (e != cudaSuccess) return cuda_fail(e, "naive: ranges");
  cudaMemcpyAsync(d_rg, rg.data(), rg.size() * 8, cudaMemcpyHostToDevice, s);
  agq_status st = naive_ring_device(world, codes, scales, n, block, d_rg, out_codes, out_scales,
                                    d_err, d_events, s);
  cudaFreeAsync(d_rg, s);
  // the host copy above must outlive the async copy
  cudaStreamSynchronize(s);
  return st;
}

// ---- multi-GPU ------------------------------------------------------------
agq_status agq_comm_unique_id(unsigned char id[128]) { return comm_unique_id(id); }
agq_status agq_comm_init(agq_comm** comm, const unsigned char id[128], int nranks, int rank,
                         int device) {
  return comm_init(comm, id, nranks, rank, device);
}
agq_status agq_comm_p2p_export(agq_comm* comm, uint64_t capacity, unsigned char handle[256]) {
  return comm_p2p_export(comm, capacity, handle);
}
agq_status agq_comm_p2p_open(agq_comm* comm, const unsigned char* handles) {
  return comm_p2p_open(comm, handles);
}
agq_status agq_comm_p2p_buffers(agq_comm* comm, uint8_t** codes, float** scales) {
  return comm_p2p_buffers(comm, codes, scales);
}
agq_status agq_comm_destroy(agq_comm* comm) { return comm_destroy(comm); }
int agq_comm_rank(const agq_comm* comm) { return comm_rank(comm); }
agq_status agq_comm_set_timeout(agq_comm* comm, double seconds) {
  if (!comm) return set_error(AGQ_ERR_INVALID_ARGUMENT, "null communicator");
  return comm_set_timeout(comm, seconds);
}
agq_status agq_comm_last_trace(agq_comm* comm, agq_trace_event* events, int cap, int* count,
                               unsigned long long* moved) {
  if (!comm || !count) return set_error(AGQ_ERR_INVALID_ARGUMENT, "null communicator");
  return comm_last_trace(comm, events, cap, count, moved);
}
int agq_comm_size(const agq_comm* comm) { return comm_size(comm); }

agq_status agq_allreduce_fp8(agq_comm* comm, uint8_t* codes, float* scales, uint64_t n,
                             uint32_t block, int algo, agq_errors* d_err, agq_stream_t stream) {
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  return allreduce_fp8(comm, codes, scales, n, block, algo, d_err, (cudaStream_t)stream);
}

agq_status agq_allreduce_naive_fp8(agq_comm* comm, uint8_t* codes, float* scales, uint64_t n,
                                   uint32_t block, agq_errors* d_err,
                                   unsigned long long* d_events, agq_stream_t stream) {
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (!d_err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "naive protocol needs an error record");
  return allreduce_naive(comm, codes, scales, n, block, d_err, d_events, (cudaStream_t)stream);
}

agq_status agq_allreduce_bf16_nccl(agq_comm* comm, void* data, uint64_t n, agq_stream_t stream) {
  return allreduce_bf16_nccl(comm, data, n, (cudaStream_t)stream);
}

// ---- host entry points --------------------------------------------------------
agq_status agq_quantize_host(const float* x, uint64_t n, int bits, uint32_t block, int codec,
                             uint8_t* codes, float* scales) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  Workspace& w = workspace();
  std::lock_guard<std::mutex> lk(w.mu);
  const uint64_t nb = (n + block - 1) / block;
  const size_t ox = 0, oc = al(n * 4), os = oc + al(n), oe = os + al(nb * 4);
  if (agq_status st = ws_reserve(w, oe + al(sizeof(agq_errors)))) return st;
  char* base = static_cast<char*>(w.dev);
  agq_errors* d_err = reinterpret_cast<agq_errors*>(base + oe);
  cudaStream_t s = w.stream;
  cudaMemcpyAsync(base + ox, x, n * 4, cudaMemcpyHostToDevice, s);
  agq_errors_reset(d_err, (agq_stream_t)s);
  agq_status st = quantize_device(base + ox, AGQ_F32, n, bits, block, codec, base + oc,
                                  AGQ_CODES_BYTES, reinterpret_cast<float*>(base + os), d_err, s);
  if (st) return st;
  agq_errors h;
  cudaMemcpyAsync(codes, base + oc, n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(scales, base + os, nb * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (agq_status e = cuda_fail(cudaStreamSynchronize(s), "quantize_host")) return e;
  return agq_errors_message(&h, AGQ_OP_QUANTIZE, nullptr, 0);
}

agq_status agq_dequantize_host(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                               uint32_t block, int codec, float* out) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  Workspace& w = workspace();
  std::lock_guard<std::mutex> lk(w.mu);
  const uint64_t nb = (n + block - 1) / block;
  const size_t oc = 0, os = al(n), oo = os + al(nb * 4), oe = oo + al(n * 4);
  if (agq_status st = ws_reserve(w, oe + al(sizeof(agq_errors)))) return st;
  char* base = static_cast<char*>(w.dev);
  agq_errors* d_err = reinterpret_cast<agq_errors*>(base + oe);
  cudaStream_t s = w.stream;
  cudaMemcpyAsync(base + oc, codes, n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(base + os, scales, nb * 4, cudaMemcpyHostToDevice, s);
  agq_errors_reset(d_err, (agq_stream_t)s);
  agq_status st = dequantize_device(base + oc, AGQ_CODES_BYTES, reinterpret_cast<float*>(base + os),
                                    n, bits, block, codec, base + oo, AGQ_F32, 1, d_err, s);
  if (st) return st;
  agq_errors h;
  cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (agq_status e = cuda_fail(cudaStreamSynchronize(s), "dequantize_host")) return e;
  if (agq_status e = agq_errors_message(&h, AGQ_OP_DEQUANTIZE, nullptr, 0)) return e;
  cudaMemcpyAsync(out, base + oo, n * 4, cudaMemcpyDeviceToHost, s);
  return cuda_fail(cudaStreamSynchronize(s), "dequantize_host");
}

agq_status agq_local_accumulate_host(const uint8_t* codes, const float* scales, uint64_t n,
                                     uint32_t block, const float* local, int precision,
                                     uint8_t* out_codes, float* out_scales) {
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  Workspace& w = workspace();
  std::lock_guard<std::mutex> lk(w.mu);
  const uint64_t nb = (n + block - 1) / block;
  const size_t oc = 0, os = al(n), ol = os + al(nb * 4), oe = ol + al(n * 4);
  if (agq_status st = ws_reserve(w, oe + al(sizeof(agq_errors)))) return st;
  char* base = static_cast<char*>(w.dev);
  agq_errors* d_err = reinterpret_cast<agq_errors*>(base + oe);
  cudaStream_t s = w.stream;
  cudaMemcpyAsync(base + oc, codes, n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(base + os, scales, nb * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(base + ol, local, n * 4, cudaMemcpyHostToDevice, s);
  agq_errors_reset(d_err, (agq_stream_t)s);
  agq_status st = accumulate_device(reinterpret_cast<uint8_t*>(base + oc),
                                    reinterpret_cast<float*>(base + os), base + ol, AGQ_F32, n,
                                    block, precision, reinterpret_cast<uint8_t*>(base + oc),
                                    reinterpret_cast<float*>(base + os), d_err, s);
  if (st) return st;
  agq_errors h;
  cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (agq_status e = cuda_fail(cudaStreamSynchronize(s), "local_accumulate_host")) return e;
  if (agq_status e = agq_errors_message(&h, AGQ_OP_ACCUMULATE, nullptr, 0)) return e;
  cudaMemcpyAsync(out_codes, base + oc, n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(out_scales, base + os, nb * 4, cudaMemcpyDeviceToHost, s);
  return cuda_fail(cudaStreamSynchronize(s), "local_accumulate_host");
}

agq_status agq_allreduce_simulated_host(int world, const uint8_t* const* codes,
                                        const float* const* scales, uint64_t n, uint32_t block,
                                        int protocol, uint8_t* out_codes, float* out_scales,
                                        uint64_t* overflow_elements, uint64_t* overflow_events) {
  if (world < 1 || world > AGQ_MAX_WORLD) return set_error(AGQ_ERR_INVALID_ARGUMENT, "no workers");
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (overflow_elements) *overflow_elements = 0;
  if (overflow_events)
    for (int r = 0; r < world; ++r) overflow_events[r] = 0;
  if (n == 0) return AGQ_OK;
  Workspace& w = workspace();
  std::lock_guard<std::mutex> lk(w.mu);
  const uint64_t nb = (n + block - 1) / block;
  const size_t per = al(n) + al(nb * 4);
  const size_t oo = per * world, oe = oo + per, ov = oe + al(sizeof(agq_errors));
  if (agq_status st = ws_reserve(w, ov + al(8 * world))) return st;
  char* base = static_cast<char*>(w.dev);
  cudaStream_t s = w.stream;
  std::vector<const uint8_t*> dc(world);
  std::vector<const float*> ds(world);
  for (int r = 0; r < world; ++r) {
    char* p = base + per * r;
    cudaMemcpyAsync(p, codes[r], n, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p + al(n), scales[r], nb * 4, cudaMemcpyHostToDevice, s);
    dc[r] = reinterpret_cast<uint8_t*>(p);
    ds[r] = reinterpret_cast<float*>(p + al(n));
  }
  agq_errors* d_err = reinterpret_cast<agq_errors*>(base + oe);
  unsigned long long* d_ev = reinterpret_cast<unsigned long long*>(base + ov);
  agq_errors_reset(d_err, (agq_stream_t)s);
  cudaMemsetAsync(d_ev, 0, 8 * world, s);
  uint8_t* ocd = reinterpret_cast<uint8_t*>(base + oo);
  float* osd = reinterpret_cast<float*>(base + oo + al(n));
  agq_status st = protocol == 0
                      ? agq_allreduce_simulated(world, dc.data(), ds.data(), n, block, ocd, osd,
                                                d_err, (agq_stream_t)s)
                      : agq_allreduce_naive_simulated(world, dc.data(), ds.data(), n, block, ocd,
                                                      osd, d_err, d_ev, (agq_stream_t)s);
  if (st) return st;
  agq_errors h;
  cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (agq_status e = cuda_fail(cudaStreamSynchronize(s), "allreduce_host")) return e;
  if (agq_status e = agq_errors_message(&h, AGQ_OP_ALLREDUCE, nullptr, 0)) return e;
  if (overflow_elements) *overflow_elements = h.saturated;
  if (overflow_events)
    cudaMemcpyAsync(overflow_events, d_ev, 8 * world, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(out_codes, ocd, n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(out_scales, osd, nb * 4, cudaMemcpyDeviceToHost, s);
  return cuda_fail(cudaStreamSynchronize(s), "allreduce_host");
}

// ---- synthetic inputs (host) ----------------------------------------------------
// tools/agq.cpp:47-65 InputSpec::materialize with rng.hpp:9-28 make_rng: the
// same libstdc++ engine and distributions, hence the same bytes as the
// reference CLI for (seed, stream 0x1D, index 0).
agq_status agq_fill_input(uint64_t seed, uint64_t stream, uint64_t index, int kind, double a,
                          double b, int out_dtype, void* out, uint64_t n) {
  if (kind < AGQ_INPUT_NORMAL || kind > AGQ_INPUT_CONST)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "unknown input kind");
  if (out_dtype != AGQ_F32 && out_dtype != AGQ_BF16)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "output dtype must be F32 or BF16");
  if (kind == AGQ_INPUT_UNIFORM && !(a <= b))
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "--uniform needs a <= b");
  if (n && !out) return set_error(AGQ_ERR_INVALID_ARGUMENT, "null output");
  auto mix = [](uint64_t z) {  // rng.hpp:10-15 splitmix64
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  std::mt19937_64 rng(mix(mix(seed ^ (stream * 0xd1342543de82ef95ULL)) + index));  // :19-28
  auto put = [&](uint64_t i, float x) {
    if (out_dtype == AGQ_F32) {
      static_cast<float*>(out)[i] = x;
    } else {  // round to nearest even (BF16-valued configs)
      uint32_t u;
      std::memcpy(&u, &x, 4);
      if ((u & 0x7fffffffu) > 0x7f800000u) u |= 0x00400000u;
      else u += 0x7fffu + ((u >> 16) & 1u);
      static_cast<uint16_t*>(out)[i] = (uint16_t)(u >> 16);
    }
  };
  if (kind == AGQ_INPUT_CONST) {
    for (uint64_t i = 0; i < n; ++i) put(i, static_cast<float>(a));
  } else if (kind == AGQ_INPUT_UNIFORM) {
    std::uniform_real_distribution<float> u(static_cast<float>(a), static_cast<float>(b));
    for (uint64_t i = 0; i < n; ++i) put(i, u(rng));
  } else {
    std::normal_distribution<float> g(static_cast<float>(a), static_cast<float>(b));
    for (uint64_t i = 0; i < n; ++i) put(i, g(rng));
  }
  return AGQ_OK;
}

// ---- DBCA control plane (dbca.hpp) ----------------------------------------------
agq_status agq_stored_activation_counts(int n_stages, int micro_batches, int interleave,
                                        int* counts) {
  // dbca.hpp:17-29 PipelineConfig::check, :34-41
  if (n_stages < 1) return set_error(AGQ_ERR_INVALID_ARGUMENT, "n_stages must be >= 1");
  if (micro_batches < 1) return set_error(AGQ_ERR_INVALID_ARGUMENT, "micro_batches must be >= 1");
  if (interleave != 2)
    return set_error(AGQ_ERR_INVALID_ARGUMENT,
                     "stored-activation counts are modeled for interleave factor 2");
  if (n_stages > 1 && micro_batches < 2 * n_stages)
    return set_error(AGQ_ERR_INVALID_ARGUMENT,
                     "steady-state counts need micro_batches >= 2 * n_stages");
  if (n_stages == 1) {
    counts[0] = 1;
    return AGQ_OK;
  }
  for (int d = 1; d <= n_stages; ++d) counts[d - 1] = 3 * n_stages - 2 * d + 1;
  return AGQ_OK;
}

agq_status agq_plan_bit_widths(int n_stages, int micro_batches, int interleave, int* counts,
                               double* raw_bits, int* assigned_bits) {
  // dbca.hpp:63-78: B_i = 4 N_max / N_i, lround, clamp [4, 8]
  if (agq_status st = agq_stored_activation_counts(n_stages, micro_batches, interleave, counts))
    return st;
  const int n_max = counts[0];
  for (int i = 0; i < n_stages; ++i) {
    raw_bits[i] = 4.0 * n_max / counts[i];
    const long r = std::lround(raw_bits[i]);
    assigned_bits[i] = (int)(r < 4 ? 4 : (r > 8 ? 8 : r));
  }
  return AGQ_OK;
}

}  // extern "C"
