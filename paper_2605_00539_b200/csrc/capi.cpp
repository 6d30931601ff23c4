// C ABI of libagq_cuda.so (include/agq_cuda.h): argument checks with the
// reference's exception texts, dispatch to the sm_100a kernels, host-buffer
// entry points for the C++ drop-in API, the DBCA bit-width planner.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
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
agq_status roundtrip_device(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                            int codec, void* codes, int layout, float* scales, void* out,
                            int out_dtype, agq_errors* err, cudaStream_t s);
agq_status dequantize_grouped_device(const agq_segment* segs, int nseg, int out_dtype, int bits,
                                     int codec, int validate, agq_errors* err, cudaStream_t s);
agq_status pack_device(const uint8_t* codes, uint64_t n, int bits, uint8_t* packed,
                       cudaStream_t s);
agq_status unpack_device(const uint8_t* packed, uint64_t n, int bits, uint8_t* codes,
                         cudaStream_t s);
agq_status accumulate_device(const uint8_t* codes, const float* scales, const void* local,
                             int local_dtype, uint64_t n, uint32_t block, int prec, uint8_t* oc,
                             float* os, agq_errors* err, cudaStream_t s, long long blk_base = 0);
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

agq_errors none_errors();
}  // namespace
const agq_errors kNoErrors = none_errors();
namespace {
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

namespace agqh {
__global__ void k_errors_reset(agq_errors* e, agq_errors none) {
  if (threadIdx.x == 0) *e = none;
}
void launch_errors_reset(agq_errors* e, cudaStream_t s) {
  static const agq_errors none = none_errors();
  k_errors_reset<<<1, 32, 0, s>>>(e, none);
  count_launch();
}
}  // namespace agqh

#ifdef AGQ_AR_PROFILE
namespace agqh {
agq_status ar_profile(unsigned long long* out);  // collective.cu, experiment builds
}
#endif
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
  // a kernel, not a pageable-host memcpy: capturable in a CUDA graph
  agqh::launch_errors_reset(d_err, (cudaStream_t)stream);
  return cuda_fail(cudaGetLastError(), "errors_reset");
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

agq_status agq_quantize_roundtrip(const void* x, int x_dtype, uint64_t n, int bits,
                                  uint32_t block, int codec, void* codes, int layout,
                                  float* scales, void* out, int out_dtype, agq_errors* d_err,
                                  agq_stream_t stream) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  return roundtrip_device(x, x_dtype, n, bits, block, codec, codes, layout, scales, out, out_dtype,
                          d_err, (cudaStream_t)stream);
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

#ifdef AGQ_AR_PROFILE
agq_status agq_ar_profile(unsigned long long* out) { return agqh::ar_profile(out); }
#endif
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
// The C++ drop-in surface (quantize.hpp:78-189, collective.hpp:128-147 over
// host std::vectors). Each call streams its tensor through a library-owned
// pipeline in block-aligned chunks: parallel host copies between the
// caller's (pageable) buffers and pinned bounce slots, H2D -> kernel -> D2H
// on one stream per slot, so the copy-in of chunk k+1, the kernels of chunk
// k and the copy-out of chunk k-1 overlap; one device error record per call
// (chunk errors carry their global block index) and one synchronisation at
// the end. Concurrent callers get separate pipelines.
}  // extern "C"

namespace agqh {
agq_status quantize_device_at(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                              int codec, void* codes, int layout, float* scales,
                              long long blk_base, agq_errors* err, cudaStream_t s);
agq_status dequantize_device_at(const void* codes, int layout, const float* scales, uint64_t n,
                                int bits, uint32_t block, int codec, void* out, int out_dtype,
                                int validate, long long blk_base, agq_errors* err,
                                cudaStream_t s);
namespace {

// Host copy of one piece. Non-temporal (streaming) stores where the CPU has
// AVX2: the destination is written without being read for ownership first
// (a third of the host memory traffic of a plain copy of a large buffer),
// which is what bounds the staging copies; sfence before the piece counts as
// done (the DMA that reads pinned staging, or the caller, comes after).
#if defined(__x86_64__)
__attribute__((target("avx2"))) void copy_stream_avx2(void* dst, const void* src, size_t n) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  const size_t nv = n / 128;
  for (size_t i = 0; i < nv; ++i, d += 128, s += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 96), e);
  }
  std::memcpy(d, s, n % 128);
  _mm_sfence();
}
bool has_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}
#endif
void copy_piece(void* dst, const void* src, size_t n) {
#if defined(__x86_64__)
  if (n >= (64u << 10) && has_avx2()) return copy_stream_avx2(dst, src, n);
#endif
  std::memcpy(dst, src, n);
}

// Persistent host copy threads: copy() splits a batch of memcpy jobs into
// >= 512 KB pieces, shares them with the workers (the caller works too) and
// returns when every piece is done. Each batch owns its counters, so a worker
// that wakes late can never touch another batch's pieces.
class CopyPool {
 public:
  struct Job {
    void* dst;
    const void* src;
    size_t bytes;
  };
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();  // never destroyed (threads detached)
    return *p;
  }
  void copy(const std::vector<Job>& jobs) {
    size_t total = 0;
    for (const Job& j : jobs) total += j.bytes;
    if (total == 0) return;
    auto b = std::make_shared<Batch>();
    const size_t piece = std::max<size_t>(kMinPiece, total / (4 * (nthreads_ + 1)) + 1);
    for (const Job& j : jobs)
      for (size_t o = 0; o < j.bytes; o += piece)
        b->pieces.push_back({static_cast<char*>(j.dst) + o, static_cast<const char*>(j.src) + o,
                             std::min(piece, j.bytes - o)});
    if (b->pieces.size() > 1 && nthreads_ > 0) {
      {
        std::lock_guard<std::mutex> lk(mu_);
        cur_ = b;
        gen_.fetch_add(1, std::memory_order_release);
      }
      if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
    }
    run(*b);
    while (b->done.load(std::memory_order_acquire) < b->pieces.size()) _mm_pause();
    std::lock_guard<std::mutex> lk(mu_);
    if (cur_ == b) cur_.reset();
  }
 private:
  struct Batch {
    std::vector<Job> pieces;
    std::atomic<size_t> next{0};
    std::atomic<size_t> done{0};
  };
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)std::min<unsigned>(7, hw > 2 ? hw / 2 : 1);
    for (int t = 0; t < nthreads_; ++t) std::thread([this] { loop(); }).detach();
  }
  static void run(Batch& b) {
    for (;;) {
      const size_t k = b.next.fetch_add(1, std::memory_order_relaxed);
      if (k >= b.pieces.size()) break;
      copy_piece(b.pieces[k].dst, b.pieces[k].src, b.pieces[k].bytes);
      b.done.fetch_add(1, std::memory_order_release);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin briefly for the next batch (a pipeline submits one per chunk),
      // then sleep
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                 std::chrono::steady_clock::now() - t0).count() < kSpinNs)
        for (int i = 0; i < 64; ++i) _mm_pause();
      std::shared_ptr<Batch> b;
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (gen_.load(std::memory_order_relaxed) == seen) {
          sleepers_.fetch_add(1, std::memory_order_acq_rel);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_relaxed) != seen; });
          sleepers_.fetch_sub(1, std::memory_order_acq_rel);
        }
        seen = gen_.load(std::memory_order_relaxed);
        b = cur_;
      }
      if (b) run(*b);
    }
  }
  // measured on the B200 box (profiles/r02_host_pipe_sweep.log): 512 KB
  // pieces balance a chunk's batch over the threads; 200 us of spinning
  // hides the wake-up latency between a pipeline's batches
  static constexpr size_t kMinPiece = 512u << 10;
  static constexpr uint64_t kSpinNs = 200000;
  int nthreads_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  std::shared_ptr<Batch> cur_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> sleepers_{0};
};

// One pipeline: kSlots slots of pinned + device staging, one stream each.
constexpr int kSlots = 4;
constexpr uint64_t kChunkElems = 2u << 20;  // 2M elements (8 MB of FP32) per chunk

struct HostPipe {
  int dev = -1;
  bool busy = false;
  cudaStream_t st[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  char* pin[kSlots] = {};
  char* dbuf[kSlots] = {};
  size_t cap = 0;
  agq_errors* d_err = nullptr;

  agq_status reserve(size_t bytes) {
    if (!st[0]) {
      for (int k = 0; k < kSlots; ++k) {
        cudaError_t e = cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "host pipeline: streams");
      }
      cudaError_t e = cudaMalloc(&d_err, sizeof(agq_errors));
      if (e != cudaSuccess) return cuda_fail(e, "host pipeline: error record");
    }
    if (cap >= bytes) return AGQ_OK;
    for (int k = 0; k < kSlots; ++k) {
      if (pin[k]) cudaFreeHost(pin[k]);
      if (dbuf[k]) cudaFree(dbuf[k]);
      pin[k] = dbuf[k] = nullptr;
    }
    cap = 0;
    for (int k = 0; k < kSlots; ++k) {
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&pin[k]), bytes, cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&dbuf[k]), bytes);
      if (e != cudaSuccess) return cuda_fail(e, "host pipeline: staging");
    }
    cap = bytes;
    return AGQ_OK;
  }
  // begin/finish jobs: pinned staging for every chunk of the call (no slot
  // reuse on the host side, so nothing waits before finish) and one event
  // per chunk
  char* big = nullptr;
  size_t big_cap = 0;
  std::vector<cudaEvent_t> cev;
  agq_status reserve_job(size_t bytes, uint64_t chunks) {
    if (big_cap < bytes) {
      if (big) cudaFreeHost(big);
      big = nullptr;
      big_cap = 0;
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&big), bytes, cudaHostAllocDefault);
      if (e != cudaSuccess) return cuda_fail(e, "host pipeline: job staging");
      big_cap = bytes;
    }
    while (cev.size() < chunks) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return cuda_fail(r, "host pipeline: events");
      cev.push_back(e);
    }
    return AGQ_OK;
  }
};

std::mutex g_pipes_mu;
std::vector<HostPipe*> g_pipes;

// Cumulative host-side time of the pipelines (agq_host_pipeline_stats).
std::atomic<unsigned long long> g_ns_copy{0}, g_ns_wait{0}, g_ns_total{0}, g_calls{0};
unsigned long long now_ns() {
  return (unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct PipeLease {
  HostPipe* p = nullptr;
  PipeLease() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_pipes_mu);
    for (HostPipe* q : g_pipes)
      if (!q->busy && q->dev == dev) {
        p = q;
        break;
      }
    if (!p) {
      p = new HostPipe();
      p->dev = dev;
      g_pipes.push_back(p);
    }
    p->busy = true;
  }
  ~PipeLease() {
    std::lock_guard<std::mutex> lk(g_pipes_mu);
    p->busy = false;
  }
};

// One chunk's staging layout: `in` bytes copied host->device before the
// kernel, `out` bytes device->host after it, both inside one slot. Inputs
// carry the caller's pointer; outputs a byte offset into output `which`
// (0: codes or values, 1: scales), resolved when the outputs are known.
struct Part {
  size_t off;  // inside the slot
  size_t bytes;
  const char* host;  // input source
  int which;         // output index
  size_t rel;        // output byte offset
};
Part in_part(size_t off, size_t bytes, const void* src) {
  return {off, bytes, static_cast<const char*>(src), -1, 0};
}
Part out_part(size_t off, size_t bytes, int which, size_t rel) {
  return {off, bytes, nullptr, which, rel};
}

// One host entry point as chunks: plan(k, in, out) fills chunk k's parts,
// launch(k, dev_slot, stream, err) enqueues its kernels.
struct OpSpec {
  uint64_t chunks = 0;
  size_t slot = 0;
  int op = 0;
  std::function<void(uint64_t, std::vector<Part>&, std::vector<Part>&)> plan;
  std::function<agq_status(uint64_t, char*, cudaStream_t, agq_errors*)> launch;
};

agq_status reset_errors(HostPipe& p) {
  return cuda_fail(cudaMemcpy(p.d_err, &kNoErrors, sizeof(agq_errors), cudaMemcpyHostToDevice),
                   "host pipeline: reset");
}

// Run the op through the slot ring: the host copies of chunk k overlap the
// transfers and kernels of chunks k-3..k-1.
agq_status run_pipeline(HostPipe& p, const OpSpec& op, char* const* outs_base) {
  if (agq_status st = p.reserve(op.slot)) return st;
  if (agq_status st = reset_errors(p)) return st;
  std::vector<std::vector<Part>> outs(kSlots);
  CopyPool& pool = CopyPool::get();
  const unsigned long long t_start = now_ns();
  unsigned long long t_copy = 0, t_wait = 0;
  for (uint64_t k = 0; k < op.chunks + kSlots; ++k) {
    const int s = (int)(k % kSlots);
    std::vector<CopyPool::Job> jobs;
    // drain the slot: chunk k - kSlots finished -> copy its results out
    if (k >= kSlots) {
      const unsigned long long t0 = now_ns();
      if (agq_status st = cuda_fail(cudaEventSynchronize(p.ev[s]), "host pipeline")) return st;
      t_wait += now_ns() - t0;
      for (const Part& o : outs[s])
        jobs.push_back({outs_base[o.which] + o.rel, p.pin[s] + o.off, o.bytes});
      outs[s].clear();
    }
    std::vector<Part> in;
    if (k < op.chunks) {
      op.plan(k, in, outs[s]);
      for (const Part& i : in) jobs.push_back({p.pin[s] + i.off, i.host, i.bytes});
    }
    const unsigned long long t1 = now_ns();
    pool.copy(jobs);
    t_copy += now_ns() - t1;
    if (k >= op.chunks) continue;
    cudaStream_t st = p.st[s];
    for (const Part& i : in)
      cudaMemcpyAsync(p.dbuf[s] + i.off, p.pin[s] + i.off, i.bytes, cudaMemcpyHostToDevice, st);
    if (agq_status r = op.launch(k, p.dbuf[s], st, p.d_err)) {
      cudaDeviceSynchronize();
      return r;
    }
    for (const Part& o : outs[s])
      cudaMemcpyAsync(p.pin[s] + o.off, p.dbuf[s] + o.off, o.bytes, cudaMemcpyDeviceToHost, st);
    if (agq_status r = cuda_fail(cudaEventRecord(p.ev[s], st), "host pipeline")) return r;
  }
  g_ns_copy += t_copy;
  g_ns_wait += t_wait;
  g_ns_total += now_ns() - t_start;
  ++g_calls;
  return AGQ_OK;
}

// A begun host call (agq_*_host_begin): every chunk's inputs staged and its
// transfers and kernels enqueued; the outputs wait in pinned staging until
// agq_host_job_finish copies them to the caller. Holds its pipeline.
constexpr size_t kJobStagingCap = 256u << 20;  // larger calls run synchronously
constexpr size_t kJobAsyncMin = 1u << 20;      // smaller calls stage on the caller's thread
}  // namespace
}  // namespace agqh

struct agq_host_job {
  agqh::PipeLease lease;
  int op = 0;
  size_t slot = 0;
  std::vector<std::vector<agqh::Part>> outs;  // per chunk
  // the staging copies and enqueues run on this thread while the caller
  // builds its result buffers; its status (and message) are read at finish
  std::thread issuer;
  agq_status issue_status = AGQ_OK;
  std::string issue_error;
  ~agq_host_job() {
    if (issuer.joinable()) issuer.join();
  }
};

namespace agqh {
namespace {

// Issue all chunks of `op`; on success `job` owns the in-flight work.
// Staging buffers, events and the error record, on the calling thread.
agq_status job_prepare(agq_host_job& job, const OpSpec& op) {
  HostPipe& p = *job.lease.p;
  if (agq_status st = p.reserve(op.slot)) return st;
  if (agq_status st = p.reserve_job(op.slot * op.chunks, op.chunks)) return st;
  if (agq_status st = reset_errors(p)) return st;
  job.op = op.op;
  job.slot = op.slot;
  job.outs.assign(op.chunks, {});
  return AGQ_OK;
}

// Stage every chunk's inputs and enqueue its transfers and kernels (the
// issuer thread).
agq_status job_issue(agq_host_job& job, const OpSpec& op) {
  HostPipe& p = *job.lease.p;
  CopyPool& pool = CopyPool::get();
  for (uint64_t k = 0; k < op.chunks; ++k) {
    const int s = (int)(k % kSlots);  // device slot: reused in stream order
    char* h = p.big + k * op.slot;
    std::vector<Part> in;
    op.plan(k, in, job.outs[k]);
    std::vector<CopyPool::Job> jobs;
    for (const Part& i : in) jobs.push_back({h + i.off, i.host, i.bytes});
    pool.copy(jobs);
    cudaStream_t st = p.st[s];
    for (const Part& i : in)
      cudaMemcpyAsync(p.dbuf[s] + i.off, h + i.off, i.bytes, cudaMemcpyHostToDevice, st);
    if (agq_status r = op.launch(k, p.dbuf[s], st, p.d_err)) {
      cudaDeviceSynchronize();
      return r;
    }
    for (const Part& o : job.outs[k])
      cudaMemcpyAsync(h + o.off, p.dbuf[s] + o.off, o.bytes, cudaMemcpyDeviceToHost, st);
    if (agq_status r = cuda_fail(cudaEventRecord(p.cev[k], st), "host pipeline")) {
      cudaDeviceSynchronize();
      return r;
    }
  }
  return AGQ_OK;
}

// Copy the outputs out, one batch per run of finished chunks (normally all
// of them: the device work ran while the caller built its result buffers).
agq_status job_finish(agq_host_job& job, char* const* outs_base) {
  HostPipe& p = *job.lease.p;
  CopyPool& pool = CopyPool::get();
  const uint64_t K = job.outs.size();
  for (uint64_t k = 0; k < K;) {
    if (agq_status st = cuda_fail(cudaEventSynchronize(p.cev[k]), "host pipeline")) return st;
    uint64_t e = k + 1;
    while (e < K && cudaEventQuery(p.cev[e]) == cudaSuccess) ++e;
    std::vector<CopyPool::Job> jobs;
    for (; k < e; ++k)
      for (const Part& o : job.outs[k])
        jobs.push_back({outs_base[o.which] + o.rel, p.big + k * job.slot + o.off, o.bytes});
    pool.copy(jobs);
  }
  return AGQ_OK;
}

// Chunk length: a multiple of the block (chunks must not split blocks) and,
// for block 128, of the 1024-element warp tile.
uint64_t chunk_elems(uint64_t n, uint32_t block) {
  uint64_t unit = block;
  if (1024 % block == 0) unit = 1024;
  uint64_t c = std::max<uint64_t>(unit, kChunkElems / unit * unit);
  return std::min<uint64_t>(c, (n + unit - 1) / unit * unit);
}

agq_status read_errors(HostPipe& p, int op) {
  agq_errors h;
  if (agq_status st = cuda_fail(cudaMemcpy(&h, p.d_err, sizeof(h), cudaMemcpyDeviceToHost),
                                "host pipeline: errors"))
    return st;
  return agq_errors_message(&h, op, nullptr, 0);
}

// The host entry points as chunked ops (slot layouts: inputs first, outputs
// after them, so a slot's next inputs can be staged while its outputs drain).
OpSpec quantize_spec(const float* x, uint64_t n, int bits, uint32_t block, int codec) {
  const uint64_t ce = chunk_elems(n, block);
  const size_t oc = al(ce * 4), os = oc + al(ce);
  OpSpec op;
  op.chunks = (n + ce - 1) / ce;
  op.slot = os + al((ce / block + 1) * 4);
  op.op = AGQ_OP_QUANTIZE;
  op.plan = [=](uint64_t k, std::vector<Part>& in, std::vector<Part>& out) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    in.push_back(in_part(0, len * 4, x + e0));
    out.push_back(out_part(oc, len, 0, e0));
    out.push_back(out_part(os, (len + block - 1) / block * 4, 1, e0 / block * 4));
  };
  op.launch = [=](uint64_t k, char* d, cudaStream_t s, agq_errors* err) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    return quantize_device_at(d, AGQ_F32, len, bits, block, codec, d + oc, AGQ_CODES_BYTES,
                              reinterpret_cast<float*>(d + os), (long long)(e0 / block), err, s);
  };
  return op;
}

OpSpec dequantize_spec(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                       uint32_t block, int codec) {
  const uint64_t ce = chunk_elems(n, block);
  const size_t os = al(ce), oo = os + al((ce / block + 1) * 4);
  OpSpec op;
  op.chunks = (n + ce - 1) / ce;
  op.slot = oo + al(ce * 4);
  op.op = AGQ_OP_DEQUANTIZE;
  op.plan = [=](uint64_t k, std::vector<Part>& in, std::vector<Part>& out) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    in.push_back(in_part(0, len, codes + e0));
    in.push_back(in_part(os, (len + block - 1) / block * 4, scales + e0 / block));
    out.push_back(out_part(oo, len * 4, 0, e0 * 4));
  };
  op.launch = [=](uint64_t k, char* d, cudaStream_t s, agq_errors* err) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    return dequantize_device_at(d, AGQ_CODES_BYTES, reinterpret_cast<float*>(d + os), len, bits,
                                block, codec, d + oo, AGQ_F32, 1, (long long)(e0 / block), err, s);
  };
  return op;
}

OpSpec roundtrip_spec(const float* x, uint64_t n, int bits, uint32_t block, int codec) {
  const uint64_t ce = chunk_elems(n, block);
  // [x | reconstruction | codes | scales]: the codes never cross PCIe
  const size_t oo = al(ce * 4), oc = oo + al(ce * 4), os = oc + al(ce);
  OpSpec op;
  op.chunks = (n + ce - 1) / ce;
  op.slot = os + al((ce / block + 1) * 4);
  op.op = AGQ_OP_QUANTIZE;
  op.plan = [=](uint64_t k, std::vector<Part>& in, std::vector<Part>& out) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    in.push_back(in_part(0, len * 4, x + e0));
    out.push_back(out_part(oo, len * 4, 0, e0 * 4));
  };
  op.launch = [=](uint64_t k, char* d, cudaStream_t s, agq_errors* err) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    // quantize with the chunk's global block indices for the errors
    if (agq_status r = quantize_device_at(d, AGQ_F32, len, bits, block, codec, d + oc,
                                          AGQ_CODES_BYTES, reinterpret_cast<float*>(d + os),
                                          (long long)(e0 / block), err, s))
      return r;
    return dequantize_device_at(d + oc, AGQ_CODES_BYTES, reinterpret_cast<float*>(d + os), len,
                                bits, block, codec, d + oo, AGQ_F32, 0, (long long)(e0 / block),
                                err, s);
  };
  return op;
}

OpSpec accumulate_spec(const uint8_t* codes, const float* scales, uint64_t n, uint32_t block,
                       const float* local, int precision) {
  const uint64_t ce = chunk_elems(n, block);
  const size_t os = al(ce), ol = os + al((ce / block + 1) * 4), oc = ol + al(ce * 4);
  const size_t oo = oc + al(ce);
  OpSpec op;
  op.chunks = (n + ce - 1) / ce;
  op.slot = oo + al((ce / block + 1) * 4);
  op.op = AGQ_OP_ACCUMULATE;
  op.plan = [=](uint64_t k, std::vector<Part>& in, std::vector<Part>& out) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    const uint64_t nb = (len + block - 1) / block;
    in.push_back(in_part(0, len, codes + e0));
    in.push_back(in_part(os, nb * 4, scales + e0 / block));
    in.push_back(in_part(ol, len * 4, local + e0));
    out.push_back(out_part(oc, len, 0, e0));
    out.push_back(out_part(oo, nb * 4, 1, e0 / block * 4));
  };
  op.launch = [=](uint64_t k, char* d, cudaStream_t s, agq_errors* err) {
    const uint64_t e0 = k * ce, len = std::min(ce, n - e0);
    return accumulate_device(reinterpret_cast<uint8_t*>(d), reinterpret_cast<float*>(d + os),
                             d + ol, AGQ_F32, len, block, precision,
                             reinterpret_cast<uint8_t*>(d + oc), reinterpret_cast<float*>(d + oo),
                             err, s, (long long)(e0 / block));
  };
  return op;
}

// The synchronous entry: one pipeline pass, one sync, the error record.
agq_status run_sync(const OpSpec& op, void* out0, void* out1) {
  PipeLease lease;
  HostPipe& p = *lease.p;
  char* base[2] = {static_cast<char*>(out0), static_cast<char*>(out1)};
  if (agq_status st = run_pipeline(p, op, base)) return st;
  return read_errors(p, op.op);
}

// The begin entry: *job = nullptr (nothing issued) when the call's staging
// would exceed kJobStagingCap — the caller then uses the synchronous entry.
agq_status run_begin(const OpSpec& op, agq_host_job** job) {
  if (op.slot * op.chunks > kJobStagingCap) return AGQ_OK;
  auto j = std::make_unique<agq_host_job>();
  if (agq_status st = job_prepare(*j, op)) return st;
  int dev = 0;
  cudaGetDevice(&dev);
  agq_host_job* jp = j.get();
  if (op.slot * op.chunks < kJobAsyncMin) {  // small call: a thread costs more than it hides
    if (agq_status st = job_issue(*jp, op)) return st;
    *job = j.release();
    return AGQ_OK;
  }
  try {
    jp->issuer = std::thread([jp, op, dev] {
      cudaSetDevice(dev);
      jp->issue_status = job_issue(*jp, op);
      if (jp->issue_status != AGQ_OK) jp->issue_error = agq_last_error();
    });
  } catch (...) {  // no thread available: issue on the caller's thread
    if (agq_status st = job_issue(*jp, op)) return st;
  }
  *job = j.release();
  return AGQ_OK;
}

}  // namespace
}  // namespace agqh

extern "C" {

agq_status agq_host_pipeline_stats(double* out, int reset) {
  // [pipeline seconds, host copy seconds, event-wait seconds, calls]
  if (out) {
    out[0] = g_ns_total.load() * 1e-9;
    out[1] = g_ns_copy.load() * 1e-9;
    out[2] = g_ns_wait.load() * 1e-9;
    out[3] = (double)g_calls.load();
  }
  if (reset) g_ns_total = g_ns_copy = g_ns_wait = g_calls = 0;
  return AGQ_OK;
}

agq_status agq_host_copy(void* dst, const void* src, uint64_t bytes) {
  if (bytes == 0) return AGQ_OK;
  if (!dst || !src) return set_error(AGQ_ERR_INVALID_ARGUMENT, "agq_host_copy: null buffer");
  CopyPool::get().copy({{dst, src, (size_t)bytes}});
  return AGQ_OK;
}

agq_status agq_quantize_host(const float* x, uint64_t n, int bits, uint32_t block, int codec,
                             uint8_t* codes, float* scales) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_sync(quantize_spec(x, n, bits, block, codec), codes, scales);
}

agq_status agq_dequantize_host(const uint8_t* codes, const float* scales, uint64_t n, int bits,
                               uint32_t block, int codec, float* out) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_sync(dequantize_spec(codes, scales, n, bits, block, codec), out, nullptr);
}

agq_status agq_roundtrip_host(const float* x, uint64_t n, int bits, uint32_t block, int codec,
                              float* out) {
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_sync(roundtrip_spec(x, n, bits, block, codec), out, nullptr);
}

agq_status agq_local_accumulate_host(const uint8_t* codes, const float* scales, uint64_t n,
                                     uint32_t block, const float* local, int precision,
                                     uint8_t* out_codes, float* out_scales) {
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_sync(accumulate_spec(codes, scales, n, block, local, precision), out_codes,
                  out_scales);
}

agq_status agq_quantize_host_begin(const float* x, uint64_t n, int bits, uint32_t block,
                                   int codec, agq_host_job** job) {
  if (!job) return set_error(AGQ_ERR_INVALID_ARGUMENT, "agq_*_host_begin: null job");
  *job = nullptr;
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_begin(quantize_spec(x, n, bits, block, codec), job);
}

agq_status agq_dequantize_host_begin(const uint8_t* codes, const float* scales, uint64_t n,
                                     int bits, uint32_t block, int codec, agq_host_job** job) {
  if (!job) return set_error(AGQ_ERR_INVALID_ARGUMENT, "agq_*_host_begin: null job");
  *job = nullptr;
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_begin(dequantize_spec(codes, scales, n, bits, block, codec), job);
}

agq_status agq_roundtrip_host_begin(const float* x, uint64_t n, int bits, uint32_t block,
                                    int codec, agq_host_job** job) {
  if (!job) return set_error(AGQ_ERR_INVALID_ARGUMENT, "agq_*_host_begin: null job");
  *job = nullptr;
  if (agq_status st = check_args(bits, block, codec)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_begin(roundtrip_spec(x, n, bits, block, codec), job);
}

agq_status agq_local_accumulate_host_begin(const uint8_t* codes, const float* scales, uint64_t n,
                                           uint32_t block, const float* local, int precision,
                                           agq_host_job** job) {
  if (!job) return set_error(AGQ_ERR_INVALID_ARGUMENT, "agq_*_host_begin: null job");
  *job = nullptr;
  if (agq_status st = check_args(8, block, AGQ_CODEC_FP8_E4M3)) return st;
  if (agq_status st = check_device()) return st;
  if (n == 0) return AGQ_OK;
  return run_begin(accumulate_spec(codes, scales, n, block, local, precision), job);
}

agq_status agq_host_job_finish(agq_host_job* job, void* out0, void* out1) {
  if (!job) return AGQ_OK;
  std::unique_ptr<agq_host_job> j(job);
  if (j->issuer.joinable()) j->issuer.join();  // every chunk staged and enqueued
  if (j->issue_status != AGQ_OK) return set_error(j->issue_status, j->issue_error.c_str());
  if (!out0) {  // cancelled: drain the work, keep the pipeline consistent
    for (uint64_t k = 0; k < j->outs.size(); ++k) cudaEventSynchronize(j->lease.p->cev[k]);
    return AGQ_OK;
  }
  char* base[2] = {static_cast<char*>(out0), static_cast<char*>(out1)};
  if (agq_status st = job_finish(*j, base)) return st;
  return read_errors(*j->lease.p, j->op);
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
