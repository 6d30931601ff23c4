/*
 * agq_cuda.h — C ABI of the B200-native AGoQ quantization hot path.
 *
 * One shared library (paper_2605_00539_b200/libagq_cuda.so). Plain pointers
 * and sizes only; no C++ or torch types cross this boundary. Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/agq/).
 *
 * Conventions
 *  - Device entry points (agq_quantize, agq_dequantize, ...) take DEVICE
 *    pointers, are ordered on `stream` and never synchronize. Argument errors
 *    the reference reports before touching data (check_codec_args,
 *    quantize.hpp:64-74) are returned synchronously as AGQ_ERR_INVALID_ARGUMENT
 *    with the reference's message in agq_last_error(). Data-dependent errors
 *    (non-finite input, bad scales, fp32 overflow) are recorded by the kernels
 *    in a device-resident agq_errors record that the caller resets with
 *    agq_errors_reset() and reads after the stream completes;
 *    agq_errors_message() turns it into the reference's exception text.
 *  - Host entry points (*_host) take HOST pointers (pinned or pageable), stage
 *    through a library-owned device workspace on the given device, synchronize,
 *    and return the reference's error status/message directly. They are what
 *    the C++ drop-in headers (include/agq_b200/) call.
 *  - Packed code layout = tensor_io.hpp:63-80 pack_codes (LSB-first bitstream
 *    at `bits` bits per element); with block 128 every block is 16*bits bytes.
 *  - The product path has no CPU fallback: without a usable sm_100 device the
 *    device entry points return AGQ_ERR_CUDA.
 */
#ifndef AGQ_CUDA_H
#define AGQ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* agq_stream_t; /* == cudaStream_t */

typedef enum {
  AGQ_OK = 0,
  AGQ_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  AGQ_ERR_RUNTIME = 2,          /* std::runtime_error in the reference */
  AGQ_ERR_CUDA = 3,
  AGQ_ERR_NCCL = 4
} agq_status;

/* quantize.hpp:15-19 CodecKind */
typedef enum {
  AGQ_CODEC_SYMMETRIC_LINEAR = 0,
  AGQ_CODEC_FP4_E2M1 = 1,
  AGQ_CODEC_FP8_E4M3 = 2
} agq_codec;

typedef enum { AGQ_F32 = 0, AGQ_BF16 = 1 } agq_dtype;
typedef enum { AGQ_CODES_PACKED = 0, AGQ_CODES_BYTES = 1 } agq_code_layout;

/* collective.hpp:99 AccumulatePrecision */
typedef enum { AGQ_ACC_FP32 = 0, AGQ_ACC_BF16 = 1, AGQ_ACC_FP16 = 2 } agq_acc_precision;

/* Device-resident error record. "None" is INT64_MAX for the *_block/_index
 * fields and 0 for the flags/counters. */
typedef struct {
  long long nonfinite_block;   /* quantize.hpp:106-110 lowest block with a non-finite element */
  long long bad_scale_block;   /* quantize.hpp:170-175 lowest block with scale <0 or non-finite */
  long long bad_code_index;    /* quantize.hpp:165-169 lowest element with code >= 2^bits */
  long long nonfinite_local;   /* collective.hpp:138-139 lowest non-finite local gradient index */
  long long overflow_block;    /* collective.hpp:278-281 fp32 overflow in the local reduce */
  unsigned long long saturated; /* collective.hpp:390-398 naive-protocol saturation count */
} agq_errors;

/* ---- library ------------------------------------------------------------ */
const char* agq_version(void);
/* Thread-local message of the last failing call on this thread. */
const char* agq_last_error(void);
/* 1 if the current device is sm_100 and the kernels loaded, else 0. */
int agq_device_ok(void);
/* Number of kernels this library launched in this process (all streams). */
unsigned long long agq_launch_count(void);

agq_status agq_errors_reset(agq_errors* d_err, agq_stream_t stream);
/* Translate a HOST copy of the record into the reference's status + text
 * (priority follows the reference's check order). */
agq_status agq_errors_message(const agq_errors* h_err, int op, char* msg,
                              size_t msglen);
enum { AGQ_OP_QUANTIZE = 0, AGQ_OP_DEQUANTIZE = 1, AGQ_OP_ACCUMULATE = 2,
       AGQ_OP_ALLREDUCE = 3 };

/* ---- sizes --------------------------------------------------------------- */
uint64_t agq_num_blocks(uint64_t n, uint32_t block);
uint64_t agq_packed_bytes(uint64_t n, int bits); /* (n*bits+7)/8 */

/* quantize.hpp:64-74 detail::check_codec_args */
agq_status agq_check_codec_args(int bits, uint32_t block, int codec);

/* ---- L1 block codec (device) -------------------------------------------- */
/* Replaces quantize_blockwise (quantize.hpp:78-138) + pack_codes
 * (tensor_io.hpp:63-80). x: n elements of x_dtype. codes: packed bitstream
 * (agq_packed_bytes(n,bits) bytes) or one byte per element. scales:
 * agq_num_blocks(n, block) floats (= block absmax). */
agq_status agq_quantize(const void* x, int x_dtype, uint64_t n, int bits,
                        uint32_t block, int codec, void* codes, int layout,
                        float* scales, agq_errors* d_err, agq_stream_t stream);

/* Replaces validate + dequantize_blockwise (quantize.hpp:157-189).
 * out: n elements of out_dtype (F32 = bit-exact reference values; BF16 =
 * round-to-nearest-even of them). validate != 0 performs the reference's
 * code-range / scale checks into d_err. */
agq_status agq_dequantize(const void* codes, int layout, const float* scales,
                          uint64_t n, int bits, uint32_t block, int codec,
                          void* out, int out_dtype, int validate,
                          agq_errors* d_err, agq_stream_t stream);

/* quantize + the reconstruction dequantize_blockwise gives for its codes in
 * one call (quantize.hpp:193-196 roundtrip_relative_delta; the C1 round
 * trip). SymmetricLinear BF16 in / out with block 128 and packed codes runs
 * as ONE kernel pass (x read once); everything else as quantize followed by
 * dequantize. Outputs are bit-identical to those two calls. */
agq_status agq_quantize_roundtrip(const void* x, int x_dtype, uint64_t n, int bits,
                                  uint32_t block, int codec, void* codes, int layout,
                                  float* scales, void* out, int out_dtype,
                                  agq_errors* d_err, agq_stream_t stream);

/* One stored tensor of a layer (layers.hpp:148-163 SavedEntry::quantized):
 * block 128, SymmetricLinear unless codec says otherwise. */
typedef struct {
  const void* x;     /* quantize: input; dequantize: output */
  void* codes;       /* packed */
  float* scales;
  uint64_t n;
} agq_segment;

/* Grouped launch over the tensors one pipeline stage stores (dbca.hpp:172-177
 * stage_policy -> layers.hpp:64-75 agoq_default(bits), layers.hpp:266-301
 * the stored set of every layer of the stage). All segments share
 * bits/codec/dtype; block is 128. Any segment count: up to 8 segments go
 * into one launch, larger groups are split. Error indices in d_err are
 * group-global (blocks / elements counted over the segments in order).
 * validate != 0 performs the reference's dequantize-time checks
 * (quantize.hpp:157-179: code range, finite non-negative scales). */
agq_status agq_quantize_grouped(const agq_segment* segs, int nseg, int x_dtype,
                                int bits, int codec, agq_errors* d_err,
                                agq_stream_t stream);
agq_status agq_dequantize_grouped(const agq_segment* segs, int nseg,
                                  int out_dtype, int bits, int codec,
                                  int validate, agq_errors* d_err,
                                  agq_stream_t stream);

/* tensor_io.hpp:63-100 on device */
agq_status agq_pack_codes(const uint8_t* codes, uint64_t n, int bits,
                          uint8_t* packed, agq_stream_t stream);
agq_status agq_unpack_codes(const uint8_t* packed, uint64_t n, int bits,
                            uint8_t* codes, agq_stream_t stream);

/* ---- L2a gradient path (device) ----------------------------------------- */
/* Replaces local_accumulate (collective.hpp:128-147): FP8-E4M3 main gradient
 * (codes one byte per element, block absmax scales) + local gradient
 * (F32 or BF16) -> dequantize, add (optionally rounded to BF16/FP16),
 * fresh-absmax FP8 requantize. out_* may alias codes/scales (in place). */
agq_status agq_fp8_accumulate(const uint8_t* codes, const float* scales,
                              const void* local, int local_dtype, uint64_t n,
                              uint32_t block, int precision,
                              uint8_t* out_codes, float* out_scales,
                              agq_errors* d_err, agq_stream_t stream);

/* Local reduce of the decomposed all-reduce (collective.hpp:250-284):
 * acc = +0.0f; acc += dequant(piece_s) for s = 0..npieces-1 in order; fp32
 * overflow -> d_err->overflow_block; fresh-absmax FP8 requant written to all
 * nout destinations (local and/or peer-mapped pointers). len elements,
 * block-aligned start. npieces, nout <= AGQ_MAX_WORLD. */
#define AGQ_MAX_WORLD 16
agq_status agq_fp8_reduce_requant(int npieces, const uint8_t* const* piece_codes,
                                  const float* const* piece_scales,
                                  uint64_t len, uint32_t block, int nout,
                                  uint8_t* const* out_codes,
                                  float* const* out_scales, agq_errors* d_err,
                                  agq_stream_t stream);

/* collective.hpp:23-39 ChunkAssignment::block_aligned; ranges = 2*workers. */
agq_status agq_chunk_assignment(uint64_t n, uint32_t block, int workers,
                                uint64_t* ranges);

/* In-process simulation on ONE device, same contract as
 * allreduce_decomposed(std::vector<WorkerState>&) (collective.hpp:226-333):
 * `world` FP8 gradients (device pointers) -> the reduced tensor every worker
 * ends up with. */
agq_status agq_allreduce_simulated(int world, const uint8_t* const* codes,
                                   const float* const* scales, uint64_t n,
                                   uint32_t block, uint8_t* out_codes,
                                   float* out_scales, agq_errors* d_err,
                                   agq_stream_t stream);

/* The overflow-prone strawman allreduce_naive_fp8 (collective.hpp:338-431),
 * simulated on one device; saturation count into d_err->saturated
 * (elements that ever saturated, = CollectiveResult::overflow_elements). */
agq_status agq_allreduce_naive_simulated(int world, const uint8_t* const* codes,
                                         const float* const* scales, uint64_t n,
                                         uint32_t block, uint8_t* out_codes,
                                         float* out_scales, agq_errors* d_err,
                                         unsigned long long* d_events /* world, or NULL */,
                                         agq_stream_t stream);

/* ---- multi-GPU decomposed all-reduce (one process per GPU) --------------- */
typedef struct agq_comm agq_comm;
enum { AGQ_AR_NCCL = 0, AGQ_AR_FUSED_P2P = 1, AGQ_AR_PUSH_P2P = 2, AGQ_AR_ONESHOT_P2P = 3 };

agq_status agq_comm_unique_id(unsigned char id[128]);
/* Collective over all ranks (NCCL communicator). device = CUDA ordinal.
 * id == NULL creates a P2P-only communicator (no NCCL): only
 * AGQ_AR_FUSED_P2P / AGQ_AR_PUSH_P2P after p2p_export/open; it also allows
 * several ranks on one GPU (which NCCL refuses). */
agq_status agq_comm_init(agq_comm** comm, const unsigned char id[128],
                         int nranks, int rank, int device);
/* Peer-memory setup for AGQ_AR_FUSED_P2P / AGQ_AR_PUSH_P2P: export this
 * rank's IPC handle, then open every peer's. Handles are exchanged by the
 * caller (any transport). capacity = max element count per all-reduce; the
 * symmetric buffer holds the gradient (capacity * (1 + 4/128) bytes) plus
 * the push algorithm's inbox (one chunk per sender, about the same again). */
agq_status agq_comm_p2p_export(agq_comm* comm, uint64_t capacity,
                               unsigned char handle[256]);
agq_status agq_comm_p2p_open(agq_comm* comm, const unsigned char* handles
                             /* nranks * 256 bytes, rank order */);
/* The symmetric (IPC-exported) FP8 gradient buffers of this rank: write the
 * gradient here and pass these pointers to agq_allreduce_fp8 to run the fused
 * path fully in place (other pointers are copied in and out). */
agq_status agq_comm_p2p_buffers(agq_comm* comm, uint8_t** codes, float** scales);
agq_status agq_comm_destroy(agq_comm* comm);
int agq_comm_rank(const agq_comm* comm);
int agq_comm_size(const agq_comm* comm);
/* Device barrier timeout of the P2P algorithms (default 300 s). A barrier
 * that times out (a peer that never arrived) makes the call report
 * "all-reduce aborted: peer did not arrive (timeout)" and marks the
 * communicator failed on every rank: later P2P calls fail fast; destroy and
 * re-create the communicator. */
agq_status agq_comm_set_timeout(agq_comm* comm, double seconds);

/* One message of the decomposed all-reduce, as collective.hpp:50-57
 * TraceEvent (phase 0 = "all_to_all", 1 = "all_gather"; payload = codes +
 * 4 bytes per block scale, collective.hpp:195-206 deliver). */
typedef struct {
  int phase;
  int sender;
  int receiver;
  int reserved;
  uint64_t chunk_start;
  uint64_t chunk_len;
  uint64_t payload_bytes;
} agq_trace_event;

/* The messages this rank took part in during its last agq_allreduce_fp8
 * call, recorded by the code that issued the transfers (NCCL: every
 * send this rank posted; fused P2P: the chunk-r pulls from every peer and
 * the pushes of the reduced chunk; push P2P: the scatters and pushes). The
 * union over all ranks, sorted by (phase, sender, receiver), is the
 * reference's MessageTrace. *count = number of events (may exceed cap).
 * moved (2 entries, or NULL): for the P2P algorithms the kernel's own
 * counters of the phase-1 traffic (elements, block scales), synchronising
 * the call's stream; zeros for NCCL. */
agq_status agq_comm_last_trace(agq_comm* comm, agq_trace_event* events, int cap,
                               int* count, unsigned long long* moved);

/* Replaces allreduce_decomposed for real ranks: in-place on this rank's FP8
 * gradient (codes one byte/element + block scales). All ranks call it with
 * the same n/block. algo = AGQ_AR_NCCL (grouped send/recv all-to-all +
 * reduce-requant kernel + ncclAllGather), AGQ_AR_FUSED_P2P (one kernel per
 * rank: pull pieces over NVLink, reduce, push results) or AGQ_AR_PUSH_P2P
 * (two kernels per rank, every NVLink transfer a store: scatter pieces into
 * the owners' inboxes, then reduce from local memory and push results) or
 * AGQ_AR_ONESHOT_P2P (small messages, n <= 4 Mi elements: every rank stores
 * its whole gradient into every peer's inbox and reduces all blocks locally;
 * one exchange, no end barrier, (P-1)x the wire bytes). All four give
 * bit-identical results. The P2P algorithms keep their epoch on the device
 * and allocate nothing per call, so they can be captured in a CUDA graph.
 * Collective contract: every rank issues the same sequence of P2P calls on
 * a communicator (same n, block, algorithm), each rank on one stream; the
 * calls of one rank must not run concurrently (they share the symmetric
 * buffer, its inboxes and the epoch). */
agq_status agq_allreduce_fp8(agq_comm* comm, uint8_t* codes, float* scales,
                             uint64_t n, uint32_t block, int algo,
                             agq_errors* d_err, agq_stream_t stream);

/* Replaces allreduce_naive_fp8 (collective.hpp:338-431) for real ranks: the
 * overflow-prone strawman, in place on this rank's FP8 gradient. P-1 NCCL
 * ring steps, each adding in FP8 at the receiver's ORIGINAL scales, then an
 * all-gather (chunk c from rank (c-1) mod P, with that rank's scales).
 * d_err->saturated (caller-reset) = CollectiveResult::overflow_elements,
 * identical on every rank; *d_events (caller-zeroed, or NULL) += this
 * rank's CollectiveResult::overflow_events entry. */
agq_status agq_allreduce_naive_fp8(agq_comm* comm, uint8_t* codes, float* scales,
                                   uint64_t n, uint32_t block, agq_errors* d_err,
                                   unsigned long long* d_events,
                                   agq_stream_t stream);

/* The baseline the north star compares against: ncclAllReduce(bf16, sum). */
agq_status agq_allreduce_bf16_nccl(agq_comm* comm, void* data, uint64_t n,
                                   agq_stream_t stream);

/* ---- host entry points (C++ drop-in surface) ----------------------------- */
agq_status agq_quantize_host(const float* x, uint64_t n, int bits,
                             uint32_t block, int codec, uint8_t* codes,
                             float* scales);
agq_status agq_dequantize_host(const uint8_t* codes, const float* scales,
                               uint64_t n, int bits, uint32_t block, int codec,
                               float* out);
/* quantize then dequantize of host FP32 values, the codes kept on the device
 * (quantize.hpp:193-196 roundtrip_relative_delta's reconstruction). */
agq_status agq_roundtrip_host(const float* x, uint64_t n, int bits, uint32_t block,
                              int codec, float* out);
agq_status agq_local_accumulate_host(const uint8_t* codes, const float* scales,
                                     uint64_t n, uint32_t block,
                                     const float* local, int precision,
                                     uint8_t* out_codes, float* out_scales);
/* Split form of the four entries above, for callers that allocate their
 * result buffers after the call starts (the drop-in API value-initialises
 * its result vectors: that host work overlaps the transfers and kernels).
 * *_begin returns at once: a library thread stages the inputs (they must
 * stay valid and unchanged until finish) and enqueues every chunk; *job is
 * NULL when nothing was issued (n == 0, or
 * the call's staging exceeds the library's 256 MB job cap — use the
 * synchronous entry then). agq_host_job_finish waits, copies the results to
 * out0 (codes or values) / out1 (scales, or NULL), reports the same errors
 * as the synchronous entry and frees the job; out0 == NULL cancels it. */
typedef struct agq_host_job agq_host_job;
agq_status agq_quantize_host_begin(const float* x, uint64_t n, int bits, uint32_t block,
                                   int codec, agq_host_job** job);
agq_status agq_dequantize_host_begin(const uint8_t* codes, const float* scales,
                                     uint64_t n, int bits, uint32_t block, int codec,
                                     agq_host_job** job);
agq_status agq_roundtrip_host_begin(const float* x, uint64_t n, int bits, uint32_t block,
                                    int codec, agq_host_job** job);
agq_status agq_local_accumulate_host_begin(const uint8_t* codes, const float* scales,
                                           uint64_t n, uint32_t block,
                                           const float* local, int precision,
                                           agq_host_job** job);
agq_status agq_host_job_finish(agq_host_job* job, void* out0, void* out1);
/* Diagnostics of the host-buffer pipelines: out[0..3] = cumulative seconds
 * inside the pipelines, of host copies (caller <-> pinned staging), waiting
 * for device work, and the number of calls; reset != 0 zeroes them. */
agq_status agq_host_pipeline_stats(double* out, int reset);
/* The host pipelines' staging copy (caller memory <-> pinned slots): the
 * library's copy threads plus the caller, streaming stores. Exported so a
 * caller can measure the host-memory rate that bounds the *_host entries. */
agq_status agq_host_copy(void* dst, const void* src, uint64_t bytes);
agq_status agq_allreduce_simulated_host(int world, const uint8_t* const* codes,
                                        const float* const* scales, uint64_t n,
                                        uint32_t block, int protocol /*0 dec,1 naive*/,
                                        uint8_t* out_codes, float* out_scales,
                                        uint64_t* overflow_elements,
                                        uint64_t* overflow_events /* world, or NULL */);

/* ---- synthetic inputs (host) ---------------------------------------------- */
/* tools/agq.cpp:47-65 InputSpec::materialize + rng.hpp:9-28 make_rng(seed,
 * stream, index): std::mt19937_64(derive_seed(...)) driving
 * std::normal_distribution<float>(a, b) (the CLI: a=0, b=1, stream 0x1D,
 * index 0), std::uniform_real_distribution<float>(a, b) or the constant a —
 * the reference's bytes (same libstdc++). out: HOST buffer of n F32 values,
 * or BF16 = their round-to-nearest-even. All-reduce worker r of the CLI uses
 * seed + r (agq.cpp:279). */
enum { AGQ_INPUT_NORMAL = 0, AGQ_INPUT_UNIFORM = 1, AGQ_INPUT_CONST = 2 };
agq_status agq_fill_input(uint64_t seed, uint64_t stream, uint64_t index, int kind,
                          double a, double b, int out_dtype, void* out, uint64_t n);

/* ---- L2b control plane (dbca.hpp, host) ---------------------------------- */
/* dbca.hpp:34-41 stored_activation_counts; counts[n_stages]. */
agq_status agq_stored_activation_counts(int n_stages, int micro_batches,
                                        int interleave, int* counts);
/* dbca.hpp:63-78 plan_bit_widths. */
agq_status agq_plan_bit_widths(int n_stages, int micro_batches, int interleave,
                               int* counts, double* raw_bits,
                               int* assigned_bits);

#ifdef __cplusplus
}
#endif
#endif /* AGQ_CUDA_H */
