/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the AGoQ hot path.
 *
 * Plain-C restatement of the reference algorithm in
 * /root/reference/proj/include/agq/{fp8,quantize,tensor_io,collective,dbca}.hpp.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it (as the checker). The product library never links it.
 * Pinned against the reference itself (oracle/_ref, built from the reference
 * headers by oracle/Makefile) and against the reference tests' known-answer
 * vectors (tests/golden/, tests/test_oracle.py).
 */
#ifndef AGQ_ORACLE_H
#define AGQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_RUNTIME_ERROR = 2 };
enum { ORC_LINEAR = 0, ORC_FP4 = 1, ORC_FP8 = 2 };
enum { ORC_ACC_FP32 = 0, ORC_ACC_BF16 = 1, ORC_ACC_FP16 = 2 };

/* fp8.hpp */
uint8_t oracle_fp8_encode(double v, int* overflow);
double oracle_fp8_decode(uint8_t b);
uint8_t oracle_fp4_encode(double v);
double oracle_fp4_decode(uint8_t c);

/* quantize.hpp */
double oracle_code_unit_value(int codec, int bits, uint8_t code);
int oracle_check_codec_args(int bits, uint32_t block, int codec, char* err,
                            size_t errlen);
int oracle_quantize(const float* x, size_t n, int bits, uint32_t block,
                    int codec, uint8_t* codes, float* scales, char* err,
                    size_t errlen);
int oracle_dequantize(const uint8_t* codes, const float* scales, size_t n,
                      int bits, uint32_t block, int codec, float* out,
                      char* err, size_t errlen);

/* tensor_io.hpp */
size_t oracle_pack_codes(const uint8_t* codes, size_t n, int bits,
                         uint8_t* out);
int oracle_unpack_codes(const uint8_t* bytes, size_t nbytes, int bits,
                        size_t count, uint8_t* out);
size_t oracle_dump_size(size_t n, int bits, uint32_t block, int ndim);
int oracle_dump(const uint8_t* codes, const float* scales, size_t n, int bits,
                uint32_t block, int codec, const uint64_t* shape, int ndim,
                uint8_t* out);

/* collective.hpp */
float oracle_round_bf16(float x);
float oracle_round_fp16(float x);
int oracle_local_accumulate(const uint8_t* codes, const float* scales,
                            size_t n, uint32_t block, const float* local,
                            int precision, uint8_t* out_codes,
                            float* out_scales, char* err, size_t errlen);
void oracle_chunk_assignment(size_t n, uint32_t block, int workers,
                             uint64_t* ranges);
int oracle_allreduce_oracle(int world, size_t n, uint32_t block,
                            const uint8_t* const* codes,
                            const float* const* scales, float* out, char* err,
                            size_t errlen);
int oracle_allreduce_decomposed(int world, size_t n, uint32_t block,
                                const uint8_t* const* codes,
                                const float* const* scales,
                                uint8_t* out_codes, float* out_scales,
                                char* err, size_t errlen);
int oracle_allreduce_naive(int world, size_t n, uint32_t block,
                           const uint8_t* const* codes,
                           const float* const* scales, uint8_t* out_codes,
                           float* out_scales, uint64_t* overflow_elements,
                           char* err, size_t errlen);

/* dbca.hpp (Eigen-free restatement of the planner) */
int oracle_stored_activation_counts(int n_stages, int micro_batches,
                                    int interleave, int* counts);
int oracle_plan_bit_widths(int n_stages, int micro_batches, int interleave,
                           int* counts, double* raw_bits, int* assigned);
int oracle_plan_reuse(int low_n, int low_mb, int high_n, int high_mb,
                      int* applied, double* peak, double* uniform4_peak,
                      int* pass);

#ifdef __cplusplus
}
#endif
#endif
