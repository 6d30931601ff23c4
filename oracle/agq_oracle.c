/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain C restatement) of the AGoQ
 * quantization hot path. See agq_oracle.h for the usage rules. Each function
 * cites the reference file:line it follows; paths are relative to
 * /root/reference/proj/include/agq/. Compile with -ffp-contract=off so every
 * double/float operation rounds exactly where the reference's does.
 */
#include "agq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int set_err(char* err, size_t errlen, int code, const char* msg) {
  if (err && errlen) {
    strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

/* ---- fp8.hpp:32-66 fp8_encode ------------------------------------------ */
uint8_t oracle_fp8_encode(double v, int* overflow) {
  if (overflow) *overflow = 0;
  const uint8_t sign = signbit(v) ? 0x80 : 0x00;
  if (isnan(v)) return (uint8_t)(sign | 0x7f); /* :33-36 */
  const double a = fabs(v);
  if (a > 448.0) { /* :39-42 saturate, flag overflow */
    if (overflow) *overflow = 1;
    return (uint8_t)(sign | 0x7e);
  }
  if (a < 0x1p-6) { /* :43-52 subnormal quantum 2^-9, RNE via nearbyint */
    const int q = (int)nearbyint(a * 0x1p9);
    if (q == 0) return sign;
    if (q < 8) return (uint8_t)(sign | q);
    return (uint8_t)(sign | (1 << 3));
  }
  int e = ilogb(a); /* :53-65 */
  int q = (int)nearbyint(ldexp(a, 3 - e));
  if (q == 16) {
    q = 8;
    ++e;
  }
  return (uint8_t)(sign | ((uint8_t)(e + 7) << 3) | (uint8_t)(q - 8));
}

/* fp8.hpp:68-84 fp8_decode */
double oracle_fp8_decode(uint8_t b) {
  const int sign = (b & 0x80) != 0;
  const int ef = (b >> 3) & 0xf, m = b & 7;
  if (ef == 0xf && m == 7) return copysign(NAN, sign ? -1.0 : 1.0);
  const double mag = ef == 0 ? m * 0x1p-9 : ldexp(8 + m, ef - 10);
  return sign ? -mag : mag;
}

/* fp8.hpp:87-114 E2M1 */
static const double kFp4Mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
uint8_t oracle_fp4_encode(double v) {
  const uint8_t sign = signbit(v) ? 0x8 : 0x0;
  const double a = fabs(v);
  if (a >= 6.0) return (uint8_t)(sign | 0x7);
  int best = 0;
  double best_dist = a;
  for (int i = 1; i < 8; ++i) {
    const double d = fabs(a - kFp4Mag[i]);
    if (d < best_dist || (d == best_dist && (i % 2 == 0))) {
      best_dist = d;
      best = i;
    }
  }
  if (best == 0) return 0; /* -0 -> +0 (:107) */
  return (uint8_t)(sign | best);
}
double oracle_fp4_decode(uint8_t c) {
  const double m = kFp4Mag[c & 7];
  return (c & 8) ? -m : m;
}

/* ---- quantize.hpp ------------------------------------------------------- */
static int levels_of(int bits) { return (1 << (bits - 1)) - 1; } /* :62 */

/* quantize.hpp:64-74 */
int oracle_check_codec_args(int bits, uint32_t block, int codec, char* err,
                            size_t errlen) {
  char buf[96];
  if (bits < 4 || bits > 8) {
    snprintf(buf, sizeof buf, "bit_width must be in [4, 8], got %d", bits);
    return set_err(err, errlen, ORC_INVALID_ARGUMENT, buf);
  }
  if (block == 0)
    return set_err(err, errlen, ORC_INVALID_ARGUMENT, "block_size must be >= 1");
  if (codec == ORC_FP8 && bits != 8)
    return set_err(err, errlen, ORC_INVALID_ARGUMENT,
                   "fp8_e4m3 requires bit_width 8");
  if (codec == ORC_FP4 && bits != 4)
    return set_err(err, errlen, ORC_INVALID_ARGUMENT,
                   "fp4_e2m1 requires bit_width 4");
  return ORC_OK;
}

/* quantize.hpp:78-138 quantize_blockwise (shape = {n}) */
int oracle_quantize(const float* x, size_t n, int bits, uint32_t block,
                    int codec, uint8_t* codes, float* scales, char* err,
                    size_t errlen) {
  int st = oracle_check_codec_args(bits, block, codec, err, errlen);
  if (st) return st;
  const size_t nb = (n + block - 1) / block;
  const int L = levels_of(bits);
  const uint8_t zero_code = codec == ORC_LINEAR ? (uint8_t)L : 0;
  for (size_t b = 0; b < nb; ++b) {
    const size_t begin = b * block;
    const size_t end = begin + block < n ? begin + block : n;
    float absmax = 0.0f;
    for (size_t i = begin; i < end; ++i) { /* :106-112 */
      if (!isfinite(x[i])) {
        char buf[96];
        snprintf(buf, sizeof buf, "non-finite input element in block %zu", b);
        return set_err(err, errlen, ORC_INVALID_ARGUMENT, buf);
      }
      const float ax = fabsf(x[i]);
      absmax = absmax > ax ? absmax : ax; /* std::max(absmax, fabs) */
    }
    scales[b] = absmax;
    if (absmax == 0.0f) { /* :114-117 */
      for (size_t i = begin; i < end; ++i) codes[i] = zero_code;
      continue;
    }
    for (size_t i = begin; i < end; ++i) { /* :118-135 */
      const double t = (double)x[i] / absmax;
      switch (codec) {
        case ORC_LINEAR: {
          int k = (int)nearbyint(t * L);
          if (k < -L) k = -L;
          if (k > L) k = L;
          codes[i] = (uint8_t)(k + L);
          break;
        }
        case ORC_FP4:
          codes[i] = oracle_fp4_encode(t * 6.0);
          break;
        default:
          codes[i] = oracle_fp8_encode(t * 448.0, NULL);
      }
    }
  }
  return ORC_OK;
}

/* quantize.hpp:142-155 */
double oracle_code_unit_value(int codec, int bits, uint8_t code) {
  switch (codec) {
    case ORC_LINEAR: {
      const int L = levels_of(bits);
      return (double)((int)code - L) / L;
    }
    case ORC_FP4:
      return oracle_fp4_decode(code) / 6.0;
    default:
      return oracle_fp8_decode(code) / 448.0;
  }
}

/* quantize.hpp:157-176 validate + :178-189 dequantize_blockwise */
int oracle_dequantize(const uint8_t* codes, const float* scales, size_t n,
                      int bits, uint32_t block, int codec, float* out,
                      char* err, size_t errlen) {
  int st = oracle_check_codec_args(bits, block, codec, err, errlen);
  if (st) return st;
  const size_t nb = (n + block - 1) / block;
  const uint32_t limit = 1u << bits;
  char buf[96];
  for (size_t i = 0; i < n; ++i)
    if (codes[i] >= limit) {
      snprintf(buf, sizeof buf, "quantized tensor: code out of range at %zu", i);
      return set_err(err, errlen, ORC_INVALID_ARGUMENT, buf);
    }
  for (size_t b = 0; b < nb; ++b) {
    const float s = scales[b];
    if (!(s >= 0.0f) || !isfinite(s)) {
      snprintf(buf, sizeof buf, "quantized tensor: bad scale at block %zu", b);
      return set_err(err, errlen, ORC_INVALID_ARGUMENT, buf);
    }
  }
  for (size_t i = 0; i < n; ++i) {
    const double scale = scales[i / block];
    out[i] = (float)(oracle_code_unit_value(codec, bits, codes[i]) * scale);
  }
  return ORC_OK;
}

/* ---- tensor_io.hpp:63-100 LSB-first bitstream ---------------------------- */
size_t oracle_pack_codes(const uint8_t* codes, size_t n, int bits,
                         uint8_t* out) {
  size_t k = 0;
  uint32_t acc = 0;
  int nbits = 0;
  for (size_t i = 0; i < n; ++i) {
    acc |= (uint32_t)(codes[i] & ((1u << bits) - 1)) << nbits;
    nbits += bits;
    while (nbits >= 8) {
      out[k++] = (uint8_t)(acc & 0xff);
      acc >>= 8;
      nbits -= 8;
    }
  }
  if (nbits > 0) out[k++] = (uint8_t)(acc & 0xff);
  return k;
}

int oracle_unpack_codes(const uint8_t* bytes, size_t nbytes, int bits,
                        size_t count, uint8_t* out) {
  uint32_t acc = 0;
  int nbits = 0;
  size_t pos = 0;
  for (size_t i = 0; i < count; ++i) {
    while (nbits < bits) {
      if (pos >= nbytes) return ORC_RUNTIME_ERROR; /* "packed codes truncated" */
      acc |= (uint32_t)bytes[pos++] << nbits;
      nbits += 8;
    }
    out[i] = (uint8_t)(acc & ((1u << bits) - 1));
    acc >>= bits;
    nbits -= bits;
  }
  return ORC_OK;
}

/* tensor_io.hpp:16-21,102-122: "AGQT", u16 version 1, u8 codec, u8 bits,
 * u32 block, u8 ndim, u64 dims, f32 scales, packed codes (little-endian). */
size_t oracle_dump_size(size_t n, int bits, uint32_t block, int ndim) {
  return 4 + 2 + 1 + 1 + 4 + 1 + 8 * (size_t)ndim +
         4 * ((n + block - 1) / block) + (n * bits + 7) / 8;
}

static void put_le(uint8_t** p, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) *(*p)++ = (uint8_t)(v >> (8 * i));
}

int oracle_dump(const uint8_t* codes, const float* scales, size_t n, int bits,
                uint32_t block, int codec, const uint64_t* shape, int ndim,
                uint8_t* out) {
  uint8_t* p = out;
  memcpy(p, "AGQT", 4);
  p += 4;
  put_le(&p, 1, 2);
  put_le(&p, (uint64_t)codec, 1);
  put_le(&p, (uint64_t)bits, 1);
  put_le(&p, block, 4);
  put_le(&p, (uint64_t)ndim, 1);
  for (int d = 0; d < ndim; ++d) put_le(&p, shape[d], 8);
  const size_t nb = (n + block - 1) / block;
  for (size_t b = 0; b < nb; ++b) {
    uint32_t u;
    memcpy(&u, &scales[b], 4);
    put_le(&p, u, 4);
  }
  p += oracle_pack_codes(codes, n, bits, p);
  return (int)(p - out);
}

/* ---- collective.hpp ------------------------------------------------------ */
/* :101-110 integer RNE on the fp32 bits */
float oracle_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t lsb = (u >> 16) & 1;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  float out;
  memcpy(&out, &u, 4);
  return out;
}

/* :112-123 custom fp16 RNE, saturating at 65520 -> 65504 */
float oracle_round_fp16(float x) {
  if (x == 0.0f || !isfinite(x)) return x;
  const double a = fabs((double)x);
  const double sign = x < 0.0f ? -1.0 : 1.0;
  if (a >= 65520.0) return (float)(sign * 65504.0);
  if (a < 0x1p-14) return (float)(sign * nearbyint(a * 0x1p24) * 0x1p-24);
  const int e = ilogb(a);
  const double q = nearbyint(ldexp(a, 10 - e));
  return (float)(sign * ldexp(q, e - 10));
}

/* :128-147 local_accumulate (main must be FP8 E4M3; checked by caller) */
int oracle_local_accumulate(const uint8_t* codes, const float* scales,
                            size_t n, uint32_t block, const float* local,
                            int precision, uint8_t* out_codes,
                            float* out_scales, char* err, size_t errlen) {
  float* vals = (float*)malloc(n ? n * sizeof(float) : 1);
  int st = oracle_dequantize(codes, scales, n, 8, block, ORC_FP8, vals, err,
                             errlen);
  if (st) {
    free(vals);
    return st;
  }
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(local[i])) {
      free(vals);
      return set_err(err, errlen, ORC_INVALID_ARGUMENT,
                     "non-finite local gradient element");
    }
    float s = vals[i] + local[i];
    if (precision == ORC_ACC_BF16) s = oracle_round_bf16(s);
    if (precision == ORC_ACC_FP16) s = oracle_round_fp16(s);
    vals[i] = s;
  }
  st = oracle_quantize(vals, n, 8, block, ORC_FP8, out_codes, out_scales, err,
                       errlen);
  free(vals);
  return st;
}

/* :23-39 ChunkAssignment::block_aligned */
void oracle_chunk_assignment(size_t n, uint32_t block, int workers,
                             uint64_t* ranges) {
  const size_t blocks = (n + block - 1) / block;
  size_t next = 0;
  for (int r = 0; r < workers; ++r) {
    const size_t share = blocks / workers + ((size_t)r < blocks % workers);
    const size_t begin = next * block < n ? next * block : n;
    next += share;
    const size_t end = next * block < n ? next * block : n;
    ranges[2 * r] = begin;
    ranges[2 * r + 1] = end;
  }
}

/* :212-221 allreduce_oracle: fp32 sum of dequantized inputs, ascending rank,
 * starting at +0.0f */
int oracle_allreduce_oracle(int world, size_t n, uint32_t block,
                            const uint8_t* const* codes,
                            const float* const* scales, float* out, char* err,
                            size_t errlen) {
  float* piece = (float*)malloc(n ? n * sizeof(float) : 1);
  for (size_t i = 0; i < n; ++i) out[i] = 0.0f;
  for (int r = 0; r < world; ++r) {
    int st = oracle_dequantize(codes[r], scales[r], n, 8, block, ORC_FP8,
                               piece, err, errlen);
    if (st) {
      free(piece);
      return st;
    }
    for (size_t i = 0; i < n; ++i) out[i] += piece[i];
  }
  free(piece);
  return ORC_OK;
}

/* :226-333 allreduce_decomposed. Every owner chunk is block aligned and the
 * per-element sum order is ascending sender rank from +0.0f (:256-277), so
 * chunk r's reduced codes/scales are quantize(sum) over [begin_r, end_r);
 * the all-gather reassembles them in place (:303-331). */
int oracle_allreduce_decomposed(int world, size_t n, uint32_t block,
                                const uint8_t* const* codes,
                                const float* const* scales,
                                uint8_t* out_codes, float* out_scales,
                                char* err, size_t errlen) {
  for (int r = 0; r < world; ++r) { /* check_workers :158-168 */
    float* tmp = (float*)malloc(n ? n * sizeof(float) : 1);
    int st = oracle_dequantize(codes[r], scales[r], n, 8, block, ORC_FP8, tmp,
                               err, errlen);
    free(tmp);
    if (st) return st;
  }
  uint64_t* ranges = (uint64_t*)malloc(sizeof(uint64_t) * 2 * world);
  oracle_chunk_assignment(n, block, world, ranges);
  int st = ORC_OK;
  for (int r = 0; r < world && st == ORC_OK; ++r) {
    const size_t begin = ranges[2 * r], end = ranges[2 * r + 1];
    if (begin == end) continue;
    const size_t len = end - begin, b0 = begin / block;
    const size_t nbl = (len + block - 1) / block;
    float* acc = (float*)calloc(len, sizeof(float));
    float* piece = (float*)malloc(len * sizeof(float));
    for (int s = 0; s < world; ++s) {
      oracle_dequantize(codes[s] + begin, scales[s] + b0, len, 8, block,
                        ORC_FP8, piece, NULL, 0);
      for (size_t i = 0; i < len; ++i) acc[i] += piece[i];
    }
    for (size_t i = 0; i < len; ++i)
      if (!isfinite(acc[i])) {
        st = set_err(err, errlen, ORC_RUNTIME_ERROR,
                     "all-reduce aborted: fp32 overflow during local reduce");
        break;
      }
    if (st == ORC_OK)
      st = oracle_quantize(acc, len, 8, block, ORC_FP8, out_codes + begin,
                           out_scales + b0, err, errlen);
    (void)nbl;
    free(acc);
    free(piece);
  }
  free(ranges);
  return st;
}

/* :338-431 allreduce_naive_fp8 ring strawman: P-1 steps adding in FP8 at the
 * receiver's original fixed scale, sticky per-element saturation flags. */
int oracle_allreduce_naive(int world, size_t n, uint32_t block,
                           const uint8_t* const* codes,
                           const float* const* scales, uint8_t* out_codes,
                           float* out_scales, uint64_t* overflow_elements,
                           char* err, size_t errlen) {
  for (int r = 0; r < world; ++r) {
    float* tmp = (float*)malloc(n ? n * sizeof(float) : 1);
    int st = oracle_dequantize(codes[r], scales[r], n, 8, block, ORC_FP8, tmp,
                               err, errlen);
    free(tmp);
    if (st) return st;
  }
  const size_t nb = (n + block - 1) / block;
  uint64_t* ranges = (uint64_t*)malloc(sizeof(uint64_t) * 2 * world);
  oracle_chunk_assignment(n, block, world, ranges);
  uint8_t** wc = (uint8_t**)malloc(sizeof(uint8_t*) * world);
  float** ws = (float**)malloc(sizeof(float*) * world);
  uint8_t* sat = (uint8_t*)calloc(n ? n : 1, 1);
  uint8_t* msg_codes = (uint8_t*)malloc(n ? n : 1);
  float* msg_scales = (float*)malloc(sizeof(float) * (nb ? nb : 1));
  for (int r = 0; r < world; ++r) {
    wc[r] = (uint8_t*)malloc(n ? n : 1);
    ws[r] = (float*)malloc(sizeof(float) * (nb ? nb : 1));
    memcpy(wc[r], codes[r], n);
    memcpy(ws[r], scales[r], sizeof(float) * nb);
  }
  /* Messages are snapshots taken before any receiver updates (:359-368). */
  uint8_t** oc = (uint8_t**)malloc(sizeof(uint8_t*) * world);
  float** os = (float**)malloc(sizeof(float*) * world);
  for (int r = 0; r < world; ++r) {
    oc[r] = (uint8_t*)malloc(n ? n : 1);
    os[r] = (float*)malloc(sizeof(float) * (nb ? nb : 1));
  }
  for (int step = 0; step < world - 1; ++step) {
    for (int r = 0; r < world; ++r) {
      memcpy(oc[r], wc[r], n);
      memcpy(os[r], ws[r], sizeof(float) * nb);
    }
    for (int r = 0; r < world; ++r) {
      const int from = (r - 1 + world) % world;
      const int chunk = ((r - step - 1) % world + world) % world;
      const size_t begin = ranges[2 * chunk], end = ranges[2 * chunk + 1];
      for (size_t i = begin; i < end; ++i) {
        const size_t blk = i / block;
        const float in_scale = os[from][blk];
        const double incoming =
            oracle_code_unit_value(ORC_FP8, 8, oc[from][i]) * in_scale;
        const double local =
            oracle_code_unit_value(ORC_FP8, 8, wc[r][i]) * ws[r][blk];
        const double sum = incoming + local;
        const float scale = scales[r][blk];
        const double unit = scale == 0.0f ? 0.0 : sum / scale;
        int over = (scale == 0.0f && sum != 0.0);
        int ovf = 0;
        const uint8_t c = oracle_fp8_encode(unit * 448.0, &ovf);
        if (ovf) over = 1;
        if (over) sat[i] = 1;
        wc[r][i] = c;
        ws[r][blk] = scale;
      }
    }
  }
  for (int chunk = 0; chunk < world; ++chunk) {
    const int owner = world == 1 ? 0 : (chunk - 1 + world) % world;
    const size_t begin = ranges[2 * chunk], end = ranges[2 * chunk + 1];
    if (begin == end) continue;
    memcpy(out_codes + begin, wc[owner] + begin, end - begin);
    const size_t b0 = begin / block, b1 = (end + block - 1) / block;
    memcpy(out_scales + b0, ws[owner] + b0, sizeof(float) * (b1 - b0));
  }
  uint64_t cnt = 0;
  for (size_t i = 0; i < n; ++i) cnt += sat[i];
  if (overflow_elements) *overflow_elements = cnt;
  for (int r = 0; r < world; ++r) {
    free(wc[r]);
    free(ws[r]);
    free(oc[r]);
    free(os[r]);
  }
  free(wc);
  free(ws);
  free(oc);
  free(os);
  free(sat);
  free(msg_codes);
  free(msg_scales);
  free(ranges);
  (void)err;
  (void)errlen;
  return ORC_OK;
}

/* ---- dbca.hpp ------------------------------------------------------------ */
/* :17-29 PipelineConfig::check + :34-41 stored_activation_counts */
int oracle_stored_activation_counts(int n_stages, int micro_batches,
                                    int interleave, int* counts) {
  if (n_stages < 1 || micro_batches < 1 || interleave != 2)
    return ORC_INVALID_ARGUMENT;
  if (n_stages > 1 && micro_batches < 2 * n_stages) return ORC_INVALID_ARGUMENT;
  if (n_stages == 1) {
    counts[0] = 1;
    return ORC_OK;
  }
  for (int d = 1; d <= n_stages; ++d) counts[d - 1] = 3 * n_stages - 2 * d + 1;
  return ORC_OK;
}

/* :63-78 plan_bit_widths: raw = 4 Nmax / Ni, lround, clamp [4, 8] */
int oracle_plan_bit_widths(int n_stages, int micro_batches, int interleave,
                           int* counts, double* raw_bits, int* assigned) {
  int st = oracle_stored_activation_counts(n_stages, micro_batches, interleave,
                                           counts);
  if (st) return st;
  const int n = n_stages;
  const int n_max = counts[0];
  for (int i = 0; i < n; ++i) {
    raw_bits[i] = 4.0 * n_max / counts[i];
    const int r = (int)lround(raw_bits[i]);
    assigned[i] = r < 4 ? 4 : (r > 8 ? 8 : r);
  }
  return ORC_OK;
}

/* :139-168 plan_reuse_check */
int oracle_plan_reuse(int low_n, int low_mb, int high_n, int high_mb,
                      int* applied, double* peak, double* uniform4_peak,
                      int* pass) {
  if (low_n > high_n) return ORC_INVALID_ARGUMENT;
  int lc[64], la[64], hc[64];
  double lr[64];
  if (low_n > 64 || high_n > 64) return ORC_INVALID_ARGUMENT;
  int st = oracle_plan_bit_widths(low_n, low_mb, 2, lc, lr, la);
  if (st) return st;
  st = oracle_stored_activation_counts(high_n, high_mb, 2, hc);
  if (st) return st;
  for (int i = 0; i < high_n; ++i) applied[i] = 4;
  for (int i = 0; i < low_n; ++i) applied[high_n - 1 - i] = la[low_n - 1 - i];
  *peak = 0.0;
  *uniform4_peak = 0.0;
  for (int i = 0; i < high_n; ++i) {
    const double bp = (double)hc[i] * applied[i];
    if (bp > *peak) *peak = bp;
    if (hc[i] * 4.0 > *uniform4_peak) *uniform4_peak = hc[i] * 4.0;
  }
  *pass = 1;
  for (int i = 0; i < high_n; ++i)
    if ((double)hc[i] * applied[i] > *uniform4_peak + hc[i]) *pass = 0;
  return ORC_OK;
}
