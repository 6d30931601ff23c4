// Device building blocks of the FP8 gradient path shared by the accumulate,
// reduce-requant and fused all-reduce kernels (see grad_codec.cu).
#pragma once
#include "agq_common.cuh"

namespace agqk {

// collective.hpp:101-110 round_bf16 (integer RNE on the fp32 bits)
__device__ __forceinline__ float round_bf16_ref(float x) {
  uint32_t u = f2u(x);
  u += 0x7fffu + ((u >> 16) & 1u);
  return u2f(u & 0xffff0000u);
}
// collective.hpp:112-123 round_fp16: RNE to fp16, but |x| >= 65520 saturates
// to +-65504 (not inf); zero and non-finite pass through.
__device__ __forceinline__ float round_fp16_ref(float x) {
  if (x == 0.0f || !(fabsf(x) <= 3.402823466e38f)) return x;
  if (fabsf(x) >= 65520.0f) return copysignf(65504.0f, x);
  return __half2float(__float2half_rn(x));
}

template <int PREC>
__device__ __forceinline__ float apply_prec(float s) {
  if (PREC == AGQ_ACC_BF16) return round_bf16_ref(s);
  if (PREC == AGQ_ACC_FP16) return round_fp16_ref(s);
  return s;
}
// round_bf16_ref / round_fp16_ref of 16 FINITE sums in pairs: cvt.rn.bf16x2
// (RNE; overflow to inf like the integer rule) and cvt.rn.satfinite.f16x2
// (RNE; |x| >= 65520 -> +-65504, the reference's saturation), then back to
// FP32 exactly.
template <int PREC>
__device__ __forceinline__ void round_pairs16(float (&v)[16]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t d;
    if (PREC == AGQ_ACC_BF16) {
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(v[2 * k + 1]), "f"(v[2 * k]));
      v[2 * k] = u2f(d << 16);
      v[2 * k + 1] = u2f(d & 0xffff0000u);
    } else {
      asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(v[2 * k + 1]), "f"(v[2 * k]));
      asm("{\n.reg .b16 a, b;\nmov.b32 {a, b}, %2;\ncvt.f32.f16 %0, a;\ncvt.f32.f16 %1, b;\n}"
          : "=f"(v[2 * k]), "=f"(v[2 * k + 1])
          : "r"(d));
    }
  }
}

// Exact FP8 decode with an FP32 block scale, (float)(fl64(e4m3(c)/448)*(double)s):
// a shared table of the signed unit values fl64(e4m3(c)/448) for every code
// (NaN for 0x7f/0xff) + DMUL + F2F. (A 16-entry table with two DMULs and an
// integer double->float rounding are verified equal in
// tests/cpp/numerics_check.cpp and measured slower,
// profiles/r01_microbench_fp8_decode_variants.log.)
constexpr int kDqTable = 256;
__device__ __forceinline__ void fill_fp8_dq_table(double* t) {
  for (int c = threadIdx.x; c < 256; c += blockDim.x)
    t[c] = ((c & 0x7f) == 0x7f) ? __longlong_as_double(0x7ff8000000000000LL)
                                : (double)e4m3_value((uint32_t)c) / 448.0;
}
__device__ __forceinline__ float fp8_dequant(uint32_t c, double sd, const double* t, bool) {
  return d2f_rn(dmul(t[c & 0xffu], sd));
}
// Signed-LUT decode: one LDS.64 + DMUL + F2F, the sign rides in the table
// (-0.0 * s = -0.0 as in the reference).
__device__ __forceinline__ float fp8_dq_lut(uint32_t c, double sd, const double* t) {
  return d2f_rn(dmul(t[c & 0xffu], sd));
}
// byte k of w (PRMT)
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)k);
}

// Gradient decode through a per-block 8-entry table (dq_tab_accum) where the
// block allows it, else the 256-entry signed unit table; both exact. The
// multi-piece reduce kernels and the FP32-local K3 use the block table
// (profiles/r01_reduce_tab_ab.log, r01_acc_tab_ab2.log).
// ---- f16-route block-table decode (every code, no per-code safety test) ----
// The hardware cvt.rn.f16x2.e4m3x2 gives every E4M3 value v exactly; as an
// FP32 value v = sign * (1 + M/8) * 2^X with a 3-bit M for EVERY code
// (normal, subnormal: m * 2^-9 renormalised, zero: 0). The reference's
// (float)(fl64(v / 448) * (double)s) = fl32(fl64((8+M)/7) * s) * 2^(X-9)
// (powers of two commute with both roundings while the results stay normal,
// i.e. s in [2^-60, 2^60], dq_fast), so with the block table
// T[M] = fl32(fl64((8+M)/7) * s) * 2^-9 the decode is T[M] * (v & sign|exp),
// an exact product, added with one FFMA. Zero codes give +-0 exactly, NaN
// codes an infinite product (the sum is then non-finite: the reference's
// abort). Table address from the f16 mantissa bits.
__device__ __forceinline__ float fp8_tab_entry_f16(double t8, float s) {
  return fmul(fp8_tab_entry(t8, s), 0x1p-9f);  // exact: the entry is a normal float
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
// acc[4i + b] = fadd(acc[4i + b], dq(code b of w[i])) through this lane's
// block table at shared address tb_s (8 floats, 32-byte aligned, so the
// entry address is one LOP3: (mantissa bits & 0x1c) | tb_s).
template <int NW>
__device__ __forceinline__ void dq_f16_accum(const uint32_t (&w)[NW], uint32_t tb_s,
                                             float (&acc)[4 * NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    uint32_t h[2];
    asm("{\n.reg .b16 lo, hi;\nmov.b32 {lo, hi}, %2;\ncvt.rn.f16x2.e4m3x2 %0, lo;\n"
        "cvt.rn.f16x2.e4m3x2 %1, hi;\n}"
        : "=r"(h[0]), "=r"(h[1])
        : "r"(w[i]));
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      // sign | exponent of both halves (one LOP3), then to FP32: p = +-2^X
      // exactly (every E4M3 value is an f16 normal or zero; NaN -> inf)
      float p0, p1;
      asm("{\n.reg .b16 a, b;\nmov.b32 {a, b}, %2;\ncvt.f32.f16 %0, a;\ncvt.f32.f16 %1, b;\n}"
          : "=f"(p0), "=f"(p1)
          : "r"(h[k] & 0xfc00fc00u));
      // f16 mantissa bits 7-9 (23-25) -> byte offset M * 4; the second shift
      // as a multiply-high (FMA pipe) to offload the integer ALU pipe
      const float e0 = lds_f32(((h[k] >> 5) & 0x1cu) | tb_s);
      const float e1 = lds_f32((__umulhi(h[k], 1u << 11) & 0x1cu) | tb_s);
      const f32x2 a = fma2(pk2(e0, e1), pk2(p0, p1),
                           pk2(acc[4 * i + 2 * k], acc[4 * i + 2 * k + 1]));
      up2(a, acc[4 * i + 2 * k], acc[4 * i + 2 * k + 1]);
    }
  }
}

// A block scale for which the block-table decode is exact (zero blocks excluded).
__device__ __forceinline__ bool dq_fast(float s) { return s >= kFastLo && s <= kFastHi; }

// acc[e] = fadd(acc[e], dequant(code e of w, sc)) for the N codes of one
// block piece through the 256-entry table (zero / subnormal / NaN codes and
// extreme scales). (Rounding part of the elements on the integer pipes
// instead of F2F measured slower, profiles/r01_dq_split.log.)
template <int N>
__device__ __forceinline__ void dq_accum(const uint32_t (&w)[N / 4], float sc, const double* t,
                                         float (&acc)[N]) {
  const double sd = (double)sc;
#pragma unroll
  for (int e = 0; e < N; ++e) acc[e] = fadd(acc[e], fp8_dq_lut(byte_of(w[e >> 2], e & 3), sd, t));
}

// Requantize 16 fp32 values of a block whose absmax is `a` (all 8 threads of
// the block agree on a): returns 4 words of codes (element e in byte e).
//
// Fast scales: the hardware RNE conversion of s*inv*(1 +- 2^-21). The two
// perturbed products bracket y = 448 s / a (their relative offsets exceed the
// 2^-22 error of fl(fl(448/a) s)), so when both convert to the same code C,
// every value in between — y included — rounds to C, which is then the
// reference's code (a tie would split the bracket). Pairs whose brackets
// split (an E4M3 midpoint within ~2^-20 relative of y) are recomputed with
// the exact comparison fp8_code. Subnormal E4M3 and saturation need no
// special case: RNE with satfinite is monotone over the whole range.
template <int NW>  // NW code words = 4 * NW values
__device__ __forceinline__ void fp8_requant_words(const float (&v)[4 * NW], float a,
                                                  uint32_t (&w)[NW]) {
  if (a == 0.0f) {
#pragma unroll
    for (int k = 0; k < NW; ++k) w[k] = 0u;
    return;
  }
  if (fast_scale(a)) {
    const float inv = fdiv(448.0f, a);
    const float ip = fmul(inv, 1.0f + 0x1p-21f), im = fmul(inv, 1.0f - 0x1p-21f);
    const f32x2 ip2 = pk2(ip, ip), im2 = pk2(im, im);
    uint32_t wm[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      // 4 codes per word: two paired conversions, halves joined by one PRMT
      float p[4], m[4];
      up2(mul2(pk2(v[4 * k], v[4 * k + 1]), ip2), p[0], p[1]);
      up2(mul2(pk2(v[4 * k + 2], v[4 * k + 3]), ip2), p[2], p[3]);
      up2(mul2(pk2(v[4 * k], v[4 * k + 1]), im2), m[0], m[1]);
      up2(mul2(pk2(v[4 * k + 2], v[4 * k + 3]), im2), m[2], m[3]);
      w[k] = cvt_e4m3x4(p[0], p[1], p[2], p[3]);
      wm[k] = cvt_e4m3x4(m[0], m[1], m[2], m[3]);
    }
    // one word-level test; pairs whose brackets split are recomputed exactly
    uint32_t diff = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) diff |= w[k] ^ wm[k];
    if (diff) {  // rare; unrolled so v/w stay in registers
#pragma unroll
      for (int k = 0; k < 2 * NW; ++k) {
        const int sh = (k & 1) * 16;
        if (((w[k >> 1] ^ wm[k >> 1]) >> sh) & 0xffffu) {
          const uint32_t c2 = fp8_code(v[2 * k], a, inv) | (fp8_code(v[2 * k + 1], a, inv) << 8);
          w[k >> 1] = (w[k >> 1] & ~(0xffffu << sh)) | (c2 << sh);
        }
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      w[k] = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) w[k] |= encode_double(2, 8, v[4 * k + e], a) << (8 * e);
    }
  }
}
__device__ __forceinline__ void fp8_requant16(const float (&v)[16], float a, uint32_t (&w)[4]) {
  fp8_requant_words<4>(v, a, w);
}

// |x| bits of the block absmax: the maximum of (bits << 1) (the shift drops
// the sign; IMAD.SHL on the FMA pipe instead of a LOP3 on the integer ALU)
// then >> 1. Non-finite values (inf / NaN) compare above every finite one.
__device__ __forceinline__ uint32_t absmax_bits16(const float (&v)[16]) {
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) m = max(m, f2u(v[e]) * 2u);
  m >>= 1;
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 4));
  return m;
}

// K4 piece table: pieces in ascending sender rank; outputs possibly remote.
struct PieceTable {
  const uint8_t* codes[AGQ_MAX_WORLD];
  const float* scales[AGQ_MAX_WORLD];
  uint8_t* out_codes[AGQ_MAX_WORLD];
  float* out_scales[AGQ_MAX_WORLD];
  int np, nout;
};

// Fill this warp's per-piece block tables (dq_f16_accum) after the previous
// group's lookups are done: 8 lanes per 128-block, lane l builds entry (l & 7)
// of warp-local block l / 8, so a piece table is 4 blocks x 8 entries. Blocks
// past the end build from scale 0 (unused).
template <int NP>
__device__ __forceinline__ void build_tables(float* wtab, const float (&sc)[NP]) {
  const int lane = threadIdx.x & 31;
  const double t8 = fp8_t8(lane & 7);
  __syncwarp();
#pragma unroll
  for (int p = 0; p < NP; ++p) wtab[p * 32 + lane] = fp8_tab_entry_f16(t8, sc[p]);
  __syncwarp();
}
// shared address of this lane's block table for piece p
__device__ __forceinline__ uint32_t lane_tab(const float* wtab, int p) {
  return (uint32_t)__cvta_generic_to_shared(wtab + p * 32 + ((threadIdx.x & 31) >> 3) * 8);
}

// Bad block scale of the all-reduce's inputs: the reference validates the
// workers in order (collective.hpp:158-168 check_workers -> validate), so the
// error is the lowest block of the lowest sender with a bad scale; the record
// holds (sender << 40) | block and agq_errors_message prints the block.
__device__ __forceinline__ long long bad_scale_key(uint32_t piece_mask, long long blk) {
  return ((long long)(__ffs(piece_mask) - 1) << 40) | blk;
}
__device__ __forceinline__ uint32_t bad_scale_bit(float s, int p) {
  return (uint32_t)(!(s >= 0.0f) || !(s <= 3.402823466e38f)) << p;
}

// Absmax, error records, FP8 requant and the stores of one 16-element group.
__device__ __forceinline__ void reduce_finish(const PieceTable& pt, uint64_t e0, uint64_t len,
                                              bool whole, bool in_range, uint64_t blk,
                                              uint32_t sbad, float (&acc)[16],
                                              long long blk_base, agq_errors* err);

// Decode + FP32 sum + requant + stores of one 16-element group whose NP
// pieces' code words (cv) and block scales (sc) are already in registers.
// Every lane of the warp must call (the table build synchronises the warp).
template <int NP>
__device__ __forceinline__ void reduce_compute(const PieceTable& pt, uint64_t e0, uint64_t len,
                                               bool whole, const uint4 (&cv)[NP],
                                               const float (&sc)[NP], long long blk_base,
                                               const double* t16, agq_errors* err, float* wtab) {
  const uint64_t blk = e0 / kBlock;
  const bool in_range = e0 < len;
  float acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
  uint32_t sbad = 0;
  if (wtab != nullptr) build_tables<NP>(wtab, sc);  // all lanes
  if (in_range) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      sbad |= bad_scale_bit(sc[p], p);
      const uint32_t w[4] = {cv[p].x, cv[p].y, cv[p].z, cv[p].w};
      if (wtab != nullptr && dq_fast(sc[p])) {
        dq_f16_accum<4>(w, lane_tab(wtab, p), acc);
      } else {
        dq_accum<16>(w, sc[p], t16, acc);
      }
    }
    // elements past the end contribute nothing to the absmax
    if (!whole)
      for (int e = 0; e < 16; ++e)
        if (e0 + e >= len) acc[e] = 0.0f;
  }
  reduce_finish(pt, e0, len, whole, in_range, blk, sbad, acc, blk_base, err);
}

// ---------------------------------------------------------------------------
// K4: block-128 reduce-requant, 16 elements per thread, direct loads.
// ---------------------------------------------------------------------------
// One 16-element group: loads of every piece first (memory-level
// parallelism), then the fp32 sum in ascending piece order from +0.0f.
// wtab (NP > 0): this warp's block tables, NP x 32 floats (4 blocks x 8
// entries per piece), or nullptr for the full-table decode only. Every lane
// of the warp must call (the table build synchronises the warp).
template <int NP>
__device__ __forceinline__ void reduce_group(const PieceTable& pt, uint64_t g, uint64_t len,
                                             long long blk_base, const double* t16,
                                             agq_errors* err, bool vec, float* wtab = nullptr) {
  const uint64_t e0 = g * 16;
  const uint64_t blk = e0 / kBlock;
  const bool in_range = e0 < len;
  const bool whole = vec && e0 + 16 <= len;
  if constexpr (NP > 0) {
    uint4 cv[NP];
    float sc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      cv[p] = make_uint4(0, 0, 0, 0);
      // every lane of an existing block loads its scale: a lane past the end
      // of a partial last block still builds its table entry for the others
      sc[p] = blk * kBlock < len ? pt.scales[p][blk] : 0.0f;
      if (!in_range) continue;
      if (whole) {
        cv[p] = *reinterpret_cast<const uint4*>(pt.codes[p] + e0);
      } else {
        uint32_t w[4] = {0, 0, 0, 0};
        for (int e = 0; e < 16 && e0 + e < len; ++e)
          w[e >> 2] |= (uint32_t)pt.codes[p][e0 + e] << (8 * (e & 3));
        cv[p] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    reduce_compute<NP>(pt, e0, len, whole, cv, sc, blk_base, t16, err, wtab);
  } else {
    const int np = pt.np;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
    uint32_t sbad = 0;
    if (in_range) {
#pragma unroll 1
      for (int p = 0; p < np; ++p) {
        const float scp = pt.scales[p][blk];
        sbad |= bad_scale_bit(scp, p);
        uint32_t w[4] = {0, 0, 0, 0};
        if (whole) {
          const uint4 v = *reinterpret_cast<const uint4*>(pt.codes[p] + e0);
          w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {
          for (int e = 0; e < 16 && e0 + e < len; ++e)
            w[e >> 2] |= (uint32_t)pt.codes[p][e0 + e] << (8 * (e & 3));
        }
        dq_accum<16>(w, scp, t16, acc);
      }
      if (!whole)
        for (int e = 0; e < 16; ++e)
          if (e0 + e >= len) acc[e] = 0.0f;
    }
    reduce_finish(pt, e0, len, whole, in_range, blk, sbad, acc, blk_base, err);
  }
}

__device__ __forceinline__ void reduce_finish(const PieceTable& pt, uint64_t e0, uint64_t len,
                                              bool whole, bool in_range, uint64_t blk,
                                              uint32_t sbad, float (&acc)[16],
                                              long long blk_base, agq_errors* err) {
  const uint32_t m = absmax_bits16(acc);
  const int sub = threadIdx.x & 7;
  if (in_range && sub == 0) {
    if (sbad) err_min(&err->bad_scale_block, bad_scale_key(sbad, blk_base + (long long)blk));
    if (m >= 0x7f800000u) err_min(&err->overflow_block, blk_base + (long long)blk);
  }
  if (!in_range) return;
  const float a = u2f(m);
  uint32_t ow[4];
  if (m >= 0x7f800000u) {
    ow[0] = ow[1] = ow[2] = ow[3] = 0;
  } else {
    fp8_requant16(acc, a, ow);
  }
  for (int o = 0; o < pt.nout; ++o) {
    if (whole) {
      *reinterpret_cast<uint4*>(pt.out_codes[o] + e0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    } else {
      for (int e = 0; e < 16 && e0 + e < len; ++e)
        pt.out_codes[o][e0 + e] = (uint8_t)(ow[e >> 2] >> (8 * (e & 3)));
    }
    if (sub == 0) pt.out_scales[o][blk] = a;
  }
}

}  // namespace agqk
