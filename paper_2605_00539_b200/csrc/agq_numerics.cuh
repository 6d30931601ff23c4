// Exact-rounding element functions for the AGoQ block codecs.
//
// Every function here reproduces, bit for bit, the reference's double-
// precision formulas in /root/reference/proj/include/agq/quantize.hpp:118-135
// (encode) and :142-155,184-186 (decode) while running in FP32 on the fast
// path. They are __host__ __device__ so the SAME source is compiled for the
// host and checked exhaustively against the reference in
// tests/test_numerics.py (tools/numerics_check.cpp) before any GPU run.
//
// Preconditions of the fast paths (checked per block by the kernels, which
// fall back to the literal double-precision formula otherwise):
//   * block absmax a is finite and in [2^-60, 2^60]  (kFastLo..kFastHi)
//   * linear_code_bf16 / dq_*_bf16scale: x and a are BF16-representable.
#pragma once

#include <stdint.h>
#include <math.h>
#include <string.h>

#if defined(__CUDACC__)
#define AGQ_HD __host__ __device__ __forceinline__
#else
#define AGQ_HD inline
#endif

namespace agqk {

constexpr float kFastLo = 0x1p-60f;
constexpr float kFastHi = 0x1p60f;

// ---- primitive ops with explicit rounding (no FMA contraction) ----------
AGQ_HD float fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
AGQ_HD float fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
AGQ_HD float ffma(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
  return __fmaf_rn(a, b, c);
#else
  return fmaf(a, b, c);
#endif
}
AGQ_HD float fdiv(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdiv_rn(a, b);
#else
  return a / b;
#endif
}
AGQ_HD int rint_int(float v) {  // round to nearest, ties to even
#if defined(__CUDA_ARCH__)
  return __float2int_rn(v);
#else
  return (int)nearbyintf(v);
#endif
}
AGQ_HD float ffloor(float v) { return floorf(v); }

// Round-to-nearest-even to an integer for |v| < 2^22 with one FP32 add: the
// sum v + 1.5*2^23 is rounded by the adder (RNE, ties to even because the
// magic constant is even) and its low mantissa bits hold the integer.
constexpr float kMagicRound = 12582912.0f;   // 1.5 * 2^23, bits 0x4B400000
constexpr uint32_t kMagicBits = 0x4B400000u;
AGQ_HD uint32_t f2u(float f);
AGQ_HD float u2f(uint32_t u);
AGQ_HD uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
AGQ_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}
AGQ_HD double u64_to_d(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
AGQ_HD uint64_t d_to_u64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}
AGQ_HD float d2f_rn(double d) {
#if defined(__CUDA_ARCH__)
  return __double2float_rn(d);
#else
  return (float)d;
#endif
}
AGQ_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}

AGQ_HD int levels_of(int bits) { return (1 << (bits - 1)) - 1; }

AGQ_HD bool fast_scale(float a) { return a >= kFastLo && a <= kFastHi; }

// ---- SymmetricLinear encode (quantize.hpp:122-126) -----------------------
// Reference: k = nearbyint(fl64(fl64(x / a) * L)), which equals RNE of the
// real x*L/a (ties -> even) because the double error (2^-52) is far below
// the distance of any non-tie quotient from a half-integer.
//
// BF16 path: x*L and r are exact in FP32; one Newton step on v = x*(L/a)
// lands exactly on the half-integer at ties and within 2^-23 relative of
// the quotient otherwise (any non-tie quotient of BF16 operands is >= 2^-16
// relative from a half-integer), so rint() is exact.
// inv = fl32(L / a), rcp = fl32(1 / a).
AGQ_HD int linear_k_bf16(float x, float a, float inv, float rcp, float Lf) {
  const float v = fmul(x, inv);
  const float xl = fmul(x, Lf);            // exact: 8-bit x times 7-bit L
  const float r = ffma(-v, a, xl);         // exact residual x*L - v*a
  const float v2 = ffma(r, rcp, v);        // v + r/a: corrected quotient
  return (int)(f2u(fadd(v2, kMagicRound)) - kMagicBits);
}

// General FP32 path: decide against the candidate boundary h = floor(v)+1/2
// with an exact two-product comparison of x*L and h*a.
AGQ_HD int linear_k_f32(float x, float a, float inv, float Lf) {
  const float v = fmul(x, inv);
  const float f = ffloor(v);
  const float h = fadd(f, 0.5f);
  const float Q = fmul(h, a);
  const float q = ffma(h, a, -Q);          // h*a = Q + q exactly
  const float D = ffma(x, Lf, -Q);         // x*L - Q (exact near a tie)
  const int fi = (int)f;
  const int up = (D > q) | ((D == q) & (fi & 1));
  return fi + up;
}

// ---- FP8 E4M3 encode (quantize.hpp:131-133 + fp8.hpp:32-66) -------------
// Reference: fp8_encode(fl64(fl64(x / a) * 448)). At exact midpoints of the
// E4M3 grid, the two double roundings push the 14 mantissa-6/7 midpoints of
// exponent fields 1..14 UP to the odd code; every other midpoint is RNE.
// (Measured against the reference in tests/test_numerics.py.)
AGQ_HD uint32_t fp8_tie_up(uint32_t c_lo) {
  const uint32_t e = c_lo >> 3, m = c_lo & 7;
  return (c_lo & 1) | (uint32_t)(m == 6 && e >= 1 && e <= 14);
}

// Magnitude code of y = 448*|x|/a (0..0x7e): candidate interval from the
// FP32 estimate v, decided by an exact comparison of 448|x| with the
// interval's midpoint times a. ax = |x|, inv = fl32(448 / a).
AGQ_HD uint32_t fp8_mag_code(float ax, float a, float inv) {
  const float v = fmul(ax, inv);
  uint32_t c_lo;
  float M;
  if (v >= 0x1p-6f) {
    const uint32_t u = f2u(v);
    c_lo = (u >> 20) - (120u << 3);
    M = u2f((u & 0xfff00000u) | 0x00080000u);
    if (c_lo >= 0x7eu) {  // top of the format: nothing above 448
      c_lo = 0x7eu;
      M = 464.0f;
    }
  } else {
    c_lo = (uint32_t)fmul(v, 512.0f);  // truncation, 0..7
    M = fmul(fadd((float)c_lo, 0.5f), 0x1p-9f);
  }
  const float Q = fmul(M, a);
  const float q = ffma(M, a, -Q);
  const float D = ffma(ax, 448.0f, -Q);
  const uint32_t gt = D > q, eq = D == q;
  return c_lo + (gt | (eq & fp8_tie_up(c_lo)));
}

AGQ_HD uint32_t fp8_code(float x, float a, float inv448) {
  const uint32_t sign = (f2u(x) >> 24) & 0x80u;
  return sign | fp8_mag_code(fabsf(x), a, inv448);
}

// Hardware RNE-to-E4M3 with saturation at 448 (cvt.rn.satfinite.e4m3x2.f32)
// for two values; the host emulation is the reference's own RNE on the
// exactly-converted double (fp8.hpp:32-66 is pure RNE on its argument).
AGQ_HD uint32_t fp8_encode_double(double v);
#if defined(__CUDACC__)
// Four values -> four E4M3 codes in one word (element 0 in the low byte):
// two paired conversions, the halves joined in the register move.
__device__ __forceinline__ uint32_t cvt_e4m3x4(float a, float b, float c, float d) {
  uint32_t r;
  asm("{\n.reg .b16 lo, hi;\ncvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\n"
      "cvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\nmov.b32 %0, {lo, hi};\n}"
      : "=r"(r)
      : "f"(a), "f"(b), "f"(c), "f"(d));
  return r;
}
#endif
AGQ_HD uint32_t cvt_e4m3x2(float lo, float hi) {
#if defined(__CUDA_ARCH__)
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
#else
  return fp8_encode_double((double)lo) | (fp8_encode_double((double)hi) << 8);
#endif
}

// v = x * fl32(448/a) is within 2.0001 ulp(v) of y = 448x/a, so RNE(v) can
// differ from the reference only if a grid midpoint lies within 2 ulp of v
// (low 20 mantissa bits within +-2 of 0x80000) or v is in the E4M3 subnormal
// range. `near` flags a conservative superset (+-3) that takes fp8_code.
AGQ_HD bool fp8_near(float v) {
  const uint32_t au = f2u(v) & 0x7fffffffu;
  return ((au & 0xfffffu) - 0x7fffdu) < 7u || au < 0x3c800000u;
}

// ---- FP4 E2M1 encode (quantize.hpp:128-130 + fp8.hpp:94-109) -------------
// Nearest of {0,.5,1,1.5,2,3,4,6} for y = 6|x|/a, ties to the even index,
// -0 -> +0. Exact comparisons of 6|x| against the 7 midpoints times a.
AGQ_HD bool exact_gt_ge(float ax, float K, float M, float a, bool ge) {
  // sign(ax*K - M*a) via two-products; returns ax*K > M*a (or >= if ge).
  const float Q = fmul(M, a);
  const float q = ffma(M, a, -Q);
  const float D = ffma(ax, K, -Q);
  return ge ? (D >= q) : (D > q);
}

AGQ_HD uint32_t fp4_code(float x, float a) {
  const float ax = fabsf(x);
  uint32_t idx = 0;
  idx += exact_gt_ge(ax, 6.0f, 0.25f, a, false);
  idx += exact_gt_ge(ax, 6.0f, 0.75f, a, true);
  idx += exact_gt_ge(ax, 6.0f, 1.25f, a, false);
  idx += exact_gt_ge(ax, 6.0f, 1.75f, a, true);
  idx += exact_gt_ge(ax, 6.0f, 2.5f, a, false);
  idx += exact_gt_ge(ax, 6.0f, 3.5f, a, true);
  idx += exact_gt_ge(ax, 6.0f, 5.0f, a, false);
  if (idx == 0) return 0;
  return ((f2u(x) >> 28) & 0x8u) | idx;
}

// ---- literal double-precision encode (slow path, any finite a > 0) --------
AGQ_HD uint32_t fp8_encode_double(double v) {  // fp8.hpp:32-66, finite v
  const uint32_t sign = (d_to_u64(v) >> 56) & 0x80u;
  const double a = fabs(v);
  if (a > 448.0) return sign | 0x7eu;
  if (a < 0x1p-6) {
    const int q = (int)nearbyint(a * 0x1p9);
    if (q == 0) return sign;
    if (q < 8) return sign | (uint32_t)q;
    return sign | 8u;
  }
  int e = ilogb(a);
  int q = (int)nearbyint(ldexp(a, 3 - e));
  if (q == 16) {
    q = 8;
    ++e;
  }
  return sign | ((uint32_t)(e + 7) << 3) | (uint32_t)(q - 8);
}

AGQ_HD uint32_t fp4_encode_double(double v) {  // fp8.hpp:94-109
  const uint32_t sign = (d_to_u64(v) >> 60) & 0x8u;
  const double a = fabs(v);
  if (a >= 6.0) return sign | 7u;
  const double mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  int best = 0;
  double best_dist = a;
  for (int i = 1; i < 8; ++i) {
    const double d = fabs(a - mag[i]);
    if (d < best_dist || (d == best_dist && (i % 2 == 0))) {
      best_dist = d;
      best = i;
    }
  }
  if (best == 0) return 0;
  return sign | (uint32_t)best;
}

// codec: 0 linear, 1 fp4, 2 fp8. a > 0 finite.
AGQ_HD uint32_t encode_double(int codec, int bits, float x, float a) {
  const double t = (double)x / (double)a;
  if (codec == 0) {
    const int L = levels_of(bits);
    int k = (int)nearbyint(t * L);
    k = k < -L ? -L : (k > L ? L : k);
    return (uint32_t)(k + L);
  }
  if (codec == 1) return fp4_encode_double(t * 6.0);
  return fp8_encode_double(t * 448.0);
}

// One element, any FP32 x, block absmax a > 0 (finite). `inv` is the
// per-block reciprocal constant of the codec: L/a, 448/a (unused for fp4).
AGQ_HD uint32_t encode_f32(int codec, int bits, float x, float a, float inv) {
  if (!fast_scale(a)) return encode_double(codec, bits, x, a);
  if (codec == 0) {
    const int L = levels_of(bits);
    return (uint32_t)(linear_k_f32(x, a, inv, (float)L) + L);
  }
  if (codec == 1) return fp4_code(x, a);
  return fp8_code(x, a, inv);
}

AGQ_HD float codec_inv(int codec, int bits, float a) {
  if (codec == 0) return fdiv((float)levels_of(bits), a);
  if (codec == 2) return fdiv(448.0f, a);
  return fdiv(6.0f, a);
}

// ---- decode (quantize.hpp:142-155 code_unit_value, :184-186) -------------
// Reference: out = (float)(unit(c) * (double)scale), unit(c) in double.

// Hardware E2M1 conversion of a pair (cvt.rn.satfinite.e2m1x2.f32: RNE on
// the E2M1 grid, ties to the even code, saturate at 6, sign kept so -0 and
// negative underflow give 0x8): low nibble = lo. Host: the same rounding.
AGQ_HD uint32_t e2m1_rne_signed(float v) {  // host model of one lane of the cvt
  const float grid[8] = {0.0f, 0.5f, 1.0f, 1.5f, 2.0f, 3.0f, 4.0f, 6.0f};
  const float a = fabsf(v);
  uint32_t best = 7;
  if (a < 6.0f) {
    for (uint32_t i = 0; i < 7; ++i) {
      const float mid = 0.5f * (grid[i] + grid[i + 1]);  // exact in binary
      if (a < mid || (a == mid && (i & 1u) == 0)) {
        best = i;
        break;
      }
    }
  }
  return ((f2u(v) >> 28) & 0x8u) | best;
}
AGQ_HD uint32_t cvt_e2m1x2(float lo, float hi) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("{\n.reg .b8 t;\n"
      "cvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n"
      "mov.b32 %0, {t, 0, 0, 0};\n}"
      : "=r"(r)
      : "f"(hi), "f"(lo));
  return r & 0xffu;
#else
  return e2m1_rne_signed(lo) | (e2m1_rne_signed(hi) << 4);
#endif
}

// E4M3 magnitude of a code as float (exact).
AGQ_HD float e4m3_value(uint32_t c) {
  const uint32_t e = (c >> 3) & 0xfu, m = c & 7u;
  float mag = e == 0 ? fmul((float)m, 0x1p-9f)
                     : u2f(((e + 120u) << 23) | (m << 20));
  return (c & 0x80u) ? -mag : mag;
}
AGQ_HD float e2m1_value(uint32_t c) {
  const uint32_t i = c & 7u;
  const float mag = i < 4 ? fmul((float)i, 0.5f) : (i == 4 ? 2.0f : (i == 5 ? 3.0f : (i == 6 ? 4.0f : 6.0f)));
  return (c & 8u) ? -mag : mag;
}

// Literal reference formula (exact by construction). unit computed in double
// exactly as code_unit_value does.
AGQ_HD double unit_value_double(int codec, int bits, uint32_t c) {
  if (codec == 0) {
    const int L = levels_of(bits);
    return (double)((int)c - L) / L;
  }
  if (codec == 1) return (double)e2m1_value(c) / 6.0;
  const uint32_t e = (c >> 3) & 0xfu, m = c & 7u;
  if (e == 15 && m == 7) return (c & 0x80u) ? -NAN : NAN;
  return (double)e4m3_value(c) / 448.0;
}
AGQ_HD float dequant_double(int codec, int bits, uint32_t c, float s) {
  return d2f_rn(dmul(unit_value_double(codec, bits, c), (double)s));
}

// E4M3 unit values factor as U[c] = fl64(e4m3(c)/448) = T16[idx]*2^k with
// 16 doubles T16 = {fl64((8+m)/448), m<8} U {fl64(m/448), m<8} (exact power-
// of-two scaling in double): idx = m (+8 if subnormal), k = max(e,1) - 10.
// out = (float)(fl64(T16[idx]*s) * 2^k): the power-of-two DMUL is exact, so
// this equals the reference's (float)(U[c]*(double)s) for every FP32 s.
AGQ_HD double fp8_t16(int idx) {
  return idx < 8 ? (double)(8 + idx) / 448.0 : (double)(idx - 8) / 448.0;
}
AGQ_HD float fp8_dequant_t16(uint32_t c, double sd, const double* t16) {
  const uint32_t e = (c >> 3) & 0xfu, m = c & 7u;
  const uint32_t idx = m | (e == 0 ? 8u : 0u);
  const int k = (int)(e == 0 ? 1u : e) - 10;
  const double p = dmul(t16[idx], sd);
  const double pw = u64_to_d((uint64_t)(k + 1023) << 52);
  const float mag = d2f_rn(dmul(p, pw));
  const uint32_t nan = ((c & 0x7fu) == 0x7fu) ? 0x7fc00000u : 0u;
  return u2f((f2u(mag) | nan) ^ ((c & 0x80u) << 24));
}

// Same value without the (slow, 1/16-rate) F2F.F32.F64: P = fl64(T16*s) by
// one DMUL, then the power-of-two factor and round-to-nearest-even to FP32
// done on the bit pattern (valid while the result is a normal float, i.e. for
// block scales in [2^-60, 2^60]; P >= 0 because T16 >= 0 and s >= 0).
AGQ_HD float fp8_dequant_t16i(uint32_t c, double sd, const double* t16) {
  const uint32_t e = (c >> 3) & 0xfu, m = c & 7u;
  const uint32_t idx = m | (e == 0 ? 8u : 0u);
  const uint32_t ke = e == 0 ? 1u : e;  // 2^(ke-10)
  const uint64_t u = d_to_u64(dmul(t16[idx], sd));
  const uint64_t r = u + 0x0FFFFFFFull + ((u >> 29) & 1u);  // RNE at bit 29
  uint32_t f = (uint32_t)(r >> 29) - ((uint32_t)(1023 - 127 + 10 - (int)ke) << 23);
  f = (c & 0x7fu) == 0 ? 0u : f;
  f = (c & 0x7fu) == 0x7fu ? 0x7fc00000u : f;
  return u2f(f ^ ((c & 0x80u) << 24));
}

// RNE of a double to float on the bit pattern, for |p| = 0 or a normal float
// result (block scales in [2^-60, 2^60] guarantee that for every non-NaN
// E4M3 code times its scale): re-bias the exponent in the high word (clamped
// at 0 so +-0 stays 0), add half-minus-one + the guard LSB at bit 29 with
// carry, funnel-shift, restore the sign. A NaN input (E4M3 code 0x7f/0xff)
// saturates to a non-finite float (inf or NaN), which keeps every sum it
// enters non-finite — the only property the reduce paths observe. About 9
// integer ops instead of one
// F2F.F32.F64 (a 1/16-rate pipe); exact, see tests/cpp/numerics_check.cpp.
AGQ_HD float d2f_rn_bits(double p) {
  const uint64_t u = d_to_u64(p);
  const uint32_t lo = (uint32_t)u, hi = (uint32_t)(u >> 32);
  int32_t hb = (int32_t)(hi & 0x7fffffffu) - (int32_t)((1023 - 127) << 20);
  hb = hb < 0 ? 0 : (hb > 0x0FF00000 ? 0x0FF00000 : hb);  // NaN/huge -> non-finite
  const uint64_t mag = ((uint64_t)(uint32_t)hb << 32) | lo;
  const uint64_t r = mag + 0x0FFFFFFFull + ((lo >> 29) & 1u);
  return u2f((uint32_t)(r >> 29) | (hi & 0x80000000u));
}

// Per-block FP8 decode table (gradient paths). For a normal E4M3 code
// (exponent field e in 1..15, mantissa m) fl64(v/448) = fl64((8+m)/7)*2^(e-16)
// exactly, and power-of-two scaling commutes with both roundings while the
// float result stays normal, which block scales in [2^-60, 2^60] guarantee.
// So (float)(fl64(v/448)*s) = F[m] * 2^(e-16) with the 8-entry block table
// F[m] = (float)(fl64((8+m)/7) * s): one DMUL + F2F per entry instead of per
// element, and an exact FMUL per element. Zero/subnormal (e = 0) and NaN
// codes are excluded (callers route them to the full table).
AGQ_HD double fp8_t8(int m) { return (double)(8 + m) / 7.0; }
AGQ_HD float fp8_tab_entry(double t8, float s) { return d2f_rn(dmul(t8, (double)s)); }
// signed 2^(e-16) for code byte c (e >= 1): sign and exponent field moved
// into a float's sign and exponent with one arithmetic shift
AGQ_HD float fp8_pow2(uint32_t c) {
  const uint32_t y = (uint32_t)((int32_t)(c << 24) >> 4);
  return u2f((y & 0x87800000u) + 0x37800000u);
}
AGQ_HD float fp8_dq_tab(uint32_t c, const float* tab) { return fmul(tab[c & 7u], fp8_pow2(c)); }
// nonzero iff one of the 4 code bytes of w is zero/subnormal (e = 0) or NaN
AGQ_HD uint32_t fp8_tab_unsafe(uint32_t w) {
  const uint32_t u = w & 0x78787878u;
  const uint32_t z = (u - 0x01010101u) & ~u;            // byte with e == 0
  const uint32_t nn = (w & 0x7f7f7f7fu) + 0x01010101u;  // byte with low 7 bits all 1
  return (z | nn) & 0x80808080u;
}

// Fast path for BF16-valued scales in [2^-60, 2^60]: p = g*s is exact in
// FP32 (g has <= 8 significant bits), and the reference value equals the
// correctly rounded quotient p / den, computed by one Markstein correction
// with rden = fl32(1/den). Verified exhaustively over every code and every
// BF16 scale in range for every codec/width (tests/test_numerics.py).
// Sign handled outside so that -0 survives (the reference keeps -0.0 for the
// negative-zero FP4/FP8 codes).
AGQ_HD float div_const_rn(float p, float den, float rden) {
  const float ap = fabsf(p);
  const float q0 = fmul(ap, rden);
  const float r = ffma(-q0, den, ap);
  const float m = ffma(r, rden, q0);
  return u2f(f2u(m) | (f2u(p) & 0x80000000u));
}

AGQ_HD float dq_linear_bf16scale(int cprime, float s, float Lf, float rL) {
  return div_const_rn(fmul((float)cprime, s), Lf, rL);
}

AGQ_HD bool is_bf16_value(float s) { return (f2u(s) & 0xffffu) == 0; }

}  // namespace agqk
