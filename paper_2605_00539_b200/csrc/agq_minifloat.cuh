// Fast exact activation paths for the FP4 E2M1 and FP8 E4M3 codecs
// (quantize.hpp:128-133, :142-155, :178-189): one warp lane row = 32
// consecutive elements of one block.
//
// Encode: the hardware RNE/satfinite conversion of y*(1 +- 2^-21), y =
// x * fl(den/a) (den = 6 or 448), brackets the exact y = den*x/a (the
// product's relative error is below 2^-22), so when both ends convert to the
// same code that code is the reference's RNE of y (a midpoint splits the
// bracket); split pairs are recomputed with the exact comparisons
// (fp4_code / fp8_code). FP4 additionally maps -0 (0x8) to +0 as the
// reference does.
//
// Decode: codes -> f16x2 in hardware (exact for every E2M1 / E4M3 value),
// f16 -> f32, then (v*s)/den with the Markstein correction proven equal to
// (float)(fl64(v/den)*s) for BF16-valued scales in [2^-60, 2^60]; the
// correction is sign-symmetric, so only -0 needs its sign restored.
#pragma once

#include "agq_grad.cuh"

namespace agqk {

// (lo, hi) values of a pair of E2M1 codes (low nibble = lo)
__device__ __forceinline__ void e2m1x2_to_f32(uint32_t b8, float& lo, float& hi) {
  uint32_t h;
  asm("{\n.reg .b8 t;\nmov.b32 {t, _, _, _}, %1;\ncvt.rn.f16x2.e2m1x2 %0, t;\n}"
      : "=r"(h)
      : "r"(b8));
  lo = __half2float(__ushort_as_half((unsigned short)(h & 0xffffu)));
  hi = __half2float(__ushort_as_half((unsigned short)(h >> 16)));
}
// (lo, hi) values of a pair of E4M3 codes (low byte = lo)
__device__ __forceinline__ void e4m3x2_to_f32(uint32_t b16, float& lo, float& hi) {
  uint32_t h;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"((unsigned short)b16));
  lo = __half2float(__ushort_as_half((unsigned short)(h & 0xffffu)));
  hi = __half2float(__ushort_as_half((unsigned short)(h >> 16)));
}

// exact per-nibble / per-byte "equals 0x8 / 0x08" masks (no cross-field carry)
__device__ __forceinline__ uint32_t nibbles_eq8(uint32_t w) {
  const uint32_t t = w ^ 0x88888888u;
  return ~(((t & 0x77777777u) + 0x77777777u) | t) & 0x88888888u;
}
__device__ __forceinline__ uint32_t bytes_eq8(uint32_t w) {
  const uint32_t t = w ^ 0x08080808u;
  return (~(((t & 0x7f7f7f7fu) + 0x7f7f7f7fu) | t) & 0x80808080u) >> 4;
}

// Byte / nibble "field != 0" masks (bit 7 of each byte / bit 3 of each
// nibble), exact (no carry between fields).
__device__ __forceinline__ uint32_t bytes_nz(uint32_t t) {
  return (((t & 0x7f7f7f7fu) + 0x7f7f7f7fu) | t) & 0x80808080u;
}
__device__ __forceinline__ uint32_t nibbles_nz(uint32_t t) {
  return (((t & 0x77777777u) + 0x77777777u) | t) & 0x88888888u;
}

// BF16 x and BF16-valued a: den*x and M*a (M an E4M3 / E2M1 midpoint) have
// at most ~13 significant bits, so y = den*x/a is either exactly a midpoint
// or at least ~2^-13 (relative) away from every midpoint — far outside the
// 2^-21 bracket. A split bracket is therefore an exact tie between the two
// adjacent codes wm (smaller magnitude) and wp, resolved branch-free with the
// reference's tie rule.
// E2M1: ties to the even code.
__device__ __forceinline__ uint32_t fp4_resolve_ties(uint32_t wp, uint32_t wm, bool bytes) {
  if (bytes) {  // one code per byte
    const uint32_t split = bytes_nz(wp ^ wm);
    const uint32_t pick = split & ((wm & 0x01010101u) << 7);  // wm odd -> wp
    const uint32_t m = (pick >> 7) * 0xffu;
    return (wp & m) | (wm & ~m);
  }
  const uint32_t split = nibbles_nz(wp ^ wm);
  const uint32_t pick = split & ((wm & 0x11111111u) << 3);
  const uint32_t m = (pick >> 3) * 0xfu;
  return (wp & m) | (wm & ~m);
}
// E4M3 (fp8.hpp:32-66 via fl64 double rounding): ties to even, except the 14
// midpoints between mantissa 6 and 7 in exponent fields 1..14, which go to
// the odd code.
__device__ __forceinline__ uint32_t fp8_resolve_ties(uint32_t wp, uint32_t wm) {
  const uint32_t split = bytes_nz(wp ^ wm);
  const uint32_t L = wm & 0x7f7f7f7fu;
  const uint32_t odd = (L & 0x01010101u) << 7;
  const uint32_t is6 = ~bytes_nz((L & 0x07070707u) ^ 0x06060606u) & 0x80808080u;
  const uint32_t e = (L >> 3) & 0x0f0f0f0fu;
  const uint32_t mid_exp = bytes_nz(e) & bytes_nz(e ^ 0x0f0f0f0fu);  // e in 1..14
  const uint32_t pick = split & (odd | (is6 & mid_exp));
  const uint32_t m = (pick >> 7) * 0xffu;
  return (wp & m) | (wm & ~m);
}

// FP4 E2M1 encode of 16 consecutive values of a lane row into PACK / 2 words
// (PACK 4: two codes per byte, 8: one code per byte). a > 0.
template <int PACK, bool BF16IN>
__device__ __forceinline__ void fp4_encode16(const float (&v)[16], float a,
                                             uint32_t (&w)[PACK / 2]) {
  constexpr int NWD = PACK / 2;
  if (!fast_scale(a)) {
#pragma unroll
    for (int k = 0; k < NWD; ++k) w[k] = 0u;
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e * PACK / 32] |= encode_double(1, 4, v[e], a) << ((e * PACK) & 31);
    return;
  }
  const float inv = fdiv(6.0f, a);
  const float ip = fmul(inv, 1.0f + 0x1p-21f), im = fmul(inv, 1.0f - 0x1p-21f);
  const f32x2 ip2 = pk2(ip, ip), im2 = pk2(im, im);
  uint32_t wm[NWD];
#pragma unroll
  for (int k = 0; k < NWD; ++k) w[k] = wm[k] = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const f32x2 x = pk2(v[2 * k], v[2 * k + 1]);
    float p0, p1, m0, m1;
    up2(mul2(x, ip2), p0, p1);
    up2(mul2(x, im2), m0, m1);
    uint32_t cp = cvt_e2m1x2(p0, p1), cm = cvt_e2m1x2(m0, m1);
    if constexpr (PACK == 8) {  // one code per byte
      cp = (cp & 0xfu) | ((cp & 0xf0u) << 4);
      cm = (cm & 0xfu) | ((cm & 0xf0u) << 4);
      w[k >> 1] |= cp << (16 * (k & 1));
      wm[k >> 1] |= cm << (16 * (k & 1));
    } else {
      w[k >> 2] |= cp << (8 * (k & 3));
      wm[k >> 2] |= cm << (8 * (k & 3));
    }
  }
  if constexpr (BF16IN) {  // a split is an exact tie: branch-free
#pragma unroll
    for (int k = 0; k < NWD; ++k) w[k] = fp4_resolve_ties(w[k], wm[k], PACK == 8);
  } else {
  uint32_t diff = 0;
#pragma unroll
  for (int k = 0; k < NWD; ++k) diff |= w[k] ^ wm[k];
  if (diff) {  // rare; unrolled so v/w stay in registers
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      constexpr uint32_t kField = PACK == 8 ? 0xffffu : 0xffu;
      const int wi = PACK == 8 ? (k >> 1) : (k >> 2);
      const int sh = PACK == 8 ? 16 * (k & 1) : 8 * (k & 3);
      if (((w[wi] ^ wm[wi]) >> sh) & kField) {
        const uint32_t c0 = fp4_code(v[2 * k], a), c1 = fp4_code(v[2 * k + 1], a);
        const uint32_t f = PACK == 8 ? (c0 | (c1 << 8)) : (c0 | (c1 << 4));
        w[wi] = (w[wi] & ~(kField << sh)) | (f << sh);
      }
    }
  }
  }
  // the hardware keeps the sign of zero; the reference encodes -0 as 0
#pragma unroll
  for (int k = 0; k < NWD; ++k) w[k] &= ~(PACK == 8 ? bytes_eq8(w[k]) : nibbles_eq8(w[k]));
}

// FP8 E4M3 encode of 16 values into 4 words. BF16 inputs: bracket + exact
// tie rule, branch-free; FP32 inputs: fp8_requant_words (exact fallback).
template <bool BF16IN>
__device__ __forceinline__ void fp8_encode16(const float (&v)[16], float a, uint32_t (&w)[4]) {
  if constexpr (!BF16IN) {
    fp8_requant_words<4>(v, a, w);
  } else {
    if (!fast_scale(a)) {
      fp8_requant_words<4>(v, a, w);  // literal double path inside
      return;
    }
    const float inv = fdiv(448.0f, a);
    const float ip = fmul(inv, 1.0f + 0x1p-21f), im = fmul(inv, 1.0f - 0x1p-21f);
    const f32x2 ip2 = pk2(ip, ip), im2 = pk2(im, im);
    uint32_t wm[4];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const f32x2 x = pk2(v[2 * k], v[2 * k + 1]);
      float p0, p1, m0, m1;
      up2(mul2(x, ip2), p0, p1);
      up2(mul2(x, im2), m0, m1);
      const uint32_t cp = cvt_e4m3x2(p0, p1), cm = cvt_e4m3x2(m0, m1);
      if (k & 1) {
        w[k >> 1] |= cp << 16;
        wm[k >> 1] |= cm << 16;
      } else {
        w[k >> 1] = cp;
        wm[k >> 1] = cm;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = fp8_resolve_ties(w[k], wm[k]);
  }
}

// Decode elements [e0, e0 + N) of a lane row (CODEC 1: E2M1 at PACK 4 or 8
// bits per code; CODEC 2: E4M3, one byte per code) for a fast BF16-valued
// scale s; FP8 rows holding a NaN code take the per-element path instead.
template <int CODEC, int PACK, int N>
__device__ __forceinline__ void minifloat_decode(const uint32_t (&w)[PACK], int e0, float s,
                                                 float (&v)[N]) {
  constexpr float kDen = CODEC == 2 ? 448.0f : 6.0f;
  const f32x2 s2 = pk2(s, s), den2 = pk2(-kDen, -kDen), rden2 = pk2(1.0f / kDen, 1.0f / kDen);
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const int pe = e0 / 2 + i;  // pair index in the row
    float lo, hi;
    if constexpr (CODEC == 2) {
      e4m3x2_to_f32((w[pe >> 1] >> (16 * (pe & 1))) & 0xffffu, lo, hi);
    } else if constexpr (PACK == 8) {
      const uint32_t h = (w[pe >> 1] >> (16 * (pe & 1))) & 0xffffu;
      e2m1x2_to_f32((h & 0xfu) | ((h >> 4) & 0xf0u), lo, hi);
    } else {
      e2m1x2_to_f32((w[pe >> 2] >> (8 * (pe & 3))) & 0xffu, lo, hi);
    }
    const f32x2 p = mul2(pk2(lo, hi), s2);
    const f32x2 q0 = mul2(p, rden2);
    const f32x2 r = fma2(q0, den2, p);
    float m0, m1, p0, p1;
    up2(fma2(r, rden2, q0), m0, m1);
    up2(p, p0, p1);
    // sign-symmetric correction: only -0 (p = -0) needs its sign back
    v[2 * i] = u2f(f2u(m0) | (f2u(p0) & 0x80000000u));
    v[2 * i + 1] = u2f(f2u(m1) | (f2u(p1) & 0x80000000u));
  }
}

// any E4M3 NaN code (0x7f / 0xff) in the row
template <int PACK>
__device__ __forceinline__ bool fp8_row_has_nan(const uint32_t (&w)[PACK]) {
  uint32_t any = 0;
#pragma unroll
  for (int k = 0; k < PACK; ++k) any |= (w[k] & 0x7f7f7f7fu) + 0x01010101u;
  return (any & 0x80808080u) != 0;
}

}  // namespace agqk
