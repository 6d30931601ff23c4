// Drop-in for agq/fp8.hpp (E4M3 / E2M1 scalar formats), host side.
// Same names and semantics as /root/reference/proj/include/agq/fp8.hpp:14-114:
// RNE encode with saturation (+overflow flag) for E4M3, nearest-with-ties-to-
// even-index for E2M1. The GPU kernels use csrc/agq_numerics.cuh instead.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>

namespace agq {

struct Fp8Value {
  std::uint8_t byte = 0;
  friend bool operator==(Fp8Value a, Fp8Value b) { return a.byte == b.byte; }
};

namespace fp8 {
constexpr double kMaxFinite = 448.0;
constexpr double kMinSubnormal = 0x1p-9;
constexpr double kMinNormal = 0x1p-6;
constexpr std::uint8_t kNaNByte = 0x7f;
constexpr std::uint8_t kMaxFiniteByte = 0x7e;
}  // namespace fp8

struct Fp8EncodeResult {
  Fp8Value value;
  bool overflow = false;
};

inline Fp8EncodeResult fp8_encode(double v) {
  const std::uint8_t s = std::signbit(v) ? 0x80 : 0x00;
  if (std::isnan(v)) return {Fp8Value{static_cast<std::uint8_t>(s | fp8::kNaNByte)}, false};
  const double m = std::fabs(v);
  if (m > fp8::kMaxFinite)
    return {Fp8Value{static_cast<std::uint8_t>(s | fp8::kMaxFiniteByte)}, true};
  if (m < fp8::kMinNormal) {  // quantum 2^-9; a quotient of 8 is the smallest normal
    const int q = static_cast<int>(std::nearbyint(std::ldexp(m, 9)));
    return {Fp8Value{static_cast<std::uint8_t>(s | (q > 8 ? 8 : q))}, false};
  }
  int e = std::ilogb(m);
  int q = static_cast<int>(std::nearbyint(std::ldexp(m, 3 - e)));  // 8..16
  if (q == 16) {
    q = 8;
    ++e;
  }
  return {Fp8Value{static_cast<std::uint8_t>(s | ((e + 7) << 3) | (q - 8))}, false};
}

inline double fp8_decode(Fp8Value b) {
  const int ef = (b.byte >> 3) & 0xf, mant = b.byte & 7;
  const bool neg = (b.byte & 0x80) != 0;
  if (ef == 0xf && mant == 7)
    return std::copysign(std::numeric_limits<double>::quiet_NaN(), neg ? -1.0 : 1.0);
  const double mag = ef == 0 ? mant * fp8::kMinSubnormal : std::ldexp(8 + mant, ef - 10);
  return neg ? -mag : mag;
}

namespace fp4 {
constexpr double kMaxFinite = 6.0;
inline constexpr double kMagnitude[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
}  // namespace fp4

inline std::uint8_t fp4_encode(double v) {
  const std::uint8_t s = std::signbit(v) ? 0x8 : 0x0;
  const double m = std::fabs(v);
  if (m >= fp4::kMaxFinite) return s | 0x7;
  // midpoints 0.25 .75 1.25 1.75 2.5 3.5 5; a tie goes to the even index
  static constexpr double kMid[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
  int idx = 0;
  for (int i = 0; i < 7; ++i)
    if (m > kMid[i] || (m == kMid[i] && ((i + 1) % 2 == 0))) idx = i + 1;
  return idx == 0 ? 0 : static_cast<std::uint8_t>(s | idx);
}

inline double fp4_decode(std::uint8_t code) {
  const double m = fp4::kMagnitude[code & 7];
  return (code & 8) ? -m : m;
}

}  // namespace agq
