"""Scalar E4M3 / E2M1 formats (fp8.hpp:14-114) on the host.

These are the reference's scalar conversions for host-side use (tables,
validation, the drop-in API). The device kernels use agq_numerics.cuh.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

kMaxFinite = 448.0
kNaNByte = 0x7F
kMaxFiniteByte = 0x7E
kFp4Magnitude = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)


@dataclass(frozen=True)
class Fp8EncodeResult:
    byte: int
    overflow: bool = False


def _rne(x: float) -> int:
    return int(round(x))  # Python round() is round-half-even


def fp8_encode(v: float) -> Fp8EncodeResult:
    """fp8.hpp:32-66: RNE, saturation to +-448 with an overflow flag."""
    sign = 0x80 if math.copysign(1.0, v) < 0 else 0
    if math.isnan(v):
        return Fp8EncodeResult(sign | kNaNByte)
    a = abs(v)
    if a > kMaxFinite:
        return Fp8EncodeResult(sign | kMaxFiniteByte, True)
    if a < 2.0 ** -6:
        q = _rne(a * 512.0)
        if q == 0:
            return Fp8EncodeResult(sign)
        return Fp8EncodeResult(sign | (q if q < 8 else 8))
    m, e = math.frexp(a)  # a = m 2^e, m in [0.5, 1)
    exp = e - 1
    q = _rne(math.ldexp(a, 3 - exp))
    if q == 16:
        q, exp = 8, exp + 1
    return Fp8EncodeResult(sign | ((exp + 7) << 3) | (q - 8))


def fp8_decode(b: int) -> float:
    """fp8.hpp:68-84."""
    sign = (b & 0x80) != 0
    ef, m = (b >> 3) & 0xF, b & 7
    if ef == 0xF and m == 7:
        return math.copysign(math.nan, -1.0 if sign else 1.0)
    mag = m * 2.0 ** -9 if ef == 0 else math.ldexp(8 + m, ef - 10)
    return -mag if sign else mag


def fp4_encode(v: float) -> int:
    """fp8.hpp:94-109: nearest E2M1, ties to the even index, -0 -> +0."""
    sign = 0x8 if math.copysign(1.0, v) < 0 else 0
    a = abs(v)
    if a >= 6.0:
        return sign | 7
    best, best_d = 0, a
    for i in range(1, 8):
        d = abs(a - kFp4Magnitude[i])
        if d < best_d or (d == best_d and i % 2 == 0):
            best, best_d = i, d
    return 0 if best == 0 else sign | best


def fp4_decode(c: int) -> float:
    m = kFp4Magnitude[c & 7]
    return -m if c & 8 else m
