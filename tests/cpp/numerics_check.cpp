// Exhaustive host-side check of the device element functions in
// paper_2605_00539_b200/csrc/agq_numerics.cuh (compiled here for the host,
// same source as the kernels) against the CPU oracle (oracle/liboracle.so,
// itself pinned to the reference by tests/test_oracle.py).
//
// Domains:
//   * encode, BF16 inputs: every BF16 x with |x| <= a, for every BF16
//     mantissa a in [1,2) and for a at the fast-path range edges.
//   * encode, FP32 inputs: random x plus adversarial near-boundary x.
//   * decode: every code x every BF16 scale in the fast range (BF16 path),
//     random FP32 scales (double path).
// Exit status 0 iff zero mismatches. Prints one line per category.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../oracle/agq_oracle.h"
#include "../../paper_2605_00539_b200/csrc/agq_numerics.cuh"

using namespace agqk;

static float bf16_to_f(uint16_t h) { return u2f((uint32_t)h << 16); }

// Reference code for x in a block whose absmax is exactly a (|x| <= a).
static uint8_t ref_code(int codec, int bits, float x, float a) {
  float blk[2] = {x, a};
  uint8_t c[2];
  float s;
  oracle_quantize(blk, 2, bits, 2, codec, c, &s, nullptr, 0);
  return c[0];
}

static long long g_fail = 0;

static void report(const char* what, long long n, long long bad) {
  std::printf("%-58s cases=%-10lld mismatches=%lld\n", what, n, bad);
  g_fail += bad;
}

// Fast-path device encode for BF16 operands (what the activation kernel runs).
static uint32_t dev_code_bf16(int codec, int bits, float x, float a) {
  const float inv = codec_inv(codec, bits, a);
  if (codec == 0) {
    // kernel form: one division per block, inv = L * (1/a)
    const int L = levels_of(bits);
    const float rcp = fdiv(1.0f, a);
    return (uint32_t)(linear_k_bf16(x, a, fmul((float)L, rcp), rcp, (float)L) + L);
  }
  return encode_f32(codec, bits, x, a, inv);
}

static void check_encode_bf16(int codec, int bits, float a_exp_scale,
                              const char* label) {
  long long n = 0, bad = 0, printed = 0;
  for (int am = 0; am < 128; ++am) {
    const float a = ldexpf(bf16_to_f((uint16_t)(0x3f80 | am)), (int)a_exp_scale);
    for (uint32_t h = 0; h < 0x8000; ++h) {
      const float ax = bf16_to_f((uint16_t)h);
      if (!(ax <= a)) continue;
      for (int sgn = 0; sgn < 2; ++sgn) {
        const float x = sgn ? -ax : ax;
        const uint8_t want = ref_code(codec, bits, x, a);
        const uint32_t got = dev_code_bf16(codec, bits, x, a);
        ++n;
        if (got != want) {
          ++bad;
          if (printed++ < 5)
            std::printf("  %s b=%d x=%a a=%a want=%u got=%u\n", label, bits,
                        x, a, want, got);
        }
      }
    }
  }
  char buf[128];
  std::snprintf(buf, sizeof buf, "encode bf16 %s bits=%d a*2^%d", label, bits,
                (int)a_exp_scale);
  report(buf, n, bad);
}

static void check_encode_f32(int codec, int bits, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> ua(0.5f, 4.0f);
  std::uniform_int_distribution<int> ue(-55, 55);
  std::uniform_real_distribution<float> ux(-1.0f, 1.0f);
  long long n = 0, bad = 0, printed = 0;
  const int L = levels_of(bits);
  for (int it = 0; it < 400000; ++it) {
    const float a = ldexpf(ua(rng), ue(rng));
    const float inv = codec_inv(codec, bits, a);
    float xs[24];
    int k = 0;
    xs[k++] = a * ux(rng);
    xs[k++] = -a;
    xs[k++] = a;
    // adversarial: near a decision boundary of the codec
    double bnd;
    if (codec == 0) {
      const int j = (int)(rng() % (2 * L)) - L;
      bnd = (j + 0.5) * (double)a / L;
    } else if (codec == 2) {
      const int c = (int)(rng() % 0x7e);
      bnd = (oracle_fp8_decode((uint8_t)c) + oracle_fp8_decode((uint8_t)(c + 1))) /
            2.0 * (double)a / 448.0;
    } else {
      static const double mids[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
      bnd = mids[rng() % 7] * (double)a / 6.0;
    }
    float b0 = (float)bnd;
    for (int d = -8; d <= 8; ++d) {
      float y = b0;
      if (d > 0) for (int t = 0; t < d; ++t) y = nextafterf(y, INFINITY);
      if (d < 0) for (int t = 0; t < -d; ++t) y = nextafterf(y, -INFINITY);
      if (std::fabs(y) <= a && k < 24) xs[k++] = (rng() & 1) ? y : -y;
    }
    for (int i = 0; i < k; ++i) {
      const float x = xs[i];
      const uint8_t want = ref_code(codec, bits, x, a);
      const uint32_t got = encode_f32(codec, bits, x, a, inv);
      ++n;
      if (got != want) {
        ++bad;
        if (printed++ < 5)
          std::printf("  f32 codec=%d b=%d x=%a a=%a want=%u got=%u\n", codec,
                      bits, x, a, want, got);
      }
    }
  }
  char buf[128];
  std::snprintf(buf, sizeof buf, "encode f32 codec=%d bits=%d (random+adversarial)",
                codec, bits);
  report(buf, n, bad);
}

// Exact ties between E4M3 neighbours: reference resolution per lower code.
static void check_fp8_ties() {
  long long n = 0, bad = 0;
  for (uint32_t c = 0; c < 0x7e; ++c) {
    const double m = (oracle_fp8_decode((uint8_t)c) +
                      oracle_fp8_decode((uint8_t)(c + 1))) / 2.0;
    // a = 448 scale, x = m exactly representable as float
    const float x = (float)m, a = 448.0f;
    if ((double)x != m) continue;
    const uint8_t want = ref_code(2, 8, x, a);
    const uint32_t got = fp8_code(x, a, fdiv(448.0f, a));
    ++n;
    if (got != want) {
      ++bad;
      std::printf("  tie c=%02x want=%02x got=%02x\n", c, want, got);
    }
  }
  report("fp8 exact midpoints (a=448)", n, bad);
}

static void check_decode(int codec, int bits) {
  long long n = 0, bad = 0, printed = 0;
  const int ncodes = 1 << bits;
  for (int e = -60; e < 60; ++e) {
    for (int sm = 0; sm < 128; ++sm) {
      const float s = ldexpf(bf16_to_f((uint16_t)(0x3f80 | sm)), e);
      std::vector<uint8_t> codes(ncodes);
      for (int c = 0; c < ncodes; ++c) codes[c] = (uint8_t)c;
      std::vector<float> want(ncodes);
      // one block holding every code, scale s
      oracle_dequantize(codes.data(), &s, ncodes, bits, ncodes, codec,
                        want.data(), nullptr, 0);
      for (int c = 0; c < ncodes; ++c) {
        float got;
        if (codec == 0) {
          const int L = levels_of(bits);
          got = dq_linear_bf16scale(c - L, s, (float)L, 1.0f / (float)L);
        } else if (codec == 1) {
          got = div_const_rn(fmul(e2m1_value(c), s), 6.0f, 1.0f / 6.0f);
        } else {
          if ((c & 0x7f) == 0x7f) continue;  // NaN codes handled separately
          got = div_const_rn(fmul(e4m3_value(c), s), 448.0f, 1.0f / 448.0f);
        }
        ++n;
        if (f2u(got) != f2u(want[c])) {
          ++bad;
          if (printed++ < 5)
            std::printf("  dq codec=%d b=%d c=%d s=%a want=%a got=%a\n", codec,
                        bits, c, s, want[c], got);
        }
      }
    }
  }
  char buf[128];
  std::snprintf(buf, sizeof buf, "decode bf16-scale fast path codec=%d bits=%d", codec,
                bits);
  report(buf, n, bad);
}

static void check_decode_double(uint64_t seed) {
  std::mt19937_64 rng(seed);
  long long n = 0, bad = 0;
  for (int it = 0; it < 20000; ++it) {
    const float s = u2f((uint32_t)(rng() % 0x7f000000u));
    uint8_t codes[256];
    float want[256];
    for (int c = 0; c < 256; ++c) codes[c] = (uint8_t)c;
    oracle_dequantize(codes, &s, 256, 8, 256, 2, want, nullptr, 0);
    for (int c = 0; c < 256; ++c) {
      if ((c & 0x7f) == 0x7f) continue;
      const float got = dequant_double(2, 8, c, s);
      ++n;
      if (f2u(got) != f2u(want[c])) ++bad;
    }
  }
  report("decode fp8 double path, random fp32 scales", n, bad);
}

// Blocks outside the fast range go through the literal double formula.
static void check_extreme(uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> ux(-1.0f, 1.0f);
  const float as[] = {0x1p-140f, 0x1.3p-127f, 0x1p-100f, 0x1.7p-61f,
                      0x1.1p61f,  0x1p100f,    0x1.fffffep127f};
  long long n = 0, bad = 0, dn = 0, dbad = 0;
  for (float a : as) {
    for (int codec = 0; codec < 3; ++codec)
      for (int bits = (codec == 2 ? 8 : 4); bits <= (codec == 1 ? 4 : 8); ++bits) {
        const float inv = codec_inv(codec, bits, a);
        for (int it = 0; it < 20000; ++it) {
          float x = a * ux(rng);
          if (it == 0) x = a;
          if (it == 1) x = -a;
          const uint8_t want = ref_code(codec, bits, x, a);
          const uint32_t got = encode_f32(codec, bits, x, a, inv);
          ++n;
          bad += got != want;
        }
        // decode with the same extreme scale
        const int nc = 1 << bits;
        std::vector<uint8_t> codes(nc);
        std::vector<float> want(nc);
        for (int c = 0; c < nc; ++c) codes[c] = (uint8_t)c;
        oracle_dequantize(codes.data(), &a, nc, bits, nc, codec, want.data(),
                          nullptr, 0);
        for (int c = 0; c < nc; ++c) {
          if (codec == 2 && (c & 0x7f) == 0x7f) continue;
          ++dn;
          dbad += f2u(dequant_double(codec, bits, c, a)) != f2u(want[c]);
        }
      }
  }
  report("encode slow path, extreme block scales", n, bad);
  report("decode double path, extreme scales, all codecs", dn, dbad);
}

// Fast FP8 encoder (hardware cvt on v + near-midpoint routing to fp8_code).
static uint32_t fp8_fast(float x, float a, float inv) {
  const float v = fmul(x, inv);
  if (fp8_near(v)) return fp8_code(x, a, inv);
  return cvt_e4m3x2(v, 0.0f) & 0xffu;
}

static void check_fp8_fast(uint64_t seed) {
  long long n = 0, bad = 0;
  // exhaustive BF16 domain at a in [1,2)
  for (int am = 0; am < 128; ++am) {
    const float a = bf16_to_f((uint16_t)(0x3f80 | am));
    const float inv = fdiv(448.0f, a);
    for (uint32_t h = 0; h < 0x8000; ++h) {
      const float ax = bf16_to_f((uint16_t)h);
      if (!(ax <= a)) continue;
      for (int sg = 0; sg < 2; ++sg) {
        const float x = sg ? -ax : ax;
        ++n;
        bad += fp8_fast(x, a, inv) != ref_code(2, 8, x, a);
      }
    }
  }
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> ua(0.5f, 4.0f);
  std::uniform_int_distribution<int> ue(-55, 55);
  std::uniform_real_distribution<float> ux(-1.0f, 1.0f);
  for (int it = 0; it < 300000; ++it) {
    const float a = ldexpf(ua(rng), ue(rng));
    const float inv = fdiv(448.0f, a);
    const int c = (int)(rng() % 0x7e);
    const double bnd = (oracle_fp8_decode((uint8_t)c) + oracle_fp8_decode((uint8_t)(c + 1))) /
                       2.0 * (double)a / 448.0;
    float y = (float)bnd;
    for (int d = 0; d < 6; ++d) y = nextafterf(y, -INFINITY);
    for (int d = -6; d <= 6; ++d, y = nextafterf(y, INFINITY)) {
      if (!(std::fabs(y) <= a)) continue;
      const float x = (rng() & 1) ? y : -y;
      ++n;
      bad += fp8_fast(x, a, inv) != ref_code(2, 8, x, a);
    }
    const float x = a * ux(rng);
    ++n;
    bad += fp8_fast(x, a, inv) != ref_code(2, 8, x, a);
  }
  report("fp8 fast encoder (cvt + near routing), bf16 exhaustive + f32", n, bad);
}

// Exact FP8 decode with FP32 scales from the 16-entry table (gradient path)
static void check_fp8_t16(uint64_t seed) {
  double t16[16];
  for (int i = 0; i < 16; ++i) t16[i] = fp8_t16(i);
  std::mt19937_64 rng(seed);
  long long n = 0, bad = 0;
  for (int it = 0; it < 40000; ++it) {
    float s = u2f((uint32_t)(rng() % 0x7f800000u));
    if (it < 4) s = it == 0 ? 0.0f : (it == 1 ? 1.4e-45f : (it == 2 ? 3.4e38f : 1.0f));
    uint8_t codes[256];
    float want[256];
    for (int c = 0; c < 256; ++c) codes[c] = (uint8_t)c;
    oracle_dequantize(codes, &s, 256, 8, 256, 2, want, nullptr, 0);
    for (int c = 0; c < 256; ++c) {
      const float got = fp8_dequant_t16(c, (double)s, t16);
      ++n;
      if ((c & 0x7f) == 0x7f) {
        bad += !(got != got) || ((f2u(got) >> 31) != (uint32_t)(c >> 7));
        continue;
      }
      bad += f2u(got) != f2u(want[c]);
    }
  }
  report("fp8 decode via T16 table, fp32 scales (random + extremes)", n, bad);
}

static void check_fp8_t16i(uint64_t seed) {
  double t16[16];
  for (int i = 0; i < 16; ++i) t16[i] = fp8_t16(i);
  std::mt19937_64 rng(seed);
  long long n = 0, bad = 0;
  for (int it = 0; it < 40000; ++it) {
    // fast-path scale range [2^-60, 2^60]
    const float s = ldexpf(1.0f + (float)(rng() % 8388608u) / 8388608.0f, (int)(rng() % 120) - 60);
    uint8_t codes[256];
    float want[256];
    for (int c = 0; c < 256; ++c) codes[c] = (uint8_t)c;
    oracle_dequantize(codes, &s, 256, 8, 256, 2, want, nullptr, 0);
    for (int c = 0; c < 256; ++c) {
      const float got = fp8_dequant_t16i(c, (double)s, t16);
      ++n;
      if ((c & 0x7f) == 0x7f) {
        bad += !(got != got);
        continue;
      }
      bad += f2u(got) != f2u(want[c]);
    }
  }
  report("fp8 decode via T16 + integer rounding, scales in [2^-60,2^60]", n, bad);
}

// Bracketing encoder of the gradient kernels (agq_grad.cuh fp8_requant16):
// cvt(s*inv*(1+2^-21)) == cvt(s*inv*(1-2^-21)) -> that code, else fp8_code.
static uint32_t fp8_bracket(float x, float a) {
  const float inv = fdiv(448.0f, a);
  const float ip = fmul(inv, 1.0f + 0x1p-21f), im = fmul(inv, 1.0f - 0x1p-21f);
  const uint32_t cp = cvt_e4m3x2(fmul(x, ip), 0.0f) & 0xffu;
  const uint32_t cm = cvt_e4m3x2(fmul(x, im), 0.0f) & 0xffu;
  return cp == cm ? cp : fp8_code(x, a, inv);
}

static void check_fp8_bracket(uint64_t seed) {
  long long n = 0, bad = 0, split = 0;
  for (int am = 0; am < 128; ++am) {
    const float a = bf16_to_f((uint16_t)(0x3f80 | am));
    for (uint32_t h = 0; h < 0x8000; ++h) {
      const float ax = bf16_to_f((uint16_t)h);
      if (!(ax <= a)) continue;
      for (int sg = 0; sg < 2; ++sg) {
        const float x = sg ? -ax : ax;
        ++n;
        bad += fp8_bracket(x, a) != ref_code(2, 8, x, a);
      }
    }
  }
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> ua(0.5f, 4.0f);
  std::uniform_int_distribution<int> ue(-55, 55);
  std::uniform_real_distribution<float> ux(-1.0f, 1.0f);
  for (int it = 0; it < 400000; ++it) {
    const float a = ldexpf(ua(rng), ue(rng));
    const int c = (int)(rng() % 0x7e);
    const double bnd = (oracle_fp8_decode((uint8_t)c) + oracle_fp8_decode((uint8_t)(c + 1))) /
                       2.0 * (double)a / 448.0;
    float y = (float)bnd;
    for (int d = 0; d < 6; ++d) y = nextafterf(y, -INFINITY);
    for (int d = -6; d <= 6; ++d, y = nextafterf(y, INFINITY)) {
      if (!(std::fabs(y) <= a)) continue;
      const float x = (rng() & 1) ? y : -y;
      ++n;
      bad += fp8_bracket(x, a) != ref_code(2, 8, x, a);
    }
    for (int k = 0; k < 4; ++k) {
      const float x = a * ux(rng) * (k == 3 ? 1e-4f : 1.0f);
      ++n;
      bad += fp8_bracket(x, a) != ref_code(2, 8, x, a);
    }
  }
  (void)split;
  report("fp8 bracketing encoder (gradient requant), bf16 exhaustive + f32", n, bad);
}

// Integer double->float rounding used for half of the gradient decodes
static void check_d2f_bits(uint64_t seed) {
  std::mt19937_64 rng(seed);
  long long n = 0, bad = 0;
  double lut[256];
  for (int c = 0; c < 256; ++c) lut[c] = oracle_code_unit_value(2, 8, (uint8_t)c);
  for (int it = 0; it < 40000; ++it) {
    const float s = ldexpf(1.0f + (float)(rng() % 8388608u) / 8388608.0f, (int)(rng() % 120) - 60);
    uint8_t codes[256];
    float want[256];
    for (int c = 0; c < 256; ++c) codes[c] = (uint8_t)c;
    oracle_dequantize(codes, &s, 256, 8, 256, 2, want, nullptr, 0);
    for (int c = 0; c < 256; ++c) {
      ++n;
      const float got = d2f_rn_bits(lut[c] * (double)s);
      if ((c & 0x7f) == 0x7f)
        bad += std::isfinite(got);  // NaN codes: any non-finite value
      else
        bad += f2u(got) != f2u(want[c]);
    }
  }
  // random doubles in the normal-float range, ties at bit 29 included
  for (int it = 0; it < 2000000; ++it) {
    uint64_t u = rng();
    const int e = 1023 - 120 + (int)(rng() % 240);
    u = (u & 0x800FFFFFFFFFFFFFull) | ((uint64_t)e << 52);
    if (it % 4 == 0) u = (u & ~0x1FFFFFFFull) | 0x10000000ull;  // exact tie
    const double d = u64_to_d(u);
    ++n;
    bad += f2u(d2f_rn_bits(d)) != f2u((float)d);
  }
  report("double->float integer RNE (gradient decode), incl. ties", n, bad);
}

// Per-block 8-entry decode table (K3/K4 gradient decode)
static void check_fp8_tab(uint64_t seed) {
  std::mt19937_64 rng(seed);
  long long n = 0, bad = 0, unsafe_ok = 0;
  double t8[8];
  for (int m = 0; m < 8; ++m) t8[m] = fp8_t8(m);
  // the unsafe-byte detector against a per-byte definition, all 2^16 byte pairs x 4 positions
  for (uint32_t a = 0; a < 256; ++a)
    for (uint32_t b = 0; b < 256; ++b) {
      const uint32_t w = a | (b << 8) | (0x40u << 16) | (0x3au << 24);
      auto uns = [](uint32_t c) { return ((c & 0x78u) == 0) || ((c & 0x7fu) == 0x7fu); };
      const bool want = uns(a) || uns(b);
      const uint32_t w2 = (a << 16) | (b << 24) | 0x4040u;
      ++n;
      bad += (fp8_tab_unsafe(w) != 0) != want;
      bad += (fp8_tab_unsafe(w2) != 0) != want;
      unsafe_ok += want;
    }
  auto run_scale = [&](float s) {
    uint8_t codes[256];
    float want[256];
    for (int c = 0; c < 256; ++c) codes[c] = (uint8_t)c;
    oracle_dequantize(codes, &s, 256, 8, 256, 2, want, nullptr, 0);
    float tab[8];
    for (int m = 0; m < 8; ++m) tab[m] = fp8_tab_entry(t8[m], s);
    for (int c = 0; c < 256; ++c) {
      if ((c & 0x78) == 0 || (c & 0x7f) == 0x7f) continue;
      ++n;
      bad += f2u(fp8_dq_tab((uint32_t)c, tab)) != f2u(want[c]);
    }
  };
  // every BF16 scale in [2^-60, 2^60] and random FP32 scales there
  for (int e = -60; e < 60; ++e)
    for (int k = 0; k < 128; ++k) run_scale(ldexpf(1.0f + k / 128.0f, e));
  run_scale(0x1p60f);
  for (int it = 0; it < 200000; ++it)
    run_scale(ldexpf(1.0f + (float)(rng() % 8388608u) / 8388608.0f, (int)(rng() % 120) - 60));
  report("fp8 decode via 8-entry block table (+ unsafe-byte detector)", n, bad);
}

int main() {
  check_fp8_tab(43);
  check_d2f_bits(41);
  check_fp8_bracket(31);
  check_fp8_t16(5);
  check_fp8_t16i(6);
  check_fp8_fast(21);
  check_extreme(11);
  check_fp8_ties();
  for (int bits = 4; bits <= 8; ++bits) check_encode_bf16(0, bits, 0, "linear");
  check_encode_bf16(0, 4, -59, "linear");
  check_encode_bf16(0, 8, 59, "linear");
  check_encode_bf16(2, 8, 0, "fp8");
  check_encode_bf16(2, 8, -59, "fp8");
  check_encode_bf16(2, 8, 59, "fp8");
  check_encode_bf16(1, 4, 0, "fp4");
  for (int bits = 4; bits <= 8; ++bits) check_encode_f32(0, bits, 100 + bits);
  check_encode_f32(2, 8, 7);
  check_encode_f32(1, 4, 8);
  for (int bits = 4; bits <= 8; ++bits) check_decode(0, bits);
  check_decode(1, 4);
  check_decode(2, 8);
  check_decode_double(3);
  std::printf("TOTAL mismatches=%lld\n", g_fail);
  return g_fail == 0 ? 0 : 1;
}
