// L1 block codec on sm_100a: block-absmax quantize + LSB-first packing (K1)
// and unpack + dequantize (K2).
//
// Reference: /root/reference/proj/include/agq/quantize.hpp:78-189 and
// tensor_io.hpp:63-100. Results are bit-identical to quantize_blockwise /
// dequantize_blockwise + pack_codes (tests/test_gpu_codec.py).
//
// Fast path (block 128, 32-byte aligned activations and 16-byte aligned
// codes / scales, whole 1024-element warp
// tiles): warp-autonomous persistent kernels. Each warp streams its own tiles;
// each lane loads its 32 consecutive elements with 256-bit loads (next tile
// in flight in registers; every 32-byte sector read once, no shared-memory
// staging), 4 lanes per 128-element block: two shuffles give the
// block absmax and a lane's 32 codes are exactly `bits` 32-bit words of the
// packed stream. No CTA-wide barrier. (CTA-wide TMA bulk-copy, per-warp TMA
// and cp.async rings were built, verified bit-exact and measured slower:
// DESIGN.md section 4.)
//
// Generic path (any block size / alignment / the tail after the last full
// tile): warp-per-block absmax, thread-per-output-byte encode+pack and
// thread-per-element decode, same element functions (agq_numerics.cuh).
#include <cstdlib>
#include <utility>

#include "agq_common.cuh"
#include "agq_minifloat.cuh"

namespace agqk {

template <int CB, int NW, int NC, int... J>
__device__ __forceinline__ void pack_chunks(uint32_t (&w)[NW], const uint64_t (&pk)[NC],
                                            std::integer_sequence<int, J...>) {
  (or_bits<J * CB, NW>(w, pk[J]), ...);
}
template <int CB, int NW, int NC, int... J>
__device__ __forceinline__ void unpack_chunks(const uint32_t (&w)[NW], uint64_t (&pk)[NC],
                                              std::integer_sequence<int, J...>) {
  ((pk[J] = get_bits<J * CB, CB, NW>(w)), ...);
}

// ---------------------------------------------------------------------------
// K1: quantize
// ---------------------------------------------------------------------------
template <typename Tin>
struct InTraits;
template <>
struct InTraits<__nv_bfloat16> {
  static constexpr int kChunks = 4;  // 16-byte chunks per thread row
  static constexpr int kStages = 4;
  static constexpr bool kBf16 = true;
};
template <>
struct InTraits<float> {
  static constexpr int kChunks = 8;
  static constexpr int kStages = 3;
  static constexpr bool kBf16 = false;
};

template <int BITS, int CODEC, bool BF16IN>
__device__ __forceinline__ uint32_t encode_one(float x, float a, float inv,
                                               float rcp, bool fast) {
  if (CODEC == 0) {
    constexpr int L = (1 << (BITS - 1)) - 1;
    if (fast) {
      if (BF16IN) return (uint32_t)(linear_k_bf16(x, a, inv, rcp, (float)L) + L);
      return (uint32_t)(linear_k_f32(x, a, inv, (float)L) + L);
    }
    return encode_double(0, BITS, x, a);
  } else if (CODEC == 1) {
    return fast ? fp4_code(x, a) : encode_double(1, 4, x, a);
  } else {
    return fast ? fp8_code(x, a, inv) : encode_double(2, 8, x, a);
  }
}

__device__ __noinline__ uint32_t encode_slow(int codec, int bits, float x, float a) {
  return encode_double(codec, bits, x, a);
}

// Same encode, written straight into the lane's PACK output words (32 codes,
// LSB-first): the pair (lo, hi) becomes ((f2u(hi) << PACK) + f2u(lo) +
// kOff * (1 + 2^PACK)) mod 2^32 = (k1 + L) << PACK | (k0 + L), since
// f2u(magic + k) = kMagicBits + k and kMagicBits + kOff = L; pair K is then
// added at bit 2*PACK*K (fields are disjoint, so add = or), which compiles
// to one LEA per pair (+ one LEA.HI where a pair straddles two words)
// instead of 64-bit chunk accumulators re-split into words.
template <int PACK, int K>
__device__ __forceinline__ void put_pair(uint32_t (&words)[PACK], uint32_t p) {
  constexpr int o = 2 * PACK * K, w = o / 32, sh = o % 32;
  // funnel shift + add (integer ALU, LEA) rather than an IMAD on the FMA
  // pipe the encode keeps busy (profiles/r02_quant_alu_pack_ab.log)
  words[w] += sh ? __funnelshift_l(0u, p, sh) : p;
  if constexpr (sh + 2 * PACK > 32) words[w + 1] += p >> (32 - sh);
}
template <int BITS, int PACK, int J = 0>
__device__ __forceinline__ void encode_linear_bf16_words(const uint4 (&ch)[4], const f32x2& inv2,
                                                         const f32x2& rcp2, const f32x2& na2,
                                                         uint32_t (&words)[PACK]) {
  constexpr int L = (1 << (BITS - 1)) - 1;
  constexpr uint32_t kOff = (uint32_t)L - kMagicBits;
  constexpr uint32_t kPairOff = kOff + (kOff << PACK);
  const f32x2 L2 = pk2((float)L, (float)L), mg2 = pk2(kMagicRound, kMagicRound);
  const uint32_t wv[4] = {ch[J].x, ch[J].y, ch[J].z, ch[J].w};
  uint32_t pr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // low half to FP32 with a byte permute (integer ALU) instead of the
    // shift the compiler issues as IMAD on the FMA pipe the encode keeps
    // 70% busy (C2 quant +2-3%, profiles/r02_quant_prmt_unpack_ab.log)
    const f32x2 x = pk2(u2f(__byte_perm(wv[k], 0u, 0x1044)), u2f(wv[k] & 0xffff0000u));
    const f32x2 v = mul2(x, inv2);
    const f32x2 xl = mul2(x, L2);
    const f32x2 r = fma2(v, na2, xl);
    const f32x2 v2 = fma2(r, rcp2, v);
    float lo, hi;
    up2(add2(v2, mg2), lo, hi);
    pr[k] = __funnelshift_l(0u, f2u(hi), PACK) + f2u(lo) + kPairOff;
  }
  put_pair<PACK, 4 * J + 0>(words, pr[0]);
  put_pair<PACK, 4 * J + 1>(words, pr[1]);
  put_pair<PACK, 4 * J + 2>(words, pr[2]);
  put_pair<PACK, 4 * J + 3>(words, pr[3]);
  if constexpr (J < 3) encode_linear_bf16_words<BITS, PACK, J + 1>(ch, inv2, rcp2, na2, words);
}

// ---------------------------------------------------------------------------
// K1 (warp-autonomous variant): every warp streams its own 1024-element tiles
// — each lane's 32 consecutive elements by 256-bit loads (next tile
// prefetched into registers while the current one is encoded), codes written
// straight from registers (PACK 32-bit words per lane, contiguous per warp).
// No shared memory, no barrier. (Round 1 staged coalesced 128-bit loads
// through a swizzled shared slot: 3% slower, profiles/r02_act_ldg256.log.)
// ---------------------------------------------------------------------------
constexpr int kWarpElems = 1024;
constexpr int kWarpsPerCta = 8;
// Resident CTAs per SM of the BF16 act kernels (measured best,
// profiles/r01_microbench_act_minb*); FP32-I/O instances run at 2. The
// macros exist only for experiment builds (Makefile `variant`).
#ifndef AGQ_QUANT_MINB
#define AGQ_QUANT_MINB 3
#endif
#ifndef AGQ_DEQUANT_MINB
#define AGQ_DEQUANT_MINB 3
#endif
constexpr int kQuantMinB = AGQ_QUANT_MINB;
constexpr int kDequantMinB = AGQ_DEQUANT_MINB;

// FP32 rows (128 B per lane) are moved through a private shared slot: a
// lane's four 256-bit accesses at a 128-byte stride measured 10-20% slower
// than coalesced 128-bit accesses + a swizzled transposition
// (profiles/r02_f32_staging_ab.log); BF16 rows (64 B) go direct.
// Swizzle: lane row r (kChunks 16-byte chunks) keeps chunk c at slot
// (c + rot(r)) mod kChunks, so the coalesced side (8 lanes = one 128-byte
// phase) and the per-row side (8 rows, same chunk) are both conflict free.
template <int kChunks>
__device__ __forceinline__ uint32_t swz_off(uint32_t row, uint32_t c) {
  const uint32_t rot = kChunks == 4 ? (row >> 1) : row;
  return row * (kChunks * 16) + ((c + rot) & (kChunks - 1)) * 16;
}
// Byte offset in the swizzled tile of the 16-byte chunk at natural offset `o`.
template <int kChunks>
__device__ __forceinline__ uint32_t swz_of_linear(uint32_t o) {
  return swz_off<kChunks>(o / (kChunks * 16), (o / 16) & (kChunks - 1));
}

struct TileRef {
  int g;
  uint64_t lt;
};

// Tiles in flight per warp (profiles/r01_quant_prefetch_ab.log,
// r01_dequant_prefetch_ab.log; dequant 2 -> 3 after the 256-bit stores:
// b=4 dequant 103 -> 97 us on 235M elements, profiles/r02_dequant_pf_ab.log).
#ifndef AGQ_QUANT_PF
#define AGQ_QUANT_PF 1
#endif
#ifndef AGQ_DEQUANT_PF
#define AGQ_DEQUANT_PF 3
#endif
constexpr int kQuantPrefetch = AGQ_QUANT_PF;
constexpr int kDequantPrefetch = AGQ_DEQUANT_PF;
// Incremental locate for a warp whose tiles only move forward (t += grid
// warps): the current segment's [begin, end) tile range lives in registers,
// so a tile costs one compare (no parameter-bank load in front of the
// prefetch address) and the table is read only when crossing a boundary —
// instead of a select chain over every segment per tile.
struct SegCursor {
  int g = 0;
  uint64_t begin = 0, end = 0;
};
__device__ __forceinline__ TileRef locate_from(const SegTable& st, uint64_t t, SegCursor& c) {
  if (c.end == 0) {  // first tile of this warp
    c.g = seg_of(st, t);
    c.begin = st.tile_begin[c.g];
    c.end = st.tile_begin[c.g + 1];
  }
  while (t >= c.end) {
    ++c.g;
    c.begin = c.end;
    c.end = st.tile_begin[c.g + 1];
  }
  return {c.g, t - c.begin};
}

template <int BITS, int PACK, int CODEC, typename Tin>
__device__ __forceinline__ void encode_row(const uint4 (&ch)[InTraits<Tin>::kChunks], float a,
                                           bool zero, bool fast, uint32_t (&words)[PACK]) {
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr int kPerChunk = 32 / kChunks;
  constexpr int kChunkBits = kPerChunk * PACK;
  constexpr int L = (1 << (BITS - 1)) - 1;
  constexpr uint32_t kZeroCode = CODEC == 0 ? (uint32_t)L : 0u;
  uint64_t pk[kChunks];
  if (zero) {
    uint64_t zc = 0;
#pragma unroll
    for (int e = 0; e < kPerChunk; ++e) zc |= (uint64_t)kZeroCode << (e * PACK);
#pragma unroll
    for (int j = 0; j < kChunks; ++j) pk[j] = zc;
  } else if (fast) {
    if constexpr (CODEC == 0 && TR::kBf16) {
      const float rcp = fdiv(1.0f, a);  // one division per block: inv = L * (1/a)
      const float inv = fmul((float)L, rcp);
#pragma unroll
      for (int k = 0; k < PACK; ++k) words[k] = 0;
      encode_linear_bf16_words<BITS, PACK>(ch, pk2(inv, inv), pk2(rcp, rcp), pk2(-a, -a), words);
      return;
    } else if constexpr (CODEC != 0) {
      // two independent halves of 16 values (register pressure)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[16];
#pragma unroll
        for (int j = 0; j < kChunks / 2; ++j) {
          const uint4 c4 = ch[h * (kChunks / 2) + j];
          const uint32_t wv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if constexpr (TR::kBf16) {
              v[8 * j + 2 * k] = u2f(wv[k] << 16);
              v[8 * j + 2 * k + 1] = u2f(wv[k] & 0xffff0000u);
            } else {
              v[4 * j + k] = u2f(wv[k]);
            }
          }
        }
        uint32_t hw[PACK / 2];
        if constexpr (CODEC == 2) {
          static_assert(PACK == 8, "E4M3 codes are one byte");
          fp8_encode16<TR::kBf16>(v, a, hw);
        } else {
          fp4_encode16<PACK, TR::kBf16>(v, a, hw);
        }
#pragma unroll
        for (int k = 0; k < PACK / 2; ++k) words[h * (PACK / 2) + k] = hw[k];
      }
      return;
    } else {
      const float inv = codec_inv(CODEC, BITS, a);
#pragma unroll
      for (int j = 0; j < kChunks; ++j) {
        const uint32_t wv[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
        uint64_t acc = 0;
#pragma unroll
        for (int e = 0; e < kPerChunk; ++e) {
          float x;
          if constexpr (TR::kBf16)
            x = u2f((e & 1) ? (wv[e >> 1] & 0xffff0000u) : (wv[e >> 1] << 16));
          else
            x = u2f(wv[e]);
          acc |= (uint64_t)encode_one<BITS, CODEC, TR::kBf16>(x, a, inv, 0.0f, true) << (e * PACK);
        }
        pk[j] = acc;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const uint32_t wv[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
      uint64_t acc = 0;
#pragma unroll
      for (int e = 0; e < kPerChunk; ++e) {
        float x;
        if constexpr (TR::kBf16)
          x = u2f((e & 1) ? (wv[e >> 1] & 0xffff0000u) : (wv[e >> 1] << 16));
        else
          x = u2f(wv[e]);
        acc |= (uint64_t)encode_slow(CODEC, BITS, x, a) << (e * PACK);
      }
      pk[j] = acc;
    }
  }
#pragma unroll
  for (int k = 0; k < PACK; ++k) words[k] = 0;
  pack_chunks<kChunkBits>(words, pk, std::make_integer_sequence<int, kChunks>{});
}

// Per-tile compute of the warp-autonomous quantizer: lane row `ch` (32
// consecutive elements, 4 lanes per 128-block) -> block absmax (2 shuffles),
// packed codes straight to HBM, one scale per 4 lanes.
template <int BITS, int PACK, int CODEC, typename Tin>
__device__ __forceinline__ void quant_tile(const SegTable& st, agq_errors* err, const TileRef& tr,
                                           int lane, const uint4 (&ch)[InTraits<Tin>::kChunks],
                                           uint32_t (&words)[PACK], float& a) {
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr uint32_t kCodeB = kWarpElems * PACK / 8;
  uint32_t m;
  if constexpr (TR::kBf16) {
    uint32_t mm = 0;
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      mm = __vmaxu2(mm, ch[j].x & 0x7fff7fffu);
      mm = __vmaxu2(mm, ch[j].y & 0x7fff7fffu);
      mm = __vmaxu2(mm, ch[j].z & 0x7fff7fffu);
      mm = __vmaxu2(mm, ch[j].w & 0x7fff7fffu);
    }
    m = max(mm & 0xffffu, mm >> 16) << 16;
  } else {
    m = 0;
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      m = max(m, ch[j].x & 0x7fffffffu);
      m = max(m, ch[j].y & 0x7fffffffu);
      m = max(m, ch[j].z & 0x7fffffffu);
      m = max(m, ch[j].w & 0x7fffffffu);
    }
  }
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
  a = u2f(m);
  if (m >= 0x7f800000u && (lane & 3) == 0)
    err_min(&err->nonfinite_block, (long long)(st.block_base[tr.g] + tr.lt * 8 + (lane >> 2)));
  encode_row<BITS, PACK, CODEC, Tin>(ch, a, m == 0, fast_scale(a), words);
  uint32_t* cdst = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(st.codes[tr.g]) +
                                               tr.lt * kCodeB) + lane * PACK;
  if constexpr (PACK % 4 == 0) {
#pragma unroll
    for (int k = 0; k < PACK / 4; ++k)
      *reinterpret_cast<uint4*>(cdst + 4 * k) =
          make_uint4(words[4 * k], words[4 * k + 1], words[4 * k + 2], words[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < PACK; ++k) cdst[k] = words[k];
  }
  if ((lane & 3) == 0) st.scales[tr.g][tr.lt * 8 + (lane >> 2)] = a;
}

template <int BITS, int PACK, int CODEC, typename Tin>
__global__ void __launch_bounds__(kWarpsPerCta * 32,
                                  sizeof(Tin) != 2 ? 2 : kQuantMinB)
    k_quant_warp(SegTable st, agq_errors* err) {
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel's outputs (our inputs) are visible
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tin);    // 2 KB / 4 KB
  constexpr bool kStaged = kChunks == 8;                    // FP32 rows
  __shared__ __align__(16) unsigned char sbuf[kStaged ? kWarpsPerCta : 1][kStaged ? kTileB : 16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sbuf[kStaged ? warp : 0];
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;

  // BF16: the lane's row (32 consecutive values, 64 B) with two 256-bit
  // loads, every 32-byte sector of the tile read once; FP32: coalesced
  // 128-bit loads, transposed through the shared slot
  auto load = [&](TileRef tr, uint4 (&buf)[kChunks]) {
    const unsigned char* src = static_cast<const unsigned char*>(st.src[tr.g]) + tr.lt * kTileB;
    if constexpr (kStaged) {
#pragma unroll
      for (int j = 0; j < kChunks; ++j) buf[j] = ldg128_stream(src + j * 512 + lane * 16);
    } else {
#pragma unroll
      for (int h = 0; h < kChunks / 2; ++h) {
        uint32_t w[8];
        ldg256_stream(src + lane * (kChunks * 16) + 32 * h, w);
        buf[2 * h] = make_uint4(w[0], w[1], w[2], w[3]);
        buf[2 * h + 1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
  };
  constexpr int kPf = kQuantPrefetch;  // tiles in flight per warp (registers)
  uint4 buf[kPf][kChunks];
  TileRef curq[kPf];
  SegCursor gseg;
#pragma unroll
  for (int d = 0; d < kPf; ++d) {
    curq[d] = TileRef{0, 0};
    if (t + d * nw < total) {
      curq[d] = locate_from(st, t + d * nw, gseg);
      load(curq[d], buf[d]);
    }
  }
  for (; t < total; t += nw) {
    uint4 ch[kChunks];
    if constexpr (kStaged) {
#pragma unroll
      for (int j = 0; j < kChunks; ++j)
        sts128(wb + swz_of_linear<kChunks>(j * 512 + lane * 16), buf[0][j]);
      __syncwarp();
    } else {
#pragma unroll
      for (int j = 0; j < kChunks; ++j) ch[j] = buf[0][j];
    }
    const TileRef tr = curq[0];
#pragma unroll
    for (int d = 0; d + 1 < kPf; ++d) {
#pragma unroll
      for (int j = 0; j < kChunks; ++j) buf[d][j] = buf[d + 1][j];
      curq[d] = curq[d + 1];
    }
    if (t + kPf * nw < total) {
      curq[kPf - 1] = locate_from(st, t + kPf * nw, gseg);
      load(curq[kPf - 1], buf[kPf - 1]);
    }
    if constexpr (kStaged) {
#pragma unroll
      for (int j = 0; j < kChunks; ++j) ch[j] = lds128(wb + swz_off<kChunks>(lane, j));
      __syncwarp();
    }
    uint32_t words[PACK];
    float a;
    quant_tile<BITS, PACK, CODEC, Tin>(st, err, tr, lane, ch, words, a);
  }
}

// K2 warp-autonomous variant: lane loads its PACK code words (+ block scale),
// next tile prefetched, decodes 32 values and writes them with 256-bit
// stores (64 or 128 contiguous bytes per lane).
template <int BITS, int PACK, int CODEC, typename Tout>
__global__ void __launch_bounds__(kWarpsPerCta * 32, sizeof(Tout) == 2 ? kDequantMinB : 2)
    k_dequant_warp(SegTable st, int validate, agq_errors* err);

// ---------------------------------------------------------------------------
// K2: dequantize
// ---------------------------------------------------------------------------
template <typename Tout>
struct OutTraits;
template <>
struct OutTraits<__nv_bfloat16> {
  static constexpr int kChunks = 4;
};
template <>
struct OutTraits<float> {
  static constexpr int kChunks = 8;
};

// Decode of one code with the block constants (exact, see agq_numerics.cuh).
template <int BITS, int CODEC>
__device__ __forceinline__ float decode_one(uint32_t c, float s, bool fast,
                                            const double* fp8lut) {
  if (CODEC == 0) {
    constexpr int L = (1 << (BITS - 1)) - 1;
    if (fast) return dq_linear_bf16scale((int)c - L, s, (float)L, 1.0f / (float)L);
    return dequant_double(0, BITS, c, s);
  } else if (CODEC == 1) {
    if (fast) return div_const_rn(fmul(e2m1_value(c), s), 6.0f, 1.0f / 6.0f);
    return dequant_double(1, 4, c, s);
  } else {
    if ((c & 0x7fu) == 0x7fu) return u2f(0x7fc00000u | ((c & 0x80u) << 24));
    if (fast) return div_const_rn(fmul(e4m3_value(c), s), 448.0f, 1.0f / 448.0f);
    const float mag = d2f_rn(dmul(fp8lut[c & 0x7fu], (double)s));
    return u2f(f2u(mag) | ((c & 0x80u) << 24));
  }
}

// SymmetricLinear, BF16-valued fast scale: c' = c - L as an exact float via
// the magic add (no I2F), p = c' s exact, then the Markstein-corrected
// division by L (agq_numerics.cuh:dq_linear_bf16scale) on pairs. Linear codes
// never produce -0, so the division needs no sign handling here.
// The magic exponent bits in a register the optimiser cannot see through, so
// mask-and-or of a code compiles to one LOP3 (x & mask) | R (a LOP3 takes one
// immediate only).
__constant__ uint32_t c_magic_bits = kMagicBits;
__device__ __forceinline__ uint32_t opaque_magic() { return c_magic_bits; }


// Code e (LSB-first, PACK bits) of a lane row held in PACK 32-bit words;
// with e a compile-time constant after unrolling this is one SHF (or one
// funnel shift where the code straddles two words). High bits are garbage:
// callers mask.
template <int PACK>
__device__ __forceinline__ uint32_t code_at(const uint32_t (&w)[PACK], int e) {
  const int o = e * PACK, wi = o >> 5, sh = o & 31;
  if (sh == 0) return w[wi];
  if (sh + PACK > 32) return __funnelshift_r(w[wi], w[wi + 1], sh);
  return w[wi] >> sh;
}
// decode_linear_fast for elements [e0, e0 + NPER) straight from the words
template <int BITS, int PACK, int NPER>
__device__ __forceinline__ void decode_linear_words(const uint32_t (&w)[PACK], int e0, float s,
                                                    float (&v)[NPER]) {
  constexpr int L = (1 << (BITS - 1)) - 1;
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  const f32x2 s2 = pk2(s, s);
  const f32x2 off2 = pk2(-(kMagicRound + (float)L), -(kMagicRound + (float)L));
  const f32x2 den2 = pk2(-(float)L, -(float)L), rden2 = pk2(1.0f / L, 1.0f / L);
  const uint32_t mb = opaque_magic();
#pragma unroll
  for (int e = 0; e < NPER; e += 2) {
    const uint32_t c0 = (code_at<PACK>(w, e0 + e) & kMask) | mb;
    const uint32_t c1 = (code_at<PACK>(w, e0 + e + 1) & kMask) | mb;
    const f32x2 cp = add2(pk2(u2f(c0), u2f(c1)), off2);
    const f32x2 p = mul2(cp, s2);
    const f32x2 q0 = mul2(p, rden2);
    const f32x2 r = fma2(q0, den2, p);
    up2(fma2(r, rden2, q0), v[e], v[e + 1]);
  }
}

// round-to-nearest-even to bf16 with the reference's integer rule
// (collective.hpp:101-110; identical to cvt.rn for non-NaN values, and keeps
// the quiet-NaN payload the reference produces).
__device__ __forceinline__ uint32_t bf16_bits_rne(float f) {
  uint32_t u = f2u(f);
  u += 0x7fffu + ((u >> 16) & 1u);
  return u >> 16;
}

template <int BITS, int PACK, int CODEC, typename Tout>
__global__ void __launch_bounds__(kWarpsPerCta * 32, sizeof(Tout) == 2 ? kDequantMinB : 2)
    k_dequant_warp(SegTable st, int validate, agq_errors* err) {
  pdl_launch_dependents();
  constexpr int kChunks = OutTraits<Tout>::kChunks;
  constexpr int kPerChunk = 32 / kChunks;
  constexpr int kChunkBits = kPerChunk * PACK;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tout);
  constexpr uint32_t kCodeB = kWarpElems * PACK / 8;
  constexpr bool kBf16Out = sizeof(Tout) == 2;
  constexpr bool kStaged = !kBf16Out;  // FP32 rows: through the shared slot
  __shared__ __align__(16) unsigned char sbuf[kStaged ? kWarpsPerCta : 1][kStaged ? kTileB : 16];
  __shared__ double fp8lut[CODEC == 2 ? 128 : 1];
  // exact unit values fl64(unit(c)) for the FP32-scale path (linear / FP4):
  // one LDS.64 + DMUL + F2F per element instead of a double division
  constexpr int kU = CODEC == 0 ? (1 << BITS) : (CODEC == 1 ? 16 : 1);
  __shared__ double ulut[kU];
  // FP8 with FP32 block scales: per-block 8-entry tables (F[m] / 2, see
  // agq_numerics.cuh:fp8_dq_tab), 8 blocks per warp tile
  __shared__ __align__(32) float dqtab[CODEC == 2 ? kWarpsPerCta * 64 : 1];
  if (CODEC == 2) {
    fill_fp8_unit_lut(fp8lut);
  } else {
    for (int c = threadIdx.x; c < kU; c += blockDim.x) ulut[c] = unit_value_double(CODEC, BITS, c);
  }
  __syncthreads();
  // the table fills above touch no global memory, so they overlap the tail
  // of the previous kernel (C1 dequantize 8.65 -> 8.55 us,
  // profiles/r02_dequant_late_pdl_wait_ab.log); everything below may read
  // its outputs
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sbuf[kStaged ? warp : 0];
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  auto load = [&](TileRef tr, uint32_t (&w)[PACK], float& sc) {
    const unsigned char* src = static_cast<const unsigned char*>(st.codes[tr.g]) + tr.lt * kCodeB;
    if constexpr (PACK % 4 == 0) {
#pragma unroll
      for (int k = 0; k < PACK / 4; ++k) {
        const uint4 v = ldg128_stream(src + lane * PACK * 4 + k * 16);
        w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
      }
    } else if constexpr (PACK % 2 == 0) {  // 8-byte aligned lane rows (b = 6)
      const uint2* s64 = reinterpret_cast<const uint2*>(src + lane * PACK * 4);
#pragma unroll
      for (int k = 0; k < PACK / 2; ++k) {
        const uint2 v = __ldg(s64 + k);
        w[2 * k] = v.x;
        w[2 * k + 1] = v.y;
      }
    } else {
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src) + lane * PACK;
#pragma unroll
      for (int k = 0; k < PACK; ++k) w[k] = __ldg(s32 + k);
    }
    sc = __ldg(st.scales[tr.g] + tr.lt * 8 + (lane >> 2));
  };
  // kDequantPrefetch tiles in flight per warp (codes + scale are <= 9
  // registers per tile, so extra tiles in flight are cheap and cover the
  // load latency the kernel otherwise stalls on)
  constexpr int kPf = kDequantPrefetch;
  uint32_t words[kPf][PACK];
  float scq[kPf];
  TileRef curq[kPf];
  SegCursor gseg;
#pragma unroll
  for (int d = 0; d < kPf; ++d) {
    scq[d] = 0.f;
    curq[d] = TileRef{0, 0};
    if (t + d * nw < total) {
      curq[d] = locate_from(st, t + d * nw, gseg);
      load(curq[d], words[d], scq[d]);
    }
  }
  for (; t < total; t += nw) {
    uint32_t cw[PACK];
#pragma unroll
    for (int k = 0; k < PACK; ++k) cw[k] = words[0][k];
    const float s = scq[0];
    const TileRef tr = curq[0];
#pragma unroll
    for (int d = 0; d + 1 < kPf; ++d) {  // shift the queue (register renames)
#pragma unroll
      for (int k = 0; k < PACK; ++k) words[d][k] = words[d + 1][k];
      scq[d] = scq[d + 1];
      curq[d] = curq[d + 1];
    }
    if (t + kPf * nw < total) {
      curq[kPf - 1] = locate_from(st, t + kPf * nw, gseg);
      load(curq[kPf - 1], words[kPf - 1], scq[kPf - 1]);
    }
    if (validate) {
      if ((!(s >= 0.0f) || !(s <= 3.402823466e38f)) && (lane & 3) == 0)
        err_min(&err->bad_scale_block, (long long)(st.block_base[tr.g] + tr.lt * 8 + (lane >> 2)));
      if constexpr (PACK == 8 && BITS < 8) {
        uint32_t bad = 0;
#pragma unroll
        for (int k = 0; k < PACK; ++k) bad |= cw[k] & (0x01010101u * (0xffu << BITS & 0xffu));
        if (bad) {
#pragma unroll 1
          for (int e = 0; e < 32; ++e) {
            const uint32_t c = (cw[e >> 2] >> ((e & 3) * 8)) & 0xffu;
            if (c >> BITS) {
              err_min(&err->bad_code_index,
                      (long long)((st.block_base[tr.g] + tr.lt * 8) * kBlock + lane * 32 + e));
              break;
            }
          }
        }
      }
    }
    const bool fast = is_bf16_value(s) && fast_scale(s);
    // FP4 / FP8 rows decode through the hardware minifloat conversion; FP8
    // rows holding a NaN code keep the per-element path (NaN payloads)
    bool mfast = false;
    if constexpr (CODEC != 0) {
      if constexpr (CODEC == 2) mfast = fast && !fp8_row_has_nan<PACK>(cw);
      else mfast = fast;
    }
    bool tfast = false;  // FP8, FP32 scale: block-table decode (f16 route)
    uint32_t tb = 0;
    if constexpr (CODEC == 2) {
      float* wt = dqtab + (threadIdx.x >> 5) * 64;
      const int j0 = (lane & 3) * 2;
      __syncwarp();  // the previous tile's lookups are done
      wt[(lane >> 2) * 8 + j0] = fp8_tab_entry_f16(fp8_t8(j0), s);
      wt[(lane >> 2) * 8 + j0 + 1] = fp8_tab_entry_f16(fp8_t8(j0 + 1), s);
      __syncwarp();
      // NaN codes keep the per-element path (the reference's NaN payload)
      tfast = !fast && dq_fast(s) && !fp8_row_has_nan<PACK>(cw);
      tb = (uint32_t)__cvta_generic_to_shared(wt + (lane >> 2) * 8);
    }
    uint64_t pk[kChunks];
    unpack_chunks<kChunkBits>(cw, pk, std::make_integer_sequence<int, kChunks>{});
    // BF16: the lane's 32 outputs (64 B) go out as two 256-bit stores;
    // FP32: staged, then coalesced 128-bit stores
    unsigned char* dst = static_cast<unsigned char*>(st.dst[tr.g]) + tr.lt * kTileB;
    uint4 prev = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      float v[kPerChunk];
      if (CODEC == 2 && tfast) {
#pragma unroll
        for (int q = 0; q < kPerChunk / 4; ++q) {
          const uint32_t w1[1] = {cw[(j * kPerChunk) / 4 + q]};
          // -0.0f + d = d for every d, signed zeros included
          float a4[4] = {-0.0f, -0.0f, -0.0f, -0.0f};
          dq_f16_accum<1>(w1, tb, a4);
#pragma unroll
          for (int e = 0; e < 4; ++e) v[4 * q + e] = a4[e];
        }
      } else if (CODEC == 0 && fast) {
        decode_linear_words<BITS, PACK, kPerChunk>(cw, j * kPerChunk, s, v);
      } else if (CODEC != 0 && mfast) {
        minifloat_decode<CODEC == 0 ? 1 : CODEC, PACK, kPerChunk>(cw, j * kPerChunk, s, v);
      } else if (fast) {
#pragma unroll
        for (int e = 0; e < kPerChunk; ++e) {
          const uint32_t c = (uint32_t)(pk[j] >> (e * PACK)) & ((1u << BITS) - 1u);
          v[e] = decode_one<BITS, CODEC>(c, s, true, fp8lut);
        }
      } else {
        const double sd = (double)s;
#pragma unroll
        for (int e = 0; e < kPerChunk; ++e) {
          const uint32_t c = (uint32_t)(pk[j] >> (e * PACK)) & ((1u << BITS) - 1u);
          if constexpr (CODEC == 2) {  // = decode_slow, inlined
            const uint32_t sg = (c & 0x80u) << 24;
            v[e] = (c & 0x7fu) == 0x7fu ? u2f(0x7fc00000u | sg)
                                         : u2f(f2u(d2f_rn(dmul(fp8lut[c & 0x7fu], sd))) | sg);
          } else {
            v[e] = d2f_rn(dmul(ulut[c], sd));  // = dequant_double, tabled
          }
        }
      }
      uint4 o;
      if constexpr (kBf16Out) {
        uint32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (CODEC == 2 && !mfast && !tfast)
            h[k] = bf16_bits_rne(v[2 * k]) | (bf16_bits_rne(v[2 * k + 1]) << 16);
          else {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
            h[k] = *reinterpret_cast<uint32_t*>(&b2);
          }
        }
        o = make_uint4(h[0], h[1], h[2], h[3]);
      } else {
        o = make_uint4(f2u(v[0]), f2u(v[1]), f2u(v[2]), f2u(v[3]));
      }
      if constexpr (kStaged)
        sts128(wb + swz_off<kChunks>(lane, j), o);
      else if (j & 1)
        stg256(dst + lane * (kChunks * 16) + (j >> 1) * 32, prev, o);
      else
        prev = o;
    }
    if constexpr (kStaged) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kChunks; ++j)
        *reinterpret_cast<uint4*>(dst + j * 512 + lane * 16) =
            lds128(wb + swz_of_linear<kChunks>(j * 512 + lane * 16));
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// K1+K2 fused round trip (SymmetricLinear, BF16 in / out, packed codes): the
// quantize pass also writes the reconstruction dequantize_blockwise would
// give for its codes (quantize.hpp:193-196 roundtrip_relative_delta; the
// C1 config), straight from the lane's code words in registers. One read of
// x, codes + scales + reconstruction written: 2 + b/8 + 4/128 + 2 bytes per
// element instead of the two calls' 2 * (2 + b/8 + 4/128). Bit-identical to
// k_quant_warp followed by k_dequant_warp (same encode, same decode).
// ---------------------------------------------------------------------------
__device__ __noinline__ float dequant_linear_slow(int bits, uint32_t c, float s) {
  return dequant_double(0, bits, c, s);
}

#ifndef AGQ_RT_MINB
#define AGQ_RT_MINB 2
#endif
template <int BITS>
__global__ void __launch_bounds__(kWarpsPerCta * 32, AGQ_RT_MINB)
    k_roundtrip_warp(SegTable st, agq_errors* err) {
  pdl_launch_dependents();
  pdl_wait();
  using Tin = __nv_bfloat16;
  constexpr int kChunks = 4;
  constexpr uint32_t kTileB = kWarpElems * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  auto load = [&](TileRef tr, uint4 (&buf)[kChunks]) {  // the lane's 64-byte row
    const unsigned char* src = static_cast<const unsigned char*>(st.src[tr.g]) + tr.lt * kTileB +
                               lane * 64;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t w[8];
      ldg256_stream(src + 32 * h, w);
      buf[2 * h] = make_uint4(w[0], w[1], w[2], w[3]);
      buf[2 * h + 1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  };
  uint4 buf[kChunks];
  TileRef nxt{0, 0};
  SegCursor gseg;
  if (t < total) {
    nxt = locate_from(st, t, gseg);
    load(nxt, buf);
  }
  for (; t < total; t += nw) {
    uint4 ch[kChunks];
#pragma unroll
    for (int j = 0; j < kChunks; ++j) ch[j] = buf[j];
    const TileRef tr = nxt;
    if (t + nw < total) {
      nxt = locate_from(st, t + nw, gseg);
      load(nxt, buf);
    }
    uint32_t words[BITS];
    float a;
    quant_tile<BITS, BITS, 0, Tin>(st, err, tr, lane, ch, words, a);
    // the reconstruction of this lane's 32 codes: two 256-bit stores
    const bool fast = fast_scale(a);  // a is BF16-valued (absmax of BF16 values)
    unsigned char* dst = static_cast<unsigned char*>(st.dst[tr.g]) + tr.lt * kTileB + lane * 64;
    uint4 prev = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      float v[8];
      if (fast) {
        decode_linear_words<BITS, BITS, 8>(words, j * 8, a, v);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = dequant_linear_slow(BITS, (code_at<BITS>(words, j * 8 + e)) & ((1u << BITS) - 1u), a);
      }
      uint32_t h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
        h[k] = *reinterpret_cast<uint32_t*>(&b2);
      }
      const uint4 o = make_uint4(h[0], h[1], h[2], h[3]);
      if (j & 1)
        stg256(dst + (j >> 1) * 32, prev, o);
      else
        prev = o;
    }
  }
}

// ---------------------------------------------------------------------------
// Generic kernels (any block size, alignment, tails)
// ---------------------------------------------------------------------------
template <typename Tin>
__device__ __forceinline__ float load_in(const Tin* x, uint64_t i) {
  if constexpr (sizeof(Tin) == 2)
    return u2f((uint32_t)reinterpret_cast<const uint16_t*>(x)[i] << 16);
  else
    return x[i];
}

// One warp per block: absmax (as |x| bits), non-finite detection.
template <typename Tin>
__global__ void k_absmax_generic(const Tin* x, uint64_t n, uint32_t block,
                                 uint64_t nblocks, float* scales,
                                 long long blk_base, agq_errors* err) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t b = warp; b < nblocks; b += nwarps) {
    const uint64_t beg = b * block;
    const uint64_t end = min(n, beg + block);
    uint32_t m = 0;
    for (uint64_t i = beg + lane; i < end; i += 32) m = max(m, f2u(load_in(x, i)) & 0x7fffffffu);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      scales[b] = u2f(m);
      if (m >= 0x7f800000u) err_min(&err->nonfinite_block, blk_base + (long long)b);
    }
  }
}

__device__ __forceinline__ uint32_t encode_generic(int codec, int bits, float x,
                                                   float a) {
  if (a == 0.0f) return codec == 0 ? (uint32_t)levels_of(bits) : 0u;
  if (!(a <= 3.402823466e38f)) return 0u;  // non-finite block: error recorded
  return encode_f32(codec, bits, x, a, codec_inv(codec, bits, a));
}

// One thread per output byte of the LSB-first stream (tensor_io.hpp:69-77).
template <typename Tin>
__global__ void k_encode_packed_generic(const Tin* x, uint64_t n, int bits,
                                        uint32_t block, int codec,
                                        const float* scales, uint8_t* packed) {
  const uint64_t nbytes = (n * bits + 7) / 8;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nbytes;
       j += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t bit0 = j * 8;
    const uint64_t e0 = bit0 / bits;
    const uint64_t e1 = min(n - 1, (bit0 + 7) / bits);
    uint32_t byte = 0;
    for (uint64_t e = e0; e <= e1; ++e) {
      const uint32_t c = encode_generic(codec, bits, load_in(x, e), scales[e / block]);
      const long long off = (long long)(e * bits) - (long long)bit0;
      byte |= off >= 0 ? (c << off) : (c >> (-off));
    }
    packed[j] = (uint8_t)(byte & 0xffu);
  }
}

template <typename Tin>
__global__ void k_encode_bytes_generic(const Tin* x, uint64_t n, int bits,
                                       uint32_t block, int codec,
                                       const float* scales, uint8_t* codes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * (uint64_t)blockDim.x)
    codes[i] = (uint8_t)encode_generic(codec, bits, load_in(x, i), scales[i / block]);
}

__device__ __forceinline__ uint32_t read_code(const uint8_t* codes, int layout,
                                              int bits, uint64_t i) {
  if (layout == AGQ_CODES_BYTES) return codes[i];
  const uint64_t bit = i * bits;
  const uint64_t byte = bit >> 3;
  uint32_t v = codes[byte];
  if ((bit & 7) + bits > 8) v |= (uint32_t)codes[byte + 1] << 8;
  return (v >> (bit & 7)) & ((1u << bits) - 1u);
}

template <typename Tout>
__global__ void k_dequant_generic(const uint8_t* codes, int layout,
                                  const float* scales, uint64_t n, int bits,
                                  uint32_t block, int codec, Tout* out,
                                  int validate, long long elem_base,
                                  agq_errors* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint32_t c = read_code(codes, layout, bits, i);
    const float s = scales[i / block];
    if (validate) {
      if (c >> bits) err_min(&err->bad_code_index, elem_base + (long long)i);
      if ((i % block) == 0 && (!(s >= 0.0f) || !(s <= 3.402823466e38f)))
        err_min(&err->bad_scale_block, (elem_base + (long long)i) / block);
    }
    const uint32_t cc = c & ((1u << bits) - 1u);
    float v;
    if (codec == 2 && (cc & 0x7fu) == 0x7fu)
      v = u2f(0x7fc00000u | ((cc & 0x80u) << 24));
    else
      v = dequant_double(codec, bits, cc, s);
    if constexpr (sizeof(Tout) == 2)
      reinterpret_cast<uint16_t*>(out)[i] = (uint16_t)bf16_bits_rne(v);
    else
      out[i] = v;
  }
}

__global__ void k_pack_generic(const uint8_t* codes, uint64_t n, int bits,
                               uint8_t* packed) {
  const uint64_t nbytes = (n * bits + 7) / 8;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nbytes;
       j += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t bit0 = j * 8;
    const uint64_t e0 = bit0 / bits;
    const uint64_t e1 = min(n - 1, (bit0 + 7) / bits);
    uint32_t byte = 0;
    for (uint64_t e = e0; e <= e1; ++e) {
      const uint32_t c = codes[e] & ((1u << bits) - 1u);
      const long long off = (long long)(e * bits) - (long long)bit0;
      byte |= off >= 0 ? (c << off) : (c >> (-off));
    }
    packed[j] = (uint8_t)(byte & 0xffu);
  }
}

__global__ void k_unpack_generic(const uint8_t* packed, uint64_t n, int bits,
                                 uint8_t* codes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * (uint64_t)blockDim.x)
    codes[i] = (uint8_t)read_code(packed, AGQ_CODES_PACKED, bits, i);
}

}  // namespace agqk

// ===========================================================================
// Host launchers
// ===========================================================================
namespace agqh {
using namespace agqk;

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// the lane rows of the activations are read / written with 256-bit accesses
bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

int gen_grid(uint64_t work, int threads) {
  const uint64_t g = (work + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Launch with programmatic stream serialization (PDL): the kernel's launch
// and prologue overlap the previous kernel's tail; the kernels wait
// (griddepcontrol.wait) before touching global memory (profiles/r01_pdl_ab.log).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem,
                             cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
// resident CTAs per SM of a kernel (queried once per instantiation)
template <typename K>
int occupancy_of(K k, int block, size_t smem) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block, smem);
  return occ < 1 ? 1 : occ;
}

template <int BITS, int PACK, int CODEC, typename Tin>
agq_status launch_quant_warp(const SegTable& st, agq_errors* err, cudaStream_t s) {
  auto k = k_quant_warp<BITS, PACK, CODEC, Tin>;
  static const int occ = occupancy_of(k, kWarpsPerCta * 32, 0);
  const uint64_t tiles = st.tile_begin[st.nseg];
  const uint64_t want = (tiles + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  cudaError_t e = launch_pdl(k, (int)(want < cap ? want : cap), kWarpsPerCta * 32, 0, s, st, err);
  count_launch();
  return cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "quantize: launch");
}

template <int BITS, int PACK, int CODEC, typename Tout>
agq_status launch_dequant_warp(const SegTable& st, int validate, agq_errors* err, cudaStream_t s) {
  auto k = k_dequant_warp<BITS, PACK, CODEC, Tout>;
  static const int occ = occupancy_of(k, kWarpsPerCta * 32, 0);
  const uint64_t tiles = st.tile_begin[st.nseg];
  const uint64_t want = (tiles + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  cudaError_t e = launch_pdl(k, (int)(want < cap ? want : cap), kWarpsPerCta * 32, 0, s, st,
                                   validate, err);
  count_launch();
  return cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "dequantize: launch");
}

template <int PACK, typename Tin>
agq_status quant_dispatch_bits(int bits, int codec, const SegTable& st,
                               agq_errors* err, cudaStream_t s) {
  if (codec == AGQ_CODEC_FP8_E4M3) return launch_quant_warp<8, 8, 2, Tin>(st, err, s);
  if (codec == AGQ_CODEC_FP4_E2M1) return launch_quant_warp<4, PACK == 8 ? 8 : 4, 1, Tin>(st, err, s);
  switch (bits) {
    case 4: return launch_quant_warp<4, PACK == 8 ? 8 : 4, 0, Tin>(st, err, s);
    case 5: return launch_quant_warp<5, PACK == 8 ? 8 : 5, 0, Tin>(st, err, s);
    case 6: return launch_quant_warp<6, PACK == 8 ? 8 : 6, 0, Tin>(st, err, s);
    case 7: return launch_quant_warp<7, PACK == 8 ? 8 : 7, 0, Tin>(st, err, s);
    default: return launch_quant_warp<8, 8, 0, Tin>(st, err, s);
  }
}

template <int PACK, typename Tout>
agq_status dequant_dispatch_bits(int bits, int codec, const SegTable& st,
                                 int validate, agq_errors* err, cudaStream_t s) {
  if (codec == AGQ_CODEC_FP8_E4M3) return launch_dequant_warp<8, 8, 2, Tout>(st, validate, err, s);
  if (codec == AGQ_CODEC_FP4_E2M1) return launch_dequant_warp<4, PACK == 8 ? 8 : 4, 1, Tout>(st, validate, err, s);
  switch (bits) {
    case 4: return launch_dequant_warp<4, PACK == 8 ? 8 : 4, 0, Tout>(st, validate, err, s);
    case 5: return launch_dequant_warp<5, PACK == 8 ? 8 : 5, 0, Tout>(st, validate, err, s);
    case 6: return launch_dequant_warp<6, PACK == 8 ? 8 : 6, 0, Tout>(st, validate, err, s);
    case 7: return launch_dequant_warp<7, PACK == 8 ? 8 : 7, 0, Tout>(st, validate, err, s);
    default: return launch_dequant_warp<8, 8, 0, Tout>(st, validate, err, s);
  }
}

template <typename Tin>
agq_status quant_generic(const Tin* x, uint64_t n, int bits, uint32_t block,
                         int codec, void* codes, int layout, float* scales,
                         long long blk_base, agq_errors* err, cudaStream_t s) {
  const uint64_t nb = (n + block - 1) / block;
  k_absmax_generic<Tin><<<gen_grid(nb * 32, 256), 256, 0, s>>>(x, n, block, nb, scales,
                                                              blk_base, err);
  count_launch();
  if (layout == AGQ_CODES_PACKED) {
    const uint64_t nbytes = (n * bits + 7) / 8;
    k_encode_packed_generic<Tin><<<gen_grid(nbytes, 256), 256, 0, s>>>(
        x, n, bits, block, codec, scales, static_cast<uint8_t*>(codes));
  } else {
    k_encode_bytes_generic<Tin><<<gen_grid(n, 256), 256, 0, s>>>(
        x, n, bits, block, codec, scales, static_cast<uint8_t*>(codes));
  }
  count_launch();
  return cuda_fail(cudaGetLastError(), "quantize (generic): launch");
}

}  // namespace

namespace {

// One tensor: whole warp tiles through the warp kernel, the rest (any block
// size, unaligned pointers, the ragged tail) through the generic kernels.
// blk_base offsets the block / element indices the error record reports
// (the position of this tensor inside a grouped call).
agq_status quantize_one(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                        int codec, void* codes, int layout, float* scales, long long blk_base,
                        agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  const int pack = layout == AGQ_CODES_PACKED ? bits : 8;
  uint64_t ntiles = 0;
  if (block == (uint32_t)kBlock && aligned32(x) && aligned16(codes) && aligned16(scales))
    ntiles = n / (uint64_t)kWarpElems;
  if (ntiles > 0) {
    SegTable st{};
    st.src[0] = x;
    st.codes[0] = codes;
    st.scales[0] = scales;
    st.tile_begin[1] = ntiles;
    st.block_base[0] = (uint64_t)blk_base;
    st.nseg = 1;
    agq_status r;
    if (x_dtype == AGQ_BF16)
      r = layout == AGQ_CODES_PACKED ? quant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, err, s)
                                     : quant_dispatch_bits<8, __nv_bfloat16>(bits, codec, st, err, s);
    else
      r = layout == AGQ_CODES_PACKED ? quant_dispatch_bits<0, float>(bits, codec, st, err, s)
                                     : quant_dispatch_bits<8, float>(bits, codec, st, err, s);
    if (r != AGQ_OK) return r;
  }
  const uint64_t done = ntiles * (uint64_t)kWarpElems;
  if (done == n) return AGQ_OK;
  // tail (block-aligned start, byte-aligned in the packed stream)
  const uint64_t rest = n - done;
  const long long bb = blk_base + (long long)(done / block);
  void* ctail = static_cast<uint8_t*>(codes) + (done * pack) / 8;
  if (x_dtype == AGQ_BF16)
    return quant_generic(reinterpret_cast<const __nv_bfloat16*>(x) + done, rest, bits, block,
                         codec, ctail, layout, scales + done / block, bb, err, s);
  return quant_generic(reinterpret_cast<const float*>(x) + done, rest, bits, block, codec, ctail,
                       layout, scales + done / block, bb, err, s);
}

agq_status dequantize_one(const void* codes, int layout, const float* scales, uint64_t n,
                          int bits, uint32_t block, int codec, void* out, int out_dtype,
                          int validate, long long blk_base, agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  const int pack = layout == AGQ_CODES_PACKED ? bits : 8;
  uint64_t ntiles = 0;
  if (block == (uint32_t)kBlock && aligned32(out) && aligned16(codes) && aligned16(scales))
    ntiles = n / (uint64_t)kWarpElems;
  if (ntiles > 0) {
    SegTable st{};
    st.codes[0] = const_cast<void*>(codes);
    st.scales[0] = const_cast<float*>(scales);
    st.dst[0] = out;
    st.tile_begin[1] = ntiles;
    st.block_base[0] = (uint64_t)blk_base;
    st.nseg = 1;
    agq_status r;
    if (out_dtype == AGQ_BF16)
      r = layout == AGQ_CODES_PACKED
              ? dequant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, validate, err, s)
              : dequant_dispatch_bits<8, __nv_bfloat16>(bits, codec, st, validate, err, s);
    else
      r = layout == AGQ_CODES_PACKED ? dequant_dispatch_bits<0, float>(bits, codec, st, validate, err, s)
                                     : dequant_dispatch_bits<8, float>(bits, codec, st, validate, err, s);
    if (r != AGQ_OK) return r;
  }
  const uint64_t done = ntiles * (uint64_t)kWarpElems;
  if (done == n) return AGQ_OK;
  const uint64_t rest = n - done;
  const uint8_t* ctail = static_cast<const uint8_t*>(codes) + (done * pack) / 8;
  const float* stail = scales + done / block;
  const long long ebase = blk_base * (long long)block + (long long)done;
  if (out_dtype == AGQ_BF16)
    k_dequant_generic<__nv_bfloat16><<<gen_grid(rest, 256), 256, 0, s>>>(
        ctail, layout, stail, rest, bits, block, codec,
        static_cast<__nv_bfloat16*>(out) + done, validate, ebase, err);
  else
    k_dequant_generic<float><<<gen_grid(rest, 256), 256, 0, s>>>(
        ctail, layout, stail, rest, bits, block, codec, static_cast<float*>(out) + done,
        validate, ebase, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "dequantize (generic): launch");
}

bool seg_tiled(const agq_segment& g) {
  return aligned32(g.x) && aligned16(g.codes) && aligned16(g.scales);
}

// Grouped launch (the tensors one pipeline stage stores, any count): the
// whole warp tiles of up to kMaxSeg segments per launch (a segment table in
// the parameter bank), tails individually. Error indices are group-global:
// blocks (elements for a bad code) counted over the segments in order.
template <bool QUANT>
agq_status grouped(const agq_segment* segs, int nseg, int dtype, int bits, int codec,
                   int validate, agq_errors* err, cudaStream_t s) {
  uint64_t blocks = 0;
  int i0 = 0;
  while (i0 < nseg) {
    SegTable st{};
    uint64_t tiles = 0, b = blocks;
    int k = 0, i = i0;
    for (; i < nseg && k < kMaxSeg; ++i) {
      const uint64_t nt = seg_tiled(segs[i]) ? segs[i].n / (uint64_t)kWarpElems : 0;
      if (nt > 0) {
        if (QUANT) st.src[k] = segs[i].x;
        else st.dst[k] = const_cast<void*>(segs[i].x);
        st.codes[k] = segs[i].codes;
        st.scales[k] = segs[i].scales;
        st.tile_begin[k] = tiles;
        st.block_base[k] = b;
        tiles += nt;
        ++k;
      }
      b += (segs[i].n + kBlock - 1) / kBlock;
    }
    st.tile_begin[k] = tiles;
    st.nseg = k;
    if (k > 0) {
      agq_status r;
      if (QUANT)
        r = dtype == AGQ_BF16 ? quant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, err, s)
                              : quant_dispatch_bits<0, float>(bits, codec, st, err, s);
      else
        r = dtype == AGQ_BF16
                ? dequant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, validate, err, s)
                : dequant_dispatch_bits<0, float>(bits, codec, st, validate, err, s);
      if (r != AGQ_OK) return r;
    }
    // tails of the same segments
    for (int j = i0; j < i; ++j) {
      const uint64_t done = seg_tiled(segs[j]) ? segs[j].n / kWarpElems * kWarpElems : 0;
      const long long bb = (long long)(blocks + done / kBlock);
      blocks += (segs[j].n + kBlock - 1) / kBlock;
      if (done == segs[j].n) continue;
      const size_t esz = dtype == AGQ_BF16 ? 2 : 4;
      void* x = static_cast<char*>(const_cast<void*>(segs[j].x)) + done * esz;
      uint8_t* c = static_cast<uint8_t*>(segs[j].codes) + done * bits / 8;
      float* sc = segs[j].scales + done / kBlock;
      agq_status r =
          QUANT ? quantize_one(x, dtype, segs[j].n - done, bits, kBlock, codec, c,
                               AGQ_CODES_PACKED, sc, bb, err, s)
                : dequantize_one(c, AGQ_CODES_PACKED, sc, segs[j].n - done, bits, kBlock, codec,
                                 x, dtype, validate, bb, err, s);
      if (r != AGQ_OK) return r;
    }
    i0 = i;
  }
  return AGQ_OK;
}

}  // namespace

agq_status quantize_device(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                           int codec, void* codes, int layout, float* scales, agq_errors* err,
                           cudaStream_t s) {
  return quantize_one(x, x_dtype, n, bits, block, codec, codes, layout, scales, 0, err, s);
}

agq_status dequantize_device(const void* codes, int layout, const float* scales, uint64_t n,
                             int bits, uint32_t block, int codec, void* out, int out_dtype,
                             int validate, agq_errors* err, cudaStream_t s) {
  return dequantize_one(codes, layout, scales, n, bits, block, codec, out, out_dtype, validate, 0,
                        err, s);
}

// Chunked host entry points: blk_base = block index of element 0 in the
// error record.
agq_status quantize_device_at(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                              int codec, void* codes, int layout, float* scales,
                              long long blk_base, agq_errors* err, cudaStream_t s) {
  return quantize_one(x, x_dtype, n, bits, block, codec, codes, layout, scales, blk_base, err, s);
}

agq_status dequantize_device_at(const void* codes, int layout, const float* scales, uint64_t n,
                                int bits, uint32_t block, int codec, void* out, int out_dtype,
                                int validate, long long blk_base, agq_errors* err,
                                cudaStream_t s) {
  return dequantize_one(codes, layout, scales, n, bits, block, codec, out, out_dtype, validate,
                        blk_base, err, s);
}

// quantize + the reconstruction (the round trip) in one pass where the fast
// kernel applies (SymmetricLinear, BF16 in / out, block 128, packed, aligned
// whole warp tiles); the rest as quantize followed by dequantize.
agq_status roundtrip_device(const void* x, int x_dtype, uint64_t n, int bits, uint32_t block,
                            int codec, void* codes, int layout, float* scales, void* out,
                            int out_dtype, agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  uint64_t ntiles = 0;
  if (x_dtype == AGQ_BF16 && out_dtype == AGQ_BF16 && codec == AGQ_CODEC_SYMMETRIC_LINEAR &&
      layout == AGQ_CODES_PACKED && block == (uint32_t)kBlock && aligned32(x) && aligned16(codes) &&
      aligned16(scales) && aligned32(out))
    ntiles = n / (uint64_t)kWarpElems;
  if (ntiles > 0) {
    SegTable st{};
    st.src[0] = x;
    st.codes[0] = codes;
    st.scales[0] = scales;
    st.dst[0] = out;
    st.tile_begin[1] = ntiles;
    st.nseg = 1;
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kern) {
      static const int occ = occupancy_of(kern, kWarpsPerCta * 32, 0);
      const uint64_t want = (ntiles + kWarpsPerCta - 1) / kWarpsPerCta;
      const uint64_t cap = (uint64_t)num_sms() * occ;
      e = launch_pdl(kern, (int)(want < cap ? want : cap), kWarpsPerCta * 32, 0, s, st, err);
    };
    switch (bits) {
      case 4: go(k_roundtrip_warp<4>); break;
      case 5: go(k_roundtrip_warp<5>); break;
      case 6: go(k_roundtrip_warp<6>); break;
      case 7: go(k_roundtrip_warp<7>); break;
      default: go(k_roundtrip_warp<8>); break;
    }
    count_launch();
    if (agq_status r = cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "roundtrip: launch"))
      return r;
  }
  const uint64_t done = ntiles * (uint64_t)kWarpElems;
  if (done == n) return AGQ_OK;
  const int pack = layout == AGQ_CODES_PACKED ? bits : 8;
  const size_t ei = x_dtype == AGQ_BF16 ? 2 : 4, eo = out_dtype == AGQ_BF16 ? 2 : 4;
  const void* xr = static_cast<const char*>(x) + done * ei;
  void* cr = static_cast<uint8_t*>(codes) + done * pack / 8;
  float* sr = scales + done / block;
  void* orr = static_cast<char*>(out) + done * eo;
  const long long bb = (long long)(done / block);
  if (agq_status r = quantize_one(xr, x_dtype, n - done, bits, block, codec, cr, layout, sr, bb, err, s))
    return r;
  return dequantize_one(cr, layout, sr, n - done, bits, block, codec, orr, out_dtype, 0, bb, err,
                        s);
}

agq_status quantize_grouped_device(const agq_segment* segs, int nseg, int x_dtype, int bits,
                                   int codec, agq_errors* err, cudaStream_t s) {
  return grouped<true>(segs, nseg, x_dtype, bits, codec, 0, err, s);
}

agq_status dequantize_grouped_device(const agq_segment* segs, int nseg, int out_dtype, int bits,
                                     int codec, int validate, agq_errors* err, cudaStream_t s) {
  return grouped<false>(segs, nseg, out_dtype, bits, codec, validate, err, s);
}

agq_status pack_device(const uint8_t* codes, uint64_t n, int bits, uint8_t* packed,
                       cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  k_pack_generic<<<gen_grid((n * bits + 7) / 8, 256), 256, 0, s>>>(codes, n, bits, packed);
  count_launch();
  return cuda_fail(cudaGetLastError(), "pack: launch");
}

agq_status unpack_device(const uint8_t* packed, uint64_t n, int bits, uint8_t* codes,
                         cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  k_unpack_generic<<<gen_grid(n, 256), 256, 0, s>>>(packed, n, bits, codes);
  count_launch();
  return cuda_fail(cudaGetLastError(), "unpack: launch");
}

}  // namespace agqh
