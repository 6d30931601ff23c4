// L1 block codec on sm_100a: block-absmax quantize + LSB-first packing (K1)
// and unpack + dequantize (K2).
//
// Reference: /root/reference/proj/include/agq/quantize.hpp:78-189 and
// tensor_io.hpp:63-100. Results are bit-identical to quantize_blockwise /
// dequantize_blockwise + pack_codes (tests/test_gpu_codec.py).
//
// Fast path (block 128, 16-byte aligned buffers, full 8192-element tiles):
// persistent CTAs stream tiles through a STAGES-deep ring of shared-memory
// buffers filled by 1-D TMA bulk copies (cp.async.bulk + mbarrier) and drain
// packed codes / scales / outputs back with bulk stores. Each thread owns 32
// consecutive elements (4 threads per 128-element block): two shuffles give
// the block absmax and a thread's 32 codes are exactly `bits` 32-bit words of
// the packed stream. The shared-memory rows are read in a per-thread rotated
// chunk order (bank-conflict free) and put back in order with selects.
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

// SymmetricLinear, BF16 input, fast block scale: linear_k_bf16 on element
// pairs with packed FP32x2 arithmetic, RNE-to-integer by the magic add.
// Identical per-lane operations to agq_numerics.cuh:linear_k_bf16 (which the
// host test verifies exhaustively); codes land at PACK bits per element.
template <int BITS, int PACK>
__device__ __forceinline__ void encode_linear_bf16_fast(const uint4 (&ch)[4], float a, float inv,
                                                        float rcp, uint64_t (&pk)[4]) {
  constexpr int L = (1 << (BITS - 1)) - 1;
  const f32x2 inv2 = pk2(inv, inv), rcp2 = pk2(rcp, rcp), na2 = pk2(-a, -a);
  const f32x2 L2 = pk2((float)L, (float)L), mg2 = pk2(kMagicRound, kMagicRound);
  constexpr uint32_t kOff = (uint32_t)L - kMagicBits;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t wv[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f32x2 x = pk2(u2f(wv[k] << 16), u2f(wv[k] & 0xffff0000u));
      const f32x2 v = mul2(x, inv2);
      const f32x2 xl = mul2(x, L2);
      const f32x2 r = fma2(v, na2, xl);
      const f32x2 v2 = fma2(r, rcp2, v);
      float lo, hi;
      up2(add2(v2, mg2), lo, hi);
      const uint32_t c0 = f2u(lo) + kOff, c1 = f2u(hi) + kOff;
      acc |= (uint64_t)(c0 | (c1 << PACK)) << (2 * k * PACK);
    }
    pk[j] = acc;
  }
}

// Same encode, written straight into the lane's PACK output words (32 codes,
// LSB-first): the pair (lo, hi) becomes ((f2u(hi) << PACK) + f2u(lo) +
// kOff * (1 + 2^PACK)) mod 2^32 = (k1 + L) << PACK | (k0 + L), since
// f2u(magic + k) = kMagicBits + k and kMagicBits + kOff = L; pair K is then
// added at bit 2*PACK*K (fields are disjoint, so add = or), which compiles
// to one LEA per pair (+ one LEA.HI where a pair straddles two words)
// instead of 64-bit chunk accumulators re-split into words.
#ifndef AGQ_QUANT_WORDS
#define AGQ_QUANT_WORDS 1
#endif
template <int PACK, int K>
__device__ __forceinline__ void put_pair(uint32_t (&words)[PACK], uint32_t p) {
  constexpr int o = 2 * PACK * K, w = o / 32, sh = o % 32;
  words[w] += p << sh;
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
    const f32x2 x = pk2(u2f(wv[k] << 16), u2f(wv[k] & 0xffff0000u));
    const f32x2 v = mul2(x, inv2);
    const f32x2 xl = mul2(x, L2);
    const f32x2 r = fma2(v, na2, xl);
    const f32x2 v2 = fma2(r, rcp2, v);
    float lo, hi;
    up2(add2(v2, mg2), lo, hi);
    pr[k] = (f2u(hi) << PACK) + f2u(lo) + kPairOff;
  }
  put_pair<PACK, 4 * J + 0>(words, pr[0]);
  put_pair<PACK, 4 * J + 1>(words, pr[1]);
  put_pair<PACK, 4 * J + 2>(words, pr[2]);
  put_pair<PACK, 4 * J + 3>(words, pr[3]);
  if constexpr (J < 3) encode_linear_bf16_words<BITS, PACK, J + 1>(ch, inv2, rcp2, na2, words);
}

// PACK: bits per stored code (BITS for the packed stream, 8 for one byte per
// element).
template <int BITS, int PACK, int CODEC, typename Tin>
__global__ void __launch_bounds__(kThreads)
    k_quant_tiled(SegTable st, agq_errors* err) {
  using TR = InTraits<Tin>;
  constexpr int kStages = TR::kStages;
  constexpr int kChunks = TR::kChunks;
  constexpr int kPerChunk = 32 / kChunks;               // elements per chunk
  constexpr uint32_t kInBytes = kTileElems * sizeof(Tin);
  constexpr uint32_t kCodeBytes = kTileElems * PACK / 8;
  constexpr int kChunkBits = kPerChunk * PACK;         // <= 64
  constexpr int L = (1 << (BITS - 1)) - 1;
  constexpr uint32_t kZeroCode = CODEC == 0 ? (uint32_t)L : 0u;

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* in_buf = smem;
  unsigned char* out_buf = smem + kStages * kInBytes;
  float* sc_buf = reinterpret_cast<float*>(out_buf + 2 * kCodeBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sc_buf + 2 * kTileBlocks);

  const int tid = threadIdx.x;
  const uint64_t ntiles = st.tile_begin[st.nseg];
  const uint64_t policy = policy_evict_first();

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_load = [&](uint64_t t, int s) {
    const int g = seg_of(st, t);
    const unsigned char* src = static_cast<const unsigned char*>(st.src[g]) +
                               (t - st.tile_begin[g]) * kInBytes;
    mbar_arrive_expect_tx(&full[s], kInBytes);
    bulk_g2s(in_buf + s * kInBytes, src, kInBytes, &full[s], policy);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const uint64_t t = blockIdx.x + (uint64_t)s * gridDim.x;
      if (t < ntiles) issue_load(t, s);
    }
  }

  const int rot = kChunks == 4 ? ((tid >> 1) & 3) : (tid & 7);
  const int lblk = tid >> 2;  // block within the tile

  for (uint64_t it = 0;; ++it) {
    const uint64_t t = blockIdx.x + it * gridDim.x;
    if (t >= ntiles) break;
    const int s = (int)(it % kStages);
    const uint32_t parity = (uint32_t)((it / kStages) & 1);
    mbar_wait(&full[s], parity);

    // ---- load my 32 elements, chunk j of the rotated order = chunk (j+rot)
    const unsigned char* row = in_buf + s * kInBytes + tid * (32 * sizeof(Tin));
    uint4 ch[kChunks];
#pragma unroll
    for (int j = 0; j < kChunks; ++j)
      ch[j] = lds128(row + ((j + rot) & (kChunks - 1)) * 16);

    // ---- block absmax on |x| bit patterns (integer max; NaN/Inf sort high)
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
    const float a = u2f(m);
    const int g = seg_of(st, t);
    const uint64_t tile_in_seg = t - st.tile_begin[g];
    if (m >= 0x7f800000u && (tid & 3) == 0)
      err_min(&err->nonfinite_block,
              (long long)(st.block_base[g] + tile_in_seg * kTileBlocks + lblk));

    const bool zero = (m == 0);
    const bool fast = fast_scale(a);
    float inv = 0.f, rcp = 0.f;
    if (!zero) {
      inv = codec_inv(CODEC, BITS, a);
      if (CODEC == 0 && TR::kBf16) rcp = fdiv(1.0f, a);
    }

    // ---- encode + pack each chunk (kPerChunk codes -> kChunkBits bits).
    // The fast/slow/zero choice is block-uniform: branch once, not per element.
    uint64_t pk[kChunks];
    if (zero) {
      uint64_t zc = 0;
#pragma unroll
      for (int e = 0; e < kPerChunk; ++e) zc |= (uint64_t)kZeroCode << (e * PACK);
#pragma unroll
      for (int j = 0; j < kChunks; ++j) pk[j] = zc;
    } else if (fast) {
      if constexpr (CODEC == 0 && TR::kBf16) {
        encode_linear_bf16_fast<BITS, PACK>(ch, a, inv, rcp, pk);
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
            acc |= (uint64_t)encode_one<BITS, CODEC, TR::kBf16>(x, a, inv, rcp, true) << (e * PACK);
          }
          pk[j] = acc;
        }
      }
    } else {
#pragma unroll 1
      for (int j = 0; j < kChunks; ++j) {
        const uint32_t wv[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
        uint64_t acc = 0;
#pragma unroll 1
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
    // undo the rotation: pk[(j + rot)] must hold chunk j
    if constexpr (kChunks == 4) rotr4(pk, rot); else rotr8(pk, rot);

    uint32_t words[PACK] = {};
    pack_chunks<kChunkBits>(words, pk, std::make_integer_sequence<int, kChunks>{});

    // ---- stage out: wait until the bulk store of two tiles ago released it
    const int ob = (int)(it & 1);
    if (tid == 0) bulk_wait_read<1>();
    __syncthreads();
    uint32_t* ow = reinterpret_cast<uint32_t*>(out_buf + ob * kCodeBytes) + tid * PACK;
    if constexpr (PACK % 4 == 0) {
#pragma unroll
      for (int k = 0; k < PACK / 4; ++k)
        sts128(ow + 4 * k, make_uint4(words[4 * k], words[4 * k + 1],
                                      words[4 * k + 2], words[4 * k + 3]));
    } else {
#pragma unroll
      for (int k = 0; k < PACK; ++k) ow[k] = words[k];
    }
    if ((tid & 3) == 0) sc_buf[ob * kTileBlocks + lblk] = a;
    fence_proxy_async_smem();
    __syncthreads();

    if (tid == 0) {
      unsigned char* cdst = static_cast<unsigned char*>(st.codes[g]) + tile_in_seg * kCodeBytes;
      float* sdst = st.scales[g] + tile_in_seg * kTileBlocks;
      bulk_s2g(cdst, out_buf + ob * kCodeBytes, kCodeBytes);
      bulk_s2g(sdst, sc_buf + ob * kTileBlocks, kTileBlocks * 4);
      bulk_commit();
      const uint64_t nt = t + (uint64_t)kStages * gridDim.x;
      if (nt < ntiles) issue_load(nt, s);
    }
  }
  if (tid == 0) bulk_wait_all<0>();
}

// ---------------------------------------------------------------------------
// K1 (warp-autonomous variant): every warp streams its own 1024-element tiles
// — coalesced 128-bit global loads (next tile prefetched into registers while
// the current one is encoded), staged through a private 2 KB shared-memory
// slot so each lane reads its 32 consecutive elements conflict-free, codes
// written straight from registers (PACK 32-bit words per lane, contiguous per
// warp). No CTA-wide barrier anywhere; only __syncwarp.
// ---------------------------------------------------------------------------
constexpr int kWarpElems = 1024;
constexpr int kWarpsPerCta = 8;
#ifndef AGQ_QUANT_MINB
#define AGQ_QUANT_MINB 3
#endif
#ifndef AGQ_QUANT_MINB_FP4
#define AGQ_QUANT_MINB_FP4 AGQ_QUANT_MINB
#endif
#ifndef AGQ_DEQUANT_MINB
#define AGQ_DEQUANT_MINB 3
#endif

// Shared-memory swizzle of a warp tile: lane row r (32 elements = kChunks
// 16-byte chunks) keeps chunk c at slot (c + rot(r)) mod kChunks, so the
// coalesced writes (8 lanes = one 128-byte phase) and the per-row reads
// (8 rows, same chunk) are both bank-conflict free, and every lane sees its
// own row in natural order.
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
__device__ __forceinline__ TileRef locate(const SegTable& st, uint64_t t) {
  if (st.nseg == 1) return {0, t};
  const int g = seg_of(st, t);
  return {g, t - st.tile_begin[g]};
}

#ifndef AGQ_DQ_PREFETCH
#define AGQ_DQ_PREFETCH 2
#endif
#ifndef AGQ_FP8_DQ_TAB
#define AGQ_FP8_DQ_TAB 1  // FP8 dequant with FP32 scales via per-block tables
#endif
#ifndef AGQ_MINIFLOAT_FAST
#define AGQ_MINIFLOAT_FAST 1  // FP4/FP8 activation rows via the hardware conversions
#endif
#ifndef AGQ_Q_PREFETCH
#define AGQ_Q_PREFETCH 1
#endif
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
    if constexpr (CODEC == 0 && TR::kBf16 && AGQ_QUANT_WORDS) {
      const float rcp = fdiv(1.0f, a);  // one division per block: inv = L * (1/a)
      const float inv = fmul((float)L, rcp);
#pragma unroll
      for (int k = 0; k < PACK; ++k) words[k] = 0;
      encode_linear_bf16_words<BITS, PACK>(ch, pk2(inv, inv), pk2(rcp, rcp), pk2(-a, -a), words);
      return;
    } else if constexpr (CODEC == 0 && TR::kBf16) {
      const float rcp = fdiv(1.0f, a);
      encode_linear_bf16_fast<BITS, PACK>(ch, a, fmul((float)L, rcp), rcp, pk);
    } else if constexpr (CODEC != 0 && AGQ_MINIFLOAT_FAST) {
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
                                           int lane, const uint4 (&ch)[InTraits<Tin>::kChunks]) {
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
  const float a = u2f(m);
  if (m >= 0x7f800000u && (lane & 3) == 0)
    err_min(&err->nonfinite_block, (long long)(st.block_base[tr.g] + tr.lt * 8 + (lane >> 2)));
  uint32_t words[PACK];
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
                                  sizeof(Tin) != 2 ? 2 : CODEC == AGQ_CODEC_FP4_E2M1 ? AGQ_QUANT_MINB_FP4 : AGQ_QUANT_MINB)
    k_quant_warp(SegTable st, agq_errors* err) {
  pdl_launch_dependents();
  pdl_wait();  // the previous kernel's outputs (our inputs) are visible
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tin);    // 2 KB / 4 KB
  __shared__ __align__(16) unsigned char sbuf[kWarpsPerCta][kTileB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sbuf[warp];
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;

  auto load = [&](TileRef tr, uint4 (&buf)[kChunks]) {
    const unsigned char* src = static_cast<const unsigned char*>(st.src[tr.g]) + tr.lt * kTileB;
#pragma unroll
    for (int j = 0; j < kChunks; ++j) buf[j] = ldg128_stream(src + j * 512 + lane * 16);
  };
  constexpr int kPf = AGQ_Q_PREFETCH;  // tiles in flight per warp (registers)
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
#pragma unroll
    for (int j = 0; j < kChunks; ++j) sts128(wb + swz_of_linear<kChunks>(j * 512 + lane * 16), buf[0][j]);
    __syncwarp();
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
    uint4 ch[kChunks];
#pragma unroll
    for (int j = 0; j < kChunks; ++j) ch[j] = lds128(wb + swz_off<kChunks>(lane, j));
    __syncwarp();

    quant_tile<BITS, PACK, CODEC, Tin>(st, err, tr, lane, ch);
  }
}

// K1, cp.async ring variant (AGQ_ACT_KERNEL=cpa): each warp keeps
// AGQ_CPA_STAGES tiles in flight with 16-byte cp.async copies written straight
// into its swizzled shared slots (no register staging, no STS), waits for the
// oldest group, reads its row conflict-free and refills the slot.
#ifndef AGQ_CPA_STAGES
#define AGQ_CPA_STAGES 3
#endif
template <int BITS, int PACK, int CODEC, typename Tin>
__global__ void __launch_bounds__(kWarpsPerCta * 32, sizeof(Tin) == 2 ? AGQ_QUANT_MINB : 2)
    k_quant_cpa(SegTable st, agq_errors* err) {
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr int kStg = AGQ_CPA_STAGES;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tin);
  extern __shared__ __align__(128) unsigned char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = dsm + warp * kStg * kTileB;
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  // per-lane swizzled shared offsets (constant), one tile ref per slot, the
  // loop unrolled by the ring depth so the slot index is a constant
  const uint32_t wb_s = (uint32_t)__cvta_generic_to_shared(wb);
  uint32_t sw[kChunks], rd[kChunks];
#pragma unroll
  for (int j = 0; j < kChunks; ++j) {
    sw[j] = swz_of_linear<kChunks>(j * 512 + lane * 16);
    rd[j] = swz_off<kChunks>(lane, j);
  }
  TileRef trq[kStg];
  SegCursor cur;
  auto issue = [&](uint64_t tt, int slot) {
    if (tt < total) {
      trq[slot] = locate_from(st, tt, cur);
      const unsigned char* src = static_cast<const unsigned char*>(st.src[trq[slot].g]) +
                                 trq[slot].lt * kTileB + lane * 16;
      const uint32_t base = wb_s + slot * kTileB;
#pragma unroll
      for (int j = 0; j < kChunks; ++j) cp_async16_s(base + sw[j], src + j * 512);
    }
    cp_async_commit();  // always: keeps the group count uniform
  };
#pragma unroll
  for (int d = 0; d < kStg; ++d) issue(t + d * nw, d);
  while (t < total) {
#pragma unroll
    for (int slot = 0; slot < kStg; ++slot) {
      if (t >= total) break;
      cp_async_wait<kStg - 1>();
      __syncwarp();
      const TileRef tr = trq[slot];
      const uint32_t base = wb_s + slot * kTileB;
      uint4 ch[kChunks];
#pragma unroll
      for (int j = 0; j < kChunks; ++j) ch[j] = lds128_s(base + rd[j]);
      __syncwarp();
      issue(t + kStg * nw, slot);
      quant_tile<BITS, PACK, CODEC, Tin>(st, err, tr, lane, ch);
      t += nw;
    }
  }
  cp_async_wait<0>();
}

// K1, per-warp TMA ring variant (AGQ_ACT_KERNEL=wtma): each warp owns
// kWStages 2 KB shared slots filled by 1-D bulk copies that lane 0 keeps in
// flight (one mbarrier per slot), so up to kWStages tiles per warp are in
// flight without any register prefetch. Rows are read in a per-lane rotated
// chunk order (the bulk copy cannot swizzle) and put back with selects.
constexpr int kWStages = 4;

template <int BITS, int PACK, int CODEC, typename Tin>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 3)
    k_quant_wtma(SegTable st, agq_errors* err) {
  using TR = InTraits<Tin>;
  constexpr int kChunks = TR::kChunks;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tin);
  constexpr uint32_t kCodeB = kWarpElems * PACK / 8;
  extern __shared__ __align__(128) unsigned char dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* slots = dsm + warp * kWStages * kTileB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + kWarpsPerCta * kWStages * kTileB) + warp * kWStages;
  if (lane == 0) {
    for (int s2 = 0; s2 < kWStages; ++s2) mbar_init(&bars[s2], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t total = st.tile_begin[st.nseg];
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  const uint64_t first = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  const uint64_t policy = policy_evict_first();
  auto issue = [&](uint64_t t, int slot) {
    const TileRef tr = locate(st, t);
    mbar_arrive_expect_tx(&bars[slot], kTileB);
    bulk_g2s(slots + slot * kTileB,
             static_cast<const unsigned char*>(st.src[tr.g]) + tr.lt * kTileB, kTileB, &bars[slot],
             policy);
  };
  if (lane == 0)
    for (int s2 = 0; s2 < kWStages; ++s2) {
      const uint64_t t = first + (uint64_t)s2 * nw;
      if (t < total) issue(t, s2);
    }
  const int rot = kChunks == 4 ? ((lane >> 1) & 3) : (lane & 7);
  for (uint64_t it = 0;; ++it) {
    const uint64_t t = first + it * nw;
    if (t >= total) break;
    const int slot = (int)(it % kWStages);
    mbar_wait(&bars[slot], (uint32_t)((it / kWStages) & 1));
    uint4 ch[kChunks];
    const unsigned char* row = slots + slot * kTileB + lane * (32 * sizeof(Tin));
#pragma unroll
    for (int j = 0; j < kChunks; ++j) ch[j] = lds128(row + ((j + rot) & (kChunks - 1)) * 16);
    __syncwarp();
    if (lane == 0) {
      const uint64_t nt = t + (uint64_t)kWStages * nw;
      if (nt < total) issue(nt, slot);
    }
    // back to natural chunk order (slot j holds chunk j + rot)
    if constexpr (kChunks == 4) rotr4(ch, rot); else rotr8(ch, rot);
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
    const float a = u2f(m);
    const TileRef tr = locate(st, t);
    if (m >= 0x7f800000u && (lane & 3) == 0)
      err_min(&err->nonfinite_block, (long long)(st.block_base[tr.g] + tr.lt * 8 + (lane >> 2)));
    uint32_t words[PACK];
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
}

// K2 warp-autonomous variant: lane loads its PACK code words (+ block scale),
// next tile prefetched, decodes 32 values, stages the 2/4 KB warp output in
// shared memory and writes it back with coalesced 128-bit stores.
template <int BITS, int PACK, int CODEC, typename Tout>
__global__ void __launch_bounds__(kWarpsPerCta * 32, sizeof(Tout) == 2 ? AGQ_DEQUANT_MINB : 2)
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

__device__ __noinline__ float decode_slow(int codec, int bits, uint32_t c, float s,
                                         const double* fp8lut) {
  if (codec == 2) {
    if ((c & 0x7fu) == 0x7fu) return u2f(0x7fc00000u | ((c & 0x80u) << 24));
    const float mag = d2f_rn(dmul(fp8lut[c & 0x7fu], (double)s));
    return u2f(f2u(mag) | ((c & 0x80u) << 24));
  }
  return dequant_double(codec, bits, c, s);
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

template <int BITS, int PACK, int NPER>
__device__ __forceinline__ void decode_linear_fast(uint64_t bits, float s, float (&v)[NPER]) {
  constexpr int L = (1 << (BITS - 1)) - 1;
  const f32x2 s2 = pk2(s, s);
  const f32x2 off2 = pk2(-(kMagicRound + (float)L), -(kMagicRound + (float)L));
  const f32x2 den2 = pk2(-(float)L, -(float)L), rden2 = pk2(1.0f / L, 1.0f / L);
  const uint32_t mb = opaque_magic();
#pragma unroll
  for (int e = 0; e < NPER; e += 2) {
    const uint32_t c0 = (uint32_t)(bits >> (e * PACK)) & ((1u << BITS) - 1u);
    const uint32_t c1 = (uint32_t)(bits >> ((e + 1) * PACK)) & ((1u << BITS) - 1u);
    const f32x2 cp = add2(pk2(u2f(mb | c0), u2f(mb | c1)), off2);
    const f32x2 p = mul2(cp, s2);
    const f32x2 q0 = mul2(p, rden2);
    const f32x2 r = fma2(q0, den2, p);
    up2(fma2(r, rden2, q0), v[e], v[e + 1]);
  }
}

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
__global__ void __launch_bounds__(kThreads)
    k_dequant_tiled(SegTable st, int validate, agq_errors* err) {
  constexpr int kStages = 4;
  constexpr int kChunks = OutTraits<Tout>::kChunks;
  constexpr int kPerChunk = 32 / kChunks;
  constexpr uint32_t kCodeBytes = kTileElems * PACK / 8;
  constexpr uint32_t kStageBytes = kCodeBytes + kTileBlocks * 4;
  constexpr uint32_t kOutBytes = kTileElems * sizeof(Tout);
  constexpr int kChunkBits = kPerChunk * PACK;
  constexpr bool kBf16Out = sizeof(Tout) == 2;

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* in_buf = smem;                                // stages
  unsigned char* out_buf = smem + kStages * kStageBytes;       // 2 x out
  uint64_t* full = reinterpret_cast<uint64_t*>(out_buf + 2 * kOutBytes);
  double* fp8lut = reinterpret_cast<double*>(full + kStages);

  const int tid = threadIdx.x;
  const uint64_t ntiles = st.tile_begin[st.nseg];
  const uint64_t policy = policy_evict_first();
  if (CODEC == 2) fill_fp8_unit_lut(fp8lut);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_load = [&](uint64_t t, int s) {
    const int g = seg_of(st, t);
    const uint64_t lt = t - st.tile_begin[g];
    unsigned char* dst = in_buf + s * kStageBytes;
    mbar_arrive_expect_tx(&full[s], kStageBytes);
    bulk_g2s(dst, static_cast<const unsigned char*>(st.codes[g]) + lt * kCodeBytes,
             kCodeBytes, &full[s], policy);
    bulk_g2s(dst + kCodeBytes, st.scales[g] + lt * kTileBlocks, kTileBlocks * 4,
             &full[s], policy);
  };
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const uint64_t t = blockIdx.x + (uint64_t)s * gridDim.x;
      if (t < ntiles) issue_load(t, s);
    }
  }

  const int rot = kChunks == 4 ? ((tid >> 1) & 3) : (tid & 7);
  const int lblk = tid >> 2;

  for (uint64_t it = 0;; ++it) {
    const uint64_t t = blockIdx.x + it * gridDim.x;
    if (t >= ntiles) break;
    const int s = (int)(it % kStages);
    mbar_wait(&full[s], (uint32_t)((it / kStages) & 1));
    const unsigned char* sb = in_buf + s * kStageBytes;
    const uint32_t* wsrc = reinterpret_cast<const uint32_t*>(sb) + tid * PACK;
    uint32_t words[PACK];
    if constexpr (PACK % 4 == 0) {
#pragma unroll
      for (int k = 0; k < PACK / 4; ++k) {
        const uint4 v = lds128(wsrc + 4 * k);
        words[4 * k] = v.x; words[4 * k + 1] = v.y;
        words[4 * k + 2] = v.z; words[4 * k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < PACK; ++k) words[k] = wsrc[k];
    }
    const float sc = reinterpret_cast<const float*>(sb + kCodeBytes)[lblk];
    const int g = seg_of(st, t);
    const uint64_t lt = t - st.tile_begin[g];

    if (validate) {
      if (!(sc >= 0.0f) || !(sc <= 3.402823466e38f)) {
        if ((tid & 3) == 0)
          err_min(&err->bad_scale_block,
                  (long long)(st.block_base[g] + lt * kTileBlocks + lblk));
      }
      if constexpr (PACK == 8 && BITS < 8) {
        uint32_t bad = 0;
#pragma unroll
        for (int k = 0; k < PACK; ++k) bad |= words[k] & (0x01010101u * (0xffu << BITS & 0xffu));
        if (bad) {
          // lowest offending element of this thread
#pragma unroll 1
          for (int e = 0; e < 32; ++e) {
            const uint32_t c = (words[e >> 2] >> ((e & 3) * 8)) & 0xffu;
            if (c >> BITS) {
              err_min(&err->bad_code_index,
                      (long long)((st.block_base[g] + lt * kTileBlocks) * kBlock + tid * 32 + e));
              break;
            }
          }
        }
      }
    }

    const bool fast = is_bf16_value(sc) && fast_scale(sc);
    uint64_t pk[kChunks];
    unpack_chunks<kChunkBits>(words, pk, std::make_integer_sequence<int, kChunks>{});
    // rotated order: slot j holds chunk (j + rot)
    if constexpr (kChunks == 4) rotl4(pk, rot); else rotl8(pk, rot);

    const int ob = (int)(it & 1);
    if (tid == 0) bulk_wait_read<1>();
    __syncthreads();
    unsigned char* orow = out_buf + ob * kOutBytes + tid * (32 * sizeof(Tout));
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      float v[kPerChunk];
      if (CODEC == 0 && fast) {
        decode_linear_fast<BITS, PACK, kPerChunk>(pk[j], sc, v);
      } else if (fast) {
#pragma unroll
        for (int e = 0; e < kPerChunk; ++e) {
          const uint32_t c = (uint32_t)(pk[j] >> (e * PACK)) & ((1u << BITS) - 1u);
          v[e] = decode_one<BITS, CODEC>(c, sc, true, fp8lut);
        }
      } else {
#pragma unroll 1
        for (int e = 0; e < kPerChunk; ++e) {
          const uint32_t c = (uint32_t)(pk[j] >> (e * PACK)) & ((1u << BITS) - 1u);
          v[e] = decode_slow(CODEC, BITS, c, sc, fp8lut);
        }
      }
      uint4 o;
      if constexpr (kBf16Out) {
        uint32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (CODEC == 2)
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
      sts128(orow + ((j + rot) & (kChunks - 1)) * 16, o);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      unsigned char* dst = static_cast<unsigned char*>(st.dst[g]) + lt * kOutBytes;
      bulk_s2g(dst, out_buf + ob * kOutBytes, kOutBytes);
      bulk_commit();
      const uint64_t nt = t + (uint64_t)kStages * gridDim.x;
      if (nt < ntiles) issue_load(nt, s);
    }
  }
  if (tid == 0) bulk_wait_all<0>();
}

template <int BITS, int PACK, int CODEC, typename Tout>
__global__ void __launch_bounds__(kWarpsPerCta * 32, sizeof(Tout) == 2 ? AGQ_DEQUANT_MINB : 2)
    k_dequant_warp(SegTable st, int validate, agq_errors* err) {
  pdl_launch_dependents();
  pdl_wait();
  constexpr int kChunks = OutTraits<Tout>::kChunks;
  constexpr int kPerChunk = 32 / kChunks;
  constexpr int kChunkBits = kPerChunk * PACK;
  constexpr uint32_t kTileB = kWarpElems * sizeof(Tout);
  constexpr uint32_t kCodeB = kWarpElems * PACK / 8;
  constexpr bool kBf16Out = sizeof(Tout) == 2;
  __shared__ __align__(16) unsigned char sbuf[kWarpsPerCta][kTileB];
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sbuf[warp];
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
  // AGQ_DQ_PREFETCH tiles in flight per warp (codes + scale are <= 9
  // registers per tile, so a second tile in flight is cheap and covers the
  // load latency the kernel otherwise stalls on)
  constexpr int kPf = AGQ_DQ_PREFETCH;
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
    if constexpr (CODEC != 0 && AGQ_MINIFLOAT_FAST) {
      if constexpr (CODEC == 2) mfast = fast && !fp8_row_has_nan<PACK>(cw);
      else mfast = fast;
    }
    bool tfast = false;  // FP8, FP32 scale: block-table decode
    uint32_t tb_s = 0;
    if constexpr (CODEC == 2 && AGQ_FP8_DQ_TAB) {
      float* wt = dqtab + (threadIdx.x >> 5) * 64;
      const int j0 = (lane & 3) * 2;
      __syncwarp();  // the previous tile's lookups are done
      wt[(lane >> 2) * 8 + j0] = fp8_tab_entry_half(fp8_t8(j0), s);
      wt[(lane >> 2) * 8 + j0 + 1] = fp8_tab_entry_half(fp8_t8(j0 + 1), s);
      __syncwarp();
      uint32_t unsafe = 0;
#pragma unroll
      for (int k = 0; k < PACK; ++k) unsafe |= fp8_tab_unsafe(cw[k]);
      tfast = !fast && dq_fast(s) && unsafe == 0;
      tb_s = (uint32_t)__cvta_generic_to_shared(wt + (lane >> 2) * 8);
    }
    uint64_t pk[kChunks];
    unpack_chunks<kChunkBits>(cw, pk, std::make_integer_sequence<int, kChunks>{});
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      float v[kPerChunk];
      if (CODEC == 2 && tfast) {
#pragma unroll
        for (int q = 0; q < kPerChunk / 4; ++q) {
          const uint32_t w1[1] = {cw[(j * kPerChunk) / 4 + q]};
          float a4[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // + 0.0f: exact (entries are never 0)
          dq_tab_accum<1>(w1, tb_s, a4);
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
      sts128(wb + swz_off<kChunks>(lane, j), o);
    }
    __syncwarp();
    unsigned char* dst = static_cast<unsigned char*>(st.dst[tr.g]) + tr.lt * kTileB;
#pragma unroll
    for (int j = 0; j < kChunks; ++j)
      *reinterpret_cast<uint4*>(dst + j * 512 + lane * 16) =
          lds128(wb + swz_of_linear<kChunks>(j * 512 + lane * 16));
    __syncwarp();
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

// Activation-kernel variant: warp-autonomous (default) or the CTA-wide TMA
// bulk-copy pipeline; AGQ_ACT_KERNEL=tma selects the latter.
bool act_warp() {
  static const bool w = [] {
    const char* e = getenv("AGQ_ACT_KERNEL");
    return !(e && e[0] == 't');
  }();
  return w;
}
bool act_wtma() {
  static const bool w = [] {
    const char* e = getenv("AGQ_ACT_KERNEL");
    return e && e[0] == 'w' && e[1] == 't';
  }();
  return w;
}
uint64_t act_unit() { return act_warp() ? (uint64_t)kWarpElems : (uint64_t)kTileElems; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename K>
int grid_for(K kernel, size_t smem, uint64_t ntiles) {
  static_assert(sizeof(K) > 0, "");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (occ < 1) occ = 1;
  const uint64_t g = (uint64_t)num_sms() * (uint64_t)occ;
  return (int)(ntiles < g ? ntiles : g);
}

template <typename K>
cudaError_t prep(K kernel, size_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int gen_grid(uint64_t work, int threads) {
  const uint64_t g = (work + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int BITS, int PACK, int CODEC, typename Tin>
agq_status launch_quant_tiled(const SegTable& st, agq_errors* err, cudaStream_t s) {
  using TR = InTraits<Tin>;
  const size_t smem = TR::kStages * (size_t)kTileElems * sizeof(Tin) +
                      2 * (size_t)kTileElems * PACK / 8 + 2 * kTileBlocks * 4 +
                      TR::kStages * 8;
  auto k = k_quant_tiled<BITS, PACK, CODEC, Tin>;
  cudaError_t e = prep(k, smem);
  if (e != cudaSuccess) return cuda_fail(e, "quantize: smem attribute");
  const int grid = grid_for(k, smem, st.tile_begin[st.nseg]);
  k<<<grid, kThreads, smem, s>>>(st, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "quantize: launch");
}

template <int BITS, int PACK, int CODEC, typename Tin>
agq_status launch_quant_wtma(const SegTable& st, agq_errors* err, cudaStream_t s) {
  auto k = k_quant_wtma<BITS, PACK, CODEC, Tin>;
  const size_t smem = (size_t)kWarpsPerCta * kWStages * (kWarpElems * sizeof(Tin) + 8);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "quantize: smem attribute");
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarpsPerCta * 32, smem);
  if (occ < 1) occ = 1;
  const uint64_t tiles = st.tile_begin[st.nseg];
  const uint64_t want = (tiles + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  k<<<(int)(want < cap ? want : cap), kWarpsPerCta * 32, smem, s>>>(st, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "quantize: launch");
}

template <int BITS, int PACK, int CODEC, typename Tin>
agq_status launch_quant_cpa(const SegTable& st, agq_errors* err, cudaStream_t s) {
  auto k = k_quant_cpa<BITS, PACK, CODEC, Tin>;
  const size_t smem = (size_t)kWarpsPerCta * AGQ_CPA_STAGES * kWarpElems * sizeof(Tin);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarpsPerCta * 32, smem);
  if (occ < 1) occ = 1;
  const uint64_t tiles = st.tile_begin[st.nseg];
  const uint64_t want = (tiles + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  k<<<(int)(want < cap ? want : cap), kWarpsPerCta * 32, smem, s>>>(st, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "quantize: launch");
}

bool act_cpa() {
  static const bool v = [] {
    const char* e = getenv("AGQ_ACT_KERNEL");
    return e && strcmp(e, "cpa") == 0;
  }();
  return v;
}

// Launch with programmatic stream serialization (PDL) unless AGQ_PDL=0: the
// kernel's launch and prologue overlap the previous kernel's tail; the
// kernels wait (griddepcontrol.wait) before touching global memory.
bool act_pdl() {
  static const bool v = [] {
    const char* e = getenv("AGQ_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*k)(KArgs...), int grid, int block, size_t smem,
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
  cfg.numAttrs = act_pdl() ? 1 : 0;
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
  if (act_wtma()) return launch_quant_wtma<BITS, PACK, CODEC, Tin>(st, err, s);
  if (act_cpa()) return launch_quant_cpa<BITS, PACK, CODEC, Tin>(st, err, s);
  auto k = k_quant_warp<BITS, PACK, CODEC, Tin>;
  static const int occ = occupancy_of(k, kWarpsPerCta * 32, 0);
  const uint64_t tiles = st.tile_begin[st.nseg];
  const uint64_t want = (tiles + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  cudaError_t e = launch_maybe_pdl(k, (int)(want < cap ? want : cap), kWarpsPerCta * 32, 0, s, st, err);
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
  cudaError_t e = launch_maybe_pdl(k, (int)(want < cap ? want : cap), kWarpsPerCta * 32, 0, s, st,
                                   validate, err);
  count_launch();
  return cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "dequantize: launch");
}

template <int PACK, typename Tin>
agq_status quant_dispatch_bits(int bits, int codec, const SegTable& st,
                               agq_errors* err, cudaStream_t s) {
  if (codec == AGQ_CODEC_FP8_E4M3) return act_warp() ? launch_quant_warp<8, 8, 2, Tin>(st, err, s) : launch_quant_tiled<8, 8, 2, Tin>(st, err, s);
  if (codec == AGQ_CODEC_FP4_E2M1) return act_warp() ? launch_quant_warp<4, PACK == 8 ? 8 : 4, 1, Tin>(st, err, s) : launch_quant_tiled<4, PACK == 8 ? 8 : 4, 1, Tin>(st, err, s);
  switch (bits) {
    case 4: return act_warp() ? launch_quant_warp<4, PACK == 8 ? 8 : 4, 0, Tin>(st, err, s) : launch_quant_tiled<4, PACK == 8 ? 8 : 4, 0, Tin>(st, err, s);
    case 5: return act_warp() ? launch_quant_warp<5, PACK == 8 ? 8 : 5, 0, Tin>(st, err, s) : launch_quant_tiled<5, PACK == 8 ? 8 : 5, 0, Tin>(st, err, s);
    case 6: return act_warp() ? launch_quant_warp<6, PACK == 8 ? 8 : 6, 0, Tin>(st, err, s) : launch_quant_tiled<6, PACK == 8 ? 8 : 6, 0, Tin>(st, err, s);
    case 7: return act_warp() ? launch_quant_warp<7, PACK == 8 ? 8 : 7, 0, Tin>(st, err, s) : launch_quant_tiled<7, PACK == 8 ? 8 : 7, 0, Tin>(st, err, s);
    default: return act_warp() ? launch_quant_warp<8, 8, 0, Tin>(st, err, s) : launch_quant_tiled<8, 8, 0, Tin>(st, err, s);
  }
}

template <int BITS, int PACK, int CODEC, typename Tout>
agq_status launch_dequant_tiled(const SegTable& st, int validate, agq_errors* err,
                                cudaStream_t s) {
  const size_t smem = 4 * ((size_t)kTileElems * PACK / 8 + kTileBlocks * 4) +
                      2 * (size_t)kTileElems * sizeof(Tout) + 4 * 8 + 128 * 8;
  auto k = k_dequant_tiled<BITS, PACK, CODEC, Tout>;
  cudaError_t e = prep(k, smem);
  if (e != cudaSuccess) return cuda_fail(e, "dequantize: smem attribute");
  const int grid = grid_for(k, smem, st.tile_begin[st.nseg]);
  k<<<grid, kThreads, smem, s>>>(st, validate, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "dequantize: launch");
}

template <int PACK, typename Tout>
agq_status dequant_dispatch_bits(int bits, int codec, const SegTable& st,
                                 int validate, agq_errors* err, cudaStream_t s) {
  if (codec == AGQ_CODEC_FP8_E4M3) return act_warp() ? launch_dequant_warp<8, 8, 2, Tout>(st, validate, err, s) : launch_dequant_tiled<8, 8, 2, Tout>(st, validate, err, s);
  if (codec == AGQ_CODEC_FP4_E2M1) return act_warp() ? launch_dequant_warp<4, PACK == 8 ? 8 : 4, 1, Tout>(st, validate, err, s) : launch_dequant_tiled<4, PACK == 8 ? 8 : 4, 1, Tout>(st, validate, err, s);
  switch (bits) {
    case 4: return act_warp() ? launch_dequant_warp<4, PACK == 8 ? 8 : 4, 0, Tout>(st, validate, err, s) : launch_dequant_tiled<4, PACK == 8 ? 8 : 4, 0, Tout>(st, validate, err, s);
    case 5: return act_warp() ? launch_dequant_warp<5, PACK == 8 ? 8 : 5, 0, Tout>(st, validate, err, s) : launch_dequant_tiled<5, PACK == 8 ? 8 : 5, 0, Tout>(st, validate, err, s);
    case 6: return act_warp() ? launch_dequant_warp<6, PACK == 8 ? 8 : 6, 0, Tout>(st, validate, err, s) : launch_dequant_tiled<6, PACK == 8 ? 8 : 6, 0, Tout>(st, validate, err, s);
    case 7: return act_warp() ? launch_dequant_warp<7, PACK == 8 ? 8 : 7, 0, Tout>(st, validate, err, s) : launch_dequant_tiled<7, PACK == 8 ? 8 : 7, 0, Tout>(st, validate, err, s);
    default: return act_warp() ? launch_dequant_warp<8, 8, 0, Tout>(st, validate, err, s) : launch_dequant_tiled<8, 8, 0, Tout>(st, validate, err, s);
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

agq_status quantize_device(const void* x, int x_dtype, uint64_t n, int bits,
                           uint32_t block, int codec, void* codes, int layout,
                           float* scales, agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  const int pack = layout == AGQ_CODES_PACKED ? bits : 8;
  const size_t esz = x_dtype == AGQ_BF16 ? 2 : 4;
  uint64_t ntiles = 0;
  if (block == (uint32_t)kBlock && aligned16(x) && aligned16(codes) && aligned16(scales))
    ntiles = n / act_unit();
  if (ntiles > 0) {
    SegTable st{};
    st.src[0] = x;
    st.codes[0] = codes;
    st.scales[0] = scales;
    st.tile_begin[0] = 0;
    st.tile_begin[1] = ntiles;
    st.block_base[0] = 0;
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
  const uint64_t done = ntiles * act_unit();
  if (done == n) return AGQ_OK;
  // tail (block-aligned start, byte-aligned in the packed stream)
  const uint64_t rest = n - done;
  const long long bb = (long long)(done / block);
  void* ctail = static_cast<uint8_t*>(codes) + (done * pack) / 8;
  if (x_dtype == AGQ_BF16)
    return quant_generic(reinterpret_cast<const __nv_bfloat16*>(x) + done, rest, bits, block,
                         codec, ctail, layout, scales + done / block, bb, err, s);
  return quant_generic(reinterpret_cast<const float*>(x) + done, rest, bits, block, codec, ctail,
                       layout, scales + done / block, bb, err, s);
  (void)esz;
}

agq_status dequantize_device(const void* codes, int layout, const float* scales,
                             uint64_t n, int bits, uint32_t block, int codec,
                             void* out, int out_dtype, int validate,
                             agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  const int pack = layout == AGQ_CODES_PACKED ? bits : 8;
  uint64_t ntiles = 0;
  if (block == (uint32_t)kBlock && aligned16(out) && aligned16(codes) && aligned16(scales))
    ntiles = n / act_unit();
  if (ntiles > 0) {
    SegTable st{};
    st.codes[0] = const_cast<void*>(codes);
    st.scales[0] = const_cast<float*>(scales);
    st.dst[0] = out;
    st.tile_begin[1] = ntiles;
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
  const uint64_t done = ntiles * act_unit();
  if (done == n) return AGQ_OK;
  const uint64_t rest = n - done;
  const uint8_t* ctail = static_cast<const uint8_t*>(codes) + (done * pack) / 8;
  const float* stail = scales + done / block;
  if (out_dtype == AGQ_BF16)
    k_dequant_generic<__nv_bfloat16><<<gen_grid(rest, 256), 256, 0, s>>>(
        ctail, layout, stail, rest, bits, block, codec,
        static_cast<__nv_bfloat16*>(out) + done, validate, (long long)done, err);
  else
    k_dequant_generic<float><<<gen_grid(rest, 256), 256, 0, s>>>(
        ctail, layout, stail, rest, bits, block, codec, static_cast<float*>(out) + done,
        validate, (long long)done, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "dequantize (generic): launch");
}

agq_status quantize_grouped_device(const agq_segment* segs, int nseg, int x_dtype,
                                   int bits, int codec, agq_errors* err,
                                   cudaStream_t s) {
  // Full tiles of every segment in one launch; tails individually.
  SegTable st{};
  uint64_t tiles = 0, blocks = 0;
  int k = 0;
  for (int i = 0; i < nseg; ++i) {
    const uint64_t nt = aligned16(segs[i].x) && aligned16(segs[i].codes) &&
                                aligned16(segs[i].scales)
                            ? segs[i].n / act_unit()
                            : 0;
    if (nt > 0) {
      if (k == kMaxSeg) return set_error(AGQ_ERR_INVALID_ARGUMENT, "too many segments");
      st.src[k] = segs[i].x;
      st.codes[k] = segs[i].codes;
      st.scales[k] = segs[i].scales;
      st.tile_begin[k] = tiles;
      st.block_base[k] = blocks;
      tiles += nt;
      ++k;
    }
    blocks += (segs[i].n + kBlock - 1) / kBlock;
  }
  st.tile_begin[k] = tiles;
  st.nseg = k;
  if (k > 0) {
    agq_status r = x_dtype == AGQ_BF16
                       ? quant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, err, s)
                       : quant_dispatch_bits<0, float>(bits, codec, st, err, s);
    if (r != AGQ_OK) return r;
  }
  for (int i = 0; i < nseg; ++i) {
    const bool tiled = aligned16(segs[i].x) && aligned16(segs[i].codes) && aligned16(segs[i].scales);
    const uint64_t done = tiled ? (segs[i].n / act_unit()) * act_unit() : 0;
    if (done == segs[i].n) continue;
    const size_t esz = x_dtype == AGQ_BF16 ? 2 : 4;
    agq_status r = quantize_device(static_cast<const char*>(segs[i].x) + done * esz, x_dtype,
                                   segs[i].n - done, bits, kBlock, codec,
                                   static_cast<uint8_t*>(segs[i].codes) + done * bits / 8,
                                   AGQ_CODES_PACKED, segs[i].scales + done / kBlock, err, s);
    if (r != AGQ_OK) return r;
  }
  return AGQ_OK;
}

agq_status dequantize_grouped_device(const agq_segment* segs, int nseg, int out_dtype,
                                     int bits, int codec, cudaStream_t s) {
  SegTable st{};
  uint64_t tiles = 0;
  int k = 0;
  for (int i = 0; i < nseg; ++i) {
    const bool tiled = aligned16(segs[i].x) && aligned16(segs[i].codes) && aligned16(segs[i].scales);
    const uint64_t nt = tiled ? segs[i].n / act_unit() : 0;
    if (nt > 0) {
      if (k == kMaxSeg) return set_error(AGQ_ERR_INVALID_ARGUMENT, "too many segments");
      st.codes[k] = segs[i].codes;
      st.scales[k] = segs[i].scales;
      st.dst[k] = const_cast<void*>(segs[i].x);
      st.tile_begin[k] = tiles;
      tiles += nt;
      ++k;
    }
  }
  st.tile_begin[k] = tiles;
  st.nseg = k;
  if (k > 0) {
    agq_status r = out_dtype == AGQ_BF16
                       ? dequant_dispatch_bits<0, __nv_bfloat16>(bits, codec, st, 0, nullptr, s)
                       : dequant_dispatch_bits<0, float>(bits, codec, st, 0, nullptr, s);
    if (r != AGQ_OK) return r;
  }
  for (int i = 0; i < nseg; ++i) {
    const bool tiled = aligned16(segs[i].x) && aligned16(segs[i].codes) && aligned16(segs[i].scales);
    const uint64_t done = tiled ? (segs[i].n / act_unit()) * act_unit() : 0;
    if (done == segs[i].n) continue;
    const size_t esz = out_dtype == AGQ_BF16 ? 2 : 4;
    agq_status r = dequantize_device(
        static_cast<const uint8_t*>(segs[i].codes) + done * bits / 8, AGQ_CODES_PACKED,
        segs[i].scales + done / kBlock, segs[i].n - done, bits, kBlock, codec,
        static_cast<char*>(const_cast<void*>(segs[i].x)) + done * esz, out_dtype, 0, nullptr, s);
    if (r != AGQ_OK) return r;
  }
  return AGQ_OK;
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
