// L2a gradient path on sm_100a: fused FP8-E4M3 accumulate (K3) and the
// local reduce + requantize of the decomposed all-reduce (K4).
//
// Reference: /root/reference/proj/include/agq/collective.hpp:101-147
// (round_bf16/round_fp16, local_accumulate) and :250-284 (local reduce).
// Both produce codes/scales bit-identical to the reference:
//   dequant  = (float)(fl64(e4m3(c)/448) * (double)scale)   (DMUL + F2F)
//   sum      = fp32 adds in the reference's order (+0.0f first for K4)
//   requant  = fresh block absmax, exact E4M3 rounding (agq_numerics.cuh)
//
// K3 (block 128): warp-autonomous persistent kernel, 16 elements per lane
// (8 lanes per block), one pass over HBM: 1 + 4/128 bytes in, 4 (or 2) bytes
// of local gradient in, 1 + 4/128 out. (A TMA tile pipeline was built,
// verified bit-exact and measured slower.)
//
// K4 uses plain 128-bit loads so that any piece may live in another GPU's
// memory (NVLink peer pointers) — the fused all-reduce runs the same code.
#include <cstdlib>

#include "agq_grad.cuh"

namespace agqk {

// ---------------------------------------------------------------------------
// K3: each warp streams 512-element tiles
// (16 per lane, 8 lanes per 128-block). Codes (16 B/lane), the block scale
// and the lane's 16 local values (one or two 256-bit loads: 32 B of BF16 or
// 64 B of FP32, every 32-byte sector read once) are loaded straight to
// registers, the next tile's while the current one is computed. No shared-
// memory staging and no CTA-wide barrier.
// ---------------------------------------------------------------------------
constexpr int kAccWarpElems = 512;
constexpr int kAccWarps = 8;

// A non-finite block sum: a non-finite local gradient makes it so; tell the
// two reference errors apart (collective.hpp:138-139 vs the requant's block
// error) by re-reading this lane's 16 local values.
template <bool BF16L>
__device__ __noinline__ void acc_report_nonfinite(const unsigned char* lp, int lane, uint64_t t,
                                                  uint64_t gblk, long long eb, agq_errors* err) {
  uint32_t lbad = 0;
  for (int e = 0; e < 16; ++e) {
    const uint32_t u = BF16L ? (uint32_t)reinterpret_cast<const uint16_t*>(lp)[e] << 16
                             : reinterpret_cast<const uint32_t*>(lp)[e];
    lbad |= (uint32_t)((u & 0x7f800000u) == 0x7f800000u) << e;
  }
  if (lbad)
    err_min(&err->nonfinite_local,
            eb * kBlock + (long long)(t * kAccWarpElems + lane * 16 + (__ffs(lbad) - 1)));
  if ((lane & 7) == 0) err_min(&err->nonfinite_block, eb + (long long)gblk);
}

// Three resident CTAs per SM (24 warps).
template <bool BF16L, int PREC>
__global__ void __launch_bounds__(kAccWarps * 32, 3)
    k_accumulate_warp(const uint8_t* codes, const float* scales, const void* local,
                      uint64_t ntiles, uint8_t* out_codes, float* out_scales, long long eb,
                      agq_errors* err) {
  // eb: block index of element 0 in the error record (chunked host calls)
  constexpr int kLW = BF16L ? 8 : 16;  // 32-bit words of local gradient per lane
  constexpr uint32_t kLocTileB = kAccWarpElems * (BF16L ? 2 : 4);  // 1 KB / 2 KB
  __shared__ double t16[kDqTable];
  __shared__ float btab[kAccWarps][32];  // per warp: 4 blocks x 8 table entries
  fill_fp8_dq_table(t16);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double t8 = fp8_t8(lane & 7);  // lane 8b+j builds entry j of block b
  const uint32_t mytab = (uint32_t)__cvta_generic_to_shared(&btab[warp][lane & ~7]);
  const uint64_t nw = (uint64_t)gridDim.x * kAccWarps;
  uint64_t t = (uint64_t)blockIdx.x * kAccWarps + warp;
  const unsigned char* lbase = static_cast<const unsigned char*>(local) + lane * (kLW * 4);

  // one tile in flight per warp beyond the one being computed
  uint4 pc;             // 16 codes
  float ps;             // block scale
  uint32_t pl[kLW];     // 16 local values
  auto load = [&](uint64_t tt) {
    pc = ldg128_stream(codes + tt * kAccWarpElems + lane * 16);
    ps = __ldg(scales + tt * 4 + (lane >> 3));
#pragma unroll
    for (int h = 0; h < kLW / 8; ++h) ldg256_stream(lbase + tt * kLocTileB + h * 32, pl + 8 * h);
  };
  if (t < ntiles) load(t);
  for (; t < ntiles; t += nw) {
    const uint32_t cw[4] = {pc.x, pc.y, pc.z, pc.w};
    const float sc = ps;
    float l[16];
#pragma unroll
    for (int k = 0; k < kLW; ++k) {
      if constexpr (BF16L) {
        l[2 * k] = u2f(pl[k] << 16);
        l[2 * k + 1] = u2f(pl[k] & 0xffff0000u);
      } else {
        l[k] = u2f(pl[k]);
      }
    }
    btab[warp][lane] = fp8_tab_entry_f16(t8, sc);  // T[M] (dq_f16_accum)
    __syncwarp();
    if (t + nw < ntiles) load(t + nw);
    const uint64_t gblk = t * 4 + (lane >> 3);
    if ((!(sc >= 0.0f) || !(sc <= 3.402823466e38f)) && (lane & 7) == 0)
      err_min(&err->bad_scale_block, eb + (long long)gblk);
    float v[16];
    // block-table decode of every code (f16 route, exact; the 256-entry
    // table of exact units only for zero / extreme block scales):
    // v = l + dq (exact product, one rounding: = fadd(dq, l))
    if (dq_fast(sc)) {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = l[e];
      dq_f16_accum<4>(cw, mytab, v);
    } else {  // zero block or an extreme scale: full table
      const double sd = (double)sc;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        v[e] = fadd(fp8_dq_lut(byte_of(cw[e >> 2], e & 3), sd, t16), l[e]);
    }
    // Rounding to BF16 / FP16 (collective.hpp:141-142) is monotone and odd,
    // so the absmax of the rounded sums is the rounded absmax of the raw
    // sums: one scalar rounding for the block scale, the values in pairs by
    // the hardware conversions (identical to round_bf16 / round_fp16 for
    // every finite sum; a non-finite sum is an error either way).
    const uint32_t mr = absmax_bits16(v);
    const uint32_t m = f2u(apply_prec<PREC>(u2f(mr)));
    if (mr >= 0x7f800000u || m >= 0x7f800000u)  // rare: out of line, not if-converted
      acc_report_nonfinite<BF16L>(lbase + t * kLocTileB, lane, t, gblk, eb, err);
    if constexpr (PREC != AGQ_ACC_FP32) round_pairs16<PREC>(v);
    uint32_t ow[4];
    fp8_requant16(v, u2f(m), ow);
    *reinterpret_cast<uint4*>(out_codes + t * kAccWarpElems + lane * 16) =
        make_uint4(ow[0], ow[1], ow[2], ow[3]);
    if ((lane & 7) == 0) out_scales[gblk] = u2f(m);
    __syncwarp();  // btab is rewritten by the next tile
  }
}

// ---------------------------------------------------------------------------
// Generic accumulate / reduce (any block size): one warp per block, two
// passes (absmax, then encode from recomputed — identical — sums).
// ---------------------------------------------------------------------------
template <int PREC>
__global__ void k_accumulate_generic(const uint8_t* codes, const float* scales,
                                     const void* local, int bf16l, uint64_t n,
                                     uint32_t block, uint64_t nblocks, uint8_t* out_codes,
                                     float* out_scales, long long elem_base,
                                     agq_errors* err) {
  __shared__ double lut[kDqTable];
  fill_fp8_dq_table(lut);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  auto loc = [&](uint64_t i) -> float {
    return bf16l ? u2f((uint32_t)static_cast<const uint16_t*>(local)[i] << 16)
                 : static_cast<const float*>(local)[i];
  };
  for (uint64_t b = warp; b < nblocks; b += nwarps) {
    const uint64_t beg = b * block, end = min(n, beg + block);
    const float sc = scales[b];
    const long long gb = (elem_base + (long long)beg) / block;
    if (lane == 0 && (!(sc >= 0.0f) || !(sc <= 3.402823466e38f))) err_min(&err->bad_scale_block, gb);
    const double sd = (double)sc;
    uint32_t m = 0;
    for (uint64_t i = beg + lane; i < end; i += 32) {
      const float l = loc(i);
      if ((f2u(l) & 0x7f800000u) == 0x7f800000u) err_min(&err->nonfinite_local, elem_base + (long long)i);
      const float s = apply_prec<PREC>(fadd(fp8_dequant(codes[i], sd, lut, dq_fast(sc)), l));
      m = max(m, f2u(s) & 0x7fffffffu);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float a = u2f(m);
    if (lane == 0 && m >= 0x7f800000u) err_min(&err->nonfinite_block, gb);
    const bool ok = m < 0x7f800000u;
    const float inv = ok && m ? fdiv(448.0f, a) : 0.0f;
    for (uint64_t i = beg + lane; i < end; i += 32) {
      const float s = apply_prec<PREC>(fadd(fp8_dequant(codes[i], sd, lut, dq_fast(sc)), loc(i)));
      out_codes[i] = (uint8_t)(m == 0 || !ok ? 0u : encode_f32(2, 8, s, a, inv));
    }
    __syncwarp();
    if (lane == 0) out_scales[b] = a;
  }
}

__global__ void k_reduce_generic(PieceTable pt, uint64_t len, uint32_t block, uint64_t nblocks,
                                 long long blk_base, agq_errors* err) {
  __shared__ double lut[kDqTable];
  fill_fp8_dq_table(lut);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t b = warp; b < nblocks; b += nwarps) {
    const uint64_t beg = b * block, end = min(len, beg + block);
    uint32_t m = 0, sbad = 0;
    for (int p = 0; p < pt.np; ++p) sbad |= bad_scale_bit(pt.scales[p][b], p);
    if (lane == 0 && sbad) err_min(&err->bad_scale_block, bad_scale_key(sbad, blk_base + (long long)b));
    for (uint64_t i = beg + lane; i < end; i += 32) {
      float acc = 0.0f;
      for (int p = 0; p < pt.np; ++p)
        acc = fadd(acc, fp8_dequant(pt.codes[p][i], (double)pt.scales[p][b], lut, dq_fast(pt.scales[p][b])));
      m = max(m, f2u(acc) & 0x7fffffffu);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float a = u2f(m);
    if (lane == 0 && m >= 0x7f800000u) err_min(&err->overflow_block, blk_base + (long long)b);
    const bool ok = m < 0x7f800000u;
    const float inv = ok && m ? fdiv(448.0f, a) : 0.0f;
    for (uint64_t i = beg + lane; i < end; i += 32) {
      float acc = 0.0f;
      for (int p = 0; p < pt.np; ++p)
        acc = fadd(acc, fp8_dequant(pt.codes[p][i], (double)pt.scales[p][b], lut, dq_fast(pt.scales[p][b])));
      const uint8_t c = (uint8_t)(m == 0 || !ok ? 0u : encode_f32(2, 8, acc, a, inv));
      for (int o = 0; o < pt.nout; ++o) pt.out_codes[o][i] = c;
    }
    __syncwarp();
    if (lane == 0)
      for (int o = 0; o < pt.nout; ++o) pt.out_scales[o][b] = a;
  }
}

template <int NP>
__global__ void __launch_bounds__(256, 1)
    k_reduce128(PieceTable pt, uint64_t len, long long blk_base, int vec, agq_errors* err) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[NP > 0 ? 8 * NP * 32 : 1];  // 8 warps x NP pieces x 32 entries
  fill_fp8_dq_table(lut);
  __syncthreads();
  const uint64_t nblocks = (len + kBlock - 1) / kBlock;
  const uint64_t ngroups = nblocks * 8;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  float* wtab = NP > 0 ? btab + (threadIdx.x >> 5) * NP * 32 : nullptr;
  // warp-uniform trip count so the 8-lane shuffles always have all lanes
  const uint64_t gpad = (ngroups + 31) / 32 * 32;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < gpad; g += stride)
    reduce_group<NP>(pt, g, g < ngroups ? len : 0, blk_base, lut, err, vec != 0, wtab);
}

// K4 with a per-warp cp.async ring (LDGSTS): the NP pieces' code words
// (16 B per lane per piece) and block scales of warp-group i+S-1 are in
// flight while warp-group i (512 elements = 4 blocks) is decoded, so a warp
// keeps HBM requests outstanding through its arithmetic. Whole 512-element
// warp-groups only (16-byte aligned pointers); the ragged tail goes through
// reduce_group. Pieces are decoded one at a time straight from the ring slot
// with the f16-route block tables (dq_f16_accum: no per-code safety test, a
// register footprint independent of NP), summed from +0.0f in ascending
// piece order, so bit-identical to reduce_group.
// W warps per CTA: small CTAs pack more warps per SM under the shared-memory
// limit of the ring (P = 8: 4-warp CTAs, 5 per SM = 20 warps, vs 2 x 8).
template <int NP>
struct RedCfg {
  static constexpr int kWarps = NP <= 4 ? 8 : 4;
  static constexpr int kMinBlocks = NP <= 4 ? 3 : 5;
};
template <int NP, int S>
__global__ void __launch_bounds__(RedCfg<NP>::kWarps * 32, RedCfg<NP>::kMinBlocks)
    k_reduce128_pipe(PieceTable pt, uint64_t len, long long blk_base, agq_errors* err) {
  constexpr int W = RedCfg<NP>::kWarps;
  extern __shared__ __align__(16) unsigned char ring_smem[];
  __shared__ double lut[kDqTable];
  __shared__ __align__(32) float btab[W * NP * 32];
  fill_fp8_dq_table(lut);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr uint32_t kSlot = NP * 512 + NP * 16;  // codes, then 4 scales per piece
  unsigned char* ring = ring_smem + (size_t)warp * S * kSlot;
  float* wtab = btab + warp * NP * 32;
  const uint32_t mytab = (uint32_t)__cvta_generic_to_shared(wtab + (lane >> 3) * 8);
  const double t8 = fp8_t8(lane & 7);  // lane 8b + j builds entry j of block b
  const uint64_t nwg = len / 512;      // whole warp-groups; the tail is another launch
  const uint64_t wstride = gridDim.x * (uint64_t)W;
  auto issue = [&](uint64_t gi, int k) {
    if (gi < nwg) {
      unsigned char* sl = ring + k * kSlot;
#pragma unroll
      for (int p = 0; p < NP; ++p) cp_async16(sl + p * 512 + lane * 16, pt.codes[p] + gi * 512 + lane * 16);
      // block scales one float per lane: a chunk's scale pointer (e.g. the
      // owner's slice of its own gradient) need not be 16-byte aligned
      if (lane < 4 * NP) cp_async4(sl + NP * 512 + lane * 4, pt.scales[lane >> 2] + gi * 4 + (lane & 3));
    }
    cp_async_commit();
  };
  uint64_t wg = blockIdx.x * (uint64_t)W + warp;
#pragma unroll
  for (int k = 0; k < S - 1; ++k) issue(wg + k * wstride, k);
  int slot = 0;
  for (; wg < nwg; wg += wstride) {
    __syncwarp();  // every lane is done reading the slot refilled next (and the tables)
    issue(wg + (S - 1) * wstride, slot == 0 ? S - 1 : slot - 1);
    cp_async_wait<S - 1>();
    __syncwarp();
    const unsigned char* sl = ring + slot * kSlot;
    const float* scs = reinterpret_cast<const float*>(sl + NP * 512) + (lane >> 3);
    bool fast = true;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float sc = scs[p * 4];
      wtab[p * 32 + lane] = fp8_tab_entry_f16(t8, sc);
      fast = fast && dq_fast(sc);
    }
    __syncwarp();
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
    uint32_t sbad = 0;
    if (__all_sync(0xffffffffu, fast)) {  // every piece of the warp-group: table decode
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const uint4 cv = lds128(sl + p * 512 + lane * 16);
        const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
        dq_f16_accum<4>(w, mytab + p * 128, acc);
      }
    } else {  // a zero / extreme / bad block scale somewhere: per piece
#pragma unroll 1
      for (int p = 0; p < NP; ++p) {
        const uint4 cv = lds128(sl + p * 512 + lane * 16);
        const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
        const float sc = scs[p * 4];
        sbad |= bad_scale_bit(sc, p);
        if (dq_fast(sc))
          dq_f16_accum<4>(w, mytab + p * 128, acc);
        else
          dq_accum<16>(w, sc, lut, acc);
      }
    }
    reduce_finish(pt, wg * 512 + lane * 16, len, true, true, (wg * 512 + lane * 16) / kBlock, sbad,
                  acc, blk_base, err);
    slot = slot == S - 1 ? 0 : slot + 1;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// allreduce_naive_fp8 strawman (collective.hpp:338-431), simulated on one
// device: P-1 ring steps adding in FP8 at the receiver's ORIGINAL scales.
// One thread per element runs the ring for that element (elements are
// independent; each step reads the snapshot of the previous step).
// ---------------------------------------------------------------------------
__global__ void k_naive_ring(PieceTable pt, uint64_t n, uint32_t block, const uint64_t* ranges,
                             uint8_t* out_codes, float* out_scales, agq_errors* err,
                             unsigned long long* events) {
  __shared__ double lut[128];
  fill_fp8_unit_lut(lut);
  __syncthreads();
  const int P = pt.np;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * (uint64_t)blockDim.x) {
    const uint64_t blk = i / block;
    int chunk = 0;
    for (int c = 0; c < P; ++c)
      if (i >= ranges[2 * c] && i < ranges[2 * c + 1]) chunk = c;
    // working state of every rank for this element
    uint8_t wc[AGQ_MAX_WORLD];
    float ws[AGQ_MAX_WORLD];
    for (int r = 0; r < P; ++r) {
      wc[r] = pt.codes[r][i];
      ws[r] = pt.scales[r][blk];
    }
    bool sat = false;
    for (int step = 0; step < P - 1; ++step) {
      // rank r updates chunk (r - step - 1) mod P with the message of r-1
      uint8_t nc[AGQ_MAX_WORLD];
      for (int r = 0; r < P; ++r) nc[r] = wc[r];
      for (int r = 0; r < P; ++r) {
        const int ch = ((r - step - 1) % P + P) % P;
        if (ch != chunk) continue;
        const int from = (r - 1 + P) % P;
        const double unit_in = lut[wc[from] & 0x7f] * (wc[from] & 0x80 ? -1.0 : 1.0);
        const double inc = unit_in * (double)ws[from];
        const double loc = lut[wc[r] & 0x7f] * (wc[r] & 0x80 ? -1.0 : 1.0) * (double)ws[r];
        const double sum = inc + loc;
        const float scale = pt.scales[r][blk];
        const double unit = scale == 0.0f ? 0.0 : sum / (double)scale;
        bool over = (scale == 0.0f && sum != 0.0);
        const double w = unit * 448.0;
        if (fabs(w) > 448.0) over = true;
        nc[r] = (uint8_t)fp8_encode_double(w);
        if (over) {
          sat = true;
          if (events) atomicAdd(&events[r], 1ull);
        }
      }
      for (int r = 0; r < P; ++r) wc[r] = nc[r];
    }
    const int owner = P == 1 ? 0 : (chunk - 1 + P) % P;
    out_codes[i] = wc[owner];
    if (i % block == 0 || i == ranges[2 * chunk]) out_scales[blk] = pt.scales[owner][blk];
    if (sat) atomicAdd(&err->saturated, 1ull);
  }
}

// One ring step of allreduce_naive_fp8 on a REAL rank (collective.hpp:373-400):
// add the chunk message of rank r-1 into this rank's working codes, re-encode
// at this rank's ORIGINAL scales (scales never change in the naive protocol,
// so they are read-only here). The sticky per-element saturation flag
// (collective.hpp:390-398) travels with the chunk as a bitmask, bit j =
// element begin+j: in_sat (NULL on step 0) | this step's overflows -> out_sat.
// On the final step the owner adds the popcount to err->saturated instead.
// One warp per 32 elements (one mask word).
__global__ void k_naive_step(const uint8_t* in_codes, const float* in_scales,
                             const uint32_t* in_sat, uint8_t* codes, const float* scales,
                             uint32_t* out_sat, uint64_t len, uint32_t block,
                             unsigned long long* saturated, unsigned long long* events) {
  __shared__ double lut[128];
  fill_fp8_unit_lut(lut);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nwords = (len + 31) / 32;
  const uint64_t nwarps = gridDim.x * (uint64_t)(blockDim.x >> 5);
  unsigned long long my_events = 0, my_sat = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < nwords;
       w += nwarps) {
    const uint64_t j = w * 32 + lane;
    bool over = false;
    if (j < len) {
      const uint64_t b = j / block;
      const uint8_t ci = in_codes[j], cl = codes[j];
      const double inc = lut[ci & 0x7f] * (ci & 0x80 ? -1.0 : 1.0) * (double)in_scales[b];
      const double loc = lut[cl & 0x7f] * (cl & 0x80 ? -1.0 : 1.0) * (double)scales[b];
      const double sum = inc + loc;
      const float scale = scales[b];
      const double unit = scale == 0.0f ? 0.0 : sum / (double)scale;
      over = (scale == 0.0f && sum != 0.0);
      const double v = unit * 448.0;
      if (fabs(v) > 448.0) over = true;
      codes[j] = (uint8_t)fp8_encode_double(v);
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, over);
    if (lane == 0) {
      my_events += __popc(mask);
      const uint32_t sticky = mask | (in_sat ? in_sat[w] : 0u);
      if (out_sat) out_sat[w] = sticky;
      else my_sat += __popc(sticky);
    }
  }
  if (lane == 0) {
    if (events && my_events) atomicAdd(events, my_events);
    if (saturated && my_sat) atomicAdd(saturated, my_sat);
  }
}

}  // namespace agqk

// ===========================================================================
// Host launchers
// ===========================================================================
namespace agqh {
using namespace agqk;

namespace {
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// K3 reads a lane's local-gradient row with 256-bit loads
bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
int gen_grid(uint64_t work, int threads) {
  const uint64_t g = (work + threads - 1) / threads;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// K4: the cp.async ring kernel (2 stages; 3 tie, 4 lose at P = 8,
// profiles/r01_reduce_pipe_ab.log) for 16-byte aligned pieces of >= 512
// elements, else the direct-load kernel.
constexpr int kRedStages = 2;

template <int NP, int S>
bool launch_reduce_pipe(const PieceTable& pt, uint64_t len, long long bb, agq_errors* err,
                        cudaStream_t s) {
  auto k = k_reduce128_pipe<NP, S>;
  constexpr int W = RedCfg<NP>::kWarps;
  const size_t smem = (size_t)W * S * (NP * 512 + NP * 16);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, W * 32, smem);
  if (occ < 1) return false;
  const uint64_t want = (len / 512 + W - 1) / W;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  const int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  k<<<grid, W * 32, smem, s>>>(pt, len, bb, err);
  return true;
}

template <int NP>
void launch_reduce128(const PieceTable& pt, uint64_t len, long long bb, int vec, agq_errors* err,
                      cudaStream_t s) {
  if constexpr (NP > 0) {
    if (vec && len >= 512 && launch_reduce_pipe<NP, kRedStages>(pt, len, bb, err, s)) {
      const uint64_t done = len / 512 * 512;
      if (done == len) return;
      // ragged tail (< 512 elements): the direct-load kernel on the rest
      PieceTable tp = pt;
      for (int p = 0; p < pt.np; ++p) {
        tp.codes[p] += done;
        tp.scales[p] += done / kBlock;
      }
      for (int o = 0; o < pt.nout; ++o) {
        tp.out_codes[o] += done;
        tp.out_scales[o] += done / kBlock;
      }
      k_reduce128<NP><<<1, 256, 0, s>>>(tp, len - done, bb + (long long)(done / kBlock), 1, err);
      count_launch();
      return;
    }
  }
  const uint64_t groups = (len + kBlock - 1) / kBlock * 8;
  int grid = gen_grid(groups, 256);
  k_reduce128<NP><<<grid, 256, 0, s>>>(pt, len, bb, vec, err);
}
}  // namespace

namespace {
template <bool BF16L, int PREC>
agq_status launch_acc_warp(const uint8_t* codes, const float* scales, const void* local,
                           uint64_t ntiles, uint8_t* oc, float* os, long long eb,
                           agq_errors* err, cudaStream_t s) {
  auto k = k_accumulate_warp<BF16L, PREC>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kAccWarps * 32, 0);
  if (occ < 1) occ = 1;
  const uint64_t want = (ntiles + kAccWarps - 1) / kAccWarps;
  const uint64_t cap = (uint64_t)num_sms() * occ;
  k<<<(int)(want < cap ? want : cap), kAccWarps * 32, 0, s>>>(codes, scales, local, ntiles, oc,
                                                              os, eb, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "accumulate: launch");
}

template <bool BF16L>
agq_status acc_warp_prec(int prec, const uint8_t* codes, const float* scales, const void* local,
                         uint64_t ntiles, uint8_t* oc, float* os, long long eb, agq_errors* err,
                         cudaStream_t s) {
  if (prec == AGQ_ACC_BF16) return launch_acc_warp<BF16L, AGQ_ACC_BF16>(codes, scales, local, ntiles, oc, os, eb, err, s);
  if (prec == AGQ_ACC_FP16) return launch_acc_warp<BF16L, AGQ_ACC_FP16>(codes, scales, local, ntiles, oc, os, eb, err, s);
  return launch_acc_warp<BF16L, AGQ_ACC_FP32>(codes, scales, local, ntiles, oc, os, eb, err, s);
}
}  // namespace

// blk_base: block index of element 0 in the error record (the offset of a
// chunk inside the caller's tensor; 0 for a whole-tensor call).
agq_status accumulate_device(const uint8_t* codes, const float* scales, const void* local,
                             int local_dtype, uint64_t n, uint32_t block, int prec,
                             uint8_t* oc, float* os, agq_errors* err, cudaStream_t s,
                             long long blk_base) {
  if (n == 0) return AGQ_OK;
  const bool bf16l = local_dtype == AGQ_BF16;
  const uint64_t unit = kAccWarpElems;
  uint64_t ntiles = 0;
  if (block == (uint32_t)kBlock && aligned16(codes) && aligned16(scales) && aligned32(local) &&
      aligned16(oc) && aligned16(os))
    ntiles = n / unit;
  if (ntiles) {
    const agq_status r =
        bf16l ? acc_warp_prec<true>(prec, codes, scales, local, ntiles, oc, os, blk_base, err, s)
              : acc_warp_prec<false>(prec, codes, scales, local, ntiles, oc, os, blk_base, err, s);
    if (r != AGQ_OK) return r;
  }
  const uint64_t done = ntiles * unit;
  if (done == n) return AGQ_OK;
  const uint64_t rest = n - done, nb = (rest + block - 1) / block;
  const void* ltail = static_cast<const char*>(local) + done * (bf16l ? 2 : 4);
  const int grid = gen_grid(nb * 32, 256);
  const long long base = blk_base * (long long)block + (long long)done;
  if (prec == AGQ_ACC_BF16)
    k_accumulate_generic<AGQ_ACC_BF16><<<grid, 256, 0, s>>>(codes + done, scales + done / block, ltail,
        bf16l, rest, block, nb, oc + done, os + done / block, base, err);
  else if (prec == AGQ_ACC_FP16)
    k_accumulate_generic<AGQ_ACC_FP16><<<grid, 256, 0, s>>>(codes + done, scales + done / block, ltail,
        bf16l, rest, block, nb, oc + done, os + done / block, base, err);
  else
    k_accumulate_generic<AGQ_ACC_FP32><<<grid, 256, 0, s>>>(codes + done, scales + done / block, ltail,
        bf16l, rest, block, nb, oc + done, os + done / block, base, err);
  count_launch();
  return cuda_fail(cudaGetLastError(), "accumulate (generic): launch");
}

agq_status reduce_requant_device(int np, const uint8_t* const* pc, const float* const* ps,
                                 uint64_t len, uint32_t block, int nout, uint8_t* const* oc,
                                 float* const* os, long long blk_base, agq_errors* err,
                                 cudaStream_t s) {
  if (len == 0) return AGQ_OK;
  PieceTable pt{};
  pt.np = np;
  pt.nout = nout;
  bool vec = true;
  for (int p = 0; p < np; ++p) {
    pt.codes[p] = pc[p];
    pt.scales[p] = ps[p];
    vec = vec && aligned16(pc[p]);
  }
  for (int o = 0; o < nout; ++o) {
    pt.out_codes[o] = oc[o];
    pt.out_scales[o] = os[o];
    vec = vec && aligned16(oc[o]);
  }
  if (block == (uint32_t)kBlock) {
    switch (np) {
      case 1: launch_reduce128<1>(pt, len, blk_base, vec, err, s); break;
      case 2: launch_reduce128<2>(pt, len, blk_base, vec, err, s); break;
      case 3: launch_reduce128<3>(pt, len, blk_base, vec, err, s); break;
      case 4: launch_reduce128<4>(pt, len, blk_base, vec, err, s); break;
      case 5: launch_reduce128<5>(pt, len, blk_base, vec, err, s); break;
      case 6: launch_reduce128<6>(pt, len, blk_base, vec, err, s); break;
      case 7: launch_reduce128<7>(pt, len, blk_base, vec, err, s); break;
      case 8: launch_reduce128<8>(pt, len, blk_base, vec, err, s); break;
      default: launch_reduce128<0>(pt, len, blk_base, vec, err, s); break;
    }
  } else {
    const uint64_t nb = (len + block - 1) / block;
    k_reduce_generic<<<gen_grid(nb * 32, 256), 256, 0, s>>>(pt, len, block, nb, blk_base, err);
  }
  count_launch();
  return cuda_fail(cudaGetLastError(), "reduce-requant: launch");
}

agq_status naive_ring_device(int world, const uint8_t* const* codes, const float* const* scales,
                             uint64_t n, uint32_t block, const uint64_t* d_ranges,
                             uint8_t* oc, float* os, agq_errors* err, unsigned long long* events,
                             cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  PieceTable pt{};
  pt.np = world;
  for (int r = 0; r < world; ++r) {
    pt.codes[r] = codes[r];
    pt.scales[r] = scales[r];
  }
  k_naive_ring<<<gen_grid(n, 256), 256, 0, s>>>(pt, n, block, d_ranges, oc, os, err, events);
  count_launch();
  return cuda_fail(cudaGetLastError(), "naive ring: launch");
}

agq_status naive_step_device(const uint8_t* in_codes, const float* in_scales,
                             const uint32_t* in_sat, uint8_t* codes, const float* scales,
                             uint32_t* out_sat, uint64_t len, uint32_t block,
                             unsigned long long* saturated, unsigned long long* events,
                             cudaStream_t s) {
  if (len == 0) return AGQ_OK;
  k_naive_step<<<gen_grid((len + 31) / 32 * 32, 256), 256, 0, s>>>(
      in_codes, in_scales, in_sat, codes, scales, out_sat, len, block, saturated, events);
  count_launch();
  return cuda_fail(cudaGetLastError(), "naive ring step: launch");
}

}  // namespace agqh
