// Multi-GPU decomposed 8-bit all-reduce (collective.hpp:226-333 for real
// ranks, one process per GPU).
//
// AGQ_AR_NCCL (v1): chunk r of every rank goes to rank r with grouped
//   ncclSend/ncclRecv (the all-to-all), rank r runs the K4 reduce-requant
//   kernel over its chunk (pieces in ascending sender rank, in place), then a
//   second grouped send/recv broadcasts every reduced chunk straight into
//   place on all ranks (the all-gather).
// AGQ_AR_FUSED_P2P (v2): every rank's FP8 gradient lives in a symmetric,
//   IPC-mapped buffer. ONE kernel per rank pulls chunk r from all peers over
//   NVLink (peer loads), reduces in FP32 in ascending rank order, requantizes,
//   and pushes the result into chunk r of every peer's buffer (peer stores):
//   the transfer overlaps the reduction tile by tile. Chunk r of peer s is
//   read and written only by rank r, so the only cross-GPU synchronisation is
//   a start barrier (inputs final) and an end barrier (all chunks written),
//   both as system-scope release/acquire flags with a timeout.
//
// Chunk ownership follows ChunkAssignment::block_aligned (collective.hpp:
// 23-39); results do not depend on it (per-block reduce, sender-rank order).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "agq_grad.cuh"

namespace agqh {
agq_status reduce_requant_device(int np, const uint8_t* const* pc, const float* const* ps,
                                 uint64_t len, uint32_t block, int nout, uint8_t* const* oc,
                                 float* const* os, long long blk_base, agq_errors* err,
                                 cudaStream_t s);
void chunk_ranges(uint64_t n, uint32_t block, int workers, uint64_t* ranges);
agq_status naive_step_device(const uint8_t* in_codes, const float* in_scales,
                             const uint32_t* in_sat, uint8_t* codes, const float* scales,
                             uint32_t* out_sat, uint64_t len, uint32_t block,
                             unsigned long long* saturated, unsigned long long* events,
                             cudaStream_t s);
}  // namespace agqh

// NCCL is resolved at run time: reuse the libnccl.so.2 already loaded in the
// process (e.g. torch's) so two NCCL builds never mix, else load the system
// one. The library itself therefore loads without NCCL present.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId;
  decltype(&ncclCommInitRank) CommInitRank;
  decltype(&ncclCommDestroy) CommDestroy;
  decltype(&ncclGroupStart) GroupStart;
  decltype(&ncclGroupEnd) GroupEnd;
  decltype(&ncclSend) Send;
  decltype(&ncclRecv) Recv;
  decltype(&ncclAllReduce) AllReduce;
  decltype(&ncclGetErrorString) GetErrorString;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
#define AGQ_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    AGQ_NCCL_SYM(GetUniqueId);
    AGQ_NCCL_SYM(CommInitRank);
    AGQ_NCCL_SYM(CommDestroy);
    AGQ_NCCL_SYM(GroupStart);
    AGQ_NCCL_SYM(GroupEnd);
    AGQ_NCCL_SYM(Send);
    AGQ_NCCL_SYM(Recv);
    AGQ_NCCL_SYM(AllReduce);
    AGQ_NCCL_SYM(GetErrorString);
#undef AGQ_NCCL_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart &&
             api.GroupEnd && api.Send && api.Recv && api.AllReduce && api.GetErrorString;
  });
  return api;
}
}  // namespace

// Symmetric buffer layout (identical offsets on every rank).
namespace {
constexpr size_t kFlagsBytes = 4096;  // ready[16] | done[16] | err words
constexpr int kReadyOff = 0, kDoneOff = 16, kScatterOff = 32;
size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

struct agq_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 0, rank = 0, device = 0;
  // v1 workspace
  uint8_t* recv_codes = nullptr;
  float* recv_scales = nullptr;
  uint64_t recv_chunk_cap = 0;  // elements per peer slot
  // naive-ring workspace: one incoming chunk + two saturation bitmasks
  uint8_t* ring_codes = nullptr;
  float* ring_scales = nullptr;
  uint32_t* ring_sat = nullptr;
  uint64_t ring_cap = 0;  // elements
  // v2 symmetric memory
  unsigned char* sym = nullptr;
  size_t sym_bytes = 0;
  uint64_t sym_cap = 0;  // elements
  unsigned char* peer[AGQ_MAX_WORLD] = {};
  bool p2p_ready = false;
  unsigned int* done_counter = nullptr;  // local, per kernel
  uint64_t epoch = 0;
};

namespace agqk {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct FusedArgs {
  unsigned char* base[AGQ_MAX_WORLD];  // symmetric buffer of every rank (self included)
  uint64_t scales_off, codes_off;      // byte offsets inside the buffer
  uint64_t begin, len;                 // my chunk (elements, block aligned)
  uint64_t epoch;
  unsigned int* done_counter;
  agq_errors* err;
  int rank, P;
  int copy_only;
};

// Spin until flag >= epoch; returns false on timeout (20 s).
__device__ bool wait_flag(const uint64_t* f, uint64_t epoch) {
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(f) < epoch) {
    if (globaltimer() - t0 > 20000000000ull) return false;
    __nanosleep(200);
  }
  return true;
}

// AGQ_P2P_COPYONLY=1 (measurement only): identical NVLink traffic, no
// dequant/reduce/requant — bounds the transfer-only time of the kernel.
// One 16-element group of the fused all-reduce with every pointer in
// registers (compile-time NP): chunk r of every rank is read over NVLink
// (rank order = ascending sender rank), reduced from +0.0f in FP32, requantized
// and written back in place to all ranks.
template <int NP>
__device__ __forceinline__ void fused_group(unsigned char* const (&base)[NP], uint64_t coff,
                                            uint64_t soff, uint64_t g, uint64_t len,
                                            long long blk_base, const double* t16,
                                            agq_errors* err, float* wtab) {
  const uint64_t e0 = g * 16;
  const uint64_t blk = e0 / kBlock;
  // chunk-relative addresses from one common offset per array
  auto cbase = [&](int p) { return base[p] + coff; };
  auto sbase = [&](int p) { return reinterpret_cast<float*>(base[p] + soff); };
  const bool in_range = e0 < len;
  const bool whole = e0 + 16 <= len;
  float acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
  uint32_t sbad = 0;
  {
    uint4 cv[NP];
    float sc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      cv[p] = make_uint4(0, 0, 0, 0);
      sc[p] = blk * kBlock < len ? sbase(p)[blk] : 0.0f;  // whole block's lanes (tables)
      if (!in_range) continue;
      if (whole) {
        cv[p] = *reinterpret_cast<const uint4*>(cbase(p) + e0);
      } else {
        uint32_t w[4] = {0, 0, 0, 0};
        for (int e = 0; e < 16 && e0 + e < len; ++e)
          w[e >> 2] |= (uint32_t)cbase(p)[e0 + e] << (8 * (e & 3));
        cv[p] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    if (AGQ_RED_TAB) build_tables<NP, 8>(wtab, sc);  // every lane of the warp
    if (in_range) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        sbad |= !(sc[p] >= 0.0f) || !(sc[p] <= 3.402823466e38f);
        const uint32_t w[4] = {cv[p].x, cv[p].y, cv[p].z, cv[p].w};
        if (AGQ_RED_TAB && dq_fast(sc[p]) && fp8_tab_ok16(w))
          dq_tab_accum<4>(w, tab_addr<8>(wtab, p), acc);
        else
          dq_accum<16>(w, sc[p], t16, acc);
      }
      if (!whole)
        for (int e = 0; e < 16; ++e)
          if (e0 + e >= len) acc[e] = 0.0f;
    }
  }
  const uint32_t m = absmax_bits16(acc);
  const int sub = threadIdx.x & 7;
  if (in_range && sub == 0) {
    if (sbad) err_min(&err->bad_scale_block, blk_base + (long long)blk);
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
#pragma unroll
  for (int o = 0; o < NP; ++o) {
    if (whole) {
      *reinterpret_cast<uint4*>(cbase(o) + e0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    } else {
      for (int e = 0; e < 16 && e0 + e < len; ++e) cbase(o)[e0 + e] = (uint8_t)(ow[e >> 2] >> (8 * (e & 3)));
    }
    if (sub == 0) sbase(o)[blk] = a;
  }
}

// 8 elements per thread (16 lanes per block) for large worlds: half the
// per-piece registers so NP = 5..8 keeps two CTAs per SM without spills.
template <int NP>
__device__ __forceinline__ void fused_group8(unsigned char* const (&base)[NP], uint64_t coff,
                                             uint64_t soff, uint64_t g, uint64_t len,
                                             long long blk_base, const double* t16,
                                             agq_errors* err, float* wtab) {
  const uint64_t e0 = g * 8;
  const uint64_t blk = e0 / kBlock;
  const bool in_range = e0 < len;
  const bool whole = e0 + 8 <= len;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  uint32_t sbad = 0;
  {
    uint2 cv[NP];
    float sc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      cv[p] = make_uint2(0, 0);
      sc[p] = blk * kBlock < len ? reinterpret_cast<const float*>(base[p] + soff)[blk] : 0.0f;
      if (!in_range) continue;
      if (whole) {
        cv[p] = *reinterpret_cast<const uint2*>(base[p] + coff + e0);
      } else {
        uint32_t w[2] = {0, 0};
        for (int e = 0; e < 8 && e0 + e < len; ++e)
          w[e >> 2] |= (uint32_t)base[p][coff + e0 + e] << (8 * (e & 3));
        cv[p] = make_uint2(w[0], w[1]);
      }
    }
    if (AGQ_RED_TAB) build_tables<NP, 16>(wtab, sc);  // every lane of the warp
    if (in_range) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        sbad |= !(sc[p] >= 0.0f) || !(sc[p] <= 3.402823466e38f);
        const uint32_t w[2] = {cv[p].x, cv[p].y};
        if (AGQ_RED_TAB && dq_fast(sc[p]) && fp8_tab_ok8(w))
          dq_tab_accum<2>(w, tab_addr<16>(wtab, p), acc);
        else
          dq_accum<8>(w, sc[p], t16, acc);
      }
      if (!whole)
        for (int e = 0; e < 8; ++e)
          if (e0 + e >= len) acc[e] = 0.0f;
    }
  }
  const uint32_t m = absmax_bits8(acc);
  const int sub = threadIdx.x & 15;
  if (in_range && sub == 0) {
    if (sbad) err_min(&err->bad_scale_block, blk_base + (long long)blk);
    if (m >= 0x7f800000u) err_min(&err->overflow_block, blk_base + (long long)blk);
  }
  if (!in_range) return;
  const float a = u2f(m);
  uint32_t ow[2];
  if (m >= 0x7f800000u) {
    ow[0] = ow[1] = 0;
  } else {
    fp8_requant8(acc, a, ow);
  }
#pragma unroll
  for (int o = 0; o < NP; ++o) {
    if (whole) {
      *reinterpret_cast<uint2*>(base[o] + coff + e0) = make_uint2(ow[0], ow[1]);
    } else {
      for (int e = 0; e < 8 && e0 + e < len; ++e)
        base[o][coff + e0 + e] = (uint8_t)(ow[e >> 2] >> (8 * (e & 3)));
    }
    if (sub == 0) reinterpret_cast<float*>(base[o] + soff)[blk] = a;
  }
}

// End of an all-reduce epoch (every CTA calls it): the last CTA of this
// rank's grid to finish publishes "done" to every rank and waits for all of
// them, so the kernel completes only when every rank has finished writing
// into this rank's buffer (and reading from it). A local-reduce overflow is
// shared with every rank first (collective.hpp:278-281 aborts all ranks).
template <class Args>
__device__ __forceinline__ void epoch_end(const Args& a) {
  unsigned char* const* base = a.base;
  const int P = a.P, rank = a.rank;
  const uint64_t epoch = a.epoch;
  unsigned int* done_counter = a.done_counter;
  agq_errors* err = a.err;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned int prev = atomicAdd(done_counter, 1u);
  if (prev != gridDim.x * gridDim.y - 1) return;
  __threadfence_system();
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(base[rank]);
  const long long ov = *reinterpret_cast<volatile long long*>(&err->overflow_block);
  for (int s = 0; s < P; ++s) {
    uint64_t* peer_flags = reinterpret_cast<uint64_t*>(base[s]);
    if (ov != kNone) atomicMin(reinterpret_cast<long long*>(peer_flags + 64 + rank), ov);
  }
  __threadfence_system();
  for (int s = 0; s < P; ++s)
    st_release_sys(reinterpret_cast<uint64_t*>(base[s]) + kDoneOff + rank, epoch);
  bool fine = true;
  for (int s = 0; s < P; ++s)
    if (!wait_flag(my_flags + kDoneOff + s, epoch)) fine = false;
  for (int s = 0; s < P; ++s) {
    const long long o = *reinterpret_cast<volatile long long*>(my_flags + 64 + s);
    if (o != kNone) err_min(&err->overflow_block, o);
    // reset for the next epoch
    *reinterpret_cast<volatile long long*>(my_flags + 64 + s) = kNone;
  }
  if (!fine) err_min(&err->overflow_block, -1);
  *done_counter = 0u;
}

#ifndef AGQ_P2P_MINB
#define AGQ_P2P_MINB 2
#endif
template <int NP, int EPT>
__global__ void __launch_bounds__(256, AGQ_P2P_MINB) k_fused_allreduce(FusedArgs a) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * (NP > 0 ? NP : 1) * 32];  // 8 warps x NP pieces x 32 entries
  __shared__ int ok;
  fill_fp8_dq_table(lut);
  float* wtab = btab + (threadIdx.x >> 5) * (NP > 0 ? NP : 1) * 32;
  const int tid = threadIdx.x;
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(a.base[a.rank]);
  // start barrier: announce "my input is final" to every rank, then wait for
  // every rank's announcement (each CTA waits; only CTA 0 announces).
  if (blockIdx.x == 0 && tid < a.P)
    st_release_sys(reinterpret_cast<uint64_t*>(a.base[tid]) + kReadyOff + a.rank, a.epoch);
  if (tid == 0) {
    ok = 1;
    for (int s = 0; s < a.P; ++s)
      if (!wait_flag(my_flags + kReadyOff + s, a.epoch)) ok = 0;
  }
  __syncthreads();
  if (!ok) {
    if (tid == 0) err_min(&a.err->overflow_block, -1);
    return;
  }

  const uint64_t b0 = a.begin / kBlock;
  const uint64_t nblocks = (a.len + kBlock - 1) / kBlock;
  const uint64_t ngroups = nblocks * 8;
  const uint64_t gpad = (ngroups + 31) / 32 * 32;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  if constexpr (NP > 0) {
    unsigned char* bs[NP];
#pragma unroll
    for (int s = 0; s < NP; ++s) bs[s] = a.base[s];
    const uint64_t coff = a.codes_off + a.begin, soff = a.scales_off + 4 * b0;
    if (a.copy_only) {
      for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < ngroups; g += stride) {
        const uint64_t e0 = g * 16;
        if (e0 + 16 > a.len) continue;
        uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const uint4 v = *reinterpret_cast<const uint4*>(bs[p] + coff + e0);
          x.x ^= v.x; x.y ^= v.y; x.z ^= v.z; x.w ^= v.w;
        }
#pragma unroll
        for (int o = 0; o < NP; ++o) *reinterpret_cast<uint4*>(bs[o] + coff + e0) = x;
      }
    } else {
      if constexpr (EPT == 8) {
        const uint64_t ng8 = nblocks * 16, gp8 = (ng8 + 31) / 32 * 32;
        for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gp8; g += stride)
          fused_group8<NP>(bs, coff, soff, g, g < ng8 ? a.len : 0, (long long)b0, lut, a.err, wtab);
      } else {
        for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride)
          fused_group<NP>(bs, coff, soff, g, g < ngroups ? a.len : 0, (long long)b0, lut, a.err, wtab);
      }
    }
  } else {
    PieceTable pt;
    pt.np = a.P;
    pt.nout = a.P;
    for (int s = 0; s < a.P; ++s) {
      pt.codes[s] = a.base[s] + a.codes_off + a.begin;
      pt.scales[s] = reinterpret_cast<const float*>(a.base[s] + a.scales_off) + b0;
      pt.out_codes[s] = a.base[s] + a.codes_off + a.begin;
      pt.out_scales[s] = reinterpret_cast<float*>(a.base[s] + a.scales_off) + b0;
    }
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride)
      reduce_group<0>(pt, g, g < ngroups ? a.len : 0, (long long)b0, lut, a.err, true);
  }

  epoch_end(a);
}

// ---------------------------------------------------------------------------
// Fused all-reduce, TMA-pipelined variant (AGQ_P2P_TMA=1): the same pull /
// reduce / push as k_fused_allreduce, but each warp keeps kStages warp tiles
// (512 elements = 4 blocks) of every piece in flight with 1-D bulk copies
// from the peers' buffers (lane 0 issues NP x (512 B codes + a 32 B aligned
// window holding the tile's 4 scales) per stage, one mbarrier per stage), so
// the NVLink pull latency overlaps the decode/reduce/requant of earlier
// tiles instead of sitting in front of every group. The partial last tile
// uses the per-thread path.
// ---------------------------------------------------------------------------
template <int NP>
struct TmaCfg {
  static constexpr int kStages = NP <= 4 ? 4 : 3;
  static constexpr uint32_t kPiece = 512 + 32;
  static constexpr uint32_t kStage = NP * kPiece;
  static constexpr uint32_t kWarpBytes = kStages * kStage;
  static constexpr size_t kSmem = 8 * (size_t)kWarpBytes;
};

// Decode + reduce (ascending piece order from +0.0f), requantize and store to
// every rank one whole 16-element group whose codes/scales are in registers.
template <int NP>
__device__ __forceinline__ void reduce_store16(unsigned char* const (&bs)[NP], uint64_t coff,
                                               uint64_t soff, uint64_t e0,
                                               const uint32_t (&cw)[NP][4], const float (&sc)[NP],
                                               long long blk_base, const double* t16,
                                               agq_errors* err, float* wtab) {
  const uint64_t blk = e0 / kBlock;
  float acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
  uint32_t sbad = 0;
  if (AGQ_RED_TAB) build_tables<NP, 8>(wtab, sc);
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    sbad |= !(sc[p] >= 0.0f) || !(sc[p] <= 3.402823466e38f);
    if (AGQ_RED_TAB && dq_fast(sc[p]) && fp8_tab_ok16(cw[p]))
      dq_tab_accum<4>(cw[p], tab_addr<8>(wtab, p), acc);
    else
      dq_accum<16>(cw[p], sc[p], t16, acc);
  }
  const uint32_t m = absmax_bits16(acc);
  const int sub = threadIdx.x & 7;
  if (sub == 0) {
    if (sbad) err_min(&err->bad_scale_block, blk_base + (long long)blk);
    if (m >= 0x7f800000u) err_min(&err->overflow_block, blk_base + (long long)blk);
  }
  const float a = u2f(m);
  uint32_t ow[4];
  if (m >= 0x7f800000u) {
    ow[0] = ow[1] = ow[2] = ow[3] = 0;
  } else {
    fp8_requant16(acc, a, ow);
  }
#pragma unroll
  for (int o = 0; o < NP; ++o) {
    *reinterpret_cast<uint4*>(bs[o] + coff + e0) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    if (sub == 0) reinterpret_cast<float*>(bs[o] + soff)[blk] = a;
  }
}

template <int NP>
__global__ void __launch_bounds__(256, 1) k_fused_tma(FusedArgs a) {
  using C = TmaCfg<NP>;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * NP * 32];
  __shared__ __align__(8) uint64_t bars[8 * C::kStages];
  __shared__ int ok;
  fill_fp8_dq_table(lut);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(a.base[a.rank]);
  if (blockIdx.x == 0 && tid < a.P)
    st_release_sys(reinterpret_cast<uint64_t*>(a.base[tid]) + kReadyOff + a.rank, a.epoch);
  if (tid == 0) {
    ok = 1;
    for (int s = 0; s < a.P; ++s)
      if (!wait_flag(my_flags + kReadyOff + s, a.epoch)) ok = 0;
  }
  __syncthreads();
  if (!ok) {
    if (tid == 0) err_min(&a.err->overflow_block, -1);
    return;
  }
  // the peers' data was published to the generic proxy; the bulk copies
  // below read it through the async proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");

  unsigned char* bs[NP];
#pragma unroll
  for (int s = 0; s < NP; ++s) bs[s] = a.base[s];
  const uint64_t b0 = a.begin / kBlock;
  const uint64_t coff = a.codes_off + a.begin, soff = a.scales_off + 4 * b0;
  float* wtab = btab + warp * NP * 32;
  unsigned char* ring = dsm + warp * C::kWarpBytes;
  uint64_t* wb = bars + warp * C::kStages;
  if (lane == 0) {
    for (int s = 0; s < C::kStages; ++s) mbar_init(&wb[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t ntile = a.len / 512;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  const uint64_t gw = (uint64_t)blockIdx.x * 8 + warp;
  const uint64_t policy = policy_evict_first();
  auto issue = [&](uint64_t w, int s) {
    if (lane == 0 && w < ntile) {
      unsigned char* stg = ring + s * C::kStage;
      mbar_arrive_expect_tx(&wb[s], C::kStage);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        bulk_g2s(stg + p * C::kPiece, bs[p] + coff + w * 512, 512, &wb[s], policy);
        const uint64_t sa = reinterpret_cast<uint64_t>(bs[p] + soff + 16 * w);
        bulk_g2s(stg + p * C::kPiece + 512, reinterpret_cast<const void*>(sa & ~15ull), 32, &wb[s],
                 policy);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < C::kStages; ++s) issue(gw + s * nw, s);
  uint32_t phase = 0;
  int s = 0;
  for (uint64_t w = gw; w < ntile; w += nw) {
    mbar_wait(&wb[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const unsigned char* stg = ring + s * C::kStage;
    // every rank's buffer has the same layout: the window offset is common
    const int so = (int)(((a.scales_off + 4 * b0 + 16 * w) & 15u) >> 2) + (lane >> 3);
    uint32_t cw[NP][4];
    float sc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint4 v = lds128(stg + p * C::kPiece + lane * 16);
      cw[p][0] = v.x; cw[p][1] = v.y; cw[p][2] = v.z; cw[p][3] = v.w;
      sc[p] = reinterpret_cast<const float*>(stg + p * C::kPiece + 512)[so];
    }
    __syncwarp();  // the stage is free again
    issue(w + C::kStages * nw, s);
    s = s + 1 == C::kStages ? 0 : s + 1;
    reduce_store16<NP>(bs, coff, soff, w * 512 + lane * 16, cw, sc, (long long)b0, lut, a.err,
                       wtab);
  }
  // the partial last tile: per-thread path (whole warps, tables)
  const uint64_t nblocks = (a.len + kBlock - 1) / kBlock;
  const uint64_t ngroups = nblocks * 8;
  const uint64_t g0 = ntile * 32;
  if (g0 < ngroups) {
    const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
    const uint64_t gpad = g0 + (ngroups - g0 + 31) / 32 * 32;
    for (uint64_t g = g0 + blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride)
      fused_group<NP>(bs, a.codes_off + a.begin, a.scales_off + 4 * b0, g, g < ngroups ? a.len : 0,
                      (long long)b0, lut, a.err, wtab);
  }
  epoch_end(a);
}

// ---------------------------------------------------------------------------
// Push all-reduce (AGQ_AR_PUSH_P2P): the same decomposition with every NVLink
// transfer a fire-and-forget store (SM stores reach 690 GB/s per direction on
// this NVSwitch, pulls 655, profiles/r01_nvlink_probe_n4.log) and no load on
// a reduction's critical path crossing NVLink:
//   1. k_push_scatter: chunk q of my gradient -> inbox slot [me] of rank q;
//      the last CTA publishes "scattered" to every rank.
//   2. k_push_reduce: wait for every rank's "scattered", reduce my chunk from
//      P local pieces (my own + P-1 inbox slots, HBM) in ascending sender
//      rank, requantize, store the result into every rank's buffer; the epoch
//      end barrier (epoch_end) keeps the next call's scatter out of inboxes
//      still being read.
// ---------------------------------------------------------------------------
struct PushArgs {
  unsigned char* base[AGQ_MAX_WORLD];
  uint64_t scales_off, codes_off;              // my gradient in the symmetric buffer
  uint64_t in_scales_off, in_codes_off;        // inbox (P slots, indexed by sender)
  uint64_t slot_scales, slot_codes;            // bytes per inbox slot
  uint64_t rg[2 * AGQ_MAX_WORLD];              // chunk [begin, end) per owner (elements)
  uint64_t epoch;
  unsigned int* done_counter;
  agq_errors* err;
  int rank, P;
};

__global__ void __launch_bounds__(256) k_push_scatter(PushArgs a) {
  const int q = (a.rank + 1 + (int)blockIdx.y) % a.P;  // staggered peers
  const uint64_t b = a.rg[2 * q], len = a.rg[2 * q + 1] - b;
  const unsigned char* src = a.base[a.rank] + a.codes_off + b;
  unsigned char* dst = a.base[q] + a.in_codes_off + (uint64_t)a.rank * a.slot_codes;
  const uint64_t nv = len / 16;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = gridDim.x * (uint64_t)blockDim.x;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  uint64_t i = tid;
  for (; i + 3 * nth < nv; i += 4 * nth) {  // 4 independent 16-byte loads in flight
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ldg128_stream(s4 + i + u * nth);
#pragma unroll
    for (int u = 0; u < 4; ++u) d4[i + u * nth] = v[u];
  }
  for (; i < nv; i += nth) d4[i] = ldg128_stream(s4 + i);
  for (uint64_t j = nv * 16 + tid; j < len; j += nth) dst[j] = src[j];
  // block scales of chunk q
  const uint64_t nbq = (len + kBlock - 1) / kBlock;
  const float* ss = reinterpret_cast<const float*>(a.base[a.rank] + a.scales_off) + b / kBlock;
  float* ds = reinterpret_cast<float*>(a.base[q] + a.in_scales_off +
                                       (uint64_t)a.rank * a.slot_scales);
  for (uint64_t j = tid; j < nbq; j += nth) ds[j] = ss[j];
  // publish "scattered" once every CTA's stores are performed system-wide
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(a.done_counter, 1u);
    if (prev == gridDim.x * gridDim.y - 1) {
      __threadfence_system();
      for (int s = 0; s < a.P; ++s)
        if (s != a.rank)
          st_release_sys(reinterpret_cast<uint64_t*>(a.base[s]) + kScatterOff + a.rank, a.epoch);
      *a.done_counter = 0u;
    }
  }
}

// pt: pieces in ascending sender rank (my own chunk, else my inbox slot of
// that sender) and outputs = chunk [me] of every rank's buffer; built on the
// host so it stays in the parameter bank.
template <int NP>
#ifndef AGQ_PUSH_MINB
#define AGQ_PUSH_MINB 2  // 3 measured equal at 4 GPUs and spills the NP = 8 instance
#endif
__global__ void __launch_bounds__(256, AGQ_PUSH_MINB) k_push_reduce(PushArgs a, PieceTable pt) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * (NP > 0 ? NP : 1) * 32];
  __shared__ int ok;
  fill_fp8_dq_table(lut);
  const int tid = threadIdx.x;
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(a.base[a.rank]);
  if (tid == 0) {
    ok = 1;
    for (int s = 0; s < a.P; ++s)
      if (s != a.rank && !wait_flag(my_flags + kScatterOff + s, a.epoch)) ok = 0;
  }
  __syncthreads();
  if (!ok) {
    if (tid == 0) err_min(&a.err->overflow_block, -1);
    epoch_end(a);
    return;
  }
  const uint64_t begin = a.rg[2 * a.rank], len = a.rg[2 * a.rank + 1] - begin;
  const uint64_t b0 = begin / kBlock;
  const uint64_t nblocks = (len + kBlock - 1) / kBlock;
  const uint64_t ngroups = nblocks * 8;
  const uint64_t gpad = (ngroups + 31) / 32 * 32;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  float* wtab = NP > 0 ? btab + (tid >> 5) * NP * 32 : nullptr;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride)
    reduce_group<NP>(pt, g, g < ngroups ? len : 0, (long long)b0, lut, a.err, true, wtab);
  epoch_end(a);
}

__global__ void k_init_flags(uint64_t* flags) {
  const int i = threadIdx.x;
  if (i < 64) flags[i] = 0;
  else if (i < 64 + AGQ_MAX_WORLD) flags[i] = (uint64_t)kNone;
}

}  // namespace agqk

namespace agqh {
using namespace agqk;

namespace {
agq_status nccl_fail(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return AGQ_OK;
  if (!nccl().ok) return set_error(AGQ_ERR_NCCL, "libnccl.so.2 not available");
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, nccl().GetErrorString(r));
  return set_error(AGQ_ERR_NCCL, buf);
}
}  // namespace

agq_status comm_unique_id(unsigned char id[128]) {
  if (!nccl().ok) return set_error(AGQ_ERR_NCCL, "libnccl.so.2 not available");
  ncclUniqueId u;
  agq_status st = nccl_fail(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  if (st) return st;
  memcpy(id, u.internal, 128);
  return AGQ_OK;
}

agq_status comm_init(agq_comm** out, const unsigned char id[128], int nranks, int rank,
                     int device) {
  if (nranks < 1 || nranks > AGQ_MAX_WORLD || rank < 0 || rank >= nranks)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "need at least one worker");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "comm_init: cudaSetDevice");
  if (!nccl().ok) return set_error(AGQ_ERR_NCCL, "libnccl.so.2 not available");
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  agq_comm* c = new agq_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  agq_status st = nccl_fail(nccl().CommInitRank(&c->nccl, nranks, u, rank), "ncclCommInitRank");
  if (st) {
    delete c;
    return st;
  }
  e = cudaMalloc(&c->done_counter, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->done_counter, 0, sizeof(unsigned int));
  if (e != cudaSuccess) return cuda_fail(e, "comm_init: counter");
  *out = c;
  return AGQ_OK;
}

// Symmetric buffer: [flags 4 KB | scales | codes | inbox scales | inbox codes],
// the inbox holding P slots of one chunk each (push algorithm).
struct SymLayout {
  uint64_t scales_off, codes_off, in_scales_off, in_codes_off, slot_scales, slot_codes, bytes;
};
SymLayout sym_layout(uint64_t capacity, int P) {
  SymLayout L{};
  const uint64_t nb = (capacity + kBlock - 1) / kBlock;
  const uint64_t chunk_blocks = (nb + P - 1) / P;
  L.scales_off = kFlagsBytes;
  L.codes_off = L.scales_off + round_up(nb * 4, 256);
  L.in_scales_off = L.codes_off + round_up(capacity, 256);
  L.slot_scales = round_up(chunk_blocks * 4, 256);
  L.in_codes_off = L.in_scales_off + (uint64_t)P * L.slot_scales;
  L.slot_codes = round_up(chunk_blocks * kBlock, 256);
  L.bytes = L.in_codes_off + (uint64_t)P * L.slot_codes;
  return L;
}

agq_status comm_p2p_export(agq_comm* c, uint64_t capacity, unsigned char handle[256]) {
  const size_t bytes = sym_layout(capacity, c->nranks).bytes;
  if (c->sym && c->sym_bytes >= bytes) {
    // keep the existing mapping
  } else {
    if (c->sym) {
      cudaFree(c->sym);
      c->sym = nullptr;
    }
    cudaError_t e = cudaMalloc(&c->sym, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "p2p_export: cudaMalloc");
    c->sym_bytes = bytes;
    k_init_flags<<<1, 128>>>(reinterpret_cast<uint64_t*>(c->sym));
    count_launch();
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "p2p_export: init");
  }
  c->sym_cap = capacity;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->sym);
  if (e != cudaSuccess) return cuda_fail(e, "p2p_export: cudaIpcGetMemHandle");
  memset(handle, 0, 256);
  memcpy(handle, &h, sizeof(h));
  memcpy(handle + 128, &c->sym_bytes, sizeof(size_t));
  return AGQ_OK;
}

agq_status comm_p2p_open(agq_comm* c, const unsigned char* handles) {
  for (int s = 0; s < c->nranks; ++s) {
    if (s == c->rank) {
      c->peer[s] = c->sym;
      continue;
    }
    if (c->peer[s] && c->peer[s] != c->sym) cudaIpcCloseMemHandle(c->peer[s]);
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 256 * s, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "p2p_open: cudaIpcOpenMemHandle");
    c->peer[s] = static_cast<unsigned char*>(p);
  }
  c->p2p_ready = true;
  return AGQ_OK;
}

agq_status comm_p2p_buffers(agq_comm* c, uint8_t** codes, float** scales) {
  if (!c->sym) return set_error(AGQ_ERR_INVALID_ARGUMENT, "p2p buffers not exported");
  const SymLayout L = sym_layout(c->sym_cap, c->nranks);
  *scales = reinterpret_cast<float*>(c->sym + L.scales_off);
  *codes = c->sym + L.codes_off;
  return AGQ_OK;
}

agq_status comm_destroy(agq_comm* c) {
  if (!c) return AGQ_OK;
  cudaSetDevice(c->device);
  for (int s = 0; s < c->nranks; ++s)
    if (c->peer[s] && c->peer[s] != c->sym) cudaIpcCloseMemHandle(c->peer[s]);
  if (c->sym) cudaFree(c->sym);
  if (c->recv_codes) cudaFree(c->recv_codes);
  if (c->recv_scales) cudaFree(c->recv_scales);
  if (c->ring_codes) cudaFree(c->ring_codes);
  if (c->ring_scales) cudaFree(c->ring_scales);
  if (c->ring_sat) cudaFree(c->ring_sat);
  if (c->done_counter) cudaFree(c->done_counter);
  if (c->nccl) nccl().CommDestroy(c->nccl);
  delete c;
  return AGQ_OK;
}

int comm_rank(const agq_comm* c) { return c->rank; }
int comm_size(const agq_comm* c) { return c->nranks; }

namespace {

agq_status allreduce_nccl(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                          agq_errors* err, cudaStream_t s) {
  const int P = c->nranks, r = c->rank;
  std::vector<uint64_t> rg(2 * P);
  chunk_ranges(n, block, P, rg.data());
  uint64_t maxlen = 0;
  for (int q = 0; q < P; ++q) maxlen = std::max(maxlen, rg[2 * q + 1] - rg[2 * q]);
  const uint64_t maxblk = (maxlen + block - 1) / block;
  if (c->recv_chunk_cap < maxlen || !c->recv_codes) {
    if (c->recv_codes) cudaFree(c->recv_codes);
    if (c->recv_scales) cudaFree(c->recv_scales);
    c->recv_codes = nullptr;
    c->recv_scales = nullptr;
    const uint64_t slots = P > 1 ? P - 1 : 1;
    const uint64_t cap = round_up(maxlen ? maxlen : 1, 256);
    cudaError_t e = cudaMalloc(&c->recv_codes, slots * cap);
    if (e == cudaSuccess) e = cudaMalloc(&c->recv_scales, slots * round_up(cap / 128 * 4 + 1024, 256));
    if (e != cudaSuccess) return cuda_fail(e, "allreduce: workspace");
    c->recv_chunk_cap = cap;
  }
  const uint64_t cap = c->recv_chunk_cap;
  const uint64_t scap = round_up(cap / 128 * 4 + 1024, 256) / 4;
  (void)maxblk;
  auto slot = [&](int q) { return q < r ? q : q - 1; };
  const uint64_t br = rg[2 * r], er = rg[2 * r + 1], lr = er - br;
  const uint64_t nbr = (lr + block - 1) / block;
  // 1) all-to-all of chunk q -> rank q
  agq_status st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const uint64_t bq = rg[2 * q], lq = rg[2 * q + 1] - bq;
    if (lq) {
      nccl().Send(codes + bq, lq, ncclUint8, q, c->nccl, s);
      nccl().Send(scales + bq / block, (lq + block - 1) / block, ncclFloat32, q, c->nccl, s);
    }
    if (lr) {
      nccl().Recv(c->recv_codes + slot(q) * cap, lr, ncclUint8, q, c->nccl, s);
      nccl().Recv(c->recv_scales + slot(q) * scap, nbr, ncclFloat32, q, c->nccl, s);
    }
  }
  st = nccl_fail(nccl().GroupEnd(), "all-to-all");
  if (st) return st;
  // 2) local reduce of chunk r, pieces in ascending sender rank, in place
  if (lr) {
    std::vector<const uint8_t*> pc(P);
    std::vector<const float*> ps(P);
    for (int q = 0; q < P; ++q) {
      if (q == r) {
        pc[q] = codes + br;
        ps[q] = scales + br / block;
      } else {
        pc[q] = c->recv_codes + slot(q) * cap;
        ps[q] = c->recv_scales + slot(q) * scap;
      }
    }
    uint8_t* oc = codes + br;
    float* os = scales + br / block;
    st = reduce_requant_device(P, pc.data(), ps.data(), lr, block, 1, &oc, &os,
                               (long long)(br / block), err, s);
    if (st) return st;
  }
  // share an overflow with every rank (collective.hpp:278-281 aborts all)
  if (err) {
    st = nccl_fail(nccl().AllReduce(&err->overflow_block, &err->overflow_block, 1, ncclInt64,
                                 ncclMin, c->nccl, s),
                   "overflow flag");
    if (st) return st;
  }
  // 3) all-gather: reduced chunk r -> every rank, received in place
  st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const uint64_t bq = rg[2 * q], lq = rg[2 * q + 1] - bq;
    if (lr) {
      nccl().Send(codes + br, lr, ncclUint8, q, c->nccl, s);
      nccl().Send(scales + br / block, nbr, ncclFloat32, q, c->nccl, s);
    }
    if (lq) {
      nccl().Recv(codes + bq, lq, ncclUint8, q, c->nccl, s);
      nccl().Recv(scales + bq / block, (lq + block - 1) / block, ncclFloat32, q, c->nccl, s);
    }
  }
  return nccl_fail(nccl().GroupEnd(), "all-gather");
}

// Elements per thread: 16 (measured ~10% faster than 8 at 4 GPUs,
// profiles/r01_p2p_ept_ctas_n4.log; with the block-table decode the NP = 8
// instance fits 128 registers without spills). AGQ_P2P_EPT=8 selects the
// 8-element kernel (16 lanes per block) for comparison.
int fused_ept(int P) {
  (void)P;
  static const int forced = [] {
    const char* e = getenv("AGQ_P2P_EPT");
    return e ? atoi(e) : 0;
  }();
  return forced == 8 ? 8 : 16;
}

bool fused_tma() {
  static const bool v = [] {
    const char* e = getenv("AGQ_P2P_TMA");
    return e && e[0] == '1';
  }();
  return v;
}
template <int NP>
void launch_fused_tma(const FusedArgs& a, cudaStream_t s) {
  using C = TmaCfg<NP>;
  static const int occ = [] {
    cudaFuncSetAttribute(k_fused_tma<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::kSmem);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused_tma<NP>, 256, C::kSmem);
    return o < 1 ? 1 : o;
  }();
  k_fused_tma<NP><<<num_sms() * occ, 256, C::kSmem, s>>>(a);
}
template <int NP>
void launch_fused(const FusedArgs& a, int grid, cudaStream_t s) {
  if constexpr (NP > 0) {
    if (fused_tma()) return launch_fused_tma<NP>(a, s);
  }
  if (fused_ept(a.P) == 8)
    k_fused_allreduce<NP, 8><<<grid, 256, 0, s>>>(a);
  else
    k_fused_allreduce<NP, 16><<<grid, 256, 0, s>>>(a);
}

agq_status allreduce_p2p(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                         agq_errors* err, cudaStream_t s) {
  if (!c->p2p_ready) return set_error(AGQ_ERR_INVALID_ARGUMENT, "p2p buffers not opened");
  if (block != (uint32_t)kBlock) return set_error(AGQ_ERR_INVALID_ARGUMENT, "fused all-reduce needs block 128");
  if (n > c->sym_cap) return set_error(AGQ_ERR_INVALID_ARGUMENT, "all-reduce larger than p2p capacity");
  if (!err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "fused all-reduce needs an error record");
  uint8_t* sc_codes;
  float* sc_scales;
  comm_p2p_buffers(c, &sc_codes, &sc_scales);
  const uint64_t nb = (n + block - 1) / block;
  const bool inplace = codes == sc_codes && scales == sc_scales;
  if (!inplace) {
    cudaMemcpyAsync(sc_codes, codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(sc_scales, scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  const int P = c->nranks, r = c->rank;
  std::vector<uint64_t> rg(2 * P);
  chunk_ranges(n, block, P, rg.data());
  FusedArgs a{};
  for (int q = 0; q < P; ++q) a.base[q] = c->peer[q];
  a.scales_off = (uint64_t)(reinterpret_cast<unsigned char*>(sc_scales) - c->sym);
  a.codes_off = (uint64_t)(reinterpret_cast<unsigned char*>(sc_codes) - c->sym);
  a.begin = rg[2 * r];
  a.len = rg[2 * r + 1] - rg[2 * r];
  a.epoch = ++c->epoch;
  a.done_counter = c->done_counter;
  a.err = err;
  a.rank = r;
  a.P = P;
  static const int copy_only = getenv("AGQ_P2P_COPYONLY") ? 1 : 0;
  a.copy_only = copy_only;
  const uint64_t groups = (a.len + kBlock - 1) / kBlock * (fused_ept(P) == 8 && P <= 8 ? 16 : 8);
  uint64_t grid = (groups + 255) / 256;
  // co-resident grid (256 threads, small smem); AGQ_P2P_CTAS_PER_SM tunes it
  static const int per_sm = [] {
    const char* e = getenv("AGQ_P2P_CTAS_PER_SM");
    const int v = e ? atoi(e) : 2;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
  }();
  const uint64_t cap = (uint64_t)num_sms() * per_sm;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  switch (P) {
    case 1: launch_fused<1>(a, (int)grid, s); break;
    case 2: launch_fused<2>(a, (int)grid, s); break;
    case 3: launch_fused<3>(a, (int)grid, s); break;
    case 4: launch_fused<4>(a, (int)grid, s); break;
    case 5: launch_fused<5>(a, (int)grid, s); break;
    case 6: launch_fused<6>(a, (int)grid, s); break;
    case 7: launch_fused<7>(a, (int)grid, s); break;
    case 8: launch_fused<8>(a, (int)grid, s); break;
    default: launch_fused<0>(a, (int)grid, s); break;
  }
  count_launch();
  agq_status st = cuda_fail(cudaGetLastError(), "fused all-reduce: launch");
  if (st) return st;
  if (!inplace) {
    cudaMemcpyAsync(codes, sc_codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(scales, sc_scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  return AGQ_OK;
}

template <int NP>
void launch_push_reduce(const PushArgs& a, const PieceTable& pt, int grid, cudaStream_t s) {
  k_push_reduce<NP><<<grid, 256, 0, s>>>(a, pt);
}

agq_status allreduce_push(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                          agq_errors* err, cudaStream_t s) {
  if (!c->p2p_ready) return set_error(AGQ_ERR_INVALID_ARGUMENT, "p2p buffers not opened");
  if (block != (uint32_t)kBlock) return set_error(AGQ_ERR_INVALID_ARGUMENT, "push all-reduce needs block 128");
  if (n > c->sym_cap) return set_error(AGQ_ERR_INVALID_ARGUMENT, "all-reduce larger than p2p capacity");
  if (!err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "push all-reduce needs an error record");
  const SymLayout L = sym_layout(c->sym_cap, c->nranks);
  uint8_t* sc_codes = c->sym + L.codes_off;
  float* sc_scales = reinterpret_cast<float*>(c->sym + L.scales_off);
  const uint64_t nb = (n + block - 1) / block;
  const bool inplace = codes == sc_codes && scales == sc_scales;
  if (!inplace) {
    cudaMemcpyAsync(sc_codes, codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(sc_scales, scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  const int P = c->nranks, r = c->rank;
  std::vector<uint64_t> rg(2 * P);
  chunk_ranges(n, block, P, rg.data());
  PushArgs a{};
  for (int q = 0; q < P; ++q) a.base[q] = c->peer[q];
  for (int q = 0; q < 2 * P; ++q) a.rg[q] = rg[q];
  a.scales_off = L.scales_off;
  a.codes_off = L.codes_off;
  a.in_scales_off = L.in_scales_off;
  a.in_codes_off = L.in_codes_off;
  a.slot_scales = L.slot_scales;
  a.slot_codes = L.slot_codes;
  a.epoch = ++c->epoch;
  a.done_counter = c->done_counter;
  a.err = err;
  a.rank = r;
  a.P = P;
  uint64_t maxlen = 0;
  for (int q = 0; q < P; ++q) maxlen = std::max<uint64_t>(maxlen, rg[2 * q + 1] - rg[2 * q]);
  // scatter: ~2 CTAs per SM in total across the P-1 peers
  uint64_t gx = (maxlen / 16 + 1023) / 1024;
  const uint64_t cap_x = std::max<uint64_t>(1, (uint64_t)num_sms() * 2 / (P - 1));
  gx = std::min<uint64_t>(std::max<uint64_t>(gx, 1), cap_x);
  // AGQ_PUSH_TIMING=1 (diagnostics only): per-phase device time on stderr
  static const bool timing = getenv("AGQ_PUSH_TIMING") != nullptr;
  cudaEvent_t ev[3];
  if (timing) {
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[0], s);
  }
  k_push_scatter<<<dim3((unsigned)gx, (unsigned)(P - 1)), 256, 0, s>>>(a);
  count_launch();
  if (timing) cudaEventRecord(ev[1], s);
  agq_status st = cuda_fail(cudaGetLastError(), "push all-reduce: scatter launch");
  if (st) return st;
  PieceTable pt{};
  pt.np = P;
  pt.nout = P;
  const uint64_t begin = rg[2 * r];
  for (int q = 0; q < P; ++q) {
    if (q == r) {
      pt.codes[q] = c->peer[r] + L.codes_off + begin;
      pt.scales[q] = reinterpret_cast<const float*>(c->peer[r] + L.scales_off) + begin / kBlock;
    } else {
      pt.codes[q] = c->peer[r] + L.in_codes_off + (uint64_t)q * L.slot_codes;
      pt.scales[q] = reinterpret_cast<const float*>(c->peer[r] + L.in_scales_off +
                                                    (uint64_t)q * L.slot_scales);
    }
    pt.out_codes[q] = c->peer[q] + L.codes_off + begin;
    pt.out_scales[q] = reinterpret_cast<float*>(c->peer[q] + L.scales_off) + begin / kBlock;
  }
  const uint64_t groups = (rg[2 * r + 1] - rg[2 * r] + kBlock - 1) / kBlock * 8;
  uint64_t grid = (groups + 255) / 256;
  grid = std::min<uint64_t>(std::max<uint64_t>(grid, 1), (uint64_t)num_sms() * AGQ_PUSH_MINB);
  switch (P) {
    case 2: launch_push_reduce<2>(a, pt, (int)grid, s); break;
    case 3: launch_push_reduce<3>(a, pt, (int)grid, s); break;
    case 4: launch_push_reduce<4>(a, pt, (int)grid, s); break;
    case 5: launch_push_reduce<5>(a, pt, (int)grid, s); break;
    case 6: launch_push_reduce<6>(a, pt, (int)grid, s); break;
    case 7: launch_push_reduce<7>(a, pt, (int)grid, s); break;
    case 8: launch_push_reduce<8>(a, pt, (int)grid, s); break;
    default: return set_error(AGQ_ERR_INVALID_ARGUMENT, "push all-reduce: world size 2..8");
  }
  count_launch();
  st = cuda_fail(cudaGetLastError(), "push all-reduce: reduce launch");
  if (st) return st;
  if (timing) {
    cudaEventRecord(ev[2], s);
    cudaEventSynchronize(ev[2]);
    float t1 = 0, t2 = 0;
    cudaEventElapsedTime(&t1, ev[0], ev[1]);
    cudaEventElapsedTime(&t2, ev[1], ev[2]);
    fprintf(stderr, "push all-reduce rank %d n=%llu: scatter %.3f ms, reduce+gather %.3f ms\n", r,
            (unsigned long long)n, t1, t2);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  if (!inplace) {
    cudaMemcpyAsync(codes, sc_codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(scales, sc_scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  return AGQ_OK;
}

}  // namespace

agq_status allreduce_fp8(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                         int algo, agq_errors* err, cudaStream_t s) {
  if (n == 0) return AGQ_OK;
  if (c->nranks == 1) {
    // P = 1: the reference still re-quantizes acc = 0 + dequant (signed
    // zeros normalise), so run the reduce with one piece.
    const uint8_t* pc = codes;
    const float* ps = scales;
    return reduce_requant_device(1, &pc, &ps, n, block, 1, &codes, &scales, 0, err, s);
  }
  if (algo == AGQ_AR_FUSED_P2P) return allreduce_p2p(c, codes, scales, n, block, err, s);
  if (algo == AGQ_AR_PUSH_P2P) return allreduce_push(c, codes, scales, n, block, err, s);
  return allreduce_nccl(c, codes, scales, n, block, err, s);
}

// allreduce_naive_fp8 (collective.hpp:338-431) on real ranks: P-1 ring
// steps (rank r sends chunk (r-step) mod P to r+1 and folds chunk
// (r-step-1) mod P from r-1 into its own codes at its original scales), the
// saturation bitmask riding along with each chunk, then an all-gather in
// which rank r contributes chunk (r+1) mod P with ITS scales. err->saturated
// = CollectiveResult::overflow_elements (summed over ranks: each chunk's
// final owner counts it); *events = this rank's overflow_events entry.
agq_status allreduce_naive(agq_comm* c, uint8_t* codes, float* scales, uint64_t n,
                           uint32_t block, agq_errors* err, unsigned long long* events,
                           cudaStream_t s) {
  if (n == 0 || c->nranks == 1) return AGQ_OK;
  const int P = c->nranks, r = c->rank;
  std::vector<uint64_t> rg(2 * P);
  chunk_ranges(n, block, P, rg.data());
  uint64_t maxlen = 0;
  for (int q = 0; q < P; ++q) maxlen = std::max(maxlen, rg[2 * q + 1] - rg[2 * q]);
  const uint64_t cap = round_up(maxlen ? maxlen : 1, 256);
  const uint64_t words = cap / 32;
  if (c->ring_cap < cap) {
    if (c->ring_codes) cudaFree(c->ring_codes);
    if (c->ring_scales) cudaFree(c->ring_scales);
    if (c->ring_sat) cudaFree(c->ring_sat);
    c->ring_codes = nullptr;
    c->ring_scales = nullptr;
    c->ring_sat = nullptr;
    c->ring_cap = 0;
    cudaError_t e = cudaMalloc(&c->ring_codes, cap);
    if (e == cudaSuccess) e = cudaMalloc(&c->ring_scales, (cap / block + 2) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&c->ring_sat, 2 * words * 4);
    if (e != cudaSuccess) return cuda_fail(e, "naive all-reduce: workspace");
    c->ring_cap = cap;
  }
  const int to = (r + 1) % P, from = (r - 1 + P) % P;
  uint32_t* sat_mine = c->ring_sat;            // mask of the chunk folded last step
  uint32_t* sat_in = c->ring_sat + c->ring_cap / 32;  // mask arriving with the message
  for (int step = 0; step < P - 1; ++step) {
    const int cs = ((r - step) % P + P) % P, cr = ((r - step - 1) % P + P) % P;
    const uint64_t bs = rg[2 * cs], ls = rg[2 * cs + 1] - bs;
    const uint64_t br = rg[2 * cr], lr = rg[2 * cr + 1] - br;
    agq_status st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
    if (st) return st;
    if (ls) {
      nccl().Send(codes + bs, ls, ncclUint8, to, c->nccl, s);
      nccl().Send(scales + bs / block, (ls + block - 1) / block, ncclFloat32, to, c->nccl, s);
      if (step) nccl().Send(sat_mine, (ls + 31) / 32, ncclUint32, to, c->nccl, s);
    }
    if (lr) {
      nccl().Recv(c->ring_codes, lr, ncclUint8, from, c->nccl, s);
      nccl().Recv(c->ring_scales, (lr + block - 1) / block, ncclFloat32, from, c->nccl, s);
      if (step) nccl().Recv(sat_in, (lr + 31) / 32, ncclUint32, from, c->nccl, s);
    }
    st = nccl_fail(nccl().GroupEnd(), "naive ring step");
    if (st) return st;
    const bool last = step == P - 2;
    st = naive_step_device(c->ring_codes, c->ring_scales, step ? sat_in : nullptr, codes + br,
                           scales + br / block, last ? nullptr : sat_mine, lr, block,
                           last ? &err->saturated : nullptr, events, s);
    if (st) return st;
  }
  agq_status st = nccl_fail(nccl().AllReduce(&err->saturated, &err->saturated, 1, ncclUint64,
                                             ncclSum, c->nccl, s),
                            "saturation count");
  if (st) return st;
  // all-gather: rank q owns chunk (q+1) mod P
  const int co = (r + 1) % P;
  const uint64_t bo = rg[2 * co], lo = rg[2 * co + 1] - bo;
  st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const int cq = (q + 1) % P;
    const uint64_t bq = rg[2 * cq], lq = rg[2 * cq + 1] - bq;
    if (lo) {
      nccl().Send(codes + bo, lo, ncclUint8, q, c->nccl, s);
      nccl().Send(scales + bo / block, (lo + block - 1) / block, ncclFloat32, q, c->nccl, s);
    }
    if (lq) {
      nccl().Recv(codes + bq, lq, ncclUint8, q, c->nccl, s);
      nccl().Recv(scales + bq / block, (lq + block - 1) / block, ncclFloat32, q, c->nccl, s);
    }
  }
  return nccl_fail(nccl().GroupEnd(), "naive all-gather");
}

agq_status allreduce_bf16_nccl(agq_comm* c, void* data, uint64_t n, cudaStream_t s) {
  return nccl_fail(nccl().AllReduce(data, data, n, ncclBfloat16, ncclSum, c->nccl, s),
                   "ncclAllReduce(bf16)");
}

}  // namespace agqh
