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
// AGQ_AR_PUSH_P2P (v3): the same decomposition with every NVLink transfer a
//   store: scatter chunk q into rank q's inbox, then reduce from local memory
//   and store the result into every rank's buffer.
// AGQ_AR_ONESHOT_P2P (v4, small messages): every rank stores its whole
//   gradient into every peer's double-buffered inbox with LL stores (payload
//   word + epoch in each 8-byte half) and reduces all blocks itself; no fence,
//   no barrier (k_oneshot_ll).
// The epoch of the P2P algorithms lives on the device (each call reads it
//   and its last CTA stores it), so captured CUDA graphs replay correctly.
//
// Failure handling: a timed-out barrier (a peer that never arrived) records
// overflow_block = -1 (agq_errors_message: "peer did not arrive") and marks
// the communicator failed on every rank (a sticky flag each kernel checks
// first), so later calls fail fast instead of reading stale peer data.
// Data errors are shared: every rank reports the same bad-scale / overflow
// error, as the reference aborts all workers (collective.hpp:158-168,
// :278-281).
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
agq_status comm_destroy(agq_comm* c);
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
constexpr size_t kFlagsBytes = 4096;
// u64 words of the flags page
constexpr int kReadyOff = 0;       // [16] start barrier, epoch per sender
constexpr int kDoneOff = 16;       // [16] end barrier, epoch per sender
constexpr int kScatteredOff = 32;  // [16] push algorithm: inbox slot written
constexpr int kFailOff = 48;       // sticky: a barrier of this communicator timed out
constexpr int kErrOff = 64;        // [2] min overflow block / min bad-scale key of
                                   // the group (peers atomicMin into them)
size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

struct agq_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 0, rank = 0, device = 0;
  uint64_t timeout_ns = 300ull * 1000000000ull;  // device barrier timeout
  // v1 workspace: P-1 receive slots of one chunk (codes + block scales)
  uint8_t* recv_codes = nullptr;
  float* recv_scales = nullptr;
  uint64_t recv_chunk_cap = 0;  // elements per slot
  uint64_t recv_scale_cap = 0;  // floats per slot
  // naive-ring workspace: one incoming chunk + two saturation bitmasks
  uint8_t* ring_codes = nullptr;
  float* ring_scales = nullptr;
  uint32_t* ring_sat = nullptr;
  uint64_t ring_cap = 0;  // elements
  uint32_t ring_block = 0;
  // v2/v3 symmetric memory
  unsigned char* sym = nullptr;
  size_t sym_bytes = 0;
  uint64_t sym_cap = 0;  // elements
  unsigned char* peer[AGQ_MAX_WORLD] = {};
  bool p2p_ready = false;
  unsigned int* done_counter = nullptr;  // local, one per kernel in flight
  // local: the last completed P2P epoch. The kernels read it (+1 = this
  // call's epoch) and the last CTA of the call stores it, so the epoch lives
  // on the device and a captured CUDA graph replays correctly.
  uint64_t* epoch_ctr = nullptr;
  // device: two [elements, blocks] records of the phase-1 traffic, used by
  // alternate epochs; each kernel zeroes the other one for the next call
  unsigned long long* stats = nullptr;
  // message trace of the last all-reduce issued by this rank
  std::vector<agq_trace_event> trace;
  int trace_algo = -1;
  cudaStream_t trace_stream = nullptr;
};

namespace agqk {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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
  uint64_t* epoch_ctr;                 // last completed epoch (this rank, local)
  uint64_t timeout_ns;
  unsigned int* done_counter;
  unsigned long long* stats;           // [elements, blocks] pulled from the peers
  agq_errors* err;
  int rank, P;
};

#ifdef AGQ_AR_PROFILE
// experiment builds: globaltimer stamps of the last fused call
__device__ unsigned long long g_ar_prof[8];
#define AR_STAMP(i) (g_ar_prof[i] = globaltimer())
#else
#define AR_STAMP(i) ((void)0)
#endif

// This call's epoch: one past the last completed one (stored by the
// previous call's last CTA, a kernel earlier on this stream).
__device__ __forceinline__ uint64_t call_epoch(const uint64_t* ctr) { return __ldcg(ctr) + 1; }

// Spin until *f >= epoch. False on timeout or when the communicator has
// been marked failed (by this rank or a peer).
__device__ bool wait_flag(const uint64_t* f, uint64_t epoch, const uint64_t* fail,
                          uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(f) < epoch) {
    if (ld_acquire_sys(fail) != 0) return false;
    if (globaltimer() - t0 > timeout_ns) return false;
    __nanosleep(200);
  }
  return true;
}

// Mark the communicator failed on every rank (sticky, see agq_comm_set_timeout).
template <class Args>
__device__ void mark_failed(const Args& a) {
  for (int s = 0; s < a.P; ++s) st_release_sys(reinterpret_cast<uint64_t*>(a.base[s]) + kFailOff, 1);
  err_min(&a.err->overflow_block, -1);
}

// Start barrier of a P2P epoch (thread 0 of each CTA; CTA 0 announces).
template <class Args>
__device__ bool start_barrier(const Args& a, int wait_off, bool skip_self, uint64_t ep) {
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(a.base[a.rank]);
  // set by an earlier call (a previous kernel): a relaxed load suffices
  if (ld_relaxed_sys(my_flags + kFailOff) != 0) return false;
  bool ok = true;
  for (int s = 0; s < a.P; ++s)
    if (!(skip_self && s == a.rank) &&
        !wait_flag(my_flags + wait_off + s, ep, my_flags + kFailOff, a.timeout_ns))
      ok = false;
  return ok;
}

// One 16-element group of the fused all-reduce with every pointer in
// registers (compile-time NP): chunk r of every rank is read over NVLink
// (rank order = ascending sender rank), reduced from +0.0f in FP32,
// requantized and written back in place to all ranks.
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
    build_tables<NP>(wtab, sc);  // every lane of the warp
    if (in_range) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        sbad |= bad_scale_bit(sc[p], p);
        const uint32_t w[4] = {cv[p].x, cv[p].y, cv[p].z, cv[p].w};
        if (dq_fast(sc[p]))
          dq_f16_accum<4>(w, lane_tab(wtab, p), acc);
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


// End of an all-reduce epoch. EVERY CTA calls it exactly once (also after a
// failed start), so the per-kernel CTA counter always returns to zero. The
// last CTA of this rank's grid shares this rank's data errors with every
// rank, publishes "done" to every rank and waits for all of them, so the
// kernel completes only when every rank has finished writing into (and
// reading from) this rank's buffer; then it merges the peers' errors.
// cta_stats (shared, or nullptr): this CTA's [elements, blocks] moved per
// peer, added to the communicator's counters once per CTA.
template <class Args>
__device__ __forceinline__ void epoch_end(const Args& a, uint64_t ep, bool ok,
                                          const unsigned long long* cta_stats = nullptr) {
  unsigned char* const* base = a.base;
  const int P = a.P, rank = a.rank;
  agq_errors* err = a.err;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (cta_stats != nullptr && cta_stats[0] != 0) {  // read from each of the P - 1 peers
    atomicAdd(&a.stats[2 * (ep & 1)], cta_stats[0] * (a.P - 1));
    atomicAdd(&a.stats[2 * (ep & 1) + 1], cta_stats[1] * (a.P - 1));
  }
  const unsigned int prev = atomicAdd(a.done_counter, 1u);
  if (prev != gridDim.x * gridDim.y - 1) return;
  AR_STAMP(3);
  // One system fence: it acquires every CTA's writes (each fenced before its
  // increment, observed through the counter) and this rank's error record,
  // and orders all of it before the relaxed "done" stores below (a release
  // per store would cost one system fence per peer: ~2 us each).
  __threadfence_system();
  uint64_t* my_flags = reinterpret_cast<uint64_t*>(base[rank]);
  // a CTA that failed its start barrier recorded -1 (min over the record)
  const long long ov = *reinterpret_cast<volatile long long*>(&err->overflow_block);
  if (ok && ov != -1) {
    const long long bs = *reinterpret_cast<volatile long long*>(&err->bad_scale_block);
    if (ov != kNone || bs != kNone) {  // rare: share this rank's data errors before "done"
      for (int s = 0; s < P; ++s) {
        long long* pe = reinterpret_cast<long long*>(base[s]) + kErrOff;
        if (ov != kNone) atomicMin(pe, ov);
        if (bs != kNone) atomicMin(pe + 1, bs);
      }
      __threadfence_system();
    }
    for (int s = 0; s < P; ++s)
      st_relaxed_sys(reinterpret_cast<uint64_t*>(base[s]) + kDoneOff + rank, ep);
    bool fine = true;
    AR_STAMP(4);
    for (int s = 0; s < P; ++s)
      if (!wait_flag(my_flags + kDoneOff + s, ep, my_flags + kFailOff, a.timeout_ns))
        fine = false;
    AR_STAMP(5);
    // one 16-byte read and reset of both words (peers enter the next epoch's
    // end only after this kernel: their start barrier needs our next "ready")
    long long e0, e1;
    asm volatile("ld.volatile.global.v2.s64 {%0, %1}, [%2];"
                 : "=l"(e0), "=l"(e1) : "l"(my_flags + kErrOff) : "memory");
    if (e0 != kNone) err_min(&err->overflow_block, e0);
    if (e1 != kNone) err_min(&err->bad_scale_block, e1);
    if (e0 != kNone || e1 != kNone)
      asm volatile("st.volatile.global.v2.s64 [%0], {%1, %1};"
                   :: "l"(my_flags + kErrOff), "l"(kNone) : "memory");
    if (!fine) mark_failed(a);
  } else {
    mark_failed(a);
  }
  __threadfence();
  // the next epoch's traffic record (this one stays readable for last_trace)
  a.stats[2 * ((ep + 1) & 1)] = 0ull;
  a.stats[2 * ((ep + 1) & 1) + 1] = 0ull;
  *a.epoch_ctr = ep;     // every CTA of this call has read it (they all arrived)
  AR_STAMP(6);
  *a.done_counter = 0u;  // both read by the next kernel on this stream
}

template <int NP>
__global__ void __launch_bounds__(256, 2) k_fused_allreduce(FusedArgs a) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * (NP > 0 ? NP : 1) * 32];  // 8 warps x NP pieces x 32 entries
  __shared__ int ok;
  __shared__ unsigned long long cta_stats[2];
  const int tid = threadIdx.x;
  if (tid == 0 && blockIdx.x == 0) AR_STAMP(0);
  const uint64_t ep = call_epoch(a.epoch_ctr);
  // start barrier: announce "my input is final" to every rank (CTA 0, before
  // anything else), then wait for every rank's announcement (each CTA)
  if (blockIdx.x == 0 && tid < a.P)
    st_release_sys(reinterpret_cast<uint64_t*>(a.base[tid]) + kReadyOff + a.rank, ep);
  fill_fp8_dq_table(lut);
  float* wtab = btab + (threadIdx.x >> 5) * (NP > 0 ? NP : 1) * 32;
  if (tid < 2) cta_stats[tid] = 0ull;
  if (tid == 0) {
    ok = start_barrier(a, kReadyOff, false, ep) ? 1 : 0;
    if (!ok) err_min(&a.err->overflow_block, -1);
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x == 0) AR_STAMP(1);
  if (!ok) {
    epoch_end(a, ep, false);
    return;
  }

  const uint64_t b0 = a.begin / kBlock;
  const uint64_t nblocks = (a.len + kBlock - 1) / kBlock;
  const uint64_t ngroups = nblocks * 8;
  const uint64_t gpad = (ngroups + 31) / 32 * 32;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  unsigned long long n_el = 0, n_blk = 0;  // what this thread moved per peer
  if constexpr (NP > 0) {
    unsigned char* bs[NP];
#pragma unroll
    for (int s = 0; s < NP; ++s) bs[s] = a.base[s];
    const uint64_t coff = a.codes_off + a.begin, soff = a.scales_off + 4 * b0;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride) {
      const uint64_t len = g < ngroups ? a.len : 0;
      fused_group<NP>(bs, coff, soff, g, len, (long long)b0, lut, a.err, wtab);
      if (g * 16 < len) {
        n_el += min((uint64_t)16, len - g * 16);
        n_blk += (tid & 7) == 0;
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
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + tid; g < gpad; g += stride) {
      const uint64_t len = g < ngroups ? a.len : 0;
      reduce_group<0>(pt, g, len, (long long)b0, lut, a.err, true);
      if (g * 16 < len) {
        n_el += min((uint64_t)16, len - g * 16);
        n_blk += (tid & 7) == 0;
      }
    }
  }
  // per-warp sums -> the communicator's counters (trace of what was moved)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    n_el += __shfl_xor_sync(0xffffffffu, n_el, o);
    n_blk += __shfl_xor_sync(0xffffffffu, n_blk, o);
  }
  if ((tid & 31) == 0 && n_el) {
    atomicAdd(&cta_stats[0], n_el);
    atomicAdd(&cta_stats[1], n_blk);
  }
  if (tid == 0 && blockIdx.x == 0) AR_STAMP(2);
  epoch_end(a, ep, true, cta_stats);
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
  uint64_t* epoch_ctr;                         // last completed epoch (this rank, local)
  uint64_t timeout_ns;
  unsigned int* done_counter;
  unsigned long long* stats;                   // [elements, blocks] scattered (all peers)
  agq_errors* err;
  int rank, P;
};

__global__ void __launch_bounds__(256) k_push_scatter(PushArgs a) {
  const uint64_t ep = call_epoch(a.epoch_ctr);  // k_push_reduce stores it
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
  // what this thread moved (16-byte vectors, tail bytes, scales), per warp
  unsigned long long n_el = 0, n_blk = 0;
  if (tid < nv) n_el += 16 * ((nv - 1 - tid) / nth + 1);
  if (nv * 16 + tid < len) n_el += (len - nv * 16 - 1 - tid) / nth + 1;
  if (tid < nbq) n_blk += (nbq - 1 - tid) / nth + 1;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    n_el += __shfl_xor_sync(0xffffffffu, n_el, o);
    n_blk += __shfl_xor_sync(0xffffffffu, n_blk, o);
  }
  if ((threadIdx.x & 31) == 0 && (n_el | n_blk)) {
    atomicAdd(&a.stats[2 * (ep & 1)], n_el);
    atomicAdd(&a.stats[2 * (ep & 1) + 1], n_blk);
  }
  // publish "scattered" once every CTA's stores are performed system-wide
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(a.done_counter, 1u);
    if (prev == gridDim.x * gridDim.y - 1) {
      __threadfence_system();
      for (int s = 0; s < a.P; ++s)
        if (s != a.rank)
          st_release_sys(reinterpret_cast<uint64_t*>(a.base[s]) + kScatteredOff + a.rank, ep);
      *a.done_counter = 0u;
    }
  }
}


// pt: pieces in ascending sender rank (my own chunk, else my inbox slot of
// that sender) and outputs = chunk [me] of every rank's buffer; built on the
// host so it stays in the parameter bank. 2 CTAs per SM (3 measured equal at
// 4 GPUs and spills the NP = 8 instance).
template <int NP>
__global__ void __launch_bounds__(256, 2) k_push_reduce(PushArgs a, PieceTable pt) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * (NP > 0 ? NP : 1) * 32];
  __shared__ int ok;
  fill_fp8_dq_table(lut);
  const int tid = threadIdx.x;
  const uint64_t ep = call_epoch(a.epoch_ctr);
  if (tid == 0) {
    ok = start_barrier(a, kScatteredOff, true, ep) ? 1 : 0;
    if (!ok) err_min(&a.err->overflow_block, -1);
  }
  __syncthreads();
  if (!ok) {
    epoch_end(a, ep, false);
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
  epoch_end(a, ep, true);
}

// ---------------------------------------------------------------------------
// One-shot all-reduce (AGQ_AR_ONESHOT_P2P), the small-message algorithm: one
// exchange instead of two and no barrier. Every rank stores its WHOLE
// gradient into every peer's inbox (slot [me] of the half selected by the
// epoch's parity), then reduces ALL blocks itself (own gradient + P-1 inbox
// slots, ascending sender rank): the same per-block arithmetic as the
// decomposed protocol, so bit-identical results, and every rank sees every
// data error (no error exchange). A peer can write a half again only two
// epochs later, after its call in between consumed this rank's data of that
// epoch, i.e. after this rank finished reading the half.
// 2(P-1)x the wire bytes of the decomposed protocol: small messages only.
// ---------------------------------------------------------------------------
struct OneShotArgs {
  unsigned char* base[AGQ_MAX_WORLD];
  uint64_t scales_off, codes_off;  // my gradient in the symmetric buffer
  uint64_t os_off;                 // inbox region: [parity][sender] slots
  uint64_t n;
  uint64_t* epoch_ctr;
  uint64_t timeout_ns;
  unsigned int* done_counter;
  unsigned long long* stats;
  agq_errors* err;
  int rank, P;
};

// One-shot, LL flavour (single kernel, no fence, no flag word): every
// 4-byte payload word travels with the epoch in the same 8-byte half of a
// 16-byte store, so a receiver polls the data itself and knows it is this
// call's as soon as the epoch matches (8-byte stores arrive whole over
// NVLink). Per group of 16 codes: two 16-byte stores per peer; per block
// scale: one 8-byte store. Each thread first sends all its groups, then
// receives and reduces them, so no thread waits on data a later phase of
// its own peer thread would send.
struct OneShotLL {
  uint64_t slot_bytes, codes_bytes;  // per sender slot: [codes LL | scales LL]
};
__device__ __forceinline__ void st_ll4(void* p, uint32_t a, uint32_t b, uint32_t f) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %3, %2, %3};" ::"l"(p), "r"(a), "r"(b),
               "r"(f)
               : "memory");
}
__device__ __forceinline__ void st_ll2(void* p, uint32_t a, uint32_t f) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(f) : "memory");
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_v2(const void* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}

template <int NP>
__global__ void __launch_bounds__(256, 2)
    k_oneshot_ll(OneShotArgs a, OneShotLL ll, const __grid_constant__ PieceTable out) {
  __shared__ double lut[kDqTable];
  __shared__ float btab[8 * NP * 32];
  const int tid = threadIdx.x, sub = tid & 7;
  const uint64_t ep = call_epoch(a.epoch_ctr);
  const uint32_t f = (uint32_t)ep;
  const uint64_t n = a.n, ngroups = (n + 15) / 16, gpad = (ngroups + 31) / 32 * 32;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  const uint64_t g0 = blockIdx.x * (uint64_t)blockDim.x + tid;
  const unsigned char* my_codes = a.base[a.rank] + a.codes_off;
  const float* my_scales = reinterpret_cast<const float*>(a.base[a.rank] + a.scales_off);
  auto slot = [&](int dst, int sender) {
    return a.base[dst] + a.os_off + ((ep & 1) * a.P + sender) * ll.slot_bytes;
  };
  auto my_group = [&](uint64_t g) {
    uint32_t w[4] = {0, 0, 0, 0};
    const uint64_t e0 = g * 16;
    if (e0 + 16 <= n) {
      const uint4 v = *reinterpret_cast<const uint4*>(my_codes + e0);
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      for (int e = 0; e < 16 && e0 + e < n; ++e) w[e >> 2] |= (uint32_t)my_codes[e0 + e] << (8 * (e & 3));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  };
  // 1) send: my groups (and my blocks' scales) to every peer
  for (uint64_t g = g0; g < ngroups; g += stride) {
    const uint4 v = my_group(g);
    const uint64_t blk = g / 8;
    const bool send_scale = sub == 0;  // group 8b carries block b's scale
    const uint32_t sc = send_scale ? f2u(my_scales[blk]) : 0u;
#pragma unroll
    for (int d = 1; d < NP; ++d) {
      const int q = (a.rank + d) % NP;
      unsigned char* sl = slot(q, a.rank);
      st_ll4(sl + g * 32, v.x, v.y, f);
      st_ll4(sl + g * 32 + 16, v.z, v.w, f);
      if (send_scale) st_ll2(sl + ll.codes_bytes + blk * 8, sc, f);
    }
  }
  fill_fp8_dq_table(lut);  // (after the sends: they do not need it)
  __syncthreads();
  // 2) receive + reduce (ascending sender rank), result into my gradient
  const uint64_t* fail = reinterpret_cast<const uint64_t*>(a.base[a.rank]) + kFailOff;
  bool ok = true;
  float* wtab = btab + (tid >> 5) * NP * 32;
  for (uint64_t g = g0; g < gpad; g += stride) {
    const uint64_t e0 = g * 16, blk = e0 / kBlock;
    const bool in_range = g < ngroups;
    const bool blk_exists = blk * kBlock < n;
    uint4 cv[NP];
    float sc[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      cv[p] = make_uint4(0, 0, 0, 0);
      sc[p] = 0.0f;
      if (p == a.rank) {
        if (blk_exists) sc[p] = my_scales[blk];
        if (in_range) cv[p] = my_group(g);
        continue;
      }
      const unsigned char* sl = slot(a.rank, p);
      const uint64_t t0 = globaltimer();
      for (uint32_t spin = 0;; ++spin) {
        bool ready = true;
        if (blk_exists) {
          const uint2 s2 = ld_v2(sl + ll.codes_bytes + blk * 8);
          if (s2.y == f) sc[p] = u2f(s2.x); else ready = false;
        }
        if (in_range) {
          const uint4 lo = ld_v4(sl + g * 32), hi = ld_v4(sl + g * 32 + 16);
          if (lo.y == f && lo.w == f && hi.y == f && hi.w == f)
            cv[p] = make_uint4(lo.x, lo.z, hi.x, hi.z);
          else
            ready = false;
        }
        if (ready) break;
        if ((spin & 255) == 255 &&
            (ld_relaxed_sys(fail) != 0 || globaltimer() - t0 > a.timeout_ns)) {
          ok = false;
          break;
        }
      }
    }
    reduce_compute<NP>(out, e0, in_range ? n : 0, in_range && e0 + 16 <= n, cv, sc, 0, lut, a.err,
                       wtab);
  }
  if (!ok) err_min(&a.err->overflow_block, -1);
  if (g0 == 0) {  // per peer: the whole tensor
    atomicAdd(&a.stats[2 * (ep & 1)], (unsigned long long)n * (NP - 1));
    atomicAdd(&a.stats[2 * (ep & 1) + 1], (unsigned long long)((n + kBlock - 1) / kBlock) * (NP - 1));
  }
  __syncthreads();
  if (tid != 0) return;
  __threadfence();  // this CTA's error-record updates before its count (release)
  const unsigned int prev = atomicAdd(a.done_counter, 1u);
  if (prev != gridDim.x - 1) return;
  __threadfence();
  if (ld_relaxed_sys(reinterpret_cast<const uint64_t*>(&a.err->overflow_block)) == (uint64_t)-1)
    mark_failed(a);
  a.stats[2 * ((ep + 1) & 1)] = 0ull;
  a.stats[2 * ((ep + 1) & 1) + 1] = 0ull;
  *a.epoch_ctr = ep;
  *a.done_counter = 0u;
}

__global__ void k_init_flags(uint64_t* flags) {
  const int i = threadIdx.x;  // 128 threads: the flag words in use
  flags[i] = (i == kErrOff || i == kErrOff + 1) ? (uint64_t)kNone : 0;
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

// id == nullptr: a P2P-only communicator (no NCCL communicator; the NVLink
// algorithms only). Also what lets several ranks share one GPU, which NCCL
// refuses.
agq_status comm_init(agq_comm** out, const unsigned char id[128], int nranks, int rank,
                     int device) {
  if (nranks < 1 || nranks > AGQ_MAX_WORLD || rank < 0 || rank >= nranks)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "need at least one worker");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "comm_init: cudaSetDevice");
  agq_comm* c = new agq_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (id != nullptr) {
    if (!nccl().ok) {
      delete c;
      return set_error(AGQ_ERR_NCCL, "libnccl.so.2 not available");
    }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    agq_status st = nccl_fail(nccl().CommInitRank(&c->nccl, nranks, u, rank), "ncclCommInitRank");
    if (st) {
      delete c;
      return st;
    }
  }
  e = cudaMalloc(&c->done_counter, 64);  // [0]: CTA counter, [8..15]: epoch
  if (e == cudaSuccess) e = cudaMemset(c->done_counter, 0, 64);
  c->epoch_ctr = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(c->done_counter) + 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->stats, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->stats, 0, 4 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    comm_destroy(c);
    return cuda_fail(e, "comm_init: counters");
  }
  *out = c;
  return AGQ_OK;
}

agq_status comm_set_timeout(agq_comm* c, double seconds) {
  if (!(seconds > 0.0) || seconds > 1e6)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "timeout must be in (0, 1e6] seconds");
  c->timeout_ns = (uint64_t)(seconds * 1e9);
  return AGQ_OK;
}

// Symmetric buffer: [flags 4 KB | scales | codes | inbox scales | inbox codes],
// the inbox holding P slots of one chunk each (push algorithm).
struct SymLayout {
  uint64_t scales_off, codes_off, in_scales_off, in_codes_off, slot_scales, slot_codes;
  // one-shot inboxes (LL format): 2 halves x P slots of [codes 32 B per
  // 16-code group | scales 8 B per block] for up to ll_cap elements
  uint64_t ll_off, ll_cap, ll_codes_bytes, ll_slot_bytes;
  uint64_t bytes;
};
constexpr uint64_t kOneShotLLMaxElems = 1u << 20;
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
  L.ll_off = L.in_codes_off + (uint64_t)P * L.slot_codes;
  L.ll_cap = std::min<uint64_t>(capacity, kOneShotLLMaxElems);
  L.ll_codes_bytes = round_up((L.ll_cap + 15) / 16 * 32, 256);
  L.ll_slot_bytes = L.ll_codes_bytes + round_up((L.ll_cap + kBlock - 1) / kBlock * 8, 256);
  L.bytes = L.ll_off + 2 * (uint64_t)P * L.ll_slot_bytes;
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
    {  // LL inboxes: no stale word may carry a future epoch
      const SymLayout L = sym_layout(capacity, c->nranks);
      e = cudaMemset(c->sym + L.ll_off, 0, L.bytes - L.ll_off);
      if (e != cudaSuccess) return cuda_fail(e, "p2p_export: LL inbox");
    }
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
  if (c->stats) cudaFree(c->stats);
  if (c->nccl) nccl().CommDestroy(c->nccl);
  delete c;
  return AGQ_OK;
}

int comm_rank(const agq_comm* c) { return c->rank; }
int comm_size(const agq_comm* c) { return c->nranks; }

namespace {

// One chunk message (collective.hpp:195-206 deliver: payload = codes + 4 *
// scales of the block-aligned chunk).
agq_trace_event chunk_event(int phase, int sender, int receiver, uint64_t begin, uint64_t len,
                            uint32_t block) {
  agq_trace_event e;
  e.phase = phase;
  e.sender = sender;
  e.receiver = receiver;
  e.chunk_start = begin;
  e.chunk_len = len;
  e.payload_bytes = len + 4 * ((len + block - 1) / block);
  return e;
}

// Share this rank's data errors with every rank (min over ranks): the
// reference's workers all abort on the same bad scale / overflow.
agq_status share_errors(agq_comm* c, agq_errors* err, cudaStream_t s) {
  if (!err) return AGQ_OK;
  agq_status st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
  if (st) return st;
  nccl().AllReduce(&err->overflow_block, &err->overflow_block, 1, ncclInt64, ncclMin, c->nccl, s);
  nccl().AllReduce(&err->bad_scale_block, &err->bad_scale_block, 1, ncclInt64, ncclMin, c->nccl,
                   s);
  return nccl_fail(nccl().GroupEnd(), "error flags");
}

agq_status allreduce_nccl(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                          agq_errors* err, cudaStream_t s) {
  const int P = c->nranks, r = c->rank;
  std::vector<uint64_t> rg(2 * P);
  chunk_ranges(n, block, P, rg.data());
  uint64_t maxlen = 0;
  for (int q = 0; q < P; ++q) maxlen = std::max(maxlen, rg[2 * q + 1] - rg[2 * q]);
  // receive slots sized for this call's chunk and block size
  const uint64_t cap = round_up(maxlen ? maxlen : 1, 256);
  const uint64_t scap = round_up((cap + block - 1) / block, 64);
  if (!c->recv_codes || c->recv_chunk_cap < cap || c->recv_scale_cap < scap) {
    if (c->recv_codes) cudaFree(c->recv_codes);
    if (c->recv_scales) cudaFree(c->recv_scales);
    c->recv_codes = nullptr;
    c->recv_scales = nullptr;
    c->recv_chunk_cap = c->recv_scale_cap = 0;
    const uint64_t slots = P > 1 ? P - 1 : 1;
    cudaError_t e = cudaMalloc(&c->recv_codes, slots * cap);
    if (e == cudaSuccess) e = cudaMalloc(&c->recv_scales, slots * scap * 4);
    if (e != cudaSuccess) return cuda_fail(e, "allreduce: workspace");
    c->recv_chunk_cap = cap;
    c->recv_scale_cap = scap;
  }
  const uint64_t ccap = c->recv_chunk_cap, sccap = c->recv_scale_cap;
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
      c->trace.push_back(chunk_event(0, r, q, bq, lq, block));
    }
    if (lr) {
      nccl().Recv(c->recv_codes + slot(q) * ccap, lr, ncclUint8, q, c->nccl, s);
      nccl().Recv(c->recv_scales + slot(q) * sccap, nbr, ncclFloat32, q, c->nccl, s);
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
        pc[q] = c->recv_codes + slot(q) * ccap;
        ps[q] = c->recv_scales + slot(q) * sccap;
      }
    }
    uint8_t* oc = codes + br;
    float* os = scales + br / block;
    st = reduce_requant_device(P, pc.data(), ps.data(), lr, block, 1, &oc, &os,
                               (long long)(br / block), err, s);
    if (st) return st;
  }
  // every rank raises the same error (collective.hpp:158-168, :278-281)
  st = share_errors(c, err, s);
  if (st) return st;
  // 3) all-gather: reduced chunk r -> every rank, received in place
  st = nccl_fail(nccl().GroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    const uint64_t bq = rg[2 * q], lq = rg[2 * q + 1] - bq;
    if (lr) {
      nccl().Send(codes + br, lr, ncclUint8, q, c->nccl, s);
      nccl().Send(scales + br / block, nbr, ncclFloat32, q, c->nccl, s);
      c->trace.push_back(chunk_event(1, r, q, br, lr, block));
    }
    if (lq) {
      nccl().Recv(codes + bq, lq, ncclUint8, q, c->nccl, s);
      nccl().Recv(scales + bq / block, (lq + block - 1) / block, ncclFloat32, q, c->nccl, s);
    }
  }
  return nccl_fail(nccl().GroupEnd(), "all-gather");
}

// Fused kernel grid: 2 co-resident CTAs per SM (256 threads, small smem).
constexpr int kP2PCtasPerSm = 2;

template <int NP>
void launch_fused(const FusedArgs& a, int grid, cudaStream_t s) {
  k_fused_allreduce<NP><<<grid, 256, 0, s>>>(a);
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
  a.epoch_ctr = c->epoch_ctr;
  a.timeout_ns = c->timeout_ns;
  a.done_counter = c->done_counter;
  a.stats = c->stats;
  a.err = err;
  a.rank = r;
  a.P = P;
  // trace: rank r pulls chunk r from every peer (sender s -> receiver r) and
  // pushes the reduced chunk r to every peer (sender r -> receiver s)
  for (int q = 0; q < P; ++q)
    if (q != r && a.len) c->trace.push_back(chunk_event(0, q, r, a.begin, a.len, block));
  for (int q = 0; q < P; ++q)
    if (q != r && a.len) c->trace.push_back(chunk_event(1, r, q, a.begin, a.len, block));
  const uint64_t groups = (a.len + kBlock - 1) / kBlock * 8;
  uint64_t grid = (groups + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * kP2PCtasPerSm;
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
  const int P = c->nranks, r = c->rank;
  if (P > 8) return set_error(AGQ_ERR_INVALID_ARGUMENT, "push all-reduce: world size 2..8");
  const SymLayout L = sym_layout(c->sym_cap, c->nranks);
  uint8_t* sc_codes = c->sym + L.codes_off;
  float* sc_scales = reinterpret_cast<float*>(c->sym + L.scales_off);
  const uint64_t nb = (n + block - 1) / block;
  const bool inplace = codes == sc_codes && scales == sc_scales;
  if (!inplace) {
    cudaMemcpyAsync(sc_codes, codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(sc_scales, scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
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
  a.epoch_ctr = c->epoch_ctr;
  a.timeout_ns = c->timeout_ns;
  a.done_counter = c->done_counter;
  a.stats = c->stats;
  a.err = err;
  a.rank = r;
  a.P = P;
  uint64_t maxlen = 0;
  for (int q = 0; q < P; ++q) maxlen = std::max<uint64_t>(maxlen, rg[2 * q + 1] - rg[2 * q]);
  const uint64_t begin = rg[2 * r], len = rg[2 * r + 1] - begin;
  for (int q = 0; q < P; ++q) {
    const uint64_t lq = rg[2 * q + 1] - rg[2 * q];
    if (q != r && lq) c->trace.push_back(chunk_event(0, r, q, rg[2 * q], lq, block));
  }
  for (int q = 0; q < P; ++q)
    if (q != r && len) c->trace.push_back(chunk_event(1, r, q, begin, len, block));
  // scatter: ~2 CTAs per SM in total across the P-1 peers
  uint64_t gx = (maxlen / 16 + 1023) / 1024;
  const uint64_t cap_x = std::max<uint64_t>(1, (uint64_t)num_sms() * 2 / (P - 1));
  gx = std::min<uint64_t>(std::max<uint64_t>(gx, 1), cap_x);
  k_push_scatter<<<dim3((unsigned)gx, (unsigned)(P - 1)), 256, 0, s>>>(a);
  count_launch();
  agq_status st = cuda_fail(cudaGetLastError(), "push all-reduce: scatter launch");
  if (st) return st;
  PieceTable pt{};
  pt.np = P;
  pt.nout = P;
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
  const uint64_t groups = (len + kBlock - 1) / kBlock * 8;
  uint64_t grid = (groups + 255) / 256;
  grid = std::min<uint64_t>(std::max<uint64_t>(grid, 1), (uint64_t)num_sms() * 2);
  // the scatter kernel reset the CTA counter; the reduce kernel reuses it
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
  if (!inplace) {
    cudaMemcpyAsync(codes, sc_codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(scales, sc_scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  return AGQ_OK;
}

agq_status allreduce_oneshot(agq_comm* c, uint8_t* codes, float* scales, uint64_t n,
                             uint32_t block, agq_errors* err, cudaStream_t s) {
  if (!c->p2p_ready) return set_error(AGQ_ERR_INVALID_ARGUMENT, "p2p buffers not opened");
  if (block != (uint32_t)kBlock) return set_error(AGQ_ERR_INVALID_ARGUMENT, "one-shot all-reduce needs block 128");
  if (!err) return set_error(AGQ_ERR_INVALID_ARGUMENT, "one-shot all-reduce needs an error record");
  const int P = c->nranks, r = c->rank;
  if (P > 8) return set_error(AGQ_ERR_INVALID_ARGUMENT, "one-shot all-reduce: world size 1..8");
  const SymLayout L = sym_layout(c->sym_cap, P);
  if (n > L.ll_cap)
    return set_error(AGQ_ERR_INVALID_ARGUMENT, "one-shot all-reduce: more than its inbox (1 Mi elements)");
  uint8_t* sc_codes = c->sym + L.codes_off;
  float* sc_scales = reinterpret_cast<float*>(c->sym + L.scales_off);
  const uint64_t nb = (n + block - 1) / block;
  const bool inplace = codes == sc_codes && scales == sc_scales;
  if (!inplace) {
    cudaMemcpyAsync(sc_codes, codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(sc_scales, scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  OneShotArgs a{};
  for (int q = 0; q < P; ++q) a.base[q] = c->peer[q];
  a.scales_off = L.scales_off;
  a.codes_off = L.codes_off;
  a.os_off = L.ll_off;
  a.n = n;
  a.epoch_ctr = c->epoch_ctr;
  a.timeout_ns = c->timeout_ns;
  a.done_counter = c->done_counter;
  a.stats = c->stats;
  a.err = err;
  a.rank = r;
  a.P = P;
  OneShotLL ll{L.ll_slot_bytes, L.ll_codes_bytes};
  PieceTable out{};
  out.np = P;
  out.nout = 1;
  out.out_codes[0] = c->peer[r] + L.codes_off;
  out.out_scales[0] = reinterpret_cast<float*>(c->peer[r] + L.scales_off);
  // trace: the whole tensor from this rank to every peer
  for (int q = 0; q < P; ++q)
    if (q != r) c->trace.push_back(chunk_event(0, r, q, 0, n, block));
  uint64_t grid = ((n + 15) / 16 + 255) / 256;
  grid = std::min<uint64_t>(std::max<uint64_t>(grid, 1), (uint64_t)num_sms() * 2);
  switch (P) {
    case 1: k_oneshot_ll<1><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 2: k_oneshot_ll<2><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 3: k_oneshot_ll<3><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 4: k_oneshot_ll<4><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 5: k_oneshot_ll<5><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 6: k_oneshot_ll<6><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    case 7: k_oneshot_ll<7><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
    default: k_oneshot_ll<8><<<(int)grid, 256, 0, s>>>(a, ll, out); break;
  }
  count_launch();
  if (agq_status st = cuda_fail(cudaGetLastError(), "one-shot all-reduce: launch")) return st;
  if (!inplace) {
    cudaMemcpyAsync(codes, sc_codes, n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(scales, sc_scales, nb * 4, cudaMemcpyDeviceToDevice, s);
  }
  return AGQ_OK;
}

}  // namespace

agq_status allreduce_fp8(agq_comm* c, uint8_t* codes, float* scales, uint64_t n, uint32_t block,
                         int algo, agq_errors* err, cudaStream_t s) {
  c->trace.clear();
  c->trace_algo = algo;
  c->trace_stream = s;
  if (n == 0) return AGQ_OK;
  if (c->nranks == 1 && algo == AGQ_AR_NCCL) {
    // P = 1: the reference still re-quantizes acc = 0 + dequant (signed
    // zeros normalise), so run the reduce with one piece. No messages.
    const uint8_t* pc = codes;
    const float* ps = scales;
    return reduce_requant_device(1, &pc, &ps, n, block, 1, &codes, &scales, 0, err, s);
  }
  if (algo == AGQ_AR_ONESHOT_P2P) return allreduce_oneshot(c, codes, scales, n, block, err, s);
  if (algo == AGQ_AR_FUSED_P2P || algo == AGQ_AR_PUSH_P2P) {
    // one rank: the fused kernel (barriers and reduce with itself); the
    // push algorithm has no peer to scatter to
    return algo == AGQ_AR_FUSED_P2P || c->nranks == 1
               ? allreduce_p2p(c, codes, scales, n, block, err, s)
               : allreduce_push(c, codes, scales, n, block, err, s);
  }
  if (!c->nccl) return set_error(AGQ_ERR_INVALID_ARGUMENT, "communicator has no NCCL (P2P only)");
  return allreduce_nccl(c, codes, scales, n, block, err, s);
}

#ifdef AGQ_AR_PROFILE
agq_status ar_profile(unsigned long long* out) {
  cudaDeviceSynchronize();
  return cuda_fail(cudaMemcpyFromSymbol(out, g_ar_prof, sizeof(g_ar_prof)), "ar_profile");
}
#endif

agq_status comm_last_trace(agq_comm* c, agq_trace_event* events, int cap, int* count,
                           unsigned long long* moved) {
  *count = (int)c->trace.size();
  for (int i = 0; i < (int)c->trace.size() && i < cap; ++i) events[i] = c->trace[i];
  if (moved) {
    moved[0] = moved[1] = 0;
    if (c->trace_algo == AGQ_AR_FUSED_P2P || c->trace_algo == AGQ_AR_PUSH_P2P ||
        c->trace_algo == AGQ_AR_ONESHOT_P2P) {
      // kernel-side counters of the last P2P call (elements, blocks)
      if (c->trace_stream) cudaStreamSynchronize(c->trace_stream);
      uint64_t ep = 0;  // the last completed epoch: its counters
      cudaError_t e = cudaMemcpy(&ep, c->epoch_ctr, sizeof ep, cudaMemcpyDeviceToHost);
      if (e == cudaSuccess)
        e = cudaMemcpy(moved, c->stats + 2 * (ep & 1), 2 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e, "last_trace: counters");
    }
  }
  return AGQ_OK;
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
  if (!c->nccl) return set_error(AGQ_ERR_INVALID_ARGUMENT, "communicator has no NCCL (P2P only)");
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
  if (!c->nccl) return set_error(AGQ_ERR_INVALID_ARGUMENT, "communicator has no NCCL (P2P only)");
  return nccl_fail(nccl().AllReduce(data, data, n, ncclBfloat16, ncclSum, c->nccl, s),
                   "ncclAllReduce(bf16)");
}

}  // namespace agqh
