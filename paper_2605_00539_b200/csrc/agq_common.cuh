// Shared definitions of the AGoQ sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/agq_cuda.h"
#include "agq_numerics.cuh"
#include "agq_ptx.cuh"

namespace agqk {

constexpr int kBlock = 128;          // block size of every fast path
constexpr int kTileBlocks = 64;      // blocks per tile
constexpr int kTileElems = kTileBlocks * kBlock;  // 8192 elements
constexpr int kThreads = 256;        // 32 consecutive elements per thread
// Segments per grouped launch; larger groups are split into launches of 8
// (a 32-entry table measured 3-4% slower kernels: C1 round trip 19.9 vs 18.7
// us, profiles/r02_ab_segtable.log).
#ifndef AGQ_MAX_SEG
#define AGQ_MAX_SEG 8
#endif
constexpr int kMaxSeg = AGQ_MAX_SEG;
constexpr long long kNone = 0x7fffffffffffffffLL;

// A list of equally-coded tensors processed by one launch (grouped launch of
// the tensors one pipeline stage stores).
// tile_begin is a prefix sum over whole warp tiles; block_base the
// group-global index of each segment's first block (error reporting).
struct SegTable {
  const void* src[kMaxSeg];
  void* codes[kMaxSeg];
  float* scales[kMaxSeg];
  void* dst[kMaxSeg];
  uint64_t tile_begin[kMaxSeg + 1];
  uint64_t block_base[kMaxSeg];
  int nseg;
};

__device__ __forceinline__ int seg_of(const SegTable& st, uint64_t t) {
  int s = 0;
#pragma unroll
  for (int j = 1; j < kMaxSeg; ++j)
    if (j < st.nseg && t >= st.tile_begin[j]) s = j;
  return s;
}

__device__ __forceinline__ void err_min(long long* field, long long v) {
  if (field) atomicMin(field, v);
}

// OR a value of at most 64 significant bits into a little-endian word array
// at compile-time bit offset OFF.
template <int OFF, int NW>
__device__ __forceinline__ void or_bits(uint32_t (&acc)[NW], uint64_t v) {
  constexpr int w = OFF / 32, sh = OFF % 32;
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  if constexpr (sh == 0) {
    acc[w] |= lo;
    if constexpr (w + 1 < NW) acc[w + 1] |= hi;
  } else {
    acc[w] |= lo << sh;
    if constexpr (w + 1 < NW) acc[w + 1] |= (lo >> (32 - sh)) | (hi << sh);
    if constexpr (w + 2 < NW) acc[w + 2] |= hi >> (32 - sh);
  }
}

// Extract bits [OFF, OFF + NB) (NB <= 64) of a little-endian word array.
template <int OFF, int NB, int NW>
__device__ __forceinline__ uint64_t get_bits(const uint32_t (&acc)[NW]) {
  constexpr int w = OFF / 32, sh = OFF % 32;
  uint64_t v = acc[w] >> sh;
  if constexpr (w + 1 < NW) v |= (uint64_t)acc[w + 1] << (32 - sh);
  if constexpr (sh > 0 && w + 2 < NW) v |= (uint64_t)acc[w + 2] << (64 - sh);
  if constexpr (NB < 64) v &= ((uint64_t)1 << NB) - 1;
  return v;
}

// Exact FP8 E4M3 unit values fl64(e4m3(c) / 448) (quantize.hpp:151-153) for
// the positive codes, built per CTA in shared memory with the reference's own
// double division (IEEE, correctly rounded on device as on host).
__device__ __forceinline__ void fill_fp8_unit_lut(double* lut) {
  for (int c = threadIdx.x; c < 128; c += blockDim.x)
    lut[c] = (c == 0x7f) ? __longlong_as_double(0x7ff8000000000000LL)
                         : (double)e4m3_value((uint32_t)c) / 448.0;
}

}  // namespace agqk

// Host-side launch accounting and helpers shared by the .cu files.
namespace agqh {
void count_launch();
int num_sms();
agq_status cuda_fail(cudaError_t e, const char* what);
agq_status set_error(agq_status st, const char* msg);
}  // namespace agqh
