// NVLink access-pattern probe (single process, all visible GPUs, peer access):
// per-GPU bandwidth of the exchange patterns a decomposed all-reduce can use.
//   pull : every GPU reads its own 1/P slice from every peer (LDG on peer ptrs)
//   push : every GPU writes its 1/P slices to every peer (STG on peer ptrs)
//   both : pull and push at the same time (the fused kernel's traffic)
//   ce   : the same all-to-all with cudaMemcpyPeerAsync (copy engines)
// Reports GB/s per GPU per direction (bytes crossing this GPU's links).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

struct Ptrs {
  uint4* buf[8];
};

// mode 0 pull, 1 push, 2 both. Each GPU has `src` (P slices of S bytes) and
// `dst` (P slices). pull: dst_me[s] <- src_s[me]; push: dst_r[me] <- src_me[r].
__global__ void xfer(Ptrs src, Ptrs dst, int me, int P, size_t slice_vec, int mode, int unroll) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  for (int k = 1; k < P; ++k) {
    const int peer = (me + k) % P;
    if (mode == 0 || mode == 2) {  // pull my slice from peer
      const uint4* s = src.buf[peer] + me * slice_vec;
      uint4* d = dst.buf[me] + peer * slice_vec;
      for (size_t i = tid; i < slice_vec; i += nth * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * nth < slice_vec) v[u] = s[i + u * nth];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * nth < slice_vec) d[i + u * nth] = v[u];
      }
    }
    if (mode == 1 || mode == 2) {  // push peer's slice to peer
      const uint4* s = src.buf[me] + peer * slice_vec;
      uint4* d = dst.buf[peer] + (P + me) * slice_vec;  // second half of dst
      for (size_t i = tid; i < slice_vec; i += nth * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * nth < slice_vec) v[u] = s[i + u * nth];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * nth < slice_vec) d[i + u * nth] = v[u];
      }
    }
  }
}

// mode 4: pull with 1-D TMA bulk copies (cp.async.bulk global -> shared, one
// mbarrier per stage, lane 0 of each warp keeps kSt stages of kChunk bytes in
// flight per peer round-robin); the data is then stored to local HBM so the
// traffic pattern matches "pull + local write".
constexpr int kSt = 4, kChunk = 4096;
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__global__ void tma_pull(Ptrs src, Ptrs dst, int me, int P, size_t slice) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  unsigned char* ring = sm + warp * kSt * kChunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + nwarps * kSt * kChunk) + warp * kSt;
  if (lane == 0)
    for (int s = 0; s < kSt; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const size_t per_peer = slice / kChunk;             // chunks per peer slice
  const size_t total = per_peer * (P - 1);
  const size_t gw = (size_t)blockIdx.x * nwarps + warp, nw = (size_t)gridDim.x * nwarps;
  auto addr = [&](size_t c, const unsigned char*& s, unsigned char*& d) {
    const int k = (int)(c % (P - 1)) + 1, peer = (me + k) % P;
    const size_t off = (c / (P - 1)) * kChunk;
    s = reinterpret_cast<const unsigned char*>(src.buf[peer]) + me * slice + off;
    d = reinterpret_cast<unsigned char*>(dst.buf[me]) + peer * slice + off;
  };
  auto issue = [&](size_t c, int st) {
    if (lane == 0 && c < total) {
      const unsigned char* s; unsigned char* d; addr(c, s, d);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[st])), "r"(kChunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(ring + st * kChunk)), "l"(s), "r"(kChunk), "r"(su32(&bars[st])) : "memory");
    }
  };
  size_t c = gw;
  for (int st = 0; st < kSt; ++st) issue(c + st * nw, st);
  uint32_t phase = 0;
  int st = 0;
  for (; c < total; c += nw) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bars[st])), "r"((phase >> st) & 1u) : "memory");
    phase ^= 1u << st;
    const unsigned char* s; unsigned char* d; addr(c, s, d);
    const uint4* r4 = reinterpret_cast<const uint4*>(ring + st * kChunk);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int i = lane; i < kChunk / 16; i += 32) d4[i] = r4[i];
    __syncwarp();
    issue(c + kSt * nw, st);
    st = st + 1 == kSt ? 0 : st + 1;
  }
}

int main(int argc, char** argv) {
  int P = 0;
  CK(cudaGetDeviceCount(&P));
  if (P > 8) P = 8;
  const size_t slice = (argc > 1 ? atoll(argv[1]) : (256ull << 20));  // bytes per slice
  const size_t slice_vec = slice / 16;
  Ptrs src{}, dst{};
  std::vector<cudaStream_t> st(P);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < P; ++h)
      if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src.buf[g], slice * P));
    CK(cudaMalloc(&dst.buf[g], slice * 2 * P));
    CK(cudaMemset(src.buf[g], g, slice * P));
    CK(cudaStreamCreate(&st[g]));
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"pull (peer LDG)", "push (peer STG)", "pull+push"};
  const int tma_warps = 8;
  const size_t tma_smem = tma_warps * (kSt * kChunk + kSt * 8);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(tma_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem));
  }
  for (int mode = 0; mode < 5; ++mode) {
    for (int grid_mult : {1, 2, 4}) {
      if (mode == 3 && grid_mult > 1) break;
      std::vector<cudaEvent_t> a(P), b(P);
      for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < P; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < P; ++g) {
          CK(cudaSetDevice(g));
          cudaEventCreate(&a[g]);
          cudaEventCreate(&b[g]);
          cudaEventRecord(a[g], st[g]);
          if (mode < 3) {
            xfer<<<sms * grid_mult, 512, 0, st[g]>>>(src, dst, g, P, slice_vec, mode, 4);
          } else if (mode == 4) {
            tma_pull<<<sms * grid_mult, tma_warps * 32, tma_smem, st[g]>>>(src, dst, g, P, slice);
          } else {
            for (int k = 1; k < P; ++k) {
              const int peer = (g + k) % P;
              cudaMemcpyPeerAsync((char*)dst.buf[g] + peer * slice, g,
                                  (char*)src.buf[peer] + g * slice, peer, slice, st[g]);
            }
          }
          cudaEventRecord(b[g], st[g]);
        }
        float worst = 0;
        for (int g = 0; g < P; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(b[g]));
          float ms;
          cudaEventElapsedTime(&ms, a[g], b[g]);
          if (ms > worst) worst = ms;
        }
        if (rep == 2) {
          const double per_dir = (mode == 2 ? 2.0 : 1.0) * (P - 1) * (double)slice;
          printf("P=%d %-16s grid=%3dxSM slice=%zuMB: %.3f ms, %.1f GB/s per GPU per direction\n",
                 P, mode == 3 ? "copy engines" : (mode == 4 ? "pull (TMA bulk)" : names[mode]),
                 grid_mult, slice >> 20, worst, per_dir / (worst * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
