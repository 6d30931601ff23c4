// NVLink access-pattern probe (single process, all visible GPUs, peer access):
// per-GPU bandwidth of the exchange patterns a decomposed all-reduce can use.
//   pull : every GPU reads its own 1/P slice from every peer (LDG on peer ptrs)
//   push : every GPU writes its 1/P slices to every peer (STG on peer ptrs)
//   both : pull and push at the same time (the fused kernel's traffic)
//   ce   : the same all-to-all with cudaMemcpyPeerAsync (copy engines)
// Reports GB/s per GPU per direction (bytes crossing this GPU's links).
#include <cuda_runtime.h>

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
  for (int mode = 0; mode < 4; ++mode) {
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
                 P, mode == 3 ? "copy engines" : names[mode], grid_mult, slice >> 20, worst,
                 per_dir / (worst * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
