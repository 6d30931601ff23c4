// Throughput probe (ops/clk/SM) of the instructions the gradient path can
// use to reproduce the reference's double arithmetic: DMUL, F2F.F32.F64,
// F2F.F64.F32, FMUL, LDS.64 with random indices.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, const double* tab, int iters) {
  __shared__ double lut[128];
  if (threadIdx.x < 128) lut[threadIdx.x] = tab[threadIdx.x];
  __syncthreads();
  double d[8];
  float f[8];
  unsigned x = threadIdx.x * 2654435761u;
  for (int i = 0; i < 8; ++i) { d[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-7; f[i] = (float)d[i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) d[i] = __dmul_rn(d[i], 1.0000001);
      if (OP == 1) f[i] = __double2float_rn(d[i] + (double)f[i] * 0.0);  // F2F + (DFMA)
      if (OP == 2) f[i] = __fmul_rn(f[i], 1.0000001f);
      if (OP == 3) { x = x * 1664525u + 1013904223u; d[i] += lut[(x >> 9) & 127]; }
      if (OP == 4) f[i] = __double2float_rn(d[i] * (1.0 + it));
      if (OP == 5) d[i] = (double)f[i] + d[i];
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, float* out, double* tab, int sms, double clk_ghz) {
  const int iters = 4096, blocks = sms * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, tab, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(out, tab, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)blocks * threads * iters * 8;
  printf("%-28s %8.2f Gop/s  %6.2f ops/clk/SM (at %.2f GHz)\n", name, ops / ms / 1e6,
         ops / (ms * 1e-3) / sms / (clk_ghz * 1e9), clk_ghz);
}

int main() {
  float* out;
  double* tab;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaMalloc(&tab, 128 * 8);
  cudaMemset(tab, 0, 128 * 8);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double g = clk / 1e6;
  run<0>("DMUL", out, tab, sms, g);
  run<1>("F2F.F32.F64 (+DFMA)", out, tab, sms, g);
  run<4>("DMUL + F2F.F32.F64", out, tab, sms, g);
  run<5>("F2F.F64.F32 + DADD", out, tab, sms, g);
  run<2>("FMUL", out, tab, sms, g);
  run<3>("LDS.64 random + DADD", out, tab, sms, g);
  return 0;
}
