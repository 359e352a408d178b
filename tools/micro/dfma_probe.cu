// Probe: fp64 FMA throughput per SM (independent chains, full occupancy).
#include <cstdio>
__global__ void dfma(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 42.0) out[0] = 1.0;
}
__global__ void ffma(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 42.0f) out[0] = 1.0f;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int occ : {1, 2, 4, 8}) {
      dim3 grid(sms * occ);
      dfma<<<grid, 256>>>(d, 100);
      cudaEventRecord(e0);
      dfma<<<grid, 256>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)grid.x * 256 * 8 * iters;
      printf("fp64 occ %d: %.1f TFMA/s = %.1f TFLOP/s\n", occ, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
      ffma<<<grid, 256>>>((float*)d, 100);
      cudaEventRecord(e0);
      ffma<<<grid, 256>>>((float*)d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("fp32 occ %d: %.1f TFMA/s = %.1f TFLOP/s\n", occ, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
    }
  }
  return 0;
}
