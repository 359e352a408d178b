// Probe: cycles of the block-level primitives used by block_lam_max.
#include <cstdio>
#include "common.cuh"
using namespace cb;

__global__ void probe(double* out, long long* cyc) {
  __shared__ double red[40];
  __shared__ double B[16 * 17], B2[16 * 17];
  for (int e = threadIdx.x; e < 16 * 17; e += blockDim.x) B[e] = 1.0 / (1 + e);
  __syncthreads();
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < 100; ++it) acc = block_max(acc, red) * 0.5;
  long long t1 = clock64();
  for (int it = 0; it < 100; ++it) acc += block_sum(acc, red) * 1e-3;
  long long t2 = clock64();
  for (int it = 0; it < 100; ++it) { __syncthreads(); acc += red[it & 31]; }
  long long t3 = clock64();
  for (int it = 0; it < 100; ++it) acc += warp_max(acc);
  long long t4 = clock64();
  for (int it = 0; it < 100; ++it) acc += sq_tiles<1>(B, B2, 10, 11, red) * 1e-9;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = acc;
    cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 100;
    cyc[3] = (t4 - t3) / 100; cyc[4] = (t5 - t4) / 100;
  }
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8); cudaMalloc(&c, 64);
  for (int nt : {32, 128, 256}) {
    for (int w = 0; w < 2; ++w) probe<<<1, nt>>>(d, c);
    cudaDeviceSynchronize();
    long long h[5];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%3d block_max=%lld block_sum=%lld syncthreads=%lld warp_max=%lld sq_tiles(R=10)=%lld cycles\n",
           nt, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
