// Probe: cycles and squaring passes of block_lam_max on one gram-product
// matrix (standalone; build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -I paper_2302_05119_b200/csrc tools/micro/lammax_probe.cu -o /tmp/lammax_probe).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "common.cuh"
using namespace cb;

__global__ void probe(const double* g, int R, double* out, long long* cyc) {
  extern __shared__ double sm[];
  const int ld = lm_ld(R);
  const int Rp = (R + 3) & ~3;
  double* A = sm;
  double* B = A + Rp * ld;
  double* B2 = B + lm_bsize(R);
  double* vec = B2 + lm_bsize(R);
  double* red = vec + 128;
  for (int e = threadIdx.x; e < Rp * ld; e += blockDim.x) {
    int i = e / ld, j = e - i * ld;
    A[e] = (i < R && j < R) ? g[i * R + j] : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
  double v = block_lam_max(A, R, B, B2, vec, red);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = v; cyc[blockIdx.x] = t1 - t0; }
}

int main() {
  for (int R : {5, 10, 16, 30, 40, 64}) {
    std::vector<double> a((R + 3) * R), gm(R * R);
    srand(R);
    for (auto& x : a) x = rand() / (double)RAND_MAX;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        double s = 0;
        for (int k = 0; k < R + 3; ++k) s += a[k * R + i] * a[k * R + j];
        gm[i * R + j] = s;
      }
    double *dg, *dout; long long* dc;
    cudaMalloc(&dg, sizeof(double) * R * R); cudaMalloc(&dout, 8); cudaMalloc(&dc, 8);
    cudaMemcpy(dg, gm.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice);
    size_t smem = sizeof(double) * lm_smem_doubles(R);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 3; ++w) probe<<<1, 256, smem>>>(dg, R, dout, dc);
    cudaDeviceSynchronize();

    probe<<<1, 256, smem>>>(dg, R, dout, dc);
    cudaDeviceSynchronize();
    int passes = 0;
    double v; long long c;
    cudaMemcpy(&v, dout, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("R=%2d lambda=%.15e cycles=%lld passes=%d (%s)\n", R, v, c, passes, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
