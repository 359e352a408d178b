// Cycles per tcgen05.mma.kind::i8 (M = 128, K = 32) as a function of N, with A
// from shared memory or TMEM: one CTA per SM issues `reps` back-to-back MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2302_05119_b200/csrc imma_probe.cu -o imma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace cb;

__global__ void __launch_bounds__(128, 1) k(int N, int a_tmem, int reps, int nmma, int ndist, long long* out) {
  extern __shared__ unsigned char raw[];
  const uint32_t r32 = smem_u32(raw);
  unsigned char* sm = raw + (((r32 + 1023u) & ~1023u) - r32);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t base = smem_u32(sm);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int j = 0; j < nmma; ++j) {
        const uint64_t B = sdesc_k_sw32(base + 16384 + (r & 3) * 8192);
        const uint32_t dcol = tmem + (uint32_t)((j % ndist) * N);
        if (a_tmem) mma_i8_ts(dcol, tmem + 480 + 8 * (j & 1), B, idesc, 1u);
        else mma_i8_ss(dcol, sdesc_k_sw32(base + (j & 3) * 4096), B, idesc, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 2000;
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int ndist : {1, 2, 3})
    for (int N : {16, 48, 96, 144, 256}) {
      if (ndist * N > 480) continue;
      const int nmma = 6;
      k<<<148, 128, 100 * 1024>>>(N, a_tmem, reps, nmma, ndist, d);
      cudaDeviceSynchronize();
      long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("A from %s  N %3d, %d independent accumulators: %.1f clk per MMA (M=128, K=32, i8)  %s\n", a_tmem ? "TMEM" : "smem", N, ndist, (double)h / reps / nmma,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
