// Probe: how fast can a B200 stream a 40 MB fp32 tensor (c2: 10 blocks of
// 100^3) from HBM (L2 flushed before every launch) while doing R = 10 fp64
// FMAs per element, with different load strategies.  Column-accumulate shape
// of the T pass: out[r][j] = sum_i2 X[j + J i2] a[i2][r].
//   A: LDG.64 pairs, register prefetch PD rows, warp tasks of 64 j
//   B: CTA-wide bulk-copy ring (one 1-D copy per row of JT elements)
//   C: pure read (sum) with LDG.128, grid-stride: the bandwidth ceiling
#include <cstdio>
#include <cstdint>
#include <vector>
#include "tma.cuh"
using namespace cb;

constexpr int R = 10;
constexpr long long S = 10, I0 = 100, I1 = 100, I2 = 100, J = I0 * I1;

__global__ void flush_k(float* f, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += gridDim.x * 256LL) f[i] += 1.f;
}

template <int PD>
__global__ void __launch_bounds__(256, 2) kA(const float* X, const double* A, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntask = S * (J / 64);
  for (long long t = blockIdx.x * 8LL + warp; t < ntask; t += gridDim.x * 8LL) {
    const long long s = t / (J / 64), j0 = (t % (J / 64)) * 64;
    const float* xs = X + s * J * I2 + j0 + 2 * lane;
    double a0[R], a1[R];
    for (int r = 0; r < R; ++r) { a0[r] = 0; a1[r] = 0; }
    float2 xb[PD];
#pragma unroll
    for (int p = 0; p < PD; ++p) xb[p] = __ldg(reinterpret_cast<const float2*>(xs + J * p));
    for (int i2 = 0; i2 < I2; i2 += PD) {
#pragma unroll
      for (int p = 0; p < PD; ++p) {
        if (i2 + p < I2) {
          const double x0 = xb[p].x, x1 = xb[p].y;
          if (i2 + p + PD < I2) xb[p] = __ldg(reinterpret_cast<const float2*>(xs + J * (i2 + p + PD)));
          const double* ar = A + (i2 + p) * R;
#pragma unroll
          for (int r = 0; r < R; ++r) { const double av = __ldg(ar + r); a0[r] = fma(x0, av, a0[r]); a1[r] = fma(x1, av, a1[r]); }
        }
      }
    }
    double v = 0;
    for (int r = 0; r < R; ++r) v += a0[r] + a1[r];
    out[t * 32 + lane] = v;
  }
}

// B: CTA of 256 threads, tile JT = 256*TJ columns, ring NST stages x CH rows
template <int TJ, int CH, int NST, bool FMA>
__global__ void __launch_bounds__(256, 1) kB(const float* X, const double* A, double* out) {
  constexpr int JT = 256 * TJ;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float* ring = reinterpret_cast<float*>(sm + 128);
  const long long ntile = S * ((J + JT - 1) / JT);
  if (threadIdx.x == 0) { for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1); mbar_fence_init(); }
  __syncthreads();
  uint32_t ph = 0;
  for (long long t = blockIdx.x; t < ntile; t += gridDim.x) {
    const long long tpb = (J + JT - 1) / JT;
    const long long s = t / tpb, j0 = (t % tpb) * JT;
    const int jl = (int)(J - j0 < JT ? J - j0 : JT);
    const float* xs = X + s * J * I2 + j0;
    const int nst = (int)((I2 + CH - 1) / CH);
    auto issue = [&](int k) {
      const int q = k % NST;
      const int r0 = k * CH, nr = (int)(I2 - r0 < CH ? I2 - r0 : CH);
      mbar_arrive_expect_tx(&bar[q], nr * jl * 4);
      for (int rr = 0; rr < nr; ++rr) bulk_g2s(ring + ((size_t)q * CH + rr) * JT, xs + J * (r0 + rr), jl * 4, &bar[q]);
    };
    if (threadIdx.x == 0) for (int k = 0; k < nst && k < NST; ++k) issue(k);
    double acc[TJ][R];
    for (int a = 0; a < TJ; ++a) for (int r = 0; r < R; ++r) acc[a][r] = 0;
    for (int k = 0; k < nst; ++k) {
      const int q = k % NST;
      mbar_wait(&bar[q], (ph >> q) & 1u);
      ph ^= 1u << q;
      const int r0 = k * CH, nr = (int)(I2 - r0 < CH ? I2 - r0 : CH);
      for (int rr = 0; rr < nr; ++rr) {
        const float* xr = ring + ((size_t)q * CH + rr) * JT;
        if (FMA) {
          const double* ar = A + (r0 + rr) * R;
          double av[R];
#pragma unroll
          for (int r = 0; r < R; ++r) av[r] = __ldg(ar + r);
#pragma unroll
          for (int a = 0; a < TJ; ++a) {
            const double x = xr[threadIdx.x + a * 256];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[a][r] = fma(x, av[r], acc[a][r]);
          }
        } else {
#pragma unroll
          for (int a = 0; a < TJ; ++a) acc[a][0] += xr[threadIdx.x + a * 256];
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && k + NST < nst) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(k + NST); }
    }
    double v = 0;
    for (int a = 0; a < TJ; ++a) for (int r = 0; r < R; ++r) v += acc[a][r];
    out[t * 256 + threadIdx.x] = v;
  }
}


template <int TJ, int CH, int NST, int MODE>
__global__ void __launch_bounds__(256, 1) kD(const float* X, const double* A, double* out) {
  constexpr int JT = 256 * TJ;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  double* As = reinterpret_cast<double*>(sm + 128);            // I2 x 10 (padded to 10)
  float* ring = reinterpret_cast<float*>(sm + 128 + I2 * R * 8);
  for (int e = threadIdx.x; e < I2 * R; e += 256) As[e] = A[e];
  const long long ntile = S * ((J + JT - 1) / JT);
  if (threadIdx.x == 0) { for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1); mbar_fence_init(); }
  __syncthreads();
  uint32_t ph = 0;
  for (long long t = blockIdx.x; t < ntile; t += gridDim.x) {
    const long long tpb = (J + JT - 1) / JT;
    const long long s = t / tpb, j0 = (t % tpb) * JT;
    const int jl = (int)(J - j0 < JT ? J - j0 : JT);
    const float* xs = X + s * J * I2 + j0;
    const int nst = (int)((I2 + CH - 1) / CH);
    auto issue = [&](int k) {
      const int q = k % NST;
      const int r0 = k * CH, nr = (int)(I2 - r0 < CH ? I2 - r0 : CH);
      mbar_arrive_expect_tx(&bar[q], nr * jl * 4);
      for (int rr = 0; rr < nr; ++rr) bulk_g2s(ring + ((size_t)q * CH + rr) * JT, xs + J * (r0 + rr), jl * 4, &bar[q]);
    };
    if (threadIdx.x == 0) for (int k = 0; k < nst && k < NST; ++k) issue(k);
    double acc[TJ][R];
    float accf[TJ][R];
    for (int a = 0; a < TJ; ++a) for (int r = 0; r < R; ++r) { acc[a][r] = 0; accf[a][r] = 0; }
    for (int k = 0; k < nst; ++k) {
      const int q = k % NST;
      mbar_wait(&bar[q], (ph >> q) & 1u);
      ph ^= 1u << q;
      const int r0 = k * CH, nr = (int)(I2 - r0 < CH ? I2 - r0 : CH);
#pragma unroll 2
      for (int rr = 0; rr < nr; ++rr) {
        const float* xr = ring + ((size_t)q * CH + rr) * JT;
        const double2* ar = reinterpret_cast<const double2*>(As + (r0 + rr) * R);
        double av[R];
#pragma unroll
        for (int r = 0; r < R / 2; ++r) { const double2 v = ar[r]; av[2 * r] = v.x; av[2 * r + 1] = v.y; }
#pragma unroll
        for (int a = 0; a < TJ; ++a) {
          if (MODE == 2) {
            const float x = xr[threadIdx.x + a * 256];
#pragma unroll
            for (int r = 0; r < R; ++r) accf[a][r] = fmaf(x, (float)av[r], accf[a][r]);
          } else {
            const double x = MODE == 1 ? 1.0000001 : (double)xr[threadIdx.x + a * 256];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[a][r] = fma(x, av[r], acc[a][r]);
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && k + NST < nst) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(k + NST); }
    }
    double v = 0;
    for (int a = 0; a < TJ; ++a) for (int r = 0; r < R; ++r) v += acc[a][r] + accf[a][r];
    out[t * 256 + threadIdx.x] = v;
  }
}

__global__ void kC(const float4* X, long long n4, double* out) {
  double v = 0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += gridDim.x * 256LL) {
    const float4 x = __ldg(X + i);
    v += x.x + x.y + x.z + x.w;
  }
  out[blockIdx.x * 256 + threadIdx.x] = v;
}

int main() {
  const long long n = S * J * I2;
  float* X; double* A; double* out; float* fl;
  cudaMalloc(&X, n * 4); cudaMalloc(&A, I2 * R * 8); cudaMalloc(&out, 64 << 20);
  const long long nfl = 64LL << 20;
  cudaMalloc(&fl, nfl * 4);
  cudaMemset(X, 0, n * 4); cudaMemset(A, 0, I2 * R * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9, tot = 0;
    for (int it = 0; it < 8; ++it) {
      flush_k<<<592, 256>>>(fl, nfl);
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = ms < best ? ms : best; tot += ms; }
    }
    printf("%-40s best %7.2f us  avg %7.2f us  (%6.0f GB/s)  %s\n", name, best * 1e3, tot / 6 * 1e3,
           n * 4 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("C: pure read LDG.128 grid 148*8", [&] { kC<<<148 * 8, 256>>>((const float4*)X, n / 4, out); });
  timeit("C: pure read LDG.128 grid 148*32", [&] { kC<<<148 * 32, 256>>>((const float4*)X, n / 4, out); });
  timeit("A: LDG pairs PD=4", [&] { kA<4><<<296, 256>>>(X, A, out); });
  timeit("A: LDG pairs PD=8", [&] { kA<8><<<296, 256>>>(X, A, out); });
  timeit("A: LDG pairs PD=16", [&] { kA<16><<<296, 256>>>(X, A, out); });
  {
    auto k = kB<4, 4, 4, true>; size_t sm = 128 + 4 * 4 * 1024 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ4 CH4 NST4 fma (fiber2-like)", [&] { k<<<148, 256, sm>>>(X, A, out); });
    auto kr = kB<4, 4, 4, false>;
    cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ4 CH4 NST4 read-only", [&] { kr<<<148, 256, sm>>>(X, A, out); });
  }
  {
    auto k = kB<2, 8, 4, true>; size_t sm = 128 + 4 * 8 * 512 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ2 CH8 NST4 fma", [&] { k<<<148, 256, sm>>>(X, A, out); });
    auto kr = kB<2, 8, 4, false>;
    cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ2 CH8 NST4 read-only", [&] { kr<<<148, 256, sm>>>(X, A, out); });
  }
  {
    auto k = kB<1, 16, 4, true>; size_t sm = 128 + 4 * 16 * 256 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ1 CH16 NST4 fma (2 CTA/SM)", [&] { k<<<296, 256, sm>>>(X, A, out); });
    auto kr = kB<1, 16, 4, false>;
    cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("B: TJ1 CH16 NST4 read-only (2 CTA/SM)", [&] { kr<<<296, 256, sm>>>(X, A, out); });
  }

  {
    size_t sm = 128 + I2 * R * 8 + 4 * 4 * 1024 * 4;
    auto k0 = kD<4, 4, 4, 0>, k1 = kD<4, 4, 4, 1>, k2 = kD<4, 4, 4, 2>;
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    timeit("D: TJ4 A in smem, fp64 fma", [&] { k0<<<148, 256, sm>>>(X, A, out); });
    timeit("D: TJ4 A in smem, fp64 fma const x", [&] { k1<<<148, 256, sm>>>(X, A, out); });
    timeit("D: TJ4 A in smem, fp32 fma", [&] { k2<<<148, 256, sm>>>(X, A, out); });
    size_t sm2 = 128 + I2 * R * 8 + 4 * 8 * 512 * 4;
    auto k3 = kD<2, 8, 4, 0>;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    timeit("D: TJ2 CH8 A in smem fp64 (2 CTA/SM)", [&] { k3<<<296, 256, sm2>>>(X, A, out); });
    auto k4 = kD<2, 8, 4, 0>;
    timeit("D: TJ2 CH8 A in smem fp64 (3 CTA/SM)", [&] { k4<<<444, 256, sm2>>>(X, A, out); });
  }
  return 0;
}
