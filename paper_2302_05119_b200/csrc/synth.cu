// Seeded synthetic blocks generated on the device.
//
// Reference: the ground-truth generator `generate` (pkg/src/concpd/synth.py:77-112)
// builds X_s = [[lam; A_0, ..., A_{N-1}]] from seeded factors and corrupts it
// with `add_noise` (pkg/src/concpd/metrics.py:207-223: additive Gaussian noise
// of power mean(X^2) / 10^(SNR/10), clipped at 0).  The BASELINE configs add
// two variants (configs.py): the block scaled by 1/max and clipped to [0, 1]
// (c3) and multiplicative log-normal noise X exp(sigma Z) (c4).
//
// The factors are drawn on the host by numpy from the reference's SeedSequence
// children (bit-identical to the host generator); only the O(|M| R) part runs
// here: the reconstruction (fp64 arithmetic) and the noise.  Gaussian draws
// come from a counter-based Philox4x32-10 stream keyed by (seed, block) with
// the element index as counter, so a block is the same whatever the launch
// shape or the order blocks are generated in.  The noise realisation is NOT
// numpy's (a sequential PCG64 ziggurat stream cannot be split): device blocks
// feed throughput runs; parity runs keep the host generator.
//
// Layout: X first-index-fastest, X[i0 + I0 j] with j the flattened index of
// modes 1..N-1 (mode 1 fastest).  A CTA owns SYN_COLS consecutive columns j
// and SYN_THREADS consecutive rows i0: the column weights
// w[j][r] = lam_r prod_{n>=1} A_n[i_n(j), r] are staged in shared memory, a
// thread keeps its A_0 row in registers, and x = sum_r A_0[i0, r] w[j][r] is
// one fp64 FMA chain per element (a broadcast shared load per FMA).  Stores of
// a column are coalesced over i0.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"

namespace cb {

constexpr int SYN_THREADS = 256;
constexpr int SYN_COLS = 32;

struct SynthArgs {
  const double* A[CB_MAX_ORDER];
  const double* lam;          // may be null: unit weights
  int64_t dims[CB_MAX_ORDER];
  int order, R;
  int64_t J;                  // prod of dims[1..]
  // fill pass
  void* out;
  int dtype;
  int noise;                  // 0 none, 1 add + clip >= 0, 2 add + clip [0, 1], 3 x exp(sigma z)
  double scale, sigma;
  uint32_t key0, key1, blk;
  // stats pass: per-CTA partials {sum x^2, max x}; residual pass: the
  // tensor X (dtype) and partials {sum (X - x)^2, sum X^2}
  double* part;
  const void* X;
};

// Philox4x32-10 (Salmon et al., SC'11), counter (c0..c3), key (k0, k1)
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// standard normal for element `idx` of block `blk` (Box-Muller, fp64)
__device__ __forceinline__ double normal_at(uint64_t idx, uint32_t blk, uint32_t k0, uint32_t k1) {
  const uint4 v = philox4x32(make_uint4((uint32_t)idx, (uint32_t)(idx >> 32), blk, 0x5EEDu), k0, k1);
  // 53-bit uniforms, u1 in (0, 1]
  const double u1 = ((double)(((uint64_t)v.x << 21) ^ (v.y >> 11)) + 1.0) * 0x1p-53;
  const double u2 = (double)(((uint64_t)v.z << 21) ^ (v.w >> 11)) * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

template <int RB, int PASS>
__global__ void __launch_bounds__(SYN_THREADS) k_synth(SynthArgs a) {
  __shared__ double w[SYN_COLS][RB];
  __shared__ double red[2][SYN_THREADS / 32];
  const int64_t I0 = a.dims[0];
  const int64_t j0 = (int64_t)blockIdx.x * SYN_COLS;
  const int ncol = (int)(a.J - j0 < SYN_COLS ? a.J - j0 : SYN_COLS);
  // column weights (zero past R)
  for (int e = threadIdx.x; e < SYN_COLS * RB; e += SYN_THREADS) {
    const int cj = e / RB, r = e - cj * RB;
    double v = 0.0;
    if (cj < ncol && r < a.R) {
      v = a.lam ? a.lam[r] : 1.0;
      int64_t j = j0 + cj;
      for (int n = 1; n < a.order; ++n) {
        const int64_t in = j % a.dims[n];
        j /= a.dims[n];
        v *= a.A[n][in * a.R + r];
      }
    }
    w[cj][r] = v;
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.y * SYN_THREADS + threadIdx.x;
  double ar[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) ar[r] = (i0 < I0 && r < a.R) ? a.A[0][i0 * a.R + r] : 0.0;
  double ss = 0.0, mx = 0.0;
  if (i0 < I0) {
    for (int cj = 0; cj < ncol; ++cj) {
      double x0 = 0.0, x1 = 0.0;   // two chains (latency), fixed order
#pragma unroll
      for (int r = 0; r < RB; r += 2) {
        x0 = fma(ar[r], w[cj][r], x0);
        if (r + 1 < RB) x1 = fma(ar[r + 1], w[cj][r + 1], x1);
      }
      double x = x0 + x1;
      if (PASS == 0) {
        ss = fma(x, x, ss);
        mx = fmax(mx, x);
      } else if (PASS == 2) {
        const uint64_t idx = (uint64_t)i0 + (uint64_t)I0 * (uint64_t)(j0 + cj);
        const double t = a.dtype == CB_F32 ? (double)static_cast<const float*>(a.X)[idx]
                                           : static_cast<const double*>(a.X)[idx];
        const double d = t - x;
        ss = fma(d, d, ss);
        mx = fma(t, t, mx);
      } else {
        const uint64_t idx = (uint64_t)i0 + (uint64_t)I0 * (uint64_t)(j0 + cj);
        x *= a.scale;
        if (a.noise == 1 || a.noise == 2) {
          x += a.sigma * normal_at(idx, a.blk, a.key0, a.key1);
          x = x < 0.0 ? 0.0 : x;
          if (a.noise == 2) x = x > 1.0 ? 1.0 : x;
        } else if (a.noise == 3) {
          x *= exp(a.sigma * normal_at(idx, a.blk, a.key0, a.key1));
        }
        if (a.dtype == CB_F32) static_cast<float*>(a.out)[idx] = (float)x;
        else static_cast<double*>(a.out)[idx] = x;
      }
    }
  }
  if (PASS != 1) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    ss = warp_sum(ss);
    mx = PASS == 0 ? warp_max(mx) : warp_sum(mx);
    if (lane == 0) { red[0][wid] = ss; red[1][wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0, m = 0.0;
      for (int k = 0; k < SYN_THREADS / 32; ++k) {
        s += red[0][k];
        m = PASS == 0 ? fmax(m, red[1][k]) : m + red[1][k];
      }
      const int64_t p = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      a.part[2 * p] = s;
      a.part[2 * p + 1] = m;
    }
  }
}

// fixed-order fold of the per-CTA partials (one warp, lanes strided, then
// the lanes in order); second component: max (stats) or sum (residual)
__global__ void k_synth_fold(const double* part, int64_t n, double* out2, int second_sum) {
  double s = 0.0, m = 0.0;
  for (int64_t p = threadIdx.x; p < n; p += 32) {
    s += part[2 * p];
    m = second_sum ? m + part[2 * p + 1] : fmax(m, part[2 * p + 1]);
  }
  __shared__ double ls[32], lm[32];
  ls[threadIdx.x] = s;
  lm[threadIdx.x] = m;
  __syncwarp();
  if (threadIdx.x == 0) {
    double t = 0.0, u = 0.0;
    for (int k = 0; k < 32; ++k) { t += ls[k]; u = second_sum ? u + lm[k] : fmax(u, lm[k]); }
    out2[0] = t;
    out2[1] = u;
  }
}

template <int PASS>
static void synth_dispatch(const SynthArgs& a, dim3 grid, cudaStream_t st) {
  if (a.R <= 8) k_synth<8, PASS><<<grid, SYN_THREADS, 0, st>>>(a);
  else if (a.R <= 16) k_synth<16, PASS><<<grid, SYN_THREADS, 0, st>>>(a);
  else if (a.R <= 32) k_synth<32, PASS><<<grid, SYN_THREADS, 0, st>>>(a);
  else if (a.R <= 40) k_synth<40, PASS><<<grid, SYN_THREADS, 0, st>>>(a);
  else k_synth<64, PASS><<<grid, SYN_THREADS, 0, st>>>(a);
}

static int synth_args(SynthArgs& a, int order, const int64_t* dims, const double* const* factors,
                      const double* weights, int rank, dim3& grid) {
  CB_ARG(order >= 1 && order <= CB_MAX_ORDER, "order %d outside [1, %d]", order, CB_MAX_ORDER);
  CB_ARG(rank >= 1 && rank <= CB_MAX_RANK, "rank %d outside [1, %d]", rank, CB_MAX_RANK);
  a.order = order;
  a.R = rank;
  a.lam = weights;
  a.J = 1;
  for (int n = 0; n < order; ++n) {
    CB_ARG(dims[n] >= 1, "dims must be positive");
    a.dims[n] = dims[n];
    a.A[n] = factors[n];
    if (n > 0) a.J *= dims[n];
  }
  const int64_t gx = (a.J + SYN_COLS - 1) / SYN_COLS;
  const int64_t gy = (dims[0] + SYN_THREADS - 1) / SYN_THREADS;
  CB_ARG(gx < (1LL << 31) && gy < 65536, "block too large for the generator grid");
  grid = dim3((unsigned)gx, (unsigned)gy);
  return CB_OK;
}

}  // namespace cb

using namespace cb;

extern "C" {

int cb_synth_stats(int order, const int64_t* dims, const double* const* factors,
                   const double* weights, int rank, double* out2, void* stream) {
  CB_ARG(dims && factors && out2, "null argument");
  SynthArgs a{};
  dim3 grid;
  int rc = synth_args(a, order, dims, factors, weights, rank, grid);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t np = (int64_t)grid.x * grid.y;
  CB_CUDA(cudaMallocAsync((void**)&a.part, sizeof(double) * 2 * np, st));
  synth_dispatch<0>(a, grid, st);
  k_synth_fold<<<1, 32, 0, st>>>(a.part, np, out2, 0);
  count_launch(2);
  CB_CHECK_LAUNCH();
  CB_CUDA(cudaFreeAsync(a.part, st));
  return CB_OK;
}

int cb_synth_fill(int dtype, void* out, int order, const int64_t* dims,
                  const double* const* factors, const double* weights, int rank, double scale,
                  int noise, double sigma, uint64_t seed, int block, void* stream) {
  CB_ARG(out && dims && factors, "null argument");
  CB_ARG(dtype == CB_F32 || dtype == CB_F64, "bad dtype");
  CB_ARG(noise >= 0 && noise <= 3, "noise kind %d outside [0, 3]", noise);
  SynthArgs a{};
  dim3 grid;
  int rc = synth_args(a, order, dims, factors, weights, rank, grid);
  if (rc) return rc;
  a.out = out;
  a.dtype = dtype;
  a.noise = noise;
  a.scale = scale;
  a.sigma = sigma;
  a.key0 = (uint32_t)seed;
  a.key1 = (uint32_t)(seed >> 32);
  a.blk = (uint32_t)block;
  synth_dispatch<1>(a, grid, (cudaStream_t)stream);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

/* out2 = {||X - [[weights; factors]]||^2, ||X||^2} by the generator's tiled
 * reconstruction (no dense model is formed). */
int cb_model_residual(int dtype, const void* X, int order, const int64_t* dims,
                      const double* const* factors, const double* weights, int rank,
                      double* out2, void* stream) {
  CB_ARG(X && dims && factors && out2, "null argument");
  CB_ARG(dtype == CB_F32 || dtype == CB_F64, "bad dtype");
  SynthArgs a{};
  dim3 grid;
  int rc = synth_args(a, order, dims, factors, weights, rank, grid);
  if (rc) return rc;
  a.X = X;
  a.dtype = dtype;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t np = (int64_t)grid.x * grid.y;
  CB_CUDA(cudaMallocAsync((void**)&a.part, sizeof(double) * 2 * np, st));
  synth_dispatch<2>(a, grid, st);
  k_synth_fold<<<1, 32, 0, st>>>(a.part, np, out2, 1);
  count_launch(2);
  CB_CHECK_LAUNCH();
  CB_CUDA(cudaFreeAsync(a.part, st));
  return CB_OK;
}

}  // extern "C"
