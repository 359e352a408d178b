// Post-solve quality metrics on the device.
//
// Reference: pkg/src/concpd/metrics.py:71-156 — rel_err / ten_fit (per-block
// ||M - M^||/||M|| averaged), psnr (10 log10(peak^2 / mse)), and the
// permutation/scale-invariant performance index of a factor matrix
// (G = |pinv(E) T|, row/column max-normalised off-peak mass), averaged per
// mode by pi_per_mode.  The tensor-sized work (c5: 16 GB) streams once; the
// Kruskal-model residual reuses the generator's tiled reconstruction
// (cb_model_residual, synth.cu).
//
// Performance index: pinv(E) T = (E^T E)^{-1} E^T T for a full-column-rank E
// (I_n x R, I_n >= R), formed as two fp64 grams and an LU solve with partial
// pivoting in shared memory, one CTA per (estimate, truth) pair; a pivot test
// flags rank-deficient estimates (the reference warns there and its value is
// "not meaningful", metrics.py:104-110).
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"

namespace cb {

// ---- ||A - B||^2 and ||A||^2 of two dense buffers (fixed-order partials) ----
template <typename TA, typename TB>
__global__ void __launch_bounds__(256) k_diff_sq(const TA* __restrict__ A, const TB* __restrict__ B,
                                                 int64_t n, double* __restrict__ part) {
  __shared__ double red[40];
  double d2 = 0.0, a2 = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double a = (double)A[e], d = a - (double)B[e];
    d2 = fma(d, d, d2);
    a2 = fma(a, a, a2);
  }
  d2 = block_sum(d2, red);
  a2 = block_sum(a2, red);
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = d2; part[2 * blockIdx.x + 1] = a2; }
}

__global__ void k_fold2(const double* __restrict__ part, int n, double* __restrict__ out2) {
  if (threadIdx.x != 0) return;
  double s = 0.0, t = 0.0;
  for (int p = 0; p < n; ++p) { s += part[2 * p]; t += part[2 * p + 1]; }
  out2[0] = s;
  out2[1] = t;
}

// ---- performance index, one CTA per pair ----
struct PiPair {
  const double* E;
  const double* T;
  int64_t rows;
};

__global__ void __launch_bounds__(256) k_perf_index(const PiPair* __restrict__ pairs, int R,
                                                    double* __restrict__ out, int* __restrict__ deficient) {
  extern __shared__ double sm[];
  double* A = sm;                  // R x R: E^T E, LU in place
  double* B = A + R * R;           // R x R: E^T T, then the solution X
  double* rmax = B + R * R;        // R
  double* cmax = rmax + R;         // R
  double* red = cmax + R;          // 40
  __shared__ int piv[64];
  __shared__ int s_p;
  const PiPair pr = pairs[blockIdx.x];
  for (int e = threadIdx.x; e < 2 * R * R; e += blockDim.x) {
    const int which = e / (R * R), q = e - which * R * R;
    const int i = q / R, j = q - i * R;
    const double* Y = which ? pr.T : pr.E;
    double g = 0.0;
    for (int64_t k = 0; k < pr.rows; ++k) g = fma(pr.E[k * R + i], Y[k * R + j], g);
    (which ? B : A)[q] = g;
  }
  __syncthreads();
  // LU with partial pivoting (first max |a_ik|)
  for (int k = 0; k < R; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double best = fabs(A[k * R + k]);
      for (int i = k + 1; i < R; ++i) {
        const double a = fabs(A[i * R + k]);
        if (a > best) { best = a; p = i; }
      }
      s_p = p;
      piv[k] = p;
    }
    __syncthreads();
    const int p = s_p;
    if (p != k)
      for (int j = threadIdx.x; j < R; j += blockDim.x) {
        double t = A[k * R + j]; A[k * R + j] = A[p * R + j]; A[p * R + j] = t;
        t = B[k * R + j]; B[k * R + j] = B[p * R + j]; B[p * R + j] = t;
      }
    __syncthreads();
    const double d = A[k * R + k];
    for (int i = k + 1 + threadIdx.x; i < R; i += blockDim.x) A[i * R + k] /= d;
    __syncthreads();
    const int m = R - k - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      A[i * R + j] -= A[i * R + k] * A[k * R + j];
    }
    __syncthreads();
  }
  // rank test on the pivots of the gram (their ratio ~ sigma_min^2 / sigma_max^2)
  if (threadIdx.x == 0) {
    double lo = INFINITY, hi = 0.0;
    for (int k = 0; k < R; ++k) { const double v = fabs(A[k * R + k]); lo = fmin(lo, v); hi = fmax(hi, v); }
    const double tol = (double)(pr.rows > R ? pr.rows : R) * 2.220446049250313e-16;
    deficient[blockIdx.x] = !(lo > hi * tol * tol * R);
  }
  // one right-hand side (column of B) per thread: forward / back substitution
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    for (int r = 0; r < R; ++r) {
      double a = B[r * R + j];
      for (int q = 0; q < r; ++q) a -= A[r * R + q] * B[q * R + j];
      B[r * R + j] = a;
    }
    for (int r = R - 1; r >= 0; --r) {
      double a = B[r * R + j];
      for (int q = r + 1; q < R; ++q) a -= A[r * R + q] * B[q * R + j];
      B[r * R + j] = a / A[r * R + r];
    }
  }
  __syncthreads();
  // G = |X|; row / column maxima (0 -> 1)
  for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) {
    const bool row = i < R;
    const int k = row ? i : i - R;
    double m = 0.0;
    for (int q = 0; q < R; ++q) m = fmax(m, fabs(row ? B[k * R + q] : B[q * R + k]));
    (row ? rmax : cmax)[k] = m == 0.0 ? 1.0 : m;
  }
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < 2 * R; i += blockDim.x) {
    const bool row = i < R;
    const int k = row ? i : i - R;
    double s = 0.0;
    for (int q = 0; q < R; ++q)
      s += row ? fabs(B[k * R + q]) / rmax[k] : fabs(B[q * R + k]) / cmax[k];
    s -= 1.0;
    acc += s > 0.0 ? s : 0.0;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc / (2.0 * R * (R - 1));
}

}  // namespace cb

using namespace cb;

extern "C" {

int cb_diff_sq(int dtype_a, const void* A, int dtype_b, const void* B, int64_t n, double* out2,
               void* stream) {
  CB_ARG(A && B && out2 && n >= 0, "bad argument");
  CB_ARG((dtype_a == CB_F32 || dtype_a == CB_F64) && (dtype_b == CB_F32 || dtype_b == CB_F64),
         "bad dtype");
  cudaStream_t st = (cudaStream_t)stream;
  const int np = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + 255) / 256));
  double* part;
  CB_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * 2 * np, st));
  if (dtype_a == CB_F32 && dtype_b == CB_F32)
    k_diff_sq<float, float><<<np, 256, 0, st>>>((const float*)A, (const float*)B, n, part);
  else if (dtype_a == CB_F32)
    k_diff_sq<float, double><<<np, 256, 0, st>>>((const float*)A, (const double*)B, n, part);
  else if (dtype_b == CB_F32)
    k_diff_sq<double, float><<<np, 256, 0, st>>>((const double*)A, (const float*)B, n, part);
  else
    k_diff_sq<double, double><<<np, 256, 0, st>>>((const double*)A, (const double*)B, n, part);
  k_fold2<<<1, 32, 0, st>>>(part, np, out2);
  count_launch(2);
  CB_CHECK_LAUNCH();
  CB_CUDA(cudaFreeAsync(part, st));
  return CB_OK;
}

int cb_performance_index(int n_pairs, const double* const* estimated, const double* const* truth,
                         const int64_t* rows, int rank, double* out, int* deficient,
                         void* stream) {
  CB_ARG(n_pairs >= 1 && estimated && truth && rows && out && deficient, "bad argument");
  CB_ARG(rank >= 2 && rank <= CB_MAX_RANK, "rank %d outside [2, %d]", rank, CB_MAX_RANK);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<PiPair> h(n_pairs);
  for (int p = 0; p < n_pairs; ++p) {
    CB_ARG(rows[p] >= 1, "empty factor");
    h[p] = PiPair{estimated[p], truth[p], rows[p]};
  }
  PiPair* d;
  CB_CUDA(cudaMallocAsync((void**)&d, sizeof(PiPair) * n_pairs, st));
  CB_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(PiPair) * n_pairs, cudaMemcpyHostToDevice, st));
  const size_t smem = sizeof(double) * (2 * (size_t)rank * rank + 2 * rank + 40);
  CB_CUDA(cudaFuncSetAttribute(k_perf_index, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_perf_index<<<n_pairs, 256, smem, st>>>(d, rank, out, deficient);
  count_launch(1);
  CB_CHECK_LAUNCH();
  // the pair table must outlive the kernel: free in stream order
  CB_CUDA(cudaFreeAsync(d, st));
  return CB_OK;
}

}  // extern "C"
