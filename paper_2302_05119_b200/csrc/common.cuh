// Shared device helpers for the concpd B200 kernels (sm_100a).
//
// Conventions (reference: pkg/src/concpd/tensor_ops.py:1-15):
//   * tensors are dense, first-index-fastest (Fortran) order;
//   * factor matrices are fp64, row-major I_n x R (a row = one index of mode n);
//   * R x R gram products are fp64 row-major.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#ifndef CB_MAX_ORDER
#define CB_MAX_ORDER 8
#endif
#define CB_MAX_RANK 64
#define CB_THREADS 256

namespace cb {

// ----------------------------------------------------------------------------
// deterministic block reductions (fixed shuffle tree, fixed warp order)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum over the whole block; result broadcast to every thread.  `red` must hold
// >= 33 doubles of shared memory.  Deterministic for a fixed blockDim.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? red[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// ----------------------------------------------------------------------------
// scalar rules of the APG iteration (solver.py:265-274)
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ double t_next(double t) {
  return 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
}
__host__ __device__ __forceinline__ double extrap_weight(double w_hat, double lp, double lc,
                                                         double delta_w) {
  if (lc <= 0.0 || lp <= 0.0) return 0.0;
  double cap = delta_w * sqrt(lp / lc);
  return w_hat < cap ? w_hat : cap;   // min(w_hat, cap); ties pick w_hat (same value)
}

// ----------------------------------------------------------------------------
// largest eigenvalue of a symmetric R x R matrix (R <= 64), whole block.
//
// Replaces tensor_ops.py:127-140 (LAPACK syevd).  Method: repeated squaring of
// the power-of-two-normalised matrix drives B -> projector onto the top
// eigenspace in O(log) steps (gap-independent up to 2^60), a column of the
// limit is the eigenvector estimate, and the Rayleigh quotient with the
// original matrix gives the eigenvalue to ~1 ulp * R.  Negative-dominant or
// +-lambda tie inputs (not produced by the solver, whose matrices are PSD
// Schur products) are handled by a shift and a second pass.
//
// smem: A (R*ld), B, B2 each R*ld doubles with ld = Rp+1, Rp = round_up(R,4);
//       vec >= 2*64 doubles, red >= 33 doubles.
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ int lm_ld(int R) { return ((R + 3) & ~3) + 1; }

__device__ inline double block_dominant_rq(const double* A, int R, int ld, double* B, double* B2,
                                    double* vec, double* red, double shift, double* resid_out) {
  const int tid = threadIdx.x;
  const int Rp = (R + 3) & ~3;
  const int nt = Rp >> 2;
  // B = (A + shift I) scaled by a power of two so max |B| in [0.5, 1)
  double m = 0.0;
  for (int e = tid; e < R * R; e += blockDim.x) {
    int i = e / R, j = e - i * R;
    double v = A[i * ld + j] + (i == j ? shift : 0.0);
    m = fmax(m, fabs(v));
  }
  m = block_max(m, red);
  if (m == 0.0) { if (resid_out) *resid_out = 0.0; return 0.0; }
  int ex; frexp(m, &ex);
  for (int e = tid; e < Rp * ld; e += blockDim.x) {
    int i = e / ld, j = e - i * ld;
    double v = 0.0;
    if (i < R && j < R) v = ldexp(A[i * ld + j] + (i == j ? shift : 0.0), -ex);
    B[e] = v;
  }
  __syncthreads();
  for (int it = 0; it < 64; ++it) {
    // B2 = B * B via 4x4 register tiles (B symmetric: row i . row j)
    double lmax = 0.0;
    for (int t = tid; t < nt * nt; t += blockDim.x) {
      int ti = t / nt, tj = t - ti * nt;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      const double* ri = B + (4 * ti) * ld;
      const double* rj = B + (4 * tj) * ld;
      for (int k = 0; k < Rp; ++k) {
        double x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) { x[a] = ri[a * ld + k]; y[a] = rj[a * ld + k]; }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          B2[(4 * ti + a) * ld + 4 * tj + b] = acc[a][b];
          lmax = fmax(lmax, fabs(acc[a][b]));
        }
    }
    lmax = block_max(lmax, red);   // includes a __syncthreads after B2 writes
    if (lmax == 0.0) break;        // nilpotent-like underflow; keep previous B
    int e2; frexp(lmax, &e2);
    double diff = 0.0;
    for (int e = tid; e < Rp * ld; e += blockDim.x) {
      int i = e / ld, j = e - i * ld;
      if (i < Rp && j < Rp) {
        double v = ldexp(B2[e], -e2);
        diff = fmax(diff, fabs(v - B[e]));
        B[e] = v;
      }
    }
    diff = block_max(diff, red);
    if (diff < 1e-13 && it >= 1) break;
  }
  // eigenvector estimate: the column of the limit with the largest diagonal
  __shared__ int s_jbest;
  if (tid == 0) {
    int jb = 0;
    double best = -1.0;
    for (int j = 0; j < R; ++j) {
      double d = B[j * ld + j];
      if (d > best) { best = d; jb = j; }
    }
    s_jbest = jb;
  }
  __syncthreads();
  const int jb = s_jbest;
  double* v = vec;
  double* av = vec + 64;
  for (int i = tid; i < R; i += blockDim.x) v[i] = B[i * ld + jb];
  __syncthreads();
  // one power step with the original (shifted) matrix sharpens the vector
  for (int i = tid; i < R; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(A[i * ld + k] + (i == k ? shift : 0.0), v[k], s);
    av[i] = s;
  }
  __syncthreads();
  double nrm = 0.0;
  for (int i = tid; i < R; i += blockDim.x) nrm = fmax(nrm, fabs(av[i]));
  nrm = block_max(nrm, red);
  if (nrm > 0.0) {
    int en; frexp(nrm, &en);
    for (int i = tid; i < R; i += blockDim.x) v[i] = ldexp(av[i], -en);
    __syncthreads();
  }
  for (int i = tid; i < R; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(A[i * ld + k] + (i == k ? shift : 0.0), v[k], s);
    av[i] = s;
  }
  __syncthreads();
  double num = 0.0, den = 0.0;
  for (int i = tid; i < R; i += blockDim.x) { num = fma(v[i], av[i], num); den = fma(v[i], v[i], den); }
  num = block_sum(num, red);
  den = block_sum(den, red);
  double rho = den > 0.0 ? num / den : 0.0;
  if (resid_out) {
    double r2 = 0.0;
    for (int i = tid; i < R; i += blockDim.x) { double d = av[i] - rho * v[i]; r2 = fma(d, d, r2); }
    r2 = block_sum(r2, red);
    *resid_out = den > 0.0 ? sqrt(r2 / den) : 0.0;
  }
  return rho;
}

// lambda_max(A) clamped at 0 (0 for the exact zero matrix).  A in smem with
// leading dimension lm_ld(R).  All threads of the block must call it.
__device__ inline double block_lam_max(const double* A, int R, double* B, double* B2, double* vec,
                                double* red) {
  const int ld = lm_ld(R);
  double resid;
  double rho = block_dominant_rq(A, R, ld, B, B2, vec, red, 0.0, &resid);
  double amax = 0.0;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    int i = e / R, j = e - i * R;
    amax = fmax(amax, fabs(A[i * ld + j]));
  }
  amax = block_max(amax, red);
  if (amax == 0.0) return 0.0;
  // PSD / positive-dominant fast path: a converged eigenpair with rho >= 0 is
  // the spectral radius, hence lambda_max.
  if (rho >= 0.0 && resid <= 1e-10 * amax * R) return rho;
  // otherwise shift by a spectral-radius bound so A + sI is PSD
  double s = rho < 0.0 && resid <= 1e-10 * amax * R ? -rho : amax * R;
  double rho2 = block_dominant_rq(A, R, ld, B, B2, vec, red, s, nullptr);
  double lm = rho2 - s;
  return lm > 0.0 ? lm : 0.0;
}

}  // namespace cb
