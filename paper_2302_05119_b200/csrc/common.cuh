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

// Programmatic dependent launch: kernels of the iteration are launched with
// programmatic stream serialization, so a kernel's CTAs may be scheduled while
// its predecessor drains; every kernel therefore waits here (first statement)
// before touching anything the predecessor wrote.  A no-op for ordinary
// launches.
// The trigger (launch_dependents) is issued first: the next kernel's CTAs are
// scheduled as soon as every CTA of this one is running, and sit in their own
// griddep_wait() until this grid has completed and flushed (the wait, not
// the trigger, carries the memory ordering), so the launch latency of the
// serial iteration chain overlaps the running kernel.  CB_NO_EARLY_TRIGGER
// builds keep the implicit trigger at exit.
__device__ __forceinline__ void griddep_wait() {
#ifndef CB_NO_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// The wait without the early trigger, for the persistent streaming kernels
// (one CTA per SM for milliseconds): dependents launched early would sit
// resident beside them for the whole stream and slow it (measured on the ALS
// mode-2 pass: 9.0 -> 4.9 ms with its contraction kernel launched at exit).
__device__ __forceinline__ void griddep_wait_no_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Asynchronous global -> shared staging (LDGSTS): every thread issues its
// 8-byte copies without waiting, so a staging loop costs one memory latency
// instead of one per iteration.  Complete with cp_async8_wait() and a barrier.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_wait() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// dst[e] = src[e], e < n, all threads of the block (no wait)
__device__ __forceinline__ void stage_async(double* dst, const double* src, long long n) {
  for (long long e = threadIdx.x; e < n; e += blockDim.x) cp_async8(dst + e, src + e);
}

// Phase timestamps (profiling builds of a run: Ctx.dbg non-null): block 0
// accumulates the time between consecutive PH() marks into dbg[slot].
struct PhaseClock {
  unsigned long long last = 0;
  long long last_clk = 0;
  __device__ __forceinline__ unsigned long long now() const {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  }
  __device__ __forceinline__ void start(const double* dbg) {
    if (dbg && blockIdx.x == 0) { __syncthreads(); last = now(); last_clk = clock64(); }
  }
  // dbg[slot] += ns, dbg[32 + slot] += SM cycles (their ratio is the clock)
  __device__ __forceinline__ void mark(double* dbg, int slot) {
    if (dbg && blockIdx.x == 0) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long t = now();
        const long long k = clock64();
        dbg[slot] += (double)(t - last);
        dbg[32 + slot] += (double)(k - last_clk);
        // restart after the read-modify-write: its global round trip is
        // charged to no phase
        last = now();
        last_clk = clock64();
      }
    }
  }
};


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
// the matrix drives B -> (normalised) projector onto the top eigenspace in
// O(log(1/gap)) squarings (<= 64 squarings resolve any gap >= 2^-60); the
// column of the limit with the largest diagonal is the eigenvector estimate;
// one power step and the Rayleigh quotient with the original matrix give the
// eigenvalue to ~R ulp.  Negative-dominant or +-lambda tie inputs (never
// produced by the solver, whose matrices are PSD Schur products) are handled
// by a spectral-radius shift and a second pass.
//
// Latency is what matters here (one call per block per mode on the
// iteration's critical path), so every thread of the block owns fixed entries
// of B (1x1 for R <= 16, 2x2 register tiles above) for the whole call: the
// squarings, renormalisation and convergence test need no index arithmetic
// and one block reduction each.  Two squarings per convergence test.
//
// smem: A  Rp4 x lm_ld(R)   (caller's matrix, Rp4 = round_up(R, 4))
//       B, B2  Rp2 x lm_bld(R) each (Rp2 = round_up(R, 2))
//       vec >= 128 doubles, red >= 40 doubles
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ int lm_ld(int R) { return ((R + 3) & ~3) + 1; }
__host__ __device__ __forceinline__ int lm_rp2(int R) { return (R + 1) & ~1; }
__host__ __device__ __forceinline__ int lm_bld(int R) { return lm_rp2(R) + 1; }
__host__ __device__ __forceinline__ int lm_bsize(int R) { return lm_rp2(R) * lm_bld(R); }

// Approximate block max of nonnegative doubles: the high 32 bits of an IEEE
// double order like the value, so one redux.sync per warp and one across the
// warp maxima give max(v) truncated to 20 mantissa bits (relative error
// < 2^-20).  Used only for rescaling and convergence tests, where that is
// plenty; far cheaper than a shuffle tree on doubles.
__device__ __forceinline__ double block_max_approx(double v, unsigned* ured) {
  const unsigned key = (unsigned)(__double_as_longlong(v) >> 32);
  const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  if (lane == 0) ured[wid] = wmax;
  __syncthreads();
  unsigned m = lane < nw ? ured[lane] : 0u;
  m = __reduce_max_sync(0xffffffffu, m);
  __syncthreads();   // ured may be reused by the next call
  return __longlong_as_double((long long)((unsigned long long)m << 32));
}
// exact warp max of nonnegative doubles via two 32-bit redux steps on the bit
// pattern (high word, then the low word among the lanes holding the max high)
__device__ __forceinline__ unsigned long long warp_max_bits(unsigned long long k) {
  const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}
// two exact maxima (nonnegative doubles) in one barrier round
__device__ __forceinline__ void block_max2_exact(double a, double b, unsigned* ured, double* ma,
                                                 double* mb) {
  unsigned long long* ub = reinterpret_cast<unsigned long long*>(ured);
  const unsigned long long ka = warp_max_bits((unsigned long long)__double_as_longlong(a));
  const unsigned long long kb = warp_max_bits((unsigned long long)__double_as_longlong(b));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { ub[wid] = ka; ub[8 + wid] = kb; }
  __syncthreads();
  unsigned long long xa = lane < nw ? ub[lane] : 0ull, xb = lane < nw ? ub[8 + lane] : 0ull;
  xa = warp_max_bits(xa);
  xb = warp_max_bits(xb);
  __syncthreads();
  *ma = __longlong_as_double((long long)xa);
  *mb = __longlong_as_double((long long)xb);
}

// B2 = B * B for symmetric B (Rp2 x Rp2, leading dim bld): entry (i,j) is
// row i . row j.  Thread tile list: tiles t = tid, tid + nthr, ... of the
// (Rp2/TS)^2 grid, TS x TS entries each.  Ends with a block barrier.
template <int TS>
__device__ __forceinline__ void sq_tiles(const double* B, double* B2, int Rp2, int bld) {
  const int nt = Rp2 / TS;
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
    const int ti = t / nt, tj = t - ti * nt;
    double acc[TS][TS], acc2[TS][TS];
#pragma unroll
    for (int a = 0; a < TS; ++a)
#pragma unroll
      for (int b = 0; b < TS; ++b) { acc[a][b] = 0.0; acc2[a][b] = 0.0; }
    const double* ri = B + (TS * ti) * bld;
    const double* rj = B + (TS * tj) * bld;
    int k = 0;
    for (; k + 2 <= Rp2; k += 2) {   // two independent FMA chains
#pragma unroll
      for (int a = 0; a < TS; ++a)
#pragma unroll
        for (int b = 0; b < TS; ++b) {
          acc[a][b] = fma(ri[a * bld + k], rj[b * bld + k], acc[a][b]);
          acc2[a][b] = fma(ri[a * bld + k + 1], rj[b * bld + k + 1], acc2[a][b]);
        }
    }
#pragma unroll
    for (int a = 0; a < TS; ++a)
#pragma unroll
      for (int b = 0; b < TS; ++b) B2[(TS * ti + a) * bld + TS * tj + b] = acc[a][b] + acc2[a][b];
  }
  __syncthreads();
}

static __device__ __noinline__ void eigen_tail(const double* A, int R, int ld, const double* B, int bld,
                                  double* vec, double* red, double shift);

static __device__ __noinline__ double dominant_rq(const double* A, int R, int ld, double* B, double* B2,
                                     double* vec, double* red, double shift, double* resid_out,
                                     double* dbg = nullptr, double* m_out = nullptr) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  PhaseClock pc;
  pc.start(dbg);
  const int Rp2 = lm_rp2(R), bld = lm_bld(R);
  unsigned* ured = reinterpret_cast<unsigned*>(red);   // 64 words = 32 doubles
  double m = 0.0;
  for (int e = tid; e < R * R; e += nthr) {
    const int i = e / R, j = e - i * R;
    m = fmax(m, fabs(A[i * ld + j] + (i == j ? shift : 0.0)));
  }
  m = block_max_approx(m, ured);
  if (m_out) *m_out = m;
  if (m == 0.0) { if (resid_out) *resid_out = 0.0; return 0.0; }
  const double inv0 = 1.0 / m;
  for (int e = tid; e < Rp2 * bld; e += nthr) {
    const int i = e / bld, j = e - i * bld;
    double v = 0.0;
    if (i < R && j < R) v = (A[i * ld + j] + (i == j ? shift : 0.0)) * inv0;
    B[e] = v;
  }
  __syncthreads();
  pc.mark(dbg, 10);
  // passes of four squarings (B -> B^16); after each pass the eigenpair is
  // extracted and accepted once its residual ||Av - rho v|| / ||v|| is below
  // 1e-9 ||A||, i.e. the Rayleigh quotient is within ~1e-18 ||A||^2 / gap of
  // lambda_max.  For the solver's matrices one pass is the norm.
  double rho = 0.0, resid = 0.0;
  for (int pass = 0; pass < 16; ++pass) {
    if (pass > 0) {
      // rescale B (entries <= Rp2^15 after a pass) before squaring again
      double mb = 0.0;
      for (int e = tid; e < Rp2 * Rp2; e += nthr) {
        const int i = e / Rp2, j = e - i * Rp2;
        mb = fmax(mb, fabs(B[i * bld + j]));
      }
      mb = block_max_approx(mb, ured);
      if (!(mb > 0.0) || !isfinite(mb)) break;
      const double ib = 1.0 / mb;
      for (int e = tid; e < Rp2 * Rp2; e += nthr) {
        const int i = e / Rp2, j = e - i * Rp2;
        B[i * bld + j] *= ib;
      }
      __syncthreads();
      pc.mark(dbg, 13);
    }
    if (R <= 16) {
      sq_tiles<1>(B, B2, Rp2, bld); sq_tiles<1>(B2, B, Rp2, bld);
      sq_tiles<1>(B, B2, Rp2, bld); sq_tiles<1>(B2, B, Rp2, bld);
    } else {
      sq_tiles<2>(B, B2, Rp2, bld); sq_tiles<2>(B2, B, Rp2, bld);
      sq_tiles<2>(B, B2, Rp2, bld); sq_tiles<2>(B2, B, Rp2, bld);
    }
    pc.mark(dbg, 11);
    eigen_tail(A, R, ld, B, bld, vec, red, shift);
    rho = red[36];
    resid = red[37];
    __syncthreads();
    pc.mark(dbg, 12);
    if (resid <= 1e-9 * m) break;
  }
  if (resid_out) *resid_out = resid;
  return rho;
}

// warp 0: eigenvector from the column of B with the largest diagonal, one
// power step with the original (shifted) matrix, Rayleigh quotient and
// residual -> red[36], red[37]; ends with a block barrier
static __device__ __noinline__ void eigen_tail(const double* A, int R, int ld, const double* B, int bld,
                                  double* vec, double* red, double shift) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    int jb = 0;
    {
      double best = -1.0;
      for (int j = 0; j < R; ++j) {
        const double d = B[j * bld + j];
        if (d > best) { best = d; jb = j; }
      }
    }
    double* v = vec;
    double* av = vec + 64;
    for (int i = lane; i < R; i += 32) v[i] = B[i * bld + jb];
    __syncwarp();
    double nrm = 0.0;
    for (int i = lane; i < R; i += 32) {
      double s = 0.0;
      for (int k = 0; k < R; ++k) s = fma(A[i * ld + k] + (i == k ? shift : 0.0), v[k], s);
      av[i] = s;
      nrm = fmax(nrm, fabs(s));
    }
    nrm = warp_max(nrm);
    __syncwarp();
    if (nrm > 0.0) {
      const double inv = 1.0 / nrm;
      for (int i = lane; i < R; i += 32) v[i] = av[i] * inv;
      __syncwarp();
    }
    double num = 0.0, den = 0.0;
    for (int i = lane; i < R; i += 32) {
      double s = 0.0;
      for (int k = 0; k < R; ++k) s = fma(A[i * ld + k] + (i == k ? shift : 0.0), v[k], s);
      av[i] = s;
      num = fma(v[i], s, num);
      den = fma(v[i], v[i], den);
    }
    num = warp_sum(num);
    den = warp_sum(den);
    const double rho = den > 0.0 ? num / den : 0.0;
    double r2 = 0.0;
    for (int i = lane; i < R; i += 32) { const double d = av[i] - rho * v[i]; r2 = fma(d, d, r2); }
    r2 = warp_sum(r2);
    if (lane == 0) {
      red[36] = rho;
      red[37] = den > 0.0 ? sqrt(r2 / den) : 0.0;
    }
  }
  __syncthreads();
}

// lambda_max(A) clamped at 0 (0 for the exact zero matrix).  A in smem with
// leading dimension lm_ld(R).  All threads of the block must call it; the
// result is returned to every thread.
static __device__ __noinline__ double block_lam_max(const double* A, int R, double* B, double* B2, double* vec,
                                       double* red, double* dbg = nullptr) {
  const int ld = lm_ld(R);
  double resid;
  // the unshifted pass's max |A| is the amax of the acceptance test (the
  // same block_max_approx of the same entries; no second reduction)
  double amax = 0.0;
  const double rho = dominant_rq(A, R, ld, B, B2, vec, red, 0.0, &resid, dbg, &amax);
  PhaseClock pc;
  pc.start(dbg);
  pc.mark(dbg, 14);
  if (amax == 0.0) return 0.0;
  // PSD / positive-dominant path: a converged eigenpair with rho >= 0 is the
  // spectral radius, hence lambda_max
  if (rho >= 0.0 && resid <= 1e-10 * amax * R) return rho;
  // otherwise shift by a spectral-radius bound so A + sI is PSD
  const double s = (rho < 0.0 && resid <= 1e-10 * amax * R) ? -rho : 2.0 * amax * R;
  const double rho2 = dominant_rq(A, R, ld, B, B2, vec, red, s, nullptr);
  pc.mark(dbg, 15);
  const double lm = rho2 - s;
  return lm > 0.0 ? lm : 0.0;
}

// lambda_max of the same matrix slot as the previous call (a step matrix of
// one block and mode, or its core gram): power steps from the slot's last
// eigenvector `warm` (64 doubles, global; zero = none yet), accepted with
// block_lam_max's test (rho >= 0, ||A v - rho v|| / ||v|| <= 1e-10 max|A| R),
// at most 10 steps while the residual keeps shrinking fast; otherwise the
// squaring solve.  The accepted eigenvector is
// stored back.  The APG's matrices move little between iterations, so one
// or two steps usually pass the test (c5: top-two ratio ~0.03).
static __device__ __noinline__ double block_lam_max_warm(const double* A, int R, double* B, double* B2,
                                                        double* vec, double* red, double* warm,
                                                        int* miss) {
  // small ranks: the squaring solve (R^3 per squaring) costs less than a few
  // barrier-bound power steps (measured on c2, R = 10)
  if (R <= 16) return block_lam_max(A, R, B, B2, vec, red);
  const int ld = lm_ld(R);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  double* v = vec;
  double* w = vec + 64;
  unsigned* ured = reinterpret_cast<unsigned*>(red);
  double m = 0.0;
  for (int e = tid; e < R * R; e += nthr) {
    const int i = e / R, j = e - i * R;
    m = fmax(m, fabs(A[i * ld + j]));
  }
  m = block_max_approx(m, ured);
  if (m == 0.0) return 0.0;
  // a slot whose spectrum defeated the warm steps recently (clustered top
  // eigenvalues) goes straight to the squaring solve; retried every 8 calls
  const int skip = *miss;
  __syncthreads();
  if (skip > 0) {
    if (tid == 0) *miss = skip - 1;
    const double lam = block_lam_max(A, R, B, B2, vec, red);
    for (int i = tid; i < R; i += nthr) warm[i] = vec[i];
    __syncthreads();
    return lam;
  }
  for (int i = tid; i < R; i += nthr) v[i] = warm[i];
  __syncthreads();
  double prev_resid = INFINITY;
  for (int it = 0; it < 10; ++it) {
    for (int i = wid; i < R; i += nw) {
      double a = 0.0;
      for (int j = lane; j < R; j += 32) a = fma(A[i * ld + j], v[j], a);
      a = warp_sum(a);
      if (lane == 0) w[i] = a;
    }
    __syncthreads();
    if (wid == 0) {
      double num = 0.0, den = 0.0, wm = 0.0;
      for (int i = lane; i < R; i += 32) {
        num = fma(v[i], w[i], num);
        den = fma(v[i], v[i], den);
        wm = fmax(wm, fabs(w[i]));
      }
      num = warp_sum(num);
      den = warp_sum(den);
      wm = warp_max(wm);
      const double rho = den > 0.0 ? num / den : 0.0;
      double r2 = 0.0;
      for (int i = lane; i < R; i += 32) {
        const double d = w[i] - rho * v[i];
        r2 = fma(d, d, r2);
      }
      r2 = warp_sum(r2);
      __syncwarp();
      if (wm > 0.0)
        for (int i = lane; i < R; i += 32) v[i] = w[i] / wm;
      if (lane == 0) {
        red[36] = rho;
        red[37] = den > 0.0 ? sqrt(r2 / den) : INFINITY;
        red[38] = (den > 0.0 && wm > 0.0) ? 1.0 : 0.0;
      }
    }
    __syncthreads();
    const double rho = red[36], resid = red[37];
    const bool live = red[38] > 0.0;
    __syncthreads();
    if (!live) break;
    if (rho >= 0.0 && resid <= 1e-10 * m * R) {
      for (int i = tid; i < R; i += nthr) warm[i] = v[i];
      return rho;
    }
    // a slowly shrinking residual means clustered top eigenvalues: the
    // squaring solve is cheaper than more steps
    if (it >= 2 && resid > 0.5 * prev_resid) break;
    prev_resid = resid;
  }
  if (tid == 0) *miss = 8;
  const double lam = block_lam_max(A, R, B, B2, vec, red);
  // the squaring solve leaves its eigenvector in vec[0..R)
  for (int i = tid; i < R; i += nthr) warm[i] = vec[i];
  __syncthreads();
  return lam;
}

// shared memory (doubles) of block_lam_max for rank R: A, B, B2, vec, red
__host__ __device__ __forceinline__ int lm_smem_doubles(int R) {
  return ((R + 3) & ~3) * lm_ld(R) + 2 * lm_bsize(R) + 128 + 40;
}

}  // namespace cb
