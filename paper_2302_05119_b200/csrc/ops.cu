// Operator-level kernels and their C-ABI entry points (include/concpd_b200.h).
//
// These are the building blocks the reference exposes as plain functions
// (tensor_ops.py:19-28, solver.py:34-52).  They are batched/general (any
// order <= 8, rank <= 64) rather than tuned: the solver engine (engine.cu)
// uses its own fused, tiled kernels for the iteration.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <vector>

#include "common.cuh"
#include "status.h"
#include "ops_internal.h"

namespace cb {

static thread_local char g_err[1024] = "";
static thread_local long long g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
            what, file, line);
  return CB_ERR_CUDA;
}

void count_launch(long long n) { g_launches += n; }

// ----------------------------------------------------------------------------
// Khatri-Rao rows with the FIRST matrix fastest:
//   out[q, r] = prod_m mats[m][idx_m(q), r],  q = i_0 + rows_0 * (i_1 + ...)
// ----------------------------------------------------------------------------
__global__ void kr_first_fastest_kernel(KrArgs a, double* __restrict__ out, int64_t nrows) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = nrows * a.rank;
  for (; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = e / a.rank;
    int r = (int)(e - q * a.rank);
    double v = 1.0;
    int64_t rem = q;
    for (int m = 0; m < a.nmats; ++m) {
      int64_t i = rem % a.rows[m];
      rem /= a.rows[m];
      v = (m == 0) ? a.mats[m][i * a.rank + r] : v * a.mats[m][i * a.rank + r];
    }
    out[e] = v;
  }
}

int launch_kr_first_fastest(const KrArgs& a, double* out, cudaStream_t st) {
  int64_t nrows = 1;
  for (int m = 0; m < a.nmats; ++m) nrows *= a.rows[m];
  int64_t total = nrows * a.rank;
  if (total == 0) return CB_OK;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  kr_first_fastest_kernel<<<blocks, 256, 0, st>>>(a, out, nrows);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

// ----------------------------------------------------------------------------
// generic MTTKRP: one CTA per output row i_n.  The tensor is viewed as
// L x I_n x H (L = prod of modes before n, H = prod after); KR rows of the
// left and right mode groups are precomputed (KRl: L x R, KRh: H x R).
// Deterministic: per-thread partial sums in fixed order, fixed block tree.
// ----------------------------------------------------------------------------
template <typename TE, int RB>
__global__ void __launch_bounds__(256) mttkrp_generic_kernel(MttJob j) {
  __shared__ double red[8][RB + 1];
  const int64_t row = blockIdx.x;
  const int R = j.R;
  const TE* X = reinterpret_cast<const TE*>(j.X);
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0;
  const int64_t LH = j.L * j.H;
  for (int64_t q = threadIdx.x; q < LH; q += blockDim.x) {
    int64_t h = q / j.L;
    int64_t l = q - h * j.L;
    double x = (double)X[l + j.L * (row + j.In * h)];
    const double* kl = j.KRl ? j.KRl + l * R : nullptr;
    const double* kh = j.KRh ? j.KRh + h * R : nullptr;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < R) {
        double k = 1.0;
        if (kl) k = kl[r];
        if (kh) k = kl ? k * kh[r] : kh[r];
        acc[r] = fma(x, k, acc[r]);
      }
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    double v = warp_sum(acc[r]);
    if (lane == 0) red[wid][r] = v;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    j.out[row * R + threadIdx.x] = s;
  }
}

template <typename TE>
static void launch_mtt_generic_t(const MttJob& j, cudaStream_t st) {
  dim3 grid((unsigned)j.In);
  if (j.R <= 8) mttkrp_generic_kernel<TE, 8><<<grid, 256, 0, st>>>(j);
  else if (j.R <= 16) mttkrp_generic_kernel<TE, 16><<<grid, 256, 0, st>>>(j);
  else if (j.R <= 32) mttkrp_generic_kernel<TE, 32><<<grid, 256, 0, st>>>(j);
  else mttkrp_generic_kernel<TE, 64><<<grid, 256, 0, st>>>(j);
}

int launch_mttkrp_generic(int dtype, const MttJob& j, cudaStream_t st) {
  if (j.In == 0) return CB_OK;
  if (dtype == CB_F32) launch_mtt_generic_t<float>(j, st);
  else launch_mtt_generic_t<double>(j, st);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

// Build KRl/KRh scratch and run the generic MTTKRP for one tensor.  `scratch`
// must hold (L + H) * R doubles.
int mttkrp_one(int dtype, const void* X, int order, const int64_t* dims,
               const double* const* factors, int rank, int mode, double* out,
               double* scratch, cudaStream_t st) {
  int64_t L = 1, H = 1;
  for (int m = 0; m < mode; ++m) L *= dims[m];
  for (int m = mode + 1; m < order; ++m) H *= dims[m];
  MttJob j{};
  j.X = X; j.L = L; j.In = dims[mode]; j.H = H; j.R = rank; j.out = out;
  j.KRl = nullptr; j.KRh = nullptr;
  if (mode > 0) {
    KrArgs a{};
    a.nmats = mode; a.rank = rank;
    for (int m = 0; m < mode; ++m) { a.mats[m] = factors[m]; a.rows[m] = dims[m]; }
    int rc = launch_kr_first_fastest(a, scratch, st);
    if (rc) return rc;
    j.KRl = scratch;
  }
  if (mode < order - 1) {
    KrArgs a{};
    a.nmats = order - 1 - mode; a.rank = rank;
    for (int m = mode + 1; m < order; ++m) {
      a.mats[m - mode - 1] = factors[m];
      a.rows[m - mode - 1] = dims[m];
    }
    int rc = launch_kr_first_fastest(a, scratch + L * rank, st);
    if (rc) return rc;
    j.KRh = scratch + L * rank;
  }
  if (L * H == 0) {  // empty contraction: zeros
    CB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * dims[mode] * rank, st));
    return CB_OK;
  }
  return launch_mttkrp_generic(dtype, j, st);
}

// ----------------------------------------------------------------------------
// hadamard product of (cross) grams, thread per output entry, mode order
// ----------------------------------------------------------------------------
__global__ void hadamard_gram_kernel(HgArgs a, double* __restrict__ out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.ra * a.rb) return;
  int p = e / a.rb, q = e - p * a.rb;
  double prod = 0.0;
  bool first = true;
  for (int m = 0; m < a.nmodes; ++m) {
    if (m == a.skip) continue;
    const double* A = a.A[m];
    const double* B = a.B[m];
    double g = 0.0;
    for (int64_t i = 0; i < a.rows[m]; ++i) g = fma(A[i * a.ra + p], B[i * a.rb + q], g);
    prod = first ? g : prod * g;
    first = false;
  }
  out[e] = prod;
}

// ----------------------------------------------------------------------------
// batched spectral norm: one CTA per matrix
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) spectral_batched_kernel(const double* __restrict__ g,
                                                               int R, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int ld = lm_ld(R);
  const int Rp = (R + 3) & ~3;
  double* A = sm;
  double* B = A + Rp * ld;
  double* B2 = B + lm_bsize(R);
  double* vec = B2 + lm_bsize(R);
  double* red = vec + 128;
  const double* gb = g + (int64_t)blockIdx.x * R * R;
  for (int e = threadIdx.x; e < Rp * ld; e += blockDim.x) {
    int i = e / ld, j = e - i * ld;
    A[e] = (i < R && j < R) ? gb[i * R + j] : 0.0;
  }
  __syncthreads();
  double v = block_lam_max(A, R, B, B2, vec, red);
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

size_t lam_max_smem_bytes(int R) { return sizeof(double) * (size_t)lm_smem_doubles(R); }

// ----------------------------------------------------------------------------
// tensor statistics: sum of squares, min, non-finite count (two-stage)
// ----------------------------------------------------------------------------
template <typename TE>
__global__ void __launch_bounds__(256) tensor_stats_kernel(const TE* __restrict__ X, int64_t n,
                                                           double* __restrict__ part) {
  __shared__ double red[40];
  double ss = 0.0, mn = INFINITY, bad = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = (double)X[i];
    if (!isfinite(x)) { bad += 1.0; continue; }
    ss = fma(x, x, ss);
    mn = fmin(mn, x);
  }
  ss = block_sum(ss, red);
  bad = block_sum(bad, red);
  mn = -block_max(-mn, red);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = ss;
    part[3 * blockIdx.x + 1] = mn;
    part[3 * blockIdx.x + 2] = bad;
  }
}

// fixed-order second stage: thread t sums parts t, t+256, ...; then the
// deterministic block tree
__global__ void __launch_bounds__(256) stats_final_kernel(const double* __restrict__ part,
                                                          int nparts, double* __restrict__ out3) {
  __shared__ double red[40];
  double ss = 0.0, mn = INFINITY, bad = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
    ss += part[3 * p];
    mn = fmin(mn, part[3 * p + 1]);
    bad += part[3 * p + 2];
  }
  ss = block_sum(ss, red);
  bad = block_sum(bad, red);
  mn = -block_max(-mn, red);
  if (threadIdx.x == 0) {
    out3[0] = ss;
    out3[1] = mn;
    out3[2] = bad;
  }
}

int tensor_stats(int dtype, const void* X, int64_t n, double* out3, double* part, int nparts,
                 cudaStream_t st) {
  if (dtype == CB_F32)
    tensor_stats_kernel<float><<<nparts, 256, 0, st>>>((const float*)X, n, part);
  else
    tensor_stats_kernel<double><<<nparts, 256, 0, st>>>((const double*)X, n, part);
  stats_final_kernel<<<1, 256, 0, st>>>(part, nparts, out3);
  count_launch(2);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

// Loads the stats kernels now (lazy module loading otherwise loads a kernel
// at its first launch, which waits for every copy in flight: the staged ALS
// start launches them beside the uploads)
void tensor_stats_preload() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tensor_stats_kernel<float>);
  cudaFuncGetAttributes(&fa, tensor_stats_kernel<double>);
  cudaFuncGetAttributes(&fa, stats_final_kernel);
}

// ----------------------------------------------------------------------------
// explicit Kruskal residual || X - [[w; U]] ||^2, generic order (two-stage)
// ----------------------------------------------------------------------------
template <typename TE>
__global__ void __launch_bounds__(256) kruskal_resid_kernel(ResidArgs a, const TE* __restrict__ X,
                                                            double* __restrict__ part) {
  __shared__ double red[40];
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx[CB_MAX_ORDER];
    int64_t rem = e;
    for (int m = 0; m < a.order; ++m) { idx[m] = rem % a.dims[m]; rem /= a.dims[m]; }
    double model = 0.0;
    for (int r = 0; r < a.R; ++r) {
      double v = a.w ? a.w[r] : 1.0;
      for (int m = 0; m < a.order; ++m) v *= a.U[m][idx[m] * a.R + r];
      model += v;
    }
    double d = (double)X[e] - model;
    acc = fma(d, d, acc);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(256) sum_parts_kernel(const double* __restrict__ part,
                                                        int nparts, double* __restrict__ out) {
  __shared__ double red[40];
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += part[p];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

int kruskal_residual(int dtype, const ResidArgs& a, const void* X, double* out, double* part,
                     int nparts, cudaStream_t st) {
  if (dtype == CB_F32)
    kruskal_resid_kernel<float><<<nparts, 256, 0, st>>>(a, (const float*)X, part);
  else
    kruskal_resid_kernel<double><<<nparts, 256, 0, st>>>(a, (const double*)X, part);
  sum_parts_kernel<<<1, 256, 0, st>>>(part, nparts, out);
  count_launch(2);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

// ----------------------------------------------------------------------------
// small dense helpers
// ----------------------------------------------------------------------------
__global__ void rowdot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              int64_t rows, int R, double* __restrict__ out) {
  __shared__ double red[40];
  const int r = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) s = fma(a[i * R + r], b[i * R + r], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[r] = s;
}

__global__ void gemm_small_kernel(int ta, int tb, int m, int n, int k, double alpha,
                                  const double* __restrict__ A, int lda,
                                  const double* __restrict__ B, int ldb, double beta,
                                  double* __restrict__ C, int ldc) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  int i = e / n, j = e - i * n;
  double s = 0.0;
  for (int p = 0; p < k; ++p) {
    double av = ta ? A[p * lda + i] : A[i * lda + p];
    double bv = tb ? B[j * ldb + p] : B[p * ldb + j];
    s = fma(av, bv, s);
  }
  double c = alpha * s;
  if (beta != 0.0) c = fma(beta, C[i * ldc + j], c);
  C[i * ldc + j] = c;
}

__global__ void factor_gradient_kernel(const double* __restrict__ uh, int64_t rows,
                                       const double* __restrict__ g,
                                       const double* __restrict__ mtt,
                                       const double* __restrict__ lam, int R,
                                       double* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * R) return;
  int64_t i = e / R;
  int r = (int)(e - i * R);
  double s = 0.0;
  for (int q = 0; q < R; ++q) s = fma(uh[i * R + q], g[q * R + r] * (lam[q] * lam[r]), s);
  out[e] = s - mtt[e] * lam[r];
}

}  // namespace cb

// ============================================================================
// C ABI
// ============================================================================
using namespace cb;

extern "C" {

const char* cb_last_error(void) { return g_err; }
int cb_abi_version(void) { return CB_ABI_VERSION; }
long long cb_launch_count(void) { return g_launches; }
void cb_launch_count_reset(void) { g_launches = 0; }

int cb_mttkrp(int dtype, const void* X, int order, const int64_t* dims,
              const double* const* factors, int rank, int mode, double* out, void* stream) {
  CB_ARG(order >= 1 && order <= CB_MAX_ORDER, "order %d outside [1, %d]", order, CB_MAX_ORDER);
  CB_ARG(rank >= 1 && rank <= CB_MAX_RANK, "rank %d outside [1, %d]", rank, CB_MAX_RANK);
  CB_ARG(mode >= 0 && mode < order, "mode %d out of range for order-%d tensor", mode, order);
  CB_ARG(dtype == CB_F32 || dtype == CB_F64, "bad dtype %d", dtype);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t L = 1, H = 1;
  for (int m = 0; m < mode; ++m) L *= dims[m];
  for (int m = mode + 1; m < order; ++m) H *= dims[m];
  double* scratch = nullptr;
  size_t sbytes = sizeof(double) * (size_t)(L + H) * rank;
  CB_CUDA(cudaMallocAsync((void**)&scratch, sbytes, st));
  int rc = mttkrp_one(dtype, X, order, dims, factors, rank, mode, out, scratch, st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int cb_khatri_rao(const double* const* mats, int nmats, const int64_t* rows, int rank,
                  double* out, void* stream) {
  CB_ARG(nmats >= 1 && nmats <= CB_MAX_ORDER, "khatri_rao needs 1..%d matrices", CB_MAX_ORDER);
  CB_ARG(rank >= 1, "rank must be >= 1");
  KrArgs a{};
  a.nmats = nmats; a.rank = rank;
  for (int m = 0; m < nmats; ++m) {   // reference order: first slowest -> reverse
    a.mats[m] = mats[nmats - 1 - m];
    a.rows[m] = rows[nmats - 1 - m];
  }
  return launch_kr_first_fastest(a, out, (cudaStream_t)stream);
}

int cb_hadamard_gram(const double* const* mats, const double* const* mats2,
                     const int64_t* rows, int nmodes, int skip, int ra, int rb, double* out,
                     void* stream) {
  CB_ARG(nmodes >= 1 && nmodes <= CB_MAX_ORDER, "bad mode count %d", nmodes);
  int kept = 0;
  for (int m = 0; m < nmodes; ++m) kept += (m != skip);
  CB_ARG(kept > 0, "no matrices left after skip");
  HgArgs a{};
  a.nmodes = nmodes; a.skip = skip; a.ra = ra; a.rb = rb;
  for (int m = 0; m < nmodes; ++m) {
    a.A[m] = mats[m];
    a.B[m] = mats2 ? mats2[m] : mats[m];
    a.rows[m] = rows[m];
  }
  int n = ra * rb;
  if (n == 0) return CB_OK;
  hadamard_gram_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(a, out);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

int cb_spectral_norm_batched(const double* g, int r, int batch, double* out, void* stream) {
  CB_ARG(r >= 1 && r <= CB_MAX_RANK, "matrix size %d outside [1, %d]", r, CB_MAX_RANK);
  if (batch <= 0) return CB_OK;
  size_t sm = lam_max_smem_bytes(r);
  CB_CUDA(cudaFuncSetAttribute(spectral_batched_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  spectral_batched_kernel<<<batch, 256, sm, (cudaStream_t)stream>>>(g, r, out);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

int cb_tensor_stats(int dtype, const void* X, int64_t n, double* out3, void* stream) {
  CB_ARG(dtype == CB_F32 || dtype == CB_F64, "bad dtype %d", dtype);
  cudaStream_t st = (cudaStream_t)stream;
  int nparts = (int)((n + 255) / 256);
  if (nparts > 148 * 8) nparts = 148 * 8;
  if (nparts < 1) nparts = 1;
  double* part = nullptr;
  CB_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * 3 * nparts, st));
  int rc = tensor_stats(dtype, X, n, out3, part, nparts, st);
  cudaFreeAsync(part, st);
  return rc;
}

int cb_kruskal_residual(int dtype, const void* X, int order, const int64_t* dims,
                        const double* const* factors, const double* weights, int rank,
                        double* out, void* stream) {
  CB_ARG(order >= 1 && order <= CB_MAX_ORDER, "bad order %d", order);
  cudaStream_t st = (cudaStream_t)stream;
  ResidArgs a{};
  a.order = order; a.R = rank; a.w = weights; a.n = 1;
  for (int m = 0; m < order; ++m) { a.dims[m] = dims[m]; a.U[m] = factors[m]; a.n *= dims[m]; }
  int nparts = (int)((a.n + 255) / 256);
  if (nparts > 148 * 8) nparts = 148 * 8;
  if (nparts < 1) nparts = 1;
  double* part = nullptr;
  CB_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * nparts, st));
  int rc = kruskal_residual(dtype, a, X, out, part, nparts, st);
  cudaFreeAsync(part, st);
  return rc;
}

int cb_rowdot(const double* a, const double* b, int64_t rows, int r, double* out, void* stream) {
  if (r <= 0) return CB_OK;
  rowdot_kernel<<<r, 256, 0, (cudaStream_t)stream>>>(a, b, rows, r, out);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

int cb_gemm(int ta, int tb, int m, int n, int k, double alpha, const double* a, int lda,
            const double* b, int ldb, double beta, double* c, int ldc, void* stream) {
  if (m <= 0 || n <= 0) return CB_OK;
  gemm_small_kernel<<<(m * n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

int cb_factor_gradient(const double* u_hat, int64_t rows, const double* gram_skip,
                       const double* mtt, const double* lam, int r, double* out,
                       void* stream) {
  int64_t n = rows * r;
  if (n == 0) return CB_OK;
  factor_gradient_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      u_hat, rows, gram_skip, mtt, lam, r, out);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

}  // extern "C"
