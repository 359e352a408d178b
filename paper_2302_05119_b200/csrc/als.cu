// CP-ALS compression engine (lraCoNCPD-APG stage 1), batched over blocks.
//
// Restates cpd_als (pkg/src/concpd/cpd_als.py:52-120) on the device: per
// sweep and mode an MTTKRP, the Hadamard product of the other grams, the
// ridge 1e-12 tr(v)/R, an LU-with-partial-pivoting solve (the reference uses
// LAPACK gesv) and a gram refresh; after each sweep the explicit residual
// ||M - [[U]]|| and the per-block stop rule |rel_prev - rel| < tol.
// 3-way blocks use the fiber / contract / slab kernels (two tensor passes per
// sweep: the residual rides on the next sweep's fiber pass); other orders use
// the generic MTTKRP and residual kernels.
//
// fp32-storage throughput mode with ranks > 16 (c5): both tensor passes of a
// sweep are register-tiled fp64 GEMMs over TMA boxes (xslab5.cu: mode-2
// D = X_r A0, and T = X x3 A2), and the residual is the gram expansion
// ||M||^2 - 2 <A2, MTT2> + 1^T (G0 * G1 * G2) 1 (mathematically the explicit
// residual; its rounding, ~1e-16 ||M||^2 / res relative, is far below the
// fp32 storage rounding these blocks already carry).  The fp64 parity mode
// keeps the explicit residual.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "engine_host.h"
#include "ops_internal.h"
#include "status.h"
#include "xoz.h"
#include "xslab5.h"

namespace cb {

struct AlsState {
  int tsel;
  int any_active;
  int error;        // CB_ERR_DIVERGED
  int err_block;
  int err_sweep;
};

struct AlsCtx {
  int S, N, max_iter;
  double tol;
  const long long* dims;
  const int* R;
  double* const* U;        // S*N
  double* const* UT;       // S*N transposed factors [r][I_n], written by the solve (3-way)
  double* const* G;        // S*N
  double* const* MTT;      // S
  int* active;             // S
  int* n_iter;             // S
  int* converged;          // S
  double* rel;             // S current rel err
  double* norm;            // S ||M||
  double* hist;            // S * max_iter
  double* res;             // S (generic residuals, or the gram expansion)
  const double* nsq;       // S ||M||^2
  int res_expand;          // residual from the gram expansion (k_als_solve, last mode)
  const double* rpart;     // fiber residual partials
  const int* fib_first;
  const double* slab_part;
  const int* slab_first;
  const int* slab_nchunk;
  int slab_sb;
  int fast3;
  AlsState* st;
};

// u = solve(v + ridge I, mtt^T)^T, v = hadamard_{m != n} G_m (cpd_als.py:94-104)
__global__ void __launch_bounds__(256) k_als_solve(AlsCtx c, int n, int src) {
  const int s = blockIdx.x;
  if (!c.active[s]) return;
  extern __shared__ double sm[];
  const int R = c.R[s];
  const int N = c.N;
  const long long In = c.dims[s * N + n];
  double* A = sm;                 // R x R (LU in place)
  int* piv = reinterpret_cast<int*>(A + R * R);
  double* red = A + R * R + (R + 1) / 2 + 1;
  __shared__ double s_ridge;
  __shared__ int s_p;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double v = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) v *= c.G[s * N + m][e];
    A[e] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < R; ++i) tr += A[i * R + i];
    s_ridge = 1e-12 * tr / R;
  }
  __syncthreads();
  const double ridge = s_ridge;
  double* U = c.U[s * N + n];
  double* Ut = c.UT ? c.UT[s * N + n] : nullptr;
  if (!(ridge > 0.0)) {
    // the Khatri-Rao columns vanish: any factor fits, the reference takes 0
    for (long long e = threadIdx.x; e < In * R; e += blockDim.x) U[e] = 0.0;
    if (Ut)
      for (long long e = threadIdx.x; e < In * R; e += blockDim.x) Ut[e] = 0.0;
  } else {
    for (int i = threadIdx.x; i < R; i += blockDim.x) A[i * R + i] += ridge;
    __syncthreads();
    // LU with partial pivoting (getrf order: first max |a_ik| as pivot)
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
          const double t = A[k * R + j];
          A[k * R + j] = A[p * R + j];
          A[p * R + j] = t;
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
    // each row of mtt is one right-hand side
    const double* M = c.MTT[s];
    for (long long i = threadIdx.x; i < In; i += blockDim.x) {
      double y[CB_MAX_RANK];
      for (int r = 0; r < R; ++r) {
        if (src == 0) {
          y[r] = M[i * R + r];
        } else {
          const int sb = c.slab_sb;
          const long long g = i / sb;
          const int mm = (int)(i - g * sb);
          const int nch = c.slab_nchunk[s];
          const long long base = c.slab_first[s] + g * nch;
          double a = 0.0;
          for (int ch = 0; ch < nch; ++ch) a += c.slab_part[((base + ch) * sb + mm) * RSTRIDE + r];
          y[r] = a;
        }
      }
      for (int k = 0; k < R; ++k) {
        const int p = piv[k];
        if (p != k) { const double t = y[k]; y[k] = y[p]; y[p] = t; }
      }
      for (int r = 0; r < R; ++r) {
        double a = y[r];
        for (int q = 0; q < r; ++q) a -= A[r * R + q] * y[q];
        y[r] = a;
      }
      for (int r = R - 1; r >= 0; --r) {
        double a = y[r];
        for (int q = r + 1; q < R; ++q) a -= A[r * R + q] * y[q];
        y[r] = a / A[r * R + r];
      }
      for (int r = 0; r < R; ++r) U[i * R + r] = y[r];
      if (Ut)
        for (int r = 0; r < R; ++r) Ut[r * In + i] = y[r];
    }
  }
  __syncthreads();
  // gram refresh (cpd_als.py:106) and divergence flag
  double* Gn = c.G[s * N + n];
  double bad = 0.0;
  if (Ut) {
    // from the transposed copy: the two columns of an entry are contiguous
    // (one warp per entry p <= q, lanes over the rows, mirrored)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int p = 0; p < R; ++p) {
      const double* ap = Ut + (long long)p * In;
      for (int q = p + wid; q < R; q += nw) {
        const double* bq = Ut + (long long)q * In;
        double g = 0.0;
        for (long long i = lane; i < In; i += 32) g = fma(ap[i], bq[i], g);
        g = warp_sum(g);
        if (lane == 0) {
          Gn[p * R + q] = g;
          Gn[q * R + p] = g;
          if (!isfinite(g)) bad = 1.0;
        }
      }
    }
  } else {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int p = e / R, q = e - p * R;
      double g = 0.0;
      for (long long i = 0; i < In; ++i) g = fma(U[i * R + p], U[i * R + q], g);
      Gn[e] = g;
      if (!isfinite(g)) bad = 1.0;
    }
  }
  bad = block_max(bad, red);
  if (threadIdx.x == 0 && bad > 0.0) c.converged[s] = -1;   // diverged marker
  if (c.res_expand && n == N - 1) {
    // ||M - [[U]]||^2 = ||M||^2 - 2 sum_ir U[i,r] MTT[i,r] + 1^T (had_m G_m) 1
    __syncthreads();
    const double* M = c.MTT[s];
    double in = 0.0;
    for (long long e = threadIdx.x; e < In * R; e += blockDim.x) in = fma(U[e], M[e], in);
    in = block_sum(in, red);
    double ms = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      double v = 1.0;
      for (int m = 0; m < N; ++m) v *= c.G[s * N + m][e];
      ms += v;
    }
    ms = block_sum(ms, red);
    if (threadIdx.x == 0) c.res[s] = c.nsq[s] - 2.0 * in + ms;
  }
}

// initial grams G_n = U_n^T U_n of every (block, mode) in one launch
// (cpd_als.py:82), the same in-order row sums as the solve's gram refresh
__global__ void __launch_bounds__(256) k_als_init_grams(AlsCtx c) {
  const int s = blockIdx.x / c.N, n = blockIdx.x - (blockIdx.x / c.N) * c.N;
  const int R = c.R[s];
  const long long In = c.dims[s * c.N + n];
  const double* U = c.U[s * c.N + n];
  double* Gn = c.G[s * c.N + n];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int p = e / R, q = e - p * R;
    double g = 0.0;
    for (long long i = 0; i < In; ++i) g = fma(U[i * R + p], U[i * R + q], g);
    Gn[e] = g;
  }
}

// deferred start (cb_als_desc.ready_events): blocks [lo, hi) have arrived:
// their norms and initial rel err from the device stats (1, or 0 for a zero
// tensor: cpd_als.py:84-86), the activity flags, and the mask of exactly
// these blocks for their first T pass
__global__ void k_als_activate(AlsCtx c, int lo, int hi, const double* stats, double* nsq,
                               int* mask) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= c.S) return;
  const bool in = s >= lo && s < hi;
  mask[s] = in ? 1 : 0;
  if (!in) return;
  if (stats[3 * s + 2] > 0.0) {
    // non-finite values: reported by cb_als_run
    if (atomicCAS(&c.st->error, 0, CB_ERR_ARG) == 0) { c.st->err_block = s; c.st->err_sweep = 0; }
    c.active[s] = 0;
    mask[s] = 0;
    return;
  }
  const double nr = sqrt(stats[3 * s]);
  c.norm[s] = nr;
  nsq[s] = stats[3 * s];
  c.rel[s] = nr == 0.0 ? 0.0 : 1.0;
  c.active[s] = c.max_iter > 0 ? 1 : 0;
  if (c.active[s]) c.st->any_active = 1;
}

// the sweep state into the pinned host copy by a kernel store (not a D2H
// copy: while uploads are in flight a copy-engine transfer queues behind them)
__global__ void k_als_state_to_host(const AlsState* d, AlsState* h) { *h = *d; }

// per-sweep bookkeeping: residual -> rel err, history, stop rule (cpd_als.py:107-117)
__global__ void k_als_control(AlsCtx c, int init) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  AlsState* st = c.st;
  int any = 0;
  for (int s = 0; s < c.S; ++s) {
    if (!c.active[s]) continue;
    if (!init) {
      if (c.converged[s] == -1) {
        if (!st->error) { st->error = CB_ERR_DIVERGED; st->err_block = s; st->err_sweep = c.n_iter[s] + 1; }
        c.active[s] = 0;
        continue;
      }
      double res = 0.0;
      if (c.fast3 && !c.res_expand) {
        res = c.rpart[s];   // per-block total folded by the fiber kernel
      } else {
        res = c.res[s];
      }
      const int it = c.n_iter[s] + 1;
      c.n_iter[s] = it;
      const double nr = c.norm[s];
      const double rel = nr > 0.0 ? sqrt(res > 0.0 ? res : 0.0) / nr : 0.0;
      c.hist[(long long)s * c.max_iter + it - 1] = rel;
      const bool stop = fabs(c.rel[s] - rel) < c.tol;
      c.rel[s] = rel;
      if (stop) { c.converged[s] = 1; c.active[s] = 0; }
      else if (it >= c.max_iter) c.active[s] = 0;
    } else if (c.max_iter <= 0) {
      c.active[s] = 0;
    }
    any |= c.active[s];
  }
  st->tsel ^= 1;   // the fiber pass wrote the other T buffer
  st->any_active = any;
}

}  // namespace cb

using namespace cb;

struct cb_als {
  cudaStream_t st = nullptr;
  cb::Sl5Plan* sl5 = nullptr;   // fp64 mode-2 MTTKRP for ranks > 16 (xslab5.cu)
  cb::OzPlan* oz = nullptr;     // both passes on the tensor cores over packed byte planes (xoz.cu)
  // deferred start: per-block upload events, blocks [0, started) are running
  bool deferred = false;
  bool released = false;        // cb_als_release_scratch was called
  std::vector<cudaEvent_t> ready;
  int started = 0;
  double* d_stats = nullptr;
  double* d_stats_part = nullptr;
  double* d_nsq = nullptr;
  int* d_mask = nullptr;
  int S = 0, N = 0, dtype = CB_F64, max_iter = 0, rmax = 1, rb = 8, fast3 = 0, pc = 0;
  double tol = 1e-4;
  std::vector<long long> dims;
  std::vector<int> R;
  std::vector<const void*> X;
  std::vector<void*> allocs;
  std::vector<double*> h_U, h_MTT;
  AlsCtx ctx{};
  XArgs xa{};
  XTables tab;
  FibUnit* d_fib = nullptr;
  SlabUnit* d_slab = nullptr;
  RowUnit *d_c0 = nullptr, *d_c1 = nullptr;
  AlsState* d_state = nullptr;
  AlsState* h_state = nullptr;
  AlsState* h_state_dev = nullptr;   // device address of the pinned host copy
  double* kr_scratch = nullptr;
  double* res_part = nullptr;
  int res_nparts = 0;
  size_t solve_smem = 0;
  bool tma = false;
};

namespace cb {

static int als_residuals(cb_als* h) {
  for (int s = 0; s < h->S; ++s) {
    ResidArgs a{};
    a.order = h->N; a.R = h->R[s]; a.n = 1; a.w = nullptr;
    for (int m = 0; m < h->N; ++m) {
      a.dims[m] = h->dims[s * h->N + m];
      a.U[m] = h->h_U[s * h->N + m];
      a.n *= a.dims[m];
    }
    int rc = kruskal_residual(h->dtype, a, h->X[s], h->ctx.res + s, h->res_part, h->res_nparts, h->st);
    if (rc) return rc;
  }
  return CB_OK;
}

static int als_sweep(cb_als* h) {
  cudaStream_t st = h->st;
  for (int n = 0; n < h->N; ++n) {
    int src = 0;
    if (h->fast3) {
      if (n < 2) {
        launch_contract(h->pc, n, h->xa, n == 0 ? h->d_c0 : h->d_c1,
                        (int)(n == 0 ? h->tab.c0.size() : h->tab.c1.size()), st);
      } else {
        if (h->oz) {
          // exact int8 slice GEMM over the packed planes (xoz.cu), written into MTT
          int rc = oz_mode2(h->oz, h->xa.U, h->xa.active, h->xa.MTT, st, h->xa.UT);
          if (rc) return rc;
        } else if (h->sl5) {
          // fp64 GEMM-tiled mode-2 MTTKRP (xslab5.cu), written into MTT
          int rc = sl5_mode2(h->sl5, h->xa.U, h->xa.active, h->xa.MTT, st);
          if (rc) return rc;
        } else {
          launch_slab(h->pc, h->rb, h->tma, h->xa, h->d_slab, (int)h->tab.slab.size(), h->tab, st);
          src = h->tab.slab_direct ? 0 : 1;   // the row-dot kernel writes MTT itself
        }
      }
      CB_CHECK_LAUNCH();
    } else {
      for (int s = 0; s < h->S; ++s) {
        std::vector<const double*> f(h->N);
        for (int m = 0; m < h->N; ++m) f[m] = h->h_U[s * h->N + m];
        int rc = mttkrp_one(h->dtype, h->X[s], h->N, reinterpret_cast<const int64_t*>(&h->dims[s * h->N]), f.data(), h->R[s], n,
                            h->h_MTT[s], h->kr_scratch, st);
        if (rc) return rc;
      }
    }
    k_als_solve<<<h->S, 256, h->solve_smem, st>>>(h->ctx, n, src);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  if (h->fast3 && h->ctx.res_expand) {
    // T for the next sweep (GEMM pass); the residual came from the expansion
    int rc = h->oz ? oz_tpass(h->oz, h->xa.U, h->xa.active, h->xa.T0, h->xa.T1, h->xa.tsel, 1, st)
                   : sl5_tpass(h->sl5, h->xa.U, h->xa.active, h->xa.T0, h->xa.T1, h->xa.tsel, 1, st);
    if (rc) return rc;
    CB_CHECK_LAUNCH();
  } else if (h->fast3) {
    XArgs a = h->xa;
    a.t_other = 1;
    launch_fiber(h->pc, h->rb, h->tma, 1, 0, 1, a, h->d_fib, (int)h->tab.fib.size(), h->tab, st);
    CB_CHECK_LAUNCH();
  } else {
    int rc = als_residuals(h);
    if (rc) return rc;
  }
  k_als_control<<<1, 32, 0, st>>>(h->ctx, 0);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

}  // namespace cb

extern "C" {

int cb_als_destroy(cb_als* h) {
  if (!h) return CB_OK;
  if (h->st) cudaStreamSynchronize(h->st);
  dfree_all(h->allocs);
  cb::sl5_plan_destroy(h->sl5);
  cb::oz_plan_destroy(h->oz);
  if (h->h_state) cudaFreeHost(h->h_state);
  delete h;
  return CB_OK;
}

// would cb_als_create take the staged path (start each block at its
// ready_event) for these blocks?  (3-way fp32 storage, fp64-grade arithmetic,
// ranks and mode sizes the plane GEMMs support)
int cb_als_staged_ok(const cb_als_desc* d) {
  if (!d || d->n_blocks < 1 || d->order != 3 || d->dtype != CB_F32 || d->compute == 1) return 0;
  const int S = d->n_blocks;
  std::vector<long long> dims(d->dims, d->dims + 3 * S);
  std::vector<int> R(d->ranks, d->ranks + S);
  int rmax = 1;
  for (int s = 0; s < S; ++s) {
    if (R[s] < 1 || R[s] > CB_MAX_RANK) return 0;
    rmax = std::max(rmax, R[s]);
  }
  std::vector<const void*> X(S, reinterpret_cast<const void*>(16));   // alignment only
  if (!oz_supported(S, X.data(), dims.data(), R.data())) return 0;
  XTables tab;
  build_xtables(S, dims.data(), R.data(), rank_bucket(rmax), PC_F32_F64, tab,
                d->total_blocks > S ? d->total_blocks : S);
  return tab.slab_direct ? 0 : 1;
}

int cb_als_create(const cb_als_desc* d, void* stream, cb_als** out) {
  CB_ARG(d && out, "null descriptor");
  *out = nullptr;
  CB_ARG(d->n_blocks >= 1, "no tensors");
  CB_ARG(d->order >= 1 && d->order <= CB_MAX_ORDER, "order %d outside [1, %d]", d->order, CB_MAX_ORDER);
  CB_ARG(d->tol > 0.0, "tol must be positive");
  CB_ARG(d->max_iter >= 0, "max_iter must be >= 0");
  cb_als* h = new cb_als();
  h->st = (cudaStream_t)stream;
  h->S = d->n_blocks; h->N = d->order; h->dtype = d->dtype; h->tol = d->tol;
  h->pc = d->dtype == CB_F64 ? PC_F64 : (d->compute == 1 ? PC_F32 : PC_F32_F64);
  h->max_iter = d->max_iter;
  const int S = h->S, N = h->N;
  h->dims.assign(d->dims, d->dims + S * N);
  h->R.assign(d->ranks, d->ranks + S);
  h->X.assign(d->tensors, d->tensors + S);
  for (int s = 0; s < S; ++s) {
    if (h->R[s] < 1 || h->R[s] > CB_MAX_RANK) {
      delete h;
      set_error("rank %d outside [1, %d]", d->ranks[s], CB_MAX_RANK);
      return CB_ERR_UNSUPPORTED;
    }
    h->rmax = std::max(h->rmax, h->R[s]);
  }
  h->fast3 = (N == 3);
  h->rb = rank_bucket(h->rmax);
  cudaStream_t st = h->st;
  set_alloc_stream(st);
  std::vector<void*>& A = h->allocs;
  int rc;
#define TRY(x) do { rc = (x); if (rc) { cb_als_destroy(h); return rc; } } while (0)
  std::vector<double*> U(S * N), G(S * N), MTT(S), UT(S * N, nullptr);
  std::vector<double> norms(S);
  for (int s = 0; s < S; ++s) {
    long long mI = 0;
    for (int n = 0; n < N; ++n) {
      const long long In = h->dims[s * N + n];
      mI = std::max(mI, In);
      TRY(dalloc((void**)&U[s * N + n], sizeof(double) * In * h->R[s], A));
      TRY(dalloc((void**)&G[s * N + n], sizeof(double) * h->R[s] * h->R[s], A));
      if (h->fast3) TRY(dalloc((void**)&UT[s * N + n], sizeof(double) * In * h->R[s], A));
    }
    TRY(dalloc((void**)&MTT[s], sizeof(double) * mI * h->R[s], A));
  }
  h->h_U = U;
  h->h_MTT = MTT;
  AlsCtx& c = h->ctx;
  c.S = S; c.N = N; c.max_iter = h->max_iter; c.tol = h->tol; c.fast3 = h->fast3;
  long long* dd; int* dr;
  TRY(upload(h->dims, &dd, A, st)); c.dims = dd;
  TRY(upload(h->R, &dr, A, st)); c.R = dr;
  double** p;
  TRY(upload(U, &p, A, st)); c.U = p;
  c.UT = nullptr;
  if (h->fast3) { TRY(upload(UT, &p, A, st)); c.UT = p; }
  TRY(upload(G, &p, A, st)); c.G = p;
  TRY(upload(MTT, &p, A, st)); c.MTT = p;
  TRY(dalloc((void**)&c.active, sizeof(int) * S, A));
  TRY(dalloc((void**)&c.n_iter, sizeof(int) * S, A));
  TRY(dalloc((void**)&c.converged, sizeof(int) * S, A));
  TRY(dalloc((void**)&c.rel, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.norm, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.hist, sizeof(double) * S * std::max(h->max_iter, 1), A));
  TRY(dalloc((void**)&c.res, sizeof(double) * S, A));
  TRY(dalloc((void**)&h->d_state, sizeof(AlsState), A));
  c.st = h->d_state;
  CB_CUDA(cudaMallocHost((void**)&h->h_state, sizeof(AlsState)));
  memset(h->h_state, 0, sizeof(AlsState));
  CB_CUDA(cudaHostGetDevicePointer((void**)&h->h_state_dev, h->h_state, 0));
  // unit tables and the tensor-core plan first: its allocations (the byte
  // planes: 34 GB on c5, ~0.1 s of host time) then run while the caller's
  // host->device copies of the blocks are still in flight on `st`, ahead of
  // the synchronisation below; its pack kernels queue behind those copies
  if (h->fast3) {
    build_xtables(S, h->dims.data(), h->R.data(), h->rb, h->pc, h->tab,
                  d->total_blocks > S ? d->total_blocks : S);
    h->tma = tma_rows_ok(S, h->dims.data(), h->X.data(), h->dtype == CB_F32 ? 4 : 8);
    // fp32 storage with fp64-grade arithmetic, ranks in (16, 48]: both tensor
    // passes of a sweep as exact int8 slice GEMMs over byte planes packed once
    // (xoz.cu).  T is then written unsplit whatever the fiber table chose.
    if (h->pc == PC_F32_F64 && !h->tab.slab_direct &&
        oz_supported(S, h->X.data(), h->dims.data(), h->R.data())) {
      if (oz_plan_create(S, h->X.data(), h->dims.data(), h->R.data(), st, &h->oz,
                         d->ready_events != nullptr) != CB_OK)
        h->oz = nullptr;
      if (h->oz) {
        h->tab.nsplit.assign(S, 1);
        h->tab.fib_unsplit = 1;
      }
    }
  }
  // blocks still uploading (ready_events): the plane-GEMM path starts each
  // block as it arrives (cb_als_run); any other path waits for all of them here
  if (d->ready_events) {
    h->ready.resize(S);
    for (int s = 0; s < S; ++s) h->ready[s] = (cudaEvent_t)d->ready_events[s];
    h->deferred = h->oz != nullptr;
    if (h->deferred) {
      // every kernel of the staged run is loaded now, before the caller
      // starts the uploads: with lazy module loading a kernel's first launch
      // waits for all copies in flight
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, k_als_activate);
      cudaFuncGetAttributes(&fa, k_als_state_to_host);
      cudaFuncGetAttributes(&fa, k_als_solve);
      cudaFuncGetAttributes(&fa, k_als_control);
      tensor_stats_preload();
      contract_preload();
      oz_preload(h->oz);
    }
    if (!h->deferred) {
      // cb_als_staged_ok said yes but the plan could not be built (device
      // memory): the caller falls back to uploading first (the events may
      // not have been recorded yet, so nothing can be read here)
      cb_als_destroy(h);
      set_error("staged start unavailable (the plane-GEMM plan could not be created)");
      return CB_ERR_UNSUPPORTED;
    }
  }
  // the starting factors (pageable host memory: these copies wait for the
  // stream, so they come after every allocation above)
  for (int s = 0; s < S; ++s)
    for (int n = 0; n < N; ++n)
      CB_CUDA(cudaMemcpyAsync(U[s * N + n], d->init[s * N + n],
                              sizeof(double) * h->dims[s * N + n] * h->R[s],
                              cudaMemcpyHostToDevice, st));
  // norms and the initial rel err (1, or 0 for a zero tensor: cpd_als.py:84-86)
  if (h->deferred) {
    // per arriving range in cb_als_run (k_als_activate), from device stats
    TRY(dalloc((void**)&h->d_stats, sizeof(double) * 3 * S, A));
    TRY(dalloc((void**)&h->d_stats_part, sizeof(double) * 3 * 148 * 8, A));
    TRY(dalloc((void**)&h->d_nsq, sizeof(double) * S, A));
    TRY(dalloc((void**)&h->d_mask, sizeof(int) * S, A));
    c.nsq = h->d_nsq;
  } else {
    double* stats;
    TRY(dalloc((void**)&stats, sizeof(double) * 3 * S, A));
    double* part;
    TRY(dalloc((void**)&part, sizeof(double) * 3 * 148 * 8, A));
    for (int s = 0; s < S; ++s) {
      long long n = 1;
      for (int m = 0; m < N; ++m) n *= h->dims[s * N + m];
      int np = (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + 255) / 256));
      TRY(tensor_stats(h->dtype, h->X[s], n, stats + 3 * s, part, np, st));
    }
    std::vector<double> hs(3 * S);
    CB_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(double) * 3 * S, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
    std::vector<double> rel0(S);
    std::vector<int> act(S, h->max_iter > 0 ? 1 : 0);
    for (int s = 0; s < S; ++s) {
      if (hs[3 * s + 2] > 0.0) {
        cb_als_destroy(h);
        set_error("tensor contains non-finite values");
        return CB_ERR_ARG;
      }
      norms[s] = sqrt(hs[3 * s]);
      rel0[s] = norms[s] == 0.0 ? 0.0 : 1.0;
    }
    CB_CUDA(cudaMemcpyAsync(c.norm, norms.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    std::vector<double> sq(S);
    for (int s = 0; s < S; ++s) sq[s] = hs[3 * s];
    double* dnsq;
    TRY(dalloc((void**)&dnsq, sizeof(double) * S, A));
    CB_CUDA(cudaMemcpyAsync(dnsq, sq.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    c.nsq = dnsq;
    CB_CUDA(cudaMemcpyAsync(c.rel, rel0.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaMemcpyAsync(c.active, act.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaStreamSynchronize(st));
  }
  // initial grams (cpd_als.py:82): one launch for every (block, mode)
  k_als_init_grams<<<S * N, 256, 0, st>>>(h->ctx);
  count_launch(1);
  CB_CHECK_LAUNCH();
  if (h->fast3) {
    prepare_slab(h->pc, h->rb, h->tma, h->tab);
    prepare_fiber(h->pc, h->rb, h->tma, h->tab);
    TRY(upload(h->tab.fib, &h->d_fib, A, st));
    TRY(upload(h->tab.slab, &h->d_slab, A, st));
    TRY(upload(h->tab.c0, &h->d_c0, A, st));
    TRY(upload(h->tab.c1, &h->d_c1, A, st));
    int* di;
    TRY(upload(h->tab.fib_first, &di, A, st)); c.fib_first = di;
    TRY(upload(h->tab.slab_first, &di, A, st)); c.slab_first = di;
    TRY(upload(h->tab.slab_nchunk, &di, A, st)); c.slab_nchunk = di;
    c.slab_sb = h->tab.sb;
    int* d_ns;
    TRY(upload(h->tab.nsplit, &d_ns, A, st));
    double *bpart, *rpart, *spart, *bsum, *rsum;
    int* blk_cnt;
    TRY(dalloc((void**)&bpart, sizeof(double) * h->tab.fib.size() * RSTRIDE, A));
    TRY(dalloc((void**)&rpart, sizeof(double) * h->tab.fib.size(), A));
    TRY(dalloc((void**)&bsum, sizeof(double) * S * RSTRIDE, A));
    TRY(dalloc((void**)&rsum, sizeof(double) * S, A));
    TRY(dalloc((void**)&blk_cnt, sizeof(int) * S, A));
    TRY(dalloc((void**)&spart,
               h->oz ? 8 : sizeof(double) * h->tab.slab.size() * h->tab.sb * RSTRIDE, A));
    c.rpart = rsum;
    c.slab_part = spart;
    std::vector<void*> T0(S), T1(S);
    const int eb = pc_compute_bytes(h->pc);
    if (h->oz) {
      // one unsplit T per block out of a single allocation: the T pass writes
      // every element before the contractions read it (no memset), and the
      // sweep is strictly sequential, so the two T selectors share a buffer
      size_t tot = 0;
      std::vector<size_t> ofs(S);
      for (int s = 0; s < S; ++s) {
        ofs[s] = tot;
        tot += ((size_t)h->R[s] * h->dims[3 * s] * h->dims[3 * s + 1] * eb + 255) & ~(size_t)255;
      }
      char* tbuf = nullptr;
      const cudaError_t te = cudaMalloc((void**)&tbuf, tot);
      if (te != cudaSuccess) {
        cb_als_destroy(h);
        return cuda_fail(te, "cudaMalloc (T buffers)", __FILE__, __LINE__);
      }
      A.push_back(tbuf);
      for (int s = 0; s < S; ++s) T0[s] = T1[s] = tbuf + ofs[s];
    } else {
      for (int s = 0; s < S; ++s) {
        const size_t tb = (size_t)h->tab.nsplit[s] * h->R[s] * h->dims[3 * s] * h->dims[3 * s + 1] * eb;
        TRY(dalloc(&T0[s], tb, A));
        TRY(dalloc(&T1[s], tb, A));
      }
    }
    void **pt0, **pt1;
    TRY(upload(T0, &pt0, A, st));
    TRY(upload(T1, &pt1, A, st));
    const void** pX;
    TRY(upload(h->X, &pX, A, st));
    XArgs& xa = h->xa;
    xa.X = pX; xa.dims = c.dims; xa.R = c.R; xa.U = (const double* const*)c.U; xa.LAM = nullptr;
    xa.UT = (const double* const*)c.UT;
    xa.T0 = pt0; xa.T1 = pt1; xa.tsel = &h->d_state->tsel; xa.t_other = 0;
    xa.nsplit = d_ns; xa.bpart = bpart; xa.rpart = rpart; xa.slab_part = spart;
    xa.MTT = c.MTT; xa.gate = nullptr; xa.active = c.active;
    xa.ktime = nullptr;
    xa.slab_stage_rows = h->tab.slab_rows;
    // fp64 arithmetic with ranks > 16: the GEMM-tiled mode-2 pass
    if (!h->oz && h->pc == PC_F32_F64 && !h->tab.slab_direct &&
        sl5_supported(S, h->X.data(), h->dims.data(), h->R.data())) {
      if (sl5_plan_create(S, h->X.data(), h->dims.data(), h->R.data(), st, &h->sl5) != CB_OK)
        h->sl5 = nullptr;
    }
    // both passes as GEMMs (unsplit T) with the gram-expansion residual
    c.res_expand = (h->oz || (h->sl5 && sl5_tpass_ok(h->sl5) && h->tab.fib_unsplit)) ? 1 : 0;
    {
      int* d_s3;
      TRY(upload(h->tab.s3_first, &d_s3, A, st));
      xa.s3_first = d_s3;
      int* d_f3;
      TRY(upload(h->tab.f3_first, &d_f3, A, st));
      xa.f3_first = d_f3;
    }
    xa.fib_first = c.fib_first; xa.blk_cnt = blk_cnt; xa.bsum = bsum; xa.rsum = rsum;
  } else {
    size_t kr = 0;
    for (int s = 0; s < S; ++s)
      for (int n = 0; n < N; ++n) {
        long long Lp = 1, Hp = 1;
        for (int m = 0; m < n; ++m) Lp *= h->dims[s * N + m];
        for (int m = n + 1; m < N; ++m) Hp *= h->dims[s * N + m];
        kr = std::max(kr, (size_t)(Lp + Hp) * h->R[s]);
      }
    TRY(dalloc((void**)&h->kr_scratch, sizeof(double) * kr, A));
    h->res_nparts = 148 * 4;
    TRY(dalloc((void**)&h->res_part, sizeof(double) * h->res_nparts, A));
  }
  h->solve_smem = sizeof(double) * ((size_t)h->rmax * h->rmax + h->rmax + 48);
  CB_CUDA(cudaFuncSetAttribute(k_als_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->solve_smem));
  // initial T buffer (X x_3 U_2 of the starting factors); deferred: per
  // arriving range in cb_als_run
  if (h->deferred) {
  } else if (h->fast3 && c.res_expand) {
    TRY(h->oz ? oz_tpass(h->oz, h->xa.U, h->xa.active, h->xa.T0, h->xa.T1, h->xa.tsel, 1, st)
              : sl5_tpass(h->sl5, h->xa.U, h->xa.active, h->xa.T0, h->xa.T1, h->xa.tsel, 1, st));
    CB_CHECK_LAUNCH();
  } else if (h->fast3) {
    XArgs a = h->xa;
    a.t_other = 1;
    launch_fiber(h->pc, h->rb, h->tma, 1, 0, 0, a, h->d_fib, (int)h->tab.fib.size(), h->tab, st);
    CB_CHECK_LAUNCH();
  }
  if (!h->deferred) {
    k_als_control<<<1, 32, 0, st>>>(h->ctx, 1);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
#undef TRY
  *out = h;
  return CB_OK;
}

// deferred start: activate the blocks [started, upto) that have arrived:
// stats, exponents + byte planes, norms / flags, their first T pass
static int als_activate(cb_als* h, int upto) {
  cudaStream_t st = h->st;
  const int lo = h->started;
  for (int s = lo; s < upto; ++s) {
    CB_CUDA(cudaStreamWaitEvent(st, h->ready[s], 0));
    long long n = 1;
    for (int m = 0; m < h->N; ++m) n *= h->dims[s * h->N + m];
    const int np = (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + 255) / 256));
    int rc = tensor_stats(h->dtype, h->X[s], n, h->d_stats + 3 * s, h->d_stats_part, np, st);
    if (rc) return rc;
  }
  int rc = oz_pack_range(h->oz, lo, upto, st);
  if (rc) return rc;
  k_als_activate<<<(h->S + 127) / 128, 128, 0, st>>>(h->ctx, lo, upto, h->d_stats, h->d_nsq,
                                                    h->d_mask);
  count_launch(1);
  CB_CHECK_LAUNCH();
  rc = oz_tpass(h->oz, h->xa.U, h->d_mask, h->xa.T0, h->xa.T1, h->xa.tsel, 1, st);
  if (rc) return rc;
  h->started = upto;
  return CB_OK;
}

static int als_finish(cb_als* h) {
  if (h->h_state->error == CB_ERR_ARG) {
    set_error("tensor contains non-finite values");
    return CB_ERR_ARG;
  }
  if (h->h_state->error) {
    set_error("block %d: ALS diverged to non-finite values at sweep %d", h->h_state->err_block,
              h->h_state->err_sweep);
    return CB_ERR_DIVERGED;
  }
  return CB_OK;
}

int cb_als_run(cb_als* h) {
  CB_ARG(h, "null handle");
  CB_ARG(!h->released, "cb_als_run after cb_als_release_scratch");
  if (h->deferred) {
    // start every block as its upload completes; between arrivals the
    // blocks already here sweep in short chunks
    const int S = h->S;
    h->h_state->any_active = 0;
    for (;;) {
      int upto = h->started;
      while (upto < S && cudaEventQuery(h->ready[upto]) == cudaSuccess) ++upto;
      if (upto == h->started && upto < S && !h->h_state->any_active) {
        // nothing to do until the next block is here
        CB_CUDA(cudaEventSynchronize(h->ready[upto]));
        continue;
      }
      if (upto > h->started) {
        int rc = als_activate(h, upto);
        if (rc) return rc;
      }
      const int chunk = h->started < S ? 2 : 8;
      for (int i = 0; i < chunk; ++i) {
        int rc = als_sweep(h);
        if (rc) return rc;
      }
      k_als_state_to_host<<<1, 1, 0, h->st>>>(h->d_state, h->h_state_dev);
      CB_CHECK_LAUNCH();
      CB_CUDA(cudaStreamSynchronize(h->st));
      if (h->h_state->error) break;
      if (h->started == S && !h->h_state->any_active) break;
    }
    return als_finish(h);
  }
  int sweeps = 0;
  CB_CUDA(cudaMemcpyAsync(h->h_state, h->d_state, sizeof(AlsState), cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaStreamSynchronize(h->st));
  while (h->h_state->any_active && sweeps < h->max_iter) {
    const int chunk = std::min(8, h->max_iter - sweeps);
    for (int i = 0; i < chunk; ++i) {
      int rc = als_sweep(h);
      if (rc) return rc;
    }
    sweeps += chunk;
    CB_CUDA(cudaMemcpyAsync(h->h_state, h->d_state, sizeof(AlsState), cudaMemcpyDeviceToHost, h->st));
    CB_CUDA(cudaStreamSynchronize(h->st));
  }
  return als_finish(h);
}

// frees what only the sweeps need (byte planes, D, fp64 GEMM scratch): the
// factors, histories and counters stay for cb_als_block_result /
// cb_als_factor_device.  c5: ~37 GB returned before the solver engine packs
// its own trace planes.  The handle cannot run again afterwards.
int cb_als_release_scratch(cb_als* h) {
  CB_ARG(h, "null handle");
  if (h->st) CB_CUDA(cudaStreamSynchronize(h->st));
  cb::oz_plan_destroy(h->oz);
  h->oz = nullptr;
  cb::sl5_plan_destroy(h->sl5);
  h->sl5 = nullptr;
  h->released = true;
  return CB_OK;
}

int cb_als_block_result(cb_als* h, int block, double* rel_err, int* n_iter, int* converged,
                        double* history, double* const* host_factors) {
  CB_ARG(h && block >= 0 && block < h->S, "bad block");
  const AlsCtx& c = h->ctx;
  if (rel_err) CB_CUDA(cudaMemcpyAsync(rel_err, c.rel + block, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  int it = 0, cv = 0;
  CB_CUDA(cudaMemcpyAsync(&it, c.n_iter + block, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaMemcpyAsync(&cv, c.converged + block, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaStreamSynchronize(h->st));
  if (n_iter) *n_iter = it;
  if (converged) *converged = cv == 1;
  if (history && it > 0)
    CB_CUDA(cudaMemcpyAsync(history, c.hist + (long long)block * h->max_iter, sizeof(double) * it,
                            cudaMemcpyDeviceToHost, h->st));
  if (host_factors)
    for (int n = 0; n < h->N; ++n)
      if (host_factors[n])
        CB_CUDA(cudaMemcpyAsync(host_factors[n], h->h_U[block * h->N + n],
                                sizeof(double) * h->dims[block * h->N + n] * h->R[block],
                                cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaStreamSynchronize(h->st));
  return CB_OK;
}

const double* cb_als_factor_device(cb_als* h, int block, int mode) {
  if (!h || block < 0 || block >= h->S || mode < 0 || mode >= h->N) return nullptr;
  return h->h_U[block * h->N + mode];
}

}  // extern "C"
