// Small fused kernels of the APG iteration (per-block Gram/Hadamard, Lipschitz
// constants, APG extrapolate/gradient/project, common-column aggregation,
// restart, evaluation and the device-side control rule).
//
// Reference: pkg/src/concpd/solver.py:311-624 (the _Apg state machine and the
// outer loop of solve()).  Every kernel is gated on device flags so that a
// whole iteration (including the restart branch) can be enqueued or captured
// in a CUDA graph without a host round trip.
#pragma once
#include "engine.h"
#include "../../include/concpd_b200.h"

namespace cb {

__device__ __forceinline__ bool stopped(const Ctx& c, int redo) {
  return redo ? (c.st->go_redo == 0) : (c.st->go_main == 0);
}
// np.maximum(0.0, x) semantics (NaN propagates)
__device__ __forceinline__ double pos(double x) { return x < 0.0 ? 0.0 : x; }

struct BlockSmem {
  double* lmA;    // lam_max workspace: A, B, B2, vec, red
  double* lmB;
  double* lmB2;
  double* vec;
  double* red;
  double* gr;     // gram staging 2 * gram_rows(gw) * gw
  int gw;
  double* misc;   // 4 * 64
};

// rows staged per gram chunk, double-buffered (chunk k + 1 in flight while
// chunk k is multiplied): the same shared memory as single 128 / 64-row
// chunks, so the per-block kernels keep two CTAs per SM at R = 40
__host__ __device__ __forceinline__ int gram_rows(int gw) { return gw <= 16 ? 64 : 32; }

__device__ __forceinline__ BlockSmem carve(double* sm, int rmax, int gw) {
  BlockSmem b;
  const int ld = lm_ld(rmax);
  const int Rp = (rmax + 3) & ~3;
  b.lmA = sm;
  b.lmB = b.lmA + Rp * ld;
  b.lmB2 = b.lmB + lm_bsize(rmax);
  b.vec = b.lmB2 + lm_bsize(rmax);
  b.red = b.vec + 128;
  b.gr = b.red + 40;
  b.gw = gw;
  b.misc = b.gr + 4 * gram_rows(gw) * gw;
  return b;
}

// gram staging: two buffers (double buffering) of A and B chunks
__host__ __device__ inline size_t block_smem_bytes(int rmax, int gw) {
  return sizeof(double) * ((size_t)lm_smem_doubles(rmax) + 4 * (size_t)gram_rows(gw) * gw + 4 * 64 + 8);
}

// out[P x Q] = A^T B with A rows x P, B rows x Q (row-major), whole block,
// fixed summation order over rows (deterministic: every output is one fma
// chain over the rows in order, whatever the staging).  Rows are staged in
// chunks of gram_rows(gw) (one round trip of loads per chunk); each thread
// owns a 4 x 4 register tile of outputs (16 FMAs per 8 shared loads per row).
static __device__ __noinline__ void block_gram(const double* __restrict__ A, int P, const double* __restrict__ B,
                           int Q, long long rows, double* __restrict__ out, const BlockSmem& sm) {
  const int CH = gram_rows(sm.gw);
  // a gram of one matrix with itself reads one staged copy; chunk k + 1 is
  // in flight while chunk k is multiplied (two buffers per operand)
  const bool same = (A == B) && (P == Q);
  auto bufA = [&](int b) { return sm.gr + (size_t)b * 2 * CH * sm.gw; };
  auto bufB = [&](int b) { return same ? bufA(b) : sm.gr + ((size_t)b * 2 + 1) * CH * sm.gw; };
  // small grams (P Q <= 256): one output per thread (more parallel rows
  // chains); larger: 4 x 4 tiles
  const bool t1 = P * Q <= 256;
  const int TP = t1 ? 1 : 4;
  const int ntp = (P + TP - 1) / TP, ntq = (Q + TP - 1) / TP;
  const int tile = threadIdx.x;                 // ntp * ntq <= 256 for P, Q <= 64
  const bool owner = tile < ntp * ntq;
  const int p0 = owner ? (tile / ntq) * TP : 0, q0 = owner ? (tile % ntq) * TP : 0;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  auto issue = [&](long long c0, int b) {
    const int nr = (int)(rows - c0 < CH ? rows - c0 : CH);
    stage_async(bufA(b), A + c0 * P, (long long)nr * P);
    if (!same) stage_async(bufB(b), B + c0 * Q, (long long)nr * Q);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();                 // the buffers may still be read by a previous call
  if (rows > 0) issue(0, 0);
  int buf = 0;
  for (long long c0 = 0; c0 < rows; c0 += CH, buf ^= 1) {
    const int nr = (int)(rows - c0 < CH ? rows - c0 : CH);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // chunk c0 visible to all; every thread is done with the previous chunk,
    // so its buffer takes the next one (in flight during this chunk's FMAs)
    __syncthreads();
    if (c0 + CH < rows) issue(c0 + CH, buf ^ 1);
    const double* As = bufA(buf);
    const double* Bs = bufB(buf);
    if (owner && t1) {
      double sacc = acc[0][0];
      for (int i = 0; i < nr; ++i) sacc = fma(As[i * P + p0], Bs[i * Q + q0], sacc);
      acc[0][0] = sacc;
    } else if (owner) {
      for (int i = 0; i < nr; ++i) {
        double a4[4], b4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a4[u] = p0 + u < P ? As[i * P + p0 + u] : 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v) b4[v] = q0 + v < Q ? Bs[i * Q + q0 + v] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(a4[u], b4[v], acc[u][v]);
      }
    }
  }
  if (owner && t1) {
    out[p0 * Q + q0] = acc[0][0];
  } else if (owner) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (p0 + u < P && q0 + v < Q) out[(p0 + u) * Q + q0 + v] = acc[u][v];
  }
  __syncthreads();
}

// Hadamard product of the block's grams over modes != skip (mode order,
// starting from ones: solver.py:352-358) times optional lam lam^T, into the
// lam_max matrix slot (leading dim lm_ld(R)).  Returns via smem.
static __device__ __noinline__ void build_gram_product(const Ctx& c, int s, int skip, bool times_lamlam,
                                   const BlockSmem& sm) {
  const int R = c.R[s];
  const int ld = lm_ld(R);
  const double* lam = c.LAM[s];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e - i * R;
    double v = 1.0;
    for (int m = 0; m < c.N; ++m)
      if (m != skip) v *= c.G[s * c.N + m][e];
    if (times_lamlam) v = v * (lam[i] * lam[j]);
    sm.lmA[i * ld + j] = v;
  }
  __syncthreads();
}

// step(n) = (hadamard_{m != n} G) o lam lam^T, its lambda_max and the
// Lipschitz history update (solver.py:402-406).
static __device__ __noinline__ void step_and_lipschitz(const Ctx& c, int s, int n, const BlockSmem& sm) {
  const int R = c.R[s];
  const int ld = lm_ld(R);
  PhaseClock pc;
  pc.start(c.dbg);
  build_gram_product(c, s, n, true, sm);
  double* step = c.STEP[s];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e - i * R;
    step[e] = sm.lmA[i * ld + j];
  }
  pc.mark(c.dbg, 4);
  const double lu = block_lam_max_warm(sm.lmA, R, sm.lmB, sm.lmB2, sm.vec, sm.red,
                                      c.evec + ((long long)s * (c.N + 1) + n) * 64,
                                      c.evec_miss + (long long)s * (c.N + 1) + n);
  if (threadIdx.x == 0) {
    const int idx = n * c.S + s;
    const double h = c.lipf_hist[idx];
    c.lip_w[lup_idx(c, n, c.off + s)] = isnan(h) ? lu : h;
    c.lipf_hist[idx] = lu;
    c.lip_w[lu_idx(c, n, c.off + s)] = lu;
  }
  __syncthreads();
  pc.mark(c.dbg, 5);
}

// Final per-block quantities of an evaluation: model_sq = lam^T (had G) lam and
// for lra inner = lam^T (had C)^T w~, res_t (solver.py:513-515).
static __device__ __noinline__ void final_quantities(const Ctx& c, int s, const BlockSmem& sm) {
  const int R = c.R[s];
  const int ld = lm_ld(R);
  const double* lam = c.LAM[s];
  build_gram_product(c, s, -1, false, sm);
  double* v = sm.misc;          // v = lam^T G
  double* u = sm.misc + 64;     // u = C^T w~
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    double a = 0.0;
    for (int i = 0; i < R; ++i) a = fma(lam[i], sm.lmA[i * ld + j], a);
    v[j] = a;
  }
  if (c.lra) {
    const int Rt = c.Rt[s];
    const double* tw = c.TW[s];
    for (int j = threadIdx.x; j < R; j += blockDim.x) {
      double a = 0.0;
      for (int q = 0; q < Rt; ++q) {
        double cp = 0.0;
        bool first = true;
        for (int m = 0; m < c.N; ++m) {
          const double g = c.C[s * c.N + m][q * R + j];
          cp = first ? g : cp * g;
          first = false;
        }
        a = fma(cp, tw[q], a);
      }
      u[j] = a;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double msq = 0.0;
    for (int j = 0; j < R; ++j) msq = fma(v[j], lam[j], msq);
    c.model_sq[s] = msq;
    if (c.lra) {
      double in = 0.0;
      for (int j = 0; j < R; ++j) in = fma(lam[j], u[j], in);
      c.inner[s] = in;
      c.res_t[s] = c.tsq[s] - 2.0 * in + msq;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// init: grams, cross grams, ||M~||^2, Lipschitz histories unset
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_init_block(Ctx c) {
  griddep_wait();
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, c.rmax);
  const int s = blockIdx.x;
  const int R = c.R[s];
  for (int n = 0; n < c.N; ++n) {
    const long long In = c.dims[s * c.N + n];
    block_gram(c.U[s * c.N + n], R, c.U[s * c.N + n], R, In, c.G[s * c.N + n], sm);
    if (c.lra) block_gram(c.Ut[s * c.N + n], c.Rt[s], c.U[s * c.N + n], R, In, c.C[s * c.N + n], sm);
  }
  if (threadIdx.x == 0) {
    c.lipc_hist[s] = NAN;
    for (int n = 0; n < c.N; ++n) c.lipf_hist[n * c.S + s] = NAN;
  }
  if (c.lra) {
    // ||M~||^2 = 1^T (hadamard_n Ut_n^T Ut_n) 1 (solver.py:334-337): reuse the
    // gram staging through the cross-gram slot of mode 0 as scratch
    const int Rt = c.Rt[s];
    double tot = 0.0;
    double* H = sm.misc;  // column sums, Rt <= 64
    for (int j = threadIdx.x; j < Rt; j += blockDim.x) H[j] = 0.0;
    __syncthreads();
    // build hadamard of tilde grams entry by entry (Rt^2 <= 4096)
    for (int e = threadIdx.x; e < Rt * Rt; e += blockDim.x) {
      const int p = e / Rt, q = e - p * Rt;
      double v = 0.0;
      bool first = true;
      for (int n = 0; n < c.N; ++n) {
        const double* A = c.Ut[s * c.N + n];
        const long long In = c.dims[s * c.N + n];
        double g = 0.0;
        for (long long i = 0; i < In; ++i) g = fma(A[i * Rt + p], A[i * Rt + q], g);
        v = first ? g : v * g;
        first = false;
      }
      c.qr_buf[(long long)s * c.N * QR_MAXC * QR_MAXC + e] = v;   // scratch
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double* Hm = c.qr_buf + (long long)s * c.N * QR_MAXC * QR_MAXC;
      // (1^T H) 1: column sums first, then their sum
      for (int q = 0; q < Rt; ++q) {
        double cs = 0.0;
        for (int p = 0; p < Rt; ++p) cs += Hm[p * Rt + q];
        tot += cs;
      }
      c.tsq[s] = tot;
    }
    __syncthreads();
  }
  final_quantities(c, s, sm);
  if (c.ld_pre && c.update_core) {
    const double ld = block_lam_max_warm(sm.lmA, R, sm.lmB, sm.lmB2, sm.vec, sm.red, c.evec + ((long long)s * (c.N + 1) + c.N) * 64, c.evec_miss + (long long)s * (c.N + 1) + c.N);
    if (threadIdx.x == 0) c.ldcore[s] = ld;
  }
}

// ---------------------------------------------------------------------------
// sweep begin: core update (solver.py:375-395) and the mode-0 step matrix
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sweep_begin(Ctx c, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  tl_begin(c.tl, TL_SWEEP);
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, 0);   // no gram staging
  const int s = blockIdx.x;
  const int R = c.R[s];
  const int ld = lm_ld(R);
  const double w_hat = redo ? 0.0 : c.st->w_hat;
  double* lam = c.LAM[s];
  double* lamp = c.LAMP[s];
  if (c.update_core) {
    build_gram_product(c, s, -1, false, sm);
    // main sweeps of the 3-way full path: L_d was formed beside the previous
    // evaluation's fiber pass (k_eval_side) from these same grams
    const double ldv = (!redo && c.ld_pre)
                           ? c.ldcore[s]
                           : block_lam_max_warm(sm.lmA, R, sm.lmB, sm.lmB2, sm.vec, sm.red, c.evec + ((long long)s * (c.N + 1) + c.N) * 64, c.evec_miss + (long long)s * (c.N + 1) + c.N);
    double* sc = sm.misc + 192;
    if (threadIdx.x == 0) {
      const double h = c.lipc_hist[s];
      sc[0] = isnan(h) ? ldv : h;
      c.lipc_hist[s] = ldv;
    }
    __syncthreads();
    const double ldp = sc[0];
    if (ldv == 0.0) {
      // all factor columns vanish, so does the gradient: keep lam
      for (int r = threadIdx.x; r < R; r += blockDim.x) lamp[r] = lam[r];
    } else {
      const double w = extrap_weight(w_hat, ldp, ldv, c.delta_w);
      double* lh = sm.misc;
      double* lin = sm.misc + 64;
      for (int r = threadIdx.x; r < R; r += blockDim.x) {
        lh[r] = lam[r] + w * (lam[r] - lamp[r]);
        if (!c.lra) {
          lin[r] = c.bbuf[((long long)c.st->bsel * c.S + s) * RSTRIDE + r];
        } else {
          const int Rt = c.Rt[s];
          const double* tw = c.TW[s];
          double a = 0.0;
          for (int q = 0; q < Rt; ++q) {
            double cp = 0.0;
            bool first = true;
            for (int m = 0; m < c.N; ++m) {
              const double g = c.C[s * c.N + m][q * R + r];
              cp = first ? g : cp * g;
              first = false;
            }
            a = fma(cp, tw[q], a);
          }
          lin[r] = a;
        }
      }
      __syncthreads();
      for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double g = 0.0;
        for (int j = 0; j < R; ++j) g = fma(sm.lmA[r * ld + j], lh[j], g);
        g -= lin[r];
        lamp[r] = lam[r];
        lam[r] = pos(lh[r] - g / ldv);
      }
    }
    __syncthreads();
  }
  PhaseClock pc;
  pc.start(c.dbg);
  step_and_lipschitz(c, s, 0, sm);
  pc.mark(c.dbg, 9);
  tl_end(c.tl, TL_SWEEP);
}

// sum over all blocks (global order) of the mode-n Lipschitz constants and of
// their "previous" values (solver.py:422-425)
// Called by a whole warp; lane 0 gets the sums.  The loads are issued by
// all lanes at once, the adds stay sequential in block order on lane 0.
__device__ inline void common_lip_sums(const Ctx& c, int n, double& sl, double& slp) {
  const int lane = threadIdx.x & 31;
  sl = 0.0;
  slp = 0.0;
  for (int q0 = 0; q0 < c.S_tot; q0 += 32) {
    const int q = q0 + lane;
    const double a = q < c.S_tot ? c.lip[lu_idx(c, n, q)] : 0.0;
    const double b = q < c.S_tot ? c.lip[lup_idx(c, n, q)] : 0.0;
    const int m = c.S_tot - q0 < 32 ? c.S_tot - q0 : 32;
    for (int k = 0; k < m; ++k) {
      const double ak = __shfl_sync(0xffffffffu, a, k);
      const double bk = __shfl_sync(0xffffffffu, b, k);
      sl += ak;
      slp += bk;
    }
  }
}

// new common columns of rows [r0, r0+rows): the partial gradients of the
// blocks with L_u > 0 summed in block order (solver.py:444), then the
// projected step from the extrapolated point (solver.py:447-451)
__device__ inline void common_fold(const Ctx& c, int n, int r0, int rows, double sumL, double wc) {
  const int L = c.counts[n];
  const int R0 = c.R[0];
  const double* U0c = c.U[n];
  const double* U0p = c.Up[n];
  for (int e = threadIdx.x; e < rows * L; e += blockDim.x) {
    const int il = e / L, l = e - il * L;
    const long long i = r0 + il;
    // partials of the blocks with L_u > 0, added in block order; 32 loads
    // in flight before their adds (latency, not bandwidth, bound)
    double acc = 0.0;
    const double cc = U0c[i * R0 + l], cp = U0p[i * R0 + l];
    for (int q0 = 0; q0 < c.S_tot; q0 += 32) {
      double g32[32];
      bool on[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int q = q0 + k;
        on[k] = q < c.S_tot && c.lip[lu_idx(c, n, q)] > 0.0;
        g32[k] = q < c.S_tot ? __ldcg(&c.gc_part[(long long)q * c.gc_stride + i * L + l]) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (on[k]) acc += g32[k];
    }
    const double chat = cc + wc * (cc - cp);
    const double cn = sumL > 0.0 ? pos(chat - acc / sumL) : cc;
    c.cnew[i * L + l] = cn;
    // every block's new factor is [c_new | new individual] (solver.py:452-456):
    // the shared columns go straight into the blocks' Un, so finalize reads
    // the new factor from one array
    for (int s = 0; s < c.S; ++s) c.Un[s * c.N + n][i * c.R[s] + l] = cn;
  }
}

// ---------------------------------------------------------------------------
// mode update: extrapolate, gradient, project individual columns, partial
// common gradient; the last CTA of each row tile forms the new common columns
// (solver.py:397-451).  src: 0 = MTT buffer, 1 = slab partials, 2 = lra.
// ---------------------------------------------------------------------------
// One row tile [r0, r0 + MU_ROWS) of block s: extrapolate, gradient, project
// the individual columns into Un, and the common-gradient partial into gcp
// (row-major I_n x L, this block's global slot).
// `smd` is the tile's shared scratch; returns the tile's (sumL, w_common)
// through sc_out (valid on every thread).
static __device__ __forceinline__ void mode_update_tile(const Ctx& c, int n, int redo, int src, int s,
                                                     int r0, double* smd, double* gcp,
                                                     double* sc_out, int TR = MU_ROWS) {
  const int R = c.R[s];
  const int N = c.N;
  const int L = c.counts[n];
  const long long In = c.dims[s * N + n];
  const int rows = (int)(In - r0 < TR ? In - r0 : TR);
  const double w_hat = redo ? 0.0 : c.st->w_hat;
  double* step = smd;                       // R*R
  double* uh = step + R * R;                // MU_ROWS*R
  double* mt = uh + TR * R;            // MU_ROWS*R
  double* P = mt + TR * R;             // Rt*R (lra)
  double* sc = P + (c.lra ? c.Rt[s] * R : 0);  // scalars
  const double* lam = c.LAM[s];
  if (threadIdx.x < 32) {
    double sl, slp;
    common_lip_sums(c, n, sl, slp);
    if (threadIdx.x == 0) {
      sc[0] = sl;
      sc[1] = extrap_weight(w_hat, slp, sl, c.delta_w);
      // own block: the written copy (current even where mode n is uncoupled
      // and nothing is exchanged)
      const int g = c.off + s;
      sc[2] = extrap_weight(w_hat, c.lip_w[lup_idx(c, n, g)], c.lip_w[lu_idx(c, n, g)], c.delta_w);
      sc[3] = c.lip_w[lu_idx(c, n, g)];
    }
  }
  stage_async(step, c.STEP[s], (long long)R * R);
  // lra, 3-way: the two other modes' cross grams, this tile's Ut rows and the
  // compression weights, staged with the step matrix in one round trip
  const bool lra3 = src == 2 && N == 3;
  double* Cs = sc + 8;                       // 2 x Rt*R (lra3)
  double* Uts = Cs + (lra3 ? 2 * c.Rt[s] * R : 0);   // rows x Rt
  double* tws = Uts + (lra3 ? TR * c.Rt[s] : 0); // Rt
  // this tile's current / previous rows (and block 0's common columns)
  double* Ucs = tws + (lra3 ? c.Rt[s] : 0);            // rows x R
  double* Ups = Ucs + TR * R;                      // rows x R
  double* U0s = Ups + TR * R;                      // rows x L (L > 0)
  double* U0ps = U0s + TR * L;                     // rows x L (L > 0)
  stage_async(Ucs, c.U[s * N + n] + (long long)r0 * R, (long long)rows * R);
  stage_async(Ups, c.Up[s * N + n] + (long long)r0 * R, (long long)rows * R);
  if (L > 0) {
    // block 0's common columns only (rows x L of its rows x R0)
    const int R0s = c.R[0];
    const double* g0 = c.U[n] + (long long)r0 * R0s;
    const double* g1 = c.Up[n] + (long long)r0 * R0s;
    for (int e = threadIdx.x; e < rows * L; e += blockDim.x) {
      const int il = e / L, l = e - il * L;
      cp_async8(U0s + e, g0 + (long long)il * R0s + l);
      cp_async8(U0ps + e, g1 + (long long)il * R0s + l);
    }
  }
  if (src == 0) stage_async(mt, c.MTT[s] + (long long)r0 * R, (long long)rows * R);
  if (lra3) {
    const int Rt = c.Rt[s];
    int k = 0;
    for (int m = 0; m < N; ++m)
      if (m != n) stage_async(Cs + (k++) * Rt * R, c.C[s * N + m], (long long)Rt * R);
    stage_async(Uts, c.Ut[s * N + n] + (long long)r0 * Rt, (long long)rows * Rt);
    stage_async(tws, c.TW[s], Rt);
  }
  cp_async8_wait();
  __syncthreads();
  const double sumL = sc[0], wc = sc[1], ws = sc[2], lu = sc[3];
  PhaseClock pc;
  pc.start(c.dbg);
  const double* Uc = c.U[s * N + n];
  const double* Upr = c.Up[s * N + n];
  const int R0 = c.R[0];
  const double* U0c = c.U[n];
  const double* U0p = c.Up[n];
  (void)U0c; (void)U0p; (void)Upr;
  for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
    const int il = e / R, r = e - il * R;
    const long long i = r0 + il;
    double v;
    if (r < L) {
      const double cc = U0s[il * L + r], cp = U0ps[il * L + r];
      v = cc + wc * (cc - cp);
    } else {
      const double cur = Ucs[e], prv = Ups[e];
      v = cur + ws * (cur - prv);
    }
    uh[e] = v;
    if (src == 1) {
      const int sb = c.slab_sb;
      const long long g = i / sb;
      const int m = (int)(i - g * sb);
      const int nch = c.slab_nchunk[s];
      const long long base = c.slab_first[s] + g * nch;
      double a = 0.0;
      for (int ch = 0; ch < nch; ++ch) a += c.slab_part[((base + ch) * sb + m) * RSTRIDE + r];
      mt[e] = a;
    }
  }
  if (lra3) {
    // P = C_a o C_b (mode order), then mt = (Ut o tw) P from shared memory
    const int Rt = c.Rt[s];
    for (int e = threadIdx.x; e < Rt * R; e += blockDim.x) P[e] = Cs[e] * Cs[Rt * R + e];
    for (int e = threadIdx.x; e < rows * Rt; e += blockDim.x) Uts[e] *= tws[e % Rt];
    __syncthreads();
    // 2 rows x 4 columns register tiles: six shared loads feed eight FMA
    // chains (each output keeps its q-ordered chain)
    const int RG = (R + 3) >> 2;
    const int H = (rows + 1) >> 1;
    for (int e = threadIdx.x; e < H * RG; e += blockDim.x) {
      const int i0 = e / RG, rb = (e - i0 * RG) << 2;
      const int i1 = i0 + H;
      const bool two = i1 < rows;
      const double* u0 = Uts + i0 * Rt;
      const double* u1 = Uts + (two ? i1 : i0) * Rt;
      double a[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      if (rb + 4 <= R) {
        for (int q = 0; q < Rt; ++q) {
          const double x0 = u0[q], x1 = u1[q];
          const double* pr = P + q * R + rb;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double pk = pr[k];
            a[0][k] = fma(x0, pk, a[0][k]);
            a[1][k] = fma(x1, pk, a[1][k]);
          }
        }
      } else {
        for (int q = 0; q < Rt; ++q) {
          const double x0 = u0[q], x1 = u1[q];
          const double* pr = P + q * R + rb;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (rb + k < R) {
              const double pk = pr[k];
              a[0][k] = fma(x0, pk, a[0][k]);
              a[1][k] = fma(x1, pk, a[1][k]);
            }
        }
      }
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (h2 == 1 && !two) break;
        double* mo = mt + (h2 ? i1 : i0) * R + rb;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rb + k < R) mo[k] = a[h2][k];
      }
    }
  } else if (src == 2) {
    const int Rt = c.Rt[s];
    for (int e = threadIdx.x; e < Rt * R; e += blockDim.x) {
      double v = 0.0;
      bool first = true;
      for (int m = 0; m < N; ++m) {
        if (m == n) continue;
        const double g = c.C[s * N + m][e];
        v = first ? g : v * g;
        first = false;
      }
      P[e] = first ? 1.0 : v;
    }
    __syncthreads();
    const double* Ut = c.Ut[s * N + n];
    const double* tw = c.TW[s];
    for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
      const int il = e / R, r = e - il * R;
      const long long i = r0 + il;
      double a = 0.0;
      for (int q = 0; q < Rt; ++q) a = fma(Ut[i * Rt + q] * tw[q], P[q * R + r], a);
      mt[e] = a;
    }
  }
  __syncthreads();
  pc.mark(c.dbg, 6);
  double* Un = c.Un[s * N + n];
  if (lu == 0.0) {
    for (int e = threadIdx.x; e < rows * R; e += blockDim.x) {
      const int il = e / R, r = e - il * R;
      if (r >= L) Un[(r0 + il) * (long long)R + r] = Ucs[e];
    }
  } else {
    // gradient u_hat step - mt o lam in 2 rows x 4 columns register tiles
    // (each output's q-ordered FMA chain unchanged), then the projection
    const int RG = (R + 3) >> 2;
    const int H = (rows + 1) >> 1;
    for (int e = threadIdx.x; e < H * RG; e += blockDim.x) {
      const int l0 = e / RG, rb = (e - l0 * RG) << 2;
      const int l1 = l0 + H;
      const bool two = l1 < rows;
      const double* ur0 = uh + l0 * R;
      const double* ur1 = uh + (two ? l1 : l0) * R;
      double g4[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      if (rb + 4 <= R) {
        for (int q = 0; q < R; ++q) {
          const double x0 = ur0[q], x1 = ur1[q];
          const double* sr = step + q * R + rb;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double sk = sr[k];
            g4[0][k] = fma(x0, sk, g4[0][k]);
            g4[1][k] = fma(x1, sk, g4[1][k]);
          }
        }
      } else {
        for (int q = 0; q < R; ++q) {
          const double x0 = ur0[q], x1 = ur1[q];
          const double* sr = step + q * R + rb;
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (rb + k < R) {
              const double sk = sr[k];
              g4[0][k] = fma(x0, sk, g4[0][k]);
              g4[1][k] = fma(x1, sk, g4[1][k]);
            }
        }
      }
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (h2 == 1 && !two) break;
        const int il = h2 ? l1 : l0;
        const double* ur = h2 ? ur1 : ur0;
        const long long i = r0 + il;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = rb + k;
          if (r >= R) break;
          const double g = g4[h2][k] - mt[il * R + r] * lam[r];
          if (r < L) gcp[i * L + r] = g;
          else Un[i * R + r] = pos(ur[r] - g / lu);
        }
      }
    }
  }
  sc_out[0] = sumL;
  sc_out[1] = wc;
  __syncthreads();
}

__global__ void __launch_bounds__(256, 1) k_mode_update(Ctx c, int n, int redo, int src,
                                                      const RowUnit* __restrict__ units) {
  griddep_wait();
  if (stopped(c, redo)) return;
  tl_begin(c.tl, TL_MU + n);
  extern __shared__ double smd[];
  const RowUnit u = units[blockIdx.x];
  const int s = u.s;
  const int L = c.counts[n];
  const long long In = c.dims[s * c.N + n];
  const int r0 = u.r0;
  const int TR = c.mu_rows;
  const int rows = (int)(In - r0 < TR ? In - r0 : TR);
  double sl2[2];
  mode_update_tile(c, n, redo, src, s, r0, smd, c.gc_w + (long long)(c.off + s) * c.gc_stride,
                   sl2, TR);
  const double sumL = sl2[0], wc = sl2[1];
  PhaseClock pc;
  pc.start(c.dbg);
  double* sc = smd;   // scratch reused (the tile is done)
  // sharded: the partials are all-reduced first; k_common folds them
  pc.mark(c.dbg, 7);
  tl_end(c.tl, TL_MU + n);
  if (L == 0 || c.shard) return;
  __threadfence();
  __syncthreads();
  int* flag = reinterpret_cast<int*>(sc + 4);
  if (threadIdx.x == 0) {
    const int t = r0 / TR;
    const int old = atomicAdd(&c.tile_cnt[t], 1);
    flag[0] = (old == c.S - 1);
  }
  __syncthreads();
  if (!flag[0]) return;
  __threadfence();
  // last CTA of this row tile: sum the partials in block order (solver.py:444)
  common_fold(c, n, r0, rows, sumL, wc);
  pc.mark(c.dbg, 8);
  tl_end(c.tl, TL_MU + n);
  if (threadIdx.x == 0) c.tile_cnt[r0 / TR] = 0;
}

// sharded runs: new common columns of one row tile from the all-reduced
// partials (grid: row tiles of mode n)
__global__ void __launch_bounds__(256) k_common(Ctx c, int n, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  tl_begin(c.tl, TL_COMMON + n);
  const int L = c.counts[n];
  if (L == 0) return;
  const long long In = c.dims[n];   // the common rows are shared: I_n of block 0
  const int r0 = blockIdx.x * MU_ROWS;
  if (r0 >= In) return;
  const int rows = (int)(In - r0 < MU_ROWS ? In - r0 : MU_ROWS);
  __shared__ double sc[2];
  if (threadIdx.x < 32) {
    double sl, slp;
    common_lip_sums(c, n, sl, slp);
    if (threadIdx.x == 0) {
      sc[0] = sl;
      sc[1] = extrap_weight(redo ? 0.0 : c.st->w_hat, slp, sl, c.delta_w);
    }
  }
  __syncthreads();
  common_fold(c, n, r0, rows, sc[0], sc[1]);
  tl_end(c.tl, TL_COMMON + n);
}

// ---------------------------------------------------------------------------
// finalize mode n: prev <- curr, curr <- [c_new | new individual], refresh the
// gram / cross gram (solver.py:452-457, :367-371), then the next mode's step
// matrix and Lipschitz constant, or the evaluation quantities after mode N-1.
// ---------------------------------------------------------------------------
// with_step = 0: the next mode's step matrix is left to k_step, which the 3-way
// path runs concurrently with the next MTTKRP (they share no inputs)
// The tail of a block's finalize (solver.py:402-406, :506-515): the next
// mode's step matrix and Lipschitz constant, or after the last mode the
// staged b and the evaluation quantities.  The grams of mode n are current.
static __device__ __noinline__ void finalize_tail(const Ctx& c, int n, int s, int with_step,
                                                  const BlockSmem& sm) {
  const int N = c.N;
  const int R = c.R[s];
  const long long In = c.dims[s * N + n];
  if (n + 1 < N) {
    if (with_step) step_and_lipschitz(c, s, n + 1, sm);
  } else if (!c.ld_pre) {
    if (c.b_mtt) {
      // staged core linear term b[r] = sum_i U_{N-1}[i, r] MTTKRP_{N-1}[i, r]
      // (solver.py:506-509); warp per r, lanes over rows, fixed order
      const double* Un = c.Un[s * N + n];
      const double* M = c.MTT[s];
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      for (int r = wid; r < R; r += blockDim.x >> 5) {
        double v = 0.0;
        for (long long i = lane; i < In; i += 32) v = fma(Un[i * R + r], M[i * R + r], v);
        v = warp_sum(v);
        if (lane == 0) c.fib_bpart[(long long)s * RSTRIDE + r] = v;
      }
    }
    final_quantities(c, s, sm);
  }
}

static __device__ __forceinline__ bool finalize_has_tail(const Ctx& c, int n, int with_step) {
  return (n + 1 < c.N) ? with_step != 0 : !c.ld_pre;
}

// finalize mode n (solver.py:452-457, :367-371): the new factor Un (shared
// columns already written by the fold) becomes current, the current one
// previous, the grams are refreshed, then the tail.  Grid (S, roles): role 0
// the copies, role 1 the gram U_n^T U_n, role 2 (lra) the cross gram
// Ut_n^T U_n, all from Un and independent of each other; the last role of
// a block to finish runs the tail (step matrix + lambda_max, or the
// evaluation quantities) once the grams are visible.
__global__ void __launch_bounds__(256) k_finalize(Ctx c, int n, int redo, int with_step) {
  griddep_wait();
  if (stopped(c, redo)) return;
  tl_begin(c.tl, TL_FIN + n);
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, c.rmax);
  const int s = blockIdx.x;
  const int role = blockIdx.y;
  const int N = c.N;
  const int R = c.R[s];
  const long long In = c.dims[s * N + n];
  double* Uc = c.U[s * N + n];
  double* Upr = c.Up[s * N + n];
  const double* Un = c.Un[s * N + n];
  if (role == 0) {
    // prev <- curr, curr <- new: all loads of a batch in flight before its
    // stores (the pointers may alias as far as the compiler knows)
    for (long long base = 0; base < In * R; base += 8LL * blockDim.x) {
      double cu[8], nv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long e = base + threadIdx.x + (long long)k * blockDim.x;
        if (e < In * R) { cu[k] = Uc[e]; nv[k] = Un[e]; }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long e = base + threadIdx.x + (long long)k * blockDim.x;
        if (e < In * R) { Upr[e] = cu[k]; Uc[e] = nv[k]; }
      }
    }
  } else if (role == 1) {
    block_gram(Un, R, Un, R, In, c.G[s * N + n], sm);
  } else {
    block_gram(c.Ut[s * N + n], c.Rt[s], Un, R, In, c.C[s * N + n], sm);
  }
  if (!finalize_has_tail(c, n, with_step)) {
    tl_end(c.tl, TL_FIN + n);
    return;
  }
  __threadfence();
  __syncthreads();
  int* flag = reinterpret_cast<int*>(sm.misc);
  if (threadIdx.x == 0) {
    const int old = atomicAdd(&c.fin_cnt[s], 1);
    const int last = old == (int)gridDim.y - 1;
    if (last) c.fin_cnt[s] = 0;
    flag[0] = last;
  }
  __syncthreads();
  if (!flag[0]) return;
  __threadfence();
  __syncthreads();
  finalize_tail(c, n, s, with_step, sm);
  tl_end(c.tl, TL_FIN + n);
}

// evaluation algebra of the 3-way full path, run beside the fiber pass:
// b[r] = sum_i U_{N-1}[i, r] MTTKRP_{N-1}[i, r] (solver.py:506-509), the
// evaluation quantities (final_quantities), and the next sweep's core
// Lipschitz constant lambda_max(hadamard_n G_n) (solver.py:375-379)
__device__ inline void eval_side_block(const Ctx& c, int s, const BlockSmem& sm) {
  const int N = c.N;
  const int R = c.R[s];
  const long long In = c.dims[s * N + N - 1];
  const double* Uc = c.U[s * N + N - 1];
  const double* M = c.MTT[s];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int r = wid; r < R; r += blockDim.x >> 5) {
    double v = 0.0;
    for (long long i = lane; i < In; i += 32) v = fma(Uc[i * R + r], M[i * R + r], v);
    v = warp_sum(v);
    if (lane == 0) c.fib_bpart[(long long)s * RSTRIDE + r] = v;
  }
  final_quantities(c, s, sm);   // leaves hadamard_n G_n in sm.lmA
  if (c.update_core) {
    const double ld = block_lam_max_warm(sm.lmA, R, sm.lmB, sm.lmB2, sm.vec, sm.red, c.evec + ((long long)s * (c.N + 1) + c.N) * 64, c.evec_miss + (long long)s * (c.N + 1) + c.N);
    if (threadIdx.x == 0) c.ldcore[s] = ld;
  }
}

__global__ void __launch_bounds__(256) k_eval_side(Ctx c, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, 0);   // no gram staging
  eval_side_block(c, blockIdx.x, sm);
}

// step matrix and Lipschitz constant of mode n for every block (solver.py:402-406)
__global__ void __launch_bounds__(256) k_step(Ctx c, int n, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  tl_begin(c.tl, TL_STEP + n - 1);
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, 0);   // no gram staging
  step_and_lipschitz(c, blockIdx.x, n, sm);
  tl_end(c.tl, TL_STEP + n - 1);
}

// restore curr <- prev and refresh caches (solver.py:538-543)
// gate 0: the restart branch (go_redo); gate 1: the pipelined lra rollback
// of a speculative sweep after a stop (rollback)
__global__ void __launch_bounds__(256) k_restore(Ctx c, int gate) {
  griddep_wait();
  if (gate == 0 ? c.st->go_redo == 0 : c.st->rollback == 0) return;
  extern __shared__ double smd[];
  const BlockSmem sm = carve(smd, c.rmax, c.rmax);
  const int s = blockIdx.x;
  const int N = c.N;
  const int R = c.R[s];
  for (int r = threadIdx.x; r < R; r += blockDim.x) c.LAM[s][r] = c.LAMP[s][r];
  for (int n = 0; n < N; ++n) {
    const long long In = c.dims[s * N + n];
    double* Uc = c.U[s * N + n];
    const double* Upr = c.Up[s * N + n];
    for (long long e = threadIdx.x; e < In * R; e += blockDim.x) Uc[e] = Upr[e];
  }
  __syncthreads();
  for (int n = 0; n < N; ++n) {
    const long long In = c.dims[s * N + n];
    block_gram(c.U[s * N + n], R, c.U[s * N + n], R, In, c.G[s * N + n], sm);
    if (c.lra) block_gram(c.Ut[s * N + n], c.Rt[s], c.U[s * N + n], R, In, c.C[s * N + n], sm);
  }
}

// ---------------------------------------------------------------------------
// lra QR route (solver.py:467-482): R factors of [Ut_n, U_n] by streamed
// Householder TSQR, then ||core||^2 of the (Rt+R)^N Kruskal core.
// Only blocks with res_t < 1e-3 ||M~||^2 do work.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool qr_route_needed(const Ctx& c, int s) {
  return c.res_t[s] < 1e-3 * c.tsq[s];
}

// TSQR with the running triangle on top: the rows of [Ut_n, U_n] stream in
// chunks of `ch` rows (as many as shared memory holds: 256 at Rt + R = 80);
// every chunk is annihilated against the current R by Cc Householder
// reflectors on the stacked [R; chunk] matrix.  Because R is upper
// triangular, reflector k touches only row k of R and the chunk rows.
// Blocked (compact WY): panels of QR_NB columns are factored by unblocked
// steps that touch only the panel (a step then costs two short barriers
// instead of a sweep over all trailing columns), and the trailing columns
// get the panel's block reflector I - V T V^T as three small GEMMs
// (Y = V^T A one warp per column with eight folded accumulators, Z = T^T Y,
// A -= V Z one warp per row).  The reflectors are those of the unblocked
// algorithm (c5: 1.37 -> ~0.3 ms per iteration on the QR route).  Result: R
// (Cc x Cc, upper triangular) of the QR of [Ut_n, U_n] up to row signs,
// which ||core||^2 does not see.  Grid: S * N CTAs of QR_THREADS.
constexpr int QR_THREADS = 512;
constexpr int QR_NB = 8;

// v0 / beta per column, Y (QR_NB x Cc), T, S, w, norm partials
__host__ __device__ inline long long qr_extra_doubles(int Cc) { return 10LL * Cc + 3 * 64 + 64; }

__host__ __device__ inline int qr_chunk_rows(int Cc, size_t smem_cap) {
  // R (Cc x (Cc+1)) + chunk (ch x (Cc+1)) + the panel scratch
  const long long avail =
      (long long)(smem_cap / sizeof(double)) - qr_extra_doubles(Cc) - (long long)Cc * (Cc + 1);
  long long ch = avail / (Cc + 1);
  ch = ch / 32 * 32;
  return (int)(ch > 256 ? 256 : (ch < 32 ? 32 : ch));
}

// sum over the 32 lanes of v[0..8) by recursive halving; lane l ends with the
// total of value l / 4 (fixed order: deterministic)
__device__ __forceinline__ double qr_fold8(double (&v)[8], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st;
    const int cnt = 8 >> st;
    if (cnt > 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < cnt / 2; ++i) {
        const double send = up ? v[i] : v[i + cnt / 2];
        const double keep = up ? v[i + cnt / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(QR_THREADS) k_qr_factor(Ctx c, int redo, int ch) {
  griddep_wait();
  if (stopped(c, redo)) return;
  const int s = blockIdx.x / c.N;
  const int n = blockIdx.x - s * c.N;
  if (!qr_route_needed(c, s)) return;
  extern __shared__ double smd[];
  const int R = c.R[s], Rt = c.Rt[s];
  const int Cc = Rt + R;
  const long long In = c.dims[s * c.N + n];
  const int ld = Cc + 1;
  double* Rm = smd;                      // Cc x ld, upper triangular
  double* X = Rm + Cc * ld;              // ch x ld chunk
  double* v0s = X + (long long)ch * ld;  // Cc: the R-row entry of reflector k
  double* betas = v0s + Cc;              // Cc
  double* Ym = betas + Cc;               // QR_NB x Cc
  double* Tm = Ym + QR_NB * Cc;          // QR_NB x QR_NB (upper triangular)
  double* Sm = Tm + 64;                  // QR_NB x QR_NB (V^T V, strictly upper)
  double* wp = Sm + 64;                  // QR_NB (panel step's w)
  double* red = wp + 64;                 // 2 x 32 (double-buffered column norms)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = QR_THREADS / 32;
  for (int e = threadIdx.x; e < Cc * ld; e += QR_THREADS) Rm[e] = 0.0;
  const double* A = c.Ut[s * c.N + n];
  const double* B = c.U[s * c.N + n];
  for (long long c0 = 0; c0 < In; c0 += ch) {
    const int nr = (int)(In - c0 < ch ? In - c0 : ch);
    __syncthreads();
    for (int i = wid; i < nr; i += nw)
      for (int j = lane; j < Cc; j += 32)
        X[i * ld + j] = j < Rt ? A[(c0 + i) * Rt + j] : B[(c0 + i) * R + (j - Rt)];
    __syncthreads();
    // squared norm of column 0 of the chunk (per-warp partials)
    {
      double ss = 0.0;
      for (int i = threadIdx.x; i < nr; i += QR_THREADS) ss = fma(X[i * ld], X[i * ld], ss);
      ss = warp_sum(ss);
      if (lane == 0) red[wid] = ss;
    }
    __syncthreads();
    for (int k0 = 0; k0 < Cc; k0 += QR_NB) {
      const int nb = Cc - k0 < QR_NB ? Cc - k0 : QR_NB;
      const int kend = k0 + nb;
      // ---- the panel: unblocked steps over its own columns
      for (int k = k0; k < kend; ++k) {
        const double* rk = red + (k & 1) * 32;
        double ss = 0.0;
        for (int q = 0; q < nw; ++q) ss += rk[q];
        const double x0 = Rm[k * ld + k];
        ss = fma(x0, x0, ss);
        const double nrm = sqrt(ss);
        const double alpha = x0 >= 0.0 ? -nrm : nrm;
        const double v0 = x0 - alpha;
        const double vtv = 2.0 * (ss - alpha * x0);
        const bool refl = vtv > 0.0;
        const double beta = refl ? 2.0 / vtv : 0.0;
        const int ncol = kend - k - 1;
        // w_j = beta (v0 R_kj + sum_i X_ik X_ij), one warp per panel column
        if (refl)
          for (int j = k + 1 + wid; j < kend; j += nw) {
            double a = 0.0;
            for (int i = lane; i < nr; i += 32) a = fma(X[i * ld + k], X[i * ld + j], a);
            a = warp_sum(a);
            if (lane == 0) wp[j - k0] = fma(v0, Rm[k * ld + j], a) * beta;
          }
        __syncthreads();
        // rank-1 update of the panel columns, one thread per row (row 0 =
        // row k of R); the squares of the updated column k + 1 are next
        // step's norm
        double nss = 0.0;
        if (ncol > 0) {
          for (int i = threadIdx.x; i <= nr; i += QR_THREADS) {
            double* p = i == 0 ? Rm + k * ld : X + (i - 1) * ld;
            if (refl) {
              const double vi = i == 0 ? v0 : p[k];
              for (int j = k + 1; j < kend; ++j) {
                const double x = p[j] - vi * wp[j - k0];
                p[j] = x;
                if (j == k + 1 && i > 0) nss = fma(x, x, nss);
              }
            } else if (i > 0) {
              nss = fma(p[k + 1], p[k + 1], nss);
            }
          }
          nss = warp_sum(nss);
          if (lane == 0) red[((k + 1) & 1) * 32 + wid] = nss;
        }
        if (threadIdx.x == 0) {
          Rm[k * ld + k] = refl ? alpha : x0;
          v0s[k] = refl ? v0 : 0.0;
          betas[k] = beta;
        }
        __syncthreads();
      }
      const int nt = Cc - kend;      // trailing columns
      if (nt == 0) break;
      // ---- S = strictly upper part of V^T V (the R-row parts of distinct
      // reflectors do not overlap: chunk rows only), one warp per pair;
      // the other warps start on Y = V^T A
      {
        const int npair = nb * (nb - 1) / 2;
        for (int pq = wid; pq < npair; pq += nw) {
          int a = 0, rem = pq;
          while (rem >= nb - 1 - a) { rem -= nb - 1 - a; ++a; }
          const int b = a + 1 + rem;
          double t = 0.0;
          for (int i = lane; i < nr; i += 32) t = fma(X[i * ld + k0 + a], X[i * ld + k0 + b], t);
          t = warp_sum(t);
          if (lane == 0) Sm[a * QR_NB + b] = t;
        }
        // Y[a][j] = v0_a R[k0 + a][j] + sum_i X[i][k0 + a] X[i][j]
        for (int j = kend + wid; j < Cc; j += nw) {
          double acc[QR_NB];
#pragma unroll
          for (int a = 0; a < QR_NB; ++a) acc[a] = 0.0;
          for (int i = lane; i < nr; i += 32) {
            const double xj = X[i * ld + j];
            const double* pr = X + i * ld + k0;
#pragma unroll
            for (int a = 0; a < QR_NB; ++a)
              if (a < nb) acc[a] = fma(pr[a], xj, acc[a]);
          }
          const double tot = qr_fold8(acc, lane);
          if ((lane & 3) == 0) {
            const int a = lane >> 2;
            if (a < nb) Ym[a * Cc + j] = fma(v0s[k0 + a], Rm[(k0 + a) * ld + j], tot);
          }
        }
      }
      __syncthreads();
      // ---- T (upper triangular): T_bb = beta_b, T[0:b, b] = -beta_b T[0:b,0:b] S[0:b, b]
      if (wid == 0) {
        for (int b = 0; b < nb; ++b) {
          const double bb = betas[k0 + b];
          if (lane < b) {
            double z = 0.0;
            for (int q = lane; q < b; ++q) z = fma(Tm[lane * QR_NB + q], Sm[q * QR_NB + b], z);
            Tm[lane * QR_NB + b] = -bb * z;
          } else if (lane == b) {
            Tm[b * QR_NB + b] = bb;
          }
          __syncwarp();
        }
      }
      __syncthreads();
      // ---- A -= V Z, Z = T^T Y: every warp keeps the Z columns of its
      // lanes' trailing columns in registers (j = kend + lane + 32 jj), then
      // one warp per row (rows 0..nb-1 = the panel's R rows, then the chunk
      // rows); the squares of the updated column kend are the next panel's
      // first norm
      {
        constexpr int QJ = (QR_MAXC + 31) / 32;
        double zr[QJ][QR_NB];
#pragma unroll
        for (int jj = 0; jj < QJ; ++jj) {
          const int j = kend + lane + 32 * jj;
#pragma unroll
          for (int a = 0; a < QR_NB; ++a) zr[jj][a] = 0.0;
          if (kend + 32 * jj >= Cc) continue;     // (warp-uniform) no such columns
          double y[QR_NB];
#pragma unroll
          for (int b = 0; b < QR_NB; ++b) y[b] = (b < nb && j < Cc) ? Ym[b * Cc + j] : 0.0;
#pragma unroll
          for (int a = 0; a < QR_NB; ++a) {
            double z = 0.0;
#pragma unroll
            for (int b = 0; b <= a; ++b)
              if (a < nb) z = fma(Tm[b * QR_NB + a], y[b], z);
            zr[jj][a] = z;
          }
        }
        double nss = 0.0;
        for (int i = wid; i < nb + nr; i += nw) {
          if (i < nb) {
            const double v = v0s[k0 + i];
#pragma unroll
            for (int jj = 0; jj < QJ; ++jj) {
              const int j = kend + lane + 32 * jj;
              if (j < Cc) {
                double z = 0.0;
#pragma unroll
                for (int a = 0; a < QR_NB; ++a) z = a == i ? zr[jj][a] : z;
                Rm[(k0 + i) * ld + j] -= v * z;
              }
            }
          } else {
            double* row = X + (i - nb) * ld;
            double pv[QR_NB];
#pragma unroll
            for (int a = 0; a < QR_NB; ++a) pv[a] = a < nb ? row[k0 + a] : 0.0;
#pragma unroll
            for (int jj = 0; jj < QJ; ++jj) {
              const int j = kend + lane + 32 * jj;
              if (j < Cc) {
                double x = row[j];
#pragma unroll
                for (int a = 0; a < QR_NB; ++a) x = fma(-pv[a], zr[jj][a], x);
                row[j] = x;
                if (jj == 0 && lane == 0) nss = fma(x, x, nss);
              }
            }
          }
        }
        // column kend is lane 0's first column
        if (lane == 0) red[(kend & 1) * 32 + wid] = nss;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  double* out = c.qr_buf + ((long long)s * c.N + n) * QR_MAXC * QR_MAXC;
  for (int e = threadIdx.x; e < Cc * Cc; e += QR_THREADS) {
    const int i = e / Cc, j = e - i * Cc;
    out[e] = j >= i ? Rm[i * ld + j] : 0.0;
  }
}

// 3-way ||core||^2 as a GEMM: core[(a, b), c] = sum_q P[(a, b), q] R2[c, q]
// with P[(a, b), q] = wts[q] R0[a, q] R1[b, q].  A CTA owns QRC_PAIRS (a, b)
// rows and every c; thread tile 4 pairs x ceil(K2 / 16) columns, R1 / R2
// transposed in shared memory (broadcast-friendly), the squares summed in
// registers; per-CTA partials folded in order by k_control.  Grid:
// S * qr_nchunks, qr_nchunks = ceil(max K0 K1 / QRC_PAIRS).
constexpr int QRC_PAIRS = 64;
constexpr int QRC_A = 8;      // core rows a per CTA
constexpr int QRC_CT = 8;     // max columns per thread (K2 <= 128)

template <int CT>
__global__ void __launch_bounds__(256) k_qr_core3(Ctx c, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  const int s = blockIdx.x / c.qr_nchunks;
  const int ch = blockIdx.x - s * c.qr_nchunks;
  if (!qr_route_needed(c, s)) return;
  extern __shared__ double smd[];
  const int R = c.R[s], Rt = c.Rt[s];
  const int Cc = Rt + R;
  const int K0 = (int)(c.dims[s * 3] < Cc ? c.dims[s * 3] : Cc);
  const int K1 = (int)(c.dims[s * 3 + 1] < Cc ? c.dims[s * 3 + 1] : Cc);
  const int K2 = (int)(c.dims[s * 3 + 2] < Cc ? c.dims[s * 3 + 2] : Cc);
  __shared__ double red[40];
  // this CTA: rows a in [a_lo, a_hi) of the core, every (b, c)
  const int a_lo = ch * QRC_A;
  const int a_hi = a_lo + QRC_A < K0 ? a_lo + QRC_A : K0;
  if (a_lo >= a_hi) {
    if (threadIdx.x == 0) c.qr_part[(long long)s * c.qr_nchunks + ch] = 0.0;
    return;
  }
  const int na = a_hi - a_lo;
  double* wq = smd;                      // Cc
  double* R1T = wq + Cc;                 // Cc x K1
  double* R2T = R1T + Cc * K1;           // Cc x K2
  double* R0T = R2T + Cc * K2;           // Cc x QRC_A
  const double* Rb = c.qr_buf + (long long)s * 3 * QR_MAXC * QR_MAXC;
  const long long MS = (long long)QR_MAXC * QR_MAXC;
  for (int q = threadIdx.x; q < Cc; q += blockDim.x)
    wq[q] = q < Rt ? c.TW[s][q] : -c.LAM[s][q - Rt];
  for (int e = threadIdx.x; e < Cc * K1; e += blockDim.x) {
    const int b = e / Cc, q = e - b * Cc;
    R1T[q * K1 + b] = Rb[MS + b * Cc + q];
  }
  for (int e = threadIdx.x; e < Cc * K2; e += blockDim.x) {
    const int cc = e / Cc, q = e - cc * Cc;
    R2T[q * K2 + cc] = Rb[2 * MS + cc * Cc + q];
  }
  for (int e = threadIdx.x; e < Cc * na; e += blockDim.x) {
    const int a = e / Cc, q = e - a * Cc;
    R0T[q * QRC_A + a] = Rb[(long long)(a_lo + a) * Cc + q];
  }
  __syncthreads();
  const int grp = threadIdx.x >> 4, col = threadIdx.x & 15;   // 16 pair groups x 16 columns
  const int npairs = na * K1;
  double ssq = 0.0;
  for (int p0 = 0; p0 < npairs; p0 += QRC_PAIRS) {
    int pa[4], pb[4];
    bool pv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + grp * 4 + u;
      pv[u] = p < npairs;
      const int pp = pv[u] ? p : 0;
      pa[u] = pp / K1;
      pb[u] = pp - pa[u] * K1;
    }
    double acc[4][CT];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < CT; ++v) acc[u][v] = 0.0;
    for (int q = 0; q < Cc; ++q) {
      const double wv = wq[q];
      double P[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) P[u] = wv * R0T[q * QRC_A + pa[u]] * R1T[q * K1 + pb[u]];
#pragma unroll
      for (int v = 0; v < CT; ++v) {
        const int cc = col + 16 * v;
        const double r2 = cc < K2 ? R2T[q * K2 + cc] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u][v] = fma(P[u], r2, acc[u][v]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < CT; ++v)
        if (pv[u]) ssq = fma(acc[u][v], acc[u][v], ssq);
  }
  ssq = block_sum(ssq, red);
  if (threadIdx.x == 0) c.qr_part[(long long)s * c.qr_nchunks + ch] = ssq;
}

// ||core||^2 with core[a_0..a_{N-1}] = sum_q wts[q] prod_m Rm[a_m, q],
// wts = [w~, -lam] (solver.py:476-482).  Grid: S * qr_nchunks.
__global__ void __launch_bounds__(256) k_qr_core(Ctx c, int redo) {
  griddep_wait();
  if (stopped(c, redo)) return;
  const int s = blockIdx.x / c.qr_nchunks;
  const int ch = blockIdx.x - s * c.qr_nchunks;
  if (!qr_route_needed(c, s)) return;
  __shared__ double red[40];
  __shared__ double wts[QR_MAXC];
  const int R = c.R[s], Rt = c.Rt[s];
  const int Cc = Rt + R;
  for (int q = threadIdx.x; q < Cc; q += blockDim.x)
    wts[q] = q < Rt ? c.TW[s][q] : -c.LAM[s][q - Rt];
  __syncthreads();
  long long K[CB_MAX_ORDER];
  long long total = 1;
  for (int m = 0; m < c.N; ++m) {
    const long long Im = c.dims[s * c.N + m];
    K[m] = Im < Cc ? Im : Cc;
    total *= K[m];
  }
  const double* Rb = c.qr_buf + (long long)s * c.N * QR_MAXC * QR_MAXC;
  double acc = 0.0;
  for (long long e = (long long)ch * blockDim.x + threadIdx.x; e < total;
       e += (long long)c.qr_nchunks * blockDim.x) {
    long long rem = e;
    int a[CB_MAX_ORDER];
    for (int m = 0; m < c.N; ++m) { a[m] = (int)(rem % K[m]); rem /= K[m]; }
    double v = 0.0;
    for (int q = 0; q < Cc; ++q) {
      double t = wts[q];
      for (int m = 0; m < c.N; ++m) t *= Rb[(long long)m * QR_MAXC * QR_MAXC + a[m] * Cc + q];
      v += t;
    }
    acc = fma(v, v, acc);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) c.qr_part[(long long)s * c.qr_nchunks + ch] = acc;
}

// ---------------------------------------------------------------------------
// control: evaluation totals, restart rule, histories, stop rule, momentum
// (solver.py:578-610).  One thread.
// ---------------------------------------------------------------------------
enum CtrlMode {
  CTRL_INIT = 0,      // iteration-0 evaluation (accept unconditionally)
  CTRL_DECIDE = 1,    // after the main sweep: restart or accept
  CTRL_REDO = 2,      // after the restart sweep: accept (full) / stage (lra)
  CTRL_FINISH = 3     // lra: after the original-tensor trace pass: accept
};

__device__ inline double block_res_full(const Ctx& c, int s, int bsrc) {
  // bsrc: 0 = fiber partials (fast3), 1 = c.res / c.borig (generic)
  if (c.objective == 0) {
    if (bsrc == 0) {
      return c.fib_rpart[s];   // per-block total folded by the fiber kernel
    }
    return c.res[s];
  }
  // gram expansion ||M||^2 - 2 lam^T b + lam^T (had G) lam
  const int R = c.R[s];
  const double* lam = c.LAM[s];
  const double* b = c.bbuf + ((long long)(1 - c.st->bsel) * c.S + s) * RSTRIDE;
  double lb = 0.0;
  for (int r = 0; r < R; ++r) lb = fma(lam[r], b[r], lb);
  return c.nsq[s] - 2.0 * lb + c.model_sq[s];
}

// momentum: advance t_k / w_hat here (classic order); the pipelined lra
// iteration advances them at DECIDE instead (the next sweep starts before
// this FINISH).  rollback_on_stop: that next sweep was speculative.
__device__ inline void advance_momentum(State* st) {
  const double t_new = t_next(st->t_k);
  st->w_hat = (st->t_k - 1.0) / t_new;
  st->t_k = t_new;
}

__device__ inline void accept_and_advance(const Ctx& c, double obj_int, double obj_orig, double rel,
                                   int swap_t, bool momentum = true, bool rollback_on_stop = false) {
  State* st = c.st;
  const int k = st->k;
  c.h_obj[k] = obj_int;
  c.h_orig[k] = obj_orig;
  c.h_rel[k] = rel;
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  if (k == 0) st->t0_ns = now;
  c.h_tns[k] = (double)(now - st->t0_ns);
  st->n_hist = k + 1;
  st->bsel ^= 1;
  if (swap_t) st->tsel ^= 1;
  st->go_redo = 0;
  st->obj_prev = obj_int;
  bool stop = false;
  if (k > 0) {
    if (fabs(rel - st->rel_prev) < c.tol) { stop = true; st->reason = 1; }
  }
  st->rel_prev = rel;
  if (!stop && k >= c.max_iter) { stop = true; st->reason = 0; }
  if (stop) {
    st->done = 1;
    st->go_main = 0;
    if (rollback_on_stop) st->rollback = 1;
    return;
  }
  // momentum for the next iteration (solver.py:588-590)
  if (momentum) advance_momentum(st);
  st->k = k + 1;
}

// Evaluation totals and the iteration rules.  Phase 1 (bit 0 of `phase`):
// per-block terms, thread s handles local block s, written to the global
// slots of ctl_w.  Phase 2 (bit 1): thread 0 folds the S_tot terms of ctl in
// global block order — the reference's summation order — and applies the
// restart / stop rules.  Single GPU runs both phases in one launch; sharded
// runs all-reduce ctl_w into ctl between them, so every rank folds the same
// values and takes the same decisions.
__global__ void __launch_bounds__(256) k_control(Ctx c, int mode, int bsrc, int phase) {
  griddep_wait();
  State* st = c.st;
  if (st->done) {
    // pipelined lra: the DECIDE after a stop follows the rollback restore
    // (k_restore gate 1) of the same step; clear the flag so later steps of
    // the host's polling chunk do not repeat that restore
    if (mode == CTRL_DECIDE && threadIdx.x == 0) st->rollback = 0;
    return;
  }
  if (mode == CTRL_REDO && !st->go_redo) return;
  if (!c.lra && mode == CTRL_FINISH) return;
  const int fast_t = (bsrc == 0);
  const bool lra_cmp = c.lra && (mode == CTRL_DECIDE || mode == CTRL_REDO);
  // pipelined lra (phase bit 4): FINISH reads the snapshots of its
  // iteration's lam / model_sq and leaves the momentum to DECIDE, which
  // advances it; bit 5: the stop rolls back a speculative sweep
  const bool pipe = (phase & 16) != 0;
  const bool rb_on_stop = (phase & 32) != 0;
  const int T = c.S_tot;
  tl_begin(c.tl, TL_CONTROL);
  if (phase & 1) {
    double* val = c.ctl_w;          // per-block residual (or compressed residual)
    double* relv = c.ctl_w + T;     // per-block relative error contribution
    double* rt0 = c.ctl_w + 2 * T;  // lra init: compressed residual
    for (int s = threadIdx.x; s < c.S; s += blockDim.x) {
      const int g = c.off + s;
      if (!c.lra) {
        if (fast_t) {
          double* b = c.bbuf + ((long long)(1 - st->bsel) * c.S + s) * RSTRIDE;
          const int R = c.R[s];
          for (int r = 0; r < R; ++r) b[r] = c.fib_bpart[(long long)s * RSTRIDE + r];
        }
        const double r = block_res_full(c, s, bsrc);
        val[g] = r;
        const double nrm = sqrt(c.nsq[s]);
        relv[g] = nrm > 0.0 ? sqrt(r > 0.0 ? r : 0.0) / nrm : 0.0;
      } else if (lra_cmp) {
        double rt = c.res_t[s];
        if (qr_route_needed(c, s)) {
          double a = 0.0;
          for (int ch = 0; ch < c.qr_nchunks; ++ch) a += c.qr_part[(long long)s * c.qr_nchunks + ch];
          rt = a;
        }
        val[g] = rt;
      } else {
        // original-tensor trace quantities (solver.py:519-522)
        const int R = c.R[s];
        const double* lam = pipe ? c.lam_snap + (long long)s * 64 : c.LAM[s];
        double lb = 0.0;
        for (int r = 0; r < R; ++r) {
          const double b = fast_t ? c.fib_bpart[(long long)s * RSTRIDE + r]
                                  : c.borig[(long long)s * RSTRIDE + r];
          lb = fma(lam[r], b, lb);
        }
        const double raw = c.nsq[s] - 2.0 * lb + (pipe ? c.msq_snap[s] : c.model_sq[s]);
        val[g] = raw;   // Python max(raw, 0.0) keeps NaN / +inf (checked below)
        const double nrm = sqrt(c.nsq[s]);
        const double r = raw > 0.0 ? raw : 0.0;
        relv[g] = nrm > 0.0 ? sqrt(r) / nrm : 0.0;
      }
      if (c.lra && mode == CTRL_INIT) {
        // the iteration-0 evaluation also needs the compressed residual
        double rt = c.res_t[s];
        if (qr_route_needed(c, s)) {
          double a = 0.0;
          for (int ch = 0; ch < c.qr_nchunks; ++ch) a += c.qr_part[(long long)s * c.qr_nchunks + ch];
          rt = a;
        }
        rt0[g] = rt;
      }
    }
  }
  tl_end(c.tl, TL_CONTROL);
  if (!(phase & 2)) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double* val = c.ctl;
  const double* relv = c.ctl + T;
  const double* rt0 = c.ctl + 2 * T;
  if (!c.lra) {
    double oi = 0.0, rel = 0.0;
    for (int s = 0; s < T; ++s) {
      const double r = val[s];
      if (!isfinite(r)) {
        st->error = CB_ERR_NONFINITE; st->err_block = s; st->err_iter = st->k;
        st->done = 1; st->go_main = 0; st->go_redo = 0;
        return;
      }
      oi += 0.5 * r;
      rel += relv[s];
    }
    rel /= T;
    if (mode == CTRL_DECIDE && oi >= st->obj_prev) {
      st->n_restarts += 1;
      st->go_redo = 1;
      if (c.use_cond) cudaGraphSetConditional(c.cond, 1u);   // run the restart branch
      return;
    }
    accept_and_advance(c, oi, oi, rel, fast_t);
    return;
  }
  // ---- lra ----
  if (lra_cmp) {
    double oi = 0.0;
    for (int s = 0; s < T; ++s) oi += 0.5 * (val[s] > 0.0 ? val[s] : 0.0);
    st->obj_pending = oi;
    if (mode == CTRL_DECIDE && pipe) advance_momentum(st);
    if (mode == CTRL_DECIDE && oi >= st->obj_prev) {
      st->n_restarts += 1;
      st->go_redo = 1;
      if (c.use_cond) cudaGraphSetConditional(c.cond, 1u);
    }
    return;
  }
  // CTRL_INIT or CTRL_FINISH
  double oi = st->obj_pending;
  if (mode == CTRL_INIT) {
    oi = 0.0;
    for (int s = 0; s < T; ++s) {
      const double rt = rt0[s];
      oi += 0.5 * (rt > 0.0 ? rt : 0.0);
    }
  }
  double oo = 0.0, rel = 0.0;
  for (int s = 0; s < T; ++s) {
    const double raw = val[s];
    if (raw != raw || raw == INFINITY) {
      st->error = CB_ERR_NONFINITE; st->err_block = s; st->err_iter = st->k;
      st->done = 1; st->go_main = 0; st->go_redo = 0;
      return;
    }
    oo += 0.5 * (raw > 0.0 ? raw : 0.0);
    rel += relv[s];
  }
  rel /= T;
  accept_and_advance(c, oi, oo, rel, 0, !(pipe && mode == CTRL_FINISH), rb_on_stop);
}

// pipelined lra: lam and model_sq of the iteration whose trace pass runs
// beside the next (speculative) sweep, read by its FINISH
__global__ void __launch_bounds__(64) k_pipe_snap(Ctx c) {
  griddep_wait();
  if (c.st->go_main == 0) return;
  const int s = blockIdx.x;
  const int R = c.R[s];
  for (int r = threadIdx.x; r < R; r += blockDim.x) c.lam_snap[(long long)s * 64 + r] = c.LAM[s][r];
  if (threadIdx.x == 0) c.msq_snap[s] = c.model_sq[s];
}

// emulated shard group exchange: recv_k <- sum_r send_r for every rank k
// (the sends have disjoint support, so the sum is an exact gather)
struct XsumArgs {
  const double* send[16];
  double* recv[16];
  int n;
  long long count;
};

__global__ void __launch_bounds__(256) k_xsum(XsumArgs a) {
  griddep_wait();
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < a.count; e += (long long)gridDim.x * 256) {
    double v = 0.0;
    for (int k = 0; k < a.n; ++k) v += a.send[k][e];
    for (int k = 0; k < a.n; ++k) a.recv[k][e] = v;
  }
}

}  // namespace cb
