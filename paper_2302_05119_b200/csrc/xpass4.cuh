// T pass (fiber, T = X x_3 A2, see xpass.cuh) with a warp-specialised
// bulk-copy ring: the T-only launches of the full-mode iteration in the fp32
// throughput mode (fp32 storage, fp64 arithmetic).
//
// Per unit (block s, j-tile of JT = 256 TJ columns) one producer lane streams
// the tile's rows X[j0 .. j0+JT, i2] (one 1-D bulk copy per row) through an
// F4_NST-stage ring of F4_ROWS rows; 8 consumer warps own TJ columns per
// thread and RB fp64 accumulators per column, read the stage as conflict-free
// consecutive floats plus the broadcast A2 row (staged once per unit), and
// release the stage per warp (full / empty mbarriers, no block barrier in the
// stream loop, so the next copy is issued as soon as the last warp is done).
// T[r, j] is written once, unsplit (nsplit = 1), in a fixed order: the
// result is bitwise that of fiber2_kernel's T-only path.
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include "xpass.cuh"

namespace cb {

constexpr int F4_CONS = 256;                  // consumer threads (8 warps)
constexpr int F4_THREADS = F4_CONS + 32;      // + the producer warp
constexpr int F4_ROWS = 8;                    // i2 rows per stage
constexpr int F4_NST = 5;                     // stages

template <typename TE>
__host__ __device__ constexpr size_t fiber4_smem(long long a2_rows, int rb, int tj) {
  return 128 + (size_t)F4_NST * F4_ROWS * F4_CONS * tj * sizeof(TE) + (size_t)a2_rows * rb * 8;
}

// RES: also the explicit residual sum_(j,i2) (X - [[lam; A0, A1, A2]])^2 of
// the unit into a.rpart[unit], folded per block in unit order by the last
// arriving CTA into a.rsum[s] (the ALS stop rule, cpd_als.py:101-110)
template <typename TE, int RB, int TJ, bool RES = false>
__global__ void __launch_bounds__(F4_THREADS)
fiber4_kernel(XArgs a, const FibUnit* __restrict__ units) {
  griddep_wait();
  if (gated(a)) return;
  constexpr int JT = F4_CONS * TJ;
  const FibUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  tl_begin(a.tl, TL_FIBER);
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1], I2 = a.dims[3 * s + 2];
  const long long J = I0 * I1;
  const TE* __restrict__ X = reinterpret_cast<const TE*>(a.X[s]);
  const double* __restrict__ A2 = a.U[3 * s + 2];

  extern __shared__ __align__(128) unsigned char f4sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(f4sm);
  uint64_t* empty = full + F4_NST;
  TE* xbuf = reinterpret_cast<TE*>(f4sm + 128);
  double* a2s = reinterpret_cast<double*>(f4sm + 128 + (size_t)F4_NST * F4_ROWS * JT * sizeof(TE));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long jlen = (J - u.j0) < JT ? (J - u.j0) : JT;
  const uint32_t row_bytes = (uint32_t)(jlen * sizeof(TE));
  const int nstages = (int)((I2 + F4_ROWS - 1) / F4_ROWS);
  if (threadIdx.x == 0) {
    for (int i = 0; i < F4_NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], F4_CONS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == F4_CONS / 32) {
    // ------------------------------------------------------- producer lane
    if (lane == 0) {
      for (int k = 0; k < nstages; ++k) {
        const int slot = k % F4_NST;
        mbar_wait(&empty[slot], (uint32_t)(((k / F4_NST) & 1) ^ 1));
        const long long r0 = (long long)k * F4_ROWS;
        const int nr = (int)((I2 - r0) < F4_ROWS ? (I2 - r0) : F4_ROWS);
        mbar_arrive_expect_tx(&full[slot], nr * row_bytes);
        for (int q = 0; q < nr; ++q)
          bulk_g2s(xbuf + ((size_t)slot * F4_ROWS + q) * JT, X + u.j0 + J * (r0 + q), row_bytes,
                   &full[slot]);
      }
    }
    return;
  }
  // ------------------------------------------------------------- consumers
  // the unit's A2 rows (overlapping the first copies); named barrier over the
  // consumer warps only
  for (long long e = threadIdx.x; e < I2 * RB; e += F4_CONS) {
    const long long q = e / RB;
    const int r = (int)(e - q * RB);
    a2s[e] = r < R ? A2[q * R + r] : 0.0;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(F4_CONS) : "memory");
  long long jq[TJ];
  bool ok[TJ];
#pragma unroll
  for (int t = 0; t < TJ; ++t) {
    jq[t] = u.j0 + threadIdx.x + (long long)t * F4_CONS;
    ok[t] = jq[t] < J;
  }
  double acc[TJ][RB];
#pragma unroll
  for (int t = 0; t < TJ; ++t)
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[t][r] = 0.0;
  // RES: the model's row weights lam_r A0[i0, r] A1[i1, r] of this column
  double w[RES ? TJ : 1][RES ? RB : 1];
  double res = 0.0;
  if constexpr (RES) {
    const double* lam = a.LAM ? a.LAM[s] : nullptr;
    const double* A0 = a.U[3 * s];
    const double* A1 = a.U[3 * s + 1];
#pragma unroll
    for (int t = 0; t < TJ; ++t) {
      const long long i1 = ok[t] ? jq[t] / I0 : 0;
      const long long i0 = ok[t] ? jq[t] - i1 * I0 : 0;
#pragma unroll
      for (int r = 0; r < RB; ++r)
        w[t][r] = (r < R && ok[t]) ? (lam ? lam[r] : 1.0) * A0[i0 * R + r] * A1[i1 * R + r] : 0.0;
    }
  }
  for (int k = 0; k < nstages; ++k) {
    const int slot = k % F4_NST;
    const long long r0 = (long long)k * F4_ROWS;
    const int nr = (int)((I2 - r0) < F4_ROWS ? (I2 - r0) : F4_ROWS);
    mbar_wait(&full[slot], (uint32_t)((k / F4_NST) & 1));
    const TE* xs = xbuf + (size_t)slot * F4_ROWS * JT + threadIdx.x;
    const double* as = a2s + r0 * RB;
#pragma unroll 2
    for (int q = 0; q < nr; ++q) {
      double x[TJ];
#pragma unroll
      for (int t = 0; t < TJ; ++t) x[t] = (double)xs[q * JT + t * F4_CONS];
      double av[RB];
      load_row<double, RB>(as + q * RB, av);
      // all RB columns: the staged A2 rows are zero past R (no predicates in
      // the FMA stream)
#pragma unroll
      for (int r = 0; r < RB; ++r) {
#pragma unroll
        for (int t = 0; t < TJ; ++t) acc[t][r] = fma(x[t], av[r], acc[t][r]);
      }
      if constexpr (RES) {
#pragma unroll
        for (int t = 0; t < TJ; ++t) {
          double m = 0.0;
#pragma unroll
          for (int r = 0; r < RB; ++r) m = fma(w[t][r], av[r], m);
          if (ok[t]) { const double d = x[t] - m; res = fma(d, d, res); }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  double* T = reinterpret_cast<double*>(tbuf(a, s));
#pragma unroll
  for (int t = 0; t < TJ; ++t)
    if (ok[t]) {
#pragma unroll
      for (int r = 0; r < RB; ++r)
        if (r < R) T[(long long)r * J + jq[t]] = acc[t][r];
    }
  if constexpr (RES) {
    // unit partial: warp sums, then the 8 warps in order (consumers only)
    __shared__ double red4[F4_CONS / 32];
    __shared__ int last4;
    for (int o = 16; o; o >>= 1) res += __shfl_xor_sync(0xffffffffu, res, o);
    if (lane == 0) red4[warp] = res;
    asm volatile("bar.sync 1, %0;" ::"r"(F4_CONS) : "memory");
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < F4_CONS / 32; ++q) t += red4[q];
      a.rpart[blockIdx.x] = t;
      __threadfence();
      const int first = a.fib_first[s], nunits = a.fib_first[s + 1] - first;
      last4 = atomicAdd(&a.blk_cnt[s], 1) == nunits - 1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(F4_CONS) : "memory");
    if (last4 && threadIdx.x == 0) {
      // the block's units in unit order
      __threadfence();
      const int first = a.fib_first[s], nunits = a.fib_first[s + 1] - first;
      double t = 0.0;
      for (int q = 0; q < nunits; ++q) t += __ldcg(&a.rpart[first + q]);
      a.rsum[s] = t;
      a.blk_cnt[s] = 0;
    }
  }
  tl_end(a.tl, TL_FIBER);
}

}  // namespace cb
