// Tensor-streaming kernels of the 3-way fast path (the only kernels that read
// the dense blocks).  All batched over the S blocks of a solve, ragged shapes
// handled through per-launch unit tables.
//
// Notation per block s: X is I0 x I1 x I2, first index fastest; J = I0*I1;
// element (i0,i1,i2) lives at j + J*i2 with j = i0 + I0*i1.  Factors A0, A1,
// A2 are fp64 row-major (I_n x R).  TE = storage/compute type of the tensor
// (float in the fp32 throughput mode, double in the fp64 parity mode).
//
//  fiber  : T[j, r] = sum_{i2} X[j, i2] A2[i2, r]         ("X x_3 A2")
//           + optional per-unit partials of
//             b[r]  = sum_j A0[i0,r] A1[i1,r] T[j,r]       (core linear term,
//                      solver.py:506-511, and the lra trace pass :519-522)
//             res   = sum (X - [[lam; A0,A1,A2]])^2         (explicit residual,
//                      solver.py:500-505)
//  slab   : M2[i2, r] = sum_j X[j, i2] A0[i0,r] A1[i1,r]   (mode-2 MTTKRP,
//                      solver.py:409-412 with n = N-1)
//  contract0 : M0[i0, r] = sum_{i1} T[i0 + I0 i1, r] A1[i1, r]  (mode-0 MTTKRP)
//  contract1 : M1[i1, r] = sum_{i0} T[i0 + I0 i1, r] A0[i0, r]  (mode-1 MTTKRP)
//
// Modes 0 and 1 of a Gauss-Seidel sweep both contract X with the SAME A2
// (A2 only changes at mode 2), so one fiber pass serves both: a full-mode
// iteration streams each block twice (fiber + slab) instead of N = 3 times,
// and the explicit objective rides along the fiber pass for free.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace cb {

constexpr int FIB_THREADS = 256;
constexpr int FIB_CHUNK = 32;     // i2 rows of A2 staged in smem per step
constexpr int SLAB_THREADS = 256;
constexpr int RSTRIDE = 64;       // per-unit partial stride (>= max rank)

struct FibUnit { int s; int split; long long j0; };
struct SlabUnit { int s; int g0; long long k0; long long k1; };
struct RowUnit { int s; int r0; };

struct XArgs {
  const void* const* X;          // per block tensor
  const long long* dims;         // S*3
  const int* R;                  // per block rank
  const double* const* U;        // S*3 current factors
  const double* const* LAM;      // S weights (nullptr entries -> unit weights)
  void* const* T0;               // per block T buffers [nsplit][R][J], double-buffered:
  void* const* T1;               //   buffer index = (*tsel) ^ t_other
  const int* tsel;
  int t_other;
  const int* nsplit;             // per block fiber splits
  double* bpart;                 // [unit][RSTRIDE]
  double* rpart;                 // [unit]
  double* slab_part;             // [unit][SB][RSTRIDE]
  double* const* MTT;            // per block I_n x R output (contract kernels)
  const int* gate;               // if non-null and *gate == 0 -> skip (flag gating)
  const int* active;             // per-block activity (ALS); nullptr -> all active
  // per-block totals of the fiber partials, formed by the last CTA of each
  // block in unit order (deterministic): bsum[s][RSTRIDE], rsum[s]
  const int* fib_first;          // S+1 unit ranges
  int* blk_cnt;                  // S arrival counters (self-resetting)
  double* bsum;
  double* rsum;
  unsigned long long* ktime;     // profiling only: [0] fiber, [1] slab accumulators
  long long slab_stage_rows;     // factor rows the slab kernel may stage in smem (0: none)
};

// In-kernel wall time of a whole launch (first CTA start -> last CTA end),
// accumulated into kt[0] (ns), kt[1] (launches); kt[2], kt[3] scratch.
// Profiling builds of a run only (ktime non-null).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktime_begin(unsigned long long* kt) {
  if (kt && threadIdx.x == 0) atomicMin(&kt[2], gtimer());
}
__device__ __forceinline__ void ktime_end(unsigned long long* kt) {
  if (!kt) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(&kt[3], 1ull) + 1;
    if (done == gridDim.x) {
      const unsigned long long t = gtimer();
      kt[0] += t - kt[2];
      kt[1] += 1;
      kt[2] = ~0ull;
      kt[3] = 0;
    }
  }
}

__device__ __forceinline__ bool gated(const XArgs& a) {
  return a.gate != nullptr && *a.gate == 0;
}
__device__ __forceinline__ void* tbuf(const XArgs& a, int s) {
  const int sel = (a.tsel ? *a.tsel : 0) ^ a.t_other;
  return sel ? a.T1[s] : a.T0[s];
}

// ---------------------------------------------------------------------------
// fiber pass
// ---------------------------------------------------------------------------
// TMA variant: the unit's X rows (j-tile of 256 elements per i2 row) stream
// through a FIB_NST-stage ring of FIB_CH-row stages filled by 1-D bulk copies
// (cp.async.bulk, issued by one thread, completing on an mbarrier), so each
// CTA keeps FIB_NST * FIB_CH * 1 KB (fp32) in flight independent of its
// thread count.  Requires 16-B aligned rows (host checks; else TMA=false).
constexpr int FIB_CH = 8;
constexpr int FIB_NST = 4;

template <typename TE, typename TC, int RB>
__host__ __device__ constexpr size_t fiber_tma_smem() {
  return 128 + (size_t)FIB_NST * FIB_CH * FIB_THREADS * sizeof(TE) +
         (size_t)FIB_NST * FIB_CH * RB * sizeof(TC);
}

template <typename TE, typename TC, int RB, bool STORE_T, bool WANT_B, bool WANT_RES, bool TMA>
__global__ void __launch_bounds__(FIB_THREADS)
fiber_kernel(XArgs a, const FibUnit* __restrict__ units) {
  if (gated(a)) return;
  const FibUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  ktime_begin(a.ktime);
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1], I2 = a.dims[3 * s + 2];
  const long long J = I0 * I1;
  const int ns = a.nsplit[s];
  const long long per = (I2 + ns - 1) / ns;
  const long long i2b = (long long)u.split * per;
  const long long i2e = i2b + per < I2 ? i2b + per : I2;
  const TE* __restrict__ X = reinterpret_cast<const TE*>(a.X[s]);
  const double* __restrict__ A0 = a.U[3 * s];
  const double* __restrict__ A1 = a.U[3 * s + 1];
  const double* __restrict__ A2 = a.U[3 * s + 2];

  __shared__ TC a2s[FIB_CHUNK][RB];
  __shared__ double red[FIB_THREADS / 32][RB + 1];

  const long long j = u.j0 + threadIdx.x;
  const bool valid = j < J;
  long long i0 = 0, i1 = 0;
  if (valid) { i1 = j / I0; i0 = j - i1 * I0; }

  TC acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = TC(0);
  TC w[WANT_RES ? RB : 1];
  double res = 0.0;
  if constexpr (WANT_RES) {
    const double* lam = a.LAM ? a.LAM[s] : nullptr;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      double v = 0.0;
      if (r < R && valid) v = (lam ? lam[r] : 1.0) * A0[i0 * R + r] * A1[i1 * R + r];
      w[r] = (TC)v;
    }
  }

  if constexpr (TMA) {
    extern __shared__ __align__(128) unsigned char fsm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(fsm);
    TE* xbuf = reinterpret_cast<TE*>(fsm + 128);
    TC* a2t = reinterpret_cast<TC*>(fsm + 128 + (size_t)FIB_NST * FIB_CH * FIB_THREADS * sizeof(TE));
    const long long jt = (J - u.j0) < FIB_THREADS ? (J - u.j0) : FIB_THREADS;
    const uint32_t row_bytes = (uint32_t)(jt * sizeof(TE));
    const int nstages = (int)((i2e - i2b + FIB_CH - 1) / FIB_CH);
    auto issue = [&](int k) {
      const int slot = k % FIB_NST;
      const long long r0 = i2b + (long long)k * FIB_CH;
      const int nr = (int)((i2e - r0) < FIB_CH ? (i2e - r0) : FIB_CH);
      mbar_arrive_expect_tx(&bar[slot], nr * row_bytes);
      for (int q = 0; q < nr; ++q)
        bulk_g2s(xbuf + ((size_t)slot * FIB_CH + q) * FIB_THREADS, X + u.j0 + J * (r0 + q),
                 row_bytes, &bar[slot]);
    };
    if (threadIdx.x == 0) {
      for (int st = 0; st < FIB_NST; ++st) mbar_init(&bar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < nstages && k < FIB_NST; ++k) issue(k);
    for (int k = 0; k < nstages; ++k) {
      const int slot = k % FIB_NST;
      const long long r0 = i2b + (long long)k * FIB_CH;
      const int nr = (int)((i2e - r0) < FIB_CH ? (i2e - r0) : FIB_CH);
      TC* as = a2t + (size_t)slot * FIB_CH * RB;
      for (int e = threadIdx.x; e < FIB_CH * RB; e += FIB_THREADS) {
        const int q = e / RB, r = e - q * RB;
        as[e] = (q < nr && r < R) ? (TC)A2[(r0 + q) * R + r] : TC(0);
      }
      __syncthreads();
      mbar_wait(&bar[slot], (uint32_t)((k / FIB_NST) & 1));
      if (valid) {
        const TE* xs = xbuf + (size_t)slot * FIB_CH * FIB_THREADS + threadIdx.x;
        for (int q = 0; q < nr; ++q) {
          const TC x = (TC)xs[q * FIB_THREADS];
          TC m = TC(0);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (r < R) {
              acc[r] = fma(x, as[q * RB + r], acc[r]);
              if constexpr (WANT_RES) m = fma(w[r], as[q * RB + r], m);
            }
          }
          if constexpr (WANT_RES) { double d = (double)x - (double)m; res = fma(d, d, res); }
        }
      }
      __syncthreads();   // slot fully consumed
      if (threadIdx.x == 0 && k + FIB_NST < nstages) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + FIB_NST);
      }
    }
  } else
  for (long long c0 = i2b; c0 < i2e; c0 += FIB_CHUNK) {
    const int nc = (int)((i2e - c0) < FIB_CHUNK ? (i2e - c0) : FIB_CHUNK);
    __syncthreads();
    for (int e = threadIdx.x; e < FIB_CHUNK * RB; e += FIB_THREADS) {
      int q = e / RB, r = e - q * RB;
      a2s[q][r] = (q < nc && r < R) ? (TC)A2[(c0 + q) * R + r] : TC(0);
    }
    __syncthreads();
    if (valid) {
      const TE* xp = X + j + J * c0;
      int q = 0;
      for (; q + 4 <= nc; q += 4) {
        TC x[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t] = (TC)__ldcs(xp + J * (q + t));
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          TC m = TC(0);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (r < R) {   // uniform: skips the bucket's padding columns
              acc[r] = fma(x[t], a2s[q + t][r], acc[r]);
              if constexpr (WANT_RES) m = fma(w[r], a2s[q + t][r], m);
            }
          }
          if constexpr (WANT_RES) { double d = (double)x[t] - (double)m; res = fma(d, d, res); }
        }
      }
      for (; q < nc; ++q) {
        TC x = (TC)__ldcs(xp + J * q);
        TC m = TC(0);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          if (r < R) {
            acc[r] = fma(x, a2s[q][r], acc[r]);
            if constexpr (WANT_RES) m = fma(w[r], a2s[q][r], m);
          }
        }
        if constexpr (WANT_RES) { double d = (double)x - (double)m; res = fma(d, d, res); }
      }
    }
  }

  if constexpr (STORE_T) if (valid) {
    TC* T = reinterpret_cast<TC*>(tbuf(a, s)) + (long long)u.split * R * J;
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < R) T[(long long)r * J + j] = acc[r];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if constexpr (WANT_B) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      double v = 0.0;
      if (valid && r < R) v = (double)acc[r] * (A0[i0 * R + r] * A1[i1 * R + r]);
      v = warp_sum(v);
      if (lane == 0) red[wid][r] = v;
    }
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int q = 0; q < FIB_THREADS / 32; ++q) t += red[q][threadIdx.x];
      a.bpart[(long long)blockIdx.x * RSTRIDE + threadIdx.x] = t;
    }
  }
  if constexpr (WANT_RES) {
    __syncthreads();
    double v = warp_sum(res);
    if (lane == 0) red[wid][0] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < FIB_THREADS / 32; ++q) t += red[q][0];
      a.rpart[blockIdx.x] = t;
    }
  }
  if constexpr (WANT_B || WANT_RES) {
    // the last CTA of block s folds the per-unit partials in unit order
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    const int first = a.fib_first[s], nunits = a.fib_first[s + 1] - first;
    if (threadIdx.x == 0) s_last = (atomicAdd(&a.blk_cnt[s], 1) == nunits - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      if constexpr (WANT_B) {
        // thread (r, c): contiguous quarter c of the unit range, then the four
        // quarter sums in order
        __shared__ double qs[4][RB];
        const int r = threadIdx.x & 63, c = threadIdx.x >> 6;
        if (r < R) {
          const int q0 = (int)((long long)nunits * c / 4), q1 = (int)((long long)nunits * (c + 1) / 4);
          double t = 0.0;
#pragma unroll 4
          for (int q = q0; q < q1; ++q) t += __ldcg(&a.bpart[(long long)(first + q) * RSTRIDE + r]);
          qs[c][r] = t;
        }
        __syncthreads();
        if (threadIdx.x < R)
          a.bsum[(long long)s * RSTRIDE + threadIdx.x] =
              ((qs[0][threadIdx.x] + qs[1][threadIdx.x]) + qs[2][threadIdx.x]) + qs[3][threadIdx.x];
      }
      if constexpr (WANT_RES) {
        double t = 0.0;
        for (int q = threadIdx.x; q < nunits; q += FIB_THREADS) t += __ldcg(&a.rpart[first + q]);
        t = block_sum(t, &red[0][0]);
        if (threadIdx.x == 0) a.rsum[s] = t;
      }
      if (threadIdx.x == 0) a.blk_cnt[s] = 0;
    }
  }
  ktime_end(a.ktime);
}

// ---------------------------------------------------------------------------
// slab pass: each unit = (block, SB consecutive i2 slabs, j-range [k0, k1))
// ---------------------------------------------------------------------------
template <typename TE, typename TC, int RB, int SB>
__global__ void __launch_bounds__(SLAB_THREADS)
slab_kernel(XArgs a, const SlabUnit* __restrict__ units) {
  if (gated(a)) return;
  const SlabUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  ktime_begin(a.ktime ? a.ktime + 4 : nullptr);
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1], I2 = a.dims[3 * s + 2];
  const long long J = I0 * I1;
  const TE* __restrict__ X = reinterpret_cast<const TE*>(a.X[s]);
  const double* __restrict__ A0 = a.U[3 * s];
  const double* __restrict__ A1 = a.U[3 * s + 1];

  extern __shared__ __align__(16) unsigned char smraw[];
  // factor rows staged r-major (a0s[r][i0]): lanes of a warp walk consecutive
  // i0, so every smem read below is conflict-free (a row-major copy would put
  // all 32 lanes on one bank)
  TC* a0s = reinterpret_cast<TC*>(smraw);          // RB x I0
  TC* a1s = a0s + I0 * RB;                         // RB x I1
  for (long long e = threadIdx.x; e < I0 * RB; e += SLAB_THREADS) {
    const int r = (int)(e / I0);
    const long long i = e - r * I0;
    a0s[e] = r < R ? (TC)A0[i * R + r] : TC(0);
  }
  for (long long e = threadIdx.x; e < I1 * RB; e += SLAB_THREADS) {
    const int r = (int)(e / I1);
    const long long i = e - r * I1;
    a1s[e] = r < R ? (TC)A1[i * R + r] : TC(0);
  }
  __syncthreads();

  int nsl = (int)(I2 - u.g0 < SB ? I2 - u.g0 : SB);
  TC acc[SB][RB];
#pragma unroll
  for (int m = 0; m < SB; ++m)
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[m][r] = TC(0);

  long long k = u.k0 + threadIdx.x;
  long long i1 = k / I0, i0 = k - i1 * I0;
  const long long st1 = SLAB_THREADS / I0, st0 = SLAB_THREADS - st1 * I0;
  const TE* xb = X + J * u.g0;
  for (; k < u.k1; k += SLAB_THREADS) {
    TC x[SB];
#pragma unroll
    for (int m = 0; m < SB; ++m) x[m] = (m < nsl) ? (TC)__ldcs(xb + J * m + k) : TC(0);
    const TC* p0 = a0s + i0;
    const TC* p1 = a1s + i1;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < R) {   // uniform: skips the bucket's padding columns
        TC kr = p0[r * I0] * p1[r * I1];
#pragma unroll
        for (int m = 0; m < SB; ++m) acc[m][r] = fma(x[m], kr, acc[m][r]);
      }
    }
    i0 += st0; i1 += st1;
    if (i0 >= I0) { i0 -= I0; i1 += 1; }
  }

  __shared__ double red[SLAB_THREADS / 32][SB * RB + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < SB; ++m)
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < R) {
        double v = warp_sum((double)acc[m][r]);
        if (lane == 0) red[wid][m * RB + r] = v;
      }
    }
  __syncthreads();
  for (int e = threadIdx.x; e < SB * RB; e += SLAB_THREADS) {
    double t = 0.0;
    for (int q = 0; q < SLAB_THREADS / 32; ++q) t += red[q][e];
    int m = e / RB, r = e - m * RB;
    a.slab_part[((long long)blockIdx.x * SB + m) * RSTRIDE + r] = t;
  }
  ktime_end(a.ktime ? a.ktime + 4 : nullptr);
}

// ---------------------------------------------------------------------------
// contractions of T (mode 0 / mode 1 MTTKRP), fp64 outputs into MTT[s];
// TE here is the storage type of T (= the fiber pass compute type)
// ---------------------------------------------------------------------------
template <typename TE>
__global__ void __launch_bounds__(256)
contract0_kernel(XArgs a, const RowUnit* __restrict__ units) {
  if (gated(a)) return;
  const RowUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1];
  const long long J = I0 * I1;
  // unit = (block, r, 32 consecutive i0); threads = 32 i0 lanes x 8 i1 groups
  const int r = u.r0 >> 20;
  const long long i0 = (u.r0 & 0xFFFFF) + (threadIdx.x & 31);
  const int grp = threadIdx.x >> 5;
  const double* A1 = a.U[3 * s + 1];
  const TE* T = reinterpret_cast<const TE*>(tbuf(a, s));
  const int ns = a.nsplit[s];
  double acc = 0.0;
  if (i0 < I0) {
    for (int sp = 0; sp < ns; ++sp) {
      const TE* Tr = T + ((long long)sp * R + r) * J + i0;
#pragma unroll 4
      for (long long i1 = grp; i1 < I1; i1 += 8) acc = fma((double)Tr[I0 * i1], A1[i1 * R + r], acc);
    }
  }
  __shared__ double part[8][33];
  part[grp][threadIdx.x & 31] = acc;
  __syncthreads();
  if (threadIdx.x < 32 && i0 < I0) {
    double t = 0.0;
    for (int g = 0; g < 8; ++g) t += part[g][threadIdx.x];
    a.MTT[s][i0 * R + r] = t;
  }
}

template <typename TE>
__global__ void __launch_bounds__(256)
contract1_kernel(XArgs a, const RowUnit* __restrict__ units) {
  if (gated(a)) return;
  const RowUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1];
  const long long J = I0 * I1;
  const int lane = threadIdx.x & 31;
  const long long p = (long long)u.r0 + (threadIdx.x >> 5);   // p = i1 * R + r
  if (p >= I1 * R) return;
  const long long i1 = p / R, r = p - i1 * R;
  const double* A0 = a.U[3 * s];
  const TE* T = reinterpret_cast<const TE*>(tbuf(a, s));
  const int ns = a.nsplit[s];
  double acc = 0.0;
  for (int sp = 0; sp < ns; ++sp) {
    const TE* Tr = T + ((long long)sp * R + r) * J + I0 * i1;
    for (long long i0 = lane; i0 < I0; i0 += 32) acc = fma((double)Tr[i0], A0[i0 * R + r], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) a.MTT[s][i1 * R + r] = acc;
}

}  // namespace cb
