// Register-tiled, bulk-copy-fed streaming kernels of the 3-way fast path.
//
// Both passes are skinny GEMMs over the dense block (see xpass.cuh for the
// notation):
//   fiber : T[j, r]  = sum_{i2} X[j, i2] A2[i2, r]      M = j (contiguous), K = i2
//   slab  : M2[i2, r] = sum_j X[j, i2] KR[j, r]          M = i2, K = j (contiguous),
//           KR[j, r] = A0[i0(j), r] A1[i1(j), r]
// N = R is small (5..64), so these run on CUDA cores with register tiles that
// reuse every operand fetched from shared memory: a fiber thread owns TJ
// columns j (TJ x R accumulators), a slab thread owns TM slabs i2 (TM x R
// accumulators); the R-wide A2 / KR rows are read as 16-byte vectors and
// shared by the TJ (TM) FMAs.  X streams through a multi-stage shared-memory
// ring filled by 1-D bulk copies (cp.async.bulk + mbarrier), so the bytes in
// flight per SM do not depend on register pressure; where rows are not 16-byte
// aligned the same kernels read X directly from global memory instead.
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include "xpass.cuh"

namespace cb {

constexpr int X2_THREADS = 256;
constexpr int F2_CH = 4;     // fiber: i2 rows per stage
constexpr int F2_NST = 4;    // fiber: stages in flight
constexpr int S2_NST = 3;    // slab: stages in flight

// register tile sizes: keep TJ*RB (TM*RB) accumulators within ~48 fp64 / 96 fp32
__host__ __device__ constexpr int x2_tile(int rb, int tc_bytes) {
  return tc_bytes == 8 ? (rb <= 12 ? 4 : rb <= 24 ? 2 : 1) : (rb <= 24 ? 4 : rb <= 48 ? 2 : 1);
}

// dynamic smem: X ring + the unit's A2 rows (max_rows x RB, TC), staged once
template <typename TE, typename TC, int RB>
__host__ __device__ constexpr size_t fiber2_smem(long long max_rows, int tj) {
  return 128 + (size_t)F2_NST * F2_CH * X2_THREADS * tj * sizeof(TE) +
         (size_t)max_rows * RB * sizeof(TC);
}

// slab: j elements per stage
__host__ __device__ constexpr int s2_kc(int rb, int tc_bytes) { return rb * tc_bytes <= 128 ? 512 : 256; }

// dynamic smem: X ring + (optionally) A0 / A1 rows (kr_rows x RB, TC)
template <typename TE, typename TC, int RB>
__host__ __device__ constexpr size_t slab2_smem(long long kr_rows) {
  return 128 + (size_t)S2_NST * x2_tile(RB, sizeof(TC)) * s2_kc(RB, sizeof(TC)) * sizeof(TE) +
         (size_t)kr_rows * RB * sizeof(TC);
}

// R-wide row of TC values from shared memory as 16-byte vectors
template <typename TC, int RB>
__device__ __forceinline__ void load_row(const TC* __restrict__ p, TC (&v)[RB]) {
  // 16-byte vectors while they fit (rows must start 16-byte aligned when
  // RB * sizeof(TC) is a multiple of 16), then a scalar tail
  constexpr int PER = 16 / sizeof(TC);
  if constexpr ((RB * sizeof(TC)) % 16 != 0) {
#pragma unroll
    for (int r = 0; r < RB; ++r) v[r] = p[r];
    return;
  }
#pragma unroll
  for (int q = 0; q < RB / PER; ++q) {
    if constexpr (sizeof(TC) == 8) {
      const double2 t = reinterpret_cast<const double2*>(p)[q];
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    } else {
      const float4 t = reinterpret_cast<const float4*>(p)[q];
      v[4 * q] = t.x;
      v[4 * q + 1] = t.y;
      v[4 * q + 2] = t.z;
      v[4 * q + 3] = t.w;
    }
  }
}

// ---------------------------------------------------------------------------
// fiber pass, unit = (block, i2 split, j-tile of 256*TJ columns)
// ---------------------------------------------------------------------------
template <typename TE, typename TC, int RB, bool STORE_T, bool WANT_B, bool WANT_RES, int TJ_>
__global__ void __launch_bounds__(X2_THREADS)
fiber2_kernel(XArgs a, const FibUnit* __restrict__ units, int use_tma) {
  griddep_wait();
  constexpr int TJ = TJ_;
  constexpr int JT = X2_THREADS * TJ;
  if (gated(a)) return;
  const FibUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  ktime_begin(a.ktime);
  tl_begin(a.tl, TL_FIBER);
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

  extern __shared__ __align__(128) unsigned char fsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(fsm);
  TE* xbuf = reinterpret_cast<TE*>(fsm + 128);
  TC* a2t = reinterpret_cast<TC*>(fsm + 128 + (size_t)F2_NST * F2_CH * JT * sizeof(TE));
  __shared__ double red[X2_THREADS / 32][RB + 1];

  long long jq[TJ];
  bool ok[TJ];
  long long i0q[TJ], i1q[TJ];
#pragma unroll
  for (int t = 0; t < TJ; ++t) {
    jq[t] = u.j0 + threadIdx.x + (long long)t * X2_THREADS;
    ok[t] = jq[t] < J;
    i1q[t] = ok[t] ? jq[t] / I0 : 0;
    i0q[t] = ok[t] ? jq[t] - i1q[t] * I0 : 0;
  }
  TC acc[TJ][RB];
#pragma unroll
  for (int t = 0; t < TJ; ++t)
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[t][r] = TC(0);
  TC w[WANT_RES ? TJ : 1][WANT_RES ? RB : 1];
  double res = 0.0;
  if constexpr (WANT_RES) {
    const double* lam = a.LAM ? a.LAM[s] : nullptr;
#pragma unroll
    for (int t = 0; t < TJ; ++t)
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double v = 0.0;
        if (r < R && ok[t]) v = (lam ? lam[r] : 1.0) * A0[i0q[t] * R + r] * A1[i1q[t] * R + r];
        w[t][r] = (TC)v;
      }
  }

  const long long jlen = (J - u.j0) < JT ? (J - u.j0) : JT;
  const uint32_t row_bytes = (uint32_t)(jlen * sizeof(TE));
  const int nstages = (int)((i2e - i2b + F2_CH - 1) / F2_CH);
  auto issue = [&](int k) {
    const int slot = k % F2_NST;
    const long long r0 = i2b + (long long)k * F2_CH;
    const int nr = (int)((i2e - r0) < F2_CH ? (i2e - r0) : F2_CH);
    mbar_arrive_expect_tx(&bar[slot], nr * row_bytes);
    for (int q = 0; q < nr; ++q)
      bulk_g2s(xbuf + ((size_t)slot * F2_CH + q) * JT, X + u.j0 + J * (r0 + q), row_bytes,
               &bar[slot]);
  };
  if (use_tma) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < F2_NST; ++st) mbar_init(&bar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < nstages && k < F2_NST; ++k) issue(k);
  }
  // all A2 rows of the unit in one round trip (overlapping the first copies);
  // the stage loop below then touches global memory only through the TMA ring
  {
    const long long nrow = i2e - i2b;
    for (long long e = threadIdx.x; e < nrow * RB; e += X2_THREADS) {
      const long long q = e / RB;
      const int r = (int)(e - q * RB);
      a2t[e] = r < R ? (TC)A2[(i2b + q) * R + r] : TC(0);
    }
  }
  __syncthreads();
  for (int k = 0; k < nstages; ++k) {
    const int slot = k % F2_NST;
    const long long r0 = i2b + (long long)k * F2_CH;
    const int nr = (int)((i2e - r0) < F2_CH ? (i2e - r0) : F2_CH);
    const TC* as = a2t + (size_t)k * F2_CH * RB;
    if (use_tma) mbar_wait(&bar[slot], (uint32_t)((k / F2_NST) & 1));
    const TE* xs = xbuf + (size_t)slot * F2_CH * JT + threadIdx.x;
#pragma unroll 2
    for (int q = 0; q < nr; ++q) {
      TC x[TJ];
#pragma unroll
      for (int t = 0; t < TJ; ++t) {
        if (use_tma) x[t] = (TC)xs[q * JT + t * X2_THREADS];
        else x[t] = ok[t] ? (TC)__ldcs(X + jq[t] + J * (r0 + q)) : TC(0);
      }
      TC av[RB];
      load_row<TC, RB>(as + q * RB, av);
      TC m[WANT_RES ? TJ : 1];
#pragma unroll
      for (int t = 0; t < (WANT_RES ? TJ : 1); ++t) m[t] = TC(0);
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (r < R) {
#pragma unroll
          for (int t = 0; t < TJ; ++t) {
            acc[t][r] = fma(x[t], av[r], acc[t][r]);
            if constexpr (WANT_RES) m[t] = fma(w[t][r], av[r], m[t]);
          }
        }
      }
      if constexpr (WANT_RES) {
#pragma unroll
        for (int t = 0; t < TJ; ++t)
          if (ok[t]) { const double d = (double)x[t] - (double)m[t]; res = fma(d, d, res); }
      }
    }
    if (use_tma) {
      __syncthreads();   // slot fully consumed
      if (threadIdx.x == 0 && k + F2_NST < nstages) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + F2_NST);
      }
    }
  }

  if constexpr (STORE_T) {
    TC* T = reinterpret_cast<TC*>(tbuf(a, s)) + (long long)u.split * R * J;
#pragma unroll
    for (int t = 0; t < TJ; ++t)
      if (ok[t]) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (r < R) T[(long long)r * J + jq[t]] = acc[t][r];
      }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if constexpr (WANT_B) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < R) {
        double v = 0.0;
#pragma unroll
        for (int t = 0; t < TJ; ++t)
          if (ok[t]) v = fma((double)acc[t][r], A0[i0q[t] * R + r] * A1[i1q[t] * R + r], v);
        v = warp_sum(v);
        if (lane == 0) red[wid][r] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int q = 0; q < X2_THREADS / 32; ++q) t += red[q][threadIdx.x];
      a.bpart[(long long)blockIdx.x * RSTRIDE + threadIdx.x] = t;
    }
  }
  if constexpr (WANT_RES) {
    __syncthreads();
    const double v = warp_sum(res);
    if (lane == 0) red[wid][0] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < X2_THREADS / 32; ++q) t += red[q][0];
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
        for (int q = threadIdx.x; q < nunits; q += X2_THREADS) t += __ldcg(&a.rpart[first + q]);
        t = block_sum(t, &red[0][0]);
        if (threadIdx.x == 0) a.rsum[s] = t;
      }
      if (threadIdx.x == 0) a.blk_cnt[s] = 0;
    }
  }
  ktime_end(a.ktime);
  tl_end(a.tl, TL_FIBER);
}

// ---------------------------------------------------------------------------
// slab pass, unit = (block, TM consecutive i2 slabs, j-range [k0, k1))
// Per stage the CTA forms KR for KC consecutive j (factor rows read through
// L1: consecutive j share the A1 row) and streams the TM slab rows of that
// j-range.
// ---------------------------------------------------------------------------
template <typename TE, typename TC, int RB>
__global__ void __launch_bounds__(X2_THREADS)
slab2_kernel(XArgs a, const SlabUnit* __restrict__ units, int use_tma) {
  griddep_wait();
  constexpr int TM = x2_tile(RB, sizeof(TC));
  constexpr int S2_KC = s2_kc(RB, sizeof(TC));
  constexpr int PER_T = S2_KC / X2_THREADS;   // j per thread per stage
  if (gated(a)) return;
  const SlabUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  ktime_begin(a.ktime ? a.ktime + 4 : nullptr);
  tl_begin(a.tl, TL_SLAB);
  const int R = a.R[s];
  const long long I0 = a.dims[3 * s], I1 = a.dims[3 * s + 1], I2 = a.dims[3 * s + 2];
  const long long J = I0 * I1;
  const TE* __restrict__ X = reinterpret_cast<const TE*>(a.X[s]);
  const double* __restrict__ A0 = a.U[3 * s];
  const double* __restrict__ A1 = a.U[3 * s + 1];
  const int nsl = (int)(I2 - u.g0 < TM ? I2 - u.g0 : TM);

  extern __shared__ __align__(128) unsigned char ssm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(ssm);
  TE* xbuf = reinterpret_cast<TE*>(ssm + 128);                       // [NST][TM][KC]
  TC* a0s = reinterpret_cast<TC*>(ssm + 128 + (size_t)S2_NST * TM * S2_KC * sizeof(TE));  // [I0][RB]
  TC* a1s = a0s + (size_t)I0 * RB;                                                        // [I1][RB]
  __shared__ double red[X2_THREADS / 32][RB + 1];
  // factor rows staged once when they fit (stage_ab); otherwise read via L1
  const bool stage_ab = a.slab_stage_rows >= I0 + I1;
  const long long nk = u.k1 - u.k0;
  const int nstages = (int)((nk + S2_KC - 1) / S2_KC);
  auto issue = [&](int k) {
    const int slot = k % S2_NST;
    const long long kb = u.k0 + (long long)k * S2_KC;
    const long long len = (u.k1 - kb) < S2_KC ? (u.k1 - kb) : S2_KC;
    const uint32_t bytes = (uint32_t)(len * sizeof(TE));
    mbar_arrive_expect_tx(&bar[slot], nsl * bytes);
    for (int m = 0; m < nsl; ++m)
      bulk_g2s(xbuf + ((size_t)slot * TM + m) * S2_KC, X + J * (u.g0 + m) + kb, bytes, &bar[slot]);
  };
  if (use_tma) {
    if (threadIdx.x == 0) {
      for (int st = 0; st < S2_NST; ++st) mbar_init(&bar[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < nstages && k < S2_NST; ++k) issue(k);
  }
  TC acc[TM][RB];
#pragma unroll
  for (int m = 0; m < TM; ++m)
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[m][r] = TC(0);
  if (stage_ab) {
    for (long long e = threadIdx.x; e < (I0 + I1) * RB; e += X2_THREADS) {
      const long long i = e / RB;
      const int r = (int)(e - i * RB);
      a0s[e] = r < R ? (TC)(i < I0 ? A0[i * R + r] : A1[(i - I0) * R + r]) : TC(0);
    }
  }
  __syncthreads();

  for (int k = 0; k < nstages; ++k) {
    const int slot = k % S2_NST;
    const long long kb = u.k0 + (long long)k * S2_KC;
    const int len = (int)((u.k1 - kb) < S2_KC ? (u.k1 - kb) : S2_KC);
    if (use_tma) mbar_wait(&bar[slot], (uint32_t)((k / S2_NST) & 1));
    const TE* xs = xbuf + (size_t)slot * TM * S2_KC;
#pragma unroll
    for (int p = 0; p < PER_T; ++p) {
      const int q = threadIdx.x + p * X2_THREADS;
      if (q < len) {
        TC x[TM];
#pragma unroll
        for (int m = 0; m < TM; ++m) {
          if (m < nsl) x[m] = use_tma ? (TC)xs[m * S2_KC + q] : (TC)__ldcs(X + J * (u.g0 + m) + kb + q);
          else x[m] = TC(0);
        }
        // KR row of this j in registers: A0[i0, :] * A1[i1, :]
        const long long j = kb + q;
        const long long i1 = j / I0, i0 = j - i1 * I0;
        TC kr[RB];
        if (stage_ab) {
          TC b1[RB];
          load_row<TC, RB>(a0s + (size_t)i0 * RB, kr);
          load_row<TC, RB>(a1s + (size_t)i1 * RB, b1);
#pragma unroll
          for (int r = 0; r < RB; ++r) kr[r] *= b1[r];
        } else {
#pragma unroll
          for (int r = 0; r < RB; ++r)
            kr[r] = r < R ? (TC)(__ldg(A0 + i0 * R + r) * __ldg(A1 + i1 * R + r)) : TC(0);
        }
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (r < R) {
#pragma unroll
            for (int m = 0; m < TM; ++m) acc[m][r] = fma(x[m], kr[r], acc[m][r]);
          }
      }
    }
    if (use_tma) {
      __syncthreads();   // slot fully consumed
      if (threadIdx.x == 0 && k + S2_NST < nstages) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S2_NST);
      }
    }
  }

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < TM; ++m) {
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < R) {
        const double v = warp_sum((double)acc[m][r]);
        if (lane == 0) red[wid][r] = v;
      }
    __syncthreads();
    if (threadIdx.x < R) {
      double t = 0.0;
      for (int q = 0; q < X2_THREADS / 32; ++q) t += red[q][threadIdx.x];
      a.slab_part[((long long)blockIdx.x * TM + m) * RSTRIDE + threadIdx.x] = t;
    }
    __syncthreads();
  }
  ktime_end(a.ktime ? a.ktime + 4 : nullptr);
  tl_end(a.tl, TL_SLAB);
}

}  // namespace cb
