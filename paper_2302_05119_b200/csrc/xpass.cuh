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

constexpr int RSTRIDE = 64;       // per-unit partial stride (>= max rank)

struct FibUnit { int s; int split; long long j0; };
struct SlabUnit { int s; int g0; long long k0; long long k1; };
struct RowUnit { int s; int r0; };

struct XArgs {
  const void* const* X;          // per block tensor
  const long long* dims;         // S*3
  const int* R;                  // per block rank
  const double* const* U;        // S*3 current factors
  const double* const* UT;       // optional transposed factors [r][I_n] (ALS: written by its solve), or null
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
  unsigned long long* tl;        // profiling only: iteration timeline (TlSlot)
  long long slab_stage_rows;     // factor rows the slab kernel may stage in smem (0: none)
  const int* s3_first;           // slab3: S+1 cumulative slab counts (task ranges)
  const int* f3_first;           // fiber3: S+1 cumulative fiber-row counts
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

// Iteration timeline (profiling only; tl non-null): per kernel slot, the
// earliest CTA start (tl[2*slot], atomicMin) and the latest CTA end seen by
// thread 0 (tl[2*slot+1], atomicMax).
__device__ __forceinline__ void tl_begin(unsigned long long* tl, int slot) {
  if (tl && threadIdx.x == 0) atomicMin(&tl[2 * slot], gtimer());
}
__device__ __forceinline__ void tl_end(unsigned long long* tl, int slot) {
  if (tl && threadIdx.x == 0) atomicMax(&tl[2 * slot + 1], gtimer());
}
enum TlSlot {
  TL_SWEEP = 0, TL_C0 = 1, TL_C1 = 2, TL_SLAB = 3, TL_FIBER = 4, TL_MU = 5, TL_FIN = 8,
  TL_STEP = 11, TL_CONTROL = 14, TL_COMMON = 15, TL_QR = 18, TL_RESTORE = 20, TL_TRACE = 21,
  TL_PREP = 22, TL_NSLOT = 24
};

__device__ __forceinline__ bool gated(const XArgs& a) {
  return a.gate != nullptr && *a.gate == 0;
}
__device__ __forceinline__ void* tbuf(const XArgs& a, int s) {
  const int sel = (a.tsel ? *a.tsel : 0) ^ a.t_other;
  return sel ? a.T1[s] : a.T0[s];
}

// ---------------------------------------------------------------------------
// contractions of T (mode 0 / mode 1 MTTKRP), fp64 outputs into MTT[s];
// TE here is the storage type of T (= the fiber pass compute type)
// ---------------------------------------------------------------------------
template <typename TE>
__global__ void __launch_bounds__(256)
contract0_kernel(XArgs a, const RowUnit* __restrict__ units) {
  griddep_wait();
  if (gated(a)) return;
  const RowUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  tl_begin(a.tl, TL_C0);
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
  tl_end(a.tl, TL_C0);
}

template <typename TE>
__global__ void __launch_bounds__(256)
contract1_kernel(XArgs a, const RowUnit* __restrict__ units) {
  griddep_wait();
  if (gated(a)) return;
  const RowUnit u = units[blockIdx.x];
  const int s = u.s;
  if (a.active && !a.active[s]) return;
  tl_begin(a.tl, TL_C1);
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
  if (a.UT) {
    // column r of A0 from the transposed copy: both operands contiguous
    const double* A0t = a.UT[3 * s] + r * I0;
    for (int sp = 0; sp < ns; ++sp) {
      const TE* Tr = T + ((long long)sp * R + r) * J + I0 * i1;
      for (long long i0 = lane; i0 < I0; i0 += 32) acc = fma((double)Tr[i0], A0t[i0], acc);
    }
  } else {
    for (int sp = 0; sp < ns; ++sp) {
      const TE* Tr = T + ((long long)sp * R + r) * J + I0 * i1;
      for (long long i0 = lane; i0 < I0; i0 += 32) acc = fma((double)Tr[i0], A0[i0 * R + r], acc);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) a.MTT[s][i1 * R + r] = acc;
  tl_end(a.tl, TL_C1);
}

}  // namespace cb
