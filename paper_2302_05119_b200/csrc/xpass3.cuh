// Mode-2 MTTKRP of the 3-way fast path as warp-level row dot products.
//
//   M2[i2, r] = sum_{i1} A1[i1, r] * sum_{i0} X[i0, i1, i2] A0[i0, r]
//
// One warp owns one task (block s, slab i2) and walks its I1 rows; a row
// X[:, i1, i2] is I0 contiguous elements, lane l holding i0 = l + 32k
// (k < NSLOT).  The lane keeps its A0 rows in registers for the whole task,
// so a row costs NSLOT * RB fp64 FMAs per lane with no shared-memory traffic;
// the R partial dot products are then folded across the warp by a recursive-
// halving butterfly (VP - VP/32 shuffles for VP padded values instead of
// 5 per value), after which lane l holds value (l * VP) / 32, scales it by
// A1[i1, r] and accumulates.  Rows are prefetched PD deep into registers.
// The task writes M2[i2, :] straight into MTT[s] (no partials, no second
// pass) in a fixed order: bitwise deterministic.
//
// Replaces the KR-row formulation (xpass2.cuh slab2_kernel) where it applies:
// I0 <= 32 * NSLOT (NSLOT <= 4) and rank bucket <= 16.
#pragma once
#include "xpass.cuh"

namespace cb {

constexpr int S3_WARPS = 4;
constexpr int S3_HDR = 256;  // mbarriers: S3_WARPS x ring slots (<= 4) x 8 B
constexpr int S3_PD = 3;    // rows prefetched ahead per warp

__host__ __device__ constexpr int s3_vp(int rb) { return rb <= 8 ? 8 : 16; }

// sum over the 32 lanes of v[0..VP); returns the total of value (lane*VP)/32
template <int VP>
__device__ __forceinline__ double warp_fold(double (&v)[VP], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st;
    const int c = VP >> st;
    if (c > 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < c / 2; ++i) {
        const double send = up ? v[i] : v[i + c / 2];
        const double keep = up ? v[i + c / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  return v[0];
}

// tasks: global slab index t in [0, ntasks); block s owns [task_first[s], task_first[s+1]).
// Per task the lane accumulates, over the I1 rows, acc[k][r] += x[i0_k] A1[i1, r]
// (A1 row: broadcast L1 read, prefetched one row ahead); at the end of the
// task it forms v[r] = sum_k A0[i0_k, r] acc[k][r] and folds v across the warp
// once.  RING > 0: the task's rows (one contiguous span of X) stream through a
// private RING-stage shared-memory ring of `rows` rows per stage, one bulk
// copy per stage issued by lane 0 (needs 16-B aligned rows); RING == 0: rows
// are prefetched S3_PD deep into registers with __ldg.
template <typename TE, int RB, int NSLOT, int RING>
__global__ void __launch_bounds__(S3_WARPS * 32, 3)
slab3_kernel(XArgs a, const int* __restrict__ task_first, int S, int ntasks, int rows,
             int a1_rows) {
  griddep_wait();
  if (gated(a)) return;
  tl_begin(a.tl, TL_SLAB);
  constexpr int VP = s3_vp(RB);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int vi = (lane * VP) >> 5;                 // value index this lane ends with
  const bool writer = (lane & ((32 / VP) - 1)) == 0;
  extern __shared__ __align__(128) unsigned char s3sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(s3sm) + warp * (RING > 0 ? RING : 1);
  // per warp: A1 copy [a1_rows][RB] (fp64, zero-padded), then the X ring
  double* a1s = reinterpret_cast<double*>(s3sm + S3_HDR) + (size_t)warp * a1_rows * RB;
  TE* ring_base = reinterpret_cast<TE*>(reinterpret_cast<double*>(s3sm + S3_HDR) +
                                        (size_t)S3_WARPS * a1_rows * RB);
  int cur = -1;
  const TE* X = nullptr;
  const double* A0 = nullptr;
  long long I0 = 0, J = 0;
  int I1 = 0, R = 0;
  int s = 0;
  uint32_t phase_bits = 0;      // RING: parity per ring slot
  if constexpr (RING > 0) {
    if (lane == 0)
      for (int q = 0; q < RING; ++q) mbar_init(&bar[q], 1);
    mbar_fence_init();
    __syncwarp();
  }
  for (int t = blockIdx.x * S3_WARPS + warp; t < ntasks; t += gridDim.x * S3_WARPS) {
    while (s + 1 < S && t >= task_first[s + 1]) ++s;
    if (a.active && !a.active[s]) continue;
    if (s != cur) {
      cur = s;
      R = a.R[s];
      I0 = a.dims[3 * s];
      I1 = (int)a.dims[3 * s + 1];
      J = I0 * I1;
      X = reinterpret_cast<const TE*>(a.X[s]);
      A0 = a.U[3 * s];
      const double* A1 = a.U[3 * s + 1];
      __syncwarp();
      for (long long e = lane; e < (long long)I1 * RB; e += 32) {
        const long long q = e / RB;
        const int r = (int)(e - q * RB);
        a1s[e] = r < R ? __ldg(A1 + q * R + r) : 0.0;
      }
      __syncwarp();
    }
    const long long i2 = t - task_first[s];
    const TE* xs = X + i2 * J;
    double acc[NSLOT][RB];
#pragma unroll
    for (int k = 0; k < NSLOT; ++k)
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[k][r] = 0.0;
    auto row = [&](const TE* xr, int i1, bool from_ring) {
      double an[RB];            // A1 row (broadcast shared-memory read)
      load_row<double, RB>(a1s + (size_t)i1 * RB, an);
#pragma unroll
      for (int k = 0; k < NSLOT; ++k) {
        const long long i0 = lane + 32 * k;
        const double x = i0 < I0 ? (double)(from_ring ? xr[i0] : __ldg(xr + i0)) : 0.0;
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[k][r] = fma(x, an[r], acc[k][r]);
      }
    };
    if constexpr (RING > 0) {
      const long long stage_elems = (long long)rows * I0;
      TE* ring = ring_base + (size_t)warp * RING * stage_elems;
      const int nst = (I1 + rows - 1) / rows;
      auto issue = [&](int k) {
        const int q = k % RING;
        const int r0 = k * rows;
        const int nr = I1 - r0 < rows ? I1 - r0 : rows;
        const uint32_t bytes = (uint32_t)(nr * I0 * sizeof(TE));
        mbar_arrive_expect_tx(&bar[q], bytes);
        bulk_g2s(ring + (size_t)q * stage_elems, xs + (long long)r0 * I0, bytes, &bar[q]);
      };
      if (lane == 0)
        for (int k = 0; k < nst && k < RING; ++k) issue(k);
      for (int k = 0; k < nst; ++k) {
        const int q = k % RING;
        mbar_wait(&bar[q], (phase_bits >> q) & 1u);
        phase_bits ^= 1u << q;
        const TE* xr = ring + (size_t)q * stage_elems;
        const int r0 = k * rows;
        const int nr = I1 - r0 < rows ? I1 - r0 : rows;
        for (int rr = 0; rr < nr; ++rr) row(xr + (size_t)rr * I0, r0 + rr, true);
        __syncwarp();   // slot consumed by every lane
        if (lane == 0 && k + RING < nst) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(k + RING);
        }
      }
    } else {
      for (int i1 = 0; i1 < I1; ++i1) row(xs + (long long)i1 * I0, i1, false);
    }
    // v[r] = sum_k A0[i0_k, r] acc[k][r], then one warp fold
    double v[VP];
#pragma unroll
    for (int r = 0; r < VP; ++r) v[r] = 0.0;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
      const long long i0 = lane + 32 * k;
      if (i0 < I0) {
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (r < R) v[r] = fma(__ldg(A0 + i0 * R + r), acc[k][r], v[r]);
      }
    }
    const double w = warp_fold<VP>(v, lane);
    if (writer && vi < R) a.MTT[s][i2 * R + vi] = w;
  }
  tl_end(a.tl, TL_SLAB);
}

constexpr int S3_RING = 3;

// rows per ring stage (~2 KB per stage) and the kernel's dynamic smem
inline int slab3_rows(long long max_i0, int elem) {
  const long long per = 2048 / (max_i0 * elem);
  return (int)(per < 1 ? 1 : per);
}
inline size_t slab3_smem(long long max_i0, int elem, int rows, long long a1_rows, int rb,
                         bool ring) {
  return S3_HDR + (size_t)S3_WARPS * a1_rows * rb * 8 +
         (ring ? (size_t)S3_WARPS * S3_RING * rows * max_i0 * elem : 0);
}

// Sizing rule of the unsplit T pass (T = X x3 A2 written once per block,
// the fiber4 kernel of xpass4.cuh): A2 staged per warp must fit.
constexpr int F3_WARPS = 8;
constexpr int F3_CH = 64;        // j per unit of the f3 table

inline size_t fiber3_smem(long long a2_rows, int rb) {
  return (size_t)F3_WARPS * a2_rows * rb * 8;
}

// usable for these shapes?  (all blocks)
inline bool slab3_ok(int S, const long long* dims, int rb) {
  if (rb > 16) return false;
  for (int s = 0; s < S; ++s)
    if (dims[3 * s] > 128) return false;
  return true;
}

inline int slab3_nslot(int S, const long long* dims) {
  long long m = 1;
  for (int s = 0; s < S; ++s) m = dims[3 * s] > m ? dims[3 * s] : m;
  return (int)((m + 31) / 32);
}

}  // namespace cb
