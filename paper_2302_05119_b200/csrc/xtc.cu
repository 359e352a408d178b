// Tensor-core trace pass: b_s[r] = sum X_s[i0,i1,i2] A0[i0,r] A1[i1,r] A2[i2,r]
// (reference: core_linear_term, solver.py:215-218; lra trace b_orig,
// solver.py:519-522) for 3-way fp32 blocks, on the 5th-generation tensor
// cores with EXACT integer accumulation.
//
// Formulation.  View block s as the row-major matrix Xr (rows = (i1,i2),
// J = I1*I2 rows; K = i0, I0 columns).  Then
//      D = A0^T . Xr^T      (R x J, a GEMM with K = I0)
//      b[r] = sum_rows A1[i1,r] A2[i2,r] D[r,row]   (fp64 epilogue)
// The reference computes in fp64; this pass reaches ~2^-22 relative per
// product with zero bias, via fixed-point byte slices and int8 MMAs:
//   * X: one exponent per block (max|X| = m 2^eX, m in [0.5, 1)), q =
//     rint(x 2^(22-eX)) = a0 2^16 + a1 2^8 + a2 with balanced signed bytes
//     (a0 in [-64, 64]).  The three byte planes are written ONCE per solve
//     (k_xtc_pack) in the MMA's shared-memory layout (K-major rows of 32
//     bytes, 32-byte swizzle), tile by tile: an iteration then streams 3
//     bytes per element instead of 4 and does no conversion work.
//   * A0: one exponent per column, p = rint(u 2^(22-eU_r)) as balanced
//     signed bytes p = b0 2^16 + b1 2^8 + b2 (b0 in [-64, 64]), per call.
//   * sum_k q_k p_k = 2^32 L0 + 2^24 L1 + 2^16 L2 + (dropped levels 3-4),
//     L0 = a0.b0, L1 = a0.b1 + a1.b0, L2 = a0.b2 + a1.b1 + a2.b0 (exact
//     int32; |L| < 2^31 for I0 <= 32768).  The dropped terms are products of
//     two balanced signed digits, ~2^-21 of a product, zero-mean.
//   * operand roles.  A kind::i8 MMA of M = 128, K = 32 costs ~220 cycles
//     whatever its N (tools/micro/imma_probe.cu), so the X rows go on N
//     (256 per instruction) and the factor on M: the three slices of a column
//     are stacked along M with a level's rows together, image rows
//     [0 (Rp); 0 (Rp); b0; b1; b2; 0], Rp = R rounded up to 8, 3 Rp <= 128.
//     The M = 128 window starting at row (2 - i) Rp is the operand for plane
//     a_i: window 2 Rp = [b0; b1; b2], window Rp = [0; b0; b1], window 0 =
//     [0; 0; b0], so three MMAs per K step accumulate D lanes [l Rp, (l+1) Rp)
//     = level l for 256 rows of X (the lanes past 3 Rp collect dropped-level
//     products and are not read).
// Error: unbiased rounding of x (2^-23 of the block max) and u (2^-23 of the
// column max); measured ~1e-8 relative on b.  The lra objective's
// cancellation (res ~ 1% of |M|^2 at 20 dB) turns that into ~1e-6 on RelErr,
// inside the fp32-mode 1e-4 (tests/test_gpu_xtc.py, tests/test_gpu_solve.py).
//
// Kernel (persistent, one CTA per SM, 320 threads):
//   warp 9  : producer - 24 KB bulk copies (one K = 32 step of a 256-row
//             tile, three planes) into an NST-stage ring, plus the block's
//             factor image (prepared by k_xtc_prep) per segment;
//   warp 8  : MMA issuer - one lane issues tcgen05.mma (both operands from
//             shared memory), tcgen05.commit frees ring stages / publishes D;
//   warps 0-7: epilogue, one TMEM lane quarter x one half of the 256 columns
//             each: a thread owns (level, r), walks its 128 rows with the
//             weights A1[i1,r] (fp32, L2-resident, prefetched a batch ahead)
//             and A2[i2,r], and keeps sum_rows w L in fp64 (int32 -> fp64
//             exactly through the fp64 adder).
// TMEM: 2 D buffers x 256 columns.
// Units of 4 tiles (never straddling a block) are the partial granularity:
// partials are reduced in fixed order and folded per block in unit order by
// the last arriving CTA, so b is bitwise independent of the grid size and
// of how blocks are sharded over GPUs.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "engine_host.h"
#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"
#include "tc.cuh"
#include "xtc.h"

namespace cb {

constexpr int XTC_NT = 256;                       // X rows per tile (MMA N)
constexpr int XTC_SX = 3;                         // byte planes of X
constexpr int XTC_PIECE = XTC_NT * 32;            // 8 KB: one plane of one K = 32 step
constexpr int XTC_STAGE = XTC_SX * XTC_PIECE;     // 24 KB per ring stage
constexpr int XTC_TPU = 4;                        // tiles per unit
constexpr int XTC_MAX_I0 = 512;
constexpr int XTC_MAX_R = 40;                     // 3 levels x Rp lanes <= 128
constexpr int XTC_XBITS = 22;
constexpr int XTC_UBITS = 22;
constexpr int XTC_WBITS = 26;                     // A1 row weights: |w| <= 2^26
constexpr int XTC_WB = 16;        // columns per epilogue batch
constexpr int XTC_THREADS = 320;  // 8 epilogue warps, MMA, producer
constexpr int XTC_SMEM_MAX = 227 * 1024;

struct XtcBlock {
  long long I0, I1, I2, J;
  int R, ntiles, nk;
  int ex;                 // fixed-point exponent of X
  int ufirst, nunits;
  int bimg_bytes;
  // per-call operands, two sets: the pipelined iteration prepares the next
  // trace's set while the current trace still reads the other
  double* aux[2];         // [64] scale_r
  int* w1[2];             // [I1][Rp] = rint(A1[i1, r] 2^(26 - e1_r)): 27-bit fixed-point row weights
                          // (zero-padded columns); 2^(e1_r - 26) is folded into aux
  float* w2[2];           // [I2][Rp] = A2[i2, r]
  unsigned char* bimg[2]; // [nk][2 Rp + 128 rows][32 B] (K-major, 32-B swizzle)
  const float* X;         // the block (read by the pack kernel only)
  unsigned char* planes;  // [ntiles][nk][3 planes][256 rows x 32 B]
};

struct XtcUnit { int s, t0, t1, u; };

struct XtcArgs {
  const XtcBlock* blk;
  const XtcUnit* units;
  int nunits;
  int nst;
  int bimg_max;
  int Rp;                 // lanes per level (max rank rounded up to 8)
  const int* par;         // operand set the trace reads (device; flipped by k_xtc_flip)
  int wr_other;           // prep: write the other set (pipelined), else the current one
  double* part;           // [unit][64]
  int* cnt;               // per-block arrival counters (self-resetting)
  double* bsum;           // [s][RSTRIDE]
  const int* gate;
  unsigned long long* tl; // iteration timeline (profiling) or null
};

struct XtcPlan {
  int S = 0, Rp = 0, nst = 0, grid = 0, nunits = 0, bimg_max = 0, ntiles = 0;
  int grid_cap = 0;          // > 0: at most this many CTAs (SMs left to concurrent work)
  size_t smem = 0;
  double bytes = 0.0;        // algorithmic: sum_s |X_s| x 4
  double stream_bytes = 0.0; // plane bytes one launch streams
  std::vector<void*> allocs;
  XtcBlock* blk = nullptr;
  XtcUnit* units = nullptr;
  double* part = nullptr;
  int* cnt = nullptr;
  int* par = nullptr;        // current operand set (device)
  unsigned int* maxbits = nullptr;
  unsigned long long* tl = nullptr;   // iteration timeline (profiling)
};

// --------------------------------------------------------------------------
// one-time: per-block max |X| (as float bits), the exponent eX, the planes
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_xtc_maxabs(const float* __restrict__ X, long long n,
                                                    unsigned int* out) {
  float m = 0.0f;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    m = fmaxf(m, fabsf(X[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__global__ void k_xtc_set_ex(XtcBlock* blk, const unsigned int* maxbits, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const float m = __uint_as_float(maxbits[s]);
  int e = 0;
  if (m > 0.0f && isfinite(m)) frexpf(m, &e);   // m = f 2^e, f in [0.5, 1)
  blk[s].ex = e;
}

// byte `byte` of four words as one word (k increasing with the address)
__device__ __forceinline__ uint32_t pick4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                          int byte) {
  const uint32_t sel = (uint32_t)byte | ((uint32_t)(byte + 4) << 4);
  return __byte_perm(__byte_perm(t0, t1, sel), __byte_perm(t2, t3, sel), 0x5410);
}

// grid (max tiles, 1, S), 256 threads: each warp transposes its 32 rows of a
// K = 32 step through shared memory (k is contiguous in X), thread m then
// owns row m: q + 0x8080 = a0 2^16 + (a1 + 128) 2^8 + (a2 + 128)
__global__ void __launch_bounds__(XTC_NT) k_xtc_pack(const XtcBlock* blk) {
  const XtcBlock& b = blk[blockIdx.z];
  const int t = blockIdx.x;
  if (t >= b.ntiles) return;
  __shared__ float tile[XTC_NT][33];
  const int m = threadIdx.x;
  const int warp = m >> 5, lane = m & 31;
  const float sx = ldexpf(1.0f, XTC_XBITS - b.ex);
  const float* __restrict__ X = b.X;
  const int sw = (m >> 2) & 1;
  for (int c = 0; c < b.nk; ++c) {
    const int kk = c * 32 + lane;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const long long rr = (long long)t * XTC_NT + warp * 32 + r;
      tile[warp * 32 + r][lane] = (rr < b.J && kk < b.I0) ? __ldcs(X + rr * b.I0 + kk) : 0.0f;
    }
    __syncwarp();
    uint32_t q[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) q[k] = (uint32_t)(__float2int_rn(tile[m][k] * sx) + 0x8080);
    __syncwarp();
    unsigned char* dst = b.planes + ((long long)t * b.nk + c) * XTC_STAGE + m * 32;
#pragma unroll
    for (int i = 0; i < XTC_SX; ++i) {
      uint32_t w[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        w[g] = pick4(q[4 * g], q[4 * g + 1], q[4 * g + 2], q[4 * g + 3], 2 - i);
        if (i > 0) w[g] ^= 0x80808080u;
      }
      uint4* d = reinterpret_cast<uint4*>(dst + i * XTC_PIECE);
      d[sw] = make_uint4(w[0], w[1], w[2], w[3]);
      d[sw ^ 1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
}

// --------------------------------------------------------------------------
// per call: A0 -> the stacked signed byte-slice image (the MMA's M-side
// operand, exactly the shared-memory layout), column scales, A1/A2 as fp32
// --------------------------------------------------------------------------
// grid (S, 4): parts 0 / 1 write the two halves of the factor image (part 0
// also the column scales), part 2 the A1 weights, part 3 the A2 weights
__global__ void __launch_bounds__(256) k_xtc_prep(XtcArgs a, const double* const* U) {
  griddep_wait();
  if (a.gate && *a.gate == 0) return;
  tl_begin(a.tl, TL_PREP);
  const int s = blockIdx.x;
  const int part = blockIdx.y;
  const XtcBlock b = a.blk[s];
  const int set = (*a.par) ^ a.wr_other;
  unsigned char* bimg = b.bimg[set];
  const double* A0 = U[3 * s];
  const double* A1 = U[3 * s + 1];
  const double* A2 = U[3 * s + 2];
  const int R = b.R, Rp = a.Rp;
  const int I0 = (int)b.I0;
  const long long I1 = b.I1, I2 = b.I2;
  const int SR = 2 * Rp + 128;        // image rows per K step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int eu[64];              // column exponents of A0
  __shared__ int e1[64];              // column exponents of A1
  // column exponent of an I x R factor: max |.| = m 2^e, m in [0.5, 1)
  auto col_exps = [&](const double* A, long long I, int* out) {
    for (int r = warp; r < Rp; r += 8) {
      double m = 0.0;
      if (r < R)
        for (long long i = lane; i < I; i += 32) m = fmax(m, fabs(A[i * R + r]));
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        int e = 0;
        if (m > 0.0) frexp(m, &e);
        out[r] = e;
      }
    }
  };
  if (part <= 1) {
    col_exps(A0, I0, eu);
    if (part == 0) col_exps(A1, I1, e1);
    __syncthreads();
    // rows [2 Rp + l Rp + n] = slice l of column n; everything else stays zero
    // (the image is zeroed at plan creation and only these bytes are rewritten)
    const int kmax = b.nk * 32;
    const int khalf = (b.nk + 1) / 2 * 32;
    const int k_lo = part == 0 ? 0 : khalf, k_hi = part == 0 ? min(khalf, kmax) : kmax;
    for (int e = k_lo * Rp + threadIdx.x; e < k_hi * Rp; e += 256) {
      const int k = e / Rp, n = e - (e / Rp) * Rp;
      long long p = 0;
      if (k < I0 && n < R) p = llrint(ldexp(A0[(long long)k * R + n], XTC_UBITS - eu[n]));
      const long long d2 = ((p + 128) & 255) - 128;
      const long long p1 = (p - d2) >> 8;
      const long long d1 = ((p1 + 128) & 255) - 128;
      const long long d0 = (p1 - d1) >> 8;
      const int c = k >> 5, kk = k & 31;
      // rows of 32 bytes, 16-byte halves swapped on rows with bit 2 set
      // (Swizzle<1,4,3>; the K-step images start on multiples of 256 bytes)
      auto put = [&](int l, long long d) {
        const int row = (2 + l) * Rp + n;
        const long long off =
            ((long long)c * SR + row) * 32 + (((kk >> 4) ^ ((row >> 2) & 1)) << 4) + (kk & 15);
        bimg[off] = (unsigned char)(signed char)d;
      };
      put(0, d0);
      put(1, d1);
      put(2, d2);
    }
    if (part == 0 && threadIdx.x < 64) {
      const int r = threadIdx.x;
      // q p = 2^16 (2^16 L0 + 2^8 L1 + L2); the A1 weights carry 2^(26 - e1)
      b.aux[set][r] =
          r < R ? ldexp(1.0, 16 + b.ex - XTC_XBITS + eu[r] - XTC_UBITS + e1[r] - XTC_WBITS) : 0.0;
    }
  } else if (part == 2) {
    // A1 as 27-bit fixed point per column: the epilogue multiplies the int32
    // levels by it in integer arithmetic (one IMAD.WIDE per row instead of
    // conversions and fp64 FMAs, which share their pipe with the MMAs)
    col_exps(A1, I1, e1);
    __syncthreads();
    for (long long e = threadIdx.x; e < I1 * Rp; e += 256) {
      const long long i = e / Rp;
      const int r = (int)(e - i * Rp);
      b.w1[set][e] = r < R ? (int)llrint(ldexp(A1[i * R + r], XTC_WBITS - e1[r])) : 0;
    }
  } else {
    for (long long e = threadIdx.x; e < I2 * Rp; e += 256) {
      const long long i = e / Rp;
      const int r = (int)(e - i * Rp);
      b.w2[set][e] = r < R ? (float)A2[i * R + r] : 0.0f;
    }
  }
  tl_end(a.tl, TL_PREP);
}

// the set just prepared becomes the one the next trace reads
__global__ void k_xtc_flip(int* par, const int* gate) {
  griddep_wait();
  if (gate && *gate == 0) return;
  if (threadIdx.x == 0) *par ^= 1;
}

// --------------------------------------------------------------------------
// the streaming MMA kernel
// --------------------------------------------------------------------------
// int32 -> double through the fp64 adder (exact): 2^52 + 2^31 + x
__device__ __forceinline__ double i2d_exact(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
}

template <int RP>
__global__ void __launch_bounds__(XTC_THREADS, 1) k_xtc_trace(XtcArgs a) {
  griddep_wait_no_trigger();
  if (a.gate && *a.gate == 0) return;
  tl_begin(a.tl, TL_TRACE);
  constexpr int NE = 256;            // epilogue threads
  constexpr int WMMA = 8, WTMA = 9;
  extern __shared__ unsigned char xtc_raw[];
  const uint32_t raw_u32 = smem_u32(xtc_raw);
  unsigned char* sm = xtc_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int nst = a.nst;
  constexpr int Rp = RP;
  constexpr int SR = 2 * Rp + 128;
  unsigned char* ring = sm;
  unsigned char* bimg = sm + (size_t)nst * XTC_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bimg + a.bimg_max);
  uint64_t* full = bars;
  uint64_t* empty = bars + nst;
  uint64_t* d_full = empty + nst;
  uint64_t* d_empty = d_full + 2;
  uint64_t* b_full = d_empty + 2;
  uint64_t* b_empty = b_full + 1;
  double* red = reinterpret_cast<double*>(b_empty + 1);      // [2 column halves][128 lanes]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + 256);
  int* shflag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int set = *a.par;
  const int G = gridDim.x;
  const int u_begin = (int)((long long)blockIdx.x * a.nunits / G);
  const int u_end = (int)((long long)(blockIdx.x + 1) * a.nunits / G);

  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], NE); }
    mbar_init(b_full, 1);
    mbar_init(b_empty, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == WTMA) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int st = 0, ph = 0, seg = 0, cur = -1;
      const uint64_t pol = l2_evict_first_policy();
      for (int u = u_begin; u < u_end; ++u) {
        const XtcUnit un = a.units[u];
        const XtcBlock& b = a.blk[un.s];
        const int nk = b.nk;
        if (un.s != cur) {
          mbar_wait(b_empty, (seg & 1) ^ 1);
          const int bytes = b.bimg_bytes;
          mbar_arrive_expect_tx(b_full, (uint32_t)bytes);
          for (int off = 0; off < bytes; off += 32768)
            bulk_g2s(bimg + off, b.bimg[set] + off, (uint32_t)min(32768, bytes - off), b_full);
          cur = un.s;
          ++seg;
        }
        for (int t = un.t0; t < un.t1; ++t) {
          const unsigned char* src = b.planes + (long long)t * nk * XTC_STAGE;
          for (int c = 0; c < nk; ++c) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], XTC_STAGE);
            bulk_g2s_hint(ring + (size_t)st * XTC_STAGE, src + (size_t)c * XTC_STAGE, XTC_STAGE,
                          &full[st], pol);
            if (++st == nst) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == WMMA) {
    // --------------------------------------------------------- MMA issuer
    // D lanes [l Rp, (l+1) Rp) += level l: plane a_i against the image window
    // starting at row (2 - i) Rp
    constexpr uint32_t idesc = idesc_i8(XTC_NT, 1, 1);
    int st = 0, ph = 0, seg = 0, cur = -1, tl = 0;
    const uint32_t bbase = smem_u32(bimg);
    const uint32_t rbase = smem_u32(ring);
    for (int u = u_begin; u < u_end; ++u) {
      const XtcUnit un = a.units[u];
      const XtcBlock& b = a.blk[un.s];
      const int nk = b.nk;
      if (un.s != cur) {
        mbar_wait(b_full, seg & 1);
        tc_fence_after();
        cur = un.s;
        ++seg;
      }
      const bool last_seg = (u + 1 == u_end) || a.units[u + 1].s != un.s;
      for (int t = un.t0; t < un.t1; ++t, ++tl) {
        const int buf = tl & 1;
        mbar_wait(&d_empty[buf], ((tl >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dc = tmem + (uint32_t)(buf * XTC_NT);
        for (int c = 0; c < nk; ++c) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t xb = rbase + (uint32_t)st * XTC_STAGE;
            const uint32_t fb = bbase + (uint32_t)(c * SR * 32);
            mma_i8_ss(dc, sdesc_k_sw32(fb + 2 * Rp * 32), sdesc_k_sw32(xb), idesc, c > 0 ? 1u : 0u);
            mma_i8_ss(dc, sdesc_k_sw32(fb + Rp * 32), sdesc_k_sw32(xb + XTC_PIECE), idesc, 1u);
            mma_i8_ss(dc, sdesc_k_sw32(fb), sdesc_k_sw32(xb + 2 * XTC_PIECE), idesc, 1u);
            tc_commit(&empty[st]);
            if (c == nk - 1) {
              tc_commit(&d_full[buf]);
              if (t == un.t1 - 1 && last_seg) tc_commit(b_empty);
            }
          }
          __syncwarp();
          if (++st == nst) { st = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 0-7)
    // warp = (column half ch, lane quarter wq); the thread's TMEM lane is
    // (level, r); it walks the 128 rows of its half in order, rows advancing
    // i1 first: inner = sum_i1 A1[i1,r] L (per i2 stretch, four interleaved
    // partial sums combined in a fixed order), acc += A2[i2,r] inner
    const int et = threadIdx.x;
    const int ch = warp >> 2;
    const int wq = warp & 3;
    const int L = wq * 32 + lane;
    const int lev = L / RP;
    const int r = L - lev * RP;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    double acc = 0.0;
    int tl = 0;
    for (int u = u_begin; u < u_end; ++u) {
      const XtcUnit un = a.units[u];
      const XtcBlock& b = a.blk[un.s];
      const int I1 = (int)b.I1;
      const long long J = b.J;
      // idle lanes (past the three levels, or columns >= R) read the zero
      // padding columns of the weight tables / a valid address and weigh
      // their products by zero
      const bool act = lev < 3 && r < b.R;
      const int* __restrict__ w1p = b.w1[set] + (act ? r : 0);
      const float* __restrict__ w2p = b.w2[set] + (act ? r : 0);
      const float wm = act ? 1.0f : 0.0f;
      for (int t = un.t0; t < un.t1; ++t, ++tl) {
        const int buf = tl & 1;
        const long long row0 = (long long)t * XTC_NT + ch * 128;
        int i2 = (int)(row0 / I1);
        int i1 = (int)(row0 - (long long)i2 * I1);
        const int nrow = (int)max(0LL, min(128LL, J - row0));   // rows of this half that exist
        // a batch is plain when all its rows exist and share one i2
        auto plain = [&](int j0, int i1s) { return j0 + XTC_WB <= nrow && i1s + XTC_WB <= I1; };
        // weights of a batch of columns: A1[i1s + j (wrapping), r]
        auto load_w1 = [&](int j0, int i1s, int (&w)[XTC_WB]) {
          if (plain(j0, i1s)) {
            const int* p = w1p + (long long)i1s * RP;
#pragma unroll
            for (int j = 0; j < XTC_WB; ++j) w[j] = __ldg(p + j * RP);
          } else {
#pragma unroll
            for (int j = 0; j < XTC_WB; ++j) {
              int i = i1s + j;
              if (i >= I1) i -= I1;   // one wrap at most (I1 >= XTC_WB)
              w[j] = j0 + j < nrow ? __ldg(w1p + (long long)i * RP) : 0;
            }
          }
        };
        int wc[XTC_WB], wn[XTC_WB];
        load_w1(0, i1, wc);
        float w2 = nrow > 0 ? wm * __ldg(w2p + (long long)i2 * RP) : 0.0f;
        // sum_i1 w L exactly in int64 (|w L| < 2^51, <= 128 rows), four
        // interleaved chains
        long long in0 = 0, in1 = 0, in2 = 0, in3 = 0;
        mbar_wait(&d_full[buf], (tl >> 1) & 1);
        tc_fence_after();
        const uint32_t dc = trow + (uint32_t)(buf * XTC_NT + ch * 128);
#pragma unroll 1
        for (int j0 = 0; j0 < 128; j0 += XTC_WB) {
          uint32_t v[XTC_WB];
          tmem_ld16(dc + j0, v);
          // next batch's weights while the TMEM load is in flight
          int i1n = i1 + XTC_WB;
          if (i1n >= I1) i1n -= I1;
          if (j0 + XTC_WB < 128) load_w1(j0 + XTC_WB, i1n, wn);
          tmem_wait_ld();
          if (plain(j0, i1)) {
#pragma unroll
            for (int j = 0; j < XTC_WB; j += 4) {
              in0 += (long long)wc[j] * (int)v[j];
              in1 += (long long)wc[j + 1] * (int)v[j + 1];
              in2 += (long long)wc[j + 2] * (int)v[j + 2];
              in3 += (long long)wc[j + 3] * (int)v[j + 3];
            }
            i1 += XTC_WB;
            if (i1 == I1) {
              acc = fma((double)w2, (double)((in0 + in1) + (in2 + in3)), acc);
              in0 = in1 = in2 = in3 = 0;
              i1 = 0;
              ++i2;
              w2 = j0 + XTC_WB < nrow ? wm * __ldg(w2p + (long long)i2 * RP) : 0.0f;
            }
          } else {
            // the batch crosses into the next i2 or past the block's rows
#pragma unroll
            for (int j = 0; j < XTC_WB; ++j) {
              in0 += (long long)wc[j] * (int)v[j];
              if (++i1 == I1) {
                acc = fma((double)w2, (double)((in0 + in1) + (in2 + in3)), acc);
                in0 = in1 = in2 = in3 = 0;
                i1 = 0;
                ++i2;
                w2 = j0 + j + 1 < nrow ? wm * __ldg(w2p + (long long)i2 * RP) : 0.0f;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < XTC_WB; ++j) wc[j] = wn[j];
        }
        acc = fma((double)w2, (double)((in0 + in1) + (in2 + in3)), acc);
        tc_fence_before();
        mbar_arrive(&d_empty[buf]);
        if (t == un.t1 - 1) {
          // unit done: levels and column halves combined in fixed order
          red[ch * 128 + L] = acc;
          acc = 0.0;
          named_bar(1, NE);
          if (et < b.R) {
            const double s0 = red[et] + red[128 + et];
            const double s1 = red[RP + et] + red[128 + RP + et];
            const double s2 = red[2 * RP + et] + red[128 + 2 * RP + et];
            a.part[(long long)un.u * 64 + et] = fma(s0, 65536.0, fma(s1, 256.0, s2)) * b.aux[set][et];
            __threadfence();
          }
          named_bar(1, NE);
          if (et == 0) {
            const int prev = atomicAdd(&a.cnt[un.s], 1);
            const int last = prev == b.nunits - 1;
            if (last) a.cnt[un.s] = 0;
            *shflag = last;
          }
          named_bar(1, NE);
          if (*shflag) {
            __threadfence();
            if (et < b.R) {
              double s = 0.0;
              for (int k = 0; k < b.nunits; ++k)
                s += __ldcg(&a.part[(long long)(b.ufirst + k) * 64 + et]);
              a.bsum[(long long)un.s * RSTRIDE + et] = s;
            }
          }
          // red / shflag are reused only after the next unit's barriers
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  tl_end(a.tl, TL_TRACE);
}

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
bool xtc_supported(int S, const void* const* X, const long long* dims, const int* R) {
  for (int s = 0; s < S; ++s) {
    const long long I0 = dims[3 * s], I1 = dims[3 * s + 1], I2 = dims[3 * s + 2];
    if (I0 < 1 || I1 < 1 || I2 < 1) return false;
    if (I0 > XTC_MAX_I0) return false;
    if (I1 * I2 >= (1LL << 31)) return false;
    if (R[s] < 1 || R[s] > XTC_MAX_R) return false;   // three levels of Rp lanes in M = 128
    if (I1 < XTC_WB) return false;        // a weight batch wraps i1 at most once
    if ((reinterpret_cast<uintptr_t>(X[s]) & 3) != 0) return false;
  }
  return true;
}

static size_t xtc_smem_for(int nst, int bimg_max) {
  return 1024 + (size_t)nst * XTC_STAGE + bimg_max + 8 * (2 * nst + 6) + 256 * 8 + 16;
}

int xtc_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                    cudaStream_t st, XtcPlan** out) {
  *out = nullptr;
  // this plan's buffers are zeroed on the stream that then fills and uses them
  set_alloc_stream(st);
  XtcPlan* p = new XtcPlan();
  p->S = S;
  int rmax = 1;
  for (int s = 0; s < S; ++s) rmax = std::max(rmax, R[s]);
  p->Rp = (rmax + 7) / 8 * 8;
  const int Rp = p->Rp;
  const int SR = 2 * Rp + 128;
  std::vector<XtcBlock> hb(S);
  std::vector<XtcUnit> hu;
  long long w_elems = 0;
  long long bimg_total = 0;
  size_t plane_bytes = 0;
  int ntmax = 1;
  for (int s = 0; s < S; ++s) {
    XtcBlock& b = hb[s];
    b.I0 = dims[3 * s]; b.I1 = dims[3 * s + 1]; b.I2 = dims[3 * s + 2];
    b.J = b.I1 * b.I2;
    b.R = R[s];
    b.ntiles = (int)((b.J + XTC_NT - 1) / XTC_NT);
    b.nk = (int)((b.I0 + 31) / 32);
    b.ex = 0;
    b.bimg_bytes = b.nk * SR * 32;
    p->bimg_max = std::max(p->bimg_max, b.bimg_bytes);
    b.ufirst = (int)hu.size();
    p->ntiles += b.ntiles;
    ntmax = std::max(ntmax, b.ntiles);
    for (int t = 0; t < b.ntiles; t += XTC_TPU)
      hu.push_back({s, t, std::min(b.ntiles, t + XTC_TPU), (int)hu.size()});
    b.nunits = (int)hu.size() - b.ufirst;
    w_elems += (long long)Rp * (b.I1 + b.I2);
    bimg_total += b.bimg_bytes;
    plane_bytes += (size_t)b.ntiles * b.nk * XTC_STAGE;
    p->bytes += (double)b.I0 * (double)b.J * 4.0;
  }
  p->stream_bytes = (double)plane_bytes;
  p->nunits = (int)hu.size();
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  p->grid = std::max(1, std::min(nsm, p->nunits));
  // shared memory: the factor image, then as many ring stages (<= 6) as fit
  const long long room = (long long)XTC_SMEM_MAX - (long long)xtc_smem_for(0, p->bimg_max);
  const int nst = (int)std::min<long long>(6, room / (XTC_STAGE + 16));
  if (nst < 2) {
    const int bm = p->bimg_max;
    delete p;
    set_error("xtc: operand image too large (%d bytes)", bm);
    return CB_ERR_UNSUPPORTED;
  }
  p->nst = nst;
  p->smem = xtc_smem_for(nst, p->bimg_max);
  // device buffers
  std::vector<void*>& A = p->allocs;
  int rc = CB_OK;
#define XTRY(x) do { rc = (x); if (rc) { xtc_plan_destroy(p); return rc; } } while (0)
#define XCUDA(x)                                                       \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      xtc_plan_destroy(p);                                             \
      return cuda_fail(e_, #x, __FILE__, __LINE__);                    \
    }                                                                  \
  } while (0)
  double* aux = nullptr;
  float* wts = nullptr;
  unsigned char* bimg = nullptr;
  unsigned char* planes = nullptr;
  // every plane byte is written by the pack kernel: no memset
  XCUDA(cudaMalloc((void**)&planes, plane_bytes));
  A.push_back(planes);
  XTRY(dalloc((void**)&p->blk, sizeof(XtcBlock) * S, A));
  XTRY(dalloc((void**)&p->units, sizeof(XtcUnit) * hu.size(), A));
  XTRY(dalloc((void**)&p->part, sizeof(double) * 64 * hu.size(), A));
  XTRY(dalloc((void**)&p->cnt, sizeof(int) * S, A));
  XTRY(dalloc((void**)&p->maxbits, sizeof(unsigned int) * S, A));
  XTRY(dalloc((void**)&p->par, sizeof(int), A));
  XTRY(dalloc((void**)&aux, sizeof(double) * 2 * 64 * S, A));
  XTRY(dalloc((void**)&wts, sizeof(float) * 2 * w_elems, A));
  XTRY(dalloc((void**)&bimg, (size_t)2 * bimg_total, A));   // zeroed: the image's zero rows
  long long wo = 0, bo = 0;
  size_t po = 0;
  for (int s = 0; s < S; ++s) {
    XtcBlock& b = hb[s];
    for (int k = 0; k < 2; ++k) {
      b.aux[k] = aux + 64LL * (2 * s + k);
      b.w1[k] = reinterpret_cast<int*>(wts + k * w_elems + wo);
      b.w2[k] = wts + k * w_elems + wo + (long long)Rp * b.I1;
      b.bimg[k] = bimg + (size_t)k * bimg_total + bo;
    }
    wo += (long long)Rp * (b.I1 + b.I2);
    b.X = reinterpret_cast<const float*>(X[s]);
    b.planes = planes + po;
    po += (size_t)b.ntiles * b.nk * XTC_STAGE;
    bo += b.bimg_bytes;
  }
  XCUDA(cudaMemcpyAsync(p->blk, hb.data(), sizeof(XtcBlock) * S, cudaMemcpyHostToDevice, st));
  XCUDA(cudaMemcpyAsync(p->units, hu.data(), sizeof(XtcUnit) * hu.size(), cudaMemcpyHostToDevice, st));
  for (int s = 0; s < S; ++s) {
    const long long n = hb[s].I0 * hb[s].J;
    const int grid = (int)std::max(1LL, std::min((n + 255) / 256, (long long)nsm * 8));
    k_xtc_maxabs<<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(X[s]), n, p->maxbits + s);
  }
  k_xtc_set_ex<<<(S + 127) / 128, 128, 0, st>>>(p->blk, p->maxbits, S);
  k_xtc_pack<<<dim3((unsigned)ntmax, 1, S), XTC_NT, 0, st>>>(p->blk);
  XCUDA(cudaGetLastError());
  count_launch(S + 2);
#define XTC_ATTR(RPV)                                                                       \
  XCUDA(cudaFuncSetAttribute(k_xtc_trace<RPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)p->smem))
  switch (Rp) {
    case 8: XTC_ATTR(8); break;
    case 16: XTC_ATTR(16); break;
    case 24: XTC_ATTR(24); break;
    case 32: XTC_ATTR(32); break;
    default: XTC_ATTR(40); break;
  }
#undef XTC_ATTR
#undef XTRY
#undef XCUDA
  *out = p;
  return CB_OK;
}

void xtc_plan_destroy(XtcPlan* p) {
  if (!p) return;
  dfree_all(p->allocs);
  delete p;
}

double xtc_bytes(const XtcPlan* p) { return p ? p->bytes : 0.0; }

double xtc_stream_bytes(const XtcPlan* p) { return p ? p->stream_bytes : 0.0; }

void xtc_set_grid_cap(XtcPlan* p, int cap) {
  if (p) p->grid_cap = cap;
}

void xtc_set_timeline(XtcPlan* p, unsigned long long* tl) {
  if (p) p->tl = tl;
}

// parts: 1 = operand prep only (snapshots the factors), 2 = the streaming
// pass only (reads only the prepared operands), 3 = both
int xtc_flip(XtcPlan* p, const int* gate, cudaStream_t st) {
  CB_CUDA(launch_k(k_xtc_flip, dim3(1), dim3(32), 0, st, p->par, gate));
  count_launch(1);
  return CB_OK;
}

int xtc_trace(XtcPlan* p, const double* const* U_dev, const int* gate, double* bsum,
              cudaStream_t st, int parts, int other) {
  XtcArgs a{};
  a.par = p->par;
  a.wr_other = other ? 1 : 0;
  a.blk = p->blk;
  a.units = p->units;
  a.nunits = p->nunits;
  a.nst = p->nst;
  a.bimg_max = p->bimg_max;
  a.Rp = p->Rp;
  a.part = p->part;
  a.cnt = p->cnt;
  a.bsum = bsum;
  a.gate = gate;
  a.tl = p->tl;
  if (parts & 1) {
    CB_CUDA(launch_k(k_xtc_prep, dim3(p->S, 4), dim3(256), 0, st, a, U_dev));
    count_launch(1);
  }
  if (parts & 2) {
    const int grid = p->grid_cap > 0 ? std::min(p->grid, p->grid_cap) : p->grid;
    // (launching it at the highest scheduling priority, so that its static
    // partition is placed before the sweep's CTAs, measured slower on c5)
    switch (p->Rp) {
      case 8: CB_CUDA(launch_k(k_xtc_trace<8>, dim3(grid), dim3(XTC_THREADS), p->smem, st, a)); break;
      case 16: CB_CUDA(launch_k(k_xtc_trace<16>, dim3(grid), dim3(XTC_THREADS), p->smem, st, a)); break;
      case 24: CB_CUDA(launch_k(k_xtc_trace<24>, dim3(grid), dim3(XTC_THREADS), p->smem, st, a)); break;
      case 32: CB_CUDA(launch_k(k_xtc_trace<32>, dim3(grid), dim3(XTC_THREADS), p->smem, st, a)); break;
      default: CB_CUDA(launch_k(k_xtc_trace<40>, dim3(grid), dim3(XTC_THREADS), p->smem, st, a)); break;
    }
    count_launch(1);
  }
  return CB_OK;
}

}  // namespace cb

// ---------------------------------------------------------------------------
// C ABI: batched core linear term on the tensor cores (operator-level entry,
// reference core_linear_term, solver.py:215-218)
// ---------------------------------------------------------------------------
extern "C" int cb_core_linear_term_tc(int n_blocks, const void* const* tensors,
                                      const int64_t* dims, const double* const* factors,
                                      const int* ranks, double* out, void* stream) {
  using namespace cb;
  CB_ARG(n_blocks >= 1 && tensors && dims && factors && ranks && out, "null argument");
  std::vector<long long> d(dims, dims + 3 * n_blocks);
  if (!xtc_supported(n_blocks, tensors, d.data(), ranks)) {
    set_error("tensor-core trace pass does not support these blocks");
    return CB_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  XtcPlan* p = nullptr;
  int rc = xtc_plan_create(n_blocks, tensors, d.data(), ranks, st, &p);
  if (rc) return rc;
  const double** dU = nullptr;
  cudaError_t e = cudaMalloc((void**)&dU, sizeof(double*) * 3 * n_blocks);
  if (e != cudaSuccess) {
    xtc_plan_destroy(p);
    return cuda_fail(e, "cudaMalloc", __FILE__, __LINE__);
  }
  e = cudaMemcpyAsync(dU, factors, sizeof(double*) * 3 * n_blocks, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) rc = xtc_trace(p, dU, nullptr, out, st);
  if (e == cudaSuccess && !rc) e = cudaStreamSynchronize(st);
  cudaFree(dU);
  xtc_plan_destroy(p);
  if (e != cudaSuccess) return cuda_fail(e, "xtc trace", __FILE__, __LINE__);
  return rc;
}
