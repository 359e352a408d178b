// ALS compression passes on the tensor cores at fp64-grade accuracy
// (reference: cpd_als.py:90-104, the MTTKRP of each mode inside a sweep).
//
// A sweep streams each block twice (DESIGN 5.3): T = X x3 A2 (modes 0 and 1
// are contractions of T) and D = X_r A0 (mode 2 is a contraction of D).  Both
// are GEMMs with a long M (160000 rows at c5), a short K (400) and N = R
// (40); in fp64 FMAs they are compute bound (58% of the DFMA peak, 15 ms per
// pass of 64 c5 blocks).  Here they run as EXACT integer GEMMs on tcgen05
// kind::i8:
//
//   * X (fp32, one exponent per block: |x| < 2^ex) is fixed point q =
//     rint(x 2^(30-ex)) = a0 2^24 + a1 2^16 + a2 2^8 + a3 with balanced signed
//     bytes (a0 in [-64, 64]); q is EXACT for every fp32 value >= 2^(ex-7)
//     and within 2^(ex-31) otherwise.  The four byte planes are written once
//     per compression (k_oz_pack) in the MMA's shared-memory layout (K-major
//     rows of 32 bytes, 32-byte swizzle), tile by tile, for both forms (rows
//     (i0,i1) with K = i2, and rows (i1,i2) with K = i0): a pass is then
//     16 KB bulk copies -> MMAs -> epilogue, with no conversion work and no
//     strided access.  A sweep count of ~36 amortises the pack (two extra
//     streams of X) to ~3% of the compression.
//   * the factor (fp64, one exponent per column) is p = rint(u 2^(38-eu)) as
//     five balanced bytes b0..b4, rebuilt per pass (k_oz_prep).
//   * q p = sum_{i,j} a_i b_j 2^(8 (7-i-j)); the levels l = i + j <= 4 are
//     kept: four MMAs per K = 32 step, a_i x [b_0 | .. | b_{4-i}] into the
//     int32 accumulator columns of levels i..4 (exact: |L_l| < 2^31 for
//     K < 32768).  The dropped levels (>= 5) are products of balanced
//     zero-mean digits, ~2^-40 of a product.
//   * epilogue: the five levels through the fp64 adder (exact int -> fp64),
//     Horner in fp64, the column scale, one coalesced fp64 store per column.
// Error per output: ~1e-13 relative (factor rounding 2^-39 of the column
// maximum, shared by a column; dropped levels), against ~1e-15 of the fp64
// FMA GEMM; tests/test_gpu_xtc.py holds the ALS histories to 1e-10 and the
// factors to 1e-8 against the fp64-storage explicit-residual ALS.
//
// Kernel (persistent, one CTA per SM, 320 threads): warp 9 streams the plane
// stages and the block's factor image (1-D bulk copies on mbarriers), warp 8
// issues the MMAs (A and B from shared memory, D double-buffered in TMEM),
// warps 0-7 are the epilogue (one TMEM lane quarter each, half the columns).
#include <cuda.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "act_tiles.cuh"
#include "engine_host.h"
#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"
#include "tc.cuh"
#include "xoz.h"

namespace cb {

constexpr int OZ_M = 128;                       // rows per tile (MMA M)
constexpr int OZ_SX = 4;                        // byte planes of X
constexpr int OZ_SB = 5;                        // byte slices of the factor = levels kept
constexpr int OZ_PIECE = OZ_M * 32;             // 4 KB: one plane of one K = 32 step
constexpr int OZ_STAGE = OZ_SX * OZ_PIECE;      // 16 KB per ring stage
constexpr int OZ_THREADS = 320;
constexpr int OZ_SMEM_MAX = 227 * 1024;
constexpr int OZ_XBITS = 30;
constexpr int OZ_UBITS = 38;

struct OzForm {
  long long J;             // rows
  long long rs, ks;        // element strides of (row, k) in X
  int K, nt, nk;           // contraction length, tiles, K = 32 steps
  unsigned char* planes;   // [nt][nk][4 planes][128 rows x 32 B]
  unsigned char* bimg;     // [nk][5 N rows][32 B]
  double* scale;           // [64]
};

struct OzBlock {
  const float* X;
  int R, ex;
  int fac[2];              // factor each form contracts with (2, 0)
  long long I1, I2;
  double* D;               // [R][J] of form 1
  OzForm f[2];             // 0: T pass (rows i0 + I0 i1, K = i2); 1: D pass (rows i1 + I1 i2, K = i0)
};

struct OzArgs {
  const OzBlock* blk;
  int S, form, nst, bimg_max;
  const int* active;
  void* const* T0;
  void* const* T1;
  const int* tsel;
  int t_other;
  const double* const* U;
  const double* const* UT;   // transposed factors [r][I_n] (written by the ALS solve) or null
  double* const* mtt;
  long long i2max;
};

struct OzPlan {
  int S = 0, N = 0, grid = 1;
  int nst[2] = {0, 0}, bimg_max[2] = {0, 0};
  size_t smem[2] = {0, 0};
  long long i2max = 1;
  double bytes[2] = {0.0, 0.0};
  std::vector<void*> allocs;
  OzBlock* blk = nullptr;
  unsigned int* maxbits = nullptr;
  int nsm = 148, ntmax[2] = {1, 1};
  std::vector<const float*> X;       // host copies for the pack launches
  std::vector<long long> elems;
};

// --------------------------------------------------------------------------
// one-time: block exponents and the byte planes
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_oz_maxabs(const float* __restrict__ X, long long n,
                                                   unsigned int* out) {
  float m = 0.0f;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    m = fmaxf(m, fabsf(X[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__global__ void k_oz_set_ex(OzBlock* blk, const unsigned int* maxbits, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const float m = __uint_as_float(maxbits[s]);
  int e = 0;
  if (m > 0.0f && isfinite(m)) frexpf(m, &e);   // m = f 2^e, f in [0.5, 1)
  blk[s].ex = e;
}

// byte `byte` of four words as one word (k increasing with the address)
__device__ __forceinline__ uint32_t oz_pick(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                            int byte) {
  const uint32_t sel = (uint32_t)byte | ((uint32_t)(byte + 4) << 4);
  return __byte_perm(__byte_perm(t0, t1, sel), __byte_perm(t2, t3, sel), 0x5410);
}

// grid (max tiles, 1, S), 128 threads: thread m owns row m of the tile
template <int FORM>
__global__ void __launch_bounds__(OZ_M) k_oz_pack(const OzBlock* blk) {
  const OzBlock& b = blk[blockIdx.z];
  const OzForm& f = b.f[FORM];
  const int t = blockIdx.x;
  if (t >= f.nt) return;
  __shared__ float tile[FORM == 1 ? OZ_M : 1][33];
  const int m = threadIdx.x;
  const int warp = m >> 5, lane = m & 31;
  const long long row = (long long)t * OZ_M + m;
  const float sx = ldexpf(1.0f, OZ_XBITS - b.ex);
  const float* __restrict__ X = b.X;
  const int sw = (m >> 2) & 1;
  for (int c = 0; c < f.nk; ++c) {
    float v[32];
    if (FORM == 0) {
      // rows are contiguous in memory: coalesced across the threads
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int kk = c * 32 + k;
        v[k] = (row < f.J && kk < f.K) ? __ldcs(X + row + (long long)kk * f.ks) : 0.0f;
      }
    } else {
      // k is contiguous: each warp transposes its 32 rows through shared memory
      const int kk = c * 32 + lane;
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        const long long rr = (long long)t * OZ_M + warp * 32 + r;
        tile[warp * 32 + r][lane] = (rr < f.J && kk < f.K) ? __ldcs(X + rr * f.rs + kk) : 0.0f;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = tile[m][k];
      __syncwarp();
    }
    uint32_t q[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) q[k] = (uint32_t)(__float2int_rn(v[k] * sx) + 0x808080);
    unsigned char* dst = f.planes + ((long long)t * f.nk + c) * OZ_STAGE + m * 32;
#pragma unroll
    for (int i = 0; i < OZ_SX; ++i) {
      uint32_t w[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        w[g] = oz_pick(q[4 * g], q[4 * g + 1], q[4 * g + 2], q[4 * g + 3], 3 - i);
        if (i > 0) w[g] ^= 0x80808080u;
      }
      uint4* d = reinterpret_cast<uint4*>(dst + i * OZ_PIECE);
      d[sw] = make_uint4(w[0], w[1], w[2], w[3]);
      d[sw ^ 1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
}

// --------------------------------------------------------------------------
// per pass: the factor as five balanced byte slices in the MMA B layout
// --------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(256) k_oz_prep(OzArgs a) {
  griddep_wait();
  const int s = blockIdx.x;
  if (a.active && !a.active[s]) return;
  const OzBlock& b = a.blk[s];
  const OzForm& f = b.f[a.form];
  const double* A = a.U[3 * s + b.fac[a.form]];
  const int R = b.R, K = f.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int eu[64];
  for (int r = warp; r < N; r += 8) {
    double m = 0.0;
    if (r < R)
      for (int i = lane; i < K; i += 32) m = fmax(m, fabs(A[(long long)i * R + r]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      int e = 0;
      if (m > 0.0 && isfinite(m)) frexp(m, &e);
      eu[r] = e;
    }
  }
  __syncthreads();
  const int kmax = f.nk * 32;
  for (int e = threadIdx.x; e < kmax * N; e += 256) {
    const int k = e / N, n = e - (e / N) * N;
    long long p = 0;
    if (k < K && n < R) p = llrint(ldexp(A[(long long)k * R + n], OZ_UBITS - eu[n]));
    signed char d[OZ_SB];
#pragma unroll
    for (int j = OZ_SB - 1; j > 0; --j) {
      const long long dj = ((p + 128) & 255) - 128;
      d[j] = (signed char)dj;
      p = (p - dj) >> 8;
    }
    d[0] = (signed char)p;
    // K step c: 5 N rows of 32 bytes ([b0 | .. | b4], slice j at rows j N + n),
    // 16-byte halves swapped on rows with bit 2 set (32-byte swizzle)
    const int c = k >> 5, kk = k & 31;
    const long long off =
        ((long long)c * OZ_SB * N + n) * 32 + (((kk >> 4) ^ ((n >> 2) & 1)) << 4) + (kk & 15);
#pragma unroll
    for (int j = 0; j < OZ_SB; ++j) f.bimg[off + (long long)j * N * 32] = (unsigned char)d[j];
  }
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    f.scale[r] = r < R ? ldexp(1.0, 24 + b.ex - OZ_XBITS + eu[r] - OZ_UBITS) : 0.0;
  }
}

// int32 -> double through the fp64 adder (exact): 2^52 + 2^31 + x
__device__ __forceinline__ double oz_i2d(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
}

// --------------------------------------------------------------------------
// the streaming GEMM: out[r][row] = scale_r sum_l L_l[row, r] 2^(8 (4 - l))
// --------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(OZ_THREADS, 1) k_oz_gemm(OzArgs a) {
  griddep_wait_no_trigger();
  constexpr int NH = N / 2;          // columns per epilogue group
  constexpr int WMMA = 8, WTMA = 9;
  constexpr int DW = OZ_SB * N;      // accumulator columns per buffer
  extern __shared__ unsigned char oz_raw[];
  const uint32_t raw_u32 = smem_u32(oz_raw);
  unsigned char* sm = oz_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int nst = a.nst;
  unsigned char* ring = sm;
  unsigned char* bimg = sm + (size_t)nst * OZ_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(bimg + a.bimg_max);
  uint64_t* empty = full + nst;
  uint64_t* d_full = empty + nst;
  uint64_t* d_empty = d_full + 2;
  uint64_t* b_full = d_empty + 2;
  uint64_t* b_empty = b_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int form = a.form;
  auto ntl = [&](int s) -> long long { return a.blk[s].f[form].nt; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], 256); }
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
      for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
           act_tiles_next(it, a.active, a.S, ntl)) {
        const OzForm& f = a.blk[it.s].f[form];
        if (it.s != cur) {
          mbar_wait(b_empty, (seg & 1) ^ 1);
          const int bytes = f.nk * OZ_SB * N * 32;
          mbar_arrive_expect_tx(b_full, (uint32_t)bytes);
          for (int off = 0; off < bytes; off += 32768)
            bulk_g2s(bimg + off, f.bimg + off, (uint32_t)min(32768, bytes - off), b_full);
          cur = it.s;
          ++seg;
        }
        const unsigned char* src = f.planes + it.t * f.nk * (long long)OZ_STAGE;
        for (int c = 0; c < f.nk; ++c) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], OZ_STAGE);
          bulk_g2s(ring + (size_t)st * OZ_STAGE, src + (size_t)c * OZ_STAGE, OZ_STAGE, &full[st]);
          if (++st == nst) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == WMMA) {
    // --------------------------------------------------------- MMA issuer
    int st = 0, ph = 0, seg = 0, cur = -1, tl = 0;
    const uint32_t bbase = smem_u32(bimg);
    const uint32_t rbase = smem_u32(ring);
    for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
         act_tiles_next(it, a.active, a.S, ntl), ++tl) {
      const OzForm& f = a.blk[it.s].f[form];
      const int nk = f.nk;
      if (it.s != cur) {
        mbar_wait(b_full, seg & 1);
        tc_fence_after();
        cur = it.s;
        ++seg;
      }
      // the CTA's next tile (if any) belongs to another block: release B
      const bool last_of_seg = it.left == 1 || it.t + 1 >= f.nt;
      const int buf = tl & 1;
      mbar_wait(&d_empty[buf], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dc = tmem + (uint32_t)(buf * DW);
      for (int c = 0; c < nk; ++c) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ab = rbase + (uint32_t)st * OZ_STAGE;
          const uint64_t B = sdesc_k_sw32(bbase + (uint32_t)c * OZ_SB * N * 32);
          // D[levels i..4] += a_i [b_0 | .. | b_{4-i}]
          mma_i8_ss(dc, sdesc_k_sw32(ab), B, idesc_i8(5 * N, 1, 1), c > 0 ? 1u : 0u);
          mma_i8_ss(dc + N, sdesc_k_sw32(ab + OZ_PIECE), B, idesc_i8(4 * N, 1, 1), 1u);
          mma_i8_ss(dc + 2 * N, sdesc_k_sw32(ab + 2 * OZ_PIECE), B, idesc_i8(3 * N, 1, 1), 1u);
          mma_i8_ss(dc + 3 * N, sdesc_k_sw32(ab + 3 * OZ_PIECE), B, idesc_i8(2 * N, 1, 1), 1u);
          tc_commit(&empty[st]);
          if (c == nk - 1) {
            tc_commit(&d_full[buf]);
            if (last_of_seg) tc_commit(b_empty);
          }
        }
        __syncwarp();
        if (++st == nst) { st = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------- epilogue (warps 0-7)
    const int eg = warp >> 2;
    const int wq = warp & 3;
    const int m = wq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    const int sel = (a.tsel ? *a.tsel : 0) ^ a.t_other;
    int tl = 0;
    for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
         act_tiles_next(it, a.active, a.S, ntl), ++tl) {
      const OzBlock& b = a.blk[it.s];
      const OzForm& f = b.f[form];
      const int R = b.R;
      const long long J = f.J;
      double* out = form == 0 ? reinterpret_cast<double*>(sel ? a.T1[it.s] : a.T0[it.s]) : b.D;
      const double* __restrict__ scale = f.scale;
      const int buf = tl & 1;
      const long long row = it.t * OZ_M + m;
      const bool valid = row < J;
      mbar_wait(&d_full[buf], (tl >> 1) & 1);
      tc_fence_after();
      const uint32_t dc = trow + (uint32_t)(buf * DW);
#pragma unroll
      for (int cg = 0; cg < NH / 8; ++cg) {
        const int col0 = eg * NH + cg * 8;
        uint32_t l0[8], l1[8], l2[8], l3[8], l4[8];
        tmem_ld8(dc + col0, l0);
        tmem_ld8(dc + N + col0, l1);
        tmem_ld8(dc + 2 * N + col0, l2);
        tmem_ld8(dc + 3 * N + col0, l3);
        tmem_ld8(dc + 4 * N + col0, l4);
        double sc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) sc[j] = __ldg(scale + col0 + j);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          double v = fma(oz_i2d(l0[j]), 256.0, oz_i2d(l1[j]));
          v = fma(v, 256.0, oz_i2d(l2[j]));
          v = fma(v, 256.0, oz_i2d(l3[j]));
          v = fma(v, 256.0, oz_i2d(l4[j]));
          const int r = col0 + j;
          if (valid && r < R) out[(long long)r * J + row] = v * sc[j];
        }
      }
      tc_fence_before();
      mbar_arrive(&d_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// M2[i2, r] = sum_{i1} A1[i1, r] D[r][i1 + I1 i2]: one warp per (s, i2, r),
// fixed-order lane sums and butterfly (deterministic)
__global__ void __launch_bounds__(256) k_oz_contract(OzArgs a) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)a.S * a.i2max * 64;
  for (long long w = (blockIdx.x * 256LL + threadIdx.x) >> 5; w < nw;
       w += ((long long)gridDim.x * 256) >> 5) {
    const int s = (int)(w / (a.i2max * 64));
    const long long rem = w - (long long)s * a.i2max * 64;
    const long long i2 = rem >> 6;
    const int r = (int)(rem & 63);
    if (a.active && !a.active[s]) continue;
    const OzBlock& b = a.blk[s];
    if (i2 >= b.I2 || r >= b.R) continue;
    const double* d = b.D + (long long)r * b.f[1].J + i2 * b.I1;
    double v = 0.0;
    if (a.UT) {
      // column r of A1 from the transposed copy: both operands contiguous
      const double* A1t = a.UT[3 * s + 1] + (long long)r * b.I1;
      for (long long i1 = lane; i1 < b.I1; i1 += 32) v = fma(A1t[i1], d[i1], v);
    } else {
      const double* A1 = a.U[3 * s + 1];
      for (long long i1 = lane; i1 < b.I1; i1 += 32) v = fma(A1[i1 * b.R + r], d[i1], v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) a.mtt[s][i2 * b.R + r] = v;
  }
}

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
static int oz_bucket(int rmax) { return rmax <= 16 ? 16 : (rmax <= 32 ? 32 : 48); }

static size_t oz_smem_for(int nst, int bimg_bytes) {
  return 1024 + (size_t)nst * OZ_STAGE + bimg_bytes + 8 * (2 * nst + 6) + 16;
}

static int oz_stages(int bimg_bytes) {
  const long long room = (long long)OZ_SMEM_MAX - (long long)oz_smem_for(0, bimg_bytes);
  return (int)std::min<long long>(8, room / (OZ_STAGE + 16));
}

bool oz_supported(int S, const void* const* X, const long long* dims, const int* R) {
  int rmax = 1;
  for (int s = 0; s < S; ++s) rmax = std::max(rmax, R[s]);
  if (rmax <= 16 || rmax > 48) return false;
  const int N = oz_bucket(rmax);
  for (int s = 0; s < S; ++s) {
    const long long I0 = dims[3 * s], I1 = dims[3 * s + 1], I2 = dims[3 * s + 2];
    if (I0 < 1 || I1 < 1 || I2 < 1 || R[s] < 1) return false;
    if (I0 * I1 >= (1LL << 31) || I1 * I2 >= (1LL << 31)) return false;
    if (I0 >= 32768 || I2 >= 32768) return false;   // int32 level sums
    for (long long K : {I0, I2}) {
      const int nk = (int)((K + 31) / 32);
      if (oz_stages(nk * OZ_SB * N * 32) < 3) return false;
    }
    if ((reinterpret_cast<uintptr_t>(X[s]) & 3) != 0) return false;
  }
  return true;
}

int oz_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                   cudaStream_t st, OzPlan** out, bool defer_pack) {
  *out = nullptr;
  // this plan's buffers are zeroed on the stream that then fills and uses them
  set_alloc_stream(st);
  OzPlan* p = new OzPlan();
  p->S = S;
  int rmax = 1;
  for (int s = 0; s < S; ++s) rmax = std::max(rmax, R[s]);
  p->N = oz_bucket(rmax);
  const int N = p->N;
  std::vector<OzBlock> hb(S);
  std::vector<void*>& A = p->allocs;
  int rc = CB_OK;
#define OTRY(x) do { rc = (x); if (rc) { oz_plan_destroy(p); return rc; } } while (0)
#define OCUDA(x)                                                        \
  do {                                                                  \
    cudaError_t e_ = (x);                                               \
    if (e_ != cudaSuccess) {                                            \
      oz_plan_destroy(p);                                               \
      return cuda_fail(e_, #x, __FILE__, __LINE__);                     \
    }                                                                   \
  } while (0)
  long long ntmax[2] = {1, 1};
  size_t plane_bytes = 0, bimg_bytes = 0;
  for (int s = 0; s < S; ++s) {
    OzBlock& b = hb[s];
    const long long I0 = dims[3 * s], I1 = dims[3 * s + 1], I2 = dims[3 * s + 2];
    b.X = reinterpret_cast<const float*>(X[s]);
    b.R = R[s];
    b.ex = 0;
    b.fac[0] = 2;
    b.fac[1] = 0;
    b.I1 = I1;
    b.I2 = I2;
    b.f[0].J = I0 * I1; b.f[0].rs = 1;  b.f[0].ks = I0 * I1; b.f[0].K = (int)I2;
    b.f[1].J = I1 * I2; b.f[1].rs = I0; b.f[1].ks = 1;       b.f[1].K = (int)I0;
    for (int f = 0; f < 2; ++f) {
      OzForm& F = b.f[f];
      F.nt = (int)((F.J + OZ_M - 1) / OZ_M);
      F.nk = (F.K + 31) / 32;
      ntmax[f] = std::max<long long>(ntmax[f], F.nt);
      p->bimg_max[f] = std::max(p->bimg_max[f], F.nk * OZ_SB * N * 32);
      p->bytes[f] += (double)F.nt * F.nk * OZ_STAGE;
      plane_bytes += (size_t)F.nt * F.nk * OZ_STAGE;
      bimg_bytes += (size_t)F.nk * OZ_SB * N * 32;
    }
    p->i2max = std::max(p->i2max, I2);
  }
  // planes (every byte is written by the pack kernels: no memset), factor
  // images, column scales, D
  unsigned char* planes = nullptr;
  OCUDA(cudaMalloc((void**)&planes, plane_bytes));
  A.push_back(planes);
  unsigned char* bimg = nullptr;
  double* scale = nullptr;
  OTRY(dalloc((void**)&bimg, bimg_bytes, A));
  OTRY(dalloc((void**)&scale, sizeof(double) * 128 * S, A));
  size_t po = 0, bo = 0;
  size_t d_elems = 0;
  for (int s = 0; s < S; ++s) d_elems += (size_t)hb[s].R * hb[s].f[1].J;
  double* dbuf = nullptr;
  OCUDA(cudaMalloc((void**)&dbuf, sizeof(double) * d_elems));
  A.push_back(dbuf);
  size_t dofs = 0;
  for (int s = 0; s < S; ++s) {
    OzBlock& b = hb[s];
    for (int f = 0; f < 2; ++f) {
      OzForm& F = b.f[f];
      F.planes = planes + po;
      po += (size_t)F.nt * F.nk * OZ_STAGE;
      F.bimg = bimg + bo;
      bo += (size_t)F.nk * OZ_SB * N * 32;
      F.scale = scale + 128 * s + 64 * f;
    }
    b.D = dbuf + dofs;
    dofs += (size_t)b.R * b.f[1].J;
  }
  OTRY(dalloc((void**)&p->blk, sizeof(OzBlock) * S, A));
  OTRY(dalloc((void**)&p->maxbits, sizeof(unsigned int) * S, A));
  OCUDA(cudaMemcpyAsync(p->blk, hb.data(), sizeof(OzBlock) * S, cudaMemcpyHostToDevice, st));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  p->grid = nsm;
  p->nsm = nsm;
  p->ntmax[0] = (int)ntmax[0];
  p->ntmax[1] = (int)ntmax[1];
  p->X.assign(S, nullptr);
  p->elems.assign(S, 0);
  for (int s = 0; s < S; ++s) {
    p->X[s] = hb[s].X;
    p->elems[s] = hb[s].f[0].J * hb[s].f[0].K;
  }
  if (!defer_pack) {
    rc = oz_pack_range(p, 0, S, st);
    if (rc) { oz_plan_destroy(p); return rc; }
  }
  for (int f = 0; f < 2; ++f) {
    p->nst[f] = oz_stages(p->bimg_max[f]);
    if (p->nst[f] < 3) {
      oz_plan_destroy(p);
      set_error("oz: factor image too large (%d bytes)", p->bimg_max[f]);
      return CB_ERR_UNSUPPORTED;
    }
    p->smem[f] = oz_smem_for(p->nst[f], p->bimg_max[f]);
  }
  const int smem_max = (int)std::max(p->smem[0], p->smem[1]);
  switch (N) {
    case 16: OCUDA(cudaFuncSetAttribute(k_oz_gemm<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max)); break;
    case 32: OCUDA(cudaFuncSetAttribute(k_oz_gemm<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max)); break;
    default: OCUDA(cudaFuncSetAttribute(k_oz_gemm<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max)); break;
  }
#undef OTRY
#undef OCUDA
  *out = p;
  return CB_OK;
}

// block exponents and byte planes of blocks [lo, hi) (their tensors must be
// readable in stream order on `st`)
int oz_pack_range(OzPlan* p, int lo, int hi, cudaStream_t st) {
  if (hi <= lo) return CB_OK;
  for (int s = lo; s < hi; ++s) {
    const long long n = p->elems[s];
    const int grid = (int)std::max(1LL, std::min((n + 255) / 256, (long long)p->nsm * 8));
    k_oz_maxabs<<<grid, 256, 0, st>>>(p->X[s], n, p->maxbits + s);
  }
  const int nb = hi - lo;
  k_oz_set_ex<<<(nb + 127) / 128, 128, 0, st>>>(p->blk + lo, p->maxbits + lo, nb);
  k_oz_pack<0><<<dim3((unsigned)p->ntmax[0], 1, nb), OZ_M, 0, st>>>(p->blk + lo);
  k_oz_pack<1><<<dim3((unsigned)p->ntmax[1], 1, nb), OZ_M, 0, st>>>(p->blk + lo);
  CB_CHECK_LAUNCH();
  count_launch(nb + 3);
  return CB_OK;
}

// loads every kernel of the passes now (see tensor_stats_preload)
void oz_preload(const OzPlan* p) {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_oz_maxabs);
  cudaFuncGetAttributes(&fa, k_oz_set_ex);
  cudaFuncGetAttributes(&fa, k_oz_pack<0>);
  cudaFuncGetAttributes(&fa, k_oz_pack<1>);
  cudaFuncGetAttributes(&fa, k_oz_contract);
  switch (p->N) {
    case 16: cudaFuncGetAttributes(&fa, k_oz_prep<16>); cudaFuncGetAttributes(&fa, k_oz_gemm<16>); break;
    case 32: cudaFuncGetAttributes(&fa, k_oz_prep<32>); cudaFuncGetAttributes(&fa, k_oz_gemm<32>); break;
    default: cudaFuncGetAttributes(&fa, k_oz_prep<48>); cudaFuncGetAttributes(&fa, k_oz_gemm<48>); break;
  }
}

void oz_plan_destroy(OzPlan* p) {
  if (!p) return;
  dfree_all(p->allocs);
  delete p;
}

double oz_pass_bytes(const OzPlan* p, int form) { return p ? p->bytes[form & 1] : 0.0; }

static int oz_go(OzPlan* p, OzArgs& a, cudaStream_t st) {
  const int f = a.form;
  a.blk = p->blk;
  a.S = p->S;
  a.nst = p->nst[f];
  a.bimg_max = p->bimg_max[f];
  a.i2max = p->i2max;
  switch (p->N) {
    case 16:
      CB_CUDA(launch_k(k_oz_prep<16>, dim3(p->S), dim3(256), 0, st, a));
      CB_CUDA(launch_k(k_oz_gemm<16>, dim3(p->grid), dim3(OZ_THREADS), p->smem[f], st, a));
      break;
    case 32:
      CB_CUDA(launch_k(k_oz_prep<32>, dim3(p->S), dim3(256), 0, st, a));
      CB_CUDA(launch_k(k_oz_gemm<32>, dim3(p->grid), dim3(OZ_THREADS), p->smem[f], st, a));
      break;
    default:
      CB_CUDA(launch_k(k_oz_prep<48>, dim3(p->S), dim3(256), 0, st, a));
      CB_CUDA(launch_k(k_oz_gemm<48>, dim3(p->grid), dim3(OZ_THREADS), p->smem[f], st, a));
      break;
  }
  count_launch(2);
  return CB_OK;
}

int oz_tpass(OzPlan* p, const double* const* U_dev, const int* active, void* const* T0,
             void* const* T1, const int* tsel, int t_other, cudaStream_t st) {
  OzArgs a;
  memset(&a, 0, sizeof(a));
  a.form = 0;
  a.U = U_dev;
  a.active = active;
  a.T0 = T0;
  a.T1 = T1;
  a.tsel = tsel;
  a.t_other = t_other;
  return oz_go(p, a, st);
}

int oz_mode2(OzPlan* p, const double* const* U_dev, const int* active, double* const* mtt,
             cudaStream_t st, const double* const* UT_dev) {
  OzArgs a;
  memset(&a, 0, sizeof(a));
  a.form = 1;
  a.U = U_dev;
  a.UT = UT_dev;
  a.active = active;
  a.mtt = mtt;
  int rc = oz_go(p, a, st);
  if (rc) return rc;
  const long long warps = (long long)p->S * p->i2max * 64;
  const int grid = (int)std::max(1LL, std::min((warps * 32 + 255) / 256, 148LL * 16));
  CB_CUDA(launch_k(k_oz_contract, dim3(grid), dim3(256), 0, st, a));
  count_launch(1);
  return CB_OK;
}

}  // namespace cb
