// Mode-2 MTTKRP for ranks > 16 in fp64 arithmetic (the ALS compression's
// default path; cpd_als.py:92-94 with n = 2):
//
//   M2[i2, r] = sum_{i1} A1[i1, r] D[(i1, i2), r],   D = X_r . A0
//
// with X_r the block viewed as rows (i1, i2) of I0 contiguous elements.  The
// row-dot mode-2 kernel (xpass3.cuh) keeps NSLOT x RB accumulators per lane
// and stops at RB = 16; the KR-row kernel (xpass2.cuh slab2) re-forms an R-wide
// KR row per element and runs at a few % of the fp64 peak for R = 40.  Here the
// dominant contraction is a plain register-tiled fp64 GEMM:
//
//   k_sl5_dpass: one CTA per 128-row tile (persistent over tiles), a producer
//     lane streams 128 x 32 fp32 boxes (2-D tensor map, 128-byte swizzle)
//     through a 4-stage full/empty mbarrier ring; 256 consumer threads own 2
//     rows x RB/4 columns each, read their rows as swizzle-aware float4 and
//     the A0 rows (staged once per block segment, fp64) as broadcast vectors;
//     D is written once (fp64, [r][row]), coalesced.
//   k_sl5_contract: one warp per (block, i2, r): the I1-long contiguous dot of
//     D with A1[:, r], fixed-order warp sum.  Deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "engine_host.h"
#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"
#include "tma.cuh"
#include "xslab5.h"
#include "act_tiles.cuh"

namespace cb {

constexpr int SL5_M = 128;                     // rows per tile
constexpr int SL5_KC = 32;                     // fp32 K per box
constexpr int SL5_BOX = SL5_M * SL5_KC * 4;    // 16 KB
constexpr int SL5_NST = 4;
constexpr int SL5_CONS = 256;
constexpr int SL5_THREADS = SL5_CONS + 32;
constexpr int SL5_SMEM_MAX = 227 * 1024;

struct Sl5Block {
  long long I0, I1, I2, J;   // J = I1 * I2 rows
  int R, ntiles, nch;
  double* D;                 // [R][J]
};

struct Sl5Tile { int s, t; };

struct Sl5Args {
  const CUtensorMap* tmaps;
  const Sl5Block* blk;
  const Sl5Tile* tiles;
  int ntiles;
  const double* const* U;    // S*3 factors
  const int* active;
  double* const* mtt;        // S outputs (I2 x R)
  int S;
  long long i2max;
  const int* gate;           // skip when *gate == 0 (the engine's gated restart copies)
};

struct Sl5Plan {
  int S = 0, rb = 0, grid = 0, ntiles = 0;
  long long i2max = 1;
  size_t smem = 0;
  std::vector<void*> allocs;
  CUtensorMap* tmaps = nullptr;
  Sl5Block* blk = nullptr;
  Sl5Tile* tiles = nullptr;
  // T pass (T = X x3 A2) as a GEMM over (J x I2) boxes; off when it does
  // not fit (tg_ok false)
  bool tg_ok = false;
  int tg_rb = 0, tg_grid = 0, tg_ntiles = 0;
  size_t tg_smem = 0;
  CUtensorMap* tg_maps = nullptr;
  Sl5Tile* tg_tiles = nullptr;
};

// ----------------------------------------------------------------------------
// T pass as a register-tiled fp64 GEMM (the ALS sweep's second X stream):
//   T[r][j] = sum_{i2} X[j + J i2] A2[i2, r],   j = i0 + I0 i1,  J = I0 I1
// X viewed as I2 rows of J contiguous fp32 values; a producer lane streams
// TG_M x TG_KC boxes (j fastest, no swizzle) through a 4-stage mbarrier
// ring; 256 consumers own 4 consecutive j (one float4 per i2 row) x RB/8
// columns; A2 (fp64, zero-padded) is staged per block; T is written once,
// fp64, into the buffer the contract kernels read ([R][J], unsplit).
// ----------------------------------------------------------------------------
__device__ __forceinline__ void sl5_tma(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

constexpr int TG_M = 128;                      // j per tile
constexpr int TG_KC = 32;                      // i2 rows per box
constexpr int TG_BOX = TG_M * TG_KC * 4;       // 16 KB
constexpr int TG_NST = 4;

struct TgArgs {
  const CUtensorMap* tmaps;
  const Sl5Block* blk;
  const Sl5Tile* tiles;
  int ntiles;
  const double* const* U;    // S*3 factors (A2 = U[3 s + 2])
  const int* active;
  void* const* T0;           // T buffers, index (*tsel) ^ t_other
  void* const* T1;
  const int* tsel;
  int t_other;
  int S;
};

template <int RB>
__global__ void __launch_bounds__(SL5_THREADS, 1) k_tg_pass(TgArgs a) {
  griddep_wait();
  constexpr int CG = RB / 8;                   // columns per thread
  extern __shared__ unsigned char tg_raw[];
  const uint32_t raw_u32 = smem_u32(tg_raw);
  unsigned char* sm = tg_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  unsigned char* ring = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + TG_NST * TG_BOX);
  uint64_t* empty = full + TG_NST;
  double* a2s = reinterpret_cast<double*>(empty + TG_NST + 2);   // [I2pad][RB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sel = (a.tsel ? *a.tsel : 0) ^ a.t_other;
  auto ntl = [&](int s) -> long long {
    return (a.blk[s].I0 * a.blk[s].I1 + TG_M - 1) / TG_M;
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < TG_NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], SL5_CONS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == SL5_CONS / 32) {
    if (lane == 0) {
      int st = 0, ph = 0;
      for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
           act_tiles_next(it, a.active, a.S, ntl)) {
        const Sl5Tile tt{it.s, (int)it.t};
        const int nch = (int)((a.blk[tt.s].I2 + TG_KC - 1) / TG_KC);
        const CUtensorMap* tm = a.tmaps + tt.s;
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], TG_BOX);
          sl5_tma(ring + (size_t)st * TG_BOX, tm, tt.t * TG_M, c * TG_KC, &full[st]);
          if (++st == TG_NST) { st = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  // 2 consecutive j (one float2 per i2 row) x RB/4 columns per thread: one
  // fp32 -> fp64 conversion feeds RB/4 FMAs (the conversions share the
  // fp64 pipe with the FMAs)
  constexpr int CG2 = RB / 4;
  const int jg = threadIdx.x & 63;             // j = 2 jg, 2 jg + 1 of the tile
  const int cg = threadIdx.x >> 6;             // columns [cg CG2, (cg + 1) CG2)
  int st = 0, ph = 0, cur = -1;
  for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
       act_tiles_next(it, a.active, a.S, ntl)) {
    const Sl5Tile tt{it.s, (int)it.t};
    const Sl5Block& b = a.blk[tt.s];
    const int nch = (int)((b.I2 + TG_KC - 1) / TG_KC);
    const int R = b.R;
    const long long J = b.I0 * b.I1;
    if (tt.s != cur) {
      asm volatile("bar.sync 1, %0;" ::"r"(SL5_CONS) : "memory");
      cur = tt.s;
      const double* A2 = a.U[3 * tt.s + 2];
      const int kpad = nch * TG_KC;
      for (int e = threadIdx.x; e < kpad * RB; e += SL5_CONS) {
        const int k = e / RB, r = e - (e / RB) * RB;
        a2s[e] = (k < b.I2 && r < R) ? A2[(long long)k * R + r] : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(SL5_CONS) : "memory");
    }
    double acc[2][CG2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < CG2; ++v) acc[u][v] = 0.0;
    for (int c = 0; c < nch; ++c) {
      mbar_wait(&full[st], ph);
      const float* tile = reinterpret_cast<const float*>(ring + (size_t)st * TG_BOX);
      const double* ar = a2s + (size_t)c * TG_KC * RB + cg * CG2;
#pragma unroll 4
      for (int k = 0; k < TG_KC; ++k) {
        const float2 x2 = *reinterpret_cast<const float2*>(tile + k * TG_M + 2 * jg);
        const double x0 = x2.x, x1 = x2.y;
        double av[CG2];
#pragma unroll
        for (int v = 0; v < CG2; ++v) av[v] = ar[k * RB + v];
#pragma unroll
        for (int v = 0; v < CG2; ++v) {
          acc[0][v] = fma(x0, av[v], acc[0][v]);
          acc[1][v] = fma(x1, av[v], acc[1][v]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == TG_NST) { st = 0; ph ^= 1; }
    }
    double* T = reinterpret_cast<double*>(sel ? a.T1[tt.s] : a.T0[tt.s]);
    const long long j0 = (long long)tt.t * TG_M + 2 * jg;
#pragma unroll
    for (int v = 0; v < CG2; ++v) {
      const int r = cg * CG2 + v;
      if (r >= R) continue;
      double* dst = T + (long long)r * J + j0;
      if (j0 + 1 < J) {
        reinterpret_cast<double2*>(dst)[0] = make_double2(acc[0][v], acc[1][v]);
      } else if (j0 < J) {
        dst[0] = acc[0][v];
      }
    }
  }
}

template <int RB>
__global__ void __launch_bounds__(SL5_THREADS, 1) k_sl5_dpass(Sl5Args a) {
  griddep_wait();
  if (a.gate && *a.gate == 0) return;
  constexpr int CG = RB / 4;                   // columns per thread
  extern __shared__ unsigned char sl5_raw[];
  const uint32_t raw_u32 = smem_u32(sl5_raw);
  unsigned char* sm = sl5_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  unsigned char* ring = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + SL5_NST * SL5_BOX);
  uint64_t* empty = full + SL5_NST;
  double* a0s = reinterpret_cast<double*>(empty + SL5_NST + 2);   // [I0 + pad][RB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto ntl = [&](int s) -> long long { return a.blk[s].ntiles; };
  if (threadIdx.x == 0) {
    for (int i = 0; i < SL5_NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], SL5_CONS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == SL5_CONS / 32) {
    // ------------------------------------------------------- producer lane
    if (lane == 0) {
      int st = 0, ph = 0;
      for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
           act_tiles_next(it, a.active, a.S, ntl)) {
        const Sl5Tile tt{it.s, (int)it.t};
        const int nch = a.blk[tt.s].nch;
        const CUtensorMap* tm = a.tmaps + tt.s;
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], SL5_BOX);
          sl5_tma(ring + (size_t)st * SL5_BOX, tm, c * SL5_KC, tt.t * SL5_M, &full[st]);
          if (++st == SL5_NST) { st = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int rg = threadIdx.x & 63;             // rows rg, rg + 64 of the tile
  const int cg = threadIdx.x >> 6;             // columns [cg CG, (cg + 1) CG)
  int st = 0, ph = 0, cur = -1;
  for (ActTiles it = act_tiles_begin(a.active, a.S, ntl); it.left > 0;
       act_tiles_next(it, a.active, a.S, ntl)) {
    const Sl5Tile tt{it.s, (int)it.t};
    const Sl5Block& b = a.blk[tt.s];
    const int nch = b.nch;
    const int R = b.R;
    if (tt.s != cur) {
      // the block's A0 (fp64, zero-padded to nch * 32 rows and RB columns)
      asm volatile("bar.sync 1, %0;" ::"r"(SL5_CONS) : "memory");
      cur = tt.s;
      const double* A0 = a.U[3 * tt.s];
      const int kpad = nch * SL5_KC;
      for (int e = threadIdx.x; e < kpad * RB; e += SL5_CONS) {
        const int k = e / RB, r = e - (e / RB) * RB;
        a0s[e] = (k < b.I0 && r < R) ? A0[(long long)k * R + r] : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(SL5_CONS) : "memory");
    }
    double acc[2][CG];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < CG; ++j) acc[i][j] = 0.0;
    for (int c = 0; c < nch; ++c) {
      mbar_wait(&full[st], ph);
      const unsigned char* tile = ring + (size_t)st * SL5_BOX;
#pragma unroll 2
      for (int k4 = 0; k4 < SL5_KC / 4; ++k4) {
        // 16-byte chunk k4 of rows rg and rg + 64 (128-byte swizzle)
        const float4 x0 = *reinterpret_cast<const float4*>(tile + rg * 128 + ((k4 ^ (rg & 7)) << 4));
        const float4 x1 =
            *reinterpret_cast<const float4*>(tile + (rg + 64) * 128 + ((k4 ^ (rg & 7)) << 4));
        const double xa[4] = {x0.x, x0.y, x0.z, x0.w};
        const double xb[4] = {x1.x, x1.y, x1.z, x1.w};
        const double* ar = a0s + (size_t)(c * SL5_KC + k4 * 4) * RB + cg * CG;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          double av[CG];
#pragma unroll
          for (int j = 0; j < CG; ++j) av[j] = ar[kk * RB + j];
#pragma unroll
          for (int j = 0; j < CG; ++j) {
            acc[0][j] = fma(xa[kk], av[j], acc[0][j]);
            acc[1][j] = fma(xb[kk], av[j], acc[1][j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == SL5_NST) { st = 0; ph ^= 1; }
    }
    const long long r0 = (long long)tt.t * SL5_M;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const long long row = r0 + rg + 64 * i;
      if (row < b.J) {
#pragma unroll
        for (int j = 0; j < CG; ++j) {
          const int r = cg * CG + j;
          if (r < R) b.D[(long long)r * b.J + row] = acc[i][j];
        }
      }
    }
  }
}

// M2[i2, r] = sum_{i1} A1[i1, r] D[r][i1 + I1 i2]: one warp per (s, i2, r)
__global__ void __launch_bounds__(256) k_sl5_contract(Sl5Args a) {
  griddep_wait();
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)a.S * a.i2max * 64;
  for (long long w = (blockIdx.x * 256LL + threadIdx.x) >> 5; w < nw;
       w += ((long long)gridDim.x * 256) >> 5) {
    const int s = (int)(w / (a.i2max * 64));
    const long long rem = w - (long long)s * a.i2max * 64;
    const long long i2 = rem >> 6;
    const int r = (int)(rem & 63);
    if (a.active && !a.active[s]) continue;
    const Sl5Block& b = a.blk[s];
    if (i2 >= b.I2 || r >= b.R) continue;
    const double* A1 = a.U[3 * s + 1];
    const double* d = b.D + (long long)r * b.J + i2 * b.I1;
    double v = 0.0;
    for (long long i1 = lane; i1 < b.I1; i1 += 32) v = fma(A1[i1 * b.R + r], d[i1], v);
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) a.mtt[s][i2 * b.R + r] = v;
  }
}

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
static int sl5_rb(int rmax) {
  if (rmax <= 8) return 8;
  if (rmax <= 12) return 12;
  if (rmax <= 16) return 16;
  if (rmax <= 24) return 24;
  if (rmax <= 32) return 32;
  if (rmax <= 40) return 40;
  if (rmax <= 48) return 48;
  return 64;
}

static size_t sl5_smem(long long kpad, int rb) {
  return 1024 + (size_t)SL5_NST * SL5_BOX + 8 * (2 * SL5_NST + 2) + (size_t)kpad * rb * 8;
}

bool sl5_supported(int S, const void* const* X, const long long* dims, const int* R) {
  int rmax = 1;
  long long kmax = 1;
  for (int s = 0; s < S; ++s) {
    const long long I0 = dims[3 * s];
    if (I0 < 1 || I0 % 4 != 0) return false;
    if (dims[3 * s + 1] * dims[3 * s + 2] >= (1LL << 31)) return false;
    if (R[s] < 1 || R[s] > 64) return false;
    if ((reinterpret_cast<uintptr_t>(X[s]) & 15) != 0) return false;
    rmax = std::max(rmax, R[s]);
    kmax = std::max(kmax, (I0 + SL5_KC - 1) / SL5_KC * SL5_KC);
  }
  return sl5_smem(kmax, sl5_rb(rmax)) <= (size_t)SL5_SMEM_MAX;
}

typedef CUresult (*Sl5EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int sl5_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                    cudaStream_t st, Sl5Plan** out) {
  *out = nullptr;
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fnp, 12000, cudaEnableDefault,
                                       &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return CB_ERR_CUDA;
  }
  Sl5EncodeFn enc = reinterpret_cast<Sl5EncodeFn>(fnp);
  set_alloc_stream(st);   // buffers zeroed on the stream that uses them
  Sl5Plan* p = new Sl5Plan();
  p->S = S;
  int rmax = 1;
  long long kmax = 1;
  for (int s = 0; s < S; ++s) rmax = std::max(rmax, R[s]);
  p->rb = sl5_rb(rmax);
  std::vector<Sl5Block> hb(S);
  std::vector<Sl5Tile> ht;
  std::vector<CUtensorMap> hm(S);
  std::vector<void*>& A = p->allocs;
  for (int s = 0; s < S; ++s) {
    Sl5Block& b = hb[s];
    b.I0 = dims[3 * s]; b.I1 = dims[3 * s + 1]; b.I2 = dims[3 * s + 2];
    b.J = b.I1 * b.I2;
    b.R = R[s];
    b.ntiles = (int)((b.J + SL5_M - 1) / SL5_M);
    b.nch = (int)((b.I0 + SL5_KC - 1) / SL5_KC);
    kmax = std::max(kmax, (long long)b.nch * SL5_KC);
    p->i2max = std::max(p->i2max, b.I2);
    for (int t = 0; t < b.ntiles; ++t) ht.push_back({s, t});
    int rc = dalloc((void**)&b.D, sizeof(double) * (size_t)b.R * b.J, A);
    if (rc) { sl5_plan_destroy(p); return rc; }
    cuuint64_t gdim[2] = {(cuuint64_t)b.I0, (cuuint64_t)b.J};
    cuuint64_t gstride[1] = {(cuuint64_t)b.I0 * 4};
    cuuint32_t box[2] = {SL5_KC, SL5_M};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&hm[s], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(X[s]), gdim, gstride,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      sl5_plan_destroy(p);
      set_error("cuTensorMapEncodeTiled failed for block %d", s);
      return CB_ERR_CUDA;
    }
  }
  p->ntiles = (int)ht.size();
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  p->grid = std::max(1, std::min(nsm, p->ntiles));
  p->smem = sl5_smem(kmax, p->rb);
  int rc = CB_OK;
  if ((rc = dalloc((void**)&p->tmaps, sizeof(CUtensorMap) * S, A)) ||
      (rc = dalloc((void**)&p->blk, sizeof(Sl5Block) * S, A)) ||
      (rc = dalloc((void**)&p->tiles, sizeof(Sl5Tile) * ht.size(), A))) {
    sl5_plan_destroy(p);
    return rc;
  }
  CB_CUDA(cudaMemcpyAsync(p->tmaps, hm.data(), sizeof(CUtensorMap) * S, cudaMemcpyHostToDevice, st));
  CB_CUDA(cudaMemcpyAsync(p->blk, hb.data(), sizeof(Sl5Block) * S, cudaMemcpyHostToDevice, st));
  CB_CUDA(cudaMemcpyAsync(p->tiles, ht.data(), sizeof(Sl5Tile) * ht.size(), cudaMemcpyHostToDevice, st));
#define SL5_ATTR(RBV)                                                                   \
  CB_CUDA(cudaFuncSetAttribute(k_sl5_dpass<RBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)p->smem))
  switch (p->rb) {
    case 8: SL5_ATTR(8); break;
    case 12: SL5_ATTR(12); break;
    case 16: SL5_ATTR(16); break;
    case 24: SL5_ATTR(24); break;
    case 32: SL5_ATTR(32); break;
    case 40: SL5_ATTR(40); break;
    case 48: SL5_ATTR(48); break;
    default: SL5_ATTR(64); break;
  }
#undef SL5_ATTR
  // ---- T pass GEMM: J % 4 == 0 (16-byte rows of the (J x I2) view), R > 8,
  // staging within shared memory
  {
    long long i2pad = 1;
    bool ok = true;
    for (int s = 0; s < S; ++s) {
      const long long J = dims[3 * s] * dims[3 * s + 1];
      ok = ok && J % 4 == 0 && R[s] > 8;
      i2pad = std::max(i2pad, (dims[3 * s + 2] + TG_KC - 1) / TG_KC * TG_KC);
    }
    const int trb = p->rb < 16 ? 16 : (p->rb == 12 ? 16 : p->rb);
    const size_t tsm = 1024 + (size_t)TG_NST * TG_BOX + 8 * (2 * TG_NST + 2) + (size_t)i2pad * trb * 8;
    if (ok && tsm <= (size_t)SL5_SMEM_MAX) {
      std::vector<CUtensorMap> tm(S);
      std::vector<Sl5Tile> tt;
      for (int s = 0; s < S && ok; ++s) {
        const long long J = dims[3 * s] * dims[3 * s + 1];
        for (long long t = 0; t < (J + TG_M - 1) / TG_M; ++t) tt.push_back({s, (int)t});
        cuuint64_t gdim[2] = {(cuuint64_t)J, (cuuint64_t)dims[3 * s + 2]};
        cuuint64_t gstride[1] = {(cuuint64_t)J * 4};
        cuuint32_t box[2] = {TG_M, TG_KC};
        cuuint32_t estr[2] = {1, 1};
        ok = enc(&tm[s], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(X[s]), gdim,
                 gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
      if (ok) {
        p->tg_rb = trb;
        p->tg_smem = tsm;
        p->tg_ntiles = (int)tt.size();
        p->tg_grid = std::max(1, std::min(nsm, p->tg_ntiles));
        if ((rc = dalloc((void**)&p->tg_maps, sizeof(CUtensorMap) * S, A)) ||
            (rc = dalloc((void**)&p->tg_tiles, sizeof(Sl5Tile) * tt.size(), A))) {
          sl5_plan_destroy(p);
          return rc;
        }
        CB_CUDA(cudaMemcpyAsync(p->tg_maps, tm.data(), sizeof(CUtensorMap) * S,
                                cudaMemcpyHostToDevice, st));
        CB_CUDA(cudaMemcpyAsync(p->tg_tiles, tt.data(), sizeof(Sl5Tile) * tt.size(),
                                cudaMemcpyHostToDevice, st));
#define TG_ATTR(RBV)                                                                      \
  CB_CUDA(cudaFuncSetAttribute(k_tg_pass<RBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)p->tg_smem))
        switch (p->tg_rb) {
          case 16: TG_ATTR(16); break;
          case 24: TG_ATTR(24); break;
          case 32: TG_ATTR(32); break;
          case 40: TG_ATTR(40); break;
          case 48: TG_ATTR(48); break;
          default: TG_ATTR(64); break;
        }
#undef TG_ATTR
        p->tg_ok = true;
      }
    }
  }
  *out = p;
  return CB_OK;
}

bool sl5_tpass_ok(const Sl5Plan* p) { return p && p->tg_ok; }

int sl5_tpass(Sl5Plan* p, const double* const* U_dev, const int* active, void* const* T0,
              void* const* T1, const int* tsel, int t_other, cudaStream_t st) {
  if (!p->tg_ok) {
    set_error("T-pass GEMM not available for these blocks");
    return CB_ERR_UNSUPPORTED;
  }
  TgArgs a;
  memset(&a, 0, sizeof(a));
  a.tmaps = p->tg_maps;
  a.blk = p->blk;
  a.tiles = p->tg_tiles;
  a.ntiles = p->tg_ntiles;
  a.U = U_dev;
  a.active = active;
  a.T0 = T0;
  a.T1 = T1;
  a.tsel = tsel;
  a.t_other = t_other;
  a.S = p->S;
  switch (p->tg_rb) {
    case 16: CB_CUDA(launch_k(k_tg_pass<16>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
    case 24: CB_CUDA(launch_k(k_tg_pass<24>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
    case 32: CB_CUDA(launch_k(k_tg_pass<32>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
    case 40: CB_CUDA(launch_k(k_tg_pass<40>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
    case 48: CB_CUDA(launch_k(k_tg_pass<48>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
    default: CB_CUDA(launch_k(k_tg_pass<64>, dim3(p->tg_grid), dim3(SL5_THREADS), p->tg_smem, st, a)); break;
  }
  count_launch(1);
  return CB_OK;
}

void sl5_plan_destroy(Sl5Plan* p) {
  if (!p) return;
  dfree_all(p->allocs);
  delete p;
}

int sl5_mode2(Sl5Plan* p, const double* const* U_dev, const int* active, double* const* mtt,
              cudaStream_t st, const int* gate) {
  Sl5Args a;
  memset(&a, 0, sizeof(a));
  a.tmaps = p->tmaps;
  a.blk = p->blk;
  a.tiles = p->tiles;
  a.ntiles = p->ntiles;
  a.U = U_dev;
  a.active = active;
  a.mtt = mtt;
  a.S = p->S;
  a.i2max = p->i2max;
  a.gate = gate;
  switch (p->rb) {
    case 8: CB_CUDA(launch_k(k_sl5_dpass<8>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 12: CB_CUDA(launch_k(k_sl5_dpass<12>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 16: CB_CUDA(launch_k(k_sl5_dpass<16>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 24: CB_CUDA(launch_k(k_sl5_dpass<24>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 32: CB_CUDA(launch_k(k_sl5_dpass<32>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 40: CB_CUDA(launch_k(k_sl5_dpass<40>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    case 48: CB_CUDA(launch_k(k_sl5_dpass<48>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
    default: CB_CUDA(launch_k(k_sl5_dpass<64>, dim3(p->grid), dim3(SL5_THREADS), p->smem, st, a)); break;
  }
  const long long warps = (long long)p->S * p->i2max * 64;
  const int grid = (int)std::max(1LL, std::min((warps * 32 + 255) / 256, 148LL * 16));
  CB_CUDA(launch_k(k_sl5_contract, dim3(grid), dim3(256), 0, st, a));
  count_launch(2);
  return CB_OK;
}

}  // namespace cb
