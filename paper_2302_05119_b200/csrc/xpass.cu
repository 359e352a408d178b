// Launchers and unit tables of the tensor-streaming kernels (xpass2.cuh,
// xpass.cuh), shared by the solver (engine.cu) and ALS (als.cu) engines.
// Kept in their own translation unit: they hold every template instantiation
// of the streaming kernels.
//
// Precision codes (storage type of the tensor, arithmetic of the pass):
//   PC_F64     fp64 storage, fp64 arithmetic (parity mode)
//   PC_F32_F64 fp32 storage, fp64 arithmetic (throughput mode default: half the
//              bytes, reference-grade sums so the restart rule sees the same
//              objective the reference does)
//   PC_F32     fp32 storage, fp32 arithmetic (trace-only / large-rank passes)
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "engine_host.h"
#include "launch.cuh"
#include "ops_internal.h"
#include "status.h"
#include "xpass2.cuh"
#include "xpass3.cuh"
#include "xpass4.cuh"

namespace cb {

int rank_bucket(int r) {
  return r <= 8 ? 8 : r <= 10 ? 10 : r <= 12 ? 12 : r <= 16 ? 16 : r <= 24 ? 24 : r <= 32 ? 32
         : r <= 40 ? 40 : 64;
}
int pc_compute_bytes(int pc) { return pc == PC_F32 ? 4 : 8; }
static int pc_storage_bytes(int pc) { return pc == PC_F64 ? 8 : 4; }

// ---- dispatch helpers: F(TE, TC, RB) over the precision code and bucket ----
#define CB_RB_SWITCH(RBV, CALL)                     \
  switch (RBV) {                                    \
    case 8: { constexpr int RB = 8; CALL; } break;  \
    case 10: { constexpr int RB = 10; CALL; } break; \
    case 12: { constexpr int RB = 12; CALL; } break; \
    case 16: { constexpr int RB = 16; CALL; } break; \
    case 24: { constexpr int RB = 24; CALL; } break; \
    case 32: { constexpr int RB = 32; CALL; } break; \
    case 40: { constexpr int RB = 40; CALL; } break; \
    default: { constexpr int RB = 64; CALL; } break; \
  }

// n < 0: set the dynamic shared-memory attribute (call outside graph capture)
template <typename TE, typename TC, int RB, bool T, bool B, bool S, int TJ>
static void fib2_go_tj(bool tma, const XArgs& a, const FibUnit* u, int n, const XTables& t,
                       cudaStream_t st) {
  const size_t sm = fiber2_smem<TE, TC, RB>(t.fib_rows, TJ);
  if (n < 0) {
    cudaFuncSetAttribute(fiber2_kernel<TE, TC, RB, T, B, S, TJ>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    return;
  }
  launch_k(fiber2_kernel<TE, TC, RB, T, B, S, TJ>, dim3(n), dim3(X2_THREADS), sm, st, a, u,
           tma ? 1 : 0);
}

// the fiber tile TJ (columns per thread) is chosen by build_xtables: the
// register-budget default x2_tile, halved when that leaves SMs idle
template <typename TE, typename TC, int RB, bool T, bool B, bool S>
static void fib2_go(bool tma, const XArgs& a, const FibUnit* u, int n, const XTables& t,
                    cudaStream_t st) {
  constexpr int TD = x2_tile(RB, sizeof(TC));
  if (t.fib_tj >= TD) fib2_go_tj<TE, TC, RB, T, B, S, TD>(tma, a, u, n, t, st);
  else if (t.fib_tj == 3) fib2_go_tj<TE, TC, RB, T, B, S, (TD >= 3 ? 3 : 1)>(tma, a, u, n, t, st);
  else if (t.fib_tj == 2) fib2_go_tj<TE, TC, RB, T, B, S, (TD >= 2 ? 2 : 1)>(tma, a, u, n, t, st);
  else fib2_go_tj<TE, TC, RB, T, B, S, 1>(tma, a, u, n, t, st);
}

template <typename TE, typename TC, int RB>
static void fib2_combo(bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                       const FibUnit* u, int n, const XTables& t, cudaStream_t st) {
  // (T, B, RES) combinations used by the engines; T-only runs the RES variant
  if (want_t && want_b && want_res) fib2_go<TE, TC, RB, true, true, true>(tma, a, u, n, t, st);
  else if (want_t && want_b) fib2_go<TE, TC, RB, true, true, false>(tma, a, u, n, t, st);
  else if (want_t && want_res) fib2_go<TE, TC, RB, true, false, true>(tma, a, u, n, t, st);
  else if (want_t) fib2_go<TE, TC, RB, true, false, false>(tma, a, u, n, t, st);
  else fib2_go<TE, TC, RB, false, true, false>(tma, a, u, n, t, st);
}

static void fiber_dispatch(int pc, int rb, bool tma, int want_t, int want_b, int want_res,
                           const XArgs& a, const FibUnit* u, int n, const XTables& t,
                           cudaStream_t st) {
  if (pc == PC_F32) {
    CB_RB_SWITCH(rb, (fib2_combo<float, float, RB>(tma, want_t, want_b, want_res, a, u, n, t, st)));
  } else if (pc == PC_F32_F64) {
    CB_RB_SWITCH(rb, (fib2_combo<float, double, RB>(tma, want_t, want_b, want_res, a, u, n, t, st)));
  } else {
    CB_RB_SWITCH(rb, (fib2_combo<double, double, RB>(tma, want_t, want_b, want_res, a, u, n, t, st)));
  }
}

// warp-specialised T pass (xpass4.cuh): T-only launches, fp32 storage with
// fp64 arithmetic, unsplit T, rank bucket <= 16, bulk-copy rows
static bool fiber4_ok(int pc, int rb, bool tma, const XTables& t) {
  return pc == PC_F32_F64 && rb <= 16 && tma && t.fiber_direct && t.fib4_tj > 0;
}

template <int RB, int TJ>
static void fiber4_go(const XArgs& a, const FibUnit* u, int n, const XTables& t, cudaStream_t st,
                      bool prep) {
  const size_t sm = fiber4_smem<float>(t.fib_rows, RB, TJ);
  if (prep) {
    cudaFuncSetAttribute(fiber4_kernel<float, RB, TJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    return;
  }
  launch_k(fiber4_kernel<float, RB, TJ>, dim3(n), dim3(F4_THREADS), sm, st, a, u);
}

template <int RB>
static void fiber4_tj(const XArgs& a, const FibUnit* u, int n, const XTables& t, cudaStream_t st,
                      bool prep) {
  if (t.fib4_tj >= 4) fiber4_go<RB, 4>(a, u, n, t, st, prep);
  else if (t.fib4_tj == 3) fiber4_go<RB, 3>(a, u, n, t, st, prep);
  else if (t.fib4_tj == 2) fiber4_go<RB, 2>(a, u, n, t, st, prep);
  else fiber4_go<RB, 1>(a, u, n, t, st, prep);
}

static void fiber4_dispatch(int rb, const XArgs& a, const FibUnit* u, int n, const XTables& t,
                            cudaStream_t st, bool prep) {
  if (rb <= 8) fiber4_tj<8>(a, u, n, t, st, prep);
  else if (rb <= 10) fiber4_tj<10>(a, u, n, t, st, prep);
  else if (rb <= 12) fiber4_tj<12>(a, u, n, t, st, prep);
  else fiber4_tj<16>(a, u, n, t, st, prep);
}

// T + explicit residual (the ALS sweep's fiber pass) for ranks > 16 on the
// fiber4 ring, over the fiber2 unit table (same units, same partial slots)
static bool fiber4res_ok(int pc, int rb, bool tma, const XTables& t) {
  return pc == PC_F32_F64 && rb >= 24 && tma && t.fib_unsplit &&
         t.fib_tj == x2_tile(rb, 8);
}

template <int RB>
static void fiber4res_go(const XArgs& a, const FibUnit* u, int n, const XTables& t,
                         cudaStream_t st, bool prep) {
  constexpr int TJ = x2_tile(RB, 8);
  const size_t sm = fiber4_smem<float>(t.fib_rows, RB, TJ);
  if (prep) {
    cudaFuncSetAttribute(fiber4_kernel<float, RB, TJ, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    return;
  }
  launch_k(fiber4_kernel<float, RB, TJ, true>, dim3(n), dim3(F4_THREADS), sm, st, a, u);
}

static void fiber4res_dispatch(int rb, const XArgs& a, const FibUnit* u, int n, const XTables& t,
                               cudaStream_t st, bool prep) {
  if (rb <= 24) fiber4res_go<24>(a, u, n, t, st, prep);
  else if (rb <= 32) fiber4res_go<32>(a, u, n, t, st, prep);
  else if (rb <= 40) fiber4res_go<40>(a, u, n, t, st, prep);
  else fiber4res_go<64>(a, u, n, t, st, prep);
}

void prepare_fiber(int pc, int rb, bool tma, const XTables& t) {
  XArgs a{};
  if (fiber4_ok(pc, rb, tma, t)) fiber4_dispatch(rb, a, nullptr, 0, t, 0, true);
  if (fiber4res_ok(pc, rb, tma, t)) fiber4res_dispatch(rb, a, nullptr, 0, t, 0, true);
  const int combos[5][3] = {{1, 1, 1}, {1, 1, 0}, {1, 0, 1}, {1, 0, 0}, {0, 1, 0}};
  for (auto& c : combos) fiber_dispatch(pc, rb, tma, c[0], c[1], c[2], a, nullptr, -1, t, 0);
}

void launch_fiber(int pc, int rb, bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                  const FibUnit* u, int n, const XTables& t, cudaStream_t st) {
  if (want_t && want_res && !want_b && n > 0 && fiber4res_ok(pc, rb, tma, t)) {
    fiber4res_dispatch(rb, a, u, n, t, st, false);
    count_launch(1);
    return;
  }
  if (want_t && !want_b && !want_res && n > 0 && t.d_fib4 && fiber4_ok(pc, rb, tma, t)) {
    fiber4_dispatch(rb, a, t.d_fib4, (int)t.fib4.size(), t, st, false);
    count_launch(1);
    return;
  }
  if (n <= 0) return;
  fiber_dispatch(pc, rb, tma, want_t, want_b, want_res, a, u, n, t, st);
  count_launch(1);
}

template <typename TE, int RB>
static void slab3_go(bool tma, const XArgs& a, const XTables& t, cudaStream_t st, bool prep) {
  const int ntasks = t.s3_first.back();
  const int S = (int)t.s3_first.size() - 1;
  const int grid = std::max(1, std::min((ntasks + S3_WARPS - 1) / S3_WARPS, 148 * 4));
  const int rows = slab3_rows(t.s3_max_i0, (int)sizeof(TE));
  const int a1r = (int)t.s3_a1_rows;
  const size_t sm = slab3_smem(t.s3_max_i0, (int)sizeof(TE), rows, a1r, RB, tma);
#define S3_LAUNCH(NS)                                                                            \
  do {                                                                                           \
    if (tma) {                                                                                   \
      if (prep) {                                                                                \
        cudaFuncSetAttribute(slab3_kernel<TE, RB, NS, S3_RING>,                                  \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);              \
        return;                                                                                  \
      }                                                                                          \
      launch_k(slab3_kernel<TE, RB, NS, S3_RING>, dim3(grid), dim3(S3_WARPS * 32), sm, st, a,    \
               a.s3_first, S, ntasks, rows, a1r);                                                \
    } else {                                                                                     \
      if (prep) {                                                                                \
        cudaFuncSetAttribute(slab3_kernel<TE, RB, NS, 0>,                                        \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);              \
        return;                                                                                  \
      }                                                                                          \
      launch_k(slab3_kernel<TE, RB, NS, 0>, dim3(grid), dim3(S3_WARPS * 32), sm, st, a,          \
               a.s3_first, S, ntasks, rows, a1r);                                                \
    }                                                                                            \
  } while (0)
  switch (t.s3_nslot) {
    case 1: S3_LAUNCH(1); break;
    case 2: S3_LAUNCH(2); break;
    case 3: S3_LAUNCH(3); break;
    default: S3_LAUNCH(4); break;
  }
#undef S3_LAUNCH
}

template <typename TE>
static void slab3_dispatch(int rb, bool tma, const XArgs& a, const XTables& t, cudaStream_t st,
                           bool prep) {
  if (rb <= 8) slab3_go<TE, 8>(tma, a, t, st, prep);
  else if (rb <= 10) slab3_go<TE, 10>(tma, a, t, st, prep);
  else if (rb <= 12) slab3_go<TE, 12>(tma, a, t, st, prep);
  else slab3_go<TE, 16>(tma, a, t, st, prep);
}

template <typename TE, typename TC, int RB>
static void slab2_go(bool tma, const XArgs& a, const SlabUnit* u, int n, const XTables& t,
                     cudaStream_t st) {
  const size_t sm = slab2_smem<TE, TC, RB>(t.slab_rows);
  if (n < 0) {
    cudaFuncSetAttribute(slab2_kernel<TE, TC, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    return;
  }
  launch_k(slab2_kernel<TE, TC, RB>, dim3(n), dim3(X2_THREADS), sm, st, a, u, tma ? 1 : 0);
}

static void slab_dispatch(int pc, int rb, bool tma, const XArgs& a, const SlabUnit* u, int n,
                          const XTables& t, cudaStream_t st) {
  if (pc == PC_F32) {
    CB_RB_SWITCH(rb, (slab2_go<float, float, RB>(tma, a, u, n, t, st)));
  } else if (pc == PC_F32_F64) {
    CB_RB_SWITCH(rb, (slab2_go<float, double, RB>(tma, a, u, n, t, st)));
  } else {
    CB_RB_SWITCH(rb, (slab2_go<double, double, RB>(tma, a, u, n, t, st)));
  }
}

void prepare_slab(int pc, int rb, bool tma, const XTables& t) {
  XArgs a{};
  if (t.slab_direct) {
    const bool ring = tma && t.s3_tma;
    if (pc == PC_F64) slab3_dispatch<double>(t.f3_rb, ring, a, t, 0, true);
    else slab3_dispatch<float>(t.f3_rb, ring, a, t, 0, true);
    return;
  }
  slab_dispatch(pc, rb, tma, a, nullptr, -1, t, 0);
}

void launch_slab(int pc, int rb, bool tma, const XArgs& a, const SlabUnit* u, int n,
                 const XTables& t, cudaStream_t st) {
  if (t.slab_direct) {
    // fp64 arithmetic (the row-dot kernel has no fp32-arithmetic variant)
    const bool ring = tma && t.s3_tma;
    if (pc == PC_F64) slab3_dispatch<double>(t.f3_rb, ring, a, t, st, false);
    else slab3_dispatch<float>(t.f3_rb, ring, a, t, st, false);
    count_launch(1);
    return;
  }
  if (n <= 0) return;
  slab_dispatch(pc, rb, tma, a, u, n, t, st);
  count_launch(1);
}

void launch_contract(int pc, int mode, const XArgs& a, const RowUnit* u, int n,
                     cudaStream_t st) {
  if (n <= 0) return;
  const bool tf = pc == PC_F32;   // T is stored in the fiber pass arithmetic type
  if (mode == 0) {
    if (tf) launch_k(contract0_kernel<float>, dim3(n), dim3(256), 0, st, a, u);
    else launch_k(contract0_kernel<double>, dim3(n), dim3(256), 0, st, a, u);
  } else {
    if (tf) launch_k(contract1_kernel<float>, dim3(n), dim3(256), 0, st, a, u);
    else launch_k(contract1_kernel<double>, dim3(n), dim3(256), 0, st, a, u);
  }
  count_launch(1);
}

void contract_preload() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, contract0_kernel<float>);
  cudaFuncGetAttributes(&fa, contract0_kernel<double>);
  cudaFuncGetAttributes(&fa, contract1_kernel<float>);
  cudaFuncGetAttributes(&fa, contract1_kernel<double>);
}

bool tma_rows_ok(int S, const long long* dims, const void* const* X, int elem_bytes) {
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    if ((J * elem_bytes) % 16 != 0) return false;
    if (((uintptr_t)X[s]) % 16 != 0) return false;
  }
  return true;
}

// Work units.  The decomposition of a block depends only on that block's
// shape and on `s_total` (the number of blocks of the whole solve), so every
// block is reduced in the same order whether it runs alone or in a shard.
void build_xtables(int S, const long long* dims, const int* R, int rb, int pc, XTables& t,
                   int s_total) {
  const int tcb = pc_compute_bytes(pc);
  const int tile = x2_tile(rb, tcb);
  const long long target_per_block = (148LL * 2 + s_total - 1) / std::max(s_total, 1);
  // warp-task T pass (xpass3.cuh) where the shapes allow it; it writes T
  // unsplit, so every T producer then uses nsplit = 1
  {
    long long a2r = 1;
    for (int s = 0; s < S; ++s) a2r = std::max(a2r, dims[3 * s + 2]);
    t.f3_a2_rows = a2r;
    int rmax = 1;
    for (int s = 0; s < S; ++s) rmax = std::max(rmax, R[s]);
    t.f3_rb = rmax <= 8 ? 8 : rmax <= 10 ? 10 : rmax <= 12 ? 12 : 16;
    // pair loads / stores need even J; A2 copies must fit (2 CTAs per SM)
    bool even = true;
    for (int s = 0; s < S; ++s) even = even && (dims[3 * s] * dims[3 * s + 1]) % 2 == 0;
    const int f3rb = rmax <= 8 ? 8 : rmax <= 10 ? 10 : rmax <= 12 ? 12 : 16;
    t.fiber_direct = (pc != PC_F32 && rmax <= 16 && even &&
                      fiber3_smem(a2r, f3rb) <= 96 * 1024) ? 1 : 0;
    t.f3_first.assign(S + 1, 0);
    for (int s = 0; s < S; ++s) {
      const long long J = dims[3 * s] * dims[3 * s + 1];
      t.f3_first[s + 1] = t.f3_first[s] + (int)((J + F3_CH - 1) / F3_CH);
    }
  }
  t.fib.clear(); t.fib_first.assign(S + 1, 0); t.nsplit.assign(S, 1);
  // fiber tile: the register-budget tile (fiber2 units)
  t.fib_tj = tile;
  const long long JT = (long long)X2_THREADS * t.fib_tj;
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    const long long I2 = dims[3 * s + 2];
    const long long tiles = (J + JT - 1) / JT;
    int ns = 1;
    while (!t.fiber_direct && tiles * ns < target_per_block && I2 / (ns * 2) >= 2 * F2_CH) ns *= 2;
    t.nsplit[s] = ns;
    t.fib_first[s] = (int)t.fib.size();
    for (int sp = 0; sp < ns; ++sp)
      for (long long j0 = 0; j0 < J; j0 += JT) t.fib.push_back(FibUnit{s, sp, j0});
  }
  t.fib_first[S] = (int)t.fib.size();
  t.fib_unsplit = 1;
  for (int s = 0; s < S; ++s) t.fib_unsplit = t.fib_unsplit && t.nsplit[s] == 1;
  // fiber4 units: the tile minimising waves x TJ over this engine's blocks,
  // a wave being 148 CTAs (one per SM).  Counting several resident CTAs per
  // SM instead (c2: TJ 1, 4 CTAs per SM) made the kernel faster (34 -> 25 us)
  // but the step slower (6.33k -> 6.17k it/s): the T pass runs on the side
  // stream beside k_sweep_begin / k_step, the critical path, and at 4 CTAs
  // per SM it leaves those R x R kernels no SM (profiles/r01h_*).
  t.fib4.clear();
  t.fib4_tj = 0;
  if (t.fiber_direct && pc == PC_F32_F64 && rb <= 16) {
    long long best = -1;
    for (int c : {4, 3, 2, 1}) {
      long long u = 0;
      for (int s = 0; s < S; ++s) {
        const long long J = dims[3 * s] * dims[3 * s + 1];
        u += (J + 256LL * c - 1) / (256LL * c);
      }
      const long long slots = 148LL;
      const long long cost = ((u + slots - 1) / slots) * c;
      if (best < 0 || cost < best) { best = cost; t.fib4_tj = c; }
    }
    const long long JT4 = 256LL * t.fib4_tj;
    for (int s = 0; s < S; ++s) {
      const long long J = dims[3 * s] * dims[3 * s + 1];
      for (long long j0 = 0; j0 < J; j0 += JT4) t.fib4.push_back(FibUnit{s, 0, j0});
    }
  }
  t.sb = tile;
  const int kc = s2_kc(rb, tcb);
  t.slab.clear(); t.slab_first.assign(S, 0); t.slab_nchunk.assign(S, 1);
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    const long long I2 = dims[3 * s + 2];
    const long long groups = (I2 + tile - 1) / tile;
    int nch = 1;
    while (groups * nch < target_per_block && J / (nch * 2) >= 2 * kc) nch *= 2;
    t.slab_nchunk[s] = nch;
    t.slab_first[s] = (int)t.slab.size();
    // chunk boundaries on multiples of the stage width keep bulk copies aligned
    long long per = (J + nch - 1) / nch;
    per = (per + kc - 1) / kc * kc;
    for (long long g0 = 0; g0 < I2; g0 += tile)
      for (int ch = 0; ch < nch; ++ch) {
        const long long k0 = std::min(J, ch * per), k1 = std::min(J, k0 + per);
        t.slab.push_back(SlabUnit{s, (int)g0, k0, k1});
      }
  }
  t.c0.clear(); t.c1.clear();
  for (int s = 0; s < S; ++s) {
    for (int r = 0; r < R[s]; ++r)
      for (long long i0 = 0; i0 < dims[3 * s]; i0 += 32) t.c0.push_back(RowUnit{s, (int)((r << 20) | i0)});
    const long long n1 = dims[3 * s + 1] * R[s];
    for (long long p = 0; p < n1; p += 8) t.c1.push_back(RowUnit{s, (int)p});
  }
  // shared-memory staging of factor rows: A2 rows of a fiber unit always; the
  // A0/A1 rows of the slab kernel when they fit beside its X ring
  t.fib_rows = 0;
  long long ab = 0;
  for (int s = 0; s < S; ++s) {
    const long long I2 = dims[3 * s + 2];
    t.fib_rows = std::max(t.fib_rows, (I2 + t.nsplit[s] - 1) / t.nsplit[s]);
    ab = std::max(ab, dims[3 * s] + dims[3 * s + 1]);
  }
  const long long ring = 128 + (long long)S2_NST * tile * kc * pc_storage_bytes(pc);
  t.slab_rows = (ring + ab * rb * tcb <= 200 * 1024) ? ab : 0;
  // row-dot mode-2 kernel where the shapes allow it (arithmetic always fp64)
  t.slab_direct = (pc != PC_F32 && slab3_ok(S, dims, rb)) ? 1 : 0;
  t.s3_nslot = slab3_nslot(S, dims);
  t.s3_a1_rows = 1;
  for (int s = 0; s < S; ++s) t.s3_a1_rows = std::max(t.s3_a1_rows, dims[3 * s + 1]);
  // per-warp A1 copies must fit beside the ring
  if ((size_t)S3_WARPS * t.s3_a1_rows * t.f3_rb * 8 > 96 * 1024) t.slab_direct = 0;
  t.s3_max_i0 = 1;
  t.s3_tma = 1;
  for (int s = 0; s < S; ++s) {
    t.s3_max_i0 = std::max(t.s3_max_i0, dims[3 * s]);
    // every row (and so every stage) 16-B aligned
    if ((dims[3 * s] * pc_storage_bytes(pc)) % 16 != 0) t.s3_tma = 0;
  }
  t.s3_first.assign(S + 1, 0);
  for (int s = 0; s < S; ++s) t.s3_first[s + 1] = t.s3_first[s] + (int)dims[3 * s + 2];
}

}  // namespace cb
