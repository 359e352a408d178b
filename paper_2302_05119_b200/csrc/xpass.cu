// Launchers and unit tables of the tensor-streaming kernels (xpass.cuh),
// shared by the solver (engine.cu) and ALS (als.cu) engines.  Kept in their
// own translation unit: they hold every template instantiation of the
// streaming kernels.
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "engine_host.h"
#include "ops_internal.h"
#include "status.h"

namespace cb {

// Precision codes of the streaming kernels: storage type of the tensor and
// arithmetic type of the contraction.
//   PC_F64     fp64 storage, fp64 arithmetic (parity mode)
//   PC_F32_F64 fp32 storage, fp64 arithmetic (throughput mode default: half the
//              bytes, reference-grade sums so the restart rule sees the same
//              objective the reference does)
//   PC_F32     fp32 storage, fp32 arithmetic (trace-only / large-rank passes)
// n < 0: set the dynamic shared memory attribute (outside graph capture)
template <typename TE, typename TC, int RB, bool T, bool B, bool S>
static void fib_launch(bool tma, const XArgs& a, const FibUnit* u, int n, cudaStream_t st) {
  if (tma) {
    constexpr size_t sm = fiber_tma_smem<TE, TC, RB>();
    if (n < 0) {
      cudaFuncSetAttribute(fiber_kernel<TE, TC, RB, T, B, S, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      return;
    }
    fiber_kernel<TE, TC, RB, T, B, S, true><<<n, FIB_THREADS, sm, st>>>(a, u);
  } else {
    if (n < 0) return;
    fiber_kernel<TE, TC, RB, T, B, S, false><<<n, FIB_THREADS, 0, st>>>(a, u);
  }
}

template <typename TE, typename TC, int RB>
static void launch_fiber_t(bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                           const FibUnit* u, int n, cudaStream_t st) {
  if (want_t && want_b && want_res) fib_launch<TE, TC, RB, true, true, true>(tma, a, u, n, st);
  else if (want_t && want_b) fib_launch<TE, TC, RB, true, true, false>(tma, a, u, n, st);
  else if (want_t && want_res) fib_launch<TE, TC, RB, true, false, true>(tma, a, u, n, st);
  else if (want_t) fib_launch<TE, TC, RB, true, false, false>(tma, a, u, n, st);
  else fib_launch<TE, TC, RB, false, true, false>(tma, a, u, n, st);
}

template <typename TE, typename TC>
static void launch_fiber_r(int rb, bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                           const FibUnit* u, int n, cudaStream_t st) {
  switch (rb) {
    case 8: launch_fiber_t<TE, TC, 8>(tma, want_t, want_b, want_res, a, u, n, st); break;
    case 16: launch_fiber_t<TE, TC, 16>(tma, want_t, want_b, want_res, a, u, n, st); break;
    case 32: launch_fiber_t<TE, TC, 32>(tma, want_t, want_b, want_res, a, u, n, st); break;
    case 40: launch_fiber_t<TE, TC, 40>(tma, want_t, want_b, want_res, a, u, n, st); break;
    default: launch_fiber_t<TE, TC, 64>(tma, want_t, want_b, want_res, a, u, n, st); break;
  }
}

static void fiber_dispatch(int pc, int rb, bool tma, int want_t, int want_b, int want_res,
                           const XArgs& a, const FibUnit* u, int n, cudaStream_t st) {
  if (pc == PC_F32) launch_fiber_r<float, float>(rb, tma, want_t, want_b, want_res, a, u, n, st);
  else if (pc == PC_F32_F64) launch_fiber_r<float, double>(rb, tma, want_t, want_b, want_res, a, u, n, st);
  else launch_fiber_r<double, double>(rb, tma, want_t, want_b, want_res, a, u, n, st);
}

bool tma_rows_ok(int S, const long long* dims, const void* const* X, int elem_bytes) {
  if (getenv("CB_NO_TMA")) return false;
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    if ((J * elem_bytes) % 16 != 0) return false;
    if (((uintptr_t)X[s]) % 16 != 0) return false;
  }
  return true;
}

void prepare_fiber(int pc, int rb, bool tma) {
  XArgs a{};
  const int combos[5][3] = {{1, 1, 1}, {1, 1, 0}, {1, 0, 1}, {1, 0, 0}, {0, 1, 0}};
  for (auto& c : combos) fiber_dispatch(pc, rb, tma, c[0], c[1], c[2], a, nullptr, -1, 0);
}

void launch_fiber(int pc, int rb, bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                  const FibUnit* u, int n, cudaStream_t st) {
  if (n <= 0) return;
  fiber_dispatch(pc, rb, tma, want_t, want_b, want_res, a, u, n, st);
  count_launch(1);
}

template <typename TE, typename TC, int RB, int SB>
static void launch_slab_t(const XArgs& a, const SlabUnit* u, int n, size_t sm, cudaStream_t st) {
  if (n < 0) {   // attribute setup call (outside any graph capture)
    cudaFuncSetAttribute(slab_kernel<TE, TC, RB, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    return;
  }
  slab_kernel<TE, TC, RB, SB><<<n, SLAB_THREADS, sm, st>>>(a, u);
}

int slab_sb_for(int rb, int tc_bytes) {
  const int sb = rb <= 8 ? 8 : rb <= 16 ? 4 : rb <= 32 ? 2 : 1;
  return tc_bytes == 8 && sb > 1 ? sb / 2 : sb;
}

template <typename TE, typename TC>
static void launch_slab_r(int rb, const XArgs& a, const SlabUnit* u, int n, size_t sm,
                          cudaStream_t st) {
  constexpr bool D = sizeof(TC) == 8;
  switch (rb) {
    case 8: launch_slab_t<TE, TC, 8, D ? 4 : 8>(a, u, n, sm, st); break;
    case 16: launch_slab_t<TE, TC, 16, D ? 2 : 4>(a, u, n, sm, st); break;
    case 32: launch_slab_t<TE, TC, 32, D ? 1 : 2>(a, u, n, sm, st); break;
    case 40: launch_slab_t<TE, TC, 40, 1>(a, u, n, sm, st); break;
    default: launch_slab_t<TE, TC, 64, 1>(a, u, n, sm, st); break;
  }
}

static void slab_dispatch(int pc, int rb, const XArgs& a, const SlabUnit* u, int n, size_t sm,
                          cudaStream_t st) {
  if (pc == PC_F32) launch_slab_r<float, float>(rb, a, u, n, sm, st);
  else if (pc == PC_F32_F64) launch_slab_r<float, double>(rb, a, u, n, sm, st);
  else launch_slab_r<double, double>(rb, a, u, n, sm, st);
}

void prepare_slab(int pc, int rb, size_t sm) {
  XArgs a{};
  slab_dispatch(pc, rb, a, nullptr, -1, sm, 0);
}

void launch_slab(int pc, int rb, const XArgs& a, const SlabUnit* u, int n, size_t sm,
                 cudaStream_t st) {
  if (n <= 0) return;
  slab_dispatch(pc, rb, a, u, n, sm, st);
  count_launch(1);
}

void launch_contract(int pc, int mode, const XArgs& a, const RowUnit* u, int n,
                     cudaStream_t st) {
  if (n <= 0) return;
  const bool tf = pc == PC_F32;   // T is stored in the fiber pass arithmetic type
  if (mode == 0) {
    if (tf) contract0_kernel<float><<<n, 256, 0, st>>>(a, u);
    else contract0_kernel<double><<<n, 256, 0, st>>>(a, u);
  } else {
    if (tf) contract1_kernel<float><<<n, 256, 0, st>>>(a, u);
    else contract1_kernel<double><<<n, 256, 0, st>>>(a, u);
  }
  count_launch(1);
}

int pc_compute_bytes(int pc) { return pc == PC_F32 ? 4 : 8; }

int rank_bucket(int r) { return r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : r <= 40 ? 40 : 64; }

void build_xtables(int S, const long long* dims, const int* R, int rb, int pc, XTables& t) {
  const int target = 148 * 4;
  long long tiles = 0;
  for (int s = 0; s < S; ++s) tiles += (dims[3 * s] * dims[3 * s + 1] + FIB_THREADS - 1) / FIB_THREADS;
  t.fib.clear(); t.fib_first.assign(S + 1, 0); t.nsplit.assign(S, 1);
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    const long long I2 = dims[3 * s + 2];
    int ns = 1;
    while (tiles * ns < target && I2 / (ns * 2) >= 16) ns *= 2;
    t.nsplit[s] = ns;
    t.fib_first[s] = (int)t.fib.size();
    for (int sp = 0; sp < ns; ++sp)
      for (long long j0 = 0; j0 < J; j0 += FIB_THREADS) t.fib.push_back(FibUnit{s, sp, j0});
  }
  t.fib_first[S] = (int)t.fib.size();
  t.sb = slab_sb_for(rb, pc_compute_bytes(pc));
  long long groups = 0;
  for (int s = 0; s < S; ++s) groups += (dims[3 * s + 2] + t.sb - 1) / t.sb;
  t.slab.clear(); t.slab_first.assign(S, 0); t.slab_nchunk.assign(S, 1);
  long long maxI01 = 0;
  for (int s = 0; s < S; ++s) {
    const long long J = dims[3 * s] * dims[3 * s + 1];
    const long long I2 = dims[3 * s + 2];
    int nch = 1;
    while (groups * nch < target && J / (nch * 2) >= 4 * SLAB_THREADS) nch *= 2;
    t.slab_nchunk[s] = nch;
    t.slab_first[s] = (int)t.slab.size();
    const long long per = (J + nch - 1) / nch;
    for (long long g0 = 0; g0 < I2; g0 += t.sb)
      for (int ch = 0; ch < nch; ++ch) {
        long long k0 = ch * per, k1 = std::min(J, k0 + per);
        t.slab.push_back(SlabUnit{s, (int)g0, k0, k1});
      }
    maxI01 = std::max(maxI01, dims[3 * s] + dims[3 * s + 1]);
  }
  t.slab_smem = (size_t)maxI01 * rb * pc_compute_bytes(pc);
  t.c0.clear(); t.c1.clear();
  for (int s = 0; s < S; ++s) {
    for (int r = 0; r < R[s]; ++r)
      for (long long i0 = 0; i0 < dims[3 * s]; i0 += 32) t.c0.push_back(RowUnit{s, (int)((r << 20) | i0)});
    const long long n1 = dims[3 * s + 1] * R[s];
    for (long long p = 0; p < n1; p += 8) t.c1.push_back(RowUnit{s, (int)p});
  }
}

}  // namespace cb
