// Host-side helpers shared by the solver (engine.cu) and ALS (als.cu) engines.
#pragma once
#include <vector>

#include "status.h"
#include "xpass.cuh"

namespace cb {

struct XTables {
  std::vector<FibUnit> fib;
  std::vector<int> fib_first;   // S+1
  std::vector<int> nsplit;      // S
  std::vector<SlabUnit> slab;
  std::vector<int> slab_first;  // S
  std::vector<int> slab_nchunk; // S
  std::vector<RowUnit> c0, c1;
  int sb = 1;
  int fib_tj = 1;             // fiber tile: columns per thread (JT = 256 * fib_tj)
  // fiber4 (xpass4.cuh) T-only units: its own tile (T is per column, so the
  // tile does not change any bit; chosen to fill the SMs)
  std::vector<FibUnit> fib4;
  int fib4_tj = 0;
  int fib_unsplit = 0;              // every block's fiber units cover all of I2 (nsplit 1)
  const FibUnit* d_fib4 = nullptr;   // device copy (set by the engine)
  long long fib_rows = 0;    // max i2 rows of a fiber unit (A2 rows staged per CTA)
  long long slab_rows = 0;   // A0+A1 rows the slab kernel stages (0: read through L1)
  // row-dot mode-2 kernel (xpass3.cuh): writes MTT[s] directly when set
  int slab_direct = 0;
  int s3_nslot = 0;
  int s3_tma = 0;             // rows 16-B aligned: bulk-copy ring usable
  long long s3_max_i0 = 1;
  long long s3_a1_rows = 1;
  std::vector<int> s3_first;  // S+1
  // warp-task T pass (xpass3.cuh fiber3_kernel) for T-only fiber launches
  int fiber_direct = 0;
  int f3_rb = 16;             // exact small rank bucket of the T pass (8, 10, 12, 16)
  int f3_tma = 0;
  long long f3_a2_rows = 1;
  std::vector<int> f3_first;  // S+1 cumulative I1 (task ranges)
};

enum { PC_F64 = 0, PC_F32_F64 = 1, PC_F32 = 2 };
int pc_compute_bytes(int pc);
void build_xtables(int S, const long long* dims, const int* R, int rb, int pc, XTables& t,
                   int s_total);
int rank_bucket(int r);
// Streaming kernel launches: `t` supplies the unit shapes; n < 0 (prepare_*)
// only sets the kernels' shared-memory attributes (outside graph capture).
void launch_fiber(int pc, int rb, bool tma, int want_t, int want_b, int want_res, const XArgs& a,
                  const FibUnit* u, int n, const XTables& t, cudaStream_t st);
void prepare_fiber(int pc, int rb, bool tma, const XTables& t);
// 16-byte aligned rows for the bulk-copy (TMA) streaming path
bool tma_rows_ok(int S, const long long* dims, const void* const* X, int elem_bytes);
void prepare_slab(int pc, int rb, bool tma, const XTables& t);
void launch_slab(int pc, int rb, bool tma, const XArgs& a, const SlabUnit* u, int n,
                 const XTables& t, cudaStream_t st);
void launch_contract(int pc, int mode, const XArgs& a, const RowUnit* u, int n,
                     cudaStream_t st);
void contract_preload();   // load the contraction kernels now (lazy module loading)
int dalloc(void** p, size_t bytes, std::vector<void*>& allocs);
void dfree_all(std::vector<void*>& allocs);
void set_alloc_stream(cudaStream_t st);

template <typename T>
int upload(const std::vector<T>& v, T** d, std::vector<void*>& allocs, cudaStream_t st) {
  *d = nullptr;
  if (v.empty()) return CB_OK;
  int rc = dalloc((void**)d, sizeof(T) * v.size(), allocs);
  if (rc) return rc;
  CB_CUDA(cudaMemcpyAsync(*d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  return CB_OK;
}

}  // namespace cb
