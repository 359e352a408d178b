// Internal (non-ABI) declarations shared between ops.cu and engine.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace cb {

struct KrArgs {
  const double* mats[CB_MAX_ORDER];
  int64_t rows[CB_MAX_ORDER];
  int nmats;
  int rank;
};

struct MttJob {
  const void* X;
  int64_t L, In, H;
  const double* KRl;
  const double* KRh;
  double* out;
  int R;
};

struct HgArgs {
  const double* A[CB_MAX_ORDER];
  const double* B[CB_MAX_ORDER];
  int64_t rows[CB_MAX_ORDER];
  int nmodes, skip, ra, rb;
};

struct ResidArgs {
  const double* U[CB_MAX_ORDER];
  const double* w;
  int64_t dims[CB_MAX_ORDER];
  int64_t n;
  int order, R;
};

void count_launch(long long n);
int launch_kr_first_fastest(const KrArgs& a, double* out, cudaStream_t st);
int launch_mttkrp_generic(int dtype, const MttJob& j, cudaStream_t st);
int mttkrp_one(int dtype, const void* X, int order, const int64_t* dims,
               const double* const* factors, int rank, int mode, double* out,
               double* scratch, cudaStream_t st);
int tensor_stats(int dtype, const void* X, int64_t n, double* out3, double* part, int nparts,
                 cudaStream_t st);
void tensor_stats_preload();
int kruskal_residual(int dtype, const ResidArgs& a, const void* X, double* out, double* part,
                     int nparts, cudaStream_t st);
size_t lam_max_smem_bytes(int R);

}  // namespace cb
