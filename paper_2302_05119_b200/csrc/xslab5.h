// fp64 mode-2 MTTKRP for ranks > 16 (ALS compression default path), see
// xslab5.cu.
#pragma once
#include <cuda_runtime.h>

namespace cb {

struct Sl5Plan;

// fp32 blocks, I0 % 4 == 0, rank <= 64, A0 staging within shared memory
bool sl5_supported(int S, const void* const* X, const long long* dims, const int* R);
int sl5_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                    cudaStream_t st, Sl5Plan** out);
void sl5_plan_destroy(Sl5Plan* p);
// mtt[s] (device array of S pointers) <- M2 (I2 x R) of every active block
int sl5_mode2(Sl5Plan* p, const double* const* U_dev, const int* active, double* const* mtt,
              cudaStream_t st, const int* gate = nullptr);

// T = X x3 A2 of every active block as an fp64 GEMM (the ALS sweep's T pass),
// written unsplit into T buffer (*tsel) ^ t_other; available when
// sl5_tpass_ok (J % 4 == 0, rank > 8, A2 staging fits)
bool sl5_tpass_ok(const Sl5Plan* p);
int sl5_tpass(Sl5Plan* p, const double* const* U_dev, const int* active, void* const* T0,
              void* const* T1, const int* tsel, int t_other, cudaStream_t st);

}  // namespace cb
