// ALS compression passes of ranks > 16 on the tensor cores at fp64-grade
// accuracy (cpd_als.py:90-104): both tensor streams of a sweep,
//
//   T[r][j]  = sum_{i2} X[j + J i2] A2[i2, r]          (j = i0 + I0 i1)
//   D[r][m]  = sum_{i0} X[i0 + I0 m] A0[i0, r]         (m = i1 + I1 i2)
//
// as exact int8 slice GEMMs (tcgen05 kind::i8, int32 accumulators) over a
// block image that is packed ONCE per compression: X as four signed byte
// planes per form (30-bit fixed point, exact for fp32 values within 2^-6 of
// the block maximum), already in the MMA's shared-memory layout, so a pass
// is bulk copy -> MMA -> fp64 epilogue with no conversion work.  See xoz.cu.
#pragma once
#include <cuda_runtime.h>

namespace cb {

struct OzPlan;

// fp32 blocks of order 3, 16 < max rank <= 48, operand images within shared
// memory (I0, I2 <= ~670 at rank 40), rows < 2^31
bool oz_supported(int S, const void* const* X, const long long* dims, const int* R);
// allocates and packs the byte planes of both forms (enqueued on `st`);
// defer_pack: allocate only, the caller packs block ranges as their tensors
// arrive (oz_pack_range)
int oz_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                   cudaStream_t st, OzPlan** out, bool defer_pack = false);
int oz_pack_range(OzPlan* p, int lo, int hi, cudaStream_t st);
// load the passes' kernels now (a first launch beside copies in flight would
// wait for them: lazy module loading)
void oz_preload(const OzPlan* p);
void oz_plan_destroy(OzPlan* p);
// T = X x3 A2 of every active block, written unsplit ([R][J] fp64) into T
// buffer (*tsel) ^ t_other
int oz_tpass(OzPlan* p, const double* const* U_dev, const int* active, void* const* T0,
             void* const* T1, const int* tsel, int t_other, cudaStream_t st);
// mtt[s] (device array of S pointers) <- M2 (I2 x R) of every active block;
// UT_dev: optional transposed factors [r][I_n] (contiguous A1 columns)
int oz_mode2(OzPlan* p, const double* const* U_dev, const int* active, double* const* mtt,
             cudaStream_t st, const double* const* UT_dev = nullptr);
// bytes one pass streams (all blocks active)
double oz_pass_bytes(const OzPlan* p, int form);

}  // namespace cb
