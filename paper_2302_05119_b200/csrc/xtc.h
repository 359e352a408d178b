// Tensor-core trace pass (tcgen05 kind::i8, exact int32 accumulation over
// byte-sliced fixed-point operands) for 3-way fp32 blocks:
//
//   b_s[r] = sum_{i0,i1,i2} X_s[i0,i1,i2] A0[i0,r] A1[i1,r] A2[i2,r]
//
// the core linear term of the reference (`solver.py:215-218`, staged at
// `:506-511`) and the lra original-tensor trace term (`solver.py:519-522`).
// See xtc.cu for the algorithm and DESIGN.md §5 for the roofline.
#pragma once
#include <cuda_runtime.h>

#include "xpass.cuh"

namespace cb {

struct XtcPlan;

// usable for these blocks?  fp32 storage, I0 <= 512, I1 >= 16, rank <= 40
// (three byte levels of a column stacked along the MMA's M = 128)
bool xtc_supported(int S, const void* const* X, const long long* dims, const int* R);

// plan for S blocks (device fp32 tensors X[s], dims S x 3, ranks R[s]):
// unit tables, the per-block fixed-point exponent of X (one max|X| pass) and
// the three byte planes of every block (one pack pass), enqueued on `st`;
// operand images and partial buffers
int xtc_plan_create(int S, const void* const* X, const long long* dims, const int* R,
                    cudaStream_t st, XtcPlan** out);
void xtc_plan_destroy(XtcPlan* p);

// b_s into bsum[s * RSTRIDE + r] (r < R[s]); factors from U (device array of
// S*3 pointers, the engine's XArgs.U), skipped when *gate == 0 (gate may be
// null).  Two launches: operand prep + the streaming MMA kernel.
// parts: 1 = operand prep only (snapshots the factors), 2 = the streaming
// pass only (reads only the prepared operands), 3 = both.  The operands
// exist twice: with other = 1 the prep writes the set the trace is NOT
// reading (the pipelined iteration prepares trace k+1 while trace k streams);
// xtc_flip then makes that set current.
int xtc_trace(XtcPlan* p, const double* const* U_dev, const int* gate, double* bsum,
              cudaStream_t st, int parts = 3, int other = 0);
int xtc_flip(XtcPlan* p, const int* gate, cudaStream_t st);

// cap the streaming kernel's persistent grid (0: one CTA per SM), leaving
// SMs to work that runs beside it (the pipelined lra sweep)
void xtc_set_grid_cap(XtcPlan* p, int cap);
// per-launch timeline slots (TL_TRACE, TL_PREP) of the solver's profiling mode
void xtc_set_timeline(XtcPlan* p, unsigned long long* tl);

// algorithmic bytes of one xtc_trace call (sum_s |X_s| * 4: every element of
// the fp32 blocks once) and the bytes it actually streams (three byte planes
// per element plus tile padding)
double xtc_bytes(const XtcPlan* p);
double xtc_stream_bytes(const XtcPlan* p);

}  // namespace cb
