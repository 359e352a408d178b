/*
 * concpd_b200 — C ABI of the B200-native CoNCPD-APG / lraCoNCPD-APG hot path.
 *
 * Drop-in boundary for the reference package `concpd` (arXiv 2302.05119,
 * /root/reference/pkg/src/concpd).  The reference is pure Python/numpy with no
 * FFI of its own; these entry points are what a ctypes binding inside the
 * reference would call.  Every function cites the
 * reference interface it replaces.
 *
 * Conventions
 *   - Tensors: dense, first-index-fastest (Fortran) order, fp32 or fp64
 *     (`cb_dtype`), device pointers owned by the caller
 *     (tensor_ops.py:1-15 layout convention).
 *   - Factor matrices: fp64, row-major I_n x R (numpy C order of an
 *     (I_n, R) array).  Gram / step matrices: fp64 row-major R x R.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Operator
 *     calls are asynchronous on that stream; engine calls synchronise only
 *     where documented.
 *   - Every call returns a cb_status; on failure cb_last_error() returns a
 *     thread-local message.  No global mutable state: handles are re-entrant
 *     per solve (the reference's bench runs solves from a thread pool,
 *     cli.py:277-282).
 *   - Nothing here falls back to the CPU.
 */
#ifndef CONCPD_B200_H
#define CONCPD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CB_ABI_VERSION 2   /* 2: cb_als_desc.ready_events, cb_als_staged_ok, cb_als_release_scratch */

typedef enum {
  CB_OK = 0,
  CB_ERR_ARG = 1,          /* invalid argument -> ValueError in the Python host      */
  CB_ERR_CUDA = 2,         /* CUDA runtime failure                                   */
  CB_ERR_NONFINITE = 3,    /* non-finite objective -> FloatingPointError (solver.py:523-527) */
  CB_ERR_UNSUPPORTED = 4,  /* shape outside the kernels' limits (rank > 64, order > 8)  */
  CB_ERR_DIVERGED = 5,     /* ALS non-finite grams -> ValueError (cpd_als.py:107-108)  */
  CB_ERR_STATE = 6         /* handle used out of order                               */
} cb_status;

typedef enum { CB_F32 = 0, CB_F64 = 1 } cb_dtype;

const char* cb_last_error(void);
int cb_abi_version(void);
/* number of this library's kernels launched by the calling thread since the
 * last reset (the bench's "gpu_launches" evidence). */
long long cb_launch_count(void);
void cb_launch_count_reset(void);

/* ------------------------------------------------------------------------
 * Operator level (device pointers in, device pointers out, async on stream)
 * ---------------------------------------------------------------------- */

/* out[I_mode x rank] = X_(mode) . KR_{-mode}; `factors` is a host array of
 * `order` device pointers.  Replaces solver.py:243-245 factor_linear_term
 * (and the matricize/factors_khatri_rao pair tensor_ops.py:45-54, 88-95). */
int cb_mttkrp(int dtype, const void* X, int order, const int64_t* dims,
              const double* const* factors, int rank, int mode, double* out,
              void* stream);

/* Batched core linear term b_s = (A0 (.) A1 (.) A2 of block s)^T vec(X_s) on the
 * tensor cores (tcgen05 kind::i8, exact int32 accumulation over byte-sliced
 * fixed-point operands, ~2^-20 relative per product, unbiased).  fp32 3-way
 * blocks (I0 % 4 == 0, I0 <= 512, rank <= 64); `tensors` and `factors` are
 * host arrays of device pointers (n_blocks and 3*n_blocks), `dims` is
 * n_blocks x 3, out is a device array of n_blocks x 64 doubles (row s holds
 * b_s[0..rank_s)).  Synchronous.  Replaces solver.py:215-218
 * core_linear_term (and the lra trace term solver.py:519-522). */
int cb_core_linear_term_tc(int n_blocks, const void* const* tensors, const int64_t* dims,
                           const double* const* factors, const int* ranks, double* out,
                           void* stream);

/* Khatri-Rao product of `nmats` row-major matrices (first slowest), out has
 * prod(rows) x rank entries.  Replaces tensor_ops.py:66-85 khatri_rao. */
int cb_khatri_rao(const double* const* mats, int nmats, const int64_t* rows, int rank,
                  double* out, void* stream);

/* out[ra x rb] = hadamard_{m != skip} mats[m]^T mats2[m] (mats2 NULL -> mats),
 * product taken in mode order; skip < 0 means none.
 * Replaces tensor_ops.py:98-124 hadamard_gram. */
int cb_hadamard_gram(const double* const* mats, const double* const* mats2,
                     const int64_t* rows, int nmodes, int skip, int ra, int rb,
                     double* out, void* stream);

/* out[b] = max(lambda_max(g_b), 0), 0 for an all-zero matrix; g is batch x r x r,
 * r <= 64.  Replaces tensor_ops.py:127-140 spectral_norm (LAPACK syevd). */
int cb_spectral_norm_batched(const double* g, int r, int batch, double* out, void* stream);

/* out3 = {sum of squares, min value, count of non-finite values} of X[0:n] in
 * fp64.  Feeds CoupledProblem.validate (solver.py:114-117) and ||M||^2
 * (solver.py:327). */
int cb_tensor_stats(int dtype, const void* X, int64_t n, double* out3, void* stream);

/* *out = || X - [[weights; factors]] ||_F^2 by an explicit streaming residual.
 * Replaces the residual of solver.py:194-202 objective(). */
int cb_kruskal_residual(int dtype, const void* X, int order, const int64_t* dims,
                        const double* const* factors, const double* weights, int rank,
                        double* out, void* stream);

/* out[r] = sum_i a[i,r] * b[i,r]  (einsum "ir,ir->r", solver.py:218, :507-511). */
int cb_rowdot(const double* a, const double* b, int64_t rows, int r, double* out,
              void* stream);

/* C = alpha * op(A) op(B) + beta * C, fp64 row-major, small shapes.  Used by
 * the operator-level lra linear terms and gradients (solver.py:205-251). */
int cb_gemm(int trans_a, int trans_b, int m, int n, int k, double alpha, const double* a,
            int lda, const double* b, int ldb, double beta, double* c, int ldc,
            void* stream);

/* out = u_hat (gram_skip o lam lam^T) - mtt o lam  (solver.py:232-240). */
int cb_factor_gradient(const double* u_hat, int64_t rows, const double* gram_skip,
                       const double* mtt, const double* lam, int r, double* out,
                       void* stream);

/* ------------------------------------------------------------------------
 * Seeded synthetic blocks on the device (the input pipeline).
 * X = [[weights; factors]] (weights NULL = ones), fp64 arithmetic, written
 * first-index-fastest.  Replaces the O(|M| R) part of synth.generate
 * (synth.py:77-112: reconstruct, kruskal.py:112-119) and add_noise
 * (metrics.py:207-223); the factors are drawn by the caller (numpy, the
 * reference's SeedSequence children).
 * ---------------------------------------------------------------------- */

/* out2 (device, 2 doubles) = {sum of x^2, max x} of the clean block
 * (add_noise's signal power mean(X^2) = out2[0] / |M|, metrics.py:218). */
int cb_synth_stats(int order, const int64_t* dims, const double* const* factors,
                   const double* weights, int rank, double* out2, void* stream);

/* out = noise(scale * X): noise 0 none; 1 + sigma z then clip at 0
 * (metrics.py:220-221); 2 + sigma z then clip to [0, 1]; 3 * exp(sigma z).
 * z: standard normals from Philox4x32-10 keyed by `seed`, counter = (element
 * index, block), so a block does not depend on launch shape or block order. */
int cb_synth_fill(int dtype, void* out, int order, const int64_t* dims,
                  const double* const* factors, const double* weights, int rank, double scale,
                  int noise, double sigma, uint64_t seed, int block, void* stream);

/* ------------------------------------------------------------------------
 * Post-solve metrics on the device (metrics.py:71-156).
 * ---------------------------------------------------------------------- */

/* out2 (device) = {||X - [[weights; factors]]||^2, ||X||^2}: rel_err / psnr of
 * a Kruskal model without forming it (metrics.py:51-81, :140-156). */
int cb_model_residual(int dtype, const void* X, int order, const int64_t* dims,
                      const double* const* factors, const double* weights, int rank,
                      double* out2, void* stream);

/* out2 (device) = {||A - B||^2, ||A||^2} of two dense buffers of n elements
 * (rel_err / psnr of a dense reconstruction). */
int cb_diff_sq(int dtype_a, const void* A, int dtype_b, const void* B, int64_t n, double* out2,
               void* stream);

/* Performance index of n_pairs (estimate, truth) factor pairs (device,
 * row-major rows[p] x rank, rank >= 2): out[p] (device) as in
 * performance_index (metrics.py:84-124) with pinv(E) T = (E^T E)^{-1} E^T T;
 * deficient[p] (device) = 1 where E looks rank-deficient (the reference's
 * warning). */
int cb_performance_index(int n_pairs, const double* const* estimated, const double* const* truth,
                         const int64_t* rows, int rank, double* out, int* deficient,
                         void* stream);

/* ------------------------------------------------------------------------
 * CP-ALS compression engine (cpd_als.py:52-120), batched over blocks.
 * Each block is an independent ALS fit with its own stop rule.
 * ---------------------------------------------------------------------- */
typedef struct cb_als cb_als;

typedef struct {
  int n_blocks;
  int order;                      /* <= 8                                   */
  const int64_t* dims;            /* host, n_blocks*order                   */
  const int* ranks;               /* host, n_blocks (<= 64)                 */
  int dtype;                      /* cb_dtype of the tensors                */
  const void* const* tensors;     /* host array of device pointers          */
  const double* const* init;      /* host array (n_blocks*order) of host
                                     I_n x R row-major initial factors      */
  double tol;                     /* AlsOptions.tol                         */
  int max_iter;                   /* AlsOptions.max_iter                    */
  int compute;                    /* fp32 storage only: 0 (and 2) = fp64-grade
                                     arithmetic in the tensor passes (3-way
                                     blocks of ranks in (16, 48]: exact int8
                                     slice GEMMs on the tensor cores over
                                     byte planes packed once, csrc/xoz.cu;
                                     else fp64 FMAs), 1 = fp32 arithmetic   */
  int total_blocks;               /* blocks of the whole (sharded) problem;
                                     fixes each block's work decomposition so
                                     a shard reproduces the unsharded bits
                                     (0 = n_blocks)                          */
  const void* const* ready_events; /* optional, host array of n_blocks
                                     cudaEvent_t in block order: tensors[s] may
                                     be read once ready_events[s] has completed
                                     (its upload is still in flight on another
                                     stream).  cb_als_run then starts each
                                     block's compression as it arrives, beside
                                     the remaining uploads (blocks are fitted
                                     independently: same results).  Only for
                                     blocks cb_als_staged_ok accepts
                                     (CB_ERR_UNSUPPORTED otherwise, also when
                                     the plan's memory cannot be allocated:
                                     create again without events once the
                                     uploads are done).  NULL: the tensors
                                     are ready in stream order               */
} cb_als_desc;

int cb_als_create(const cb_als_desc* desc, void* stream, cb_als** out);
/* frees the sweep workspace (byte planes, GEMM scratch) once cb_als_run has
 * finished; results and device factors stay valid, the handle cannot run
 * again */
int cb_als_release_scratch(cb_als* h);
/* 1 if cb_als_create would start these blocks one by one at their
 * ready_events (only then may the events be recorded after the create: the
 * engine reads no tensor before cb_als_run); needs dims, ranks, dtype,
 * compute, total_blocks only */
int cb_als_staged_ok(const cb_als_desc* desc);
/* runs every block to convergence or max_iter; synchronises the stream */
int cb_als_run(cb_als* h);
/* per block: rel_err, n_iter, converged flag, and the rel-err history
 * (history capacity max_iter doubles); factors copied to host row-major. */
int cb_als_block_result(cb_als* h, int block, double* rel_err, int* n_iter, int* converged,
                        double* history, double* const* host_factors);
/* device pointer of the fitted factor (block, mode), valid until destroy */
const double* cb_als_factor_device(cb_als* h, int block, int mode);
int cb_als_destroy(cb_als* h);

/* ------------------------------------------------------------------------
 * APG solver engine (solver.py:546-624 with the _Apg state machine
 * solver.py:311-543), device-resident: sweep, evaluation, restart rule and
 * stop rule all run on the GPU; the host only launches and polls a flag.
 * ---------------------------------------------------------------------- */
typedef struct cb_solver cb_solver;

typedef struct {
  int n_blocks;                   /* blocks owned by this process            */
  int order;
  const int64_t* dims;            /* host, n_blocks*order                    */
  const int* ranks;               /* host, n_blocks                          */
  const int* coupled;             /* host, order (L_n)                       */
  int lra;                        /* 0 = CoNCPD-APG, 1 = lraCoNCPD-APG       */
  int update_core;                /* 0 = fixed-core variant                  */
  int dtype;                      /* tensor storage dtype                    */
  const void* const* tensors;     /* host array of device pointers           */
  const double* const* init_factors;  /* host (n_blocks*order) host arrays   */
  const double* const* init_weights;  /* host (n_blocks) host arrays         */
  const int* tilde_ranks;             /* lra: host, n_blocks                 */
  const double* const* tilde_factors; /* lra: host array of DEVICE pointers  */
  const double* const* tilde_weights; /* lra: host array of HOST arrays      */
  int objective;                  /* 0 = explicit residual, 1 = gram expansion */
  int compute;                    /* fp32 storage only: 0 = fp64 arithmetic in
                                     the tensor passes, 1 = fp32 arithmetic,
                                     2 = fp64 arithmetic except the lra trace
                                     pass, which runs on the tensor cores
                                     (cb_core_linear_term_tc's algorithm)     */
  double delta_w;
  double tol;
  int max_iter;
  /* multi-GPU block sharding (world_size 1: all NULL/0).  Each rank owns the
   * contiguous blocks [block_offset, block_offset + n_blocks) of
   * total_blocks; the per-mode Lipschitz sums, common-column gradient
   * partials and per-block evaluation terms are all-reduced (solver.py:422-451,
   * :593-610).  nccl_comm NULL with world_size > 1: one rank of an emulated
   * group on one GPU, driven by cb_group_step / cb_group_run. */
  int world_size;
  int rank_id;
  void* nccl_comm;                /* ncclComm_t created by cb_nccl_comm_init */
  int total_blocks;               /* S over all ranks                        */
  int block_offset;               /* global index of this rank's first block */
  /* lra with the tensor-core trace pass: iteration k's trace pass streams
   * beside iteration k+1's sweep (results bitwise those of the serial order).
   * 0 = auto (on when the trace pass streams >= 64 MB), 1 = on, 2 = off. */
  int pipeline;
  /* SMs the pipelined trace pass leaves to the sweep beside it (0 = auto,
   * ceil(S / 3), at most a third of the SMs) */
  int pipeline_reserve;
} cb_solver_desc;

typedef struct {
  int n_iter;
  int n_restarts;
  int done;
  int reason;                     /* 0 max_iterations, 1 tolerance           */
  int error;                      /* 0 ok, CB_ERR_NONFINITE                  */
  int error_block;
  int error_iter;
} cb_solver_summary;

int cb_solver_create(const cb_solver_desc* desc, void* stream, cb_solver** out);
/* run up to `iters` more iterations (device stops early at tolerance);
 * synchronises and reports the summary. */
int cb_solver_run(cb_solver* h, int iters, cb_solver_summary* summary);
/* enqueue exactly one APG iteration (sweep, evaluation, restart rule, stop
 * rule) without synchronising: the bench's timed step. */
int cb_solver_step_async(cb_solver* h);
int cb_solver_summary_get(cb_solver* h, cb_solver_summary* summary);
/* per accepted iteration 0..n_iter: internal objective, original-tensor
 * objective, RelErr, device timestamp (ns) */
int cb_solver_history(cb_solver* h, double* obj_int, double* obj_orig, double* rel,
                      double* t_ns, int cap);
int cb_solver_block_factors(cb_solver* h, int block, double* const* host_factors,
                            double* host_weights);
/* CUDA-event timing of the tensor-streaming kernels (events on the solve
 * stream around every launch): on/off, and per kind (0 = all, 1 = fiber pass,
 * 2 = slab pass) the accumulated milliseconds, launches and algorithmic bytes. */
int cb_solver_set_timing(cb_solver* h, int on);
/* per-launch profile of whole iterations (events after every launch, no CUDA
 * graph while on): on=1 starts, on=0 stops and writes "label count ms" lines */
int cb_solver_profile(cb_solver* h, int on, char* out, int cap);
int cb_solver_timing(cb_solver* h, int kind, double* ms, long long* launches, double* bytes);
/* iteration timeline (profiling): op 1 enables (re-captures the iteration
 * graph with in-kernel timestamps) and resets, 2 resets, 0 synchronises and
 * copies per kernel slot {earliest CTA start, latest CTA end} (globaltimer
 * ns, 2*24 entries; slot ids in csrc/xpass.cuh TlSlot), -1 disables. */
int cb_solver_timeline(cb_solver* h, int op, unsigned long long* out, int cap);
int cb_solver_destroy(cb_solver* h);

/* Emulated shard group: the handles of ranks 0..n-1 (created with
 * world_size n, nccl_comm NULL, on ONE stream) run the sharded program one
 * segment at a time with the exchanges done by a summing kernel between
 * segments — the multi-GPU code path verified on a single GPU.
 * program 0 = iteration-0 evaluation, 1 = one APG iteration. */
#define CB_MAX_GROUP 16
int cb_group_step(cb_solver* const* handles, int n, int program);
int cb_group_run(cb_solver* const* handles, int n, int iters, cb_solver_summary* summary);

/* NCCL communicator for the block-sharded multi-GPU path. `unique_id` is the
 * 128-byte ncclUniqueId produced on rank 0 (cb_nccl_unique_id) and broadcast
 * by the caller (torch.distributed). */
int cb_nccl_unique_id(void* out128);
int cb_nccl_comm_init(const void* unique_id128, int world_size, int rank, void** comm);
int cb_nccl_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* CONCPD_B200_H */
