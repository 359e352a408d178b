// Device-side state and kernel argument structs of the APG solver engine.
#pragma once
#include <vector>

#include "common.cuh"
#include "xpass.cuh"

namespace cb {

constexpr int MU_ROWS = 32;        // rows per mode-update CTA
constexpr int QR_MAXC = 128;       // R~ + R limit of the QR route

// Iteration state living in device memory; only the control kernel writes it.
struct State {
  int k;              // iteration being computed (1-based); 0 during init
  int go_main;        // 1 while not done (gates main-path kernels)
  int go_redo;        // 1 iff the current iteration restarts (gates redo kernels)
  int done;
  int reason;         // 0 max_iterations, 1 tolerance
  int n_restarts;
  int error, err_block, err_iter;
  int tsel, bsel;     // accepted T / b buffers
  int n_hist;         // history entries written (n_iter + 1)
  int rollback;       // pipelined lra: the stop came after a speculative sweep (undo it)
  double t_k;
  double w_hat;       // extrapolation weight of the current (main) sweep
  double rel_prev;    // RelErr of the last accepted iteration
  double obj_prev;    // objective_history[-1]
  double obj_pending; // lra: compressed objective of the accepted sweep
  unsigned long long t0_ns;
};

struct Ctx {
  int S, N, lra, update_core, objective, fast3, max_iter, rmax;
  int counts[CB_MAX_ORDER];
  double delta_w, tol;
  const long long* dims;      // S*N
  const int* R;               // S
  const int* Rt;              // S (lra)
  double* const* U;           // S*N current factors
  double* const* Up;          // S*N previous factors
  double* const* Un;          // S*N staging of the new individual columns
  double* const* G;           // S*N grams R x R
  double* const* C;           // S*N cross grams R~ x R (lra)
  double* const* Ut;          // S*N compression factors I_n x R~ (lra)
  double* const* LAM;         // S
  double* const* LAMP;        // S
  double* const* TW;          // S compression weights (lra)
  double* const* STEP;        // S step matrices of the current mode
  double* const* MTT;         // S MTTKRP outputs of the current mode (I_n x R)
  double* lipc_hist;          // S (NaN = unset)
  double* dbg;                // phase-time accumulators (profiling only) or null
  double* lipf_hist;          // N*S
  double* evec;               // S*(N+1)*64 warm eigenvectors (step matrices, core)
  int* evec_miss;             // S*(N+1) calls left before the warm path is retried
  int* fin_cnt;               // S arrival counters of k_finalize's roles (self-resetting)
  // Block sharding (one process per GPU, blocks [off, off+S) of S_tot).  Every
  // quantity that couples blocks lives in a GLOBAL-slot array indexed by the
  // global block number; a rank writes only its own slots into the *_w copy,
  // whose other slots stay zero, and an all-reduce (sum) of the *_w copy into
  // the read copy is then an exact all-gather.  Single GPU: *_w == read copy.
  int S_tot, off, shard;
  // Lipschitz constants, per mode n: lu at [n*2*S_tot + g], lup at
  // [n*2*S_tot + S_tot + g]  (lup = the "previous" constant used this sweep)
  double* lip;
  double* lip_w;
  double* ctl;                // 3*S_tot per-block evaluation terms
  double* ctl_w;
  double* nsq;                // S ||M_s||^2
  double* bbuf;               // 2 * S * RSTRIDE staged core linear terms
  double* model_sq;           // S lam^T (hadamard G) lam
  double* lam_snap;           // S * 64: lam of the iteration whose trace is in flight (pipelined lra)
  double* msq_snap;           // S: its model_sq
  double* inner;              // S (lra) lam^T (hadamard C)^T w~
  double* res_t;              // S (lra) compressed residual by expansion
  double* tsq;                // S (lra) ||M~||^2
  double* res;                // S explicit residuals (generic path)
  double* borig;              // S * RSTRIDE (generic lra trace / generic full b)
  double* gc_part;            // S_tot * gc_stride common-gradient partials (global slots)
  double* gc_w;
  double* cnew;             // I_n x L_n new common columns
  int* tile_cnt;              // per row tile arrival counters
  long long gc_stride;
  double* qr_buf;             // S*N*QR_MAXC*QR_MAXC R factors
  double* qr_part;            // S*qr_nchunks partial core sums
  int qr_nchunks;
  int mu_rows;                // rows per k_mode_update tile (MU_ROWS, or 64 for lra 3-way)
  int* qr_need;               // S flags: QR route taken this evaluation
  double* fib_bpart;          // per-block fiber totals: b (S x RSTRIDE)
  double* fib_rpart;          //   and explicit residual (S)
  const int* fib_first;       // S+1 unit ranges
  double* slab_part;
  const int* slab_first;      // S
  const int* slab_nchunk;     // S
  int slab_sb;
  State* st;
  double* h_obj;              // max_iter+1 histories
  double* h_orig;
  double* h_rel;
  double* h_tns;
  // graph-captured iterations: the restart branch is the body of a
  // conditional (IF) node that k_control switches on
  cudaGraphConditionalHandle cond;
  int use_cond;
  unsigned long long* tl;     // profiling only: iteration timeline (TlSlot)
  int b_mtt;                  // b from the last mode's MTTKRP in k_finalize (3-way row-dot path)
  // 3-way full path: the evaluation's per-block algebra (b, model_sq) and the
  // NEXT iteration's core Lipschitz constant run in k_eval_side beside the
  // fiber pass; k_sweep_begin then reads ldcore instead of a lambda_max
  int ld_pre;
  double* ldcore;             // S
  unsigned* gbar;             // grid-barrier counter of k_mode_fused (monotonic)
};

__host__ __device__ inline long long lu_idx(const Ctx& c, int n, int g) {
  return (long long)n * 2 * c.S_tot + g;
}
__host__ __device__ inline long long lup_idx(const Ctx& c, int n, int g) {
  return (long long)n * 2 * c.S_tot + c.S_tot + g;
}

}  // namespace cb
