// APG solver engine: host orchestration + C ABI (cb_solver_*).
//
// Mirrors solve() (pkg/src/concpd/solver.py:546-624).  The whole iteration —
// core update, N mode updates with common-column aggregation, evaluation,
// restart branch and stop rule — is enqueued without host round trips; for
// the 3-way fast path one iteration is captured once in a CUDA graph and
// replayed.  The host polls the device `done` flag every few iterations.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "engine_kernels.cuh"
#include "ops_internal.h"
#include "status.h"
#include "engine_host.h"
#include "launch.cuh"
#include "nccl_shim.h"
#include "xtc.h"

namespace cb {


static thread_local cudaStream_t g_alloc_stream = nullptr;

// Small buffers (an engine has thousands: per-block factors, grams, tables)
// are carved from 32 MB chunks, one cudaMalloc + one memset per chunk instead
// of one per buffer (c5: ~0.25 s of host time per solve); the chunk belongs
// to the handle whose `allocs` it was pushed to and is freed with it.
static thread_local struct {
  std::vector<void*>* owner;
  char* base;
  size_t off, cap;
} g_chunk = {nullptr, nullptr, 0, 0};

constexpr size_t DALLOC_CHUNK = 32u << 20;
constexpr size_t DALLOC_SMALL = 2u << 20;

int dalloc(void** p, size_t bytes, std::vector<void*>& allocs) {
  *p = nullptr;
  if (bytes == 0) bytes = 8;
  if (bytes <= DALLOC_SMALL) {
    const size_t need = (bytes + 255) & ~(size_t)255;
    if (g_chunk.owner != &allocs || g_chunk.off + need > g_chunk.cap) {
      void* base = nullptr;
      CB_CUDA(cudaMalloc(&base, DALLOC_CHUNK));
      allocs.push_back(base);
      CB_CUDA(cudaMemsetAsync(base, 0, DALLOC_CHUNK, g_alloc_stream));
      g_chunk.owner = &allocs;
      g_chunk.base = static_cast<char*>(base);
      g_chunk.off = 0;
      g_chunk.cap = DALLOC_CHUNK;
    }
    *p = g_chunk.base + g_chunk.off;
    g_chunk.off += need;
    return CB_OK;
  }
  CB_CUDA(cudaMalloc(p, bytes));
  allocs.push_back(*p);
  CB_CUDA(cudaMemsetAsync(*p, 0, bytes, g_alloc_stream));
  return CB_OK;
}

// frees a handle's buffers (and forgets its chunk: a later handle's `allocs`
// may live at the same address)
void dfree_all(std::vector<void*>& allocs) {
  for (void* p : allocs) cudaFree(p);
  allocs.clear();
  if (g_chunk.owner == &allocs) g_chunk.owner = nullptr;
}

void set_alloc_stream(cudaStream_t st) {
  g_alloc_stream = st;
  g_chunk.owner = nullptr;
}

}  // namespace cb

using namespace cb;

struct cb_solver {
  cudaStream_t st = nullptr;
  bool redo_reprep = false;   // pipelined lra: the restart branch re-prepares the trace operands
  // side stream of the 3-way full path: the MTTKRP of mode n runs on it
  // concurrently with mode n's step matrix / lambda_max on `st` (fork/join by
  // events, captured as parallel graph branches)
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t st3 = nullptr;     // capture stream of the conditional restart body
  cudaStream_t st_main = nullptr; // the iteration's stream while a body is captured
  bool cond_capture = false;
  bool in_body = false;
  int S = 0, N = 0, lra = 0, update_core = 1, dtype = CB_F64, objective = 0, fast3 = 0, pc = 0;
  int rmax = 1, rtmax = 0, rb = 8, max_iter = 0;
  double delta_w = 0.9999, tol = 1e-8;
  std::vector<long long> dims;
  std::vector<int> R, Rt;
  int counts[CB_MAX_ORDER] = {0};
  std::vector<const void*> X;
  std::vector<void*> allocs;
  Ctx ctx{};
  XArgs xa_main{}, xa_redo{};
  XTables tab;
  FibUnit* d_fib = nullptr;
  SlabUnit* d_slab = nullptr;
  RowUnit *d_c0 = nullptr, *d_c1 = nullptr;
  std::vector<RowUnit*> d_rows;
  std::vector<int> n_rows;
  State* d_state = nullptr;
  State* h_state = nullptr;     // pinned mirror
  size_t blk_smem = 0, mu_smem = 0, qr_smem = 0, qrc_smem = 0;
  size_t blk_smem_ng = 0;      // per-block kernels without gram staging
  int qr_ch = 32;             // TSQR chunk rows (k_qr_factor)
  bool qr_core3 = false;      // 3-way GEMM-form ||core||^2 (k_qr_core3)
  int qrc_ct = 8;             // its columns per thread
  std::vector<double*> h_U;     // device pointer tables mirrored on host
  std::vector<double*> h_MTT;
  std::vector<double*> h_LAM;
  long long launches_per_iter = 0;
  double* kr_scratch = nullptr; // generic path
  double* res_part = nullptr;
  int res_nparts = 0;
  cudaGraphExec_t gexec = nullptr;
  bool graph_ok = true;
  bool timing = false;
  bool profile = false;
  bool tma = false;             // bulk-copy streaming path usable
  std::vector<cudaEvent_t> mpool;
  std::vector<const char*> mlabels;
  size_t mused = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;     // per event pair: 1 fiber, 2 slab
  size_t ev_used = 0;
  double t_ms = 0.0, t_bytes = 0.0;
  long long t_launches = 0;
  long long elem_total = 0;
  int elem_bytes = 8;
  int iters_enqueued = 0;
  bool init_done = false;
  // ---- block sharding (see Ctx::S_tot).  With an NCCL communicator the
  // exchanges are all-reduces enqueued in stream order (and captured in the
  // iteration graph).  Without one (world > 1, comm null) the handle is one
  // rank of an EMULATED group driven by cb_group_step: every handle of the
  // group enqueues the program one segment at a time on the same stream and
  // the exchanges between segments are done by k_xsum.
  // shard: the sharded program (exchanges, separate send copies) runs; also
  // with world 1 when a communicator is given (the NCCL path on one GPU)
  int world = 1, rank = 0, S_tot = 0, off = 0, shard = 0;
  void* comm = nullptr;
  int seg_cur = 0, seg_want = -1;   // -1: emit everything; -2: count segments
  struct Xchg { double* send; double* recv; long long count; };
  std::vector<Xchg> pending;
  cb::XtcPlan* xtc = nullptr;  // tensor-core lra trace pass (compute code 2)
  // pipelined lra (single GPU, tensor-core trace): the trace pass of
  // iteration k streams beside the sweep of k+1 (see enqueue_pipe_step)
  bool pipe = false;
  bool pipe_pending = false;     // an iteration's trace + FINISH not yet enqueued
  cudaGraphExec_t gexec_pipe = nullptr;
  long long launches_per_pipe = 0;
};

namespace cb {

// does the current program position belong to the segment being enqueued?
static inline bool emit(const cb_solver* h) {
  return h->seg_want == -1 || h->seg_cur == h->seg_want;
}

static int begin_cond_body(cb_solver* h);
static int end_cond_body(cb_solver* h);

// exchange point: recv <- sum over ranks of send (count doubles); closes the
// current segment.  Inside a captured conditional restart body the NCCL call
// is issued in the parent graph between two bodies (collectives stay out of
// conditional nodes; every rank runs the same graph).  There it also runs
// when no restart happens: the send buffers are then unchanged since their
// last exchange, so the all-reduce rewrites recv with the values it holds.
static int xchg(cb_solver* h, double* send, double* recv, long long count) {
  if (!h->shard) return CB_OK;
  if (h->comm) {
    if (emit(h)) {
      const bool split = h->in_body && h->cond_capture;
      int rc;
      if (split && (rc = end_cond_body(h))) return rc;
      NcclApi& api = nccl_api();
      ncclResult_t r = api.ncclAllReduce(send, recv, (size_t)count, ncclFloat64, ncclSum,
                                         (ncclComm_t)h->comm, h->st);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
      if (split && (rc = begin_cond_body(h))) return rc;
    }
  } else if (h->seg_cur == h->seg_want) {
    h->pending.push_back(cb_solver::Xchg{send, recv, count});
  }
  h->seg_cur += 1;
  return CB_OK;
}

// the Lipschitz constants of mode n (before its mode update), the common
// gradient partials of mode n (after it), the per-block evaluation terms
static int xchg_lip(cb_solver* h, int n) {
  if (!h->shard || h->counts[n] == 0) return CB_OK;
  const long long o = lu_idx(h->ctx, n, 0);
  return xchg(h, h->ctx.lip_w + o, h->ctx.lip + o, 2LL * h->S_tot);
}
static int xchg_gc(cb_solver* h, int n) {
  if (!h->shard || h->counts[n] == 0) return CB_OK;
  // equal shards over NCCL: an all-gather of each rank's own contiguous
  // slot range (half the traffic of the all-reduce with zero foreign slots,
  // same result); otherwise the all-reduce
  if (h->comm && h->S_tot == h->S * h->world) {
    if (emit(h)) {
      const bool split = h->in_body && h->cond_capture;
      int rc;
      if (split && (rc = end_cond_body(h))) return rc;
      const long long cnt = (long long)h->S * h->ctx.gc_stride;
      NcclApi& api = nccl_api();
      ncclResult_t r = api.ncclAllGather(h->ctx.gc_w + (long long)h->off * h->ctx.gc_stride,
                                         h->ctx.gc_part, (size_t)cnt, ncclFloat64,
                                         (ncclComm_t)h->comm, h->st);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
      if (split && (rc = begin_cond_body(h))) return rc;
    }
    h->seg_cur += 1;
    return CB_OK;
  }
  return xchg(h, h->ctx.gc_w, h->ctx.gc_part, (long long)h->S_tot * h->ctx.gc_stride);
}

// profiling marks: an event after every launch of the iteration; the interval
// ending at a mark is charged to that mark's label (kernel time + launch gap)
static void prof(cb_solver* h, const char* label) {
  if (!h->profile || !emit(h)) return;
  if (h->mused >= h->mpool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    h->mpool.push_back(e);
  }
  cudaEvent_t e = h->mpool[h->mused++];
  cudaEventRecord(e, h->st);
  h->mlabels.push_back(label);
}

static int ev_pair(cb_solver* h, cudaEvent_t* a, cudaEvent_t* b, int kind) {
  h->ev_kind.push_back(kind);
  while (h->ev_pool.size() < h->ev_used + 2) {
    cudaEvent_t e;
    CB_CUDA(cudaEventCreate(&e));
    h->ev_pool.push_back(e);
  }
  *a = h->ev_pool[h->ev_used];
  *b = h->ev_pool[h->ev_used + 1];
  h->ev_used += 2;
  return CB_OK;
}

// stream the blocks once through the fiber kernel (optionally timed)
// timing mode brackets main-path launches only: the restart-branch copies are
// gated no-ops unless a restart happens and would dilute the average
static int enqueue_fiber(cb_solver* h, const XArgs& a, int want_t, int want_b, int want_res) {
  if (!emit(h)) return CB_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = h->timing && a.gate != &h->d_state->go_redo;
  if (timed) { int rc = ev_pair(h, &e0, &e1, 1); if (rc) return rc; CB_CUDA(cudaEventRecord(e0, h->st)); }
  launch_fiber(h->pc, h->rb, h->tma, want_t, want_b, want_res, a, h->d_fib, (int)h->tab.fib.size(),
               h->tab, h->st);
  CB_CHECK_LAUNCH();
  if (timed) { CB_CUDA(cudaEventRecord(e1, h->st)); h->t_launches += 1; h->t_bytes += (double)h->elem_total * h->elem_bytes; }
  return CB_OK;
}

static int enqueue_slab(cb_solver* h, const XArgs& a, cudaStream_t st) {
  if (!emit(h)) return CB_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = h->timing && a.gate != &h->d_state->go_redo;
  if (timed) { int rc = ev_pair(h, &e0, &e1, 2); if (rc) return rc; CB_CUDA(cudaEventRecord(e0, st)); }
  launch_slab(h->pc, h->rb, h->tma, a, h->d_slab, (int)h->tab.slab.size(), h->tab, st);
  CB_CHECK_LAUNCH();
  if (timed) { CB_CUDA(cudaEventRecord(e1, st)); h->t_launches += 1; h->t_bytes += (double)h->elem_total * h->elem_bytes; }
  return CB_OK;
}

// side-stream fork / join (no-ops outside the emitted segment)
static int fork_side(cb_solver* h) {
  if (!emit(h)) return CB_OK;
  CB_CUDA(cudaEventRecord(h->ev_fork, h->st));
  CB_CUDA(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  return CB_OK;
}
static int join_side(cb_solver* h) {
  if (!emit(h)) return CB_OK;
  CB_CUDA(cudaEventRecord(h->ev_join, h->st2));
  CB_CUDA(cudaStreamWaitEvent(h->st, h->ev_join, 0));
  return CB_OK;
}

// MTTKRP of mode n of the 3-way full path (contract from T, or the slab pass)
static int enqueue_mttkrp3(cb_solver* h, int n, const XArgs& xa, int redo, cudaStream_t st) {
  if (n < 2) {
    if (emit(h)) {
      launch_contract(h->pc, n, xa, n == 0 ? h->d_c0 : h->d_c1,
                      (int)(n == 0 ? h->tab.c0.size() : h->tab.c1.size()), st);
      CB_CHECK_LAUNCH();
    }
    prof(h, redo ? "redo:contract" : (n == 0 ? "contract0" : "contract1"));
    return CB_OK;
  }
  int rc = enqueue_slab(h, xa, st);
  prof(h, redo ? "redo:slab" : "slab");
  return rc;
}

// generic-order helpers (per-block launches, host-driven restart)
static int generic_mttkrp(cb_solver* h, int s, int n) {
  std::vector<const double*> f(h->N);
  for (int m = 0; m < h->N; ++m) f[m] = h->h_U[s * h->N + m];
  return mttkrp_one(h->dtype, h->X[s], h->N, reinterpret_cast<const int64_t*>(&h->dims[s * h->N]), f.data(), h->R[s], n,
                    h->h_MTT[s], h->kr_scratch, h->st);
}

static int generic_rowdot_into(cb_solver* h, int s, int n, double* out);
static int generic_residuals(cb_solver* h);

// one sweep (solver.py:459-463); redo = restart sweep with w_hat = 0.
// 3-way full path: mode n's MTTKRP (side stream) overlaps mode n's step
// matrix + lambda_max (k_sweep_begin for n = 0, k_step otherwise).
static int enqueue_sweep(cb_solver* h, int redo) {
  cudaStream_t st = h->st;
  const XArgs& xa = redo ? h->xa_redo : h->xa_main;
  // no side stream inside the conditional restart body (rarely executed; keeps
  // that capture single-stream)
  const bool par = h->fast3 && !h->lra && !h->in_body;
  int rc;
  if (par) {
    if ((rc = fork_side(h))) return rc;
    if ((rc = enqueue_mttkrp3(h, 0, xa, redo, h->st2))) return rc;
  }
  if (emit(h)) {
    launch_k(k_sweep_begin, dim3(h->S), dim3(256), h->blk_smem_ng, st, h->ctx, redo);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  prof(h, redo ? "redo:sweep_begin" : "sweep_begin");
  if (par && (rc = join_side(h))) return rc;
  if ((rc = xchg_lip(h, 0))) return rc;
  for (int n = 0; n < h->N; ++n) {
    int src = 0;
    if (h->lra) {
      src = 2;
    } else if (h->fast3) {
      src = (n < 2 || h->tab.slab_direct) ? 0 : 1;
      // overlapped runs enqueued this MTTKRP on the side stream already
      if (!par && (rc = enqueue_mttkrp3(h, n, xa, redo, st))) return rc;
    } else {
      for (int s = 0; s < h->S; ++s) {
        if ((rc = generic_mttkrp(h, s, n))) return rc;
      }
      prof(h, "generic_mttkrp");
    }
    const bool split = par && n + 1 < h->N;
    if (emit(h)) {
      launch_k(k_mode_update, dim3(h->n_rows[n]), dim3(256), h->mu_smem, st, h->ctx, n, redo, src, h->d_rows[n]);
      count_launch(1);
      CB_CHECK_LAUNCH();
    }
    prof(h, redo ? "redo:mode_update" : "mode_update");
    if (h->shard && h->counts[n] > 0) {
      if ((rc = xchg_gc(h, n))) return rc;
      if (emit(h)) {
        const int tiles = (int)((h->dims[n] + MU_ROWS - 1) / MU_ROWS);
        launch_k(k_common, dim3(tiles), dim3(256), 0, st, h->ctx, n, redo);
        count_launch(1);
        CB_CHECK_LAUNCH();
      }
      prof(h, redo ? "redo:common" : "common");
    }
    if (emit(h)) {
      launch_k(k_finalize, dim3(h->S, h->lra ? 3 : 2), dim3(256), h->blk_smem, st, h->ctx, n, redo,
               split ? 0 : 1);
      count_launch(1);
      CB_CHECK_LAUNCH();
    }
    prof(h, redo ? "redo:finalize" : "finalize");
    if (split) {
      if ((rc = fork_side(h))) return rc;
      if ((rc = enqueue_mttkrp3(h, n + 1, xa, redo, h->st2))) return rc;
      if (emit(h)) {
        launch_k(k_step, dim3(h->S), dim3(256), h->blk_smem_ng, st, h->ctx, n + 1, redo);
        count_launch(1);
        CB_CHECK_LAUNCH();
      }
      prof(h, redo ? "redo:step" : "step");
      if ((rc = join_side(h))) return rc;
    }
    if (n + 1 < h->N && (rc = xchg_lip(h, n + 1))) return rc;
  }
  return CB_OK;
}

static int enqueue_qr(cb_solver* h, int redo) {
  if (!emit(h)) return CB_OK;
  launch_k(k_qr_factor, dim3(h->S * h->N), dim3(QR_THREADS), h->qr_smem, h->st, h->ctx, redo,
           h->qr_ch);
  prof(h, redo ? "redo:qr_factor" : "qr_factor");
  if (h->qr_core3) {
    // columns per thread: ceil(K2 / 16) rounded to the instantiated tiles
    const dim3 g(h->S * h->ctx.qr_nchunks);
    if (h->qrc_ct <= 2) launch_k(k_qr_core3<2>, g, dim3(256), h->qrc_smem, h->st, h->ctx, redo);
    else if (h->qrc_ct <= 4) launch_k(k_qr_core3<4>, g, dim3(256), h->qrc_smem, h->st, h->ctx, redo);
    else if (h->qrc_ct <= 5) launch_k(k_qr_core3<5>, g, dim3(256), h->qrc_smem, h->st, h->ctx, redo);
    else launch_k(k_qr_core3<8>, g, dim3(256), h->qrc_smem, h->st, h->ctx, redo);
  }
  else
    launch_k(k_qr_core, dim3(h->S * h->ctx.qr_nchunks), dim3(256), 0, h->st, h->ctx, redo);
  prof(h, redo ? "redo:qr_core" : "qr_core");
  count_launch(2);
  CB_CHECK_LAUNCH();
  return CB_OK;
}

static int enqueue_control(cb_solver* h, int mode, int extra = 0) {
  const int bsrc = h->fast3 ? 0 : 1;
  if (!h->shard) {
    if (emit(h)) {
      launch_k(k_control, dim3(1), dim3(256), 0, h->st, h->ctx, mode, bsrc, 3 | extra);
      count_launch(1);
      CB_CHECK_LAUNCH();
    }
    prof(h, "control");
    return CB_OK;
  }
  if (emit(h)) {
    launch_k(k_control, dim3(1), dim3(256), 0, h->st, h->ctx, mode, bsrc, 1 | extra);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  int rc = xchg(h, h->ctx.ctl_w, h->ctx.ctl, 3LL * h->S_tot);
  if (rc) return rc;
  if (emit(h)) {
    launch_k(k_control, dim3(1), dim3(256), 0, h->st, h->ctx, mode, bsrc, 2 | extra);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  prof(h, "control");
  return CB_OK;
}

static int enqueue_restore(cb_solver* h) {
  if (emit(h)) {
    launch_k(k_restore, dim3(h->S), dim3(256), h->blk_smem, h->st, h->ctx, 0);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  prof(h, "redo:restore");
  return CB_OK;
}

// evaluation after a sweep (full mode): fiber pass (fast3) or generic terms
static int enqueue_eval_full(cb_solver* h, int redo) {
  if (h->fast3) {
    XArgs a = redo ? h->xa_redo : h->xa_main;
    a.t_other = 1;   // write the non-accepted T buffer
    int rc;
    if (!h->ctx.ld_pre)
      return enqueue_fiber(h, a, 1, h->ctx.b_mtt ? 0 : 1, h->objective == 0 ? 1 : 0);
    // per-block evaluation algebra beside the fiber pass (side stream)
    const bool par = !h->in_body;
    if (par && (rc = fork_side(h))) return rc;
    if (emit(h)) {
      launch_k(k_eval_side, dim3(h->S), dim3(256), h->blk_smem_ng, par ? h->st2 : h->st, h->ctx, redo);
      count_launch(1);
      CB_CHECK_LAUNCH();
    }
    if ((rc = enqueue_fiber(h, a, 1, 0, h->objective == 0 ? 1 : 0))) return rc;
    if (par && (rc = join_side(h))) return rc;
    return CB_OK;
  }
  // generic: b from the last mode's MTTKRP (solver.py:506-509), residuals
  for (int s = 0; s < h->S; ++s) {
    int rc = generic_rowdot_into(h, s, h->N - 1, nullptr);
    if (rc) return rc;
  }
  if (h->objective == 0) return generic_residuals(h);
  return CB_OK;
}

static int enqueue_trace_lra(cb_solver* h) {
  if (h->xtc) {
    // tensor-core trace pass (xtc.cu): b_orig of every block into fib_bpart
    if (!emit(h)) return CB_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->timing) { int rc = ev_pair(h, &e0, &e1, 1); if (rc) return rc; CB_CUDA(cudaEventRecord(e0, h->st)); }
    int rc = xtc_trace(h->xtc, h->xa_main.U, h->xa_main.gate, h->ctx.fib_bpart, h->st);
    if (rc) return rc;
    CB_CHECK_LAUNCH();
    if (h->timing) { CB_CUDA(cudaEventRecord(e1, h->st)); h->t_launches += 1; h->t_bytes += xtc_bytes(h->xtc); }
    return CB_OK;
  }
  if (h->fast3) return enqueue_fiber(h, h->xa_main, 0, 1, 0);
  for (int s = 0; s < h->S; ++s) {
    int rc = generic_mttkrp(h, s, 0);
    if (rc) return rc;
    rc = generic_rowdot_into(h, s, 0, h->ctx.borig + (long long)s * RSTRIDE);
    if (rc) return rc;
  }
  return CB_OK;
}

// one full APG iteration (solver.py:586-610), device-gated
// restart branch (solver.py:594-599): restore, sweep with w_hat = 0,
// re-evaluate, accept; every kernel is gated on go_redo
static int enqueue_pipe_prep_redo(cb_solver* h);

static int enqueue_redo_branch(cb_solver* h) {
  int rc;
  if ((rc = enqueue_restore(h))) return rc;
  if ((rc = enqueue_sweep(h, 1))) return rc;
  if (!h->lra) {
    if ((rc = enqueue_eval_full(h, 1))) return rc;
    prof(h, "redo:fiber");
  } else if ((rc = enqueue_qr(h, 1))) {
    return rc;
  }
  if (h->redo_reprep && (rc = enqueue_pipe_prep_redo(h))) return rc;
  return enqueue_control(h, CTRL_REDO);
}

// Under graph capture (h->cond_capture) the restart branch becomes the body of
// a conditional IF node (sharded: one node per stretch between exchanges), so
// an iteration without restart launches none of its ~15 kernels; otherwise it
// is enqueued inline as gated no-ops.
static int begin_cond_body(cb_solver* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CB_CUDA(cudaStreamGetCaptureInfo(h->st_main, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h->ctx.cond;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CB_CUDA(cudaGraphAddNode(&node, g, deps, nd, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CB_CUDA(cudaStreamUpdateCaptureDependencies(h->st_main, &node, 1,
                                              cudaStreamSetCaptureDependencies));
  h->st = h->st3;
  CB_CUDA(cudaStreamBeginCaptureToGraph(h->st3, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeThreadLocal));
  return CB_OK;
}

static int end_cond_body(cb_solver* h) {
  cudaGraph_t done_body;
  cudaError_t e = cudaStreamEndCapture(h->st3, &done_body);
  h->st = h->st_main;
  CB_CUDA(e);
  return CB_OK;
}

static int enqueue_redo(cb_solver* h) {
  if (!h->cond_capture) return enqueue_redo_branch(h);
  h->st_main = h->st;
  int rc = begin_cond_body(h);
  if (rc) return rc;
  h->in_body = true;
  rc = enqueue_redo_branch(h);
  h->in_body = false;
  const int rc2 = end_cond_body(h);
  return rc ? rc : rc2;
}

// one full APG iteration (solver.py:586-610), device-gated
static int enqueue_iteration(cb_solver* h) {
  int rc;
  prof(h, "(start)");
  if (!h->lra) {
    if ((rc = enqueue_sweep(h, 0))) return rc;
    if ((rc = enqueue_eval_full(h, 0))) return rc;
    prof(h, "fiber");
    if ((rc = enqueue_control(h, CTRL_DECIDE))) return rc;
    if ((rc = enqueue_redo(h))) return rc;
  } else {
    if ((rc = enqueue_sweep(h, 0))) return rc;
    if ((rc = enqueue_qr(h, 0))) return rc;
    if ((rc = enqueue_control(h, CTRL_DECIDE))) return rc;
    if ((rc = enqueue_redo(h))) return rc;
    if ((rc = enqueue_trace_lra(h))) return rc;
    prof(h, "trace_fiber");
    if ((rc = enqueue_control(h, CTRL_FINISH))) return rc;
  }
  return CB_OK;
}

// ---- pipelined lra iteration (single GPU, tensor-core trace pass) ---------
// The trace pass only feeds FINISH (trace, histories, stop rule), never the
// next sweep, so iteration k's streaming pass (16 GB on c5) runs on the side
// stream beside the sweep + QR route of iteration k+1:
//   prologue (k = 1):  sweep, qr, DECIDE (advances the momentum), redo, prep
//   step (k -> k+1):   [st2: trace(k)] || [st: sweep(k+1), qr(k+1)] -> join
//                      -> FINISH(k) (snapshots of lam_k / model_sq_k) ->
//                      rollback if it stopped (k_restore, gate 1) -> DECIDE
//                      (k+1) -> redo -> prep(k+1) + snapshots
//   drain:             trace(k), FINISH(k) (no speculative sweep to undo)
// The arithmetic is that of the classic order, so results are identical.
// Operand prep of the next trace into the set the running trace does not
// read, then (PREP_COMMIT) the lam / model_sq snapshots and the set flip.
//   PREP_MAIN:   after DECIDE / redo on the main gate (the prologue);
//   PREP_SPEC:   right after the sweep, beside the running trace: the
//                factors are final unless the iteration restarts;
//   PREP_REDO:   inside the restart branch (gate go_redo), after its sweep;
//   PREP_COMMIT: snapshots + flip only.
enum { PREP_MAIN = 0, PREP_SPEC = 1, PREP_REDO = 2, PREP_COMMIT = 3 };

static int enqueue_pipe_prep(cb_solver* h, int mode) {
  if (!emit(h)) return CB_OK;
  if (mode != PREP_COMMIT) {
    const int* gate = mode == PREP_REDO ? h->xa_redo.gate : h->xa_main.gate;
    int rc = xtc_trace(h->xtc, h->xa_main.U, gate, h->ctx.fib_bpart, h->st, 1, 1);
    if (rc) return rc;
    if (mode != PREP_MAIN) return CB_OK;
  }
  launch_k(k_pipe_snap, dim3(h->S), dim3(64), 0, h->st, h->ctx);
  count_launch(1);
  CB_CHECK_LAUNCH();
  return xtc_flip(h->xtc, h->xa_main.gate, h->st);
}

static int enqueue_pipe_prep_redo(cb_solver* h) { return enqueue_pipe_prep(h, PREP_REDO); }

static int enqueue_pipe_stream(cb_solver* h, cudaStream_t st) {
  if (!emit(h)) return CB_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->timing) { int rc = ev_pair(h, &e0, &e1, 1); if (rc) return rc; CB_CUDA(cudaEventRecord(e0, st)); }
  int rc = xtc_trace(h->xtc, h->xa_main.U, h->xa_main.gate, h->ctx.fib_bpart, st, 2);
  if (rc) return rc;
  CB_CHECK_LAUNCH();
  if (h->timing) { CB_CUDA(cudaEventRecord(e1, st)); h->t_launches += 1; h->t_bytes += xtc_bytes(h->xtc); }
  return CB_OK;
}

static int enqueue_pipe_prologue(cb_solver* h) {
  int rc;
  if ((rc = enqueue_sweep(h, 0))) return rc;
  if ((rc = enqueue_qr(h, 0))) return rc;
  if ((rc = enqueue_control(h, CTRL_DECIDE, 16))) return rc;
  if ((rc = enqueue_redo(h))) return rc;
  return enqueue_pipe_prep(h, PREP_MAIN);
}

static int enqueue_pipe_step(cb_solver* h) {
  int rc;
  if ((rc = fork_side(h))) return rc;
  if ((rc = enqueue_pipe_stream(h, h->st2))) return rc;
  if ((rc = enqueue_sweep(h, 0))) return rc;
  if ((rc = enqueue_qr(h, 0))) return rc;
  if ((rc = enqueue_pipe_prep(h, PREP_SPEC))) return rc;
  if ((rc = join_side(h))) return rc;
  if ((rc = enqueue_control(h, CTRL_FINISH, 16 | 32))) return rc;
  if (emit(h)) {
    launch_k(k_restore, dim3(h->S), dim3(256), h->blk_smem, h->st, h->ctx, 1);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  if ((rc = enqueue_control(h, CTRL_DECIDE, 16))) return rc;
  h->redo_reprep = true;     // a restarted iteration re-prepares the operands
  rc = enqueue_redo(h);
  h->redo_reprep = false;
  if (rc) return rc;
  return enqueue_pipe_prep(h, PREP_COMMIT);
}

static int pipe_drain(cb_solver* h) {
  if (!h->pipe_pending) return CB_OK;
  int rc;
  if ((rc = enqueue_pipe_stream(h, h->st))) return rc;
  if ((rc = enqueue_control(h, CTRL_FINISH, 16))) return rc;
  h->pipe_pending = false;
  return CB_OK;
}

static int read_state(cb_solver* h) {
  CB_CUDA(cudaMemcpyAsync(h->h_state, h->d_state, sizeof(State), cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaStreamSynchronize(h->st));
  return CB_OK;
}

// generic path: iteration with a host-side restart decision
static int generic_iteration(cb_solver* h) {
  int rc;
  if ((rc = enqueue_sweep(h, 0))) return rc;
  if (!h->lra) {
    if ((rc = enqueue_eval_full(h, 0))) return rc;
  } else if ((rc = enqueue_qr(h, 0))) return rc;
  if ((rc = enqueue_control(h, CTRL_DECIDE))) return rc;
  if ((rc = read_state(h))) return rc;
  if (h->h_state->go_redo) {
    launch_k(k_restore, dim3(h->S), dim3(256), h->blk_smem, h->st, h->ctx, 0);
    count_launch(1);
    CB_CHECK_LAUNCH();
    if ((rc = enqueue_sweep(h, 1))) return rc;
    if (!h->lra) {
      if ((rc = enqueue_eval_full(h, 1))) return rc;
    } else if ((rc = enqueue_qr(h, 1))) return rc;
    if ((rc = enqueue_control(h, CTRL_REDO))) return rc;
  }
  if (h->lra) {
    if ((rc = enqueue_trace_lra(h))) return rc;
    if ((rc = enqueue_control(h, CTRL_FINISH))) return rc;
  }
  return CB_OK;
}

static int generic_rowdot_into(cb_solver* h, int s, int n, double* out) {
  // b[r] = sum_i U_n[i,r] MTT[i,r]; default target: staged b buffer 1 - bsel
  // (bsel is read on the host: generic path syncs every iteration)
  double* dst = out;
  if (!dst) {
    const int bsel = h->h_state->bsel;
    dst = h->ctx.bbuf + ((long long)(1 - bsel) * h->S + s) * RSTRIDE;
  }
  return ::cb_rowdot(h->h_U[s * h->N + n], h->h_MTT[s], h->dims[s * h->N + n], h->R[s], dst,
                   (void*)h->st);
}

static int generic_residuals(cb_solver* h) {
  for (int s = 0; s < h->S; ++s) {
    ResidArgs a{};
    a.order = h->N; a.R = h->R[s]; a.n = 1;
    a.w = h->h_LAM[s];
    for (int m = 0; m < h->N; ++m) {
      a.dims[m] = h->dims[s * h->N + m];
      a.U[m] = h->h_U[s * h->N + m];
      a.n *= a.dims[m];
    }
    int rc = kruskal_residual(h->dtype, a, h->X[s], h->ctx.res + s, h->res_part, h->res_nparts, h->st);
    if (rc) return rc;
  }
  return CB_OK;
}

static int init_evaluation(cb_solver* h) {
  int rc;
  if (emit(h)) {
    launch_k(k_init_block, dim3(h->S), dim3(256), h->blk_smem, h->st, h->ctx);
    count_launch(1);
    CB_CHECK_LAUNCH();
  }
  if (!h->lra) {
    if (h->fast3) {
      XArgs a = h->xa_main;
      a.t_other = 1;
      if ((rc = enqueue_fiber(h, a, 1, 1, h->objective == 0 ? 1 : 0))) return rc;
    } else {
      // iteration 0 stages b from the mode-0 unfolding (solver.py:510-511)
      for (int s = 0; s < h->S; ++s) {
        if ((rc = generic_mttkrp(h, s, 0))) return rc;
        if ((rc = generic_rowdot_into(h, s, 0, nullptr))) return rc;
      }
      if (h->objective == 0 && (rc = generic_residuals(h))) return rc;
    }
  } else {
    if ((rc = enqueue_qr(h, 0))) return rc;
    if ((rc = enqueue_trace_lra(h))) return rc;
  }
  return enqueue_control(h, CTRL_INIT);
}

}  // namespace cb

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int cb_solver_create(const cb_solver_desc* d, void* stream, cb_solver** out) {
  CB_ARG(d && out, "null descriptor");
  *out = nullptr;
  CB_ARG(d->n_blocks >= 1, "no tensors");
  CB_ARG(d->order >= 1 && d->order <= CB_MAX_ORDER, "order %d outside [1, %d]", d->order, CB_MAX_ORDER);
  CB_ARG(d->dtype == CB_F32 || d->dtype == CB_F64, "bad dtype");
  const int world = d->world_size > 1 ? d->world_size : 1;
  const int shard = (world > 1 || d->nccl_comm) ? 1 : 0;
  if (shard) {
    CB_ARG(d->order == 3, "block-sharded solves need 3-way blocks (order %d)", d->order);
    CB_ARG(d->rank_id >= 0 && d->rank_id < world, "rank %d outside [0, %d)", d->rank_id, world);
    CB_ARG(d->block_offset >= 0 && d->block_offset + d->n_blocks <= d->total_blocks,
           "block range [%d, %d) outside the %d blocks", d->block_offset,
           d->block_offset + d->n_blocks, d->total_blocks);
    if (d->nccl_comm) {
      int rc0 = nccl_load();
      if (rc0) return rc0;
    }
  }
  cb_solver* h = new cb_solver();
  h->world = world;
  h->shard = shard;
  h->rank = shard ? d->rank_id : 0;
  h->comm = shard ? d->nccl_comm : nullptr;
  h->S_tot = shard ? d->total_blocks : d->n_blocks;
  h->off = shard ? d->block_offset : 0;
  h->st = (cudaStream_t)stream;
  h->S = d->n_blocks; h->N = d->order; h->lra = d->lra; h->update_core = d->update_core;
  h->dtype = d->dtype; h->objective = d->objective; h->delta_w = d->delta_w; h->tol = d->tol;
  h->pc = d->dtype == CB_F64 ? PC_F64 : (d->compute == 1 ? PC_F32 : PC_F32_F64);
  h->max_iter = d->max_iter;
  const int S = h->S, N = h->N;
  h->dims.assign(d->dims, d->dims + S * N);
  h->R.assign(d->ranks, d->ranks + S);
  for (int n = 0; n < N; ++n) h->counts[n] = d->coupled[n];
  h->X.assign(d->tensors, d->tensors + S);
  for (int s = 0; s < S; ++s) {
    if (h->R[s] < 1 || h->R[s] > CB_MAX_RANK) {
      delete h;
      set_error("rank %d outside [1, %d]", d->ranks[s], CB_MAX_RANK);
      return CB_ERR_UNSUPPORTED;
    }
    h->rmax = std::max(h->rmax, h->R[s]);
  }
  if (h->lra) {
    h->Rt.assign(d->tilde_ranks, d->tilde_ranks + S);
    for (int s = 0; s < S; ++s) {
      h->rtmax = std::max(h->rtmax, h->Rt[s]);
      if (h->Rt[s] + h->R[s] > QR_MAXC || h->Rt[s] > CB_MAX_RANK) {
        delete h;
        set_error("compression rank %d + rank %d exceeds the QR route limit %d", d->tilde_ranks[s],
                  d->ranks[s], QR_MAXC);
        return CB_ERR_UNSUPPORTED;
      }
    }
  } else {
    h->Rt.assign(S, 0);
  }
  h->fast3 = (N == 3);
  h->rb = rank_bucket(h->rmax);
  h->elem_bytes = h->dtype == CB_F32 ? 4 : 8;
  for (int s = 0; s < S; ++s) {
    long long e = 1;
    for (int n = 0; n < N; ++n) e *= h->dims[s * N + n];
    h->elem_total += e;
  }
  std::vector<void*>& A = h->allocs;
  cudaStream_t st = h->st;
  set_alloc_stream(st);
  int rc = CB_OK;
#define TRY(x) do { rc = (x); if (rc) { cb_solver_destroy(h); return rc; } } while (0)
  // ---- per-(s,n) factor buffers
  std::vector<double*> U(S * N), Up(S * N), Un(S * N), G(S * N), C(S * N), Ut(S * N);
  std::vector<double*> LAM(S), LAMP(S), TW(S), STEP(S), MTT(S);
  long long maxIn = 0;
  for (int s = 0; s < S; ++s) {
    const int Rs = h->R[s];
    long long mI = 0;
    for (int n = 0; n < N; ++n) {
      const long long In = h->dims[s * N + n];
      mI = std::max(mI, In);
      const size_t fb = sizeof(double) * In * Rs;
      TRY(dalloc((void**)&U[s * N + n], fb, A));
      TRY(dalloc((void**)&Up[s * N + n], fb, A));
      TRY(dalloc((void**)&Un[s * N + n], fb, A));
      TRY(dalloc((void**)&G[s * N + n], sizeof(double) * Rs * Rs, A));
      CB_CUDA(cudaMemcpyAsync(U[s * N + n], d->init_factors[s * N + n], fb, cudaMemcpyHostToDevice, st));
      CB_CUDA(cudaMemcpyAsync(Up[s * N + n], d->init_factors[s * N + n], fb, cudaMemcpyHostToDevice, st));
      if (h->lra) {
        const int Rts = h->Rt[s];
        TRY(dalloc((void**)&C[s * N + n], sizeof(double) * Rts * Rs, A));
        TRY(dalloc((void**)&Ut[s * N + n], sizeof(double) * In * Rts, A));
        CB_CUDA(cudaMemcpyAsync(Ut[s * N + n], d->tilde_factors[s * N + n], sizeof(double) * In * Rts,
                                cudaMemcpyDeviceToDevice, st));
      }
    }
    maxIn = std::max(maxIn, mI);
    TRY(dalloc((void**)&LAM[s], sizeof(double) * Rs, A));
    TRY(dalloc((void**)&LAMP[s], sizeof(double) * Rs, A));
    CB_CUDA(cudaMemcpyAsync(LAM[s], d->init_weights[s], sizeof(double) * Rs, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaMemcpyAsync(LAMP[s], d->init_weights[s], sizeof(double) * Rs, cudaMemcpyHostToDevice, st));
    TRY(dalloc((void**)&STEP[s], sizeof(double) * Rs * Rs, A));
    TRY(dalloc((void**)&MTT[s], sizeof(double) * mI * Rs, A));
    if (h->lra) {
      TRY(dalloc((void**)&TW[s], sizeof(double) * h->Rt[s], A));
      CB_CUDA(cudaMemcpyAsync(TW[s], d->tilde_weights[s], sizeof(double) * h->Rt[s], cudaMemcpyHostToDevice, st));
    }
  }
  h->h_U = U;
  h->h_MTT = MTT;
  h->h_LAM = LAM;
  Ctx& c = h->ctx;
  c.S = S; c.S_tot = h->S_tot; c.off = h->off; c.shard = shard;
  c.N = N; c.lra = h->lra; c.update_core = h->update_core; c.objective = h->objective;
  c.fast3 = h->fast3; c.max_iter = h->max_iter; c.rmax = std::max(h->rmax, h->rtmax);
  for (int n = 0; n < N; ++n) c.counts[n] = h->counts[n];
  c.delta_w = h->delta_w; c.tol = h->tol;
  long long* d_dims; int *d_R, *d_Rt;
  TRY(upload(h->dims, &d_dims, A, st)); c.dims = d_dims;
  TRY(upload(h->R, &d_R, A, st)); c.R = d_R;
  TRY(upload(h->Rt, &d_Rt, A, st)); c.Rt = d_Rt;
  double** p;
  TRY(upload(U, &p, A, st)); c.U = p;
  TRY(upload(Up, &p, A, st)); c.Up = p;
  TRY(upload(Un, &p, A, st)); c.Un = p;
  TRY(upload(G, &p, A, st)); c.G = p;
  TRY(upload(LAM, &p, A, st)); c.LAM = p;
  TRY(upload(LAMP, &p, A, st)); c.LAMP = p;
  TRY(upload(STEP, &p, A, st)); c.STEP = p;
  TRY(upload(MTT, &p, A, st)); c.MTT = p;
  if (h->lra) {
    TRY(upload(C, &p, A, st)); c.C = p;
    TRY(upload(Ut, &p, A, st)); c.Ut = p;
    TRY(upload(TW, &p, A, st)); c.TW = p;
  }
  TRY(dalloc((void**)&c.lipc_hist, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.evec, sizeof(double) * S * (N + 1) * 64, A));
  TRY(dalloc((void**)&c.evec_miss, sizeof(int) * S * (N + 1), A));
  TRY(dalloc((void**)&c.fin_cnt, sizeof(int) * S, A));
  c.dbg = nullptr;
  TRY(dalloc((void**)&c.lipf_hist, sizeof(double) * N * S, A));
  TRY(dalloc((void**)&c.ldcore, sizeof(double) * S, A));
  // coupling arrays in global block slots; separate send copies when sharded
  // (their foreign slots stay zero: the all-reduce is an exact all-gather)
  const int ST = h->S_tot;
  TRY(dalloc((void**)&c.lip, sizeof(double) * 2 * N * ST, A));
  TRY(dalloc((void**)&c.ctl, sizeof(double) * 3 * ST, A));
  c.lip_w = c.lip; c.ctl_w = c.ctl;
  if (shard) {
    TRY(dalloc((void**)&c.lip_w, sizeof(double) * 2 * N * ST, A));
    TRY(dalloc((void**)&c.ctl_w, sizeof(double) * 3 * ST, A));
  }
  TRY(dalloc((void**)&c.nsq, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.bbuf, sizeof(double) * 2 * S * RSTRIDE, A));
  TRY(dalloc((void**)&c.model_sq, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.inner, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.res_t, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.tsq, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.res, sizeof(double) * S, A));
  TRY(dalloc((void**)&c.borig, sizeof(double) * S * RSTRIDE, A));
  TRY(dalloc((void**)&c.lam_snap, sizeof(double) * S * 64, A));
  TRY(dalloc((void**)&c.msq_snap, sizeof(double) * S, A));
  int maxL = 0;
  for (int n = 0; n < N; ++n) maxL = std::max(maxL, h->counts[n]);
  c.gc_stride = maxIn * std::max(maxL, 1);
  TRY(dalloc((void**)&c.gc_part, sizeof(double) * ST * c.gc_stride, A));
  c.gc_w = c.gc_part;
  if (shard) TRY(dalloc((void**)&c.gc_w, sizeof(double) * ST * c.gc_stride, A));
  TRY(dalloc((void**)&c.cnew, sizeof(double) * c.gc_stride, A));
  TRY(dalloc((void**)&c.tile_cnt, sizeof(int) * (maxIn / MU_ROWS + 2), A));
  if (h->lra) {
    TRY(dalloc((void**)&c.qr_buf, sizeof(double) * (size_t)S * N * QR_MAXC * QR_MAXC, A));
    // ||core||^2: the GEMM form for 3-way blocks whose R1 / R2 images fit in
    // shared memory, else the generic per-entry kernel
    long long pairs = 1, k2max = 1;
    size_t qrc = 0;
    for (int s = 0; s < S; ++s) {
      const long long Cc = h->R[s] + h->Rt[s];
      if (N != 3) break;
      const long long K0 = std::min(h->dims[3 * s], Cc), K1 = std::min(h->dims[3 * s + 1], Cc);
      const long long K2 = std::min(h->dims[3 * s + 2], Cc);
      pairs = std::max(pairs, K0);
      qrc = std::max(qrc, sizeof(double) * (size_t)(Cc + Cc * K1 + Cc * K2 + Cc * QRC_A));
      k2max = std::max(k2max, K2);
      if (K2 > 16 * QRC_CT) qrc = SIZE_MAX;
    }
    h->qr_core3 = N == 3 && qrc <= 200 * 1024;
    h->qrc_ct = (int)((k2max + 15) / 16);
    h->qrc_smem = h->qr_core3 ? qrc : 0;
    c.qr_nchunks = h->qr_core3 ? (int)((pairs + QRC_A - 1) / QRC_A) : 8;
    TRY(dalloc((void**)&c.qr_part, sizeof(double) * S * c.qr_nchunks, A));
  }
  TRY(dalloc((void**)&c.h_obj, sizeof(double) * (h->max_iter + 1), A));
  TRY(dalloc((void**)&c.h_orig, sizeof(double) * (h->max_iter + 1), A));
  TRY(dalloc((void**)&c.h_rel, sizeof(double) * (h->max_iter + 1), A));
  TRY(dalloc((void**)&c.h_tns, sizeof(double) * (h->max_iter + 1), A));
  TRY(dalloc((void**)&h->d_state, sizeof(State), A));
  c.st = h->d_state;
  CB_CUDA(cudaMallocHost((void**)&h->h_state, sizeof(State)));
  memset(h->h_state, 0, sizeof(State));
  State s0{};
  s0.k = 0; s0.go_main = 1; s0.go_redo = 0; s0.t_k = 1.0; s0.w_hat = 0.0;
  s0.obj_prev = INFINITY; s0.rel_prev = 0.0;
  CB_CUDA(cudaMemcpyAsync(h->d_state, &s0, sizeof(State), cudaMemcpyHostToDevice, st));
  // ---- ||M_s||^2 (solver.py:327) with the validation statistics kernel
  {
    double* stats;
    TRY(dalloc((void**)&stats, sizeof(double) * 3 * S, A));
    double* part;
    TRY(dalloc((void**)&part, sizeof(double) * 3 * 148 * 8, A));
    for (int s = 0; s < S; ++s) {
      long long n = 1;
      for (int m = 0; m < N; ++m) n *= h->dims[s * N + m];
      int np = (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + 255) / 256));
      TRY(tensor_stats(h->dtype, h->X[s], n, stats + 3 * s, part, np, st));
    }
    // nsq[s] = stats[3s]
    std::vector<double> hs(3 * S);
    CB_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(double) * 3 * S, cudaMemcpyDeviceToHost, st));
    CB_CUDA(cudaStreamSynchronize(st));
    std::vector<double> ns(S);
    for (int s = 0; s < S; ++s) ns[s] = hs[3 * s];
    CB_CUDA(cudaMemcpyAsync(c.nsq, ns.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    CB_CUDA(cudaStreamSynchronize(st));
  }
  // ---- mode-update tile: 64 rows for the lra 3-way path (the per-tile
  // staging of the step matrix and two cross grams then serves twice the
  // rows, half the CTAs) when its shared memory fits, else MU_ROWS
  {
    int maxL = 0;
    for (int n = 0; n < N; ++n) maxL = std::max(maxL, h->counts[n]);
    const int rtm = std::max(h->rtmax, 1);
    auto mu_bytes = [&](long long tr) {
      return sizeof(double) * ((size_t)h->rmax * h->rmax + 2 * (size_t)tr * h->rmax +
                               (h->lra ? (size_t)rtm * h->rmax : 0) + 16 +
                               (h->lra && N == 3 ? 2 * (size_t)rtm * h->rmax + (size_t)tr * rtm + rtm : 0) +
                               2 * (size_t)tr * h->rmax + 2 * (size_t)tr * maxL);
    };
    c.mu_rows = (h->lra && N == 3 && mu_bytes(64) <= 200 * 1024) ? 64 : MU_ROWS;
    h->mu_smem = mu_bytes(c.mu_rows);
  }
  // ---- row-unit tables for the mode updates
  h->d_rows.assign(N, nullptr);
  h->n_rows.assign(N, 0);
  for (int n = 0; n < N; ++n) {
    std::vector<RowUnit> ru;
    for (int s = 0; s < S; ++s)
      for (long long r0 = 0; r0 < h->dims[s * N + n]; r0 += c.mu_rows) ru.push_back(RowUnit{s, (int)r0});
    h->n_rows[n] = (int)ru.size();
    TRY(upload(ru, &h->d_rows[n], A, st));
  }
  // ---- fast 3-way tables and T buffers
  std::vector<void*> T0(S, nullptr), T1(S, nullptr);
  if (h->fast3) {
    build_xtables(S, h->dims.data(), h->R.data(), h->rb, h->pc, h->tab, h->S_tot);
    TRY(upload(h->tab.fib, &h->d_fib, A, st));
    if (!h->tab.fib4.empty()) {
      FibUnit* d4;
      TRY(upload(h->tab.fib4, &d4, A, st));
      h->tab.d_fib4 = d4;
    }
    TRY(upload(h->tab.slab, &h->d_slab, A, st));
    TRY(upload(h->tab.c0, &h->d_c0, A, st));
    TRY(upload(h->tab.c1, &h->d_c1, A, st));
    int* di;
    TRY(upload(h->tab.fib_first, &di, A, st)); c.fib_first = di;
    TRY(upload(h->tab.slab_first, &di, A, st)); c.slab_first = di;
    TRY(upload(h->tab.slab_nchunk, &di, A, st)); c.slab_nchunk = di;
    int* d_ns;
    TRY(upload(h->tab.nsplit, &d_ns, A, st));
    c.slab_sb = h->tab.sb;
    h->tma = tma_rows_ok(S, h->dims.data(), h->X.data(), h->elem_bytes);
    prepare_slab(h->pc, h->rb, h->tma, h->tab);
    prepare_fiber(h->pc, h->rb, h->tma, h->tab);
    double *ubpart, *urpart;
    TRY(dalloc((void**)&ubpart, sizeof(double) * h->tab.fib.size() * RSTRIDE, A));
    TRY(dalloc((void**)&urpart, sizeof(double) * h->tab.fib.size(), A));
    TRY(dalloc((void**)&c.fib_bpart, sizeof(double) * S * RSTRIDE, A));
    TRY(dalloc((void**)&c.fib_rpart, sizeof(double) * S, A));
    int* blk_cnt;
    TRY(dalloc((void**)&blk_cnt, sizeof(int) * S, A));
    TRY(dalloc((void**)&c.slab_part, sizeof(double) * h->tab.slab.size() * h->tab.sb * RSTRIDE, A));
    if (!h->lra) {
      for (int s = 0; s < S; ++s) {
        const size_t tb = (size_t)h->tab.nsplit[s] * h->R[s] * h->dims[3 * s] * h->dims[3 * s + 1] *
                          pc_compute_bytes(h->pc);
        TRY(dalloc(&T0[s], tb, A));
        TRY(dalloc(&T1[s], tb, A));
      }
    }
    void** pv;
    TRY(upload(T0, &pv, A, st));
    void** pv1;
    TRY(upload(T1, &pv1, A, st));
    const void** pX;
    TRY(upload(h->X, &pX, A, st));
    XArgs xa{};
    xa.X = pX; xa.dims = c.dims; xa.R = c.R; xa.U = (const double* const*)c.U; xa.LAM = (const double* const*)c.LAM;
    xa.T0 = pv; xa.T1 = pv1; xa.tsel = &h->d_state->tsel; xa.t_other = 0;
    xa.nsplit = d_ns; xa.bpart = ubpart; xa.rpart = urpart; xa.slab_part = c.slab_part;
    xa.fib_first = c.fib_first; xa.blk_cnt = blk_cnt; xa.bsum = c.fib_bpart; xa.rsum = c.fib_rpart;
    xa.MTT = c.MTT; xa.active = nullptr;
    xa.ktime = nullptr;
    xa.slab_stage_rows = h->tab.slab_rows;
    {
      int* d_s3;
      TRY(upload(h->tab.s3_first, &d_s3, A, st));
      xa.s3_first = d_s3;
      int* d_f3;
      TRY(upload(h->tab.f3_first, &d_f3, A, st));
      xa.f3_first = d_f3;
    }
    // with the row-dot mode-2 kernel, the core linear term b is staged from
    // its MTTKRP output (solver.py:506-509) in k_finalize of the last mode,
    // so the evaluation fiber pass only forms T
    c.b_mtt = (h->tab.slab_direct && !h->lra) ? 1 : 0;
    c.ld_pre = c.b_mtt;
    xa.gate = &h->d_state->go_main;
    h->xa_main = xa;
    // lra trace pass on the tensor cores (compute code 2, fp32 storage)
    if (h->lra && d->compute == 2 && h->dtype == CB_F32 &&
        xtc_supported(S, h->X.data(), h->dims.data(), h->R.data())) {
      // a plan that does not fit (shared memory) leaves the CUDA-core pass
      if (xtc_plan_create(S, h->X.data(), h->dims.data(), h->R.data(), st, &h->xtc) != CB_OK)
        h->xtc = nullptr;
      // pipelined when the trace pass streams >= 32 MB (c3, c4, c5; c4, 35 MB:
      // 1710 -> 1780 it/s over its 500 iterations since the operand prep left
      // the critical path); below that the snapshot / rollback work costs
      // more than the hidden trace
      // sharded: with an NCCL communicator (the emulated group runs the
      // classic order segment by segment)
      h->pipe = h->xtc != nullptr && (!shard || d->nccl_comm) && d->pipeline != 2 &&
                (xtc_bytes(h->xtc) >= 32e6 || d->pipeline == 1);
      if (h->pipe) {
        // leave SMs for the sweep that runs beside the trace (its per-block
        // CTAs).  The trace pass stays HBM bound down to ~100 SMs (its MMA time
        // per SM is half its HBM share, its epilogue is integer), so the sweep
        // gets up to 40: c5 (S = 64) measured 2.32 ms per iteration at 32, 2.28
        // at 36, 2.29 at 40, 2.33 at 44, 2.37 at 48
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int reserve = d->pipeline_reserve > 0 ? d->pipeline_reserve : std::min(S, 40);
        reserve = std::max(0, std::min(reserve, nsm / 2));
        xtc_set_grid_cap(h->xtc, nsm - reserve);
      }
    }
    xa.gate = &h->d_state->go_redo;
    h->xa_redo = xa;
  } else {
    size_t kr = 0;
    for (int s = 0; s < S; ++s)
      for (int n = 0; n < N; ++n) {
        long long Lp = 1, Hp = 1;
        for (int m = 0; m < n; ++m) Lp *= h->dims[s * N + m];
        for (int m = n + 1; m < N; ++m) Hp *= h->dims[s * N + m];
        kr = std::max(kr, (size_t)(Lp + Hp) * h->R[s]);
      }
    TRY(dalloc((void**)&h->kr_scratch, sizeof(double) * kr, A));
    h->res_nparts = 148 * 4;
    TRY(dalloc((void**)&h->res_part, sizeof(double) * h->res_nparts, A));
  }
  // ---- shared memory sizes
  h->blk_smem = block_smem_bytes(c.rmax, c.rmax);
  h->blk_smem_ng = block_smem_bytes(c.rmax, 0);
  int maxRt = std::max(h->rtmax, 1);
  // (mu_smem: set with the mode-update tile above)
  h->qr_smem = 0;
  if (h->lra) {
    int cmax = 0;
    for (int s = 0; s < S; ++s) cmax = std::max(cmax, h->R[s] + h->Rt[s]);
    const size_t cap = 227 * 1024;
    h->qr_ch = qr_chunk_rows(cmax, cap);
    h->qr_smem = sizeof(double) * ((size_t)cmax * (cmax + 1) + (size_t)h->qr_ch * (cmax + 1) +
                                  (size_t)qr_extra_doubles(cmax));
  }
  CB_CUDA(cudaFuncSetAttribute(k_init_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem));
  CB_CUDA(cudaFuncSetAttribute(k_sweep_begin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem_ng));
  CB_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem));
  CB_CUDA(cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem_ng));
  CB_CUDA(cudaFuncSetAttribute(k_eval_side, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem_ng));
  CB_CUDA(cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking));
  CB_CUDA(cudaStreamCreateWithFlags(&h->st3, cudaStreamNonBlocking));
  CB_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CB_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CB_CUDA(cudaFuncSetAttribute(k_restore, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->blk_smem));
  CB_CUDA(cudaFuncSetAttribute(k_mode_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->mu_smem));
  if (h->lra)
  {
    CB_CUDA(cudaFuncSetAttribute(k_qr_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->qr_smem));
    if (h->qr_core3) {
      CB_CUDA(cudaFuncSetAttribute(k_qr_core3<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->qrc_smem));
      CB_CUDA(cudaFuncSetAttribute(k_qr_core3<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->qrc_smem));
      CB_CUDA(cudaFuncSetAttribute(k_qr_core3<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->qrc_smem));
      CB_CUDA(cudaFuncSetAttribute(k_qr_core3<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->qrc_smem));
    }
  }
  // ---- iteration 0 (an emulated group runs it through cb_group_step)
  if (!shard || h->comm) {
    TRY(init_evaluation(h));
    TRY(read_state(h));
    h->init_done = true;
  } else {
    CB_CUDA(cudaStreamSynchronize(st));
  }
#undef TRY
  *out = h;
  return CB_OK;
}

int cb_solver_step_async(cb_solver* h) {
  CB_ARG(h, "null handle");
  CB_ARG(!h->shard || h->comm, "emulated shard groups are stepped with cb_group_step");
  if (!h->fast3) {
    int rc = generic_iteration(h);
    return rc;
  }
  if (h->pipe && !h->timing && !h->profile) {
    if (!h->pipe_pending) {
      // a new pipeline: iteration k+1's sweep .. prep, eagerly
      int rc = enqueue_pipe_prologue(h);
      if (rc) return rc;
      h->pipe_pending = true;
      return CB_OK;
    }
    if (!h->gexec_pipe && h->graph_ok) {
      cudaGraph_t g;
      cudaError_t e = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        {
          cudaGraph_t cg;
          cudaStreamCaptureStatus cs;
          if (cudaStreamGetCaptureInfo(h->st, &cs, nullptr, &cg, nullptr, nullptr) == cudaSuccess &&
              cudaGraphConditionalHandleCreate(&h->ctx.cond, cg, 0, cudaGraphCondAssignDefault) ==
                  cudaSuccess) {
            h->ctx.use_cond = 1;
            h->cond_capture = true;
          }
        }
        const long long before = cb_launch_count();
        int rc = enqueue_pipe_step(h);
        h->launches_per_pipe = cb_launch_count() - before;
        h->ctx.use_cond = 0;
        h->cond_capture = false;
        cudaError_t e2 = cudaStreamEndCapture(h->st, &g);
        if (rc == CB_OK && e2 == cudaSuccess) {
          if (cudaGraphInstantiate(&h->gexec_pipe, g, 0) != cudaSuccess) {
            h->gexec_pipe = nullptr;
            h->graph_ok = false;
          }
          cudaGraphDestroy(g);
        } else {
          h->graph_ok = false;
        }
        cudaGetLastError();
      } else {
        h->graph_ok = false;
        cudaGetLastError();
      }
    }
    if (h->gexec_pipe) {
      CB_CUDA(cudaGraphLaunch(h->gexec_pipe, h->st));
      count_launch(h->launches_per_pipe);
      return CB_OK;
    }
    return enqueue_pipe_step(h);
  }
  if (h->pipe) {
    int rc = pipe_drain(h);   // the classic iteration (timing / profile modes)
    if (rc) return rc;
  }
  if (h->timing || h->profile) return enqueue_iteration(h);
  if (!h->gexec && h->graph_ok) {
    cudaGraph_t g;
    cudaError_t e = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      // conditional restart branch (sharded: NCCL exchanges between the bodies)
      if (!h->shard || h->comm) {
        cudaGraph_t cg;
        cudaStreamCaptureStatus cs;
        if (cudaStreamGetCaptureInfo(h->st, &cs, nullptr, &cg, nullptr, nullptr) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&h->ctx.cond, cg, 0, cudaGraphCondAssignDefault) ==
                cudaSuccess) {
          h->ctx.use_cond = 1;
          h->cond_capture = true;
        }
      }
      const long long before = cb_launch_count();
      int rc = enqueue_iteration(h);
      h->launches_per_iter = cb_launch_count() - before;
      h->ctx.use_cond = 0;
      h->cond_capture = false;
      cudaError_t e2 = cudaStreamEndCapture(h->st, &g);
      if (rc == CB_OK && e2 == cudaSuccess) {
        cudaError_t e3 = cudaGraphInstantiate(&h->gexec, g, 0);
        if (e3 != cudaSuccess) {
          h->gexec = nullptr;
          h->graph_ok = false;
        }
        cudaGraphDestroy(g);
      } else {
        h->graph_ok = false;
      }
      cudaGetLastError();
    } else {
      h->graph_ok = false;
      cudaGetLastError();
    }
  }
  if (h->gexec) {
    CB_CUDA(cudaGraphLaunch(h->gexec, h->st));
    count_launch(h->launches_per_iter);
    return CB_OK;
  }
  return enqueue_iteration(h);
}

int cb_solver_summary_get(cb_solver* h, cb_solver_summary* sum) {
  CB_ARG(h && sum, "null handle");
  int rc = pipe_drain(h);
  if (rc) return rc;
  rc = read_state(h);
  if (rc) return rc;
  const State& s = *h->h_state;
  sum->n_iter = s.n_hist > 0 ? s.n_hist - 1 : 0;
  sum->n_restarts = s.n_restarts;
  sum->done = s.done;
  sum->reason = s.reason;
  sum->error = s.error;
  sum->error_block = s.err_block;
  sum->error_iter = s.err_iter;
  return CB_OK;
}

int cb_solver_run(cb_solver* h, int iters, cb_solver_summary* sum) {
  CB_ARG(h, "null handle");
  CB_ARG(!h->shard || h->comm, "emulated shard groups run through cb_group_run");
  int rc = read_state(h);
  if (rc) return rc;
  int left = iters;
  while (left > 0 && !h->h_state->done) {
    const int chunk = std::min(left, h->fast3 ? 16 : 1);
    for (int i = 0; i < chunk; ++i) {
      rc = cb_solver_step_async(h);
      if (rc) return rc;
    }
    left -= chunk;
    rc = read_state(h);
    if (rc) return rc;
  }
  if ((rc = pipe_drain(h))) return rc;
  if (sum) return cb_solver_summary_get(h, sum);
  return CB_OK;
}

int cb_solver_history(cb_solver* h, double* obj_int, double* obj_orig, double* rel, double* t_ns,
                      int cap) {
  CB_ARG(h, "null handle");
  int rc = pipe_drain(h);
  if (rc) return rc;
  rc = read_state(h);
  if (rc) return rc;
  const int n = std::min(cap, h->h_state->n_hist);
  if (n <= 0) return CB_OK;
  if (obj_int) CB_CUDA(cudaMemcpyAsync(obj_int, h->ctx.h_obj, sizeof(double) * n, cudaMemcpyDeviceToHost, h->st));
  if (obj_orig) CB_CUDA(cudaMemcpyAsync(obj_orig, h->ctx.h_orig, sizeof(double) * n, cudaMemcpyDeviceToHost, h->st));
  if (rel) CB_CUDA(cudaMemcpyAsync(rel, h->ctx.h_rel, sizeof(double) * n, cudaMemcpyDeviceToHost, h->st));
  if (t_ns) CB_CUDA(cudaMemcpyAsync(t_ns, h->ctx.h_tns, sizeof(double) * n, cudaMemcpyDeviceToHost, h->st));
  CB_CUDA(cudaStreamSynchronize(h->st));
  return CB_OK;
}

int cb_solver_block_factors(cb_solver* h, int block, double* const* host_factors,
                            double* host_weights) {
  CB_ARG(h && block >= 0 && block < h->S, "bad block %d", block);
  {
    int rc = pipe_drain(h);
    if (rc) return rc;
  }
  for (int n = 0; n < h->N; ++n) {
    if (!host_factors || !host_factors[n]) continue;
    CB_CUDA(cudaMemcpyAsync(host_factors[n], h->h_U[block * h->N + n],
                            sizeof(double) * h->dims[block * h->N + n] * h->R[block],
                            cudaMemcpyDeviceToHost, h->st));
  }
  if (host_weights) {
    CB_CUDA(cudaMemcpyAsync(host_weights, h->h_LAM[block], sizeof(double) * h->R[block], cudaMemcpyDeviceToHost, h->st));
  }
  CB_CUDA(cudaStreamSynchronize(h->st));
  return CB_OK;
}

int cb_solver_profile(cb_solver* h, int on, char* out, int cap) {
  CB_ARG(h, "null handle");
  if (on) {
    h->profile = true;
    h->mused = 0;
    h->mlabels.clear();
    return CB_OK;
  }
  CB_CUDA(cudaStreamSynchronize(h->st));
  h->profile = false;
  // aggregate intervals (previous mark -> this mark) by this mark's label
  std::vector<std::string> names;
  std::vector<double> tot;
  std::vector<long long> cnt;
  for (size_t i = 1; i < h->mused; ++i) {
    if (strcmp(h->mlabels[i], "(start)") == 0) continue;
    float t = 0.f;
    CB_CUDA(cudaEventElapsedTime(&t, h->mpool[i - 1], h->mpool[i]));
    size_t k = 0;
    for (; k < names.size(); ++k)
      if (names[k] == h->mlabels[i]) break;
    if (k == names.size()) { names.push_back(h->mlabels[i]); tot.push_back(0.0); cnt.push_back(0); }
    tot[k] += t;
    cnt[k] += 1;
  }
  std::string s;
  char line[160];
  for (size_t k = 0; k < names.size(); ++k) {
    snprintf(line, sizeof(line), "%s %lld %.6f\n", names[k].c_str(), cnt[k], tot[k]);
    s += line;
  }
  if (h->ctx.dbg) {
    double ph[64];
    CB_CUDA(cudaMemcpy(ph, h->ctx.dbg, sizeof(ph), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 64; ++k)
      if (ph[k] > 0.0) {
        snprintf(line, sizeof(line), "phase%02d 0 %.6f\n", k, ph[k] * 1e-6);
        s += line;
      }
  }
  if (out && cap > 0) {
    strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
  }
  return CB_OK;
}

int cb_solver_timeline(cb_solver* h, int op, unsigned long long* out, int cap) {
  CB_ARG(h, "null handle");
  const size_t bytes = sizeof(unsigned long long) * 2 * TL_NSLOT;
  if (op == 1 && !h->ctx.tl) {
    CB_CUDA(cudaMalloc((void**)&h->ctx.tl, bytes));
    h->allocs.push_back(h->ctx.tl);
    h->xa_main.tl = h->ctx.tl;
    h->xa_redo.tl = h->ctx.tl;
    xtc_set_timeline(h->xtc, h->ctx.tl);
    if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }   // recapture
    if (h->gexec_pipe) { cudaGraphExecDestroy(h->gexec_pipe); h->gexec_pipe = nullptr; }
  }
  if (op == -1 && h->ctx.tl) {
    h->ctx.tl = nullptr;
    h->xa_main.tl = nullptr;
    h->xa_redo.tl = nullptr;
    xtc_set_timeline(h->xtc, nullptr);
    // both iteration graphs captured the timeline pointer: recapture them
    if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
    if (h->gexec_pipe) { cudaGraphExecDestroy(h->gexec_pipe); h->gexec_pipe = nullptr; }
    return CB_OK;
  }
  if (!h->ctx.tl) return CB_OK;
  if (op == 1 || op == 2) {
    // begin slots (even) start at ~0 for atomicMin, end slots at 0
    std::vector<unsigned long long> init(2 * TL_NSLOT);
    for (int k = 0; k < TL_NSLOT; ++k) { init[2 * k] = ~0ull; init[2 * k + 1] = 0ull; }
    CB_CUDA(cudaMemcpyAsync(h->ctx.tl, init.data(), bytes, cudaMemcpyHostToDevice, h->st));
    CB_CUDA(cudaStreamSynchronize(h->st));
    return CB_OK;
  }
  CB_CUDA(cudaStreamSynchronize(h->st));
  CB_ARG(out && cap >= 2 * TL_NSLOT, "timeline buffer needs %d entries", 2 * TL_NSLOT);
  CB_CUDA(cudaMemcpy(out, h->ctx.tl, bytes, cudaMemcpyDeviceToHost));
  return CB_OK;
}

int cb_solver_set_timing(cb_solver* h, int on) {
  CB_ARG(h, "null handle");
  h->timing = on != 0;
  h->ev_used = 0;
  h->ev_kind.clear();
  h->t_ms = 0.0; h->t_bytes = 0.0; h->t_launches = 0;
  return CB_OK;
}

int cb_solver_timing(cb_solver* h, int kind, double* ms, long long* launches, double* bytes) {
  CB_ARG(h, "null handle");
  CB_CUDA(cudaStreamSynchronize(h->st));
  double tot = 0.0;
  long long n = 0;
  for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
    if (kind != 0 && h->ev_kind[i / 2] != kind) continue;
    float t = 0.f;
    CB_CUDA(cudaEventElapsedTime(&t, h->ev_pool[i], h->ev_pool[i + 1]));
    tot += t;
    n += 1;
  }
  if (ms) *ms = tot;
  if (launches) *launches = n;
  if (bytes) *bytes = (double)n * (double)h->elem_total * h->elem_bytes;
  return CB_OK;
}

// ---- emulated shard groups (verification of the sharded program on one GPU)
int cb_group_step(cb_solver* const* hs, int n, int program) {
  CB_ARG(hs && n >= 1 && n <= CB_MAX_GROUP, "group of %d handles outside [1, %d]", n, CB_MAX_GROUP);
  CB_ARG(program == 0 || program == 1, "program %d", program);
  for (int k = 0; k < n; ++k) {
    CB_ARG(hs[k] && hs[k]->world == n && !hs[k]->comm && hs[k]->rank == k,
           "handle %d is not rank %d of an emulated group of %d", k, k, n);
    CB_ARG(hs[k]->st == hs[0]->st, "group handles must share one stream");
    CB_ARG(program == 1 || !hs[k]->init_done, "iteration 0 already evaluated");
    CB_ARG(program == 0 || hs[k]->init_done, "iteration 0 not evaluated yet");
  }
  auto run = [&](cb_solver* h, int want) -> int {
    h->seg_cur = 0;
    h->seg_want = want;
    h->pending.clear();
    int rc = program == 0 ? init_evaluation(h) : enqueue_iteration(h);
    h->seg_want = -1;
    return rc;
  };
  int rc = run(hs[0], -2);
  if (rc) return rc;
  const int nseg = hs[0]->seg_cur + 1;
  for (int seg = 0; seg < nseg; ++seg) {
    for (int k = 0; k < n; ++k) {
      if ((rc = run(hs[k], seg))) return rc;
    }
    for (size_t x = 0; x < hs[0]->pending.size(); ++x) {
      XsumArgs a{};
      a.n = n;
      a.count = hs[0]->pending[x].count;
      for (int k = 0; k < n; ++k) {
        CB_ARG(hs[k]->pending.size() == hs[0]->pending.size() && hs[k]->pending[x].count == a.count,
               "group handles disagree on the exchange program");
        a.send[k] = hs[k]->pending[x].send;
        a.recv[k] = hs[k]->pending[x].recv;
      }
      const int blocks = (int)std::min<long long>(148 * 4, (a.count + 255) / 256);
      launch_k(k_xsum, dim3(std::max(blocks, 1)), dim3(256), 0, hs[0]->st, a);
      count_launch(1);
      CB_CHECK_LAUNCH();
    }
  }
  for (int k = 0; k < n; ++k) {
    hs[k]->pending.clear();
    if (program == 0) hs[k]->init_done = true;
  }
  return CB_OK;
}

int cb_group_run(cb_solver* const* hs, int n, int iters, cb_solver_summary* sum) {
  CB_ARG(hs && n >= 1, "empty group");
  int rc;
  if (!hs[0]->init_done && (rc = cb_group_step(hs, n, 0))) return rc;
  if ((rc = read_state(hs[0]))) return rc;
  int left = iters;
  while (left > 0 && !hs[0]->h_state->done) {
    const int chunk = std::min(left, 8);
    for (int i = 0; i < chunk; ++i)
      if ((rc = cb_group_step(hs, n, 1))) return rc;
    left -= chunk;
    if ((rc = read_state(hs[0]))) return rc;
  }
  if (sum) return cb_solver_summary_get(hs[0], sum);
  return CB_OK;
}

int cb_solver_destroy(cb_solver* h) {
  if (!h) return CB_OK;
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gexec_pipe) cudaGraphExecDestroy(h->gexec_pipe);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->st2) cudaStreamDestroy(h->st2);
  if (h->st3) cudaStreamDestroy(h->st3);
  dfree_all(h->allocs);
  cb::xtc_plan_destroy(h->xtc);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  if (h->h_state) cudaFreeHost(h->h_state);
  delete h;
  return CB_OK;
}

}  // extern "C"
