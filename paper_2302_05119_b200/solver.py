"""Coupled nonnegative CP decomposition by APG — B200 drop-in for
`pkg/src/concpd/solver.py`.

The public surface is the reference's: ``CoupledProblem``, ``SolverOptions``,
``SolveResult``, ``TraceRow``, ``solve`` and the operator-level building
blocks (solver.py:34-52).  ``solve`` validates on the host, draws the
reference's seeded start (bit-identical numpy PCG64 stream), uploads the
blocks once, and hands the whole iteration to the device engine
(`cb_solver_*`, csrc/engine.cu): sweep, objective, restart rule and stop
rule all run on the GPU.  lra mode first compresses every block with the
batched device ALS (`cb_als_*`).  No code path computes on the CPU.

Additions over the reference (defaulted, so existing callers are unchanged):
``SolverOptions.precision`` ("fp64" parity mode, "fp32" throughput mode that
stores the tensors in fp32 while keeping factors and all small algebra in
fp64) and ``SolverOptions.objective`` ("auto" = explicit residual in fp64
like the reference, gram expansion in fp32; or force "explicit" /
"expansion") and ``SolverOptions.compute`` (arithmetic of the tensor passes
when the storage is fp32: "auto" = fp64 for CoNCPD-APG, whose restart rule
compares objectives that differ by ~1e-12 late in a run, and for the ALS
compression, whose fixed point is sensitive; "tc" for the lra
original-tensor trace pass of ranks > 16, which feeds the reported trace and
stop rule alone: the tensor-core pass of `cb_core_linear_term_tc`, ~2e-8
relative on b.  "fp32" forces CUDA-core fp32 arithmetic in that pass).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib as L
from .cpd_als import AlsHandle, AlsOptions, _check_feasible, als_compress_blocks, als_staged_ok
from .kruskal import CoupledFactorSet, KruskalTensor
from .tensor_ops import hadamard_gram, spectral_norm

__all__ = [
    "CoupledProblem", "SolverOptions", "core_linear_terms_tc", "SolveResult", "TraceRow", "solve", "objective",
    "core_gradient", "factor_gradient", "core_linear_term", "core_linear_term_lra",
    "factor_linear_term", "factor_linear_term_lra", "lipschitz_core", "lipschitz_factor",
    "extrapolation_weight", "t_next", "init_factors", "solve_distributed",
    "solve_emulated_shards", "shard_ranges", "ShardSpec",
]


def _is_torch(t):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(t, torch.Tensor)


@dataclass
class CoupledProblem:
    """S nonnegative tensors decomposed jointly (solver.py:60-135).

    ``tensors`` may be numpy arrays (cast to float64 like the reference,
    except float32 arrays, which are kept: the cast is exact and the fp32
    throughput mode uploads them without a float64 detour) or CUDA torch
    tensors already resident on the device (kept as given; an fp32 tensor
    stored first-index-fastest is used without any copy).
    """

    tensors: list
    ranks: list
    coupled_counts: list
    mode: str = "full"
    update_core: bool = True
    als_options: AlsOptions = None

    def __post_init__(self):
        self.tensors = [t if (_is_torch(t) or (isinstance(t, np.ndarray) and t.dtype == np.float32))
                        else np.asarray(t, dtype=float) for t in self.tensors]
        if isinstance(self.ranks, (int, np.integer)):
            self.ranks = [int(self.ranks)] * len(self.tensors)
        self.ranks = [int(r) for r in self.ranks]
        self.coupled_counts = [int(c) for c in self.coupled_counts]

    @property
    def n_blocks(self):
        return len(self.tensors)

    @property
    def order(self):
        return self.tensors[0].ndim

    def validate(self, check_values=True):
        """The reference's checks in the reference's order (solver.py:96-135):
        per block its order, then its values; then ranks and coupled counts.
        ``check_values=False`` skips the per-element finite / nonnegative scan
        (the single-process solve runs the same loop with the scan on the
        device, in the input's own dtype, right after each upload)."""
        self._validate_head()
        for s, t in enumerate(self.tensors):
            self._validate_block(s, t)
            if check_values:
                _raise_values(s, t)
        self._validate_tail()

    def _validate_head(self):
        if not self.tensors:
            raise ValueError("no tensors")
        if self.mode not in ("full", "lra"):
            raise ValueError(f"unknown mode {self.mode!r}")

    def _validate_block(self, s, t):
        order = self.tensors[0].ndim
        if t.ndim != order:
            raise ValueError(f"block {s} has order {t.ndim}, expected {order}")

    def _validate_tail(self):
        order = self.tensors[0].ndim
        if len(self.ranks) != len(self.tensors):
            raise ValueError("one rank per block required")
        if any(r < 1 for r in self.ranks):
            raise ValueError("ranks must be >= 1")
        if len(self.coupled_counts) != order:
            raise ValueError("one coupled count per mode required")
        lo = min(self.ranks)
        for n, c in enumerate(self.coupled_counts):
            if not 0 <= c <= lo:
                raise ValueError(f"coupled count {c} in mode {n} exceeds minimum rank {lo}")
            if c > 0:
                sizes = sorted({int(t.shape[n]) for t in self.tensors})
                if len(sizes) != 1:
                    raise ValueError(f"mode {n} is coupled but block sizes differ: {sizes}")


def _raise_values(s, t):
    finite, nonneg = _value_checks(t)
    if not finite:
        raise ValueError(f"block {s} contains non-finite values")
    if not nonneg:
        raise ValueError(f"block {s} contains negative entries")


def _value_checks(t):
    """(all finite, no negative entries).  Device tensors are checked by the
    library's statistics kernel; host arrays with numpy (input validation,
    not the hot path)."""
    if _is_torch(t):
        torch = D.torch_mod()
        flat = t.reshape(-1) if t.is_contiguous() else t.contiguous().reshape(-1)
        code = L.CB_F32 if flat.dtype == torch.float32 else L.CB_F64
        if flat.dtype not in (torch.float32, torch.float64):
            flat = flat.to(torch.float64)
            code = L.CB_F64
        out = torch.empty(3, dtype=torch.float64, device=flat.device)
        L.check(L.lib.cb_tensor_stats(code, D.ptr(flat), flat.numel(), D.ptr(out), D.stream()))
        ss, mn, bad = (float(v) for v in out.cpu())
        return bad == 0.0, not (mn < 0.0)
    return bool(np.isfinite(t).all()), not bool((t < 0).any())


@dataclass
class SolverOptions:
    max_iter: int = 1000
    tol: float = 1e-8
    delta_w: float = 0.9999
    seed: int = 0
    trace_every: int = 1
    precision: str = "fp64"        # "fp64" parity mode | "fp32" throughput mode
    objective: str = "auto"        # "auto" | "explicit" | "expansion"
    compute: str = "auto"          # fp32 storage: "auto" | "fp64" | "fp32" | "tc" (lra trace)
    pipeline: str = "auto"         # lra tensor-core trace beside the next sweep: "auto" | "on" | "off"
    pipeline_reserve: int = 0      # SMs the pipelined trace leaves to the sweep (0 = auto)

    def __post_init__(self):
        if self.max_iter < 0:
            raise ValueError("max_iter must be >= 0")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if not 0.0 < self.delta_w < 1.0:
            raise ValueError("delta_w must lie in (0, 1)")
        if self.trace_every < 1:
            raise ValueError("trace_every must be >= 1")
        if self.precision not in ("fp64", "fp32"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.objective not in ("auto", "explicit", "expansion"):
            raise ValueError(f"unknown objective evaluation {self.objective!r}")
        if self.compute not in ("auto", "fp64", "fp32", "tc"):
            raise ValueError(f"unknown compute type {self.compute!r}")
        if self.pipeline not in ("auto", "on", "off"):
            raise ValueError(f"unknown pipeline mode {self.pipeline!r}")


@dataclass(frozen=True)
class TraceRow:
    iteration: int
    obj_fun: float
    rel_err: float
    elapsed_s: float


@dataclass
class SolveResult:
    """Outcome of :func:`solve` (solver.py:165-186).  ``trace`` reports the
    original-tensor objective and RelErr; ``objective_history`` is the
    minimised objective (compressed in lra mode) kept non-increasing by the
    restart rule."""

    factors: CoupledFactorSet
    trace: list
    termination_reason: str
    objective_history: list = field(repr=False, default_factory=list)
    rel_err_history: list = field(repr=False, default_factory=list)
    n_iter: int = 0
    n_restarts: int = 0
    solve_seconds: float = 0.0
    compress_seconds: float = 0.0
    compression: list = None
    # additions (defaulted): ALS sweeps per block of the lra compression
    compression_iters: list = None


# ---------------------------------------------------------------------------
# scalar rules and the seeded start (host: they are not tensor arithmetic)
# ---------------------------------------------------------------------------

def t_next(t):
    """t_k = (1 + sqrt(1 + 4 t_{k-1}^2)) / 2 (solver.py:265-267)."""
    return 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))


def extrapolation_weight(w_hat, lip_prev, lip_curr, delta_w):
    """min(w_hat, delta_w sqrt(L_prev/L_curr)); 0 on degenerate blocks (solver.py:270-274)."""
    if lip_curr <= 0.0 or lip_prev <= 0.0:
        return 0.0
    return min(w_hat, delta_w * float(np.sqrt(lip_prev / lip_curr)))


def init_factors(problem, seed):
    """Uniform [0,1) start, common prefix drawn once; the draw order matches the
    reference exactly (solver.py:277-303) so GPU runs start bit-identically."""
    rng = np.random.default_rng(seed)
    counts = problem.coupled_counts
    shape0 = tuple(problem.tensors[0].shape)
    shared = [rng.random((shape0[n], counts[n])) for n in range(problem.order)]
    blocks = []
    for s in range(problem.n_blocks):
        r = problem.ranks[s]
        shp = tuple(problem.tensors[s].shape)
        facs = []
        for n in range(problem.order):
            own = rng.random((shp[n], r - counts[n]))
            facs.append(np.hstack([shared[n], own]) if counts[n] else own)
        lam = rng.random(r) if problem.update_core else np.ones(r)
        blocks.append(KruskalTensor(facs, lam))
    return CoupledFactorSet(blocks, list(counts))


# ---------------------------------------------------------------------------
# operator-level building blocks (GPU)
# ---------------------------------------------------------------------------

def _dev_tensor(t):
    dtype = "fp64"
    if _is_torch(t):
        import torch
        dtype = "fp32" if t.dtype == torch.float32 else "fp64"
    flat, dims = D.tensor_to_dev(t, dtype)
    return flat, dims, (L.CB_F32 if dtype == "fp32" else L.CB_F64)


def factor_linear_term(tensor, factors, n):
    """M_(n) U_kr^(-n) on the GPU (`cb_mttkrp`; solver.py:243-245)."""
    torch = D.torch_mod()
    flat, dims, code = _dev_tensor(tensor)
    rank = int(np.asarray(factors[0]).shape[1])
    dev = [D.to_dev_f64(f) for f in factors]
    out = torch.empty((dims[n], rank), dtype=torch.float64, device=flat.device)
    L.check(L.lib.cb_mttkrp(code, D.ptr(flat), len(dims), L.i64_array(dims),
                            L.ptr_array([D.ptr(x) for x in dev]), rank, n, D.ptr(out),
                            D.stream()))
    return D.to_host(out)


def core_linear_term(tensor, factors):
    """(U_kr)^T vec(M) through the mode-0 MTTKRP (solver.py:215-218)."""
    torch = D.torch_mod()
    flat, dims, code = _dev_tensor(tensor)
    rank = int(np.asarray(factors[0]).shape[1])
    dev = [D.to_dev_f64(f) for f in factors]
    mtt = torch.empty((dims[0], rank), dtype=torch.float64, device=flat.device)
    L.check(L.lib.cb_mttkrp(code, D.ptr(flat), len(dims), L.i64_array(dims),
                            L.ptr_array([D.ptr(x) for x in dev]), rank, 0, D.ptr(mtt),
                            D.stream()))
    out = torch.empty(rank, dtype=torch.float64, device=flat.device)
    L.check(L.lib.cb_rowdot(D.ptr(dev[0]), D.ptr(mtt), dims[0], rank, D.ptr(out), D.stream()))
    return D.to_host(out)


def core_linear_terms_tc(tensors, factor_sets):
    """Batched core linear terms b_s = (U_kr,s)^T vec(M_s) of 3-way blocks on
    the tensor cores (`cb_core_linear_term_tc`: tcgen05 kind::i8 over
    byte-sliced fixed-point operands, exact int32 accumulation, ~2^-20
    relative per product).  The tensors are cast to fp32 (the throughput-mode
    storage); returns a list of R_s-vectors (solver.py:215-218)."""
    torch = D.torch_mod()
    devs, dims, ranks, facs = [], [], [], []
    for t, fs in zip(tensors, factor_sets):
        flat, d = D.tensor_to_dev(np.asarray(t), "fp32")
        if len(d) != 3:
            raise ValueError("the tensor-core trace pass needs 3-way blocks")
        devs.append(flat)
        dims.extend(int(x) for x in d)
        ranks.append(int(np.asarray(fs[0]).shape[1]))
        facs.extend(D.to_dev_f64(f) for f in fs)
    out = torch.zeros((len(devs), 64), dtype=torch.float64, device=devs[0].device)
    L.check(L.lib.cb_core_linear_term_tc(len(devs), L.ptr_array([D.ptr(x) for x in devs]),
                                         L.i64_array(dims), L.ptr_array([D.ptr(x) for x in facs]),
                                         L.int_array(ranks), D.ptr(out), D.stream()))
    host = D.to_host(out)
    return [host[s, :r].copy() for s, r in enumerate(ranks)]


def _gemm(a, b, ta=False, tb=False, alpha=1.0):
    torch = D.torch_mod()
    da, db = D.to_dev_f64(a), D.to_dev_f64(b)
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device=da.device)
    L.check(L.lib.cb_gemm(int(ta), int(tb), m, n, k, float(alpha), D.ptr(da), a.shape[1],
                          D.ptr(db), b.shape[1], 0.0, D.ptr(out), n, D.stream()))
    return D.to_host(out)


def core_linear_term_lra(tilde, factors):
    """(hadamard U^T U~) w~ via cross grams (solver.py:221-229)."""
    cross = hadamard_gram(factors, mats2=tilde.factors)
    return _gemm(cross, tilde.weights.reshape(-1, 1))[:, 0]


def factor_linear_term_lra(tilde, factors, n):
    """(U~_n * w~) (hadamard_{m!=n} U~_m^T U_m) (solver.py:248-251)."""
    cross = hadamard_gram(tilde.factors, skip=n, mats2=factors)
    scaled = np.asarray(tilde.factors[n]) * tilde.weights
    return _gemm(scaled, cross)


def core_gradient(gram_all, lam_hat, linear):
    """gram_all lam_hat - linear (solver.py:205-212)."""
    g = _gemm(np.asarray(gram_all, dtype=float), np.asarray(lam_hat, dtype=float).reshape(-1, 1))
    return g[:, 0] - np.asarray(linear, dtype=float)


def factor_gradient(u_hat, gram_skip, mtt, lam):
    """u_hat (gram_skip o lam lam^T) - mtt o lam (`cb_factor_gradient`; solver.py:232-240)."""
    torch = D.torch_mod()
    u_hat = np.asarray(u_hat, dtype=float)
    du = D.to_dev_f64(u_hat)
    dg = D.to_dev_f64(gram_skip)
    dm = D.to_dev_f64(mtt)
    dl = D.to_dev_f64(lam)
    out = torch.empty(u_hat.shape, dtype=torch.float64, device=du.device)
    L.check(L.lib.cb_factor_gradient(D.ptr(du), u_hat.shape[0], D.ptr(dg), D.ptr(dm), D.ptr(dl),
                                     u_hat.shape[1], D.ptr(out), D.stream()))
    return D.to_host(out)


def lipschitz_core(factors):
    """lambda_max of the all-modes Hadamard gram (solver.py:254-256)."""
    return spectral_norm(hadamard_gram(factors))


def lipschitz_factor(factors, lam, n):
    """lambda_max of (hadamard_{m!=n} gram) o lam lam^T (solver.py:259-262)."""
    g = hadamard_gram(factors, skip=n) * np.outer(lam, lam)
    return spectral_norm(g)


def objective(tensors, blocks):
    """1/2 sum_s ||M_s - [[lam_s; U_s]]||^2 by explicit streaming residuals on
    the GPU (`cb_kruskal_residual`; solver.py:194-202)."""
    torch = D.torch_mod()
    total = 0.0
    for t, k in zip(tensors, blocks):
        flat, dims, code = _dev_tensor(np.asarray(t, dtype=float) if not _is_torch(t) else t)
        dev = [D.to_dev_f64(f) for f in k.factors]
        dw = D.to_dev_f64(k.weights)
        out = torch.empty(1, dtype=torch.float64, device=flat.device)
        L.check(L.lib.cb_kruskal_residual(code, D.ptr(flat), len(dims), L.i64_array(dims),
                                          L.ptr_array([D.ptr(x) for x in dev]), D.ptr(dw),
                                          k.rank, D.ptr(out), D.stream()))
        total += 0.5 * float(out.item())
    return total


# ---------------------------------------------------------------------------
# solve
# ---------------------------------------------------------------------------

class _Engine:
    """Owns one device solver handle (re-entrant: one per solve)."""

    def __init__(self, desc, stream):
        h = L.c_vp()
        L.check(L.lib.cb_solver_create(ctypes.byref(desc), stream, ctypes.byref(h)))
        self.h = h

    def run(self, iters):
        summ = L.SolverSummary()
        L.check(L.lib.cb_solver_run(self.h, int(iters), ctypes.byref(summ)))
        return summ

    def summary(self):
        summ = L.SolverSummary()
        L.check(L.lib.cb_solver_summary_get(self.h, ctypes.byref(summ)))
        return summ

    def step_async(self):
        L.check(L.lib.cb_solver_step_async(self.h))

    def history(self, n):
        oi, oo, rel, tns = (np.zeros(n) for _ in range(4))
        L.check(L.lib.cb_solver_history(self.h, oi.ctypes.data_as(L.c_dp),
                                        oo.ctypes.data_as(L.c_dp), rel.ctypes.data_as(L.c_dp),
                                        tns.ctypes.data_as(L.c_dp), n))
        return oi, oo, rel, tns

    def block(self, s, dims, rank):
        facs = [np.zeros((d, rank)) for d in dims]
        w = np.zeros(rank)
        L.check(L.lib.cb_solver_block_factors(self.h, s, L.dptr_array(facs),
                                              w.ctypes.data_as(L.c_dp)))
        return facs, w

    def set_timing(self, on):
        L.check(L.lib.cb_solver_set_timing(self.h, int(on)))

    def timing(self, kind=0):
        ms = ctypes.c_double()
        n = ctypes.c_longlong()
        b = ctypes.c_double()
        L.check(L.lib.cb_solver_timing(self.h, int(kind), ctypes.byref(ms), ctypes.byref(n),
                                       ctypes.byref(b)))
        return ms.value, n.value, b.value

    def close(self):
        if getattr(self, "h", None) and L is not None and getattr(L, "lib", None) is not None:
            L.lib.cb_solver_destroy(self.h)
        self.h = None

    def __del__(self):
        self.close()


class PreparedSolve:
    """A solve with its inputs resident on the device, split into
    prepare / iterate / collect so the bench can time the iterations alone."""

    def __init__(self, problem, opts=None, stream=None, shard=None, agree=None):
        torch = D.torch_mod()
        opts = opts if opts is not None else SolverOptions()
        # the reference's checks in its order (per block: order, values; then
        # ranks / counts).  The element scan runs on the device in each
        # block's own dtype before the downcast to `precision`; a sharded rank
        # scans its own blocks and `agree` (PreparedShardedSolve: an
        # all-reduce) makes every rank raise the same first error
        problem._validate_head()
        self.problem, self.opts = problem, opts
        S_all = problem.n_blocks
        self.shard = shard if shard is not None else ShardSpec(1, 0, 0, S_all, None)
        if not (0 <= self.shard.begin < self.shard.end <= S_all):
            raise ValueError(f"shard [{self.shard.begin}, {self.shard.end}) of {S_all} blocks is empty "
                             "or out of range")
        self.local = list(range(self.shard.begin, self.shard.end))
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        prec = opts.precision
        self.code = L.CB_F32 if prec == "fp32" else L.CB_F64
        objective_mode = opts.objective
        if objective_mode == "auto":
            objective_mode = "explicit" if prec == "fp64" else "expansion"
        # arithmetic of the tensor passes on fp32 storage: fp64 wherever the
        # result steers the iterates (full-mode MTTKRPs and objective, the ALS
        # compression); the lra trace pass only feeds the reported trace and
        # may run in fp32 for large ranks
        compute = opts.compute
        if compute == "auto":
            compute = "fp64" if (problem.mode == "full" or max(problem.ranks) <= 16) else "tc"
        self.compute_code = {"fp64": 0, "fp32": 1, "tc": 2}[compute] if prec == "fp32" else 0
        # ALS compression: fp64-grade passes (ranks in (16, 48]: exact int8
        # slice GEMMs on the tensor cores, csrc/xoz.cu; the compressed model
        # of an ill-conditioned fit moves by ~1e-5 relative under ~1e-9 MTTKRP
        # changes, so the passes keep ~1e-13) unless "fp32" is asked for
        self.als_compute_code = ({"fp32": 1}.get(opts.compute, 0)
                                 if prec == "fp32" else 0)
        S, N = len(self.local), problem.order
        with torch.cuda.stream(self.stream):
            self.dev = []
            self.dims = []
            first_bad, bad_msg = None, None     # (block, 0 order / 1 values)
            limit = len(problem.tensors)
            for g, t in enumerate(problem.tensors):
                try:
                    problem._validate_block(g, t)
                except ValueError as exc:
                    first_bad, bad_msg, limit = (g, 0), exc, g
                    break
            scan = [g for g in self.local if g < limit]
            stats = torch.empty((max(len(scan), 1), 3), dtype=torch.float64, device=D.device())
            shapes = [tuple(int(d) for d in problem.tensors[g].shape) for g in scan]
            # host-side checks that follow the value checks in the reference's
            # order (ranks / counts, then the compression's feasibility); they
            # only need the shapes
            ranks = None
            late_exc = None
            if bad_msg is None:
                try:
                    problem._validate_tail()
                    if problem.mode == "lra":
                        base = (problem.als_options if problem.als_options is not None
                                else AlsOptions())
                        ranks = [base.rank if base.rank is not None else problem.ranks[g]
                                 for g in self.local]
                        for s, (dims, r) in enumerate(zip(shapes, ranks)):
                            try:
                                _check_feasible(dims, r)
                            except ValueError as exc:
                                raise ValueError(
                                    f"compression of block {self.local[s]} failed: {exc}") from exc
                except ValueError as exc:
                    late_exc = exc
            self.als = None
            st = L.c_vp(self.stream.cuda_stream)
            als_exc = None
            als_ran = False
            t_als = 0.0
            want = torch.float32 if prec == "fp32" else torch.float64

            def _stageable(t, dims):
                return (isinstance(t, torch.Tensor) and not t.is_cuda and t.is_pinned()
                        and t.dtype == want and tuple(t.stride()) == D.fortran_strides(dims))

            # lra solves on pinned host tensors already in the solve's dtype and
            # layout (single process): the uploads run on a copy stream with an
            # event per block and the compression starts every block as it
            # arrives, beside the remaining uploads (cb_als_desc.ready_events;
            # blocks are fitted independently: same results).  Device
            # allocations synchronise with copies in flight, so all of them (the
            # blocks' buffers, then the compression engine's) come before the
            # first copy.
            staged = (ranks is not None and late_exc is None and agree is None and len(scan) > 1
                      and all(_stageable(problem.tensors[g], shapes[k])
                              for k, g in enumerate(scan))
                      and als_staged_ok(shapes, ranks, self.code, self.als_compute_code, S_all))
            copy_stream = self.stream
            if staged:
                code = L.CB_F32 if prec == "fp32" else L.CB_F64
                self.dims = list(shapes)
                self.dev = [torch.empty(int(np.prod(d)), dtype=want, device=D.device())
                            for d in shapes]
                arrived = [torch.cuda.Event() for _ in scan]
                for ev in arrived:
                    ev.record(self.stream)      # creates the event; re-recorded after its copy
                tic = time.perf_counter()
                staged_fallback = False
                try:
                    self.als = AlsHandle(self.dev, self.dims, ranks, self.code, base.tol,
                                         base.max_iter, [base.seed + g for g in self.local], st,
                                         self.als_compute_code, S_all, ready_events=arrived)
                except ValueError as exc:
                    als_exc = exc
                except NotImplementedError:
                    # the staged plan did not fit: upload first, then a plain handle
                    staged_fallback = True
                t_als = time.perf_counter() - tic
                copy_stream = torch.cuda.Stream()
                copy_stream.wait_stream(self.stream)
                with torch.cuda.stream(copy_stream):
                    for k, g in enumerate(scan):
                        t = problem.tensors[g]
                        dst = self.dev[k]
                        dst.record_stream(copy_stream)
                        dst.copy_(t.as_strided((t.numel(),), (1,)), non_blocking=True)
                        arrived[k].record(copy_stream)
                        L.check(L.lib.cb_tensor_stats(code, D.ptr(dst), dst.numel(),
                                                      D.ptr(stats[k]), D.stream()))
                if staged_fallback:
                    copy_stream.synchronize()
                    tic = time.perf_counter()
                    try:
                        self.als = AlsHandle(self.dev, self.dims, ranks, self.code, base.tol,
                                             base.max_iter, [base.seed + g for g in self.local],
                                             st, self.als_compute_code, S_all)
                    except ValueError as exc:
                        als_exc = exc
                    t_als = 0.0
                elif self.als is not None:
                    tic = time.perf_counter()
                    try:
                        # sweeps of the blocks that are here while the rest uploads
                        self.als.run()
                        als_ran = True
                    except ValueError as exc:
                        als_exc = exc
                    t_als += time.perf_counter() - tic
            else:
                # uploads and element scans of the blocks before the first order
                # error, all enqueued, one synchronisation (stats slot per block)
                for k, g in enumerate(scan):
                    t = problem.tensors[g]
                    src, dims = D.tensor_to_dev(t, D.source_dtype(t))
                    code = L.CB_F32 if D.source_dtype(t) == "fp32" else L.CB_F64
                    L.check(L.lib.cb_tensor_stats(code, D.ptr(src), src.numel(), D.ptr(stats[k]),
                                                  D.stream()))
                    flat = src if D.source_dtype(t) == prec else D.cast_flat(src, prec)
                    del src
                    self.dev.append(flat)
                    self.dims.append(dims)
                # lra stage 1 setup (solver.py:556-573) before the value checks'
                # synchronisation: the ALS engine's allocations run beside
                # whatever part of the uploads is asynchronous
                tic = time.perf_counter()
                if ranks is not None and late_exc is None:
                    try:
                        self.als = AlsHandle(self.dev, self.dims, ranks, self.code, base.tol,
                                             base.max_iter, [base.seed + g for g in self.local],
                                             st, self.als_compute_code, S_all)
                    except ValueError as exc:
                        als_exc = exc
            copy_stream.synchronize()
            self.stream.wait_stream(copy_stream)
            host = stats.cpu().numpy() if scan else np.zeros((0, 3))
            for k, g in enumerate(scan):
                if host[k, 2] != 0.0 or host[k, 1] < 0.0:
                    which = "non-finite values" if host[k, 2] != 0.0 else "negative entries"
                    first_bad, bad_msg = (g, 1), ValueError(f"block {g} contains {which}")
                    break
            if agree is not None:
                first_bad, bad_msg = agree(first_bad, bad_msg, problem)
            if bad_msg is None:
                bad_msg = late_exc
            if bad_msg is not None:
                if self.als is not None:
                    self.als.close()
                    self.als = None
                raise bad_msg
        # lra stage 1: batched device ALS (solver.py:556-573)
        self.compress_seconds = 0.0
        tilde_ranks = None
        if problem.mode == "lra":
            with torch.cuda.stream(self.stream):
                try:
                    if als_exc is not None:
                        raise als_exc
                    if not als_ran:
                        self.als.run()
                except ValueError as exc:
                    msg = str(exc)
                    blk = 0
                    if msg.startswith("block "):
                        blk = self.local[int(msg.split()[1].rstrip(":"))]
                        msg = msg.split(": ", 1)[1]
                    if self.als is not None:
                        self.als.close()
                        self.als = None
                    raise ValueError(f"compression of block {blk} failed: {msg}") from exc
            self.stream.synchronize()
            # the sweep workspace (c5: ~37 GB of byte planes and scratch) goes
            # back before the solver engine allocates its own trace planes
            self.als.release_scratch()
            # staged: the engine setup plus the run that overlapped the uploads;
            # else from the setup (beside the upload's tail) to the last sweep
            self.compress_seconds = t_als if als_ran else time.perf_counter() - tic
            tilde_ranks = ranks
        # the seeded start of ALL blocks (one PCG64 stream), then this shard's
        start = init_factors(problem, opts.seed)
        self.start = start
        local_blocks = [start.blocks[g] for g in self.local]
        desc = L.SolverDesc()
        desc.n_blocks = S
        desc.order = N
        self._keep = []
        flat_dims = [d for dims in self.dims for d in dims]
        self._keep.append(L.i64_array(flat_dims))
        desc.dims = ctypes.cast(self._keep[-1], L.c_i64p)
        self._keep.append(L.int_array([problem.ranks[g] for g in self.local]))
        desc.ranks = ctypes.cast(self._keep[-1], L.c_ip)
        self._keep.append(L.int_array(problem.coupled_counts))
        desc.coupled = ctypes.cast(self._keep[-1], L.c_ip)
        desc.lra = 1 if problem.mode == "lra" else 0
        desc.update_core = 1 if problem.update_core else 0
        desc.dtype = self.code
        self._keep.append(L.ptr_array([D.ptr(x) for x in self.dev]))
        desc.tensors = ctypes.cast(self._keep[-1], ctypes.POINTER(L.c_vp))
        init_f = [np.ascontiguousarray(f) for b in local_blocks for f in b.factors]
        init_w = [np.ascontiguousarray(b.weights) for b in local_blocks]
        self._keep.extend([init_f, init_w])
        self._keep.append(L.dptr_array(init_f))
        desc.init_factors = ctypes.cast(self._keep[-1], ctypes.POINTER(L.c_dp))
        self._keep.append(L.dptr_array(init_w))
        desc.init_weights = ctypes.cast(self._keep[-1], ctypes.POINTER(L.c_dp))
        if self.als is not None:
            self._keep.append(L.int_array(tilde_ranks))
            desc.tilde_ranks = ctypes.cast(self._keep[-1], L.c_ip)
            tptrs = [self.als.factor_device_ptr(s, n) for s in range(S) for n in range(N)]
            self._keep.append((L.c_vp * len(tptrs))(*tptrs))
            desc.tilde_factors = ctypes.cast(self._keep[-1], ctypes.POINTER(L.c_dp))
            tw = [np.ones(r) for r in tilde_ranks]
            self._keep.append(tw)
            self._keep.append(L.dptr_array(tw))
            desc.tilde_weights = ctypes.cast(self._keep[-1], ctypes.POINTER(L.c_dp))
        desc.objective = 0 if objective_mode == "explicit" else 1
        desc.compute = self.compute_code
        desc.delta_w = float(opts.delta_w)
        desc.tol = float(opts.tol)
        desc.max_iter = int(opts.max_iter)
        sh = self.shard
        desc.world_size = sh.world
        desc.rank_id = sh.rank
        desc.nccl_comm = sh.comm
        desc.total_blocks = S_all
        desc.block_offset = sh.begin
        desc.pipeline = {"auto": 0, "on": 1, "off": 2}[opts.pipeline]
        desc.pipeline_reserve = int(opts.pipeline_reserve)
        self.t0 = time.perf_counter()
        self.engine = _Engine(desc, st)
        self.tilde_ranks = tilde_ranks

    def run(self, iters=None):
        iters = self.opts.max_iter if iters is None else iters
        return self.engine.run(iters)

    def collect_local(self):
        """Summary, histories and this shard's blocks (and compressions)."""
        summ = self.engine.summary()
        solve_seconds = time.perf_counter() - self.t0
        hist = self.engine.history(summ.n_iter + 1)
        blocks = {}
        for s, g in enumerate(self.local):
            facs, w = self.engine.block(s, self.dims[s], self.problem.ranks[g])
            blocks[g] = KruskalTensor(facs, w)
        compression = None
        if self.als is not None:
            compression = {}
            for s, g in enumerate(self.local):
                facs, _, _, its, _ = self.als.block(s)
                compression[g] = KruskalTensor(facs, np.ones(self.tilde_ranks[s]))
                compression[g].als_iters = its
        return summ, hist, blocks, compression, solve_seconds

    def collect(self):
        summ, hist, blocks, compression, secs = self.collect_local()
        return _assemble(self.problem, self.opts, summ, hist, blocks, compression, secs,
                         self.compress_seconds)

    def close(self):
        self.engine.close()
        if self.als is not None:
            self.als.close()


def _assemble(problem, opts, summ, hist, blocks, compression, solve_seconds, compress_seconds):
    """SolveResult from the device summary/histories and {global block: model}."""
    if summ.error == L.CB_ERR_NONFINITE:
        raise FloatingPointError(
            f"block {summ.error_block} produced a non-finite objective "
            f"at iteration {summ.error_iter}")
    n_iter = summ.n_iter
    oi, oo, rel, tns = hist
    trace = []
    for k in range(n_iter + 1):
        last = k == n_iter and k > 0
        if k == 0 or k % opts.trace_every == 0 or last:
            trace.append(TraceRow(k, float(oo[k]), float(rel[k]), float(tns[k]) * 1e-9))
    S = problem.n_blocks
    comp = None if compression is None else [compression[g] for g in range(S)]
    comp_iters = None if comp is None else [getattr(k, "als_iters", None) for k in comp]
    reason = "tolerance" if summ.reason == 1 else "max_iterations"
    return SolveResult(
        factors=CoupledFactorSet([blocks[g] for g in range(S)], list(problem.coupled_counts)),
        trace=trace, termination_reason=reason,
        objective_history=[float(v) for v in oi[: n_iter + 1]],
        rel_err_history=[float(v) for v in rel[: n_iter + 1]],
        n_iter=n_iter, n_restarts=summ.n_restarts, solve_seconds=solve_seconds,
        compress_seconds=compress_seconds, compression=comp, compression_iters=comp_iters)


# ---------------------------------------------------------------------------
# block sharding: one process per GPU, each owning a contiguous
# range of whole blocks; the couplings (per-mode Lipschitz sums, common-column
# gradient partials, per-block evaluation terms) are all-reduced in
# global-slot arrays, so every rank folds identical values in block order and
# a sharded solve reproduces the single-GPU bits.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ShardSpec:
    world: int
    rank: int
    begin: int      # first global block of this rank
    end: int        # one past the last
    comm: object    # ncclComm_t (int address) or None: emulated group


def shard_ranges(n_blocks, world):
    """Contiguous block ranges per rank: rank r owns [r*S//P, (r+1)*S//P)."""
    if world < 1 or world > n_blocks:
        raise ValueError(f"cannot shard {n_blocks} blocks over {world} ranks")
    return [(r * n_blocks // world, (r + 1) * n_blocks // world) for r in range(world)]


def solve_emulated_shards(problem, opts=None, world=2):
    """The block-sharded program on ONE GPU: `world` engine handles, one per
    emulated rank, stepped segment by segment with the all-reduces done by a
    summing kernel between segments (`cb_group_run`).  A verification tool
    for the multi-GPU code path; results must equal `solve` bit for bit."""
    torch = D.torch_mod()
    opts = opts if opts is not None else SolverOptions()
    stream = torch.cuda.Stream()
    parts = []
    try:
        for r, (b, e) in enumerate(shard_ranges(problem.n_blocks, world)):
            parts.append(PreparedSolve(problem, opts, stream=stream,
                                       shard=ShardSpec(world, r, b, e, None)))
        hs = (L.c_vp * world)(*[p.engine.h.value for p in parts])
        summ = L.SolverSummary()
        L.check(L.lib.cb_group_run(hs, world, int(opts.max_iter), ctypes.byref(summ)))
        blocks, comp = {}, ({} if parts[0].als is not None else None)
        hist, secs = None, 0.0
        for p in parts:
            s_, h_, b_, c_, t_ = p.collect_local()
            blocks.update(b_)
            if comp is not None:
                comp.update(c_)
            if hist is None:
                summ, hist, secs = s_, h_, t_
        return _assemble(problem, opts, summ, hist, blocks, comp, secs,
                         sum(p.compress_seconds for p in parts))
    finally:
        for p in parts:
            p.close()


def _agree_first_error(first_bad, msg, problem, group):
    """Every rank raises the group's first validation error in the
    reference's order: the smallest block, an order error before a value
    error of the same block (only the owner of a block scans its values)."""
    import torch
    import torch.distributed as dist
    code = 2 * problem.n_blocks if first_bad is None else 2 * first_bad[0] + first_bad[1]
    t = torch.tensor([code], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    best = int(t.item())
    if best >= 2 * problem.n_blocks:
        return None, None
    g, kind = divmod(best, 2)
    if kind == 0:
        # every rank checks every block's order: all found it themselves
        return (g, 0), ValueError(f"block {g} has order {problem.tensors[g].ndim}, "
                                  f"expected {problem.tensors[0].ndim}")
    # a value error, found by the rank owning block g: one more exchange
    # tells the others which of the two checks failed (same message as
    # _raise_values on every rank)
    mine = first_bad is not None and first_bad == (g, 1)
    kinds = torch.tensor([(1 if "non-finite" in str(msg) else 2) if mine else 0],
                         dtype=torch.int64, device="cuda")
    dist.all_reduce(kinds, op=dist.ReduceOp.MAX, group=group)
    which = "contains non-finite values" if int(kinds.item()) == 1 else "contains negative entries"
    return (g, 1), ValueError(f"block {g} {which}")


def nccl_comm_for(group=None):
    """An NCCL communicator over the ranks of a torch.distributed group, built
    from a unique id that rank 0 creates and broadcasts (object collective)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        L.check(L.lib.cb_nccl_unique_id(uid))
    box = [bytes(uid.raw) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    uid = ctypes.create_string_buffer(box[0], 128)
    comm = L.c_vp()
    L.check(L.lib.cb_nccl_comm_init(uid, world, rank, ctypes.byref(comm)))
    return comm.value


class PreparedShardedSolve:
    """This rank's part of a block-sharded solve (torch.distributed initialised,
    one process per GPU).  `run`/`step_async` behave as in PreparedSolve; every
    rank must make the same calls."""

    def __init__(self, problem, opts=None, group=None):
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.group = group
        # a communicator even for one rank: the sharded program (exchanges in
        # the iteration graph) then runs on a single GPU too
        self.comm = nccl_comm_for(group)
        b, e = shard_ranges(problem.n_blocks, world)[rank]
        self.inner = PreparedSolve(problem, opts, shard=ShardSpec(world, rank, b, e, self.comm),
                                   agree=lambda fb, msg, prob: _agree_first_error(fb, msg, prob, group))
        self.engine, self.stream = self.inner.engine, self.inner.stream

    def run(self, iters=None):
        return self.inner.run(iters)

    def collect(self):
        """The full SolveResult on every rank (blocks gathered over the group)."""
        import torch.distributed as dist
        summ, hist, blocks, comp, secs = self.inner.collect_local()
        world = dist.get_world_size(self.group)
        if world == 1:
            merged_b, merged_c = blocks, comp
        else:
            got = [None] * world
            dist.all_gather_object(got, (blocks, comp), group=self.group)
            merged_b, merged_c = {}, (None if comp is None else {})
            for b_, c_ in got:
                merged_b.update(b_)
                if merged_c is not None:
                    merged_c.update(c_)
        return _assemble(self.inner.problem, self.inner.opts, summ, hist, merged_b, merged_c,
                         secs, self.inner.compress_seconds)

    def close(self):
        self.inner.close()
        if self.comm is not None:
            L.lib.cb_nccl_comm_destroy(L.c_vp(self.comm))
            self.comm = None


def solve_distributed(problem, opts=None, group=None):
    """Block-sharded `solve` over the ranks of a torch.distributed group (one
    process per GPU, NCCL over NVLink for the couplings).  Every rank passes
    the same problem and options and receives the full SolveResult."""
    run = PreparedShardedSolve(problem, opts, group)
    try:
        run.run()
        return run.collect()
    finally:
        run.close()


def solve(problem, opts=None):
    """Run the coupled decomposition on the GPU (drop-in for solver.py:546-624).

    Stops when the original-tensor relative error changes by less than
    ``opts.tol`` ("tolerance") or after ``opts.max_iter`` iterations
    ("max_iterations").
    """
    run = PreparedSolve(problem, opts)
    try:
        run.run()
        return run.collect()
    finally:
        run.close()
