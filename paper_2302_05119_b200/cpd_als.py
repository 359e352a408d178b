"""CP-ALS compression stage on the GPU (drop-in for `pkg/src/concpd/cpd_als.py`).

``cpd_als(t, opts)`` keeps the reference signature and result type
(cpd_als.py:17-120); the sweeps run in the batched device engine
(`cb_als_*`, csrc/als.cu).  ``als_compress_blocks`` is the batched form used
by lraCoNCPD-APG: every block is an independent fit with its own stop rule,
all advanced by the same kernel launches.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib as L
from .kruskal import KruskalTensor

__all__ = ["AlsOptions", "AlsResult", "cpd_als", "als_compress_blocks"]


@dataclass
class AlsOptions:
    """Settings of the compression fit (cpd_als.py:20-40).

    ``rank=None`` means "the block's target rank" when used by the solver; it
    must be resolved before calling :func:`cpd_als` directly.
    """

    rank: int = None
    tol: float = 1e-4
    max_iter: int = 200
    seed: int = 0

    def __post_init__(self):
        if self.rank is not None and self.rank < 1:
            raise ValueError(f"rank must be >= 1, got {self.rank}")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iter < 0:
            raise ValueError("max_iter must be >= 0")


@dataclass
class AlsResult:
    model: KruskalTensor
    rel_err: float
    rel_err_history: list = field(repr=False)
    n_iter: int = 0
    converged: bool = False


def _check_feasible(dims, rank):
    total = int(np.prod(dims))
    for n, d in enumerate(dims):
        other = total // d if d else 0
        if rank > other:
            raise ValueError(f"rank {rank} infeasible: mode-{n} system has only {other} rows")


def als_staged_ok(dims_list, ranks, dtype_code, compute_code=0, total_blocks=0):
    """Would the batched ALS start these blocks one by one at their upload
    events (`cb_als_staged_ok`)?  Only then may the uploads be enqueued after
    the engine has been created."""
    desc = L.AlsDesc()
    desc.n_blocks = len(dims_list)
    desc.order = len(dims_list[0])
    dims_c = L.i64_array([d for dims in dims_list for d in dims])
    ranks_c = L.int_array(ranks)
    desc.dims = ctypes.cast(dims_c, L.c_i64p)
    desc.ranks = ctypes.cast(ranks_c, L.c_ip)
    desc.dtype = dtype_code
    desc.compute = int(compute_code)
    desc.total_blocks = int(total_blocks or 0)
    return bool(L.lib.cb_als_staged_ok(ctypes.byref(desc)))


class AlsHandle:
    """Owns a device ALS engine; factors stay resident for the solver."""

    def __init__(self, dev_tensors, dims_list, ranks, dtype_code, tol, max_iter, seeds, stream,
                 compute_code=0, total_blocks=0, ready_events=None):
        self.S = len(dev_tensors)
        self.N = len(dims_list[0])
        self.dims = dims_list
        self.ranks = ranks
        self.max_iter = max_iter
        self._keep = list(dev_tensors)
        # initial factors: default_rng(seed).random((d, R)) per mode (cpd_als.py:81-82)
        self.init = []
        for s in range(self.S):
            gen = np.random.default_rng(seeds[s])
            self.init.extend(np.ascontiguousarray(gen.random((d, ranks[s]))) for d in dims_list[s])
        desc = L.AlsDesc()
        desc.n_blocks = self.S
        desc.order = self.N
        flat_dims = [d for dims in dims_list for d in dims]
        self._dims_c = L.i64_array(flat_dims)
        self._ranks_c = L.int_array(ranks)
        self._x_c = L.ptr_array([D.ptr(x) for x in dev_tensors])
        self._init_c = L.dptr_array(self.init)
        desc.dims = ctypes.cast(self._dims_c, L.c_i64p)
        desc.ranks = ctypes.cast(self._ranks_c, L.c_ip)
        desc.dtype = dtype_code
        desc.tensors = ctypes.cast(self._x_c, ctypes.POINTER(L.c_vp))
        desc.init = ctypes.cast(self._init_c, ctypes.POINTER(L.c_dp))
        desc.tol = float(tol)
        desc.max_iter = int(max_iter)
        desc.compute = int(compute_code)
        desc.total_blocks = int(total_blocks or 0)
        # per-block upload events (torch.cuda.Event, recorded on the copy
        # stream after each block's host->device copy): run() then starts
        # every block as it arrives
        self._events = list(ready_events) if ready_events is not None else None
        if self._events is not None:
            self._events_c = (L.c_vp * self.S)(*[L.c_vp(int(e.cuda_event)) for e in self._events])
            desc.ready_events = ctypes.cast(self._events_c, ctypes.POINTER(L.c_vp))
        h = L.c_vp()
        L.check(L.lib.cb_als_create(ctypes.byref(desc), stream, ctypes.byref(h)))
        self.h = h

    def run(self):
        L.check(L.lib.cb_als_run(self.h))

    def release_scratch(self):
        """Free the sweep workspace (byte planes, GEMM scratch); the fitted
        factors stay on the device for the solver."""
        L.check(L.lib.cb_als_release_scratch(self.h))

    def block(self, s):
        rel = ctypes.c_double()
        it = ctypes.c_int()
        conv = ctypes.c_int()
        hist = np.zeros(max(self.max_iter, 1))
        facs = [np.zeros((d, self.ranks[s])) for d in self.dims[s]]
        L.check(L.lib.cb_als_block_result(self.h, s, ctypes.byref(rel), ctypes.byref(it),
                                          ctypes.byref(conv), hist.ctypes.data_as(L.c_dp),
                                          L.dptr_array(facs)))
        return facs, float(rel.value), list(hist[: it.value]), int(it.value), bool(conv.value)

    def factor_device_ptr(self, s, n):
        return L.lib.cb_als_factor_device(self.h, s, n)

    def close(self):
        if getattr(self, "h", None) and L is not None and getattr(L, "lib", None) is not None:
            L.lib.cb_als_destroy(self.h)
        self.h = None

    def __del__(self):
        self.close()


def als_compress_blocks(dev_tensors, dims_list, ranks, tol, max_iter, seeds, dtype_code, stream,
                        compute_code=0, total_blocks=0):
    """Batched ALS over blocks; returns the live handle (factors on device).
    ``total_blocks``: blocks of the whole problem when this is one shard."""
    h = AlsHandle(dev_tensors, dims_list, ranks, dtype_code, tol, max_iter, seeds, stream,
                  compute_code, total_blocks)
    h.run()
    return h


def cpd_als(t, opts):
    """Fit an unconstrained rank-``opts.rank`` CP model to ``t`` on the GPU.

    Same contract as the reference (cpd_als.py:52-120): ValueError for
    non-finite input, an unresolved or infeasible rank, or divergence; the
    returned model has unit weights and the reported RelErr is the explicit
    residual norm ratio.
    """
    torch = D.torch_mod()
    t = np.asarray(t, dtype=float)
    if not np.isfinite(t).all():
        raise ValueError("tensor contains non-finite values")
    if opts.rank is None:
        raise ValueError("AlsOptions.rank was not resolved to an integer")
    rank = int(opts.rank)
    _check_feasible(t.shape, rank)
    dev, dims = D.tensor_to_dev(t, "fp64")
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        h = als_compress_blocks([dev], [dims], [rank], opts.tol, opts.max_iter, [opts.seed],
                                L.CB_F64, L.c_vp(stream.cuda_stream))
        facs, rel, hist, n_iter, conv = h.block(0)
        h.close()
    return AlsResult(KruskalTensor(facs, np.ones(rank)), rel, hist, n_iter=n_iter,
                     converged=conv)
