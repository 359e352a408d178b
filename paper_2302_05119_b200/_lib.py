"""ctypes binding of the C ABI (include/concpd_b200.h) — the only path to compute.

The shared library is built in-tree (``make -C paper_2302_05119_b200/csrc``,
or ``__graft_entry__.build()``) for sm_100a.  There is no CPU fallback: if the
library is missing the import fails, and if no CUDA device is present every
compute call raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CONCPD_B200_LIB", os.path.join(_HERE, "libconcpd_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"concpd_b200 native library not found at {LIB_PATH}; build it with "
        "`make -C paper_2302_05119_b200/csrc` (no CPU fallback exists)")

lib = ctypes.CDLL(LIB_PATH)

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_ip = ctypes.POINTER(ctypes.c_int)

CB_OK, CB_ERR_ARG, CB_ERR_CUDA, CB_ERR_NONFINITE, CB_ERR_UNSUPPORTED, CB_ERR_DIVERGED, \
    CB_ERR_STATE = range(7)
CB_F32, CB_F64 = 0, 1


class SolverDesc(ctypes.Structure):
    _fields_ = [
        ("n_blocks", c_int), ("order", c_int), ("dims", c_i64p), ("ranks", c_ip),
        ("coupled", c_ip), ("lra", c_int), ("update_core", c_int), ("dtype", c_int),
        ("tensors", ctypes.POINTER(c_vp)), ("init_factors", ctypes.POINTER(c_dp)),
        ("init_weights", ctypes.POINTER(c_dp)), ("tilde_ranks", c_ip),
        ("tilde_factors", ctypes.POINTER(c_dp)), ("tilde_weights", ctypes.POINTER(c_dp)),
        ("objective", c_int), ("compute", c_int), ("delta_w", c_dbl), ("tol", c_dbl), ("max_iter", c_int),
        ("world_size", c_int), ("rank_id", c_int), ("nccl_comm", c_vp),
        ("total_blocks", c_int), ("block_offset", c_int), ("pipeline", c_int),
        ("pipeline_reserve", c_int),
    ]


class SolverSummary(ctypes.Structure):
    _fields_ = [("n_iter", c_int), ("n_restarts", c_int), ("done", c_int), ("reason", c_int),
                ("error", c_int), ("error_block", c_int), ("error_iter", c_int)]


class AlsDesc(ctypes.Structure):
    _fields_ = [("n_blocks", c_int), ("order", c_int), ("dims", c_i64p), ("ranks", c_ip),
                ("dtype", c_int), ("tensors", ctypes.POINTER(c_vp)),
                ("init", ctypes.POINTER(c_dp)), ("tol", c_dbl), ("max_iter", c_int),
                ("compute", c_int), ("total_blocks", c_int),
                ("ready_events", ctypes.POINTER(c_vp))]


def _sig(name, res, args):
    fn = getattr(lib, name, None)
    if fn is None:
        return None
    fn.restype = res
    fn.argtypes = args
    return fn


_sig("cb_last_error", ctypes.c_char_p, [])
_sig("cb_abi_version", c_int, [])
_sig("cb_launch_count", ctypes.c_longlong, [])
_sig("cb_launch_count_reset", None, [])
_sig("cb_mttkrp", c_int, [c_int, c_vp, c_int, c_i64p, ctypes.POINTER(c_vp), c_int, c_int, c_vp, c_vp])
_sig("cb_core_linear_term_tc", c_int, [c_int, ctypes.POINTER(c_vp), c_i64p, ctypes.POINTER(c_vp),
                                        c_ip, c_vp, c_vp])
_sig("cb_khatri_rao", c_int, [ctypes.POINTER(c_vp), c_int, c_i64p, c_int, c_vp, c_vp])
_sig("cb_hadamard_gram", c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i64p, c_int, c_int,
                                 c_int, c_int, c_vp, c_vp])
_sig("cb_spectral_norm_batched", c_int, [c_vp, c_int, c_int, c_vp, c_vp])
_sig("cb_tensor_stats", c_int, [c_int, c_vp, c_i64, c_vp, c_vp])
_sig("cb_kruskal_residual", c_int, [c_int, c_vp, c_int, c_i64p, ctypes.POINTER(c_vp), c_vp, c_int,
                                    c_vp, c_vp])
_sig("cb_rowdot", c_int, [c_vp, c_vp, c_i64, c_int, c_vp, c_vp])
_sig("cb_gemm", c_int, [c_int, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_int, c_vp, c_int, c_dbl,
                        c_vp, c_int, c_vp])
_sig("cb_factor_gradient", c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_vp])
_sig("cb_synth_stats", c_int, [c_int, c_i64p, ctypes.POINTER(c_vp), c_vp, c_int, c_vp, c_vp])
_sig("cb_synth_fill", c_int, [c_int, c_vp, c_int, c_i64p, ctypes.POINTER(c_vp), c_vp, c_int, c_dbl,
                              c_int, c_dbl, ctypes.c_uint64, c_int, c_vp])
_sig("cb_model_residual", c_int, [c_int, c_vp, c_int, c_i64p, ctypes.POINTER(c_vp), c_vp, c_int,
                                  c_vp, c_vp])
_sig("cb_diff_sq", c_int, [c_int, c_vp, c_int, c_vp, c_i64, c_vp, c_vp])
_sig("cb_performance_index", c_int, [c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i64p,
                                     c_int, c_vp, c_vp, c_vp])
_sig("cb_als_create", c_int, [ctypes.POINTER(AlsDesc), c_vp, ctypes.POINTER(c_vp)])
_sig("cb_als_staged_ok", c_int, [ctypes.POINTER(AlsDesc)])
_sig("cb_als_release_scratch", c_int, [c_vp])
_sig("cb_als_run", c_int, [c_vp])
_sig("cb_als_block_result", c_int, [c_vp, c_int, c_dp, c_ip, c_ip, c_dp, ctypes.POINTER(c_dp)])
_sig("cb_als_factor_device", c_vp, [c_vp, c_int, c_int])
_sig("cb_als_destroy", c_int, [c_vp])
_sig("cb_solver_create", c_int, [ctypes.POINTER(SolverDesc), c_vp, ctypes.POINTER(c_vp)])
_sig("cb_solver_run", c_int, [c_vp, c_int, ctypes.POINTER(SolverSummary)])
_sig("cb_solver_step_async", c_int, [c_vp])
_sig("cb_solver_summary_get", c_int, [c_vp, ctypes.POINTER(SolverSummary)])
_sig("cb_solver_history", c_int, [c_vp, c_dp, c_dp, c_dp, c_dp, c_int])
_sig("cb_solver_block_factors", c_int, [c_vp, c_int, ctypes.POINTER(c_dp), c_dp])
_sig("cb_solver_set_timing", c_int, [c_vp, c_int])
_sig("cb_solver_profile", c_int, [c_vp, c_int, ctypes.c_char_p, c_int])
_sig("cb_solver_timing", c_int, [c_vp, c_int, c_dp, ctypes.POINTER(ctypes.c_longlong), c_dp])
_sig("cb_solver_timeline", c_int, [c_vp, c_int, ctypes.POINTER(ctypes.c_ulonglong), c_int])
_sig("cb_solver_destroy", c_int, [c_vp])
_sig("cb_group_step", c_int, [ctypes.POINTER(c_vp), c_int, c_int])
_sig("cb_group_run", c_int, [ctypes.POINTER(c_vp), c_int, c_int, ctypes.POINTER(SolverSummary)])
_sig("cb_nccl_unique_id", c_int, [c_vp])
_sig("cb_nccl_comm_init", c_int, [c_vp, c_int, c_int, ctypes.POINTER(c_vp)])
_sig("cb_nccl_comm_destroy", c_int, [c_vp])

# every symbol the header declares (checked by tests/test_boundary.py)
EXPORTED = [
    "cb_last_error", "cb_abi_version", "cb_launch_count", "cb_launch_count_reset",
    "cb_mttkrp", "cb_core_linear_term_tc", "cb_khatri_rao", "cb_hadamard_gram", "cb_spectral_norm_batched",
    "cb_tensor_stats", "cb_kruskal_residual", "cb_rowdot", "cb_gemm", "cb_factor_gradient",
    "cb_synth_stats", "cb_synth_fill", "cb_model_residual", "cb_diff_sq",
    "cb_performance_index",
    "cb_als_create", "cb_als_staged_ok", "cb_als_release_scratch", "cb_als_run", "cb_als_block_result", "cb_als_factor_device",
    "cb_als_destroy", "cb_solver_create", "cb_solver_run", "cb_solver_step_async",
    "cb_solver_summary_get", "cb_solver_history", "cb_solver_block_factors",
    "cb_solver_set_timing", "cb_solver_timing", "cb_solver_profile", "cb_solver_timeline",
    "cb_solver_destroy",
    "cb_group_step", "cb_group_run", "cb_nccl_unique_id",
    "cb_nccl_comm_init", "cb_nccl_comm_destroy",
]


def last_error():
    msg = lib.cb_last_error()
    return msg.decode() if msg else ""


def check(rc, what=""):
    """Map a cb_status to the reference's exception types."""
    if rc == CB_OK:
        return
    msg = last_error() or what
    if rc in (CB_ERR_ARG, CB_ERR_DIVERGED):
        raise ValueError(msg)
    if rc == CB_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if rc == CB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"concpd_b200 failure ({rc}): {msg}")


def i64_array(values):
    arr = (c_i64 * len(values))(*[int(v) for v in values])
    return arr


def int_array(values):
    return (c_int * len(values))(*[int(v) for v in values])


def ptr_array(ptrs):
    return (c_vp * len(ptrs))(*[int(p) if p else None for p in ptrs])


def dptr_array(arrays):
    """Host array of host double* for numpy float64 C-contiguous arrays."""
    return (c_dp * len(arrays))(*[a.ctypes.data_as(c_dp) for a in arrays])


def launch_count():
    return int(lib.cb_launch_count())


def launch_count_reset():
    lib.cb_launch_count_reset()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("concpd_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def stream_handle(torch_mod=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def as_f64_c(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))
