"""Tensor algebra operators of the reference (`pkg/src/concpd/tensor_ops.py`).

Layout conventions (tensor_ops.py:1-15) are kept exactly: first-index-fastest
vectorization, mode-n unfoldings with the remaining modes ascending (lower
fastest), Khatri-Rao products with the first matrix slowest and
``factors_khatri_rao`` in descending mode order.

``vectorize``/``unvectorize``/``matricize``/``refold`` are pure index
relabellings (no arithmetic) and are expressed as numpy reshapes.  The
arithmetic operators — ``khatri_rao``, ``factors_khatri_rao``,
``hadamard_gram``, ``spectral_norm`` — run on the GPU through the C ABI.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _lib as L

__all__ = [
    "vectorize", "unvectorize", "matricize", "refold", "khatri_rao",
    "factors_khatri_rao", "hadamard_gram", "spectral_norm",
]


def vectorize(t):
    """First-index-fastest vectorization (tensor_ops.py:31-33)."""
    return np.asarray(t).reshape(-1, order="F")


def unvectorize(v, dims):
    """Inverse of :func:`vectorize` (tensor_ops.py:36-42)."""
    v = np.asarray(v)
    dims = tuple(int(d) for d in dims)
    if v.size != int(np.prod(dims)):
        raise ValueError(f"vector of length {v.size} cannot fill dims {dims}")
    return v.reshape(dims, order="F")


def matricize(t, mode):
    """Mode-``mode`` unfolding (tensor_ops.py:45-54)."""
    t = np.asarray(t)
    if not 0 <= mode < t.ndim:
        raise ValueError(f"mode {mode} out of range for order-{t.ndim} tensor")
    return np.moveaxis(t, mode, 0).reshape((t.shape[mode], -1), order="F")


def refold(m, mode, dims):
    """Inverse of :func:`matricize` (tensor_ops.py:57-63)."""
    dims = tuple(int(d) for d in dims)
    if not 0 <= mode < len(dims):
        raise ValueError(f"mode {mode} out of range for dims {dims}")
    lead = (dims[mode],) + tuple(d for k, d in enumerate(dims) if k != mode)
    return np.moveaxis(np.asarray(m).reshape(lead, order="F"), 0, mode)


def khatri_rao(mats):
    """Column-wise Kronecker product, first matrix slowest — on the GPU
    (`cb_khatri_rao`; replaces tensor_ops.py:66-85)."""
    mats = [np.asarray(m) for m in mats]
    if not mats:
        raise ValueError("khatri_rao needs at least one matrix")
    ncols = mats[0].shape[1]
    if any(m.shape[1] != ncols for m in mats[1:]):
        raise ValueError(f"column counts differ: {[m.shape[1] for m in mats]}")
    if len(mats) > 8:
        raise ValueError("khatri_rao supports at most 8 matrices")
    torch = D.torch_mod()
    rows = [m.shape[0] for m in mats]
    nrows = int(np.prod(rows))
    if ncols == 0 or nrows == 0:
        return np.zeros((nrows, ncols))
    dev = [D.to_dev_f64(m) for m in mats]
    out = torch.empty((nrows, ncols), dtype=torch.float64, device=dev[0].device)
    L.check(L.lib.cb_khatri_rao(L.ptr_array([D.ptr(x) for x in dev]), len(dev),
                                L.i64_array(rows), ncols, D.ptr(out), D.stream()))
    return D.to_host(out)


def factors_khatri_rao(factors, skip=None):
    """Khatri-Rao of the factors in descending mode order (tensor_ops.py:88-95)."""
    mats = [f for k, f in enumerate(factors) if k != skip]
    return khatri_rao(mats[::-1])


def hadamard_gram(mats, skip=None, mats2=None):
    """Element-wise product over modes of ``mats[n].T @ mats2[n]`` — on the GPU
    (`cb_hadamard_gram`; replaces tensor_ops.py:98-124)."""
    if mats2 is None:
        mats2 = mats
    if len(mats) != len(mats2):
        raise ValueError("mats and mats2 must have the same length")
    mats = [np.asarray(a, dtype=float) for a in mats]
    mats2 = [np.asarray(b, dtype=float) for b in mats2]
    kept = [k for k in range(len(mats)) if k != skip]
    if not kept:
        raise ValueError("no matrices left after skip")
    shape = None
    for k in kept:
        if mats[k].shape[0] != mats2[k].shape[0]:
            raise ValueError(f"row counts differ in mode {k}")
        s = (mats[k].shape[1], mats2[k].shape[1])
        if shape is None:
            shape = s
        elif s != shape:
            raise ValueError(f"gram shapes differ: {shape} vs {s}")
    torch = D.torch_mod()
    da = [D.to_dev_f64(a) for a in mats]
    db = da if mats2 is mats else [D.to_dev_f64(b) for b in mats2]
    # kernels need consistent column counts per mode; skipped modes may differ
    for k in range(len(mats)):
        if k not in kept:
            da[k] = da[kept[0]]
            db[k] = db[kept[0]]
    rows = [int(da[k].shape[0]) for k in range(len(mats))]
    out = torch.empty(shape, dtype=torch.float64, device=da[kept[0]].device)
    L.check(L.lib.cb_hadamard_gram(L.ptr_array([D.ptr(x) for x in da]),
                                   L.ptr_array([D.ptr(x) for x in db]), L.i64_array(rows),
                                   len(mats), -1 if skip is None else int(skip),
                                   shape[0], shape[1], D.ptr(out), D.stream()))
    return D.to_host(out)


def spectral_norm(g):
    """Largest eigenvalue of a symmetric PSD matrix (0 for the zero matrix),
    on the GPU (`cb_spectral_norm_batched`; replaces tensor_ops.py:127-140)."""
    g = np.asarray(g, dtype=float)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {g.shape}")
    if g.shape[0] == 0:
        return 0.0
    return float(spectral_norm_batched(g[None])[0])


def spectral_norm_batched(gs):
    """lambda_max of each matrix of a (batch, R, R) stack (R <= 64)."""
    gs = np.asarray(gs, dtype=float)
    torch = D.torch_mod()
    dg = D.to_dev_f64(gs)
    out = torch.empty(gs.shape[0], dtype=torch.float64, device=dg.device)
    L.check(L.lib.cb_spectral_norm_batched(D.ptr(dg), gs.shape[1], gs.shape[0], D.ptr(out),
                                           D.stream()))
    return D.to_host(out)
