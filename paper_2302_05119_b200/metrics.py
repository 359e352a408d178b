"""Decomposition quality metrics on the GPU (`pkg/src/concpd/metrics.py:71-156`).

Same names, arguments, results and error messages as the reference's
``MetricReport``, ``rel_err``, ``ten_fit``, ``performance_index``,
``pi_per_mode`` and ``psnr``.  The tensor-sized work streams on the device:

* ``rel_err`` / ``ten_fit`` / ``psnr`` accept, for the recovered side, either
  dense tensors (numpy or torch; ``cb_diff_sq``) or Kruskal models
  (``KruskalTensor``; ``cb_model_residual`` evaluates ||M - [[lam; U]]||^2
  with the generator's tiled reconstruction, so a c5 block's 256 MB model is
  never formed).  The reference takes dense reconstructions
  (`cli.py:324`: ``[reconstruct(b) for b in blocks]``); passing the models is
  the device-native form of the same call.
* ``performance_index`` / ``pi_per_mode``: pinv(E) T as (E^T E)^{-1} E^T T,
  fp64 grams and an LU solve per (estimate, truth) pair in one launch for all
  pairs (``cb_performance_index``); equal to the reference's SVD-based pinv
  to ~cond(E)^2 x 1e-16 for full-column-rank estimates.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib as L
from .kruskal import KruskalTensor

__all__ = ["MetricReport", "rel_err", "ten_fit", "performance_index", "pi_per_mode", "psnr",
           "PSNR_CAP_DB"]

PSNR_CAP_DB = 99.0


@dataclass
class MetricReport:
    """Flat record of the per-run quality numbers (metrics.py:31-48)."""

    rel_err: float
    ten_fit: float
    obj_fun: float
    pi_per_mode: list
    elapsed_seconds: float
    psnr: float = None
    mcc: float = None


def _shape(x):
    if isinstance(x, KruskalTensor):
        return tuple(int(d) for d in x.dims)
    return tuple(int(d) for d in x.shape)


def _dev_flat(t):
    """Flat first-index-fastest device copy of a dense tensor in its own
    dtype (fp32 stays fp32), with its cb_dtype code."""
    flat, _ = D.tensor_to_dev(t, D.source_dtype(t))
    return flat, (L.CB_F32 if D.source_dtype(t) == "fp32" else L.CB_F64)


def _sq_pair(m, m_hat):
    """(||m - m_hat||^2, ||m||^2) on the device."""
    torch = D.torch_mod()
    x, code = _dev_flat(m)
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    if isinstance(m_hat, KruskalTensor):
        dims = L.i64_array(_shape(m))
        dev = [D.to_dev_f64(f) for f in m_hat.factors]
        w = D.to_dev_f64(m_hat.weights)
        L.check(L.lib.cb_model_residual(code, D.ptr(x), len(dev), dims,
                                        L.ptr_array([D.ptr(f) for f in dev]), D.ptr(w),
                                        m_hat.rank, D.ptr(out), D.stream()))
    else:
        y, ycode = _dev_flat(m_hat)
        L.check(L.lib.cb_diff_sq(code, D.ptr(x), ycode, D.ptr(y), x.numel(), D.ptr(out),
                                 D.stream()))
    d2, a2 = (float(v) for v in out.cpu())
    return d2, a2


def _norm_ratios(originals, recovered):
    if len(originals) != len(recovered):
        raise ValueError(f"{len(originals)} original blocks vs {len(recovered)} recovered")
    ratios = []
    for s, (m, m_hat) in enumerate(zip(originals, recovered)):
        if _shape(m) != _shape(m_hat):
            raise ValueError(f"block {s}: original shape {_shape(m)} != recovered {_shape(m_hat)}")
        d2, a2 = _sq_pair(m, m_hat)
        denom = float(np.sqrt(a2))
        ratios.append(0.0 if denom == 0.0 else float(np.sqrt(d2)) / denom)
    return ratios


def rel_err(originals, recovered):
    """Averaged relative reconstruction error over the blocks (metrics.py:71-76);
    zero-norm blocks contribute 0."""
    ratios = _norm_ratios(originals, recovered)
    return float(sum(ratios) / len(ratios))


def ten_fit(originals, recovered):
    """1 - rel_err (metrics.py:79-81)."""
    return 1.0 - rel_err(originals, recovered)


def _pi_batch(pairs):
    """Performance indices of (estimated, truth) matrix pairs of one rank in
    one launch; returns (values, deficient flags)."""
    torch = D.torch_mod()
    rank = int(np.asarray(pairs[0][1]).shape[1])
    es = [D.to_dev_f64(e) for e, _ in pairs]
    ts = [D.to_dev_f64(t) for _, t in pairs]
    out = torch.empty(len(pairs), dtype=torch.float64, device=es[0].device)
    bad = torch.empty(len(pairs), dtype=torch.int32, device=es[0].device)
    L.check(L.lib.cb_performance_index(len(pairs), L.ptr_array([D.ptr(x) for x in es]),
                                       L.ptr_array([D.ptr(x) for x in ts]),
                                       L.i64_array([e.shape[0] for e in es]), rank, D.ptr(out),
                                       D.ptr(bad), D.stream()))
    return [float(v) for v in out.cpu()], [bool(v) for v in bad.cpu()]


def _pi_checks(estimated, truth):
    estimated = np.asarray(estimated, dtype=float)
    truth = np.asarray(truth, dtype=float)
    if estimated.shape != truth.shape:
        raise ValueError(f"estimated shape {estimated.shape} != truth {truth.shape}")
    if truth.shape[1] == 1:
        raise ValueError("performance index is undefined for a single component")
    return estimated, truth


def _warn_deficient():
    warnings.warn("estimated factor matrix is rank-deficient; performance index is unreliable",
                  RuntimeWarning, stacklevel=3)


def performance_index(estimated, truth):
    """Permutation/scale-invariant recovery error of a factor matrix
    (metrics.py:84-124); exactly 0 when the estimate spans the truth column
    for column in any order and scaling."""
    estimated, truth = _pi_checks(estimated, truth)
    vals, bad = _pi_batch([(estimated, truth)])
    if bad[0]:
        _warn_deficient()
    return vals[0]


def pi_per_mode(estimated, truth):
    """Block-averaged performance index per mode (metrics.py:127-137); every
    (block, mode) pair of a rank in one launch."""
    if len(estimated.blocks) != len(truth.blocks):
        raise ValueError(f"{len(estimated.blocks)} estimated blocks vs {len(truth.blocks)}")
    order = truth.blocks[0].order
    pairs, where = [], []
    for n in range(order):
        for e, t in zip(estimated.blocks, truth.blocks):
            pairs.append(_pi_checks(e.factors[n], t.factors[n]))
            where.append(n)
    vals = [0.0] * len(pairs)
    by_rank = {}
    for i, (e, _) in enumerate(pairs):
        by_rank.setdefault(e.shape[1], []).append(i)
    for idx in by_rank.values():
        v, bad = _pi_batch([pairs[i] for i in idx])
        if any(bad):
            _warn_deficient()
        for i, x in zip(idx, v):
            vals[i] = x
    return [float(np.mean([v for v, w in zip(vals, where) if w == n])) for n in range(order)]


def psnr(original, recovered, peak=255.0):
    """Peak signal-to-noise ratio in dB, capped at 99 (metrics.py:140-156)."""
    if _shape(original) != _shape(recovered):
        raise ValueError(f"original shape {_shape(original)} != recovered {_shape(recovered)}")
    if peak <= 0:
        raise ValueError("peak must be positive")
    d2, _ = _sq_pair(original, recovered)
    mse = d2 / float(np.prod(_shape(original)))
    if mse == 0.0:
        return PSNR_CAP_DB
    return float(min(10.0 * np.log10(peak * peak / mse), PSNR_CAP_DB))
