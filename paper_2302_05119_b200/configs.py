"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference measures on real datasets that are not available here (Yale B,
ERP; `PAPER.md:358-359`, `PAPER.md:406`).  Seeded synthetic inputs with the
shapes and value distributions BASELINE.json names stand in for them.

Seeding follows the reference generator's SeedSequence scheme
(`pkg/src/concpd/synth.py:85-106`): child 0 draws the shared prefixes
(I_n x L_n per mode), child 1+2s draws block s's individual columns per
mode, child 2+2s drives block s's noise.  Core weights are all ones
("X_s = [[A1, A2, A3]]").  Gaussian noise follows ``add_noise`` semantics
(`pkg/src/concpd/metrics.py:218-223`: sigma^2 = mean(X^2) / 10^(SNR/10),
noise drawn over the logical shape in C order, result clipped at 0).

Tensors are returned as numpy arrays of logical shape ``dims`` stored in
Fortran (first-index-fastest) order — the physical layout the device kernels
read (`tensor_ops.py:1-15`).  This module is numpy-only (the bench's
reference arm loads it by path without the native library);
``synth.generate_config_device`` is the on-device generator of the same
recipes for throughput runs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["ConfigSpec", "CONFIGS", "generate_config", "config_tensor_block",
           "config_block_factors", "shared_prefixes"]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n_blocks: int
    dims: tuple
    rank: int
    coupled: tuple
    dtype: str            # storage / throughput dtype on the device
    mode: str             # "full" | "lra"
    max_iter: int
    factor_dist: str      # "uniform" | "gamma"
    noise: str            # "gauss" | "gauss01" | "lognormal"
    snr_db: float = None
    sigma: float = None   # log-normal noise sigma
    description: str = ""

    @property
    def tensor_bytes(self):
        per = int(np.prod(self.dims)) * (8 if self.dtype == "fp64" else 4)
        return per * self.n_blocks


CONFIGS = {
    "c1": ConfigSpec("c1", 2, (50, 50, 50), 5, (2, 2, 2), "fp64", "full", 100,
                     "uniform", "gauss", snr_db=20.0,
                     description="CoNCPD-APG CPU-runnable: S=2 50^3 fp64 R=5 L=(2,2,2) 20 dB, 100 it"),
    "c2": ConfigSpec("c2", 10, (100, 100, 100), 10, (4, 4, 4), "fp32", "full", 500,
                     "uniform", "gauss", snr_db=10.0,
                     description="CoNCPD-APG: S=10 100^3 fp32 R=10 L=(4,4,4) 10 dB, 500 it"),
    "c3": ConfigSpec("c3", 8, (112, 92, 400), 20, (20, 20, 0), "fp32", "lra", 300,
                     "uniform", "gauss01", snr_db=15.0,
                     description="lraCoNCPD-APG image-like: S=8 112x92x400 fp32 R=20 L=(20,20,0) 15 dB in [0,1], 300 it"),
    "c4": ConfigSpec("c4", 32, (64, 71, 60), 30, (10, 10, 10), "fp32", "lra", 500,
                     "gamma", "lognormal", sigma=0.2,
                     description="lraCoNCPD-APG ERP-like: S=32 64x71x60 fp32 R=30 L=(10,10,10) gamma(2,0.5), X*exp(0.2 Z), 500 it"),
    "c5": ConfigSpec("c5", 64, (400, 400, 400), 40, (10, 10, 10), "fp32", "lra", 200,
                     "uniform", "gauss", snr_db=20.0,
                     description="large lraCoNCPD-APG: S=64 400^3 fp32 R=40 L=(10,10,10) 20 dB, 200 it"),
}


def _draw(rng, dist, shape):
    if dist == "uniform":
        return rng.random(shape)
    if dist == "gamma":
        return rng.gamma(2.0, 0.5, size=shape)
    raise ValueError(f"unknown factor distribution {dist!r}")


def _reconstruct_f(factors):
    """Unit-weight Kruskal tensor in Fortran layout: X_(0) = A0 @ KR(A2, A1)^T."""
    a0, a1, a2 = factors
    r = a0.shape[1]
    kr = (a2[:, None, :] * a1[None, :, :]).reshape(-1, r)   # (i2 slow, i1 fast)
    flat = a0 @ kr.T                                         # I0 x (I1*I2), i1 fastest
    return flat.reshape(a0.shape[0], a1.shape[0], a2.shape[0], order="F")


def shared_prefixes(spec, children):
    """The common prefixes (I_n x L_n per mode) from child 0."""
    rng_c = np.random.default_rng(children[0])
    return [_draw(rng_c, spec.factor_dist, (spec.dims[n], spec.coupled[n]))
            for n in range(3)]


def config_block_factors(spec, s, children, common):
    """Block ``s``'s true factors: the common prefix plus its individual
    columns from child 1+2s (unit weights)."""
    rng_s = np.random.default_rng(children[1 + 2 * s])
    facs = []
    for n in range(3):
        own = _draw(rng_s, spec.factor_dist, (spec.dims[n], spec.rank - spec.coupled[n]))
        facs.append(np.hstack([common[n], own]) if spec.coupled[n] else own)
    return facs


def config_tensor_block(spec, s, seed=0, children=None, common=None):
    """Generate block ``s`` of a config on the host: returns (tensor_fp64_F,
    true_factors).  ``synth.generate_config_device`` runs the same recipe with
    the reconstruction and the noise on the GPU."""
    if children is None:
        children = np.random.SeedSequence(seed).spawn(2 * spec.n_blocks + 1)
    if common is None:
        common = shared_prefixes(spec, children)
    facs = config_block_factors(spec, s, children, common)
    clean = _reconstruct_f(facs)
    if spec.noise == "gauss01":
        clean = clean / clean.max()
    rng_n = np.random.default_rng(children[2 + 2 * s])
    if spec.noise in ("gauss", "gauss01"):
        p_s = float(np.mean(clean * clean))
        sigma = np.sqrt(p_s / 10.0 ** (spec.snr_db / 10.0))
        noisy = clean + rng_n.normal(0.0, sigma, clean.shape)
        noisy = np.maximum(noisy, 0.0)
        if spec.noise == "gauss01":
            noisy = np.minimum(noisy, 1.0)
    elif spec.noise == "lognormal":
        # multiplicative log-normal noise X * exp(sigma Z); the median-preserving
        # form (no -sigma^2/2 shift) is used, as documented in DESIGN.md
        noisy = clean * np.exp(spec.sigma * rng_n.standard_normal(clean.shape))
    else:
        raise ValueError(f"unknown noise {spec.noise!r}")
    return np.asfortranarray(noisy), facs


def generate_config(name, seed=0, blocks=None, dtype=None):
    """Return (tensors, spec) for a named config.

    ``tensors`` are numpy arrays (Fortran order) already rounded to the config
    storage dtype (fp32 configs: float32 arrays).  ``blocks`` selects a subset
    of block indices (the seeds of the selected blocks are unchanged).
    """
    spec = CONFIGS[name]
    children = np.random.SeedSequence(seed).spawn(2 * spec.n_blocks + 1)
    common = shared_prefixes(spec, children)
    idx = range(spec.n_blocks) if blocks is None else blocks
    want = dtype or spec.dtype
    np_dtype = np.float64 if want == "fp64" else np.float32
    out = []
    for s in idx:
        t, _ = config_tensor_block(spec, s, children=children, common=common)
        out.append(np.asfortranarray(t.astype(np_dtype)))
    return out, spec
