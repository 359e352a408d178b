"""Ground-truth coupled problems (`pkg/src/concpd/synth.py`) with the tensor
part generated on the GPU.

Same surface as the reference: ``round_half_away``, ``SynthSpec`` and
``generate(spec)`` (synth.py:25-112).  The seeded draws (common prefixes from
child 0 of ``SeedSequence(spec.seed)``, block s's individual columns and
weights from child 1+2s) are the reference's, made with numpy, so the truth
factors are bit-identical.  The O(|M| R) part — the reconstruction
X_s = [[lam; A_0, A_1, A_2]] and ``add_noise``'s Gaussian corruption
(metrics.py:207-223) — runs in ``cb_synth_stats`` / ``cb_synth_fill``
(csrc/synth.cu): fp64 reconstruction, Philox noise keyed by block s's noise
child.  The noise realisation therefore differs from numpy's PCG64 stream
(same distribution and power); parity runs that must see the reference's exact
inputs use ``generate_host``, which restates the reference generator on the
host (numpy only, bit-identical).

``generate_config_device`` does the same for the five BASELINE configs
(configs.py): device-resident fp32 blocks for throughput runs in seconds
instead of minutes of host numpy (c5: 64 x 400^3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib as L
from .configs import CONFIGS, config_block_factors, shared_prefixes
from .kruskal import CoupledFactorSet, KruskalTensor
from .solver import CoupledProblem

__all__ = ["SynthSpec", "generate", "generate_host", "round_half_away", "device_block",
           "generate_config_device"]


def round_half_away(x):
    """Nearest integer, ties away from zero (synth.py:25-27)."""
    return int(np.sign(x) * np.floor(abs(x) + 0.5))


@dataclass
class SynthSpec:
    """Recipe for one coupled synthetic problem (synth.py:30-74)."""

    n_blocks: int = 10
    size_factor: int = 2
    snr_db: float = 20.0
    seed: int = 0
    dims: tuple = None
    rank: int = None
    coupled: tuple = None

    def __post_init__(self):
        if self.n_blocks < 1:
            raise ValueError("n_blocks must be >= 1")
        if self.size_factor < 1:
            raise ValueError("size_factor must be >= 1")
        dims, rank, coupled = self.resolve()
        if len(dims) != 3 or any(d < 1 for d in dims):
            raise ValueError(f"dims must be three positive sizes, got {dims}")
        if rank < 1:
            raise ValueError(f"rank must be >= 1, got {rank}")
        if len(coupled) != 3:
            raise ValueError(f"coupled needs one count per mode, got {coupled}")
        if any(not 0 <= c <= rank for c in coupled):
            raise ValueError(f"coupled counts {coupled} must lie in [0, rank={rank}]")

    def resolve(self):
        """Final ``(dims, rank, coupled)`` after the size rules."""
        dims = self.dims
        if dims is None:
            f = self.size_factor
            dims = (8 * f, 9 * f, 10 * f)
        dims = tuple(int(d) for d in dims)
        rank = self.rank if self.rank is not None else round_half_away(dims[1] / 2)
        coupled = self.coupled
        if coupled is None:
            coupled = (round_half_away(dims[1] / 4),) * 3
        return dims, int(rank), tuple(int(c) for c in coupled)


def _truth(spec):
    """The reference's seeded draws (synth.py:87-104): truth blocks and the
    noise SeedSequence child of every block."""
    dims, rank, counts = spec.resolve()
    children = np.random.SeedSequence(spec.seed).spawn(2 * spec.n_blocks + 1)
    rng_c = np.random.default_rng(children[0])
    common = [rng_c.random((dims[n], counts[n])) for n in range(3)]
    blocks = []
    for s in range(spec.n_blocks):
        rng_s = np.random.default_rng(children[1 + 2 * s])
        facs = []
        for n in range(3):
            ind = rng_s.random((dims[n], rank - counts[n]))
            facs.append(np.hstack([common[n], ind]) if counts[n] else ind)
        lam = rng_s.uniform(0.5, 1.5, rank)
        blocks.append(KruskalTensor(facs, lam))
    return dims, rank, counts, blocks, children


def _noise_key(child):
    """64-bit Philox key of a block's noise child (deterministic in the seed)."""
    return int(child.generate_state(1, np.uint64)[0])


def device_block(factors, weights, dtype="fp32", noise="none", snr_db=None, sigma=None,
                 scale_to_max=False, key=0, block=0):
    """One block on the device: X = [[weights; factors]] (fp64 arithmetic)
    corrupted by ``noise`` ("none" | "gauss": add_noise semantics, clip at 0 |
    "gauss01": X / max(X) then Gaussian noise clipped to [0, 1] |
    "lognormal": X exp(sigma Z)).  Returns a flat first-index-fastest CUDA
    tensor and the dims."""
    torch = D.torch_mod()
    dims = tuple(int(f.shape[0]) for f in factors)
    rank = int(np.asarray(factors[0]).shape[1])
    dev = [D.to_dev_f64(f) for f in factors]
    dw = D.to_dev_f64(weights) if weights is not None else None
    fptrs = L.ptr_array([D.ptr(x) for x in dev])
    dims_c = L.i64_array(dims)
    wptr = D.ptr(dw) if dw is not None else None
    n = int(np.prod(dims))
    scale, sig, code = 1.0, 0.0, 0
    if noise in ("gauss", "gauss01") or scale_to_max:
        st = torch.empty(2, dtype=torch.float64, device=dev[0].device)
        L.check(L.lib.cb_synth_stats(len(dims), dims_c, fptrs, wptr, rank, D.ptr(st), D.stream()))
        ss, mx = (float(v) for v in st.cpu())
        if noise == "gauss01" or scale_to_max:
            scale = 1.0 / mx if mx > 0.0 else 1.0
        if noise in ("gauss", "gauss01"):
            if snr_db is None or not np.isfinite(snr_db):
                raise ValueError("gaussian noise needs a finite snr_db")
            p_s = ss * scale * scale / n          # mean(X^2) of the (scaled) clean block
            sig = float(np.sqrt(p_s / 10.0 ** (snr_db / 10.0)))
            code = 2 if noise == "gauss01" else 1
    elif noise == "lognormal":
        code, sig = 3, float(sigma)
    elif noise != "none":
        raise ValueError(f"unknown noise kind: {noise!r}")
    want = torch.float32 if dtype == "fp32" else torch.float64
    out = torch.empty(n, dtype=want, device=dev[0].device)
    L.check(L.lib.cb_synth_fill(L.CB_F32 if dtype == "fp32" else L.CB_F64, D.ptr(out), len(dims),
                                dims_c, fptrs, wptr, rank, float(scale), code, sig,
                                int(key) & ((1 << 64) - 1), int(block), D.stream()))
    return out, dims


def generate(spec, dtype="fp64"):
    """Draw the problem on the GPU; returns ``(CoupledProblem, truth)`` with
    the tensors as device-resident torch tensors of logical shape ``dims``
    (synth.py:77-112).  Truth factors equal the reference's bit for bit."""
    dims, rank, counts, blocks, children = _truth(spec)
    noiseless = spec.snr_db is None or np.isinf(spec.snr_db)
    tensors = []
    for s, k in enumerate(blocks):
        flat, d = device_block(k.factors, k.weights, dtype=dtype,
                               noise="none" if noiseless else "gauss", snr_db=spec.snr_db,
                               key=_noise_key(children[2 + 2 * s]), block=s)
        tensors.append(D.fortran_view(flat, d))
    problem = CoupledProblem(tensors, rank, list(counts))
    truth = CoupledFactorSet(blocks, list(counts))
    truth.validate()
    return problem, truth


def generate_host(spec):
    """The reference generator restated on the host (numpy; bit-identical
    inputs for parity runs): reconstruct through the mode-0 unfolding
    (kruskal.py:112-119) and ``add_noise`` (metrics.py:218-221)."""
    dims, rank, counts, blocks, children = _truth(spec)
    noiseless = spec.snr_db is None or np.isinf(spec.snr_db)
    tensors = []
    for s, k in enumerate(blocks):
        kr = (k.factors[2][:, None, :] * k.factors[1][None, :, :]).reshape(-1, rank)
        clean = ((k.factors[0] * k.weights) @ kr.T).reshape(dims, order="F")
        if noiseless:
            tensors.append(clean)
            continue
        rng = np.random.default_rng(children[2 + 2 * s])
        p_s = float(np.mean(clean * clean))
        sig = np.sqrt(p_s / 10.0 ** (spec.snr_db / 10.0))
        tensors.append(np.maximum(clean + rng.normal(0.0, sig, clean.shape), 0.0))
    problem = CoupledProblem(tensors, rank, list(counts))
    problem.validate()
    truth = CoupledFactorSet(blocks, list(counts))
    truth.validate()
    return problem, truth


def generate_config_device(name, seed=0, blocks=None, dtype=None):
    """Device-resident blocks of a BASELINE config (configs.py): the same
    seeded factors as ``configs.generate_config``, reconstruction and noise
    on the GPU.  Returns (list of flat fp32/fp64 CUDA tensors viewed with
    logical shape ``dims`` in first-index-fastest order, spec)."""
    spec = CONFIGS[name]
    children = np.random.SeedSequence(seed).spawn(2 * spec.n_blocks + 1)
    common = shared_prefixes(spec, children)
    idx = range(spec.n_blocks) if blocks is None else blocks
    want = dtype or spec.dtype
    noise = {"gauss": "gauss", "gauss01": "gauss01", "lognormal": "lognormal"}[spec.noise]
    out = []
    for s in idx:
        facs = config_block_factors(spec, s, children, common)
        flat, d = device_block(facs, None, dtype=want, noise=noise, snr_db=spec.snr_db,
                               sigma=spec.sigma, key=_noise_key(children[2 + 2 * s]), block=s)
        out.append(D.fortran_view(flat, d))
    return out, spec
