"""Input pipeline: the reference's ground-truth generator
(`pkg/src/concpd/synth.py:77-112`, `metrics.py:207-223`) restated on the
host bit-for-bit, and the device generator (csrc/synth.cu) checked against
it: the same truth factors, the fp64 reconstruction at round-off, and a
Gaussian corruption of the prescribed power (a different, counter-based
noise stream)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from store import unpack_models

SPECS = {"ladder": dict(n_blocks=2, size_factor=2, snr_db=20.0, seed=3),
         "clean": dict(n_blocks=3, size_factor=1, snr_db=None, seed=5),
         "override": dict(n_blocks=2, dims=(7, 5, 6), rank=4, coupled=(2, 0, 1),
                          snr_db=10.0, seed=11)}


@pytest.mark.parametrize("name", sorted(SPECS))
def test_host_generator_is_the_reference_bitwise(name):
    from paper_2302_05119_b200.synth import SynthSpec, generate_host
    z = np.load(os.path.join(GOLDEN, "synth.npz"))
    prob, truth = generate_host(SynthSpec(**SPECS[name]))
    for s, t in enumerate(prob.tensors):
        np.testing.assert_array_equal(np.asarray(t), z[f"{name}/t{s}"])
    for blk, (wf, ww) in zip(truth.blocks, unpack_models(f"{name}/truth", z)):
        np.testing.assert_array_equal(blk.weights, ww)
        for a, b in zip(blk.factors, wf):
            np.testing.assert_array_equal(a, b)


def test_synth_spec_rules():
    """Size rules and validation of SynthSpec (synth.py:30-74; the
    reference's test_synth.py:10-29 pins round-half-away and the ladder)."""
    from paper_2302_05119_b200.synth import SynthSpec, round_half_away
    assert [round_half_away(x) for x in (0.5, 1.5, 2.5, -0.5, -1.5, 2.4)] == [1, 2, 3, -1, -2, 2]
    assert SynthSpec(size_factor=2).resolve() == ((16, 18, 20), 9, (5, 5, 5))
    assert SynthSpec(size_factor=3).resolve() == ((24, 27, 30), 14, (7, 7, 7))
    with pytest.raises(ValueError, match="n_blocks"):
        SynthSpec(n_blocks=0)
    with pytest.raises(ValueError, match="coupled counts"):
        SynthSpec(dims=(4, 4, 4), rank=2, coupled=(3, 0, 0))


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SPECS))
def test_device_generator_matches_host(P, name):
    from paper_2302_05119_b200 import synth
    spec = synth.SynthSpec(**SPECS[name])
    hp, ht = synth.generate_host(spec)
    dp, dt = synth.generate(spec)
    for a, b in zip(ht.blocks, dt.blocks):          # truth: the same numpy draws
        np.testing.assert_array_equal(a.weights, b.weights)
        for fa, fb in zip(a.factors, b.factors):
            np.testing.assert_array_equal(fa, fb)
    for s, (th, td) in enumerate(zip(hp.tensors, dp.tensors)):
        got = td.cpu().numpy()
        assert got.shape == th.shape and (got >= 0).all()
        k = dt.blocks[s]
        clean, _ = synth.device_block(k.factors, k.weights, dtype="fp64")
        clean = clean.cpu().numpy().reshape(th.shape, order="F")
        kr = (k.factors[2][:, None, :] * k.factors[1][None, :, :]).reshape(-1, k.rank)
        ref = ((k.factors[0] * k.weights) @ kr.T).reshape(th.shape, order="F")
        np.testing.assert_allclose(clean, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
        if spec.snr_db is None:
            np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


@pytest.mark.gpu
def test_device_noise_power_and_determinism(P):
    """add_noise semantics on the device: sigma^2 = mean(X^2) / 10^(SNR/10),
    clip at 0; a block depends only on (seed, block), not on launch shape."""
    from paper_2302_05119_b200 import synth
    rng = np.random.default_rng(7)
    facs = [rng.random((d, 6)) for d in (60, 50, 40)]
    clean, dims = synth.device_block(facs, None, dtype="fp64")
    x = clean.cpu().numpy()
    snr = 10.0
    sig = np.sqrt(np.mean(x * x) / 10.0 ** (snr / 10.0))
    noisy, _ = synth.device_block(facs, None, dtype="fp64", noise="gauss", snr_db=snr, key=99, block=3)
    y = noisy.cpu().numpy()
    assert (y >= 0).all()
    d = y - x
    keep = x > 4 * sig                     # entries the clip (almost) never reaches
    z = d[keep] / sig
    tol = 5.0 / np.sqrt(z.size)            # 5 standard errors
    assert z.size > 2000
    assert abs(z.mean()) < tol and abs(z.std() - 1.0) < 2 * tol
    again, _ = synth.device_block(facs, None, dtype="fp64", noise="gauss", snr_db=snr, key=99, block=3)
    np.testing.assert_array_equal(again.cpu().numpy(), y)
    other, _ = synth.device_block(facs, None, dtype="fp64", noise="gauss", snr_db=snr, key=99, block=4)
    assert not np.array_equal(other.cpu().numpy(), y)
    # multiplicative log-normal and [0, 1] clipped variants
    ln, _ = synth.device_block(facs, None, dtype="fp64", noise="lognormal", sigma=0.2, key=1)
    r = np.log(ln.cpu().numpy() / x)
    assert abs(r.mean()) < 0.01 and abs(r.std() - 0.2) < 0.01
    g01, _ = synth.device_block(facs, None, dtype="fp32", noise="gauss01", snr_db=15.0, key=2)
    v = g01.cpu().numpy()
    assert v.min() >= 0.0 and v.max() <= 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c4"])
def test_config_device_blocks_track_host_blocks(P, name):
    """generate_config_device: same clean signal as the host config generator
    (same seeded factors), noise of the same power."""
    from paper_2302_05119_b200.configs import generate_config
    from paper_2302_05119_b200.synth import generate_config_device
    host, spec = generate_config(name, blocks=[0, 1])
    dev, _ = generate_config_device(name, blocks=[0, 1])
    for h, d in zip(host, dev):
        a = d.cpu().numpy()
        assert a.shape == h.shape and a.dtype == h.dtype
        np.testing.assert_allclose(a.mean(), h.mean(), rtol=2e-3)
        np.testing.assert_allclose(np.sqrt((a.astype(float) ** 2).mean()),
                                   np.sqrt((h.astype(float) ** 2).mean()), rtol=2e-3)
