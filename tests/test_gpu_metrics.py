"""Post-solve metrics on the GPU against the reference's own
values (tests/golden/metrics.npz from pkg/src/concpd/metrics.py:71-156)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from store import unpack_models

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


@pytest.fixture(scope="module")
def Z():
    return np.load(os.path.join(GOLDEN, "metrics.npz"))


def _models(P, Z, prefix):
    return [P.KruskalTensor(f, w) for f, w in unpack_models(prefix, Z)]


def test_rel_err_dense_and_kruskal(P, Z):
    from paper_2302_05119_b200 import metrics as M
    tensors = [Z[f"t{s}"] for s in range(3)]
    models = _models(P, Z, "models")
    dense = [P.reconstruct(k) for k in models]
    assert M.rel_err(tensors, dense) == pytest.approx(float(Z["rel_err"]), rel=1e-12)
    # the device-native form: models streamed, never formed
    assert M.rel_err(tensors, models) == pytest.approx(float(Z["rel_err"]), rel=1e-12)
    assert M.ten_fit(tensors, models) == pytest.approx(1.0 - float(Z["rel_err"]), rel=1e-12)
    with pytest.raises(ValueError, match="3 original blocks vs 2 recovered"):
        M.rel_err(tensors, models[:2])
    with pytest.raises(ValueError, match="block 1: original shape"):
        M.rel_err(tensors, [models[0], models[0], models[2]])
    assert M.rel_err([np.zeros((3, 4, 5))], [np.ones((3, 4, 5))]) == 0.0


def test_psnr(P, Z):
    from paper_2302_05119_b200 import metrics as M
    models = _models(P, Z, "models")
    t0 = Z["t0"]
    assert M.psnr(t0, P.reconstruct(models[0]), peak=2.0) == pytest.approx(float(Z["psnr"]), rel=1e-12)
    assert M.psnr(t0, models[0], peak=2.0) == pytest.approx(float(Z["psnr"]), rel=1e-12)
    assert M.psnr(t0, t0) == M.PSNR_CAP_DB
    with pytest.raises(ValueError, match="peak must be positive"):
        M.psnr(t0, t0, peak=0.0)


def test_performance_index(P, Z):
    from paper_2302_05119_b200 import metrics as M
    for i, want in enumerate(Z["pi"]):
        got = M.performance_index(Z[f"pi_e{i}"], Z[f"pi_t{i}"])
        assert got == pytest.approx(float(want), rel=1e-10, abs=1e-13)
    e = Z["pi_perm_e"]
    assert M.performance_index(e, e[:, [3, 0, 4, 1, 2]] * [2.0, 0.5, 3.0, 1.0, 7.0]) < 1e-12
    with pytest.raises(ValueError, match="single component"):
        M.performance_index(np.ones((4, 1)), np.ones((4, 1)))
    with pytest.raises(ValueError, match="estimated shape"):
        M.performance_index(np.ones((4, 2)), np.ones((5, 2)))
    with pytest.warns(RuntimeWarning, match="rank-deficient"):
        M.performance_index(np.ones((6, 3)), np.random.default_rng(0).random((6, 3)))


def test_pi_per_mode(P, Z):
    from paper_2302_05119_b200 import metrics as M
    est = P.CoupledFactorSet(_models(P, Z, "pm_est"), [0, 0, 0])
    tru = P.CoupledFactorSet(_models(P, Z, "pm_tru"), [0, 0, 0])
    np.testing.assert_allclose(M.pi_per_mode(est, tru), Z["pi_per_mode"], rtol=1e-10)


def test_metrics_of_a_c5_block_stream_on_the_device(P):
    """rel_err of a device-resident c5 block against its own truth model:
    the 256 MB model is never formed (cb_model_residual)."""
    from paper_2302_05119_b200 import metrics as M
    from paper_2302_05119_b200.configs import CONFIGS, config_block_factors, shared_prefixes
    from paper_2302_05119_b200.synth import generate_config_device
    spec = CONFIGS["c5"]
    dev, _ = generate_config_device("c5", blocks=[3])
    children = np.random.SeedSequence(0).spawn(2 * spec.n_blocks + 1)
    facs = config_block_factors(spec, 3, children, shared_prefixes(spec, children))
    err = M.rel_err(dev, [P.KruskalTensor(facs, np.ones(spec.rank))])
    # 20 dB noise: ||noise|| / ||X|| ~ 0.1 (less after clipping at 0)
    assert 0.05 < err < 0.11
