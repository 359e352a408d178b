"""GPU parity of the operator-level kernels against the reference fixtures
(tests/golden/ops.npz, produced by the reference itself) and the oracle.
fp64 throughout; tolerances are stated per assertion."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from conftest import GOLDEN
from oracle import concpd_oracle as O


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


@pytest.fixture(scope="module")
def ops():
    return np.load(os.path.join(GOLDEN, "ops.npz"))


def _case(z, c):
    p = f"case{c}"
    N = int(z[f"{p}/N"])
    facs = [z[f"{p}/f{n}"] for n in range(N)]
    tf = [z[f"{p}/tf{n}"] for n in range(N)]
    return p, N, z[f"{p}/t"], facs, tf, z[f"{p}/tw"], z[f"{p}/lam"]


def test_khatri_rao_and_grams(P, ops):
    for c in range(int(ops["ncases"])):
        p, N, t, facs, tf, tw, lam = _case(ops, c)
        # exact: products of the same two-factor terms in the same order
        np.testing.assert_allclose(P.factors_khatri_rao(facs), ops[f"{p}/kr"], rtol=1e-15, atol=0)
        np.testing.assert_allclose(P.hadamard_gram(facs), ops[f"{p}/hg"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(P.hadamard_gram(facs, mats2=tf), ops[f"{p}/hgx"],
                                   rtol=1e-12, atol=1e-12)
        for n in range(N):
            np.testing.assert_allclose(P.factors_khatri_rao(facs, skip=n), ops[f"{p}/krs{n}"],
                                       rtol=1e-15, atol=0)
            np.testing.assert_allclose(P.hadamard_gram(facs, skip=n), ops[f"{p}/hgs{n}"],
                                       rtol=1e-13, atol=1e-13)


def test_khatri_rao_worked_example(P):
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[0.0, 1.0], [1.0, 0.0]])
    want = np.array([[0.0, 2.0], [1.0, 0.0], [0.0, 4.0], [3.0, 0.0]])
    assert np.array_equal(P.khatri_rao([a, b]), want)
    with pytest.raises(ValueError):
        P.khatri_rao([np.zeros((2, 3)), np.zeros((4, 2))])


def test_mttkrp_all_modes(P, ops):
    for c in range(int(ops["ncases"])):
        p, N, t, facs, tf, tw, lam = _case(ops, c)
        for n in range(N):
            got = P.factor_linear_term(t, facs, n)
            np.testing.assert_allclose(got, ops[f"{p}/mtt{n}"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(P.core_linear_term(t, facs), ops[f"{p}/core"], rtol=1e-12,
                                   atol=1e-12)


def test_lra_linear_terms(P, ops):
    for c in range(int(ops["ncases"])):
        p, N, t, facs, tf, tw, lam = _case(ops, c)
        tilde = P.KruskalTensor(tf, tw)
        np.testing.assert_allclose(P.core_linear_term_lra(tilde, facs), ops[f"{p}/core_lra"],
                                   rtol=1e-11, atol=1e-11)
        for n in range(N):
            np.testing.assert_allclose(P.factor_linear_term_lra(tilde, facs, n),
                                       ops[f"{p}/mtt_lra{n}"], rtol=1e-11, atol=1e-11)


def test_spectral_norm_matches_eigvalsh(P, ops):
    vals = ops["psd_vals"]
    for i in range(len(vals)):
        got = P.spectral_norm(ops[f"psd{i}"])
        assert got == pytest.approx(float(vals[i]), rel=1e-13), i


def test_spectral_norm_known_values(P):
    assert P.spectral_norm(np.diag([3.0, 7.0, 1.0])) == pytest.approx(7.0, rel=1e-12)
    q = np.array([[1.0, 1.0], [1.0, -1.0]]) / np.sqrt(2.0)
    assert P.spectral_norm(q @ np.diag([1.0, 5.0]) @ q.T) == pytest.approx(5.0, rel=1e-12)
    v = np.array([1.0, 2.0, 2.0])
    assert P.spectral_norm(np.outer(v, v)) == pytest.approx(9.0, rel=1e-12)
    assert P.spectral_norm(np.zeros((4, 4))) == 0.0
    assert P.spectral_norm(np.eye(5) * 3.0) == pytest.approx(3.0, rel=1e-14)
    # indefinite input: lambda_max, not the spectral radius
    assert P.spectral_norm(np.diag([-9.0, 2.0])) == pytest.approx(2.0, rel=1e-12)
    assert P.spectral_norm(-np.eye(3)) == 0.0
    with pytest.raises(ValueError, match="square"):
        P.spectral_norm(np.ones((2, 3)))


def test_spectral_norm_random_sweep(P):
    rng = np.random.default_rng(12)
    for _ in range(30):
        r = int(rng.integers(1, 65))
        a = rng.standard_normal((r + 2, r))
        g = a.T @ a
        want = float(np.linalg.eigvalsh(g)[-1])
        assert P.spectral_norm(g) == pytest.approx(want, rel=1e-12)


def test_lipschitz_and_gradients(P, ops):
    for c in range(int(ops["ncases"])):
        p, N, t, facs, tf, tw, lam = _case(ops, c)
        assert P.lipschitz_core(facs) == pytest.approx(float(ops[f"{p}/lipc"]), rel=1e-12)
        for n in range(N):
            assert P.lipschitz_factor(facs, lam, n) == pytest.approx(float(ops[f"{p}/lipf{n}"]),
                                                                     rel=1e-12)
            gskip = O.gram_hadamard(facs, skip=n)
            mtt = O.mttkrp(t, facs, n)
            want = facs[n] @ (gskip * np.outer(lam, lam)) - mtt * lam
            np.testing.assert_allclose(P.factor_gradient(facs[n], gskip, mtt, lam), want,
                                       rtol=1e-12, atol=1e-12)
        gall = O.gram_hadamard(facs)
        lin = O.core_term(t, facs)
        np.testing.assert_allclose(P.core_gradient(gall, lam, lin), gall @ lam - lin,
                                   rtol=1e-12, atol=1e-12)


def test_objective_explicit_residual(P, ops):
    for c in range(int(ops["ncases"])):
        p, N, t, facs, tf, tw, lam = _case(ops, c)
        got = P.objective([t], [P.KruskalTensor(facs, lam)])
        assert got == pytest.approx(float(ops[f"{p}/obj"]), rel=1e-12)


def test_reconstruct(P):
    rng = np.random.default_rng(4)
    facs = [rng.random((d, 3)) for d in (4, 5, 6)]
    lam = rng.random(3)
    got = P.reconstruct(P.KruskalTensor(facs, lam))
    want = O.dense_from_model(facs, lam)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-14)


def test_cpd_als_matches_reference(P):
    from cases import als_recipes
    z = np.load(os.path.join(GOLDEN, "als.npz"))
    for name, (t, kw) in als_recipes().items():
        res = P.cpd_als(t, P.AlsOptions(**kw))
        assert res.n_iter == int(z[f"{name}/n_iter"]), name
        assert res.converged == bool(z[f"{name}/converged"]), name
        np.testing.assert_allclose(res.rel_err_history, z[f"{name}/history"], rtol=1e-8,
                                   atol=1e-12, err_msg=name)
        for n in range(int(z[f"{name}/N"])):
            np.testing.assert_allclose(res.model.factors[n], z[f"{name}/f{n}"], rtol=1e-6,
                                       atol=1e-8, err_msg=f"{name} mode {n}")
        assert res.model.weights.tolist() == [1.0] * res.model.rank


def test_cpd_als_errors(P):
    with pytest.raises(ValueError, match="infeasible"):
        P.cpd_als(np.ones((2, 2, 2)), P.AlsOptions(rank=5))
    t = np.ones((3, 3, 3))
    t[0, 0, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        P.cpd_als(t, P.AlsOptions(rank=1))
    with pytest.raises(ValueError):
        P.cpd_als(np.ones((2, 2)), P.AlsOptions())
