"""The reference's own property suites, restated against the GPU package.

SURVEY 8(c) lists the property pins the new path must pass:
* central-difference checks of every analytic gradient form — core weights,
  individual and shared factor columns, full and compressed
  (`pkg/tests/test_solver_gradients.py:124-254`,
  `pkg/tests/test_acceptance.py:143-193`);
* tensor-algebra identities at 1e-10 (`test_acceptance.py:199-239`,
  `test_solver.py:53-97`): Khatri-Rao gram = Hadamard gram, vectorised model
  = KR x weights, unfolding of the model, compressed linear terms = full
  linear terms of the surrogate, Lipschitz constants = dense spectral norms.

The instances are drawn the way those tests draw them (small random coupled
problems, data unrelated to the model, signed compressions); every operator
called here runs on the GPU through the C ABI (objective: explicit residual
kernel; MTTKRP, grams, gradients, lambda_max: cb_* kernels).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
N_MODES = 3


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


def _instance(P, i):
    rng = np.random.default_rng(1000 + i)
    dims = tuple(int(rng.integers(2, 7)) for _ in range(N_MODES))
    rank = int(rng.integers(1, 5))
    S = int(rng.integers(1, 4))
    counts = ([0] * N_MODES if i % 4 == 0 else [rank] * N_MODES if i % 4 == 1
              else [int(rng.integers(0, rank + 1)) for _ in range(N_MODES)])
    common = [rng.random((dims[n], counts[n])) for n in range(N_MODES)]
    blocks, tensors = [], []
    for _ in range(S):
        f = [np.hstack([common[n], rng.random((dims[n], rank - counts[n]))]) for n in range(N_MODES)]
        blocks.append(P.KruskalTensor(f, rng.uniform(0.5, 1.5, rank)))
        tensors.append(rng.random(dims))
    return tensors, blocks, counts


def _compressions(P, tensors, i):
    rng = np.random.default_rng(5000 + i)
    out = []
    for t in tensors:
        r = int(rng.integers(1, 4))
        out.append(P.KruskalTensor([rng.standard_normal((d, r)) for d in t.shape],
                                   rng.standard_normal(r)))
    return out


def _rel(num, ref):
    return float(np.linalg.norm(num - ref)) / max(float(np.linalg.norm(ref)), 1e-12)


def _fd(obj, get, put, h0=1e-5):
    """Central differences of obj() over the entries of get()."""
    x0 = get().copy()
    g = np.zeros(x0.size)
    for j in range(x0.size):
        h = h0 * max(1.0, abs(x0.flat[j]))
        vals = []
        for sgn in (1.0, -1.0):
            x = x0.copy()
            x.flat[j] += sgn * h
            put(x)
            vals.append(obj())
        g[j] = (vals[0] - vals[1]) / (2.0 * h)
    put(x0)
    return g.reshape(x0.shape)


def _set_cols(k, n, sl, x):
    f = k.factors[n].copy()
    f[:, sl] = x
    k.factors[n] = f


def _grad_factor(P, t_or_tilde, k, n, lra):
    lin = (P.factor_linear_term_lra(t_or_tilde, k.factors, n) if lra
           else P.factor_linear_term(t_or_tilde, k.factors, n))
    return P.factor_gradient(k.factors[n], P.hadamard_gram(k.factors, skip=n), lin, k.weights)


@pytest.mark.parametrize("i", range(6))
@pytest.mark.parametrize("lra", [False, True])
def test_core_gradient_matches_central_differences(P, i, lra):
    tensors, blocks, _ = _instance(P, i)
    data = tensors
    if lra:
        tilde = _compressions(P, tensors, i)
        data = [P.reconstruct(tk) for tk in tilde]
    for s, k in enumerate(blocks):
        fd = _fd(lambda: P.objective(data, blocks), lambda: k.weights,
                 lambda x: setattr(k, "weights", x))
        lin = (P.core_linear_term_lra(tilde[s], k.factors) if lra
               else P.core_linear_term(tensors[s], k.factors))
        got = P.core_gradient(P.hadamard_gram(k.factors), k.weights, lin)
        assert _rel(got, fd) < 1e-6, f"block {s}"


@pytest.mark.parametrize("i", range(6))
@pytest.mark.parametrize("lra", [False, True])
def test_factor_gradients_match_central_differences(P, i, lra):
    """Individual columns per block, shared columns as the block sum of the
    per-block gradients (the coupling rule, solver.py:444)."""
    tensors, blocks, counts = _instance(P, i)
    data, tilde = tensors, None
    if lra:
        tilde = _compressions(P, tensors, i)
        data = [P.reconstruct(tk) for tk in tilde]
    src = tilde if lra else tensors
    for n in range(N_MODES):
        ln = counts[n]
        for s, k in enumerate(blocks):
            if k.factors[n].shape[1] == ln:
                continue
            fd = _fd(lambda: P.objective(data, blocks), lambda: k.factors[n][:, ln:],
                     lambda x: _set_cols(k, n, slice(ln, None), x))
            got = _grad_factor(P, src[s], k, n, lra)[:, ln:]
            assert _rel(got, fd) < 1e-6, f"mode {n} block {s}"
        if ln:
            def put(x):
                for k in blocks:
                    _set_cols(k, n, slice(0, ln), x)
            fd = _fd(lambda: P.objective(data, blocks), lambda: blocks[0].factors[n][:, :ln], put)
            got = sum(_grad_factor(P, src[s], k, n, lra)[:, :ln] for s, k in enumerate(blocks))
            assert _rel(got, fd) < 1e-6, f"shared mode {n}"


@pytest.mark.parametrize("i", range(10))
def test_tensor_algebra_identities(P, i):
    rng = np.random.default_rng(100 + i)
    order = int(rng.integers(2, 5))
    dims = tuple(int(d) for d in rng.integers(2, 6, size=order))
    rank = int(rng.integers(1, 4))
    mats = [rng.standard_normal((d, rank)) for d in dims]
    w = rng.standard_normal(rank)
    model = P.KruskalTensor(mats, w)
    t = rng.standard_normal(dims)
    kr = P.factors_khatri_rao(mats)
    np.testing.assert_allclose(kr.T @ kr, P.hadamard_gram(mats), rtol=1e-10, atol=1e-10)
    full = P.reconstruct(model)
    np.testing.assert_allclose(P.vectorize(full), kr @ w, rtol=1e-10, atol=1e-10)
    assert (P.unvectorize(P.vectorize(t), dims) == t).all()
    for n in range(order):
        assert (P.refold(P.matricize(t, n), n, dims) == t).all()
        np.testing.assert_allclose(P.matricize(full, n),
                                   (mats[n] * w) @ P.factors_khatri_rao(mats, skip=n).T,
                                   rtol=1e-10, atol=1e-10)
    tr = int(rng.integers(1, 4))
    tilde = P.KruskalTensor([rng.standard_normal((d, tr)) for d in dims], rng.standard_normal(tr))
    sur = P.reconstruct(tilde)
    np.testing.assert_allclose(P.core_linear_term_lra(tilde, mats), P.core_linear_term(sur, mats),
                               rtol=1e-10, atol=1e-10)
    for n in range(order):
        np.testing.assert_allclose(P.factor_linear_term_lra(tilde, mats, n),
                                   P.factor_linear_term(sur, mats, n), rtol=1e-10, atol=1e-10)


def test_lipschitz_constants_match_dense_spectral_norms(P):
    rng = np.random.default_rng(2)
    facs = [rng.random((d, 3)) for d in (4, 5, 6)]
    kr = P.factors_khatri_rao(facs)
    assert P.lipschitz_core(facs) == pytest.approx(np.linalg.norm(kr.T @ kr, 2), rel=1e-10)
    lam = rng.uniform(0.5, 1.5, 3)
    for n in range(3):
        k = P.factors_khatri_rao(facs, skip=n)
        want = np.linalg.norm(np.diag(lam) @ k.T @ k @ np.diag(lam), 2)
        assert P.lipschitz_factor(facs, lam, n) == pytest.approx(want, rel=1e-10)
