"""Pin the CPU oracle against the REAL reference's outputs and known answers.

The fixtures under tests/golden/ were produced by tests/golden/make_golden.py
running the reference package itself; here the oracle (oracle/concpd_oracle.py)
must reproduce them.  CPU only.
"""

import glob
import os

import numpy as np
import pytest

from oracle import concpd_oracle as O
from store import tensor_fingerprint, unpack_models, unpack_solve

from conftest import GOLDEN


def _ops():
    return np.load(os.path.join(GOLDEN, "ops.npz"))


def test_known_answers_from_reference_tests():
    # KR worked example (pkg/tests/test_tensor_ops.py:124-128)
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[0.0, 1.0], [1.0, 0.0]])
    want = np.array([[0.0, 2.0], [1.0, 0.0], [0.0, 4.0], [3.0, 0.0]])
    assert np.array_equal(O.kr_columns([a, b]), want)
    # spectral norm known values (test_tensor_ops.py:229-248)
    assert O.top_eig(np.diag([3.0, 7.0, 1.0])) == pytest.approx(7.0, rel=1e-12)
    q = np.array([[1.0, 1.0], [1.0, -1.0]]) / np.sqrt(2.0)
    assert O.top_eig(q @ np.diag([1.0, 5.0]) @ q.T) == pytest.approx(5.0, rel=1e-12)
    v = np.array([1.0, 2.0, 2.0])
    assert O.top_eig(np.outer(v, v)) == pytest.approx(9.0, rel=1e-12)
    assert O.top_eig(np.zeros((4, 4))) == 0.0
    # momentum / extrapolation caps (test_solver.py:103-120)
    assert O.next_t(1.0) == pytest.approx((1 + np.sqrt(5)) / 2, rel=1e-15)
    assert O.extrap_w(0.9, 1.0, 4.0, 0.9999) == pytest.approx(0.9999 * 0.5)
    assert O.extrap_w(0.5, 4.0, 1.0, 0.9999) == 0.5
    assert O.extrap_w(0.5, 0.0, 1.0, 0.9999) == 0.0
    assert O.extrap_w(0.5, 1.0, 0.0, 0.9999) == 0.0


def test_operator_fixtures_exact():
    z = _ops()
    for c in range(int(z["ncases"])):
        p = f"case{c}"
        N = int(z[f"{p}/N"])
        t = z[f"{p}/t"]
        facs = [z[f"{p}/f{n}"] for n in range(N)]
        tf = [z[f"{p}/tf{n}"] for n in range(N)]
        tw = z[f"{p}/tw"]
        lam = z[f"{p}/lam"]
        assert np.array_equal(O.kr_desc(facs), z[f"{p}/kr"])
        assert np.array_equal(O.gram_hadamard(facs), z[f"{p}/hg"])
        assert np.array_equal(O.gram_hadamard(facs, mats2=tf), z[f"{p}/hgx"])
        np.testing.assert_allclose(O.core_term(t, facs), z[f"{p}/core"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(O.core_term_lra(tf, tw, facs), z[f"{p}/core_lra"],
                                   rtol=1e-13, atol=1e-13)
        assert O.full_objective([t], [(facs, lam)]) == pytest.approx(float(z[f"{p}/obj"]),
                                                                     rel=1e-13)
        assert O.top_eig(O.gram_hadamard(facs)) == pytest.approx(float(z[f"{p}/lipc"]),
                                                                 rel=1e-13)
        for n in range(N):
            assert np.array_equal(O.unfold(t, n), z[f"{p}/mat{n}"])
            assert np.array_equal(O.fold(O.unfold(t, n), n, t.shape), t)
            assert np.array_equal(O.kr_desc(facs, skip=n), z[f"{p}/krs{n}"])
            np.testing.assert_allclose(O.mttkrp(t, facs, n), z[f"{p}/mtt{n}"],
                                       rtol=1e-13, atol=1e-13)
            np.testing.assert_allclose(O.mttkrp_lra(tf, tw, facs, n), z[f"{p}/mtt_lra{n}"],
                                       rtol=1e-13, atol=1e-13)
            step = O.gram_hadamard(facs, skip=n) * np.outer(lam, lam)
            assert O.top_eig(step) == pytest.approx(float(z[f"{p}/lipf{n}"]), rel=1e-13)
    vals = z["psd_vals"]
    for i in range(len(vals)):
        assert O.top_eig(z[f"psd{i}"]) == pytest.approx(float(vals[i]), rel=1e-14)


def _compare_solve(got, want, rtol):
    assert got["n_iter"] == want["n_iter"]
    assert got["n_restarts"] == want["n_restarts"]
    assert got["termination_reason"] == want["termination_reason"]
    np.testing.assert_allclose(got["objective_history"], want["objective_history"],
                               rtol=rtol, atol=1e-300)
    np.testing.assert_allclose(got["rel_err_history"], want["rel_err_history"],
                               rtol=rtol, atol=1e-300)
    assert [r[0] for r in got["trace"]] == [r[0] for r in want["trace"]]
    for (fg, wg), (fw, ww) in zip(got["factors"], want["factors"]):
        np.testing.assert_allclose(wg, ww, rtol=rtol, atol=1e-12)
        for a, b in zip(fg, fw):
            np.testing.assert_allclose(a, b, rtol=rtol, atol=1e-12)


SOLVE_CASES = sorted(os.path.basename(p)[6:-4]
                     for p in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_oracle_solve_matches_reference(name):
    from cases import recipes
    tensors, pkw, skw = recipes()[name]
    z = np.load(os.path.join(GOLDEN, f"solve_{name}.npz"))
    for s, t in enumerate(tensors):
        assert np.array_equal(np.asarray(t, dtype=float), z[f"input/{s}"])
    want = unpack_solve(z)
    got = O.solve_oracle(tensors, pkw["ranks"], pkw["coupled_counts"],
                         mode=pkw.get("mode", "full"),
                         update_core=pkw.get("update_core", True), **skw)
    _compare_solve(got, want, rtol=1e-12)


def test_oracle_als_matches_reference():
    from cases import als_recipes
    z = np.load(os.path.join(GOLDEN, "als.npz"))
    for name, (t, kw) in als_recipes().items():
        assert np.array_equal(np.asarray(t, dtype=float), z[f"{name}/input"])
        got = O.als_fit(t, **kw)
        assert got["n_iter"] == int(z[f"{name}/n_iter"])
        assert got["converged"] == bool(z[f"{name}/converged"])
        np.testing.assert_allclose(got["history"], z[f"{name}/history"], rtol=1e-10,
                                   atol=1e-14)
        for n in range(int(z[f"{name}/N"])):
            np.testing.assert_allclose(got["factors"][n], z[f"{name}/f{n}"], rtol=1e-9,
                                       atol=1e-12)


def test_config_c1_oracle_matches_reference():
    from paper_2302_05119_b200.configs import CONFIGS, generate_config
    from cases import TINY_TOL
    z = np.load(os.path.join(GOLDEN, "config_c1.npz"))
    tensors, spec = generate_config("c1")
    fp = np.stack([tensor_fingerprint(t) for t in tensors])
    np.testing.assert_allclose(fp, z["fingerprints"], rtol=1e-14)
    got = O.solve_oracle(tensors, spec.rank, list(spec.coupled), mode=spec.mode,
                         max_iter=spec.max_iter, tol=TINY_TOL, seed=0)
    _compare_solve(got, unpack_solve(z), rtol=1e-10)


def test_recovery_table_known_answers():
    """pkg/test_output.txt:266-276 records the per-seed RelErr of the reference's
    recovery gate; the fixture (run here) must reproduce those printed digits."""
    printed = {0: 2.59e-06, 1: 2.46e-02, 2: 1.63e-06, 3: 2.08e-02, 4: 1.51e-05,
               5: 2.10e-06, 6: 2.56e-02, 7: 1.60e-06, 8: 2.91e-06, 9: 2.20e-02}
    path = os.path.join(GOLDEN, "recovery.npz")
    if not os.path.exists(path):
        pytest.skip("recovery fixture not generated")
    z = np.load(path)
    for seed, val in printed.items():
        assert f"{float(z[f'seed{seed}/rel']):.2e}" == f"{val:.2e}"


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_recovery_run_matches_reference(seed):
    z = np.load(os.path.join(GOLDEN, "recovery.npz"))
    tensors = [z[f"seed{seed}/input/{s}"] for s in range(3)]
    got = O.solve_oracle(tensors, 9, [4, 4, 4], seed=seed)
    assert got["n_iter"] == int(z[f"seed{seed}/n_iter"])
    np.testing.assert_allclose(got["objective_history"], z[f"seed{seed}/obj"], rtol=1e-10)
    for (fg, wg), (fw, ww) in zip(got["factors"], unpack_models(f"seed{seed}/factors", z)):
        np.testing.assert_allclose(wg, ww, rtol=1e-8, atol=1e-10)
