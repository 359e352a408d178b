"""Small seeded problem recipes shared by the golden generator and the tests.

Each recipe returns (tensors, kwargs) where kwargs are the ``CoupledProblem``
fields (ranks, coupled_counts, mode, update_core) plus the ``SolverOptions``
fields used for the golden run.  The scenarios mirror the reference's own
solver tests (`pkg/tests/test_solver.py`): noisy full/lra runs, the fixed-core
variant, restart-heavy runs, partial and zero coupling, heterogeneous ranks
and uncoupled dims, zero tensors, max_iter=0, trace thinning, orders 2 and 4.
"""

import numpy as np

TINY_TOL = float(np.nextafter(0.0, 1.0))  # "fixed iteration count" tolerance


def _rank_model(rng, dims, rank, counts, common=None):
    if common is None:
        common = [rng.random((dims[n], counts[n])) for n in range(len(dims))]
    facs = [np.hstack([common[n], rng.random((dims[n], rank - counts[n]))])
            for n in range(len(dims))]
    lam = rng.uniform(0.5, 1.5, rank)
    return facs, lam, common


def _dense(facs, lam):
    out = np.zeros(tuple(f.shape[0] for f in facs))
    for r in range(len(lam)):
        term = lam[r]
        for f in facs:
            term = np.multiply.outer(term, f[:, r])
        out += term
    return out


def _noisy(t, snr_db, seed):
    rng = np.random.default_rng(seed)
    p_s = float(np.mean(t * t))
    sigma = np.sqrt(p_s / 10.0 ** (snr_db / 10.0))
    return np.maximum(t + rng.normal(0.0, sigma, t.shape), 0.0)


def coupled(seed, S=2, dims=(6, 7, 8), rank=4, counts=(2, 2, 2), snr_db=None):
    rng = np.random.default_rng(seed)
    common = [rng.random((dims[n], counts[n])) for n in range(len(dims))]
    tensors = []
    for _ in range(S):
        facs, lam, _ = _rank_model(rng, dims, rank, counts, common)
        t = _dense(facs, lam)
        if snr_db is not None:
            t = _noisy(t, snr_db, seed + 100)
        tensors.append(t)
    return tensors


def recipes():
    """name -> (tensors, problem kwargs, solver kwargs)"""
    out = {}
    out["full_basic"] = (coupled(6, snr_db=20.0), dict(ranks=4, coupled_counts=[2, 2, 2]),
                         dict(max_iter=150, seed=1))
    out["lra_basic"] = (coupled(7, snr_db=20.0),
                        dict(ranks=4, coupled_counts=[2, 2, 2], mode="lra"),
                        dict(max_iter=150, seed=1))
    out["full_nc"] = (coupled(9, snr_db=20.0),
                      dict(ranks=4, coupled_counts=[2, 2, 2], update_core=False),
                      dict(max_iter=80, seed=3))
    out["lra_nc"] = (coupled(9, snr_db=20.0),
                     dict(ranks=4, coupled_counts=[2, 2, 2], update_core=False, mode="lra"),
                     dict(max_iter=80, seed=3))
    out["full_restarts"] = (coupled(16, snr_db=10.0), dict(ranks=4, coupled_counts=[2, 2, 2]),
                            dict(max_iter=400, seed=5))
    out["full_counts_210"] = (coupled(8, counts=(2, 1, 0)),
                              dict(ranks=4, coupled_counts=[2, 1, 0]),
                              dict(max_iter=60, seed=2))
    out["lra_counts_210"] = (coupled(8, counts=(2, 1, 0)),
                             dict(ranks=4, coupled_counts=[2, 1, 0], mode="lra"),
                             dict(max_iter=60, seed=2))
    rng = np.random.default_rng(13)
    t0 = rng.random((5, 6, 7))
    t1 = rng.random((5, 6, 9))
    out["hetero"] = ([t0, t1], dict(ranks=[3, 4], coupled_counts=[2, 2, 0]),
                     dict(max_iter=60, seed=8))
    out["zero"] = ([np.zeros((4, 5, 6)), np.zeros((4, 5, 6))],
                   dict(ranks=3, coupled_counts=[1, 1, 1]), dict(max_iter=50, seed=7))
    out["max_iter0"] = (coupled(12), dict(ranks=4, coupled_counts=[2, 2, 2]),
                        dict(max_iter=0, seed=6))
    out["trace_every"] = (coupled(15), dict(ranks=4, coupled_counts=[2, 2, 2]),
                          dict(max_iter=12, tol=TINY_TOL, seed=10, trace_every=5))
    out["full_counts_full"] = (coupled(21, rank=3, counts=(3, 3, 3), snr_db=20.0),
                               dict(ranks=3, coupled_counts=[3, 3, 3]),
                               dict(max_iter=60, seed=4))
    out["single_block"] = (coupled(22, S=1, dims=(9, 5, 7), rank=3, counts=(0, 0, 0),
                                   snr_db=20.0),
                           dict(ranks=3, coupled_counts=[0, 0, 0]),
                           dict(max_iter=80, seed=5))
    out["order4_full"] = (coupled(31, S=2, dims=(4, 5, 3, 6), rank=3, counts=(1, 1, 0, 1),
                                  snr_db=20.0),
                          dict(ranks=3, coupled_counts=[1, 1, 0, 1]),
                          dict(max_iter=40, seed=1))
    out["order4_lra"] = (coupled(31, S=2, dims=(4, 5, 3, 6), rank=3, counts=(1, 1, 0, 1),
                                 snr_db=20.0),
                         dict(ranks=3, coupled_counts=[1, 1, 0, 1], mode="lra"),
                         dict(max_iter=40, seed=1))
    out["order2_full"] = (coupled(32, S=3, dims=(7, 9), rank=3, counts=(2, 0), snr_db=20.0),
                          dict(ranks=3, coupled_counts=[2, 0]),
                          dict(max_iter=40, seed=2))
    out["lra_trace"] = (coupled(16, snr_db=20.0),
                        dict(ranks=4, coupled_counts=[2, 2, 2], mode="lra"),
                        dict(max_iter=80, seed=11))
    out["full_bigger"] = (coupled(40, S=3, dims=(20, 24, 28), rank=6, counts=(3, 3, 3),
                                  snr_db=15.0),
                          dict(ranks=6, coupled_counts=[3, 3, 3]),
                          dict(max_iter=120, seed=0))
    out["lra_bigger"] = (coupled(41, S=3, dims=(20, 24, 28), rank=6, counts=(3, 3, 3),
                                 snr_db=15.0),
                         dict(ranks=6, coupled_counts=[3, 3, 3], mode="lra"),
                         dict(max_iter=120, seed=0))
    return out


def als_recipes():
    """name -> (tensor, als kwargs) mirroring pkg/tests/test_cpd_als.py."""
    rng = np.random.default_rng(0)
    out = {}
    facs = [rng.random((d, 1)) for d in (5, 6, 4)]
    out["rank1"] = (_dense(facs, np.ones(1)), dict(rank=1, seed=1))
    rng = np.random.default_rng(1)
    facs = [rng.random((d, 9)) for d in (16, 18, 20)]
    out["rank9_deep"] = (_dense(facs, np.ones(9)), dict(rank=9, tol=1e-9, max_iter=500, seed=2))
    out["zero"] = (np.zeros((3, 4, 5)), dict(rank=2, seed=0))
    rng = np.random.default_rng(2)
    out["fullrank"] = (rng.random((6, 7, 5)), dict(rank=3, tol=1e-12, max_iter=60, seed=3))
    rng = np.random.default_rng(3)
    out["small"] = (rng.random((5, 4, 6)), dict(rank=2, seed=4))
    rng = np.random.default_rng(4)
    out["one_sweep"] = (rng.random((4, 5, 3)), dict(rank=2, max_iter=1, seed=0))
    rng = np.random.default_rng(5)
    out["order4"] = (rng.random((4, 3, 5, 3)), dict(rank=3, seed=7))
    return out
