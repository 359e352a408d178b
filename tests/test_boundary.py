"""The C-ABI boundary: the library loads on a CPU-only host, exports every
symbol include/concpd_b200.h declares, and the Python host mirrors the
reference's option/validation behaviour (no compute calls here)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2302_05119_b200 import _lib as L
    header = open(os.path.join(ROOT, "include", "concpd_b200.h")).read()
    declared = set(re.findall(r"\b(cb_[a-z0-9_]+)\s*\(", header))
    declared = {d for d in declared if not d.endswith("_t")}
    assert declared, "no declarations found"
    missing = [name for name in sorted(declared) if not hasattr(L.lib, name)]
    assert not missing, f"library is missing {missing}"
    assert set(L.EXPORTED) == declared
    assert L.lib.cb_abi_version() == 2


def test_library_is_sm100a():
    import subprocess
    from paper_2302_05119_b200 import _lib as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_launch_counter_roundtrip():
    from paper_2302_05119_b200 import _lib as L
    L.launch_count_reset()
    assert L.launch_count() == 0


def test_solver_options_validation_matches_reference():
    from paper_2302_05119_b200 import SolverOptions
    with pytest.raises(ValueError, match="max_iter"):
        SolverOptions(max_iter=-1)
    with pytest.raises(ValueError, match="tol"):
        SolverOptions(tol=0.0)
    with pytest.raises(ValueError, match="delta_w"):
        SolverOptions(delta_w=1.0)
    with pytest.raises(ValueError, match="trace_every"):
        SolverOptions(trace_every=0)
    with pytest.raises(ValueError, match="precision"):
        SolverOptions(precision="fp16")
    # additions (defaulted): arithmetic of the fp32-storage tensor passes
    for ok in ("auto", "fp64", "fp32", "tc"):
        SolverOptions(precision="fp32", compute=ok)
    with pytest.raises(ValueError, match="compute"):
        SolverOptions(compute="int8")


def test_float32_inputs_kept_and_value_checks():
    """float32 numpy blocks are kept (the cast to float64 is exact); value
    checks on host arrays give the reference's messages either way."""
    from paper_2302_05119_b200 import CoupledProblem
    x32 = np.ones((3, 4, 5), dtype=np.float32)
    p = CoupledProblem([x32], 2, [0, 0, 0])
    assert p.tensors[0].dtype == np.float32 and p.tensors[0] is x32
    p64 = CoupledProblem([x32.astype(np.int64)], 2, [0, 0, 0])
    assert p64.tensors[0].dtype == np.float64
    bad = x32.copy()
    bad[0, 0, 0] = -1.0
    with pytest.raises(ValueError, match="negative"):
        CoupledProblem([bad], 2, [0, 0, 0]).validate()
    # the single-process solve defers the element scan to the device
    CoupledProblem([bad], 2, [0, 0, 0]).validate(check_values=False)


def test_problem_validation_messages_match_reference():
    from paper_2302_05119_b200 import CoupledProblem
    good = np.ones((3, 3, 3))
    with pytest.raises(ValueError, match="negative"):
        CoupledProblem([-good], 2, [0, 0, 0]).validate()
    with pytest.raises(ValueError, match="non-finite"):
        CoupledProblem([good * np.nan], 2, [0, 0, 0]).validate()
    with pytest.raises(ValueError, match="mode"):
        CoupledProblem([good], 2, [0, 0, 0], mode="turbo").validate()
    with pytest.raises(ValueError, match="order"):
        CoupledProblem([good, np.ones((3, 3))], 2, [0, 0, 0]).validate()
    with pytest.raises(ValueError, match="rank"):
        CoupledProblem([good], 0, [0, 0, 0]).validate()
    with pytest.raises(ValueError, match="coupled count"):
        CoupledProblem([good], 2, [3, 0, 0]).validate()
    with pytest.raises(ValueError, match="one coupled count"):
        CoupledProblem([good], 2, [0, 0]).validate()
    with pytest.raises(ValueError, match="sizes differ"):
        CoupledProblem([good, np.ones((4, 3, 3))], 2, [1, 0, 0]).validate()
    with pytest.raises(ValueError, match="one rank per block"):
        CoupledProblem([good], [2, 2], [0, 0, 0]).validate()


def test_als_options_validation():
    from paper_2302_05119_b200 import AlsOptions
    with pytest.raises(ValueError):
        AlsOptions(rank=0)
    with pytest.raises(ValueError):
        AlsOptions(rank=2, tol=0.0)
    with pytest.raises(ValueError):
        AlsOptions(max_iter=-1)


def test_scalar_rules_and_seeded_start_match_oracle():
    from oracle import concpd_oracle as O
    from paper_2302_05119_b200 import CoupledProblem, extrapolation_weight, init_factors, t_next
    assert t_next(1.0) == O.next_t(1.0)
    for args in [(0.9, 1.0, 4.0, 0.9999), (0.5, 4.0, 1.0, 0.9999), (0.5, 0.0, 1.0, 0.9999)]:
        assert extrapolation_weight(*args) == O.extrap_w(*args)
    rng = np.random.default_rng(3)
    tensors = [rng.random((4, 5, 6)), rng.random((4, 5, 7))]
    prob = CoupledProblem(tensors, [3, 4], [2, 1, 0])
    got = init_factors(prob, seed=9)
    want = O.draw_init([t.shape for t in tensors], [3, 4], [2, 1, 0], True, 9)
    for blk, (facs, lam) in zip(got.blocks, want):
        assert np.array_equal(blk.weights, lam)
        for a, b in zip(blk.factors, facs):
            assert np.array_equal(a, b)


def test_layout_conventions_match_reference_fixtures():
    from paper_2302_05119_b200 import matricize, refold, unvectorize, vectorize
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "ops.npz"))
    for c in range(int(z["ncases"])):
        t = z[f"case{c}/t"]
        assert np.array_equal(unvectorize(vectorize(t), t.shape), t)
        for n in range(t.ndim):
            assert np.array_equal(matricize(t, n), z[f"case{c}/mat{n}"])
            assert np.array_equal(refold(matricize(t, n), n, t.shape), t)


def test_config_generator_fingerprints():
    from paper_2302_05119_b200.configs import generate_config
    from store import tensor_fingerprint
    from conftest import GOLDEN
    for name in ("c1", "c4"):
        z = np.load(os.path.join(GOLDEN, f"config_{name}.npz"))
        tensors, spec = generate_config(name)
        fp = np.stack([tensor_fingerprint(np.asarray(t, dtype=float)) for t in tensors])
        np.testing.assert_allclose(fp, z["fingerprints"], rtol=1e-13)
