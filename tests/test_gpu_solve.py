"""GPU parity of the full solver (CoNCPD-APG and lraCoNCPD-APG) against the
REAL reference's outputs on the same seeded inputs (tests/golden/*.npz), plus
the reference's solver invariants (pkg/tests/test_solver.py) re-run on the
GPU path.

Tolerances (north_star): fp64 mode — histories and factors within 1e-9
relative; fp32 throughput mode — within 1e-4 relative (oracle = reference in
fp64 on the fp32-rounded inputs)."""

import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from conftest import GOLDEN
from store import tensor_fingerprint, unpack_solve


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


def _rel_close(got, want, rtol, what):
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    scale = max(float(np.max(np.abs(want))) if want.size else 0.0, 1e-300)
    err = float(np.max(np.abs(got - want))) / scale if want.size else 0.0
    assert err <= rtol, f"{what}: max rel err {err:.3e} > {rtol:.1e}"
    return err


def _hist_close(got, want, rtol, what):
    """Element-wise relative error of a history (every entry on its own scale)."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    if not want.size:
        return 0.0
    # entries below 1e-12 of the history's peak are round-off residues (e.g.
    # a zero tensor's objective: the reference 1.7e-37, exact 0 here)
    floor = max(float(np.max(np.abs(want))) * 1e-12, 1e-300)
    scale = np.maximum(np.abs(want), floor)
    err = float(np.max(np.abs(got - want) / scale))
    assert err <= rtol, f"{what}: max element-wise rel err {err:.3e} > {rtol:.1e}"
    return err


def compare(res, want, rtol, prefix_only=False, factor_rtol=None):
    """Compare a SolveResult with an unpacked reference result.  Histories are
    compared element-wise over the common prefix; iteration and restart counts
    whenever the runs have the same length (always unless prefix_only)."""
    n = min(res.n_iter, want["n_iter"]) + 1
    if not prefix_only or res.n_iter == want["n_iter"]:
        assert res.n_iter == want["n_iter"]
        assert res.n_restarts == want["n_restarts"]
        assert res.termination_reason == want["termination_reason"]
    _hist_close(res.objective_history[:n], want["objective_history"][:n], rtol, "objective_history")
    _hist_close(res.rel_err_history[:n], want["rel_err_history"][:n], rtol, "rel_err_history")
    if not prefix_only:
        assert [r.iteration for r in res.trace] == [r[0] for r in want["trace"]]
        _hist_close([r.obj_fun for r in res.trace], [r[1] for r in want["trace"]], rtol, "trace obj")
        _hist_close([r.rel_err for r in res.trace], [r[2] for r in want["trace"]], rtol, "trace rel")
    if not prefix_only or factor_rtol is not None:
        ft = factor_rtol if factor_rtol is not None else rtol
        for s, (blk, (wf, ww)) in enumerate(zip(res.factors.blocks, want["factors"])):
            _rel_close(blk.weights, ww, ft, f"block {s} weights")
            for m, (a, b) in enumerate(zip(blk.factors, wf)):
                _rel_close(a, b, ft, f"block {s} mode {m} factor")


SOLVE_CASES = sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_solve_matches_reference_fp64(P, name):
    from cases import recipes
    tensors, pkw, skw = recipes()[name]
    want = unpack_solve(np.load(os.path.join(GOLDEN, f"solve_{name}.npz")))
    prob = P.CoupledProblem(tensors, pkw["ranks"], pkw["coupled_counts"],
                            mode=pkw.get("mode", "full"), update_core=pkw.get("update_core", True))
    res = P.solve(prob, P.SolverOptions(**skw))
    compare(res, want, rtol=1e-9)


def _config(P, name, precision, **opt):
    from cases import TINY_TOL
    from paper_2302_05119_b200.configs import generate_config
    z = np.load(os.path.join(GOLDEN, f"config_{name}.npz"))
    blocks = [int(b) for b in z["blocks"]] if "blocks" in z else None
    tensors, spec = generate_config(name, blocks=blocks)
    fp = np.stack([tensor_fingerprint(np.asarray(t, dtype=float)) for t in tensors])
    np.testing.assert_allclose(fp, z["fingerprints"], rtol=1e-13)
    max_iter = int(z["max_iter"]) if "max_iter" in z else spec.max_iter
    # fp32 configs: the solver gets the generator's float32 arrays (kept as
    # float32, the exact values the reference saw as float64)
    prob = P.CoupledProblem(list(tensors), spec.rank, list(spec.coupled), mode=spec.mode)
    res = P.solve(prob, P.SolverOptions(max_iter=max_iter, tol=TINY_TOL, seed=0,
                                        precision=precision, **opt))
    return res, unpack_solve(z)


def test_config_c1_fp64_matches_reference(P):
    res, want = _config(P, "c1", "fp64")
    compare(res, want, rtol=1e-9)


def _final_state(res, want, rtol):
    for s, (blk, (wf, ww)) in enumerate(zip(res.factors.blocks, want["factors"])):
        _rel_close(blk.weights, ww, rtol, f"block {s} weights")
        for m, (a, b) in enumerate(zip(blk.factors, wf)):
            _rel_close(a, b, rtol, f"block {s} mode {m}")
    assert abs(res.rel_err_history[-1] - want["rel_err_history"][-1]) <= rtol * want["rel_err_history"][-1]


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_fp32_matches_reference(P, name):
    res, want = _config(P, name, "fp32")
    # exact-zero RelErr steps may end the run at a different iteration; compare
    # the common prefix of the histories (and the counts when the lengths
    # agree), then the final state
    compare(res, want, rtol=1e-4, prefix_only=True)
    _final_state(res, want, 1e-4)


# fp64 parity mode (north_star: 1e-9): histories element-wise over the common
# prefix; factors within max(1e-9, 10x the reference's own sensitivity to a
# 1e-15 input perturbation: c2 1.75e-8, c3 4.9e-14, c4 1.5e-12)
@pytest.mark.parametrize("name,factor_rtol", [("c2", 2e-7), ("c3", 1e-9), ("c4", 1e-9)])
def test_config_fp64_matches_reference(P, name, factor_rtol):
    res, want = _config(P, name, "fp64")
    compare(res, want, rtol=1e-9, prefix_only=True)
    if res.n_iter == want["n_iter"]:
        _final_state(res, want, factor_rtol)


def test_config_c5_subset_matches_reference(P):
    """c5 (64 x 400^3, R = 40, lra) pinned on blocks {0, 1}: the reference's
    ALS compression and 30 APG iterations (tests/golden/make_golden.py
    SUBSETS) against the default throughput path (fp32 storage, fp64 ALS and
    sweep, tensor-core trace pass)."""
    res, want = _config(P, "c5", "fp32")
    compare(res, want, rtol=1e-4, factor_rtol=1e-4)
    for s, (blk, (wf, _)) in enumerate(zip(res.compression, want["compression"])):
        for m, (a, b) in enumerate(zip(blk.factors, wf)):
            _rel_close(a, b, 1e-4, f"compression block {s} mode {m}")


def test_config_c5_subset_fp64_matches_reference(P):
    """c5 blocks {0, 1} in the fp64 parity mode (fp64 storage and arithmetic
    everywhere: ALS, sweep, the trace term by the CUDA-core fiber pass):
    histories element-wise at 1e-9 (north_star), iteration / restart counts,
    factors and the compression at 1e-8."""
    res, want = _config(P, "c5", "fp64")
    compare(res, want, rtol=1e-9, factor_rtol=1e-8)
    for s, (blk, (wf, _)) in enumerate(zip(res.compression, want["compression"])):
        for m, (a, b) in enumerate(zip(blk.factors, wf)):
            _rel_close(a, b, 1e-8, f"compression block {s} mode {m}")


def test_config_c5_subset_explicit_tc(P):
    """compute="tc" asked for explicitly (the default for these ranks): the
    tensor-core trace pass and the tensor-core ALS passes."""
    res, want = _config(P, "c5", "fp32", compute="tc")
    compare(res, want, rtol=1e-4, factor_rtol=1e-4)


@pytest.mark.parametrize("opt", [dict(compute="fp32"), dict(objective="explicit")])
def test_config_c2_fp32_variants_match_reference(P, opt):
    """fp32 arithmetic in the tensor passes / the explicit-residual objective
    in the throughput mode, against the reference's c2 run: the first 100
    iterations element-wise at 1e-4 (fp32 sums move late-run objectives by
    ~1e-7, enough to flip a restart decision afterwards, DESIGN 3)."""
    res, want = _config(P, "c2", "fp32", **opt)
    n = min(100, res.n_iter, want["n_iter"]) + 1
    _hist_close(res.objective_history[:n], want["objective_history"][:n], 1e-4, "objective_history")
    _hist_close(res.rel_err_history[:n], want["rel_err_history"][:n], 1e-4, "rel_err_history")


# ---- reference solver invariants (pkg/tests/test_solver.py) on the GPU ----

def _problem(P, seed, **kw):
    from cases import coupled
    snr = kw.pop("snr_db", None)
    counts = kw.pop("counts", (2, 2, 2))
    tensors = coupled(seed, counts=counts, snr_db=snr)
    return P.CoupledProblem(tensors, 4, list(counts), **kw)


def _monotone(hist, rel_tol=1e-10):
    arr = np.asarray(hist)
    bound = rel_tol * np.maximum(np.abs(arr[:-1]), 1.0)
    assert (np.diff(arr) <= bound).all()


def test_monotone_nonnegative_and_shared_columns(P):
    for mode in ("full", "lra"):
        prob = _problem(P, 8, counts=(2, 1, 0), mode=mode, snr_db=20.0)
        res = P.solve(prob, P.SolverOptions(max_iter=60, seed=2))
        _monotone(res.objective_history)
        for blk in res.factors.blocks:
            assert blk.is_nonnegative()
        for n, ln in enumerate(prob.coupled_counts):
            for blk in res.factors.blocks[1:]:
                np.testing.assert_array_equal(blk.factors[n][:, :ln],
                                              res.factors.blocks[0].factors[n][:, :ln])


def test_deterministic_reruns(P):
    a = P.solve(_problem(P, 10, snr_db=20.0), P.SolverOptions(max_iter=50, seed=4))
    b = P.solve(_problem(P, 10, snr_db=20.0), P.SolverOptions(max_iter=50, seed=4))
    assert a.objective_history == b.objective_history
    assert a.rel_err_history == b.rel_err_history
    for ba, bb in zip(a.factors.blocks, b.factors.blocks):
        np.testing.assert_array_equal(ba.weights, bb.weights)
        for fa, fb in zip(ba.factors, bb.factors):
            np.testing.assert_array_equal(fa, fb)


def test_fixed_core_and_max_iter_zero(P):
    res = P.solve(_problem(P, 9, update_core=False, snr_db=20.0), P.SolverOptions(max_iter=80, seed=3))
    for blk in res.factors.blocks:
        np.testing.assert_array_equal(blk.weights, np.ones(4))
    prob = _problem(P, 12)
    res = P.solve(prob, P.SolverOptions(max_iter=0, seed=6))
    assert res.n_iter == 0 and res.termination_reason == "max_iterations"
    assert len(res.objective_history) == 1 and len(res.trace) == 1
    start = P.init_factors(prob, seed=6)
    for got, want in zip(res.factors.blocks, start.blocks):
        for f_got, f_want in zip(got.factors, want.factors):
            np.testing.assert_array_equal(f_got, f_want)


def test_zero_tensors(P):
    prob = P.CoupledProblem([np.zeros((4, 5, 6)), np.zeros((4, 5, 6))], 3, [1, 1, 1])
    res = P.solve(prob, P.SolverOptions(max_iter=50, seed=7))
    assert res.rel_err_history[-1] == 0.0
    assert np.isfinite(res.objective_history).all()


def test_lra_trace_reports_original_tensor_quantities(P):
    prob = _problem(P, 16, snr_db=20.0, mode="lra")
    res = P.solve(prob, P.SolverOptions(max_iter=80, seed=11))
    want_obj = P.objective(prob.tensors, res.factors.blocks)
    assert res.trace[-1].obj_fun == pytest.approx(want_obj, rel=1e-8)
    assert res.compress_seconds > 0.0
    assert len(res.compression) == prob.n_blocks


def test_device_resident_fp32_inputs(P):
    """torch CUDA fp32 tensors in first-index-fastest layout are used in place."""
    import torch
    from cases import coupled
    from paper_2302_05119_b200._device import fortran_view
    tensors = coupled(6, snr_db=20.0)
    dev = []
    for t in tensors:
        flat = torch.from_numpy(np.ravel(t.astype(np.float32), order="F")).cuda()
        dev.append(fortran_view(flat, t.shape))
    res_dev = P.solve(P.CoupledProblem(dev, 4, [2, 2, 2]),
                      P.SolverOptions(max_iter=40, seed=1, precision="fp32"))
    res_host = P.solve(P.CoupledProblem([t.astype(np.float32).astype(float) for t in tensors], 4, [2, 2, 2]),
                       P.SolverOptions(max_iter=40, seed=1, precision="fp32"))
    assert res_dev.objective_history == res_host.objective_history


def test_staged_upload_compression_equals_resident_inputs(P):
    """lra on pinned host tensors: the blocks upload on a copy stream and the
    compression starts each block as it arrives (cb_als_desc.ready_events:
    deferred stats / plane packing / first T pass per arriving range,
    csrc/als.cu).  Blocks are fitted independently, so the compression and the
    solve equal, bitwise, those of the same blocks already resident on the
    device (all blocks started together)."""
    import torch
    from paper_2302_05119_b200._device import fortran_view
    rng = np.random.default_rng(12)
    shapes = [(96, 80, 72)] * 5
    host, dev = [], []
    for d in shapes:
        f = [rng.random((n, 20)) for n in d]
        x = np.einsum("ir,jr,kr->ijk", *f) + 0.3 * rng.standard_normal(d)
        flat = torch.from_numpy(np.ravel(np.maximum(x, 0).astype(np.float32), order="F").copy())
        pinned = torch.empty_strided(d, (1, d[0], d[0] * d[1]), dtype=torch.float32, pin_memory=True)
        pinned.copy_(fortran_view(flat, d))
        host.append(pinned)
        dev.append(fortran_view(flat.cuda(), d))
    out = {}
    for name, ts in (("host", host), ("dev", dev)):
        out[name] = P.solve(P.CoupledProblem(ts, 20, [5, 5, 0], mode="lra"),
                            P.SolverOptions(max_iter=30, seed=2, precision="fp32"))
    a, b = out["host"], out["dev"]
    assert a.compression_iters == b.compression_iters
    for ca, cb in zip(a.compression, b.compression):
        for fa, fb in zip(ca.factors, cb.factors):
            np.testing.assert_array_equal(fa, fb)
    assert a.objective_history == b.objective_history
    assert a.rel_err_history == b.rel_err_history
    # a non-finite block is still reported as the reference reports it
    bad = host[3].clone().pin_memory()
    bad[1, 2, 3] = float("nan")
    with pytest.raises(ValueError, match="block 3 contains non-finite values"):
        P.solve(P.CoupledProblem(host[:3] + [bad] + host[4:], 20, [5, 5, 0], mode="lra"),
                P.SolverOptions(max_iter=3, precision="fp32"))


def test_staged_upload_edge_cases(P):
    """Staged start with heterogeneous blocks (shapes and ranks differ), an
    all-zero block (rel err 0 from the start, cpd_als.py:84-86) and a
    compression capped at zero sweeps: same results as resident inputs."""
    import torch
    from paper_2302_05119_b200._device import fortran_view
    rng = np.random.default_rng(31)
    specs = [((64, 48, 40), 18), ((80, 48, 40), 24), ((64, 48, 56), 20), ((72, 48, 40), 17)]
    host, dev, ranks = [], [], []
    for k, (d, r) in enumerate(specs):
        f = [rng.random((n, r)) for n in d]
        x = np.einsum("ir,jr,kr->ijk", *f) + 0.2 * rng.standard_normal(d)
        x = np.maximum(x, 0).astype(np.float32)
        if k == 2:
            x[:] = 0.0
        flat = torch.from_numpy(np.ravel(x, order="F").copy())
        pinned = torch.empty_strided(d, (1, d[0], d[0] * d[1]), dtype=torch.float32, pin_memory=True)
        pinned.copy_(fortran_view(flat, d))
        host.append(pinned)
        dev.append(fortran_view(flat.cuda(), d))
        ranks.append(r)
    for als in (None, P.AlsOptions(max_iter=0), P.AlsOptions(max_iter=5, tol=1e-30)):
        out = {}
        for name, ts in (("host", host), ("dev", dev)):
            out[name] = P.solve(P.CoupledProblem(ts, ranks, [0, 6, 0], mode="lra", als_options=als),
                                P.SolverOptions(max_iter=12, seed=4, precision="fp32"))
        a, b = out["host"], out["dev"]
        assert a.compression_iters == b.compression_iters
        for ca, cb in zip(a.compression, b.compression):
            for fa, fb in zip(ca.factors, cb.factors):
                np.testing.assert_array_equal(fa, fb)
        assert a.objective_history == b.objective_history
        assert a.rel_err_history == b.rel_err_history


def test_staged_upload_falls_back_when_the_plan_is_unavailable(P, monkeypatch):
    """cb_als_create with upload events refuses blocks it cannot start one by
    one (CB_ERR_UNSUPPORTED: here small ranks, in production a plan that does
    not fit in device memory); solve() then finishes the uploads and runs the
    plain compression: same results as resident inputs."""
    import torch
    from paper_2302_05119_b200 import solver as S
    from paper_2302_05119_b200._device import fortran_view
    rng = np.random.default_rng(8)
    d = (24, 20, 16)
    host, dev = [], []
    for _ in range(3):
        x = np.maximum(rng.random(d) + 0.1 * rng.standard_normal(d), 0).astype(np.float32)
        flat = torch.from_numpy(np.ravel(x, order="F").copy())
        pinned = torch.empty_strided(d, (1, d[0], d[0] * d[1]), dtype=torch.float32, pin_memory=True)
        pinned.copy_(fortran_view(flat, d))
        host.append(pinned)
        dev.append(fortran_view(flat.cuda(), d))
    want = P.solve(P.CoupledProblem(dev, 4, [2, 2, 0], mode="lra"),
                   P.SolverOptions(max_iter=15, seed=3, precision="fp32"))
    monkeypatch.setattr(S, "als_staged_ok", lambda *a, **k: True)
    got = P.solve(P.CoupledProblem(host, 4, [2, 2, 0], mode="lra"),
                  P.SolverOptions(max_iter=15, seed=3, precision="fp32"))
    assert got.compression_iters == want.compression_iters
    assert got.objective_history == want.objective_history
    assert got.rel_err_history == want.rel_err_history


def test_device_value_checks_raise_reference_messages(P):
    """The single-process solve scans the uploaded blocks on the device; the
    errors are the reference's (solver.py:114-117), with the block index."""
    rng = np.random.default_rng(4)
    good = rng.random((6, 5, 4)).astype(np.float32)
    bad = good.copy()
    bad[1, 2, 3] = -0.5
    with pytest.raises(ValueError, match="block 1 contains negative entries"):
        P.solve(P.CoupledProblem([good, bad], 2, [0, 0, 0]),
                P.SolverOptions(max_iter=2, precision="fp32"))
    nan = good.copy()
    nan[0, 0, 0] = np.nan
    with pytest.raises(ValueError, match="block 0 contains non-finite values"):
        P.solve(P.CoupledProblem([nan, good], 2, [0, 0, 0]),
                P.SolverOptions(max_iter=2, precision="fp32"))


def test_value_checks_in_input_dtype_and_reference_order(P):
    """Values are scanned in the input's own dtype before the downcast to the
    solve precision, and errors come in the reference's order (per block:
    order, values; then ranks / counts; solver.py:96-135)."""
    rng = np.random.default_rng(5)
    good = rng.random((6, 5, 4))
    tiny = good.copy()
    tiny[2, 1, 0] = -1e-300            # flushes to -0.0 in fp32: must still raise
    with pytest.raises(ValueError, match="block 1 contains negative entries"):
        P.solve(P.CoupledProblem([good, tiny], 2, [0, 0, 0]),
                P.SolverOptions(max_iter=2, precision="fp32"))
    huge = good.copy()
    huge[0, 0, 0] = 1e300              # finite in fp64 (inf after an fp32 cast)
    with pytest.raises(ValueError, match="exceeds minimum rank"):
        P.solve(P.CoupledProblem([huge, good], 2, [3, 0, 0]),
                P.SolverOptions(max_iter=2, precision="fp32"))
    # a value error of block 0 comes before a rank error, an order error of
    # block 0 before a value error of block 1
    with pytest.raises(ValueError, match="block 0 contains negative entries"):
        P.solve(P.CoupledProblem([-good, good], [0, 2], [0, 0, 0]), P.SolverOptions(max_iter=2))
    with pytest.raises(ValueError, match="block 1 has order 2"):
        P.solve(P.CoupledProblem([good, good[:, :, 0], -good], 2, [0, 0, 0]),
                P.SolverOptions(max_iter=2))
    # lra (the compression engine is set up beside the upload, before the
    # value checks complete): a value error still comes before the
    # compression's own feasibility error (solver.py:556-573)
    als = P.AlsOptions(rank=50)
    with pytest.raises(ValueError, match="block 1 contains negative entries"):
        P.solve(P.CoupledProblem([good, -good], 2, [0, 0, 0], mode="lra", als_options=als),
                P.SolverOptions(max_iter=2))
    with pytest.raises(ValueError, match="compression of block 0 failed"):
        P.solve(P.CoupledProblem([good, good], 2, [0, 0, 0], mode="lra", als_options=als),
                P.SolverOptions(max_iter=2))
    nan = good.copy()
    nan[1, 1, 1] = np.inf
    with pytest.raises(ValueError, match="block 1 contains non-finite values"):
        P.solve(P.CoupledProblem([good, nan], 2, [0, 0, 0], mode="lra"),
                P.SolverOptions(max_iter=2))
