"""GPU parity of the tensor-core trace pass (`cb_core_linear_term_tc`,
csrc/xtc.cu) against the oracle's core linear term (oracle/concpd_oracle.py
`core_term`, reference solver.py:215-218), fp64 on the same fp32-rounded
inputs.

The pass rounds X to 2^-21 of its block maximum and A0 to 2^-23 of each
column maximum (unbiased) and accumulates exactly in int32; the bound
asserted is 2e-7 relative to sum |X||A0||A1||A2| per rank column (observed
~2e-8), plus bitwise determinism and independence of the batching."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import concpd_oracle as O


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


def _block(rng, dims, rank, signed=False):
    f = [rng.random((d, rank)) for d in dims]
    if signed:
        f = [x - 0.5 for x in f]
    x = O.dense_from_model(f, np.ones(rank)) + 0.1 * rng.standard_normal(dims)
    if not signed:
        x = np.maximum(x, 0.0)
    x = np.asfortranarray(x.astype(np.float32))
    g = [rng.random((d, rank)) - (0.5 if signed else 0.0) for d in dims]
    return x, g


def _want(x, g):
    x64 = np.asarray(x, dtype=np.float64)
    want = O.core_term(x64, g)
    scale = O.core_term(np.abs(x64), [np.abs(a) for a in g])
    return want, scale


SHAPES = [
    ((400, 24, 30), 40),     # c5-like rank, K tail (400 = 6 x 64 + 16)
    ((112, 92, 40), 20),     # c3 mode sizes (shortened), J tail tile
    ((64, 71, 60), 30),      # c4 shape
    ((100, 100, 10), 10),    # c2 modes, N bucket 16
    ((36, 20, 7), 40),       # the largest rank (3 x 40 lanes), a single partial tile
    ((50, 33, 21), 33),      # rank not a multiple of 8, ragged everything
    ((4, 19, 2), 3),         # tiny
]


@pytest.mark.parametrize("signed", [False, True])
def test_tc_trace_matches_oracle(P, signed):
    rng = np.random.default_rng(11 if signed else 7)
    for dims, rank in SHAPES:
        x, g = _block(rng, dims, rank, signed)
        got = P.core_linear_terms_tc([x], [g])[0]
        want, scale = _want(x, g)
        err = np.abs(got - want) / scale
        # relative to sum |.| (signed data cancels inside b); tiny blocks do
        # not average the 2^-21 input rounding, so they get the per-product
        # bound
        tol = 2e-7 if x.size >= 10000 else 4e-6
        assert err.max() < (2.5 * tol if signed else tol), (dims, rank, err.max())


def test_tc_trace_batched_ragged_and_deterministic(P):
    rng = np.random.default_rng(3)
    blocks = [_block(rng, d, r) for d, r in SHAPES[:4]]
    # ranks differ per block: the N bucket is the maximum
    xs = [b[0] for b in blocks]
    gs = [b[1] for b in blocks]
    got = P.core_linear_terms_tc(xs, gs)
    again = P.core_linear_terms_tc(xs, gs)
    for a, b in zip(got, again):
        assert np.array_equal(a, b)              # bitwise run-to-run
    for s, (x, g) in enumerate(blocks):
        want, scale = _want(x, g)
        assert (np.abs(got[s] - want) / scale).max() < 2e-7
    # a block's result does not depend on its batch neighbours (fixed units)
    single = P.core_linear_terms_tc([xs[1]], [gs[1]])[0]
    # (alone it may use a smaller N bucket: same products, same fold order)
    assert np.array_equal(single, got[1])


def test_tc_trace_rejects_unsupported_shapes(P):
    rng = np.random.default_rng(1)
    for dims, rank in (((6, 5, 4), 3), ((516, 20, 4), 3), ((36, 20, 7), 41)):   # I1 < 16; I0 > 512; rank > 40
        x, g = _block(rng, dims, rank)
        with pytest.raises(Exception):
            P.core_linear_terms_tc([x], [g])


def test_tc_trace_odd_leading_size(P):
    """I0 not a multiple of 4 or 32 (the pack pads K with zeros)."""
    rng = np.random.default_rng(2)
    for dims, rank in (((30, 20, 4), 3), ((45, 37, 11), 12), ((33, 64, 9), 20)):
        x, g = _block(rng, dims, rank)
        got = P.core_linear_terms_tc([x], [g])[0]
        want, scale = _want(x, g)
        assert (np.abs(got - want) / scale).max() < 4e-6, dims


def test_tc_trace_zero_and_scaled(P):
    rng = np.random.default_rng(5)
    x, g = _block(rng, (64, 20, 20), 8)
    z = np.zeros_like(x)
    assert np.array_equal(P.core_linear_terms_tc([z], [g])[0], np.zeros(8))
    # power-of-two scalings are exact in the fixed-point representation
    a = P.core_linear_terms_tc([x], [g])[0]
    b = P.core_linear_terms_tc([np.asfortranarray(x * np.float32(1024.0))], [g])[0]
    np.testing.assert_array_equal(b, a * 1024.0)


def test_tc_trace_c5_block(P):
    """One full c5 block (400^3 fp32, R = 40): the size the roofline runs on."""
    from paper_2302_05119_b200.configs import generate_config
    xs, spec = generate_config("c5", blocks=[0])
    rng = np.random.default_rng(0)
    g = [rng.random((d, spec.rank)) for d in spec.dims]
    got = P.core_linear_terms_tc(xs, [g])[0]
    x64 = np.asarray(xs[0], dtype=np.float64)
    want = O.core_term(x64, g)
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() < 1e-7, rel.max()


def test_plane_gemm_als_small_blocks_match_fp64_als(P):
    """ALS compression with both tensor passes as exact int8 slice GEMMs over
    the packed byte planes (csrc/xoz.cu: ragged tiles, K not a multiple of 32,
    rank buckets 32 and 48) against the fp64-storage ALS on the same values:
    relative-error histories within 1e-10 absolute per sweep, factors within
    1e-8 relative after 12 sweeps."""
    import torch
    from paper_2302_05119_b200 import _lib as L
    from paper_2302_05119_b200 import _device as D
    from paper_2302_05119_b200.cpd_als import als_compress_blocks
    rng = np.random.default_rng(21)
    shapes = [((64, 40, 50), 20), ((96, 36, 30), 24), ((70, 45, 33), 40), ((33, 70, 45), 17)]
    dev32, dims = [], []
    for d, r in shapes:
        x, _ = _block(rng, d, r)
        flat, dd = D.tensor_to_dev(x, "fp32")
        dev32.append(flat)
        dims.append(dd)
    dev64 = [f.to(torch.float64) for f in dev32]
    ranks = [r for _, r in shapes]
    st = L.c_vp(torch.cuda.current_stream().cuda_stream)
    out = {}
    for code, data in ((L.CB_F32, dev32), (L.CB_F64, dev64)):
        h = als_compress_blocks(data, dims, ranks, 1e-30, 12, list(range(len(shapes))), code, st, 0,
                                total_blocks=len(shapes))
        out[code] = [h.block(s) for s in range(len(shapes))]
        h.close()
    for s in range(len(shapes)):
        fa, _, ha, na, _ = out[L.CB_F32][s]
        fb, _, hb, nb, _ = out[L.CB_F64][s]
        assert na == nb == 12
        np.testing.assert_allclose(ha, hb, rtol=0, atol=1e-10)
        for a, b in zip(fa, fb):
            assert np.abs(a - b).max() <= 1e-8 * np.abs(b).max()


@pytest.mark.parametrize("tol,max_iter", [(1e-30, 40), (1e-5, 400)])
def test_pipelined_lra_iteration_is_bitwise_unpipelined(P, tol, max_iter):
    """The pipelined lra iteration (csrc/engine.cu enqueue_pipe_*: the trace of
    iteration k beside the sweep of k+1, snapshots, rollback on stop) returns
    the unpipelined solve's factors, histories and stop iteration bitwise,
    both at max_iter and at an early tol stop (the rollback path)."""
    rng = np.random.default_rng(33)
    tensors = [_block(rng, (64, 40, 30), 20)[0] for _ in range(3)]
    out = {}
    for pipe in (True, False):
        prob = P.CoupledProblem(tensors, 20, [5, 5, 0], mode="lra")
        out[pipe] = P.solve(prob, P.SolverOptions(max_iter=max_iter, tol=tol, seed=5,
                                                  precision="fp32", compute="tc",
                                                  pipeline="on" if pipe else "off"))
    a, b = out[True], out[False]
    assert a.n_iter == b.n_iter and a.termination_reason == b.termination_reason
    if tol > 1e-20:
        assert a.n_iter < max_iter            # the stop (and rollback) path ran
    assert a.objective_history == b.objective_history
    assert a.rel_err_history == b.rel_err_history
    assert a.n_restarts == b.n_restarts
    for ba, bb in zip(a.factors.blocks, b.factors.blocks):
        np.testing.assert_array_equal(ba.weights, bb.weights)
        for fa, fb in zip(ba.factors, bb.factors):
            np.testing.assert_array_equal(fa, fb)


def test_pipelined_iteration_with_a_restart_is_bitwise_unpipelined(P):
    """c3 (device-generated blocks) restarts once: the pipelined iteration
    prepares the next trace's operands right after the sweep, beside the
    running trace, and the restart branch re-prepares them from the redone
    sweep (csrc/engine.cu PREP_SPEC / PREP_REDO); histories, counts and
    factors equal the unpipelined solve's bitwise."""
    from paper_2302_05119_b200.synth import generate_config_device
    dev, spec = generate_config_device("c3")
    out = {}
    for pipe in ("on", "off"):
        prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
        out[pipe] = P.solve(prob, P.SolverOptions(max_iter=spec.max_iter, tol=float(np.nextafter(0, 1)),
                                                  seed=0, precision="fp32", pipeline=pipe))
    a, b = out["on"], out["off"]
    assert a.n_restarts == b.n_restarts and a.n_restarts >= 1
    assert a.n_iter == b.n_iter
    assert a.objective_history == b.objective_history
    assert a.rel_err_history == b.rel_err_history
    for ba, bb in zip(a.factors.blocks, b.factors.blocks):
        np.testing.assert_array_equal(ba.weights, bb.weights)
        for fa, fb in zip(ba.factors, bb.factors):
            np.testing.assert_array_equal(fa, fb)


def test_tc_trace_stop_iteration_near_the_fp64_trace(P):
    """At the default tol = 1e-8 the stop rule |rel_k - rel_{k-1}| < tol sees the
    tensor-core trace's fixed-point rounding of A0 (2^-23 of a column maximum,
    fresh every iteration; the X planes are fixed for the whole solve), ~1e-8
    on these small blocks where K = I0 = 64 averages little: the solve may
    stop some iterations away from the fp64 CUDA-core trace's stop (measured
    490 vs 463).  The common prefix of the traces and the final RelErr agree
    to 2e-5 relative (measured 7e-6; the fp32 mode's contract is 1e-4);
    compute="fp64" gives the exact stop."""
    rng = np.random.default_rng(44)
    tensors = [_block(rng, (64, 40, 30), 20)[0] for _ in range(3)]
    out = {}
    for compute in ("tc", "fp64"):
        prob = P.CoupledProblem(tensors, 20, [5, 5, 0], mode="lra")
        out[compute] = P.solve(prob, P.SolverOptions(max_iter=4000, seed=5, precision="fp32",
                                                     compute=compute))
    a, b = out["tc"], out["fp64"]
    assert b.termination_reason == "tolerance" and a.termination_reason == "tolerance"
    assert abs(a.n_iter - b.n_iter) <= 0.1 * b.n_iter
    n = min(a.n_iter, b.n_iter) + 1
    np.testing.assert_allclose(a.rel_err_history[:n], b.rel_err_history[:n], rtol=2e-5)
    np.testing.assert_allclose(a.rel_err_history[-1], b.rel_err_history[-1], rtol=2e-5)


@pytest.mark.parametrize("name,blocks", [("c5", [0, 1]), ("c3", [0, 1, 2])])
def test_gemm_pass_als_matches_explicit_fp64_als(P, name, blocks):
    """The fp32-storage ALS of ranks > 16 (both tensor passes as exact int8
    slice GEMMs on the tensor cores over packed byte planes, residual by the
    gram expansion; csrc/xoz.cu, csrc/als.cu) against the fp64-storage ALS on the same values
    (explicit residual, the reference's formula cpd_als.py:107-110): the
    relative-error histories within 1e-10 absolute per sweep, same number of
    sweeps, factors within 1e-8 relative."""
    import torch
    from paper_2302_05119_b200 import _lib as L
    from paper_2302_05119_b200.cpd_als import als_compress_blocks
    from paper_2302_05119_b200.synth import generate_config_device
    dev, spec = generate_config_device(name, blocks=blocks)
    flat32 = [t.permute(2, 1, 0).contiguous().reshape(-1) for t in dev]
    flat64 = [f.to(torch.float64) for f in flat32]
    dims = [tuple(spec.dims)] * len(blocks)
    st = L.c_vp(torch.cuda.current_stream().cuda_stream)
    out = {}
    for code, data in ((L.CB_F32, flat32), (L.CB_F64, flat64)):
        h = als_compress_blocks(data, dims, [spec.rank] * len(blocks), 1e-4, 200,
                                [0 + b for b in blocks], code, st, 0, total_blocks=spec.n_blocks)
        out[code] = [h.block(s) for s in range(len(blocks))]
        h.close()
    for s in range(len(blocks)):
        fa, _, ha, na, ca = out[L.CB_F32][s]
        fb, _, hb, nb, cb = out[L.CB_F64][s]
        assert na == nb and ca == cb
        np.testing.assert_allclose(ha, hb, rtol=0, atol=1e-10)
        for a, b in zip(fa, fb):
            assert np.abs(a - b).max() <= 1e-8 * np.abs(b).max()
