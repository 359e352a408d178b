"""GPU tests of the block-sharded (multi-GPU) code path.

Only one GPU is available to the tests, so the sharded program runs as an
EMULATED group (`solve_emulated_shards`, `cb_group_run`): one engine handle
per rank, each owning a contiguous range of blocks, stepped segment by
segment on one stream with the all-reduces of the couplings (per-mode
Lipschitz sums, common-column gradient partials, per-block evaluation terms;
SURVEY 8e) done by a summing kernel between segments.  The kernels, the
global-slot exchange buffers and the segment boundaries are exactly those of
the NCCL path; only the transport differs.  Because the exchanged arrays have
disjoint support and every fold runs in global block order, a sharded solve
must reproduce the single-GPU solve BIT FOR BIT, and it is tested that way
(and against the reference fixtures through the single-GPU parity tests)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2302_05119_b200 as P
    return P


def _problem_tensors(S=5, dims=(14, 12, 16), rank=5, counts=(2, 2, 2), seed=3):
    rng = np.random.default_rng(seed)
    common = [rng.random((d, c)) for d, c in zip(dims, counts)]
    out = []
    for _ in range(S):
        facs = [np.hstack([common[n], rng.random((dims[n], rank - counts[n]))]) for n in range(3)]
        t = np.einsum("ir,jr,kr->ijk", *facs)
        out.append(np.maximum(t + 0.05 * rng.standard_normal(t.shape), 0.0))
    return out


def _same(a, b):
    assert a.n_iter == b.n_iter
    assert a.n_restarts == b.n_restarts
    assert a.termination_reason == b.termination_reason
    np.testing.assert_array_equal(a.objective_history, b.objective_history)
    np.testing.assert_array_equal(a.rel_err_history, b.rel_err_history)
    for x, y in zip(a.factors.blocks, b.factors.blocks):
        np.testing.assert_array_equal(x.weights, y.weights)
        for u, v in zip(x.factors, y.factors):
            np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("mode", ["full", "lra"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_sharded_equals_single_gpu_fp64(P, mode, world):
    tensors = _problem_tensors()
    prob = P.CoupledProblem(tensors, 5, [2, 2, 2], mode=mode)
    opts = P.SolverOptions(max_iter=60, seed=4)
    want = P.solve(prob, opts)
    got = P.solver.solve_emulated_shards(prob, opts, world=world)
    _same(got, want)


def test_sharded_equals_single_gpu_fp32_c2_blocks(P):
    """fp32 storage (throughput mode) on c2-shaped blocks, uneven shards."""
    from paper_2302_05119_b200.configs import generate_config
    tensors, spec = generate_config("c2", blocks=range(4))
    prob = P.CoupledProblem([np.asarray(t, dtype=float) for t in tensors], spec.rank,
                            list(spec.coupled), mode=spec.mode)
    opts = P.SolverOptions(max_iter=200, seed=0, precision="fp32")
    want = P.solve(prob, opts)
    got = P.solver.solve_emulated_shards(prob, opts, world=3)
    _same(got, want)
    assert want.n_restarts > 0   # the restart branch (restore + redo sweep) is exercised


def test_sharded_uncoupled_mode_and_tolerance_stop(P):
    """L_n = 0 in one mode (no exchange there) and a tolerance stop."""
    tensors = _problem_tensors(S=4, counts=(3, 0, 2))
    prob = P.CoupledProblem(tensors, 5, [3, 0, 2])
    opts = P.SolverOptions(max_iter=400, tol=1e-7, seed=2)
    want = P.solve(prob, opts)
    got = P.solver.solve_emulated_shards(prob, opts, world=2)
    _same(got, want)
    assert want.termination_reason == "tolerance"


def test_shard_argument_errors(P):
    tensors = _problem_tensors(S=2)
    prob = P.CoupledProblem(tensors, 5, [2, 2, 2])
    with pytest.raises(ValueError):
        P.solver.solve_emulated_shards(prob, P.SolverOptions(max_iter=3), world=3)


def test_nccl_path_single_rank_equals_single_gpu(P, tmp_path):
    """The NCCL transport on one GPU: a world-1 NCCL communicator makes the
    engine run the sharded program (all-reduces captured in the iteration
    graph); the result must equal the plain solve bit for bit."""
    import socket
    import torch
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        for mode in ("full", "lra"):
            tensors = _problem_tensors(S=3)
            prob = P.CoupledProblem(tensors, 5, [2, 2, 2], mode=mode)
            opts = P.SolverOptions(max_iter=40, seed=1)
            want = P.solve(prob, opts)
            got = P.solver.solve_distributed(prob, opts)
            _same(got, want)
        # restarts through the conditional restart bodies split at the NCCL
        # exchanges (fp32 storage, c2-shaped blocks)
        from paper_2302_05119_b200.configs import generate_config
        tensors, spec = generate_config("c2", blocks=range(3))
        prob = P.CoupledProblem(list(tensors), spec.rank, list(spec.coupled))
        opts = P.SolverOptions(max_iter=200, seed=0, precision="fp32")
        want = P.solve(prob, opts)
        got = P.solver.solve_distributed(prob, opts)
        _same(got, want)
        assert want.n_restarts > 0
        # the pipelined lra iteration under sharding (trace pass beside the
        # next sweep, exchanges on the sweep stream), max_iter and tol stops
        rng = np.random.default_rng(33)
        facs = lambda d: [rng.random((n, 20)) for n in d]  # noqa: E731
        blocks = []
        for _ in range(3):
            f = facs((64, 40, 30))
            t = np.einsum("ir,jr,kr->ijk", *f)
            blocks.append(np.maximum(t + 0.05 * rng.standard_normal(t.shape), 0.0).astype(np.float32))
        for tol, mi in ((1e-30, 40), (1e-5, 400)):
            prob = P.CoupledProblem(blocks, 20, [5, 5, 0], mode="lra")
            kw = dict(max_iter=mi, tol=tol, seed=5, precision="fp32", compute="tc", pipeline="on")
            want = P.solve(prob, P.SolverOptions(**kw))
            got = P.solver.solve_distributed(prob, P.SolverOptions(**kw))
            _same(got, want)
            off = P.solve(prob, P.SolverOptions(**{**kw, "pipeline": "off"}))
            _same(off, want)
    finally:
        dist.destroy_process_group()
