"""CPU tests of the block-sharded (multi-GPU) design with world_size 2 over
torch.distributed `gloo`.

The GPU engine shards blocks across ranks and exchanges exactly three kinds
of coupling data, each as an all-reduce (sum) of a GLOBAL-SLOT array whose
foreign slots are zero (csrc/engine.h, Ctx::S_tot):
  1. before the mode-n update: every block's (L_u, L_u,prev)   (solver.py:422-425)
  2. after it: every block's common-column gradient partial    (solver.py:444)
  3. per evaluation: every block's residual / RelErr terms      (solver.py:593-610)
after which every rank folds the S_tot slots in global block order.  These
tests run that protocol with real processes on the CPU: a sharded APG built
from the oracle's per-block steps, exchanging only those three arrays through
gloo, must reproduce the single-process oracle trajectory BIT FOR BIT.  They
also pin the exactness premise (a disjoint-support all-reduce is an exact
all-gather, including NaN / inf / signed zeros) and the host helpers
(`shard_ranges`)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import concpd_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    port = _free_port()
    mp.spawn(_entry, args=(fn, world, port) + args, nprocs=world, join=True)


def _entry(rank, fn, world, port, *args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _allreduce(arr):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


# ---------------------------------------------------------------------------
def test_shard_ranges():
    from paper_2302_05119_b200.solver import shard_ranges
    for S in (1, 2, 5, 10, 64):
        for P in range(1, min(S, 8) + 1):
            rs = shard_ranges(S, P)
            assert rs[0][0] == 0 and rs[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [e - b for b, e in rs]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_ranges(2, 3)


# ---------------------------------------------------------------------------
def _exactness(rank, world, S_tot):
    rng = np.random.default_rng(7)
    vals = rng.standard_normal(S_tot) * 10.0 ** rng.integers(-300, 300, S_tot)
    vals[1] = np.nan
    vals[2] = np.inf
    vals[3] = -np.inf
    vals[4] = 5e-324
    b, e = rank * S_tot // world, (rank + 1) * S_tot // world
    send = np.zeros(S_tot)
    send[b:e] = vals[b:e]
    got = _allreduce(send)
    same = (got == vals) | (np.isnan(got) & np.isnan(vals))
    assert same.all(), (rank, got, vals)


def test_global_slot_allreduce_is_exact_gather():
    _spawn(_exactness, 2, 11)


# ---------------------------------------------------------------------------
def _sharded_apg(X, ranks, counts, max_iter, seed, delta_w, lo, hi, S_tot, exchange):
    """CoNCPD-APG (full mode) over blocks [lo, hi) of S_tot, with the couplings
    exchanged through `exchange(global_slot_array) -> summed array`."""
    N = X[0].ndim
    allshapes = [None] * S_tot
    for g in range(lo, hi):
        allshapes[g] = X[g - lo].shape
    # every rank draws the whole seeded start (one PCG64 stream), keeps its own
    shapes = exchange_shapes(allshapes, exchange)
    start = O.draw_init(shapes, ranks, counts, True, seed)
    loc = range(lo, hi)
    U = {g: [f.copy() for f in start[g][0]] for g in loc}
    lam = {g: start[g][1].copy() for g in loc}
    Up = {g: [f.copy() for f in U[g]] for g in loc}
    lamp = {g: lam[g].copy() for g in loc}
    Xg = {g: X[g - lo] for g in loc}
    nsq = {g: float(np.vdot(Xg[g], Xg[g])) for g in loc}
    M0 = {g: O.unfold(Xg[g], 0) for g in loc}

    def mttkrp(g, n):
        mn = M0[g] if n == 0 else O.unfold(Xg[g], n)
        return mn @ O.kr_desc(U[g], skip=n)
    Lc = {g: None for g in loc}
    Lf = [{g: None for g in loc} for _ in range(N)]
    b = {}

    def gram(g, skip=None):
        return O._hprod([f.T @ f for f in U[g]], skip=skip)

    def evaluate(first=False):
        terms = np.zeros(2 * S_tot)
        staged = {}
        for g in loc:
            f, w = U[g], lam[g]
            kr0 = O.kr_desc(f, skip=0)
            m0 = M0[g]
            d = m0 - (f[0] * w) @ kr0.T
            r = float(np.einsum("ij,ij->", d, d))
            # b staged from the last mode's MTTKRP (iteration 0: mode 0), solver.py:506-511
            staged[g] = (np.einsum("ir,ir->r", f[0], m0 @ kr0) if first else
                         np.einsum("ir,ir->r", f[N - 1], mttkrp(g, N - 1)))
            terms[g] = r
            terms[S_tot + g] = np.sqrt(max(r, 0.0)) / np.sqrt(nsq[g])
        terms = exchange(terms)                                   # exchange 3
        oi, rel = 0.0, 0.0
        for q in range(S_tot):
            oi += 0.5 * terms[q]
            rel += terms[S_tot + q]
        return oi, rel / S_tot, staged

    def sweep(w_hat):
        for g in loc:                                             # core update (local)
            gall = gram(g)
            ld = O.top_eig(gall)
            ldp = Lc[g] if Lc[g] is not None else ld
            Lc[g] = ld
            w = O.extrap_w(w_hat, ldp, ld, delta_w)
            lh = lam[g] + w * (lam[g] - lamp[g])
            lamp[g] = lam[g]
            lam[g] = np.maximum(0.0, lh - (gall @ lh - b[g]) / ld)
        for n in range(N):
            ln = counts[n]
            lip = np.zeros(2 * S_tot)
            step = {}
            for g in loc:
                step[g] = gram(g, skip=n) * np.outer(lam[g], lam[g])
                lu = O.top_eig(step[g])
                lip[S_tot + g] = Lf[n][g] if Lf[n][g] is not None else lu
                lip[g] = lu
                Lf[n][g] = lu
            if ln > 0:
                lip = exchange(lip)                               # exchange 1
            lsum = sum(lip[q] for q in range(S_tot))
            lsump = sum(lip[S_tot + q] for q in range(S_tot))
            c0 = U[lo][n][:, :ln]
            ch = c0 + O.extrap_w(w_hat, lsump, lsum, delta_w) * (c0 - Up[lo][n][:, :ln])
            part = np.zeros((S_tot,) + ch.shape)
            own = {}
            for g in loc:
                u, lu = U[g][n], lip[g]
                if lu == 0.0:
                    own[g] = u[:, ln:].copy()
                    continue
                w = O.extrap_w(w_hat, lip[S_tot + g], lu, delta_w)
                ih = u[:, ln:] + w * (u[:, ln:] - Up[g][n][:, ln:])
                uh = np.hstack([ch, ih])
                grad = uh @ step[g] - mttkrp(g, n) * lam[g]
                part[g] = grad[:, :ln]
                own[g] = np.maximum(0.0, ih - grad[:, ln:] / lu)
            if ln > 0:
                part = exchange(part.reshape(-1)).reshape(part.shape)   # exchange 2
                acc = np.zeros_like(ch)
                for q in range(S_tot):
                    if lip[q] > 0.0:
                        acc = acc + part[q]
                cn = np.maximum(0.0, ch - acc / lsum) if lsum > 0.0 else c0.copy()
            for g in loc:
                Up[g][n] = U[g][n]
                U[g][n] = np.hstack([cn, own[g]]) if ln > 0 else own[g]

    oi, rel, staged = evaluate(first=True)
    b.update(staged)
    hist, rels, restarts, t_k = [oi], [rel], 0, 1.0
    for k in range(1, max_iter + 1):
        t_new = O.next_t(t_k)
        w_hat = (t_k - 1.0) / t_new
        t_k = t_new
        sweep(w_hat)
        oi, new_rel, staged = evaluate()
        if oi >= hist[-1]:
            restarts += 1
            for g in loc:
                lam[g] = lamp[g].copy()
                U[g] = [f.copy() for f in Up[g]]
            sweep(0.0)
            oi, new_rel, staged = evaluate()
        b.update(staged)
        hist.append(oi)
        rels.append(new_rel)
    return hist, rels, restarts, {g: (U[g], lam[g]) for g in loc}


def exchange_shapes(allshapes, exchange):
    dims = np.zeros((len(allshapes), 3))
    for g, sh in enumerate(allshapes):
        if sh is not None:
            dims[g] = sh
    dims = exchange(dims.reshape(-1)).reshape(dims.shape)
    return [tuple(int(v) for v in row) for row in dims]


def _problem(S=5, dims=(9, 8, 10), rank=4, counts=(2, 0, 1), seed=5):
    rng = np.random.default_rng(seed)
    common = [rng.random((d, c)) for d, c in zip(dims, counts)]
    out = []
    for _ in range(S):
        facs = [np.hstack([common[n], rng.random((dims[n], rank - counts[n]))]) for n in range(3)]
        t = O.dense_from_model(facs, np.ones(rank))
        out.append(np.maximum(t + 0.1 * rng.standard_normal(t.shape), 0.0))
    return out, rank, list(counts)


def _sharded_rank(rank, world, max_iter, result_dir):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)   # same BLAS blocking (summation order) as the parent's oracle run
    X, R, counts = _problem()
    S = len(X)
    lo, hi = rank * S // world, (rank + 1) * S // world
    hist, rels, restarts, blocks = _sharded_apg(X[lo:hi], [R] * S, counts, max_iter, 3, 0.9999,
                                                lo, hi, S, _allreduce)
    np.savez(os.path.join(result_dir, f"rank{rank}.npz"), hist=hist, rels=rels,
             restarts=restarts,
             **{f"U{g}_{n}": blocks[g][0][n] for g in blocks for n in range(3)},
             **{f"lam{g}": blocks[g][1] for g in blocks})


def test_sharded_protocol_reproduces_oracle_bits(tmp_path):
    """2 gloo ranks == 1 process bit for bit (the sharding changes nothing);
    the restated APG itself matches the oracle to rounding (1e-12)."""
    max_iter = 40
    _spawn(_sharded_rank, 2, max_iter, str(tmp_path))
    X, R, counts = _problem()
    S = len(X)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        one = _sharded_apg(X, [R] * S, counts, max_iter, 3, 0.9999, 0, S, S, lambda a: a)
        want = O.solve_oracle(X, R, counts, max_iter=max_iter, tol=0.0, seed=3)
    hist1, rels1, restarts1, blocks1 = one
    for rank in range(2):
        got = np.load(tmp_path / f"rank{rank}.npz")
        np.testing.assert_array_equal(got["hist"], hist1)
        np.testing.assert_array_equal(got["rels"], rels1)
        assert int(got["restarts"]) == restarts1
        lo, hi = rank * S // 2, (rank + 1) * S // 2
        for g in range(lo, hi):
            np.testing.assert_array_equal(got[f"lam{g}"], blocks1[g][1])
            for n in range(3):
                np.testing.assert_array_equal(got[f"U{g}_{n}"], blocks1[g][0][n])
    np.testing.assert_allclose(hist1, want["objective_history"], rtol=1e-12)
    np.testing.assert_allclose(rels1, want["rel_err_history"], rtol=1e-12)
    assert restarts1 == want["n_restarts"]
    for g in range(S):
        np.testing.assert_allclose(blocks1[g][1], want["factors"][g][1], rtol=1e-10, atol=1e-13)
        for n in range(3):
            np.testing.assert_allclose(blocks1[g][0][n], want["factors"][g][0][n], rtol=1e-10,
                                       atol=1e-13)
