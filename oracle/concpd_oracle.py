"""CPU ORACLE for the CoNCPD-APG / lraCoNCPD-APG hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`/root/reference/pkg/src/concpd`, arXiv 2302.05119).  It exists so that the
GPU product can be checked on the GPU box, where the reference itself is not
present.  It is NOT part of the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it, and only as the checker or the timed CPU
baseline.  The product package never imports it and has no CPU fallback.

Pinning: ``tests/golden/make_golden.py`` runs the real reference in the
build container and stores its outputs under ``tests/golden/``;
``tests/test_oracle_pinning.py`` checks every function here against those
fixtures (and against the reference's own known answers, e.g. the recovery
table in ``pkg/test_output.txt:266-276``).  Parity status: PINNED.

Every function cites the reference file:line it restates.  Arithmetic is
kept in the same order as the reference where that decides the last bits
(gram products in mode order, explicit residuals, ``eigvalsh``), so that the
oracle reproduces the reference trajectories bit-for-bit on the fixtures.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "unfold", "fold", "kr_columns", "kr_desc", "gram_hadamard", "top_eig",
    "mttkrp", "core_term", "core_term_lra", "mttkrp_lra", "full_objective",
    "next_t", "extrap_w", "draw_init", "dense_from_model", "als_fit",
    "solve_oracle",
]


# ----------------------------------------------------------------------------
# layout conventions (tensor_ops.py:1-15: first index fastest)
# ----------------------------------------------------------------------------

def unfold(t, n):
    """Mode-n unfolding, remaining modes ascending, lower fastest.
    Restates tensor_ops.py:45-54."""
    t = np.asarray(t)
    return np.moveaxis(t, n, 0).reshape((t.shape[n], -1), order="F")


def fold(m, n, dims):
    """Inverse of :func:`unfold`.  Restates tensor_ops.py:57-63."""
    dims = tuple(int(d) for d in dims)
    lead = (dims[n],) + tuple(d for k, d in enumerate(dims) if k != n)
    return np.moveaxis(np.asarray(m).reshape(lead, order="F"), 0, n)


def kr_columns(mats):
    """Column-wise Kronecker product, first matrix slowest.
    Restates tensor_ops.py:66-85."""
    acc = np.asarray(mats[0])
    cols = acc.shape[1]
    for nxt in mats[1:]:
        nxt = np.asarray(nxt)
        acc = (acc[:, None, :] * nxt[None, :, :]).reshape(-1, cols)
    return acc


def kr_desc(factors, skip=None):
    """Khatri-Rao of the factor list in descending mode order.
    Restates tensor_ops.py:88-95."""
    kept = [f for k, f in enumerate(factors) if k != skip]
    return kr_columns(kept[::-1])


def gram_hadamard(mats, skip=None, mats2=None):
    """Element-wise product over modes of mats[n].T @ mats2[n].
    Restates tensor_ops.py:98-124 (product taken in mode order)."""
    other = mats if mats2 is None else mats2
    prod = None
    for k in range(len(mats)):
        if k == skip:
            continue
        g = np.asarray(mats[k]).T @ np.asarray(other[k])
        prod = g if prod is None else prod * g
    return prod


def top_eig(g):
    """Largest eigenvalue of a symmetric PSD matrix, clamped at 0; 0 for the
    zero matrix.  Restates tensor_ops.py:127-140 (LAPACK syevd via eigvalsh)."""
    g = np.asarray(g, dtype=float)
    if not g.any():
        return 0.0
    return max(float(np.linalg.eigvalsh(g)[-1]), 0.0)


def dense_from_model(factors, weights):
    """Full tensor of a Kruskal model through the mode-0 unfolding.
    Restates kruskal.py:112-119."""
    flat = (factors[0] * weights) @ kr_desc(factors, skip=0).T
    return fold(flat, 0, tuple(f.shape[0] for f in factors))


# ----------------------------------------------------------------------------
# operator-level building blocks (solver.py:194-274)
# ----------------------------------------------------------------------------

def mttkrp(t, factors, n):
    """M_(n) @ KR_{-n}.  Restates solver.py:243-245."""
    return unfold(t, n) @ kr_desc(factors, skip=n)


def core_term(t, factors):
    """(U_kr)^T vec(M) via the mode-0 unfolding.  Restates solver.py:215-218."""
    return np.einsum("ir,ir->r", factors[0], unfold(t, 0) @ kr_desc(factors, skip=0))


def core_term_lra(tilde_factors, tilde_weights, factors):
    """Cross-gram form of the core linear term.  Restates solver.py:221-229."""
    return gram_hadamard(factors, mats2=tilde_factors) @ tilde_weights


def mttkrp_lra(tilde_factors, tilde_weights, factors, n):
    """(U~_n * w~) @ (hadamard_{m!=n} U~_m^T U_m).  Restates solver.py:248-251."""
    cross = gram_hadamard(tilde_factors, skip=n, mats2=factors)
    return (tilde_factors[n] * tilde_weights) @ cross


def full_objective(tensors, models):
    """1/2 sum_s ||M_s - [[lam; U]]||^2 by explicit residuals.
    Restates solver.py:194-202.  ``models`` is a list of (factors, weights)."""
    acc = 0.0
    for t, (facs, lam) in zip(tensors, models):
        resid = unfold(t, 0) - (facs[0] * lam) @ kr_desc(facs, skip=0).T
        acc += 0.5 * float(np.einsum("ij,ij->", resid, resid))
    return acc


def next_t(t):
    """Momentum sequence.  Restates solver.py:265-267."""
    return 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))


def extrap_w(w_hat, lip_prev, lip_curr, delta_w):
    """Capped extrapolation weight.  Restates solver.py:270-274."""
    if lip_curr <= 0.0 or lip_prev <= 0.0:
        return 0.0
    return min(w_hat, delta_w * float(np.sqrt(lip_prev / lip_curr)))


def draw_init(shapes, ranks, counts, update_core, seed):
    """Uniform[0,1) start with the common prefix drawn once.
    Restates solver.py:277-303 (draw order: common per mode; then per block
    individual columns per mode, then weights if the core is updated)."""
    gen = np.random.default_rng(seed)
    order = len(counts)
    shared = [gen.random((shapes[0][n], counts[n])) for n in range(order)]
    out = []
    for s, shp in enumerate(shapes):
        r = ranks[s]
        facs = []
        for n in range(order):
            own = gen.random((shp[n], r - counts[n]))
            facs.append(np.hstack([shared[n], own]) if counts[n] else own)
        lam = gen.random(r) if update_core else np.ones(r)
        out.append((facs, lam))
    return out


# ----------------------------------------------------------------------------
# CP-ALS compression (cpd_als.py:52-120)
# ----------------------------------------------------------------------------

def als_fit(t, rank, tol=1e-4, max_iter=200, seed=0):
    """Unconstrained rank-`rank` CP by ALS with a tiny ridge.
    Restates cpd_als.py:52-120.  Returns dict(factors, weights, rel_err,
    history, n_iter, converged)."""
    t = np.asarray(t, dtype=float)
    if not np.isfinite(t).all():
        raise ValueError("tensor contains non-finite values")
    shape = t.shape
    for n in range(t.ndim):
        if rank > t.size // shape[n]:
            raise ValueError(
                f"rank {rank} infeasible: mode-{n} system has only "
                f"{t.size // shape[n]} rows")
    gen = np.random.default_rng(seed)
    facs = [gen.random((d, rank)) for d in shape]
    grams = [f.T @ f for f in facs]
    tnorm = float(np.linalg.norm(t))
    hist = []
    rel = 0.0 if tnorm == 0.0 else 1.0
    converged = False
    sweep = 0
    for sweep in range(1, max_iter + 1):
        for n in range(t.ndim):
            kr = kr_desc(facs, skip=n)
            mn = unfold(t, n)
            rhs = mn @ kr
            v = np.ones((rank, rank))
            for m in range(t.ndim):
                if m != n:
                    v *= grams[m]
            ridge = 1e-12 * np.trace(v) / rank
            if ridge > 0.0:
                facs[n] = np.linalg.solve(v + ridge * np.eye(rank), rhs.T).T
            else:
                facs[n] = np.zeros_like(facs[n])
            grams[n] = facs[n].T @ facs[n]
        if not all(np.isfinite(g).all() for g in grams):
            raise ValueError(f"ALS diverged to non-finite values at sweep {sweep}")
        res = float(np.linalg.norm(mn - facs[t.ndim - 1] @ kr.T))
        new_rel = res / tnorm if tnorm > 0.0 else 0.0
        hist.append(new_rel)
        stop = abs(rel - new_rel) < tol
        rel = new_rel
        if stop:
            converged = True
            break
    return dict(factors=facs, weights=np.ones(rank), rel_err=rel, history=hist,
                n_iter=sweep, converged=converged)


# ----------------------------------------------------------------------------
# the APG iteration (solver.py:311-624), restated procedurally
# ----------------------------------------------------------------------------

def _hprod(mats, skip=None):
    """Hadamard product of a list of equal-shape matrices in list order,
    starting from ones (solver.py:352-358)."""
    r = mats[0].shape[0]
    out = np.ones((r, mats[0].shape[1]))
    for m, g in enumerate(mats):
        if m != skip:
            out *= g
    return out


def _cprod(mats, skip=None):
    """Hadamard product of cross grams starting from the first kept one
    (solver.py:360-365)."""
    out = None
    for m, c in enumerate(mats):
        if m != skip:
            out = c.copy() if out is None else out * c
    return out


def solve_oracle(tensors, ranks, counts, mode="full", update_core=True,
                 max_iter=1000, tol=1e-8, delta_w=0.9999, seed=0,
                 trace_every=1, als_rank=None, als_tol=1e-4, als_max_iter=200,
                 als_seed=0, on_iteration=None):
    """Coupled nonnegative CPD by APG with restart.  Restates solver.py:546-624
    (outer loop) and the ``_Apg`` state machine solver.py:311-543.

    ``on_iteration(k)`` (optional) is called after every accepted iteration
    (k = 0 after the initial evaluation); the bench uses it to time steps.

    Returns a dict with keys factors (list of (factors, weights)), objective_history,
    rel_err_history, trace (list of (iter, obj_fun, rel_err)), n_iter, n_restarts,
    termination_reason, compression (list of (factors, weights) or None).
    """
    X = [np.asarray(t, dtype=float) for t in tensors]
    S = len(X)
    N = X[0].ndim
    if isinstance(ranks, (int, np.integer)):
        ranks = [int(ranks)] * S
    ranks = [int(r) for r in ranks]
    counts = [int(c) for c in counts]

    # -- lra stage 1: per-block ALS compression (solver.py:556-573)
    tl = None
    if mode == "lra":
        tl = []
        for s in range(S):
            fit = als_fit(X[s], als_rank if als_rank is not None else ranks[s],
                          tol=als_tol, max_iter=als_max_iter, seed=als_seed + s)
            tl.append((fit["factors"], fit["weights"]))

    # -- state (solver.py:314-348)
    start = draw_init([x.shape for x in X], ranks, counts, update_core, seed)
    U = [list(f) for f, _ in start]
    lam = [w for _, w in start]
    Up = [[f.copy() for f in U[s]] for s in range(S)]
    lamp = [w.copy() for w in lam]
    M0 = [unfold(x, 0) for x in X]
    nsq = [float(np.vdot(x, x)) for x in X]
    G = [[f.T @ f for f in U[s]] for s in range(S)]
    C = None
    tsq = None
    if tl is not None:
        C = [[tf.T @ f for tf, f in zip(tl[s][0], U[s])] for s in range(S)]
        tsq = [float(np.ones(len(w)) @ gram_hadamard(tf) @ np.ones(len(w)))
               for tf, w in tl]
    b = [None] * S
    mlast = [None] * S
    mtag = [-1] * S
    it_tag = [0]
    Lcore = [None] * S
    Lfac = [[None] * S for _ in range(N)]

    def refresh(s, n):
        # solver.py:367-371
        G[s][n] = U[s][n].T @ U[s][n]
        if tl is not None:
            C[s][n] = tl[s][0][n].T @ U[s][n]

    def core_step(w_hat):
        # solver.py:375-395
        for s in range(S):
            gall = _hprod(G[s])
            ld = top_eig(gall)
            ldp = Lcore[s] if Lcore[s] is not None else ld
            Lcore[s] = ld
            cur = lam[s]
            if ld == 0.0:
                lamp[s] = cur
                lam[s] = cur.copy()
                continue
            w = extrap_w(w_hat, ldp, ld, delta_w)
            lh = cur + w * (cur - lamp[s])
            lin = b[s] if tl is None else _cprod(C[s]).T @ tl[s][1]
            g = gall @ lh - lin
            lamp[s] = cur
            lam[s] = np.maximum(0.0, lh - g / ld)

    def mode_step(n, w_hat):
        # solver.py:397-457
        ln = counts[n]
        info = []
        for s in range(S):
            step = _hprod(G[s], skip=n) * np.outer(lam[s], lam[s])
            lu = top_eig(step)
            lup = Lfac[n][s] if Lfac[n][s] is not None else lu
            Lfac[n][s] = lu
            mt = None
            if lu > 0.0:
                if tl is None:
                    kr = kr_desc(U[s], skip=n)
                    mn = M0[s] if n == 0 else unfold(X[s], n)
                    mt = mn @ kr
                    if n == N - 1:
                        mlast[s] = mt
                        mtag[s] = it_tag[0]
                else:
                    tf, tw = tl[s]
                    mt = (tf[n] * tw) @ _cprod(C[s], skip=n)
            info.append((step, lu, lup, mt))
        lsum = sum(e[1] for e in info)
        if ln > 0:
            lsum_prev = sum(e[2] for e in info)
            wc = extrap_w(w_hat, lsum_prev, lsum, delta_w)
            cc = U[0][n][:, :ln]
            cp = Up[0][n][:, :ln]
            ch = cc + wc * (cc - cp)
            gc = np.zeros_like(ch)
        own_new = []
        for s, (step, lu, lup, mt) in enumerate(info):
            u = U[s][n]
            if lu == 0.0:
                own_new.append(u[:, ln:].copy())
                continue
            w = extrap_w(w_hat, lup, lu, delta_w)
            ih = u[:, ln:] + w * (u[:, ln:] - Up[s][n][:, ln:])
            uh = np.hstack([ch, ih]) if ln > 0 else ih
            g = uh @ step - mt * lam[s]
            if ln > 0:
                gc += g[:, :ln]
            own_new.append(np.maximum(0.0, ih - g[:, ln:] / lu))
        if ln > 0:
            cn = np.maximum(0.0, ch - gc / lsum) if lsum > 0.0 else cc.copy()
        for s in range(S):
            Up[s][n] = U[s][n]
            U[s][n] = np.hstack([cn, own_new[s]]) if ln > 0 else own_new[s]
            refresh(s, n)

    def sweep(w_hat):
        # solver.py:459-463
        if update_core:
            core_step(w_hat)
        for n in range(N):
            mode_step(n, w_hat)

    def small_resid(s):
        # solver.py:467-482
        tf, tw = tl[s]
        wts = np.concatenate([tw, -lam[s]])
        rs = [np.linalg.qr(np.hstack([tf[n], U[s][n]]), mode="r") for n in range(N)]
        core = dense_from_model(rs, wts)
        return float(np.vdot(core, core))

    def evaluate():
        # solver.py:484-534
        oi = 0.0
        oo = 0.0
        rel = 0.0
        staged = [None] * S
        for s in range(S):
            w = lam[s]
            f = U[s]
            if tl is None:
                kr0 = kr_desc(f, skip=0)
                d = M0[s] - (f[0] * w) @ kr0.T
                rsq = float(np.einsum("ij,ij->", d, d))
                oi += 0.5 * rsq
                if mtag[s] == it_tag[0]:
                    staged[s] = np.einsum("ir,ir->r", f[N - 1], mlast[s])
                else:
                    staged[s] = np.einsum("ir,ir->r", f[0], M0[s] @ kr0)
            else:
                msq = float(w @ _hprod(G[s]) @ w)
                inner = float(w @ (_cprod(C[s]).T @ tl[s][1]))
                rt = tsq[s] - 2.0 * inner + msq
                if rt < 1e-3 * tsq[s]:
                    rt = small_resid(s)
                oi += 0.5 * max(rt, 0.0)
                kr0 = kr_desc(f, skip=0)
                bo = np.einsum("ir,ir->r", f[0], M0[s] @ kr0)
                rsq = max(nsq[s] - 2.0 * w @ bo + msq, 0.0)
            if not np.isfinite(rsq):
                raise FloatingPointError(
                    f"block {s} produced a non-finite objective at iteration {it_tag[0]}")
            if tl is None:
                oo = oi
            else:
                oo += 0.5 * rsq
            nrm = np.sqrt(nsq[s])
            rel += np.sqrt(max(rsq, 0.0)) / nrm if nrm > 0.0 else 0.0
        return oi, oo, rel / S, staged

    def restore():
        # solver.py:538-543
        for s in range(S):
            lam[s] = lamp[s].copy()
            for n in range(N):
                U[s][n] = Up[s][n].copy()
                refresh(s, n)

    # -- outer loop (solver.py:576-610)
    oi, oo, rel_err, staged = evaluate()
    b[:] = staged
    obj_hist = [oi]
    rel_hist = [rel_err]
    trace = [(0, oo, rel_err)]
    if on_iteration is not None:
        on_iteration(0)
    reason = "max_iterations"
    n_done = 0
    n_restarts = 0
    t_k = 1.0
    for k in range(1, max_iter + 1):
        it_tag[0] = k
        t_new = next_t(t_k)
        w_hat = (t_k - 1.0) / t_new
        t_k = t_new
        sweep(w_hat)
        oi, oo, new_rel, staged = evaluate()
        if oi >= obj_hist[-1]:
            n_restarts += 1
            restore()
            sweep(0.0)
            oi, oo, new_rel, staged = evaluate()
        b[:] = staged
        obj_hist.append(oi)
        rel_hist.append(new_rel)
        n_done = k
        last = abs(new_rel - rel_err) < tol or k == max_iter
        if k % trace_every == 0 or last:
            trace.append((k, oo, new_rel))
        if on_iteration is not None:
            on_iteration(k)
        if abs(new_rel - rel_err) < tol:
            reason = "tolerance"
            break
        rel_err = new_rel

    return dict(
        factors=[(U[s], lam[s]) for s in range(S)],
        objective_history=obj_hist,
        rel_err_history=rel_hist,
        trace=trace,
        n_iter=n_done,
        n_restarts=n_restarts,
        termination_reason=reason,
        compression=tl,
    )
