"""Flatten solver/ALS results into .npz fixtures and back (no pickle)."""

import numpy as np


def pack_models(prefix, models, out):
    """models: list of (factors list, weights)."""
    out[f"{prefix}/S"] = np.array(len(models))
    for s, (facs, w) in enumerate(models):
        out[f"{prefix}/{s}/N"] = np.array(len(facs))
        out[f"{prefix}/{s}/w"] = np.asarray(w, dtype=float)
        for n, f in enumerate(facs):
            out[f"{prefix}/{s}/f{n}"] = np.asarray(f, dtype=float)


def unpack_models(prefix, z):
    S = int(z[f"{prefix}/S"])
    models = []
    for s in range(S):
        N = int(z[f"{prefix}/{s}/N"])
        facs = [z[f"{prefix}/{s}/f{n}"] for n in range(N)]
        models.append((facs, z[f"{prefix}/{s}/w"]))
    return models


def pack_solve(res, out):
    """res: dict with the oracle's solve_oracle keys."""
    pack_models("factors", res["factors"], out)
    out["objective_history"] = np.asarray(res["objective_history"], dtype=float)
    out["rel_err_history"] = np.asarray(res["rel_err_history"], dtype=float)
    out["trace"] = np.asarray([[i, o, r] for i, o, r in res["trace"]], dtype=float)
    out["n_iter"] = np.array(res["n_iter"])
    out["n_restarts"] = np.array(res["n_restarts"])
    out["termination_reason"] = np.array(res["termination_reason"])
    if res.get("compression") is not None:
        pack_models("compression", res["compression"], out)


def unpack_solve(z):
    res = dict(
        factors=unpack_models("factors", z),
        objective_history=list(z["objective_history"]),
        rel_err_history=list(z["rel_err_history"]),
        trace=[(int(a), float(b), float(c)) for a, b, c in z["trace"]],
        n_iter=int(z["n_iter"]),
        n_restarts=int(z["n_restarts"]),
        termination_reason=str(z["termination_reason"]),
        compression=unpack_models("compression", z) if "compression/S" in z else None,
    )
    return res


def tensor_fingerprint(t):
    """Cheap, layout-independent fingerprint of a tensor's logical values."""
    t = np.asarray(t, dtype=float)
    flat = t.reshape(-1, order="F")
    idx = np.linspace(0, flat.size - 1, 16).astype(np.int64)
    return np.concatenate([[flat.sum(), float(np.vdot(flat, flat))], flat[idx]])
