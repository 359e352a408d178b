"""Diagnostic: GPU solve of a BASELINE config in several precision modes vs the
reference fixture (prints per-mode divergence)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import paper_2302_05119_b200 as P
from paper_2302_05119_b200.configs import generate_config
from store import unpack_solve
from cases import TINY_TOL

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"config_{name}.npz"))
want = unpack_solve(z)
tensors, spec = generate_config(name)
t64 = [np.asarray(t, dtype=float) for t in tensors]
print(f"{name}: reference n_iter={want['n_iter']} restarts={want['n_restarts']} rel={want['rel_err_history'][-1]:.10f}")
modes = [(p, o, c) for p, o, c in [("fp64", "explicit", "auto"), ("fp32", "expansion", "fp64"), ("fp32", "explicit", "fp64"), ("fp32", "expansion", "fp32"), ("fp32", "explicit", "fp32")]]
for prec, obj, comp in modes:
    if name == "c1" and prec == "fp32":
        continue
    for iters in ([spec.max_iter] if len(sys.argv) < 3 else [int(sys.argv[2])]):
        tic = time.perf_counter()
        res = P.solve(P.CoupledProblem(t64, spec.rank, list(spec.coupled), mode=spec.mode),
                      P.SolverOptions(max_iter=iters, tol=TINY_TOL, seed=0, precision=prec, objective=obj, compute=comp))
        dt = time.perf_counter() - tic
        n = min(res.n_iter, want["n_iter"]) + 1
        h = np.asarray(res.rel_err_history[:n]); hw = np.asarray(want["rel_err_history"][:n])
        herr = np.max(np.abs(h - hw) / hw)
        msg = f"  {prec}/{obj}/{comp} max_iter={iters}: n_iter={res.n_iter} restarts={res.n_restarts} rel={res.rel_err_history[-1]:.10f} hist_err={herr:.2e} ({dt:.2f}s)"
        if iters == spec.max_iter:
            fe = 0.0
            for blk, (wf, ww) in zip(res.factors.blocks, want["factors"]):
                fe = max(fe, np.max(np.abs(blk.weights - ww)) / np.max(np.abs(ww)))
                for a, b in zip(blk.factors, wf):
                    fe = max(fe, np.max(np.abs(a - b)) / np.max(np.abs(b)))
            msg += f" factor_err={fe:.2e}"
        print(msg, flush=True)
