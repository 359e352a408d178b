"""Diagnostic: per-iteration trace of the GPU solve vs the reference fixture."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import paper_2302_05119_b200 as P
from paper_2302_05119_b200.configs import generate_config
from store import unpack_solve
from cases import TINY_TOL
name = sys.argv[1]; iters = int(sys.argv[2])
want = unpack_solve(np.load(f"tests/golden/config_{name}.npz"))
tensors, spec = generate_config(name)
t64 = [np.asarray(t, dtype=float) for t in tensors]
runs = {}
for prec, obj in [("fp64", "explicit"), ("fp64", "expansion"), ("fp32", "explicit")]:
    res = P.solve(P.CoupledProblem(t64, spec.rank, list(spec.coupled), mode=spec.mode),
                  P.SolverOptions(max_iter=iters, tol=TINY_TOL, seed=0, precision=prec, objective=obj))
    runs[(prec, obj)] = res
    print(prec, obj, "restarts", res.n_restarts)
ro = np.asarray(want["objective_history"]); rr = np.asarray(want["rel_err_history"])
for k in range(min(iters + 1, len(ro))):
    line = f"{k:4d} ref obj {ro[k]:.16e}"
    for key, res in runs.items():
        o = res.objective_history[k]; r = res.rel_err_history[k]
        line += f" | {key[0]}/{key[1][:3]} dobj {(o-ro[k])/ro[k]:+.2e} drel {(r-rr[k])/rr[k]:+.2e}"
    print(line)
