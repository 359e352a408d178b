"""Diagnostic: explicit residual of the fiber pass vs the generic residual kernel."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05119_b200 as P
from oracle import concpd_oracle as O

for dims, R, S in [((50, 50, 50), 5, 2), ((100, 100, 100), 10, 10), ((30, 20, 40), 10, 2), ((30, 20, 40), 7, 2), ((30, 20, 40), 12, 1), ((30, 20, 40), 16, 1), ((30,20,40), 20, 1)]:
    rng = np.random.default_rng(1)
    tensors = [rng.random(dims) for _ in range(S)]
    for prec in ("fp64", "fp32"):
        for obj in ("explicit", "expansion"):
            prob = P.CoupledProblem(tensors, R, [0, 0, 0])
            res = P.solve(prob, P.SolverOptions(max_iter=0, seed=3, precision=prec, objective=obj))
            init = P.init_factors(prob, 3)
            want = O.full_objective(tensors, [(b.factors, b.weights) for b in init.blocks])
            print(dims, R, S, prec, obj, f"{res.objective_history[0]:.15e}", f"{want:.15e}", f"{abs(res.objective_history[0]-want)/want:.2e}", flush=True)
