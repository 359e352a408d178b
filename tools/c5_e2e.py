"""c5 end-to-end breakdown: host generation, solve() (upload + ALS compression
+ iterations), per phase.   python tools/c5_e2e.py [config] [iters]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200.configs import CONFIGS, generate_config
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = CONFIGS[name]
t0 = time.perf_counter()
tensors, _ = generate_config(name)
t1 = time.perf_counter()
print(f"{name}: host generation {t1 - t0:.1f} s", flush=True)
prob = P.CoupledProblem(tensors, spec.rank, list(spec.coupled), mode=spec.mode)
opts = P.SolverOptions(max_iter=iters, tol=float(np.nextafter(0, 1)), precision=spec.dtype)
torch.cuda.synchronize()
t2 = time.perf_counter()
res = P.solve(prob, opts)
t3 = time.perf_counter()
print(f"solve() {t3 - t2:.2f} s: compress {res.compress_seconds:.2f} s, iterations {res.solve_seconds:.2f} s "
      f"({res.n_iter} it, {res.n_iter / max(res.solve_seconds, 1e-9):.1f} it/s), other {t3 - t2 - res.compress_seconds - res.solve_seconds:.2f} s")
comp = res.compression
if comp:
    its = [getattr(c, "n_iter", None) for c in comp][:4]
    print("ALS sweeps (first blocks):", its)
