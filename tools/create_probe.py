"""Time cb_solver_create for the c5 problem twice (lazy module loading shows
as a first-call cost)."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2302_05119_b200 as P  # noqa: E402
from paper_2302_05119_b200 import solver as S  # noqa: E402
from paper_2302_05119_b200.synth import generate_config_device  # noqa: E402

dev, spec = generate_config_device("c5")
prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
orig = S._Engine.__init__


def timed(self, desc, stream):
    torch.cuda.synchronize()
    t = time.perf_counter()
    orig(self, desc, stream)
    torch.cuda.synchronize()
    print(f"  cb_solver_create {time.perf_counter() - t:.3f} s", flush=True)


S._Engine.__init__ = timed
for rep in range(2):
    t = time.perf_counter()
    run = S.PreparedSolve(prob, P.SolverOptions(max_iter=5, tol=float(np.nextafter(0, 1)),
                                                 precision="fp32"))
    torch.cuda.synchronize()
    print(f"PreparedSolve {rep}: {time.perf_counter() - t:.3f} s", flush=True)
    run.close()
