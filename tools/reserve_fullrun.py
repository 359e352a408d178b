"""c5 whole-run iterations/s (early iterations + the late ones on the QR
route) vs the SMs left to the sweep (pipeline_reserve)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2302_05119_b200 as P  # noqa: E402
from paper_2302_05119_b200.synth import generate_config_device  # noqa: E402

dev, spec = generate_config_device("c5")
for res in [int(x) for x in (sys.argv[1:] or ["40", "48", "56", "64"])]:
    prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
    r = P.solve(prob, P.SolverOptions(max_iter=spec.max_iter, tol=float(np.nextafter(0, 1)), seed=0,
                                      precision="fp32", pipeline_reserve=res))
    t = np.array([row.elapsed_s for row in r.trace])
    d = np.diff(t) * 1e3
    print(f"reserve {res:3d}: {r.n_iter / (t[-1] - t[0]):7.1f} it/s whole run; early {np.median(d[5:60]):.3f} ms, "
          f"late {np.median(d[150:195]):.3f} ms", flush=True)
