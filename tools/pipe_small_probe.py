"""Pipelined vs serial lra iteration on the small lra configs (c4, c3): whole
run (early iterations and the late ones on the QR route)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2302_05119_b200 as P  # noqa: E402
from paper_2302_05119_b200.synth import generate_config_device  # noqa: E402

for name in ("c4", "c3"):
    dev, spec = generate_config_device(name)
    for pipe, res in (("off", 0), ("on", 8), ("on", 16)):
        best = None
        for rep in range(2):
            prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
            r = P.solve(prob, P.SolverOptions(max_iter=spec.max_iter, tol=float(np.nextafter(0, 1)), seed=0,
                                              precision="fp32", pipeline=pipe, pipeline_reserve=res))
            t = np.array([row.elapsed_s for row in r.trace])
            d = np.diff(t) * 1e3
            cur = (r.n_iter / (t[-1] - t[0]), np.median(d[5:60]), np.median(d[-60:-5]))
            best = cur if best is None or cur[0] > best[0] else best
        print(f"{name} pipeline {pipe} reserve {res:2d}: {best[0]:7.1f} it/s whole run; early {best[1]:.3f} ms, "
              f"late {best[2]:.3f} ms", flush=True)
