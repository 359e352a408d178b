"""Per-launch profile (events after every launch) of APG iterations after
`skip` iterations, device-generated inputs.

    python tools/profile_late.py [config] [skip] [iters]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05119_b200 as P  # noqa: E402
from paper_2302_05119_b200 import _lib as L  # noqa: E402
from paper_2302_05119_b200.solver import PreparedSolve  # noqa: E402
from paper_2302_05119_b200.synth import generate_config_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 150
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev, spec = generate_config_device(name)
prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
run = PreparedSolve(prob, P.SolverOptions(max_iter=skip + iters + 8, tol=float(np.nextafter(0, 1)),
                                          precision=spec.dtype))
with torch.cuda.stream(run.stream):
    summ = run.engine.run(skip)
    print(f"after {summ.n_iter} iterations, {summ.n_restarts} restarts")
    L.check(L.lib.cb_solver_profile(run.engine.h, 1, None, 0))
    for _ in range(iters):
        run.engine.step_async()
buf = ctypes.create_string_buffer(1 << 16)
L.check(L.lib.cb_solver_profile(run.engine.h, 0, buf, len(buf)))
rows = []
for line in buf.value.decode().strip().splitlines():
    lab, n, ms = line.split()
    if not lab.startswith(("phase", "kernel:")):
        rows.append((lab, int(n), float(ms)))
tot = sum(r[2] for r in rows)
print(f"{name}: {iters} iterations after {skip}: {1e3 * tot / iters:.1f} us/iteration")
for lab, n, ms in sorted(rows, key=lambda r: -r[2]):
    print(f"  {lab:20s} {n:5d} launches  {1e3 * ms / iters:9.2f} us/it  {1e3 * ms / n:9.2f} us/launch  "
          f"{100 * ms / tot:5.1f}%")
print("restarts now", run.engine.summary().n_restarts)
run.close()
