"""c5 pipelined iteration time vs the SMs left to the sweep (pipeline_reserve)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2302_05119_b200 as P  # noqa: E402
from paper_2302_05119_b200.solver import PreparedSolve  # noqa: E402
from paper_2302_05119_b200.synth import generate_config_device  # noqa: E402

dev, spec = generate_config_device("c5")
prob = P.CoupledProblem(dev, spec.rank, list(spec.coupled), mode=spec.mode)
for res in [int(x) for x in (sys.argv[1:] or ["4", "8", "12", "16", "22", "28"])]:
    run = PreparedSolve(prob, P.SolverOptions(max_iter=60, tol=float(np.nextafter(0, 1)),
                                              precision="fp32", pipeline_reserve=res))
    with torch.cuda.stream(run.stream):
        run.engine.run(5)
        run.engine.step_async()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(run.stream):
        e0.record(run.stream)
        for _ in range(30):
            run.engine.step_async()
        e1.record(run.stream)
    torch.cuda.synchronize()
    print(f"reserve {res:3d}: {e0.elapsed_time(e1) / 30:.3f} ms/iteration", flush=True)
    run.close()
