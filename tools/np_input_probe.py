import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _device as D
from paper_2302_05119_b200.synth import generate_config_device
dev, spec = generate_config_device("c5", blocks=list(range(8)))
host = [t.cpu().numpy().copy(order="C") for t in dev]   # numpy's default layout
del dev
torch.cuda.synchronize()
for rep in range(2):
    tic = time.perf_counter()
    for h in host:
        flat, dims = D.tensor_to_dev(h, "fp32")
    torch.cuda.synchronize()
    print(f"tensor_to_dev of 8 C-ordered 400^3 fp32 numpy blocks: {time.perf_counter() - tic:.3f} s")
tic = time.perf_counter()
res = P.solve(P.CoupledProblem(host, spec.rank, list(spec.coupled), mode="lra"),
              P.SolverOptions(max_iter=20, tol=1e-300, seed=0, precision="fp32"))
print(f"solve() of 8 blocks from numpy, 20 iterations: {time.perf_counter() - tic:.3f} s")
