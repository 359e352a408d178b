"""Per-launch profile of APG iterations (CUDA events after every launch).

    python tools/profile_iter.py [config] [iters] [flush(0/1)]
"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _lib as L
from paper_2302_05119_b200.configs import CONFIGS, generate_config
from paper_2302_05119_b200.solver import PreparedSolve

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
flush_on = int(sys.argv[3]) if len(sys.argv) > 3 else 1
spec = CONFIGS[name]
nblk = int(os.environ.get("TL_BLOCKS", "0"))
tensors, _ = generate_config(name, blocks=range(nblk) if nblk else None)
prob = P.CoupledProblem([np.asarray(t, dtype=float) for t in tensors], spec.rank, list(spec.coupled), mode=spec.mode)
run = PreparedSolve(prob, P.SolverOptions(max_iter=iters + 12, tol=float(np.nextafter(0, 1)), precision=spec.dtype))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
with torch.cuda.stream(run.stream):
    run.engine.run(5)
    L.check(L.lib.cb_solver_profile(run.engine.h, 1, None, 0))
    for _ in range(iters):
        if flush_on:
            flush.fill_(1.0)
        run.engine.step_async()
buf = ctypes.create_string_buffer(1 << 16)
L.check(L.lib.cb_solver_profile(run.engine.h, 0, buf, len(buf)))
rows, phases = [], []
for line in buf.value.decode().strip().splitlines():
    lab, n, ms = line.split()
    if lab.startswith("kernel:"):
        print(f"  in-kernel time {lab[7:]}: {1e3*float(ms)/int(n):8.2f} us/launch over {n} launches")
        continue
    (phases if lab.startswith("phase") else rows).append((lab, int(n), float(ms)))
tot = sum(r[2] for r in rows)
print(f"{name}: {iters} iterations, flush={flush_on}: {1e3*tot/iters:.1f} us/iteration (excl. flush)")
for lab, n, ms in sorted(rows, key=lambda r: -r[2]):
    print(f"  {lab:20s} {n:5d} launches  {1e3*ms/iters:8.2f} us/it  {1e3*ms/n:8.2f} us/launch  {100*ms/tot:5.1f}%")
for lab, _, ms in phases:
    print(f"  {lab} (block 0, summed over launches): {1e3*ms/iters:8.2f} us/it")
run.close()
ph = {lab: ms for lab, _, ms in phases}
for k in range(32):
    a, b = ph.get(f"phase{k:02d}"), ph.get(f"phase{k+32:02d}")
    if a and b:
        print(f"  phase{k:02d}: effective SM clock {b / a / 1e3:.0f} MHz")
