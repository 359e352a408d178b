"""Timeline of one graph-launched APG iteration from in-kernel timestamps.

    python tools/timeline.py [config] [iters] [flush(0/1)]

Per kernel slot: start / end (us, relative to the first kernel start of the
iteration) averaged over `iters` iterations, plus the CUDA-event time of the
step.  Slots of kernels that did not run (restart branch) are omitted.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _lib as L
from paper_2302_05119_b200.configs import CONFIGS, generate_config
from paper_2302_05119_b200.synth import generate_config_device
from paper_2302_05119_b200.solver import PreparedSolve

NAMES = {0: "sweep_begin", 1: "contract0", 2: "contract1", 3: "slab", 4: "fiber",
         5: "mode_update0", 6: "mode_update1", 7: "mode_update2", 8: "finalize0",
         9: "finalize1", 10: "finalize2", 11: "step1", 12: "step2", 14: "control",
         15: "common0", 16: "common1", 17: "common2", 18: "qr", 20: "restore", 21: "trace",
         22: "trace_prep"}
NSLOT = 24

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
flush_on = int(sys.argv[3]) if len(sys.argv) > 3 else 1
spec = CONFIGS[name]
nblk = int(os.environ.get("TL_BLOCKS", "0"))
tensors, _ = generate_config_device(name, blocks=range(nblk) if nblk else None)
prob = P.CoupledProblem(tensors, spec.rank, list(spec.coupled), mode=spec.mode)
run = PreparedSolve(prob, P.SolverOptions(max_iter=iters + 20, tol=float(np.nextafter(0, 1)),
                                          precision=spec.dtype))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
buf = (ctypes.c_ulonglong * (2 * NSLOT))()
h = run.engine.h
acc = {}
cnt = {}
ev = []
with torch.cuda.stream(run.stream):
    L.check(L.lib.cb_solver_timeline(h, 1, None, 0))
    run.engine.run(3)                    # warm-up + capture with timestamps
    for _ in range(iters):
        if flush_on:
            flush.fill_(1.0)
        L.check(L.lib.cb_solver_timeline(h, 2, None, 0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(run.stream)
        run.engine.step_async()
        e1.record(run.stream)
        L.check(L.lib.cb_solver_timeline(h, 0, buf, 2 * NSLOT))
        ev.append(e0.elapsed_time(e1) * 1e3)
        starts = [buf[2 * k] for k in range(NSLOT) if buf[2 * k] != 2 ** 64 - 1]
        t0 = min(starts)
        for k in range(NSLOT):
            b, e = buf[2 * k], buf[2 * k + 1]
            if b == 2 ** 64 - 1 or e == 0:
                continue
            a = acc.setdefault(k, [0.0, 0.0])
            a[0] += (b - t0) / 1e3
            a[1] += (e - t0) / 1e3
            cnt[k] = cnt.get(k, 0) + 1
print(f"{name}: step (CUDA events) {np.mean(ev):.1f} us  (flush={flush_on}, {iters} iterations)")
rows = sorted(((acc[k][0] / cnt[k], acc[k][1] / cnt[k], k) for k in acc))
for b, e, k in rows:
    print(f"  {NAMES.get(k, k):14s} start {b:8.1f}  end {e:8.1f}  dur {e - b:7.1f} us")
run.close()
