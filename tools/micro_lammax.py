"""Micro-benchmark: batched lambda_max kernel (cb_spectral_norm_batched)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2302_05119_b200 import _lib as L
rng = np.random.default_rng(0)
for R, batch in [(5, 2), (10, 10), (16, 10), (20, 8), (30, 32), (40, 64), (64, 8)]:
    gs = []
    for _ in range(batch):
        a = rng.random((R + 3, R))
        g = a.T @ a
        gs.append(g * np.outer(rng.uniform(0.5, 1.5, R), rng.uniform(0.5, 1.5, R)) if False else g)
    gs = np.stack(gs)
    dg = torch.from_numpy(gs).cuda()
    out = torch.empty(batch, dtype=torch.float64, device="cuda")
    st = L.c_vp(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        L.check(L.lib.cb_spectral_norm_batched(dg.data_ptr(), R, batch, out.data_ptr(), st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        L.check(L.lib.cb_spectral_norm_batched(dg.data_ptr(), R, batch, out.data_ptr(), st))
    e1.record()
    torch.cuda.synchronize()
    want = np.array([np.linalg.eigvalsh(g)[-1] for g in gs])
    err = np.max(np.abs(out.cpu().numpy() - want) / want)
    print(f"R={R:3d} batch={batch:3d}: {e0.elapsed_time(e1)/20*1e3:8.2f} us/launch  max rel err {err:.2e}")
