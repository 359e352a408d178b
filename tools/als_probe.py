"""Batched device ALS (lra compression) on S c5-shaped blocks (device-generated
uniform data, 400^3 fp32, R~ = 40): wall time and sweeps.
    python tools/als_probe.py [S] [max_iter]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _lib as L
from paper_2302_05119_b200.cpd_als import als_compress_blocks
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 10
code = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # compute code (0: fp64-grade passes)
I, R = 400, 40
g = torch.Generator(device="cuda").manual_seed(0)
dev = [torch.rand(I * I * I, device="cuda", generator=g) for _ in range(S)]
dims = [(I, I, I)] * S
st = torch.cuda.current_stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
res = als_compress_blocks(dev, dims, [R] * S, 1e-30, mi, list(range(S)), L.CB_F32,
                          L.c_vp(st.cuda_stream), code, total_blocks=S)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"code {code}: ALS {S} blocks x {mi} sweeps: {t1 - t0:.3f} s  ({(t1 - t0) / mi * 1e3:.1f} ms per sweep, "
      f"{2 * S * I**3 * 4 / ((t1 - t0) / mi) / 1e9:.0f} GB/s for 2 passes per sweep)")
facs, rel, hist, nit, conv = res.block(0)
print(f"  block 0: rel_err {rel:.12e} after {nit} sweeps; history tail {hist[-3:]}")

