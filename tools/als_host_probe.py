"""Host-side cost of the batched device ALS on 64 c5-shaped blocks: handle
creation (allocations, plane packing, stats, initial grams), the sweeps,
result download, destruction.   python tools/als_host_probe.py [S] [sweeps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _lib as L
from paper_2302_05119_b200.cpd_als import AlsHandle

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 36
dims = tuple(int(x) for x in sys.argv[3].split("x")) if len(sys.argv) > 3 else (400, 400, 400)
R = int(sys.argv[4]) if len(sys.argv) > 4 else 40
g = torch.Generator(device="cuda").manual_seed(0)
dev = [torch.rand(dims[0] * dims[1] * dims[2], device="cuda", generator=g) for _ in range(S)]
st = L.c_vp(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    h = AlsHandle(dev, [dims] * S, [R] * S, L.CB_F32, 1e-30, mi, list(range(S)), st, 0, S)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h.run()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ptrs = [h.factor_device_ptr(s, n) for s in range(S) for n in range(3)]
    t4 = time.perf_counter()
    h.close()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"rep {rep}: create (host) {t1 - t0:.3f} s, create drain {t2 - t1:.3f} s, run {t3 - t2:.3f} s "
          f"({(t3 - t2) / mi * 1e3:.2f} ms/sweep), ptrs {t4 - t3:.4f} s, destroy {t5 - t4:.3f} s", flush=True)
