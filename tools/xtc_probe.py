"""Tensor-core trace pass on S device-resident 400^3 fp32 blocks, R = 40
(c5 block shape): per-call time through cb_core_linear_term_tc (plan setup +
max|X| pass + prep + trace).  Kernel durations come from ncu.

    python tools/xtc_probe.py [S] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2302_05119_b200 import _lib as L

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
I, R = 400, 40
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.rand(I * I * I, device="cuda", generator=g) for _ in range(S)]
fs = [torch.rand(I, R, device="cuda", dtype=torch.float64, generator=g) for _ in range(3 * S)]
out = torch.zeros(S, 64, device="cuda", dtype=torch.float64)
dims = [I] * (3 * S)
st = torch.cuda.current_stream().cuda_stream
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.check(L.lib.cb_core_linear_term_tc(S, L.ptr_array([x.data_ptr() for x in xs]),
                                         L.i64_array(dims), L.ptr_array([f.data_ptr() for f in fs]),
                                         L.int_array([R] * S), out.data_ptr(), st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gb = S * I ** 3 * 4 / 1e9
    print(f"call {i}: {ms:.3f} ms  ({gb:.2f} GB streamed twice: max|X| + trace)", flush=True)
# fp64 check of block 0 against torch
x0 = xs[0].double().reshape(I, I * I)          # [i0 fastest]: view as (i2,i1,i0)? see below
X = xs[0].double().reshape(I, I, I)            # X[i2, i1, i0] in C order == first-index-fastest
A0, A1, A2 = fs[0], fs[1], fs[2]
want = torch.einsum("cba,ar,br,cr->r", X, A0, A1, A2)
rel = ((out[0, :R] - want).abs() / want.abs()).max().item()
print(f"block 0 max rel err vs fp64 einsum: {rel:.3e}")
