"""ALS passes on the packed byte planes (csrc/xoz.cu) against the fp64-storage
ALS on the same fp32 values: per-sweep history and factor differences on a few
shapes, then timing on c5-shaped blocks.
    python tools/oz_probe.py [S_c5] [sweeps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2302_05119_b200 as P
from paper_2302_05119_b200 import _lib as L
from paper_2302_05119_b200.cpd_als import als_compress_blocks

st = L.c_vp(torch.cuda.current_stream().cuda_stream)


def model_block(rng, dims, rank, noise=0.05):
    f = [rng.random((d, rank)) for d in dims]
    x = np.einsum("ir,jr,kr->ijk", *f)
    x = np.maximum(x + noise * x.std() * rng.standard_normal(x.shape), 0.0)
    return torch.from_numpy(np.ascontiguousarray(x.transpose(2, 1, 0)).reshape(-1).astype(np.float32)).cuda()


def compare(shapes, sweeps):
    rng = np.random.default_rng(5)
    dev32 = [model_block(rng, d, r) for d, r in shapes]
    dev64 = [x.double() for x in dev32]
    dims = [d for d, _ in shapes]
    ranks = [r for _, r in shapes]
    out = {}
    for code, data in ((L.CB_F32, dev32), (L.CB_F64, dev64)):
        h = als_compress_blocks(data, dims, ranks, 1e-30, sweeps, list(range(len(shapes))), code, st, 0,
                                total_blocks=len(shapes))
        out[code] = [h.block(s) for s in range(len(shapes))]
        h.close()
    for s in range(len(shapes)):
        fa, _, ha, na, _ = out[L.CB_F32][s]
        fb, _, hb, nb, _ = out[L.CB_F64][s]
        dh = np.abs(np.asarray(ha) - np.asarray(hb)).max()
        df = max(np.abs(a - b).max() / np.abs(b).max() for a, b in zip(fa, fb))
        print(f"  {shapes[s]}: sweeps {na}/{nb}  max |dhist| {dh:.3e}  max rel dfactor {df:.3e}  rel {ha[-1]:.6e}")


print("one sweep:")
compare([((64, 40, 50), 20), ((96, 36, 30), 24), ((70, 45, 33), 40), ((33, 70, 45), 17)], 1)
print("12 sweeps:")
compare([((64, 40, 50), 20), ((96, 36, 30), 24), ((70, 45, 33), 40), ((33, 70, 45), 17), ((128, 128, 96), 40)], 12)

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 6
I, R = 400, 40
g = torch.Generator(device="cuda").manual_seed(0)
dev = [torch.rand(I * I * I, device="cuda", generator=g) for _ in range(S)]
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    res = als_compress_blocks(dev, [(I, I, I)] * S, [R] * S, 1e-30, mi, list(range(S)), L.CB_F32, st, 0,
                              total_blocks=S)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"ALS {S} c5 blocks x {mi} sweeps: {t1 - t0:.3f} s ({(t1 - t0) / mi * 1e3:.1f} ms per sweep incl. setup)")
    facs, rel, hist, nit, conv = res.block(0)
    print(f"  block 0: rel_err {rel:.12e} after {nit} sweeps")
    res.close()
