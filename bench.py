"""Benchmark: APG iterations/s of the CoNCPD-APG / lraCoNCPD-APG hot path on B200.

Default workload: BASELINE.json configs[4] ("c5"), the largest config that
fits one GPU: S=64 blocks 400^3 fp32 (16.4 GB), R=40, L_n=(10,10,10), 20 dB
noise, lraCoNCPD-APG (per-block ALS compression, then the APG iteration on the
compressed factors plus the original-tensor trace pass), seeded synthetic
inputs generated on the device.  One step = one APG
iteration over all blocks (core update, three mode updates with common-column
aggregation, compressed objective, restart rule, trace pass, stop rule).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1..c5]

Prints ONE JSON line (rank 0).  ``--gpus N`` without a torchrun environment
re-launches itself under ``torch.distributed.run`` with N ranks (one per GPU);
the config's S blocks are split over the ranks (strong scaling, NCCL
all-reduce of the coupling terms inside the iteration graph).

Timed region: exactly K steps bracketed by CUDA events on the solve stream,
after W warm-up steps plus one priming step, so every trace pass of the K
iterations runs inside the window in the pipelined lra iteration.  c5's 16 GB
exceeds L2 (126 MB) by 130x; configs below 2x L2 flush L2 with a 256 MiB write
before each step, outside the events.

``--impl reference`` times the reference algorithm on the host cores (the
oracle port, pinned to the real reference's outputs; the reference is pure
Python with no GPU path), on a bounded sample: c5 runs 1 of its 64 blocks and
extrapolates linearly in S.  It never imports the product
package or its native library.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
TINY_TOL = float(np.nextafter(0.0, 1.0))
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--cpu-iters", type=int, default=3, help="cpu_baseline APG iterations")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_configs():
    """configs.py by path: numpy only, no product package import (so the
    reference arm never maps the native library)."""
    path = os.path.join(ROOT, "paper_2302_05119_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("_bench_configs", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_bench_configs"] = mod
    spec.loader.exec_module(mod)
    return mod


def config_dict(spec, world):
    """The workload description, identical in both arms."""
    big = spec.tensor_bytes >= 2 * L2_BYTES
    return {"workload": spec.description, "name": spec.name, "n_blocks": spec.n_blocks,
            "dims": list(spec.dims), "rank": spec.rank, "coupled": list(spec.coupled),
            "mode": spec.mode, "storage": spec.dtype,
            "l2": ("inputs larger than L2 (no flush)" if big else
                   "flushed before every timed step (256 MiB write, outside the events)"),
            "parallelism": f"dp{world} over blocks" if world > 1 else "single GPU"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([int(i.get("num_threads", 1)) for i in info] or [os.cpu_count() or 1])
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU leg: the reference algorithm (oracle port) on a bounded sample
# ---------------------------------------------------------------------------

def cpu_sample(cfg, spec, iters, warmup):
    """Time the reference algorithm on the host cores (numpy/OpenBLAS, all
    threads): APG iterations/s of the whole config, ALS seconds per sweep and
    the fp64 MTTKRP GB/s of `factor_linear_term` (solver.py:243-245).  c5 runs
    one block and scales linearly in S; the others run every block.  The
    compression is bounded to 2 ALS sweeps (the per-iteration cost does not
    depend on how well the compression converged)."""
    sys.path.insert(0, ROOT)
    from oracle import concpd_oracle as O
    blocks = [0] if spec.name == "c5" else list(range(spec.n_blocks))
    scale = spec.n_blocks / len(blocks)
    tensors, _ = cfg.generate_config(spec.name, blocks=blocks)
    t64 = [np.asarray(t, dtype=np.float64) for t in tensors]
    out = {"blocks_sampled": len(blocks), "scale": scale, "cores": host_threads()}
    # MTTKRP of every mode on the first sampled block (fp64, with the
    # reference's unfolding copy)
    rng = np.random.default_rng(0)
    facs = [rng.random((d, spec.rank)) for d in spec.dims]
    gbs = []
    for n in range(3):
        tic = time.perf_counter()
        O.mttkrp(t64[0], facs, n)
        gbs.append(t64[0].size * 8 / (time.perf_counter() - tic) / 1e9)
    out["mttkrp_gbs"] = gbs
    if spec.mode == "lra":
        tic = time.perf_counter()
        fit = O.als_fit(t64[0], spec.rank, max_iter=2, seed=0)
        out["als_seconds_per_sweep_block"] = (time.perf_counter() - tic) / fit["n_iter"]
    marks = {}

    def mark(k):
        marks[k] = time.perf_counter()

    O.solve_oracle(t64, spec.rank, list(spec.coupled), mode=spec.mode,
                   max_iter=warmup + iters, tol=TINY_TOL, seed=0, als_max_iter=2,
                   on_iteration=mark)
    k0, k1 = warmup, max(marks)
    per_iter = (marks[k1] - marks[k0]) / max(k1 - k0, 1)
    out["iters_timed"] = k1 - k0
    out["seconds_per_iteration"] = per_iter * scale
    out["it_per_s"] = 1.0 / (per_iter * scale)
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = load_configs()
    spec = cfg.CONFIGS[args.config]
    c = cpu_sample(cfg, spec, args.steps, args.warmup)
    rate = c["it_per_s"]
    extrap = c["scale"] > 1
    sample = (f"{c['iters_timed']} APG iterations of {c['blocks_sampled']} of {spec.n_blocks} blocks"
              f"{', extrapolated linearly in S (BASELINE.md 2)' if extrap else ''}; fp64 "
              "numpy/OpenBLAS restatement of the reference (oracle port)")
    line = {
        "impl": "reference", "metric": "APG iterations/s", "value": rate, "unit": "it/s",
        "n_gpus": args.gpus, "steps": c["iters_timed"], "warmup": args.warmup,
        "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp64", "data": "synthetic (seeded, SURVEY 8d)",
        "config": config_dict(spec, world),
        "cpu_baseline": {"value": rate, "unit": "it/s", "cores": c["cores"], "kind": "port",
                         "sample": sample, "extrapolated": extrap,
                         "mttkrp_gbs": c["mttkrp_gbs"],
                         "als_seconds_per_sweep_block": c.get("als_seconds_per_sweep_block")},
        "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def relaunch(args):
    """--gpus N without a torchrun environment: one process per GPU."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port)] + [os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    import paper_2302_05119_b200 as P
    from paper_2302_05119_b200 import _lib as L
    from paper_2302_05119_b200.configs import CONFIGS
    from paper_2302_05119_b200.solver import PreparedShardedSolve, PreparedSolve, shard_ranges
    from paper_2302_05119_b200.synth import generate_config_device

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    spec = CONFIGS[args.config]
    prec = spec.dtype
    b0, b1 = shard_ranges(spec.n_blocks, world)[rank]
    # ---- inputs: this rank's blocks generated on the device -------------
    torch.cuda.synchronize()
    tic = time.perf_counter()
    local_dev, _ = generate_config_device(spec.name, blocks=list(range(b0, b1)))
    torch.cuda.synchronize()
    gen_seconds = time.perf_counter() - tic

    def placeholder_problem(local_tensors):
        # every block's shape (validation), data only for this rank's blocks
        ts = [torch.empty(spec.dims, device="meta") for _ in range(spec.n_blocks)]
        ts[b0:b1] = local_tensors
        return P.CoupledProblem(ts, spec.rank, list(spec.coupled), mode=spec.mode)

    W, K = args.warmup, args.steps
    KT = min(K, 10)                      # roofline (per-launch event timing) steps
    opts = P.SolverOptions(max_iter=W + K + KT + 4, tol=TINY_TOL, seed=0, precision=prec)
    problem = placeholder_problem(local_dev)
    run = PreparedShardedSolve(problem, opts) if world > 1 else PreparedSolve(problem, opts)
    stream = run.stream
    big = spec.tensor_bytes >= 2 * L2_BYTES
    flush = None if big else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(stream):
        run.engine.run(W)                       # warm-up (also captures the CUDA graph)
        run.engine.step_async()                 # priming: the pipelined iteration's prologue
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    L.launch_count_reset()
    events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        torch.cuda.synchronize()
        for e0, e1 in events:
            with torch.cuda.stream(stream):
                if flush is not None:
                    flush.fill_(1.0)            # evict the blocks from L2 (untimed)
                e0.record(stream)
                run.engine.step_async()
                e1.record(stream)
        torch.cuda.synchronize()
    launches = L.launch_count()
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in events)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    summ = run.engine.summary()
    assert summ.n_iter >= W + K, f"solve stopped early at iteration {summ.n_iter}"
    value = K / (total_ms * 1e-3)      # whole-problem iterations per second
    # ---- roofline of the dominant streaming kernel -------------------------
    # timing mode: CUDA events on the launching stream around every launch of
    # the streaming kernels (classic, unpipelined iteration order)
    run.engine.set_timing(True)
    with torch.cuda.stream(stream):
        for _ in range(KT):
            if flush is not None:
                flush.fill_(1.0)
            run.engine.step_async()
    torch.cuda.synchronize()
    kinds = {}
    for kind, name in ((1, "fiber"), (2, "slab")):
        ms, n, b = run.engine.timing(kind)
        if n:
            kinds[name] = {"ms_avg": ms / n, "launches": n, "bytes_per_launch": b / n,
                           "gbs": (b / n) / (ms / n * 1e-3) / 1e9}
    run.engine.set_timing(False)
    tc_trace = spec.mode == "lra" and getattr(run, "compute_code", 0) == 2
    run.close()
    del run, problem, local_dev
    torch.cuda.empty_cache()
    peak, peak_kind = measured_peak()
    dom_name = max(kinds, key=lambda k: kinds[k]["ms_avg"])
    dom = kinds[dom_name]
    kname = ("xtc" if tc_trace else
             ("fiber4" if (dom_name == "fiber" and spec.mode == "full" and prec == "fp32" and
                           spec.rank <= 16) else dom_name))
    traffic_tab = {
        ("c2", "slab"): (40.186624e6, "profiles/r01f_c2_streaming_ncu_summary.txt"),
        ("c2", "fiber4"): (40.100096e6 + 18.944e3, "profiles/r01f_c2_streaming_ncu_summary.txt"),
        ("c5", "xtc"): (12.794673e9 + 4.373504e6, "profiles/r02_xtc_c5_ncu_summary.txt"),
    }
    traffic, traffic_src = traffic_tab.get((spec.name, kname), (None, None))
    iter_bytes = (1 if spec.mode == "lra" else 3) * spec.tensor_bytes
    # the tensor-core trace pass streams the blocks as three signed byte
    # planes packed once per solve (256-row tiles x K steps of 32, 24 KB each):
    # fewer bytes than the algorithmic fp32 count, so `achieved` (the
    # contract's algorithmic bytes / time) can exceed the HBM peak;
    # `achieved_stream` is what the kernel actually pulls from HBM
    stream = None
    if tc_trace:
        i0, i1, i2 = spec.dims
        per_block = -(-(i1 * i2) // 256) * -(-i0 // 32) * 24576
        sb = float(per_block * (b1 - b0))
        sgbs = sb / (dom["ms_avg"] * 1e-3) / 1e9
        stream = {"bytes_per_launch": sb, "achieved_stream": sgbs, "frac_stream": sgbs / peak,
                  "note": "bytes the launch streams from HBM: 3 B per element (22-bit fixed "
                          "point, byte planes in the MMA shared-memory layout) plus tile padding"}
    roof = {"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
            "frac": dom["gbs"] / peak, "traffic": traffic, "traffic_source": traffic_src,
            "stream": stream,
            "kernel": ("k_xtc_trace (lra trace pass, tcgen05 kind::i8 tensor cores)" if tc_trace
                       else {"slab": "slab3_kernel (mode-2 MTTKRP, row-dot)",
                             "fiber": ("fiber4_kernel (T = X x3 A2, warp-specialised ring)"
                                       if kname == "fiber4" else "fiber2_kernel (T = X x3 A2)")
                             }[dom_name]),
            "bytes_per_launch": dom["bytes_per_launch"],
            "bytes_note": "algorithmic: every block element read once, sum_s |M_s| x 4 B"
                          + (" (the kernel reads a 3-byte image of it, see stream)" if tc_trace else ""),
            "peak_source": peak_kind, "kernels": kinds,
            "iteration": {"bytes": iter_bytes, "gbs": iter_bytes * value / 1e9,
                          "frac": iter_bytes * value / 1e9 / peak,
                          "note": "SURVEY 8d algorithmic bytes per iteration x iterations/s "
                                  "(the whole pipelined step)"}}
    # ---- e2e: public API on pinned host buffers ----------------------------
    e2e = None
    compress_seconds = None
    if not args.no_e2e:
        dev_again, _ = generate_config_device(spec.name, blocks=list(range(b0, b1)))
        host = []
        for t in dev_again:
            try:
                h = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, pin_memory=True)
            except RuntimeError:
                h = torch.empty_strided(t.shape, t.stride(), dtype=t.dtype)
            h.copy_(t)
            host.append(h)
        del dev_again
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        e2e_problem = placeholder_problem(host)
        e2e_opts = P.SolverOptions(max_iter=spec.max_iter, tol=TINY_TOL, seed=0, precision=prec)
        if world > 1:
            torch.distributed.barrier()
        # one complete solve(); runs shorter than 0.5 s (c1-c4) are repeated
        # and the median of 3 is reported (first-call effects are a large
        # share of a 0.1 s solve)
        runs = []
        for _ in range(3):
            torch.cuda.synchronize()
            tic = time.perf_counter()
            res = (P.solve_distributed(e2e_problem, e2e_opts) if world > 1
                   else P.solve(e2e_problem, e2e_opts))
            runs.append((time.perf_counter() - tic, res))
            if world > 1 or runs[0][0] >= 0.5:   # (sharded: one solve, same on every rank)
                break
        runs.sort(key=lambda r: r[0])
        e2e_s, res = runs[len(runs) // 2]
        e2e_runs = len(runs)
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(t.item())
        compress_seconds = res.compress_seconds
        elem = sum(int(h.numel()) for h in host)
        h2d = elem * h.element_size() * world      # every rank uploads its own blocks
        d2h = 8 * 4 * (res.n_iter + 1) + spec.n_blocks * 8 * (sum(spec.dims) * spec.rank + spec.rank)
        e2e = {"value": res.n_iter / e2e_s, "unit": "it/s",
               "h2d_bytes_per_step": h2d / max(res.n_iter, 1),
               "d2h_bytes_per_step": d2h / max(res.n_iter, 1),
               "seconds": e2e_s, "n_iter": res.n_iter, "solves_timed": e2e_runs,
               "compress_seconds": res.compress_seconds,
               "solve_seconds": res.solve_seconds,
               "als_sweeps_mean": (float(np.mean(res.compression_iters))
                                   if res.compression_iters else None),
               # the config's whole run length (late iterations included:
               # QR route, clustered spectra), device timestamps of the
               # accepted iterations, compression and setup excluded
               "iterations_per_s_full_run": (
                   res.n_iter / max(res.trace[-1].elapsed_s - res.trace[0].elapsed_s, 1e-12)
                   if len(res.trace) > 1 else None),
               "step": f"one solve() call of {res.n_iter} iterations on pinned host torch "
                       "buffers: upload, device value checks, ALS compression, engine setup, "
                       "graph capture, iterations, result download"}
        del host, e2e_problem, res
    # ---- CPU baseline: the oracle port on a bounded sample -----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_sample(load_configs(), spec, args.cpu_iters, 1)
        extrap = c["scale"] > 1
        cpu = {"value": c["it_per_s"], "unit": "it/s", "cores": c["cores"], "kind": "port",
               "sample": (f"{c['iters_timed']} APG iterations of {c['blocks_sampled']} of "
                          f"{spec.n_blocks} blocks (compression bounded to 2 ALS sweeps)"
                          f"{', extrapolated linearly in S' if extrap else ''}; fp64 "
                          "numpy/OpenBLAS restatement of the reference"),
               "extrapolated": extrap, "mttkrp_gbs": c["mttkrp_gbs"]}
        if "als_seconds_per_sweep_block" in c:
            cpu["als_seconds_per_sweep_block"] = c["als_seconds_per_sweep_block"]
            if e2e and e2e["als_sweeps_mean"]:
                cpu["compress_seconds_extrapolated"] = (c["als_seconds_per_sweep_block"] *
                                                        e2e["als_sweeps_mean"] * spec.n_blocks)
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": "APG iterations/s", "value": value, "unit": "it/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp64",
        "data": "synthetic (seeded, SURVEY 8d; generated on the device; Yale-B/ERP unavailable)",
        "config": config_dict(spec, world),
        "impl_notes": {"storage": prec, "arithmetic": "fp64 (FMA) in the sweep, the ALS and "
                       "the full-mode passes; lra trace pass and ALS compression passes on "
                       "tcgen05 int8 tensor cores (exact int32 over byte-sliced fixed point: "
                       "22/22 bits in the trace, 30/38 bits in the ALS)" if tc_trace else
                       "fp64 (FMA) accumulation"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(), "n_restarts_timed": summ.n_restarts,
        "gen_seconds": gen_seconds, "compress_seconds": compress_seconds,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    sys.path.insert(0, ROOT)
    run_ours(args)


if __name__ == "__main__":
    main()
