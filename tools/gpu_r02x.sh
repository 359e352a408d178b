#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02x
mkdir -p $O
timeout 900 python tools/reserve_sweep.py 12 14 16 18 20 22 > $O/reserve.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 600 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err
echo done
