#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/timeline.py c5 12 0 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 600 python bench.py --config c2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err
echo done
