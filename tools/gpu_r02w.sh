#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02w
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/timeline.py c5 12 0 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 600 python tools/timeline.py c4 20 0 > $O/timeline_c4.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_$c.jsonl 2> $O/bench_$c.err; done
echo done
