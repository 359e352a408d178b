#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/timeline.py c5 12 0 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 900 python tools/reserve_sweep.py 10 16 22 28 > $O/reserve.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -c 1 -o $O/xtc -f python tools/profile_late.py c5 3 1 > $O/xtc.log 2>&1
echo done
