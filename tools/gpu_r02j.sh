#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02j
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config c2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 600 python tools/profile_late.py c2 5 10 > $O/prof_c2.txt 2>&1
timeout 600 python tools/profile_late.py c4 300 3 > $O/prof_c4_late.txt 2>&1
timeout 600 python tools/profile_late.py c3 200 3 > $O/prof_c3_late.txt 2>&1
timeout 600 python tools/profile_late.py c5 150 3 > $O/prof_c5_late.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c2_launches.csv python bench.py --config c2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/c2_ncu.log 2>&1
echo done
