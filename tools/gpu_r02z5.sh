#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z5
mkdir -p $O; rm -f $O/status.txt
timeout 900 python -m pytest tests/test_gpu_xtc.py -m gpu -x -q > $O/pytest_xtc.log 2>&1; echo "pytest xtc rc=$?" >> $O/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_xtc_trace python tools/xtc_probe.py 64 2 > $O/ncu_probe.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench rc=$?" >> $O/status.txt
timeout 600 python tools/timeline.py c5 20 1 > $O/timeline_c5.txt 2>&1
timeout 900 python tools/reserve_sweep.py 16 20 24 28 32 40 > $O/reserve.txt 2>&1
cat $O/status.txt; tail -3 $O/pytest_xtc.log; grep -A3 "k_xtc_trace" $O/ncu_probe.log | tail -12; cut -c1-200 $O/bench_c5.json; tail -12 $O/timeline_c5.txt; cat $O/reserve.txt
