#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z3
mkdir -p $O; rm -f $O/status.txt
timeout 900 python -m pytest tests/test_gpu_xtc.py -m gpu -x -q > $O/pytest_xtc.log 2>&1; echo "pytest xtc rc=$?" >> $O/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench rc=$?" >> $O/status.txt
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1; echo "e2e rc=$?" >> $O/status.txt
timeout 600 python tools/timeline.py c5 20 1 > $O/timeline_c5.txt 2>&1
cat $O/status.txt; tail -5 $O/pytest_xtc.log; tail -5 $O/pytest.log; cat $O/bench_c5.json | cut -c1-700; head -20 $O/e2e_c5.txt; tail -30 $O/timeline_c5.txt
