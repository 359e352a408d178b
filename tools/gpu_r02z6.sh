#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z6
mkdir -p $O; rm -f $O/status.txt
timeout 900 python tools/reserve_sweep.py 36 40 44 48 52 56 64 72 > $O/reserve.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
cat $O/status.txt; cat $O/reserve.txt; tail -5 $O/pytest.log
