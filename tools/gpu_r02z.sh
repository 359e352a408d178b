#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z
mkdir -p $O; rm -f $O/status.txt
timeout 600 python tools/oz_probe.py 64 8 > $O/oz_probe.txt 2>&1; echo "probe rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_xtc.py tests/test_gpu_solve.py tests/test_gpu_ops.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1; echo "e2e rc=$?" >> $O/status.txt
cat $O/status.txt; tail -30 $O/oz_probe.txt; tail -5 $O/pytest.log; head -12 $O/e2e_c5.txt
