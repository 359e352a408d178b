#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02l
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mode_cluster -c 3 -o $O/mc -f python tools/profile_late.py c2 5 2 > $O/mc.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/als64.csv python tools/als_probe.py 64 40 > $O/als64.log 2>&1
timeout 600 python tools/als_probe.py 64 60 > $O/als_probe64.txt 2>&1
echo done
