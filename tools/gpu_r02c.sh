#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02c
mkdir -p $O
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
timeout 600 python tools/profile_late.py c5 3 5 > $O/prof_c5_early.txt 2>&1
timeout 600 python tools/profile_late.py c5 150 5 > $O/prof_c5_late.txt 2>&1
timeout 600 python tools/als_probe.py > $O/als_probe.txt 2>&1
echo done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/als_launches.csv python tools/als_probe.py 8 4 > $O/als_ncu.log 2>&1
echo done2
