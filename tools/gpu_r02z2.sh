#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z2
mkdir -p $O; rm -f $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/als_launches.csv python tools/als_probe.py 64 3 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
python tools/launch_summary.py $O/als_launches.csv > $O/als_launches_summary.txt 2>&1
cat $O/status.txt; head -40 $O/als_launches_summary.txt
