#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02z4
mkdir -p $O; rm -f $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -c 1 -o $O/xtc_trace -f python tools/xtc_probe.py 64 1 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/xtc_trace.ncu-rep 5 > $O/xtc_trace_summary.txt 2>&1
python tools/ncu_lines.py $O/xtc_trace.ncu-rep 40 > $O/xtc_trace_lines.txt 2>&1
cat $O/status.txt; cat $O/xtc_trace_summary.txt; head -45 $O/xtc_trace_lines.txt
