#!/bin/bash
# ncu --set full of k_mode_update / k_finalize in c5 iterations (profile mode: non-graph launches)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/muprof; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_mode_update|k_finalize" -c 40 -o $O/mu -f python tools/profile_late.py c5 20 2 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/mu.ncu-rep 50 > $O/summary.txt 2>&1
python tools/ncu_lines.py $O/mu.ncu-rep 45 >> $O/summary.txt 2>&1
rm -f $O/mu.ncu-rep
grep -v "  0.0%" $O/summary.txt | tail -75
