#!/bin/bash
# ncu --set full of k_als_solve (64 c5 blocks)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/alsprof; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_als_solve -s 3 -c 3 -o $O/solve -f python tools/als_probe.py 64 3 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/solve.ncu-rep 5 > $O/summary.txt 2>&1
python tools/ncu_lines.py $O/solve.ncu-rep 30 >> $O/summary.txt 2>&1
rm -f $O/solve.ncu-rep
grep -v "  0.0%" $O/summary.txt | tail -50
