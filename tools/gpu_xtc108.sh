#!/bin/bash
# ncu --set full of k_xtc_trace as the bench launches it in timing mode (grid capped at 148 - reserve CTAs)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/xtc108; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_xtc_trace -s 2 -c 1 -o $O/t -f python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/t.ncu-rep 5 > $O/summary.txt 2>&1
rm -f $O/t.ncu-rep
cat $O/summary.txt
