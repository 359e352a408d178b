#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/clk
mkdir -p $O
(nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > $O/smi.txt) &
SMI=$!
sleep 1
timeout 600 python tools/als_host_probe.py 64 100 > $O/als.txt 2>&1
sleep 1
kill $SMI
cat $O/als.txt; sort $O/smi.txt | uniq -c | sort -rn | head -12
