#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02i
mkdir -p $O
timeout 900 python tools/reserve_sweep.py 2 4 6 8 12 16 22 > $O/reserve.txt 2>&1
timeout 600 python tools/profile_late.py c4 300 3 > $O/prof_c4_late.txt 2>&1
timeout 600 python tools/profile_late.py c4 3 3 > $O/prof_c4_early.txt 2>&1
timeout 600 python tools/profile_late.py c3 200 3 > $O/prof_c3_late.txt 2>&1
echo done
