#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02u
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/als_probe.py 64 10 > $O/als_probe64.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
timeout 600 python tools/profile_late.py c4 300 3 > $O/prof_c4_late.txt 2>&1
timeout 600 python tools/profile_late.py c3 200 3 > $O/prof_c3_late.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(mode|final|sweep|xtc|control|qr|restore|pipe|step|init)" -c 300 --csv --log-file $O/c5_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tg_pass -c 1 -o $O/tg -f python tools/als_probe.py 64 2 > $O/tg.log 2>&1
echo done
