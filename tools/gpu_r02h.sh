#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02h
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/profile_late.py c5 150 3 > $O/prof_c5_late.txt 2>&1
timeout 600 python tools/profile_late.py c5 3 3 > $O/prof_c5_early.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 600 python bench.py --config c2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c2.jsonl 2> $O/bench_c2.err
NCU="ncu --set full --clock-control none --import-source on"
P="python tools/profile_late.py c5 150 2"
timeout 900 $NCU -k regex:k_qr_factor --launch-skip 2 -c 4 -o $O/qrf -f $P > $O/qrf.log 2>&1
timeout 900 $NCU -k regex:k_finalize -c 1 -o $O/fin -f $P > $O/fin.log 2>&1
timeout 900 $NCU -k regex:k_mode_update -c 1 -o $O/mu -f $P > $O/mu.log 2>&1
echo done
