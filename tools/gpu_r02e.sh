#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02e
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c4 > $O/e2e_c4.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c3 > $O/e2e_c3.txt 2>&1
timeout 600 python tools/profile_late.py c5 150 5 > $O/prof_c5_late.txt 2>&1
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
bash tools/sanitize.sh $O/sanitize
echo done
