#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02b
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
echo done
