#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02n
mkdir -p $O
timeout 600 python tools/timeline.py c5 12 0 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/timeline.py c2 20 1 > $O/timeline_c2.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
echo done
