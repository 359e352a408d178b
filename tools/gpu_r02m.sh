#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02m
mkdir -p $O
timeout 600 python tools/create_probe.py > $O/create.txt 2>&1
CUDA_MODULE_LOADING=EAGER timeout 600 python tools/create_probe.py > $O/create_eager.txt 2>&1
timeout 600 python tools/e2e_breakdown.py c5 > $O/e2e_c5.txt 2>&1
echo done
