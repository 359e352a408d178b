#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g
mkdir -p $O
P="python tools/profile_late.py c5 150 2"
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_qr_factor --launch-skip 2 -c 1 -o $O/qrf -f $P > $O/qrf.log 2>&1
timeout 900 $NCU -k regex:k_qr_core3 --launch-skip 2 -c 1 -o $O/qrc -f $P > $O/qrc.log 2>&1
timeout 900 $NCU -k regex:k_finalize -c 1 -o $O/fin -f $P > $O/fin.log 2>&1
timeout 900 $NCU -k regex:k_mode_update -c 1 -o $O/mu -f $P > $O/mu.log 2>&1
timeout 900 $NCU -k regex:k_xtc_trace -c 1 -o $O/xtc -f $P > $O/xtc.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_shards.py -m gpu -q -p no:cacheprovider > $O/pytest_shards.log 2>&1
echo done
